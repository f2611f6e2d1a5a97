"""CPU checks of bench.py's roofline bookkeeping (no GPU): the compulsory-bytes floor of the six
K3 GEMMs and the DRAM traffic read back from the committed ncu capture summary."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import bench  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS  # noqa: E402


def test_gemm_min_bytes_c2():
    c = CONFIGS["C2"]
    R, d, f, E = c.T * c.k, c.d, c.f, c.E
    # per GEMM: operands read once, outputs written once (bf16)
    want = 2 * (R * d + E * 2 * f * d + R * 2 * f + R * f          # up+gate -> h, act
                + R * f + E * d * f + R * d                       # down -> y
                + R * d + E * d * f + R * 2 * f + R * 2 * f       # SwiGLU bwd -> dH
                + R * 2 * f + E * 2 * f * d + R * d               # dX
                + R * 2 * f + R * d + E * 2 * f * d               # dW_ug
                + R * d + R * f + E * d * f)                      # dW_d
    assert bench.gemm_min_bytes(c) == want


def test_ncu_traffic_reads_committed_capture():
    tr = bench.ncu_traffic(CONFIGS["C2"].name, "grouped_gemm_kernel", 6)
    assert tr is not None, "profiles/ncu_traffic_C2.json missing"
    floor = bench.gemm_min_bytes(CONFIGS["C2"])
    # measured DRAM bytes can only exceed the compulsory floor (L2 re-reads), within reason
    assert floor <= tr["bytes"] < 4 * floor
    assert bench.ncu_traffic("C9-none", "grouped_gemm_kernel", 6) is None


def test_reference_arm_prints_one_json_line():
    """`bench.py --impl reference` (the driver's reference arm: the CPU oracle on the host) on a
    tiny sample prints the contract's JSON line."""
    import json
    import subprocess

    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "bench.py"), "--impl",
                        "reference", "--config", "C1", "--steps", "1", "--warmup", "0",
                        "--cpu-tokens", "64"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "impl", "cpu_baseline", "e2e", "config"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"


def test_gpus_flag_relaunches_under_torchrun():
    """`bench.py --gpus 2` without WORLD_SIZE re-executes itself under torch.distributed.run with
    two ranks (the driver may call it either way); rank 0 alone prints one line with n_gpus 2.
    Exercised through the reference arm, which needs no GPU."""
    import json
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "bench.py"), "--impl",
                        "reference", "--gpus", "2", "--config", "C1", "--steps", "1", "--warmup", "0",
                        "--cpu-tokens", "64"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


def test_world_size_must_match_gpus():
    import subprocess

    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "bench.py"), "--impl",
                        "reference", "--gpus", "4", "--config", "C1", "--steps", "1"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr
