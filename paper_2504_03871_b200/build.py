"""In-tree build of libhetermoe_kernels.so (sm_100a) with nvcc; no JIT cache is used."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build_native(force: bool = False, verbose: bool = False) -> str:
    """Run the csrc/Makefile (nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo ...)."""
    cmd = ["make", "-C", CSRC, f"NVCC={NVCC}"]
    if force:
        subprocess.run(["make", "-C", CSRC, "clean"], check=True, capture_output=not verbose)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"native build failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stdout)
    return os.path.join(HERE, "libhetermoe_kernels.so")
