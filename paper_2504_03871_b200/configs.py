"""Expert-layer configurations C1-C5 (BASELINE.json ``configs``) and seeded
synthetic inputs.

The reference's configs carry no tensor shapes (``hidden_dim`` is parsed but never used and
there is no ``d_ff``: ``/root/reference/pkg/src/zpsim/core.py:87``), so the shapes below are
defined here: C1 is the tiny parity config the survey asks the builder to create, C2 is the
Mixtral-style layer, C3 the fine-grained DeepSeek/Qwen-style layer.

Inputs are generated on the CPU with ``torch.Generator().manual_seed(seed)`` and rounded to
bf16 so the GPU path and the CPU oracle see identical bits:
x ~ N(0,1); Wg, W_gate, W_up ~ N(0, 1/d); W_down ~ N(0, 1/f); dY ~ N(0,1).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class LayerConfig:
    name: str
    E: int  # experts
    k: int  # top-k
    d: int  # model dim
    f: int  # expert hidden dim (d_ff)
    T: int  # tokens per step on one GPU

    @property
    def rows(self) -> int:
        return self.T * self.k

    def flops_fwd(self) -> float:
        return 6.0 * self.T * self.k * self.d * self.f

    def flops_bwd(self) -> float:
        return 12.0 * self.T * self.k * self.d * self.f


C1 = LayerConfig("C1-tiny", E=8, k=2, d=256, f=896, T=4096)
C2 = LayerConfig("C2-mixtral", E=8, k=2, d=4096, f=14336, T=16384)
C3 = LayerConfig("C3-finegrained", E=64, k=6, d=2048, f=1408, T=16384)

CONFIGS = {"C1": C1, "C2": C2, "C3": C3}


def with_tokens(cfg: LayerConfig, T: int) -> LayerConfig:
    return LayerConfig(cfg.name + f"-T{T}", cfg.E, cfg.k, cfg.d, cfg.f, T)


@dataclass
class LayerInputs:
    x: torch.Tensor  # [T, d] bf16
    wg: torch.Tensor  # [d, E] bf16 router weight (logits = x @ wg)
    w_gate: torch.Tensor  # [E, f, d] bf16
    w_up: torch.Tensor  # [E, f, d] bf16
    w_down: torch.Tensor  # [E, d, f] bf16
    dy: torch.Tensor  # [T, d] bf16


def make_inputs(cfg: LayerConfig, seed: int = 0, device="cpu", expert_bias=None) -> LayerInputs:
    """Seeded synthetic inputs. ``expert_bias`` (length E, optional) skews the router by adding
    ``bias[e]`` to every token's logit for expert e through a constant input feature."""
    g = torch.Generator().manual_seed(seed)
    E, d, f, T = cfg.E, cfg.d, cfg.f, cfg.T

    def n(shape, std):
        return (torch.randn(shape, generator=g, dtype=torch.float32) * std).to(torch.bfloat16)

    x = n((T, d), 1.0)
    wg = n((d, E), d ** -0.5)
    w_gate = n((E, f, d), d ** -0.5)
    w_up = n((E, f, d), d ** -0.5)
    w_down = n((E, d, f), f ** -0.5)
    dy = n((T, d), 1.0)
    if expert_bias is not None:
        # feature 0 of every token is set to 1 and Wg[0, e] carries the bias
        x[:, 0] = 1.0
        wg[0, :] = torch.as_tensor(expert_bias, dtype=torch.float32).to(torch.bfloat16)
    out = LayerInputs(x, wg, w_gate, w_up, w_down, dy)
    if device != "cpu":
        out = LayerInputs(*(t.to(device) for t in (x, wg, w_gate, w_up, w_down, dy)))
    return out


def zipf_bias(E: int, alpha: float, scale: float = 1.0):
    """Per-expert logit bias giving roughly Zipf(alpha) expert loads (C5 router skew)."""
    import math

    if alpha == 0:
        return [0.0] * E
    return [-scale * alpha * math.log(e + 1) for e in range(E)]
