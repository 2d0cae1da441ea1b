"""Algorithmic work ledger and roofline arithmetic of the MoE layer (host logic, no kernels).

Eq. 1 (§5.1): GEMM arithmetic-to-IO intensity
    I = n (6 N_k h h_i + 4h^2 + 4h^2/s) / (6 N_e h h_i + 4h^2 + 4h^2/s)
read (reading R14) as FLOPs per token (2 FLOPs/MAC x 3 expert matrices) over bf16
BYTES of weights (2 B x 3 matrices per expert); the 4h^2 and 4h^2/s terms are the attention
projections, which are outside this path.
Eq. 2: the GPU saturates when n >= (C_GPU / B_IO) (N_e / N_k); Table 2
 reproduces with binary prefixes (TFLOPS = 2^40, GB/s = 2^30), reading R15.
"""
from __future__ import annotations

import dataclasses


def expert_bytes(h: int, hi: int) -> int:
    """bf16 bytes of one SwiGLU expert: three h x h_i matrices."""
    return 6 * h * hi


def expert_flops_per_token(h: int, hi: int) -> int:
    """FLOPs of one token through one expert (2 FLOPs per multiply-add, 3 matrices)."""
    return 6 * h * hi


@dataclasses.dataclass(frozen=True)
class LayerWork:
    tokens: int
    weight_bytes: int      # host -> device bytes that must be streamed (experts with >= 1 token)
    expert_flops: int      # FLOPs of all (token, expert) pairs incl. shared experts
    router_flops: int
    gemm1_flops: int       # W1|W3 part of expert_flops
    gemm2_flops: int       # W2 part

    @property
    def flops(self) -> int:
        return self.expert_flops + self.router_flops


def layer_work(tokens: int, h: int, hi: int, num_experts: int, top_k: int, num_shared: int = 0,
               experts_hit: int | None = None) -> LayerWork:
    hit = num_experts if experts_hit is None else experts_hit
    pairs = tokens * (top_k + num_shared)
    return LayerWork(tokens=tokens,
                     weight_bytes=(hit + num_shared) * expert_bytes(h, hi),
                     expert_flops=pairs * expert_flops_per_token(h, hi),
                     router_flops=2 * tokens * h * num_experts,
                     gemm1_flops=pairs * 4 * h * hi,
                     gemm2_flops=pairs * 2 * h * hi)


def roofline_time_s(work: LayerWork, tensor_tflops: float, host_link_gbs: float) -> dict:
    """max(expert FLOPs / tensor-core peak, streamed bytes / host-link bandwidth)."""
    t_tc = work.expert_flops / (tensor_tflops * 1e12)
    t_io = work.weight_bytes / (host_link_gbs * 1e9)
    return {"t_tensor_s": t_tc, "t_host_link_s": t_io, "t_roofline_s": max(t_tc, t_io),
            "bound": "host_link" if t_io >= t_tc else "tensor"}


def eq1_intensity(n: float, num_experts: int, top_k: int, h: int, hi: int, s: float,
                  form: str = "left") -> float:
    """Eq. 1.  The paper prints two forms that disagree on the attention terms (reading R14b):
    left  = n (6 N_k h h_i + 4h^2 + 4h^2/s) / (6 N_e h h_i + 4h^2 + 4h^2/s)
    right = n (6 m N_k + 2 + 2/s) / (6 m N_e + 2 + 2/s),  m = h_i / h
    They agree on the expert terms (the only ones on this path) and on the N_k/N_e limit."""
    if form == "left":
        num = 6 * top_k * h * hi + 4 * h * h + 4 * h * h / s
        den = 6 * num_experts * h * hi + 4 * h * h + 4 * h * h / s
    elif form == "right":
        m = hi / h
        num = 6 * m * top_k + 2 + 2 / s
        den = 6 * m * num_experts + 2 + 2 / s
    else:
        raise ValueError(form)
    return n * num / den


def eq2_tokens_to_saturate(c_tflops: float, b_gbs: float, num_experts: int, top_k: int,
                           binary_prefixes: bool = True) -> float:
    """n* = (C_GPU / B_IO) (N_e / N_k)."""
    c = c_tflops * (2 ** 40 if binary_prefixes else 1e12)
    b = b_gbs * (2 ** 30 if binary_prefixes else 1e9)
    return c / b * num_experts / top_k


def model_bytes(layers: int, num_experts: int, h: int, hi: int, s: float, vocab: int) -> float:
    """bf16 model size: per layer Eq. 1's weight denominator, plus embedding and LM head."""
    per_layer = 6 * num_experts * h * hi + 4 * h * h + 4 * h * h / s
    return layers * per_layer + 2 * 2 * vocab * h


def kv_bytes_per_token(layers: int, h: int, s: float) -> float:
    """K and V, bf16, GQA group size s: 2 * 2 B * layers * h/s."""
    return 2 * 2 * layers * h / s
