"""MoE-Lens two-stage performance model (§5, Eqs. 1-14), with a
B200 calibration of the streamed MoE layer from this repo's own measurements.

Host-only arithmetic.  Equation numbers and lines refer to PAPER.md:
  Eq. 1  P:271  GEMM intensity            (ledger.eq1_intensity)
  Eq. 2  P:278  tokens to saturate the GPU (ledger.eq2_tokens_to_saturate)
  Eq. 3  P:327  PME = 2(p+g) / ((2p+g) g)
  Eq. 4  P:336  T_max = min(PME * M / delta, T_GPU)
  Eq. 5  P:369  B_Mem = B_KV + B_IO = (M / M_weight) B_IO
  Eq. 6  P:375  T_CPU = 2 s I_cpu_attn B_KV
  Eq. 7  P:406  C_KV,eff = (p+g) / (p + g/2) C_KV
  Eq. 8  P:430  q = N / sum_{i=0}^{g} ceil((p+i)/b)
  Eq. 9  P:437  g q > N / (p+g)
  Eq. 10 P:442  T1 = K g / ((K/q + g) delta) = K/(K+gq) * gq/delta
  Eq. 11 P:452  T_prefill = T_GPU p / (p+g)
  Eq. 12 P:458  It = 2g + (K p - (T_prefill + T_GPU)/2 * g) / T_prefill
  Eq. 13 P:462  T2 = K g / (It delta)
  Eq. 14 P:466  T = min(T1, T2)
Readings: Eq. 3's sum has g+1 terms but its closed form has g -- the closed form
is canonical; in §5.5 T_GPU is tokens per iteration (it is compared with q(p+g) and divides
token counts into iterations), T_GPU_iter = T_GPU[tokens/s] * delta; Eq. 13's lowercase k is K.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
from typing import Dict, List, Optional, Sequence

from . import ledger


# ----------------------------------------------------------------------------------- Stage 1
def pme(p: float, g: float) -> float:
    """Eq. 3: parallel tokens per unit of KV-cache occupancy over a sequence's lifetime."""
    if p < 1 or g < 1:
        raise ValueError("p, g >= 1")
    return 2.0 * (p + g) / ((2.0 * p + g) * g)


def weight_transfer_time(model_bytes: float, b_io: float) -> float:
    """delta = Model Size / B_IO."""
    return model_bytes / b_io


def t_max(p: float, g: float, kv_tokens: float, delta: float, t_gpu: float) -> Dict[str, float]:
    """Eq. 4 with utilisation T_max / T_GPU; kv_tokens = M (KV capacity in tokens)."""
    if kv_tokens < p + g:
        raise ValueError("workload infeasible: single sequence exceeds KV capacity")
    mem_bound = pme(p, g) * kv_tokens / delta
    t = min(mem_bound, t_gpu)
    return {"t_max": t, "utilization": t / t_gpu,
            "regime": "MemoryBound" if mem_bound < t_gpu else "GpuBound"}


def required_bandwidths(kv_bytes: float, weight_bytes: float, b_io: float) -> Dict[str, float]:
    """Eq. 5: B_KV = (M_kv / M_weight) B_IO and B_Mem = B_KV + B_IO."""
    b_kv = kv_bytes / weight_bytes * b_io
    return {"b_kv": b_kv, "b_mem": b_kv + b_io}


def required_cpu_attn_throughput(s: float, i_cpu_attn: float, b_kv: float) -> float:
    """Eq. 6: T_CPU = 2 s I_cpu_attn B_KV."""
    return 2.0 * s * i_cpu_attn * b_kv


def effective_kv_capacity(p: float, g: float, c_kv: float) -> float:
    """Eq. 7."""
    return (p + g) / (p + g / 2.0) * c_kv


def utilization_surface(p_range: Sequence[float], g_range: Sequence[float], kv_tokens: float,
                        delta: float, t_gpu: float) -> List[List[float]]:
    """Fig. 3(a): T_max / T_GPU over (p, g)."""
    return [[t_max(p, g, kv_tokens, delta, t_gpu)["utilization"] for g in g_range]
            for p in p_range]


# ----------------------------------------------------------------------------------- Stage 2
def prefill_rate(n_blocks: int, b: int, p: int, g: int) -> float:
    """Eq. 8 (q, sequences scheduled for prefill per iteration)."""
    if n_blocks < 1 or b < 1 or p < 1 or g < 1:
        raise ValueError("N, b, p, g >= 1")
    demand = sum(math.ceil((p + i) / b) for i in range(g + 1))
    if demand > n_blocks * (g + 1):
        raise ValueError("infeasible workload: one sequence's lifetime demand exceeds the cache")
    return n_blocks / demand


def t1_memory_bound(K: float, g: float, q: float, delta: float) -> float:
    """Eq. 10."""
    return K * g / ((K / q + g) * delta)


def t2_gpu_bound(K: float, p: float, g: float, t_gpu_iter: float, delta: float) -> Dict[str, float]:
    """Eqs. 11-13 (t_gpu_iter: GPU-limited tokens per iteration).  Raises if the prologue alone
    would exceed the batch (K p <= (T_prefill + T_GPU)/2 * g)."""
    t_prefill = t_gpu_iter * p / (p + g)
    main = K * p - (t_prefill + t_gpu_iter) / 2.0 * g
    if main <= 0:
        raise ValueError("not GPU-bound: the batch ends inside the pipeline prologue")
    it = 2.0 * g + main / t_prefill
    return {"t_prefill": t_prefill, "iterations": it, "t2": K * g / (it * delta)}


def predict(K: int, p: int, g: int, n_blocks: int, b: int, t_gpu: float, delta: float) -> Dict:
    """Eq. 14 with regime and utilisation (total tokens per second over the GPU ceiling)."""
    q = prefill_rate(n_blocks, b, p, g)
    t1 = t1_memory_bound(K, g, q, delta)
    t_gpu_iter = t_gpu * delta
    t2 = None
    if t_gpu_iter < q * (p + g):   # GPU-bound condition
        try:
            t2 = t2_gpu_bound(K, p, g, t_gpu_iter, delta)["t2"]
        except ValueError:
            t2 = None
    t = t1 if t2 is None else min(t1, t2)
    return {"q": q, "t1": t1, "t2": t2, "predicted_throughput": t,
            "regime": "MemoryBound" if t2 is None or t1 <= t2 else "GpuBound",
            "predicted_utilization": min(1.0, t * (p + g) / g / t_gpu)}


# ---------------------------------------------------------------- B200 streamed-layer model
@dataclasses.dataclass
class LayerCalibration:
    """Measured B200 numbers for ONE streamed MoE layer (this repo's kernels)."""
    config: str
    weight_bytes: int           # streamed per call
    host_link_gbs: float        # measured, the paper's 1 GB probe
    gpu_s_per_token: float      # slope of the profiler's GPU-time line
    gpu_intercept_s: float

    @property
    def delta_s(self) -> float:
        return self.weight_bytes / (self.host_link_gbs * 1e9)

    @property
    def t_gpu_tokens_per_s(self) -> float:
        return 1.0 / self.gpu_s_per_token

    def predicted_layer_time_s(self, n: int) -> float:
        """Stage 1 for one layer: each call takes delta while IO-bound, the GPU time otherwise."""
        return max(self.delta_s, self.gpu_intercept_s + self.gpu_s_per_token * n)

    def n_real(self) -> float:
        """Eq. 2 measured: tokens at which the GPU line meets delta."""
        return (self.delta_s - self.gpu_intercept_s) / self.gpu_s_per_token


def calibrate_from_profiler(prof: Dict, host_link_gbs: Optional[float] = None) -> LayerCalibration:
    """From `python -m paper_2504_09345_b200.profiler` output."""
    return LayerCalibration(config=prof["config"], weight_bytes=int(prof["layer_weight_bytes"]),
                            host_link_gbs=host_link_gbs or prof["eq2_inputs"]["host_link_gbs"],
                            gpu_s_per_token=prof["slope_ms_per_token"] * 1e-3,
                            gpu_intercept_s=prof["intercept_ms"] * 1e-3)


def validate_against_profiler(prof: Dict) -> Dict:
    """Predicted vs measured streamed-layer step time at every profiled token count (the B200
    analogue of the paper's 94% model accuracy)."""
    cal = calibrate_from_profiler(prof)
    rows = []
    for pt in prof["points"]:
        pred = cal.predicted_layer_time_s(pt["tokens"]) * 1e3
        rows.append({"tokens": pt["tokens"], "measured_ms": pt["step_ms"], "predicted_ms": pred,
                     "accuracy": 1.0 - abs(pred - pt["step_ms"]) / pt["step_ms"]})
    return {"config": cal.config, "delta_ms": cal.delta_s * 1e3, "n_real": cal.n_real(),
            "t_gpu_tokens_per_s": cal.t_gpu_tokens_per_s, "points": rows,
            "mean_accuracy": sum(r["accuracy"] for r in rows) / len(rows)}


def predict_expert_parallel(hidden: int, ffn: int, num_experts: int, top_k: int,
                            num_shared: int, tokens: int, world: int, link_gbs: float,
                            host_dram_gbs: float, tensor_tflops: float,
                            gemm_efficiency: float = 0.8, nvlink_gbs: float = 900.0,
                            shard_shared: bool = False) -> Dict:
    """Predicted step time / tokens per second of ONE streamed MoE layer under expert
    parallelism over `world` GPUs of one box (BASELINE.json's 1/2/4/8 B200s).

    Each rank streams its N_e / W routed experts plus the replicated shared ones (or, with
    shard_shared, its column slice of them) over its own host link; all W links draw on one host's DRAM at once (Eq. 5's logic: host
    memory must feed every stream), so a link delivers min(link, host_dram / W).  Each rank's
    expert GEMMs do 1/W of the layer's FLOPs (plus its own shared-expert work), at
    `gemm_efficiency` of the tensor peak; the token exchange (dispatch + combine, bf16 rows, the
    (W-1)/W of them that leave the rank) goes over NVLink.  The step is the slowest of the three
    pipelined streams (weights, GEMMs, exchange): step = max(t_link, t_gemm, t_a2a)."""
    if world < 1 or num_experts % world:
        raise ValueError("world must divide num_experts")
    eb = ledger.expert_bytes(hidden, ffn)
    if shard_shared and world > 1 and num_shared:
        # MOE_FLAG_SHARD_SHARED: the slowest rank holds ceil(B / W) of the B = S h_i / 128
        # column blocks of the concatenated shared FFN (include/moe.h, moe_shared_slice)
        blocks = num_shared * ffn // 128
        rank_bytes = (num_experts // world) * eb + -(-blocks // world) * 128 * 6 * hidden
    else:
        rank_bytes = (num_experts // world + num_shared) * eb
    per_link = min(link_gbs, host_dram_gbs / world)
    t_link = rank_bytes / (per_link * 1e9)
    flops = 6.0 * hidden * ffn * tokens * (top_k / world + num_shared / world)
    t_gemm = flops / (gemm_efficiency * tensor_tflops * 1e12)
    a2a_bytes = 2 * (tokens / world) * top_k * hidden * 2 * (world - 1) / world
    t_a2a = a2a_bytes / (nvlink_gbs * 1e9) if world > 1 else 0.0
    step = max(t_link, t_gemm, t_a2a)
    return {"world": world, "rank_weight_bytes": rank_bytes, "per_link_gbs": per_link,
            "t_link_ms": t_link * 1e3, "t_gemm_ms": t_gemm * 1e3, "t_a2a_ms": t_a2a * 1e3,
            "step_ms": step * 1e3, "tokens_per_s": tokens / step,
            "bound": "host_link" if step == t_link else ("tensor" if step == t_gemm else "nvlink")}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("validate", help="predicted vs measured layer time from a profiler JSON")
    a.add_argument("profiler_json")
    b = sub.add_parser("stage2", help="Eq. 14 for a workload")
    for k, d in (("K", 20000), ("p", 100), ("g", 128), ("N", 1000), ("b", 16)):
        b.add_argument(f"--{k}", type=int, default=d)
    b.add_argument("--t-gpu", type=float, required=True, help="tokens/s")
    b.add_argument("--delta", type=float, required=True, help="seconds")
    args = ap.parse_args()
    if args.cmd == "validate":
        print(json.dumps(validate_against_profiler(json.load(open(args.profiler_json))), indent=1))
    else:
        print(json.dumps(predict(args.K, args.p, args.g, args.N, args.b, args.t_gpu, args.delta)))


if __name__ == "__main__":
    main()
