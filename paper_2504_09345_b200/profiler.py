"""Pipeline profiler on B200 (§6.3, fig:profiler).

The paper's profiler "estimates n using Equation 2, then varies the number of prefilled tokens and
measures the corresponding GPU computation time ... fits a line to capture the relationship
between token count and GPU time.  It also measures the time required to transfer a layer of
weights to the GPU.  It calculates the maximum number of parallel tokens using the line's slope
and weight transfer time".  Here the "GPU computation time" of one MoE layer
call is the sum of the CUDA-event durations of its kernels (router, permute, expert GEMMs,
combine -- the events bracket the kernels only, not the waits on the copy engine), and the
"weight transfer time" is the copy stream's H2D time for the layer's experts.

    python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,65536,131072
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from typing import Sequence


def fit_line(ns: Sequence[float], ts: Sequence[float]):
    """Least-squares t = slope * n + intercept."""
    n = len(ns)
    if n < 2:
        raise ValueError("need at least two points")
    mx = sum(ns) / n
    my = sum(ts) / n
    sxx = sum((x - mx) ** 2 for x in ns)
    if sxx == 0:
        raise ValueError("token counts must differ")
    sxy = sum((x - mx) * (y - my) for x, y in zip(ns, ts))
    slope = sxy / sxx
    return slope, my - slope * mx


def n_real(slope: float, intercept: float, t_io: float) -> float:
    """Token count at which the fitted GPU time line reaches the layer's weight-transfer time."""
    if slope <= 0:
        raise ValueError("slope must be positive")
    return (t_io - intercept) / slope


def profile(config, tokens: Sequence[int], steps: int = 3, device: int = 0) -> dict:
    """config: a synth.CONFIGS name or a synth.MoEConfig (any layer shape)."""
    import numpy as np
    import torch

    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    import synth
    from . import HostExperts, MoELayer, ledger, moe_probe_h2d

    torch.cuda.set_device(device)
    cfg = synth.CONFIGS[config] if isinstance(config, str) else config
    tmax = max(tokens)
    inp = synth.gen_inputs(cfg, tokens=tmax)
    experts = HostExperts(cfg.hidden, cfg.ffn, inp.w1, inp.w3, inp.w2)
    router = torch.from_numpy(inp.router.view(np.int16)).view(torch.bfloat16).cuda()
    xall = torch.from_numpy(inp.x.view(np.int16)).view(torch.bfloat16).cuda()
    layer = MoELayer(cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k, tmax,
                     num_shared=cfg.num_shared, device=device, profile=True)
    stream = torch.cuda.Stream()
    pts = []
    for T in tokens:
        x = xall[:T]
        out = torch.empty_like(x)
        for _ in range(2):
            layer.forward(x, router, experts, out, stream=stream.cuda_stream)
        torch.cuda.synchronize()
        layer.reset_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            layer.forward(x, router, experts, out, stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        st = layer.stats()
        gpu_ms = (st["route_ms"] + st["permute_ms"] + st["gemm1_ms"] + st["gemm2_ms"] +
                  st["combine_ms"]) / steps
        pts.append({"tokens": T, "gpu_ms": gpu_ms, "h2d_ms": st["h2d_ms"] / steps,
                    "step_ms": e0.elapsed_time(e1) / steps,
                    "gemm_ms": (st["gemm1_ms"] + st["gemm2_ms"]) / steps})
    slope, icpt = fit_line([p["tokens"] for p in pts], [p["gpu_ms"] for p in pts])
    t_io = sum(p["h2d_ms"] for p in pts) / len(pts)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    tf = json.load(open(peaks_path))["bf16_tflops_sustained"] if os.path.exists(peaks_path) else 1400.0
    probe = moe_probe_h2d(device, 1 << 30, 3)
    n_eq2 = ledger.eq2_tokens_to_saturate(tf, probe, cfg.num_experts, cfg.top_k,
                                          binary_prefixes=False)
    # residuals of the line relative to each measured point (how linear GPU time is in n)
    for p in pts:
        p["fit_rel_residual"] = (p["gpu_ms"] - (slope * p["tokens"] + icpt)) / p["gpu_ms"]
    res = {"config": cfg.name, "shape": {"hidden": cfg.hidden, "ffn": cfg.ffn,
                                         "experts": cfg.num_experts, "top_k": cfg.top_k,
                                         "shared": cfg.num_shared},
           "points": pts, "slope_ms_per_token": slope, "intercept_ms": icpt,
           "t_io_ms": t_io, "n_real": n_real(slope, icpt, t_io),
           "n_eq2_estimate": n_eq2, "eq2_inputs": {"tensor_tflops": tf, "host_link_gbs": probe},
           "layer_weight_bytes": cfg.expert_bytes * (cfg.num_experts + cfg.num_shared)}
    layer.close()
    experts.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral_8x7b")
    ap.add_argument("--tokens", default="4096,16384,65536,131072")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    print(json.dumps(profile(a.config, [int(t) for t in a.tokens.split(",")], a.steps)))


if __name__ == "__main__":
    main()
