"""VSLPipe alpha / beta measurement, C1 by default.

In ONE process, on the same pinned inputs, alternating rounds so host-link drift hits every
variant alike, each round timing `steps` back-to-back e2e GPU Task B steps (2 layers cycled):
  single     moe_taskb_forward_host on all T tokens (one partition)
  ab         moe_taskb_forward2_host on T/2 + T/2 tokens (alpha, beta), one weight stream
for the event-ordered engine and the data mover (one packet in flight), plus the per-partition
token-copy latency (enqueue -> resident) of PACED calls -- each issued after the previous one
finished, as when the caller waits for CPU attention -- and the 1 GB host-link probe before and
after.
    python tools/ab_partitions.py [--config mixtral_8x7b] [--steps 10] > profiles/r02/ab.json
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral_8x7b")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--packet-mb", type=float, default=100.0)
    a = ap.parse_args()
    import numpy as np
    import torch
    import synth
    import paper_2504_09345_b200 as moe

    torch.cuda.set_device(0)
    cfg = synth.CONFIGS[a.config]
    T, h, half = cfg.tokens, cfg.hidden, cfg.tokens // 2
    layers = [synth.gen_inputs(cfg, layer=l) for l in range(2)]
    tbs = [synth.gen_taskb(cfg, l.x, layer=i) for i, l in enumerate(layers)]
    experts = [moe.HostExperts(h, cfg.ffn, l.w1, l.w3, l.w2) for l in layers]
    hls = [moe.HostLayer(h, tb.wo, tb.gamma) for tb in tbs]
    bf = lambda bits: torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)
    routers = [bf(l.router).cuda() for l in layers]
    attn = [bf(tb.attn).pin_memory() for tb in tbs]
    resid = [bf(tb.resid).cuda() for tb in tbs]
    outs = [torch.empty_like(x).pin_memory() for x in attn]
    probe0 = moe.moe_probe_h2d(0, 1 << 30, 5)
    ctxs = {m: moe.MoELayer(h, cfg.ffn, cfg.num_experts, cfg.top_k, T, num_shared=cfg.num_shared,
                            profile=True, mover=m, packet_bytes=int(a.packet_mb * 2 ** 20))
            for m in (False, True)}
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream

    def call(layer, variant, i):
        l = i % 2
        if variant == "single":
            layer.taskb_forward_host(attn[l], resid[l], hls[l], tbs[l].eps, routers[l],
                                     experts[l], outs[l], stream=sh)
        else:
            layer.taskb_forward2_host([attn[l][:half], attn[l][half:]],
                                      [resid[l][:half], resid[l][half:]], hls[l], tbs[l].eps,
                                      routers[l], experts[l], [outs[l][:half], outs[l][half:]],
                                      stream=sh)

    def timed(layer, variant):
        for i in range(2):
            call(layer, variant, i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(a.steps):
            call(layer, variant, i)
        layer.wait_output(sh)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.steps

    def paced_latency(layer, variant):
        """Token-copy latency per partition of calls issued one at a time (each after the last
        finished): the time the attention output waits behind the call's own weight copies."""
        layer.sync()
        layer.reset_stats()
        for i in range(3):
            call(layer, variant, i)
            layer.sync()
        st = layer.stats()
        return [st["part_latency_ms"][p] / max(1, st["part_copies"][p]) for p in range(2)]

    res = {f"{v}_{'mover' if m else 'events'}": [] for m in (False, True) for v in ("single", "ab")}
    for _ in range(a.rounds):
        for m in (False, True):
            for v in ("single", "ab"):
                res[f"{v}_{'mover' if m else 'events'}"].append(timed(ctxs[m], v))
    lat = {f"{v}_{'mover' if m else 'events'}": paced_latency(ctxs[m], v)
           for m in (False, True) for v in ("single", "ab")}
    probe1 = moe.moe_probe_h2d(0, 1 << 30, 5)
    med = {k: statistics.median(v) for k, v in res.items()}
    weights = cfg.expert_bytes * (cfg.num_experts + cfg.num_shared) + hls[0].nbytes
    out = {"config": cfg.name, "tokens": T, "partitions": [half, T - half], "steps": a.steps,
           "rounds": a.rounds, "packet_mb": a.packet_mb,
           "e2e_ms_per_step_median": med, "e2e_ms_per_step_all": res,
           "ab_over_single": {e: med[f"ab_{e}"] / med[f"single_{e}"] for e in ("events", "mover")},
           "weights_streamed_per_step_bytes": weights,
           "token_copy_latency_ms_paced": lat,
           "host_link_probe_gbs": [probe0, probe1],
           "link_roofline_ms": weights / (min(probe0, probe1) * 1e9) * 1e3}
    print(json.dumps(out))
    for c in ctxs.values():
        c.close()


if __name__ == "__main__":
    main()
