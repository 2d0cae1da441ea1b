"""GPU tests of the Contiguous Data Mover (MOE_FLAG_MOVER, csrc/mover.cu):
expert copies cut into packets and issued by a library thread, ordered against the GEMMs by
device counters.  The mover changes only how the bytes travel, so every output must equal the
event-ordered engine's bitwise, and the oracle within the north-star tolerance."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import GpuRun, bf16_tensor, to_f32, token_rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.mark.parametrize("inflight", ["1", "3"])
@pytest.mark.parametrize("shape,packet,slots", [
    (dict(hidden=256, ffn=384, ne=8, k=2, T=300), 64 << 10, 0),      # many packets per expert
    (dict(hidden=512, ffn=640, ne=16, k=4, T=1000, S=1), 1 << 20, 3),  # odd slot count
    (dict(hidden=256, ffn=256, ne=64, k=6, T=333, S=2), 0, 0),         # 100 MB packets, batches
])
def test_mover_parity_and_bitwise_equal(shape, packet, slots, inflight, monkeypatch):
    monkeypatch.setenv("MOE_MOVER_INFLIGHT", inflight)
    cfg = synth.MoEConfig("custom", 21, shape["hidden"], shape["ffn"], shape["ne"], shape["k"],
                          shape["T"], shape.get("S", 0))
    inp = synth.gen_inputs(cfg)
    ref = GpuRun(inp, num_slots=slots)
    out0, idx0, g0 = ref.run()
    ref.close()
    run = GpuRun(inp, packet_bytes=packet, mover=True, num_slots=slots)
    try:
        out, idx, g = run.run()
        assert torch.equal(out, out0) and torch.equal(idx, idx0) and torch.equal(g, g0)
        y_ref, idx_ref, _ = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, cfg.top_k,
                                           cfg.num_shared)
        assert np.array_equal(idx.cpu().numpy(), idx_ref)
        assert token_rel_err(to_f32(out), y_ref).max() <= TOL
        st = run.layer.stats()
        assert st["h2d_weight_bytes"] == (cfg.num_experts + cfg.num_shared) * 6 * cfg.hidden * cfg.ffn
    finally:
        run.close()


def test_mover_back_to_back_layers_and_streams():
    """Six calls over 2 layers without host syncs, alternating between two caller streams, with
    2 slots (every call re-streams every expert through recycled slots): each output equals the
    isolated call's bitwise."""
    cfg = synth.MoEConfig("custom", 22, 512, 768, 8, 2, 500)
    layers = [synth.gen_inputs(cfg, layer=l) for l in range(2)]
    iso = []
    for l in layers:
        r = GpuRun(l)
        iso.append(r.run()[0])
        r.close()
    runs = [GpuRun(l, mover=True, packet_bytes=256 << 10, num_slots=2) for l in layers]
    ctx = runs[0]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    keep = []
    for it in range(6):
        lay = layers[it % 2]
        s = streams[(it // 2) % 2]
        with torch.cuda.stream(s):
            x = bf16_tensor(lay.x)
            r = bf16_tensor(lay.router)
            o = torch.empty_like(x)
        s.synchronize()   # inputs ready before the library reads them on s
        ctx.layer.forward(x, r, runs[it % 2].experts, o, stream=s.cuda_stream)
        outs.append((it % 2, o))
        keep.append((x, r))
    ctx.layer.sync()
    torch.cuda.synchronize()
    for l, o in outs:
        assert torch.equal(o, iso[l])
    for r in runs:
        r.close()


def test_mover_host_tokens_wait_behind_one_packet():
    """The paper's reason for the mover: a latency-sensitive transfer must not queue
    behind every weight transfer already requested.  Two back-to-back host-buffer calls of a layer
    with 25 MB experts (~3.6 ms of weights per call): without the mover the second call's tokens
    wait for the first call's remaining weight copies; with it (8 MB packets, one in flight) only
    for the packet on the wire.  Outputs identical."""
    cfg = synth.MoEConfig("custom", 18, 1024, 4096, 8, 2, 512)
    inp = synth.gen_inputs(cfg)
    xh = torch.from_numpy(inp.x.view(np.int16)).view(torch.bfloat16).pin_memory()
    lat, res = {}, {}
    for mover in (False, True):
        run = GpuRun(inp, profile=True, packet_bytes=8 << 20, mover=mover)
        out_dev, _, _ = run.run()
        oh = [torch.empty_like(xh).pin_memory() for _ in range(2)]
        s = torch.cuda.current_stream()
        best = None
        for rep in range(3):
            run.layer.reset_stats()
            for o in oh:
                run.layer.forward_host(xh, run.router, run.experts, o, stream=s.cuda_stream)
            s.synchronize()
            st = run.layer.stats()
            v = st["token_latency_ms"] / st["host_calls"]
            best = v if best is None else min(best, v)
        for o in oh:
            assert torch.equal(o, out_dev.cpu())
        res[mover] = out_dev.cpu()
        lat[mover] = best
        run.close()
    print(f"mean enqueue->resident token latency: events {lat[False]:.3f} ms, mover {lat[True]:.3f} ms")
    assert torch.equal(res[False], res[True])
    assert lat[True] < lat[False]


def test_mover_taskb_and_destroy_with_work_queued():
    """GPU Task B (layer weights copied by the API thread, experts by the mover) equals the
    event-ordered engine bitwise; destroying a context right after enqueueing drains cleanly."""
    cfg = synth.MoEConfig("custom", 23, 256, 384, 8, 2, 300)
    inp = synth.gen_inputs(cfg)
    tb = synth.gen_taskb(cfg, inp.x)
    from paper_2504_09345_b200 import HostLayer
    outs = []
    for mover in (False, True):
        run = GpuRun(inp, mover=mover, packet_bytes=64 << 10)
        hl = HostLayer(cfg.hidden, tb.wo, tb.gamma)
        attn, resid = bf16_tensor(tb.attn), bf16_tensor(tb.resid)
        o = torch.empty_like(attn)
        s = torch.cuda.current_stream()
        for _ in range(3):
            run.layer.taskb_forward(attn, resid, hl, tb.eps, run.router, run.experts, o,
                                    stream=s.cuda_stream)
        s.synchronize()
        outs.append(o.clone())
        # enqueue more work and destroy without an explicit sync
        x2, o2 = bf16_tensor(inp.x), torch.empty_like(attn)
        run.layer.forward(x2, run.router, run.experts, o2, stream=s.cuda_stream)
        run.close()
        hl.close()
        s.synchronize()
    assert torch.equal(outs[0], outs[1])
