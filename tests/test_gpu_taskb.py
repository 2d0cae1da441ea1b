"""GPU parity of GPU Task B (O projection + MoE layer over all tokens; SURVEY.md §8
NEXT-2) through the C ABI against the oracle (oracle.taskb_forward and its pinned steps).

Staged bar (readings R19-R21):
  * h1 = bf16(resid + attn Wo^T): per-token max-abs error / max-abs reference <= 1e-2 (tensor-core
    fp32 vs oracle fp64 accumulation, one bf16 rounding each), and >= 97% of elements bit-equal;
  * u = RMSNorm(h1) * gamma: BIT-EXACT given the GPU's h1 (both sides use the same correctly
    rounded IEEE operations, R21);
  * routing on u: expert indices bit-exact, gates within 1e-6;
  * out = h1 + MoE(u): per-token relative error <= 2e-2 (the MoE layer's bar).
  * end to end from (attn, resid) alone: the same output bar on every token whose routing agrees
    with the pure-oracle run; tokens whose routing flips (h1 rounding moved u across a near-tie)
    must be rare (< 0.5%).
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2504_09345_b200 import (MOE_E_INVAL, MOE_E_NOT_PINNED, HostLayer, MoEError,
                                   moe_taskb_forward)

from gpu_helpers import (GpuRun, bf16_tensor, block_tokens, dev_view, sample_tokens,
                         stratified_tokens, to_f32, token_rel_err)

pytestmark = pytest.mark.gpu

TOL = 2e-2
H1_TOL = 1e-2


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


class TaskBRun:
    def __init__(self, inp, tb, force_ep=False, profile=False, max_tokens=None, **kw):
        self.inp, self.tb = inp, tb
        self.run = GpuRun(inp, force_ep=force_ep, profile=profile, max_tokens=max_tokens, **kw)
        self.layer = HostLayer(inp.cfg.hidden, tb.wo, tb.gamma)

    def forward(self, attn_bits=None, resid_bits=None, out_alias=None, layer=None):
        attn_bits = self.tb.attn if attn_bits is None else attn_bits
        resid_bits = self.tb.resid if resid_bits is None else resid_bits
        T, k = attn_bits.shape[0], self.inp.cfg.top_k
        attn, resid = bf16_tensor(attn_bits), bf16_tensor(resid_bits)
        out = {"resid": resid, "attn": attn}.get(out_alias) if out_alias else torch.empty_like(attn)
        idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
        gates = torch.empty((T, k), dtype=torch.float32, device="cuda")
        s = torch.cuda.current_stream()
        self.run.layer.taskb_forward(attn, resid, layer or self.layer, self.tb.eps,
                                     self.run.router, self.run.experts, out, idx, gates,
                                     stream=s.cuda_stream)
        s.synchronize()
        self.run.layer.sync()
        dbg = self.run.layer.debug()
        assert dbg.taskb_tokens == T
        h = self.inp.cfg.hidden
        h1 = _bits(dev_view(dbg.h1, (T, h), "<i2").clone().view(torch.int16))
        u = _bits(dev_view(dbg.moe_in, (T, h), "<i2").clone().view(torch.int16))
        return out, idx, gates, h1, u

    def close(self):
        self.layer.close()
        self.run.close()


def _check_staged(inp, tb, out, idx, gates, h1, u, rows=None):
    """Stage-by-stage parity on the token rows `rows` (all when None)."""
    cfg = inp.cfg
    sel = np.arange(tb.attn.shape[0]) if rows is None else rows
    # b1: O-projection + residual
    h1_ref = oracle.oproj_residual(tb.attn[sel], tb.resid[sel], tb.wo)
    e1 = token_rel_err(synth.bf16_bits_to_f32(h1[sel]), synth.bf16_bits_to_f32(h1_ref))
    same = np.mean(h1[sel] == h1_ref)
    assert e1.max() <= H1_TOL and same >= 0.97, f"h1: max rel {e1.max():.3e}, bit-equal {same:.4f}"
    # b2: RMSNorm -- bit-exact on the GPU's h1
    u_ref = oracle.rmsnorm(h1[sel], tb.gamma, tb.eps)
    assert np.array_equal(u[sel], u_ref), f"u: {(u[sel] != u_ref).sum()} elements differ"
    # routing on u (all tokens: cheap)
    logits = oracle.router_logits(u, inp.router)
    idx_ref, g_ref = oracle.topk_gates(logits, cfg.top_k)
    assert np.array_equal(idx.cpu().numpy(), idx_ref)
    assert np.max(np.abs(gates.cpu().numpy() - g_ref)) <= 1e-6
    # out = h1 + MoE(u)
    y = oracle.experts_combine(u[sel], inp.w1, inp.w3, inp.w2, cfg.num_experts, cfg.num_shared,
                               idx_ref[sel], g_ref[sel])
    y += synth.bf16_bits_to_f32(h1[sel])
    err = token_rel_err(to_f32(out[torch.from_numpy(sel).cuda()]), y)
    assert err.max() <= TOL, f"out: max token rel err {err.max():.3e}"
    return e1.max(), err.max()


def _inputs(hidden, ffn, ne, k, T, S=0, seed_id=9):
    cfg = synth.MoEConfig("custom", seed_id, hidden, ffn, ne, k, T, S)
    inp = synth.gen_inputs(cfg)
    return inp, synth.gen_taskb(cfg, inp.x)


@pytest.mark.parametrize("shape", [
    dict(hidden=256, ffn=384, ne=8, k=2, T=300),
    dict(hidden=512, ffn=640, ne=16, k=4, T=1000, S=1),
    dict(hidden=384, ffn=256, ne=64, k=6, T=777, S=2),
    dict(hidden=128, ffn=128, ne=4, k=2, T=1),
])
@pytest.mark.parametrize("force_ep,pair", [(False, "auto"), (True, "auto"), (False, "0"),
                                            (False, "1")])
def test_taskb_staged_parity(shape, force_ep, pair, monkeypatch):
    monkeypatch.setenv("MOE_GEMM_PAIR", pair)
    inp, tb = _inputs(shape["hidden"], shape["ffn"], shape["ne"], shape["k"], shape["T"],
                      shape.get("S", 0))
    r = TaskBRun(inp, tb, force_ep=force_ep)
    try:
        out, idx, gates, h1, u = r.forward()
        e1, e = _check_staged(inp, tb, out, idx, gates, h1, u)
        print(f"{shape} ep={force_ep} pair={pair}: h1 rel {e1:.2e}, out rel {e:.2e}")
    finally:
        r.close()


@pytest.mark.parametrize("shape", [
    dict(hidden=768, ffn=1792, ne=8, k=2, T=1100, S=1),
    dict(hidden=4096, ffn=256, ne=2, k=1, T=1100),     # O-projection: 80 pair tiles, K = 4096
])
@pytest.mark.parametrize("groupm", ["1", "3"])
def test_taskb_raster_groups(shape, groupm, monkeypatch):
    """The residual-epilogue O-projection (and the expert GEMMs) on the CTA-pair kernel with
    several raster groups per launch, the last one partial (MOE_GEMM_GROUPM)."""
    monkeypatch.setenv("MOE_GEMM_PAIR", "1")
    monkeypatch.setenv("MOE_GEMM_GROUPM", groupm)
    inp, tb = _inputs(shape["hidden"], shape["ffn"], shape["ne"], shape["k"], shape["T"],
                      shape.get("S", 0))
    r = TaskBRun(inp, tb)
    try:
        out, idx, gates, h1, u = r.forward()
        _check_staged(inp, tb, out, idx, gates, h1, u)
    finally:
        r.close()


def test_taskb_end_to_end_vs_pure_oracle():
    """From (attn, resid) alone: the whole oracle Task B vs the CUDA path."""
    inp, tb = _inputs(512, 640, 16, 4, 700, S=1)
    cfg = inp.cfg
    r = TaskBRun(inp, tb)
    try:
        out, idx, gates, h1, u = r.forward()
    finally:
        r.close()
    y, h1_ref, u_ref, idx_ref, g_ref = oracle.taskb_forward(
        tb.attn, tb.resid, tb.wo, tb.gamma, tb.eps, inp.router, inp.w1, inp.w3, inp.w2,
        cfg.top_k, cfg.num_shared)
    agree = (idx.cpu().numpy() == idx_ref).all(axis=1)
    assert agree.mean() >= 0.995, f"{(~agree).sum()} tokens routed differently"
    err = token_rel_err(to_f32(out)[agree], y[agree])
    assert err.max() <= TOL, f"max token rel err {err.max():.3e}"


@pytest.mark.parametrize("name", ["mixtral_8x7b", "dsv2_lite"])
def test_taskb_full_size(name):
    """BASELINE.json sizes: routing bit-exact on every token; the other stages on a stratified
    token set -- the first and last token of every 128-token O-projection M tile, and every
    (expert, 128-row M tile) of the MoE's permuted layout (gpu_helpers.stratified_tokens)."""
    cfg = synth.CONFIGS[name]
    inp = synth.gen_inputs(cfg)
    tb = synth.gen_taskb(cfg, inp.x)
    r = TaskBRun(inp, tb)
    try:
        out, idx, gates, h1, u = r.forward()
        sel = np.union1d(np.union1d(block_tokens(cfg.tokens),
                                    stratified_tokens(idx.cpu().numpy(), cfg.num_experts,
                                                      cfg.num_shared)),
                         sample_tokens(cfg.tokens, 16))
        e1, e = _check_staged(inp, tb, out, idx, gates, h1, u, rows=sel)
        print(f"{name}: h1 rel {e1:.2e}, out rel {e:.2e} over {len(sel)} tokens")
    finally:
        r.close()


def test_taskb_back_to_back_layers_and_in_place():
    """Alternating layer blobs (both layer slots cycle) interleaved with plain MoE calls; the
    output may alias resid (in-place residual update)."""
    inp, tb = _inputs(256, 256, 8, 2, 200, S=1)
    tb2 = synth.TaskBInputs(tb.attn, tb.resid, synth.f32_to_bf16_bits(
        -synth.bf16_bits_to_f32(tb.wo)), tb.gamma[::-1].copy(), 1e-6)
    r = TaskBRun(inp, tb)
    layer2 = HostLayer(inp.cfg.hidden, tb2.wo, tb2.gamma)
    try:
        ref1 = [t.clone() for t in r.forward()[:3]]
        r.tb = tb2
        ref2 = [t.clone() for t in r.forward(layer=layer2)[:3]]
        for it in range(3):
            r.tb = tb
            a = r.forward()
            r.run.run()                      # a plain MoE layer call in between
            r.tb = tb2
            b = r.forward(layer=layer2)
            for x, y in zip(a[:3], ref1):
                assert torch.equal(x, y), f"iteration {it}: layer 1 changed"
            for x, y in zip(b[:3], ref2):
                assert torch.equal(x, y), f"iteration {it}: layer 2 changed"
        r.tb = tb
        out, idx, gates, h1, u = r.forward(out_alias="resid")
        assert torch.equal(out, ref1[0]) and torch.equal(idx, ref1[1])
    finally:
        layer2.close()
        r.close()


def test_taskb_stats_and_errors():
    inp, tb = _inputs(256, 256, 8, 2, 64)
    r = TaskBRun(inp, tb, profile=True)
    try:
        r.run.layer.reset_stats()
        r.forward()
        st = r.run.layer.stats()
        blob = 6 * 256 * 256
        assert st["taskb_calls"] == 1 and st["calls"] == 1
        assert st["h2d_weight_bytes"] == 8 * blob + (2 * 256 * 256 + 2 * 256)
        assert st["oproj_ms"] > 0 and st["norm_ms"] > 0
        lay = r.run.layer
        attn = bf16_tensor(tb.attn)
        out = torch.empty_like(attn)

        def call(eps=1e-5, layer_ptr=r.layer.ptr, T=64, a=attn):
            moe_taskb_forward(lay.ctx, a.data_ptr(), a.data_ptr(), T, layer_ptr, eps,
                              r.run.router.data_ptr(), r.run.experts.array, 2, out.data_ptr())

        with pytest.raises(MoEError) as e:
            call(eps=-1.0)
        assert e.value.status == MOE_E_INVAL
        with pytest.raises(MoEError) as e:
            call(eps=float("nan"))
        assert e.value.status == MOE_E_INVAL
        pageable = np.zeros(2 * 256 * 256 + 2 * 256, np.uint16)
        with pytest.raises(MoEError) as e:
            call(layer_ptr=pageable.ctypes.data)
        assert e.value.status == MOE_E_NOT_PINNED
        with pytest.raises(MoEError) as e:
            call(T=65)      # > max_tokens
        assert e.value.status == MOE_E_INVAL
        call(T=0)           # no-op at W = 1
        # the context is still healthy
        a2 = r.forward()
        assert a2[0].shape == (64, 256)
    finally:
        r.close()


def test_taskb_host_entry_point_matches_device():
    """moe_taskb_forward_host (attention output and result in pinned host memory, residual on the
    device): bitwise equal to moe_taskb_forward, over back-to-back calls (both host buffers)."""
    inp, tb = _inputs(512, 640, 16, 4, 900, S=1)
    r = TaskBRun(inp, tb)
    try:
        ref = r.forward()[0].clone()
        attn_h = bf16_tensor(tb.attn, device="cpu").pin_memory()
        resid = bf16_tensor(tb.resid)
        outs = [torch.empty_like(attn_h).pin_memory() for _ in range(3)]
        s = torch.cuda.current_stream()
        for o in outs:
            r.run.layer.taskb_forward_host(attn_h, resid, r.layer, tb.eps, r.run.router,
                                           r.run.experts, o, stream=s.cuda_stream)
        s.synchronize()
        r.run.layer.sync()
        for o in outs:
            assert torch.equal(o.cuda(), ref)
        st = r.run.layer.stats()
        assert st["host_calls"] == 3 and st["taskb_calls"] == 4
    finally:
        r.close()


@pytest.mark.parametrize("shard", [False, True])
def test_taskb_local_expert_parallel_matches_single_gpu(shard):
    """GPU Task B under in-process expert parallelism (MOE_FLAG_LOCAL_EP, the P2P transport):
    each of W = 2 ranks runs the O-projection + RMSNorm on its token slice and the MoE layer
    over its N_e/W experts; every rank's output equals, bitwise, the one-GPU Task B output on
    its slice over two back-to-back calls.  shard: the shared expert split by columns over the
    ranks (MOE_FLAG_SHARD_SHARED) -- then equal up to the shared part's summation order
    (per-token relative difference <= 1e-2, routing identical)."""
    import os
    import threading
    from paper_2504_09345_b200 import HostExperts, MoELayer, shared_slice_weights
    world = 2
    inp, tb = _inputs(256, 256, 8, 2, 300, S=1)
    cfg = inp.cfg
    r = TaskBRun(inp, tb)
    try:
        ref = r.forward()[0].clone()
        router = r.run.router
        ne, nl, S, T = cfg.num_experts, cfg.num_experts // world, cfg.num_shared, cfg.tokens
        bounds = [T * q // world for q in range(world + 1)]
        key = os.urandom(128)
        exps, lays, bufs, errors = [], [], [], []
        for q in range(world):
            if shard:
                ids = list(range(q * nl, (q + 1) * nl))
                sl = shared_slice_weights(cfg.ffn, inp.w1[ne:], inp.w3[ne:], inp.w2[ne:], world, q)
            else:
                ids = list(range(q * nl, (q + 1) * nl)) + [ne + s for s in range(S)]
                sl = None
            exps.append(HostExperts(cfg.hidden, cfg.ffn, [inp.w1[i] for i in ids],
                                    [inp.w3[i] for i in ids], [inp.w2[i] for i in ids],
                                    slice_=sl))
            lays.append(MoELayer(cfg.hidden, cfg.ffn, ne, cfg.top_k, max(1, -(-T // world)),
                                 num_shared=S, world_size=world, rank=q, nccl_unique_id=key,
                                 local_ep=True, shard_shared=shard))
            a = bf16_tensor(tb.attn[bounds[q]:bounds[q + 1]])
            bufs.append((torch.cuda.Stream(), a, bf16_tensor(tb.resid[bounds[q]:bounds[q + 1]]),
                         torch.empty_like(a)))
        torch.cuda.synchronize()

        def work(q):
            try:
                s, a, res, o = bufs[q]
                for _ in range(2):
                    lays[q].taskb_forward(a, res, r.layer, tb.eps, router, exps[q], o,
                                          stream=s.cuda_stream)
                s.synchronize()
            except Exception as e:  # noqa: BLE001
                errors.append((q, repr(e)[:300]))

        th = [threading.Thread(target=work, args=(q,)) for q in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        assert not errors, errors
        for q in range(world):
            got, want = bufs[q][3], ref[bounds[q]:bounds[q + 1]]
            if shard:
                assert token_rel_err(to_f32(got), to_f32(want)).max() <= 1e-2, q
            else:
                assert torch.equal(got, want), f"rank {q} differs"
        for l in lays:
            l.close()
        for e in exps:
            e.close()
    finally:
        r.close()


def test_taskb_chained_layers():
    """NEXT-2 'chain L layers': three Task B layers back to back on one context, each layer's
    output feeding the next layer's residual stream (with a fresh attention output), all weights
    streamed (the copy stream prefetches layer l+1's Wo and experts while layer l computes).
    Each layer is checked against the oracle on the GPU's own input to that layer (staged)."""
    cfgs = [synth.MoEConfig("custom", 30 + l, 256, 384, 8, 2, 257, 1) for l in range(3)]
    inps = [synth.gen_inputs(c) for c in cfgs]
    tbs = [synth.gen_taskb(c, i.x) for c, i in zip(cfgs, inps)]
    run = GpuRun(inps[0])
    layers = [HostLayer(256, tb.wo, tb.gamma) for tb in tbs]
    from paper_2504_09345_b200 import HostExperts
    experts = [run.experts] + [HostExperts(256, 384, i.w1, i.w3, i.w2) for i in inps[1:]]
    routers = [run.router] + [bf16_tensor(i.router) for i in inps[1:]]
    try:
        resid = bf16_tensor(tbs[0].resid)
        s = torch.cuda.current_stream()
        outs, ins = [], []
        for l in range(3):   # enqueue all three layers, then synchronise once
            attn = bf16_tensor(tbs[l].attn)
            out = torch.empty_like(attn)
            idx = torch.empty((257, 2), dtype=torch.int32, device="cuda")
            run.layer.taskb_forward(attn, resid, layers[l], tbs[l].eps, routers[l], experts[l],
                                    out, idx, stream=s.cuda_stream)
            ins.append(resid)
            outs.append((out, idx))
            resid = out
        s.synchronize()
        run.layer.sync()
        for l in range(3):
            r_bits = _bits(ins[l])
            y, h1, u, idx_ref, g = oracle.taskb_forward(
                tbs[l].attn, r_bits, tbs[l].wo, tbs[l].gamma, tbs[l].eps, inps[l].router,
                inps[l].w1, inps[l].w3, inps[l].w2, 2, 1)
            out, idx = outs[l]
            agree = (idx.cpu().numpy() == idx_ref).all(axis=1)
            assert agree.mean() >= 0.99, f"layer {l}: {(~agree).sum()} tokens routed differently"
            err = token_rel_err(to_f32(out)[agree], y[agree])
            assert err.max() <= TOL, f"layer {l}: max token rel err {err.max():.3e}"
    finally:
        for hl in layers:
            hl.close()
        for e in experts[1:]:
            e.close()
        run.close()


# ------------------------------------------------- VSLPipe alpha / beta partitions (NEXT-3)
def _two_partition_run(r, tb, split, mover_note=""):
    """moe_taskb_forward2_host on rows [0, split) (alpha) and [split, T) (beta)."""
    T = tb.attn.shape[0]
    k = r.inp.cfg.top_k
    attn = [bf16_tensor(tb.attn[:split], device="cpu").pin_memory(),
            bf16_tensor(tb.attn[split:], device="cpu").pin_memory()]
    resid = [bf16_tensor(tb.resid[:split]), bf16_tensor(tb.resid[split:])]
    outs = [torch.empty_like(a).pin_memory() for a in attn]
    idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
    gates = torch.empty((T, k), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    r.run.layer.taskb_forward2_host(attn, resid, r.layer, tb.eps, r.run.router, r.run.experts,
                                    outs, idx, gates, stream=s.cuda_stream)
    r.run.layer.wait_output(s.cuda_stream)
    s.synchronize()
    r.run.layer.sync()
    return outs, idx, gates


@pytest.mark.parametrize("mover", [False, True])
@pytest.mark.parametrize("split", [400, 0, 900, 1])
def test_taskb_two_partitions_bitwise_equal_single_calls(split, mover):
    """VSLPipe's alpha / beta through ONE stream of the layer's weights
    (moe_taskb_forward2_host): each partition's output and routing are bitwise those of
    moe_taskb_forward_host on that partition alone, while the layer blob and every expert are
    copied once per call (H2D weight bytes = one layer), with and without the data mover.
    split 0 / T: one empty partition; 1: a one-token alpha."""
    inp, tb = _inputs(512, 640, 16, 4, 900, S=1)
    r = TaskBRun(inp, tb, profile=True, mover=mover, packet_bytes=1 << 20)
    try:
        T = 900
        # reference: each partition alone through the single-partition host entry point
        ref_out, ref_idx = [], []
        s = torch.cuda.current_stream()
        for lo, hi in ((0, split), (split, T)):
            if hi == lo:
                ref_out.append(None)
                continue
            a = bf16_tensor(tb.attn[lo:hi], device="cpu").pin_memory()
            o = torch.empty_like(a).pin_memory()
            idx = torch.empty((hi - lo, 4), dtype=torch.int32, device="cuda")
            r.run.layer.taskb_forward_host(a, bf16_tensor(tb.resid[lo:hi]), r.layer, tb.eps,
                                           r.run.router, r.run.experts, o, idx,
                                           stream=s.cuda_stream)
            r.run.layer.sync()
            ref_out.append(o.clone())
            ref_idx.append(idx.clone())
        r.run.layer.reset_stats()
        outs, idx, gates = _two_partition_run(r, tb, split)
        st = r.run.layer.stats()
        blob = 6 * 512 * 640
        assert st["h2d_weight_bytes"] == 17 * blob + (2 * 512 * 512 + 2 * 512), st
        assert st["taskb_calls"] == 1
        for p, (lo, hi) in enumerate(((0, split), (split, T))):
            if hi == lo:
                continue
            assert torch.equal(outs[p], ref_out[p]), f"partition {p} differs"
        assert torch.equal(idx, torch.cat(ref_idx))
        # and the whole two-partition call against the oracle, stage by stage
        out_all = torch.cat([o for o in outs if o.shape[0]]).cuda()
        dbg = r.run.layer.debug()
        h1 = _bits(dev_view(dbg.h1, (T, 512), "<i2").clone().view(torch.int16))
        u = _bits(dev_view(dbg.moe_in, (T, 512), "<i2").clone().view(torch.int16))
        _check_staged(inp, tb, out_all, idx, gates, h1, u)
    finally:
        r.close()


def test_taskb_two_partitions_beta_copy_latency_mover_vs_events():
    """Beta's attention copy is issued after the call's first expert copies were requested (its
    CPU attention finishes during alpha's GPU phase).  With the event-ordered engine it queues
    behind those expert DMAs; with the data mover (one packet in flight) it
    waits behind at most one packet -- the head-of-line blocking the mover exists to avoid.
    Measured per partition (moe_stats.part_latency_ms) over back-to-back calls; outputs equal."""
    cfg = synth.MoEConfig("custom", 41, 1024, 4096, 8, 2, 1024)   # 25 MB experts
    inp = synth.gen_inputs(cfg)
    tb = synth.gen_taskb(cfg, inp.x)
    from paper_2504_09345_b200 import HostExperts, MoELayer
    experts = HostExperts(cfg.hidden, cfg.ffn, inp.w1, inp.w3, inp.w2)
    hl = HostLayer(cfg.hidden, tb.wo, tb.gamma)
    router = bf16_tensor(inp.router)
    split = 512
    attn = [bf16_tensor(tb.attn[:split], device="cpu").pin_memory(),
            bf16_tensor(tb.attn[split:], device="cpu").pin_memory()]
    resid = [bf16_tensor(tb.resid[:split]), bf16_tensor(tb.resid[split:])]
    lat, res = {}, {}
    try:
        for mover in (False, True):
            layer = MoELayer(cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k, cfg.tokens,
                             profile=True, mover=mover, packet_bytes=4 << 20)
            outs = [[torch.empty_like(a).pin_memory() for a in attn] for _ in range(3)]
            s = torch.cuda.current_stream()
            layer.taskb_forward2_host(attn, resid, hl, tb.eps, router, experts, outs[0],
                                      stream=s.cuda_stream)   # warm-up
            layer.sync()
            layer.reset_stats()
            for o in outs:
                layer.taskb_forward2_host(attn, resid, hl, tb.eps, router, experts, o,
                                          stream=s.cuda_stream)
            layer.sync()
            st = layer.stats()
            assert st["part_copies"] == [3, 3], st["part_copies"]
            lat[mover] = [st["part_latency_ms"][p] / 3 for p in range(2)]
            res[mover] = [o.clone() for o in outs[-1]]
            for o in outs[:-1]:
                assert all(torch.equal(x, y) for x, y in zip(o, outs[-1]))
            layer.close()
        print(f"beta token-copy latency: events {lat[False][1]:.3f} ms, mover {lat[True][1]:.3f} ms;"
              f" alpha: events {lat[False][0]:.3f} ms, mover {lat[True][0]:.3f} ms")
        assert all(torch.equal(x, y) for x, y in zip(res[False], res[True]))
        assert lat[True][1] < lat[False][1]
    finally:
        hl.close()
        experts.close()
