"""Expert parallelism across PROCESSES over peer memory (MOE_FLAG_IPC_EP): one process per rank,
CUDA IPC handles exchanged through a gloo group, the P2P transport (fused permute+dispatch into
the owners' x_recv, combine reading their y_recv, device flags, no host sync per call).  On the
test box all ranks share one GPU -- same-device IPC exercises the same code as NVLink peers.
Bar: every rank's output bitwise equal to the one-GPU (non-EP) result on its token slice, which
test_gpu_parity pins to the oracle; expert indices bit-exact."""
import multiprocessing as mp
import socket

import numpy as np
import pytest
import torch

import oracle
import synth

from ep_ipc_worker import run_rank
from gpu_helpers import GpuRun, to_f32, token_rel_err

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,shape", [
    (2, dict(hidden=256, ffn=384, num_experts=8, top_k=2, tokens=600, num_shared=0)),
    (2, dict(hidden=512, ffn=256, num_experts=16, top_k=4, tokens=333, num_shared=1)),
    (4, dict(hidden=256, ffn=256, num_experts=16, top_k=2, tokens=3, num_shared=0)),  # empty ranks
])
def test_ep_ipc_processes(world, shape):
    cfg = synth.MoEConfig("custom", 17, shape["hidden"], shape["ffn"], shape["num_experts"],
                          shape["top_k"], shape["tokens"], shape["num_shared"])
    inp = synth.gen_inputs(cfg)
    full = GpuRun(inp)
    out_full, idx_full, _ = full.run()
    out_full = out_full.view(torch.int16).cpu().numpy()
    idx_full = idx_full.cpu().numpy()
    full.close()
    y_ref, idx_ref, _ = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, cfg.top_k,
                                       cfg.num_shared)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cfg_tuple = (cfg.name, cfg.config_id, cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k,
                 cfg.tokens, cfg.num_shared)
    procs = [ctx.Process(target=run_rank, args=(r, world, port, cfg_tuple, 3, 0, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            r, idx, out, comm, err = q.get(timeout=600)
            assert err is None, f"rank {r}:\n{err}"
            results[r] = (idx, out, comm)
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    T = cfg.tokens
    for r in range(world):
        lo, hi = T * r // world, T * (r + 1) // world
        idx, out, _ = results[r]
        if hi == lo:
            continue
        assert np.array_equal(idx, idx_ref[lo:hi])
        assert np.array_equal(out.reshape(hi - lo, -1), out_full[lo:hi]), f"rank {r} differs"
        y = torch.from_numpy(out.reshape(hi - lo, -1)).view(torch.bfloat16)
        assert token_rel_err(to_f32(y), y_ref[lo:hi]).max() <= 2e-2
    assert sum(results[r][2][0] for r in range(world)) == 3 * 2 * T * cfg.top_k * cfg.hidden * 2
    assert all(p.exitcode == 0 for p in procs)


def _run_ranks(world, cfg_arg, calls, timeout=900, shard=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=run_rank, args=(r, world, port, cfg_arg, calls, 0, q, shard))
             for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            r, idx, out, comm, err = q.get(timeout=timeout)
            assert err is None, f"rank {r}:\n{err}"
            results[r] = (idx, out, comm)
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    return results


@pytest.mark.parametrize("name,world", [("mixtral_8x7b", 2), ("mixtral_8x7b", 4),
                                        ("mixtral_8x7b", 8), ("mixtral_8x22b", 8),
                                        ("dbrx", 8), ("dsv2_lite", 8)])
def test_ep_ipc_full_size(name, world):
    """Expert parallelism at the BASELINE.json shapes and GPU counts (C1 at W = 2 / 4 / 8, C2-C4
    at W = 8), one PROCESS per rank sharing this GPU over CUDA IPC (the P2P transport of a
    multi-GPU box).  Each rank streams only its N_e / W experts (+ the shared ones) and owns T / W
    tokens.  Bar: every rank's expert indices bit-exact vs the oracle router on every token; its
    output bitwise equal to the one-GPU result on its slice; and, on the stratified token set
    (every (expert, 128-row M tile) of the permuted layout -- the EP receive layout holds the
    same rows in the same order), within 2e-2 of the oracle."""
    from gpu_helpers import sample_tokens, stratified_tokens
    cfg = synth.CONFIGS[name]
    inp = synth.gen_inputs(cfg)
    full = GpuRun(inp)
    out_full, _, _ = full.run()
    out_full = out_full.view(torch.int16).cpu().numpy()
    full.close()
    logits = oracle.router_logits(inp.x, inp.router)
    idx_ref, g_ref = oracle.topk_gates(logits, cfg.top_k)
    results = _run_ranks(world, name, 2)
    T = cfg.tokens
    out_ep = np.empty_like(out_full)
    for r in range(world):
        lo, hi = T * r // world, T * (r + 1) // world
        idx, out, _ = results[r]
        assert np.array_equal(idx, idx_ref[lo:hi]), f"rank {r}: routing differs"
        out_ep[lo:hi] = out.reshape(hi - lo, -1)
        assert np.array_equal(out_ep[lo:hi], out_full[lo:hi]), f"rank {r} differs from W = 1"
    sel = np.union1d(stratified_tokens(idx_ref, cfg.num_experts, cfg.num_shared),
                     sample_tokens(T, 16))
    y_ref = oracle.experts_combine(inp.x[sel], inp.w1, inp.w3, inp.w2, cfg.num_experts,
                                   cfg.num_shared, idx_ref[sel], g_ref[sel])
    y = torch.from_numpy(out_ep[sel]).view(torch.bfloat16)
    err = token_rel_err(to_f32(y), y_ref)
    print(f"{name} W={world}: max token rel err {err.max():.3e} over {len(sel)} stratified tokens")
    assert err.max() <= 2e-2
    assert sum(results[r][2][0] for r in range(world)) == 2 * 2 * T * cfg.top_k * cfg.hidden * 2


def test_ep_ipc_full_size_sharded_shared():
    """C4 (DeepSeek-V2-Lite shape: 64 routed experts top-6 + 2 shared) at W = 8 processes with
    the shared experts SHARDED (MOE_FLAG_SHARD_SHARED): each rank streams its 8
    routed experts and a 352-column slice of the 2816-wide concatenated shared FFN (17.3 MB x 8 +
    4.3 MB, vs 17.3 MB x 10 replicated), every token is gathered to every slice owner and the
    partial rows are summed in the token's rank.  Bar: routing bit-exact on every token; the
    stratified token set within 2e-2 of the oracle; host bytes summed over ranks = the
    algorithmic bytes of one layer per call (no replication)."""
    from gpu_helpers import sample_tokens, stratified_tokens
    cfg = synth.CONFIGS["dsv2_lite"]
    world = 8
    inp = synth.gen_inputs(cfg)
    logits = oracle.router_logits(inp.x, inp.router)
    idx_ref, g_ref = oracle.topk_gates(logits, cfg.top_k)
    results = _run_ranks(world, "dsv2_lite", 2, shard=True)
    T = cfg.tokens
    out_ep = np.empty((T, cfg.hidden), dtype=np.int16)
    for r in range(world):
        lo, hi = T * r // world, T * (r + 1) // world
        idx, out, _ = results[r]
        assert np.array_equal(idx, idx_ref[lo:hi]), f"rank {r}: routing differs"
        out_ep[lo:hi] = out.reshape(hi - lo, -1)
    sel = np.union1d(stratified_tokens(idx_ref, cfg.num_experts, cfg.num_shared),
                     sample_tokens(T, 16))
    y_ref = oracle.experts_combine(inp.x[sel], inp.w1, inp.w3, inp.w2, cfg.num_experts,
                                   cfg.num_shared, idx_ref[sel], g_ref[sel])
    y = torch.from_numpy(out_ep[sel]).view(torch.bfloat16)
    err = token_rel_err(to_f32(y), y_ref)
    print(f"dsv2_lite W=8 sharded shared: max token rel err {err.max():.3e} over {len(sel)} tokens")
    assert err.max() <= 2e-2
    layer_bytes = (cfg.num_experts + cfg.num_shared) * 6 * cfg.hidden * cfg.ffn
    assert sum(results[r][2][1] for r in range(world)) == 2 * layer_bytes
