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
    assert sum(results[r][2] for r in range(world)) == 3 * 2 * T * cfg.top_k * cfg.hidden * 2
    assert all(p.exitcode == 0 for p in procs)
