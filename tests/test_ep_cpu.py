"""Expert parallelism host logic on CPU (no GPU): the exchange plan `moe_ep_plan` (C ABI, host
code of the N>1 path) and a world_size-2 gloo simulation of the whole EP dataflow -- routing,
expert-sorted send buffers, count all-gather, dispatch with the plan's offsets, per-rank expert
FFNs on the received rows, combine exchange, gate-weighted combine -- checked against the
single-process oracle.  The simulation uses the oracle for the arithmetic (test infrastructure);
what it pins is the plan and the layouts the CUDA path uses (csrc/ep.cu)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2504_09345_b200 as moe
from paper_2504_09345_b200 import build as moe_build


@pytest.fixture(scope="module", autouse=True)
def _lib():
    moe_build.build()
    moe.load()


@pytest.mark.parametrize("world,ne", [(2, 8), (4, 8), (8, 8), (8, 64), (2, 16), (1, 8)])
def test_plan_consistency_brute_force(world, ne):
    rng = np.random.default_rng(world * 100 + ne)
    counts = rng.integers(0, 50, size=(world, ne)).astype(np.int32)
    counts[rng.random((world, ne)) < 0.2] = 0     # empty (rank, expert) pairs
    nl = ne // world
    plans = [moe.moe_ep_plan(world, r, ne, counts) for r in range(world)]
    for r, p in enumerate(plans):
        # send side: expert-sorted local rows, one contiguous block per (dest, local expert)
        assert np.array_equal(p["send_cnt"], counts[r])
        assert np.array_equal(p["send_off"], np.concatenate([[0], np.cumsum(counts[r])[:-1]]))
        # receive side: expert-major, then source rank
        exp_rows = sum(int(counts[s, r * nl:(r + 1) * nl].sum()) for s in range(world))
        assert p["recv_rows"] == exp_rows == p["grp_off"][-1]
        pos = 0
        for le in range(nl):
            assert p["grp_off"][le] == pos
            for s in range(world):
                assert p["recv_off"][s * nl + le] == pos
                assert p["recv_cnt"][s * nl + le] == counts[s, r * nl + le]
                pos += counts[s, r * nl + le]
    # every send (s -> d, le) is matched by the receive on d with the same count, in order
    for s in range(world):
        for d in range(world):
            for le in range(nl):
                assert plans[s]["send_cnt"][d * nl + le] == plans[d]["recv_cnt"][s * nl + le]


def test_plan_rejects_bad_arguments():
    c = np.zeros((2, 8), dtype=np.int32)
    with pytest.raises(moe.MoEError):
        moe.moe_ep_plan(3, 0, 8, np.zeros((3, 8), dtype=np.int32))   # 8 % 3 != 0
    with pytest.raises(moe.MoEError):
        moe.moe_ep_plan(2, 2, 8, c)                                  # rank out of range
    bad = c.copy()
    bad[1, 3] = -1
    with pytest.raises(moe.MoEError):
        moe.moe_ep_plan(2, 0, 8, bad)


# ------------------------------------------------------------------------------ gloo, W = 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(rank, world, outs, ins):
    """Pairwise point-to-point exchange (the gloo analogue of NCCL grouped send/recv)."""
    reqs = []
    for p in range(world):
        if p == rank:
            ins[p].copy_(outs[p])
            continue
        if outs[p].numel():
            reqs.append(dist.isend(outs[p], p))
        if ins[p].numel():
            reqs.append(dist.irecv(ins[p], p))
    for r in reqs:
        r.wait()


def _ep_worker(rank, world, port, splits, q):
    import oracle
    import synth
    import paper_2504_09345_b200 as moe_
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.MoEConfig("ep", 20, 128, 256, 8, 2, sum(splits), num_shared=1)
        inp = synth.gen_inputs(cfg)
        ne, k, nl, h = cfg.num_experts, cfg.top_k, cfg.num_experts // world, cfg.hidden
        lo = sum(splits[:rank])
        T = splits[rank]
        x = inp.x[lo:lo + T]
        # routing of the local tokens (stand-in for the GPU router: the oracle)
        idx, gates = oracle.topk_gates(oracle.router_logits(x, inp.router), k)
        # x_perm: local (t, j) rows sorted by global expert id, ascending t inside an expert
        order = sorted(((int(idx[t, j]), t, j) for t in range(T) for j in range(k)))
        pos = np.zeros((T, k), dtype=np.int64)
        x_perm = np.zeros((len(order), h), dtype=np.uint16)
        for p, (e, t, j) in enumerate(order):
            pos[t, j] = p
            x_perm[p] = x[t]
        counts = np.bincount(idx.ravel(), minlength=ne).astype(np.int32)
        allc = [torch.zeros(ne, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(counts))
        counts_all = torch.stack(allc).numpy()
        plan = moe_.moe_ep_plan(world, rank, ne, counts_all)
        # dispatch: one message per peer = concatenation of its (local expert) blocks
        send = [np.concatenate([x_perm[plan["send_off"][d * nl + le]:
                                       plan["send_off"][d * nl + le] + plan["send_cnt"][d * nl + le]]
                                for le in range(nl)]) for d in range(world)]
        recv_sizes = [int(sum(plan["recv_cnt"][s * nl + le] for le in range(nl))) for s in range(world)]
        recv = [torch.zeros((n, h), dtype=torch.int16) for n in recv_sizes]
        _exchange(rank, world, [torch.from_numpy(m.view(np.int16)).contiguous() for m in send], recv)
        x_recv = np.zeros((plan["recv_rows"], h), dtype=np.uint16)
        for s in range(world):
            m = recv[s].numpy().view(np.uint16)
            o = 0
            for le in range(nl):
                c = plan["recv_cnt"][s * nl + le]
                x_recv[plan["recv_off"][s * nl + le]:plan["recv_off"][s * nl + le] + c] = m[o:o + c]
                o += c
        # local experts over their expert-major groups
        y_recv = np.zeros((plan["recv_rows"], h), dtype=np.float32)
        for le in range(nl):
            e = rank * nl + le
            for r in range(plan["grp_off"][le], plan["grp_off"][le + 1]):
                y_recv[r] = oracle.expert_ffn(x_recv[r], inp.w1[e], inp.w3[e], inp.w2[e])
        # combine exchange: reverse of the dispatch
        back = [np.concatenate([y_recv[plan["recv_off"][s * nl + le]:
                                       plan["recv_off"][s * nl + le] + plan["recv_cnt"][s * nl + le]]
                                for le in range(nl)]) for s in range(world)]
        got = [torch.zeros((int(sum(plan["send_cnt"][d * nl + le] for le in range(nl))), h))
               for d in range(world)]
        _exchange(rank, world, [torch.from_numpy(b).contiguous() for b in back], got)
        y_perm = np.zeros((len(order), h), dtype=np.float32)
        for d in range(world):
            m = got[d].numpy()
            o = 0
            for le in range(nl):
                c = plan["send_cnt"][d * nl + le]
                y_perm[plan["send_off"][d * nl + le]:plan["send_off"][d * nl + le] + c] = m[o:o + c]
                o += c
        # gate-weighted combine + replicated shared expert
        y = np.zeros((T, h), dtype=np.float32)
        for t in range(T):
            for j in range(k):
                y[t] += gates[t, j] * y_perm[pos[t, j]]
            y[t] += oracle.expert_ffn(x[t], inp.w1[ne], inp.w3[ne], inp.w2[ne])
        y_ref, idx_ref, g_ref = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, k,
                                               n_shared=1)
        ok = (np.array_equal(idx, idx_ref[lo:lo + T]) and np.array_equal(gates, g_ref[lo:lo + T])
              and np.array_equal(y, y_ref[lo:lo + T]))
        err = float(np.abs(y - y_ref[lo:lo + T]).max()) if T else 0.0
        q.put((rank, bool(ok), err, plan["recv_rows"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("splits", [(40, 24), (0, 33)])
def test_gloo_world2_ep_dataflow_matches_oracle(splits):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, 2, port, splits, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=120) for _ in procs]
    finally:
        for p in procs:
            p.join(30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok, err, rows in res:
        assert ok, f"rank {rank}: max abs err {err}"
    assert sum(r[3] for r in res) == sum(splits) * 2
