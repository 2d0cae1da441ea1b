"""Pins of the CPU oracle (oracle/moe_oracle.c) to things other than itself.

Each test checks the oracle against what the mathematics fixes -- exact integer arithmetic,
subset enumeration, closed forms, special cases that reduce to a textbook torch fp64 routine,
exact invariants -- so that a dropped term, wrong sign/index or transposed operand fails one.
Readings R1-R10 are listed in DESIGN.md; citations are PAPER.md lines.
"""
import itertools
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from synth import bf16_bits_to_f32, f32_to_bf16_bits

pytestmark = pytest.mark.filterwarnings("ignore")


def _bf(a):
    return f32_to_bf16_bits(np.asarray(a, dtype=np.float32))


def _t64(bits):
    return torch.from_numpy(bf16_bits_to_f32(bits).astype(np.float64))


def _dense_swiglu_fp64(x_bits, w1, w3, w2):
    """Textbook SwiGLU FFN (torch fp64): W2 (silu(W1 x) * (W3 x))   -- reading R2."""
    x = _t64(x_bits)
    return (torch.nn.functional.silu(x @ _t64(w1).T) * (x @ _t64(w3).T)) @ _t64(w2).T


# ------------------------------------------------------------------------------------------
# Router logits (step a2; reading R6: fp64 accumulation)
# ------------------------------------------------------------------------------------------
def test_router_logits_exact_integers():
    """Small-integer bf16 operands: every logit is an exact integer -> compare with Python ints."""
    rng = np.random.default_rng(0)
    T, h, ne = 37, 96, 11
    xi = rng.integers(-7, 8, size=(T, h))
    wi = rng.integers(-5, 6, size=(ne, h))
    logits = oracle.router_logits(_bf(xi), _bf(wi))
    ref = np.array([[sum(int(a) * int(b) for a, b in zip(xi[t], wi[e])) for e in range(ne)]
                    for t in range(T)], dtype=np.float64)
    assert np.array_equal(logits, ref)


def test_router_logits_vs_fsum():
    """Random bf16: fp64 ascending sum within a few ulp of the correctly rounded sum (math.fsum)."""
    inp = synth.gen_inputs(synth.CONFIGS["tiny"], experts=False)
    logits = oracle.router_logits(inp.x, inp.router)
    x = bf16_bits_to_f32(inp.x).astype(np.float64)
    w = bf16_bits_to_f32(inp.router).astype(np.float64)
    for t in range(0, inp.x.shape[0], 7):
        for e in range(w.shape[0]):
            exact = math.fsum(x[t] * w[e])   # products of bf16 are exact in fp64
            assert abs(logits[t, e] - exact) <= 1e-13 * max(1.0, float(np.abs(x[t] * w[e]).sum()))


# ------------------------------------------------------------------------------------------
# Top-k selection and gates (step a3; readings R3, R5, R7)
# ------------------------------------------------------------------------------------------
def _rank_count_sets(logits, k):
    """e in S_t  <=>  #{e' : l_e' > l_e  or (l_e' == l_e and e' < e)} < k."""
    T, ne = logits.shape
    out = []
    for t in range(T):
        l = logits[t]
        s = [e for e in range(ne)
             if sum(1 for f in range(ne) if l[f] > l[e] or (l[f] == l[e] and f < e)) < k]
        out.append(sorted(s))
    return out


def _enumerate_best_subset(l, k):
    """Maximise the sum of logits over all C(N_e,k) subsets; ties -> lexicographically smallest."""
    best, best_sum = None, -math.inf
    for sub in itertools.combinations(range(len(l)), k):
        s = math.fsum(l[list(sub)])
        if s > best_sum:
            best, best_sum = sub, s
    return list(best)


@pytest.mark.parametrize("ne,k", [(8, 2), (16, 4), (9, 1), (6, 6), (12, 5)])
def test_topk_rank_count_and_enumeration(ne, k):
    rng = np.random.default_rng(ne * 100 + k)
    T = 200
    # integer-valued logits force many exact ties
    logits = rng.integers(-3, 4, size=(T, ne)).astype(np.float64)
    logits[: T // 2] += rng.standard_normal((T // 2, ne))
    idx, gates = oracle.topk_gates(logits, k)
    rc = _rank_count_sets(logits, k)
    for t in range(T):
        assert sorted(idx[t].tolist()) == rc[t]
        assert sorted(idx[t].tolist()) == _enumerate_best_subset(logits[t], k)
        # listed in rank order: (logit desc, index asc)
        for a, b in zip(idx[t][:-1], idx[t][1:]):
            assert logits[t, a] > logits[t, b] or (logits[t, a] == logits[t, b] and a < b)


def test_topk_all_ties_zero_router():
    """W_r = 0 -> all logits 0 -> idx = [0..k-1], gates 1/k."""
    inp = synth.gen_inputs(synth.CONFIGS["tiny"], experts=False)
    zero = np.zeros_like(inp.router)
    logits = oracle.router_logits(inp.x, zero)
    idx, gates = oracle.topk_gates(logits, 3)
    assert (idx == np.arange(3, dtype=np.int32)).all()
    assert np.all(gates == np.float32(1.0 / 3.0))


def test_topk_duplicate_router_rows_lowest_index_first():
    inp = synth.gen_inputs(synth.CONFIGS["tiny"], experts=False)
    r = inp.router.copy()
    r[5] = r[3]
    logits = oracle.router_logits(inp.x, r)
    idx, _ = oracle.topk_gates(logits, 2)
    both = 0
    for row in idx.tolist():
        if 3 in row and 5 in row:
            both += 1
            assert row.index(3) < row.index(5)
    # whenever 5 is selected, 3 (identical logit, lower index) must be selected as well
    for t, row in enumerate(idx.tolist()):
        if 5 in row:
            assert 3 in row


def test_gates_closed_forms():
    rng = np.random.default_rng(3)
    logits = rng.standard_normal((500, 8)) * 3
    # renormalised gates sum to 1
    _, g = oracle.topk_gates(logits, 4)
    assert np.allclose(g.astype(np.float64).sum(1), 1.0, atol=1e-6)
    # k = 1 -> gate exactly 1
    _, g1 = oracle.topk_gates(logits, 1)
    assert np.all(g1 == 1.0)
    # k = 2 -> g0 = sigmoid(l0 - l1)
    i2, g2 = oracle.topk_gates(logits, 2)
    l0 = np.take_along_axis(logits, i2[:, :1].astype(np.int64), 1)[:, 0]
    l1 = np.take_along_axis(logits, i2[:, 1:].astype(np.int64), 1)[:, 0]
    sig = 1.0 / (1.0 + np.exp(-(l0 - l1)))
    assert np.allclose(g2[:, 0], sig, rtol=1e-6, atol=0)
    assert np.allclose(g2[:, 1], 1 - sig, rtol=1e-5, atol=1e-7)
    # renormalize=0 -> full-softmax probabilities (torch.softmax), and rescaling them reproduces
    # the renormalised gates
    i4n, g4n = oracle.topk_gates(logits, 4, renormalize=False)
    full = torch.softmax(torch.from_numpy(logits), dim=1).numpy()
    assert np.allclose(g4n, np.take_along_axis(full, i4n.astype(np.int64), 1), rtol=1e-6)
    assert np.allclose(g4n / g4n.sum(1, keepdims=True), g, rtol=1e-5)


# ------------------------------------------------------------------------------------------
# Expert FFN (steps a5-a6; Eq. 1's three h x h_i matrices; reading R2)
# ------------------------------------------------------------------------------------------
def test_expert_ffn_hand_example():
    """h=2, h_i=1: W1=[1,0], W3=[0,1], x=[2,3] -> a=2, b=3, u=3*2/(1+e^-2); W2=[[1],[-0.5]]."""
    x = _bf([2.0, 3.0])
    w1 = _bf([[1.0, 0.0]])
    w3 = _bf([[0.0, 1.0]])
    w2 = _bf([[1.0], [-0.5]])
    v = oracle.expert_ffn(x, w1, w3, w2)
    u = 3.0 * 2.0 / (1.0 + math.exp(-2.0))
    assert np.allclose(v, [u, -0.5 * u], rtol=1e-6)


def test_expert_ffn_vs_torch_fp64(tiny_inputs):
    inp = tiny_inputs
    for e in (0, 5):
        for t in (0, 17, 63):
            v = oracle.expert_ffn(inp.x[t], inp.w1[e], inp.w3[e], inp.w2[e])
            ref = _dense_swiglu_fp64(inp.x[t:t + 1], inp.w1[e], inp.w3[e], inp.w2[e])[0].numpy()
            assert np.max(np.abs(v - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_expert_ffn_w2_zero_and_scaling(tiny_inputs):
    inp = tiny_inputs
    x = inp.x[3]
    zero = np.zeros_like(inp.w2[1])
    assert np.all(oracle.expert_ffn(x, inp.w1[1], inp.w3[1], zero) == 0)
    # doubling W2 (exact in bf16) doubles v exactly (linear in W2)
    w2x2 = f32_to_bf16_bits(bf16_bits_to_f32(inp.w2[1]) * 2)
    v1 = oracle.expert_ffn(x, inp.w1[1], inp.w3[1], inp.w2[1])
    v2 = oracle.expert_ffn(x, inp.w1[1], inp.w3[1], w2x2)
    assert np.array_equal(v2, 2 * v1)
    # x = 0 -> v = 0
    assert np.all(oracle.expert_ffn(np.zeros_like(x), inp.w1[1], inp.w3[1], inp.w2[1]) == 0)


# ------------------------------------------------------------------------------------------
# Whole layer (steps a2-a7)
# ------------------------------------------------------------------------------------------
def test_single_expert_top1_is_dense_ffn(tiny_inputs):
    inp = tiny_inputs
    y, idx, g = oracle.forward(inp.x, inp.router[:1], inp.w1[:1], inp.w3[:1], inp.w2[:1], top_k=1)
    assert np.all(idx == 0) and np.all(g == 1.0)
    ref = _dense_swiglu_fp64(inp.x, inp.w1[0], inp.w3[0], inp.w2[0]).numpy()
    assert np.max(np.abs(y - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_identical_experts_give_dense_ffn(tiny_inputs):
    inp = tiny_inputs
    ne = inp.cfg.num_experts
    y, _, _ = oracle.forward(inp.x, inp.router, [inp.w1[2]] * ne, [inp.w3[2]] * ne,
                             [inp.w2[2]] * ne, top_k=2)
    ref = _dense_swiglu_fp64(inp.x, inp.w1[2], inp.w3[2], inp.w2[2]).numpy()
    assert np.max(np.abs(y - ref)) <= 2e-5 * np.max(np.abs(ref))


def test_k_equals_ne_is_full_softmax_mixture(tiny_inputs):
    inp = tiny_inputs
    ne = inp.cfg.num_experts
    y, _, _ = oracle.forward(inp.x, inp.router, inp.w1[:ne], inp.w3[:ne], inp.w2[:ne], top_k=ne)
    logits = _t64(inp.x) @ _t64(inp.router).T
    p = torch.softmax(logits, dim=1)
    ref = sum(p[:, e:e + 1] * _dense_swiglu_fp64(inp.x, inp.w1[e], inp.w3[e], inp.w2[e])
              for e in range(ne)).numpy()
    assert np.max(np.abs(y - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_top2_matches_torch_mixture(tiny_inputs):
    """Top-2 layer = sum over the 2 selected experts of renormalised softmax * FFN (torch fp64)."""
    inp = tiny_inputs
    y, idx, g = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, top_k=2)
    logits = (_t64(inp.x) @ _t64(inp.router).T)
    top = torch.topk(logits, 2, dim=1)
    assert np.array_equal(np.sort(top.indices.numpy(), 1), np.sort(idx, 1))
    p = torch.softmax(top.values, dim=1)
    ffn = [_dense_swiglu_fp64(inp.x, inp.w1[e], inp.w3[e], inp.w2[e]) for e in range(8)]
    ref = torch.stack([sum(p[t, j] * ffn[int(top.indices[t, j])][t] for j in range(2))
                       for t in range(inp.x.shape[0])]).numpy()
    assert np.max(np.abs(y - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_token_permutation_equivariance(tiny_inputs):
    inp = tiny_inputs
    perm = np.random.default_rng(9).permutation(inp.x.shape[0])
    y, idx, g = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, top_k=2)
    yp, idxp, gp = oracle.forward(inp.x[perm], inp.router, inp.w1, inp.w3, inp.w2, top_k=2)
    assert np.array_equal(yp, y[perm]) and np.array_equal(idxp, idx[perm])
    assert np.array_equal(gp, g[perm])


def test_shared_experts_concatenation(tiny_inputs):
    """Two shared experts of width h_i == one shared FFN of width 2*h_i (reading R10)."""
    inp = tiny_inputs
    ne = inp.cfg.num_experts
    w1 = inp.w1[:ne] + [inp.w1[0], inp.w1[1]]
    w3 = inp.w3[:ne] + [inp.w3[0], inp.w3[1]]
    w2 = inp.w2[:ne] + [inp.w2[0], inp.w2[1]]
    y_s, idx, g = oracle.forward(inp.x, inp.router, w1, w3, w2, top_k=2, n_shared=2)
    y_0, idx0, g0 = oracle.forward(inp.x, inp.router, inp.w1[:ne], inp.w3[:ne], inp.w2[:ne], top_k=2)
    assert np.array_equal(idx, idx0) and np.array_equal(g, g0)
    cat1 = np.concatenate([inp.w1[0], inp.w1[1]], 0)
    cat3 = np.concatenate([inp.w3[0], inp.w3[1]], 0)
    cat2 = np.concatenate([inp.w2[0], inp.w2[1]], 1)
    ref = _dense_swiglu_fp64(inp.x, cat1, cat3, cat2).numpy()
    assert np.max(np.abs((y_s - y_0) - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_zero_tokens_and_invalid_args(tiny_inputs):
    inp = tiny_inputs
    y, idx, g = oracle.forward(inp.x[:0], inp.router, inp.w1, inp.w3, inp.w2, top_k=2)
    assert y.shape == (0, 128)
    with pytest.raises(ValueError):
        oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, top_k=9)   # top_k > N_e


def test_determinism(tiny_inputs):
    inp = tiny_inputs
    a = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, top_k=2)
    b = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, top_k=2)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_whole_layer_c4_slice_vs_torch_fp64():
    """SURVEY §8(c.3) 'whole layer': an independent torch fp64 implementation on a token slice of
    the C4 (DeepSeek-V2-Lite-shaped: 64 routed experts, top-6, 2 shared) workload -- routing by
    torch.topk on fp64 logits, renormalised softmax gates, SwiGLU experts, shared experts added
    with weight 1 (readings R1-R3, R10) -- against the oracle: idx equal, y within 1e-5."""
    cfg = synth.CONFIGS["dsv2_lite"]
    inp = synth.gen_inputs(cfg, tokens=48)
    y, idx, g = oracle.forward(inp.x, inp.router, inp.w1, inp.w3, inp.w2, cfg.top_k,
                               n_shared=cfg.num_shared)
    x = _t64(inp.x)
    logits = x @ _t64(inp.router).T
    top = torch.topk(logits, cfg.top_k, dim=1)     # no exact ties in this draw
    assert np.array_equal(top.indices.numpy(), idx)
    p = torch.softmax(top.values, dim=1)
    assert np.max(np.abs(p.numpy() - g)) <= 1e-6
    ref = torch.zeros(x.shape[0], cfg.hidden, dtype=torch.float64)
    used = sorted(set(idx.ravel().tolist()))
    ffn = {e: _dense_swiglu_fp64(inp.x, inp.w1[e], inp.w3[e], inp.w2[e]) for e in used}
    for t in range(x.shape[0]):
        for j in range(cfg.top_k):
            ref[t] += p[t, j] * ffn[int(top.indices[t, j])][t]
    for s in range(cfg.num_shared):
        e = cfg.num_experts + s
        ref += _dense_swiglu_fp64(inp.x, inp.w1[e], inp.w3[e], inp.w2[e])
    ref = ref.numpy()
    assert np.max(np.abs(y - ref)) <= 1e-5 * np.max(np.abs(ref))


def _rank_count_mask(logits, k):
    """Vectorised rank-count definition (numpy, independent of the oracle's C selection):
    e in S_t  <=>  #{e' : l_e' > l_e  or (l_e' == l_e and e' < e)} < k."""
    l = logits[:, None, :]          # [T, 1, e']
    m = logits[:, :, None]          # [T, e, 1]
    ne = logits.shape[1]
    lower = np.arange(ne)[None, None, :] < np.arange(ne)[None, :, None]
    above = (l > m) | ((l == m) & lower)
    return above.sum(axis=2) < k    # [T, e]


@pytest.mark.parametrize("name,k_override", [
    ("tiny", None), ("mixtral_8x7b", None), ("mixtral_8x22b", None), ("dbrx", None),
    ("dsv2_lite", None),                       # (N_e, k) = (64, 6): the C4 shape
    ("envelope_128x8", None),                  # (128, 8): the envelope maximum
])
def test_topk_on_config_logits(name, k_override):
    """Routing on REAL config logits (a token sample of every BASELINE workload's structure, plus
    the envelope maximum N_e = 128, k = 8) by two routes other than the oracle's selection loop:
    (1) the rank-count definition (PAPER.md:269 'top-N_k of N_e', reading R5's order), vectorised;
    (2) Python's sorted() with key (-logit, index) -- which also fixes the listed ORDER.  Where
    C(N_e, k) is small, (3) exhaustive subset enumeration on the first tokens as well.  Some rows
    get duplicated router rows so exact ties occur."""
    if name == "envelope_128x8":
        cfg = synth.MoEConfig("envelope_128x8", 50, 1024, 128, 128, 8, 1024)
    else:
        cfg = synth.CONFIGS[name]
    T = min(cfg.tokens, 1024)
    inp = synth.gen_inputs(cfg, tokens=T, experts=False)
    router = inp.router.copy()
    router[cfg.num_experts - 1] = router[0]           # exact ties between experts 0 and N_e - 1
    logits = oracle.router_logits(inp.x, router)
    k = cfg.top_k
    idx, gates = oracle.topk_gates(logits, k)
    mask = _rank_count_mask(logits, k)
    for t in range(T):
        assert sorted(idx[t].tolist()) == np.nonzero(mask[t])[0].tolist(), t
        ref = sorted(range(cfg.num_experts), key=lambda e: (-logits[t, e], e))[:k]
        assert idx[t].tolist() == ref, t
    if math.comb(cfg.num_experts, k) <= 2000:
        for t in range(min(T, 64)):
            assert sorted(idx[t].tolist()) == _enumerate_best_subset(logits[t], k)
    assert np.allclose(gates.astype(np.float64).sum(1), 1.0, atol=1e-6)


@pytest.mark.parametrize("name,tokens", [("mixtral_8x7b", 2), ("mixtral_8x22b", 2), ("dbrx", 1)])
def test_whole_layer_full_shape_slice_vs_torch_fp64(name, tokens):
    """SURVEY §8(c.3) 'whole layer' at the C1-C3 shapes: an independent torch fp64 layer on a
    token slice -- fp64 router matmul, selection by a stable sort on (-logit, index), softmax over
    the k selected logits, SwiGLU experts W2 (silu(W1 x) * W3 x) in fp64, gate-weighted sum
    (readings R1-R3, R5) -- against the oracle: idx equal, y within 1e-5 of the largest output.
    Only the routed experts' weights are generated (each expert's draw is independent of the
    others, synth.gen_inputs(expert_ids=...))."""
    cfg = synth.CONFIGS[name]
    head = synth.gen_inputs(cfg, tokens=tokens, experts=False)
    x = _t64(head.x)
    logits = x @ _t64(head.router).T
    order = [sorted(range(cfg.num_experts), key=lambda e: (-float(logits[t, e]), e))[:cfg.top_k]
             for t in range(tokens)]
    used = sorted({e for row in order for e in row})
    sub = synth.gen_inputs(cfg, tokens=tokens, expert_ids=used)
    assert np.array_equal(sub.x, head.x)
    w = {e: (sub.w1[i], sub.w3[i], sub.w2[i]) for i, e in enumerate(used)}
    ref = torch.zeros(tokens, cfg.hidden, dtype=torch.float64)
    for t in range(tokens):
        sel = torch.tensor([float(logits[t, e]) for e in order[t]], dtype=torch.float64)
        p = torch.softmax(sel, dim=0)
        for j, e in enumerate(order[t]):
            ref[t] += p[j] * _dense_swiglu_fp64(head.x[t:t + 1], *w[e])[0]
    # the oracle on the same tokens, routed by its own router + top-k; it reads only the routed
    # experts' weights (unrouted experts are given a stand-in that is never read)
    lg = oracle.router_logits(head.x, head.router)
    idx, g = oracle.topk_gates(lg, cfg.top_k)
    assert idx.tolist() == order
    mats = [[w.get(e, w[used[0]])[m] for e in range(cfg.num_experts)] for m in range(3)]
    y = oracle.experts_combine(head.x, mats[0], mats[1], mats[2], cfg.num_experts, 0, idx, g)
    ref = ref.numpy()
    assert np.max(np.abs(y - ref)) <= 1e-5 * np.max(np.abs(ref))
