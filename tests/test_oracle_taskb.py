"""Pins of the oracle's GPU Task B (oracle/moe_oracle.c; readings R19-R21).

Each test ties the oracle to something other than itself: special cases with exact answers
(Wo = 0 or I, one-hot attention rows that select one COLUMN of Wo^T, constant rows whose RMSNorm
is +-1), exact invariants (power-of-two scaling), and fp64 torch formulas within a rounding
bound -- chosen so that a transposed Wo, a dropped residual, a missing 1/h, a misplaced eps or
gamma, or a lost residual around the MoE fails one of them.
"""
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


def _f(bits):
    return bf16_bits_to_f32(bits).astype(np.float64)


def _rand(rng, shape, scale=1.0):
    return _bf(rng.standard_normal(shape) * scale)


def _ulp_bf16(x):
    """bf16 spacing at |x| (8 significant bits)."""
    x = np.maximum(np.abs(x), 1e-30)
    return 2.0 ** (np.floor(np.log2(x)) - 7)


# ------------------------------------------------------------------------------- b1: O-proj
def test_oproj_wo_zero_is_residual():
    rng = np.random.default_rng(1)
    T, h = 9, 64
    attn, resid = _rand(rng, (T, h)), _rand(rng, (T, h))
    h1 = oracle.oproj_residual(attn, resid, np.zeros((h, h), np.uint16))
    assert np.array_equal(h1, resid)


def test_oproj_identity_is_bf16_sum():
    """Wo = I: h1 = bf16(attn + resid) (the fp64 sum of two bf16 values is exact)."""
    rng = np.random.default_rng(2)
    T, h = 7, 32
    attn, resid = _rand(rng, (T, h)), _rand(rng, (T, h))
    h1 = oracle.oproj_residual(attn, resid, _bf(np.eye(h)))
    exact = _f(attn) + _f(resid)
    assert np.array_equal(h1, _bf(exact.astype(np.float32)))


def test_oproj_one_hot_selects_column():
    """attn[t] = e_i: h1[t, c] = bf16(Wo[c, i] + resid[t, c]) -- catches a transposed Wo."""
    rng = np.random.default_rng(3)
    h = 48
    wo = _rand(rng, (h, h))
    resid = np.zeros((h, h), np.uint16)
    attn = _bf(np.eye(h))
    h1 = oracle.oproj_residual(attn, resid, wo)
    assert np.array_equal(h1, wo.T)       # row t of h1 is column t of Wo
    assert not np.array_equal(wo, wo.T)


def test_oproj_vs_fp64_matmul():
    rng = np.random.default_rng(4)
    T, h = 13, 256
    attn, resid, wo = _rand(rng, (T, h)), _rand(rng, (T, h)), _rand(rng, (h, h), 0.05)
    h1 = _f(oracle.oproj_residual(attn, resid, wo))
    ref = (torch.from_numpy(_f(attn)) @ torch.from_numpy(_f(wo)).T).numpy() + _f(resid)
    # one bf16 rounding (+ the float step): at most one bf16 ulp
    assert np.all(np.abs(h1 - ref) <= _ulp_bf16(ref) * 0.5 + 1e-12)


# ------------------------------------------------------------------------------- b2: RMSNorm
def test_rmsnorm_constant_rows_are_unit():
    """h1 row = a (constant): mean square a^2, so u = sign(a) * gamma exactly (eps = 0)."""
    vals = [0.5, -3.0, 1.25, -0.0078125, 96.0]
    h = 64
    h1 = _bf(np.repeat(np.array(vals, np.float32)[:, None], h, axis=1))
    gamma = _bf(np.ones(h))
    u = _f(oracle.rmsnorm(h1, gamma, 0.0))
    assert np.array_equal(u, np.sign(np.array(vals))[:, None] * np.ones((1, h)))
    g2 = _bf(np.linspace(-2, 2, h))
    u2 = _f(oracle.rmsnorm(h1, g2, 0.0))
    assert np.array_equal(u2, np.sign(np.array(vals))[:, None] * _f(g2)[None, :])


def test_rmsnorm_power_of_two_scale_invariant():
    rng = np.random.default_rng(5)
    T, h = 11, 128
    x = rng.standard_normal((T, h))
    gamma = _rand(rng, (h,))
    u1 = oracle.rmsnorm(_bf(x), gamma, 0.0)
    u2 = oracle.rmsnorm(_bf(x * 8.0), gamma, 0.0)
    assert np.array_equal(u1, u2)


def test_rmsnorm_vs_fp64_formula():
    """u ~ gamma * h1 / sqrt(mean(h1^2) + eps) within two bf16 roundings."""
    rng = np.random.default_rng(6)
    T, h = 17, 512
    h1 = _rand(rng, (T, h), 3.0)
    gamma = _rand(rng, (h,))
    for eps in (1e-5, 1e-6, 4.0):
        u = _f(oracle.rmsnorm(h1, gamma, eps))
        x = _f(h1)
        ref = _f(gamma)[None, :] * x / np.sqrt((x * x).mean(axis=1, keepdims=True) + np.float32(eps))
        # n = bf16(h1 r) errs by <= 2^-8 |n| relative (half an ulp of 8 significant bits), then
        # u = bf16(gamma n) by half an ulp of u
        assert np.all(np.abs(u - ref) <= 2.0 ** -8 * 1.01 * np.abs(ref) + 0.5 * _ulp_bf16(ref))


def test_rmsnorm_eps_matters():
    """Large eps shrinks the output: r = 1/sqrt(ms + eps) (eps inside the sqrt, per token)."""
    h = 64
    h1 = _bf(np.full((1, h), 1.0))
    gamma = _bf(np.ones(h))
    u = _f(oracle.rmsnorm(h1, gamma, 3.0))  # 1 / sqrt(1 + 3) = 0.5
    assert np.array_equal(u, np.full((1, h), 0.5))


# ------------------------------------------------------------------------------- whole Task B
def _small_layer(rng, T=12, h=128, ffn=128, ne=4, k=2, S=0, w2_zero=False):
    attn, resid = _rand(rng, (T, h)), _rand(rng, (T, h))
    wo, gamma = _rand(rng, (h, h), 0.05), _bf(1.0 + 0.1 * rng.standard_normal(h))
    router = _rand(rng, (ne, h), 0.1)
    n = ne + S
    w1 = [_rand(rng, (ffn, h), 0.05) for _ in range(n)]
    w3 = [_rand(rng, (ffn, h), 0.05) for _ in range(n)]
    w2 = [(np.zeros((h, ffn), np.uint16) if w2_zero else _rand(rng, (h, ffn), 0.05))
          for _ in range(n)]
    return attn, resid, wo, gamma, router, w1, w3, w2


def test_taskb_w2_zero_is_h1():
    rng = np.random.default_rng(7)
    attn, resid, wo, gamma, router, w1, w3, w2 = _small_layer(rng, S=1, w2_zero=True)
    y, h1, u, idx, gates = oracle.taskb_forward(attn, resid, wo, gamma, 1e-5, router, w1, w3, w2,
                                                2, n_shared=1)
    assert np.array_equal(y, bf16_bits_to_f32(h1))


def test_taskb_is_composition():
    """y = h1 + MoE(u) with h1 = b1(attn, resid), u = b2(h1) and the pinned MoE oracle."""
    rng = np.random.default_rng(8)
    attn, resid, wo, gamma, router, w1, w3, w2 = _small_layer(rng, S=1)
    y, h1, u, idx, gates = oracle.taskb_forward(attn, resid, wo, gamma, 1e-5, router, w1, w3, w2,
                                                2, n_shared=1)
    assert np.array_equal(h1, oracle.oproj_residual(attn, resid, wo))
    assert np.array_equal(u, oracle.rmsnorm(h1, gamma, 1e-5))
    ym, im, gm = oracle.forward(u, router, w1, w3, w2, 2, n_shared=1)
    assert np.array_equal(idx, im) and np.array_equal(gates, gm)
    assert np.array_equal(y, bf16_bits_to_f32(h1) + ym)
    # routing happens on the normalised u, not on h1 or attn
    assert not np.array_equal(oracle.forward(h1, router, w1, w3, w2, 2, n_shared=1)[0], ym)


def test_taskb_rejects_bad_eps():
    rng = np.random.default_rng(9)
    attn, resid, wo, gamma, router, w1, w3, w2 = _small_layer(rng, T=2)
    with pytest.raises(ValueError):
        oracle.taskb_forward(attn, resid, wo, gamma, -1.0, router, w1, w3, w2, 2)
