"""Seeded synthetic inputs for the MoE-layer hot path (shared by oracle tests, GPU tests and bench).

This module holds NO arithmetic of the method (no routing, no FFN, no combine): it only draws
random numbers, rounds them to bf16 and shapes them like the paper's workloads.  Both the oracle
(``oracle/``) and the CUDA path (``paper_2504_09345_b200``) consume the identical bf16 arrays it
returns, so neither side ever computes an input for the other.

Recipe:
  * seeds: ``SeedSequence(entropy=250409345, spawn_key=(config_id, layer))`` with children
    [x, router, expert_0..N_e-1, shared_0..S-1, structure];
  * values drawn in fp32 and rounded to bf16 (round-to-nearest-even);
  * x ~ N(0,1) (unit RMS, like post-RMSNorm hidden states); W_r, W1, W3 ~ U(+-1/sqrt(h));
    W2 ~ U(+-1/sqrt(h_i))  (nn.Linear init bounds);
  * C3 (DBRX-shaped) is a mixed batch: 126 prefill prompts x 98 tokens (MTBench mean prompt
    length) followed by decode tokens; prefill tokens share a per-prompt direction;
  * C4 (DeepSeek-V2-Lite-shaped) is skewed: x = normalize(eps + gamma * u_c(t)), topic c(t) drawn
    from a Zipf(1.3) law truncated to 64 topics, u_c a router row scaled to norm sqrt(h).

bf16 values are carried as ``numpy.uint16`` bit patterns.
"""
from __future__ import annotations

import dataclasses
import math
from concurrent.futures import ThreadPoolExecutor
from typing import List, Optional

import numpy as np

ENTROPY = 250409345


@dataclasses.dataclass(frozen=True)
class MoEConfig:
    """Shape of one MoE layer (PAPER.md:269 notation: h, h_i, N_e, N_k) plus the token batch T."""

    name: str
    config_id: int
    hidden: int          # h
    ffn: int             # h_i
    num_experts: int     # N_e (routed)
    top_k: int           # N_k
    tokens: int          # T
    num_shared: int = 0  # always-on experts (C4 only)
    structure: str = "iid"  # iid | mixed | skewed

    @property
    def expert_bytes(self) -> int:
        """bf16 bytes of one expert's three matrices (W1, W3: [h_i,h]; W2: [h,h_i])."""
        return 3 * self.hidden * self.ffn * 2

    def with_tokens(self, tokens: int) -> "MoEConfig":
        return dataclasses.replace(self, tokens=tokens)


# BASELINE.json "configs", in order (config_id = index).
CONFIGS = {
    "tiny": MoEConfig("tiny", 0, 128, 256, 8, 2, 64),
    "mixtral_8x7b": MoEConfig("mixtral_8x7b", 1, 4096, 14336, 8, 2, 4096),
    "mixtral_8x22b": MoEConfig("mixtral_8x22b", 2, 6144, 16384, 8, 2, 8192),
    "dbrx": MoEConfig("dbrx", 3, 6144, 10752, 16, 4, 16384, structure="mixed"),
    "dsv2_lite": MoEConfig("dsv2_lite", 4, 2048, 1408, 64, 6, 32768, num_shared=2,
                           structure="skewed"),
}
CONFIG_ORDER = ["tiny", "mixtral_8x7b", "mixtral_8x22b", "dbrx", "dsv2_lite"]


# ---------------------------------------------------------------------------------------------
# bf16 bit helpers (representation only)
# ---------------------------------------------------------------------------------------------
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 with round-to-nearest-even; returns uint16 bit patterns (no NaN input)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = a.view(np.uint32)
    r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(a: np.ndarray) -> np.ndarray:
    """Exact upcast of bf16 bit patterns to fp32."""
    return (np.asarray(a, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


# ---------------------------------------------------------------------------------------------
# Generators
# ---------------------------------------------------------------------------------------------
@dataclasses.dataclass
class MoEInputs:
    cfg: MoEConfig
    x: np.ndarray            # [T, h]     uint16 (bf16)
    router: np.ndarray       # [N_e, h]   uint16 (bf16)
    w1: List[np.ndarray]     # N_e + S of [h_i, h] uint16; routed experts first, then shared
    w3: List[np.ndarray]     # N_e + S of [h_i, h]
    w2: List[np.ndarray]     # N_e + S of [h, h_i]
    topic: Optional[np.ndarray] = None  # C4: per-token topic id (diagnostic only)

    @property
    def num_all_experts(self) -> int:
        return self.cfg.num_experts + self.cfg.num_shared


def _seed_children(cfg: MoEConfig, layer: int) -> List[np.random.SeedSequence]:
    ss = np.random.SeedSequence(entropy=ENTROPY, spawn_key=(cfg.config_id, layer))
    n = 2 + cfg.num_experts + cfg.num_shared + 1
    return ss.spawn(n)


def _uniform_bf16(rng: np.random.Generator, shape, bound: float) -> np.ndarray:
    u = rng.random(int(np.prod(shape)), dtype=np.float32)
    u *= np.float32(2.0 * bound)
    u -= np.float32(bound)
    return f32_to_bf16_bits(u).reshape(shape)


def gen_expert(cfg: MoEConfig, child: np.random.SeedSequence):
    """One expert's canonical (PyTorch nn.Linear orientation) bf16 matrices W1, W3 [h_i,h], W2 [h,h_i]."""
    rng = np.random.default_rng(child)
    b1 = 1.0 / math.sqrt(cfg.hidden)
    b2 = 1.0 / math.sqrt(cfg.ffn)
    w1 = _uniform_bf16(rng, (cfg.ffn, cfg.hidden), b1)
    w3 = _uniform_bf16(rng, (cfg.ffn, cfg.hidden), b1)
    w2 = _uniform_bf16(rng, (cfg.hidden, cfg.ffn), b2)
    return w1, w3, w2


def gen_router(cfg: MoEConfig, layer: int = 0) -> np.ndarray:
    ch = _seed_children(cfg, layer)
    return _uniform_bf16(np.random.default_rng(ch[1]), (cfg.num_experts, cfg.hidden),
                         1.0 / math.sqrt(cfg.hidden))


def _normalize_rows(a: np.ndarray) -> np.ndarray:
    rms = np.sqrt(np.mean(a.astype(np.float64) ** 2, axis=1, keepdims=True))
    return (a / np.maximum(rms, 1e-12)).astype(np.float32)


def gen_hidden(cfg: MoEConfig, router_bits: np.ndarray, layer: int = 0, tokens: Optional[int] = None):
    """Hidden states x [T, h] (bf16 bits) with the config's structure; returns (x, topic)."""
    ch = _seed_children(cfg, layer)
    T = cfg.tokens if tokens is None else tokens
    h = cfg.hidden
    rng = np.random.default_rng(ch[0])
    srng = np.random.default_rng(ch[-1])
    eps = rng.standard_normal((T, h), dtype=np.float32)
    topic = None
    if cfg.structure == "iid":
        x = eps
    elif cfg.structure == "mixed":
        # 126 prefill prompts x 98 tokens (PAPER.md:901 MTBench mean prompt length), then decode.
        n_prompts, plen = 126, 98
        n_prefill = min(T, n_prompts * plen)
        x = eps.copy()
        n_seq = (n_prefill + plen - 1) // plen
        mu = srng.standard_normal((n_seq, h), dtype=np.float32)
        seq_of_token = np.arange(n_prefill) // plen
        x[:n_prefill] = _normalize_rows(eps[:n_prefill] + np.float32(0.5) * mu[seq_of_token])
    elif cfg.structure == "skewed":
        n_topics = min(64, cfg.num_experts)
        p = np.arange(1, n_topics + 1, dtype=np.float64) ** -1.3
        p /= p.sum()
        rank = srng.choice(n_topics, size=T, p=p)
        perm = srng.permutation(cfg.num_experts)[:n_topics]   # topic rank -> router row
        topic = perm[rank]
        u = bf16_bits_to_f32(router_bits).astype(np.float64)
        u = u / np.linalg.norm(u, axis=1, keepdims=True) * math.sqrt(h)
        gamma = 0.15
        x = _normalize_rows(eps + (gamma * u[topic]).astype(np.float32))
    else:
        raise ValueError(cfg.structure)
    return f32_to_bf16_bits(x), topic


def gen_inputs(cfg: MoEConfig, layer: int = 0, threads: int = 8, tokens: Optional[int] = None,
               experts: bool = True, expert_ids: Optional[List[int]] = None) -> MoEInputs:
    """All inputs of one layer call: x, router and (optionally) the experts' canonical weights.
    expert_ids selects a subset (indices over routed experts then shared ones, e.g. one rank's
    experts under expert parallelism); the weights of expert i never depend on the subset."""
    ch = _seed_children(cfg, layer)
    router = gen_router(cfg, layer)
    x, topic = gen_hidden(cfg, router, layer, tokens)
    w1: List[np.ndarray] = []
    w3: List[np.ndarray] = []
    w2: List[np.ndarray] = []
    if experts:
        n_all = cfg.num_experts + cfg.num_shared
        ids = list(range(n_all)) if expert_ids is None else list(expert_ids)
        kids = [ch[2 + i] for i in ids]
        with ThreadPoolExecutor(max(1, threads)) as ex:
            mats = list(ex.map(lambda c: gen_expert(cfg, c), kids))
        for a, b, c in mats:
            w1.append(a)
            w3.append(b)
            w2.append(c)
    if tokens is not None:
        cfg = cfg.with_tokens(tokens)
    return MoEInputs(cfg, x, router, w1, w3, w2, topic)


@dataclasses.dataclass
class TaskBInputs:
    """GPU Task B inputs: attention output, residual stream, Wo, RMSNorm gamma."""
    attn: np.ndarray         # [T, h] uint16 (bf16)
    resid: np.ndarray        # [T, h]
    wo: np.ndarray           # [h, h]  nn.Linear (out x in)
    gamma: np.ndarray        # [h]
    eps: float


def gen_taskb(cfg: MoEConfig, x_bits: np.ndarray, layer: int = 0) -> TaskBInputs:
    """Task B inputs around a layer's MoE hidden batch x (DESIGN.md input recipe): the residual
    stream carries the config's token structure (resid = 4 x, so the post-norm MoE input keeps
    the routing skew of the MoE-only workload), the attention output is an iid N(0, 1) per
    channel, Wo ~ U(+-1/sqrt(h)) (nn.Linear init scale), gamma ~ U(0.5, 1.5); eps 1e-5 (Mixtral)."""
    ss = np.random.SeedSequence(entropy=ENTROPY, spawn_key=(cfg.config_id, layer, 0xB))
    ra, rw, rg = [np.random.default_rng(c) for c in ss.spawn(3)]
    T, h = x_bits.shape
    attn = f32_to_bf16_bits(ra.standard_normal((T, h), dtype=np.float32))
    resid = f32_to_bf16_bits(bf16_bits_to_f32(x_bits) * np.float32(4.0))
    wo = _uniform_bf16(rw, (h, h), 1.0 / math.sqrt(h))
    g = rg.random(h, dtype=np.float32) + np.float32(0.5)
    return TaskBInputs(attn, resid, wo, f32_to_bf16_bits(g), 1e-5)
