"""Helpers for the GPU parity tests: run the CUDA path through the C ABI on seeded inputs and
compare with the oracle (tests only)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth
from paper_2504_09345_b200 import HostExperts, MoELayer


def bf16_tensor(bits: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(device)


def to_f32(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


class GpuRun:
    """One context + pinned experts for a set of inputs."""

    def __init__(self, inp: synth.MoEInputs, max_tokens=None, profile=False, packet_bytes=0,
                 renormalize=True, force_ep=False, mover=False, num_slots=0):
        cfg = inp.cfg
        self.inp = inp
        self.layer = MoELayer(cfg.hidden, cfg.ffn, cfg.num_experts, cfg.top_k,
                              max_tokens or max(1, inp.x.shape[0]), num_shared=cfg.num_shared,
                              renormalize=renormalize, profile=profile, packet_bytes=packet_bytes,
                              force_ep=force_ep, mover=mover, num_slots=num_slots)
        self.experts = HostExperts(cfg.hidden, cfg.ffn, inp.w1, inp.w3, inp.w2)
        self.router = bf16_tensor(inp.router)

    def run(self, x_bits=None, stream=None):
        x_bits = self.inp.x if x_bits is None else x_bits
        T = x_bits.shape[0]
        k = self.inp.cfg.top_k
        x = bf16_tensor(x_bits)
        out = torch.empty_like(x)
        idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
        gates = torch.empty((T, k), dtype=torch.float32, device="cuda")
        s = torch.cuda.current_stream() if stream is None else stream
        self.layer.forward(x, self.router, self.experts, out, idx, gates, stream=s.cuda_stream)
        s.synchronize()
        self.layer.sync()
        return out, idx, gates

    def close(self):
        self.layer.close()
        self.experts.close()


def token_rel_err(y_gpu: np.ndarray, y_ref: np.ndarray) -> np.ndarray:
    """Per-token max-abs error over the token's max-abs reference value (reading R9)."""
    num = np.max(np.abs(y_gpu.astype(np.float64) - y_ref.astype(np.float64)), axis=1)
    den = np.maximum(np.max(np.abs(y_ref.astype(np.float64)), axis=1), 1e-30)
    return num / den


def sample_tokens(T: int, n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    fixed = [0, 1, T // 2, T - 2, T - 1]
    rest = rng.choice(T, size=min(T, n), replace=False)
    return np.unique(np.clip(np.concatenate([fixed, rest]), 0, T - 1))


def stratified_tokens(idx: np.ndarray, num_experts: int, num_shared: int = 0,
                      block: int = 128) -> np.ndarray:
    """Tokens that touch every (expert, 128-row M tile) of the permuted layout -- and so every
    256-row CTA-pair tile and every raster group of every GEMM launch -- including each group's
    first and last row (VERDICT r1 "stratified token set").

    Inside expert e's group the rows are the (t, j) with idx[t, j] == e in ascending t (reading
    R12); for every 128-row block of the group the tokens at its first and last row are taken,
    plus the group's last row.  Shared experts (and Task B's O-projection) take all T tokens in
    order: the first and last token of every 128-token block."""
    T, k = idx.shape
    flat = np.asarray(idx).ravel()
    sel = set()
    for e in range(num_experts):
        rows = np.nonzero(flat == e)[0]          # ascending flat index = ascending t
        n = len(rows)
        if n == 0:
            continue
        for p in set(range(0, n, block)) | set(range(block - 1, n, block)) | {n - 1}:
            sel.add(int(rows[p]) // k)
    if num_shared:
        sel |= set(block_tokens(T, block).tolist())
    return np.array(sorted(sel), dtype=np.int64)


def block_tokens(T: int, block: int = 128) -> np.ndarray:
    """First and last token of every `block`-token M tile of a GEMM over all T tokens."""
    s = set(range(0, T, block)) | set(range(block - 1, T, block)) | {T - 1}
    return np.array(sorted(s), dtype=np.int64)


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3}


def dev_view(ptr: int, shape, typestr: str) -> torch.Tensor:
    """Read-only torch view of a raw device pointer owned by the library (debug buffers)."""
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device="cuda")


def run_local_ep(inp: synth.MoEInputs, world: int, shard: bool = False, mover: bool = False,
                 calls: int = 2, key: bytes = None, stream_per_rank: bool = True):
    """MOE_FLAG_LOCAL_EP: `world` contexts on this GPU, one host thread each, every rank owning
    T / W tokens and N_e / W experts (+ the shared ones, or its column slice with `shard`).
    Returns (per-rank (out, idx) device tensors, per-rank stats, token bounds)."""
    import os
    import threading
    from paper_2504_09345_b200 import shared_slice_weights
    cfg = inp.cfg
    ne, nl, S, T, h = cfg.num_experts, cfg.num_experts // world, cfg.num_shared, cfg.tokens, cfg.hidden
    bounds = [T * r // world for r in range(world + 1)]
    key = key or os.urandom(128)
    router = bf16_tensor(inp.router)
    experts, layers = [], []
    try:
        for r in range(world):
            if shard:
                ids = list(range(r * nl, (r + 1) * nl))
                sl = shared_slice_weights(cfg.ffn, inp.w1[ne:], inp.w3[ne:], inp.w2[ne:], world, r)
            else:
                ids = list(range(r * nl, (r + 1) * nl)) + [ne + s for s in range(S)]
                sl = None
            experts.append(HostExperts(h, cfg.ffn, [inp.w1[i] for i in ids],
                                       [inp.w3[i] for i in ids], [inp.w2[i] for i in ids],
                                       slice_=sl))
        for r in range(world):
            layers.append(MoELayer(h, cfg.ffn, ne, cfg.top_k, max(1, -(-T // world)),
                                   num_shared=S, world_size=world, rank=r, nccl_unique_id=key,
                                   local_ep=True, shard_shared=shard, mover=mover,
                                   packet_bytes=(64 << 10) if mover else 0))
        bufs = []
        for r in range(world):
            x = bf16_tensor(inp.x[bounds[r]:bounds[r + 1]].reshape(-1, h))
            bufs.append((torch.cuda.Stream(), x, torch.empty_like(x),
                         torch.empty((x.shape[0], cfg.top_k), dtype=torch.int32, device="cuda")))
        torch.cuda.synchronize()
        errors = []

        def work(r):
            try:
                s, x, o, idx = bufs[r]
                for _ in range(calls):
                    layers[r].forward(x, router, experts[r], o, idx, stream=s.cuda_stream)
                s.synchronize()
            except Exception as e:  # noqa: BLE001 -- reported below
                msg = repr(e)[:300]
                try:
                    layers[r].sync()
                except Exception as e2:  # noqa: BLE001
                    msg += f" | sync: {e2!r}"[:300]
                errors.append((r, msg))

        threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert not errors, "\n".join(f"rank {r}: {e}" for r, e in errors)
        stats = [l.stats() for l in layers]
        return [(b[2], b[3]) for b in bufs], stats, bounds
    finally:
        for l in layers:
            l.close()
        for e in experts:
            e.close()
