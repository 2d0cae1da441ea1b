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
