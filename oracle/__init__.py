"""CPU oracle of the MoE layer (arXiv 2504.09345, "MoE layer ... applied to all tokens").

TEST INFRASTRUCTURE ONLY: may be imported solely by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg.  The product package (paper_2504_09345_b200) never imports
it, and it never imports the product package.  The arithmetic lives in ``moe_oracle.c`` (plain C,
fp64 router, fp32 expert FFN, see its header for the step-by-step definition and citations); this
file only compiles it with gcc and marshals numpy arrays through ctypes.

Parity status of each function:
  router_logits  -- pinned (brute force / closed forms / special cases, tests/test_oracle_pins.py)
  topk_gates     -- pinned (subset enumeration, rank-count definition, ties, 2-expert sigmoid)
  expert_ffn     -- pinned (torch fp64 textbook SwiGLU, W2=0, linearity)
  forward        -- pinned (dense equivalence, k=N_e mixture, permutation equivariance, shared experts)
  oproj_residual -- pinned (Wo = 0 / I, one-hot columns, fp64 brute force; tests/test_oracle_taskb.py)
  rmsnorm        -- pinned (constant rows, power-of-2 scale invariance, gamma scaling, fp64 formula)
  taskb_forward  -- pinned (W2 = 0 -> y = h1, composition of the pinned steps)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "moe_oracle.c")
_LIB = os.path.join(_HERE, "libmoe_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile moe_oracle.c with gcc (-O2, no -ffast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        lib.moe_ref_router_logits.argtypes = [P, i64, i32, P, i32, P]
        lib.moe_ref_topk_gates.argtypes = [P, i64, i32, i32, i32, P, P]
        lib.moe_ref_expert_ffn.argtypes = [P, i32, P, P, P, i32, P, P]
        lib.moe_ref_experts_combine.argtypes = [P, i64, i32, i32, P, P, P, i32, i32, P, P, i32, P]
        lib.moe_ref_forward.argtypes = [P, i64, i32, P, i32, i32, i32, P, P, P, i32, i32, P, P, P, P]
        lib.moe_ref_forward.restype = ctypes.c_int
        lib.moe_ref_num_threads.restype = ctypes.c_int
        lib.moe_ref_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _u16(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    assert a.dtype == np.uint16, a.dtype
    return a


def num_threads() -> int:
    return _load().moe_ref_num_threads()


def set_num_threads(n: int) -> None:
    """OpenMP threads of the following oracle calls (timing only; results do not depend on it)."""
    _load().moe_ref_set_num_threads(int(n))


def router_logits(x: np.ndarray, router: np.ndarray) -> np.ndarray:
    x, router = _u16(x), _u16(router)
    T, h = x.shape
    ne = router.shape[0]
    out = np.empty((T, ne), dtype=np.float64)
    _load().moe_ref_router_logits(_ptr(x), T, h, _ptr(router), ne, _ptr(out))
    return out


def topk_gates(logits: np.ndarray, top_k: int, renormalize: bool = True):
    logits = np.ascontiguousarray(logits, dtype=np.float64)
    T, ne = logits.shape
    idx = np.empty((T, top_k), dtype=np.int32)
    gates = np.empty((T, top_k), dtype=np.float32)
    _load().moe_ref_topk_gates(_ptr(logits), T, ne, top_k, int(renormalize), _ptr(idx), _ptr(gates))
    return idx, gates


def expert_ffn(x_row: np.ndarray, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray) -> np.ndarray:
    x_row, w1, w3, w2 = _u16(x_row), _u16(w1), _u16(w3), _u16(w2)
    ffn, h = w1.shape
    u = np.empty(ffn, dtype=np.float32)
    v = np.empty(h, dtype=np.float32)
    _load().moe_ref_expert_ffn(_ptr(x_row), h, _ptr(w1), _ptr(w3), _ptr(w2), ffn, _ptr(u), _ptr(v))
    return v


def _ptr_array(mats: Sequence[np.ndarray]):
    arr = (ctypes.c_void_p * len(mats))(*[_ptr(m) for m in mats])
    return arr


def experts_combine(x, w1, w3, w2, n_experts: int, n_shared: int, idx, gates) -> np.ndarray:
    x = _u16(x)
    T, h = x.shape
    ffn = w1[0].shape[0]
    w1, w3, w2 = [_u16(m) for m in w1], [_u16(m) for m in w3], [_u16(m) for m in w2]
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    gates = np.ascontiguousarray(gates, dtype=np.float32)
    y = np.empty((T, h), dtype=np.float32)
    p1, p3, p2 = _ptr_array(w1), _ptr_array(w3), _ptr_array(w2)
    _load().moe_ref_experts_combine(_ptr(x), T, h, ffn, ctypes.addressof(p1), ctypes.addressof(p3),
                                    ctypes.addressof(p2), n_experts, n_shared, _ptr(idx),
                                    _ptr(gates), idx.shape[1], _ptr(y))
    return y


def forward(x, router, w1, w3, w2, top_k: int, n_shared: int = 0, renormalize: bool = True,
            want_logits: bool = False):
    """Whole MoE layer.  Returns (y fp32 [T,h], idx int32 [T,k], gates fp32 [T,k][, logits])."""
    x, router = _u16(x), _u16(router)
    T, h = x.shape
    ne = router.shape[0]
    ffn = w1[0].shape[0]
    assert len(w1) == ne + n_shared
    w1, w3, w2 = [_u16(m) for m in w1], [_u16(m) for m in w3], [_u16(m) for m in w2]
    y = np.empty((T, h), dtype=np.float32)
    idx = np.empty((T, top_k), dtype=np.int32)
    gates = np.empty((T, top_k), dtype=np.float32)
    logits = np.empty((T, ne), dtype=np.float64) if want_logits else None
    p1, p3, p2 = _ptr_array(w1), _ptr_array(w3), _ptr_array(w2)
    rc = _load().moe_ref_forward(_ptr(x), T, h, _ptr(router), ne, top_k, int(renormalize),
                                 ctypes.addressof(p1), ctypes.addressof(p3), ctypes.addressof(p2),
                                 ffn, n_shared, _ptr(y), _ptr(idx), _ptr(gates),
                                 _ptr(logits) if logits is not None else None)
    if rc != 0:
        raise ValueError(f"moe_ref_forward: invalid arguments (rc={rc})")
    if want_logits:
        return y, idx, gates, logits
    return y, idx, gates


# ----------------------------------------------------------------------------- GPU Task B
def _load_taskb():
    lib = _load()
    if not getattr(lib, "_taskb_ready", False):
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.moe_ref_oproj_residual.argtypes = [P, P, i64, i32, P, P]
        lib.moe_ref_rmsnorm.argtypes = [P, i64, i32, P, ctypes.c_float, P]
        lib.moe_ref_taskb_forward.argtypes = [P, P, i64, i32, P, P, ctypes.c_float, P, i32, i32,
                                              i32, P, P, P, i32, i32, P, P, P, P, P]
        lib.moe_ref_taskb_forward.restype = ctypes.c_int
        lib._taskb_ready = True
    return lib


def oproj_residual(attn, resid, wo) -> np.ndarray:
    """b1 (readings R19/R20): h1 = bf16(resid + attn Wo^T), bf16 bits [T, h]."""
    attn, resid, wo = _u16(attn), _u16(resid), _u16(wo)
    T, h = attn.shape
    h1 = np.empty((T, h), dtype=np.uint16)
    _load_taskb().moe_ref_oproj_residual(_ptr(attn), _ptr(resid), T, h, _ptr(wo), _ptr(h1))
    return h1


def rmsnorm(h1, gamma, eps: float) -> np.ndarray:
    """b2 (reading R21): u = bf16(gamma * bf16(h1 / sqrt(mean(h1^2) + eps))), bf16 bits."""
    h1, gamma = _u16(h1), _u16(gamma)
    T, h = h1.shape
    u = np.empty((T, h), dtype=np.uint16)
    _load_taskb().moe_ref_rmsnorm(_ptr(h1), T, h, _ptr(gamma), eps, _ptr(u))
    return u


def taskb_forward(attn, resid, wo, gamma, eps: float, router, w1, w3, w2, top_k: int,
                  n_shared: int = 0, renormalize: bool = True):
    """GPU Task B.  Returns (y fp32 [T,h], h1 bf16 bits, u bf16 bits, idx, gates)."""
    attn, resid, wo, gamma, router = _u16(attn), _u16(resid), _u16(wo), _u16(gamma), _u16(router)
    T, h = attn.shape
    ne = router.shape[0]
    ffn = w1[0].shape[0]
    w1, w3, w2 = [_u16(m) for m in w1], [_u16(m) for m in w3], [_u16(m) for m in w2]
    h1 = np.empty((T, h), dtype=np.uint16)
    u = np.empty((T, h), dtype=np.uint16)
    y = np.empty((T, h), dtype=np.float32)
    idx = np.empty((T, top_k), dtype=np.int32)
    gates = np.empty((T, top_k), dtype=np.float32)
    p1, p3, p2 = _ptr_array(w1), _ptr_array(w3), _ptr_array(w2)
    rc = _load_taskb().moe_ref_taskb_forward(
        _ptr(attn), _ptr(resid), T, h, _ptr(wo), _ptr(gamma), eps, _ptr(router), ne, top_k,
        int(renormalize), ctypes.addressof(p1), ctypes.addressof(p3), ctypes.addressof(p2), ffn,
        n_shared, _ptr(h1), _ptr(u), _ptr(y), _ptr(idx), _ptr(gates))
    if rc != 0:
        raise ValueError(f"moe_ref_taskb_forward: invalid arguments (rc={rc})")
    return y, h1, u, idx, gates
