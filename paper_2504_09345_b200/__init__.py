"""paper_2504_09345_b200 -- B200-native streamed-weight MoE layer (MoE-Lens, arXiv 2504.09345).

Thin ctypes binding over ``libmoe_b200.so`` (C ABI in ``include/moe.h``): argument marshalling
only -- every step of the layer (routing, permute, expert GEMMs, combine, weight streaming) runs
in the library's sm_100a kernels and copy engine.  There is no CPU or PyTorch fallback: if the
library is missing or the device is not sm_100, the calls fail loudly.

PyTorch is used by callers only for device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libmoe_b200.so")

MOE_OK = 0
MOE_E_INVAL = 1
MOE_E_CUDA = 2
MOE_E_NCCL = 3
MOE_E_NOMEM = 4
MOE_E_NOT_PINNED = 5
MOE_E_UNSUPPORTED = 6
MOE_E_STATE = 7
MOE_FLAG_PROFILE = 1
MOE_FLAG_FORCE_EP = 2
MOE_FLAG_LOCAL_EP = 4

EXPORTED = ["moe_packed_expert_bytes", "moe_pack_expert", "moe_host_alloc", "moe_host_free",
            "moe_init", "moe_layer_forward", "moe_layer_forward_host", "moe_sync", "moe_get_stats",
            "moe_reset_stats", "moe_debug_buffers", "moe_destroy", "moe_status_string",
            "moe_last_error", "moe_probe_h2d", "moe_ep_plan", "moe_nccl_unique_id",
            "moe_packed_layer_bytes", "moe_pack_layer", "moe_taskb_forward",
            "moe_taskb_forward_host", "moe_ep_ipc_handle", "moe_ep_ipc_connect",
            "moe_ep_ipc_selftest", "moe_wait_output", "moe_taskb_forward2_host",
            "moe_ep_group_size", "moe_shared_slice"]
MOE_FLAG_IPC_EP = 8
MOE_FLAG_MOVER = 16
MOE_FLAG_SHARD_SHARED = 32
MOE_IPC_HANDLE_BYTES = 512


class moe_config(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("num_experts", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("num_shared", ctypes.c_int32), ("max_tokens", ctypes.c_int32),
                ("renormalize", ctypes.c_int32), ("device", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("packet_bytes", ctypes.c_int64),
                ("flags", ctypes.c_uint32), ("num_slots", ctypes.c_int32)]


class moe_stats(ctypes.Structure):
    _fields_ = [("calls", ctypes.c_int64), ("h2d_weight_bytes", ctypes.c_int64),
                ("h2d_token_bytes", ctypes.c_int64), ("d2h_token_bytes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("gemm1_launches", ctypes.c_int64),
                ("gemm2_launches", ctypes.c_int64), ("h2d_ms", ctypes.c_double),
                ("route_ms", ctypes.c_double), ("permute_ms", ctypes.c_double),
                ("gemm1_ms", ctypes.c_double), ("gemm2_ms", ctypes.c_double),
                ("combine_ms", ctypes.c_double), ("comm_ms", ctypes.c_double),
                ("num_slots", ctypes.c_int64), ("comm_bytes", ctypes.c_int64),
                ("host_calls", ctypes.c_int64), ("token_latency_ms", ctypes.c_double),
                ("taskb_calls", ctypes.c_int64), ("oproj_ms", ctypes.c_double),
                ("norm_ms", ctypes.c_double), ("gemm1_sm_mhz", ctypes.c_double),
                ("gemm2_sm_mhz", ctypes.c_double), ("part_copies", ctypes.c_int64 * 2),
                ("part_latency_ms", ctypes.c_double * 2), ("h2d_token_ms", ctypes.c_double)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        for f in ("part_copies", "part_latency_ms"):
            d[f] = list(d[f])
        return d


class moe_debug_view(ctypes.Structure):
    _fields_ = [("counts", ctypes.c_void_p), ("offsets", ctypes.c_void_p),
                ("pos", ctypes.c_void_p), ("x_perm", ctypes.c_void_p),
                ("h_act", ctypes.c_void_p), ("y_perm", ctypes.c_void_p),
                ("rows", ctypes.c_int64), ("h1", ctypes.c_void_p), ("moe_in", ctypes.c_void_p),
                ("taskb_tokens", ctypes.c_int64)]


class MoEError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        self.status = status
        super().__init__(f"{status_string(status)}{': ' + detail if detail else ''}")


_lib = None


def load(path: str = LIB_PATH):
    """Load libmoe_b200.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2504_09345_b200.build` "
                          "(the CUDA path has no fallback)")
    lib = ctypes.CDLL(path)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.moe_packed_expert_bytes.argtypes = [i32, i32]
    lib.moe_packed_expert_bytes.restype = i64
    lib.moe_pack_expert.argtypes = [i32, i32, P, P, P, P]
    lib.moe_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
    lib.moe_host_free.argtypes = [P]
    lib.moe_init.argtypes = [ctypes.POINTER(moe_config), ctypes.POINTER(ctypes.c_void_p)]
    lib.moe_layer_forward.argtypes = [P, P, i32, P, P, i32, P, P, P, P]
    lib.moe_layer_forward_host.argtypes = [P, P, i32, P, P, i32, P, P, P, P]
    lib.moe_sync.argtypes = [P]
    lib.moe_get_stats.argtypes = [P, ctypes.POINTER(moe_stats)]
    lib.moe_reset_stats.argtypes = [P]
    lib.moe_debug_buffers.argtypes = [P, ctypes.POINTER(moe_debug_view)]
    lib.moe_destroy.argtypes = [P]
    lib.moe_status_string.argtypes = [ctypes.c_int]
    lib.moe_status_string.restype = ctypes.c_char_p
    lib.moe_last_error.argtypes = [P]
    lib.moe_last_error.restype = ctypes.c_char_p
    lib.moe_probe_h2d.argtypes = [i32, ctypes.c_size_t, i32, ctypes.POINTER(ctypes.c_double)]
    lib.moe_ep_plan.argtypes = [i32, i32, i32, P, P, P, P, P, P]
    lib.moe_ep_plan.restype = i64
    lib.moe_nccl_unique_id.argtypes = [P]
    lib.moe_packed_layer_bytes.argtypes = [i32]
    lib.moe_packed_layer_bytes.restype = i64
    lib.moe_pack_layer.argtypes = [i32, P, P, P]
    lib.moe_taskb_forward.argtypes = [P, P, P, i32, P, ctypes.c_float, P, P, i32, P, P, P, P]
    lib.moe_taskb_forward_host.argtypes = [P, P, P, i32, P, ctypes.c_float, P, P, i32, P, P, P, P]
    lib.moe_ep_ipc_handle.argtypes = [P, P]
    lib.moe_ep_ipc_connect.argtypes = [P, P]
    lib.moe_ep_ipc_selftest.argtypes = [P, ctypes.c_double]
    lib.moe_wait_output.argtypes = [P, P]
    lib.moe_ep_group_size.argtypes = [P, ctypes.POINTER(ctypes.c_int32)]
    lib.moe_taskb_forward2_host.argtypes = [P, P, P, P, P, ctypes.c_float, P, P, i32, P, P, P, P]
    lib.moe_shared_slice.argtypes = [i32, i32, i32, i32, ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int32)]
    for name in EXPORTED:
        if name not in ("moe_packed_expert_bytes", "moe_status_string", "moe_last_error",
                        "moe_ep_plan", "moe_packed_layer_bytes"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def status_string(s: int) -> str:
    return load().moe_status_string(int(s)).decode()


def _check(rc: int, ctx=None):
    if rc != MOE_OK:
        detail = load().moe_last_error(ctx).decode() if ctx else ""
        raise MoEError(rc, detail)


# ----------------------------------------------------------------------------- C ABI, 1:1
def moe_packed_expert_bytes(hidden: int, ffn: int) -> int:
    return int(load().moe_packed_expert_bytes(hidden, ffn))


def moe_pack_expert(hidden: int, ffn: int, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray,
                    dst: int) -> None:
    for a in (w1, w3, w2):
        assert a.dtype == np.uint16 and a.flags.c_contiguous
    _check(load().moe_pack_expert(hidden, ffn, w1.ctypes.data, w3.ctypes.data, w2.ctypes.data, dst))


def moe_shared_slice(ffn: int, num_shared: int, world: int, rank: int) -> tuple:
    """(col0, width): rank's columns of the concatenated shared FFN (MOE_FLAG_SHARD_SHARED)."""
    c0, w = ctypes.c_int32(), ctypes.c_int32()
    _check(load().moe_shared_slice(ffn, num_shared, world, rank, ctypes.byref(c0), ctypes.byref(w)))
    return c0.value, w.value


def shared_slice_weights(ffn: int, w1s: Sequence[np.ndarray], w3s: Sequence[np.ndarray],
                         w2s: Sequence[np.ndarray], world: int, rank: int):
    """The rank's slice of the shared experts (canonical bf16 bit patterns), or None if its width
    is 0: rows [col0, col0 + width) of the row-stacked W1 / W3 and the same columns of the
    column-concatenated W2 (include/moe.h, moe_shared_slice) -- array slicing only."""
    c0, w = moe_shared_slice(ffn, len(w1s), world, rank)
    if w == 0:
        return None
    w1 = np.ascontiguousarray(np.concatenate(list(w1s), axis=0)[c0:c0 + w])
    w3 = np.ascontiguousarray(np.concatenate(list(w3s), axis=0)[c0:c0 + w])
    w2 = np.ascontiguousarray(np.concatenate(list(w2s), axis=1)[:, c0:c0 + w])
    return w1, w3, w2


def moe_host_alloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    _check(load().moe_host_alloc(nbytes, ctypes.byref(p)))
    return p.value


def moe_host_free(ptr: int) -> None:
    _check(load().moe_host_free(ptr))


def moe_init(cfg: moe_config) -> int:
    ctx = ctypes.c_void_p()
    _check(load().moe_init(ctypes.byref(cfg), ctypes.byref(ctx)))
    return ctx.value


def moe_layer_forward(ctx: int, hidden: int, num_tokens: int, router_w: int, experts, top_k: int,
                      out: int, topk_idx: int = 0, topk_w: int = 0, stream: int = 0) -> None:
    _check(load().moe_layer_forward(ctx, hidden, num_tokens, router_w, experts, top_k, out,
                                    topk_idx or None, topk_w or None, stream or None), ctx)


def moe_layer_forward_host(ctx: int, hidden_host: int, num_tokens: int, router_w: int, experts,
                           top_k: int, out_host: int, topk_idx: int = 0, topk_w: int = 0,
                           stream: int = 0) -> None:
    _check(load().moe_layer_forward_host(ctx, hidden_host, num_tokens, router_w, experts, top_k,
                                         out_host, topk_idx or None, topk_w or None,
                                         stream or None), ctx)


def moe_packed_layer_bytes(hidden: int) -> int:
    return int(load().moe_packed_layer_bytes(hidden))


def moe_pack_layer(hidden: int, wo: np.ndarray, gamma: np.ndarray, dst: int) -> None:
    for a in (wo, gamma):
        assert a.dtype == np.uint16 and a.flags.c_contiguous
    _check(load().moe_pack_layer(hidden, wo.ctypes.data, gamma.ctypes.data, dst))


def moe_taskb_forward(ctx: int, attn: int, resid: int, num_tokens: int, layer: int, eps: float,
                      router_w: int, experts, top_k: int, out: int, topk_idx: int = 0,
                      topk_w: int = 0, stream: int = 0) -> None:
    _check(load().moe_taskb_forward(ctx, attn or None, resid or None, num_tokens, layer or None,
                                    eps, router_w, experts, top_k, out or None, topk_idx or None,
                                    topk_w or None, stream or None), ctx)


def moe_taskb_forward_host(ctx: int, attn_host: int, resid: int, num_tokens: int, layer: int,
                           eps: float, router_w: int, experts, top_k: int, out_host: int,
                           topk_idx: int = 0, topk_w: int = 0, stream: int = 0) -> None:
    _check(load().moe_taskb_forward_host(ctx, attn_host or None, resid or None, num_tokens,
                                         layer or None, eps, router_w, experts, top_k,
                                         out_host or None, topk_idx or None, topk_w or None,
                                         stream or None), ctx)


def moe_taskb_forward2_host(ctx: int, attn_host: Sequence[int], resid: Sequence[int],
                            num_tokens: Sequence[int], layer: int, eps: float, router_w: int,
                            experts, top_k: int, out_host: Sequence[int], topk_idx: int = 0,
                            topk_w: int = 0, stream: int = 0) -> None:
    """Two token partitions (alpha, beta) through one stream of the layer's weights."""
    a = (ctypes.c_void_p * 2)(*[p or None for p in attn_host])
    r = (ctypes.c_void_p * 2)(*[p or None for p in resid])
    n = (ctypes.c_int32 * 2)(*num_tokens)
    o = (ctypes.c_void_p * 2)(*[p or None for p in out_host])
    _check(load().moe_taskb_forward2_host(ctx, a, r, n, layer or None, eps, router_w, experts,
                                          top_k, o, topk_idx or None, topk_w or None,
                                          stream or None), ctx)


def moe_wait_output(ctx: int, stream: int = 0) -> None:
    _check(load().moe_wait_output(ctx, stream or None), ctx)


def moe_ep_ipc_handle(ctx: int) -> bytes:
    buf = ctypes.create_string_buffer(MOE_IPC_HANDLE_BYTES)
    _check(load().moe_ep_ipc_handle(ctx, buf), ctx)
    return buf.raw


def moe_ep_ipc_connect(ctx: int, handles: Sequence[bytes]) -> None:
    blob = b"".join(handles)
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(load().moe_ep_ipc_connect(ctx, buf), ctx)


def moe_sync(ctx: int) -> None:
    _check(load().moe_sync(ctx), ctx)


def moe_get_stats(ctx: int) -> dict:
    s = moe_stats()
    _check(load().moe_get_stats(ctx, ctypes.byref(s)), ctx)
    return s.as_dict()


def moe_reset_stats(ctx: int) -> None:
    _check(load().moe_reset_stats(ctx), ctx)


def moe_debug_buffers(ctx: int) -> moe_debug_view:
    v = moe_debug_view()
    _check(load().moe_debug_buffers(ctx, ctypes.byref(v)), ctx)
    return v


def moe_destroy(ctx: int) -> None:
    _check(load().moe_destroy(ctx))


def moe_probe_h2d(device: int = 0, nbytes: int = 1 << 30, iters: int = 5) -> float:
    g = ctypes.c_double()
    _check(load().moe_probe_h2d(device, nbytes, iters, ctypes.byref(g)))
    return g.value


def moe_ep_plan(world: int, rank: int, num_experts: int, counts: np.ndarray) -> dict:
    """Expert-parallel exchange plan (host logic in the library; see include/moe.h)."""
    counts = np.ascontiguousarray(counts, dtype=np.int32).reshape(world, num_experts)
    nl = num_experts // world if world > 0 else 0
    n = max(1, world * nl)
    out = {k: np.zeros(n, dtype=np.int32) for k in ("send_off", "send_cnt", "recv_off", "recv_cnt")}
    out["grp_off"] = np.zeros(nl + 1, dtype=np.int32)
    rows = load().moe_ep_plan(world, rank, num_experts, counts.ctypes.data,
                              out["send_off"].ctypes.data, out["send_cnt"].ctypes.data,
                              out["recv_off"].ctypes.data, out["recv_cnt"].ctypes.data,
                              out["grp_off"].ctypes.data)
    if rows < 0:
        raise MoEError(MOE_E_INVAL, "moe_ep_plan")
    out["recv_rows"] = int(rows)
    return out


def moe_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().moe_nccl_unique_id(buf))
    return buf.raw


# ----------------------------------------------------------------------------- convenience
class HostExperts:
    """Pinned, packed expert blobs of one layer (this rank's routed experts, then shared)."""

    def __init__(self, hidden: int, ffn: int, w1: Sequence[np.ndarray], w3: Sequence[np.ndarray],
                 w2: Sequence[np.ndarray], contiguous: bool = True, slice_=None):
        """contiguous: one pinned region holding every blob back to back (the library then
        moves consecutive small experts with one DMA); else one allocation per expert.
        slice_: (w1, w3, w2) of a shared-FFN slice (shared_slice_weights) appended as the last
        blob, in an allocation of its own (MOE_FLAG_SHARD_SHARED)."""
        self.hidden, self.ffn = hidden, ffn
        self.blob_bytes = moe_packed_expert_bytes(hidden, ffn)
        self.ptrs: List[int] = []
        self._allocs: List[int] = []
        self.slice_bytes = 0
        n = len(w1)
        try:
            if contiguous and n > 0:
                base = moe_host_alloc(self.blob_bytes * n)
                self._allocs.append(base)
                self.ptrs = [base + i * self.blob_bytes for i in range(n)]
            else:
                for _ in range(n):
                    self._allocs.append(moe_host_alloc(self.blob_bytes))
                self.ptrs = list(self._allocs)
            for p, a, b, c in zip(self.ptrs, w1, w3, w2):
                moe_pack_expert(hidden, ffn, np.ascontiguousarray(a), np.ascontiguousarray(b),
                                np.ascontiguousarray(c), p)
            if slice_ is not None:
                a, b, c = slice_
                width = a.shape[0]
                self.slice_bytes = moe_packed_expert_bytes(hidden, width)
                p = moe_host_alloc(self.slice_bytes)
                self._allocs.append(p)
                self.ptrs.append(p)
                moe_pack_expert(hidden, width, np.ascontiguousarray(a), np.ascontiguousarray(b),
                                np.ascontiguousarray(c), p)
        except Exception:
            self.close()
            raise
        self.array = (ctypes.c_void_p * len(self.ptrs))(*self.ptrs)

    @property
    def nbytes(self) -> int:
        n = len(self.ptrs) - (1 if self.slice_bytes else 0)
        return self.blob_bytes * n + self.slice_bytes

    def close(self):
        for p in self._allocs:
            moe_host_free(p)
        self._allocs = []
        self.ptrs = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostLayer:
    """Pinned, packed layer-wise weights of GPU Task B: Wo [h, h] then the RMSNorm gamma [h]."""

    def __init__(self, hidden: int, wo: np.ndarray, gamma: np.ndarray):
        self.hidden = hidden
        self.nbytes = moe_packed_layer_bytes(hidden)
        self.ptr = moe_host_alloc(self.nbytes)
        try:
            moe_pack_layer(hidden, np.ascontiguousarray(wo), np.ascontiguousarray(gamma), self.ptr)
        except Exception:
            self.close()
            raise

    def close(self):
        if self.ptr:
            moe_host_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MoELayer:
    """A context for one MoE layer shape on one device (see include/moe.h)."""

    def __init__(self, hidden: int, ffn: int, num_experts: int, top_k: int, max_tokens: int,
                 num_shared: int = 0, renormalize: bool = True, device: int = 0,
                 world_size: int = 1, rank: int = 0, packet_bytes: int = 0,
                 profile: bool = False, nccl_unique_id: Optional[bytes] = None,
                 force_ep: bool = False, num_slots: int = 0, local_ep: bool = False,
                 ipc_ep: bool = False, mover: bool = False, shard_shared: bool = False):
        """local_ep: in-process expert parallelism over peer memory (MOE_FLAG_LOCAL_EP);
        nccl_unique_id is then the 128-byte group key shared by the `world_size` contexts (one
        host thread each).  ipc_ep: the same transport across processes (MOE_FLAG_IPC_EP): call
        ipc_connect(all ranks' ipc_handle()) before the first forward.  mover: expert copies in
        packets through the library's data-mover thread (MOE_FLAG_MOVER).  shard_shared: the
        shared experts sharded by intermediate columns across the EP group
        (MOE_FLAG_SHARD_SHARED; pass HostExperts(..., slice_=shared_slice_weights(...)))."""
        flags = ((MOE_FLAG_PROFILE if profile else 0) | (MOE_FLAG_FORCE_EP if force_ep else 0) |
                 (MOE_FLAG_LOCAL_EP if local_ep else 0) | (MOE_FLAG_IPC_EP if ipc_ep else 0) |
                 (MOE_FLAG_MOVER if mover else 0) |
                 (MOE_FLAG_SHARD_SHARED if shard_shared else 0))
        self.cfg = moe_config(hidden, ffn, num_experts, top_k, num_shared, max_tokens,
                              int(renormalize), device, world_size, rank, None, packet_bytes,
                              flags, num_slots)
        self._uid = None
        if nccl_unique_id is not None:
            self._uid = ctypes.create_string_buffer(bytes(nccl_unique_id), len(nccl_unique_id))
            self.cfg.nccl_unique_id = ctypes.cast(self._uid, ctypes.c_void_p)
        self.ctx = moe_init(self.cfg)
        self.top_k = top_k

    def forward(self, hidden, router_w, experts: HostExperts, out, topk_idx=None, topk_w=None,
                stream: int = 0):
        """Device tensors (torch) in, device tensors out; enqueued on `stream` (raw handle)."""
        moe_layer_forward(self.ctx, hidden.data_ptr() if hidden.numel() else 0, hidden.shape[0],
                          router_w.data_ptr(),
                          experts.array, self.top_k, out.data_ptr() if out.numel() else 0,
                          topk_idx.data_ptr() if topk_idx is not None else 0,
                          topk_w.data_ptr() if topk_w is not None else 0, stream)

    def forward_host(self, hidden_host, router_w, experts: HostExperts, out_host, topk_idx=None,
                     topk_w=None, stream: int = 0):
        moe_layer_forward_host(self.ctx, hidden_host.data_ptr(), hidden_host.shape[0],
                               router_w.data_ptr(), experts.array, self.top_k,
                               out_host.data_ptr(),
                               topk_idx.data_ptr() if topk_idx is not None else 0,
                               topk_w.data_ptr() if topk_w is not None else 0, stream)

    def taskb_forward(self, attn, resid, layer: HostLayer, eps: float, router_w,
                      experts: HostExperts, out, topk_idx=None, topk_w=None, stream: int = 0):
        """GPU Task B: out = h1 + MoE(RMSNorm(h1)), h1 = resid + attn Wo^T (device tensors)."""
        T = attn.shape[0]
        moe_taskb_forward(self.ctx, attn.data_ptr() if T else 0, resid.data_ptr() if T else 0, T,
                          layer.ptr, eps, router_w.data_ptr(), experts.array, self.top_k,
                          out.data_ptr() if T else 0,
                          topk_idx.data_ptr() if topk_idx is not None else 0,
                          topk_w.data_ptr() if topk_w is not None else 0, stream)

    def taskb_forward_host(self, attn_host, resid, layer: HostLayer, eps: float, router_w,
                           experts: HostExperts, out_host, topk_idx=None, topk_w=None,
                           stream: int = 0):
        """GPU Task B with the attention output and the result in pinned host tensors."""
        T = attn_host.shape[0]
        moe_taskb_forward_host(self.ctx, attn_host.data_ptr() if T else 0,
                               resid.data_ptr() if T else 0, T, layer.ptr, eps,
                               router_w.data_ptr(), experts.array, self.top_k,
                               out_host.data_ptr() if T else 0,
                               topk_idx.data_ptr() if topk_idx is not None else 0,
                               topk_w.data_ptr() if topk_w is not None else 0, stream)

    def taskb_forward2_host(self, attn_host, resid, layer: HostLayer, eps: float, router_w,
                            experts: HostExperts, out_host, topk_idx=None, topk_w=None,
                            stream: int = 0):
        """GPU Task B over two partitions (sequences of 2 pinned host attention outputs, 2 device
        residuals, 2 pinned host outputs) with the layer's weights streamed once."""
        moe_taskb_forward2_host(
            self.ctx, [a.data_ptr() if a.shape[0] else 0 for a in attn_host],
            [r.data_ptr() if r.shape[0] else 0 for r in resid], [a.shape[0] for a in attn_host],
            layer.ptr, eps, router_w.data_ptr(), experts.array, self.top_k,
            [o.data_ptr() if o.shape[0] else 0 for o in out_host],
            topk_idx.data_ptr() if topk_idx is not None else 0,
            topk_w.data_ptr() if topk_w is not None else 0, stream)

    def group_size(self) -> int:
        """Ranks of the expert-parallel group as the transport sees them (NCCL: ncclCommCount)."""
        n = ctypes.c_int32()
        _check(load().moe_ep_group_size(self.ctx, ctypes.byref(n)), self.ctx)
        return n.value

    def wait_output(self, stream: int = 0):
        """Make `stream` wait for the result copies of the host-buffer calls issued so far."""
        moe_wait_output(self.ctx, stream)

    def ipc_handle(self) -> bytes:
        return moe_ep_ipc_handle(self.ctx)

    def ipc_connect(self, handles: Sequence[bytes]) -> None:
        moe_ep_ipc_connect(self.ctx, handles)

    def ipc_selftest(self, timeout_s: float = 5.0) -> None:
        """Collective: raises MoEError if the peer mapping does not work (see include/moe.h)."""
        _check(load().moe_ep_ipc_selftest(self.ctx, timeout_s), self.ctx)

    def sync(self):
        moe_sync(self.ctx)

    def stats(self) -> dict:
        return moe_get_stats(self.ctx)

    def reset_stats(self):
        moe_reset_stats(self.ctx)

    def debug(self) -> moe_debug_view:
        return moe_debug_buffers(self.ctx)

    def close(self):
        if self.ctx:
            moe_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
