// moe_api.cu -- C ABI (include/moe.h) and the weight-streaming engine.
//
// Streaming engine ("weights for the next execution stage are prefetched at the
// beginning of each stage by the Contiguous Data Mover ... runs asynchronously ... synchronizes
// only at the stage boundaries"; PAPER.md:823-826 pinned host weights and a GPU weight buffer of
// two units; PAPER.md:829-835 packetised transfers):
//   * N device staging slots (N = num_slots, auto ~512 MiB), each one packed expert (W13 | W2);
//   * a dedicated copy stream; the copy of streamed item q into slot q%N waits on `slot_free[q%N]`
//     (recorded after the GEMMs of item q-N) and records `ready13` / `ready2`, so the H2D of the
//     next experts overlaps the GEMMs of expert e; consecutive small experts move in one DMA;
//   * host enqueue order interleaves "GEMMs of item i" with "copy of item i+N", and a call's first
//     N copies are enqueued before its routing kernels, so the copy engine runs back-to-back
//     across experts AND across calls (cross-call prefetch of the next layer's first experts).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>

#include "engine.h"

using moe::GemmGroup;
using moe::Prof;

namespace moe {

namespace {
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
        cudaGetLastError();
    });
    return fn;
}
}  // namespace

// bf16 [rows, cols] row-major, box = box_cols columns (box_cols * 2 bytes = the swizzle span:
// 128 or 64) x box_rows rows; rows past `rows` read as zeros.
bool make_tmap_box(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                   uint32_t box_rows) {
    PFN_encodeTiled_t enc = get_encode_fn();
    if (!enc || rows == 0 || (box_cols != 64 && box_cols != 32)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// box = 64 columns (128 B, one swizzle atom) x box_rows rows.
bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    return make_tmap_box(m, base, rows, cols, 64, box_rows);
}

moe_status set_err(moe_ctx c, moe_status s, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->last_error = buf;
    }
    return s;
}

cudaEvent_t pool_get(moe_ctx c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

}  // namespace moe

namespace {

using moe::set_err;

// MOE_FLAG_SHARD_SHARED: rank r's columns of the concatenated shared FFN (include/moe.h,
// moe_shared_slice): blocks [floor(r B / W), floor((r+1) B / W)) of B = S h_i / 128.
void shared_slice_cols(int ffn, int S, int W, int r, int* col0, int* width) {
    const int64_t B = (int64_t)S * ffn / 128;
    const int64_t b0 = B * r / W, b1 = B * (r + 1) / W;
    *col0 = (int)(b0 * 128);
    *width = (int)((b1 - b0) * 128);
}

moe_status check_cfg(const moe_config* cfg) {
    if (!cfg) return MOE_E_INVAL;
    if (cfg->hidden <= 0 || cfg->ffn <= 0 || cfg->num_experts <= 0 || cfg->top_k <= 0 ||
        cfg->top_k > cfg->num_experts || cfg->num_shared < 0 || cfg->max_tokens <= 0 ||
        cfg->world_size <= 0 || cfg->rank < 0 || cfg->rank >= cfg->world_size ||
        cfg->packet_bytes < 0)
        return MOE_E_INVAL;
    if (cfg->hidden % 128 || cfg->ffn % 128 || cfg->num_experts > moe::kMaxExperts ||
        cfg->top_k > moe::kMaxTopK || cfg->num_shared > moe::kMaxShared)
        return MOE_E_UNSUPPORTED;
    if (cfg->num_experts % cfg->world_size) return MOE_E_UNSUPPORTED;
    if (cfg->world_size > 1 && !cfg->nccl_unique_id && !(cfg->flags & MOE_FLAG_IPC_EP))
        return MOE_E_INVAL;
    if (cfg->num_slots < 0 || cfg->num_slots == 1 || cfg->num_slots > moe::kMaxSlots)
        return MOE_E_INVAL;
    int s_items = cfg->num_shared;
    if (cfg->flags & MOE_FLAG_SHARD_SHARED) {
        // P2P transport only (the gather / partial sums ride the peer-memory permute / combine);
        // a slice must fit one expert slot (S <= W: at most ceil(S h_i / 128 / W) <= h_i / 128
        // blocks)
        if (cfg->world_size < 2 || !(cfg->flags & (MOE_FLAG_LOCAL_EP | MOE_FLAG_IPC_EP)) ||
            cfg->num_shared < 1 || cfg->num_shared > cfg->world_size)
            return MOE_E_UNSUPPORTED;
        int c0 = 0, w = 0;
        shared_slice_cols(cfg->ffn, cfg->num_shared, cfg->world_size, cfg->rank, &c0, &w);
        s_items = w > 0 ? 1 : 0;
    }
    if (cfg->num_slots > 2 && cfg->num_slots >= cfg->num_experts / cfg->world_size + s_items)
        return MOE_E_INVAL;  // more slots than streamed experts would let weights stay resident
    const int64_t rows = (int64_t)cfg->max_tokens * cfg->world_size * cfg->top_k +
                         (int64_t)cfg->max_tokens * std::max(cfg->num_shared, cfg->world_size);
    if (rows >= (1ll << 31)) return MOE_E_UNSUPPORTED;
    return MOE_OK;
}

typedef CUresult (*PFN_pointerGetAttribute_t)(void*, CUpointer_attribute, CUdeviceptr);

// Start address of the CUDA allocation containing p (0 if unknown).  A DMA may only be merged
// across blobs of the SAME pinned allocation: separately allocated blobs can be adjacent in the
// address space, and one cudaMemcpyAsync must not span two allocations.
uintptr_t alloc_start(const void* p) {
    static PFN_pointerGetAttribute_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &f, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_pointerGetAttribute_t>(f);
        cudaGetLastError();
    });
    CUdeviceptr start = 0;
    if (!fn || fn(&start, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, (CUdeviceptr)(uintptr_t)p) !=
                   CUDA_SUCCESS)
        return 0;
    return (uintptr_t)start;
}

// Page-locked host memory?  Checked on every call, not cached: a caller may free a blob and get
// new (possibly pageable) memory at the same address.
bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

bool is_device(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    const char* x = static_cast<const char*>(a);
    const char* y = static_cast<const char*>(b);
    return x < y + nb && y < x + na;
}

// Issue the pending batch of streamed items [pend_q0, pend_q0 + pend_n): their slots are
// adjacent (no wrap) and their host blobs contiguous, so one DMA moves them all.
moe_status flush_copies(moe_ctx c) {
    if (c->pend_n == 0) return MOE_OK;
    const int n = c->pend_n;
    const int s0 = (int)(c->pend_q0 % (uint64_t)c->nslots);
    const int64_t ib = c->pend_item, i13 = c->pend_w13;   // bytes per item / its W13 part
    if (c->mover) {   // the mover thread packetises and orders it by device counters
        for (int j = 0; j < n; ++j) {
            c->batch_q0[s0 + j] = c->pend_q0;
            c->batch_n[s0 + j] = n;
        }
        c->stats.h2d_weight_bytes += (int64_t)n * ib;
        c->pend_n = 0;
        return moe::mover_push(c, c->pend_q0, n, c->pend_src, static_cast<char*>(c->slot[s0]), ib,
                               i13);
    }
    for (int j = 0; j < n; ++j)  // each slot must have been released by its previous item's GEMMs
        MOE_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->slot_free[s0 + j], 0));
    const char* src = c->pend_src;
    char* dst = static_cast<char*>(c->slot[s0]);
    const int64_t pk = c->cfg.packet_bytes > 0 ? c->cfg.packet_bytes : INT64_MAX;
    Prof p(c, moe::kRecH2D, c->copy_stream);
    auto copy_range = [&](int64_t lo, int64_t hi) -> moe_status {
        for (int64_t o = lo; o < hi;) {
            const int64_t m = std::min(pk, hi - o);
            MOE_CUDA(c, cudaMemcpyAsync(dst + o, src + o, (size_t)m, cudaMemcpyHostToDevice,
                                        c->copy_stream));
            o += m;
        }
        return MOE_OK;
    };
    if (c->cfg.packet_bytes == 0) {
        // One DMA for the whole batch: every copy/event boundary on the copy stream costs a few
        // microseconds of idle link (measured: separate W13/W2 copies lost ~0.4% of the C1 step,
        // 17 MB per-expert copies ran at 54.0 of 55.6 GB/s).  GEMM1 then starts after the
        // batch landed -- still long before the next batch's copy ends.
        moe_status st = copy_range(0, (int64_t)n * ib);
        if (st != MOE_OK) return st;
        for (int j = 0; j < n; ++j) {
            MOE_CUDA(c, cudaEventRecord(c->ready13[s0 + j], c->copy_stream));
            MOE_CUDA(c, cudaEventRecord(c->ready2[s0 + j], c->copy_stream));
        }
    } else {  // packetised: W13 first so GEMM1 can start early
        for (int j = 0; j < n; ++j) {
            const int64_t b = (int64_t)j * ib;
            moe_status st = copy_range(b, b + i13);
            if (st != MOE_OK) return st;
            MOE_CUDA(c, cudaEventRecord(c->ready13[s0 + j], c->copy_stream));
            st = copy_range(b + i13, b + ib);
            if (st != MOE_OK) return st;
            MOE_CUDA(c, cudaEventRecord(c->ready2[s0 + j], c->copy_stream));
        }
    }
    p.end();
    for (int j = 0; j < n; ++j) {   // the GEMMs take the batch as one launch (forward_impl)
        c->batch_q0[s0 + j] = c->pend_q0;
        c->batch_n[s0 + j] = n;
    }
    c->stats.h2d_weight_bytes += (int64_t)n * ib;
    c->pend_n = 0;
    return MOE_OK;
}

// Request the copy of streamed item q (blob experts[i]) into slot q % nslots.  Requests
// are batched (see flush_copies); a batch is flushed when full, when the next item is not
// contiguous (host blob or slot), and at the end of each call.  Items are requested nslots ahead
// of their GEMMs and copy_group <= nslots, so an item's batch is always flushed before the
// compute stream waits on it.
moe_status request_copy(moe_ctx c, const void* const* experts, int i, uint64_t q) {
    const char* src = static_cast<const char*>(experts[i]);
    const int s = (int)(q % (uint64_t)c->nslots);
    // the shared slice (MOE_FLAG_SHARD_SHARED) is smaller than an expert: a batch of its own
    const bool slice = c->shard && i >= c->n_local;
    const int64_t ib = slice ? c->slice_bytes : c->blob_bytes;
    if (c->pend_n > 0) {
        const uintptr_t a0 = c->pend_base, a1 = c->call_base[i];
        const bool contiguous = !slice && c->pend_item == ib &&
                                src == c->pend_src + (int64_t)c->pend_n * c->blob_bytes &&
                                q == c->pend_q0 + (uint64_t)c->pend_n && s != 0 && a0 != 0 &&
                                a0 == a1;
        if (!contiguous || c->pend_n >= c->copy_group) {
            moe_status st = flush_copies(c);
            if (st != MOE_OK) return st;
        }
    }
    if (c->pend_n == 0) {
        c->pend_q0 = q;
        c->pend_src = src;
        c->pend_base = c->call_base[i];
        c->pend_item = ib;
        c->pend_w13 = slice ? 4ll * c->cfg.hidden * c->shard_w : c->w13_bytes;
    }
    ++c->pend_n;
    if (c->pend_n >= c->copy_group || slice) return flush_copies(c);
    return MOE_OK;
}

// Tile shape of one GEMM launch: the CTA-pair kernel (256x256 tiles on SM pairs, ~97% tensor-pipe
// activity) or the single-CTA kernel (128 x bn tiles, ~76%: shared-memory bandwidth bound, but
// half the M granularity and twice the concurrent tiles), by a wave model on the EXPECTED tiles
// of the launch's n groups: time ~ ceil(tiles / concurrent tiles) x tile width / efficiency.
// rows[i]: a group's expected rows; `routed`: the counts are a routing outcome (mean rows[i],
// spread ~ sqrt), so a group's last M tile is on average half full -- expected tiles = rows/BM
// + 1/2 -- else (shared experts, the O-projection: exactly rows[i]) tiles = ceil(rows/BM).
// (Round 1 used rows + 10% instead, which at C1 predicted 3 waves of CTA-pair tiles for GEMM2
// of two 1024-row experts where the actual routing gives 2, and so chose the slower kernel.)
bool pick_pair(moe_ctx c, const int64_t* rows, int n, int bn, int N, bool routed) {
    if (bn != 256 || N % 256 || c->pair_mode == 0) return false;
    if (c->pair_mode == 1) return true;
    const int sms = c->num_sms;
    double t1 = 0, t2 = 0;
    for (int i = 0; i < n; ++i) {
        if (rows[i] <= 0) continue;
        t1 += (routed ? rows[i] / 128.0 + 0.5 : (double)((rows[i] + 127) / 128)) * (N / bn);
        t2 += (routed ? rows[i] / 256.0 + 0.5 : (double)((rows[i] + 255) / 256)) * (N / 256);
    }
    if (t1 == 0) return false;
    const double w1 = std::ceil(t1 / sms - 1e-9) / 0.76;
    const double w2 = std::ceil(t2 / (sms / 2) - 1e-9) / 0.97;
    return w2 < w1;
}

// One expert-GEMM launch over a batch of groups on `st` (pair: tmB_pair, else tmB).
moe_status launch_grouped(moe_ctx c, int mode, int bn, const int64_t* rows, bool routed,
                          const CUtensorMap* tmA, const CUtensorMap* tmB,
                          const CUtensorMap* tmB_pair, const moe::GemmBatch& batch, int N, int K,
                          __nv_bfloat16* out, int ldo, cudaStream_t st,
                          const __nv_bfloat16* resid = nullptr) {
    const bool pair = pick_pair(c, rows, batch.n, bn, N, routed);
    MOE_CUDA(c, moe::launch_expert_gemm(mode, bn, pair, tmA, pair ? tmB_pair : tmB, batch, N, K,
                                        out, ldo, resid, c->num_sms, st));
    return MOE_OK;
}

// Optional parts of a call (GPU Task B with two token partitions, moe_taskb_forward2_host):
//   pre_route   runs after the call's first weight copies are requested and before any routing
//               (the late partition's token copy + O-projection + norm go there, so its copy
//               queues behind this call's weight requests -- the head-of-line case the data
//               mover is for);
//   split_at    0 < split_at < T: the combine runs as rows [0, split_at) then [split_at, T), with
//               split_ev recorded between them (the first partition's result copy starts while
//               the second is still being combined).
struct FwdExtra {
    std::function<moe_status()> pre_route;
    int split_at = 0;
    cudaEvent_t split_ev = nullptr;
};

// resid (Task B): added to every output row in the combine (nullptr for the plain MoE layer).
moe_status forward_impl(moe_ctx c, const __nv_bfloat16* hidden, int T, const __nv_bfloat16* wr,
                        const void* const* experts, __nv_bfloat16* out, int32_t* topk_idx,
                        float* topk_w, cudaStream_t st, bool hidden_on_copy_stream, int xb,
                        const __nv_bfloat16* resid = nullptr, const FwdExtra* ex = nullptr) {
    const moe_config& cf = c->cfg;
    const int h = cf.hidden, hi = cf.ffn, ne = cf.num_experts, k = cf.top_k, S = cf.num_shared;
    const int n_tiles = (T + moe::kRouteTile - 1) / moe::kRouteTile;
    int32_t* idx = topk_idx ? topk_idx : c->idx_ws;
    float* gates = topk_w ? topk_w : c->gates_ws;
    const uint64_t q0 = c->seq;

    // Calls share the context's workspace (routing tables, x_perm, h_act, y_perm, the host-mode
    // token buffers) and, with the mover, one compute order of the slot counters: a call on
    // another stream than the previous one first waits for it (a no-op on the same stream).
    MOE_CUDA(c, cudaStreamWaitEvent(st, c->done_ev, 0));

    // A operand of the shared experts is the hidden batch itself (per-call tensor map).
    // (T == 0 only happens under EP: the rank serves other ranks' tokens; its shared-expert
    // groups are then empty and never touch the map.)
    CUtensorMap tm_x = c->tm_xperm;
    const int Si = c->s_items;   // shared items streamed (S, or this rank's slice: 0 / 1)
    if (S > 0 && !c->shard && T > 0 && !moe::make_tmap(&tm_x, hidden, (uint64_t)T, (uint64_t)h, 128))
        return set_err(c, MOE_E_CUDA, "cuTensorMapEncodeTiled failed for hidden");

    // Streaming order: shared experts first (their GEMMs need only the hidden batch, and they are
    // the longest GEMMs -- T rows each -- so they must not sit at the end of a call where they
    // would hold slots the next call's first copies wait on), then the routed experts.
    // expert_of(i) is the index into `experts` / the group tables of streamed item i.
    auto expert_of = [&](int i) { return i < Si ? c->n_local + i : i - Si; };
    // the first nslots weight copies go ahead of routing (cross-call prefetch)
    const int ns = c->nslots;
    for (int i = 0; i < std::min(ns, c->n_all); ++i) {
        moe_status s = request_copy(c, experts, expert_of(i), q0 + i);
        if (s != MOE_OK) return s;
    }
    if (hidden_on_copy_stream) MOE_CUDA(c, cudaStreamWaitEvent(st, c->x_ready[xb], 0));
    if (ex && ex->pre_route) {
        moe_status s = ex->pre_route();
        if (s != MOE_OK) return s;
    }

    // One GEMM1 + one GEMM2 launch per DMA batch (flush_copies): the batch's experts sit in
    // adjacent slots of the staging buffer and their tiles are scheduled together (GemmBatch),
    // so many small experts no longer pay one partial last wave each.  A batch never mixes
    // shared and routed experts (different A operands and outputs).  Items [i0, i1), group
    // tables g1 (GEMM1) / g2 (GEMM2) indexed by expert_of(i).
    // The host does not know the group sizes (they live on the device), so the tile shape is
    // chosen on the expected size: T*k*W/N_e rows per routed expert (+10% for routing
    // variance), T per shared expert.
    const int64_t exp_routed = (int64_t)T * k * cf.world_size / ne;
    // Experts per GEMM launch (routed items): consecutive experts whose expected rows are small
    // share one launch -- and so one set of waves -- until a launch has ~kGemmRowsTarget rows
    // (C1: 2 experts of ~1024 rows per launch, 4 staging slots).  Bounded by half the slots, so
    // the next group's copies never wait on this group's GEMMs.
    const int gemm_items =
        (int)std::max<int64_t>(1, std::min<int64_t>(c->gemm_group_max,
                                                    (c->gemm_rows_target + exp_routed - 1) /
                                                        std::max<int64_t>(1, exp_routed)));
    const CUtensorMap* tmA_routed = &c->tm_xperm;
    __nv_bfloat16* y_routed = c->y_perm;
    auto run_items = [&](int i0, int i1, const GemmGroup* g1, const GemmGroup* g2) -> moe_status {
    for (int i = i0; i < i1;) {
        const uint64_t q = q0 + i;
        const bool shared = expert_of(i) >= c->n_local;
        // the rank's shared-FFN slice (MOE_FLAG_SHARD_SHARED): every rank's tokens gathered in
        // x_recv from row cap_recv, shard_w columns, partial rows into y_recv (peers read them)
        const bool slice = shared && c->shard;
        const int left = (shared ? Si : c->n_all) - i;   // items of this class (shared / routed)
        // the launch takes item q's whole DMA batch, or gemm_items routed items if more
        int want = std::min(left, shared ? 1 : gemm_items);
        if (c->pend_n > 0 && c->pend_q0 < q + (uint64_t)want) {  // a batch still pending: issue it
            moe_status fs = flush_copies(c);
            if (fs != MOE_OK) return fs;
        }
        const int s = (int)(q % (uint64_t)ns);
        int nb = (int)(c->batch_q0[s] + (uint64_t)c->batch_n[s] - q);
        nb = std::max(1, std::min({std::max(nb, want), left, moe::kMaxBatch}));
        moe::GemmBatch b1{}, b2{};
        b1.table = g1;
        if (c->clk_acc) {
            b1.clk = c->clk_acc;
            b2.clk = c->clk_acc + 2;
        }
        b2.table = g2;
        b1.n = b2.n = nb;
        int64_t rows[moe::kMaxBatch];
        if (c->mover) {
            if (c->mover_trace)
                fprintf(stderr, "[api] GEMMs of items [%llu, %llu): wait r13 >= %llu\n",
                        (unsigned long long)q, (unsigned long long)(q + nb), (unsigned long long)(q + nb));
            moe_status ws = moe::mover_wait(c, st, 0, q + nb);
            if (ws != MOE_OK) return ws;
        }
        for (int j = 0; j < nb; ++j) {
            const int sj = (int)((q + j) % (uint64_t)ns), e = expert_of(i + j);
            if (!c->mover) MOE_CUDA(c, cudaStreamWaitEvent(st, c->ready13[sj], 0));
            b1.idx[j] = b2.idx[j] = e;
            b1.b_row[j] = 3 * hi * sj;           // W13 of slot sj in tm_w13*
            b2.b_row[j] = slice ? 0                        // tm_w2s*[sj] starts at the W2 part
                                : 3 * h * sj + 2 * h;    // W2 of slot sj in tm_w2*
            rows[j] = slice ? (int64_t)T * cf.world_size : shared ? (int64_t)T : exp_routed;
        }
        {
            Prof p(c, moe::kRecGemm1, st);
            moe_status gs = launch_grouped(c, moe::kGemmSwiGLU, c->bn1, rows, !shared,
                                           slice ? &c->tm_xrecv : shared ? &tm_x : tmA_routed,
                                           &c->tm_w13, &c->tm_w13_pair, b1,
                                           2 * (slice ? c->shard_w : hi), h, c->h_act, hi, st);
            if (gs != MOE_OK) return gs;
            p.end();
        }
        if (c->mover) {
            moe_status ws = moe::mover_wait(c, st, 1, q + nb);
            if (ws != MOE_OK) return ws;
        } else {
            for (int j = 0; j < nb; ++j)
                MOE_CUDA(c, cudaStreamWaitEvent(st, c->ready2[(q + j) % (uint64_t)ns], 0));
        }
        {
            Prof p(c, moe::kRecGemm2, st);
            moe_status gs = launch_grouped(c, moe::kGemmPlain, c->bn2, rows, !shared, &c->tm_h,
                                           slice ? &c->tm_w2s[q % (uint64_t)ns] : &c->tm_w2,
                                           slice ? &c->tm_w2s_pair[q % (uint64_t)ns] : &c->tm_w2_pair,
                                           b2, h,
                                           slice ? c->shard_w : hi,
                                           slice ? c->y_recv : shared ? c->y_perm : y_routed, h,
                                           st);
            if (gs != MOE_OK) return gs;
            p.end();
        }
        c->stats.kernel_launches += 2;
        c->stats.gemm1_launches += 1;
        c->stats.gemm2_launches += 1;
        if (c->mover) {
            moe_status ms = moe::mover_mark_free(c, st, q + nb);
            if (ms != MOE_OK) return ms;
        } else {
            for (int j = 0; j < nb; ++j)
                MOE_CUDA(c, cudaEventRecord(c->slot_free[(q + j) % (uint64_t)ns], st));
        }
        for (int j = 0; j < nb; ++j) {   // the freed slots take the items ns ahead
            if (i + j + ns < c->n_all) {
                moe_status s2 = request_copy(c, experts, expert_of(i + j + ns), q + j + ns);
                if (s2 != MOE_OK) return s2;
            }
        }
        i += nb;
    }
    return MOE_OK;
    };

    // Shared experts first, BEFORE routing: they need only the hidden batch, so their GEMMs run
    // while the router works and their slots are free for the next copies early (the copy
    // engine never waits on the router).  Their group tables are written here (not by scan).
    if (Si > 0 && !c->shard) {
        const int hbase = (int)(c->ep ? c->cap_recv : (int64_t)T * k);
        MOE_CUDA(c, moe::launch_fill_shared_groups(c->shared_grp, c->n_local, c->n_all, S, T,
                                                   hbase, T * k, st));
        c->stats.kernel_launches += 1;
        const moe_status ss = run_items(0, Si, c->shared_grp, c->shared_grp + c->n_all);
        if (ss != MOE_OK) return ss;
    }

    {
        Prof p(c, moe::kRecRoute, st);
        int nl = 0;
        MOE_CUDA(c, moe::launch_router_topk(hidden, T, h, wr, ne, k, cf.renormalize, idx, gates,
                                            c->tile_counts, c->wr64, &nl, st));
        MOE_CUDA(c, moe::launch_scan(c->tile_counts, n_tiles, ne, T, k, S, c->tile_prefix,
                                     c->offsets, c->counts, c->grp1, c->grp2, st));
        p.end();
        c->stats.kernel_launches += nl + 1;
    }
    if (c->p2p) {   // P2P EP: counts exchange + plan before the permute writes into the owners
        Prof p(c, moe::kRecComm, st);
        moe_status s = moe::p2p_before_dispatch(c, T, st);
        if (s != MOE_OK) return s;
        p.end();
    }
    {
        Prof p(c, moe::kRecPermute, st);
        MOE_CUDA(c, moe::launch_permute(hidden, T, h, k, ne, idx, c->tile_prefix, c->offsets,
                                        c->x_perm, c->pos, c->p2p ? c->pr_x : nullptr, st));
        p.end();
        c->stats.kernel_launches += 1;
    }

    // Expert parallelism: ship each token row to the rank owning its expert.
    const GemmGroup* g1 = c->grp1;
    const GemmGroup* g2 = c->grp2;
    if (c->ep) {
        Prof p(c, moe::kRecComm, st);
        moe_status s = c->p2p ? moe::p2p_after_dispatch(c, st) : moe::ep_dispatch(c, T, st);
        if (s != MOE_OK) return s;
        p.end();
        tmA_routed = &c->tm_xrecv;
        g1 = c->ep_grp;
        g2 = c->ep_grp + c->n_all;
        y_routed = c->y_recv;
    }
    if (c->shard && Si > 0) {   // the shared slice, once every rank's tokens have arrived
        const moe_status ss = run_items(0, Si, g1, g2);
        if (ss != MOE_OK) return ss;
    }

    const moe_status rs = run_items(Si, c->n_all, g1, g2);   // the routed experts
    if (rs != MOE_OK) return rs;
    {
        moe_status fs = flush_copies(c);  // nothing may stay pending across calls
        if (fs != MOE_OK) return fs;
    }
    if (c->ep) {
        Prof p(c, moe::kRecComm, st);
        moe_status s = c->p2p ? moe::p2p_after_gemms(c, st) : moe::ep_combine(c, st);
        if (s != MOE_OK) return s;
        p.end();
    }
    {
        Prof p(c, moe::kRecCombine, st);
        // rows [r0, r1) of the call's tokens (two launches when the call is split, FwdExtra)
        auto combine = [&](int r0, int r1) -> moe_status {
            MOE_CUDA(c, moe::launch_combine(c->y_perm, c->pos + (int64_t)r0 * k, gates + (int64_t)r0 * k,
                                            r1 - r0, h, k, S, (int64_t)T * k + r0, T,
                                            resid ? resid + (int64_t)r0 * h : nullptr,
                                            out + (int64_t)r0 * h, idx + (int64_t)r0 * k, c->offsets,
                                            c->p2p ? c->pr_y : nullptr, c->shard ? r0 : -1, st));
            c->stats.kernel_launches += 1;
            return MOE_OK;
        };
        const int split = (ex && ex->split_at > 0 && ex->split_at < T) ? ex->split_at : 0;
        if (split) {
            moe_status cs = combine(0, split);
            if (cs != MOE_OK) return cs;
            if (ex->split_ev) MOE_CUDA(c, cudaEventRecord(ex->split_ev, st));
            cs = combine(split, T);
            if (cs != MOE_OK) return cs;
        } else if (T > 0) {
            moe_status cs = combine(0, T);
            if (cs != MOE_OK) return cs;
        }
        p.end();
    }
    if (c->p2p) {
        moe_status s = moe::p2p_after_combine(c, st);
        if (s != MOE_OK) return s;
    }
    c->seq = q0 + c->n_all;
    c->last_rows = (int64_t)T * (k + S);
    c->stats.calls += 1;
    MOE_CUDA(c, cudaEventRecord(c->done_ev, st));
    return MOE_OK;
}

moe_status validate_call(moe_ctx c, int32_t T, const void* router_w, const void* const* experts,
                         int32_t top_k) {
    if (!c) return MOE_E_INVAL;
    if (c->sticky != MOE_OK) return set_err(c, MOE_E_STATE, "context is in an error state");
    if (c->p2p_diag_h && (c->p2p_diag_h[0] || c->p2p_diag_h[5])) {   // an earlier call failed
        moe_sync(c);
        return c->sticky != MOE_OK ? c->sticky : MOE_E_STATE;
    }
    if (T < 0 || T > c->cfg.max_tokens)
        return set_err(c, MOE_E_INVAL, "num_tokens %d outside [0, %d]", T, c->cfg.max_tokens);
    if (top_k != c->cfg.top_k)
        return set_err(c, MOE_E_INVAL, "top_k %d != configured %d", top_k, c->cfg.top_k);
    if (T == 0 && !c->ep) return MOE_OK;
    if (!router_w || !experts) return set_err(c, MOE_E_INVAL, "NULL router_w / experts");
    if (!is_device(router_w)) return set_err(c, MOE_E_INVAL, "router_w is not device memory");
    if ((uintptr_t)router_w & 15)   // the router reads it with 16-byte vector loads
        return set_err(c, MOE_E_INVAL, "router_w must be 16-byte aligned");
    c->call_base.assign(c->n_all, 0);
    for (int i = 0; i < c->n_all; ++i) {
        if (!experts[i]) return set_err(c, MOE_E_INVAL, "experts[%d] is NULL", i);
        if (!is_pinned(experts[i]))
            return set_err(c, MOE_E_NOT_PINNED, "experts[%d] is not page-locked host memory", i);
        // start of the blob's allocation, looked up per call: one DMA may only span blobs of
        // the same allocation (request_copy)
        c->call_base[i] = alloc_start(experts[i]);
    }
    return MOE_OK;
}

// Host-buffer entry points.  Two device token buffers x_dev / out_dev alternate between calls
// (parity b = host_buffer()); allocated on first use.
moe_status host_buffer(moe_ctx c, int* b_out) {
    if (!c->x_dev[0]) {
        const size_t cap = (size_t)c->cfg.max_tokens * c->cfg.hidden * 2;
        for (int i = 0; i < 2; ++i) {
            if (cudaMalloc(&c->x_dev[i], cap) != cudaSuccess || cudaMalloc(&c->out_dev[i], cap) != cudaSuccess) {
                cudaGetLastError();
                return set_err(c, MOE_E_NOMEM, "host-mode buffers");
            }
        }
    }
    *b_out = c->host_parity;
    c->host_parity ^= 1;
    return MOE_OK;
}

// Copy `bytes` of pinned host tokens into x_dev[b] at byte offset `off` on the weight stream, in
// enqueue order with the weight copies (see engine.h token_lane), and record `ready` there.
// part: 0 / 1 -- the partition whose enqueue -> resident latency the stats attribute it to.
moe_status stage_tokens(moe_ctx c, int b, const void* host, size_t bytes, size_t off,
                        cudaEvent_t ready, int part) {
    cudaStream_t ts = c->token_lane ? c->token_stream : c->copy_stream;
    cudaEvent_t t0 = nullptr;
    const bool prof = (c->cfg.flags & MOE_FLAG_PROFILE) != 0;
    if (prof) {  // enqueue-time stamp: the clock stream is always idle
        t0 = moe::pool_get(c);
        MOE_CUDA(c, cudaEventRecord(t0, c->clock_stream));
    }
    MOE_CUDA(c, cudaStreamWaitEvent(ts, c->xbuf_free[b], 0));
    Prof pc(c, moe::kRecH2DTok, ts);   // the copy's own duration
    MOE_CUDA(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->x_dev[b]) + off, host, bytes,
                                cudaMemcpyHostToDevice, ts));
    pc.end();
    MOE_CUDA(c, cudaEventRecord(ready, ts));
    if (prof) {
        cudaEvent_t t1 = moe::pool_get(c);
        MOE_CUDA(c, cudaEventRecord(t1, ts));
        c->pending.push_back(moe::Rec{part ? moe::kRecTokenB : moe::kRecTokenA, t0, t1});
    }
    c->stats.h2d_token_bytes += (int64_t)bytes;
    c->stats.host_calls += part == 0 ? 1 : 0;
    c->stats.part_copies[part] += 1;
    return MOE_OK;
}

// Result copies of a host-buffer call into pinned host memory, on the context's D2H stream: part
// p (rows [row0[p], row0[p] + rows[p]) of out_dev[b]) starts once ev[p] -- recorded on the caller's
// stream after that part's combine -- has passed, so the copy overlaps whatever the caller's
// stream runs next (the next call's shared-expert GEMMs and routing; the second partition's
// combine).  d2h_done[b] guards out_dev[b] against the call that reuses it; out_ev is the
// completion moe_wait_output / moe_sync wait on.
moe_status copy_results(moe_ctx c, int b, int np, void* const* host, const int* row0,
                        const int* rows, const cudaEvent_t* ev) {
    const size_t rb = (size_t)c->cfg.hidden * 2;
    for (int p = 0; p < np; ++p) {
        if (rows[p] <= 0) continue;
        MOE_CUDA(c, cudaStreamWaitEvent(c->d2h_stream, ev[p], 0));
        MOE_CUDA(c, cudaMemcpyAsync(host[p], reinterpret_cast<char*>(c->out_dev[b]) + row0[p] * rb,
                                    rows[p] * rb, cudaMemcpyDeviceToHost, c->d2h_stream));
        c->stats.d2h_token_bytes += (int64_t)rows[p] * (int64_t)rb;
    }
    MOE_CUDA(c, cudaEventRecord(c->d2h_done[b], c->d2h_stream));
    MOE_CUDA(c, cudaEventRecord(c->out_ev, c->d2h_stream));
    return MOE_OK;
}

// Task B resources, allocated on the first moe_taskb_forward.  All or nothing: on any failure
// everything allocated here is released again, so the next call retries from scratch
// (taskb_ready is set only once the tensor maps are encoded).
void taskb_release(moe_ctx c) {
    for (int i = 0; i < 2; ++i) {
        cudaFree(c->lw_slot[i]);
        c->lw_slot[i] = nullptr;
        if (c->lw_ready[i]) cudaEventDestroy(c->lw_ready[i]);
        if (c->lw_free[i]) cudaEventDestroy(c->lw_free[i]);
        c->lw_ready[i] = c->lw_free[i] = nullptr;
    }
    cudaFree(c->h1_ws);
    cudaFree(c->u_ws);
    cudaFree(c->oproj_grp);
    c->h1_ws = c->u_ws = nullptr;
    c->oproj_grp = nullptr;
    c->taskb_ready = false;
    cudaGetLastError();
}

moe_status taskb_resources(moe_ctx c) {
    if (c->taskb_ready) return MOE_OK;
    const int h = c->cfg.hidden;
    const size_t act = (size_t)c->cfg.max_tokens * h * 2;
    c->layer_bytes = moe_packed_layer_bytes(h);
    bool ok = true;
    for (int i = 0; i < 2; ++i) {
        ok &= cudaMalloc((void**)&c->lw_slot[i], (size_t)c->layer_bytes) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->lw_ready[i], cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->lw_free[i], cudaEventDisableTiming) == cudaSuccess;
    }
    ok &= cudaMalloc((void**)&c->h1_ws, act) == cudaSuccess;
    ok &= cudaMalloc((void**)&c->u_ws, act) == cudaSuccess;
    ok &= cudaMalloc((void**)&c->oproj_grp, 2 * sizeof(GemmGroup)) == cudaSuccess;   // 2 partitions
    if (!ok) {
        taskb_release(c);
        return set_err(c, MOE_E_NOMEM, "Task B buffers (2 x %lld B layer slots + 2 x %zu B)",
                       (long long)c->layer_bytes, act);
    }
    bool tm = true;
    for (int i = 0; i < 2; ++i) {  // Wo [h, h]: N = h output rows, K = h
        tm &= moe::make_tmap(&c->tm_wo[i], c->lw_slot[i], (uint64_t)h, (uint64_t)h, (uint32_t)c->bn2);
        tm &= moe::make_tmap(&c->tm_wo_pair[i], c->lw_slot[i], (uint64_t)h, (uint64_t)h, 128);
    }
    if (!tm) {
        taskb_release(c);
        return set_err(c, MOE_E_CUDA, "cuTensorMapEncodeTiled failed for Wo");
    }
    c->taskb_ready = true;
    return MOE_OK;
}

// One token partition of a Task B call: its attention output (rows [base, base + T) of the
// A operand `tm_attn` maps), its residual rows, and the event that marks its attention output
// resident (nullptr: already on the device, in stream order).
struct TbPart {
    const __nv_bfloat16* resid;
    int T, base;
    cudaEvent_t ready;
};

// b1 O-projection + residual and b2 RMSNorm of one partition (rows [base, base + T) of h1 / u).
moe_status taskb_front(moe_ctx c, const CUtensorMap& tm_attn, const TbPart& pt, int lb, float eps,
                       cudaStream_t st) {
    const int h = c->cfg.hidden;
    if (pt.T == 0) return MOE_OK;
    const int gi = pt.base == 0 ? 0 : 1;   // oproj_grp entry of this partition
    MOE_CUDA(c, moe::launch_fill_group(c->oproj_grp + gi, pt.base, pt.base + pt.T, 0, st));
    if (pt.ready) MOE_CUDA(c, cudaStreamWaitEvent(st, pt.ready, 0));
    MOE_CUDA(c, cudaStreamWaitEvent(st, c->lw_ready[lb], 0));
    __nv_bfloat16* h1 = c->h1_ws + (int64_t)pt.base * h;
    {
        Prof p(c, moe::kRecOproj, st);
        moe::GemmBatch ob{};
        ob.table = c->oproj_grp + gi;
        ob.n = 1;   // idx[0] = 0, b_row[0] = 0: Wo is the whole map
        const int64_t rows = pt.T;
        moe_status gs = launch_grouped(c, moe::kGemmResidual, c->bn2, &rows, false, &tm_attn,
                                       &c->tm_wo[lb], &c->tm_wo_pair[lb], ob, h, h, h1, h, st,
                                       pt.resid);
        if (gs != MOE_OK) return gs;
        p.end();
    }
    {
        Prof p(c, moe::kRecNorm, st);
        const __nv_bfloat16* gamma =
            reinterpret_cast<const __nv_bfloat16*>(c->lw_slot[lb] + 2ll * h * h);
        MOE_CUDA(c, moe::launch_rmsnorm(h1, gamma, pt.T, h, eps, c->u_ws + (int64_t)pt.base * h, st));
        p.end();
    }
    c->stats.kernel_launches += 3;
    return MOE_OK;
}

// GPU Task B over one or two token partitions (R19-R21): b1 O-projection
// + residual, b2 RMSNorm, then the MoE layer on u with h1 as the combine's residual.  The layer
// blob and the experts are streamed ONCE for all partitions.  Partition 0's front runs as soon as
// its attention output and Wo are resident; partition 1's (`late`, the two-partition host call)
// runs after the call's first expert copies are requested -- its token copy is issued there by
// late->stage -- and the combine is split so partition 0's result can leave first (VSLPipe's
// alpha / beta).
struct TbLate {
    TbPart part;
    std::function<moe_status()> stage;   // issues partition 1's token copy
};

moe_status taskb_impl(moe_ctx c, const __nv_bfloat16* attn, const TbPart& p0, const TbLate* late,
                      const void* layer, float eps, const __nv_bfloat16* wr,
                      const void* const* experts, __nv_bfloat16* out, int32_t* topk_idx,
                      float* topk_w, cudaStream_t st, cudaEvent_t split_ev = nullptr) {
    const int h = c->cfg.hidden;
    const int T = p0.T + (late ? late->part.T : 0);
    c->stats.taskb_calls += 1;
    // h1 / u are read by the previous call's combine: order after it (see forward_impl)
    MOE_CUDA(c, cudaStreamWaitEvent(st, c->done_ev, 0));
    if (T == 0) {  // EP only: no local tokens, this rank still serves its experts
        c->last_taskb_T = 0;
        return forward_impl(c, nullptr, 0, wr, experts, nullptr, topk_idx, topk_w, st, false, 0);
    }
    CUtensorMap tm_attn;
    if (!moe::make_tmap(&tm_attn, attn, (uint64_t)T, (uint64_t)h, 128))
        return set_err(c, MOE_E_CUDA, "cuTensorMapEncodeTiled failed for attn");
    // The layer weights ride the copy stream just ahead of this call's expert weights (nothing
    // is pending between calls: forward_impl flushes at its end).
    const int lb = (int)(c->lw_seq & 1);
    c->lw_seq += 1;
    MOE_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->lw_free[lb], 0));
    {
        Prof p(c, moe::kRecH2D, c->copy_stream);
        MOE_CUDA(c, cudaMemcpyAsync(c->lw_slot[lb], layer, (size_t)c->layer_bytes,
                                    cudaMemcpyHostToDevice, c->copy_stream));
        p.end();
    }
    MOE_CUDA(c, cudaEventRecord(c->lw_ready[lb], c->copy_stream));
    c->stats.h2d_weight_bytes += c->layer_bytes;

    moe_status s = taskb_front(c, tm_attn, p0, lb, eps, st);
    if (s != MOE_OK) return s;
    FwdExtra ex;
    if (late && late->part.T > 0) {
        ex.pre_route = [&]() -> moe_status {
            moe_status ls = late->stage();
            if (ls != MOE_OK) return ls;
            ls = taskb_front(c, tm_attn, late->part, lb, eps, st);
            if (ls != MOE_OK) return ls;
            MOE_CUDA(c, cudaEventRecord(c->lw_free[lb], st));
            return MOE_OK;
        };
        ex.split_at = p0.T;
        ex.split_ev = split_ev;
    } else {
        MOE_CUDA(c, cudaEventRecord(c->lw_free[lb], st));
    }
    c->last_taskb_T = T;
    return forward_impl(c, c->u_ws, T, wr, experts, out, topk_idx, topk_w, st, false, 0, c->h1_ws,
                        &ex);
}

}  // namespace

extern "C" {

int64_t moe_packed_expert_bytes(int32_t hidden, int32_t ffn) {
    if (hidden <= 0 || ffn <= 0) return 0;
    return 6ll * hidden * ffn;
}

moe_status moe_shared_slice(int32_t ffn, int32_t num_shared, int32_t world, int32_t rank,
                            int32_t* col0, int32_t* width) {
    if (!col0 || !width || ffn <= 0 || ffn % 128 || num_shared < 1 || world < 1 || rank < 0 ||
        rank >= world)
        return MOE_E_INVAL;
    int c0 = 0, w = 0;
    shared_slice_cols(ffn, num_shared, world, rank, &c0, &w);
    *col0 = c0;
    *width = w;
    return MOE_OK;
}

moe_status moe_pack_expert(int32_t hidden, int32_t ffn, const void* w1, const void* w3,
                           const void* w2, void* dst) {
    if (!w1 || !w3 || !w2 || !dst || hidden <= 0 || ffn <= 0) return MOE_E_INVAL;
    if (ffn % 128) return MOE_E_UNSUPPORTED;
    const size_t row = (size_t)hidden * 2;  // bytes per W1/W3 row
    const char* a = static_cast<const char*>(w1);
    const char* b = static_cast<const char*>(w3);
    char* d = static_cast<char*>(dst);
    // W13: 32-row blocks = [16 rows of W1 ; the same 16 rows of W3]
    for (int j = 0; j < ffn / 16; ++j) {
        memcpy(d + (size_t)(32 * j) * row, a + (size_t)(16 * j) * row, 16 * row);
        memcpy(d + (size_t)(32 * j + 16) * row, b + (size_t)(16 * j) * row, 16 * row);
    }
    memcpy(d + (size_t)2 * ffn * row, w2, (size_t)hidden * ffn * 2);
    return MOE_OK;
}

moe_status moe_host_alloc(size_t bytes, void** ptr) {
    if (!ptr || bytes == 0) return MOE_E_INVAL;
    *ptr = nullptr;
    if (cudaHostAlloc(ptr, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        *ptr = nullptr;
        return MOE_E_NOMEM;
    }
    return MOE_OK;
}

moe_status moe_host_free(void* ptr) {
    if (!ptr) return MOE_OK;
    return cudaFreeHost(ptr) == cudaSuccess ? MOE_OK : MOE_E_CUDA;
}

moe_status moe_init(const moe_config* cfg, moe_ctx* out) {
    if (!out) return MOE_E_INVAL;
    *out = nullptr;
    moe_status s = check_cfg(cfg);
    if (s != MOE_OK) return s;
    moe_ctx c = new moe_ctx_s();
    c->cfg = *cfg;
    auto fail = [&](moe_status st) {
        moe_destroy(c);
        return st;
    };
    if (cudaSetDevice(cfg->device) != cudaSuccess) {
        cudaGetLastError();
        return fail(MOE_E_CUDA);
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess) return fail(MOE_E_CUDA);
    if (prop.major != 10) return fail(MOE_E_UNSUPPORTED);  // sm_100a kernels only
    c->num_sms = prop.multiProcessorCount;
    const int h = cfg->hidden, hi = cfg->ffn, ne = cfg->num_experts, k = cfg->top_k;
    const int S = cfg->num_shared, Tm = cfg->max_tokens, W = cfg->world_size;
    if (const char* e = getenv("MOE_GEMM_ROWS")) c->gemm_rows_target = std::max(1, atoi(e));
    c->ep = W > 1 || (cfg->flags & (MOE_FLAG_FORCE_EP | MOE_FLAG_LOCAL_EP | MOE_FLAG_IPC_EP));
    c->local_ep = (cfg->flags & MOE_FLAG_LOCAL_EP) != 0;
    c->p2p = c->local_ep || (cfg->flags & MOE_FLAG_IPC_EP) != 0;
    if (W > moe::kMaxRanks && c->p2p) return fail(MOE_E_UNSUPPORTED);
    c->n_local = ne / W;
    c->shard = (cfg->flags & MOE_FLAG_SHARD_SHARED) != 0;   // check_cfg: P2P, W > 1, S <= W
    c->s_items = S;
    if (c->shard) {
        int c0 = 0;
        for (int r = 0; r < W; ++r) {
            int w = 0;
            shared_slice_cols(hi, S, W, r, &c0, &w);
            if (w > 0) c->shard_mask |= 1u << r;
            if (r == cfg->rank) c->shard_w = w;
        }
        c->s_items = c->shard_w > 0 ? 1 : 0;
        c->slice_bytes = c->shard_w > 0 ? moe_packed_expert_bytes(h, c->shard_w) : 0;
    }
    c->n_all = c->n_local + c->s_items;
    c->w13_bytes = 4ll * h * hi;
    c->blob_bytes = moe_packed_expert_bytes(h, hi);
    c->bn1 = moe::gemm_bn_for(moe::kGemmSwiGLU, 2 * hi);
    c->bn2 = moe::gemm_bn_for(moe::kGemmPlain, h);
    if (!c->bn1 || !c->bn2) return fail(MOE_E_UNSUPPORTED);
    if (cfg->num_slots > 0) {
        c->nslots = cfg->num_slots;
    } else {  // auto: ~512 MiB of staging, 2..32 slots, fewer than the experts streamed per call
        // (measured on DSV2-Lite-size experts: 8 slots 95.1%, 16 slots 98.9%, 24-32 slots with
        // 12-16-expert DMAs 99.4% of roofline); at least two GEMM groups' worth when small
        // expert groups share a launch (forward_impl gemm_items; C1: 4 slots)
        int64_t want = (moe::kAutoSlotBytes + c->blob_bytes - 1) / c->blob_bytes;
        const int64_t rows_max = std::max<int64_t>(1, (int64_t)Tm * k * W / ne);
        const int64_t g = std::min<int64_t>((c->gemm_rows_target + rows_max - 1) / rows_max,
                                            (c->n_all - 1) / 2);
        if (g > 1) want = std::max(want, 2 * g);
        c->nslots = (int)std::max<int64_t>(
            2, std::min<int64_t>({want, (int64_t)moe::kMaxSlots, (int64_t)c->n_all - 1}));
    }
    // DMA batches of ~192 MiB, at most half the slots (two batches in flight)
    c->copy_group = (int)std::max<int64_t>(
        1, std::min<int64_t>((moe::kCopyBatchBytes + c->blob_bytes - 1) / c->blob_bytes, c->nslots / 2));
    if (const char* e = getenv("MOE_COPY_GROUP")) c->copy_group = std::max(1, std::min(atoi(e), c->nslots));
    c->gemm_group_max = std::min(c->nslots / 2, moe::kMaxBatch);
    c->cap_recv = c->ep ? (int64_t)W * Tm * k : (int64_t)Tm * k;
    // h_act rows: routed rows (received rows under EP) then S * Tm shared rows (sharded: the
    // slice's rows for all W ranks' tokens, W * Tm)
    const int64_t h_rows = c->cap_recv + (int64_t)(c->shard ? W : S) * Tm;
    c->rows_cap = (int64_t)Tm * (k + S);  // y_perm rows
    const int n_tiles = (Tm + moe::kRouteTile - 1) / moe::kRouteTile;

    auto dalloc = [&](void** p, size_t n) { return cudaMalloc(p, n) == cudaSuccess; };
    bool ok = true;
    ok &= cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) == cudaSuccess;
    {
        // Streams only where used: every extra stream shares the device's hardware work queues
        // (CUDA_DEVICE_MAX_CONNECTIONS) with the other contexts of the process.
        if (const char* e = getenv("MOE_TOKEN_LANE")) c->token_lane = atoi(e) != 0;
        if (c->token_lane) {
            int least = 0, greatest = 0;
            ok &= cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess;
            ok &= cudaStreamCreateWithPriority(&c->token_stream, cudaStreamNonBlocking, greatest) ==
                  cudaSuccess;
        }
        if (cfg->flags & MOE_FLAG_PROFILE) {
            ok &= cudaStreamCreateWithFlags(&c->clock_stream, cudaStreamNonBlocking) == cudaSuccess;
            ok &= cudaMalloc((void**)&c->clk_acc, 4 * sizeof(unsigned long long)) == cudaSuccess &&
                  cudaMemset(c->clk_acc, 0, 4 * sizeof(unsigned long long)) == cudaSuccess;
        }
        ok &= cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->out_ev, cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking) == cudaSuccess;
    }
    ok &= dalloc((void**)&c->slot_base, (size_t)c->blob_bytes * c->nslots);
    for (int i = 0; i < c->nslots; ++i) {
        c->slot[i] = c->slot_base ? c->slot_base + (size_t)i * c->blob_bytes : nullptr;
        ok &= cudaEventCreateWithFlags(&c->ready13[i], cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->ready2[i], cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->slot_free[i], cudaEventDisableTiming) == cudaSuccess;
    }
    for (int i = 0; i < 2; ++i) {
        ok &= cudaEventCreateWithFlags(&c->xbuf_free[i], cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->x_ready[i], cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->x_ready_b[i], cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->d2h_done[i], cudaEventDisableTiming) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&c->comb_ev[i], cudaEventDisableTiming) == cudaSuccess;
    }
    ok &= dalloc((void**)&c->idx_ws, sizeof(int32_t) * (size_t)Tm * k);
    ok &= dalloc((void**)&c->gates_ws, sizeof(float) * (size_t)Tm * k);
    ok &= dalloc((void**)&c->tile_counts, sizeof(int32_t) * (size_t)n_tiles * ne);
    ok &= dalloc((void**)&c->wr64, sizeof(double) * moe::router_ws_doubles(h, ne));
    ok &= dalloc((void**)&c->tile_prefix, sizeof(int32_t) * (size_t)n_tiles * ne);
    ok &= dalloc((void**)&c->offsets, sizeof(int32_t) * (size_t)(ne + 1));
    ok &= dalloc((void**)&c->counts, sizeof(int32_t) * (size_t)(ne + S));
    ok &= dalloc((void**)&c->grp1, sizeof(GemmGroup) * (size_t)(ne + S));
    ok &= dalloc((void**)&c->grp2, sizeof(GemmGroup) * (size_t)(ne + S));
    ok &= dalloc((void**)&c->shared_grp, sizeof(GemmGroup) * 2 * (size_t)c->n_all);
    ok &= dalloc((void**)&c->pos, sizeof(int32_t) * (size_t)Tm * k);
    ok &= dalloc((void**)&c->x_perm, 2 * (size_t)Tm * k * h);
    ok &= dalloc((void**)&c->h_act, 2 * (size_t)h_rows * hi);
    ok &= dalloc((void**)&c->y_perm, 2 * (size_t)c->rows_cap * h);
    if (!ok) {
        cudaGetLastError();
        return fail(MOE_E_NOMEM);
    }
    bool tm = true;
    tm &= moe::make_tmap(&c->tm_xperm, c->x_perm, (uint64_t)Tm * k, h, 128);
    tm &= moe::make_tmap(&c->tm_h, c->h_act, (uint64_t)h_rows, hi, 128);
    {   // the whole staging buffer as one W13 view and one W2 view (see engine.h)
        const uint64_t r13 = 3ull * hi * c->nslots, r2 = 3ull * h * c->nslots;
        tm &= moe::make_tmap(&c->tm_w13, c->slot_base, r13, h, (uint32_t)c->bn1);
        tm &= moe::make_tmap(&c->tm_w13_pair, c->slot_base, r13, h, 128);
        tm &= moe::make_tmap(&c->tm_w2, c->slot_base, r2, hi, (uint32_t)c->bn2);
        tm &= moe::make_tmap(&c->tm_w2_pair, c->slot_base, r2, hi, 128);
        // the slice's W2 [h, shard_w] after its W13 [2 shard_w, h], one view per slot (the
        // slice has its own launch, so the map is chosen per launch)
        for (int i = 0; c->shard_w > 0 && i < c->nslots; ++i) {
            const char* w2 = c->slot_base + (size_t)i * c->blob_bytes + 4ll * h * c->shard_w;
            tm &= moe::make_tmap(&c->tm_w2s[i], w2, (uint64_t)h, c->shard_w, (uint32_t)c->bn2);
            tm &= moe::make_tmap(&c->tm_w2s_pair[i], w2, (uint64_t)h, c->shard_w, 128);
        }
    }
    if (!tm) return fail(MOE_E_CUDA);
    if (const char* e = getenv("MOE_GEMM_PAIR")) {   // tests: force one kernel
        if (!strcmp(e, "0")) c->pair_mode = 0;
        else if (!strcmp(e, "1")) c->pair_mode = 1;
        else c->pair_mode = -1;
    }
    {
        const char* gm = getenv("MOE_GEMM_GROUPM");   // tests: raster group override
        if (moe::set_gemm_group_m(gm ? atoi(gm) : 0) != cudaSuccess) return fail(MOE_E_CUDA);
    }
    if (c->ep) {
        moe_status es = moe::ep_init(c);
        if (es != MOE_OK) return fail(es);
    }
    if (cfg->flags & MOE_FLAG_MOVER) {
        c->mover_trace = getenv("MOE_MOVER_TRACE") && atoi(getenv("MOE_MOVER_TRACE")) != 0;
        moe_status ms = moe::mover_start(c);
        if (ms != MOE_OK) return fail(ms);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(MOE_E_CUDA);
    *out = c;
    return MOE_OK;
}

moe_status moe_layer_forward(moe_ctx ctx, const void* hidden, int32_t num_tokens,
                             const void* router_w, const void* const* experts, int32_t top_k,
                             void* out, int32_t* topk_idx, float* topk_w, void* stream) {
    moe_status s = validate_call(ctx, num_tokens, router_w, experts, top_k);
    if (s != MOE_OK || (num_tokens == 0 && !ctx->ep)) return s;
    if (num_tokens > 0) {
        if (!hidden || !out) return set_err(ctx, MOE_E_INVAL, "NULL hidden / out");
        const size_t bytes = (size_t)num_tokens * ctx->cfg.hidden * 2;
        if (overlaps(hidden, bytes, out, bytes)) return set_err(ctx, MOE_E_INVAL, "out aliases hidden");
        if (((uintptr_t)hidden | (uintptr_t)out) & 15)
            return set_err(ctx, MOE_E_INVAL, "hidden/out must be 16-byte aligned");
        if (!is_device(hidden) || !is_device(out))
            return set_err(ctx, MOE_E_INVAL, "hidden/out must be device memory");
        if ((topk_idx && !is_device(topk_idx)) || (topk_w && !is_device(topk_w)))
            return set_err(ctx, MOE_E_INVAL, "topk_idx/topk_w must be device memory");
    }
    MOE_CUDA(ctx, cudaSetDevice(ctx->cfg.device));
    return forward_impl(ctx, static_cast<const __nv_bfloat16*>(hidden), num_tokens,
                        static_cast<const __nv_bfloat16*>(router_w), experts,
                        static_cast<__nv_bfloat16*>(out), topk_idx, topk_w,
                        static_cast<cudaStream_t>(stream), false, 0);
}

moe_status moe_layer_forward_host(moe_ctx ctx, const void* hidden_host, int32_t num_tokens,
                                  const void* router_w, const void* const* experts, int32_t top_k,
                                  void* out_host, int32_t* topk_idx, float* topk_w, void* stream) {
    moe_status s = validate_call(ctx, num_tokens, router_w, experts, top_k);
    if (s != MOE_OK || (num_tokens == 0 && !ctx->ep)) return s;
    moe_ctx c = ctx;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (num_tokens == 0)  // EP: this rank still serves the other ranks' tokens
        return forward_impl(c, nullptr, 0, static_cast<const __nv_bfloat16*>(router_w), experts,
                            nullptr, topk_idx, topk_w, st, false, 0);
    if (!hidden_host || !out_host) return set_err(ctx, MOE_E_INVAL, "NULL hidden / out");
    if (!is_pinned(hidden_host) || !is_pinned(out_host))
        return set_err(ctx, MOE_E_NOT_PINNED, "hidden_host/out_host must be page-locked");
    MOE_CUDA(ctx, cudaSetDevice(ctx->cfg.device));
    const size_t bytes = (size_t)num_tokens * c->cfg.hidden * 2;
    int b = 0;
    s = host_buffer(c, &b);
    if (s != MOE_OK) return s;
    s = stage_tokens(c, b, hidden_host, bytes, 0, c->x_ready[b], 0);
    if (s != MOE_OK) return s;
    // out_dev[b] is rewritten by this call's combine: the result copy of two calls ago must be out
    MOE_CUDA(c, cudaStreamWaitEvent(st, c->d2h_done[b], 0));
    s = forward_impl(c, c->x_dev[b], num_tokens, static_cast<const __nv_bfloat16*>(router_w),
                     experts, c->out_dev[b], topk_idx, topk_w, st, true, b);
    if (s != MOE_OK) return s;
    MOE_CUDA(c, cudaEventRecord(c->xbuf_free[b], st));
    MOE_CUDA(c, cudaEventRecord(c->comb_ev[0], st));
    const int r0 = 0, rows = num_tokens;
    return copy_results(c, b, 1, &out_host, &r0, &rows, c->comb_ev);
}

int64_t moe_packed_layer_bytes(int32_t hidden) {
    if (hidden <= 0) return 0;
    return 2ll * hidden * hidden + 2ll * hidden;
}

moe_status moe_pack_layer(int32_t hidden, const void* wo, const void* gamma, void* dst) {
    if (!wo || !gamma || !dst || hidden <= 0) return MOE_E_INVAL;
    const size_t wo_bytes = (size_t)hidden * hidden * 2;
    memcpy(dst, wo, wo_bytes);
    memcpy(static_cast<char*>(dst) + wo_bytes, gamma, (size_t)hidden * 2);
    return MOE_OK;
}

moe_status moe_taskb_forward(moe_ctx ctx, const void* attn, const void* resid, int32_t num_tokens,
                             const void* layer, float eps, const void* router_w,
                             const void* const* experts, int32_t top_k, void* out,
                             int32_t* topk_idx, float* topk_w, void* stream) {
    moe_status s = validate_call(ctx, num_tokens, router_w, experts, top_k);
    if (s != MOE_OK || (num_tokens == 0 && !ctx->ep)) return s;
    if (!(eps >= 0.0f) || !std::isfinite(eps))
        return set_err(ctx, MOE_E_INVAL, "eps must be finite and >= 0");
    if (num_tokens > 0) {
        if (!attn || !resid || !out || !layer)
            return set_err(ctx, MOE_E_INVAL, "NULL attn / resid / out / layer");
        if (((uintptr_t)attn | (uintptr_t)resid | (uintptr_t)out) & 15)
            return set_err(ctx, MOE_E_INVAL, "attn/resid/out must be 16-byte aligned");
        if (!is_device(attn) || !is_device(resid) || !is_device(out))
            return set_err(ctx, MOE_E_INVAL, "attn/resid/out must be device memory");
        if ((topk_idx && !is_device(topk_idx)) || (topk_w && !is_device(topk_w)))
            return set_err(ctx, MOE_E_INVAL, "topk_idx/topk_w must be device memory");
        if (!is_pinned(layer))
            return set_err(ctx, MOE_E_NOT_PINNED, "layer blob is not page-locked host memory");
    }
    MOE_CUDA(ctx, cudaSetDevice(ctx->cfg.device));
    s = taskb_resources(ctx);
    if (s != MOE_OK) return s;
    const TbPart p0{static_cast<const __nv_bfloat16*>(resid), num_tokens, 0, nullptr};
    return taskb_impl(ctx, static_cast<const __nv_bfloat16*>(attn), p0, nullptr, layer, eps,
                      static_cast<const __nv_bfloat16*>(router_w), experts,
                      static_cast<__nv_bfloat16*>(out), topk_idx, topk_w,
                      static_cast<cudaStream_t>(stream));
}

moe_status moe_taskb_forward_host(moe_ctx ctx, const void* attn_host, const void* resid,
                                  int32_t num_tokens, const void* layer, float eps,
                                  const void* router_w, const void* const* experts, int32_t top_k,
                                  void* out_host, int32_t* topk_idx, float* topk_w, void* stream) {
    const void* a[2] = {attn_host, nullptr};
    const void* r[2] = {resid, nullptr};
    const int32_t n[2] = {num_tokens, 0};
    void* o[2] = {out_host, nullptr};
    return moe_taskb_forward2_host(ctx, a, r, n, layer, eps, router_w, experts, top_k, o, topk_idx,
                                   topk_w, stream);
}

moe_status moe_taskb_forward2_host(moe_ctx ctx, const void* const attn_host[2],
                                   const void* const resid[2], const int32_t num_tokens[2],
                                   const void* layer, float eps, const void* router_w,
                                   const void* const* experts, int32_t top_k,
                                   void* const out_host[2], int32_t* topk_idx, float* topk_w,
                                   void* stream) {
    if (!ctx || !attn_host || !resid || !num_tokens || !out_host) return MOE_E_INVAL;
    if (num_tokens[0] < 0 || num_tokens[1] < 0)
        return set_err(ctx, MOE_E_INVAL, "negative partition size");
    const int T = num_tokens[0] + num_tokens[1];
    moe_status s = validate_call(ctx, T, router_w, experts, top_k);
    if (s != MOE_OK || (T == 0 && !ctx->ep)) return s;
    if (!(eps >= 0.0f) || !std::isfinite(eps))
        return set_err(ctx, MOE_E_INVAL, "eps must be finite and >= 0");
    moe_ctx c = ctx;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    MOE_CUDA(c, cudaSetDevice(c->cfg.device));
    if (!layer) return set_err(c, MOE_E_INVAL, "NULL layer");
    if (!is_pinned(layer)) return set_err(c, MOE_E_NOT_PINNED, "layer must be page-locked");
    if (T == 0) {  // EP: this rank still serves the other ranks' tokens
        s = taskb_resources(c);
        if (s != MOE_OK) return s;
        const TbPart none{nullptr, 0, 0, nullptr};
        return taskb_impl(c, nullptr, none, nullptr, layer, eps,
                          static_cast<const __nv_bfloat16*>(router_w), experts, nullptr, topk_idx,
                          topk_w, st);
    }
    for (int p = 0; p < 2; ++p) {
        if (num_tokens[p] == 0) continue;
        if (!attn_host[p] || !resid[p] || !out_host[p])
            return set_err(c, MOE_E_INVAL, "NULL attn_host / resid / out_host of partition %d", p);
        if (((uintptr_t)resid[p] & 15) || !is_device(resid[p]))
            return set_err(c, MOE_E_INVAL, "resid[%d] must be 16-byte aligned device memory", p);
        if (!is_pinned(attn_host[p]) || !is_pinned(out_host[p]))
            return set_err(c, MOE_E_NOT_PINNED, "attn_host/out_host[%d] must be page-locked", p);
    }
    if ((topk_idx && !is_device(topk_idx)) || (topk_w && !is_device(topk_w)))
        return set_err(c, MOE_E_INVAL, "topk_idx/topk_w must be device memory");
    s = taskb_resources(c);
    if (s != MOE_OK) return s;
    const size_t rb = (size_t)c->cfg.hidden * 2;
    int b = 0;
    s = host_buffer(c, &b);
    if (s != MOE_OK) return s;
    // the first non-empty partition is "alpha": its attention output goes ahead of Wo + experts
    const int pa = num_tokens[0] > 0 ? 0 : 1, pb = 1 - pa;
    const int Ta = num_tokens[pa], Tb = pa == 0 ? num_tokens[1] : 0;
    s = stage_tokens(c, b, attn_host[pa], (size_t)Ta * rb, 0, c->x_ready[b], 0);
    if (s != MOE_OK) return s;
    MOE_CUDA(c, cudaStreamWaitEvent(st, c->d2h_done[b], 0));   // out_dev[b] free (see forward)
    const TbPart p0{static_cast<const __nv_bfloat16*>(resid[pa]), Ta, 0, c->x_ready[b]};
    TbLate late;
    late.part = TbPart{static_cast<const __nv_bfloat16*>(resid[pb]), Tb, Ta, c->x_ready_b[b]};
    late.stage = [&]() {   // beta's attention output: queued behind this call's weight requests
        return stage_tokens(c, b, attn_host[pb], (size_t)Tb * rb, (size_t)Ta * rb,
                            c->x_ready_b[b], 1);
    };
    s = taskb_impl(c, c->x_dev[b], p0, Tb > 0 ? &late : nullptr, layer, eps,
                   static_cast<const __nv_bfloat16*>(router_w), experts, c->out_dev[b], topk_idx,
                   topk_w, st, c->comb_ev[0]);
    if (s != MOE_OK) return s;
    MOE_CUDA(c, cudaEventRecord(c->xbuf_free[b], st));
    MOE_CUDA(c, cudaEventRecord(c->comb_ev[Tb > 0 ? 1 : 0], st));
    void* const hosts[2] = {out_host[pa], Tb > 0 ? out_host[pb] : nullptr};
    const int row0[2] = {0, Ta}, rows[2] = {Ta, Tb};
    return copy_results(c, b, 2, hosts, row0, rows, c->comb_ev);
}

moe_status moe_wait_output(moe_ctx ctx, void* stream) {
    if (!ctx) return MOE_E_INVAL;
    MOE_CUDA(ctx, cudaSetDevice(ctx->cfg.device));
    MOE_CUDA(ctx, cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->out_ev, 0));
    return MOE_OK;
}

moe_status moe_sync(moe_ctx ctx) {
    if (!ctx) return MOE_E_INVAL;
    if (ctx->p2p_diag_h && ctx->p2p_diag_h[5]) {   // the P2P plan refused an overflow (ep_p2p.cu)
        ctx->sticky = MOE_E_STATE;
        return set_err(ctx, MOE_E_STATE,
                       "P2P EP: an expert owner would receive %lld rows > its capacity %lld "
                       "(ranks configured with different max_tokens / top_k?); the call "
                       "exchanged nothing", ctx->p2p_diag_h[6], ctx->p2p_diag_h[7]);
    }
    if (ctx->p2p_diag_h && ctx->p2p_diag_h[0]) {   // a P2P flag wait timed out (ep_p2p.cu)
        ctx->sticky = MOE_E_CUDA;
        return set_err(ctx, MOE_E_CUDA,
                       "P2P EP: rank %d timed out waiting for flag %lld of rank %lld to reach "
                       "call %lld (saw %lld)", ctx->cfg.rank, ctx->p2p_diag_h[1],
                       ctx->p2p_diag_h[2], ctx->p2p_diag_h[3], ctx->p2p_diag_h[4]);
    }
    MOE_CUDA(ctx, cudaSetDevice(ctx->cfg.device));
    if (ctx->mover) {   // every packet issued before the streams are waited on
        moe_status ms = moe::mover_drain(ctx);
        if (ms != MOE_OK) return ms;
    }
    MOE_CUDA(ctx, cudaEventSynchronize(ctx->done_ev));     // the last call (see engine.h)
    MOE_CUDA(ctx, cudaEventSynchronize(ctx->out_ev));      // its result copy (host-buffer calls)
    MOE_CUDA(ctx, cudaStreamSynchronize(ctx->copy_stream));
    if (ctx->token_stream) MOE_CUDA(ctx, cudaStreamSynchronize(ctx->token_stream));
    if (ctx->comm && moe::nccl_api()) {
        moe::ncclResult_t r = 0;
        moe::nccl_api()->CommGetAsyncError(ctx->comm, &r);
        if (r != 0) {
            ctx->sticky = MOE_E_NCCL;
            return set_err(ctx, MOE_E_NCCL, "NCCL async error: %s", moe::nccl_api()->GetErrorString(r));
        }
    }
    return ctx->sticky;
}

moe_status moe_get_stats(moe_ctx ctx, moe_stats* out) {
    if (!ctx || !out) return MOE_E_INVAL;
    moe_status s = moe_sync(ctx);
    if (s != MOE_OK) return s;
    double* bucket[moe::kRecKinds] = {&ctx->stats.h2d_ms,   &ctx->stats.route_ms,   &ctx->stats.permute_ms,
                                      &ctx->stats.gemm1_ms, &ctx->stats.gemm2_ms,   &ctx->stats.combine_ms,
                                      &ctx->stats.comm_ms,  &ctx->stats.part_latency_ms[0],
                                      &ctx->stats.part_latency_ms[1],
                                      &ctx->stats.oproj_ms, &ctx->stats.norm_ms,
                                      &ctx->stats.h2d_token_ms};
    for (const moe::Rec& r : ctx->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
            *bucket[r.kind] += ms;
            if (r.kind == moe::kRecTokenA || r.kind == moe::kRecTokenB)
                ctx->stats.token_latency_ms += ms;
        } else {
            cudaGetLastError();
        }
        ctx->ev_pool.push_back(r.a);
        ctx->ev_pool.push_back(r.b);
    }
    ctx->pending.clear();
    if (ctx->mover) ctx->stats.h2d_ms += moe::mover_take_h2d_ms(ctx, nullptr);
    ctx->stats.num_slots = ctx->nslots;
    ctx->stats.comm_bytes = ctx->comm_bytes;
    if (ctx->p2p && ctx->p2p_bytes) {   // P2P transport: counted on the device by the plan kernel
        long long b = 0;
        MOE_CUDA(ctx, cudaMemcpyAsync(&b, ctx->p2p_bytes, sizeof b, cudaMemcpyDeviceToHost,
                                      ctx->copy_stream));
        MOE_CUDA(ctx, cudaStreamSynchronize(ctx->copy_stream));
        ctx->stats.comm_bytes = b;
    }
    if (ctx->clk_acc) {   // SM clock during the expert GEMMs (in-kernel clock64 / globaltimer)
        unsigned long long v[4] = {};
        MOE_CUDA(ctx, cudaMemcpyAsync(v, ctx->clk_acc, sizeof v, cudaMemcpyDeviceToHost,
                                      ctx->copy_stream));
        MOE_CUDA(ctx, cudaStreamSynchronize(ctx->copy_stream));
        ctx->stats.gemm1_sm_mhz = v[1] ? 1e3 * (double)v[0] / (double)v[1] : 0.0;
        ctx->stats.gemm2_sm_mhz = v[3] ? 1e3 * (double)v[2] / (double)v[3] : 0.0;
    }
    *out = ctx->stats;
    return MOE_OK;
}

moe_status moe_reset_stats(moe_ctx ctx) {
    if (!ctx) return MOE_E_INVAL;
    moe_stats tmp;
    moe_status s = moe_get_stats(ctx, &tmp);
    ctx->stats = moe_stats{};
    if (ctx->clk_acc && s == MOE_OK) {
        MOE_CUDA(ctx, cudaMemsetAsync(ctx->clk_acc, 0, 4 * sizeof(unsigned long long),
                                      ctx->copy_stream));
        MOE_CUDA(ctx, cudaStreamSynchronize(ctx->copy_stream));
    }
    return s;
}

moe_status moe_debug_buffers(moe_ctx ctx, moe_debug_view* out) {
    if (!ctx || !out) return MOE_E_INVAL;
    out->counts = ctx->counts;
    out->offsets = ctx->offsets;
    out->pos = ctx->pos;
    out->x_perm = ctx->ep ? ctx->x_recv : ctx->x_perm;
    out->h_act = ctx->h_act;
    out->y_perm = ctx->y_perm;
    out->rows = ctx->ep ? ctx->last_recv_rows : ctx->last_rows;
    if (ctx->p2p && ctx->p2p_rows) {   // P2P transport: the plan kernel counted the rows
        int32_t r = 0;
        MOE_CUDA(ctx, cudaSetDevice(ctx->cfg.device));
        moe_status s = moe_sync(ctx);
        if (s != MOE_OK) return s;
        MOE_CUDA(ctx, cudaMemcpyAsync(&r, ctx->p2p_rows, sizeof r, cudaMemcpyDeviceToHost,
                                      ctx->copy_stream));
        MOE_CUDA(ctx, cudaStreamSynchronize(ctx->copy_stream));
        out->rows = r;
    }
    out->h1 = ctx->h1_ws;
    out->moe_in = ctx->u_ws;
    out->taskb_tokens = ctx->last_taskb_T;
    return MOE_OK;
}

moe_status moe_destroy(moe_ctx c) {
    if (!c) return MOE_OK;
    cudaSetDevice(c->cfg.device);
    moe::mover_stop(c);
    cudaDeviceSynchronize();
    moe::ep_destroy(c);
    for (const moe::Rec& r : c->pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    cudaFree(c->slot_base);
    for (int i = 0; i < moe::kMaxSlots; ++i) {
        cudaEvent_t evs[] = {c->ready13[i], c->ready2[i], c->slot_free[i]};
        for (cudaEvent_t e : evs)
            if (e) cudaEventDestroy(e);
    }
    for (int i = 0; i < 2; ++i) {
        cudaFree(c->x_dev[i]);
        cudaFree(c->out_dev[i]);
        cudaEvent_t evs[] = {c->xbuf_free[i], c->x_ready[i], c->lw_ready[i], c->lw_free[i],
                             c->x_ready_b[i], c->d2h_done[i], c->comb_ev[i]};
        for (cudaEvent_t e : evs)
            if (e) cudaEventDestroy(e);
        cudaFree(c->lw_slot[i]);
    }
    void* bufs[] = {c->idx_ws, c->gates_ws, c->tile_counts, c->wr64, c->tile_prefix, c->offsets, c->counts,
                    c->grp1, c->grp2, c->shared_grp, c->pos, c->x_perm, c->h_act, c->y_perm,
                    c->h1_ws, c->u_ws, c->oproj_grp, c->clk_acc};
    for (void* p : bufs) cudaFree(p);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->token_stream) cudaStreamDestroy(c->token_stream);
    if (c->clock_stream) cudaStreamDestroy(c->clock_stream);
    if (c->done_ev) cudaEventDestroy(c->done_ev);
    if (c->out_ev) cudaEventDestroy(c->out_ev);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    cudaGetLastError();
    delete c;
    return MOE_OK;
}

const char* moe_status_string(moe_status s) {
    switch (s) {
        case MOE_OK: return "MOE_OK";
        case MOE_E_INVAL: return "MOE_E_INVAL: invalid argument";
        case MOE_E_CUDA: return "MOE_E_CUDA: CUDA error";
        case MOE_E_NCCL: return "MOE_E_NCCL: NCCL error";
        case MOE_E_NOMEM: return "MOE_E_NOMEM: out of memory";
        case MOE_E_NOT_PINNED: return "MOE_E_NOT_PINNED: host buffer is not page-locked";
        case MOE_E_UNSUPPORTED: return "MOE_E_UNSUPPORTED: outside the kernels' envelope";
        case MOE_E_STATE: return "MOE_E_STATE: context in error state";
    }
    return "unknown moe_status";
}

const char* moe_last_error(moe_ctx ctx) { return ctx ? ctx->last_error.c_str() : ""; }

moe_status moe_probe_h2d(int32_t device, size_t bytes, int32_t iters, double* gbps) {
    if (!gbps || bytes == 0 || iters <= 0) return MOE_E_INVAL;
    *gbps = 0.0;
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return MOE_E_CUDA;
    }
    void* h = nullptr;
    void* d = nullptr;
    if (cudaHostAlloc(&h, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return MOE_E_NOMEM;
    }
    if (cudaMalloc(&d, bytes) != cudaSuccess) {
        cudaFreeHost(h);
        cudaGetLastError();
        return MOE_E_NOMEM;
    }
    memset(h, 1, bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);  // warm-up
    double best = 0.0;
    for (int i = 0; i < iters; ++i) {
        cudaEventRecord(a, st);
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (ms > 0) best = std::max(best, (double)bytes / (ms * 1e-3) / 1e9);
    }
    cudaError_t e = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    cudaFree(d);
    cudaFreeHost(h);
    *gbps = best;
    return e == cudaSuccess ? MOE_OK : MOE_E_CUDA;
}

}  // extern "C"
