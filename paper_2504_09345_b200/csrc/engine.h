// engine.h -- the context object behind the C ABI and helpers shared by moe_api.cu / ep.cu.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/moe.h"
#include "moe_internal.h"

namespace moe {

// kRecTokenA / B: enqueue -> resident latency of a host token copy of partition 0 / 1
enum RecKind { kRecH2D = 0, kRecRoute, kRecPermute, kRecGemm1, kRecGemm2, kRecCombine, kRecComm,
               kRecTokenA, kRecTokenB, kRecOproj, kRecNorm, kRecH2DTok, kRecKinds };

struct Rec {
    int kind;
    cudaEvent_t a, b;
};

// ------------------------------------------------------------------ NCCL (dlopen'ed, EP only)
// Minimal ABI-stable declarations (NCCL >= 2.10): we never link NCCL at build time, so the
// library loads on machines without it; expert parallelism dlopens the process's libnccl.so.2
// (the one torch.distributed already loaded, or MOE_NCCL_LIBRARY).
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
struct ncclUniqueId { char internal[128]; };
enum { kNcclInt32 = 2, kNcclBfloat16 = 9 };

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;   // optional
};
const NcclApi* nccl_api();  // nullptr if libnccl cannot be found

}  // namespace moe

namespace moe {
struct Mover;   // mover.cu: the Contiguous Data Mover thread (MOE_FLAG_MOVER)
}

struct moe_ctx_s {
    moe_config cfg{};
    int n_local = 0;       // routed experts owned by this rank
    int n_all = 0;         // n_local + s_items (items streamed per call)
    int s_items = 0;       // shared items streamed per call: num_shared, or 0/1 (sharded)
    // MOE_FLAG_SHARD_SHARED: this rank streams one slice of the concatenated
    // shared FFN, shard_w columns wide (0 = none), run over every rank's tokens.  Its W2 part
    // ([h, shard_w]) is read through tm_w2s*[s], a view of slot s's W2 part with shard_w columns
    // per row (any width: no divisibility of the slot by the row pitch is needed).
    bool shard = false;
    int shard_w = 0;
    uint32_t shard_mask = 0;          // ranks whose slice is not empty
    int64_t slice_bytes = 0;
    CUtensorMap tm_w2s[moe::kMaxSlots], tm_w2s_pair[moe::kMaxSlots];
    int64_t blob_bytes = 0, w13_bytes = 0;
    int num_sms = 148;
    int bn1 = 256, bn2 = 256;
    int64_t rows_cap = 0;  // rows of h_act / y_perm (single GPU)
    cudaStream_t copy_stream = nullptr;
    // Token copies of moe_layer_forward_host ride the weight stream, just ahead of their call's
    // weights (right for throughput).  MOE_TOKEN_LANE=1 puts them on a highest-priority stream
    // instead -- measured NOT to help: DMAs are served in submission order across streams, so a
    // priority lane needs host-paced packets (the paper's one-packet-in-flight mover,
    // PAPER.md:829-835); see DESIGN.md §7.
    cudaStream_t token_stream = nullptr;
    cudaStream_t clock_stream = nullptr;  // idle stream: events on it timestamp enqueue time
    // Recorded at the end of every call on the caller's stream: moe_sync waits on it (and the
    // copy stream) instead of the whole device -- a device-wide sync from one rank's thread
    // would also wait on the other in-process ranks' flag-wait kernels (LOCAL_EP deadlock).
    cudaEvent_t done_ev = nullptr;
    bool token_lane = false;

    // staging slots (a bounded GPU weight buffer, recycled every call)
    int nslots = 2;
    char* slot_base = nullptr;          // one allocation: slot s = slot_base + s * blob_bytes
    void* slot[moe::kMaxSlots] = {};
    // DMA coalescing: consecutive streamed items whose host blobs are contiguous and whose slots
    // are adjacent are moved by one cudaMemcpyAsync of up to copy_group experts.
    int copy_group = 1;
    // Routed experts per GEMM launch: up to gemm_group_max (half the slots) consecutive experts
    // until the launch expects gemm_rows_target rows (MOE_GEMM_ROWS overrides; forward_impl).
    int gemm_group_max = 1;
    int64_t gemm_rows_target = 2048;
    int pend_n = 0;                     // items in the pending batch
    uint64_t pend_q0 = 0;               // streamed-item index of the batch's first item
    const char* pend_src = nullptr;     // host address of the batch's first blob
    int64_t pend_item = 0, pend_w13 = 0; // bytes per item of the batch / of its W13 part
    uintptr_t pend_base = 0;            // start of that blob's pinned allocation
    cudaEvent_t ready13[moe::kMaxSlots] = {}, ready2[moe::kMaxSlots] = {};
    cudaEvent_t slot_free[moe::kMaxSlots] = {};
    uint64_t seq = 0;  // streamed-item counter across calls: item q uses slot q % nslots
    // MOE_FLAG_MOVER: expert copies go through the mover thread (mover.cu) in packets, ordered
    // against the GEMMs by device counters instead of the ready13 / ready2 / slot_free events.
    moe::Mover* mover = nullptr;
    bool mover_trace = false;   // MOE_MOVER_TRACE=1: one stderr line per GEMM wait / mover job
    // The staging buffer seen as one W13 matrix [nslots * 3 h_i, h] and one W2 matrix
    // [nslots * 3 h, h_i]: slot s's W13 starts at row 3 h_i s, its W2 at row 3 h s + 2 h, so one
    // GEMM launch can cover experts in different slots (GemmBatch::b_row).
    CUtensorMap tm_w13, tm_w2;
    CUtensorMap tm_w13_pair, tm_w2_pair;   // 128-row boxes (CTA-pair GEMM)
    // DMA batches (flush_copies): slot s holds item batch_q0[s] + j of a batch of batch_n[s]
    uint64_t batch_q0[moe::kMaxSlots] = {};
    int batch_n[moe::kMaxSlots] = {};
    // MOE_GEMM_PAIR: 0 never, 1 always, -1 auto (default): the host's wave model on the
    // EXPECTED group sizes picks the CTA-pair or the single-CTA kernel, one launch (pick_pair).
    int pair_mode = -1;

    // workspace
    int32_t* idx_ws = nullptr;
    float* gates_ws = nullptr;
    int32_t* tile_counts = nullptr;
    double* wr64 = nullptr;   // router rows widened to fp64 (router workspace)
    int32_t* tile_prefix = nullptr;
    int32_t* offsets = nullptr;
    int32_t* counts = nullptr;
    moe::GemmGroup* grp1 = nullptr;
    moe::GemmGroup* grp2 = nullptr;
    moe::GemmGroup* shared_grp = nullptr;   // [2][n_all]: shared experts' groups (before routing)
    int32_t* pos = nullptr;
    __nv_bfloat16* x_perm = nullptr;
    __nv_bfloat16* h_act = nullptr;
    __nv_bfloat16* y_perm = nullptr;
    CUtensorMap tm_xperm, tm_h;
    int64_t last_rows = 0;

    // expert parallelism (world_size > 1, or MOE_FLAG_FORCE_EP)
    bool ep = false;
    bool local_ep = false;             // MOE_FLAG_LOCAL_EP: in-process transport
    void* local_group = nullptr;       // ep.cu LocalGroup*
    moe::ncclComm_t comm = nullptr;
    int64_t cap_recv = 0;              // rows a rank can receive: W * max_tokens * top_k
    int32_t* counts_all = nullptr;     // device [W][N_e]
    int32_t* counts_all_h = nullptr;   // pinned host copy
    moe::GemmGroup* ep_grp_h = nullptr;  // pinned [2][n_all]
    moe::GemmGroup* ep_grp = nullptr;    // device [2][n_all]
    __nv_bfloat16* x_recv = nullptr;
    __nv_bfloat16* y_recv = nullptr;
    CUtensorMap tm_xrecv;
    std::vector<int32_t> send_off, send_cnt, recv_off, recv_cnt, grp_off;
    int64_t last_recv_rows = 0, comm_bytes = 0;
    // P2P transport (MOE_FLAG_LOCAL_EP: ranks in this process; MOE_FLAG_IPC_EP: ranks in other
    // processes, buffers mapped with CUDA IPC): fused permute+dispatch and combine kernels over
    // peer memory, synchronised by device flags (ep_p2p.cu) -- no host sync per call.
    bool p2p = false;
    bool p2p_ready = false;                  // peer tables filled (connect done)
    uint64_t p2p_seq = 0;                    // calls issued (flag values)
    uint64_t p2p_selftest_seq = 0;           // moe_ep_ipc_selftest tokens
    unsigned long long* p2p_flags = nullptr; // device [kP2PFlags][kMaxRanks], written by peers
    int32_t* p2p_counts = nullptr;           // device [2][W][N_e], row s written by rank s
    moe::P2PTable* p2p_tab = nullptr;        // device tables (peers' buffers in this process)
    moe::PeerRows* pr_x = nullptr;           // peers' x_recv + this rank's send bases
    moe::PeerRows* pr_y = nullptr;           // peers' y_recv + the same bases
    int32_t* p2p_rows = nullptr;             // device: rows received by the last call
    long long* p2p_bytes = nullptr;          // device: bytes moved (stats)
    unsigned long long* clk_acc = nullptr;   // device [4]: GEMM1 / GEMM2 SM cycles, ns (profile)
    void* ipc_opened[moe::kMaxRanks][4] = {};  // IPC mappings to close (MOE_FLAG_IPC_EP)
    long long* p2p_diag_h = nullptr;         // pinned, mapped: a timed-out flag wait (moe_sync)
    long long* p2p_diag_d = nullptr;
    // LOCAL_EP synchronises with events instead of device flag waits: [flag][call parity],
    // recorded by this rank, waited on by its peers after a host barrier (enqueue order) -- a
    // spinning wait kernel could share a hardware queue with the peer work it waits for when
    // several ranks run on one GPU.
    cudaEvent_t p2p_ev[moe::kP2PFlags][2] = {};

    // GPU Task B (moe_taskb_forward; allocated on first use).  The layer weights (Wo + gamma,
    // moe_packed_layer_bytes) are streamed like the experts, into two slots of their own, on the
    // same copy stream just ahead of the call's expert weights.
    int64_t layer_bytes = 0;
    bool taskb_ready = false;         // every Task B resource below allocated and mapped
    char* lw_slot[2] = {nullptr, nullptr};
    cudaEvent_t lw_ready[2] = {}, lw_free[2] = {};
    CUtensorMap tm_wo[2], tm_wo_pair[2];
    uint64_t lw_seq = 0;
    __nv_bfloat16* h1_ws = nullptr;   // [max_tokens, h] residual stream after the O-projection
    __nv_bfloat16* u_ws = nullptr;    // [max_tokens, h] normalised MoE input
    moe::GemmGroup* oproj_grp = nullptr;
    int64_t last_taskb_T = -1;

    // host-buffer mode (moe_layer_forward_host)
    __nv_bfloat16* x_dev[2] = {nullptr, nullptr};
    __nv_bfloat16* out_dev[2] = {nullptr, nullptr};
    cudaEvent_t xbuf_free[2] = {}, x_ready[2] = {};
    cudaEvent_t x_ready_b[2] = {};      // [parity] partition 1's tokens resident (2-partition Task B)
    // Result copies (device -> pinned host) run on their own stream, so the caller's stream never
    // waits for them (the next call's shared-expert GEMMs and routing start at once):
    // comb_ev[p] = partition p combined (recorded on the caller's stream); d2h_done[b] = the copy
    // out of out_dev[b] finished (the call reusing out_dev[b] waits for it); out_ev = the last
    // result copy finished (moe_wait_output, moe_sync).
    cudaStream_t d2h_stream = nullptr;
    cudaEvent_t comb_ev[2] = {}, d2h_done[2] = {};
    cudaEvent_t out_ev = nullptr;
    int host_parity = 0;

    // profiling
    std::vector<moe::Rec> pending;
    std::vector<cudaEvent_t> ev_pool;
    moe_stats stats{};

    std::vector<uintptr_t> call_base;   // this call's expert blobs -> start of their allocation
    std::string last_error;
    moe_status sticky = MOE_OK;
};

namespace moe {

moe_status set_err(moe_ctx c, moe_status s, const char* fmt, ...);
bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
cudaEvent_t pool_get(moe_ctx c);

#define MOE_CUDA(ctx, expr)                                                                  \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            if (ctx) (ctx)->sticky = MOE_E_CUDA;                                             \
            return ::moe::set_err(ctx, MOE_E_CUDA, "%s failed: %s (%s:%d)", #expr,           \
                                  cudaGetErrorString(_e), __FILE__, __LINE__);               \
        }                                                                                    \
    } while (0)

#define MOE_NCCL(ctx, expr)                                                                  \
    do {                                                                                     \
        ::moe::ncclResult_t _r = (expr);                                                     \
        if (_r != 0) {                                                                       \
            if (ctx) (ctx)->sticky = MOE_E_NCCL;                                             \
            return ::moe::set_err(ctx, MOE_E_NCCL, "%s failed: %s (%s:%d)", #expr,           \
                                  ::moe::nccl_api()->GetErrorString(_r), __FILE__, __LINE__); \
        }                                                                                    \
    } while (0)

// CUDA-event bracket around a launch when MOE_FLAG_PROFILE is set.
struct Prof {
    moe_ctx c;
    bool on;
    cudaEvent_t a = nullptr;
    int kind;
    cudaStream_t st;
    Prof(moe_ctx c_, int k, cudaStream_t s)
        : c(c_), on((c_->cfg.flags & MOE_FLAG_PROFILE) != 0), kind(k), st(s) {
        if (on) {
            a = pool_get(c);
            cudaEventRecord(a, st);
        }
    }
    void end() {
        if (on) {
            cudaEvent_t b = pool_get(c);
            cudaEventRecord(b, st);
            c->pending.push_back(Rec{kind, a, b});
        }
    }
};

// Contiguous Data Mover (mover.cu, MOE_FLAG_MOVER)
moe_status mover_start(moe_ctx c);
void mover_stop(moe_ctx c);                      // drains, joins, frees
moe_status mover_drain(moe_ctx c);               // every queued packet issued; mover errors
moe_status mover_push(moe_ctx c, uint64_t q0, int n, const char* src, char* dst, int64_t item,
                      int64_t w13);   // n items of `item` bytes (W13 part: the first w13)
moe_status mover_wait(moe_ctx c, cudaStream_t st, int which, uint64_t value);  // 0 r13, 1 r2
moe_status mover_mark_free(moe_ctx c, cudaStream_t st, uint64_t value);
double mover_take_h2d_ms(moe_ctx c, int64_t* packets);

// expert parallelism (ep.cu)
// Layer shape a rank publishes in its IPC blob (after the 4 memory handles); connect checks that
// every rank's matches its own.
struct IpcShape {
    int32_t magic, rank, world, hidden, ffn, num_experts, top_k, num_shared, max_tokens;
    int32_t shard;   // MOE_FLAG_SHARD_SHARED bit: all ranks must agree
};
IpcShape ipc_shape(moe_ctx c);
moe_status ep_init(moe_ctx c);
void ep_destroy(moe_ctx c);
// After routing/permute on `st`: exchange counts (host sync), build the plan, dispatch x_perm
// rows to their experts' ranks (NCCL grouped send/recv).
moe_status ep_dispatch(moe_ctx c, int T, cudaStream_t st);
// After the local expert GEMMs: return y_recv rows to their source ranks' y_perm.
moe_status ep_combine(moe_ctx c, cudaStream_t st);
// P2P transport steps (see ep_p2p.cu for the protocol), all on `st`:
//   before the permute: counts exchange + plan + wait until the owners' x_recv are free;
moe_status p2p_before_dispatch(moe_ctx c, int T, cudaStream_t st);
//   after the permute (which wrote into the owners' x_recv): signal + wait for all dispatches;
moe_status p2p_after_dispatch(moe_ctx c, cudaStream_t st);
//   after the expert GEMMs: signal x_recv free / y_recv ready, wait for every owner's y_recv;
moe_status p2p_after_gemms(moe_ctx c, cudaStream_t st);
//   after the combine: signal y_recv read.
moe_status p2p_after_combine(moe_ctx c, cudaStream_t st);

}  // namespace moe
