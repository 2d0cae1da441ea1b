// moe_internal.h -- shared declarations between the host engine (moe_api.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace moe {

constexpr int kRouteTile = 32;       // tokens per routing tile (router / permute granularity)
constexpr int kMaxExperts = 128;     // envelope: N_e <= 128
constexpr int kMaxTopK = 8;          // envelope: top_k <= 8
constexpr int kMaxShared = 8;
constexpr int kMaxSlots = 32;        // expert staging slots
// auto slot count: ~512 MiB of staging (2 slots for Mixtral/DBRX-size experts, 32 for
// DeepSeek-V2-Lite-size ones); coalesced H2D DMA size target ~192 MiB (C4: 12 experts per DMA
// and per grouped GEMM launch -- measured 99.45% of the link roofline vs 98.9% at 64 MiB).
constexpr int64_t kAutoSlotBytes = 512ll << 20;
constexpr int64_t kCopyBatchBytes = 192ll << 20;

// Row range of one expert group inside a GEMM's A operand, and where its output rows go.
struct GemmGroup {
    int32_t a_begin;   // first A row of the group
    int32_t a_end;     // one past the last A row
    int32_t out_base;  // output row of A row a_begin
    int32_t pad;
};

// The expert groups of one GEMM launch (kernel parameter, by value): entry i is group
// table[idx[i]] (a device table written by the routing / EP plan kernels), whose weights start
// at row b_row[i] of the launch's B tensor map (one map spans all staging slots).
constexpr int kMaxBatch = 16;
struct GemmBatch {
    const GemmGroup* table;
    int32_t idx[kMaxBatch];
    int32_t b_row[kMaxBatch];
    int32_t n;
    // clk: if non-null, CTA 0 adds its SM cycles (clock64) and elapsed ns (globaltimer) from
    // kernel entry to exit to clk[0] / clk[1] (the SM clock under power management).
    unsigned long long* clk;
};

// ------------------------------------------------------------ expert parallelism, P2P transport
constexpr int kMaxRanks = 8;         // EP group size (one B200 box)
// Row buffers of the EP group as seen by one rank (device-resident, rewritten by the plan kernel
// every call): routed row (t, j) of expert e lives in rank e / nl's buffer at row
// base[e] + (pos[t, j] - offsets[e]) -- base[e] is where this rank's block for expert e starts
// in the owner's expert-major layout (moe_ep_plan's recv_off).
// MOE_FLAG_SHARD_SHARED: every rank in shard_mask also holds a shared-FFN slice; the rows from
// cap_recv on of its x_recv / y_recv hold all ranks' tokens (rank-major, rank q's T_q tokens
// from row cap_recv + P_q, P_q = sum_{q'<q} T_q') and the slice's partial outputs for them.
// shard_row = cap_recv + P_me of THIS rank (written by the plan kernel every call), -1 = off.
struct PeerRows {
    __nv_bfloat16* rows[kMaxRanks];
    int32_t base[kMaxExperts];
    int32_t nl;
    int32_t shard_row;
    uint32_t shard_mask;
};

// Per-call synchronisation of the P2P transport: each rank owns flags[kP2PFlags][kMaxRanks]
// (uint64 call numbers) that its PEERS write (release, system scope) and it waits on (acquire).
enum P2PFlag { kFlagCounts = 0, kFlagDispatched, kFlagXFree, kFlagYReady, kFlagYDone,
               kFlagSelftest, kP2PFlags };
struct P2PTable {   // device-resident: every rank's buffers, as mapped in this process
    unsigned long long* flags[kMaxRanks];
    int32_t* counts[kMaxRanks];      // [2][W][N_e] (call parity, source rank, expert)
};
// Push this rank's per-expert counts into every peer's counts[par][me][:], then release
// kFlagCounts = seq on every peer.
cudaError_t launch_p2p_push_counts(const P2PTable* tab, const int32_t* counts, int ne, int W,
                                   int me, int par, unsigned long long seq, cudaStream_t st);
// flags[which][me] = val on every peer (after a system-scope fence).
cudaError_t launch_p2p_signal(const P2PTable* tab, int W, int me, int which,
                              unsigned long long val, cudaStream_t st);
// Spin (acquire, system scope) until my flags[which][s] >= val for every rank s; traps after
// ~20 s (a lost peer must not hang the GPU), first writing {1, which, s, val, seen} to the
// host-mapped diag[5] (nullable).
cudaError_t launch_p2p_wait(const unsigned long long* flags, int W, int which,
                            unsigned long long val, long long* diag, cudaStream_t st);
// Transport self-test (collective, once after connect): every rank writes a tagged word into
// each peer's x_recv and releases kFlagSelftest = token; then waits (acquire, NO trap: gives up
// after timeout_cycles) for every peer and checks the words it received.  *result = bitmask:
// bit s = peer s never signalled, bit 8+s = peer s's word wrong or missing.
cudaError_t launch_p2p_selftest(const P2PTable* tab, const PeerRows* pr_x,
                                const unsigned long long* my_flags, const uint32_t* my_xrecv,
                                int W, int me, unsigned long long token,
                                long long timeout_cycles, int* result, cudaStream_t st);
// From counts[par] (all ranks' per-expert counts): this rank's GEMM groups over x_recv
// (expert-major, moe_ep_plan's layout) + shared-expert groups, the send bases of pr_x / pr_y
// (where this rank's rows for expert e start in the owner's buffers), rows received (rows_out)
// and bytes sent (+= bytes_acc).  If some owner would receive more than cap_recv rows, nothing
// is dispatched (bases -1, empty groups) and diag[5..7] = {1, rows, cap_recv} (host-mapped).
// shard_item >= 0 (MOE_FLAG_SHARD_SHARED): group entry of this rank's shared slice, run over
// every rank's tokens (x_recv rows cap_recv + [0, sum_q T_q)), and pr_x / pr_y->shard_row set;
// -1 = shared experts replicated (groups over the local tokens) or none.
cudaError_t launch_p2p_plan(const int32_t* counts_par, int W, int ne, int me, int T, int k,
                            int S, long long cap_recv, int n_all, int h, GemmGroup* grp,
                            PeerRows* pr_x, PeerRows* pr_y, int32_t* rows_out,
                            long long* bytes_acc, long long* diag, int shard_item,
                            cudaStream_t st);

// ---------------------------------------------------------------------------- routing kernels
// a2+a3: router GEMM (fp64, ascending c) + warp-shuffle top-k + softmax gates + per-tile counts.
//   wr64: device workspace of router_ws_doubles(h, ne) doubles (the router rows widened to fp64
//   by the router's own first launch); *launches += the kernels enqueued.
cudaError_t launch_router_topk(const __nv_bfloat16* x, int T, int h, const __nv_bfloat16* wr,
                               int ne, int k, int renorm, int32_t* idx, float* gates,
                               int32_t* tile_counts, double* wr64, int* launches,
                               cudaStream_t st);
size_t router_ws_doubles(int h, int ne);
// Tensor map of a bf16 [rows, cols] row-major array: box_cols (64 -> 128B swizzle, 32 -> 64B
// swizzle) x box_rows, rows past `rows` read as zeros (moe_api.cu).
bool make_tmap_box(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                   uint32_t box_rows);
// Router v7 block 0: SM clock at entry, cycles to the end of compute warp 0's channel loop / to
// exit, exit ns, cycles to the last compute warp's loop end, cycles to the end of the top-k.
cudaError_t router_probe(unsigned long long out[6]);
// Round 1's router kernel (comparison only: tools/router_bench.cu, MOE_ROUTER=3).
cudaError_t launch_router_v3(const __nv_bfloat16* x, int T, int h, const __nv_bfloat16* wr,
                             int ne, int k, int renorm, int32_t* idx, float* gates,
                             int32_t* tile_counts, cudaStream_t st);
// a4 (scan): tile prefix per expert, expert offsets, per-expert counts and GEMM group tables.
//   expert_lo..expert_lo+n_local-1 are the experts whose groups are built (all of them at W=1).
cudaError_t launch_scan(const int32_t* tile_counts, int n_tiles, int ne, int T, int k,
                        int num_shared, int32_t* tile_prefix, int32_t* offsets, int32_t* counts,
                        GemmGroup* grp1, GemmGroup* grp2, cudaStream_t st);
// a4 (permute): stable position of every (t, j) and 16-byte row copies X[t] -> X_perm[pos].
//   pr != NULL (P2P expert parallelism): the row goes straight to its expert owner's x_recv
//   (PeerRows, possibly another GPU's memory) -- permute and dispatch in one kernel; each
//   thread ends with a system-scope fence so a following flag release covers its stores.
cudaError_t launch_permute(const __nv_bfloat16* x, int T, int h, int k, int ne,
                           const int32_t* idx, const int32_t* tile_prefix,
                           const int32_t* offsets, __nv_bfloat16* x_perm, int32_t* pos,
                           const PeerRows* pr, cudaStream_t st);
// a7: out[t] = sum_j g[t,j] * Y[pos[t,j]] + sum_s Y[R + s*stride + t] (+ resid[t] if resid !=
//     NULL) (fp32, fixed order) -> bf16, for the T rows starting at the given pointers (a row
//     range of a call: R = shared_base is then offset by the range's first row, stride = the
//     call's T).  pr != NULL (P2P expert parallelism): routed rows are read from their owners'
//     y_recv (PeerRows; needs idx and offsets), shared rows from y_perm.  shard_t0 >= 0
//     (MOE_FLAG_SHARD_SHARED; num_shared is then ignored): the shared part is the sum, in rank
//     order over pr->shard_mask, of row pr->shard_row + shard_t0 + t of every owner's y_recv.
cudaError_t launch_combine(const __nv_bfloat16* y_perm, const int32_t* pos, const float* gates,
                           int T, int h, int k, int num_shared, int64_t shared_base,
                           int64_t shared_stride, const __nv_bfloat16* resid, __nv_bfloat16* out,
                           const int32_t* idx, const int32_t* offsets, const PeerRows* pr,
                           int shard_t0, cudaStream_t st);
// Task B (b2): u[t] = RMSNorm(h1[t]) * gamma, reading R21:
//   r = 1 / sqrt(sum_c h1[t,c]^2 / h + eps)  (fp64),  n = bf16(float(h1 * r)),
//   u = bf16(float(gamma) * float(n))  (fp32 multiply).
cudaError_t launch_rmsnorm(const __nv_bfloat16* h1, const __nv_bfloat16* gamma, int T, int h,
                           float eps, __nv_bfloat16* u, cudaStream_t st);
// One GEMM group {a_begin, a_end, out_base} written on the stream (device-side group tables are
// how the GEMM learns its rows without a host sync).
cudaError_t launch_fill_group(GemmGroup* g, int a_begin, int a_end, int out_base, cudaStream_t st);
// Groups of the S shared experts (A = the T local tokens): GEMM1 g[n_local + s] =
// {0, T, hbase + s T} (h_act rows), GEMM2 g[n_all + n_local + s] = {hbase + s T, ... + T,
// ybase + s T} (y_perm rows).
cudaError_t launch_fill_shared_groups(GemmGroup* g, int n_local, int n_all, int S, int T,
                                      int hbase, int ybase, cudaStream_t st);

// ---------------------------------------------------------------------------- expert GEMM
enum GemmMode { kGemmSwiGLU = 0, kGemmPlain = 1, kGemmResidual = 2 };
// One launch over a batch of expert groups (GemmBatch: up to kMaxBatch experts whose tiles
// share the persistent CTAs' waves) of a5 (SwiGLU, N = 2*h_i interleaved), a6 (plain, N = h) or
// the O-projection of Task B (residual: out = bf16(A B^T + resid), N = h), on tcgen05.
//   tmA: A [rows, K] bf16 (box 64 x 128); tmB: B [N, K] bf16 (box 64 x bn, or 64 x 128 when
//   `pair`: the CTA-pair kernel, 256 x 256 tiles, bn must be 256).
//   out: bf16 [*, ldo]; SwiGLU writes N/2 columns.  resid: bf16 [*, ldo] (residual mode only,
//   else nullptr), read at the output's rows.
cudaError_t launch_expert_gemm(int mode, int bn, bool pair, const CUtensorMap* tmA,
                               const CUtensorMap* tmB, const GemmBatch& batch, int N, int K,
                               __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid, int grid,
                               cudaStream_t st);
int gemm_bn_for(int mode, int N);   // tile width used for a given mode / N (0 = unsupported)
cudaError_t set_gemm_group_m(int gm);   // raster group override (0 = kernel default; tests)

}  // namespace moe
