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
// part: 0 = every row of each group; 1 = the head (the largest multiple of 256 rows -- whole
// CTA-pair tiles); 2 = the tail (the remaining < 256 rows), so a pair-kernel launch on the head
// and a concurrent 128-row-tile launch on the tail split a group without padding it to 256.
// tail_swap (CTA-pair kernel only): a group's last partial tile of <= 128 rows runs swap-AB
// inside the same launch -- weights as the 256-row M side, the r tail tokens as an N =
// ceil(r/32)*32 side -- instead of a 256-row tile that is mostly padding; those tail tiles are
// scheduled after the full tiles onto the least-loaded CTA pairs, at an estimated `tail_cost`
// (time of a tail tile / time of a full 256x256 tile).
constexpr int kMaxBatch = 16;
constexpr int kPairRows = 256;
struct GemmBatch {
    const GemmGroup* table;
    int32_t idx[kMaxBatch];
    int32_t b_row[kMaxBatch];
    int32_t n;
    int32_t part;
    int32_t tail_swap;
    float tail_cost;
    // select > 0: the host launched BOTH the CTA-pair and the single-CTA kernel for this batch,
    // sized for `select` SMs; each evaluates the same wave model (plan_tiles, gemm.cu) on the
    // ACTUAL group sizes (device memory, no host sync) and the one not chosen exits at once.
    // bn_single: the single-CTA kernel's tile width; alt_ok: the pair launch has PairBMaps.
    int32_t select;
    int32_t bn_single;
    int32_t alt_ok;
    // clk: if non-null, CTA 0 adds its SM cycles (clock64) and elapsed ns (globaltimer) from
    // kernel entry to exit to clk[0] / clk[1] (the SM clock under power management).
    unsigned long long* clk;
    // Stream-K last wave (CTA-pair kernel, streamk != 0): when the full tiles leave a partial
    // last wave of L <= P/2 tiles on P pairs, those L tiles are cut along K into S chunks that
    // run on S*L <= P pairs at once; chunk 0's pair sums the other chunks' fp32 partials
    // (sk_ws: kStreamKUnitFloats per chunk, P chunks) after their per-CTA counters in sk_flags
    // ([P][2], zero between launches) reach S - 1, then runs the usual epilogue.
    int32_t streamk;
    float* sk_ws;
    int* sk_flags;
};
constexpr int64_t kStreamKUnitFloats = 8ll * 256 * 32;   // 256 rows x 256 fp32 columns
// Extra B maps of the CTA-pair kernel: per-CTA boxes of 112 and 96 rows for 224- and 192-wide
// tiles (chosen on the device when N divides and fewer waves result, e.g. 28672 = 128 x 224).
struct PairBMaps {
    CUtensorMap b224, b192;
};

// ------------------------------------------------------------ expert parallelism, P2P transport
constexpr int kMaxRanks = 8;         // EP group size (one B200 box)
// Row buffers of the EP group as seen by one rank (device-resident, rewritten by the plan kernel
// every call): routed row (t, j) of expert e lives in rank e / nl's buffer at row
// base[e] + (pos[t, j] - offsets[e]) -- base[e] is where this rank's block for expert e starts
// in the owner's expert-major layout (moe_ep_plan's recv_off).
struct PeerRows {
    __nv_bfloat16* rows[kMaxRanks];
    int32_t base[kMaxExperts];
    int32_t nl;
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
// and bytes sent (+= bytes_acc).
cudaError_t launch_p2p_plan(const int32_t* counts_par, int W, int ne, int me, int T, int k,
                            int S, long long cap_recv, int n_all, int h, GemmGroup* grp,
                            PeerRows* pr_x, PeerRows* pr_y, int32_t* rows_out,
                            long long* bytes_acc, cudaStream_t st);

// ---------------------------------------------------------------------------- routing kernels
// a2+a3: router GEMM (fp64, ascending c) + warp-shuffle top-k + softmax gates + per-tile counts.
cudaError_t launch_router_topk(const __nv_bfloat16* x, int T, int h, const __nv_bfloat16* wr,
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
// a7: out[t] = sum_j g[t,j] * Y[pos[t,j]] + sum_s Y[R + s*T + t] (+ resid[t] if resid != NULL)
//     (fp32, fixed order) -> bf16.  pr != NULL (P2P expert parallelism): routed rows are read
//     from their owners' y_recv (PeerRows; needs idx and offsets), shared rows from y_perm.
cudaError_t launch_combine(const __nv_bfloat16* y_perm, const int32_t* pos, const float* gates,
                           int T, int h, int k, int num_shared, int64_t shared_base,
                           const __nv_bfloat16* resid, __nv_bfloat16* out,
                           const int32_t* idx, const int32_t* offsets, const PeerRows* pr,
                           cudaStream_t st);
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
// One expert group of a5 (SwiGLU, N = 2*h_i interleaved) or a6 (plain, N = h) on tcgen05, or
// the O-projection of Task B (residual: out = bf16(A B^T + resid), N = h).
//   tmA: A [rows, K] bf16 (box 64 x 128); tmB: B [N, K] bf16 (box 64 x bn, or 64 x 128 when
//   `pair`: the CTA-pair kernel, 256 x 256 tiles, bn must be 256); group: device ptr.
//   out: bf16 [*, ldo]; SwiGLU writes N/2 columns.  resid: bf16 [*, ldo] (residual mode only,
//   else nullptr), read at the output's rows.
//   batch: the launch's expert groups (GemmBatch below): ONE persistent launch covers up to
//   kMaxBatch experts -- their tiles are scheduled together, so small experts no longer pay a
//   partial last wave each.
// Token operand of the swap-AB kernel: the same [rows, K] bf16 tensor with 64-column boxes of
// 128, 64, 32 and 16 rows, so a CTA's N/2 token rows (a multiple of 16) load in <= 4 TMA ops.
struct TokenMaps {
    CUtensorMap box[4];
};
//   tmT: tmA's tensor as TokenMaps -- the token operand of swap-AB tail tiles (pair kernel with
//   batch.tail_swap; may be nullptr otherwise).
cudaError_t launch_expert_gemm(int mode, int bn, bool pair, const CUtensorMap* tmA,
                               const CUtensorMap* tmB, const GemmBatch& batch, int N, int K,
                               __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid, int grid,
                               cudaStream_t st, const TokenMaps* tmT = nullptr,
                               const PairBMaps* alt = nullptr);
// Host model of the pair kernel's schedule (the same rule the kernel applies): the makespan in
// units of one full 256x256 tile time of a launch whose groups have rows[i] rows, N/256 weight
// tiles, on npairs CTA pairs.
double pair_makespan(const int64_t* rows, int n, int n_tiles, int npairs, bool tail_swap,
                     float tail_cost, bool streamk = false, int num_kb = 64);
bool make_token_maps(TokenMaps* t, const void* base, uint64_t rows, uint64_t cols);  // moe_api.cu
// Swap-AB CTA-pair kernel (gemm.cu): weights are the 256-row M side (tmW: box 64 x 128, M rows
// = 2 h_i for SwiGLU, h otherwise, M % 256 == 0), the group's tokens the N side, N = 32..256
// per tile (a multiple of 32).
cudaError_t launch_expert_gemm_swap(int mode, const CUtensorMap* tmW, const TokenMaps* tmX,
                                    const GemmBatch& batch, int M, int K, __nv_bfloat16* out,
                                    int ldo, const __nv_bfloat16* resid, int grid, cudaStream_t st);
int gemm_bn_for(int mode, int N);   // tile width used for a given mode / N (0 = unsupported)
// L2 policy of the GEMM operand loads for the current device: 0 evict_normal, 1 A evict_last +
// B evict_first.
cudaError_t set_gemm_l2_hints(int mode);
cudaError_t set_gemm_group_m(int gm);   // 0 = per-kernel default (MOE_GEMM_GROUPM, experiments)

}  // namespace moe
