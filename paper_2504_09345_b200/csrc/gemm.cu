// gemm.cu -- grouped bf16 expert GEMM on 5th-gen tensor cores (tcgen05 + TMEM), fed by TMA.
//
// One launch computes a batch of expert groups (steps a5 / a6 of the MoE layer; Eq. 1's
// "6 N_k h h_i" FLOPs) -- the experts one coalesced H2D copy brought in, whose
// tiles share the persistent CTAs' waves (GemmBatch):
//   a5 (kGemmSwiGLU): H[r, f] = silu(A W1^T)[r,f] * (A W3^T)[r,f]   with B = packed W13 whose
//                     32-row blocks hold 16 gate rows then the 16 matching up rows, so the
//                     SwiGLU is applied in the epilogue straight out of TMEM;
//   a6 (kGemmPlain):  Y[r, :] = A W2^T;
//   Task B O-projection (kGemmResidual): out = bf16(A Wo^T + resid).
// A rows of each group are [a_begin, a_end) (read from device memory: the routing kernels
// produce them, so no host sync is needed); rows past a_end in the last M tile are computed
// but never stored.  B rows of group i start at GemmBatch::b_row[i] of one tensor map that
// spans every staging slot.
//
// Kernels: expert_gemm_kernel (1 CTA, M = 128), expert_gemm_pair_kernel (CTA pair,
// cta_group::2, M = 256), expert_gemm_swap_kernel (weights as M, tokens as N; experimental).
// Opt-in variants of the pair kernel, each parity-tested and measured (none beat
// the default in-bench): swap-AB tail tiles (GemmBatch::tail_swap), 224/192-wide tiles
// (PairBMaps), device-side choice between the two kernels (GemmBatch::select), stream-K last
// wave (GemmBatch::streamk).  Every launch can report its SM clock (GemmBatch::clk).
// Structure of the first (persistent, one CTA per SM, 256 threads):
//   warp 0     TMA producer: A tile 128x64 and B tile BNx64 per stage, 128B swizzle
//   warp 1     MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16 per instr
//   warp 2     TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-7  epilogue: tcgen05.ld 32x32b -> fp32 math -> bf16 -> global
// Pipelines: smem full/empty mbarriers (TMA <-> MMA), TMEM full/empty (MMA <-> epilogue).
#include <algorithm>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kThreads = 256;

constexpr size_t kBatchReserve = 640;   // shared memory for BatchInfo (below)

template <int BN>
struct GemmCfg {
    static constexpr int kStages = (BN == 256) ? 4 : 6;
    static constexpr uint32_t kABytes = BM * BK * 2;
    static constexpr uint32_t kBBytes = BN * BK * 2;
    static constexpr uint32_t kTmemCols = 2 * BN;
    static constexpr size_t kSmem =
        1024 /*align slack*/ + kStages * (kABytes + kBBytes) + kBatchReserve + 256;
};

// Persistent tile order: groups of `gm` M tiles, M fastest inside a group, then N.  The ~148
// concurrently running tiles then share gm A tiles and ~148/gm B tiles, which stay in L2 (an
// M-fastest order over all M tiles thrashes L2 once m_tiles x A-tile bytes > 126 MB).
__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int gm, int& m,
                                            int& n) {
    const int group = tile / (gm * n_tiles);
    const int first = group * gm;
    const int width = min(gm, m_tiles - first);
    const int r = tile - group * gm * n_tiles;
    m = first + r % width;
    n = r / width;
}

// L2 policies of the operand loads (MOE_GEMM_L2HINT: 0 = evict_normal for both, 1 = A evict_last
// + B evict_first).  Set once per process by set_gemm_l2_hints().
__device__ int g_l2_hints = 0;
__device__ int g_group_m = 0;  // raster group override (0 = kernel default); experiments only

__device__ __forceinline__ uint64_t l2_policy_a() {
    return g_l2_hints ? ptx::policy_evict_last() : ptx::policy_evict_normal();
}
__device__ __forceinline__ uint64_t l2_policy_b() {
    return g_l2_hints ? ptx::policy_evict_first() : ptx::policy_evict_normal();
}

// SM clock probe (GemmBatch::clk): thread 0 of CTA 0 samples at entry and adds at exit.
struct ClkProbe {
    uint64_t c0 = 0, t0 = 0;
    __device__ __forceinline__ void start(const GemmBatch& b) {
        if (b.clk && blockIdx.x == 0 && threadIdx.x == 0) {
            t0 = ptx::globaltimer_ns();
            c0 = clock64();
        }
    }
    __device__ __forceinline__ void stop(const GemmBatch& b) {
        if (b.clk && blockIdx.x == 0 && threadIdx.x == 0) {
            const uint64_t c1 = clock64(), t1 = ptx::globaltimer_ns();
            atomicAdd(b.clk, (unsigned long long)(c1 - c0));
            atomicAdd(b.clk + 1, (unsigned long long)(t1 - t0));
        }
    }
};

__device__ __forceinline__ float silu_mul(float g, float u) {
    return g / (1.0f + __expf(-g)) * u;
}

// Epilogue of one accumulator row (this thread's TMEM lane): TMEM -> registers -> fp32 math ->
// bf16 -> global.  SwiGLU tiles hold gate columns [0, BN/2) and the matching up columns
// [BN/2, BN); they produce BN/2 outputs.  tcgen05.ld is warp-collective: every lane loads, only
// rows inside the group store.
template <int MODE>
__device__ __forceinline__ void epilogue_row(uint32_t taddr, bool valid, __nv_bfloat16* row_out,
                                             const __nv_bfloat16* row_res, int n, int BN) {
    if (MODE == kGemmSwiGLU) {
        // packed W13 (moe_pack_expert): 32-column blocks = 16 gate columns, then the 16 matching
        // up columns -> 16 output features per 32 accumulator columns
        __nv_bfloat16* dst = row_out + (int64_t)n * (BN / 2);
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(taddr + c, v);
            ptx::tmem_ld_wait();
            if (valid) {
                uint32_t pk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float h0 = silu_mul(__uint_as_float(v[2 * i]), __uint_as_float(v[16 + 2 * i]));
                    const float h1 = silu_mul(__uint_as_float(v[2 * i + 1]), __uint_as_float(v[17 + 2 * i]));
                    pk[i] = ptx::pack_bf16x2(h0, h1);
                }
                ptx::st_global_v4(dst + c / 2, pk[0], pk[1], pk[2], pk[3]);
                ptx::st_global_v4(dst + c / 2 + 8, pk[4], pk[5], pk[6], pk[7]);
            }
        }
    } else {
        __nv_bfloat16* dst = row_out + (int64_t)n * BN;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(taddr + c, v);
            ptx::tmem_ld_wait();
            if (valid) {
                if (MODE == kGemmResidual) {  // + residual row, one rounding (reading R20)
                    const __nv_bfloat16* src = row_res + (int64_t)n * BN + c;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int4 r = ptx::ld_nc_v4(src + 8 * i);
                        const uint32_t rw[4] = {(uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            v[8 * i + 2 * j] = __float_as_uint(__uint_as_float(v[8 * i + 2 * j]) +
                                                               __uint_as_float(rw[j] << 16));
                            v[8 * i + 2 * j + 1] = __float_as_uint(
                                __uint_as_float(v[8 * i + 2 * j + 1]) + __uint_as_float(rw[j] & 0xffff0000u));
                        }
                    }
                }
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    pk[i] = ptx::pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    ptx::st_global_v4(dst + c + 8 * i, pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
            }
        }
    }
}

// The groups of one launch (up to kMaxBatch experts whose weights sit in different staging slots
// of one tensor map), resolved once per CTA into shared memory: global tile t belongs to group
// g with first[g] <= t < first[g + 1]; inside a group tiles follow tile_coords().
// With tail swap (pair kernel): a group whose last partial tile has r <= 128 rows has m_tiles =
// rows / 256 full tiles plus n_tiles swap-AB tail tiles of tail_nc = ceil(r/32)*32 token columns;
// the tail tiles of all such groups are numbered after the full tiles (TailSched below).
struct BatchInfo {
    int n, total, n_tail_grp, plan;
    int sk_L, sk_S;            // stream-K: the last sk_L full tiles run as sk_S K-chunks each
    int first[kMaxBatch + 1];
    int m_tiles[kMaxBatch];
    int a_begin[kMaxBatch], a_end[kMaxBatch], out_base[kMaxBatch], b_row[kMaxBatch];
    int tail_nc[kMaxBatch];
    int tail_grp[kMaxBatch];   // groups with a swap tail, last group first
};
constexpr size_t kBatchSmem = (sizeof(BatchInfo) + 15) & ~size_t(15);
static_assert(kBatchSmem <= kBatchReserve, "BatchInfo does not fit its reservation");

// Tail rule shared by the kernel and the host model: rows of a group -> full 256-row tiles and
// the swap-tail width (0 = no swap tail; the partial tile, if any, is an ordinary padded tile).
__host__ __device__ __forceinline__ int tail_cols(int rows, bool tail_swap) {
    const int rem = rows % kPairRows;
    return (tail_swap && rem > 0 && rem <= 128) ? ((rem + 31) & ~31) : 0;
}

// Row ranges of the launch's groups (after the tail-split `part` cut), no tiling yet.
__device__ __forceinline__ void batch_load(BatchInfo* bi, const GemmBatch& b) {
    for (int i = 0; i < b.n; ++i) {
        GemmGroup g = b.table[b.idx[i]];
        const int head = (max(0, g.a_end - g.a_begin) / kPairRows) * kPairRows;
        if (b.part == 1) {          // whole 256-row tiles only
            g.a_end = g.a_begin + head;
        } else if (b.part == 2) {   // the remainder
            g.a_begin += head;
            g.out_base += head;
        }
        bi->a_begin[i] = g.a_begin;
        bi->a_end[i] = max(g.a_begin, g.a_end);
        bi->out_base[i] = g.out_base;
        bi->b_row[i] = b.b_row[i];
    }
    bi->n = b.n;
}

// Tiles of bm rows x n_tiles weight tiles per group, numbered group after group.
__device__ __forceinline__ void batch_tiles(BatchInfo* bi, int bm, int n_tiles, bool tail_swap) {
    int t = 0;
    for (int i = 0; i < bi->n; ++i) {
        const int rows = bi->a_end[i] - bi->a_begin[i];
        bi->tail_nc[i] = tail_cols(rows, tail_swap);
        bi->m_tiles[i] = bi->tail_nc[i] ? rows / bm : (rows + bm - 1) / bm;
        bi->first[i] = t;
        t += bi->m_tiles[i] * n_tiles;
    }
    bi->first[bi->n] = t;
    bi->total = t;
    bi->sk_L = 0;
    bi->sk_S = 1;
    int nt = 0;
    for (int i = bi->n - 1; i >= 0; --i)
        if (bi->tail_nc[i]) bi->tail_grp[nt++] = i;
    bi->n_tail_grp = nt;
}

// Stream-K plan of the pair kernel's partial last wave (GemmBatch::streamk; the host model in
// pair_makespan mirrors it): F full tiles on P pairs leave L = F % P tiles for a last wave in
// which P - L pairs would idle.  If F > P and 0 < L <= P / 2, each of those L tiles is cut into
// S = the largest power of two <= min(P / L, 4) that divides num_kb (S >= 2) K-chunks.
__host__ __device__ __forceinline__ void streamk_plan(int F, int P, int num_kb, int& L, int& S) {
    L = 0;
    S = 1;
    if (F <= P) return;
    const int l = F % P;
    if (l == 0 || l > P / 2) return;
    int s2 = 1;   // at most 4 chunks: the owner's read of the others' partials stays short
    while (s2 * 2 <= P / l && s2 * 2 <= 4 && num_kb % (s2 * 2) == 0) s2 *= 2;
    if (s2 < 2) return;
    L = l;
    S = s2;
}

__device__ __forceinline__ void batch_init(BatchInfo* bi, const GemmBatch& b, int bm,
                                           int n_tiles, bool tail_swap = false) {
    batch_load(bi, b);
    batch_tiles(bi, bm, n_tiles, tail_swap);
}

// Tile shape of a launch from the ACTUAL group sizes (both kernels evaluate it identically; see
// GemmBatch::select): wave model time ~ ceil(tiles / concurrent tiles) x tile width / tensor
// efficiency -- single-CTA 128 x bn_single tiles at 0.76 (shared-memory bound), CTA-pair
// 256 x BN tiles at 0.97, BN in {256, 224, 192} where N % BN == 0.  Returns 0 (single-CTA
// kernel) or the pair tile width; -1 if there is no work.
__device__ __forceinline__ int plan_tiles(const BatchInfo* bi, int N, int sms, int bn_single,
                                          bool allow_single, bool allow_pair, bool alt_maps) {
    int rows128 = 0, rows256 = 0;
    for (int i = 0; i < bi->n; ++i) {
        const int r = bi->a_end[i] - bi->a_begin[i];
        rows128 += (r + 127) / 128;
        rows256 += (r + 255) / 256;
    }
    if (rows128 == 0) return -1;
    int choice = -1;
    float best = 3.0e38f;
    if (allow_single && bn_single > 0) {
        const int t = rows128 * (N / bn_single), conc = sms;
        best = (float)((t + conc - 1) / conc) * ((float)bn_single / 256.f) / 0.76f;
        choice = 0;
    }
    if (allow_pair) {
        const int conc = sms / 2;
        for (int bn = 256; bn >= 192; bn -= 32) {
            if (N % bn || (bn != 256 && !alt_maps)) continue;
            const int t = rows256 * (N / bn);
            const float w = (float)((t + conc - 1) / conc) * ((float)bn / 256.f) / 0.97f;
            if (w < best * 0.999f) {
                best = w;
                choice = bn;
            }
        }
    }
    return choice;
}

__device__ __forceinline__ int batch_locate(const BatchInfo* bi, int tile, int& local) {
    int g = 0;
    while (tile >= bi->first[g + 1]) ++g;
    local = tile - bi->first[g];
    return g;
}

// Static schedule of the pair kernel (every thread of every CTA computes it identically, so no
// tile queue is needed): full tile t goes to pair t % P -- pair p has q = F / P full tiles, plus
// one more if p < r = F % P -- then the R tail tiles (cost c each, in full-tile units) are dealt
// out in rounds in order of the time a round would finish: a "light" round gives one tail to each
// pair p >= r (done at q + c*(i+1)), a "heavy" round one to each pair p < r (q + 1 + c*(i+1)).
// This is greedy least-loaded assignment for two load classes; next() yields pair p's tails.
struct TailSched {
    int R, p, q, r, nl, nh, j, li, hi;
    float c;
    __host__ __device__ void init(int F, int R_, int P, int p_, float c_) {
        R = R_; p = p_; q = F / P; r = F % P; nl = P - r; nh = r; j = 0; li = 0; hi = 0; c = c_;
    }
    __host__ __device__ bool next(int& tj) {
        while (j < R) {
            const float tl = q + c * (li + 1);
            const float th = nh ? q + 1 + c * (hi + 1) : 3.0e38f;
            const int base = j;
            if (tl <= th) {
                j += nl; ++li;
                if (p >= r && base + (p - r) < R) { tj = base + (p - r); return true; }
            } else {
                j += nh; ++hi;
                if (p < r && base + p < R) { tj = base + p; return true; }
            }
        }
        return false;
    }
};

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
expert_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ GemmBatch batch, int N, int K,
                   __nv_bfloat16* __restrict__ out, int ldo,
                   const __nv_bfloat16* __restrict__ resid) {
    using C = GemmCfg<BN>;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * C::kABytes;
    BatchInfo* bi = reinterpret_cast<BatchInfo*>(sB + S * C::kBBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(bi) + kBatchSmem);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int n_tiles = N / BN;
    ClkProbe clk;
    clk.start(batch);
    if (threadIdx.x == 0) {
        batch_init(bi, batch, BM, n_tiles);
        bi->plan = batch.select ? plan_tiles(bi, N, batch.select, BN, true, true, batch.alt_ok != 0) : 0;
    }
    __syncthreads();
    if (bi->plan != 0) return;                   // the CTA-pair kernel of this launch runs it
    const int total = bi->total;
    if ((int)blockIdx.x >= total) return;
    const int num_kb = K / BK;
    // rows per raster group: A footprint ~32 MB (measured at 65k tokens, K=4096: group 16 ->
    // 2.0 GB DRAM per launch, group 32 -> 1.08 GB; the weight tiles are re-read once per group)
    const int group_m = g_group_m > 0 ? g_group_m : ((K <= 8192) ? 32 : 8);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 4);
        }
        ptx::fence_barrier_init();
        ptx::fence_proxy_async();
    }
    if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            const uint64_t pol_a = l2_policy_a();  // A tile re-read by every N tile of the group
            const uint64_t pol_b = l2_policy_b();  // weight tile: read by the group's M tiles
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
                int m, n, local;
                const int gi = batch_locate(bi, tile, local);
                tile_coords(local, bi->m_tiles[gi], n_tiles, group_m, m, n);
                const int arow = bi->a_begin[gi] + m * BM, brow = bi->b_row[gi] + n * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1u);
                    ptx::mbar_arrive_expect_tx(&full[stage], C::kABytes + C::kBBytes);
                    ptx::tma_load_2d_hint(sA + stage * C::kABytes, &tmA, &full[stage], kb * BK,
                                          arow, pol_a);
                    ptx::tma_load_2d_hint(sB + stage * C::kBBytes, &tmB, &full[stage], kb * BK,
                                          brow, pol_b);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = ptx::umma_idesc_bf16(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], aphase ^ 1u);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(sA + stage * C::kABytes);
                    const uint32_t b0 = ptx::smem_u32(sB + stage * C::kBBytes);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const uint64_t ad = ptx::umma_desc_sw128_kmajor(a0 + kk * 32);
                        const uint64_t bd = ptx::umma_desc_sw128_kmajor(b0 + kk * 32);
                        ptx::umma_bf16(d, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                    }
                    ptx::umma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                ptx::umma_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- epilogue
        const int q = warp - 4;  // TMEM lane quadrant (warp % 4)
        int it = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            int m, n, local;
            const int gi = batch_locate(bi, tile, local);
            tile_coords(local, bi->m_tiles[gi], n_tiles, group_m, m, n);
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const int r = q * 32 + lane;
            const int arow = bi->a_begin[gi] + m * BM + r;
            const bool valid = arow < bi->a_end[gi];
            const int64_t orow = (int64_t)bi->out_base[gi] + (arow - bi->a_begin[gi]);
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
            epilogue_row<MODE>(taddr, valid, out + orow * ldo,
                               resid ? resid + orow * ldo : nullptr, n, BN);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
    clk.stop(batch);
}

// ------------------------------------------------------------------------------------------
// Swap-AB CTA-pair variant: D^T = W X^T.  The weights are the M side (a 256-row pair tile: 128
// rows per CTA, the same operand maps as the pair kernel's B), the group's tokens the N side:
// tcgen05 takes N = 16..256 in steps of 16 at run time, so a group of R rows costs
// ceil(R/32)*32 columns instead of ceil(R/256)*256 rows (C1: 1053 rows -> 1056 instead of 1280).
// Tiles are handed out round-robin over a grouped raster (SwapRR).
// Token rows are loaded in 16-row TMA boxes (a CTA holds N/2 of them).  The epilogue transposes
// through shared memory: TMEM lane = weight row (feature), column = token.
constexpr int kSwapStages = 6;
constexpr uint32_t kSwapABytes = 128 * BK * 2;      // per CTA: 128 weight rows
constexpr uint32_t kSwapBBytes = 128 * BK * 2;      // per CTA: up to 128 token rows
constexpr uint32_t kSwapEpiBytes = 4 * 32 * 33 * 4;  // per-warp transpose tiles (4 warps)
constexpr size_t kSwapSmem = 1024 + kSwapStages * (kSwapABytes + kSwapBBytes) + kSwapEpiBytes + 256;

// Round-robin tile order (tile t -> pair t % npairs) over a grouped raster: the token columns of
// a group are cut into nck near-equal chunks (<= 256 columns, multiples of 32); chunk groups of
// kSwapGroup chunks (<= 4096 tokens, ~33 MB at K = 4096) are the outer loop, weight tiles next,
// chunks innermost -- so the ~74 tiles in flight share a few weight tiles and one token group
// in L2.  (A contiguous-range-per-pair split balances work better but re-reads each weight tile
// once per chunk from DRAM: 4.5x the traffic at C1, measured.)
constexpr int kSwapGroup = 16;
struct SwapRR {
    int nck, ucols, extra, m_tiles, total, t, step, grp;
    __device__ __forceinline__ void init(int rows, int m_tiles_, int pair, int npairs) {
        grp = g_group_m > 0 ? g_group_m : kSwapGroup;
        const int upm = (rows + 31) >> 5;
        nck = (upm + 7) / 8;
        ucols = upm / nck;               // units per chunk (the first `extra` get one more)
        extra = upm % nck;
        m_tiles = m_tiles_;
        total = m_tiles * nck;
        t = pair;
        step = npairs;
    }
    __device__ __forceinline__ bool next(int& m, int& col, int& ncols) {
        if (t >= total) return false;
        const int per_group = grp * m_tiles;
        const int gidx = t / per_group, r = t % per_group;
        const int gsize = min(grp, nck - gidx * grp);
        m = r / gsize;
        const int ck = gidx * grp + r % gsize;
        col = 32 * (ck * ucols + min(ck, extra));
        ncols = 32 * (ucols + (ck < extra ? 1 : 0));
        t += step;
        return true;
    }
    __device__ __forceinline__ bool empty() const { return t >= total; }
};

// Epilogue of one swap tile, one warp (TMEM lane quadrant): 32 token columns at a time, TMEM ->
// registers -> the warp's own smem tile `wt` (32 x 33 fp32; __syncwarp only) -> 16-byte global
// stores.  fcol: first output feature of the warp's 32 lanes
//   SwiGLU: the quadrant's 32 weight rows are 16 gate rows then the 16 matching up rows
//           (moe_pack_expert's 16-row blocks) -> 16 output features;
//   Plain / Residual: 32 output features.
template <int MODE>
__device__ __forceinline__ void swap_epilogue(uint32_t taddr, int lane, int ncols, int tok0,
                                              int rows, int64_t orow0, __nv_bfloat16* out,
                                              int ldo, int fcol, const __nv_bfloat16* resid,
                                              float* wt) {
#pragma unroll 1
    for (int c = 0; c < ncols; c += 32) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(taddr + c, v);
        ptx::tmem_ld_wait();
        if (MODE == kGemmSwiGLU) {
            // lane l < 16: gate row of feature f = fcol + l; lane l + 16: the matching up row.
            // One xor-16 shuffle per pair: the gate lane finishes tokens c..c+15, the up lane
            // tokens c+16..c+31 of the same feature.
            // The results are transposed through the warp's smem tile (token-major, padded) so
            // each lane then writes one token's 16 features as two 16-byte stores.
            // Staged as bf16 (the output precision; one rounding either way) in rows of 18
            // elements: conflict-free 2-byte writes and 4-byte reads, half the smem traffic of
            // fp32 staging (this kernel is shared-memory-bandwidth sensitive).
            const bool up = lane >= 16;
            const int fl = lane & 15;
            __nv_bfloat16* wb = reinterpret_cast<__nv_bfloat16*>(wt);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float mine = __uint_as_float(up ? v[j] : v[16 + j]);
                const float x = __shfl_xor_sync(0xffffffffu, mine, 16);
                const float hv = up ? silu_mul(x, __uint_as_float(v[16 + j]))
                                    : silu_mul(__uint_as_float(v[j]), x);
                wb[(j + (up ? 16 : 0)) * 18 + fl] = __float2bfloat16_rn(hv);
            }
            __syncwarp();
            if (tok0 + c + lane < rows) {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(wb + lane * 18);
                uint32_t pk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) pk[i] = src[i];
                __nv_bfloat16* dst = out + (orow0 + c + lane) * ldo + fcol;
                ptx::st_global_v4(dst, pk[0], pk[1], pk[2], pk[3]);
                ptx::st_global_v4(dst + 8, pk[4], pk[5], pk[6], pk[7]);
            }
            __syncwarp();
        } else if (MODE == kGemmPlain) {
            // lane = output feature fcol + lane; transpose through the warp's smem tile (bf16,
            // rows of 34 elements) so each lane owns one token's 32 features: four 16-B stores.
            __nv_bfloat16* wb = reinterpret_cast<__nv_bfloat16*>(wt);
#pragma unroll
            for (int j = 0; j < 32; ++j) wb[j * 34 + lane] = __float2bfloat16_rn(__uint_as_float(v[j]));
            __syncwarp();
            if (tok0 + c + lane < rows) {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(wb + lane * 34);
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) pk[i] = src[i];
                __nv_bfloat16* dst = out + (orow0 + c + lane) * ldo + fcol;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    ptx::st_global_v4(dst + 8 * i, pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
            }
            __syncwarp();
        } else {
            // residual mode: fp32 staging so the residual is added before the single rounding
#pragma unroll
            for (int j = 0; j < 32; ++j) wt[j * 33 + lane] = __uint_as_float(v[j]);
            __syncwarp();
            if (tok0 + c + lane < rows) {
                const float* src = wt + lane * 33;
                const int64_t off = (orow0 + c + lane) * ldo + fcol;
                float f[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) f[i] = src[i];
                if (MODE == kGemmResidual) {   // + residual, one rounding (reading R20)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int4 r = ptx::ld_nc_v4(resid + off + 8 * i);
                        const uint32_t rw[4] = {(uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            f[8 * i + 2 * q] += __uint_as_float(rw[q] << 16);
                            f[8 * i + 2 * q + 1] += __uint_as_float(rw[q] & 0xffff0000u);
                        }
                    }
                }
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) pk[i] = ptx::pack_bf16x2(f[2 * i], f[2 * i + 1]);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    ptx::st_global_v4(out + off + 8 * i, pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
            }
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes 256 x 256 tiles.
// Each CTA stages its own 128 rows of A and half (128 rows) of the B tile per K step (32 KB, 6
// stages), the leader issues tcgen05.mma.cta_group::2 (M=256) reading both CTAs' smem, and each
// CTA's TMEM holds its 128 rows of the fp32 accumulator.  Per SM this halves the B bytes moved
// per MMA and doubles the bytes in flight (6 x 32 KB vs 4 x 48 KB), for large expert groups.
// Barrier protocol: full[s] (leader; arrivals: leader expect_tx + peer remote arrive; TMA bytes
// of both CTAs), empty[s] (both; MMA commit multicast), tfull[a] (both; multicast), tempty[a]
// (leader; 4 epilogue warps x 2 CTAs).
// Tail swap (batch.tail_swap): a group's last partial tile of r <= 128 rows is a swap-AB tile
// instead -- the stage's B buffer takes the weight tile exactly as for a full tile, the A buffer
// only the r tail tokens (nc/2 rows per CTA, nc = ceil(r/32)*32), and the leader issues
// D^T[256 x nc] = W X^T with the operand descriptors swapped, so the tile moves ~half the bytes
// and does nc/256 of the MMA work of a padded 256-row tile.  Its epilogue (TMEM lane = weight row)
// transposes through shared memory (swap_epilogue).  Schedule: TailSched.
constexpr int kPairStages = 6;
constexpr uint32_t kPairABytes = 128 * BK * 2;   // per CTA
constexpr uint32_t kPairBBytes = 128 * BK * 2;   // per CTA (half of a 256-row B tile)
constexpr size_t kPairSmem =
    1024 + kPairStages * (kPairABytes + kPairBBytes) + kSwapEpiBytes + kBatchReserve + 256;

// One tile of the pair kernel's sequence: a full (or padded) 256 x BN tile (nc == 0) of group gi
// at M tile m, weight tile n, over k-blocks [kb0, kb1); or a swap tail (nc > 0): token columns
// [m*256, m*256 + nc).  Stream-K chunks have unit >= 0: split tile lidx, chunk `chunk`.
struct PairTile {
    int gi, m, n, nc, kb0, kb1, unit, chunk, lidx;
};
struct PairSched {
    int t, P, Ffull, n_tiles, group_m, num_kb, pair, L, S;
    bool unit_done;
    TailSched ts;
    __device__ __forceinline__ void init(const BatchInfo* bi, int pair_, int npairs, int nt,
                                         int gm, float cost, int nkb) {
        t = pair_; P = npairs; n_tiles = nt; group_m = gm; num_kb = nkb; pair = pair_;
        L = bi->sk_L; S = bi->sk_S;
        Ffull = bi->total - L;
        unit_done = false;
        ts.init(bi->total, bi->n_tail_grp * nt, npairs, pair_, cost);
    }
    __device__ __forceinline__ void coords(const BatchInfo* bi, int tile, PairTile& o) const {
        int local;
        o.gi = batch_locate(bi, tile, local);
        tile_coords(local, bi->m_tiles[o.gi], n_tiles, group_m, o.m, o.n);
    }
    __device__ __forceinline__ bool next(const BatchInfo* bi, PairTile& o) {
        o.nc = 0; o.kb0 = 0; o.kb1 = num_kb; o.unit = -1; o.chunk = 0; o.lidx = 0;
        if (t < Ffull) {
            coords(bi, t, o);
            t += P;
            return true;
        }
        if (!unit_done && pair < L * S) {   // this pair's stream-K chunk (one per pair at most)
            unit_done = true;
            o.unit = pair;
            o.lidx = pair / S;
            o.chunk = pair % S;
            coords(bi, Ffull + o.lidx, o);
            const int per = num_kb / S;
            o.kb0 = o.chunk * per;
            o.kb1 = o.kb0 + per;
            return true;
        }
        int tj;
        if (!ts.next(tj)) return false;
        o.gi = bi->tail_grp[tj / n_tiles];
        o.n = n_tiles - 1 - tj % n_tiles;     // descending: the most recently used weights first
        o.m = bi->m_tiles[o.gi];
        o.nc = bi->tail_nc[o.gi];
        return true;
    }
};

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
expert_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ TokenMaps tmT,
                        const __grid_constant__ PairBMaps tmAlt,
                        const __grid_constant__ GemmBatch batch, int N, int K,
                        __nv_bfloat16* __restrict__ out, int ldo,
                        const __nv_bfloat16* __restrict__ resid) {
    constexpr int PM = 256, S = kPairStages, kAccCols = 256;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * kPairABytes;
    float* sE = reinterpret_cast<float*>(sB + S * kPairBBytes);
    BatchInfo* bi = reinterpret_cast<BatchInfo*>(sB + S * kPairBBytes + kSwapEpiBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(bi) + kBatchSmem);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    ClkProbe clk;
    clk.start(batch);
    if (threadIdx.x == 0) {
        batch_load(bi, batch);
        // tile width: 256, or 224 / 192 when that needs fewer waves; 0 = the single-CTA kernel
        // of this launch runs it (select), -1 = nothing to do
        const int plan = batch.select
            ? plan_tiles(bi, N, batch.select, batch.bn_single, true, true, batch.alt_ok != 0)
            : plan_tiles(bi, N, gridDim.x, 0, false, true, batch.alt_ok != 0);
        bi->plan = plan;
        if (plan > 0) {
            const bool tails = batch.tail_swap != 0 && plan == 256;
            batch_tiles(bi, PM, N / plan, tails);
            if (batch.streamk && !tails && batch.sk_ws && batch.sk_flags)
                streamk_plan(bi->total, (int)gridDim.x / 2, K / BK, bi->sk_L, bi->sk_S);
        }
    }
    __syncthreads();
    if (bi->plan <= 0) return;                   // uniform over the grid
    const int BN = bi->plan;
    const int n_tiles = N / BN;
    const CUtensorMap* mB = BN == 256 ? &tmB : (BN == 224 ? &tmAlt.b224 : &tmAlt.b192);
    const int num_kb = K / BK;
    const int group_m = g_group_m > 0 ? g_group_m : ((K <= 8192) ? 16 : 4);  // 256-row tiles
    PairSched sched0;
    sched0.init(bi, pair, npairs, n_tiles, group_m, batch.tail_cost, num_kb);
    {
        PairSched probe = sched0;
        PairTile pt;
        if (!probe.next(bi, pt)) return;         // identical in both CTAs: the pair leaves together
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(mB);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 2);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 8);
        }
        ptx::fence_barrier_init();
        ptx::fence_proxy_async();
    }
    if (warp == 2) ptx::tmem_alloc_cta2<2 * kAccCols>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------------------------------------------- TMA producer (both CTAs)
            const uint64_t pol_a = l2_policy_a();
            const uint64_t pol_b = l2_policy_b();
            const uint32_t full0 = ptx::mapa_shared(&full[0], 0);  // leader's full[0]
            int stage = 0;
            uint32_t phase = 0;
            PairSched sc = sched0;
            PairTile pt;
            while (sc.next(bi, pt)) {
                const int brow = bi->b_row[pt.gi] + pt.n * BN + (int)rank * (BN / 2);
                const int half = pt.nc >> 1;   // swap tail: token rows of this CTA
                const int arow = bi->a_begin[pt.gi] + pt.m * PM + (int)rank * (pt.nc ? half : 128);
                const uint32_t tx = pt.nc ? 2 * kPairBBytes + (uint32_t)pt.nc * BK * 2
                                          : 2 * kPairABytes + (uint32_t)BN * BK * 2;
                for (int kb = pt.kb0; kb < pt.kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1u);
                    const uint32_t fbar = full0 + stage * 8;
                    if (leader) ptx::mbar_arrive_expect_tx(&full[stage], tx);
                    else ptx::mbar_arrive_cluster(fbar);
                    ptx::tma_load_2d_cta2(sB + stage * kPairBBytes, mB, fbar, kb * BK, brow, pol_b);
                    if (!pt.nc) {
                        ptx::tma_load_2d_cta2(sA + stage * kPairABytes, &tmA, fbar, kb * BK, arow, pol_a);
                    } else {
                        uint8_t* a = sA + stage * kPairABytes;
                        for (int i = 1, r = 0; i < 4; ++i) {   // boxes of 64, 32, 16 rows
                            const int box = 128 >> i;
                            if (half - r >= box) {
                                ptx::tma_load_2d_cta2(a + r * (BK * 2), &tmT.box[i], fbar, kb * BK,
                                                      arow + r, pol_a);
                                r += box;
                            }
                        }
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            // ---------------------------------------------------- MMA issuer (leader only)
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            PairSched sc = sched0;
            PairTile pt;
            while (sc.next(bi, pt)) {
                const uint32_t idesc = ptx::umma_idesc_bf16(PM, pt.nc ? (uint32_t)pt.nc : (uint32_t)BN);
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], aphase ^ 1u);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * kAccCols;
                for (int kb = pt.kb0; kb < pt.kb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(sA + stage * kPairABytes);
                    const uint32_t b0 = ptx::smem_u32(sB + stage * kPairBBytes);
                    // swap tail: the weights (B buffer) are the MMA's A operand
                    const uint32_t x0 = pt.nc ? b0 : a0, y0 = pt.nc ? a0 : b0;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        ptx::umma_bf16_cta2(d, ptx::umma_desc_sw128_kmajor(x0 + kk * 32),
                                            ptx::umma_desc_sw128_kmajor(y0 + kk * 32), idesc,
                                            (kb != pt.kb0 || kk != 0) ? 1u : 0u);
                    ptx::umma_commit_cta2_mc(&empty[stage], 0x3);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                ptx::umma_commit_cta2_mc(&tfull[acc], 0x3);
                ++it;
            }
        }
    } else if (warp >= 4) {
        // -------------------------------------------------------- epilogue (both CTAs)
        const int q = warp - 4;
        const uint32_t tempty0 = ptx::mapa_shared(&tempty[0], 0);
        int it = 0;
        PairSched sc = sched0;
        PairTile pt;
        while (sc.next(bi, pt)) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kAccCols;
            const int gi = pt.gi;
            if (pt.unit >= 0 && pt.chunk != 0) {
                // stream-K chunk: fp32 partial of this CTA's 128 rows -> sk_ws, then count it
                const int row = (int)rank * 128 + q * 32 + lane;
                float* ws = batch.sk_ws + (int64_t)pt.unit * kStreamKUnitFloats;
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(taddr + c, v);
                    ptx::tmem_ld_wait();
                    float4* dst = reinterpret_cast<float4*>(ws + ((int64_t)(c / 32) * 256 + row) * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
                ptx::named_bar_sync(1, 128);
                if (q == 0 && lane == 0) {
                    __threadfence();
                    ptx::red_release_gpu_add(batch.sk_flags + pt.lidx * 2 + (int)rank, 1);
                }
            } else if (!pt.nc) {
                if (pt.unit >= 0) {
                    // stream-K owner (chunk 0): wait for the other S-1 chunks' partials of these
                    // rows, add them into the TMEM accumulator, then the usual epilogue
                    const int S = bi->sk_S;
                    int* flag = batch.sk_flags + pt.lidx * 2 + (int)rank;
                    if (q == 0 && lane == 0)
                        while (ptx::ld_acquire_gpu(flag) < S - 1) __nanosleep(64);
                    ptx::named_bar_sync(1, 128);
                    const int row = (int)rank * 128 + q * 32 + lane;
#pragma unroll 1
                    for (int c = 0; c < BN; c += 32) {
                        uint32_t v[32];
                        ptx::tmem_ld_32x32b_x32(taddr + c, v);
                        ptx::tmem_ld_wait();
                        // all (S-1) x 8 loads of this 32-column chunk in flight at once; fixed
                        // summation order (chunk 1, 2, 3) keeps the result deterministic
                        const float4* src = reinterpret_cast<const float4*>(
                            batch.sk_ws + (int64_t)pt.unit * kStreamKUnitFloats +
                            ((int64_t)(c / 32) * 256 + row) * 32);
                        constexpr int64_t kUnit4 = kStreamKUnitFloats / 4;
                        float4 p4[3][8];
#pragma unroll
                        for (int sc = 1; sc < 4; ++sc)
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                p4[sc - 1][i] = sc < S ? __ldcg(src + sc * kUnit4 + i)
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float4 a = p4[0][i], b = p4[1][i], d4 = p4[2][i];
                            v[4 * i] = __float_as_uint(__uint_as_float(v[4 * i]) + ((a.x + b.x) + d4.x));
                            v[4 * i + 1] = __float_as_uint(__uint_as_float(v[4 * i + 1]) + ((a.y + b.y) + d4.y));
                            v[4 * i + 2] = __float_as_uint(__uint_as_float(v[4 * i + 2]) + ((a.z + b.z) + d4.z));
                            v[4 * i + 3] = __float_as_uint(__uint_as_float(v[4 * i + 3]) + ((a.w + b.w) + d4.w));
                        }
                        ptx::tmem_st_32x32b_x32(taddr + c, v);
                    }
                    ptx::tmem_st_wait();
                    if (q == 0 && lane == 0) *flag = 0;   // ready for the next launch
                }
                const int arow = bi->a_begin[gi] + pt.m * PM + (int)rank * 128 + q * 32 + lane;
                const bool valid = arow < bi->a_end[gi];
                const int64_t orow = (int64_t)bi->out_base[gi] + (arow - bi->a_begin[gi]);
                epilogue_row<MODE>(taddr, valid, out + orow * ldo,
                                   resid ? resid + orow * ldo : nullptr, pt.n, BN);
            } else {
                // TMEM lane = weight row n*256 + rank*128 + q*32 + lane, column = tail token
                const int tok0 = pt.m * PM;
                const int fcol = (MODE == kGemmSwiGLU) ? pt.n * 128 + (int)rank * 64 + q * 16
                                                       : pt.n * 256 + (int)rank * 128 + q * 32;
                swap_epilogue<MODE>(taddr, lane, pt.nc, tok0, bi->a_end[gi] - bi->a_begin[gi],
                                    (int64_t)bi->out_base[gi] + tok0, out, ldo, fcol, resid,
                                    sE + q * (32 * 33));
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + acc * 8);
            ++it;
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_cta2<2 * kAccCols>(tmem_base);
    }
    clk.stop(batch);
}

// tmW: weights [M, K] (box 64 x 128); tmX: group tokens [*, K] (TokenMaps); M = 2 h_i (SwiGLU)
// or h (plain / residual).  out: [*, ldo], SwiGLU writes M/2 columns.
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
expert_gemm_swap_kernel(const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ TokenMaps tmX,
                        const __grid_constant__ GemmBatch batch, int M, int K,
                        __nv_bfloat16* __restrict__ out, int ldo,
                        const __nv_bfloat16* __restrict__ resid) {
    constexpr int S = kSwapStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * kSwapABytes;
    float* sE = reinterpret_cast<float*>(sB + S * kSwapBBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * kSwapBBytes + kSwapEpiBytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const GemmGroup g = batch.table[batch.idx[0]];   // one group per launch (host checks)
    const int wrow0 = batch.b_row[0];
    const int rows = g.a_end - g.a_begin;
    if (rows <= 0) return;                       // uniform over the cluster
    const int m_tiles = M / 256;
    SwapRR probe;
    probe.init(rows, m_tiles, pair, npairs);
    if (probe.empty()) return;                   // no tile for this pair: both CTAs leave
    const int num_kb = K / BK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmW);
        for (int i = 0; i < 4; ++i) ptx::prefetch_tmap(&tmX.box[i]);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 2);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 8);
        }
        ptx::fence_barrier_init();
        ptx::fence_proxy_async();
    }
    if (warp == 2) ptx::tmem_alloc_cta2<512>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------------------------------------------- TMA producer (both CTAs)
            const uint64_t pol = ptx::policy_evict_normal();
            const uint32_t full0 = ptx::mapa_shared(&full[0], 0);
            SwapRR sc = probe;
            int stage = 0;
            uint32_t phase = 0;
            int m, col, nc;
            while (sc.next(m, col, nc)) {
                const int wrow = wrow0 + m * 256 + (int)rank * 128;
                const int half = nc >> 1;                      // token rows of this CTA
                const int trow = g.a_begin + col + (int)rank * half;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1u);
                    const uint32_t fbar = full0 + stage * 8;
                    if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * kSwapABytes + (uint32_t)nc * BK * 2);
                    else ptx::mbar_arrive_cluster(fbar);
                    ptx::tma_load_2d_cta2(sA + stage * kSwapABytes, &tmW, fbar, kb * BK, wrow, pol);
                    uint8_t* b = sB + stage * kSwapBBytes;
                    for (int i = 0, r = 0; i < 4; ++i) {   // boxes of 128, 64, 32, 16 rows
                        const int box = 128 >> i;
                        if (half - r >= box) {
                            ptx::tma_load_2d_cta2(b + r * (BK * 2), &tmX.box[i], fbar, kb * BK,
                                                  trow + r, pol);
                            r += box;
                        }
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            // ---------------------------------------------------- MMA issuer (leader only)
            SwapRR sc = probe;
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            int m, col, nc;
            while (sc.next(m, col, nc)) {
                const uint32_t idesc = ptx::umma_idesc_bf16(256, (uint32_t)nc);
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], aphase ^ 1u);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * 256;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(sA + stage * kSwapABytes);
                    const uint32_t b0 = ptx::smem_u32(sB + stage * kSwapBBytes);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        ptx::umma_bf16_cta2(d, ptx::umma_desc_sw128_kmajor(a0 + kk * 32),
                                            ptx::umma_desc_sw128_kmajor(b0 + kk * 32), idesc,
                                            (kb | kk) != 0 ? 1u : 0u);
                    ptx::umma_commit_cta2_mc(&empty[stage], 0x3);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                ptx::umma_commit_cta2_mc(&tfull[acc], 0x3);
                ++it;
            }
        }
    } else if (warp >= 4) {
        // -------------------------------------------------------- epilogue (both CTAs)
        const int q = warp - 4;
        const uint32_t tempty0 = ptx::mapa_shared(&tempty[0], 0);
        SwapRR sc = probe;
        int it = 0;
        int m, col, nc;
        while (sc.next(m, col, nc)) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256;
            // weight rows of this warp: m*256 + rank*128 + q*32 + [0, 32)
            const int fcol = (MODE == kGemmSwiGLU) ? m * 128 + (int)rank * 64 + q * 16
                                                   : m * 256 + (int)rank * 128 + q * 32;
            swap_epilogue<MODE>(taddr, lane, nc, col, rows, (int64_t)g.out_base + col, out, ldo,
                                fcol, resid, sE + q * (32 * 33));
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + acc * 8);
            ++it;
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_cta2<512>(tmem_base);
    }
}

template <int MODE>
cudaError_t launch_swap(const CUtensorMap* tmW, const TokenMaps* tmX, const GemmBatch& batch,
                        int M, int K, __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid,
                        int grid, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(expert_gemm_swap_kernel<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSwapSmem);   // every launch, see launch_pair
    if (e != cudaSuccess) return e;
    expert_gemm_swap_kernel<MODE><<<grid & ~1, kThreads, kSwapSmem, st>>>(*tmW, *tmX, batch, M, K,
                                                                          out, ldo, resid);
    return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_pair(const CUtensorMap* tmA, const CUtensorMap* tmB, const TokenMaps* tmT,
                        const PairBMaps* alt, const GemmBatch& batch, int N, int K,
                        __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid, int grid,
                        cudaStream_t st) {
    // Set on every launch: the attribute is per device context, contexts may be driven from
    // several host threads (MOE_FLAG_LOCAL_EP), and the call is a cheap host-side update.
    cudaError_t e = cudaFuncSetAttribute(expert_gemm_pair_kernel<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kPairSmem);
    if (e != cudaSuccess) return e;
    TokenMaps none{};
    PairBMaps no_alt{};
    GemmBatch b = batch;
    if (!alt) b.alt_ok = 0;
    expert_gemm_pair_kernel<MODE><<<grid & ~1, kThreads, kPairSmem, st>>>(
        *tmA, *tmB, tmT ? *tmT : none, alt ? *alt : no_alt, b, N, K, out, ldo, resid);
    return cudaGetLastError();
}

template <int BN, int MODE>
cudaError_t launch_one(const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmBatch& batch,
                       int N, int K, __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid,
                        int grid, cudaStream_t st) {
    using C = GemmCfg<BN>;
    cudaError_t e = cudaFuncSetAttribute(expert_gemm_kernel<BN, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::kSmem);   // every launch, see launch_pair
    if (e != cudaSuccess) return e;
    expert_gemm_kernel<BN, MODE><<<grid, kThreads, C::kSmem, st>>>(*tmA, *tmB, batch, N, K, out, ldo, resid);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_expert_gemm_swap(int mode, const CUtensorMap* tmW, const TokenMaps* tmX,
                                    const GemmBatch& batch, int M, int K, __nv_bfloat16* out,
                                    int ldo, const __nv_bfloat16* resid, int grid, cudaStream_t st) {
    if ((mode == kGemmResidual) != (resid != nullptr) || M % 256 || K % BK || batch.n != 1)
        return cudaErrorInvalidValue;
    if (mode == kGemmSwiGLU) return launch_swap<kGemmSwiGLU>(tmW, tmX, batch, M, K, out, ldo, resid, grid, st);
    if (mode == kGemmResidual) return launch_swap<kGemmResidual>(tmW, tmX, batch, M, K, out, ldo, resid, grid, st);
    return launch_swap<kGemmPlain>(tmW, tmX, batch, M, K, out, ldo, resid, grid, st);
}

double pair_makespan(const int64_t* rows, int n, int n_tiles, int npairs, bool tail_swap,
                     float tail_cost, bool streamk, int num_kb) {
    int64_t F = 0, R = 0;
    for (int i = 0; i < n; ++i) {
        const int r = (int)std::max<int64_t>(0, rows[i]);
        const int nc = tail_cols(r, tail_swap);
        F += (int64_t)(nc ? r / kPairRows : (r + kPairRows - 1) / kPairRows) * n_tiles;
        if (nc) R += n_tiles;
    }
    if (streamk && !tail_swap) {
        int L, S;
        streamk_plan((int)F, npairs, num_kb, L, S);
        if (L > 0)   // q full waves + one 1/S-long chunk + the partial-sum fixup (~0.1 tile)
            return (double)(F / npairs) + 1.0 / S + 0.1;
    }
    double worst = 0.0;
    for (int p = 0; p < npairs; ++p) {
        TailSched ts;
        ts.init((int)F, (int)R, npairs, p, tail_cost);
        int tails = 0, tj;
        while (ts.next(tj)) ++tails;
        const double load = (double)(F / npairs + (p < F % npairs ? 1 : 0)) + tail_cost * tails;
        worst = std::max(worst, load);
    }
    return worst;
}

int gemm_bn_for(int mode, int N) {
    if (mode == kGemmSwiGLU) return (N % 256 == 0) ? 256 : 0;
    if (N % 256 == 0) return 256;
    if (N % 128 == 0) return 128;
    return 0;
}

cudaError_t launch_expert_gemm(int mode, int bn, bool pair, const CUtensorMap* tmA,
                               const CUtensorMap* tmB, const GemmBatch& batch, int N, int K,
                               __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid, int grid,
                               cudaStream_t st, const TokenMaps* tmT, const PairBMaps* alt) {
    if ((mode == kGemmResidual) != (resid != nullptr) || batch.n < 1 || batch.n > kMaxBatch)
        return cudaErrorInvalidValue;
    if (pair) {
        if (bn != 256 || (batch.tail_swap && (!tmT || batch.part != 0 || !(batch.tail_cost > 0.f))))
            return cudaErrorInvalidValue;
        if (batch.select && batch.alt_ok && !alt) return cudaErrorInvalidValue;  // plans must agree
        if (mode == kGemmSwiGLU) return launch_pair<kGemmSwiGLU>(tmA, tmB, tmT, alt, batch, N, K, out, ldo, resid, grid, st);
        if (mode == kGemmResidual) return launch_pair<kGemmResidual>(tmA, tmB, tmT, alt, batch, N, K, out, ldo, resid, grid, st);
        return launch_pair<kGemmPlain>(tmA, tmB, tmT, alt, batch, N, K, out, ldo, resid, grid, st);
    }
    if (mode == kGemmSwiGLU) {
        if (bn == 256) return launch_one<256, kGemmSwiGLU>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
    } else if (mode == kGemmResidual) {
        if (bn == 256) return launch_one<256, kGemmResidual>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
        if (bn == 128) return launch_one<128, kGemmResidual>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
    } else {
        if (bn == 256) return launch_one<256, kGemmPlain>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
        if (bn == 128) return launch_one<128, kGemmPlain>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace moe

namespace moe {
cudaError_t set_gemm_l2_hints(int mode) {
    return cudaMemcpyToSymbol(g_l2_hints, &mode, sizeof(int));
}
cudaError_t set_gemm_group_m(int gm) {
    return cudaMemcpyToSymbol(g_group_m, &gm, sizeof(int));
}
}  // namespace moe
