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
// Structure of the first (persistent, one CTA per SM, 256 threads):
//   warp 0     TMA producer: A tile 128x64 and B tile BNx64 per stage, 128B swizzle
//   warp 1     MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16 per instr
//   warp 2     TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-7  epilogue: tcgen05.ld 32x32b -> fp32 math -> bf16 -> global
// Pipelines: smem full/empty mbarriers (TMA <-> MMA), TMEM full/empty (MMA <-> epilogue).
#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kThreads = 256;

constexpr size_t kBatchReserve = 512;   // shared memory for BatchInfo (below)

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

__device__ __forceinline__ float silu_mul(float g, float u) {
    return g / (1.0f + __expf(-g)) * u;
}

// Epilogue of one accumulator row (this thread's TMEM lane): TMEM -> registers -> fp32 math ->
// bf16 -> global.  SwiGLU tiles hold gate columns [0, BN/2) and the matching up columns
// [BN/2, BN); they produce BN/2 outputs.  tcgen05.ld is warp-collective: every lane loads, only
// rows inside the group store.
template <int BN, int MODE>
__device__ __forceinline__ void epilogue_row(uint32_t taddr, bool valid, __nv_bfloat16* row_out,
                                             const __nv_bfloat16* row_res, int n) {
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
struct BatchInfo {
    int n, total;
    int first[kMaxBatch + 1];
    int m_tiles[kMaxBatch];
    int a_begin[kMaxBatch], a_end[kMaxBatch], out_base[kMaxBatch], b_row[kMaxBatch];
};
constexpr size_t kBatchSmem = (sizeof(BatchInfo) + 15) & ~size_t(15);
static_assert(kBatchSmem <= kBatchReserve, "BatchInfo does not fit its reservation");

__device__ __forceinline__ void batch_init(BatchInfo* bi, const GemmBatch& b, int bm,
                                           int n_tiles) {
    int t = 0;
    for (int i = 0; i < b.n; ++i) {
        GemmGroup g = b.table[b.idx[i]];
        const int head = (max(0, g.a_end - g.a_begin) / kPairRows) * kPairRows;
        if (b.part == 1) {          // whole 256-row tiles only
            g.a_end = g.a_begin + head;
        } else if (b.part == 2) {   // the remainder
            g.a_begin += head;
            g.out_base += head;
        }
        const int rows = max(0, g.a_end - g.a_begin);
        bi->a_begin[i] = g.a_begin;
        bi->a_end[i] = g.a_end;
        bi->out_base[i] = g.out_base;
        bi->b_row[i] = b.b_row[i];
        bi->m_tiles[i] = (rows + bm - 1) / bm;
        bi->first[i] = t;
        t += bi->m_tiles[i] * n_tiles;
    }
    bi->first[b.n] = t;
    bi->n = b.n;
    bi->total = t;
}

__device__ __forceinline__ int batch_locate(const BatchInfo* bi, int tile, int& local) {
    int g = 0;
    while (tile >= bi->first[g + 1]) ++g;
    local = tile - bi->first[g];
    return g;
}

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
    if (threadIdx.x == 0) batch_init(bi, batch, BM, n_tiles);
    __syncthreads();
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
            epilogue_row<BN, MODE>(taddr, valid, out + orow * ldo,
                                   resid ? resid + orow * ldo : nullptr, n);
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
constexpr int kPairStages = 6;
constexpr uint32_t kPairABytes = 128 * BK * 2;   // per CTA
constexpr uint32_t kPairBBytes = 128 * BK * 2;   // per CTA (half of a 256-row B tile)
constexpr size_t kPairSmem =
    1024 + kPairStages * (kPairABytes + kPairBBytes) + kBatchReserve + 256;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
expert_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ GemmBatch batch, int N, int K,
                        __nv_bfloat16* __restrict__ out, int ldo,
                        const __nv_bfloat16* __restrict__ resid) {
    constexpr int BN = 256, PM = 256, S = kPairStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * kPairABytes;
    BatchInfo* bi = reinterpret_cast<BatchInfo*>(sB + S * kPairBBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(bi) + kBatchSmem);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int n_tiles = N / BN;
    if (threadIdx.x == 0) batch_init(bi, batch, PM, n_tiles);
    __syncthreads();
    const int total = bi->total;                 // identical in both CTAs of the cluster
    if (pair >= total) return;                   // both CTAs of a pair leave together
    const int num_kb = K / BK;
    const int group_m = g_group_m > 0 ? g_group_m : ((K <= 8192) ? 16 : 4);  // 256-row tiles
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
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
    if (warp == 2) ptx::tmem_alloc_cta2<2 * BN>(tmem_slot);
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
            for (int tile = pair; tile < total; tile += npairs) {
                int m, n, local;
                const int gi = batch_locate(bi, tile, local);
                tile_coords(local, bi->m_tiles[gi], n_tiles, group_m, m, n);
                const int arow = bi->a_begin[gi] + m * PM + (int)rank * 128;
                const int brow = bi->b_row[gi] + n * BN + (int)rank * 128;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1u);
                    const uint32_t fbar = full0 + stage * 8;
                    if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (kPairABytes + kPairBBytes));
                    else ptx::mbar_arrive_cluster(fbar);
                    ptx::tma_load_2d_cta2(sA + stage * kPairABytes, &tmA, fbar, kb * BK, arow, pol_a);
                    ptx::tma_load_2d_cta2(sB + stage * kPairBBytes, &tmB, fbar, kb * BK, brow, pol_b);
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
            constexpr uint32_t idesc = ptx::umma_idesc_bf16(PM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = pair; tile < total; tile += npairs, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], aphase ^ 1u);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(sA + stage * kPairABytes);
                    const uint32_t b0 = ptx::smem_u32(sB + stage * kPairBBytes);
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
            }
        }
    } else if (warp >= 4) {
        // -------------------------------------------------------- epilogue (both CTAs)
        const int q = warp - 4;
        const uint32_t tempty0 = ptx::mapa_shared(&tempty[0], 0);
        int it = 0;
        for (int tile = pair; tile < total; tile += npairs, ++it) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            int m, n, local;
            const int gi = batch_locate(bi, tile, local);
            tile_coords(local, bi->m_tiles[gi], n_tiles, group_m, m, n);
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const int arow = bi->a_begin[gi] + m * PM + (int)rank * 128 + q * 32 + lane;
            const bool valid = arow < bi->a_end[gi];
            const int64_t orow = (int64_t)bi->out_base[gi] + (arow - bi->a_begin[gi]);
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
            epilogue_row<BN, MODE>(taddr, valid, out + orow * ldo,
                                   resid ? resid + orow * ldo : nullptr, n);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + acc * 8);
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_cta2<2 * BN>(tmem_base);
    }
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
cudaError_t launch_pair(const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmBatch& batch,
                        int N, int K, __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid,
                        int grid, cudaStream_t st) {
    // Set on every launch: the attribute is per device context, contexts may be driven from
    // several host threads (MOE_FLAG_LOCAL_EP), and the call is a cheap host-side update.
    cudaError_t e = cudaFuncSetAttribute(expert_gemm_pair_kernel<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kPairSmem);
    if (e != cudaSuccess) return e;
    expert_gemm_pair_kernel<MODE><<<grid & ~1, kThreads, kPairSmem, st>>>(*tmA, *tmB, batch, N, K,
                                                                          out, ldo, resid);
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

int gemm_bn_for(int mode, int N) {
    if (mode == kGemmSwiGLU) return (N % 256 == 0) ? 256 : 0;
    if (N % 256 == 0) return 256;
    if (N % 128 == 0) return 128;
    return 0;
}

cudaError_t launch_expert_gemm(int mode, int bn, bool pair, const CUtensorMap* tmA,
                               const CUtensorMap* tmB, const GemmBatch& batch, int N, int K,
                               __nv_bfloat16* out, int ldo, const __nv_bfloat16* resid, int grid,
                               cudaStream_t st) {
    if ((mode == kGemmResidual) != (resid != nullptr) || batch.n < 1 || batch.n > kMaxBatch)
        return cudaErrorInvalidValue;
    if (pair) {
        if (bn != 256) return cudaErrorInvalidValue;
        if (mode == kGemmSwiGLU) return launch_pair<kGemmSwiGLU>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
        if (mode == kGemmResidual) return launch_pair<kGemmResidual>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
        return launch_pair<kGemmPlain>(tmA, tmB, batch, N, K, out, ldo, resid, grid, st);
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
