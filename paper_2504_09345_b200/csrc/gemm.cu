// gemm.cu -- grouped bf16 expert GEMM on 5th-gen tensor cores (tcgen05 + TMEM), fed by TMA.
//
// One launch computes a batch of expert groups (steps a5 / a6 of the MoE layer; Eq. 1's
// "6 N_k h h_i" FLOPs) -- the experts whose weights sit in the launch's staging
// slots, whose tiles share the persistent CTAs' waves (GemmBatch):
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
// Two kernels, chosen per launch by the host's wave model (moe_api.cu pick_pair):
//   expert_gemm_kernel       1 CTA per SM, 128 x BN tiles (tcgen05.mma.cta_group::1, M = 128);
//   expert_gemm_pair_kernel  CTA pair (cluster of 2 on one TPC), 256 x 256 tiles
//                            (tcgen05.mma.cta_group::2, M = 256, 2-CTA TMA, multicast commits).
// Every launch can report its SM clock (GemmBatch::clk).  Structure of the first (persistent,
// one CTA per SM, 256 threads):
//   warp 0     TMA producer: A tile 128x64 and B tile BNx64 per stage, 128B swizzle
//   warp 1     MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16 per instr
//   warp 2     TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-7  epilogue: tcgen05.ld 32x32b -> fp32 math -> bf16 -> global
// Pipelines: smem full/empty mbarriers (TMA <-> MMA), TMEM full/empty (MMA <-> epilogue).
// (Round-1 experiments that lost to these two kernels in-bench -- swap-AB tiles, 224/192-wide
// tiles, device-side kernel choice, stream-K, a tail split -- are recorded in DESIGN.md §12 and
// were removed from the code.)
#include <algorithm>

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

// Raster group override (MOE_GEMM_GROUPM; 0 = the kernel's default).  Tests use it to put
// several raster groups -- and a partial last one -- into launches small enough for the oracle.
__device__ int g_group_m = 0;

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
struct BatchInfo {
    int n, total;
    int first[kMaxBatch + 1];
    int m_tiles[kMaxBatch];
    int a_begin[kMaxBatch], a_end[kMaxBatch], out_base[kMaxBatch], b_row[kMaxBatch];
};
constexpr size_t kBatchSmem = (sizeof(BatchInfo) + 15) & ~size_t(15);
static_assert(kBatchSmem <= kBatchReserve, "BatchInfo does not fit its reservation");

// Row ranges of the launch's groups and their tiles of bm rows x n_tiles weight tiles, numbered
// group after group (one thread).
__device__ __forceinline__ void batch_init(BatchInfo* bi, const GemmBatch& b, int bm, int n_tiles) {
    int t = 0;
    for (int i = 0; i < b.n; ++i) {
        const GemmGroup g = b.table[b.idx[i]];
        bi->a_begin[i] = g.a_begin;
        bi->a_end[i] = max(g.a_begin, g.a_end);
        bi->out_base[i] = g.out_base;
        bi->b_row[i] = b.b_row[i];
        bi->m_tiles[i] = (bi->a_end[i] - bi->a_begin[i] + bm - 1) / bm;
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
    ClkProbe clk;
    clk.start(batch);
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
            // evict_normal on both operands (measured: evict_last on A + evict_first on the
            // weights INCREASED DRAM re-reads)
            const uint64_t pol = ptx::policy_evict_normal();
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
                                          arow, pol);
                    ptx::tma_load_2d_hint(sB + stage * C::kBBytes, &tmB, &full[stage], kb * BK,
                                          brow, pol);
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
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes 256 x 256 tiles.
// Each CTA stages its own 128 rows of A and half (128 rows) of the B tile per K step (32 KB, 6
// stages), the leader issues tcgen05.mma.cta_group::2 (M=256) reading both CTAs' smem, and each
// CTA's TMEM holds its 128 rows of the fp32 accumulator.  Per SM this halves the B bytes moved
// per MMA and doubles the bytes in flight (6 x 32 KB vs 4 x 48 KB), for large expert groups.
// Barrier protocol: full[s] (leader; arrivals: leader expect_tx + peer remote arrive; TMA bytes
// of both CTAs), empty[s] (both; MMA commit multicast), tfull[a] (both; multicast), tempty[a]
// (leader; 4 epilogue warps x 2 CTAs).  The remote arrive uses default semantics: a
// `.release.cluster` arrive lowered to MEMBAR.ALL.GPU on every stage and halved throughput.
// Tiles are dealt round-robin over the pairs (tile t -> pair t % P) in tile_coords order.
constexpr int kPairStages = 6;
constexpr int kPairBN = 256;
constexpr uint32_t kPairABytes = 128 * BK * 2;   // per CTA
constexpr uint32_t kPairBBytes = 128 * BK * 2;   // per CTA (half of a 256-row B tile)
constexpr size_t kPairSmem = 1024 + kPairStages * (kPairABytes + kPairBBytes) + kBatchReserve + 256;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
expert_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ GemmBatch batch, int N, int K,
                        __nv_bfloat16* __restrict__ out, int ldo,
                        const __nv_bfloat16* __restrict__ resid) {
    constexpr int PM = 256, S = kPairStages, BN = kPairBN;
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
    ClkProbe clk;
    clk.start(batch);
    if (threadIdx.x == 0) batch_init(bi, batch, PM, n_tiles);
    __syncthreads();
    const int total = bi->total;
    if (pair >= total) return;                   // identical in both CTAs: the pair leaves together
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
            const uint64_t pol = ptx::policy_evict_normal();
            const uint32_t full0 = ptx::mapa_shared(&full[0], 0);  // leader's full[0]
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = pair; tile < total; tile += npairs) {
                int m, n, local;
                const int gi = batch_locate(bi, tile, local);
                tile_coords(local, bi->m_tiles[gi], n_tiles, group_m, m, n);
                const int brow = bi->b_row[gi] + n * BN + (int)rank * (BN / 2);
                const int arow = bi->a_begin[gi] + m * PM + (int)rank * 128;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1u);
                    const uint32_t fbar = full0 + stage * 8;
                    if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (kPairABytes + kPairBBytes));
                    else ptx::mbar_arrive_cluster(fbar);
                    ptx::tma_load_2d_cta2(sB + stage * kPairBBytes, &tmB, fbar, kb * BK, brow, pol);
                    ptx::tma_load_2d_cta2(sA + stage * kPairABytes, &tmA, fbar, kb * BK, arow, pol);
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
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
            const int arow = bi->a_begin[gi] + m * PM + (int)rank * 128 + q * 32 + lane;
            const bool valid = arow < bi->a_end[gi];
            const int64_t orow = (int64_t)bi->out_base[gi] + (arow - bi->a_begin[gi]);
            epilogue_row<MODE>(taddr, valid, out + orow * ldo,
                               resid ? resid + orow * ldo : nullptr, n, BN);
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
    clk.stop(batch);
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
    if ((mode == kGemmResidual) != (resid != nullptr) || batch.n < 1 || batch.n > kMaxBatch ||
        K % BK)
        return cudaErrorInvalidValue;
    if (pair) {
        if (bn != kPairBN || N % kPairBN) return cudaErrorInvalidValue;
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

cudaError_t set_gemm_group_m(int gm) {
    return cudaMemcpyToSymbol(g_group_m, &gm, sizeof(int));
}

}  // namespace moe
