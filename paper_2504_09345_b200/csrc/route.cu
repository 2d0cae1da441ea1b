// route.cu -- router GEMM + softmax top-k gating (a2, a3), scan + permute (a4) and the
// gate-weighted combine (a7) of the MoE layer (readings R1-R10 in DESIGN.md).
//
// Determinism / exactness by construction:
//   * router logits accumulate the exact bf16 x bf16 products in fp64 with one FMA chain per
//     (token, expert) in ascending channel order -- the same chain as the definition (R6), so
//     expert selection is bit-exact;
//   * top-k breaks ties toward the lower expert index (R5); NaN ranks last;
//   * token positions inside an expert group are ascending in t (R12), computed from per-tile
//     counts (no atomics on the data path).
#include <cfloat>
#include <cmath>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kRouterThreads = 256;
constexpr int kChunk = 64;  // channels staged per iteration (one 16-byte vector per thread of x)
constexpr int kXsPitch = kRouteTile + 1;  // padded row (doubles): conflict-free transposed stores

__device__ __forceinline__ bool ranks_above(double la, int a, double lb, int b) {
    const bool na = isnan(la), nb = isnan(lb);
    if (na || nb) return (na && nb) ? (a < b) : nb;
    if (la > lb) return true;
    if (la < lb) return false;
    return a < b;
}

__device__ __forceinline__ void bf16x8_to_f64(const int4& v, double (&o)[8]) {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(b[i]);  // exact
        o[2 * i] = (double)f.x;
        o[2 * i + 1] = (double)f.y;
    }
}

// One block = kRouteTile (32) tokens.  Warp w computes experts {w, w+8, w+16, ...} for all 32
// tokens (lane = token), EPT accumulators per thread; each accumulator is ONE fp64 FMA chain in
// ascending channel order (the definition's order, reading R6).  Staging: 64-channel chunks, one
// 16-byte x vector per thread and up to 4 router vectors, prefetched into registers one chunk
// ahead so global latency overlaps the FMA chains.
template <int EPT>
__global__ void __launch_bounds__(kRouterThreads)
router_topk_kernel(const __nv_bfloat16* __restrict__ x, int T, int h,
                   const __nv_bfloat16* __restrict__ wr, int ne, int k, int renorm,
                   int32_t* __restrict__ idx_out, float* __restrict__ gate_out,
                   int32_t* __restrict__ tile_counts) {
    __shared__ double xs[kChunk * kXsPitch];   // x tile, transposed [c][t], fp64
    __shared__ int cnt[kMaxExperts];
    extern __shared__ double dyn[];            // ws [ne][kChunk]  then logits [32][ne]
    double* ws = dyn;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t0 = blockIdx.x * kRouteTile;
    for (int e = tid; e < kMaxExperts; e += kRouterThreads) cnt[e] = 0;

    double acc[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) acc[i] = 0.0;

    // staging assignment: x vector (token xt, channels xc..xc+7); router vectors v = tid + 256 i
    const int xt = tid >> 3, xc = (tid & 7) * 8;
    const bool xvalid = t0 + xt < T;
    const int nwv = ne * (kChunk / 8);
    int4 xr = make_int4(0, 0, 0, 0);
    int4 wv[kMaxExperts * (kChunk / 8) / kRouterThreads];
    auto load = [&](int c0) {
        if (xvalid) xr = ptx::ld_nc_v4(x + (size_t)(t0 + xt) * h + c0 + xc);
#pragma unroll
        for (int i = 0; i < kMaxExperts * (kChunk / 8) / kRouterThreads; ++i) {
            const int v = tid + kRouterThreads * i;
            if (v < nwv) wv[i] = ptx::ld_nc_v4(wr + (size_t)(v >> 3) * h + c0 + (v & 7) * 8);
        }
    };
    auto store = [&]() {
        double d[8];
        bf16x8_to_f64(xr, d);
#pragma unroll
        for (int j = 0; j < 8; ++j) xs[(xc + j) * kXsPitch + xt] = d[j];
#pragma unroll
        for (int i = 0; i < kMaxExperts * (kChunk / 8) / kRouterThreads; ++i) {
            const int v = tid + kRouterThreads * i;
            if (v < nwv) {
                bf16x8_to_f64(wv[i], d);
#pragma unroll
                for (int j = 0; j < 8; ++j) ws[(v >> 3) * kChunk + (v & 7) * 8 + j] = d[j];
            }
        }
    };

    load(0);
    for (int c0 = 0; c0 < h; c0 += kChunk) {
        store();
        __syncthreads();
        if (c0 + kChunk < h) load(c0 + kChunk);   // next chunk in flight during the FMAs
#pragma unroll 8
        for (int c = 0; c < kChunk; ++c) {
            const double xv = xs[c * kXsPitch + lane];
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int e = warp + 8 * i;
                if (e < ne) acc[i] = fma(xv, ws[e * kChunk + c], acc[i]);
            }
        }
        __syncthreads();
    }
    // logits -> shared [32][ne]
    double* lg = dyn;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int e = warp + 8 * i;
        if (e < ne) lg[lane * ne + e] = acc[i];
    }
    __syncthreads();

    // warp-shuffle top-k: warp w handles tokens w, w+8, w+16, w+24 of the tile
    for (int tt = warp; tt < kRouteTile; tt += 8) {
        const int t = t0 + tt;
        if (t >= T) break;
        double v[kMaxExperts / 32];
#pragma unroll
        for (int i = 0; i < kMaxExperts / 32; ++i) {
            const int e = lane + 32 * i;
            v[i] = (e < ne) ? lg[tt * ne + e] : 0.0;
        }
        uint32_t taken = 0;
        double sel_l[kMaxTopK];
        int sel_e[kMaxTopK];
        for (int j = 0; j < k; ++j) {
            bool have = false;
            double bv = 0.0;
            int be = 0x7fffffff;
#pragma unroll
            for (int i = 0; i < kMaxExperts / 32; ++i) {
                const int e = lane + 32 * i;
                if (e < ne && !((taken >> i) & 1u)) {
                    if (!have || ranks_above(v[i], e, bv, be)) {
                        bv = v[i];
                        be = e;
                        have = true;
                    }
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int oe = __shfl_xor_sync(0xffffffffu, be, off);
                const int oh = __shfl_xor_sync(0xffffffffu, (int)have, off);
                if (oh && (!have || ranks_above(ov, oe, bv, be))) {
                    bv = ov;
                    be = oe;
                    have = true;
                }
            }
            if ((be & 31) == lane) taken |= 1u << (be >> 5);
            sel_l[j] = bv;
            sel_e[j] = be;
        }
        // softmax gates in fp64 (R3): renormalised over the k selected, or over all N_e
        const double m = sel_l[0];
        double z = 0.0;
        if (renorm) {
            for (int j = 0; j < k; ++j) z += exp(sel_l[j] - m);
        } else {
            double part = 0.0;
#pragma unroll
            for (int i = 0; i < kMaxExperts / 32; ++i) {
                const int e = lane + 32 * i;
                if (e < ne) part += exp(v[i] - m);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            z = part;
        }
        if (lane < k) {
            double mine = sel_l[0];
            int me = sel_e[0];
            for (int j = 1; j < k; ++j)
                if (j == lane) {
                    mine = sel_l[j];
                    me = sel_e[j];
                }
            idx_out[(size_t)t * k + lane] = me;
            gate_out[(size_t)t * k + lane] = (float)(exp(mine - m) / z);
            atomicAdd(&cnt[me], 1);
        }
    }
    __syncthreads();
    for (int e = tid; e < ne; e += kRouterThreads) tile_counts[(size_t)blockIdx.x * ne + e] = cnt[e];
}

// Single block of 1024 threads.  Warp w scans experts w, w+32, ... over the tiles.
__global__ void __launch_bounds__(1024)
scan_kernel(const int32_t* __restrict__ tile_counts, int n_tiles, int ne, int T, int k,
            int num_shared, int32_t* __restrict__ tile_prefix, int32_t* __restrict__ offsets,
            int32_t* __restrict__ counts, GemmGroup* __restrict__ grp1,
            GemmGroup* __restrict__ grp2) {
    __shared__ int tot[kMaxExperts];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < ne; e += 32) {
        int run = 0;
        for (int b0 = 0; b0 < n_tiles; b0 += 32) {
            const int b = b0 + lane;
            const int v = (b < n_tiles) ? tile_counts[(size_t)b * ne + e] : 0;
            int s = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int n = __shfl_up_sync(0xffffffffu, s, off);
                if (lane >= off) s += n;
            }
            if (b < n_tiles) tile_prefix[(size_t)b * ne + e] = run + s - v;
            run += __shfl_sync(0xffffffffu, s, 31);
        }
        if (lane == 0) tot[e] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int o = 0;
        for (int e = 0; e < ne; ++e) {
            offsets[e] = o;
            counts[e] = tot[e];
            grp1[e] = GemmGroup{o, o + tot[e], o, 0};
            grp2[e] = GemmGroup{o, o + tot[e], o, 0};
            o += tot[e];
        }
        offsets[ne] = o;  // == T * k
        const int R = T * k;
        for (int s = 0; s < num_shared; ++s) {
            counts[ne + s] = T;
            grp1[ne + s] = GemmGroup{0, T, R + s * T, 0};          // A = hidden itself
            grp2[ne + s] = GemmGroup{R + s * T, R + s * T + T, R + s * T, 0};
        }
    }
}

constexpr int kPermuteTokens = 16;  // tokens per permute block (half a routing tile)

__global__ void __launch_bounds__(256)
permute_kernel(const __nv_bfloat16* __restrict__ x, int T, int h, int k, int ne,
               const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_prefix,
               const int32_t* __restrict__ offsets, __nv_bfloat16* __restrict__ x_perm,
               int32_t* __restrict__ pos_out) {
    __shared__ int sidx[kRouteTile * kMaxTopK];
    __shared__ int spos[kPermuteTokens * kMaxTopK];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int parts = kRouteTile / kPermuteTokens;
    const int tile = blockIdx.x / parts, tt0 = (blockIdx.x % parts) * kPermuteTokens;
    const int tbase = tile * kRouteTile;
    const int n_pre = (tt0 + kPermuteTokens) * k;
    for (int i = tid; i < n_pre; i += 256) {
        const int t = tbase + i / k;
        sidx[i] = (t < T) ? idx[(size_t)tbase * k + i] : -1;
    }
    __syncthreads();
    for (int i = tid; i < kPermuteTokens * k; i += 256) {
        const int tt = tt0 + i / k, j = i % k, t = tbase + tt;
        if (t < T) {
            const int e = sidx[tt * k + j];
            int r = 0;
            for (int u = 0; u < tt * k; ++u) r += (sidx[u] == e);
            const int p = offsets[e] + tile_prefix[(size_t)tile * ne + e] + r;
            spos[i] = p;
            pos_out[(size_t)t * k + j] = p;
        }
    }
    __syncthreads();
    const int nvec = h / 8;  // 16-byte vectors per row
    for (int q = warp; q < kPermuteTokens; q += 8) {
        const int t = tbase + tt0 + q;
        if (t >= T) break;
        const int4* src = reinterpret_cast<const int4*>(x + (size_t)t * h);
        int dst_row[kMaxTopK];
#pragma unroll
        for (int j = 0; j < kMaxTopK; ++j) dst_row[j] = (j < k) ? spos[q * k + j] : 0;
        constexpr int U = 4;
        for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
            int4 buf[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + 32 * u;
                if (v < nvec) buf[u] = ptx::ld_nc_v4(src + v);
            }
            for (int j = 0; j < k; ++j) {
                int4* dst = reinterpret_cast<int4*>(x_perm + (size_t)dst_row[j] * h);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int v = v0 + 32 * u;
                    if (v < nvec) dst[v] = buf[u];
                }
            }
        }
    }
}

// Warp per token; lane handles 8 consecutive columns per 16-byte vector.
__global__ void __launch_bounds__(256)
combine_kernel(const __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ pos,
               const float* __restrict__ gates, int T, int h, int k, int num_shared,
               int64_t shared_base, __nv_bfloat16* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 8 + warp;
    if (t >= T) return;
    int prow[kMaxTopK];
    float g[kMaxTopK];
#pragma unroll
    for (int j = 0; j < kMaxTopK; ++j) {
        prow[j] = (j < k) ? pos[(size_t)t * k + j] : 0;
        g[j] = (j < k) ? gates[(size_t)t * k + j] : 0.f;
    }
    const int nvec = h / 8;
    for (int v = lane; v < nvec; v += 32) {
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
        for (int j = 0; j < k; ++j) {
            const int4 raw = ptx::ld_nc_v4(reinterpret_cast<const int4*>(y + (size_t)prow[j] * h) + v);
            const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(b[i]);
                acc[2 * i] = fmaf(g[j], f.x, acc[2 * i]);
                acc[2 * i + 1] = fmaf(g[j], f.y, acc[2 * i + 1]);
            }
        }
        for (int s = 0; s < num_shared; ++s) {
            const int64_t row = shared_base + (int64_t)s * T + t;
            const int4 raw = ptx::ld_nc_v4(reinterpret_cast<const int4*>(y + (size_t)row * h) + v);
            const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(b[i]);
                acc[2 * i] += f.x;
                acc[2 * i + 1] += f.y;
            }
        }
        int4 o;
        o.x = (int)ptx::pack_bf16x2(acc[0], acc[1]);
        o.y = (int)ptx::pack_bf16x2(acc[2], acc[3]);
        o.z = (int)ptx::pack_bf16x2(acc[4], acc[5]);
        o.w = (int)ptx::pack_bf16x2(acc[6], acc[7]);
        reinterpret_cast<int4*>(out + (size_t)t * h)[v] = o;
    }
}

}  // namespace

cudaError_t launch_router_topk(const __nv_bfloat16* x, int T, int h, const __nv_bfloat16* wr,
                               int ne, int k, int renorm, int32_t* idx, float* gates,
                               int32_t* tile_counts, cudaStream_t st) {
    const int n_tiles = (T + kRouteTile - 1) / kRouteTile;
    if (n_tiles == 0) return cudaSuccess;
    const size_t dyn = sizeof(double) * (size_t)ne * kChunk;  // >= 32 * ne doubles (logits too)
    const int ept = (ne + 7) / 8;
#define MOE_ROUTER(E)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = cudaFuncSetAttribute(router_topk_kernel<E>,                         \
            cudaFuncAttributeMaxDynamicSharedMemorySize,                                     \
            (int)(sizeof(double) * kMaxExperts * kChunk));                                   \
        if (e_ != cudaSuccess) return e_;                                                    \
        router_topk_kernel<E><<<n_tiles, kRouterThreads, dyn, st>>>(x, T, h, wr, ne, k,      \
                                                                     renorm, idx, gates,     \
                                                                     tile_counts);           \
    } while (0)
    if (ept <= 1) MOE_ROUTER(1);
    else if (ept <= 2) MOE_ROUTER(2);
    else if (ept <= 4) MOE_ROUTER(4);
    else if (ept <= 8) MOE_ROUTER(8);
    else MOE_ROUTER(16);
#undef MOE_ROUTER
    return cudaGetLastError();
}

cudaError_t launch_scan(const int32_t* tile_counts, int n_tiles, int ne, int T, int k,
                        int num_shared, int32_t* tile_prefix, int32_t* offsets, int32_t* counts,
                        GemmGroup* grp1, GemmGroup* grp2, cudaStream_t st) {
    scan_kernel<<<1, 1024, 0, st>>>(tile_counts, n_tiles, ne, T, k, num_shared, tile_prefix,
                                    offsets, counts, grp1, grp2);
    return cudaGetLastError();
}

cudaError_t launch_permute(const __nv_bfloat16* x, int T, int h, int k, int ne,
                           const int32_t* idx, const int32_t* tile_prefix,
                           const int32_t* offsets, __nv_bfloat16* x_perm, int32_t* pos,
                           cudaStream_t st) {
    const int n_tiles = (T + kRouteTile - 1) / kRouteTile;
    if (n_tiles == 0) return cudaSuccess;
    permute_kernel<<<n_tiles * (kRouteTile / kPermuteTokens), 256, 0, st>>>(
        x, T, h, k, ne, idx, tile_prefix, offsets, x_perm, pos);
    return cudaGetLastError();
}

cudaError_t launch_combine(const __nv_bfloat16* y_perm, const int32_t* pos, const float* gates,
                           int T, int h, int k, int num_shared, int64_t shared_base,
                           __nv_bfloat16* out, cudaStream_t st) {
    if (T == 0) return cudaSuccess;
    combine_kernel<<<(T + 7) / 8, 256, 0, st>>>(y_perm, pos, gates, T, h, k, num_shared,
                                                shared_base, out);
    return cudaGetLastError();
}

}  // namespace moe
