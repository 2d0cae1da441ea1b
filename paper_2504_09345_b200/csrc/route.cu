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
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kChunk = 64;  // channels staged per iteration (one 16-byte vector per thread of x)

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

// Warp-shuffle top-k of one block's tokens from their fp64 logits lg[kTok][ne_pad] (shared):
// warp w handles tokens w, w+nw, ...; selection by (logit desc, index asc) with NaN last (R5,
// R13); gates = fp64 softmax over the k selected (or all N_e) logits (R3); per-tile counts.
template <int TPT>
__device__ __forceinline__ void topk_tile(const double* lg, int ne_pad, int t0, int T, int ne,
                                          int k, int renorm, int32_t* __restrict__ idx_out,
                                          float* __restrict__ gate_out,
                                          int (*cnt)[kMaxExperts], int warp, int nw, int lane) {
    constexpr int kTok = kRouteTile * TPT;
    for (int tt = warp; tt < kTok; tt += nw) {
        const int t = t0 + tt;
        if (t >= T) break;
        double v[kMaxExperts / 32];
#pragma unroll
        for (int i = 0; i < kMaxExperts / 32; ++i) {
            const int e = lane + 32 * i;
            v[i] = (e < ne) ? lg[tt * ne_pad + e] : 0.0;
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
            atomicAdd(&cnt[tt / kRouteTile][me], 1);
        }
    }
}

// Router: one block = TPT x kRouteTile (32) tokens; warp w owns experts [w*EPT, (w+1)*EPT) for all
// of them (lane = token, TPT tokens per lane).  Every (token, expert) logit is ONE fp64 FMA chain
// over the channels in ascending order -- the definition's order (reading R6) -- so selection is
// bit-exact.  Per channel a lane reads its TPT x values (fp64, transposed tile) and its EPT router
// weights as EPT/2 double2 broadcasts from a [channel][expert] tile zero-padded to a multiple of
// EPT experts: TPT + EPT/2 shared-memory wavefront groups per TPT*EPT DFMAs and no branches in
// the inner loop (TPT = 2 for many experts: the kernel is shared-memory bound there -- ncu at C4:
// 70% of the smem pipe, short-scoreboard stalls -- and a second token per lane reuses every
// weight broadcast).  64-channel chunks are staged with 16-byte loads prefetched into registers
// one chunk ahead.
template <int EPT, int TPT>
__global__ void __launch_bounds__((EPT >= 8 && TPT == 1) ? 512 : 256)
router_topk_kernel(const __nv_bfloat16* __restrict__ x, int T, int h,
                   const __nv_bfloat16* __restrict__ wr, int ne, int k, int renorm,
                   int32_t* __restrict__ idx_out, float* __restrict__ gate_out,
                   int32_t* __restrict__ tile_counts) {
    constexpr int kTok = kRouteTile * TPT;      // tokens per block
    constexpr int kPitch = kTok + 1;            // padded row (doubles): conflict-free stores
    extern __shared__ __align__(16) double dyn[];
    __shared__ int cnt[TPT][kMaxExperts];
    const int nw = blockDim.x >> 5;            // warps = ne_pad / EPT
    const int ne_pad = nw * EPT;
    double* xs = dyn;                           // [kChunk][kPitch]
    double* ws = dyn + kChunk * kPitch;         // [kChunk][ne_pad], later logits [kTok][ne_pad]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
    const int t0 = blockIdx.x * kTok;
    for (int e = tid; e < TPT * kMaxExperts; e += nthr) cnt[e / kMaxExperts][e % kMaxExperts] = 0;

    double acc[TPT][EPT];
#pragma unroll
    for (int p = 0; p < TPT; ++p)
#pragma unroll
        for (int i = 0; i < EPT; ++i) acc[p][i] = 0.0;

    // x vectors per thread: the TPT = 2 variant runs with >= 3 warps (N_e > 16)
    constexpr int kMinThreads = TPT >= 2 ? 96 : 32;
    constexpr int kXV = (kTok * (kChunk / 8) + kMinThreads - 1) / kMinThreads;
    constexpr int kWV = (EPT * (kChunk / 8) + 31) / 32;  // router vectors per thread
    const int n_xv = kTok * (kChunk / 8);
    const int n_wv = ne_pad * (kChunk / 8);
    int4 xr[kXV], wv[kWV];
    // Staging maps consecutive lanes to consecutive TOKENS (x) / EXPERTS (router) at a fixed
    // 8-channel group, so the transposed fp64 stores hit consecutive shared-memory words (the
    // row-major mapping caused ~72M bank conflicts per C4 call); each lane still reads 16 B.
    auto load = [&](int c0) {
#pragma unroll
        for (int j = 0; j < kXV; ++j) {
            const int v = tid + j * nthr;
            if (v < n_xv) {
                const int t = v % kTok, cc = (v / kTok) * 8;
                xr[j] = (t0 + t < T) ? ptx::ld_nc_v4(x + (size_t)(t0 + t) * h + c0 + cc)
                                     : make_int4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int j = 0; j < kWV; ++j) {
            const int v = tid + j * nthr;
            if (v < n_wv) {
                const int e = v % ne_pad, cc = (v / ne_pad) * 8;
                wv[j] = (e < ne) ? ptx::ld_nc_v4(wr + (size_t)e * h + c0 + cc)
                                 : make_int4(0, 0, 0, 0);
            }
        }
    };
    auto store = [&]() {
        double d[8];
#pragma unroll
        for (int j = 0; j < kXV; ++j) {
            const int v = tid + j * nthr;
            if (v < n_xv) {
                const int t = v % kTok, cc = (v / kTok) * 8;
                bf16x8_to_f64(xr[j], d);
#pragma unroll
                for (int q = 0; q < 8; ++q) xs[(cc + q) * kPitch + t] = d[q];
            }
        }
#pragma unroll
        for (int j = 0; j < kWV; ++j) {
            const int v = tid + j * nthr;
            if (v < n_wv) {
                const int e = v % ne_pad, cc = (v / ne_pad) * 8;
                bf16x8_to_f64(wv[j], d);
#pragma unroll
                for (int q = 0; q < 8; ++q) ws[(cc + q) * ne_pad + e] = d[q];
            }
        }
    };

    load(0);
    const double* wbase = ws + warp * EPT;
    for (int c0 = 0; c0 < h; c0 += kChunk) {
        store();
        __syncthreads();
        if (c0 + kChunk < h) load(c0 + kChunk);   // next chunk in flight during the FMAs
#pragma unroll 8
        for (int c = 0; c < kChunk; ++c) {
            double xv[TPT];
#pragma unroll
            for (int p = 0; p < TPT; ++p) xv[p] = xs[c * kPitch + p * 32 + lane];
            if constexpr (EPT == 1) {
                const double w = wbase[c * ne_pad];
#pragma unroll
                for (int p = 0; p < TPT; ++p) acc[p][0] = fma(xv[p], w, acc[p][0]);
            } else {
                const double2* w2 = reinterpret_cast<const double2*>(wbase + c * ne_pad);
#pragma unroll
                for (int i = 0; i < EPT / 2; ++i) {
                    const double2 w = w2[i];
#pragma unroll
                    for (int p = 0; p < TPT; ++p) {
                        acc[p][2 * i] = fma(xv[p], w.x, acc[p][2 * i]);
                        acc[p][2 * i + 1] = fma(xv[p], w.y, acc[p][2 * i + 1]);
                    }
                }
            }
        }
        __syncthreads();
    }
    // logits -> shared [kTok][ne_pad]: the router tile's space when kTok <= kChunk, else the x
    // tile's (kTok * ne_pad <= kChunk * kPitch for ne_pad <= 64, which TPT = 4 requires)
    double* lg = kTok <= kChunk ? ws : xs;
#pragma unroll
    for (int p = 0; p < TPT; ++p)
#pragma unroll
        for (int i = 0; i < EPT; ++i) lg[(p * 32 + lane) * ne_pad + warp * EPT + i] = acc[p][i];
    __syncthreads();

    topk_tile<TPT>(lg, ne_pad, t0, T, ne, k, renorm, idx_out, gate_out, cnt, warp, nw, lane);
    __syncthreads();
    const int n_tiles = (T + kRouteTile - 1) / kRouteTile;
#pragma unroll
    for (int p = 0; p < TPT; ++p) {   // one row per 32-token routing tile (scan / permute grain)
        const int tile = blockIdx.x * TPT + p;
        if (tile < n_tiles)
            for (int e = tid; e < ne; e += nthr) tile_counts[(size_t)tile * ne + e] = cnt[p][e];
    }
}

// Block 0's SM clock at kernel entry / end of the channel loop (compute warp 0) / exit, and the
// entry-to-exit %globaltimer ns (router_probe(): tools only).
__device__ unsigned long long g_router_probe[8];

// Router rows widened to fp64 for router v7: wr64[c * ne_pad + e] = (double)wr[e][c] (exact), zero
// for the padding experts e >= ne.
__global__ void __launch_bounds__(256)
router_widen_kernel(const __nv_bfloat16* __restrict__ wr, int h, int ne, int ne_pad,
                    double* __restrict__ wr64) {
    const int64_t n = (int64_t)h * ne_pad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(i % ne_pad), c = (int)(i / ne_pad);
        wr64[i] = e < ne ? (double)__bfloat162float(wr[(size_t)e * h + c]) : 0.0;
    }
}

// Order-preserving 64-bit key of an fp64 logit: larger key = larger logit; -0 and +0 share a key
// (they compare equal), every NaN maps to 0 -- below -inf, so NaN ranks last (R13) and NaNs tie.
__device__ __forceinline__ uint64_t logit_key(double l) {
    uint64_t b = (uint64_t)__double_as_longlong(l);
    if (b == 0x8000000000000000ull) b = 0;                   // -0 -> +0
    b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    return isnan(l) ? 0ull : b;
}
__device__ __forceinline__ double key_logit(uint64_t k) {   // inverse (NaN for key 0)
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// Top-k of one token per thread from its fp64 logits (row of lg, shared): insertion of experts
// 0..ne-1 in ascending order into a k-deep list ranked by (key desc, index asc) -- the order
// ranks_above defines (R5, R13) -- on 64-bit integer keys, every list index a compile-time
// constant (registers only).  Gates from the selected fp64 logits exactly as in topk_tile (R3).
// (A warp-per-token shuffle selection with fp64 compares and dynamically indexed lists, and a
// token-per-thread scan with fp64 compares, both took as long as the channel loop at C4.)
template <int TPT, int G>
__device__ __forceinline__ void topk_rows(const double* lg, int pitch, int t0, int T, int ne,
                                          int k, int renorm, int32_t* __restrict__ idx_out,
                                          float* __restrict__ gate_out,
                                          int (*cnt)[kMaxExperts], int tid, int nthr) {
    // G threads (adjacent lanes) per token: thread `sub` scans experts sub, sub + G, ... into its
    // own list, then the G lists merge by xor shuffles (the order is total, so any partition of
    // the experts merges to the same top-k).  nthr and kTok * G are multiples of 32: every lane
    // of a warp runs the same trip count (full-mask shuffles).
    constexpr int kTok = kRouteTile * TPT;
    auto insert = [&](uint64_t (&sk)[kMaxTopK], int (&se)[kMaxTopK], uint64_t ck, int ce) {
#pragma unroll
        for (int j = 0; j < kMaxTopK; ++j) {
            const bool up = j < k && (ck > sk[j] || (ck == sk[j] && ce < se[j]));
            const uint64_t tk = sk[j];
            const int te = se[j];
            sk[j] = up ? ck : tk;
            se[j] = up ? ce : te;
            ck = up ? tk : ck;
            ce = up ? te : ce;
        }
    };
    for (int u = tid; u < kTok * G; u += nthr) {
        const int tt = u / G, sub = u % G;
        const int t = t0 + tt;
        const double* row = lg + tt * pitch;
        uint64_t sk[kMaxTopK];
        int se[kMaxTopK];
#pragma unroll
        for (int j = 0; j < kMaxTopK; ++j) {
            sk[j] = 0ull;
            se[j] = 0x7fffffff;   // empty: below every expert, NaN included
        }
        for (int e = sub; e < ne; e += G) insert(sk, se, logit_key(row[e]), e);
        if constexpr (G > 1) {
#pragma unroll
            for (int off = 1; off < G; off <<= 1) {
                uint64_t pk[kMaxTopK];
                int pe[kMaxTopK];
#pragma unroll
                for (int j = 0; j < kMaxTopK; ++j) {
                    pk[j] = __shfl_xor_sync(0xffffffffu, sk[j], off);
                    pe[j] = __shfl_xor_sync(0xffffffffu, se[j], off);
                }
#pragma unroll
                for (int j = 0; j < kMaxTopK; ++j) insert(sk, se, pk[j], pe[j]);
            }
        }
        if (t >= T || sub != 0) continue;
        const double m = key_logit(sk[0]);
        double ex[kMaxTopK];
        double z = 0.0;
#pragma unroll
        for (int j = 0; j < kMaxTopK; ++j) {
            ex[j] = 0.0;
            if (j < k) {
                ex[j] = exp(key_logit(sk[j]) - m);
                if (renorm) z += ex[j];
            }
        }
        if (!renorm)
            for (int e = 0; e < ne; ++e) z += exp(row[e] - m);
#pragma unroll
        for (int j = 0; j < kMaxTopK; ++j) {
            if (j < k) {
                idx_out[(size_t)t * k + j] = se[j];
                gate_out[(size_t)t * k + j] = (float)(ex[j] / z);
                atomicAdd(&cnt[tt / kRouteTile][se[j]], 1);
            }
        }
    }
}

// Router v7: the same one-FMA-chain-per-logit arithmetic (R6) with the staging taken off the
// compute warps (DESIGN.md §6 has the measurements behind each choice).
//   * the router rows are widened once per call into an fp64 [channel][N_e padded] workspace
//     (router_widen_kernel, zero rows pad N_e);
//   * one producer thread runs an S-deep mbarrier ring: per chunk of CW channels ONE 2-D TMA box
//     of x ([kTok tokens][CW channels] bf16, 128-B / 64-B swizzle, rows >= T read as zeros) and
//     ONE bulk copy of the chunk's fp64 router rows (a copy per token row made the TMA engine's
//     per-copy cost the limit: ~33 cycles per channel at C1);
//   * NW compute warps (lane = token, TPT tokens per lane; warp w = experts [w*EPT, (w+1)*EPT))
//     wait on full[s], run their chains and release the stage (empty[s]); no block barrier in
//     the channel loop.  x stays bf16 in shared memory (2 B per token-channel instead of the 8 of round 2's v6 kernel)
//     and is widened in registers (exact bf16 -> fp32 shift, F2F.F64.F32); router operands are
//     read kWD channels ahead, x one 8-channel group ahead;
//   * the stage pointer is aligned by an offset from the shared array so operand reads stay LDS
//     (an integer-rebuilt pointer compiled to generic LD: 22 vs 16 cycles per channel at C1);
//   * top-k per thread on 64-bit integer keys (topk_rows; 4 threads per token above 16 experts).
template <int EPT, int TPT, int NW, int CW>
struct RouterV7Cfg {
    static_assert(CW == 64 || CW == 32, "x chunk = one 128-B (64 ch) or 64-B (32 ch) swizzle span");
    static constexpr int kTok = kRouteTile * TPT;
    static constexpr int kNePad = NW * EPT;
    static constexpr int kXP = CW * 2;                       // bytes per staged x row (swizzled)
    static constexpr int kXBytes = kTok * kXP;
    static constexpr int kStage = (kXBytes + CW * kNePad * 8 + 1023) / 1024 * 1024;
    static constexpr int kStages = (110 * 1024 / kStage) < 2 ? 2 : ((110 * 1024 / kStage) > 8 ? 8 : 110 * 1024 / kStage);
    static constexpr int kLgPitch = kNePad + 1;              // odd pitch: conflict-free row reads
    static constexpr size_t kSmem = 1024 + ((size_t)kStages * kStage > (size_t)kTok * kLgPitch * 8
                                                ? (size_t)kStages * kStage
                                                : (size_t)kTok * kLgPitch * 8);
};

template <int EPT, int TPT, int NW, int CW>
__global__ void __launch_bounds__((NW + 1) * 32)
router_v7_kernel(const __grid_constant__ CUtensorMap tmX, int T, int h,
                 const double* __restrict__ wr64, int ne, int k, int renorm,
                 int32_t* __restrict__ idx_out, float* __restrict__ gate_out,
                 int32_t* __restrict__ tile_counts) {
    using C = RouterV7Cfg<EPT, TPT, NW, CW>;
    static_assert((EPT == 1 || EPT % 2 == 0) && CW % 8 == 0, "shape");
    constexpr int S = C::kStages, kTok = C::kTok, kNePad = C::kNePad, kXP = C::kXP;
    constexpr uint32_t kWBytes = CW * kNePad * 8;
    constexpr int kThr = (NW + 1) * 32;
    extern __shared__ uint8_t dyn7_raw[];
    // 1024-byte aligned (the TMA swizzle span) by an OFFSET from the shared array, so the compiler
    // still knows every operand pointer is shared memory (LDS); an aligned pointer rebuilt from an
    // integer made every operand read a generic LD (ncu: long-scoreboard stalls on the DFMAs).
    uint8_t* dyn7 = dyn7_raw + ((1024u - (ptx::smem_u32(dyn7_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[S], empty[S];
    __shared__ int cnt[TPT][kMaxExperts];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t0 = blockIdx.x * kTok;
    const int n_chunks = h / CW;
    const bool probe = blockIdx.x == 0 && tid == 0;
    uint64_t clk0 = 0, ns0 = 0;
    if (probe) {
        clk0 = clock64();
        ns0 = ptx::globaltimer_ns();
        g_router_probe[4] = 0;
    }
    for (int e = tid; e < TPT * kMaxExperts; e += kThr) cnt[e / kMaxExperts][e % kMaxExperts] = 0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);    // the producer's expect_tx (+ the copies' bytes)
            ptx::mbar_init(&empty[s], NW);  // one arrive per compute warp
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();

    double acc[TPT][EPT];
#pragma unroll
    for (int p = 0; p < TPT; ++p)
#pragma unroll
        for (int i = 0; i < EPT; ++i) acc[p][i] = 0.0;

    if (warp == NW) {
        // ---------------------------------------------------------------- producer (1 thread)
        if (lane == 0) {
            ptx::prefetch_tmap(&tmX);
            for (int ch = 0; ch < n_chunks; ++ch) {
                const int s = ch % S;
                ptx::mbar_wait(&empty[s], ((ch / S) & 1) ^ 1u);
                uint8_t* st = dyn7 + (size_t)s * C::kStage;
                const int c0 = ch * CW;
                ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)(C::kXBytes + kWBytes));
                ptx::tma_load_2d(st, &tmX, &full[s], c0, t0);   // rows >= T read as zeros
                ptx::bulk_g2s(st + C::kXBytes, wr64 + (size_t)c0 * kNePad, kWBytes, &full[s]);
            }
        }
    } else {
        // ---------------------------------------------------------------- compute warps
        // Explicit register pipeline inside a chunk (fully unrolled, so every ring index is a
        // compile-time constant): router operands kWD channels ahead, x one 8-channel group
        // ahead, each channel's x widened one channel ahead.  Left to the compiler, the router
        // loads were issued one channel ahead and every channel step waited a shared-memory
        // round trip (measured 34 cycles per channel at C1).
        constexpr int kWP = EPT >= 2 ? EPT / 2 : 1;      // double2 (or double) loads per channel
        constexpr int kWD = EPT >= 8 ? 2 : 4;             // router channels in flight
        for (int ch = 0; ch < n_chunks; ++ch) {
            const int s = ch % S;
            ptx::mbar_wait(&full[s], (ch / S) & 1);
            const uint8_t* st = dyn7 + (size_t)s * C::kStage;
            // x tile: token row r at r * kXP, its 16-byte group g at (g ^ swz(r)) * 16 (the TMA
            // swizzle: 128B span -> r & 7, 64B span -> (r >> 1) & 3): lanes hit 8 distinct groups
            const uint8_t* xr = st + lane * kXP;
            const double* wc = reinterpret_cast<const double*>(st + C::kXBytes) + warp * EPT;
            double2 wv[kWD][kWP];
            auto loadw = [&](int c, int slot) {
                const double* wrow = wc + c * kNePad;
#pragma unroll
                for (int i = 0; i < kWP; ++i) {
                    if constexpr (EPT == 1) wv[slot][i].x = wrow[0];
                    else wv[slot][i] = reinterpret_cast<const double2*>(wrow)[i];
                }
            };
            constexpr int kXG = 3;                            // x groups (8 channels) in flight
            int4 xv[kXG][TPT];
            auto loadx = [&](int g, int slot) {
#pragma unroll
                for (int p = 0; p < TPT; ++p)
                    xv[slot][p] = *reinterpret_cast<const int4*>(
                        xr + p * 32 * kXP + ((g ^ (CW == 64 ? (lane & 7) : ((lane >> 1) & 3))) * 16));
            };
            constexpr int kXL = 4;                            // channels widened ahead
            double xd[kXL + 1][TPT];
            auto widen = [&](int c, int slot) {   // exact: bf16 -> fp32 (shift) -> fp64
#pragma unroll
                for (int p = 0; p < TPT; ++p) {
                    const int4& v = xv[(c >> 3) % kXG][p];
                    const int qq = c & 7;
                    const uint32_t w32 = (qq >> 1) == 0 ? (uint32_t)v.x
                                       : (qq >> 1) == 1 ? (uint32_t)v.y
                                       : (qq >> 1) == 2 ? (uint32_t)v.z
                                                        : (uint32_t)v.w;
                    xd[slot][p] = (double)__uint_as_float((qq & 1) ? (w32 & 0xffff0000u) : (w32 << 16));
                }
            };
            loadx(0, 0);
            if (CW > 8) loadx(1, 1);
#pragma unroll
            for (int c = 0; c < kWD; ++c) loadw(c, c);
#pragma unroll
            for (int c = 0; c < kXL; ++c) widen(c, c);
#pragma unroll
            for (int c = 0; c < CW; ++c) {   // channel c0 + c: ascending in every chain
                if ((c & 7) == 0 && c + 16 < CW) loadx((c >> 3) + 2, ((c >> 3) + 2) % kXG);
                if (c + kXL < CW) widen(c + kXL, (c + kXL) % (kXL + 1));
                const int xs = c % (kXL + 1);
#pragma unroll
                for (int i = 0; i < kWP; ++i) {
#pragma unroll
                    for (int p = 0; p < TPT; ++p) {
                        if constexpr (EPT == 1) {
                            acc[p][0] = fma(xd[xs][p], wv[c % kWD][0].x, acc[p][0]);
                        } else {
                            acc[p][2 * i] = fma(xd[xs][p], wv[c % kWD][i].x, acc[p][2 * i]);
                            acc[p][2 * i + 1] = fma(xd[xs][p], wv[c % kWD][i].y, acc[p][2 * i + 1]);
                        }
                    }
                }
                if (c + kWD < CW) loadw(c + kWD, c % kWD);
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[s]);
        }
        if (probe) g_router_probe[1] = clock64() - clk0;
        if (blockIdx.x == 0 && lane == 0) atomicMax(&g_router_probe[4], (unsigned long long)clock64());
    }
    __syncthreads();   // every stage consumed: the ring's memory holds the logits now
    double* lg = reinterpret_cast<double*>(dyn7);   // [kTok][kLgPitch]
    if (warp < NW) {
#pragma unroll
        for (int p = 0; p < TPT; ++p)
#pragma unroll
            for (int i = 0; i < EPT; ++i) lg[(p * 32 + lane) * C::kLgPitch + warp * EPT + i] = acc[p][i];
    }
    __syncthreads();
    if (ne > 16)   // 4 threads per token: a serial scan of 64 experts took 19% of C4's block time
        topk_rows<TPT, 4>(lg, C::kLgPitch, t0, T, ne, k, renorm, idx_out, gate_out, cnt, tid, kThr);
    else
        topk_rows<TPT, 1>(lg, C::kLgPitch, t0, T, ne, k, renorm, idx_out, gate_out, cnt, tid, kThr);
    __syncthreads();
    if (probe) g_router_probe[5] = clock64() - clk0;
    const int n_tiles = (T + kRouteTile - 1) / kRouteTile;
#pragma unroll
    for (int p = 0; p < TPT; ++p) {
        const int tile = blockIdx.x * TPT + p;
        if (tile < n_tiles)
            for (int e = tid; e < ne; e += kThr) tile_counts[(size_t)tile * ne + e] = cnt[p][e];
    }
    if (probe) {
        g_router_probe[4] -= clk0;
        g_router_probe[0] = clk0;
        g_router_probe[2] = clock64() - clk0;
        g_router_probe[3] = ptx::globaltimer_ns() - ns0;
    }
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
               int32_t* __restrict__ pos_out, const PeerRows* __restrict__ pr) {
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
        __nv_bfloat16* dst_ptr[kMaxTopK];
#pragma unroll
        for (int j = 0; j < kMaxTopK; ++j) {
            dst_ptr[j] = x_perm;
            if (j < k) {
                const int p = spos[q * k + j];
                if (pr) {   // straight into the expert owner's x_recv (P2P dispatch)
                    const int e = sidx[(tt0 + q) * k + j];
                    const int b = pr->base[e];   // -1: the plan refused the exchange (overflow)
                    dst_ptr[j] = b < 0 ? nullptr
                                       : pr->rows[e / pr->nl] + (size_t)(b + p - offsets[e]) * h;
                } else {
                    dst_ptr[j] = x_perm + (size_t)p * h;
                }
            }
        }
        // MOE_FLAG_SHARD_SHARED: the row also goes to every shared-slice owner (the gather)
        const uint32_t smask = (pr && pr->shard_row >= 0) ? pr->shard_mask : 0u;
        // 8 vectors (4 KB per warp) in flight; the destination loop is unrolled over kMaxTopK so
        // dst_ptr stays in registers (a loop to the run-time k indexed it from a local-memory
        // stack frame)
        constexpr int U = 8;
        for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
            int4 buf[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + 32 * u;
                if (v < nvec) buf[u] = ptx::ld_nc_v4(src + v);
            }
#pragma unroll
            for (int j = 0; j < kMaxTopK; ++j) {
                int4* dst = reinterpret_cast<int4*>(dst_ptr[j]);
                if (j < k && dst) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int v = v0 + 32 * u;
                        if (v < nvec) dst[v] = buf[u];
                    }
                }
            }
            for (uint32_t m = smask; m; m &= m - 1) {
                const int d = __ffs(m) - 1;
                int4* dst = reinterpret_cast<int4*>(pr->rows[d] + (size_t)(pr->shard_row + t) * h);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int v = v0 + 32 * u;
                    if (v < nvec) dst[v] = buf[u];
                }
            }
        }
    }
    if (pr) __threadfence_system();   // peer stores performed before the dispatch flag release
}

// Warp per (token, 1/split of its row); lane = 8 consecutive columns per 16-byte vector, two
// vectors per iteration with all their row loads issued first.  split (host) makes >= ~8k warps
// so small calls still keep enough loads in flight (C1: 4096 tokens -> half rows); a warp per
// 256 columns was measured slower at C1 (32 vs 23 us: each warp paid the pos -> row dependent
// round trips for a single vector per lane).
template <int K>   // top_k (compile time: the row loads of a batch sit in K * 2 registers x4)
__global__ void __launch_bounds__(256)
combine_kernel(const __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ pos,
               const float* __restrict__ gates, int T, int h, int num_shared,
               int64_t shared_base, int64_t shared_stride, const __nv_bfloat16* __restrict__ resid,
               __nv_bfloat16* __restrict__ out, const int32_t* __restrict__ idx,
               const int32_t* __restrict__ offsets, const PeerRows* __restrict__ pr,
               int shard_t0, int split) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nvec = h / 8;
    const int64_t gw = (int64_t)blockIdx.x * 8 + warp;
    const int t = (int)(gw / split);
    if (t >= T) return;
    const int per = nvec / split;               // vectors of this warp's part of the row
    const int v0 = (int)(gw % split) * per;
    const __nv_bfloat16* prow[K];
    float g[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        prow[j] = y;
        g[j] = 0.f;
        {
            const int p = pos[(size_t)t * K + j];
            g[j] = gates[(size_t)t * K + j];
            if (pr) {   // the expert owner's y_recv (P2P combine)
                const int e = idx[(size_t)t * K + j];
                const int b = pr->base[e];
                if (b < 0) {   // the plan refused the exchange (overflow): contributes nothing
                    prow[j] = y;
                    g[j] = 0.f;
                    continue;
                }
                prow[j] = pr->rows[e / pr->nl] + (size_t)(b + p - offsets[e]) * h;
            } else {
                prow[j] = y + (size_t)p * h;
            }
        }
    }
    constexpr int U = K <= 2 ? 4 : 2;   // U x K row vectors in flight per lane
    for (int vb = v0 + lane; vb < v0 + per; vb += 32 * U) {
        int4 raw[U][K];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (vb + 32 * u < v0 + per)
                    raw[u][j] = ptx::ld_nc_v4(reinterpret_cast<const int4*>(prow[j]) + vb + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = vb + 32 * u;
            if (v >= v0 + per) break;
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll
            for (int j = 0; j < K; ++j) {   // fixed j order (R10)
                {
                    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw[u][j]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 f = __bfloat1622float2(b[i]);
                        acc[2 * i] = fmaf(g[j], f.x, acc[2 * i]);
                        acc[2 * i + 1] = fmaf(g[j], f.y, acc[2 * i + 1]);
                    }
                }
            }
            // weight-1 rows after the routed terms, in call order: shared experts (or their
            // sharded partial rows, rank order), then Task B's residual
            auto add_row = [&](const __nv_bfloat16* row) {
                const int4 r = ptx::ld_nc_v4(reinterpret_cast<const int4*>(row) + v);
                const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 f = __bfloat1622float2(b[i]);
                    acc[2 * i] += f.x;
                    acc[2 * i + 1] += f.y;
                }
            };
            if (shard_t0 >= 0) {
                for (uint32_t m = pr->shard_mask; m; m &= m - 1)
                    add_row(pr->rows[__ffs(m) - 1] + (size_t)(pr->shard_row + shard_t0 + t) * h);
            } else {
                for (int s2 = 0; s2 < num_shared; ++s2)
                    add_row(y + (size_t)(shared_base + (int64_t)s2 * shared_stride + t) * h);
            }
            if (resid) add_row(resid + (size_t)t * h);
            int4 o;
            o.x = (int)ptx::pack_bf16x2(acc[0], acc[1]);
            o.y = (int)ptx::pack_bf16x2(acc[2], acc[3]);
            o.z = (int)ptx::pack_bf16x2(acc[4], acc[5]);
            o.w = (int)ptx::pack_bf16x2(acc[6], acc[7]);
            reinterpret_cast<int4*>(out + (size_t)t * h)[v] = o;
        }
    }
}

}  // namespace

// Router v3 (round 1; MOE_ROUTER=3 for comparison): x and router tiles staged in shared memory.
cudaError_t launch_router_v3(const __nv_bfloat16* x, int T, int h, const __nv_bfloat16* wr,
                            int ne, int k, int renorm, int32_t* idx, float* gates,
                            int32_t* tile_counts, cudaStream_t st) {
    const int n_tiles = (T + kRouteTile - 1) / kRouteTile;
    if (n_tiles == 0) return cudaSuccess;
    // EPT experts per warp: few experts -> fewer per warp, so a 32-token tile still spreads over
    // several warps (C1's 4096 tokens are only 128 tiles); more experts -> more per warp (fewer
    // x loads per DFMA).  Measured per call (profiles/r01/router_ept): N_e = 8 (C1): EPT 1 / 2
    // 0.15 ms, 4 0.18, 8 0.44; N_e = 16 (DBRX): EPT 2 0.64 ms, 4 0.52, 8 0.70.
    int ept = ne <= 8 ? 1 : (ne <= 16 ? 4 : 8);
    if (const char* e = getenv("MOE_ROUTER_EPT")) {   // experiments: 1, 2, 4 or 8
        const int v = atoi(e);
        const int bound = v >= 8 ? 512 : 256;          // the kernel's __launch_bounds__
        if ((v == 1 || v == 2 || v == 4 || v == 8) && ((ne + v - 1) / v) * 32 <= bound) ept = v;
    }
    const int nw = (ne + ept - 1) / ept;
    const int ne_pad = nw * ept;
    // two tokens per lane where the kernel is shared-memory bound (8 experts per warp, 3..8 warps:
    // the staging of the 64-token x tile is sized for >= 96 threads, kMinThreads)
    // (4 tokens per lane measured slower at C4: 0.84 vs 0.79 ms -- 180 registers, fewer warps)
    const int tpt = (ept == 8 && nw >= 3 && nw <= 8) ? 2 : 1;
    const size_t dyn = sizeof(double) * (size_t)(kChunk * (kRouteTile * tpt + 1) + kChunk * ne_pad);
    const int smem_max = (int)(sizeof(double) * (kChunk * (2 * kRouteTile + 1) + kChunk * kMaxExperts));
    const int blocks = (T + kRouteTile * tpt - 1) / (kRouteTile * tpt);
#define MOE_ROUTER(E, P)                                                                     \
    do {                                                                                     \
        cudaError_t e_ = cudaFuncSetAttribute(router_topk_kernel<E, P>,                      \
            cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);                          \
        if (e_ != cudaSuccess) return e_;                                                    \
        router_topk_kernel<E, P><<<blocks, nw * 32, dyn, st>>>(x, T, h, wr, ne, k, renorm,   \
                                                               idx, gates, tile_counts);     \
    } while (0)
    if (ept == 1) MOE_ROUTER(1, 1);
    else if (ept == 2) MOE_ROUTER(2, 1);
    else if (ept == 4) MOE_ROUTER(4, 1);
    else if (tpt == 2) MOE_ROUTER(8, 2);
    else MOE_ROUTER(8, 1);
#undef MOE_ROUTER
    return cudaGetLastError();
}

// N_e padded to the v7 bucket's NW * EPT (every EPT override of a bucket pads to the same width)
static int router_ne_pad(int ne) {
    int p = 8;
    while (p < ne) p *= 2;
    return p;
}

size_t router_ws_doubles(int h, int ne) { return (size_t)h * router_ne_pad(ne); }

cudaError_t router_probe(unsigned long long out[4]) {
    return cudaMemcpyFromSymbol(out, g_router_probe, 6 * sizeof(unsigned long long));
}

cudaError_t launch_router_topk(const __nv_bfloat16* x, int T, int h, const __nv_bfloat16* wr,
                               int ne, int k, int renorm, int32_t* idx, float* gates,
                               int32_t* tile_counts, double* wr64, int* launches,
                               cudaStream_t st) {
    const int n_tiles = (T + kRouteTile - 1) / kRouteTile;
    if (n_tiles == 0) return cudaSuccess;
    // MOE_ROUTER: unset / 7 = v7, 3 = round 1's kernel (comparisons; N_e <= 64)
    const char* ver = getenv("MOE_ROUTER");
    int none = 0;
    if (!launches) launches = &none;
    if (ver && atoi(ver) == 3) {
        *launches += 1;
        return launch_router_v3(x, T, h, wr, ne, k, renorm, idx, gates, tile_counts, st);
    }
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (!ver || atoi(ver) == 7) {
        const char* ev = getenv("MOE_ROUTER_EPT");
        const int ept = ev ? atoi(ev) : 0;
        int tpt = 4;
        while (tpt > 1 && (T + kRouteTile * tpt - 1) / (kRouteTile * tpt) < sms) tpt >>= 1;
        if (const char* e = getenv("MOE_ROUTER_TPT")) {
            const int v = atoi(e);
            if (v == 1 || v == 2 || v == 4) tpt = v;
        }
        if (tpt == 4 && (ne > 16 || ept == 8)) tpt = 2;   // 4 tokens x 8 experts per lane spill
        const int blocks = (T + kRouteTile * tpt - 1) / (kRouteTile * tpt);
        cudaError_t err = cudaSuccess;
#define MOE_ROUTER7(E, P, N, CW_)                                                            \
    do {                                                                                     \
        using C7 = RouterV7Cfg<E, P, N, CW_>;                                                \
        if (h % CW_ || C7::kNePad != ne_pad) return cudaErrorInvalidValue;                  \
        CUtensorMap tmX;                                                                     \
        if (!make_tmap_box(&tmX, x, (uint64_t)T, (uint64_t)h, CW_, C7::kTok))                \
            return cudaErrorInvalidValue;                                                    \
        err = cudaFuncSetAttribute(router_v7_kernel<E, P, N, CW_>,                           \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                                   (int)C7::kSmem);                                          \
        if (err != cudaSuccess) return err;                                                  \
        router_v7_kernel<E, P, N, CW_><<<blocks, (N + 1) * 32, C7::kSmem, st>>>(             \
            tmX, T, h, wr64, ne, k, renorm, idx, gates, tile_counts);                            \
    } while (0)
#define MOE_ROUTER7_TPT(E, N, CW_)                                                           \
    do {                                                                                     \
        if (tpt == 1) MOE_ROUTER7(E, 1, N, CW_);                                             \
        else if (tpt == 2) MOE_ROUTER7(E, 2, N, CW_);                                        \
        else {                                                                               \
            if constexpr (E < 8) MOE_ROUTER7(E, 4, N, CW_);                                  \
            else return cudaErrorInvalidValue;   /* 4 x 8 chains per lane: capped above */   \
        }                                                                                    \
    } while (0)
        if (!wr64) return cudaErrorInvalidValue;
        const int ne_pad = router_ne_pad(ne);
        router_widen_kernel<<<(int)std::min<int64_t>(((int64_t)h * ne_pad + 255) / 256, 1184), 256, 0, st>>>(
            wr, h, ne, ne_pad, wr64);
        *launches += 2;
        if (ne <= 8 && ept == 1) MOE_ROUTER7_TPT(1, 8, 64);
        else if (ne <= 8 && ept == 4) MOE_ROUTER7_TPT(4, 2, 64);
        else if (ne <= 8 && ept == 8) MOE_ROUTER7_TPT(8, 1, 64);
        else if (ne <= 8) MOE_ROUTER7_TPT(2, 4, 64);
        else if (ne <= 16 && ept == 8) MOE_ROUTER7_TPT(8, 2, 64);
        else if (ne <= 16) MOE_ROUTER7_TPT(4, 4, 64);
        else if (ne <= 32) MOE_ROUTER7_TPT(8, 4, 64);
        else if (ne <= 64) MOE_ROUTER7_TPT(8, 8, 32);
        else MOE_ROUTER7_TPT(8, 16, 32);
#undef MOE_ROUTER7_TPT
#undef MOE_ROUTER7
        return cudaGetLastError();
    }
    return cudaErrorInvalidValue;   // MOE_ROUTER=<unknown>
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
                           const PeerRows* pr, cudaStream_t st) {
    const int n_tiles = (T + kRouteTile - 1) / kRouteTile;
    if (n_tiles == 0) return cudaSuccess;
    permute_kernel<<<n_tiles * (kRouteTile / kPermuteTokens), 256, 0, st>>>(
        x, T, h, k, ne, idx, tile_prefix, offsets, x_perm, pos, pr);
    return cudaGetLastError();
}

cudaError_t launch_combine(const __nv_bfloat16* y_perm, const int32_t* pos, const float* gates,
                           int T, int h, int k, int num_shared, int64_t shared_base,
                           int64_t shared_stride, const __nv_bfloat16* resid, __nv_bfloat16* out,
                           const int32_t* idx, const int32_t* offsets, const PeerRows* pr,
                           int shard_t0, cudaStream_t st) {
    if (T == 0) return cudaSuccess;
    if (shard_t0 >= 0 && !pr) return cudaErrorInvalidValue;
    // parts per row: >= ~8k warps in flight, each part a multiple of 32 vectors
    int split = 1;
    while (split < 8 && (int64_t)T * split < 8192 && (h / 8) % (64 * split) == 0) split *= 2;
    const int64_t warps = (int64_t)T * split;
    const unsigned blocks = (unsigned)((warps + 7) / 8);
#define MOE_COMBINE(KK)                                                                      \
    combine_kernel<KK><<<blocks, 256, 0, st>>>(y_perm, pos, gates, T, h, num_shared,         \
                                               shared_base, shared_stride, resid, out, idx,  \
                                               offsets, pr, shard_t0, split)
    switch (k) {
        case 1: MOE_COMBINE(1); break;
        case 2: MOE_COMBINE(2); break;
        case 3: MOE_COMBINE(3); break;
        case 4: MOE_COMBINE(4); break;
        case 5: MOE_COMBINE(5); break;
        case 6: MOE_COMBINE(6); break;
        case 7: MOE_COMBINE(7); break;
        case 8: MOE_COMBINE(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef MOE_COMBINE
    return cudaGetLastError();
}

}  // namespace moe
