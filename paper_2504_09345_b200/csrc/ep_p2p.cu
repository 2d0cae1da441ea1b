// ep_p2p.cu -- expert parallelism over peer memory (NVLink P2P across the GPUs of one box, or
// the same GPU for in-process ranks): the dispatch is fused into the permute kernel (each token
// row is written straight into its expert owner's x_recv) and the combine reads the owners'
// y_recv directly -- no staging copies, no collective library, no host synchronisation.
//
// Per call n on rank r (all on r's compute stream, in this order):
//   push counts[n%2][r] to every peer, release kFlagCounts = n      (p2p_push_counts)
//   wait kFlagCounts >= n from every rank                           (p2p_wait)
//   plan: GEMM groups over x_recv + send bases                       (p2p_plan)
//   wait kFlagXFree >= n-1 (owners finished GEMM1 of call n-1)
//   permute+dispatch into the owners' x_recv, release kFlagDispatched = n
//   wait kFlagDispatched >= n, wait kFlagYDone >= n-1 (sources finished reading y_recv of n-1)
//   expert GEMMs (weights streamed as usual) -> y_recv
//   release kFlagXFree = n, kFlagYReady = n; wait kFlagYReady >= n
//   combine reading the owners' y_recv, release kFlagYDone = n
// Every wait is for a signal its peers issue EARLIER in their own program order (or in call n-1),
// so the protocol cannot deadlock; the counts buffer is double-buffered by call parity.
#include "moe_internal.h"

namespace moe {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void p2p_push_counts_kernel(const P2PTable* __restrict__ tab,
                                       const int32_t* __restrict__ counts, int ne, int W, int me,
                                       int par, unsigned long long seq) {
    for (int i = threadIdx.x; i < W * ne; i += blockDim.x) {
        const int d = i / ne, e = i % ne;
        tab->counts[d][((size_t)par * W + me) * ne + e] = counts[e];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < W) st_release_sys(tab->flags[threadIdx.x] + kFlagCounts * kMaxRanks + me, seq);
}

__global__ void p2p_signal_kernel(const P2PTable* __restrict__ tab, int W, int me, int which,
                                  unsigned long long val) {
    if (threadIdx.x < W) {
        __threadfence_system();
        st_release_sys(tab->flags[threadIdx.x] + which * kMaxRanks + me, val);
    }
}

__global__ void p2p_wait_kernel(const unsigned long long* __restrict__ flags, int W, int which,
                                unsigned long long val, long long* __restrict__ diag) {
    if (threadIdx.x < W) {
        const unsigned long long* f = flags + which * kMaxRanks + threadIdx.x;
        const long long t0 = clock64();
        unsigned long long v;
        while ((v = ld_acquire_sys(f)) < val) {
            __nanosleep(256);
            if (clock64() - t0 > 40000000000ll) {   // ~20 s: a peer is gone or the group is stuck
                if (diag) {   // host-mapped: survives the trap, reported by moe_sync
                    diag[1] = which;
                    diag[2] = threadIdx.x;
                    diag[3] = (long long)val;
                    diag[4] = (long long)v;
                    __threadfence_system();
                    diag[0] = 1;
                    __threadfence_system();
                }
                __trap();
            }
        }
    }
    __syncthreads();
}

__global__ void p2p_plan_kernel(const int32_t* __restrict__ counts, int W, int ne, int me, int T,
                                int k, int S, long long cap_recv, int n_all, int h,
                                GemmGroup* __restrict__ grp, PeerRows* __restrict__ pr_x,
                                PeerRows* __restrict__ pr_y, int32_t* __restrict__ rows_out,
                                long long* __restrict__ bytes_acc,
                                long long* __restrict__ diag, int shard_item) {
    const int nl = ne / W;
    // Every owner must be able to hold the rows routed to it: each rank checks every owner's
    // total (the counts are the same on every rank, so all ranks agree).  With consistent
    // configurations (max_tokens, top_k equal on all ranks; checked at connect) this cannot
    // fail; if it does, nothing is dispatched (send bases -1, empty groups) instead of writing
    // past a peer's buffer, and moe_sync reports the overflow.
    __shared__ long long worst;
    if (threadIdx.x == 0) worst = 0;
    __syncthreads();
    for (int d = threadIdx.x; d < W; d += blockDim.x) {
        long long tot = 0;
        for (int q = 0; q < W; ++q)
            for (int l = 0; l < nl; ++l) tot += counts[(size_t)q * ne + d * nl + l];
        atomicMax(&worst, tot);
    }
    __syncthreads();
    const bool overflow = worst > cap_recv;
    // send bases: where this rank's block for expert e = d*nl + le starts in owner d's x_recv
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        const int d = e / nl, le = e % nl;
        long long b = 0;
        for (int l = 0; l < le; ++l)
            for (int q = 0; q < W; ++q) b += counts[(size_t)q * ne + d * nl + l];
        for (int q = 0; q < me; ++q) b += counts[(size_t)q * ne + e];
        pr_x->base[e] = overflow ? -1 : (int32_t)b;
        pr_y->base[e] = overflow ? -1 : (int32_t)b;
    }
    if (threadIdx.x == 0) {
        if (overflow && diag) {   // host-mapped: reported by moe_sync / the next call
            diag[6] = worst;
            diag[7] = cap_recv;
            __threadfence_system();
            diag[5] = 1;
            __threadfence_system();
        }
        // receive side: expert-major groups (local expert, source rank, source token order)
        int off = 0;
        for (int le = 0; le < nl; ++le) {
            int cnt = 0;
            for (int q = 0; q < W; ++q) cnt += counts[(size_t)q * ne + me * nl + le];
            if (overflow) cnt = 0;
            grp[le] = GemmGroup{off, off + cnt, off, 0};
            grp[n_all + le] = grp[le];
            off += cnt;
        }
        *rows_out = off;
        long long shard_rows = 0;
        if (shard_item >= 0) {
            // MOE_FLAG_SHARD_SHARED: rank q's tokens sit at rows cap_recv + P_q of every slice
            // owner's x_recv / y_recv (P_q = sum of the earlier ranks' T; T_q = its routed rows
            // / k, read from the counts every rank already has)
            long long P = 0, tot = 0;
            for (int q = 0; q < W; ++q) {
                long long rq = 0;
                for (int e = 0; e < ne; ++e) rq += counts[(size_t)q * ne + e];
                if (q < me) P += rq / k;
                tot += rq / k;
            }
            pr_x->shard_row = pr_y->shard_row = (int32_t)(cap_recv + P);
            if ((pr_x->shard_mask >> me) & 1u) {   // this rank's slice over all W ranks' tokens
                const int hb = (int)cap_recv;
                grp[shard_item] = GemmGroup{hb, (int)(hb + tot), hb, 0};
                grp[n_all + shard_item] = GemmGroup{hb, (int)(hb + tot), hb, 0};
            }
            shard_rows = (long long)__popc(pr_x->shard_mask) * T;
        } else {
            for (int s = 0; s < S; ++s) {   // shared experts (replicated): the local tokens
                const int hb = (int)(cap_recv + (long long)s * T);
                grp[nl + s] = GemmGroup{0, T, hb, 0};
                grp[n_all + nl + s] = GemmGroup{hb, hb + T, T * k + s * T, 0};
            }
        }
        long long sent = 0;
        for (int e = 0; e < ne; ++e) sent += counts[(size_t)me * ne + e];
        // rows written to the owners + read back in the combine (and the shared gather / sum)
        if (!overflow) *bytes_acc += 2 * (sent + shard_rows) * h * 2;
    }
}

__global__ void p2p_selftest_kernel(const P2PTable* __restrict__ tab,
                                    const PeerRows* __restrict__ pr_x,
                                    const unsigned long long* __restrict__ my_flags,
                                    const uint32_t* __restrict__ my_xrecv, int W, int me,
                                    unsigned long long token, long long timeout_cycles,
                                    int* __restrict__ result) {
    const int d = threadIdx.x;
    if (d == 0) *result = 0;
    if (d < W) {   // my word in peer d's x_recv: tag | (me << 8) | d
        volatile uint32_t* w = reinterpret_cast<uint32_t*>(pr_x->rows[d]) + me;
        *w = 0x5E1F0000u | ((uint32_t)me << 8) | (uint32_t)d;
    }
    __threadfence_system();
    __syncthreads();
    if (d < W) st_release_sys(tab->flags[d] + kFlagSelftest * kMaxRanks + me, token);
    if (d < W) {
        const unsigned long long* f = my_flags + kFlagSelftest * kMaxRanks + d;
        const long long t0 = clock64();
        bool ok = true;
        while (ld_acquire_sys(f) < token) {
            __nanosleep(256);
            if (clock64() - t0 > timeout_cycles) {
                ok = false;
                break;
            }
        }
        if (!ok) {
            atomicOr(result, 1 << d);
        } else {
            const uint32_t want = 0x5E1F0000u | ((uint32_t)d << 8) | (uint32_t)me;
            if (reinterpret_cast<const volatile uint32_t*>(my_xrecv)[d] != want)
                atomicOr(result, 1 << (8 + d));
        }
    }
}

}  // namespace

cudaError_t launch_p2p_selftest(const P2PTable* tab, const PeerRows* pr_x,
                                const unsigned long long* my_flags, const uint32_t* my_xrecv,
                                int W, int me, unsigned long long token,
                                long long timeout_cycles, int* result, cudaStream_t st) {
    p2p_selftest_kernel<<<1, 32, 0, st>>>(tab, pr_x, my_flags, my_xrecv, W, me, token,
                                          timeout_cycles, result);
    return cudaGetLastError();
}

cudaError_t launch_p2p_push_counts(const P2PTable* tab, const int32_t* counts, int ne, int W,
                                   int me, int par, unsigned long long seq, cudaStream_t st) {
    p2p_push_counts_kernel<<<1, 256, 0, st>>>(tab, counts, ne, W, me, par, seq);
    return cudaGetLastError();
}

cudaError_t launch_p2p_signal(const P2PTable* tab, int W, int me, int which,
                              unsigned long long val, cudaStream_t st) {
    p2p_signal_kernel<<<1, 32, 0, st>>>(tab, W, me, which, val);
    return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const unsigned long long* flags, int W, int which,
                            unsigned long long val, long long* diag, cudaStream_t st) {
    p2p_wait_kernel<<<1, 32, 0, st>>>(flags, W, which, val, diag);
    return cudaGetLastError();
}

cudaError_t launch_p2p_plan(const int32_t* counts_par, int W, int ne, int me, int T, int k,
                            int S, long long cap_recv, int n_all, int h, GemmGroup* grp,
                            PeerRows* pr_x, PeerRows* pr_y, int32_t* rows_out,
                            long long* bytes_acc, long long* diag, int shard_item,
                            cudaStream_t st) {
    p2p_plan_kernel<<<1, 128, 0, st>>>(counts_par, W, ne, me, T, k, S, cap_recv, n_all, h, grp,
                                       pr_x, pr_y, rows_out, bytes_acc, diag, shard_item);
    return cudaGetLastError();
}

}  // namespace moe
