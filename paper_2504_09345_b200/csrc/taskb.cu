// taskb.cu -- token-wise kernels of GPU Task B ("GPU Task B (GB), which includes
// the O projection and MoE layer, is applied to all tokens").  The O-projection itself runs on
// the expert GEMM (gemm.cu, residual epilogue); this file holds the post-attention RMSNorm that
// sits between it and the MoE layer in the Mixtral/DBRX block (readings R19-R21).
#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

// Warp per token, 8 tokens per 256-thread block; lane handles 8 consecutive columns per 16-byte
// vector.  Arithmetic is fixed by reading R21 and uses only correctly rounded IEEE operations
// (explicit _rn intrinsics, no contraction), so the result does not depend on the GPU:
//   ss = sum_c h1[t,c]^2 in fp64 (butterfly order; every square is exact in fp64),
//   r  = 1 / sqrt(ss / h + eps),  n = bf16(float(h1 * r)),  u = bf16(float(gamma) * float(n)).
__global__ void __launch_bounds__(256)
rmsnorm_kernel(const __nv_bfloat16* __restrict__ h1, const __nv_bfloat16* __restrict__ gamma,
               int T, int h, double eps, __nv_bfloat16* __restrict__ u) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 8 + warp;
    if (t >= T) return;
    const int4* row = reinterpret_cast<const int4*>(h1 + (size_t)t * h);
    const int4* gv = reinterpret_cast<const int4*>(gamma);
    int4* dst = reinterpret_cast<int4*>(u + (size_t)t * h);
    const int nvec = h / 8;
    double ss = 0.0;
    for (int v = lane; v < nvec; v += 32) {
        const int4 raw = row[v];
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(b[i]);
            ss = __dadd_rn(ss, __dmul_rn((double)f.x, (double)f.x));
            ss = __dadd_rn(ss, __dmul_rn((double)f.y, (double)f.y));
        }
    }
    // xor butterfly: partners add the same two values (a+b == b+a), so all lanes agree bitwise
#pragma unroll
    for (int o = 16; o; o >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    const double r = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(ss, (double)h), eps)));
    for (int v = lane; v < nvec; v += 32) {
        const int4 raw = row[v];
        const int4 graw = gv[v];
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
        const __nv_bfloat162* g = reinterpret_cast<const __nv_bfloat162*>(&graw);
        uint32_t o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(b[i]);
            const float2 w = __bfloat1622float2(g[i]);
            const float n0 = __bfloat162float(__float2bfloat16_rn(__double2float_rn(__dmul_rn((double)f.x, r))));
            const float n1 = __bfloat162float(__float2bfloat16_rn(__double2float_rn(__dmul_rn((double)f.y, r))));
            o[i] = ptx::pack_bf16x2(__fmul_rn(w.x, n0), __fmul_rn(w.y, n1));
        }
        dst[v] = make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]);
    }
}

__global__ void fill_group_kernel(GemmGroup* g, int a_begin, int a_end, int out_base) {
    *g = GemmGroup{a_begin, a_end, out_base, 0};
}

__global__ void fill_shared_groups_kernel(GemmGroup* g, int n_local, int n_all, int S, int T,
                                          int hbase, int ybase) {
    const int s = threadIdx.x;
    if (s < S) {
        const int hb = hbase + s * T;
        g[n_local + s] = GemmGroup{0, T, hb, 0};
        g[n_all + n_local + s] = GemmGroup{hb, hb + T, ybase + s * T, 0};
    }
}

}  // namespace

cudaError_t launch_rmsnorm(const __nv_bfloat16* h1, const __nv_bfloat16* gamma, int T, int h,
                           float eps, __nv_bfloat16* u, cudaStream_t st) {
    if (T == 0) return cudaSuccess;
    if (h % 8) return cudaErrorInvalidValue;
    rmsnorm_kernel<<<(T + 7) / 8, 256, 0, st>>>(h1, gamma, T, h, (double)eps, u);
    return cudaGetLastError();
}

cudaError_t launch_fill_group(GemmGroup* g, int a_begin, int a_end, int out_base, cudaStream_t st) {
    fill_group_kernel<<<1, 1, 0, st>>>(g, a_begin, a_end, out_base);
    return cudaGetLastError();
}

cudaError_t launch_fill_shared_groups(GemmGroup* g, int n_local, int n_all, int S, int T,
                                      int hbase, int ybase, cudaStream_t st) {
    fill_shared_groups_kernel<<<1, 32, 0, st>>>(g, n_local, n_all, S, T, hbase, ybase);
    return cudaGetLastError();
}

}  // namespace moe
