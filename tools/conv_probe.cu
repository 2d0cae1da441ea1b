// conv_probe.cu -- latency of the router's per-channel operations on this GPU (tools only):
// F2F.F64.F32 (bf16 -> fp64 widening), the shared-memory load round trip, and the DFMA chain.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/conv_probe.cu -o build/conv_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// dependent F2F.F64.F32 -> (hi word) -> shift chain: cycles per step = F2F latency + one ALU op
__global__ void f2f_chain(unsigned* out, int iters, long long* cyc) {
    unsigned x = 0x3f80u + threadIdx.x;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const double d = (double)__uint_as_float(x << 16);
        x = (unsigned)__double2hiint(d) >> 13;   // depends on the conversion
    }
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

// dependent shared-memory loads (pointer chase): cycles per step = LDS latency
__global__ void lds_chain(unsigned* out, int iters, long long* cyc) {
    __shared__ unsigned s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    unsigned j = threadIdx.x;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) j = s[j];
    const long long t1 = clock64();
    out[threadIdx.x] = j;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

// the router's step: acc = fma(widen(x_c), w_c, acc) with x_c, w_c independent of acc (x from a
// register stream, w from shared memory): cycles per step with everything off the chain
__global__ void router_step(double* out, int iters, long long* cyc) {
    __shared__ double w[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) w[i] = 1.0 + i * 1e-6;
    __syncthreads();
    double acc = 0;
    unsigned x = 0x3f80u + threadIdx.x;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < iters; ++i) {
        const double xd = (double)__uint_as_float((x + i) << 16);
        acc = fma(xd, w[i & 255], acc);
    }
    const long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

// F2F throughput: 8 independent conversions per step, `warps` warps on one SM
__global__ void f2f_tput(double* out, int iters, long long* cyc) {
    unsigned x[8];
    double s[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { x[j] = 0x3f80u + threadIdx.x + j; s[j] = 0; }
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] += (double)__uint_as_float((x[j] + i) << 16);
    }
    const long long t1 = clock64();
    double t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += s[j];
    out[threadIdx.x] = t;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <typename K, typename T>
void run(const char* name, K kern, int threads, int iters, double per) {
    T* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(T) * 1024);
    cudaMalloc(&cyc, sizeof(long long));
    kern<<<1, threads>>>(out, iters, cyc);
    kern<<<1, threads>>>(out, iters, cyc);
    long long c = 0;
    cudaError_t e = cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    printf("%-44s threads %4d: %.2f cycles per step (%s)\n", name, threads, (double)c / iters / per,
           cudaGetErrorString(e));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<decltype(&f2f_chain), unsigned>("F2F.F64.F32 + shift chain", f2f_chain, 32, 1 << 14, 1);
    run<decltype(&lds_chain), unsigned>("LDS pointer chase", lds_chain, 32, 1 << 14, 1);
    run<decltype(&router_step), double>("router step (widen + LDS + DFMA)", router_step, 32, 1 << 14, 1);
    run<decltype(&router_step), double>("router step (widen + LDS + DFMA)", router_step, 128, 1 << 14, 1);
    run<decltype(&f2f_tput), double>("F2F + DADD, 8 independent (per conversion)", f2f_tput, 32, 1 << 12, 8);
    run<decltype(&f2f_tput), double>("F2F + DADD, 8 independent (per conversion)", f2f_tput, 128, 1 << 12, 8);
    run<decltype(&f2f_tput), double>("F2F + DADD, 8 independent (per conversion)", f2f_tput, 512, 1 << 12, 8);
    return 0;
}
