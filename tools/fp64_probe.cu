// fp64_probe.cu -- DFMA latency / throughput on this GPU (router design input; tools only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_probe.cu -o build/fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_chain(double* out, int iters, long long* cycles) {
    double a[CHAINS];
    const double x = 1.0000001 + threadIdx.x * 1e-9, y = 0.9999999;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = c * 1e-3;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = fma(a[c], x, y);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int CHAINS>
void run(int blocks, int threads, int iters) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long));
    dfma_chain<CHAINS><<<blocks, threads>>>(out, iters, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_chain<CHAINS><<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    const double dfma = (double)blocks * threads * iters * CHAINS;
    printf("chains/thread %2d blocks %4d threads %4d: %.2f cycles per dependent step (block 0), "
           "%.2f TFLOP/s fp64 (FMA = 2)\n", CHAINS, blocks, threads, (double)c / iters,
           2.0 * dfma / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<1>(1, 32, 1 << 16);     // latency: one warp, one chain
    run<4>(1, 32, 1 << 16);
    run<8>(1, 32, 1 << 16);
    run<1>(148, 128, 1 << 14);  // one chain per lane, 4 warps per SM
    run<1>(148, 256, 1 << 14);
    run<2>(148, 256, 1 << 14);
    run<4>(148, 256, 1 << 14);
    run<8>(148, 256, 1 << 14);
    run<4>(296, 512, 1 << 13);
    return 0;
}
