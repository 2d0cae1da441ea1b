// router_bench.cu -- time the router + top-k kernel alone on random bf16 inputs (tools only).
// usage: router_bench T h N_e k [iters]   (MOE_ROUTER=3 / MOE_ROUTER_EPT / MOE_ROUTER_TPT select
// the kernel as in the library)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc
//        tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "moe_internal.h"

__global__ void fill(__nv_bfloat16* p, size_t n, unsigned seed, float scale) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned x = (unsigned)i * 2654435761u ^ seed;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        p[i] = __float2bfloat16(((x & 0xFFFFFF) / 16777216.0f - 0.5f) * scale);
    }
}

int main(int argc, char** argv) {
    const int T = argc > 1 ? atoi(argv[1]) : 4096, h = argc > 2 ? atoi(argv[2]) : 4096;
    const int ne = argc > 3 ? atoi(argv[3]) : 8, k = argc > 4 ? atoi(argv[4]) : 2;
    const int iters = argc > 5 ? atoi(argv[5]) : 20;
    __nv_bfloat16 *x, *w;
    int32_t *idx, *tc;
    float* g;
    cudaMalloc(&x, (size_t)T * h * 2);
    cudaMalloc(&w, (size_t)ne * h * 2);
    cudaMalloc(&idx, (size_t)T * k * 4);
    cudaMalloc(&g, (size_t)T * k * 4);
    cudaMalloc(&tc, (size_t)((T + 31) / 32) * ne * 4);
    double* wr64;
    cudaMalloc(&wr64, sizeof(double) * moe::router_ws_doubles(h, ne));
    int nl = 0;
    fill<<<1024, 256>>>(x, (size_t)T * h, 1, 3.f);
    fill<<<64, 256>>>(w, (size_t)ne * h, 2, 0.03f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // launches captured in a CUDA graph: the timing excludes the host-side launch path
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int i = 0; i < 3; ++i) moe::launch_router_topk(x, T, h, w, ne, k, 1, idx, g, tc, wr64, &nl, s);
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < iters; ++i) moe::launch_router_topk(x, T, h, w, ne, k, 1, idx, g, tc, wr64, &nl, s);
    cudaStreamEndCapture(s, &graph);
    cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphLaunch(exec, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(exec, s);
    cudaEventRecord(e1, s);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err == cudaSuccess) err = cudaGetLastError();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // bitwise check against round 1's kernel (v3) on the same inputs
    int32_t* idx3;
    float* g3;
    cudaMalloc(&idx3, (size_t)T * k * 4);
    cudaMalloc(&g3, (size_t)T * k * 4);
    moe::launch_router_v3(x, T, h, w, ne, k, 1, idx3, g3, tc, 0);
    cudaDeviceSynchronize();
    std::vector<int32_t> a((size_t)T * k), b((size_t)T * k);
    std::vector<float> ga((size_t)T * k), gb((size_t)T * k);
    cudaMemcpy(a.data(), idx, a.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), idx3, b.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ga.data(), g, ga.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(gb.data(), g3, gb.size() * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < a.size(); ++i) bad += (a[i] != b[i]) || (memcmp(&ga[i], &gb[i], 4) != 0);
    const double dfma = (double)T * ne * h;
    printf("router T=%d h=%d N_e=%d k=%d [MOE_ROUTER=%s EPT=%s TPT=%s LANES=%s]: %.1f us  %.2f TFLOP/s fp64 (%s; %zu of %zu idx/gates differ from v3)\n",
           T, h, ne, k, getenv("MOE_ROUTER") ? getenv("MOE_ROUTER") : "default",
           getenv("MOE_ROUTER_EPT") ? getenv("MOE_ROUTER_EPT") : "auto",
           getenv("MOE_ROUTER_TPT") ? getenv("MOE_ROUTER_TPT") : "auto",
           getenv("MOE_ROUTER_LANES") ? getenv("MOE_ROUTER_LANES") : "auto", 1e3 * ms / iters,
           2 * dfma / (ms / iters * 1e-3) / 1e12, cudaGetErrorString(err), bad, a.size());
    unsigned long long pr[6] = {0, 0, 0, 0, 0, 0};
    if ((!getenv("MOE_ROUTER") || atoi(getenv("MOE_ROUTER")) == 7) && ne <= 64 && moe::router_probe(pr) == cudaSuccess && pr[3])
        printf("    block 0: %llu cycles (loop %llu = %.1f per channel, last warp %llu, top-k done %llu), %.2f us, %.0f MHz\n",
               pr[2], pr[1], (double)pr[1] / h, pr[4], pr[5], pr[3] * 1e-3, (double)pr[2] / pr[3] * 1e3);
    return 0;
}
