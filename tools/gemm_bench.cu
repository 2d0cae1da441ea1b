// gemm_bench.cu -- microbenchmark of the expert GEMM kernels on one synthetic group (tools only):
//   pair  : tokens as M (CTA pair, 256x256 tiles), weights as N
//   single: tokens as M (1 CTA, 128x256 tiles)
// usage: gemm_bench ROWS [K=4096] [NW=28672] [MODE=0 swiglu|1 plain] [ITERS=20]
// (ROWS may be a comma-separated list of groups, all in ONE launch)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc
//        tools/gemm_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/gemm_bench
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "moe_internal.h"

namespace moe {
bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
}

int main(int argc, char** argv) {
    std::vector<int> rlist;
    for (const char* p = argc > 1 ? argv[1] : "1053"; *p;) {
        rlist.push_back(atoi(p));
        while (*p && *p != ',') ++p;
        if (*p == ',') ++p;
    }
    const int K = argc > 2 ? atoi(argv[2]) : 4096;
    const int NW = argc > 3 ? atoi(argv[3]) : 28672;
    const int mode = argc > 4 ? atoi(argv[4]) : 0;
    const int iters = argc > 5 ? atoi(argv[5]) : 20;
    const int n = (int)rlist.size();
    int rows = 0;
    std::vector<moe::GemmGroup> g(n);
    for (int i = 0; i < n; ++i) {
        g[i] = moe::GemmGroup{rows, rows + rlist[i], rows, 0};
        rows += rlist[i];
    }
    __nv_bfloat16 *A, *B, *out;
    cudaMalloc(&A, (size_t)rows * K * 2);
    cudaMalloc(&B, (size_t)n * NW * K * 2);
    const int ocols = mode == 0 ? NW / 2 : NW;
    cudaMalloc(&out, (size_t)rows * ocols * 2);
    cudaMemset(A, 0, (size_t)rows * K * 2);
    cudaMemset(B, 0, (size_t)n * NW * K * 2);
    moe::GemmGroup* dg;
    cudaMalloc(&dg, sizeof(moe::GemmGroup) * n);
    cudaMemcpy(dg, g.data(), sizeof(moe::GemmGroup) * n, cudaMemcpyHostToDevice);
    moe::GemmBatch b{};
    b.table = dg;
    b.n = n;
    for (int i = 0; i < n; ++i) {
        b.idx[i] = i;
        b.b_row[i] = i * NW;
    }
    CUtensorMap tA, tB, tB128;
    moe::make_tmap(&tA, A, rows, K, 128);
    moe::make_tmap(&tB, B, (uint64_t)n * NW, K, 256);
    moe::make_tmap(&tB128, B, (uint64_t)n * NW, K, 128);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double flops = (double)rows * NW * K * 2.0;
    const char* names[2] = {"pair", "single"};
    for (int v = 0; v < 2; ++v) {
        auto launch = [&]() {
            if (v == 0) return moe::launch_expert_gemm(mode, 256, true, &tA, &tB128, b, NW, K, out, ocols, nullptr, sms, 0);
            return moe::launch_expert_gemm(mode, 256, false, &tA, &tB, b, NW, K, out, ocols, nullptr, sms, 0);
        };
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < iters; ++i) launch();
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-6s groups=%d rows=%d K=%d N=%d mode=%d: %.1f us  %.0f TFLOP/s  (%s)\n", names[v], n,
               rows, K, NW, mode, 1e3 * ms / iters, flops / (ms / iters * 1e-3) / 1e12,
               cudaGetErrorString(err));
    }
    cudaFree(A); cudaFree(B); cudaFree(out); cudaFree(dg);
    return 0;
}
