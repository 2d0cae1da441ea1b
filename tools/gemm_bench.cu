// gemm_bench.cu -- microbenchmark of the expert GEMM kernels on one synthetic group (tools only):
//   pair  : tokens as M (CTA pair, 256x256 tiles), weights as N
//   single: tokens as M (1 CTA, 128x256 tiles)
//   swap  : weights as M (CTA pair), tokens as N (32..256 per tile)
//   pairts: pair kernel with swap-AB tail tiles (GemmBatch::tail_swap, cost $TAILCOST or 0.6)
//   pairalt: pair kernel that may pick 224 / 192-wide tiles (PairBMaps)
//   auto  : pair + single kernel launched together, the device picks (GemmBatch::select)
// usage: gemm_bench ROWS [K=4096] [NW=28672] [MODE=0 swiglu|1 plain] [ITERS=20]
// (ROWS may be a comma-separated list)
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
    const float tail_cost = getenv("TAILCOST") ? (float)atof(getenv("TAILCOST")) : 0.6f;
    for (int rows : rlist) {
    __nv_bfloat16 *A, *B, *out;
    cudaMalloc(&A, (size_t)rows * K * 2);
    cudaMalloc(&B, (size_t)NW * K * 2);
    const int ocols = mode == 0 ? NW / 2 : NW;
    cudaMalloc(&out, (size_t)rows * ocols * 2);
    cudaMemset(A, 0, (size_t)rows * K * 2);
    cudaMemset(B, 0, (size_t)NW * K * 2);
    moe::GemmGroup g{0, rows, 0, 0};
    moe::GemmGroup* dg;
    cudaMalloc(&dg, sizeof g);
    cudaMemcpy(dg, &g, sizeof g, cudaMemcpyHostToDevice);
    moe::GemmBatch b{};
    b.table = dg;
    b.n = 1;
    CUtensorMap tA, tB, tB128, tW;
    moe::TokenMaps tX;
    moe::make_tmap(&tA, A, rows, K, 128);
    moe::make_tmap(&tB, B, NW, K, 256);
    moe::make_tmap(&tB128, B, NW, K, 128);
    moe::make_tmap(&tW, B, NW, K, 128);
    moe::make_token_maps(&tX, A, rows, K);
    moe::PairBMaps alt;
    moe::make_tmap(&alt.b224, B, NW, K, 112);
    moe::make_tmap(&alt.b192, B, NW, K, 96);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double flops = (double)rows * NW * K * 2.0;
    const char* names[6] = {"pair", "single", "swap", "pairts", "pairalt", "auto"};
    for (int v = 0; v < 6; ++v) {
        auto launch = [&]() {
            if (v == 4) {
                moe::GemmBatch ba = b;
                ba.alt_ok = 1;
                return moe::launch_expert_gemm(mode, 256, true, &tA, &tB128, ba, NW, K, out, ocols, nullptr, sms, 0, nullptr, &alt);
            }
            if (v == 5) {
                moe::GemmBatch ba = b;
                ba.alt_ok = 1;
                ba.select = sms;
                ba.bn_single = 256;
                cudaError_t e = moe::launch_expert_gemm(mode, 256, true, &tA, &tB128, ba, NW, K, out, ocols, nullptr, sms, 0, nullptr, &alt);
                if (e != cudaSuccess) return e;
                return moe::launch_expert_gemm(mode, 256, false, &tA, &tB, ba, NW, K, out, ocols, nullptr, sms, 0);
            }
            if (v == 3) {
                moe::GemmBatch bt = b;
                bt.tail_swap = 1;
                bt.tail_cost = tail_cost;
                return moe::launch_expert_gemm(mode, 256, true, &tA, &tB128, bt, NW, K, out, ocols, nullptr, sms, 0, &tX);
            }
            if (v == 0) return moe::launch_expert_gemm(mode, 256, true, &tA, &tB128, b, NW, K, out, ocols, nullptr, sms, 0);
            if (v == 1) return moe::launch_expert_gemm(mode, 256, false, &tA, &tB, b, NW, K, out, ocols, nullptr, sms, 0);
            return moe::launch_expert_gemm_swap(mode, &tW, &tX, b, NW, K, out, ocols, nullptr, sms, 0);
        };
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < iters; ++i) launch();
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-6s rows=%d K=%d N=%d mode=%d: %.1f us  %.0f TFLOP/s  (%s)\n", names[v], rows, K, NW,
               mode, 1e3 * ms / iters, flops / (ms / iters * 1e-3) / 1e12, cudaGetErrorString(err));
    }
    cudaFree(A); cudaFree(B); cudaFree(out); cudaFree(dg);
    }
    return 0;
}
