/*
 * moe_layer.c -- the C ABI (include/moe.h) used from plain C99, no Python: one streamed MoE
 * layer call on host token buffers (moe_layer_forward_host), inputs from files.
 *
 *   usage: moe_layer <dir> <hidden> <ffn> <experts> <top_k> <shared> <tokens>
 *   reads  <dir>/x.bin       bf16 [tokens, hidden]
 *          <dir>/router.bin  bf16 [experts, hidden]
 *          <dir>/experts.bin per expert (routed, then shared): W1 [ffn, hidden], W3 [ffn, hidden],
 *                            W2 [hidden, ffn], bf16 row-major (nn.Linear orientation)
 *   writes <dir>/out.bin     bf16 [tokens, hidden]
 *          <dir>/idx.bin     int32 [tokens, top_k]
 *
 * Build: gcc -std=c99 -O2 -I include -I /usr/local/cuda/include examples/moe_layer.c \
 *            -L paper_2504_09345_b200 -lmoe_b200 -L /usr/local/cuda/lib64 -lcudart -o moe_layer
 * (tests/test_abi_cpu.py builds it; tests/test_gpu_parity.py runs it against the oracle.)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "moe.h"

static int read_file(const char* dir, const char* name, void* dst, size_t bytes) {
    char path[4096];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE* f = fopen(path, "rb");
    if (!f) return -1;
    const size_t n = fread(dst, 1, bytes, f);
    fclose(f);
    return n == bytes ? 0 : -1;
}

static int write_file(const char* dir, const char* name, const void* src, size_t bytes) {
    char path[4096];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE* f = fopen(path, "wb");
    if (!f) return -1;
    const size_t n = fwrite(src, 1, bytes, f);
    fclose(f);
    return n == bytes ? 0 : -1;
}

#define CHECK(expr)                                                                   \
    do {                                                                              \
        moe_status s_ = (expr);                                                       \
        if (s_ != MOE_OK) {                                                           \
            fprintf(stderr, "%s: %s (%s)\n", #expr, moe_status_string(s_),           \
                    ctx ? moe_last_error(ctx) : "");                                  \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

int main(int argc, char** argv) {
    moe_ctx ctx = NULL;
    if (argc != 8) {
        fprintf(stderr, "usage: %s <dir> <hidden> <ffn> <experts> <top_k> <shared> <tokens>\n", argv[0]);
        return 2;
    }
    const char* dir = argv[1];
    const int h = atoi(argv[2]), hi = atoi(argv[3]), ne = atoi(argv[4]), k = atoi(argv[5]);
    const int S = atoi(argv[6]), T = atoi(argv[7]);
    const int n_all = ne + S;
    const size_t wbytes = (size_t)hi * h * 2, xbytes = (size_t)T * h * 2;

    moe_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.hidden = h;
    cfg.ffn = hi;
    cfg.num_experts = ne;
    cfg.top_k = k;
    cfg.num_shared = S;
    cfg.max_tokens = T;
    cfg.renormalize = 1;
    cfg.world_size = 1;
    CHECK(moe_init(&cfg, &ctx));

    /* pinned, packed expert blobs (moe_pack_expert from the canonical matrices) */
    const int64_t blob = moe_packed_expert_bytes(h, hi);
    void** blobs = calloc((size_t)n_all, sizeof(void*));
    uint8_t* canon = malloc(3 * wbytes * (size_t)n_all);
    if (!blobs || !canon || read_file(dir, "experts.bin", canon, 3 * wbytes * (size_t)n_all)) {
        fprintf(stderr, "cannot read experts.bin\n");
        return 1;
    }
    for (int i = 0; i < n_all; ++i) {
        const uint8_t* e = canon + 3 * wbytes * (size_t)i;
        CHECK(moe_host_alloc((size_t)blob, &blobs[i]));
        CHECK(moe_pack_expert(h, hi, e, e + wbytes, e + 2 * wbytes, blobs[i]));
    }
    free(canon);

    /* router on the device; tokens and result in pinned host memory */
    void *router_h = malloc((size_t)ne * h * 2), *router_d = NULL, *x_h = NULL, *out_h = NULL;
    int32_t* idx_d = NULL;
    if (!router_h || read_file(dir, "router.bin", router_h, (size_t)ne * h * 2)) return 1;
    if (cudaMalloc(&router_d, (size_t)ne * h * 2) != cudaSuccess ||
        cudaMemcpy(router_d, router_h, (size_t)ne * h * 2, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMalloc((void**)&idx_d, sizeof(int32_t) * (size_t)T * k) != cudaSuccess) {
        fprintf(stderr, "CUDA allocation failed\n");
        return 1;
    }
    CHECK(moe_host_alloc(xbytes, &x_h));
    CHECK(moe_host_alloc(xbytes, &out_h));
    if (read_file(dir, "x.bin", x_h, xbytes)) return 1;

    CHECK(moe_layer_forward_host(ctx, x_h, T, router_d, (const void* const*)blobs, k, out_h,
                                 idx_d, NULL, NULL));
    CHECK(moe_sync(ctx));   /* out_h is complete after moe_sync */

    int32_t* idx_h = malloc(sizeof(int32_t) * (size_t)T * k);
    if (!idx_h || cudaMemcpy(idx_h, idx_d, sizeof(int32_t) * (size_t)T * k,
                             cudaMemcpyDeviceToHost) != cudaSuccess)
        return 1;
    if (write_file(dir, "out.bin", out_h, xbytes) || write_file(dir, "idx.bin", idx_h, sizeof(int32_t) * (size_t)T * k))
        return 1;

    moe_stats st;
    CHECK(moe_get_stats(ctx, &st));
    printf("moe_layer: %d tokens, %d experts (+%d shared), top-%d: %lld weight bytes streamed\n",
           T, ne, S, k, (long long)st.h2d_weight_bytes);
    CHECK(moe_destroy(ctx));
    for (int i = 0; i < n_all; ++i) moe_host_free(blobs[i]);
    moe_host_free(x_h);
    moe_host_free(out_h);
    cudaFree(router_d);
    cudaFree(idx_d);
    free(blobs);
    free(router_h);
    free(idx_h);
    return 0;
}
