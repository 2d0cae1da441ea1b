/*
 * moe_oracle.c -- plain, slow, obviously-correct CPU oracle of the MoE layer that MoE-Lens
 * (arXiv 2504.09345) leaves to the GPU ("GPU Task B ... MoE layer ... applied to all tokens",
 * PAPER.md:636).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header, table or helper with
 * paper_2504_09345_b200/ (the CUDA path) and never includes anything from it.
 *
 * What it computes (the paper defers the layer's math to prior work; DESIGN.md
 * "Readings" R1-R10 give the standard Mixtral/DBRX block this follows):
 *   1. router logits  l[t,e] = sum_{c=0}^{h-1} (double)x[t,c] * (double)Wr[e,c], ascending c, fp64
 *      ("routing each input through a small subset of expert networks", PAPER.md:37;
 *       N_e experts, top-N_k per token, dimension h).  Reading R6: fp64.
 *   2. S_t = first N_k experts under the order (l desc, e asc)  (reading R5: lowest index wins ties).
 *   3. gates g[t,j] = exp(l_j - l_0) / sum_j' exp(l_j' - l_0)  over the selected experts (fp64,
 *      stored fp32) when renormalize=1 (reading R3); softmax over all N_e otherwise.
 *   4. expert e on token t (three h x h_i matrices per expert, Eq. 1 "6 N_k h h_i"):
 *      a = W1_e x_t, b = W3_e x_t, u = silu(a) * b, v = W2_e u   (reading R2), fp32 ascending sums.
 *   5. y_t = sum_{j=0}^{N_k-1} g[t,j] v_{t,j}  (fixed j order)  +  sum_s v_{t,s}  for shared experts
 *      (weight 1, not renormalised; reading R10).
 * bf16 operands are given as uint16 bit patterns and upcast exactly.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline float bf16_to_f32(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

int moe_ref_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the following calls (bench.py's one-thread baseline); the
 * arithmetic is per output element and does not depend on it. */
void moe_ref_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Step 1: router logits, fp64 accumulation in ascending c.  logits: [T, n_experts]. */
void moe_ref_router_logits(const uint16_t* x, int64_t T, int32_t h, const uint16_t* router,
                           int32_t n_experts, double* logits) {
    int64_t t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < T; ++t) {
        for (int32_t e = 0; e < n_experts; ++e) {
            double acc = 0.0;
            for (int32_t c = 0; c < h; ++c)
                acc += (double)bf16_to_f32(x[t * h + c]) * (double)bf16_to_f32(router[(int64_t)e * h + c]);
            logits[t * n_experts + e] = acc;
        }
    }
}

/* "a ranks above b": larger logit, or equal logit and smaller index.  NaN ranks last. */
static int ranks_above(double la, int32_t a, double lb, int32_t b) {
    if (isnan(lb) && !isnan(la)) return 1;
    if (isnan(la)) return isnan(lb) ? (a < b) : 0;
    if (la > lb) return 1;
    if (la < lb) return 0;
    return a < b;
}

/* Steps 2-3: top-k selection (l desc, e asc) and softmax gates.  idx, gates: [T, top_k]. */
void moe_ref_topk_gates(const double* logits, int64_t T, int32_t n_experts, int32_t top_k,
                        int32_t renormalize, int32_t* idx, float* gates) {
    int64_t t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < T; ++t) {
        const double* l = logits + t * n_experts;
        int32_t chosen[64 + 1];
        unsigned char taken[1024];
        memset(taken, 0, sizeof taken);
        for (int32_t j = 0; j < top_k; ++j) {
            int32_t best = -1;
            for (int32_t e = 0; e < n_experts; ++e) {
                if (taken[e]) continue;
                if (best < 0 || ranks_above(l[e], e, l[best], best)) best = e;
            }
            taken[best] = 1;
            chosen[j] = best;
            idx[t * top_k + j] = best;
        }
        double m = l[chosen[0]];
        double z = 0.0;
        if (renormalize) {
            for (int32_t j = 0; j < top_k; ++j) z += exp(l[chosen[j]] - m);
        } else {
            for (int32_t e = 0; e < n_experts; ++e) z += exp(l[e] - m);
        }
        for (int32_t j = 0; j < top_k; ++j) gates[t * top_k + j] = (float)(exp(l[chosen[j]] - m) / z);
    }
}

/* Step 4: one token through one SwiGLU expert, fp32.  u: scratch [ffn]; v: out [h]. */
void moe_ref_expert_ffn(const uint16_t* x_row, int32_t h, const uint16_t* w1, const uint16_t* w3,
                        const uint16_t* w2, int32_t ffn, float* u, float* v) {
    for (int32_t i = 0; i < ffn; ++i) {
        float a = 0.0f, b = 0.0f;
        for (int32_t c = 0; c < h; ++c) {
            float xc = bf16_to_f32(x_row[c]);
            a += bf16_to_f32(w1[(int64_t)i * h + c]) * xc;
            b += bf16_to_f32(w3[(int64_t)i * h + c]) * xc;
        }
        float silu = a / (1.0f + expf(-a));
        u[i] = silu * b;
    }
    for (int32_t r = 0; r < h; ++r) {
        float acc = 0.0f;
        for (int32_t i = 0; i < ffn; ++i) acc += bf16_to_f32(w2[(int64_t)r * ffn + i]) * u[i];
        v[r] = acc;
    }
}

/* Step 5 given routing: y[t] = sum_j g[t,j] * FFN_{idx[t,j]}(x_t) + sum_s FFN_shared_s(x_t).
 * w1/w3/w2: arrays of (n_experts + n_shared) pointers, routed experts first.  y: [T, h] fp32. */
void moe_ref_experts_combine(const uint16_t* x, int64_t T, int32_t h, int32_t ffn,
                             const uint16_t* const* w1, const uint16_t* const* w3,
                             const uint16_t* const* w2, int32_t n_experts, int32_t n_shared,
                             const int32_t* idx, const float* gates, int32_t top_k, float* y) {
    int64_t t;
#pragma omp parallel
    {
        float* u = (float*)malloc(sizeof(float) * (size_t)ffn);
        float* v = (float*)malloc(sizeof(float) * (size_t)h);
#pragma omp for schedule(dynamic, 1)
        for (t = 0; t < T; ++t) {
            const uint16_t* xr = x + t * h;
            float* yr = y + t * h;
            for (int32_t c = 0; c < h; ++c) yr[c] = 0.0f;
            for (int32_t j = 0; j < top_k; ++j) {
                int32_t e = idx[t * top_k + j];
                float g = gates[t * top_k + j];
                moe_ref_expert_ffn(xr, h, w1[e], w3[e], w2[e], ffn, u, v);
                for (int32_t c = 0; c < h; ++c) yr[c] += g * v[c];
            }
            for (int32_t s = 0; s < n_shared; ++s) {
                int32_t e = n_experts + s;
                moe_ref_expert_ffn(xr, h, w1[e], w3[e], w2[e], ffn, u, v);
                for (int32_t c = 0; c < h; ++c) yr[c] += v[c];
            }
        }
        free(u);
        free(v);
    }
}

/* The whole layer.  logits (optional, may be NULL): [T, n_experts] fp64.  Returns 0 on success,
 * 1 on invalid arguments (top_k outside [1, min(n_experts, 64)], n_experts > 1024, etc.). */
int moe_ref_forward(const uint16_t* x, int64_t T, int32_t h, const uint16_t* router,
                    int32_t n_experts, int32_t top_k, int32_t renormalize,
                    const uint16_t* const* w1, const uint16_t* const* w3, const uint16_t* const* w2,
                    int32_t ffn, int32_t n_shared, float* y, int32_t* idx, float* gates,
                    double* logits) {
    if (T < 0 || h <= 0 || ffn <= 0 || n_experts <= 0 || n_experts > 1024 || top_k < 1 ||
        top_k > n_experts || top_k > 64 || n_shared < 0)
        return 1;
    if (T == 0) return 0;
    double* l = logits ? logits : (double*)malloc(sizeof(double) * (size_t)T * (size_t)n_experts);
    if (!l) return 2;
    moe_ref_router_logits(x, T, h, router, n_experts, l);
    moe_ref_topk_gates(l, T, n_experts, top_k, renormalize, idx, gates);
    moe_ref_experts_combine(x, T, h, ffn, w1, w3, w2, n_experts, n_shared, idx, gates, top_k, y);
    if (!logits) free(l);
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * GPU Task B ("GPU Task B (GB), which includes the O projection and MoE layer, is
 * applied to all tokens").  Between the two the standard pre-norm decoder block of the paper's
 * models (Mixtral, DBRX) has a residual add and the post-attention RMSNorm; DESIGN.md readings:
 *   R19  h1 = resid + attn Wo^T (Wo [h, h], nn.Linear out x in); y = h1 + MoE(u).
 *   R20  h1 is stored as bf16 (the model's residual stream dtype), rounded once:
 *        h1 = bf16(float(sum_i attn[t,i] Wo[c,i] + resid[t,c])), the sum in fp64, ascending i.
 *   R21  u = RMSNorm(h1) * gamma:  r = 1 / sqrt(sum_c h1^2 / h + eps) (fp64, ascending c),
 *        n = bf16(float(h1 * r)),  u = bf16(float(gamma) * float(n))  (fp32 multiply).
 * bf16 rounding is round-to-nearest-even (NaN kept quiet).
 * ------------------------------------------------------------------------------------------ */
static uint16_t f32_to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, sizeof u);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* NaN */
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

/* b1 (R19, R20).  attn, resid, h1: [T, h] bf16 bits; wo: [h, h] bf16 bits. */
void moe_ref_oproj_residual(const uint16_t* attn, const uint16_t* resid, int64_t T, int32_t h,
                            const uint16_t* wo, uint16_t* h1) {
    int64_t t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < T; ++t) {
        for (int32_t c = 0; c < h; ++c) {
            double acc = 0.0;
            for (int32_t i = 0; i < h; ++i)
                acc += (double)bf16_to_f32(attn[t * h + i]) * (double)bf16_to_f32(wo[(int64_t)c * h + i]);
            acc += (double)bf16_to_f32(resid[t * h + c]);
            h1[t * h + c] = f32_to_bf16((float)acc);
        }
    }
}

/* b2 (R21).  h1, u: [T, h] bf16 bits; gamma: [h] bf16 bits. */
void moe_ref_rmsnorm(const uint16_t* h1, int64_t T, int32_t h, const uint16_t* gamma, float eps,
                     uint16_t* u) {
    int64_t t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < T; ++t) {
        double ss = 0.0;
        for (int32_t c = 0; c < h; ++c) {
            const double x = (double)bf16_to_f32(h1[t * h + c]);
            ss += x * x;
        }
        const double r = 1.0 / sqrt(ss / (double)h + (double)eps);
        for (int32_t c = 0; c < h; ++c) {
            const double x = (double)bf16_to_f32(h1[t * h + c]);
            const float n = bf16_to_f32(f32_to_bf16((float)(x * r)));
            u[t * h + c] = f32_to_bf16(bf16_to_f32(gamma[c]) * n);
        }
    }
}

/* The whole Task B: h1 (b1), u (b2), the MoE layer on u, y = float(h1) + MoE(u) (fp32).
 * h1, u: [T, h] bf16 bits out; y: [T, h] fp32 out; idx/gates as moe_ref_forward. */
int moe_ref_taskb_forward(const uint16_t* attn, const uint16_t* resid, int64_t T, int32_t h,
                          const uint16_t* wo, const uint16_t* gamma, float eps,
                          const uint16_t* router, int32_t n_experts, int32_t top_k,
                          int32_t renormalize, const uint16_t* const* w1, const uint16_t* const* w3,
                          const uint16_t* const* w2, int32_t ffn, int32_t n_shared, uint16_t* h1,
                          uint16_t* u, float* y, int32_t* idx, float* gates) {
    if (T < 0 || h <= 0 || !(eps >= 0.0f)) return 1;
    if (T == 0) return 0;
    moe_ref_oproj_residual(attn, resid, T, h, wo, h1);
    moe_ref_rmsnorm(h1, T, h, gamma, eps, u);
    int rc = moe_ref_forward(u, T, h, router, n_experts, top_k, renormalize, w1, w3, w2, ffn,
                             n_shared, y, idx, gates, NULL);
    if (rc != 0) return rc;
    for (int64_t i = 0; i < T * (int64_t)h; ++i) y[i] = bf16_to_f32(h1[i]) + y[i];
    return 0;
}
