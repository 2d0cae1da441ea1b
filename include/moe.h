/*
 * moe.h -- C ABI of the B200-native streamed-weight MoE layer (arXiv 2504.09345, "MoE-Lens").
 *
 * The operation ("GPU Task B (GB), which includes the O projection and MoE layer,
 * is applied to all tokens"; reading R1-R10 in DESIGN.md fix the layer's math, which the paper
 * defers to prior work):
 *
 *   logits[t,e] = sum_c x[t,c] * Wr[e,c]                  (router GEMM, fp64 accumulation)
 *   S_t         = top-k experts by (logit desc, index asc) (softmax top-k gating)
 *   g[t,j]      = softmax over the k selected logits       (renormalised; cfg.renormalize)
 *   y[t]        = sum_j g[t,j] * W2_e (silu(W1_e x_t) * W3_e x_t)  + shared experts (weight 1)
 *
 * Expert weights live in pinned host memory ("All weights are stored in pinned CPU memory",
 * PAPER.md:823) and are streamed into a bounded GPU buffer ("two times the model weight size
 * divided by the number of layers", PAPER.md:824-825 -- here N expert-sized slots, at most
 * ~512 MiB, always fewer than the experts of a call) on every call, prefetched ahead by an
 * asynchronous copy stream.
 *
 * Conventions (all entry points):
 *   - No C++ types or exceptions cross this boundary.  Every entry point returns a moe_status.
 *   - Validation is synchronous and happens before anything is enqueued; on MOE_E_INVAL nothing
 *     is written.  Asynchronous CUDA errors surface at the next call or at moe_sync().
 *   - Ownership: the caller owns every pointer it passes (hidden, router_w, out, topk_*, host
 *     expert blobs).  The library owns its workspace, the staging slots, its internal streams,
 *     events and (world_size > 1) its NCCL communicator.
 *   - Lifetime: calls are asynchronous w.r.t. the host.  Host expert blobs and every argument
 *     buffer must stay valid and unmodified until `stream` has passed the call (or moe_sync()).
 *   - A context is bound to one device and is not thread-safe.
 *   - Determinism: for fixed inputs and world_size the outputs are bitwise reproducible.
 */
#ifndef MOE_B200_H_
#define MOE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct moe_ctx_s* moe_ctx;

typedef enum {
    MOE_OK = 0,
    MOE_E_INVAL = 1,        /* bad argument: shape, top_k, num_tokens > max_tokens, aliasing    */
    MOE_E_CUDA = 2,         /* CUDA runtime/driver error (detail in moe_last_error)              */
    MOE_E_NCCL = 3,         /* NCCL error (world_size > 1)                                       */
    MOE_E_NOMEM = 4,        /* device or pinned-host allocation failed                           */
    MOE_E_NOT_PINNED = 5,   /* an expert blob is pageable host memory                            */
    MOE_E_UNSUPPORTED = 6,  /* shape outside the kernels' envelope (see moe_config)              */
    MOE_E_STATE = 7         /* call on a context in an error state / wrong order                 */
} moe_status;

/* Flags for moe_config.flags */
#define MOE_FLAG_PROFILE 1u  /* record CUDA events around every kernel and copy (moe_get_stats) */
#define MOE_FLAG_FORCE_EP 2u /* world_size == 1: still run the expert-parallel exchange through a
                                one-rank NCCL communicator (tests the EP path on one GPU)        */
#define MOE_FLAG_LOCAL_EP 4u /* expert parallelism among `world_size` contexts of ONE process
                                (one host thread per rank; the GPUs of one box, or one GPU):
                                the P2P transport -- the permute kernel writes each token row
                                straight into its expert owner's receive buffer, the combine
                                kernel reads the owners' results, device flags order the calls
                                (no host sync, no NCCL).  nccl_unique_id points to a 128-byte
                                group key shared by the ranks.                                    */
#define MOE_FLAG_IPC_EP 8u   /* the P2P transport across PROCESSES (one per GPU, e.g. torchrun):
                                buffers are shared with CUDA IPC -- call moe_ep_ipc_handle on
                                every rank, all-gather the handles, then moe_ep_ipc_connect
                                before the first forward call.  Takes precedence over NCCL.      */
#define MOE_FLAG_MOVER 16u   /* the Contiguous Data Mover: expert copies are cut
                                into packets of packet_bytes (0 = 100 MB) and issued by a
                                library thread with at most one packet in flight (
                                MOE_MOVER_INFLIGHT=n for n), so a caller's token copy
                                (moe_layer_forward_host) waits behind one packet, not behind
                                every expert copy already requested.  The copies and the GEMMs
                                are ordered by device counters (stream memory operations);
                                MOE_E_UNSUPPORTED if the driver lacks them.                      */
#define MOE_FLAG_SHARD_SHARED 32u /* shared experts SHARDED across the expert-parallel group
                                 instead of replicated on every rank.  Needs
                                the P2P transport (LOCAL_EP / IPC_EP), world_size > 1 and
                                1 <= num_shared <= world_size.  The S
                                shared experts are one FFN of width S*ffn (their concatenation,
                                DESIGN.md reading R10) and a SwiGLU FFN is a sum over blocks of
                                its intermediate columns:  W2 (silu(W1 x) * W3 x) =
                                sum_B W2[:,B] (silu(W1[B] x) * W3[B] x).  Rank r streams only
                                the column slice moe_shared_slice() gives it (~S*ffn/W wide, so
                                the per-rank host bytes are the algorithmic total / W); the
                                permute kernel also writes every local token row into every
                                slice owner (the all-gather, over peer memory), each owner runs
                                its slice over all ranks' tokens, and the combine kernel of the
                                token's rank adds the owners' partial rows in rank order (fp32)
                                -- the reduce-scatter.  Output differs from the replicated
                                layout by summation order only (within the same 2e-2 bar).      */

/*
 * Layer configuration.  Envelope of the sm_100a kernels (MOE_E_UNSUPPORTED otherwise):
 *   hidden % 128 == 0, ffn % 128 == 0, 1 <= num_experts <= 128, 1 <= top_k <= min(num_experts, 8),
 *   0 <= num_shared <= 8, max_tokens >= 1.
 * Multi-GPU expert parallelism (world_size > 1): num_experts % world_size == 0; rank r owns the
 * routed experts [r*N_e/W, (r+1)*N_e/W); shared experts are replicated on every rank, or
 * sharded by intermediate columns with MOE_FLAG_SHARD_SHARED.
 */
typedef struct {
    int32_t hidden;           /* h                                          */
    int32_t ffn;              /* h_i  (expert intermediate dimension)                          */
    int32_t num_experts;      /* N_e  routed experts                                           */
    int32_t top_k;            /* N_k  experts per token                                        */
    int32_t num_shared;       /* always-on experts with weight 1 (DeepSeek-style; 0 = none)    */
    int32_t max_tokens;       /* per-rank token capacity used to size the workspace            */
    int32_t renormalize;      /* 1: gates = softmax over the top-k (sum to 1); 0: full softmax */
    int32_t device;           /* CUDA device ordinal                                           */
    int32_t world_size;       /* expert-parallel group size; 1 = single GPU                    */
    int32_t rank;             /* this process's rank in the group                              */
    const void* nccl_unique_id; /* 128-byte ncclUniqueId (world_size > 1), else NULL           */
    int64_t packet_bytes;     /* 0 = one DMA per expert; else H2D packets of this size          */
    uint32_t flags;           /* MOE_FLAG_*                                                    */
    int32_t num_slots;        /* expert staging slots, 2..32 (must be < streamed experts per
                                 call when > 2); 0 = auto: enough slots to hold ~512 MiB of
                                 weights (2 for Mixtral-size experts, 32 for DeepSeek-V2-Lite-
                                 size ones).  The paper's buffer is two LAYERS;
                                 slots are recycled every call, so weights are always re-streamed. */
} moe_config;

/* Packed host blob of one expert (produced by moe_pack_expert, consumed by the copy engine):
 *   [ W13 : 2*h_i rows x h bf16, gate/up rows interleaved in blocks of 16 rows:
 *           rows [32j, 32j+16) = W1 rows [16j, 16j+16), rows [32j+16, 32j+32) = W3 rows
 *           [16j, 16j+16) -- every 32 accumulator columns (tokens-as-M GEMM) or every warp's
 *           32 TMEM lanes (weights-as-M GEMM) hold matching gate and up rows, so the SwiGLU is
 *           applied in the GEMM epilogue in either operand role ]
 *   [ W2  : h rows x h_i bf16 (canonical nn.Linear orientation) ]
 * Size in bytes = 6 * h * h_i  (Eq. 1 denominator per expert). */
int64_t moe_packed_expert_bytes(int32_t hidden, int32_t ffn);

/* Host-side, synchronous.  Canonical bf16 (uint16 bit patterns) W1,W3: [h_i, h] row-major,
 * W2: [h, h_i] row-major  ->  dst (moe_packed_expert_bytes bytes, any host memory).
 * MOE_E_INVAL on NULL pointers or non-positive / unsupported shapes. */
moe_status moe_pack_expert(int32_t hidden, int32_t ffn, const void* w1, const void* w3,
                           const void* w2, void* dst);

/* MOE_FLAG_SHARD_SHARED: the columns [*col0, *col0 + *width) of the concatenated shared
 * intermediate dimension (num_shared * ffn wide; shared expert s holds columns [s*ffn,
 * (s+1)*ffn)) that rank `rank` of `world` serves.  The concatenation's B = num_shared*ffn/128
 * blocks of 128 columns are split evenly in rank order: rank r takes blocks
 * [floor(r*B/W), floor((r+1)*B/W)), so widths differ by at most 128 and may be 0.
 * The rank's slice blob is moe_pack_expert(hidden, *width, W1s, W3s, W2s) with W1s / W3s = rows
 * [col0, col0 + width) of the shared experts' row-stacked W1 / W3 ([S*ffn, h]) and W2s = columns
 * [col0, col0 + width) of their column-concatenated W2 ([h, S*ffn]); it is the last entry of the
 * rank's `experts` array (no entry when *width == 0).  Host-only, synchronous.
 * MOE_E_INVAL on NULL outputs, ffn % 128 != 0, num_shared < 1, world < 1 or rank outside
 * [0, world). */
moe_status moe_shared_slice(int32_t ffn, int32_t num_shared, int32_t world, int32_t rank,
                            int32_t* col0, int32_t* width);

/* Pinned host allocation helpers (cudaHostAlloc, portable).  The blobs passed to
 * moe_layer_forward must be page-locked; these are one way to get such memory. */
moe_status moe_host_alloc(size_t bytes, void** ptr);
moe_status moe_host_free(void* ptr);

/* Create a context on cfg->device: validates cfg, allocates the workspace for max_tokens
 * tokens, cfg->num_slots (0 = auto, ~512 MiB) staging slots of moe_packed_expert_bytes each, the
 * copy stream and events, and (world_size > 1) the NCCL communicator.  *out is NULL on failure:
 * MOE_E_INVAL (bad cfg), MOE_E_UNSUPPORTED (outside the envelope or not an sm_100 device),
 * MOE_E_NOMEM, MOE_E_CUDA, MOE_E_NCCL. */
moe_status moe_init(const moe_config* cfg, moe_ctx* out);

/*
 * One MoE layer over this rank's tokens, enqueued on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  Returns after enqueueing (asynchronous).
 *   hidden      device bf16 [num_tokens, h] row-major (local tokens); must not alias `out`.
 *   num_tokens  0 <= T <= max_tokens (0 = no-op).
 *   router_w    device bf16 [N_e, h] row-major (all routed experts, on every rank).
 *   experts     host array of (N_e/W + num_shared) pointers to PINNED packed blobs: this rank's
 *               routed experts in increasing expert id, then the shared experts.  With
 *               MOE_FLAG_SHARD_SHARED: N_e/W routed blobs, then the rank's shared slice blob
 *               (moe_shared_slice) if its width is not 0.
 *   top_k       must equal cfg->top_k.
 *   out         device bf16 [num_tokens, h].
 *   topk_idx    optional device int32 [num_tokens, top_k] (NULL = not returned): the selected
 *               experts of each token in rank order (logit desc, index asc).
 *   topk_w      optional device fp32 [num_tokens, top_k]: the gates, same order.
 * Errors: MOE_E_INVAL (shapes/aliasing/NULL), MOE_E_NOT_PINNED, MOE_E_CUDA, MOE_E_NCCL.
 */
moe_status moe_layer_forward(moe_ctx ctx, const void* hidden, int32_t num_tokens,
                             const void* router_w, const void* const* experts, int32_t top_k,
                             void* out, int32_t* topk_idx, float* topk_w, void* stream);

/*
 * Same as moe_layer_forward with HOST token buffers: hidden_host (pinned bf16 [T,h]) is copied
 * to the device on the copy stream ahead of the call's expert weights, and the result is copied
 * back into out_host (pinned bf16 [T,h]) on the library's result-copy stream once the call's
 * combine has run -- work enqueued on `stream` after the call does NOT wait for that copy.
 * out_host is complete when moe_sync() returns, or once `stream` passes a moe_wait_output()
 * issued after the call.  topk_* are optional DEVICE buffers as above (written in `stream`
 * order).  End-to-end entry point (bench "e2e").
 */
moe_status moe_layer_forward_host(moe_ctx ctx, const void* hidden_host, int32_t num_tokens,
                                  const void* router_w, const void* const* experts, int32_t top_k,
                                  void* out_host, int32_t* topk_idx, float* topk_w, void* stream);

/*
 * GPU Task B: "GPU Task B (GB), which includes the O projection and MoE
 * layer, is applied to all tokens"; the layer-wise weights are streamed from host
 * memory like the experts ("weights ... are placed in CPU memory ... transferred to the GPU
 * layer by layer").  Around the two operations sits the standard pre-norm decoder
 * block of the paper's models (Mixtral/DBRX; readings R19-R21):
 *   h1 = bf16(resid + attn Wo^T)                     O-projection + residual (one rounding)
 *   u  = RMSNorm(h1) * gamma                         post-attention norm (R21 arithmetic)
 *   out = bf16(h1 + MoE(u))                          the MoE layer of moe_layer_forward + residual
 *
 * Packed layer blob (pinned host): Wo bf16 [h, h] row-major (nn.Linear out x in), then gamma
 * bf16 [h]; moe_packed_layer_bytes(h) = 2h^2 + 2h bytes.
 */
int64_t moe_packed_layer_bytes(int32_t hidden);
moe_status moe_pack_layer(int32_t hidden, const void* wo, const void* gamma, void* dst);

/*
 * One Task B over this rank's tokens, enqueued on `stream` (asynchronous, like
 * moe_layer_forward; the two share the context's staging and must be issued in program order).
 *   attn        device bf16 [T, h]: attention output (heads concatenated), the O-proj input.
 *   resid       device bf16 [T, h]: residual stream entering the block's attention half.
 *   layer       pinned host packed layer blob (above), streamed each call into one of two
 *               device slots ahead of this call's expert weights.
 *   eps         RMSNorm epsilon (>= 0, finite).
 *   router_w, experts, top_k, topk_idx, topk_w: as moe_layer_forward (routing is on u).
 *   out         device bf16 [T, h]; may alias attn and/or resid (both are consumed first).
 * The intermediate h1 and u of the last call are exposed by moe_debug_buffers.
 * Errors: MOE_E_INVAL, MOE_E_NOT_PINNED, MOE_E_NOMEM (first call allocates 2 layer slots and
 * 2 x max_tokens x h bf16 of workspace), MOE_E_CUDA, MOE_E_NCCL.
 */
moe_status moe_taskb_forward(moe_ctx ctx, const void* attn, const void* resid, int32_t num_tokens,
                             const void* layer, float eps, const void* router_w,
                             const void* const* experts, int32_t top_k, void* out,
                             int32_t* topk_idx, float* topk_w, void* stream);

/*
 * Same as moe_taskb_forward with the attention output and the result in HOST memory -- the
 * paper's pipeline, where attention runs on the CPU and its output is moved
 * to the GPU for Task B.  attn_host (pinned bf16 [T, h]) is copied on the copy stream ahead of
 * the call's layer and expert weights; out_host (pinned bf16 [T, h]) receives the result (D2H
 * ordered on `stream`).  resid stays on the device (the residual stream lives on the GPU).
 * End-to-end entry point of `bench.py --taskb` ("e2e").
 */
moe_status moe_taskb_forward_host(moe_ctx ctx, const void* attn_host, const void* resid,
                                  int32_t num_tokens, const void* layer, float eps,
                                  const void* router_w, const void* const* experts, int32_t top_k,
                                  void* out_host, int32_t* topk_idx, float* topk_w, void* stream);

/* Enqueue on `stream` a wait for the result copies (into out_host) of every host-buffer call
 * issued so far on this context; `stream` may be any stream of the context's device. */
moe_status moe_wait_output(moe_ctx ctx, void* stream);

/*
 * GPU Task B over TWO token partitions through ONE stream of the layer's weights -- VSLPipe's
 * alpha / beta groups ("partitions them into two groups, alpha and beta ... In
 * each phase, CPU-side attention computations for one partition run concurrently with GPU-side
 * GEMM operations for the other"; the data mover keeps the attention transfers from being
 * head-of-line blocked by weight packets).  Partition p in {0 = alpha,
 * 1 = beta} has num_tokens[p] >= 0 tokens; attn_host[p] (pinned bf16 [T_p, h]), resid[p] (device
 * bf16 [T_p, h]) and out_host[p] (pinned bf16 [T_p, h]) as moe_taskb_forward_host.  Order:
 *   alpha's attention copy; Wo|gamma (streamed once); alpha's O-projection + norm; the call's first
 *   expert copies; THEN beta's attention copy (with MOE_FLAG_MOVER it waits behind at most one
 *   weight packet, else behind those expert copies); beta's O-projection + norm; routing over
 *   T_0 + T_1 tokens; every expert streamed once, its GEMMs covering both partitions' rows;
 *   alpha's rows combined first and copied back while beta's rows are combined.
 * topk_idx / topk_w: optional device [T_0 + T_1, k], alpha's rows then beta's.  The outputs are
 * bitwise those of moe_taskb_forward_host on each partition in turn, for one layer's weight
 * traffic.  T_0 + T_1 <= max_tokens; either may be 0 (then this is moe_taskb_forward_host).
 * Per-partition token-copy latencies: moe_stats.part_latency_ms (MOE_FLAG_PROFILE).
 */
moe_status moe_taskb_forward2_host(moe_ctx ctx, const void* const attn_host[2],
                                   const void* const resid[2], const int32_t num_tokens[2],
                                   const void* layer, float eps, const void* router_w,
                                   const void* const* experts, int32_t top_k,
                                   void* const out_host[2], int32_t* topk_idx, float* topk_w,
                                   void* stream);

/* Block until all work of the context is done; returns the first pending async error. */
moe_status moe_sync(moe_ctx ctx);

/* Per-context counters.  Times are sums of CUDA-event durations (MOE_FLAG_PROFILE only; 0
 * otherwise), measured on the stream each kernel / copy was launched on. */
typedef struct {
    int64_t calls;
    int64_t h2d_weight_bytes;     /* expert bytes copied host -> device                       */
    int64_t h2d_token_bytes;      /* hidden bytes copied (moe_layer_forward_host)             */
    int64_t d2h_token_bytes;      /* output bytes copied back (moe_layer_forward_host)        */
    int64_t kernel_launches;      /* launches of this library's kernels                       */
    int64_t gemm1_launches, gemm2_launches;
    double h2d_ms;                /* sum of weight-copy durations (copy stream)               */
    double route_ms, permute_ms, gemm1_ms, gemm2_ms, combine_ms, comm_ms;
    int64_t num_slots;            /* expert staging slots in use                              */
    int64_t comm_bytes;           /* bytes this rank sent in EP dispatch + combine            */
    int64_t host_calls;           /* host-buffer calls (moe_*_host)                            */
    double token_latency_ms;      /* sum over host calls: enqueue -> tokens resident on the GPU */
    int64_t taskb_calls;          /* moe_taskb_forward calls (each also counts in `calls`)    */
    double oproj_ms, norm_ms;     /* Task B: O-projection GEMM, RMSNorm                       */
    /* Mean SM clock while the expert GEMMs ran (MOE_FLAG_PROFILE): clock64 cycles / globaltimer
     * ns of CTA 0 from its first to its last instruction, summed over launches -- the clock the
     * tensor-core roofline of those kernels must be scaled to (power management).  0 = none. */
    double gemm1_sm_mhz, gemm2_sm_mhz;
    /* Host token copies per partition (0: the only / alpha partition, 1: beta of
     * moe_taskb_forward2_host) and their summed enqueue -> resident latency (MOE_FLAG_PROFILE);
     * token_latency_ms is their total. */
    int64_t part_copies[2];
    double part_latency_ms[2];
    double h2d_token_ms;          /* sum of host token copy durations (MOE_FLAG_PROFILE)        */
} moe_stats;

moe_status moe_get_stats(moe_ctx ctx, moe_stats* out);   /* synchronises the context */
moe_status moe_reset_stats(moe_ctx ctx);

/* Device pointers into the workspace of the last call (debugging / white-box tests). */
typedef struct {
    const int32_t* counts;      /* [N_e_local + num_shared] rows per expert of the last call  */
    const int32_t* offsets;     /* [N_e + 1] exclusive scan of routed counts (local view)     */
    const int32_t* pos;         /* [T, top_k] row of (t, j) in the permuted layout            */
    const void* x_perm;         /* bf16 [rows, h]  permuted tokens                            */
    const void* h_act;          /* bf16 [rows, h_i] silu(W1 x) * W3 x                         */
    const void* y_perm;         /* bf16 [rows, h]  gate-scaled expert outputs                 */
    int64_t rows;               /* rows used by the last call                                 */
    const void* h1;             /* bf16 [T, h] Task B: residual stream after the O-projection */
    const void* moe_in;         /* bf16 [T, h] Task B: RMSNorm output u (the MoE input)       */
    int64_t taskb_tokens;       /* T of the last moe_taskb_forward (-1: none yet)             */
} moe_debug_view;
moe_status moe_debug_buffers(moe_ctx ctx, moe_debug_view* out);

/* Release everything owned by the context (synchronises first).  NULL is a no-op. */
moe_status moe_destroy(moe_ctx ctx);

const char* moe_status_string(moe_status s);
const char* moe_last_error(moe_ctx ctx);   /* detail of the last failure ("" if none) */

/*
 * Expert-parallel exchange plan (host-only, deterministic).  Rank r owns routed
 * experts [r*n_local, (r+1)*n_local), n_local = num_experts / world.  Given counts[W][N_e] (rows
 * each rank routes to each expert, all-gathered), fills for `rank`:
 *   send_off[d*n_local + le], send_cnt[...]  rows of this rank's expert-sorted x_perm that go to
 *                                            (destination rank d, its local expert le);
 *   recv_off[s*n_local + le], recv_cnt[...]  where rows from (source rank s, local expert le)
 *                                            land in x_recv, laid out expert-major
 *                                            (local expert, then source rank, then token);
 *   grp_off[n_local + 1]                     expert group boundaries in x_recv.
 * The combine exchange is the exact reverse (recv_* -> send_*).  Returns the number of rows this
 * rank receives, or -1 on invalid arguments.
 */
int64_t moe_ep_plan(int32_t world, int32_t rank, int32_t num_experts, const int32_t* counts,
                    int32_t* send_off, int32_t* send_cnt, int32_t* recv_off, int32_t* recv_cnt,
                    int32_t* grp_off);

/* MOE_FLAG_IPC_EP bootstrap.  moe_ep_ipc_handle writes this rank's MOE_IPC_HANDLE_BYTES-byte
 * blob (CUDA IPC handles of its receive buffers, counts and flags, then its layer shape and
 * max_tokens); the caller all-gathers the blobs of all ranks (rank order) and passes them to
 * moe_ep_ipc_connect, which checks that every rank runs the same layer shape and max_tokens
 * (MOE_E_INVAL otherwise: the receive buffers are sized W x max_tokens x top_k rows) and maps
 * the peers' buffers (cudaIpcOpenMemHandle, peer access enabled lazily).  MOE_E_STATE if the
 * context is not an IPC_EP context or is already connected.  If a call nevertheless routes more
 * rows to an owner than it can hold, nothing is exchanged and moe_sync / the next call return
 * MOE_E_STATE. */
#define MOE_IPC_HANDLE_BYTES 512
moe_status moe_ep_ipc_handle(moe_ctx ctx, void* out);
moe_status moe_ep_ipc_connect(moe_ctx ctx, const void* all_handles);
/* Collective check of a connected IPC_EP group (call on every rank): each rank writes a tagged
 * word into every peer's receive buffer and releases a flag; each then waits up to timeout_s for
 * all peers (no trap) and verifies what it received.  MOE_E_NCCL (with the failing peers in
 * moe_last_error) if any peer did not signal or its data did not arrive -- the caller can then
 * fall back to the NCCL transport with a new context. */
moe_status moe_ep_ipc_selftest(moe_ctx ctx, double timeout_s);

/* Ranks of the context's expert-parallel group as its transport sees them: ncclCommCount of the
 * NCCL communicator, world_size for the P2P transports, 1 without expert parallelism. */
moe_status moe_ep_group_size(moe_ctx ctx, int32_t* nranks);

/* 128-byte ncclUniqueId for moe_config.nccl_unique_id (call on one rank, broadcast to all).
 * MOE_E_NCCL if libnccl.so.2 cannot be loaded. */
moe_status moe_nccl_unique_id(void* out128);

/* Host-link probe, the paper's method ("B_IO ... based on 1GB tensor transfers"):
 * `iters` pinned host->device copies of `bytes` on `device`; returns the best GB/s (1e9 B/s). */
moe_status moe_probe_h2d(int32_t device, size_t bytes, int32_t iters, double* gbps);

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H_ */
