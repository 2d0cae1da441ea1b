// ep.cu -- expert parallelism over the GPUs of one box (BASELINE.json north_star: "shards experts
// across the 8 GPUs of one B200 box, so each GPU pulls only its own experts over its own host
// link, and exchanges tokens with an NCCL all-to-all dispatch and combine over NVLink").
//
// Per call on rank r (W ranks, n_local = N_e / W experts each, T_r local tokens):
//   router/top-k/permute on the local tokens      -> x_perm sorted by GLOBAL expert id, so the
//                                                    rows for rank d are one contiguous block
//   all-gather of the per-expert counts            -> counts_all [W][N_e] on the host
//   moe_ep_plan (host, deterministic)              -> send/recv offsets, expert-major x_recv
//   dispatch: one point-to-point transfer per (peer, local expert) with rows > 0
//   local expert GEMMs over x_recv (only this rank's experts, streamed over its own host link)
//   combine exchange: the exact reverse, into the source rank's y_perm at the rows permute gave
//   local gate-weighted combine
// The per-call host sync (after the count all-gather) happens after the call's first weight
// copies are enqueued, so the copy engine keeps streaming while the host waits.
//
// Two transports share the plan and the layouts:
//   NCCL  (default): ncclAllGather + grouped ncclSend/ncclRecv on the caller's stream.
//   local (MOE_FLAG_LOCAL_EP): W contexts of one process, one host thread per rank; counts are
//         exchanged through host memory and rows are PULLED with device-to-device copies from
//         the peers' buffers between host barriers.  It exists to run the multi-rank EP path on
//         a single GPU (tests); it is synchronous and not a performance path.
#include <dlfcn.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "engine.h"

namespace moe {

// ------------------------------------------------------------------------------ NCCL loader
const NcclApi* nccl_api() {
    static NcclApi api;
    static bool ok = false;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = getenv("MOE_NCCL_LIBRARY");
        void* h = nullptr;
        if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.handle = h;
#define LOAD(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym))
        LOAD(GetUniqueId, "ncclGetUniqueId");
        LOAD(CommInitRank, "ncclCommInitRank");
        LOAD(CommDestroy, "ncclCommDestroy");
        LOAD(CommGetAsyncError, "ncclCommGetAsyncError");
        LOAD(AllGather, "ncclAllGather");
        LOAD(Send, "ncclSend");
        LOAD(Recv, "ncclRecv");
        LOAD(GroupStart, "ncclGroupStart");
        LOAD(GroupEnd, "ncclGroupEnd");
        LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
        ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.CommGetAsyncError &&
             api.AllGather && api.Send && api.Recv && api.GroupStart && api.GroupEnd &&
             api.GetErrorString;
    });
    return ok ? &api : nullptr;
}

// ------------------------------------------------------------------------ local transport
namespace {

struct LocalGroup {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<moe_ctx> ranks;
    std::vector<int32_t> counts;  // [W][N_e]

    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

std::mutex g_groups_mu;
std::map<std::string, std::shared_ptr<LocalGroup>> g_groups;

LocalGroup* local_group(moe_ctx c) { return static_cast<LocalGroup*>(c->local_group); }

// Rows of x_perm (sorted by global expert) that rank s holds for expert e: exclusive scan.
int64_t send_offset(const int32_t* counts, int ne, int s, int e) {
    int64_t o = 0;
    for (int i = 0; i < e; ++i) o += counts[(size_t)s * ne + i];
    return o;
}
// Row of x_recv on rank d where (source s, local expert le) lands (expert-major layout).
int64_t recv_offset(const int32_t* counts, int ne, int W, int d, int s, int le) {
    const int nl = ne / W;
    int64_t o = 0;
    for (int l = 0; l < le; ++l)
        for (int q = 0; q < W; ++q) o += counts[(size_t)q * ne + d * nl + l];
    for (int q = 0; q < s; ++q) o += counts[(size_t)q * ne + d * nl + le];
    return o;
}

}  // namespace

// --------------------------------------------------------------------------------- init/teardown
moe_status ep_init(moe_ctx c) {
    const moe_config& cf = c->cfg;
    const int W = cf.world_size, ne = cf.num_experts;
    bool ok = true;
    ok &= cudaMalloc((void**)&c->counts_all, sizeof(int32_t) * (size_t)W * ne) == cudaSuccess;
    ok &= cudaHostAlloc((void**)&c->counts_all_h, sizeof(int32_t) * (size_t)W * ne, 0) == cudaSuccess;
    ok &= cudaMalloc((void**)&c->ep_grp, sizeof(GemmGroup) * 2 * (size_t)c->n_all) == cudaSuccess;
    ok &= cudaHostAlloc((void**)&c->ep_grp_h, sizeof(GemmGroup) * 2 * (size_t)c->n_all, 0) == cudaSuccess;
    ok &= cudaMalloc((void**)&c->x_recv, 2 * (size_t)c->cap_recv * cf.hidden) == cudaSuccess;
    ok &= cudaMalloc((void**)&c->y_recv, 2 * (size_t)c->cap_recv * cf.hidden) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        return set_err(c, MOE_E_NOMEM, "EP buffers");
    }
    if (!make_tmap(&c->tm_xrecv, c->x_recv, (uint64_t)c->cap_recv, cf.hidden, 128) ||
        !make_token_maps(&c->tm_xrecv_t, c->x_recv, (uint64_t)c->cap_recv, cf.hidden))
        return set_err(c, MOE_E_CUDA, "tensor map x_recv");
    const int np = W * c->n_local;
    c->send_off.assign(np, 0);
    c->send_cnt.assign(np, 0);
    c->recv_off.assign(np, 0);
    c->recv_cnt.assign(np, 0);
    c->grp_off.assign(c->n_local + 1, 0);

    if (c->local_ep) {
        if (!cf.nccl_unique_id) return set_err(c, MOE_E_INVAL, "LOCAL_EP needs a group key");
        const std::string key(static_cast<const char*>(cf.nccl_unique_id), 128);
        std::lock_guard<std::mutex> lk(g_groups_mu);
        auto& g = g_groups[key];
        if (!g) {
            g = std::make_shared<LocalGroup>();
            g->world = W;
            g->ranks.assign(W, nullptr);
            g->counts.assign((size_t)W * ne, 0);
        }
        if (g->world != W || g->ranks[cf.rank]) return set_err(c, MOE_E_INVAL, "LOCAL_EP group mismatch");
        g->ranks[cf.rank] = c;
        c->local_group = g.get();
        return MOE_OK;
    }
    const NcclApi* n = nccl_api();
    if (!n) return set_err(c, MOE_E_NCCL, "libnccl.so.2 not found (set MOE_NCCL_LIBRARY)");
    ncclUniqueId id;
    if (cf.nccl_unique_id) {
        memcpy(&id, cf.nccl_unique_id, sizeof id);
    } else {  // world_size == 1 with MOE_FLAG_FORCE_EP: a private one-rank communicator
        MOE_NCCL(c, n->GetUniqueId(&id));
    }
    MOE_NCCL(c, n->CommInitRank(&c->comm, W, id, cf.rank));
    return MOE_OK;
}

void ep_destroy(moe_ctx c) {
    if (c->comm && nccl_api()) nccl_api()->CommDestroy(c->comm);
    c->comm = nullptr;
    if (c->local_group) {
        std::lock_guard<std::mutex> lk(g_groups_mu);
        for (auto it = g_groups.begin(); it != g_groups.end(); ++it) {
            if (it->second.get() == c->local_group) {
                it->second->ranks[c->cfg.rank] = nullptr;
                bool empty = true;
                for (moe_ctx r : it->second->ranks) empty &= (r == nullptr);
                if (empty) g_groups.erase(it);
                break;
            }
        }
        c->local_group = nullptr;
    }
    cudaFree(c->counts_all);
    cudaFreeHost(c->counts_all_h);
    cudaFree(c->ep_grp);
    cudaFreeHost(c->ep_grp_h);
    cudaFree(c->x_recv);
    cudaFree(c->y_recv);
    c->counts_all = nullptr;
    c->counts_all_h = nullptr;
    c->ep_grp = c->ep_grp_h = nullptr;
    c->x_recv = c->y_recv = nullptr;
    cudaGetLastError();
}

// --------------------------------------------------------------------------------- dispatch
moe_status ep_dispatch(moe_ctx c, int T, cudaStream_t st) {
    const moe_config& cf = c->cfg;
    const int W = cf.world_size, ne = cf.num_experts, nl = c->n_local, h = cf.hidden;
    const int k = cf.top_k, S = cf.num_shared, rank = cf.rank;
    const size_t row = (size_t)h;

    // 1. counts exchange -> host
    if (c->local_ep) {
        LocalGroup* g = local_group(c);
        MOE_CUDA(c, cudaMemcpyAsync(c->counts_all_h + (size_t)rank * ne, c->counts,
                                    sizeof(int32_t) * ne, cudaMemcpyDeviceToHost, st));
        MOE_CUDA(c, cudaStreamSynchronize(st));  // also: this rank's x_perm is complete
        {
            std::lock_guard<std::mutex> lk(g->m);
            memcpy(g->counts.data() + (size_t)rank * ne, c->counts_all_h + (size_t)rank * ne,
                   sizeof(int32_t) * ne);
        }
        g->barrier();
        {
            std::lock_guard<std::mutex> lk(g->m);
            memcpy(c->counts_all_h, g->counts.data(), sizeof(int32_t) * (size_t)W * ne);
        }
        g->barrier();  // everyone has read the counts before any rank's next call overwrites them
    } else {
        const NcclApi* n = nccl_api();
        MOE_NCCL(c, n->AllGather(c->counts, c->counts_all, (size_t)ne, kNcclInt32, c->comm, st));
        MOE_CUDA(c, cudaMemcpyAsync(c->counts_all_h, c->counts_all, sizeof(int32_t) * (size_t)W * ne,
                                    cudaMemcpyDeviceToHost, st));
        MOE_CUDA(c, cudaStreamSynchronize(st));
    }
    // 2. plan + GEMM group tables: routed local experts over x_recv; shared experts over the
    //    local tokens
    const int64_t R = moe_ep_plan(W, rank, ne, c->counts_all_h, c->send_off.data(),
                                  c->send_cnt.data(), c->recv_off.data(), c->recv_cnt.data(),
                                  c->grp_off.data());
    if (R < 0 || R > c->cap_recv) return set_err(c, MOE_E_STATE, "EP plan: %lld rows", (long long)R);
    c->last_recv_rows = R;
    GemmGroup* g1 = c->ep_grp_h;
    GemmGroup* g2 = c->ep_grp_h + c->n_all;
    for (int le = 0; le < nl; ++le) {
        g1[le] = GemmGroup{c->grp_off[le], c->grp_off[le + 1], c->grp_off[le], 0};
        g2[le] = g1[le];
    }
    for (int s = 0; s < S; ++s) {
        const int hb = (int)(c->cap_recv + (int64_t)s * T);   // h_act rows of shared expert s
        g1[nl + s] = GemmGroup{0, T, hb, 0};
        g2[nl + s] = GemmGroup{hb, hb + T, T * k + s * T, 0};  // -> y_perm shared rows
    }
    MOE_CUDA(c, cudaMemcpyAsync(c->ep_grp, c->ep_grp_h, sizeof(GemmGroup) * 2 * (size_t)c->n_all,
                                cudaMemcpyHostToDevice, st));
    // 3. rows: x_perm blocks -> the owners' x_recv (expert-major)
    int64_t bytes = 0;
    if (c->local_ep) {
        LocalGroup* g = local_group(c);
        for (int s = 0; s < W; ++s) {
            const moe_ctx peer = g->ranks[s];
            for (int le = 0; le < nl; ++le) {
                const int i = s * nl + le;
                const int32_t cnt = c->recv_cnt[i];
                if (cnt <= 0) continue;
                const int64_t src = send_offset(c->counts_all_h, ne, s, rank * nl + le);
                MOE_CUDA(c, cudaMemcpyAsync(c->x_recv + (size_t)c->recv_off[i] * row,
                                            peer->x_perm + (size_t)src * row,
                                            (size_t)cnt * row * 2, cudaMemcpyDeviceToDevice, st));
            }
        }
        for (int i = 0; i < W * nl; ++i) bytes += (int64_t)c->send_cnt[i] * h * 2;
        MOE_CUDA(c, cudaStreamSynchronize(st));
        g->barrier();  // all pulls done: peers may reuse x_perm
    } else {
        const NcclApi* n = nccl_api();
        MOE_NCCL(c, n->GroupStart());
        for (int p = 0; p < W; ++p) {
            for (int le = 0; le < nl; ++le) {
                const int i = p * nl + le;
                if (c->send_cnt[i] > 0) {
                    MOE_NCCL(c, n->Send(c->x_perm + (size_t)c->send_off[i] * row,
                                        (size_t)c->send_cnt[i] * row, kNcclBfloat16, p, c->comm, st));
                    bytes += (int64_t)c->send_cnt[i] * h * 2;
                }
                if (c->recv_cnt[i] > 0)
                    MOE_NCCL(c, n->Recv(c->x_recv + (size_t)c->recv_off[i] * row,
                                        (size_t)c->recv_cnt[i] * row, kNcclBfloat16, p, c->comm, st));
            }
        }
        MOE_NCCL(c, n->GroupEnd());
    }
    c->comm_bytes += bytes;
    return MOE_OK;
}

// --------------------------------------------------------------------------------- combine
moe_status ep_combine(moe_ctx c, cudaStream_t st) {
    const moe_config& cf = c->cfg;
    const int W = cf.world_size, nl = c->n_local, h = cf.hidden, ne = cf.num_experts;
    const int rank = cf.rank;
    const size_t row = (size_t)h;
    int64_t bytes = 0;
    if (c->local_ep) {
        LocalGroup* g = local_group(c);
        MOE_CUDA(c, cudaStreamSynchronize(st));  // this rank's y_recv is complete
        g->barrier();                            // ... and every peer's
        for (int d = 0; d < W; ++d) {            // pull my rows back from each expert owner
            const moe_ctx peer = g->ranks[d];
            for (int le = 0; le < nl; ++le) {
                const int i = d * nl + le;
                const int32_t cnt = c->send_cnt[i];
                if (cnt <= 0) continue;
                const int64_t src = recv_offset(c->counts_all_h, ne, W, d, rank, le);
                MOE_CUDA(c, cudaMemcpyAsync(c->y_perm + (size_t)c->send_off[i] * row,
                                            peer->y_recv + (size_t)src * row,
                                            (size_t)cnt * row * 2, cudaMemcpyDeviceToDevice, st));
            }
        }
        for (int i = 0; i < W * nl; ++i) bytes += (int64_t)c->recv_cnt[i] * h * 2;
        MOE_CUDA(c, cudaStreamSynchronize(st));
        g->barrier();  // all pulls done: peers may reuse y_recv
    } else {
        const NcclApi* n = nccl_api();
        MOE_NCCL(c, n->GroupStart());
        for (int p = 0; p < W; ++p) {
            for (int le = 0; le < nl; ++le) {
                const int i = p * nl + le;
                if (c->recv_cnt[i] > 0) {  // rows computed here for source p go back to it
                    MOE_NCCL(c, n->Send(c->y_recv + (size_t)c->recv_off[i] * row,
                                        (size_t)c->recv_cnt[i] * row, kNcclBfloat16, p, c->comm, st));
                    bytes += (int64_t)c->recv_cnt[i] * h * 2;
                }
                if (c->send_cnt[i] > 0)
                    MOE_NCCL(c, n->Recv(c->y_perm + (size_t)c->send_off[i] * row,
                                        (size_t)c->send_cnt[i] * row, kNcclBfloat16, p, c->comm, st));
            }
        }
        MOE_NCCL(c, n->GroupEnd());
    }
    c->comm_bytes += bytes;
    return MOE_OK;
}

}  // namespace moe

extern "C" {

int64_t moe_ep_plan(int32_t world, int32_t rank, int32_t num_experts, const int32_t* counts,
                    int32_t* send_off, int32_t* send_cnt, int32_t* recv_off, int32_t* recv_cnt,
                    int32_t* grp_off) {
    if (world <= 0 || rank < 0 || rank >= world || num_experts <= 0 || num_experts % world ||
        !counts || !send_off || !send_cnt || !recv_off || !recv_cnt || !grp_off)
        return -1;
    const int nl = num_experts / world;
    const int32_t* mine = counts + (size_t)rank * num_experts;
    // send side: this rank's x_perm is sorted by global expert id
    int64_t off = 0;
    for (int e = 0; e < num_experts; ++e) {
        if (mine[e] < 0) return -1;
        send_off[e] = (int32_t)off;  // e == d * nl + le
        send_cnt[e] = mine[e];
        off += mine[e];
    }
    // receive side: expert-major (local expert, then source rank, then source token order)
    int64_t pos = 0;
    for (int le = 0; le < nl; ++le) {
        grp_off[le] = (int32_t)pos;
        for (int s = 0; s < world; ++s) {
            const int32_t cnt = counts[(size_t)s * num_experts + rank * nl + le];
            if (cnt < 0) return -1;
            recv_off[s * nl + le] = (int32_t)pos;
            recv_cnt[s * nl + le] = cnt;
            pos += cnt;
        }
    }
    grp_off[nl] = (int32_t)pos;
    return pos;
}

moe_status moe_nccl_unique_id(void* out128) {
    if (!out128) return MOE_E_INVAL;
    const moe::NcclApi* n = moe::nccl_api();
    if (!n) return MOE_E_NCCL;
    moe::ncclUniqueId id;
    if (n->GetUniqueId(&id) != 0) return MOE_E_NCCL;
    memcpy(out128, &id, sizeof id);
    return MOE_OK;
}

}  // extern "C"
