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
//   NCCL  (default): ncclAllGather + grouped ncclSend/ncclRecv on the caller's stream, one host
//         sync per call (the counts, for the plan).
//   P2P   (MOE_FLAG_LOCAL_EP: ranks are contexts of this process; MOE_FLAG_IPC_EP: ranks are
//         processes, buffers mapped with CUDA IPC): every rank holds device pointers to every
//         rank's x_recv / y_recv / counts / flags; the permute kernel writes rows straight into
//         the owners' x_recv, the combine kernel reads the owners' y_recv, and device flags
//         order the calls (ep_p2p.cu) -- no host sync, no staging copies.
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
        LOAD(CommCount, "ncclCommCount");
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
    // MOE_FLAG_SHARD_SHARED: W * max_tokens more rows for every rank's tokens (x_recv) and the
    // shared slice's partial outputs for them (y_recv), both read / written by peers
    const int64_t rows = c->cap_recv + (c->shard ? (int64_t)W * cf.max_tokens : 0);
    ok &= cudaMalloc((void**)&c->x_recv, 2 * (size_t)rows * cf.hidden) == cudaSuccess;
    ok &= cudaMalloc((void**)&c->y_recv, 2 * (size_t)rows * cf.hidden) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        return set_err(c, MOE_E_NOMEM, "EP buffers");
    }
    if (!make_tmap(&c->tm_xrecv, c->x_recv, (uint64_t)rows, cf.hidden, 128))
        return set_err(c, MOE_E_CUDA, "tensor map x_recv");
    const int np = W * c->n_local;
    c->send_off.assign(np, 0);
    c->send_cnt.assign(np, 0);
    c->recv_off.assign(np, 0);
    c->recv_cnt.assign(np, 0);
    c->grp_off.assign(c->n_local + 1, 0);

    if (c->p2p) {
        bool pk = true;
        pk &= cudaMalloc((void**)&c->p2p_flags, sizeof(unsigned long long) * kP2PFlags * kMaxRanks) == cudaSuccess;
        pk &= cudaMalloc((void**)&c->p2p_counts, sizeof(int32_t) * 2 * (size_t)W * ne) == cudaSuccess;
        pk &= cudaMalloc((void**)&c->p2p_tab, sizeof(P2PTable)) == cudaSuccess;
        pk &= cudaMalloc((void**)&c->pr_x, sizeof(PeerRows)) == cudaSuccess;
        pk &= cudaMalloc((void**)&c->pr_y, sizeof(PeerRows)) == cudaSuccess;
        pk &= cudaMalloc((void**)&c->p2p_rows, sizeof(int32_t)) == cudaSuccess;
        pk &= cudaMalloc((void**)&c->p2p_bytes, sizeof(long long)) == cudaSuccess;
        pk &= cudaHostAlloc((void**)&c->p2p_diag_h, 8 * sizeof(long long), cudaHostAllocMapped) == cudaSuccess;
        if (pk) {
            memset(c->p2p_diag_h, 0, 8 * sizeof(long long));
            pk &= cudaHostGetDevicePointer((void**)&c->p2p_diag_d, c->p2p_diag_h, 0) == cudaSuccess;
        }
        if (!pk) {
            cudaGetLastError();
            return set_err(c, MOE_E_NOMEM, "P2P EP buffers");
        }
        pk &= cudaMemset(c->p2p_flags, 0, sizeof(unsigned long long) * kP2PFlags * kMaxRanks) == cudaSuccess;
        pk &= cudaMemset(c->p2p_counts, 0, sizeof(int32_t) * 2 * (size_t)W * ne) == cudaSuccess;
        pk &= cudaMemset(c->p2p_rows, 0, sizeof(int32_t)) == cudaSuccess;
        pk &= cudaMemset(c->p2p_bytes, 0, sizeof(long long)) == cudaSuccess;
        pk &= cudaDeviceSynchronize() == cudaSuccess;
        if (!pk) return set_err(c, MOE_E_CUDA, "P2P EP init");
        if (!c->local_ep) return MOE_OK;   // IPC: moe_ep_ipc_connect maps the peers
        for (int f = 0; f < kP2PFlags; ++f)
            for (int p = 0; p < 2; ++p)
                if (cudaEventCreateWithFlags(&c->p2p_ev[f][p], cudaEventDisableTiming) != cudaSuccess)
                    return set_err(c, MOE_E_CUDA, "P2P EP events");
    }
    if (c->local_ep) {
        if (!cf.nccl_unique_id) return set_err(c, MOE_E_INVAL, "LOCAL_EP needs a group key");
        const std::string key(static_cast<const char*>(cf.nccl_unique_id), 128);
        std::lock_guard<std::mutex> lk(g_groups_mu);
        auto& g = g_groups[key];
        if (!g) {
            g = std::make_shared<LocalGroup>();
            g->world = W;
            g->ranks.assign(W, nullptr);
        }
        if (g->world != W || g->ranks[cf.rank]) return set_err(c, MOE_E_INVAL, "LOCAL_EP group mismatch");
        for (moe_ctx p : g->ranks) {   // the exchange assumes one layer shape on every rank
            if (!p) continue;
            const moe_config& o = p->cfg;
            if (o.hidden != cf.hidden || o.ffn != cf.ffn || o.num_experts != cf.num_experts ||
                o.top_k != cf.top_k || o.num_shared != cf.num_shared ||
                o.max_tokens != cf.max_tokens ||
                (o.flags & MOE_FLAG_SHARD_SHARED) != (cf.flags & MOE_FLAG_SHARD_SHARED))
                return set_err(c, MOE_E_INVAL, "LOCAL_EP rank %d: layer shape / max_tokens differ "
                               "(or MOE_FLAG_SHARD_SHARED) from rank %d's", cf.rank, o.rank);
        }
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
    for (int d = 0; d < kMaxRanks; ++d)
        for (int i = 0; i < 4; ++i)
            if (c->ipc_opened[d][i]) {
                cudaIpcCloseMemHandle(c->ipc_opened[d][i]);
                c->ipc_opened[d][i] = nullptr;
            }
    void* pbufs[] = {c->p2p_flags, c->p2p_counts, c->p2p_tab, c->pr_x, c->pr_y, c->p2p_rows,
                     c->p2p_bytes};
    for (void* p : pbufs) cudaFree(p);
    for (int f = 0; f < kP2PFlags; ++f)
        for (int p = 0; p < 2; ++p)
            if (c->p2p_ev[f][p]) {
                cudaEventDestroy(c->p2p_ev[f][p]);
                c->p2p_ev[f][p] = nullptr;
            }
    if (c->p2p_diag_h) cudaFreeHost(c->p2p_diag_h);
    c->p2p_diag_h = nullptr;
    c->p2p_diag_d = nullptr;
    c->p2p_flags = nullptr;
    c->p2p_counts = nullptr;
    c->p2p_tab = nullptr;
    c->pr_x = c->pr_y = nullptr;
    c->p2p_rows = nullptr;
    c->p2p_bytes = nullptr;
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
    {
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
    {
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
    {
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

// ---------------------------------------------------------------------------- P2P transport
IpcShape ipc_shape(moe_ctx c) {
    const moe_config& cf = c->cfg;
    return IpcShape{0x4D6F4533, cf.rank, cf.world_size, cf.hidden, cf.ffn, cf.num_experts,
                    cf.top_k, cf.num_shared, cf.max_tokens,
                    (int32_t)(cf.flags & MOE_FLAG_SHARD_SHARED)};
}

namespace {

// This rank's device tables, filled from the peers' buffers as mapped in this process.
// Uploaded on `st` (stream-ordered before the kernels that read them): a legacy-stream copy
// could wait on peers' flag-wait kernels and deadlock the group.
moe_status p2p_upload(moe_ctx c, unsigned long long* const* flags, int32_t* const* counts,
                      __nv_bfloat16* const* xr, __nv_bfloat16* const* yr, cudaStream_t st) {
    const int W = c->cfg.world_size;
    P2PTable tab{};
    PeerRows px{}, py{};
    for (int d = 0; d < W; ++d) {
        tab.flags[d] = flags[d];
        tab.counts[d] = counts[d];
        px.rows[d] = xr[d];
        py.rows[d] = yr[d];
    }
    px.nl = py.nl = c->n_local;
    px.shard_row = py.shard_row = -1;   // set per call by the plan kernel when sharded
    px.shard_mask = py.shard_mask = c->shard ? c->shard_mask : 0u;
    MOE_CUDA(c, cudaMemcpyAsync(c->p2p_tab, &tab, sizeof tab, cudaMemcpyHostToDevice, st));
    MOE_CUDA(c, cudaMemcpyAsync(c->pr_x, &px, sizeof px, cudaMemcpyHostToDevice, st));
    MOE_CUDA(c, cudaMemcpyAsync(c->pr_y, &py, sizeof py, cudaMemcpyHostToDevice, st));
    MOE_CUDA(c, cudaStreamSynchronize(st));   // the host structs go out of scope
    c->p2p_ready = true;
    return MOE_OK;
}

// LOCAL_EP: wait until every rank of the group exists (first call only), then map them.
moe_status p2p_connect_local(moe_ctx c, cudaStream_t st) {
    LocalGroup* g = local_group(c);
    g->barrier();
    const int W = c->cfg.world_size;
    unsigned long long* flags[kMaxRanks];
    int32_t* counts[kMaxRanks];
    __nv_bfloat16 *xr[kMaxRanks], *yr[kMaxRanks];
    {
        std::lock_guard<std::mutex> lk(g->m);
        for (int d = 0; d < W; ++d) {
            const moe_ctx p = g->ranks[d];
            if (!p) return set_err(c, MOE_E_STATE, "LOCAL_EP rank %d missing", d);
            if (p->cfg.device != c->cfg.device) {   // ranks on different GPUs of the box
                int can = 0;
                MOE_CUDA(c, cudaDeviceCanAccessPeer(&can, c->cfg.device, p->cfg.device));
                if (!can)
                    return set_err(c, MOE_E_UNSUPPORTED, "LOCAL_EP: device %d cannot access "
                                   "peer device %d", c->cfg.device, p->cfg.device);
                const cudaError_t e = cudaDeviceEnablePeerAccess(p->cfg.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else MOE_CUDA(c, e);
            }
            flags[d] = p->p2p_flags;
            counts[d] = p->p2p_counts;
            xr[d] = p->x_recv;
            yr[d] = p->y_recv;
        }
    }
    return p2p_upload(c, flags, counts, xr, yr, st);
}

// Sync point `which` of call `val`.  IPC: device flags (release / acquire, system scope).
// LOCAL: an event recorded on this rank's stream; the waiters pass a host barrier (so every
// rank has enqueued its record, in program order before this wait) and enqueue stream waits.
moe_status p2p_signal(moe_ctx c, int which, unsigned long long val, cudaStream_t st) {
    if (c->local_ep) {
        MOE_CUDA(c, cudaEventRecord(c->p2p_ev[which][val & 1], st));
        return MOE_OK;
    }
    MOE_CUDA(c, launch_p2p_signal(c->p2p_tab, c->cfg.world_size, c->cfg.rank, which, val, st));
    c->stats.kernel_launches += 1;
    return MOE_OK;
}

moe_status p2p_wait(moe_ctx c, int which, unsigned long long val, cudaStream_t st) {
    if (val == 0) return MOE_OK;   // call 0 never happened
    const int W = c->cfg.world_size;
    if (c->local_ep) {
        LocalGroup* g = local_group(c);
        g->barrier();
        for (int d = 0; d < W; ++d)
            if (d != c->cfg.rank)
                MOE_CUDA(c, cudaStreamWaitEvent(st, g->ranks[d]->p2p_ev[which][val & 1], 0));
        return MOE_OK;
    }
    MOE_CUDA(c, launch_p2p_wait(c->p2p_flags, W, which, val, c->p2p_diag_d, st));
    c->stats.kernel_launches += 1;
    return MOE_OK;
}

#define P2P_TRY(expr)                           \
    do {                                        \
        moe_status _s = (expr);                 \
        if (_s != MOE_OK) return _s;            \
    } while (0)

}  // namespace

moe_status p2p_before_dispatch(moe_ctx c, int T, cudaStream_t st) {
    if (!c->p2p_ready) {
        if (!c->local_ep)
            return set_err(c, MOE_E_STATE, "IPC_EP context not connected (moe_ep_ipc_connect)");
        moe_status s = p2p_connect_local(c, st);
        if (s != MOE_OK) return s;
    }
    const moe_config& cf = c->cfg;
    const int W = cf.world_size, ne = cf.num_experts, me = cf.rank;
    const unsigned long long seq = ++c->p2p_seq;
    const int par = (int)(seq & 1);
    static const bool trace = getenv("MOE_P2P_TRACE") != nullptr;
    if (trace) fprintf(stderr, "[p2p] rank %d call %llu T=%d stream=%p\n", me, seq, T, (void*)st);
    // the push kernel also releases kFlagCounts on every peer (used by IPC; harmless in LOCAL)
    MOE_CUDA(c, launch_p2p_push_counts(c->p2p_tab, c->counts, ne, W, me, par, seq, st));
    c->stats.kernel_launches += 2;
    if (c->local_ep) MOE_CUDA(c, cudaEventRecord(c->p2p_ev[kFlagCounts][par], st));
    P2P_TRY(p2p_wait(c, kFlagCounts, seq, st));
    MOE_CUDA(c, launch_p2p_plan(c->p2p_counts + (size_t)par * W * ne, W, ne, me, T, cf.top_k,
                                cf.num_shared, c->cap_recv, c->n_all, cf.hidden, c->ep_grp,
                                c->pr_x, c->pr_y, c->p2p_rows, c->p2p_bytes, c->p2p_diag_d,
                                c->shard ? c->n_local : -1, st));
    P2P_TRY(p2p_wait(c, kFlagXFree, seq - 1, st));
    return MOE_OK;
}

moe_status p2p_after_dispatch(moe_ctx c, cudaStream_t st) {
    const unsigned long long seq = c->p2p_seq;
    P2P_TRY(p2p_signal(c, kFlagDispatched, seq, st));
    P2P_TRY(p2p_wait(c, kFlagDispatched, seq, st));
    P2P_TRY(p2p_wait(c, kFlagYDone, seq - 1, st));
    return MOE_OK;
}

moe_status p2p_after_gemms(moe_ctx c, cudaStream_t st) {
    const unsigned long long seq = c->p2p_seq;
    P2P_TRY(p2p_signal(c, kFlagXFree, seq, st));
    P2P_TRY(p2p_signal(c, kFlagYReady, seq, st));
    P2P_TRY(p2p_wait(c, kFlagYReady, seq, st));
    return MOE_OK;
}

moe_status p2p_after_combine(moe_ctx c, cudaStream_t st) {
    return p2p_signal(c, kFlagYDone, c->p2p_seq, st);
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

moe_status moe_ep_group_size(moe_ctx c, int32_t* nranks) {
    if (!c || !nranks) return MOE_E_INVAL;
    *nranks = c->ep ? c->cfg.world_size : 1;
    if (c->comm && moe::nccl_api() && moe::nccl_api()->CommCount) {
        int n = 0;
        MOE_NCCL(c, moe::nccl_api()->CommCount(c->comm, &n));
        *nranks = n;
    }
    return MOE_OK;
}

moe_status moe_ep_ipc_handle(moe_ctx c, void* out) {
    if (!c || !out) return MOE_E_INVAL;
    if (!c->p2p || c->local_ep) return moe::set_err(c, MOE_E_STATE, "not an IPC_EP context");
    MOE_CUDA(c, cudaSetDevice(c->cfg.device));
    void* bufs[4] = {c->x_recv, c->y_recv, c->p2p_counts, c->p2p_flags};
    static_assert(4 * sizeof(cudaIpcMemHandle_t) + sizeof(moe::IpcShape) <= MOE_IPC_HANDLE_BYTES,
                  "IPC blob size");
    char* o = static_cast<char*>(out);
    memset(o, 0, MOE_IPC_HANDLE_BYTES);
    for (int i = 0; i < 4; ++i) {
        cudaIpcMemHandle_t hnd;
        MOE_CUDA(c, cudaIpcGetMemHandle(&hnd, bufs[i]));
        memcpy(o + i * sizeof hnd, &hnd, sizeof hnd);
    }
    const moe::IpcShape sh = moe::ipc_shape(c);
    memcpy(o + 4 * sizeof(cudaIpcMemHandle_t), &sh, sizeof sh);
    return MOE_OK;
}

moe_status moe_ep_ipc_connect(moe_ctx c, const void* all) {
    if (!c || !all) return MOE_E_INVAL;
    if (!c->p2p || c->local_ep || c->p2p_ready)
        return moe::set_err(c, MOE_E_STATE, "not an unconnected IPC_EP context");
    MOE_CUDA(c, cudaSetDevice(c->cfg.device));
    const int W = c->cfg.world_size, me = c->cfg.rank;
    // every rank must run the same layer shape and capacity (the receive buffers are sized for
    // W x max_tokens x top_k rows), in rank order
    const moe::IpcShape mine = moe::ipc_shape(c);
    for (int d = 0; d < W; ++d) {
        moe::IpcShape o;
        memcpy(&o, static_cast<const char*>(all) + (size_t)d * MOE_IPC_HANDLE_BYTES +
                       4 * sizeof(cudaIpcMemHandle_t), sizeof o);
        moe::IpcShape want = mine;
        want.rank = d;
        if (memcmp(&o, &want, sizeof o) != 0)
            return moe::set_err(c, MOE_E_INVAL, "IPC_EP: rank %d's blob (magic %x, rank %d, W %d, "
                                "h %d, h_i %d, N_e %d, k %d, S %d, max_tokens %d, shard %d) does "
                                "not match this rank's layer", d, o.magic, o.rank, o.world,
                                o.hidden, o.ffn, o.num_experts, o.top_k, o.num_shared,
                                o.max_tokens, o.shard);
    }
    unsigned long long* flags[moe::kMaxRanks];
    int32_t* counts[moe::kMaxRanks];
    __nv_bfloat16 *xr[moe::kMaxRanks], *yr[moe::kMaxRanks];
    for (int d = 0; d < W; ++d) {
        if (d == me) {
            xr[d] = c->x_recv;
            yr[d] = c->y_recv;
            counts[d] = c->p2p_counts;
            flags[d] = c->p2p_flags;
            continue;
        }
        void* p[4];
        for (int i = 0; i < 4; ++i) {
            cudaIpcMemHandle_t hnd;
            memcpy(&hnd, static_cast<const char*>(all) + (size_t)d * MOE_IPC_HANDLE_BYTES + i * sizeof hnd,
                   sizeof hnd);
            MOE_CUDA(c, cudaIpcOpenMemHandle(&p[i], hnd, cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened[d][i] = p[i];
        }
        xr[d] = static_cast<__nv_bfloat16*>(p[0]);
        yr[d] = static_cast<__nv_bfloat16*>(p[1]);
        counts[d] = static_cast<int32_t*>(p[2]);
        flags[d] = static_cast<unsigned long long*>(p[3]);
    }
    return moe::p2p_upload(c, flags, counts, xr, yr, c->copy_stream);
}

moe_status moe_ep_ipc_selftest(moe_ctx c, double timeout_s) {
    if (!c) return MOE_E_INVAL;
    if (!c->p2p || c->local_ep || !c->p2p_ready)
        return moe::set_err(c, MOE_E_STATE, "not a connected IPC_EP context");
    MOE_CUDA(c, cudaSetDevice(c->cfg.device));
    int* d_res = nullptr;
    int h_res = -1;
    MOE_CUDA(c, cudaMalloc((void**)&d_res, sizeof(int)));
    const long long cycles = (long long)(timeout_s * 2.0e9);   // SM clock <= 2 GHz
    cudaError_t e = moe::launch_p2p_selftest(c->p2p_tab, c->pr_x, c->p2p_flags,
                                             reinterpret_cast<const uint32_t*>(c->x_recv),
                                             c->cfg.world_size, c->cfg.rank,
                                             ++c->p2p_selftest_seq, cycles, d_res, c->copy_stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&h_res, d_res, sizeof(int), cudaMemcpyDeviceToHost, c->copy_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->copy_stream);
    cudaFree(d_res);
    MOE_CUDA(c, e);
    if (h_res != 0)
        return moe::set_err(c, MOE_E_NCCL, "P2P self-test failed on rank %d (mask 0x%x: low byte "
                            "= peers that never signalled, high byte = peers whose rows did not "
                            "arrive)", c->cfg.rank, h_res);
    return MOE_OK;
}
}  // extern "C"
