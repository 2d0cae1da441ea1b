// mover.cu -- the Contiguous Data Mover (§6.5), B200 version (MOE_FLAG_MOVER).
//
// "a dedicated Contiguous Data Mover, running on a separate thread ... The execution pipeline
// pushes weight transfer requests to the data mover at layer-wise granularity, while the data
// mover internally performs fine-grained transfers ... It first partitions the requested weights
// into small packets and issues one packet transfer at a time to the runtime.  This strategy
// prevents contention with other CPU-GPU transfers ... Issuing all weight transfers at once would
// lead to head-of-line blocking, delaying latency-sensitive compute transfers ... a 100MB packet
// size".
//
// Here: the engine's copy requests (flush_copies: a batch of streamed experts) become jobs on a
// queue; a native thread cuts each job into packets (cfg.packet_bytes, default 100 MB) and keeps
// at most `inflight` packets (default 1, the paper's "one packet at a time") submitted to the copy
// engine, waiting on the oldest packet's event before issuing the next.  A token copy issued by
// the caller (moe_layer_forward_host) therefore queues behind at most `inflight` packets instead
// of behind every expert copy already requested.
//
// Ordering between the thread and the streams is by monotone counters in device memory, written
// and awaited with stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32, GEQ,
// wrap-aware), never by events: the thread issues copies asynchronously to the API thread, so an
// event re-recorded by a later call could otherwise be waited on by an earlier copy.
//   flags[0] r13  = streamed items whose W13 part is resident   (copy stream writes)
//   flags[1] r2   = streamed items fully resident               (copy stream writes)
//   flags[2] free = streamed items whose GEMMs are done          (compute stream writes)
// Item q may overwrite slot q % nslots once free >= q - nslots + 1; GEMM1 of items [q, q + n)
// waits r13 >= q + n, GEMM2 waits r2 >= q + n.  Items are copied and computed in order, so one
// counter per kind suffices.
// A stream wait must never name work that has not been SUBMITTED yet: streams share a small set
// of hardware queues, and a wait at the head of one blocks whatever is queued behind it -- here,
// possibly the very packet it waits for (measured: C1 hung with the compute stream's wait for
// r13 >= 1 enqueued before the mover had submitted item 0's last packet).  So the API thread
// first waits on the HOST until the mover has submitted the write it will wait for (sub13 / sub2),
// which paces moe_layer_forward by the mover (it returns once its last packet is submitted); the
// copy stream's wait on `free` only ever names GEMMs enqueued before the job was pushed.
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>

#include "engine.h"

namespace moe {

namespace {
typedef CUresult (*PFN_streamValue32_t)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct ValueOps {
    PFN_streamValue32_t wait = nullptr, write = nullptr;
};

const ValueOps& value_ops() {
    static ValueOps ops;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.wait = reinterpret_cast<PFN_streamValue32_t>(p);
        p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.write = reinterpret_cast<PFN_streamValue32_t>(p);
        cudaGetLastError();
    });
    return ops;
}

constexpr unsigned kWaitGeq = 0x0;     // CU_STREAM_WAIT_VALUE_GEQ
constexpr unsigned kWriteDefault = 0x0;
constexpr int kMaxInflight = 8;

struct Job {
    uint64_t q0;
    int n;
    const char* src;
    char* dst;
    int64_t item, w13;   // bytes per item / of its W13 part (a shared-FFN slice is smaller)
};
}  // namespace

struct Mover {
    int device = 0;
    int nslots = 2;
    int64_t blob = 0, w13 = 0, packet = 0;
    int inflight = 1;
    cudaStream_t copy = nullptr;
    uint32_t* flags = nullptr;   // device [3]: r13, r2, free

    std::thread th;
    std::mutex mu;
    std::condition_variable cv, idle_cv;
    std::deque<Job> queue;
    bool stop = false, busy = false;
    moe_status err = MOE_OK;
    std::string err_msg;
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> recs;   // H2D brackets (profile mode)

    std::condition_variable sub_cv;
    uint64_t sub[2] = {0, 0};   // items whose r13 / r2 write has been submitted (host view)

    cudaEvent_t ev[kMaxInflight] = {};
    int ev_head = 0, ev_n = 0;
    uint64_t packets = 0;
    bool trace = false;   // MOE_MOVER_TRACE=1: one stderr line per job / packet wait

    bool fail(const char* what, cudaError_t e) {
        std::lock_guard<std::mutex> g(mu);
        if (err == MOE_OK) {
            err = MOE_E_CUDA;
            err_msg = std::string("data mover: ") + what + ": " + cudaGetErrorString(e);
        }
        sub_cv.notify_all();
        return false;
    }
    bool fail_cu(const char* what, CUresult r) {
        std::lock_guard<std::mutex> g(mu);
        if (err == MOE_OK) {
            err = MOE_E_CUDA;
            err_msg = std::string("data mover: ") + what + " failed (CUresult " + std::to_string((int)r) + ")";
        }
        sub_cv.notify_all();
        return false;
    }

    // one packet: at most `inflight` submitted and not yet complete
    bool issue(char* dst, const char* src, int64_t bytes) {
        if (ev_n == inflight) {
            if (trace) fprintf(stderr, "[mover] packet %llu: wait for the oldest in flight\n", (unsigned long long)packets);
            cudaError_t e = cudaEventSynchronize(ev[ev_head]);
            if (e != cudaSuccess) return fail("cudaEventSynchronize", e);
            ev_head = (ev_head + 1) % inflight;
            --ev_n;
        }
        cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, copy);
        if (e != cudaSuccess) return fail("cudaMemcpyAsync", e);
        e = cudaEventRecord(ev[(ev_head + ev_n) % inflight], copy);
        if (e != cudaSuccess) return fail("cudaEventRecord", e);
        ++ev_n;
        ++packets;
        return true;
    }

    bool write_flag(int i, uint64_t v) {
        CUresult r = value_ops().write((CUstream)copy, (CUdeviceptr)(flags + i), (cuuint32_t)v,
                                       kWriteDefault);
        if (r != CUDA_SUCCESS) return fail_cu("cuStreamWriteValue32", r);
        {
            std::lock_guard<std::mutex> g(mu);
            sub[i] = v;
        }
        sub_cv.notify_all();
        return true;
    }

    bool run(const Job& j) {
        cudaEvent_t a = nullptr, b = nullptr;
        // the batch's slots are free once the items nslots earlier finished their GEMMs
        const int64_t need = (int64_t)j.q0 + j.n - nslots;
        if (trace)
            fprintf(stderr, "[mover] job items [%llu, %llu): copy stream waits free >= %lld\n",
                    (unsigned long long)j.q0, (unsigned long long)(j.q0 + j.n), (long long)need);
        if (need > 0) {
            CUresult r = value_ops().wait((CUstream)copy, (CUdeviceptr)(flags + 2),
                                          (cuuint32_t)(uint64_t)need, kWaitGeq);
            if (r != CUDA_SUCCESS) return fail_cu("cuStreamWaitValue32", r);
        }
        if (prof && (cudaEventCreate(&a) != cudaSuccess || cudaEventRecord(a, copy) != cudaSuccess))
            return fail("profile event", cudaGetLastError());
        // The job's items are contiguous in host memory and in the staging buffer: one byte range
        // cut into packets regardless of item boundaries (small experts share packets); after each
        // packet the counters advance over the items whose W13 part / whole blob it completed.
        const int64_t total = (int64_t)j.n * j.item;
        int done13 = 0, done2 = 0;
        for (int64_t o = 0; o < total;) {
            const int64_t e = std::min(total, o + packet);
            if (!issue(j.dst + o, j.src + o, e - o)) return false;
            o = e;
            int n13 = done13, n2 = done2;
            while (n13 < j.n && (int64_t)n13 * j.item + j.w13 <= e) ++n13;
            while (n2 < j.n && (int64_t)(n2 + 1) * j.item <= e) ++n2;
            if (n13 > done13 && !write_flag(0, j.q0 + n13)) return false;
            if (n2 > done2 && !write_flag(1, j.q0 + n2)) return false;
            done13 = n13;
            done2 = n2;
        }
        if (prof) {
            if (cudaEventCreate(&b) != cudaSuccess || cudaEventRecord(b, copy) != cudaSuccess)
                return fail("profile event", cudaGetLastError());
            std::lock_guard<std::mutex> g(mu);
            recs.emplace_back(a, b);
        }
        return true;
    }

    void loop() {
        cudaSetDevice(device);
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> g(mu);
                cv.wait(g, [&] { return stop || !queue.empty(); });
                if (queue.empty()) break;   // stop requested and nothing left
                j = queue.front();
                queue.pop_front();
                busy = true;
            }
            bool ok;
            {
                std::lock_guard<std::mutex> g(mu);
                ok = err == MOE_OK;
            }
            if (ok) run(j);   // after an error the queue is drained without copying
            {
                std::lock_guard<std::mutex> g(mu);
                busy = false;
                if (queue.empty()) idle_cv.notify_all();
            }
        }
    }
};

moe_status mover_start(moe_ctx c) {
    const ValueOps& ops = value_ops();
    if (!ops.wait || !ops.write)
        return set_err(c, MOE_E_UNSUPPORTED, "data mover: stream memory operations unavailable");
    Mover* m = new Mover();
    m->device = c->cfg.device;
    m->nslots = c->nslots;
    m->blob = c->blob_bytes;
    m->w13 = c->w13_bytes;
    m->packet = c->cfg.packet_bytes > 0 ? c->cfg.packet_bytes : (int64_t)100 << 20;
    m->inflight = 1;
    if (const char* e = getenv("MOE_MOVER_INFLIGHT")) m->inflight = std::max(1, std::min(atoi(e), kMaxInflight));
    m->copy = c->copy_stream;
    m->prof = (c->cfg.flags & MOE_FLAG_PROFILE) != 0;
    m->trace = getenv("MOE_MOVER_TRACE") && atoi(getenv("MOE_MOVER_TRACE")) != 0;
    bool ok = cudaMalloc((void**)&m->flags, 4 * sizeof(uint32_t)) == cudaSuccess &&
              cudaMemset(m->flags, 0, 4 * sizeof(uint32_t)) == cudaSuccess &&
              cudaDeviceSynchronize() == cudaSuccess;
    for (int i = 0; ok && i < m->inflight; ++i)
        ok = cudaEventCreateWithFlags(&m->ev[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        for (cudaEvent_t e : m->ev)
            if (e) cudaEventDestroy(e);
        cudaFree(m->flags);
        delete m;
        return set_err(c, MOE_E_NOMEM, "data mover: flags / events");
    }
    m->th = std::thread([m] { m->loop(); });
    c->mover = m;
    return MOE_OK;
}

moe_status mover_drain(moe_ctx c) {
    Mover* m = c->mover;
    if (!m) return MOE_OK;
    std::unique_lock<std::mutex> g(m->mu);
    m->idle_cv.wait(g, [&] { return m->queue.empty() && !m->busy; });
    if (m->err != MOE_OK) {
        c->sticky = m->err;
        return set_err(c, m->err, "%s", m->err_msg.c_str());
    }
    return MOE_OK;
}

void mover_stop(moe_ctx c) {
    Mover* m = c->mover;
    if (!m) return;
    {
        std::lock_guard<std::mutex> g(m->mu);
        m->stop = true;
    }
    m->cv.notify_all();
    if (m->th.joinable()) m->th.join();
    cudaStreamSynchronize(m->copy);
    for (cudaEvent_t e : m->ev)
        if (e) cudaEventDestroy(e);
    for (auto& r : m->recs) {
        cudaEventDestroy(r.first);
        cudaEventDestroy(r.second);
    }
    cudaFree(m->flags);
    delete m;
    c->mover = nullptr;
}

moe_status mover_push(moe_ctx c, uint64_t q0, int n, const char* src, char* dst, int64_t item,
                      int64_t w13) {
    Mover* m = c->mover;
    {
        std::lock_guard<std::mutex> g(m->mu);
        if (m->err != MOE_OK) {
            c->sticky = m->err;
            return set_err(c, m->err, "%s", m->err_msg.c_str());
        }
        m->queue.push_back(Job{q0, n, src, dst, item, w13});
    }
    m->cv.notify_one();
    return MOE_OK;
}

moe_status mover_wait(moe_ctx c, cudaStream_t st, int which, uint64_t value) {
    Mover* m = c->mover;
    {   // the write this stream wait names must already be submitted (see the header)
        std::unique_lock<std::mutex> g(m->mu);
        m->sub_cv.wait(g, [&] { return m->sub[which] >= value || m->err != MOE_OK; });
        if (m->err != MOE_OK) {
            c->sticky = m->err;
            return set_err(c, m->err, "%s", m->err_msg.c_str());
        }
    }
    CUresult r = value_ops().wait((CUstream)st, (CUdeviceptr)(m->flags + which),
                                  (cuuint32_t)value, kWaitGeq);
    if (r != CUDA_SUCCESS) {
        c->sticky = MOE_E_CUDA;
        return set_err(c, MOE_E_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
    }
    return MOE_OK;
}

moe_status mover_mark_free(moe_ctx c, cudaStream_t st, uint64_t value) {
    CUresult r = value_ops().write((CUstream)st, (CUdeviceptr)(c->mover->flags + 2),
                                   (cuuint32_t)value, kWriteDefault);
    if (r != CUDA_SUCCESS) {
        c->sticky = MOE_E_CUDA;
        return set_err(c, MOE_E_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
    }
    return MOE_OK;
}

double mover_take_h2d_ms(moe_ctx c, int64_t* packets) {
    Mover* m = c->mover;
    if (!m) return 0.0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> recs;
    {
        std::lock_guard<std::mutex> g(m->mu);
        recs.swap(m->recs);
        if (packets) *packets = (int64_t)m->packets;
    }
    double ms = 0.0;
    for (auto& r : recs) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, r.first, r.second) == cudaSuccess) ms += t;
        else cudaGetLastError();
        cudaEventDestroy(r.first);
        cudaEventDestroy(r.second);
    }
    return ms;
}

}  // namespace moe
