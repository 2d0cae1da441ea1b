// sync_probe.cu -- does a cudaDeviceSynchronize in one host thread block another thread's CUDA
// calls?  Thread A: a kernel on s1 spins on a device flag, then cudaDeviceSynchronize.  Thread B,
// 200 ms later: variant 0 cudaMemcpyAsync + flag write (cudaMemcpyAsync of the flag value);
// variant 1 first cudaEventSynchronize on an already-complete event; variant 2 cudaEventQuery.
// Prints the time thread B's calls took.  (tools only)
#include <chrono>
#include <cstdio>
#include <thread>
#include <cuda_runtime.h>

__global__ void spin(volatile unsigned* f) {
    long long t0 = clock64();
    while (*f == 0) {
        if (clock64() - t0 > 4000000000ll) { printf("spin timeout\n"); return; }
    }
}

int main() {
    unsigned* f; cudaMalloc(&f, 4);
    unsigned* h; cudaMallocHost(&h, 4); *h = 1;
    char *d, *hb; cudaMalloc(&d, 64 << 20); cudaMallocHost(&hb, 64 << 20);
    for (int v = 0; v < 3; ++v) {
        cudaMemset(f, 0, 4); cudaDeviceSynchronize();
        cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
        cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, s2); cudaEventSynchronize(e);
        spin<<<1, 1, 0, s1>>>(f);
        auto t0 = std::chrono::steady_clock::now();
        std::thread b([&] {
            std::this_thread::sleep_for(std::chrono::milliseconds(200));
            auto a = std::chrono::steady_clock::now();
            if (v == 1) cudaEventSynchronize(e);
            if (v == 2) cudaEventQuery(e);
            auto m = std::chrono::steady_clock::now();
            cudaMemcpyAsync(d, hb, 64 << 20, cudaMemcpyHostToDevice, s2);
            cudaMemcpyAsync(f, h, 4, cudaMemcpyHostToDevice, s2);
            auto z = std::chrono::steady_clock::now();
            printf("variant %d: thread B first call %.3f ms, copies enqueued after %.3f ms\n", v,
                   std::chrono::duration<double, std::milli>(m - a).count(),
                   std::chrono::duration<double, std::milli>(z - a).count());
        });
        cudaDeviceSynchronize();
        auto t1 = std::chrono::steady_clock::now();
        b.join();
        printf("variant %d: device sync returned after %.1f ms (%s)\n", v,
               std::chrono::duration<double, std::milli>(t1 - t0).count(), cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
    }
    return 0;
}
