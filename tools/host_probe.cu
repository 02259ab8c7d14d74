// Host-side copy probe for the pageable drop-in path: host memcpy bandwidth
// by thread count, cudaHostRegister cost, pageable vs pinned H2D / D2H.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/host_probe.cu -o gpurun_out/host_probe -lpthread
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void* big(size_t bytes, bool touch) {
    void* p = nullptr;
    posix_memalign(&p, 2 << 20, bytes);
    madvise(p, bytes, MADV_HUGEPAGE);
    if (touch) memset(p, 1, bytes);
    return p;
}

static void pcopy(char* dst, const char* src, size_t bytes, int nt) {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        size_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
        th.emplace_back([=] { memcpy(dst + a, src + a, b - a); });
    }
    for (auto& x : th) x.join();
}

int main() {
    const size_t G = (size_t)1 << 30;
    char* src = (char*)big(G, true);
    char* dst = (char*)big(G, true);
    printf("hw threads %u\n", std::thread::hardware_concurrency());
    for (int nt : {1, 2, 4, 8, 12, 16, 24, 32}) {
        pcopy(dst, src, G, nt);
        double t0 = now();
        pcopy(dst, src, G, nt);
        double t = now() - t0;
        printf("memcpy 1 GiB touched->touched %2d threads: %7.2f ms  %6.1f GB/s\n", nt, t, G / t / 1e6);
    }
    for (int nt : {1, 4, 8, 16}) {
        char* fresh = (char*)big(G, false);
        double t0 = now();
        pcopy(fresh, src, G, nt);
        double t = now() - t0;
        printf("memcpy 1 GiB into fresh (first touch) %2d threads: %7.2f ms\n", nt, t);
        free(fresh);
    }
    char* pin;
    cudaMallocHost(&pin, G);
    memset(pin, 0, G);
    for (int nt : {4, 8, 16}) {
        pcopy(pin, src, G, nt);
        double t0 = now();
        pcopy(pin, src, G, nt);
        double t = now() - t0;
        printf("memcpy 1 GiB pageable->pinned %2d threads: %7.2f ms  %6.1f GB/s\n", nt, t, G / t / 1e6);
    }
    char* dev;
    cudaMalloc(&dev, G);
    cudaStream_t s, s2;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        cudaMemcpyAsync(dev, pin, G, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        double t1 = now();
        cudaMemcpyAsync(dev, src, G, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        double t2 = now();
        cudaMemcpyAsync(pin, dev, G, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        double t3 = now();
        cudaMemcpyAsync(dst, dev, G, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        double t4 = now();
        printf("H2D pinned %.2f ms, H2D pageable %.2f ms, D2H pinned %.2f ms, D2H pageable %.2f ms\n", t1 - t0, t2 - t1,
               t3 - t2, t4 - t3);
    }
    for (int rep = 0; rep < 2; ++rep) {
        char* fresh = (char*)big(G, true);
        double t0 = now();
        cudaError_t e = cudaHostRegister(fresh, G, cudaHostRegisterDefault);
        double t1 = now();
        cudaMemcpyAsync(dev, fresh, G, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        double t2 = now();
        cudaHostUnregister(fresh);
        double t3 = now();
        printf("cudaHostRegister 1 GiB (THP) %.2f ms (%s), H2D %.2f ms, unregister %.2f ms\n", t1 - t0, cudaGetErrorString(e),
               t2 - t1, t3 - t2);
        free(fresh);
    }
    {
        void* p = malloc(G);   // plain malloc, 4 KiB pages unless THP=always
        memset(p, 1, G);
        double t0 = now();
        cudaError_t e = cudaHostRegister(p, G, cudaHostRegisterDefault);
        double t1 = now();
        cudaHostUnregister(p);
        double t2 = now();
        printf("cudaHostRegister 1 GiB (malloc) %.2f ms (%s), unregister %.2f ms\n", t1 - t0, cudaGetErrorString(e), t2 - t1);
        free(p);
    }
    // staged pipeline: pageable -> pinned ring (T threads) -> device, 8 MiB chunks
    for (int nt : {4, 8, 16}) {
        for (size_t chunk : {(size_t)4 << 20, (size_t)16 << 20}) {
            const int R = 4;
            cudaEvent_t ev[R];
            for (int i = 0; i < R; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
            double t0 = now();
            for (size_t o = 0, i = 0; o < G; o += chunk, ++i) {
                char* buf = pin + (i % R) * chunk;
                cudaEventSynchronize(ev[i % R]);
                pcopy(buf, src + o, chunk, nt);
                cudaMemcpyAsync(dev + o, buf, chunk, cudaMemcpyHostToDevice, s);
                cudaEventRecord(ev[i % R], s);
            }
            cudaStreamSynchronize(s);
            double t = now() - t0;
            printf("staged H2D 1 GiB, %2d threads, %2zu MiB chunks: %.2f ms (%.1f GB/s)\n", nt, chunk >> 20, t, G / t / 1e6);
        }
    }
    return 0;
}
