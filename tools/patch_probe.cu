// Scattered 8-byte writes from the GPU into pinned host memory (the edit-record
// patch of a corrected field, ~4.4 M edits over 1 GiB): time vs the host's own
// threaded patch.  nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/patch_probe.cu -o /tmp/patch_probe -lpthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <algorithm>
__global__ void k_patch(const long long* ids, const double* vals, long long m, double* g) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        g[ids[i]] = vals[i];
}
static double now() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    const long long n = 512LL * 512 * 512, m = 4368697;
    double* g;
    cudaMallocHost(&g, n * 8);
    memset(g, 0, n * 8);
    std::vector<long long> ids(m);
    std::vector<double> vals(m);
    srand(1);
    long long pos = 0;
    for (long long i = 0; i < m; ++i) { pos += 1 + rand() % 60; ids[i] = pos % n; vals[i] = i; }
    std::sort(ids.begin(), ids.end());
    long long *dids; double* dvals;
    cudaMalloc(&dids, m * 8); cudaMalloc(&dvals, m * 8);
    cudaMemcpy(dids, ids.data(), m * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dvals, vals.data(), m * 8, cudaMemcpyHostToDevice);
    double* gd = nullptr;
    cudaError_t e = cudaHostGetDevicePointer((void**)&gd, g, 0);
    printf("device pointer %s (same=%d)\n", cudaGetErrorString(e), gd == g);
    for (int blocks : {148, 592, 2368}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaDeviceSynchronize();
            double t0 = now();
            k_patch<<<blocks, 256>>>(dids, dvals, m, gd);
            cudaDeviceSynchronize();
            printf("gpu patch %d blocks: %.2f ms (%s)\n", blocks, now() - t0, cudaGetErrorString(cudaGetLastError()));
        }
    }
    long long bad = 0;
    for (long long i = 0; i < m; ++i) bad += g[ids[i]] != vals[i] && (i + 1 == m || ids[i + 1] != ids[i]);
    printf("mismatches %lld\n", bad);
    for (int nt : {8, 16}) {
        double t0 = now();
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t) th.emplace_back([&, t] {
            const long long a = m * t / nt, b = m * (t + 1) / nt;
            for (long long i = a; i < b; ++i) { if (i + 32 < b) __builtin_prefetch(g + ids[i + 32], 1, 0); g[ids[i]] = vals[i]; }
        });
        for (auto& x : th) x.join();
        printf("host patch %d threads: %.2f ms\n", nt, now() - t0);
    }
    return 0;
}
