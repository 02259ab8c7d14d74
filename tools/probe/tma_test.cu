// Standalone TMA probe: stage one 34x34 f64 box with NaN OOB fill and compare.
#include <cstdio>
#include <vector>
#include <cmath>
#include <cstdlib>
#include "../../paper_2601_01787_b200/csrc/tma.cuh"
using namespace pmsz;
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int x, int y, int z, int bx) {
    __shared__ __align__(128) double buf[34 * 34 + 16];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = smem_u32(&bar);
    if (threadIdx.x == 0) {
        mbar_init(b, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(b, bx * 34 * 8);
        tma_load_3d(smem_u32(buf), &tm, x, y, z, b);
    }
    mbar_wait(b, 0);
    for (int i = threadIdx.x; i < bx * 34; i += blockDim.x) out[i] = buf[i];
}
static bool encode(CUtensorMap* m, const void* base, int nx, int ny, int nz, int bx, int by, int fill, int l2) {
    auto enc = tma_encoder();
    const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t strides[2] = {(cuuint64_t)(nx * 8), (cuuint64_t)(nx * ny * 8)};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
               fill ? CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA : CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode r=%d\n", (int)r);
    return r == CUDA_SUCCESS;
}
int main(int argc, char** argv) {
    const int fill = atoi(argv[1]), l2 = atoi(argv[2]), bxa = atoi(argv[3]), mode = atoi(argv[4]);
    const int nx = 64, ny = 48, nz = 8;
    std::vector<double> h((size_t)nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 34 * 34 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    CUtensorMap m;
    bool ok = encode(&m, d, nx, ny, nz, bxa, 34, fill, l2);
    printf("encode ok=%d\n", ok);
    int bad = 0;
    const int X[3] = {-1, 31, 40}, Y[3] = {-1, 15, 20}, Z[3] = {-1, 3, 8};
    for (int t = mode; t < 3; ++t) {
        k<<<1, 128>>>(m, o, X[t], Y[t], Z[t], bxa);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("launch %d: %s\n", t, cudaGetErrorString(e)); return 1; }
        std::vector<double> r(34 * 34);
        cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
        for (int j = 0; j < 34; ++j)
            for (int i = 0; i < bxa; ++i) {
                const int gx = X[t] + i, gy = Y[t] + j, gz = Z[t];
                const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz;
                const double want = in ? h[gx + (size_t)nx * (gy + (size_t)ny * gz)] : (fill ? NAN : 0.0);
                const double got = r[j * bxa + i];
                if (in || !fill ? got != want : !std::isnan(got)) { if (bad < 5) printf("t%d (%d,%d): got %g want %g\n", t, i, j, got, want); ++bad; }
            }
    }
    printf("bad=%d\n", bad);
    return bad != 0;
}
