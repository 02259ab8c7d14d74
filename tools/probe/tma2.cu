// TMA probe variants: 1 = 1-D cp.async.bulk; 2 = tensor map in global memory; 3 = param map, 2-D box
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2601_01787_b200/csrc/tma.cuh"
using namespace pmsz;
__device__ __forceinline__ void bulk_1d(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__global__ void k1(const double* src, double* out) {
    __shared__ __align__(128) double buf[256];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = smem_u32(&bar);
    if (threadIdx.x == 0) { mbar_init(b, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) { mbar_expect_tx(b, 2048); bulk_1d(smem_u32(buf), src, 2048, b); }
    mbar_wait(b, 0);
    out[threadIdx.x] = buf[threadIdx.x];
}
__global__ void k2(const CUtensorMap* tmg, double* out) {
    __shared__ __align__(128) double buf[34 * 34];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = smem_u32(&bar);
    if (threadIdx.x == 0) { mbar_init(b, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(tmg) : "memory");
        mbar_expect_tx(b, 34 * 34 * 8);
        tma_load_3d(smem_u32(buf), tmg, 0, 0, 0, b);
    }
    mbar_wait(b, 0);
    for (int i = threadIdx.x; i < 34 * 34; i += blockDim.x) out[i] = buf[i];
}
__global__ void k4(const __grid_constant__ CUtensorMap tm, double* out, int x, int y, int z) {
    __shared__ __align__(128) double buf[34 * 34];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = smem_u32(&bar);
    if (threadIdx.x == 0) { mbar_init(b, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(b, 34 * 34 * 8);
        tma_load_3d(smem_u32(buf), &tm, x, y, z, b);
    }
    mbar_wait(b, 0);
    for (int i = threadIdx.x; i < 34 * 34; i += blockDim.x) out[i] = buf[i];
}
__global__ void k5(const CUtensorMap* tmg, double* out, int x, int y, int z) {
    __shared__ __align__(128) double buf[34 * 34];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = smem_u32(&bar);
    if (threadIdx.x == 0) { mbar_init(b, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(b, 34 * 34 * 8);
        tma_load_3d(smem_u32(buf), tmg, x, y, z, b);
    }
    mbar_wait(b, 0);
    for (int i = threadIdx.x; i < 34 * 34; i += blockDim.x) out[i] = buf[i];
}
__global__ void k3(const __grid_constant__ CUtensorMap tm, double* out) {
    __shared__ __align__(128) double buf[34 * 34];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = smem_u32(&bar);
    if (threadIdx.x == 0) { mbar_init(b, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(b, 34 * 34 * 8);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(b) : "memory");
    }
    mbar_wait(b, 0);
    for (int i = threadIdx.x; i < 34 * 34; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
    const int mode = atoi(argv[1]);
    const int nx = 64, ny = 48, nz = 8;
    std::vector<double> h((size_t)nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 34 * 34 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    std::vector<double> r(34 * 34);
    if (mode == 1) {
        k1<<<1, 256>>>(d + 64, o);
    } else if (mode == 2) {
        CUtensorMap m;
        printf("enc %d\n", (int)tma_field_map(&m, d, false, nx, ny, nz, 34, 34));
        CUtensorMap* g;
        cudaMalloc(&g, sizeof(m));
        cudaMemcpy(g, &m, sizeof(m), cudaMemcpyHostToDevice);
        k2<<<1, 128>>>(g, o);
    } else if (mode >= 4) {
        CUtensorMap m;
        printf("enc %d\n", (int)tma_field_map(&m, d, false, nx, ny, nz, 34, 34));
        const int x = atoi(argv[2]), y = atoi(argv[3]), z = atoi(argv[4]);
        if (mode == 4) k4<<<1, 128>>>(m, o, x, y, z);
        else {
            CUtensorMap* g;
            cudaMalloc(&g, sizeof(m));
            cudaMemcpy(g, &m, sizeof(m), cudaMemcpyHostToDevice);
            k5<<<1, 128>>>(g, o, x, y, z);
        }
    } else {
        auto enc = tma_encoder();
        CUtensorMap m;
        const cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)(ny * nz)};
        const cuuint64_t strides[1] = {(cuuint64_t)(nx * 8)};
        const cuuint32_t box[2] = {34, 34};
        const cuuint32_t es[2] = {1, 1};
        printf("enc r=%d\n", (int)enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
        k3<<<1, 128>>>(m, o);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e) return 1;
    cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
    printf("r[0]=%g r[1]=%g r[34]=%g\n", r[0], r[1], r[34]);
    return 0;
}
