// tma.cuh -- Tensor Memory Accelerator plumbing for the tiled sweeps (sm_100a):
// host-side tensor maps of a (nx, ny, nz) x-fastest field and the device-side
// mbarrier / cp.async.bulk.tensor wrappers.
//
// A 3-D tiled tensor map with a (bx, by, 1) box stages one plane of a CTA's
// column (its halo included) with ONE instruction issued by one thread; cells
// outside the field are filled with NaN by the TMA unit (OOB fill), which is
// exactly the "missing neighbour" encoding of fold_scan (common.cuh).
// Restrictions of the hardware: every global stride (nx * elem, nx * ny * elem
// bytes) must be a multiple of 16 (plans whose field does not qualify use the
// cp.async stager of tiles.cuh), and the innermost box origin must be 16-byte
// aligned -- an odd x origin of an f64 box is an illegal instruction, so the
// boxes start at the even (f64) / multiple-of-4 (f32) column left of x0 - 1.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace pmsz {

// ---- host ------------------------------------------------------------------
inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

inline bool tma_strides_ok(int64_t nx, int64_t ny, size_t elem) {
    return ((size_t)nx * elem) % 16 == 0 && ((size_t)nx * (size_t)ny * elem) % 16 == 0;
}

// Tensor map of field `base` (f64 or f32) with a (bx, by, 1) box, NaN OOB fill.
inline bool tma_field_map(CUtensorMap* m, const void* base, bool f32, int64_t nx, int64_t ny, int64_t nz,
                          uint32_t bx, uint32_t by) {
    const size_t elem = f32 ? 4 : 8;
    if (!tma_strides_ok(nx, ny, elem) || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t strides[2] = {(cuuint64_t)(nx * elem), (cuuint64_t)(nx * ny * elem)};
    const cuuint32_t box[3] = {bx, by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base),
               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA) == CUDA_SUCCESS;
}

// Tensor map of a u8 field (the f-code) with a (bx, by, 1) box.
inline bool tma_u8_map(CUtensorMap* m, const void* base, int64_t nx, int64_t ny, int64_t nz, uint32_t bx, uint32_t by) {
    if (!tma_strides_ok(nx, ny, 1) || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t strides[2] = {(cuuint64_t)nx, (cuuint64_t)(nx * ny)};
    const cuuint32_t box[3] = {bx, by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor map of a bit field viewed as u32 words (nwx words per row).
inline bool tma_u32_map(CUtensorMap* m, const void* base, int64_t nwx, int64_t ny, int64_t nz, uint32_t bx, uint32_t by) {
    if (!tma_strides_ok(nwx, ny, 4) || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)nwx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t strides[2] = {(cuuint64_t)(nwx * 4), (cuuint64_t)(nwx * ny * 4)};
    const cuuint32_t box[3] = {bx, by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- device ----------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Wait for the phase with `parity` to complete.  The suspend-time hint lets
// the hardware park the warp until the phase flips instead of spinning (a
// spinning producer or consumer would steal issue slots from the others).
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(0x989680u)
            : "memory");
    } while (!done);
}
// One 3-D box load (x, y, z = box origin, may be negative / past the end).
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* m, int x, int y, int z, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}

}  // namespace pmsz
