// common.cuh -- stencil, total order and proposal primitives shared by the
// pMSz kernels (sm_100a).
//
// Semantics follow /root/reference/pkg/src/topocorrect:
//   * Freudenthal 14-stencil and (value, id) order: grid.py:24-32,111-118.
//   * The neighbours of one centre are visited in ASCENDING ID ORDER, which is
//     the lexicographic (dz, dy, dx) order of the offsets for every grid
//     shape.  "rank" below is that position (0..13); the centre
//     itself sorts between rank 6 (-x) and rank 7 (+x).  Visiting in rank
//     order turns the reference's (value, id) tie-break into a plain ">="
//     (running max keeps the later = larger id on ties) and "<" (running min
//     keeps the earlier = smaller id), exactly topology.py:64-80.
//   * Out-of-domain neighbours are padded with NaN: every ordered f64
//     comparison with NaN is false, so they never win either chain.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>

namespace pmsz {

// Programmatic dependent launch (sm_90+): a kernel of the loop is launched
// with programmatic stream serialisation, so its launch is processed while
// the previous kernel drains; every such kernel waits here, first thing,
// until the previous grid has completed and its writes are visible (a no-op
// when it was launched the ordinary way).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    static const bool on = !(getenv("PMSZ_PDL") && atoi(getenv("PMSZ_PDL")) == 0);
    if (!on) {
        kern<<<grid, block, smem, s>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...) != cudaSuccess) {
        cudaGetLastError();   // (a driver without programmatic launch: the ordinary one)
        kern<<<grid, block, smem, s>>>(args...);
    }
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per call site and
// device (it is per device, and a host call per launch costs the launch
// path several microseconds): `done` is the call site's device bitmask.
template <typename F>
inline void smem_attr_once(F* fn, int bytes, unsigned long long& done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done & bit) return;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess) done |= bit;
}

// Offsets in ascending-id (rank) order, packed 2 bits per rank (value + 1) so
// a run-time rank costs a shift and a mask, no memory table:
//   dx: -1 0 -1 0 | -1 0 -1 1 0 1 | 0 1 0 1
//   dy: -1 -1 0 0 | -1 -1 0 0 1 1 | 0 0 1 1
//   dz: -1 -1 -1 -1 | 0 0 0 0 0 0 | 1 1 1 1
constexpr unsigned kPackDX = 0u | (1u << 2) | (0u << 4) | (1u << 6) | (0u << 8) | (1u << 10) | (0u << 12) |
                             (2u << 14) | (1u << 16) | (2u << 18) | (1u << 20) | (2u << 22) | (1u << 24) | (2u << 26);
constexpr unsigned kPackDY = 0u | (0u << 2) | (1u << 4) | (1u << 6) | (0u << 8) | (0u << 10) | (1u << 12) |
                             (1u << 14) | (2u << 16) | (2u << 18) | (1u << 20) | (1u << 22) | (2u << 24) | (2u << 26);
constexpr unsigned kPackDZ = 0u | (0u << 2) | (0u << 4) | (0u << 6) | (1u << 8) | (1u << 10) | (1u << 12) |
                             (1u << 14) | (1u << 16) | (1u << 18) | (2u << 20) | (2u << 22) | (2u << 24) | (2u << 26);
__host__ __device__ constexpr int rank_dx(int r) { return (int)((kPackDX >> (2 * r)) & 3u) - 1; }
__host__ __device__ constexpr int rank_dy(int r) { return (int)((kPackDY >> (2 * r)) & 3u) - 1; }
__host__ __device__ constexpr int rank_dz(int r) { return (int)((kPackDZ >> (2 * r)) & 3u) - 1; }
// Centre sorts above ranks 0..6 and below ranks 7..13.
constexpr int kCenterBelow = 6;
constexpr uint8_t kExtremum = 15;
// f-code of a robust centre (tiles.cuh, acc_robust): never evaluated
constexpr uint8_t kRobust = 0xEE;

struct Dom {
    int64_t nx, ny, nz;   // domain (ext) extents
    int64_t sy, sz;       // strides: 1, nx, nx*ny
    int64_t n;
    int64_t lo[3], hi[3]; // core (centre) box
    int32_t shl[3], shh[3]; // shared band widths (block mode)
    double xi, tau;
    double lxi;           // subtracted from the apply's f operand: xi, or 0 when the caller passes L itself
    int extrema_only;
    // exact 32-bit division by the strides (ids < 2^32): q = umulhi64(m, c)
    // with m = ceil(2^64 / stride) (Lemire-Kaser-Kurz); 0 encodes stride 1
    uint64_t msy, msz;
};

__host__ __device__ inline uint64_t div_magic(uint64_t dv) { return dv <= 1 ? 0 : ~0ull / dv + 1; }
__device__ __forceinline__ uint32_t fast_div(uint32_t c, uint64_t m) {
    return m ? (uint32_t)__umul64hi(m, (uint64_t)c) : c;
}

__device__ __forceinline__ double nan64() { return __longlong_as_double(0x7ff8000000000000ll); }

// Read-only loads pinned at their program position (asm volatile), used for
// software prefetching: ptxas may not sink them to the first use.
__device__ __forceinline__ uint32_t ld_nc_u8(const uint8_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_nc_f64(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// Order-preserving 64-bit key of a finite double (min-merge by atomicMin).
// Proposals are g[a] - tau with tau > 0, which is never -0.0.
__device__ __forceinline__ unsigned long long okey(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}
constexpr unsigned long long kNoProposal = 0xffffffffffffffffull;

// Result of the steepest-neighbour scan of one centre.
struct Scan {
    double vc;        // centre value
    double vmax;      // value of the (value,id)-largest neighbour
    double vmin;      // value of the (value,id)-smallest neighbour
    int rmax, rmin;   // their ranks
    bool is_max, is_min;
};

__device__ __forceinline__ uint8_t scan_code(const Scan& s) {
    uint8_t lo = s.is_max ? kExtremum : (uint8_t)s.rmax;
    uint8_t hi = s.is_min ? kExtremum : (uint8_t)s.rmin;
    return (uint8_t)(lo | (hi << 4));
}

// Fold 14 neighbour values (rank order, NaN = absent) into a Scan.
__device__ __forceinline__ Scan fold_scan(double vc, const double (&nv)[14]) {
    Scan s;
    s.vc = vc;
    double bmax = -__longlong_as_double(0x7ff0000000000000ll);  // -inf
    double bmin = __longlong_as_double(0x7ff0000000000000ll);   // +inf
    int rmax = 15, rmin = 15;
#pragma unroll
    for (int r = 0; r < 14; ++r) {
        const double v = nv[r];
        const bool tmax = v >= bmax;
        bmax = tmax ? v : bmax;
        rmax = tmax ? r : rmax;
        const bool tmin = v < bmin;
        bmin = tmin ? v : bmin;
        rmin = tmin ? r : rmin;
    }
    s.vmax = bmax; s.vmin = bmin; s.rmax = rmax; s.rmin = rmin;
    // topology.py:79-80
    s.is_max = (bmax < vc) || (bmax == vc && rmax <= kCenterBelow);
    s.is_min = (bmin > vc) || (bmin == vc && rmin > kCenterBelow);
    return s;
}

// One (value, rank) match; the right operand always holds the higher ranks,
// so ties go right for the max (larger id) and left for the min (smaller id).
__device__ __forceinline__ void mmax(double& v, int& r, double v2, int r2) {
    const bool t = v2 >= v;
    v = t ? v2 : v;
    r = t ? r2 : r;
}
__device__ __forceinline__ void mmin(double& v, int& r, double v2, int r2) {
    const bool t = v2 < v;
    v = t ? v2 : v;
    r = t ? r2 : r;
}

// fold_scan (common.cuh) for a complete ring (no missing neighbour) as a
// balanced tree: the same argmax / argmin under the (value, rank) order.
__device__ __forceinline__ Scan tree_scan(double vc, const double (&nv)[14]) {
    double ax[7], an[7];
    int rx[7], rn[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        // one compare serves both sides (no NaN here): ties -> right for the
        // max (larger id), left for the min (smaller id)
        const bool t = nv[2 * k + 1] >= nv[2 * k];
        ax[k] = t ? nv[2 * k + 1] : nv[2 * k];
        rx[k] = 2 * k + (t ? 1 : 0);
        an[k] = t ? nv[2 * k] : nv[2 * k + 1];
        rn[k] = 2 * k + (t ? 0 : 1);
    }
    mmax(ax[0], rx[0], ax[1], rx[1]); mmin(an[0], rn[0], an[1], rn[1]);   // 0-3
    mmax(ax[2], rx[2], ax[3], rx[3]); mmin(an[2], rn[2], an[3], rn[3]);   // 4-7
    mmax(ax[4], rx[4], ax[5], rx[5]); mmin(an[4], rn[4], an[5], rn[5]);   // 8-11
    mmax(ax[0], rx[0], ax[2], rx[2]); mmin(an[0], rn[0], an[2], rn[2]);   // 0-7
    mmax(ax[4], rx[4], ax[6], rx[6]); mmin(an[4], rn[4], an[6], rn[6]);   // 8-13
    mmax(ax[0], rx[0], ax[4], rx[4]); mmin(an[0], rn[0], an[4], rn[4]);   // 0-13
    Scan s;
    s.vc = vc;
    s.vmax = ax[0]; s.vmin = an[0]; s.rmax = rx[0]; s.rmin = rn[0];
    s.is_max = (ax[0] < vc) || (ax[0] == vc && rx[0] <= kCenterBelow);   // topology.py:79
    s.is_min = (an[0] > vc) || (an[0] == vc && rn[0] > kCenterBelow);    // topology.py:80
    return s;
}

__device__ __forceinline__ void coords(const Dom& d, int64_t c, int64_t& x, int64_t& y, int64_t& z) {
    const uint32_t cc = (uint32_t)c;
    const uint32_t zz = fast_div(cc, d.msz);
    const uint32_t r = cc - zz * (uint32_t)d.sz;
    const uint32_t yy = fast_div(r, d.msy);
    x = (int64_t)(r - yy * (uint32_t)d.sy);
    y = (int64_t)yy;
    z = (int64_t)zz;
}

__device__ __forceinline__ bool in_dom(const Dom& d, int64_t x, int64_t y, int64_t z) {
    return x >= 0 && x < d.nx && y >= 0 && y < d.ny && z >= 0 && z < d.nz;
}

__host__ __device__ __forceinline__ int64_t rank_off(const Dom& d, int r) {
    return (int64_t)rank_dx(r) + (int64_t)rank_dy(r) * d.sy + (int64_t)rank_dz(r) * d.sz;
}

// The 14 neighbour values of centre c = (x,y,z) in rank order, NaN outside
// the domain.  Interior centres (the common case) take plain pointer
// arithmetic -- 3 planes x 3 rows around c -- instead of 14 bounds checks.
template <class Ld>
__device__ __forceinline__ void load_ring(const Dom& d, const double* g, int64_t c, int64_t x, int64_t y, int64_t z,
                                          double (&nv)[14], Ld ld) {
    const double* p0 = g + c;
    if (x > 0 && x + 1 < d.nx && y > 0 && y + 1 < d.ny && z > 0 && z + 1 < d.nz) {
        const double* dn = p0 - d.sz;
        const double* up = p0 + d.sz;
        nv[0] = ld(dn - d.sy - 1); nv[1] = ld(dn - d.sy); nv[2] = ld(dn - 1); nv[3] = ld(dn);
        nv[4] = ld(p0 - d.sy - 1); nv[5] = ld(p0 - d.sy); nv[6] = ld(p0 - 1); nv[7] = ld(p0 + 1);
        nv[8] = ld(p0 + d.sy); nv[9] = ld(p0 + d.sy + 1);
        nv[10] = ld(up); nv[11] = ld(up + 1); nv[12] = ld(up + d.sy); nv[13] = ld(up + d.sy + 1);
    } else {
#pragma unroll
        for (int r = 0; r < 14; ++r) {
            const bool ok = in_dom(d, x + rank_dx(r), y + rank_dy(r), z + rank_dz(r));
            nv[r] = ok ? ld(p0 + rank_off(d, r)) : nan64();
        }
    }
}

// Gather-based scan of centre (x,y,z) from global memory (sparse sweeps and
// domain edges).
__device__ __forceinline__ Scan gather_scan(const Dom& d, const double* __restrict__ g,
                                            int64_t x, int64_t y, int64_t z) {
    const int64_t c = x + y * d.sy + z * d.sz;
    double nv[14];
#pragma unroll
    for (int r = 0; r < 14; ++r) {
        const bool ok = in_dom(d, x + rank_dx(r), y + rank_dy(r), z + rank_dz(r));
        nv[r] = ok ? __ldg(g + c + rank_off(d, r)) : nan64();
    }
    return fold_scan(__ldg(g + c), nv);
}

}  // namespace pmsz
