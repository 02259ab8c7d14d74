// qsweep.cuh -- tiled detection sweep over a per-plane queue of FRAGILE centres
// (K1 full / masked, K4 count).
//
// K0 marks a centre robust (f-code kRobust) when the largest and the smallest
// member of its closed 1-ring in f lead the runners-up by more than 2 xi
// (tiles.cuh, acc_robust): every g of the loop stays in [f - xi, f + xi], so a
// robust centre's steepest directions and extremum flags never differ from
// f's and none of the six rules (correction.py:169-229) can fire there.  On
// the benchmark field ~80 % of the centres are robust, but they are spread
// over every warp, so skipping them inside the shared-fold sweep of tiles.cuh
// saves nothing.  Here the fold work is compacted instead:
//
//   * one thread stages each plane of the CTA's 32 x 32 column (36 x 34 with
//     the halo) by TMA into a shared ring, a few planes ahead; every g value
//     is read from HBM once per CTA, and the tensor map's NaN fill encodes the
//     neighbours outside the field;
//   * per plane, each thread tests its four centres' f-codes (prefetched two
//     planes ahead) and the fragile ones are appended to a shared queue
//     (warp ballot + one shared atomic per warp);
//   * the queue is evaluated densely, one centre per thread: 15 shared loads,
//     a balanced-tree (value, rank) fold (depth 4 instead of 14) and the
//     f-code comparison.
//
// The fold work per voxel drops by the robust fraction, and the sweep streams
// g at close to the HBM rate (9 B per voxel: g + f-code).
#pragma once
#include "tiles.cuh"
#include "tma.cuh"
#include <algorithm>

namespace pmsz {

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

// ---------------------------------------------------------------------------
// TMA-staged queue sweep.  A CTA owns a 32 x 32 column of centres (thread
// (tx, ty) owns x = tx and rows 4 ty .. 4 ty + 3) and marches its z chunk.
// Thread 0 stages each 36 x 34 plane (halo included, NaN outside the field)
// with one cp.async.bulk.tensor into a 6-slot ring, 3 planes ahead, completion
// on a per-slot mbarrier.  One __syncthreads per plane: at step k the CTA
// enqueues the fragile centres of plane zb + k and evaluates the queue of
// plane zb + k - 1 (queues and counters rotate so the barrier separates every
// writer from its readers).
constexpr int kQX = 32, kQY = 32, kQRowsPerThread = 4;
// TMA boxes must start on a 16-byte boundary: a staged row covers the even
// x0 - 1 - (x0 - 1 odd) .. + 35 (36 f64 = 288 B), the halo column x0 - 1 at xo.
constexpr int kQPX = kQX + 4, kQPY = kQY + 2, kQPlane = kQPX * kQPY;   // 36 x 34
constexpr int kQPlaneStride = ((kQPlane * 8 + 127) / 128) * 128 / 8;   // doubles, 128-B aligned slots
constexpr int kQSlots = 6, kQAhead = 3;
constexpr int kQCapT = kQX * kQY;
static_assert(kQAhead <= kQSlots - 3, "a refilled slot must be out of use");
struct QSmem {
    double plane[kQSlots][kQPlaneStride];
    uint8_t code[kQSlots][kQX * kQY];   // f-code tiles (kCodeTma)
    uint32_t queue[2][kQCapT];          // staged cell | f-code << 16
    unsigned long long bar[kQSlots];
    unsigned cnt[3];
};
constexpr size_t kQSmemBytes = sizeof(QSmem);

// kCodeTma: the f-code tile of every plane comes with the g plane (one more
// TMA box; needs x0 % 16 == 0 and nx % 16 == 0), else the codes (and, masked,
// the dirty words) are loaded per thread two planes ahead.
template <bool kCount, bool kMasked, bool kExtrema, bool kCodeTma>
__global__ void __launch_bounds__(256, 3) k_qsweep_tma(Dom d, const __grid_constant__ CUtensorMap tm,
                                                       const __grid_constant__ CUtensorMap tmc,
                                                       DetectOp<kCount, kMasked, kExtrema> op, int zchunk) {
    using Op = DetectOp<kCount, kMasked, kExtrema>;
    static_assert(!(kCodeTma && kMasked), "masked sweeps load their dirty words per thread");
    extern __shared__ __align__(1024) unsigned char qraw[];   // TMA destinations: 128-B aligned slots
    QSmem& S = *reinterpret_cast<QSmem*>(qraw);
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * kQX + tx, lane = tid & 31;
    const int64_t x0 = d.lo[0] + (int64_t)blockIdx.x * kQX;
    const int64_t y0 = d.lo[1] + (int64_t)blockIdx.y * kQY;
    const int64_t zb = d.lo[2] + (int64_t)blockIdx.z * zchunk;
    const int64_t ze = min(zb + (int64_t)zchunk, d.hi[2]);
    const int K = (int)(ze - zb);
    const int64_t sy = d.sy, sz = d.sz;
    const int64_t xs = (x0 - 1) & ~int64_t(1);   // even box origin
    const int xo = (int)(x0 - 1 - xs);          // column of x0 - 1 in a staged row
    const unsigned bar0 = smem_u32(&S.bar[0]);
    const unsigned pl0 = smem_u32(&S.plane[0][0]);
    const unsigned cd0 = smem_u32(&S.code[0][0]);
    constexpr unsigned kBytes = kQPlane * 8;
    // plane index i = p - (zb - 1), i in [0, K + 1]; slot i % kQSlots, use i / kQSlots
    auto issue = [&](int i) {
        const int slot = i % kQSlots;
        const bool codes = kCodeTma && i >= 1 && i <= K;   // centre planes carry their f-code tile
        mbar_expect_tx(bar0 + 8 * slot, kBytes + (codes ? kQX * kQY : 0));
        tma_load_3d(pl0 + slot * kQPlaneStride * 8, &tm, (int)xs, (int)(y0 - 1), (int)(zb - 1 + i),
                    bar0 + 8 * slot);
        if (codes) tma_load_3d(cd0 + slot * kQX * kQY, &tmc, (int)x0, (int)y0, (int)(zb - 1 + i), bar0 + 8 * slot);
    };
    auto wait_plane = [&](int i) { mbar_wait(bar0 + 8 * (i % kQSlots), (unsigned)((i / kQSlots) & 1)); };
    if (tid == 0) {
        for (int s = 0; s < kQSlots; ++s) mbar_init(bar0 + 8 * s, 1);
        mbar_fence_init();
        S.cnt[0] = S.cnt[1] = S.cnt[2] = 0;
        for (int i = 0; i <= kQAhead && i <= K + 1; ++i) issue(i);
    }
    op.begin();
    const bool edge_xy = x0 == 0 || x0 + kQX >= d.nx || y0 == 0 || y0 + kQY >= d.ny;
    const int64_t x = x0 + tx, yr = y0 + kQRowsPerThread * ty;
    const bool live_x = x < d.hi[0];
    bool live[kQRowsPerThread];
#pragma unroll
    for (int r = 0; r < kQRowsPerThread; ++r) live[r] = live_x && yr + r < d.hi[1];
    // ids < 2^32 (plan limit): 32-bit index arithmetic
    const uint32_t cbase = (uint32_t)(x + yr * sy + zb * sz);   // centre of row 0 at plane zb
    const uint32_t sy32 = (uint32_t)sy, sz32 = (uint32_t)sz;
    // f-codes (and dirty words) two planes ahead (per-thread path)
    typename Op::Pre p0[kQRowsPerThread], p1[kQRowsPerThread];
    if (!kCodeTma) {
#pragma unroll
        for (int r = 0; r < kQRowsPerThread; ++r) {
            p0[r] = op.fetch(cbase + r * sy32, live[r]);
            p1[r] = op.fetch(cbase + r * sy32 + sz32, live[r] && zb + 1 < ze);
        }
    }
    __syncthreads();
    for (int k = 0; k <= K; ++k) {
        if (k == 0) { wait_plane(0); wait_plane(1); }
        else wait_plane(k + 1);
        __syncthreads();
        if (tid == 0) {
            if (k + 1 + kQAhead <= K + 1) issue(k + 1 + kQAhead);
            S.cnt[(k + 1) % 3] = 0;
        }
        if (k < K) {
            // enqueue the live, fragile (and dirty) centres of plane zb + k
            const uint32_t cz = cbase + (uint32_t)k * sz32;
            uint32_t code[kQRowsPerThread];
            bool want[kQRowsPerThread];
            if (kCodeTma) {
                const uint8_t* ct = S.code[(k + 1) % kQSlots];
#pragma unroll
                for (int r = 0; r < kQRowsPerThread; ++r) {
                    code[r] = ct[(kQRowsPerThread * ty + r) * kQX + tx];
                    want[r] = live[r] && code[r] != kRobust;
                }
            } else {
                typename Op::Pre p2[kQRowsPerThread];
#pragma unroll
                for (int r = 0; r < kQRowsPerThread; ++r)
                    p2[r] = op.fetch(cz + r * sy32 + 2 * sz32, live[r] && zb + k + 2 < ze);
#pragma unroll
                for (int r = 0; r < kQRowsPerThread; ++r) {
                    code[r] = p0[r].code & 0xffu;
                    want[r] = op.wants(p0[r]);
                    p0[r] = p1[r];
                    p1[r] = p2[r];
                }
            }
            unsigned bal[kQRowsPerThread], tot = 0;
#pragma unroll
            for (int r = 0; r < kQRowsPerThread; ++r) {
                bal[r] = __ballot_sync(0xffffffffu, want[r]);
                tot += __popc(bal[r]);
            }
            unsigned base = 0;
            if (lane == 0 && tot) base = atomicAdd(&S.cnt[k % 3], tot);
            base = __shfl_sync(0xffffffffu, base, 0);
            const unsigned below = (1u << lane) - 1u;
            uint32_t* q = S.queue[k & 1];
#pragma unroll
            for (int r = 0; r < kQRowsPerThread; ++r) {
                if (want[r]) {
                    const unsigned at = base + __popc(bal[r] & below);
                    q[at] = (uint32_t)((kQRowsPerThread * ty + r + 1) * kQPX + xo + 1 + tx) | (code[r] << 16);
                }
                base += __popc(bal[r]);
            }
        }
        if (k >= 1) {
            // evaluate the queue of plane zc = zb + k - 1 (planes i = k - 1, k, k + 1)
            const int64_t zc = zb + k - 1;
            const unsigned n = S.cnt[(k - 1) % 3];
            const uint32_t* q = S.queue[(k - 1) & 1];
            const uint32_t cpl = (uint32_t)(x0 + y0 * sy + zc * sz);   // centre id of tile cell (0, 0)
            const double* dn = S.plane[(k - 1) % kQSlots];
            const double* ct = S.plane[k % kQSlots];
            const double* up = S.plane[(k + 1) % kQSlots];
            const bool interior = !edge_xy && zc >= 1 && zc + 1 < d.nz;
            for (unsigned e = tid; e < n; e += kQX * kQY / kQRowsPerThread) {
                const uint32_t ent = q[e];
                const int cell = (int)(ent & 0xffffu);
                double nv[14];
                nv[0] = dn[cell - kQPX - 1]; nv[1] = dn[cell - kQPX]; nv[2] = dn[cell - 1]; nv[3] = dn[cell];
                nv[4] = ct[cell - kQPX - 1]; nv[5] = ct[cell - kQPX]; nv[6] = ct[cell - 1]; nv[7] = ct[cell + 1];
                nv[8] = ct[cell + kQPX]; nv[9] = ct[cell + kQPX + 1];
                nv[10] = up[cell]; nv[11] = up[cell + 1]; nv[12] = up[cell + kQPX]; nv[13] = up[cell + kQPX + 1];
                const double vc = ct[cell];
                const Scan s = interior ? tree_scan(vc, nv) : fold_scan(vc, nv);   // NaN = outside the field
                const int ly = cell / kQPX, lx = cell - ly * kQPX;
                op.evaluate(d, (int64_t)(cpl + (uint32_t)(ly - 1) * sy32 + (uint32_t)(lx - 1 - xo)), s, (uint8_t)(ent >> 16));
            }
        }
    }
    op.finish();
}

inline void qsweep_grid(const Dom& d, dim3& grid, int& zchunk) {
    const int64_t cx = d.hi[0] - d.lo[0], cy = d.hi[1] - d.lo[1], cz = d.hi[2] - d.lo[2];
    const int64_t tiles = ((cx + kQX - 1) / kQX) * ((cy + kQY - 1) / kQY);
    // z chunks of ~64 planes unless that leaves fewer than ~6 waves of
    // 148 SMs x 3 CTAs; never below 16 planes
    const int64_t want = (148 * 3 * 6 + tiles - 1) / tiles;
    int64_t chunks = std::max<int64_t>((cz + 63) / 64, std::min<int64_t>(want, cz / 16));
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, cz));
    zchunk = (int)std::max<int64_t>(1, (cz + chunks - 1) / chunks);
    chunks = (cz + zchunk - 1) / zchunk;
    grid = dim3((unsigned)((cx + kQX - 1) / kQX), (unsigned)((cy + kQY - 1) / kQY), (unsigned)chunks);
}

template <bool kCount, bool kMasked, bool kExtrema>
inline bool launch_qsweep(const Dom& d, const double* g, const Work& w, cudaStream_t s, const uint32_t* dirty) {
    CUtensorMap tm, tmc;
    if (!tma_field_map(&tm, g, false, d.nx, d.ny, d.nz, kQPX, kQPY)) return false;
    // f-code tiles by TMA: 16-byte aligned tile origins and strides
    const bool code_tma = !kMasked && d.lo[0] % 16 == 0 && tma_u8_map(&tmc, w.code, d.nx, d.ny, d.nz, kQX, kQY);
    if (!code_tma) tmc = tm;
    using Op = DetectOp<kCount, kMasked, kExtrema>;
    dim3 grid;
    int zchunk;
    qsweep_grid(d, grid, zchunk);
    Op op{w, dirty, 0};
    const dim3 block(kQX, kQY / kQRowsPerThread, 1);
    if (code_tma) {
        auto kern = k_qsweep_tma<kCount, kMasked, kExtrema, !kMasked>;
        static bool attr = false;
        if (!attr) attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQSmemBytes) == cudaSuccess;
        kern<<<grid, block, kQSmemBytes, s>>>(d, tm, tmc, op, zchunk);
    } else {
        auto kern = k_qsweep_tma<kCount, kMasked, kExtrema, false>;
        static bool attr = false;
        if (!attr) attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQSmemBytes) == cudaSuccess;
        kern<<<grid, block, kQSmemBytes, s>>>(d, tm, tmc, op, zchunk);
    }
    return true;
}

// K1 full / masked and K4 count sweeps (dirty: masked sweep over its bits).
// Returns false when the field cannot be described by a tensor map (odd
// extents): the caller then takes the cp.async sweep of tiles.cuh.
template <bool kCount>
inline bool launch_sweep_q(const Dom& d, const double* g, const Work& w, cudaStream_t s,
                           const uint32_t* dirty = nullptr) {
    if (kCount) return launch_qsweep<true, false, false>(d, g, w, s, nullptr);
    if (dirty && d.extrema_only) return launch_qsweep<false, true, true>(d, g, w, s, dirty);
    if (dirty) return launch_qsweep<false, true, false>(d, g, w, s, dirty);
    if (d.extrema_only) return launch_qsweep<false, false, true>(d, g, w, s, nullptr);
    return launch_qsweep<false, false, false>(d, g, w, s, nullptr);
}

}  // namespace pmsz
