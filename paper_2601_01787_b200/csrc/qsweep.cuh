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
//   * per plane, each consumer warp tests its 4 x 32 centres' f-codes (TMA
//     tiles, or per lane two planes ahead) and appends the fragile ones to its
//     own shared queue (ballots, no atomics);
//   * the warp evaluates its queue densely, one centre per lane: 15 shared
//     loads, a balanced-tree (value, rank) fold (depth 4 instead of 14) and
//     the f-code comparison;
//   * no block barrier: full / empty mbarriers per slot hand the planes from
//     the producer to the consumers and back.
//
// The fold work per voxel drops by the robust fraction, and the sweep streams
// g at close to the HBM rate (9 B per voxel: g + f-code).
#pragma once
#include "tiles.cuh"
#include "tma.cuh"
#include <algorithm>

namespace pmsz {

// ---------------------------------------------------------------------------
// TMA-staged queue sweep.  A CTA owns a 32 x 32 column of centres (consumer
// warp w owns rows 4 w .. 4 w + 3, lane = x) and marches its z chunk; a
// producer warp stages each 36 x 34 plane (halo included, NaN outside the
// field) with one cp.async.bulk.tensor into a 6-slot ring.
constexpr int kQX = 32, kQY = 32, kQRowsPerThread = 4;
// TMA boxes must start on a 16-byte boundary: a staged row covers the even
// x0 - 1 - (x0 - 1 odd) .. + 35 (36 f64 = 288 B), the halo column x0 - 1 at xo.
constexpr int kQPX = kQX + 4, kQPY = kQY + 2, kQPlane = kQPX * kQPY;   // 36 x 34
constexpr int kQPlaneStride = ((kQPlane * 8 + 127) / 128) * 128 / 8;   // doubles, 128-B aligned slots
// Closed ring of the staged cell `cell` (kQPX-wide rows) of planes dn / ct / up.
__device__ __forceinline__ void ring_from_smem(const double* dn, const double* ct, const double* up, int cell,
                                               double (&nv)[14], double& vc) {
    nv[0] = dn[cell - kQPX - 1]; nv[1] = dn[cell - kQPX]; nv[2] = dn[cell - 1]; nv[3] = dn[cell];
    nv[4] = ct[cell - kQPX - 1]; nv[5] = ct[cell - kQPX]; nv[6] = ct[cell - 1]; nv[7] = ct[cell + 1];
    nv[8] = ct[cell + kQPX]; nv[9] = ct[cell + kQPX + 1];
    nv[10] = up[cell]; nv[11] = up[cell + 1]; nv[12] = up[cell + kQPX]; nv[13] = up[cell + kQPX + 1];
    vc = ct[cell];
}

#ifndef PMSZ_QSLOTS
#define PMSZ_QSLOTS 6   // plane slots of the ring (3 in use + look-ahead)
#endif
#ifndef PMSZ_QMINB
#define PMSZ_QMINB 3    // resident CTAs per SM
#endif
constexpr int kQSlots = PMSZ_QSLOTS;
constexpr int kQConsumers = kQY / kQRowsPerThread;   // consumer warps (4 rows x 32 columns each)
constexpr int kQThreads = (kQConsumers + 1) * 32;     // + one producer warp
struct QSmem {
    double plane[kQSlots][kQPlaneStride];
    uint8_t code[kQSlots][kQX * kQY];                  // f-code tiles
    uint32_t dirty[kQSlots][kQY * 4];                  // dirty-bitmap tiles (masked): 4 words / row
    uint32_t queue[kQConsumers][kQRowsPerThread * 32 + 32];   // per-warp queue: tile index | f-code << 16 | plane bit << 24
    unsigned long long full[kQSlots];                  // TMA landed
    unsigned long long empty[kQSlots];                 // every consumer warp is done with the slot
};
constexpr size_t kQSmemBytes = sizeof(QSmem);

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Producer / consumer pipeline without block barriers.  Warp 8 (one lane)
// streams the CTA's planes into a 6-slot ring: plane index i = p - (zb - 1)
// goes to slot i % 6 once every consumer warp has released index i - 6.
// Consumer warp w owns rows 4 w .. 4 w + 3 of the 32 x 32 column: per centre
// plane zb + k it waits for index k + 2, queues its fragile centres in its own
// shared queue, evaluates them one per lane and releases index k.
//
// The f-code tile of every centre plane (and, masked, its dirty words) comes
// with the g plane as one more TMA box (needs x0 % 16 == 0 and nx % 16 == 0;
// launch_qsweep falls back to tiles.cuh otherwise).
template <bool kCount, bool kMasked, bool kExtrema>
__global__ void __launch_bounds__(kQThreads, PMSZ_QMINB) k_qsweep_tma(Dom d, const __grid_constant__ CUtensorMap tm,
                                                             const __grid_constant__ CUtensorMap tmc,
                                                             const __grid_constant__ CUtensorMap tmd,
                                                             DetectOp<kCount, kMasked, kExtrema> op, int zchunk) {
    pdl_wait();   // (programmatic dependent launch)
    using Op = DetectOp<kCount, kMasked, kExtrema>;
    extern __shared__ __align__(1024) unsigned char qraw[];   // TMA destinations: 128-B aligned slots
    QSmem& S = *reinterpret_cast<QSmem*>(qraw);
    const int tx = threadIdx.x, ty = threadIdx.y;   // ty = warp
    const int64_t x0 = d.lo[0] + (int64_t)blockIdx.x * kQX;
    const int64_t y0 = d.lo[1] + (int64_t)blockIdx.y * kQY;
    const int64_t zb = d.lo[2] + (int64_t)blockIdx.z * zchunk;
    const int64_t ze = min(zb + (int64_t)zchunk, d.hi[2]);
    const int K = (int)(ze - zb);
    const int64_t sy = d.sy, sz = d.sz;
    const uint32_t sy32 = (uint32_t)sy, sz32 = (uint32_t)sz;
    const int64_t xs = (x0 - 1) & ~int64_t(1);   // even box origin
    const int xo = (int)(x0 - 1 - xs);          // column of x0 - 1 in a staged row
    const unsigned full0 = smem_u32(&S.full[0]), empty0 = smem_u32(&S.empty[0]);
    if (ty == kQConsumers && tx == 0) {
        for (int s = 0; s < kQSlots; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, kQConsumers);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (ty == kQConsumers) {
        // ---- producer ----
        if (tx == 0) {
            const unsigned pl0 = smem_u32(&S.plane[0][0]), cd0 = smem_u32(&S.code[0][0]);
            for (int i = 0; i <= K + 1; ++i) {
                const int slot = i % kQSlots;
                if (i >= kQSlots) mbar_wait(empty0 + 8 * slot, (unsigned)((i / kQSlots - 1) & 1));
                const bool codes = i >= 1 && i <= K;   // centre planes carry their f-code tile
                const bool dirt = codes && kMasked;                 // ... and their dirty words
                mbar_expect_tx(full0 + 8 * slot, kQPlane * 8 + (codes ? kQX * kQY : 0) + (dirt ? kQY * 16 : 0));
                tma_load_3d(pl0 + slot * kQPlaneStride * 8, &tm, (int)xs, (int)(y0 - 1), (int)(zb - 1 + i),
                            full0 + 8 * slot);
                if (codes)
                    tma_load_3d(cd0 + slot * kQX * kQY, &tmc, (int)x0, (int)y0, (int)(zb - 1 + i), full0 + 8 * slot);
                if (dirt)
                    tma_load_3d(smem_u32(&S.dirty[slot][0]), &tmd, (int)((x0 >> 5) & ~int64_t(3)), (int)y0,
                                (int)(zb - 1 + i), full0 + 8 * slot);
            }
        }
        return;
    }
    // ---- consumers ----
    auto wait_plane = [&](int i) { mbar_wait(full0 + 8 * (i % kQSlots), (unsigned)((i / kQSlots) & 1)); };
    op.begin();
    const int lane = tx;
    const bool edge_xy = x0 == 0 || x0 + kQX >= d.nx || y0 == 0 || y0 + kQY >= d.ny;
    const int64_t x = x0 + tx, yr = y0 + kQRowsPerThread * ty;
    const bool live_x = x < d.hi[0];
    bool live[kQRowsPerThread];
#pragma unroll
    for (int r = 0; r < kQRowsPerThread; ++r) live[r] = live_x && yr + r < d.hi[1];
    // ids < 2^32 (plan limit): 32-bit index arithmetic
    const uint32_t ctile = (uint32_t)(x0 + y0 * sy + zb * sz);  // tile cell (0, 0) at plane zb
    uint32_t* q = S.queue[ty];
    const unsigned below = (1u << lane) - 1u;
    // Carry-over: a step evaluates only whole batches of 32 queued centres;
    // the (< 32) leftovers of plane zb + k wait for step k + 1 (entry bit 24
    // marks them), so the lanes stay busy although a warp queues only ~26
    // fragile centres per plane.  A carried entry needs planes k .. k + 2 one
    // step longer: a warp releases index k - 1 after step k.
    unsigned carry = 0;
    wait_plane(0);
    wait_plane(1);
    for (int k = 0; k < K; ++k) {
        // centre plane zc = zb + k: planes i = k, k + 1, k + 2
        wait_plane(k + 2);
        uint32_t code[kQRowsPerThread];
        bool want[kQRowsPerThread];
        {
            const uint8_t* ctl = S.code[(k + 1) % kQSlots];
            const uint32_t* dtl = S.dirty[(k + 1) % kQSlots] + ((x0 >> 5) & 3);
#pragma unroll
            for (int r = 0; r < kQRowsPerThread; ++r) {
                code[r] = ctl[(kQRowsPerThread * ty + r) * kQX + tx];
                want[r] = live[r] && code[r] != kRobust;
                if (kMasked) want[r] = want[r] && ((dtl[(kQRowsPerThread * ty + r) * 4] >> tx) & 1u);
            }
        }
        // q[0 .. carry) holds plane k - 1's leftovers; append plane k behind them
        unsigned n = carry;
#pragma unroll
        for (int r = 0; r < kQRowsPerThread; ++r) {
            const unsigned bal = __ballot_sync(0xffffffffu, want[r]);
            if (want[r]) q[n + __popc(bal & below)] = (uint32_t)(r * kQX + tx) | (code[r] << 16) | (1u << 24);
            n += __popc(bal);
        }
        __syncwarp();
        // whole batches (they include every carried entry: carry < 32); a short
        // queue waits for the next plane unless it holds carried entries; all at the end
        const unsigned m = (k == K - 1) ? n : (n >= 32 ? (n & ~31u) : (carry ? n : 0u));
        const int64_t zc = zb + k;
        const bool int_cur = !edge_xy && zc >= 1 && zc + 1 < d.nz;
        const bool int_prev = !edge_xy && zc - 1 >= 1 && zc < d.nz;
        const uint32_t cpl = ctile + (uint32_t)(kQRowsPerThread * ty) * sy32 + (uint32_t)k * sz32;
        for (unsigned e = lane; e < m; e += 32) {
            const uint32_t ent = q[e];
            const int cur = (int)((ent >> 24) & 1u);   // 1: plane k, 0: carried from plane k - 1
            const int base = k - 1 + cur;               // plane index of the entry's z - 1
            const int r = (int)((ent & 0xffffu) >> 5), lx = (int)(ent & 31u);
            const int cell = (kQRowsPerThread * ty + r + 1) * kQPX + xo + 1 + lx;
            double nv[14], vc;
            ring_from_smem(S.plane[base % kQSlots], S.plane[(base + 1) % kQSlots], S.plane[(base + 2) % kQSlots], cell,
                           nv, vc);
            const bool interior = cur ? int_cur : int_prev;
            const Scan s = interior ? tree_scan(vc, nv) : fold_scan(vc, nv);   // NaN = outside the field
            op.evaluate(d, (int64_t)(cpl - (cur ? 0u : sz32) + (uint32_t)r * sy32 + (uint32_t)lx), s,
                        (uint8_t)(ent >> 16));
        }
        __syncwarp();
        // leftovers of plane k move to the front, marked as carried
        const unsigned left = n - m;
        uint32_t mv = 0;
        if (lane < left) mv = q[m + lane] & ~(1u << 24);
        __syncwarp();
        if (lane < left) q[lane] = mv;
        carry = left;
        __syncwarp();
        if (lane == 0 && k >= 1) mbar_arrive(empty0 + 8 * ((k - 1) % kQSlots));   // index k - 1 is done
    }
    op.finish();
}

// A masked queue sweep stages its dirty words by TMA: bitmap rows must be whole
// 16-byte groups of words (nx % 128 == 0) and tiles must start on a word.
inline bool qsweep_masked_ok(const Dom& d) { return d.nx % 128 == 0 && d.lo[0] % 32 == 0; }

inline void qsweep_grid(const Dom& d, dim3& grid, int& zchunk) {
    const int64_t cx = d.hi[0] - d.lo[0], cy = d.hi[1] - d.lo[1], cz = d.hi[2] - d.lo[2];
    const int64_t tiles = ((cx + kQX - 1) / kQX) * ((cy + kQY - 1) / kQY);
    // z chunks of ~64 planes unless that leaves fewer than ~6 waves of
    // 148 SMs x 3 CTAs; never below 16 planes (a CTA stages zchunk + 2 planes)
    const int64_t want = (148 * 3 * 6 + tiles - 1) / tiles;
    int64_t chunks = std::max<int64_t>((cz + 63) / 64, std::min<int64_t>(want, cz / 16));
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, cz));
    zchunk = (int)std::max<int64_t>(1, (cz + chunks - 1) / chunks);
    static const int zc_env = getenv("PMSZ_SWEEP_ZCHUNK") ? atoi(getenv("PMSZ_SWEEP_ZCHUNK")) : 0;
    if (zc_env > 0) zchunk = (int)std::min<int64_t>(zc_env, cz);
    chunks = (cz + zchunk - 1) / zchunk;
    grid = dim3((unsigned)((cx + kQX - 1) / kQX), (unsigned)((cy + kQY - 1) / kQY), (unsigned)chunks);
}

template <bool kCount, bool kMasked, bool kExtrema>
inline bool launch_qsweep(const Dom& d, const double* g, const Work& w, cudaStream_t s, const uint32_t* dirty) {
    CUtensorMap tm, tmc, tmd;
    if (!tma_field_map(&tm, g, false, d.nx, d.ny, d.nz, kQPX, kQPY)) return false;
    // f-code tiles by TMA: 16-byte aligned tile origins and strides; masked
    // sweeps also stage their dirty words (bitmap rows of whole words)
    bool code_tma = d.lo[0] % 16 == 0 && tma_u8_map(&tmc, w.code, d.nx, d.ny, d.nz, kQX, kQY);
    if (kMasked) code_tma = code_tma && qsweep_masked_ok(d) && tma_u32_map(&tmd, dirty, d.nx / 32, d.ny, d.nz, 4, kQY);
    else tmd = tm;
    // Without TMA tiles the per-lane code (and dirty-word) loads sit on the
    // critical path of every plane; the shared-fold cp.async sweep of
    // tiles.cuh (which also skips robust centres) is faster there.
    if (!code_tma) return false;
    using Op = DetectOp<kCount, kMasked, kExtrema>;
    dim3 grid;
    int zchunk;
    qsweep_grid(d, grid, zchunk);
    Op op{w, dirty, 0};
    const dim3 block(kQX, kQConsumers + 1, 1);
    auto kern = k_qsweep_tma<kCount, kMasked, kExtrema>;
    static unsigned long long attr = 0;
    smem_attr_once(kern, (int)kQSmemBytes, attr);
    pdl_launch(kern, grid, block, kQSmemBytes, s, d, tm, tmc, tmd, op, zchunk);
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
