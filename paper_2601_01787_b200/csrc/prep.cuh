// prep.cuh -- K0 as a TMA-staged screen + queue kernel.
//
// K0 (correction.py:52-60,118-122,404-405) validates the pair, copies
// g <- fhat and builds the f-code (field_scan(original)).  The f-code is only
// ever read at centres that can mismatch, and K0 decides which those are
// (tiles.cuh, acc_robust): a centre is robust when the largest and the
// smallest member of its closed 1-ring in f lead the runners-up by more than
// 2 xi.  So instead of an exact (value, rank) fold at every centre, this
// kernel runs
//
//   * a cheap SCREEN at every centre: the top-2 and bottom-2 values of the
//     closed ring, no ranks -- min / max only (FMNMX / FMNMX3 on f32 fields),
//     with the 2 x 2 boxes of every plane shared by the three centres whose
//     rings contain them (one box per centre per plane);
//   * the exact f-code only for the fragile centres, from a per-plane queue
//     (the balanced-tree fold of qsweep.cuh on the staged values).
//
// Cells outside the field are NaN (TMA fill).  min / max ignore NaN, and a
// NaN can only duplicate a real value into a runner-up slot: the screen's
// gaps never exceed the true gaps, so a NaN can make a robust centre look
// fragile (it then gets its exact code), never the reverse.
#pragma once
#include "qsweep.cuh"

#ifndef PMSZ_PREP_MINB
#define PMSZ_PREP_MINB 3   // resident K0 CTAs per SM for f32 fields (smem allows 3)
#endif

namespace pmsz {

template <typename V> __device__ __forceinline__ V vmx(V a, V b);
template <typename V> __device__ __forceinline__ V vmn(V a, V b);
template <> __device__ __forceinline__ float vmx<float>(float a, float b) { return fmaxf(a, b); }
template <> __device__ __forceinline__ float vmn<float>(float a, float b) { return fminf(a, b); }
template <> __device__ __forceinline__ double vmx<double>(double a, double b) { return fmax(a, b); }
template <> __device__ __forceinline__ double vmn<double>(double a, double b) { return fmin(a, b); }

// x-pair: (hi, lo); its runner-up on the max side is lo and vice versa.
template <typename V>
struct P2 {
    V hi, lo;
};
template <typename V>
__device__ __forceinline__ P2<V> p2(V a, V b) { return P2<V>{vmx(a, b), vmn(a, b)}; }

// Top-2 / bottom-2 of a group.
template <typename V>
struct T2 {
    V mx, sx, mn, sn;
};
template <typename V>
__device__ __forceinline__ T2<V> box2(const P2<V>& a, const P2<V>& b) {
    return T2<V>{vmx(a.hi, b.hi), vmx(vmx(vmn(a.hi, b.hi), a.lo), b.lo),
                 vmn(a.lo, b.lo), vmn(vmn(vmx(a.lo, b.lo), a.hi), b.hi)};
}
template <typename V>
__device__ __forceinline__ void merge2(T2<V>& A, const T2<V>& G) {
    A.sx = vmx(vmx(A.sx, G.sx), vmn(A.mx, G.mx));
    A.mx = vmx(A.mx, G.mx);
    A.sn = vmn(vmn(A.sn, G.sn), vmx(A.mn, G.mn));
    A.mn = vmn(A.mn, G.mn);
}
template <typename V>
__device__ __forceinline__ void merge2(T2<V>& A, const P2<V>& P) { merge2(A, T2<V>{P.hi, P.lo, P.lo, P.hi}); }
template <typename V>
__device__ __forceinline__ void merge2(T2<V>& A, V v) {
    A.sx = vmx(A.sx, vmn(A.mx, v));
    A.mx = vmx(A.mx, v);
    A.sn = vmn(A.sn, vmx(A.mn, v));
    A.mn = vmn(A.mn, v);
}

// Robust iff both leads exceed 2 xi plus rounding slack (the bound of
// acc_robust in tiles.cuh, evaluated with directed rounding so that the f32
// comparison is conservative): thr = RU(2 xi (1 + 2^-30)).
__device__ __forceinline__ bool robust2(const T2<float>& a, float thr, double) {
    return a.sx < __fsub_rd(a.mx, thr) && a.sn > __fadd_ru(a.mn, thr);
}
__device__ __forceinline__ bool robust2(const T2<double>& a, double thr, double) {
    // f64 fields: the one-ulp rounding of f - xi is not absorbed by an f64
    // ulp of the difference, so add 2^-50 |v| explicitly
    return a.sx < __dsub_rd(__dsub_rd(a.mx, thr), 0x1p-50 * fabs(a.mx)) &&
           a.sn > __dadd_ru(__dadd_ru(a.mn, thr), 0x1p-50 * fabs(a.mn));
}

// f64 fields screened in f32 (k_prep_q): rounding to f32 is monotone, so the
// f32 top-2 / bottom-2 are the images of the f64 ones, each within 2^-24 |v|;
// the gap test absorbs both roundings (and the 2^-50 |v| of robust2's f64
// form) in 2^-22 max|v| plus an absolute 2^-120 for subnormal images.  Values
// beyond the f32 range become +-inf and fail the test (fragile: exact code).
__device__ __forceinline__ bool robust2_narrowed(const T2<float>& a, float thr32) {
    const float sx = __fadd_ru(__fmul_ru(0x1p-22f, fmaxf(fabsf(a.mx), fabsf(a.sx))), 0x1p-120f);
    const float sn = __fadd_ru(__fmul_ru(0x1p-22f, fmaxf(fabsf(a.mn), fabsf(a.sn))), 0x1p-120f);
    return a.sx < __fsub_rd(__fsub_rd(a.mx, thr32), sx) && a.sn > __fadd_ru(__fadd_ru(a.mn, thr32), sn);
}

// Extrema-only mode compares the extremum flags alone, so a side
// is also robust when the centre c trails the ring's largest (smallest)
// member by more than 2 xi: c can then never be the maximum (minimum) for any
// g in [f - xi, f + xi].  Per side: the ordinary lead test OR that one.
__device__ __forceinline__ bool robust_extrema(const T2<float>& a, float fc, float thr) {
    const float hi = __fsub_rd(a.mx, thr), lo = __fadd_ru(a.mn, thr);
    return fminf(a.sx, fc) < hi && fmaxf(a.sn, fc) > lo;
}
// (f64 fields screened in f32: the slack of robust2_narrowed, over c too)
__device__ __forceinline__ bool robust_extrema_narrowed(const T2<float>& a, float fc, float thr32) {
    const float afc = fabsf(fc);
    const float sx = __fadd_ru(__fmul_ru(0x1p-22f, fmaxf(fmaxf(fabsf(a.mx), fabsf(a.sx)), afc)), 0x1p-120f);
    const float sn = __fadd_ru(__fmul_ru(0x1p-22f, fmaxf(fmaxf(fabsf(a.mn), fabsf(a.sn)), afc)), 0x1p-120f);
    return fminf(a.sx, fc) < __fsub_rd(__fsub_rd(a.mx, thr32), sx) &&
           fmaxf(a.sn, fc) > __fadd_ru(__fadd_ru(a.mn, thr32), sn);
}

// Exact f-code of a queued centre (fold_scan / tree_scan on V values; NaN =
// outside the field, only in the fold).
template <typename V>
__device__ __forceinline__ uint8_t fold_code(V vc, const V (&nv)[14]) {
    V bmax = -vinf<V>(), bmin = vinf<V>();
    int rmax = 15, rmin = 15;
#pragma unroll
    for (int r = 0; r < 14; ++r) {
        const V v = nv[r];
        const bool tmax = v >= bmax;
        bmax = tmax ? v : bmax;
        rmax = tmax ? r : rmax;
        const bool tmin = v < bmin;
        bmin = tmin ? v : bmin;
        rmin = tmin ? r : rmin;
    }
    const bool is_max = (bmax < vc) || (bmax == vc && rmax <= kCenterBelow);   // topology.py:79
    const bool is_min = (bmin > vc) || (bmin == vc && rmin > kCenterBelow);    // topology.py:80
    return (uint8_t)((is_max ? kExtremum : rmax) | ((is_min ? kExtremum : rmin) << 4));
}
template <typename V>
__device__ __forceinline__ void tmax(V& v, int& r, V v2, int r2) {
    const bool t = v2 >= v;
    v = t ? v2 : v;
    r = t ? r2 : r;
}
template <typename V>
__device__ __forceinline__ void tmin(V& v, int& r, V v2, int r2) {
    const bool t = v2 < v;
    v = t ? v2 : v;
    r = t ? r2 : r;
}
template <typename V>
__device__ __forceinline__ uint8_t tree_code(V vc, const V (&nv)[14]) {
    V ax[7], an[7];
    int rx[7], rn[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const bool t = nv[2 * k + 1] >= nv[2 * k];
        ax[k] = t ? nv[2 * k + 1] : nv[2 * k];
        rx[k] = 2 * k + (t ? 1 : 0);
        an[k] = t ? nv[2 * k] : nv[2 * k + 1];
        rn[k] = 2 * k + (t ? 0 : 1);
    }
    tmax(ax[0], rx[0], ax[1], rx[1]); tmin(an[0], rn[0], an[1], rn[1]);
    tmax(ax[2], rx[2], ax[3], rx[3]); tmin(an[2], rn[2], an[3], rn[3]);
    tmax(ax[4], rx[4], ax[5], rx[5]); tmin(an[4], rn[4], an[5], rn[5]);
    tmax(ax[0], rx[0], ax[2], rx[2]); tmin(an[0], rn[0], an[2], rn[2]);
    tmax(ax[4], rx[4], ax[6], rx[6]); tmin(an[4], rn[4], an[6], rn[6]);
    tmax(ax[0], rx[0], ax[4], rx[4]); tmin(an[0], rn[0], an[4], rn[4]);
    const bool is_max = (ax[0] < vc) || (ax[0] == vc && rx[0] <= kCenterBelow);
    const bool is_min = (an[0] > vc) || (an[0] == vc && rn[0] > kCenterBelow);
    return (uint8_t)((is_max ? kExtremum : rx[0]) | ((is_min ? kExtremum : rn[0]) << 4));
}

// ---- layout ------------------------------------------------------------------
// f planes: 32 x 32 centres + halo; the TMA box starts 16-byte aligned, so a
// staged row begins kPA(T) - 1 cells left of x0 - 1 (T = f32: 4 per 16 B).
template <typename T> struct PrepGeo {
    static constexpr int kAlign = 16 / (int)sizeof(T);                      // cells per 16 B
    static constexpr int kPX = ((kQX + 1 + kAlign) + kAlign - 1) / kAlign * kAlign;   // 40 (f32) / 36 (f64)
    static constexpr int kPY = kQY + 2;
    static constexpr int kPlane = kPX * kPY;
    static constexpr int kStride = ((kPlane * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
    static constexpr int kSlots = 5;   // f planes in use k-1 .. k+2, one more in flight
    static constexpr int kHSlots = 4;  // fhat planes (with halo) in use k-1 .. k+1, one more in flight
};
template <typename T>
struct PrepSmem {
    using G = PrepGeo<T>;
    T plane[G::kSlots][G::kStride];
    double fh[G::kHSlots][kQPlaneStride];   // fhat = g of iteration 1, staged like qsweep.cuh
    uint16_t queue[2][kQX * kQY];   // code-tile index (row * 32 + x) of fragile centres
    unsigned long long bar[G::kSlots];
    unsigned long long hbar[G::kHSlots];
    unsigned cnt[3];
};

struct PrepArgs {
    double* g;          // may alias fhat (then no copy)
    uint8_t* code;
    uint32_t* frag;     // null: no robustness test (every centre gets its code)
    DevCounters* ctr;
    double xi;
    double thr;         // RU(2 xi (1 + 2^-30)) in the field's precision (f32 fields: rounded up)
    int frag_direct;    // nx % 32 == 0: a warp's ballot is exactly one bitmap word
    // fused first detection sweep (g = fhat): the fragile centres of the core
    // box are compared with their f-code right here (null: not fused)
    uint32_t* det;
    int extrema_only;
    int64_t core_lo[3], core_hi[3];
    int z0, z1;         // centre planes of this launch (z-slab launches overlap the input copy)
};

template <typename FT, bool kScreen, bool kDetect, bool kExtrema>
__global__ void __launch_bounds__(256, sizeof(FT) == 4 ? PMSZ_PREP_MINB : 2) k_prep_q(Dom d, const __grid_constant__ CUtensorMap tf,
                                                   const __grid_constant__ CUtensorMap th, PrepArgs a, int zchunk) {
    pdl_wait();   // (programmatic dependent launch)
    using G = PrepGeo<FT>;
    extern __shared__ __align__(1024) unsigned char praw[];
    PrepSmem<FT>& S = *reinterpret_cast<PrepSmem<FT>*>(praw);
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * kQX + tx, lane = tid & 31;
    // 32-bit coordinates (extents < 2^31, ids < 2^32: plan limits): fewer
    // registers than int64 in this register-bound kernel
    const int x0 = (int)blockIdx.x * kQX, y0 = (int)blockIdx.y * kQY;
    const int zb = a.z0 + (int)blockIdx.z * zchunk;
    const int K = min(zb + zchunk, a.z1) - zb;
    const uint32_t sy = (uint32_t)d.sy, sz = (uint32_t)d.sz;
    const int xs = (x0 - 1) & ~(G::kAlign - 1);
    const int xo = (int)(x0 - 1 - xs);   // column of x0 - 1 in a staged row
    const unsigned bar0 = smem_u32(&S.bar[0]), hbar0 = smem_u32(&S.hbar[0]);
    const unsigned pl0 = smem_u32(&S.plane[0][0]), fh0 = smem_u32(&S.fh[0][0]);
    // plane index i = p - (zb - 1), i in [0, K + 1], for f and fhat alike
    const int xh = (x0 - 1) & ~1;   // fhat boxes (f64): even origin
    const int xho = (int)(x0 - 1 - xh);
    auto issue = [&](int i) {
        const int s = i % G::kSlots;
        mbar_expect_tx(bar0 + 8 * s, G::kPlane * (unsigned)sizeof(FT));
        tma_load_3d(pl0 + s * G::kStride * (unsigned)sizeof(FT), &tf, (int)xs, (int)(y0 - 1), (int)(zb - 1 + i),
                    bar0 + 8 * s);
    };
    auto issue_h = [&](int j) {
        const int s = j % G::kHSlots;
        mbar_expect_tx(hbar0 + 8 * s, kQPlane * 8);
        tma_load_3d(fh0 + s * kQPlaneStride * 8, &th, (int)xh, (int)(y0 - 1), (int)(zb - 1 + j), hbar0 + 8 * s);
    };
    auto wait_plane = [&](int i) { mbar_wait(bar0 + 8 * (i % G::kSlots), (unsigned)((i / G::kSlots) & 1)); };
    auto wait_h = [&](int j) { mbar_wait(hbar0 + 8 * (j % G::kHSlots), (unsigned)((j / G::kHSlots) & 1)); };
    if (tid == 0) {
        for (int s = 0; s < G::kSlots; ++s) mbar_init(bar0 + 8 * s, 1);
        for (int s = 0; s < G::kHSlots; ++s) mbar_init(hbar0 + 8 * s, 1);
        mbar_fence_init();
        S.cnt[0] = S.cnt[1] = S.cnt[2] = 0;
        for (int i = 0; i <= 2 && i <= K + 1; ++i) issue(i);
        for (int j = 0; j <= 1 && j <= K + 1; ++j) issue_h(j);
    }
    const int x = x0 + tx, yr = y0 + kQRowsPerThread * ty;
    const bool live_x = x < d.nx;
    bool live[kQRowsPerThread];
#pragma unroll
    for (int r = 0; r < kQRowsPerThread; ++r) live[r] = live_x && yr + r < d.ny;
    const uint32_t c0 = (uint32_t)x + (uint32_t)yr * sy + (uint32_t)zb * sz;   // row-0 centre at plane zb
    const int col = xo + tx;                 // staged column of x - 1
    const int row0 = kQRowsPerThread * ty;   // staged row of y_0 - 1
    unsigned nfrag = 0, ndet = 0;
    using V = FT;       // staged values (exact f-codes of the fragile centres)
    using SV = float;   // screen values: f32 for both field types (robust2_narrowed for f64)

    // The closed ring of centre (x, y_r, p) is covered by four 2 x 2 boxes:
    // D = lb of plane p-1, the in-plane part lb + rb of plane p (they share the
    // centre itself, which is harmless -- a duplicated member can only lower
    // the screen's gaps, never raise them), and U = rb of plane p+1.
    // Plane p's shared groups for this thread's four centres, streamed row by
    // row: for centre r, emit(r, lb, rb, rp, leaf) with
    //   lb = 2 x 2 box at (x-1, y_r-1)  (D of plane p+1, in-plane of p)
    //   rb = 2 x 2 box at (x, y_r)      (U of plane p-1)
    //   rp = x-pair (x, y_r+1)-(x+1, y_r+1), leaf = (x+1, y_r)
    auto plane_groups = [&](const V* P, auto&& emit) {
        const V* row = P + row0 * G::kPX + col;
        SV l = (SV)row[0], m = (SV)row[1], rr = (SV)row[2];
        P2<SV> pl = p2(l, m), pr = p2(m, rr), pl1;
        SV leaf_prev = rr;
#pragma unroll
        for (int j = 1; j < kQRowsPerThread + 2; ++j) {
            row += G::kPX;
            l = (SV)row[0]; m = (SV)row[1];
            const SV rn = (SV)row[2];
            const P2<SV> pln = p2(l, m), prn = p2(m, rn);
            if (j >= 2) emit(j - 2, box2(pl1, pl), box2(pr, prn), prn, leaf_prev);
            pl1 = pl; pl = pln;
            pr = prn;
            leaf_prev = rn;
        }
        // centre r = kQRowsPerThread - 1 needs the lb of rows (3, 4): emitted above with j = 5
    };
    __syncthreads();
    // prologue: D boxes of plane zb - 1, partial rings of plane zb
    T2<SV> lbprev[kQRowsPerThread], acc[kQRowsPerThread];
    const float thr32 = sizeof(FT) == 4 ? (float)a.thr : __double2float_ru(a.thr);
    wait_plane(0);
    wait_plane(1);
    wait_h(0);
    plane_groups(S.plane[0], [&](int r, const T2<SV>& lb, const T2<SV>&, const P2<SV>&, SV) { lbprev[r] = lb; });
    plane_groups(S.plane[1], [&](int r, const T2<SV>& lb, const T2<SV>& rb, const P2<SV>&, SV) {
        acc[r] = lbprev[r];
        merge2(acc[r], lb);
        merge2(acc[r], rb);
        lbprev[r] = lb;
    });
    for (int k = 0; k <= K; ++k) {
        // step k: finalise + enqueue centre plane zb + k (needs f plane index k + 2),
        //         exact codes of the queue of plane zb + k - 1 (indices k - 1 .. k + 1)
        if (k < K) wait_plane(k + 2);
        wait_h(k + 1);
        __syncthreads();
        if (tid == 0) {
            if (k + 3 <= K + 1) issue(k + 3);
            if (k + 2 <= K + 1) issue_h(k + 2);
            S.cnt[(k + 1) % 3] = 0;
        }
        if (k < K) {
            const V* ctr_plane = S.plane[(k + 1) % G::kSlots];
            const double* fht = S.fh[(k + 1) % G::kHSlots] + kQPX + xho + 1 + tx;   // fhat at (x, y_0 - 1)
            const uint32_t cz = c0 + (uint32_t)k * sz;
            bool want[kQRowsPerThread];
            plane_groups(S.plane[(k + 2) % G::kSlots],
                         [&](int r, const T2<SV>& lb, const T2<SV>& rb, const P2<SV>& rp, SV leaf) {
                merge2(acc[r], rb);   // U group: the ring of centre r is complete
                const uint32_t c = cz + r * sy;
                bool robust = kScreen && (sizeof(FT) == 4 ? robust2(acc[r], thr32, a.xi)
                                                          : robust2_narrowed(acc[r], thr32));
                if (kExtrema && kScreen && !robust) {
                    const SV fcv = (SV)ctr_plane[(row0 + r + 1) * G::kPX + col + 1];
                    robust = sizeof(FT) == 4 ? robust_extrema(acc[r], fcv, thr32)
                                             : robust_extrema_narrowed(acc[r], fcv, thr32);
                }
                want[r] = live[r] && !robust;
                if (live[r]) {
                    // validation (correction.py:52-60), hazard H6, g <- fhat
                    const double fv = (double)ctr_plane[(row0 + r + 1) * G::kPX + col + 1];
                    const double hv = fht[(row0 + r) * kQPX];
                    // one predicate on the fast path: NaN / Inf fail every
                    // comparison, so `ok` implies all four tests below pass
                    const bool ok = fabs(fv - hv) <= a.xi && hv >= fv - a.xi && hv <= fv + a.xi;
                    if (!ok) {   // rare (an invalid pair): count straight into the counters
                        if (!isfinite(fv) || !isfinite(hv)) atomicAdd(&a.ctr->nonfinite, 1ull);
                        if (fabs(fv - hv) > a.xi) {
                            atomicAdd(&a.ctr->bound_viol, 1ull);
                            atomicMin(&a.ctr->bound_first, (unsigned long long)c);
                        }
                        if (hv < fv - a.xi) atomicAdd(&a.ctr->floor_viol, 1ull);
                        if (hv > fv + a.xi) atomicAdd(&a.ctr->upper_viol, 1ull);
                    }
                    if (robust) a.code[c] = kRobust;
                }
                // partial ring of the same column at plane zb + k + 1
                acc[r] = lbprev[r];
                merge2(acc[r], lb);
                merge2(acc[r], rb);
                lbprev[r] = lb;
            });
            if (a.g != nullptr) {
#pragma unroll
                for (int r = 0; r < kQRowsPerThread; ++r)
                    if (live[r]) a.g[cz + r * sy] = fht[(row0 + r) * kQPX];
            }
            // fragile bitmap and queue
            unsigned bal[kQRowsPerThread], tot = 0;
#pragma unroll
            for (int r = 0; r < kQRowsPerThread; ++r) {
                bal[r] = __ballot_sync(0xffffffffu, want[r]);
                tot += __popc(bal[r]);
            }
            if (kScreen && a.frag_direct) {
                // one word per row: lane r stores row r's ballot
                if (lane < kQRowsPerThread && yr + lane < d.ny) {
                    unsigned b = bal[0];
#pragma unroll
                    for (int r = 1; r < kQRowsPerThread; ++r) b = lane == r ? bal[r] : b;
                    a.frag[(cz - (uint32_t)tx + (uint32_t)lane * sy) >> 5] = b;
                }
            } else if (kScreen && lane == 0) {
#pragma unroll
                for (int r = 0; r < kQRowsPerThread; ++r) {
                    const uint32_t cw = cz + r * sy;   // id of lane 0's centre
                    if (bal[r]) {
                        const unsigned sh = cw & 31;
                        atomicOr(a.frag + (cw >> 5), bal[r] << sh);
                        if (sh && (bal[r] >> (32 - sh))) atomicOr(a.frag + (cw >> 5) + 1, bal[r] >> (32 - sh));
                    }
                }
            }
            nfrag += lane == 0 ? tot : 0u;   // want = live && !robust
            unsigned base = 0;
            if (lane == 0 && tot) base = atomicAdd(&S.cnt[k % 3], tot);
            base = __shfl_sync(0xffffffffu, base, 0);
            const unsigned below = (1u << lane) - 1u;
            uint16_t* q = S.queue[k & 1];
#pragma unroll
            for (int r = 0; r < kQRowsPerThread; ++r) {
                if (want[r]) q[base + __popc(bal[r] & below)] = (uint16_t)((row0 + r) * kQX + tx);
                base += __popc(bal[r]);
            }
        }
        if (k >= 1) {
            // exact f-codes of the fragile centres of plane zc = zb + k - 1
            const int zc = zb + k - 1;
            const unsigned n = S.cnt[(k - 1) % 3];
            const uint16_t* q = S.queue[(k - 1) & 1];
            const V* dn = S.plane[(k - 1) % G::kSlots];
            const V* ct = S.plane[k % G::kSlots];
            const V* up = S.plane[(k + 1) % G::kSlots];
            const bool edge = x0 == 0 || x0 + kQX >= d.nx || y0 == 0 || y0 + kQY >= d.ny || zc == 0 || zc + 1 >= d.nz;
            const uint32_t cpl = c0 - (uint32_t)tx - (uint32_t)(kQRowsPerThread * ty) * sy + (uint32_t)(k - 1) * sz;
            for (unsigned e = tid; e < n; e += 256) {
                const int idx = q[e];
                const int ly = idx >> 5, lx = idx & 31;
                const int cell = (ly + 1) * G::kPX + xo + 1 + lx;
                V nv[14];
                nv[0] = dn[cell - G::kPX - 1]; nv[1] = dn[cell - G::kPX]; nv[2] = dn[cell - 1]; nv[3] = dn[cell];
                nv[4] = ct[cell - G::kPX - 1]; nv[5] = ct[cell - G::kPX]; nv[6] = ct[cell - 1]; nv[7] = ct[cell + 1];
                nv[8] = ct[cell + G::kPX]; nv[9] = ct[cell + G::kPX + 1];
                nv[10] = up[cell]; nv[11] = up[cell + 1]; nv[12] = up[cell + G::kPX]; nv[13] = up[cell + G::kPX + 1];
                const V vc = ct[cell];
                const uint8_t fc = edge ? fold_code<V>(vc, nv) : tree_code<V>(vc, nv);
                const uint32_t c = cpl + ly * sy + lx;
                a.code[c] = fc;
                if (kDetect) {
                    // the first detection sweep (g = fhat) of this centre
                    const int gx = x0 + lx, gy = y0 + ly;
                    if (gx >= a.core_lo[0] && gx < a.core_hi[0] && gy >= a.core_lo[1] && gy < a.core_hi[1] &&
                        zc >= a.core_lo[2] && zc < a.core_hi[2]) {
                        double hv[14], hc;
                        ring_from_smem(S.fh[(k - 1) % G::kHSlots], S.fh[k % G::kHSlots], S.fh[(k + 1) % G::kHSlots],
                                       (ly + 1) * kQPX + xho + 1 + lx, hv, hc);
                        const uint8_t gc = scan_code(edge ? fold_scan(hc, hv) : tree_scan(hc, hv));
                        const bool mismatch = a.extrema_only
                                                  ? (((gc & 15) == kExtremum) != ((fc & 15) == kExtremum) ||
                                                     ((gc >> 4) == kExtremum) != ((fc >> 4) == kExtremum))
                                                  : gc != fc;
                        if (mismatch) {
                            atomicOr(a.det + (c >> 5), 1u << (c & 31));
                            ++ndet;
                        }
                    }
                }
            }
        }
    }
    const unsigned nfr = __reduce_add_sync(0xffffffffu, nfrag);
    const unsigned nd = __reduce_add_sync(0xffffffffu, ndet);
    if (lane == 0) {
        if (nd) atomicAdd(&a.ctr->ndetect, (unsigned long long)nd);
        if (nfr) atomicAdd(&a.ctr->nfragile, (unsigned long long)nfr);
    }
}

// Launch K0 over the whole domain (ghost layers included: the f-code of a
// block's ext field is scan_neighbors(f_ext), parallel.py:212).  Returns false
// when the fields cannot be described by tensor maps (the caller then runs
// the shared-fold K0 of tiles.cuh).
template <typename FT>
inline bool launch_prep_q(const Dom& d, const FT* f, const double* fh, double* g, uint8_t* code, uint32_t* frag,
                          DevCounters* ctr, uint32_t* det, cudaStream_t s, int64_t z0 = 0, int64_t z1 = -1,
                          bool pdl = true) {
    if (z1 < 0) z1 = d.nz;
    using G = PrepGeo<FT>;
    CUtensorMap tf, th;
    if (!tma_field_map(&tf, f, sizeof(FT) == 4, d.nx, d.ny, d.nz, G::kPX, G::kPY)) return false;
    if (!tma_field_map(&th, fh, false, d.nx, d.ny, d.nz, kQPX, kQPY)) return false;
    PrepArgs a;
    a.g = (g != fh) ? g : nullptr;
    a.code = code;
    a.frag = frag;
    a.ctr = ctr;
    a.xi = d.xi;
    const double t = 2.0 * d.xi * (1.0 + 0x1p-30);
    if (sizeof(FT) == 4) {
        float t32 = (float)t;
        if ((double)t32 < t) t32 = nextafterf(t32, INFINITY);
        a.thr = (double)t32;
    } else {
        a.thr = nextafter(t, INFINITY);
    }
    a.frag_direct = (d.nx % 32) == 0;
    a.det = det;
    a.extrema_only = d.extrema_only;
    for (int ax = 0; ax < 3; ++ax) { a.core_lo[ax] = d.lo[ax]; a.core_hi[ax] = d.hi[ax]; }
    a.z0 = (int)z0;
    a.z1 = (int)z1;
    const int64_t nzr = z1 - z0;
    Dom all = d;
    for (int ax = 0; ax < 3; ++ax) all.lo[ax] = 0;
    all.hi[0] = d.nx; all.hi[1] = d.ny; all.hi[2] = d.nz;
    const int64_t tiles = ((d.nx + kQX - 1) / kQX) * ((d.ny + kQY - 1) / kQY);
    const int64_t want = (148 * 2 * 6 + tiles - 1) / tiles;
    // z chunks of at most 24 planes: the ~+8 % halo re-reads cost less than
    // the tail of fewer, longer CTAs (512^3: 1.33 ms at 64 planes, 1.27 at 20-26)
    int64_t chunks = std::max<int64_t>((nzr + 23) / 24, std::min<int64_t>(want, nzr / 16));
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, nzr));
    int zchunk = (int)std::max<int64_t>(1, (nzr + chunks - 1) / chunks);
    static const int zc_env = getenv("PMSZ_PREP_ZCHUNK") ? atoi(getenv("PMSZ_PREP_ZCHUNK")) : 0;
    if (zc_env > 0) zchunk = (int)std::min<int64_t>(zc_env, nzr);
    chunks = (nzr + zchunk - 1) / zchunk;
    const dim3 grid((unsigned)((d.nx + kQX - 1) / kQX), (unsigned)((d.ny + kQY - 1) / kQY), (unsigned)chunks);
    const dim3 block(kQX, kQY / kQRowsPerThread, 1);
    const size_t smem = sizeof(PrepSmem<FT>);
#define PMSZ_LAUNCH_PREP(R, D)                                                    \
    {                                                                             \
        static unsigned long long attr = 0;                                      \
        smem_attr_once(k_prep_q<FT, R, D, E>, (int)smem, attr);                  \
        if (pdl)   /* (the slab launches wait on copy events: ordinary launches) */             \
            pdl_launch(k_prep_q<FT, R, D, E>, grid, block, smem, s, all, tf, th, a, zchunk);      \
        else                                                                                       \
            k_prep_q<FT, R, D, E><<<grid, block, smem, s>>>(all, tf, th, a, zchunk);              \
    }
    if (frag && det && d.extrema_only) { constexpr bool E = true; PMSZ_LAUNCH_PREP(true, true); }
    else if (frag && d.extrema_only) { constexpr bool E = true; PMSZ_LAUNCH_PREP(true, false); }
    else if (frag && det) { constexpr bool E = false; PMSZ_LAUNCH_PREP(true, true); }
    else if (frag) { constexpr bool E = false; PMSZ_LAUNCH_PREP(true, false); }
    else if (det) { constexpr bool E = false; PMSZ_LAUNCH_PREP(false, true); }
    else { constexpr bool E = false; PMSZ_LAUNCH_PREP(false, false); }
#undef PMSZ_LAUNCH_PREP
    return true;
}

}  // namespace pmsz
