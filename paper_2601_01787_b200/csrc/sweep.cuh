// sweep.cuh -- detection / proposal / apply kernels of the correction loop.
//
// K1  detect+propose : per centre, steepest-neighbour scan of g, compare with
//                      the packed f-code, and on a mismatch run the six rules of
//                      correction.py:169-229, min-merging every
//                      proposal g[a]-tau into prop[t] with a 64-bit atomicMin on
//                      an order-preserving key.  The first proposer of a target
//                      appends it to the work list (warp-aggregated).
// K2  apply          : over the work list, g' = max(min(g, p), f - xi)
//                      (correction.py:239), edit counting, per-vertex edit
//                      counts, ever-edited bitmap, dirty 1-ring for the next
//                      incremental sweep, shared_dirty (parallel.py:249-250).
// K4  verify         : the K1 scan in counting mode (correction.py:424-426).
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace pmsz {
namespace cg = cooperative_groups;

struct DevCounters {
    unsigned long long nwork;        // targets in the work list
    unsigned long long nedits;       // edits of the iteration
    unsigned long long ndetect;      // centres with >= 1 detection
    unsigned long long shared_dirty;
    unsigned long long nact[2];      // dirty-list lengths (ping-pong)
    unsigned long long maxcount;     // max per-vertex edit count
    unsigned long long kinds[6];     // verify: per-kind detection counts
    unsigned long long bound_viol;
    unsigned long long bound_first;
    unsigned long long floor_viol;
    unsigned long long upper_viol;
    unsigned long long nonfinite;
    unsigned long long changed;      // merge helpers
    unsigned long long scratch[4];
};

struct Work {
    unsigned long long* prop;   // n, kNoProposal when idle
    uint32_t* work;             // target list (cap n)
    uint32_t* act[2];           // dirty centre lists
    uint32_t* actbits;          // n bits
    uint32_t* editbits;         // n bits: ever edited
    uint16_t* counts;           // per-vertex edit counts
    uint8_t* code;              // packed f-code
    uint8_t* edited_mask;       // optional per-iteration mask
    DevCounters* ctr;
    unsigned long long act_cap;
    int incremental;
};

// Warp-aggregated append: returns the slot of this thread in `counter`.
__device__ __forceinline__ unsigned long long agg_append(unsigned long long* counter) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(counter, (unsigned long long)g.size());
    base = g.shfl(base, 0);
    return base + g.thread_rank();
}

__device__ __forceinline__ void propose(const Work& w, int64_t t, double val) {
    const unsigned long long k = okey(val);
    // Skip the atomic when the current value already dominates (exact: min-merge).
    if (k >= w.prop[t]) return;
    const unsigned long long old = atomicMin(w.prop + t, k);
    if (old == kNoProposal) {
        const unsigned long long slot = agg_append(&w.ctr->nwork);
        w.work[slot] = (uint32_t)t;
    }
}

// Mismatch between the g-scan and the f-code, i.e. "some rule fires".
__device__ __forceinline__ bool code_mismatch(const Dom& d, uint8_t gcode, uint8_t fcode) {
    if (!d.extrema_only) return gcode != fcode;
    const bool gx = (gcode & 15) == kExtremum, fx = (fcode & 15) == kExtremum;
    const bool gn = (gcode >> 4) == kExtremum, fn = (fcode >> 4) == kExtremum;
    return (gx != fx) || (gn != fn);
}

// The six rules for centre c (correction.py:169-229).  kCount:
// count detections per kind instead of proposing (verify sweep).
template <bool kCount>
__device__ __noinline__ void rules(const Dom& d, const double* __restrict__ g, const Work& w,
                                   const Scan& s, uint8_t fcode, int64_t c,
                                   int64_t x, int64_t y, int64_t z) {
    const int fr = fcode & 15, fs = fcode >> 4;
    const bool fmax = fr == kExtremum, fmin = fs == kExtremum;
    const bool k_fpmax = s.is_max && !fmax;
    const bool k_fnmax = fmax && !s.is_max;
    const bool k_fpmin = s.is_min && !fmin;
    const bool k_fnmin = fmin && !s.is_min;
    const bool k_asc = !d.extrema_only && !fmax && s.rmax != fr;
    const bool k_desc = !d.extrema_only && !fmin && s.rmin != fs;
    if (kCount) {
        if (k_fpmax) atomicAdd(&w.ctr->kinds[0], 1ull);
        if (k_fnmax) atomicAdd(&w.ctr->kinds[1], 1ull);
        if (k_fpmin) atomicAdd(&w.ctr->kinds[2], 1ull);
        if (k_fnmin) atomicAdd(&w.ctr->kinds[3], 1ull);
        if (k_asc) atomicAdd(&w.ctr->kinds[4], 1ull);
        if (k_desc) atomicAdd(&w.ctr->kinds[5], 1ull);
        return;
    }
    if (!(k_fpmax | k_fnmax | k_fpmin | k_fnmin | k_asc | k_desc)) return;
    atomicAdd(&w.ctr->ndetect, 1ull);
    const double tau = d.tau;
    // FALSE_MAXIMUM: target c, anchor f.nmax(c)          (correction.py:213-215)
    if (k_fpmax) propose(w, c, __ldg(g + c + rank_off(d, fr)) - tau);
    // MISSING_MAXIMUM: anchor c, targets above c            (correction.py:216-218)
    if (k_fnmax) {
        const double vc = s.vc, val = vc - tau;
#pragma unroll 1
        for (int r = 0; r < 14; ++r) {
            if (!in_dom(d, x + rank_dx(r), y + rank_dy(r), z + rank_dz(r))) continue;
            const int64_t j = c + rank_off(d, r);
            const double vj = __ldg(g + j);
            if (vj > vc || (vj == vc && r > kCenterBelow)) propose(w, j, val);
        }
    }
    // ASC_ORDER: anchor a = f.nmax(c), targets above a     (correction.py:225-227)
    if (k_asc) {
        const double va = __ldg(g + c + rank_off(d, fr)), val = va - tau;
#pragma unroll 1
        for (int r = 0; r < 14; ++r) {
            if (!in_dom(d, x + rank_dx(r), y + rank_dy(r), z + rank_dz(r))) continue;
            const int64_t j = c + rank_off(d, r);
            const double vj = __ldg(g + j);
            if (vj > va || (vj == va && r > fr)) propose(w, j, val);
        }
    }
    // FALSE_MINIMUM: anchor c, target f.nmin(c)            (correction.py:219-221)
    if (k_fpmin) propose(w, c + rank_off(d, fs), s.vc - tau);
    // MISSING_MINIMUM: anchor g.nmin(c), target c           (correction.py:222-224)
    if (k_fnmin) propose(w, c, s.vmin - tau);
    // DESC_ORDER: anchor g.nmin(c), target f.nmin(c)        (correction.py:228-229)
    if (k_desc) propose(w, c + rank_off(d, fs), s.vmin - tau);
}

// ---------------------------------------------------------------------------
// K1/K4 full sweep over the core box, one thread per centre (gather form).
template <bool kCount>
__global__ void __launch_bounds__(256) k_sweep_gather(Dom d, const double* __restrict__ g, Work w) {
    const int64_t x = d.lo[0] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t y = d.lo[1] + (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    const int64_t z = d.lo[2] + (int64_t)blockIdx.z;
    if (x >= d.hi[0] || y >= d.hi[1]) return;
    const int64_t c = x + y * d.sy + z * d.sz;
    const Scan s = gather_scan(d, g, x, y, z);
    const uint8_t fc = w.code[c];
    if (code_mismatch(d, scan_code(s), fc)) rules<kCount>(d, g, w, s, fc, c, x, y, z);
}

// K1 sparse sweep over the dirty-centre list (grid-stride; count read on device).
__global__ void __launch_bounds__(256) k_sweep_sparse(Dom d, const double* __restrict__ g, Work w,
                                                     int cur) {
    const unsigned long long n = min(w.ctr->nact[cur], w.act_cap);
    const uint32_t* list = w.act[cur];
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int64_t c = list[i];
        atomicAnd(w.actbits + (c >> 5), ~(1u << (c & 31)));
        int64_t x, y, z;
        coords(d, c, x, y, z);
        const Scan s = gather_scan(d, g, x, y, z);
        const uint8_t fc = w.code[c];
        if (code_mismatch(d, scan_code(s), fc)) rules<false>(d, g, w, s, fc, c, x, y, z);
    }
}

__device__ __forceinline__ bool in_core(const Dom& d, int64_t x, int64_t y, int64_t z) {
    return x >= d.lo[0] && x < d.hi[0] && y >= d.lo[1] && y < d.hi[1] && z >= d.lo[2] && z < d.hi[2];
}

__device__ __forceinline__ bool in_shared(const Dom& d, int64_t x, int64_t y, int64_t z) {
    return (x < d.shl[0]) || (x >= d.nx - d.shh[0]) || (y < d.shl[1]) || (y >= d.ny - d.shh[1]) ||
           (z < d.shl[2]) || (z >= d.nz - d.shh[2]);
}

// Add the closed 1-ring of v (restricted to core centres) to the dirty list `nxt`.
__device__ __forceinline__ void mark_ring(const Dom& d, const Work& w, int64_t v, int nxt) {
    int64_t x, y, z;
    coords(d, v, x, y, z);
#pragma unroll 1
    for (int r = -1; r < 14; ++r) {
        const int64_t px = x + (r < 0 ? 0 : rank_dx(r));
        const int64_t py = y + (r < 0 ? 0 : rank_dy(r));
        const int64_t pz = z + (r < 0 ? 0 : rank_dz(r));
        if (!in_core(d, px, py, pz)) continue;
        const int64_t u = px + py * d.sy + pz * d.sz;
        const uint32_t bit = 1u << (u & 31);
        if (__ldcg(w.actbits + (u >> 5)) & bit) continue;
        const uint32_t old = atomicOr(w.actbits + (u >> 5), bit);
        if (old & bit) continue;
        const unsigned long long slot = agg_append(&w.ctr->nact[nxt]);
        if (slot < w.act_cap) w.act[nxt][slot] = (uint32_t)u;
    }
}

// K2 apply over the work list.
template <typename FT>
__global__ void __launch_bounds__(256) k_apply(Dom d, const FT* __restrict__ f, double* __restrict__ g,
                                               Work w, int nxt) {
    const unsigned long long n = w.ctr->nwork;
    unsigned long long my_edits = 0;
    unsigned int my_max = 0;
    bool my_shared = false;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int64_t t = w.work[i];
        const double p = okey_inv(w.prop[t]);
        w.prop[t] = kNoProposal;
        const double gt = g[t];
        const double lower = (double)f[t] - d.xi;           // BoundsField.lower (correction.py:122)
        const double m = (p < gt) ? p : gt;                  // np.minimum(g, prop)
        const double nv = (m < lower) ? lower : m;           // np.maximum(., lower)
        if (nv != gt) {
            g[t] = nv;
            ++my_edits;
            const unsigned int cnt = (unsigned int)w.counts[t] + 1u;
            w.counts[t] = (uint16_t)min(cnt, 65535u);
            my_max = max(my_max, cnt);
            atomicOr(w.editbits + (t >> 5), 1u << (t & 31));
            if (w.edited_mask) w.edited_mask[t] = 1;
            int64_t x, y, z;
            coords(d, t, x, y, z);
            my_shared |= in_shared(d, x, y, z);
            if (w.incremental) mark_ring(d, w, t, nxt);
        }
    }
    // Block-level reduction of the counters, one atomic per warp.
    const unsigned long long we = __reduce_add_sync(0xffffffffu, (unsigned)my_edits);
    const unsigned int wm = __reduce_max_sync(0xffffffffu, my_max);
    const unsigned int ws = __reduce_or_sync(0xffffffffu, my_shared ? 1u : 0u);
    if ((threadIdx.x & 31) == 0) {
        if (we) atomicAdd(&w.ctr->nedits, we);
        if (wm) atomicMax(&w.ctr->maxcount, (unsigned long long)wm);
        if (ws) atomicOr(&w.ctr->shared_dirty, 1ull);
    }
}

}  // namespace pmsz
