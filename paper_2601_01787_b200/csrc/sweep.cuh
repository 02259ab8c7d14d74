// sweep.cuh -- detection / proposal / apply kernels of the correction loop.
//
// K1  detect+propose : per centre, steepest-neighbour scan of g, compare with
//                      the packed f-code, and on a mismatch run the six rules of
//                      correction.py:169-229 on the register-resident
//                      neighbour values.  Every proposal g[a]-tau is min-merged
//                      into prop[t] by a fire-and-forget 64-bit RED.MIN on an
//                      order-preserving key (exactly np.minimum.at) and t is
//                      flagged in the `touched` bitmap (RED.OR).  Sparse sweeps
//                      additionally append first-touched targets to a work list.
// K2  apply          : over the touched targets, g' = max(min(g, p), f - xi)
//                      (correction.py:239), edit counting, per-vertex edit
//                      counts, ever-edited bitmap, dirty 1-ring for the next
//                      incremental sweep, shared_dirty (parallel.py:249-250).
// K4  verify         : the K1 scan in counting mode (correction.py:424-426).
#pragma once
#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>
#include "common.cuh"

namespace pmsz {
namespace cg = cooperative_groups;

struct DevCounters {
    unsigned long long nwork;        // targets in the work list (sparse mode)
    unsigned long long nedits;       // edits of the iteration
    unsigned long long ndetect;      // centres with >= 1 detection
    unsigned long long shared_dirty;
    unsigned long long ndefer;       // mismatching centres handed from a tiled sweep to k_defer
    unsigned long long nelist;       // edits recorded for list-mode ring marking
    unsigned long long nact[2];      // dirty-list lengths (ping-pong)
    unsigned long long maxcount;     // max per-vertex edit count
    unsigned long long kinds[6];     // verify: per-kind detection counts
    unsigned long long bound_viol;
    unsigned long long bound_first;
    unsigned long long floor_viol;
    unsigned long long upper_viol;
    unsigned long long nonfinite;
    unsigned long long nfragile;     // K0: centres that are not robust
    unsigned long long changed;      // merge helpers
    unsigned long long scratch[4];
};

struct Work {
    unsigned long long* prop;   // n, kNoProposal when idle
    uint32_t* touched;          // n bits: has a pending proposal
    uint32_t* work;             // target list (sparse mode)
    uint32_t* act[2];           // dirty centre lists
    uint32_t* actbits;          // n bits
    uint32_t* editbits;         // n bits: ever edited
    uint32_t* detbits;          // n bits: centre had a detection at its latest evaluation
    uint32_t* iteredit;         // n bits: edited in this iteration (bitmap-mode marking)
    uint32_t* elist;            // edits of a list-mode iteration (ring marking input)
    void* counts;               // per-vertex edit counts MINUS ONE where editbits is set (0 elsewhere): u16, or u32 when counts32
    int counts32;               // the iteration cap exceeds 65535 (a vertex is edited at most once per iteration)
    uint8_t* code;              // packed f-code
    const uint32_t* frag;       // n bits: fragile centres (K0); null = every centre is evaluated
    uint8_t* edited_mask;       // optional per-iteration mask
    DevCounters* ctr;
    unsigned long long act_cap;
    unsigned long long mark_limit;  // K2 skips ring marking above this many detections
    int64_t nwords;
    int incremental;
    int track;                  // append first-touched targets to `work`
    int first_apply;            // the run's first apply: no vertex was edited before (counts / editbits not read)
};

// Warp-aggregated append: returns the slot of this thread in `counter`.
__device__ __forceinline__ unsigned long long agg_append(unsigned long long* counter) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(counter, (unsigned long long)g.size());
    base = g.shfl(base, 0);
    return base + g.thread_rank();
}

// Proposal g[a]-tau -> prop[t]: min-merge by RED.MIN on the order key (exactly
// np.minimum.at) and flag t in the touched bitmap (RED.OR).  Nothing returns,
// so a thread's proposals are all in flight at once.
__device__ __forceinline__ void propose_red(const Work& w, int64_t t, double val) {
    atomicMin(w.prop + t, okey(val));
    atomicOr(w.touched + (t >> 5), 1u << (t & 31));
}

struct EmitRed {
    const Work& w;
    __device__ __forceinline__ void operator()(int64_t t, double val) { propose_red(w, t, val); }
};

// Sparse sweeps also remember their targets; flush() reserves the thread's
// slots of the work list with one warp-aggregated atomic.  Duplicates across
// centres are resolved in K2 (first to clear the touched bit applies).
struct EmitList {
    const Work& w;
    uint32_t t[18];
    int n;
    __device__ __forceinline__ void operator()(int64_t tt, double val) {
        propose_red(w, tt, val);
        t[n++] = (uint32_t)tt;
    }
    __device__ __forceinline__ void flush() {
        cg::coalesced_group g = cg::coalesced_threads();
        const unsigned mine = (unsigned)n;
        const unsigned before = cg::exclusive_scan(g, mine);
        const unsigned total = g.shfl(before + mine, g.size() - 1);
        unsigned long long base = 0;
        if (g.thread_rank() == 0 && total) base = atomicAdd(&w.ctr->nwork, (unsigned long long)total);
        base = g.shfl(base, 0) + before;
        for (int i = 0; i < n; ++i) w.work[base + i] = t[i];
    }
};

// Mismatch between the g-scan and the f-code, i.e. "some rule fires".
__device__ __forceinline__ bool code_mismatch(const Dom& d, uint8_t gcode, uint8_t fcode) {
    if (fcode == kRobust) return false;   // robust centres never mismatch (tiles.cuh, acc_robust)
    if (!d.extrema_only) return gcode != fcode;
    const bool gx = (gcode & 15) == kExtremum, fx = (fcode & 15) == kExtremum;
    const bool gn = (gcode >> 4) == kExtremum, fn = (fcode >> 4) == kExtremum;
    return (gx != fx) || (gn != fn);
}

__device__ __forceinline__ double pick(const double (&nv)[14], int r) {
    double v = nv[0];
#pragma unroll
    for (int k = 1; k < 14; ++k) v = (r == k) ? nv[k] : v;
    return v;
}

// The six rules for centre c (correction.py:169-229) on the
// snapshot values nv[] (rank order, NaN = outside the domain).  kCount:
// count detections per kind instead of proposing (verify sweep).
template <bool kCount, class Emit>
__device__ __forceinline__ void rules(const Dom& d, const Work& w, const Scan& s, const double (&nv)[14],
                                      uint8_t fcode, int64_t c, Emit& propose) {
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
    const double tau = d.tau;
    const double vc = s.vc;
    // FALSE_MAXIMUM: target c, anchor f.nmax(c)              (correction.py:213-215)
    // ASC_ORDER: anchor a = f.nmax(c), targets above a         (correction.py:225-227)
    // MISSING_MAXIMUM: anchor c, targets above c               (correction.py:216-218)
    if (k_fpmax || k_asc) {
        const double va = pick(nv, fr);
        if (k_fpmax) propose(c, va - tau);
        if (k_asc) {
            const double val = va - tau;
#pragma unroll
            for (int r = 0; r < 14; ++r) {
                const double vj = nv[r];
                if (vj > va || (vj == va && r > fr)) propose(c + rank_off(d, r), val);
            }
        }
    }
    if (k_fnmax) {
        const double val = vc - tau;
#pragma unroll
        for (int r = 0; r < 14; ++r) {
            const double vj = nv[r];
            if (vj > vc || (vj == vc && r > kCenterBelow)) propose(c + rank_off(d, r), val);
        }
    }
    // FALSE_MINIMUM: anchor c, target f.nmin(c)               (correction.py:219-221)
    if (k_fpmin) propose(c + rank_off(d, fs), vc - tau);
    // MISSING_MINIMUM: anchor g.nmin(c), target c              (correction.py:222-224)
    if (k_fnmin) propose(c, s.vmin - tau);
    // DESC_ORDER: anchor g.nmin(c), target f.nmin(c)           (correction.py:228-229)
    if (k_desc) propose(c + rank_off(d, fs), s.vmin - tau);
}

// Rule evaluation of the centres a tiled sweep found mismatching (their ids are
// in w.work[0 .. ndefer)); one thread per centre, neighbours gathered from g.
__global__ void __launch_bounds__(256) k_defer(Dom d, const double* __restrict__ g, Work w) {
    pdl_wait();   // (programmatic dependent launch)
    const unsigned long long n = w.ctr->ndefer;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int64_t c = w.work[i];
        const uint8_t fc = w.code[c];
        int64_t x, y, z;
        coords(d, c, x, y, z);
        double nv[14];
        // interior centres (all but the domain faces): plain pointer arithmetic
        // and the balanced-tree fold; faces: bounds checks and the NaN fold
        load_ring(d, g, c, x, y, z, nv, [](const double* q) { return __ldg(q); });
        const double vc = __ldg(g + c);
        const bool interior = x > 0 && x + 1 < d.nx && y > 0 && y + 1 < d.ny && z > 0 && z + 1 < d.nz;
        const Scan s = interior ? tree_scan(vc, nv) : fold_scan(vc, nv);
        EmitRed emit{w};
        rules<false>(d, w, s, nv, fc, c, emit);
    }
}

// K1 sparse sweep over the dirty-centre list (grid-stride; count read on device).
// `sorted`: the list was compacted from actbits (ascending ids, bits already
// cleared), so neighbouring threads gather neighbouring cache lines.
__device__ __forceinline__ void sweep_sparse_range(const Dom& d, const double* __restrict__ g, const Work& w,
                                                   int cur, bool sorted, unsigned long long i,
                                                   unsigned long long stride) {
    const unsigned long long n = min(__ldcg(&w.ctr->nact[cur]), w.act_cap);
    const uint32_t* list = w.act[cur];
    for (; i < n; i += stride) {
        const int64_t c = __ldcg(list + i);
        if (!sorted) atomicAnd(w.actbits + (c >> 5), ~(1u << (c & 31)));
        int64_t x, y, z;
        coords(d, c, x, y, z);
        double nv[14];
        load_ring(d, g, c, x, y, z, nv, [](const double* q) { return __ldcg(q); });
        const Scan s = fold_scan(__ldcg(g + c), nv);
        const uint8_t fc = w.code[c];
        const uint32_t bit = 1u << (c & 31);
        if (code_mismatch(d, scan_code(s), fc)) {
            atomicOr(w.detbits + (c >> 5), bit);
            atomicAdd(&w.ctr->ndetect, 1ull);
            EmitList emit{w, {}, 0};
            rules<false>(d, w, s, nv, fc, c, emit);
            emit.flush();
        } else if (__ldcg(w.detbits + (c >> 5)) & bit) {
            atomicAnd(w.detbits + (c >> 5), ~bit);
        }
    }
}

// Detection + rules over an ascending centre list (a masked iteration's
// compacted dirty set): one thread per centre, __ldg gathers, proposals by RED
// into prop / touched (the apply compacts touched afterwards), detection bits
// set or cleared.  The simple form of k_gather (gather.cuh).
__global__ void __launch_bounds__(256) k_sweep_list(Dom d, const double* __restrict__ g, Work w,
                                                    const uint32_t* __restrict__ list,
                                                    const unsigned long long* __restrict__ count) {
    pdl_wait();   // (programmatic dependent launch)
    const unsigned long long n = *count;
    unsigned ndet = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int64_t c = list[i];
        int64_t x, y, z;
        coords(d, c, x, y, z);
        if (!(x >= d.lo[0] && x < d.hi[0] && y >= d.lo[1] && y < d.hi[1] && z >= d.lo[2] && z < d.hi[2])) continue;
        const uint8_t fc = w.code[c];
        if (fc == kRobust) continue;
        double nv[14];
        load_ring(d, g, c, x, y, z, nv, [](const double* q) { return __ldg(q); });
        const Scan s = fold_scan(__ldg(g + c), nv);
        const uint32_t bit = 1u << (c & 31);
        if (code_mismatch(d, scan_code(s), fc)) {
            ++ndet;
            atomicOr(w.detbits + (c >> 5), bit);
            EmitRed emit{w};
            rules<false>(d, w, s, nv, fc, c, emit);
        } else if (__ldg(w.detbits + (c >> 5)) & bit) {
            atomicAnd(w.detbits + (c >> 5), ~bit);
        }
    }
    const unsigned t = __reduce_add_sync(0xffffffffu, ndet);
    if (t && (threadIdx.x & 31) == 0) atomicAdd(&w.ctr->ndetect, (unsigned long long)t);
}

__global__ void __launch_bounds__(256) k_sweep_sparse(Dom d, const double* __restrict__ g, Work w, int cur,
                                                     int sorted) {
    pdl_wait();   // (programmatic dependent launch)
    sweep_sparse_range(d, g, w, cur, sorted != 0, (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x,
                       (unsigned long long)gridDim.x * blockDim.x);
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
        if (w.frag && !(__ldg(w.frag + (u >> 5)) & bit)) continue;   // robust: never evaluated
        if (__ldcg(w.actbits + (u >> 5)) & bit) continue;
        const uint32_t old = atomicOr(w.actbits + (u >> 5), bit);
        if (old & bit) continue;
        const unsigned long long slot = agg_append(&w.ctr->nact[nxt]);
        if (slot < w.act_cap) w.act[nxt][slot] = (uint32_t)u;
    }
}

struct ApplyAcc {
    unsigned long long edits = 0;
    unsigned int maxc = 0;
    bool shared = false;
};

// Apply the merged proposal at t (correction.py:239) and do the bookkeeping.
// Dirty marking of the next incremental sweep: none, explicit 1-ring lists
// (small edit sets -> sparse sweep), or the per-iteration edit bitmap that the
// dilation kernel turns into the mask of a masked tiled sweep (large sets).
enum { kMarkNone = 0, kMarkList = 1, kMarkBits = 2 };

// Operands of one target, loaded before any of them is used so a thread keeps
// several scattered targets in flight.
struct TargetOps {
    unsigned long long key;
    double gt, fv;
    unsigned int cnt;
};
template <typename FT>
__device__ __forceinline__ TargetOps load_target_nokey(const FT* __restrict__ f, const double* __restrict__ g,
                                                       const Work& w, int64_t t) {
    unsigned int cnt = 0;
    if (!w.first_apply) {
        const uint32_t ew = __ldcg(w.editbits + (t >> 5));
        const unsigned int extra = w.counts32 ? __ldcg((const unsigned int*)w.counts + t)
                                              : (unsigned int)__ldcg((const uint16_t*)w.counts + t);
        cnt = ((ew >> (t & 31)) & 1u) ? extra + 1u : 0u;
    }
    return TargetOps{kNoProposal, __ldcg(g + t), (double)f[t], cnt};
}

template <typename FT>
__device__ __forceinline__ TargetOps load_target(const FT* __restrict__ f, const double* __restrict__ g,
                                                 const Work& w, int64_t t) {
    TargetOps op = load_target_nokey(f, g, w, t);
    op.key = __ldcg(w.prop + t);
    return op;
}

template <typename FT>
__device__ __forceinline__ void apply_target(const Dom& d, const FT* __restrict__ f, double* __restrict__ g,
                                             const Work& w, int64_t t, int mark, int nxt, ApplyAcc& acc,
                                             const TargetOps& op) {
    const double p = okey_inv(op.key);
    w.prop[t] = kNoProposal;
    const double gt = op.gt;
    const double lower = op.fv - d.lxi;                  // BoundsField.lower (correction.py:122)
    const double m = (p < gt) ? p : gt;                  // np.minimum(g, prop)
    const double nv = (m < lower) ? lower : m;           // np.maximum(., lower)
    if (nv != gt) {
        g[t] = nv;
        ++acc.edits;
        const unsigned int cnt = op.cnt + 1u;
        if (op.cnt) {   // a re-edit: store the extra count (cnt - 1 <= iterations <= 65535 for u16)
            if (w.counts32) ((unsigned int*)w.counts)[t] = cnt - 1u;
            else ((uint16_t*)w.counts)[t] = (uint16_t)(cnt - 1u);
        }
        acc.maxc = max(acc.maxc, cnt);
        atomicOr(w.editbits + (t >> 5), 1u << (t & 31));
        if (w.edited_mask) w.edited_mask[t] = 1;
        int64_t x, y, z;
        coords(d, t, x, y, z);
        acc.shared |= in_shared(d, x, y, z);
        // list mode: the 1-rings are marked by k_mark_list, one thread per member
        if (mark == kMarkList) w.elist[agg_append(&w.ctr->nelist)] = (uint32_t)t;
        else if (mark == kMarkBits) atomicOr(w.iteredit + (t >> 5), 1u << (t & 31));
    }
}

// The marking mode follows from the number of targets (an upper bound of the
// edits): 15 ring entries per edit must fit the list budget.
__device__ __forceinline__ int apply_marks(const Work& w) {
    if (!w.incremental) return kMarkNone;
    const int mode = (__ldcg(&w.ctr->nwork) * 15ull <= w.mark_limit) ? kMarkList : kMarkBits;
    if (blockIdx.x == 0 && threadIdx.x == 0) w.ctr->scratch[3] = (unsigned long long)mode;
    return mode;
}

__device__ __forceinline__ void flush_acc(const Work& w, const ApplyAcc& a) {
    const unsigned long long we = __reduce_add_sync(0xffffffffu, (unsigned)a.edits);
    const unsigned int wm = __reduce_max_sync(0xffffffffu, a.maxc);
    const unsigned int ws = __reduce_or_sync(0xffffffffu, a.shared ? 1u : 0u);
    if ((threadIdx.x & 31) == 0) {
        if (we) atomicAdd(&w.ctr->nedits, we);
        if (wm) atomicMax(&w.ctr->maxcount, (unsigned long long)wm);
        if (ws) atomicOr(&w.ctr->shared_dirty, 1ull);
    }
}

// K2 over the target list (compacted from the touched bitmap after a tiled
// sweep, or appended by first touch in a sparse sweep).
// kB: targets in flight per thread (more memory parallelism, more registers).
template <int kB, typename FT>
__device__ __forceinline__ void apply_range(const Dom& d, const FT* __restrict__ f, double* __restrict__ g,
                                            const Work& w, int nxt, int mark, unsigned long long i0,
                                            unsigned long long stride) {
    const unsigned long long n = __ldcg(&w.ctr->nwork);
    ApplyAcc acc;
    for (; i0 < n; i0 += kB * stride) {
        int64_t t[kB];
        bool ok[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            ok[k] = i0 + k * stride < n;
            t[k] = ok[k] ? (int64_t)__ldcg(w.work + i0 + k * stride) : 0;
        }
        if (w.track) {
            // sparse lists may repeat a target: the thread that clears its
            // touched bit owns it (compacted lists have their bits cleared)
#pragma unroll
            for (int k = 0; k < kB; ++k) {
                const uint32_t bit = 1u << (t[k] & 31);
                if (ok[k]) ok[k] = (atomicAnd(w.touched + (t[k] >> 5), ~bit) & bit) != 0;
            }
        }
        TargetOps ops[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k)
            if (ok[k]) ops[k] = load_target(f, g, w, t[k]);
#pragma unroll
        for (int k = 0; k < kB; ++k)
            if (ok[k]) apply_target(d, f, g, w, t[k], mark, nxt, acc, ops[k]);
    }
    flush_acc(w, acc);
}

template <typename FT>
__global__ void __launch_bounds__(256) k_apply_list(Dom d, const FT* __restrict__ f, double* __restrict__ g,
                                                    Work w, int nxt) {
    pdl_wait();   // (programmatic dependent launch)
    const int mark = apply_marks(w);
    apply_range<8>(d, f, g, w, nxt, mark, (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x,
                (unsigned long long)gridDim.x * blockDim.x);
}

// 1-ring marking of the edits of a list-mode iteration: thread i marks ring
// member (i % 15) of edit (i / 15).  The dirty set always goes to actbits; it
// is appended to the list act[nxt] only when short (`append`) -- a long list
// is compacted from actbits in ascending order before its sweep anyway, and
// appending millions of entries through one counter serialises on it.
__device__ __forceinline__ bool mark_appends(const Work& w, unsigned long long list_limit) {
    return __ldcg(&w.ctr->nelist) * 15ull <= list_limit;
}

__device__ __forceinline__ void mark_list_range(const Dom& d, const Work& w, int nxt, bool append,
                                                unsigned long long i, unsigned long long stride) {
    const unsigned long long n = __ldcg(&w.ctr->nelist) * 15ull;
    for (; i < n; i += stride) {
        const int64_t v = __ldcg(w.elist + i / 15);
        const int r = (int)(i % 15) - 1;
        int64_t x, y, z;
        coords(d, v, x, y, z);
        const int64_t px = x + (r < 0 ? 0 : rank_dx(r));
        const int64_t py = y + (r < 0 ? 0 : rank_dy(r));
        const int64_t pz = z + (r < 0 ? 0 : rank_dz(r));
        if (!in_core(d, px, py, pz)) continue;
        const int64_t u = px + py * d.sy + pz * d.sz;
        const uint32_t bit = 1u << (u & 31);
        if (w.frag && !(__ldg(w.frag + (u >> 5)) & bit)) continue;   // robust: never evaluated
        if (!append) {
            atomicOr(w.actbits + (u >> 5), bit);
            continue;
        }
        if (atomicOr(w.actbits + (u >> 5), bit) & bit) continue;
        const unsigned long long slot = agg_append(&w.ctr->nact[nxt]);
        if (slot < w.act_cap) w.act[nxt][slot] = (uint32_t)u;
    }
}

__global__ void __launch_bounds__(256) k_mark_list(Dom d, Work w, int nxt, unsigned long long list_limit) {
    pdl_wait();   // (programmatic dependent launch)
    mark_list_range(d, w, nxt, mark_appends(w, list_limit), (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x,
                    (unsigned long long)gridDim.x * blockDim.x);
}

}  // namespace pmsz
