// tiles.cuh -- z-marching tiled full-domain scans (K0 prepare, K1 detect, K4 verify).
//
// A CTA owns a 32 x 16 column of the core box and marches a chunk of z
// planes.  Each plane of the tile plus its one-voxel halo (34 x 18 cells) is
// staged once into an 8-slot shared-memory ring with cp.async, 5 planes ahead
// of the compute, so every value is read from HBM once per CTA (halo re-reads
// of neighbouring CTAs hit L2).
//
// Shared partial extrema (the 14-neighbour fold without redundant work).
// In rank order (ascending id, common.cuh) the neighbours of c = (x,y,z) fall
// into six contiguous groups:
//   ranks 0-3   the 2x2 box of plane z-1 at corner (x-1, y-1)        "D"
//   ranks 4-5   the x-pair (x-1, y-1)-(x, y-1) of plane z              H
//   rank  6, 7  (x-1, y) and (x+1, y) of plane z
//   ranks 8-9   the x-pair (x, y+1)-(x+1, y+1) of plane z              H
//   ranks 10-13 the 2x2 box of plane z+1 at corner (x, y)              "U"
// A box of plane p is the U group of centre (x, y, p-1) and the D group of
// centre (x+1, y+1, p+1); x-pairs feed the boxes and the in-plane groups.  A
// thread owns the two centres (x, y) and (x, y+1), so it evaluates six x-pairs
// and four boxes per plane and folds every group once: 20 (value, rank)
// compare-selects per centre instead of 26, and 5 shared loads instead of 14.
// Each plane is read exactly once (when it is "plane z+1" of the centres being
// finalised); the D groups and in-plane partial folds are carried in registers.
//
// Missing neighbours (outside the domain) are +-inf leaves in CTAs whose halo
// leaves the domain (a uniform per-CTA flag), and whole missing planes are
// skipped by uniform branches, so interior CTAs carry no padding logic.
//
// The per-centre global operands (f-code, fhat, dirty bit) are prefetched two
// planes ahead.  Centres whose g-code differs from the f-code are appended to
// a compact list (warp-aggregated) and their rules run in k_defer, one thread
// per centre, instead of diverging inside the sweep.
#pragma once
#include "sweep.cuh"

namespace pmsz {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T>
__device__ __forceinline__ void cp_async_t(T* dst, const T* src) {
    if (sizeof(T) == 8) cp_async8(dst, src); else cp_async4(dst, src);
}

constexpr int kTX = 32, kTY = 8, kThreads = kTX * kTY;   // threads
constexpr int kRows = 2 * kTY;                            // tile rows (2 centres / thread)
constexpr int kPX = kTX + 2, kPY = kRows + 2, kPlane = kPX * kPY;   // 34 x 18 = 612 cells
constexpr int kCopies = (kPlane + kThreads - 1) / kThreads;        // 3 copy slots / thread
constexpr int kAhead = 5;
constexpr int kSlots = 8;
static_assert(kAhead + 2 <= kSlots && (kSlots & (kSlots - 1)) == 0, "ring");

// The folds run in the type of the staged field: f32 originals are folded in
// f32 (the f32 -> f64 promotion is exact and monotone, so ranks and
// extremum flags are identical) -- no conversions, single-register selects.
template <typename V> __device__ __forceinline__ V vinf();
template <> __device__ __forceinline__ double vinf<double>() { return __longlong_as_double(0x7ff0000000000000ll); }
template <> __device__ __forceinline__ float vinf<float>() { return __int_as_float(0x7f800000); }

// A leaf value as seen by the max fold (-inf if missing) and the min fold (+inf).
template <typename V>
struct Leaf {
    V mx, mn;
};
template <bool kEdge, typename V>
__device__ __forceinline__ Leaf<V> leaf(V v, bool miss) {
    if (!kEdge) return Leaf<V>{v, v};
    return Leaf<V>{miss ? -vinf<V>() : v, miss ? vinf<V>() : v};
}

// x-pair (left = lower id): winner bit 1 = right.
template <typename V>
struct Pair {
    V mx, mn;
    int bx, bn;
    V sx, sn;   // the loser of each side (second extrema, K0's robustness test)
};
template <typename V>
__device__ __forceinline__ Pair<V> xpair(const Leaf<V>& l, const Leaf<V>& r) {
    Pair<V> p;
    const bool tx = r.mx >= l.mx;   // ties -> larger id
    p.mx = tx ? r.mx : l.mx;
    p.bx = tx;
    const bool tn = r.mn < l.mn;    // ties -> smaller id
    p.mn = tn ? r.mn : l.mn;
    p.bn = tn;
    p.sx = min(l.mx, r.mx);
    p.sn = max(l.mn, r.mn);
    return p;
}

// 2x2 box from the x-pairs of rows r (lo) and r+1 (hi): corner 0..3 in id order.
// sx / sn: the second largest / smallest value of the group (K0's robustness
// test).
template <typename V>
struct Quad {
    V mx, mn;
    int cx, cn;
    V sx, sn;
};
template <bool kSecond, typename V>
__device__ __forceinline__ Quad<V> ybox(const Pair<V>& lo, const Pair<V>& hi) {
    Quad<V> b;
    const bool tx = hi.mx >= lo.mx;
    b.mx = tx ? hi.mx : lo.mx;
    b.cx = tx ? 2 + hi.bx : lo.bx;
    const bool tn = hi.mn < lo.mn;
    b.mn = tn ? hi.mn : lo.mn;
    b.cn = tn ? 2 + hi.bn : lo.bn;
    if (kSecond) {
        b.sx = max(min(lo.mx, hi.mx), max(lo.sx, hi.sx));
        b.sn = min(max(lo.mn, hi.mn), min(lo.sn, hi.sn));
    }
    return b;
}
template <typename V>
__device__ __forceinline__ Quad<V> missing_quad() {
    return Quad<V>{-vinf<V>(), vinf<V>(), 0, 0, -vinf<V>(), vinf<V>()};
}

// Running fold in ascending rank order (sx / sn: running second extrema).
template <typename V>
struct Acc {
    V mx, mn;
    int rx, rn;
    V sx, sn;
};
template <typename V>
__device__ __forceinline__ Acc<V> acc_from(const Quad<V>& b) { return Acc<V>{b.mx, b.mn, b.cx, b.cn, b.sx, b.sn}; }
template <bool kSecond, typename V>
__device__ __forceinline__ void acc_pair(Acc<V>& a, const Pair<V>& p, int base) {
    if (kSecond) {
        a.sx = max(max(a.sx, p.sx), min(a.mx, p.mx));
        a.sn = min(min(a.sn, p.sn), max(a.mn, p.mn));
    }
    const bool tx = p.mx >= a.mx;
    a.mx = tx ? p.mx : a.mx;
    a.rx = tx ? base + p.bx : a.rx;
    const bool tn = p.mn < a.mn;
    a.mn = tn ? p.mn : a.mn;
    a.rn = tn ? base + p.bn : a.rn;
}
template <bool kSecond, typename V>
__device__ __forceinline__ void acc_leaf(Acc<V>& a, const Leaf<V>& l, int rank) {
    if (kSecond) {
        a.sx = max(a.sx, min(a.mx, l.mx));
        a.sn = min(a.sn, max(a.mn, l.mn));
    }
    const bool tx = l.mx >= a.mx;
    a.mx = tx ? l.mx : a.mx;
    a.rx = tx ? rank : a.rx;
    const bool tn = l.mn < a.mn;
    a.mn = tn ? l.mn : a.mn;
    a.rn = tn ? rank : a.rn;
}
template <bool kSecond, typename V>
__device__ __forceinline__ void acc_quad(Acc<V>& a, const Quad<V>& b, int base) {
    if (kSecond) {
        a.sx = max(max(a.sx, b.sx), min(a.mx, b.mx));
        a.sn = min(min(a.sn, b.sn), max(a.mn, b.mn));
    }
    const bool tx = b.mx >= a.mx;
    a.mx = tx ? b.mx : a.mx;
    a.rx = tx ? base + b.cx : a.rx;
    const bool tn = b.mn < a.mn;
    a.mn = tn ? b.mn : a.mn;
    a.rn = tn ? base + b.cn : a.rn;
}
template <typename V>
__device__ __forceinline__ Scan acc_scan(const Acc<V>& a, V vc) {
    Scan s;
    s.vc = (double)vc;
    s.vmax = (double)a.mx;
    s.vmin = (double)a.mn;
    s.rmax = a.rx;
    s.rmin = a.rn;
    s.is_max = (a.mx < vc) || (a.mx == vc && a.rx <= kCenterBelow);   // topology.py:79
    s.is_min = (a.mn > vc) || (a.mn == vc && a.rn > kCenterBelow);    // topology.py:80
    return s;
}

// Robustness of a centre (K0): the largest and the smallest member of its
// closed 1-ring lead the runners-up by more than 2 xi (plus rounding slack).
// Every g of the loop satisfies L <= g <= fhat with |f - fhat| <= xi, i.e.
// f - xi <= g <= f + xi up to rounding, so such a centre's steepest ascent and
// descent (and extremum flags) are those of f in every iteration: it can never
// mismatch, its rules never fire, and no sweep needs to evaluate it.
__device__ __forceinline__ double robust_margin(double xi, double v) {
    return 2.0 * xi * (1.0 + 0x1p-40) + 0x1p-40 * fabs(v) + 0x1p-1000;
}
template <typename V>
__device__ __forceinline__ bool acc_robust(const Acc<V>& a, V vc, double xi) {
    const double mxc = (double)max(a.mx, vc), sxc = (double)max(a.sx, min(a.mx, vc));
    const double mnc = (double)min(a.mn, vc), snc = (double)min(a.sn, max(a.mn, vc));
    return (mxc - sxc > robust_margin(xi, mxc)) && (snc - mnc > robust_margin(xi, mnc));
}

__device__ __forceinline__ void count_kinds(const Dom& d, const Work& w, const Scan& s, uint8_t fcode) {
    if (fcode == kRobust) return;
    const int fr = fcode & 15, fs = fcode >> 4;
    const bool fmax = fr == kExtremum, fmin = fs == kExtremum;
    if (s.is_max && !fmax) atomicAdd(&w.ctr->kinds[0], 1ull);
    if (fmax && !s.is_max) atomicAdd(&w.ctr->kinds[1], 1ull);
    if (s.is_min && !fmin) atomicAdd(&w.ctr->kinds[2], 1ull);
    if (fmin && !s.is_min) atomicAdd(&w.ctr->kinds[3], 1ull);
    if (!d.extrema_only && !fmax && s.rmax != fr) atomicAdd(&w.ctr->kinds[4], 1ull);
    if (!d.extrema_only && !fmin && s.rmin != fs) atomicAdd(&w.ctr->kinds[5], 1ull);
}

// ---------------------------------------------------------------------------
// Ops: what happens to a finalised centre.  fetch() issues the per-centre
// global loads (two planes ahead); center() consumes them.

// K1 / K4: detection against the f-code.  kMasked: `dirty` restricts the
// centres to those whose bit is set (masked sweep of an incremental
// iteration; their detection bits were cleared by the dilation kernel).
// kExtrema: the extrema-only mismatch test.  Both are template
// parameters so the plain full sweep carries none of their logic.
template <bool kCount, bool kMasked = false, bool kExtrema = false>
struct DetectOp {
    static constexpr bool kSecond = false;
    Work w;
    const uint32_t* dirty;
    unsigned ndet;
    struct Pre {
        uint32_t code;   // f-code byte; 0x100 = not a live centre
        uint32_t word;   // dirty-bitmap word (masked sweep)
        uint32_t sh;     // bit of the centre in `word`
    };
    __device__ __forceinline__ void begin() { ndet = 0; }
    // loads issued now, consumed two planes later
    __device__ __forceinline__ Pre fetch(int64_t c, bool live) const {
        if (!live) return Pre{0x100u, 0u, 0u};
        if (!kMasked) return Pre{ld_nc_u8(w.code + c), 1u, 0u};
        return Pre{ld_nc_u8(w.code + c), ld_nc_u32(dirty + (c >> 5)), (uint32_t)(c & 31)};
    }
    // robust centres (K0) never mismatch and are never evaluated
    __device__ __forceinline__ bool wants(const Pre& p) const {
        if (!kMasked) return !(p.code & 0x100u) && p.code != kRobust;
        return !(p.code & 0x100u) && p.code != kRobust && ((p.word >> p.sh) & 1u);
    }
    __device__ __forceinline__ bool skippable() const { return kMasked; }
    __device__ __forceinline__ void center(const Dom& d, int64_t c, const Acc<double>& a, double vc, const Pre& p) {
        evaluate(d, c, acc_scan(a, vc), (uint8_t)p.code);
    }
    // the g-scan s of centre c against its f-code fc
    __device__ __forceinline__ void evaluate(const Dom& d, int64_t c, const Scan& s, uint8_t fc) {
        const uint8_t gc = scan_code(s);
        const bool mismatch = kExtrema ? (((gc & 15) == kExtremum) != ((fc & 15) == kExtremum) ||
                                          ((gc >> 4) == kExtremum) != ((fc >> 4) == kExtremum))
                                       : gc != fc;
        if (!mismatch) return;
        ++ndet;
        if (kCount) count_kinds(d, w, s, fc);
        else atomicOr(w.detbits + (c >> 5), 1u << (c & 31));   // RED; k_defer picks it up
    }
    __device__ __forceinline__ void finish() {
        if (!kCount) {
            const unsigned t = __reduce_add_sync(0xffffffffu, ndet);
            if (t && (threadIdx.x & 31) == 0) atomicAdd(&w.ctr->ndetect, (unsigned long long)t);
        }
    }
};

// K0: validate the pair (correction.py:52-60, hazard H6), build the f-code
// (field_scan(original), correction.py:404) and copy g <- fhat (:405).
struct PrepOp {
    static constexpr bool kSecond = true;   // second extrema for the robustness test
    const double* fh;
    double* g;
    uint8_t* code;
    uint32_t* frag;   // fragile bitmap (zeroed by the caller); null: robustness off
    DevCounters* ctr;
    double xi;
    unsigned bound, floorv, upper, nonfin, nfrag;
    struct Pre {
        double hv;
    };
    __device__ __forceinline__ void begin() { bound = floorv = upper = nonfin = nfrag = 0; }
    __device__ __forceinline__ Pre fetch(int64_t c, bool live) const { return Pre{live ? ld_nc_f64(fh + c) : 0.0}; }
    __device__ __forceinline__ bool wants(const Pre&) const { return true; }
    __device__ __forceinline__ bool skippable() const { return false; }
    template <typename V>
    __device__ __forceinline__ void center(const Dom&, int64_t c, const Acc<V>& a, V vc, const Pre& p) {
        const double fv = (double)vc;
        const double hv = p.hv;
        nonfin += (!isfinite(fv) || !isfinite(hv)) ? 1u : 0u;
        if (fabs(fv - hv) > xi) {
            ++bound;
            atomicMin(&ctr->bound_first, (unsigned long long)c);
        }
        floorv += hv < fv - xi ? 1u : 0u;
        upper += hv > fv + xi ? 1u : 0u;
        if (g != fh) g[c] = hv;
        const bool robust = frag != nullptr && acc_robust(a, vc, xi);
        code[c] = robust ? kRobust : scan_code(acc_scan(a, vc));
        if (frag) {
            // fragile bitmap: a full warp holds 32 consecutive ids of one row
            // (lane = x - x0), i.e. at most two words -> two RED.OR by lane 0
            nfrag += robust ? 0u : 1u;
            const unsigned lane = threadIdx.x & 31;
            if (__activemask() == 0xffffffffu) {
                const unsigned bal = __ballot_sync(0xffffffffu, !robust);
                const int64_t c0 = c - lane;
                const unsigned sh = (unsigned)(c0 & 31);
                if (lane == 0 && bal) {
                    if (bal << sh) atomicOr(frag + (c0 >> 5), bal << sh);
                    if (sh && (bal >> (32 - sh))) atomicOr(frag + (c0 >> 5) + 1, bal >> (32 - sh));
                }
            } else if (!robust) {
                atomicOr(frag + (c >> 5), 1u << (c & 31));
            }
        }
    }
    __device__ __forceinline__ void finish() {
        const unsigned b = __reduce_add_sync(0xffffffffu, bound);
        const unsigned fl = __reduce_add_sync(0xffffffffu, floorv);
        const unsigned up = __reduce_add_sync(0xffffffffu, upper);
        const unsigned nf = __reduce_add_sync(0xffffffffu, nonfin);
        const unsigned nfr = __reduce_add_sync(0xffffffffu, nfrag);
        if ((threadIdx.x & 31) == 0) {
            if (nfr) atomicAdd(&ctr->nfragile, (unsigned long long)nfr);
            if (b) atomicAdd(&ctr->bound_viol, (unsigned long long)b);
            if (fl) atomicAdd(&ctr->floor_viol, (unsigned long long)fl);
            if (up) atomicAdd(&ctr->upper_viol, (unsigned long long)up);
            if (nf) atomicAdd(&ctr->nonfinite, (unsigned long long)nf);
        }
    }
};

// ---------------------------------------------------------------------------
// Per-plane work of one thread: six x-pairs, two U boxes, two D boxes and the
// in-plane groups of its two centres.
template <typename V>
struct PlaneOut {
    Quad<V> ua, ub;           // U groups of centres (x, ya) and (x, yb) at plane p-1
    Quad<V> da, db;           // D groups of the same centres at plane p+1
    Pair<V> h1, h2, h5, h6;   // in-plane x-pairs of plane p
    Leaf<V> b, c, i, j;       // in-plane singles of plane p
    V fa, fb;                 // centre values at plane p
};

template <bool kEdge, bool kSecond, typename V>
__device__ __forceinline__ PlaneOut<V> plane_work(const V* __restrict__ s, int cell, bool mxl, bool mxr, bool myl,
                                                  bool myb, bool my2) {
    // column x-1: rows ya-1, ya, yb; column x: ya-1..ya+2; column x+1: ya..ya+2
    const Leaf<V> a = leaf<kEdge>(s[cell - kPX - 1], mxl || myl);
    const Leaf<V> b = leaf<kEdge>(s[cell - 1], mxl);
    const Leaf<V> c = leaf<kEdge>(s[cell + kPX - 1], mxl || myb);
    const Leaf<V> e = leaf<kEdge>(s[cell - kPX], myl);
    const V fv = s[cell];
    const V gv = s[cell + kPX];
    const Leaf<V> f{fv, fv};
    const Leaf<V> g = leaf<kEdge>(gv, myb);
    const Leaf<V> h = leaf<kEdge>(s[cell + 2 * kPX], my2);
    const Leaf<V> i = leaf<kEdge>(s[cell + 1], mxr);
    const Leaf<V> j = leaf<kEdge>(s[cell + kPX + 1], mxr || myb);
    const Leaf<V> k = leaf<kEdge>(s[cell + 2 * kPX + 1], mxr || my2);
    PlaneOut<V> o;
    o.h1 = xpair(a, e);   // (x-1, ya-1)
    o.h2 = xpair(b, f);   // (x-1, ya)
    const Pair<V> h3 = xpair(c, g);   // (x-1, yb)
    const Pair<V> h4 = xpair(f, i);   // (x, ya)
    o.h5 = xpair(g, j);   // (x, yb)
    o.h6 = xpair(h, k);   // (x, ya+2)
    o.ua = ybox<kSecond>(h4, o.h5);
    o.ub = ybox<kSecond>(o.h5, o.h6);
    o.da = ybox<kSecond>(o.h1, o.h2);
    o.db = ybox<kSecond>(o.h2, h3);
    o.b = b; o.c = c; o.i = i; o.j = j;
    o.fa = fv;
    o.fb = gv;
    return o;
}

// Partial fold of the groups of ranks 0..9 (D, in-plane).
template <bool kSecond, typename V>
__device__ __forceinline__ Acc<V> partial_a(const Quad<V>& d, const PlaneOut<V>& o) {
    Acc<V> a = acc_from(d);
    acc_pair<kSecond>(a, o.h1, 4);
    acc_leaf<kSecond>(a, o.b, 6);
    acc_leaf<kSecond>(a, o.i, 7);
    acc_pair<kSecond>(a, o.h5, 8);
    return a;
}
template <bool kSecond, typename V>
__device__ __forceinline__ Acc<V> partial_b(const Quad<V>& d, const PlaneOut<V>& o) {
    Acc<V> a = acc_from(d);
    acc_pair<kSecond>(a, o.h2, 4);
    acc_leaf<kSecond>(a, o.c, 6);
    acc_leaf<kSecond>(a, o.j, 7);
    acc_pair<kSecond>(a, o.h6, 8);
    return a;
}

// Copy-slot bookkeeping of one CTA: each thread owns up to kCopies cells of the
// 34 x 18 staged plane; their source offsets are fixed along z.
// Halo cells outside the domain are never staged (leaves flag them missing).
// The source pointers advance by one plane per call; the destination is the
// shared byte address of the thread's cell in slot 0 plus slot * plane size.
template <typename T>
struct Stager {
    const T* p[kCopies];
    unsigned valid;    // bit q: cell q exists and lies in the domain
    unsigned dst0;     // shared address of cell `tid` in slot 0
    int64_t sz;
    __device__ __forceinline__ void init(const Dom& d, const T* src, T* sm0, int64_t x0, int64_t y0, int64_t z,
                                         int tid) {
        sz = d.sz;
        valid = 0;
        dst0 = (unsigned)__cvta_generic_to_shared(sm0 + tid);
#pragma unroll
        for (int q = 0; q < kCopies; ++q) {
            const int e = tid + q * kThreads;
            p[q] = src;
            if (e < kPlane) {
                const int py = e / kPX, px = e - py * kPX;
                const int64_t gx = x0 - 1 + px, gy = y0 - 1 + py;
                if (gx >= 0 && gx < d.nx && gy >= 0 && gy < d.ny) {
                    p[q] = src + gx + gy * d.sy + z * d.sz;
                    valid |= 1u << q;
                }
            }
        }
    }
    // stage the current plane into `slot` (if `on`) and advance to the next plane
    __device__ __forceinline__ void stage(int slot, bool on) {
        const unsigned dst = dst0 + (unsigned)(slot * kPlane * (int)sizeof(T));
#pragma unroll
        for (int q = 0; q < kCopies; ++q) {
            if (on && ((valid >> q) & 1u)) {
                const unsigned a = dst + (unsigned)(q * kThreads * (int)sizeof(T));
                if (sizeof(T) == 8)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(p[q]));
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(a), "l"(p[q]));
            }
            p[q] += sz;
        }
    }
};

template <bool kEdge, typename T, class Op>
__device__ __forceinline__ void tiled_body(const Dom& d, T (*sm)[kPlane], Stager<T>& st, Op& op, int64_t x0,
                                           int64_t y0, int64_t zb, int64_t ze) {
    constexpr bool kSecond = Op::kSecond;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t x = x0 + tx, ya = y0 + 2 * ty, yb = ya + 1;
    const int cell = (2 * ty + 1) * kPX + (tx + 1);
    // domain-edge flags of this thread's halo (only used when kEdge)
    const bool mxl = x - 1 < 0, mxr = x + 1 >= d.nx, myl = ya - 1 < 0, myb = yb >= d.ny, my2 = ya + 2 >= d.ny;
    // interior CTAs (kEdge == false) have every centre inside the core box
    const bool live_a = !kEdge || (x < d.hi[0] && ya < d.hi[1]);
    const bool live_b = !kEdge || (x < d.hi[0] && yb < d.hi[1]);
    const int64_t sz = d.sz, sy = d.sy;
    int64_t ca = x + ya * sy + zb * sz;   // centre A of the current plane; centre B = A + sy

    // per-centre operands, two planes ahead
    typename Op::Pre pa0 = op.fetch(ca, live_a);
    typename Op::Pre pb0 = op.fetch(ca + sy, live_b);
    typename Op::Pre pa1 = op.fetch(ca + sz, live_a && zb + 1 < ze);
    typename Op::Pre pb1 = op.fetch(ca + sy + sz, live_b && zb + 1 < ze);

    // prologue: plane zb-1 (D groups), plane zb (partial folds)
    cp_async_wait<kAhead>();
    __syncthreads();
    Quad<T> da, db;
    if (zb - 1 >= 0) {
        const PlaneOut<T> o = plane_work<kEdge, kSecond>(sm[0], cell, mxl, mxr, myl, myb, my2);
        da = o.da;
        db = o.db;
    } else {
        da = db = missing_quad<T>();
    }
    Acc<T> pa, pb;
    T fa, fb;
    {
        const PlaneOut<T> o = plane_work<kEdge, kSecond>(sm[1], cell, mxl, mxr, myl, myb, my2);
        pa = partial_a<kSecond>(da, o);
        pb = partial_b<kSecond>(db, o);
        da = o.da;
        db = o.db;
        fa = o.fa;
        fb = o.fb;
    }
    // planes up to zstop are staged (plane ze is the last one read)
    const int64_t zstop = min(ze, d.nz - 1);
    int k = 0;
    // one plane step; kUp: plane z+1 lies in the domain (false only for z = nz-1)
    auto step = [&](auto up_tag, int64_t z) {
        constexpr bool kUp = decltype(up_tag)::value;
        cp_async_wait<kAhead - 1>();   // plane z+1 has landed
        __syncthreads();               // ... for every thread; iteration z-1 is done
        // refill: plane z+1+kAhead replaces plane z+1+kAhead-kSlots (long consumed)
        st.stage((k + 2 + kAhead) & (kSlots - 1), z + 1 + kAhead <= zstop);
        cp_async_commit();
        const typename Op::Pre pa2 = op.fetch(ca + 2 * sz, live_a && z + 2 < ze);
        const typename Op::Pre pb2 = op.fetch(ca + sy + 2 * sz, live_b && z + 2 < ze);
        // masked sweep: a warp whose centres at planes z, z+1, z+2 are all clean
        // skips the plane; the state it leaves stale (partial folds for z+1, D
        // groups for z+2, centre values) is only ever read for those clean centres
        bool work = true;
        if (op.skippable())
            work = __any_sync(0xffffffffu, op.wants(pa0) || op.wants(pb0) || op.wants(pa1) || op.wants(pb1) ||
                                               op.wants(pa2) || op.wants(pb2));
        PlaneOut<T> o;
        if (kUp && work) o = plane_work<kEdge, kSecond>(sm[(k + 2) & (kSlots - 1)], cell, mxl, mxr, myl, myb, my2);
        if (work && live_a && op.wants(pa0)) {
            Acc<T> a = pa;
            if (kUp) acc_quad<kSecond>(a, o.ua, 10);
            op.center(d, ca, a, fa, pa0);
        }
        if (work && live_b && op.wants(pb0)) {
            Acc<T> a = pb;
            if (kUp) acc_quad<kSecond>(a, o.ub, 10);
            op.center(d, ca + sy, a, fb, pb0);
        }
        if (kUp && work) {
            pa = partial_a<kSecond>(da, o);
            pb = partial_b<kSecond>(db, o);
            da = o.da;
            db = o.db;
            fa = o.fa;
            fb = o.fb;
        }
        pa0 = pa1; pb0 = pb1;
        pa1 = pa2; pb1 = pb2;
        ca += sz;
        ++k;
    };
    const int64_t zmain = min(ze, d.nz - 1);   // centres with plane z+1 in the domain
    for (int64_t z = zb; z < zmain; ++z) step(std::true_type{}, z);
    if (zmain < ze) step(std::false_type{}, zmain);   // the last plane of the domain
}

template <typename T, class Op>
__global__ void __launch_bounds__(kThreads, 2) k_tiled(Dom d, const T* __restrict__ src, Op op, int zchunk) {
    __shared__ __align__(16) T sm[kSlots][kPlane];
    const int tid = threadIdx.y * kTX + threadIdx.x;
    const int64_t x0 = d.lo[0] + (int64_t)blockIdx.x * kTX;
    const int64_t y0 = d.lo[1] + (int64_t)blockIdx.y * kRows;
    const int64_t zb = d.lo[2] + (int64_t)blockIdx.z * zchunk;
    const int64_t ze = min(zb + (int64_t)zchunk, d.hi[2]);
    Stager<T> st;
    st.init(d, src, &sm[0][0], x0, y0, zb - 1, tid);
    op.begin();
    // plane z' lives in slot (z' - zb + 1) & (kSlots - 1); the stager walks
    // the planes zb-1, zb, zb+1, ... in order
    const int64_t zstop = min(ze, d.nz - 1);
    st.stage(0, zb - 1 >= 0);
    st.stage(1, true);
    cp_async_commit();
#pragma unroll
    for (int j = 1; j <= kAhead; ++j) {
        st.stage(j + 1, zb + j <= zstop);
        cp_async_commit();
    }
    // halo leaves the domain, or the tile leaves the core box?  (uniform per CTA)
    const bool edge = x0 == 0 || x0 + kTX >= d.nx || y0 == 0 || y0 + kRows >= d.ny || x0 + kTX > d.hi[0] ||
                      y0 + kRows > d.hi[1];
    if (edge)
        tiled_body<true>(d, sm, st, op, x0, y0, zb, ze);
    else
        tiled_body<false>(d, sm, st, op, x0, y0, zb, ze);
    cp_async_wait<0>();
    op.finish();
}

inline void tiled_grid(const Dom& d, dim3& grid, int& zchunk) {
    const int64_t cx = d.hi[0] - d.lo[0], cy = d.hi[1] - d.lo[1], cz = d.hi[2] - d.lo[2];
    const int64_t tiles = ((cx + kTX - 1) / kTX) * ((cy + kRows - 1) / kRows);
    // z chunks of ~64 planes (3% halo re-read) unless that leaves fewer than
    // ~8 waves of 148 SMs x 2 CTAs; never below 16 planes
    const int64_t want = (148 * 2 * 8 + tiles - 1) / tiles;
    int64_t chunks = std::max<int64_t>((cz + 63) / 64, std::min<int64_t>(want, cz / 16));
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, cz));
    zchunk = (int)std::max<int64_t>(1, (cz + chunks - 1) / chunks);
    chunks = (cz + zchunk - 1) / zchunk;
    grid = dim3((unsigned)((cx + kTX - 1) / kTX), (unsigned)((cy + kRows - 1) / kRows), (unsigned)chunks);
}

template <bool kCount, bool kMasked, bool kExtrema>
inline void launch_detect(const Dom& d, const double* g, const Work& w, cudaStream_t s, const uint32_t* dirty) {
    dim3 grid;
    int zchunk;
    tiled_grid(d, grid, zchunk);
    using Op = DetectOp<kCount, kMasked, kExtrema>;
    Op op{w, dirty, 0};
    k_tiled<double, Op><<<grid, dim3(kTX, kTY, 1), 0, s>>>(d, g, op, zchunk);
}

// kCount: the K4 count sweep (all six kinds, unmasked).
template <bool kCount>
inline void launch_sweep_full(const Dom& d, const double* g, const Work& w, cudaStream_t s,
                              const uint32_t* dirty = nullptr) {
    if (kCount) launch_detect<true, false, false>(d, g, w, s, nullptr);
    else if (dirty && d.extrema_only) launch_detect<false, true, true>(d, g, w, s, dirty);
    else if (dirty) launch_detect<false, true, false>(d, g, w, s, dirty);
    else if (d.extrema_only) launch_detect<false, false, true>(d, g, w, s, nullptr);
    else launch_detect<false, false, false>(d, g, w, s, nullptr);
}

template <typename FT>
inline void launch_prep(const Dom& d, const FT* f, const double* fh, double* g, uint8_t* code, uint32_t* frag,
                        DevCounters* ctr, cudaStream_t s) {
    // K0 scans the whole domain (ghost layers included): the f-code of a block's
    // ext field is scan_neighbors(f_ext, ext_dims) (parallel.py:212).
    Dom all = d;
    for (int a = 0; a < 3; ++a) all.lo[a] = 0;
    all.hi[0] = d.nx;
    all.hi[1] = d.ny;
    all.hi[2] = d.nz;
    dim3 grid;
    int zchunk;
    tiled_grid(all, grid, zchunk);
    PrepOp op{fh, g, code, frag, ctr, d.xi, 0, 0, 0, 0, 0};
    k_tiled<FT, PrepOp><<<grid, dim3(kTX, kTY, 1), 0, s>>>(all, f, op, zchunk);
}

}  // namespace pmsz
