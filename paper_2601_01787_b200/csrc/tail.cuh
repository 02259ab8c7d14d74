// tail.cuh -- the list-mode iterations of the correction loop in ONE
// persistent cooperative kernel.
//
// After the first one or two sweeps the dirty set collapses to a few thousand
// centres and every iteration is latency bound: a sparse sweep, an apply and a
// ring marking of a few microseconds each, plus a host round trip to read the
// edit count and choose the next iteration's form.  k_tail runs those
// iterations back to back on a grid that is co-resident on all 148 SMs, with
// three grid barriers per iteration instead of three launches and a host
// synchronisation:
//
//   S  sparse sweep of the dirty list act[cur]  -> proposals, target list
//   |  grid barrier
//   A  apply the merged proposals (K2)         -> edits, elist
//   |  grid barrier
//   M  1-ring marking of the edits             -> act[nxt]
//   |  grid barrier; every CTA reads the same final counters and takes the
//      same decision: stop (zero edits), hand back to the host (the edit set
//      grew past the list budget, the next dirty list is large enough to be
//      worth sorting first -- see sort_pending -- or the iteration budget is
//      spent), or go on.
//
// The arithmetic is the list-mode iteration of iterate_once unchanged (same
// device functions), so results are bit-identical whichever form runs an
// iteration.  Mutable data are read with ld.global.cg (L2) only.
//
// Counter lifetimes (each is reset in a phase where nobody can still read
// the previous value, so no extra barrier is needed):
//   nwork   written S, read A, reset M      ndetect written S, read A, reset M
//   nedits  written A, read M, reset S'     nelist  written A, read M, reset S'
//   nact[nxt] reset A, written M, read after the M barrier and in S'
#pragma once
#include <cooperative_groups.h>
#include "sweep.cuh"

namespace pmsz {

enum : unsigned long long { kTailConverged = 1, kTailBits = 2, kTailOverflow = 3, kTailBudget = 4, kTailSort = 5,
                            kTailSmall = 6 /* the dirty list fits k_tail1, which runs next on the stream */ };

struct TailState {
    unsigned long long iterations;   // iterations run by this launch
    unsigned long long exit;         // kTail*
    unsigned long long cur;          // dirty list the next iteration would sweep
    unsigned long long pending;      // its length
    unsigned long long last_edits;
    unsigned long long last_detect;
    unsigned long long shared_or;    // shared_dirty of any iteration
    unsigned long long detections;   // sum over iterations
    unsigned long long appended;     // the pending dirty set is listed (else: actbits only, `pending` a bound)
};

// In-tail rebuild of a long dirty list: the ascending compaction of actbits
// into `list` (bits cleared).  Every WARP of the grid owns one contiguous
// sub-chunk of words, so the walk needs only warp scans; the per-warp counts
// stay in shared memory across the grid barrier that separates counting from
// writing, the per-CTA totals go through `counts`.  Every CTA then knows the
// total and takes the same decision.
constexpr int kTailWarps = 8;

__device__ __forceinline__ int64_t tail_warp_chunk(int64_t nwords) {
    const int64_t nw = (int64_t)gridDim.x * kTailWarps;
    return ((nwords + nw - 1) / nw + 31) / 32 * 32;
}

__device__ __forceinline__ unsigned long long tail_chunk_count(const uint32_t* bits, int64_t nwords,
                                                               unsigned long long* counts, unsigned* warp_cnt) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t chunk = tail_warp_chunk(nwords);
    const int64_t w0 = ((int64_t)blockIdx.x * kTailWarps + wid) * chunk, w1 = min(w0 + chunk, nwords);
    unsigned t = 0;
    for (int64_t base = w0; base < w1; base += 8 * 32) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {   // 8 independent loads in flight
            const int64_t q = base + k * 32 + lane;
            v[k] = q < w1 ? __ldcg(bits + q) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) t += __popc(v[k]);
    }
    t = __reduce_add_sync(0xffffffffu, t);
    if (lane == 0) warp_cnt[wid] = t;
    __syncthreads();
    unsigned long long s = 0;
    for (int q = 0; q < kTailWarps; ++q) s += warp_cnt[q];
    if (threadIdx.x == 0) counts[blockIdx.x] = s;
    return s;
}

__device__ __forceinline__ void tail_chunk_write(uint32_t* bits, int64_t nwords, unsigned long long cta_pos,
                                                 const unsigned* warp_cnt, uint32_t* list) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t chunk = tail_warp_chunk(nwords);
    const int64_t w0 = ((int64_t)blockIdx.x * kTailWarps + wid) * chunk, w1 = min(w0 + chunk, nwords);
    unsigned long long pos0 = cta_pos;
    for (int q = 0; q < wid; ++q) pos0 += warp_cnt[q];
    for (int64_t base = w0; base < w1; base += 8 * 32) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t q = base + k * 32 + lane;
            v[k] = q < w1 ? __ldcg(bits + q) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t q = base + k * 32 + lane;
            uint32_t m = v[k];
            if (m) bits[q] = 0u;
            const unsigned c = __popc(m);
            unsigned sc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, sc, o);
                if (lane >= o) sc += y;
            }
            unsigned long long pos = pos0 + sc - c;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                list[pos++] = (uint32_t)(q * 32 + b);
            }
            pos0 += __shfl_sync(0xffffffffu, sc, 31);
        }
    }
}

template <typename FT>
__global__ void __launch_bounds__(256) k_tail(Dom d, const FT* __restrict__ f, double* g, Work w, int cur,
                                              int sorted, unsigned long long sort_min, unsigned long long dense_min,
                                              unsigned long long* __restrict__ chunk_counts, long long budget,
                                              unsigned long long* __restrict__ hist, TailState* ts,
                                              unsigned long long* __restrict__ trace, unsigned long long small_max) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned warp_cnt[kTailWarps];
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const bool leader = tid == 0;
    DevCounters* c = w.ctr;
    w.track = 1;
    unsigned long long shared_or = 0, detections = 0;
    for (long long it = 0;; ++it) {
        const int nxt = cur ^ 1;
        // ---- S ---------------------------------------------------------------
        if (trace && leader && it == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[8190] = t;
        }
        if (leader && it > 0) {
            c->nedits = 0;
            c->nelist = 0;
            c->shared_dirty = 0;
        }
        sweep_sparse_range(d, g, w, cur, sorted != 0, tid, stride);
        grid.sync();
        if (trace && leader && it < 4) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[8000 + 2 * it] = t;
        }
        // ---- A ---------------------------------------------------------------
        const unsigned long long ndet = __ldcg(&c->ndetect);
        if (leader) c->nact[nxt] = 0;
        const int mark = apply_marks(w);
        apply_range<4>(d, f, g, w, nxt, mark, tid, stride);
        grid.sync();
        if (trace && leader && it < 4) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[8001 + 2 * it] = t;
        }
        // ---- M ---------------------------------------------------------------
        const unsigned long long nedits = __ldcg(&c->nedits);
        shared_or |= __ldcg(&c->shared_dirty);
        detections += ndet;
        if (leader) {
            hist[it] = nedits;
            c->nwork = 0;
            c->ndetect = 0;
        }
        const unsigned long long nel = __ldcg(&c->nelist);
        const bool append = nel * 15ull <= sort_min;
        if (mark == kMarkList) mark_list_range(d, w, nxt, append, tid, stride);
        grid.sync();
        // ---- decide ------------------------------------------------------------
        const unsigned long long nact = __ldcg(&c->nact[nxt]);
        if (trace && leader) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[2 * it] = t;
            trace[2 * it + 1] = nact;
        }
        unsigned long long exit = 0, pending = append ? nact : nel * 15ull;   // a bound when only actbits was marked
        bool listed = append;
        if (nedits == 0) exit = kTailConverged;
        else if (mark != kMarkList) exit = kTailBits;
        else if (nact > w.act_cap) exit = kTailOverflow;
        else if (it + 1 >= budget) exit = kTailBudget;
        else if (append && nact <= small_max) exit = kTailSmall;   // k_tail1 takes over on the device
        else if (!append || nact > sort_min) {
            // a long dirty set: rebuild the list sorted from actbits here, or
            // hand it to the host's gather path when it is longer still
            tail_chunk_count(w.actbits, w.nwords, chunk_counts, warp_cnt);
            grid.sync();
            unsigned long long total = 0, before = 0;
            for (unsigned q = 0; q < gridDim.x; ++q) {
                const unsigned long long v = __ldcg(chunk_counts + q);
                total += v;
                before += q < blockIdx.x ? v : 0ull;
            }
            if (total > dense_min) {
                exit = kTailSort;   // the set stays in actbits (exact count in `pending`)
                pending = total;
                listed = false;
            } else {
                tail_chunk_write(w.actbits, w.nwords, before, warp_cnt, w.act[nxt]);
                if (leader) c->nact[nxt] = total;
                grid.sync();
                sorted = 1;
            }
        } else {
            sorted = 0;
        }
        if (exit) {
            if (leader) {
                ts->iterations = (unsigned long long)(it + 1);
                ts->exit = exit;
                ts->cur = (unsigned long long)nxt;
                ts->pending = pending;
                ts->last_edits = nedits;
                ts->last_detect = ndet;
                ts->shared_or = shared_or;
                ts->detections = detections;
                ts->appended = listed ? 1ull : 0ull;
                c->ndetect = ndet;   // the host reads the last iteration's counters
            }
            return;
        }
        cur = nxt;
    }
}

}  // namespace pmsz

namespace pmsz {

// ---------------------------------------------------------------------------
// k_tail1: the small-dirty-set iterations in ONE CTA.
//
// Late in the loop an iteration sweeps a few hundred centres and applies a
// few dozen edits; the grid-wide tail above then pays its three grid
// barriers and ~20 dependent L2 round trips per iteration (~15 us at 512^3).
// Here one 1024-thread CTA keeps the dirty set, the proposal targets and the
// iteration's edits in shared memory, and an iteration is two phases with
// one L2 round trip each (plus the wait for the proposals' reductions):
//
//   S  ring gather + detection + rules of every dirty centre; proposals go to
//      prop[] by RED.MIN as everywhere else, the target ids into a shared
//      hash set (first insert wins, no global work list)
//   A  per target: the apply operands AND the fragile bits of its closed
//      1-ring are loaded together; the apply (K2 arithmetic), and for an edit
//      the ring's core, fragile members go straight into a second shared
//      hash set -> the next dirty list (the M phase of k_tail, fused)
//
// Same device functions as the list-mode iteration (load_ring, fold_scan,
// rules, the apply arithmetic of apply_target), so results are bit-identical.
// The entry list's actbits are cleared on entry; on a hand-back the pending
// list is written to act[cur ^ 1] with its actbits set, exactly the state a
// list-mode iteration leaves.  Overflow of any shared structure falls back to
// the global structures (work list + touched bits for targets, mark_ring for
// the next dirty set) and hands back to the host.
constexpr int kT1Threads = 1024;
constexpr int kT1Dirty = 4096;      // dirty-list capacity (ping-pong)
// (shared memory: 32 KB dirty lists + 64 KB keys + 3 x 32 KB sets = 192 KB of the 227 KB)
constexpr int kT1Set = 8192;        // hash sets (targets / next dirty); power of two
constexpr int kT1SetBits = 13;
constexpr uint32_t kT1Empty = 0xffffffffu;
// hand-over threshold of the grid tail: the one-CTA iteration beats the grid
// barriers below about a thousand dirty centres (PMSZ_TAIL1_MAX overrides)
constexpr int kT1Handover = 512;

struct T1Smem {
    uint32_t dirty[2][kT1Dirty];
    unsigned long long tkey[kT1Set];   // min-merged proposal key of each target slot (kNoProposal when free)
    uint32_t tset[kT1Set];
    uint32_t dset[kT1Set];
    uint32_t edits[kT1Set];
    unsigned nd[2];
    unsigned nedit, ndet, shared, maxc, ovf_tgt, ovf_edit, ovf_mark;
};
constexpr size_t kT1SmemBytes = sizeof(T1Smem);

// 1 = inserted, 0 = present, 2 = no free slot within the probe limit; *at = the slot
__device__ __forceinline__ int t1_insert(uint32_t* set, uint32_t u, uint32_t* at = nullptr) {
    const uint32_t h = (u * 2654435761u) >> (32 - kT1SetBits);
#pragma unroll 1
    for (int k = 0; k < 64; ++k) {
        const uint32_t slot = (h + (uint32_t)k) & (uint32_t)(kT1Set - 1);
        const uint32_t old = atomicCAS(set + slot, kT1Empty, u);
        if (old == kT1Empty || old == u) {
            if (at) *at = slot;
            return old == kT1Empty ? 1 : 0;
        }
    }
    return 2;
}

// Proposals are min-merged in shared memory (the target's slot key; exactly
// np.minimum.at, like the RED.MIN of the other forms); global prop is left
// untouched, so no fence is needed before the apply.  A full set falls back
// to prop + touched + the global work list (a target is either in the set
// for all its proposals or for none: slots never free during the sweep).
struct EmitT1 {
    const Work& w;
    T1Smem& S;
    bool issued = false;   // this thread issued global RED.MINs (overflow)
    __device__ __forceinline__ void operator()(int64_t t, double val) {
        uint32_t slot;
        if (t1_insert(S.tset, (uint32_t)t, &slot) != 2) {
            atomicMin(S.tkey + slot, okey(val));
            return;
        }
        atomicMin(w.prop + t, okey(val));
        issued = true;
        S.ovf_tgt = 1;
        const uint32_t bit = 1u << (t & 31);
        if (!(atomicOr(w.touched + (t >> 5), bit) & bit)) w.work[agg_append(&w.ctr->nwork)] = (uint32_t)t;
    }
};

// Apply target t (apply_target's arithmetic) and, for an edit, put the core,
// fragile members of its closed 1-ring into the next dirty set.  The fragile
// words of the ring are loaded with the apply operands (one round trip).
template <typename FT>
__device__ __forceinline__ void t1_apply_mark(const Dom& d, const FT* __restrict__ f, double* __restrict__ g,
                                              const Work& w, T1Smem& S, int b, unsigned dcap, int64_t t,
                                              ApplyAcc& acc, bool smem_key, unsigned long long key) {
    int64_t x, y, z;
    coords(d, t, x, y, z);
    uint32_t fw[15];
#pragma unroll
    for (int r = -1; r < 14; ++r) {
        const int64_t px = x + (r < 0 ? 0 : rank_dx(r)), py = y + (r < 0 ? 0 : rank_dy(r)),
                      pz = z + (r < 0 ? 0 : rank_dz(r));
        const int64_t u = px + py * d.sy + pz * d.sz;
        fw[r + 1] = !in_core(d, px, py, pz) ? 0u : (w.frag ? __ldg(w.frag + (u >> 5)) : ~0u);
    }
    TargetOps op;
    if (smem_key) {   // the proposal is in shared memory; global prop stays all-ones
        op = load_target_nokey(f, g, w, t);
        op.key = key;
    } else {
        op = load_target(f, g, w, t);
        w.prop[t] = kNoProposal;
    }
    const double p = okey_inv(op.key);
    const double gt = op.gt;
    const double lower = op.fv - d.lxi;                  // BoundsField.lower (correction.py:122)
    const double m = (p < gt) ? p : gt;                  // np.minimum(g, prop)
    const double nv = (m < lower) ? lower : m;           // np.maximum(., lower)
    if (nv == gt) return;
    g[t] = nv;
    ++acc.edits;
    const unsigned int cnt = op.cnt + 1u;
    if (op.cnt) {   // a re-edit: store the extra count (apply_target)
        if (w.counts32) ((unsigned int*)w.counts)[t] = cnt - 1u;
        else ((uint16_t*)w.counts)[t] = (uint16_t)(cnt - 1u);
    }
    acc.maxc = max(acc.maxc, cnt);
    atomicOr(w.editbits + (t >> 5), 1u << (t & 31));
    acc.shared |= in_shared(d, x, y, z);
    const unsigned k = atomicAdd(&S.nedit, 1u);
    if (k < (unsigned)kT1Set) {
        S.edits[k] = (uint32_t)t;
    } else {   // edit list full: the global one (marked globally at the hand-back)
        S.ovf_edit = 1;
        w.elist[agg_append(&w.ctr->nelist)] = (uint32_t)t;
    }
#pragma unroll
    for (int r = -1; r < 14; ++r) {
        const int64_t u = t + (r < 0 ? 0 : rank_off(d, r));
        if (!((fw[r + 1] >> (u & 31)) & 1u)) continue;   // outside the core, or robust (never evaluated)
        const int ins = t1_insert(S.dset, (uint32_t)u);
        if (ins == 1) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(w.code + u));   // read by the next sweep
            const unsigned q = atomicAdd(&S.nd[b ^ 1], 1u);
            if (q < dcap) S.dirty[b ^ 1][q] = (uint32_t)u;
            else S.ovf_mark = 1;
        } else if (ins == 2) {
            S.ovf_mark = 1;
        }
    }
}

// chained != 0: launched right behind k_tail on the stream; runs only if that
// launch handed over (exit kTailSmall), continuing its iteration count,
// history and flags, so the hand-over costs no host round trip.
template <typename FT>
__global__ void __launch_bounds__(kT1Threads, 1) k_tail1(Dom d, const FT* __restrict__ f, double* g, Work w, int cur,
                                                         long long budget, unsigned long long* __restrict__ hist,
                                                         TailState* ts, unsigned long long* __restrict__ trace,
                                                         int chained) {
    pdl_wait();   // (programmatic dependent launch)
    extern __shared__ __align__(16) unsigned char t1raw[];
    T1Smem& S = *reinterpret_cast<T1Smem*>(t1raw);
    const int tid = threadIdx.x;
    DevCounters* c = w.ctr;
    long long it0 = 0;
    unsigned long long shared_or = 0, detections = 0;
    if (chained) {
        if (ts->exit != kTailSmall) return;
        cur = (int)ts->cur;
        it0 = (long long)ts->iterations;
        shared_or = ts->shared_or;
        detections = ts->detections;
        hist += it0;
        budget -= it0;
    }
    const int xl = cur ^ 1;   // global list a hand-back leaves the pending dirty set in
    // dirty-list capacity: the shared list, and the global list a hand-back fills
    const unsigned dcap = (unsigned)min((unsigned long long)kT1Dirty, w.act_cap);
    const unsigned n0 = (unsigned)min(__ldcg(&c->nact[cur]), (unsigned long long)dcap);
    for (unsigned i = tid; i < n0; i += kT1Threads) {
        const uint32_t u = __ldcg(w.act[cur] + i);
        S.dirty[0][i] = u;
        atomicAnd(w.actbits + (u >> 5), ~(1u << (u & 31)));
    }
    for (int i = tid; i < kT1Set; i += kT1Threads) {
        S.tset[i] = kT1Empty;
        S.tkey[i] = kNoProposal;
    }
    if (tid == 0) {
        S.nd[0] = n0;
        S.nd[1] = 0;
        S.ovf_tgt = S.ovf_edit = S.ovf_mark = 0;
        S.nedit = S.ndet = S.shared = S.maxc = 0;
        c->nact[xl] = 0;
        c->nwork = 0;
        c->nelist = 0;
        if (trace) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[8190] = t;
        }
    }
    int b = 0;
    for (long long it = 0;; ++it) {
        for (int i = tid; i < kT1Set; i += kT1Threads) S.dset[i] = kT1Empty;   // filled by A
        __syncthreads();
        // ---- S: detection + rules of the dirty list ----------------------------
        const unsigned nd = S.nd[b];
        unsigned mydet = 0;
        bool issued = false;
        for (unsigned i = tid; i < nd; i += kT1Threads) {
            const int64_t cc = S.dirty[b][i];
            int64_t x, y, z;
            coords(d, cc, x, y, z);
            double nv[14];
            load_ring(d, g, cc, x, y, z, nv, [](const double* q) { return __ldcg(q); });
            const double vc = __ldcg(g + cc);
            const uint8_t fc = __ldg(w.code + cc);
            const Scan s = fold_scan(vc, nv);
            const uint32_t bit = 1u << (cc & 31);
            if (code_mismatch(d, scan_code(s), fc)) {
                atomicOr(w.detbits + (cc >> 5), bit);
                ++mydet;
                EmitT1 emit{w, S};
                rules<false>(d, w, s, nv, fc, cc, emit);
                issued = issued || emit.issued;
            } else {
                atomicAnd(w.detbits + (cc >> 5), ~bit);   // (a reduction: no round trip)
            }
        }
        mydet = __reduce_add_sync(0xffffffffu, mydet);
        if ((tid & 31) == 0 && mydet) atomicAdd(&S.ndet, mydet);
        if (issued) __threadfence();   // this thread's RED.MINs are performed before anyone reads prop
        __syncthreads();
        // ---- A: apply every target, mark the rings of the edits -------------------
        ApplyAcc acc;
        for (int slot = tid; slot < kT1Set; slot += kT1Threads) {
            const uint32_t t = S.tset[slot];
            if (t == kT1Empty) continue;
            const unsigned long long key = S.tkey[slot];
            S.tset[slot] = kT1Empty;   // empty again for the next S
            S.tkey[slot] = kNoProposal;
            t1_apply_mark(d, f, g, w, S, b, dcap, (int64_t)t, acc, true, key);
        }
        if (S.ovf_tgt) {
            const unsigned long long n = __ldcg(&c->nwork);
            for (unsigned long long i = tid; i < n; i += kT1Threads) {
                const int64_t t = __ldcg(w.work + i);
                const uint32_t bit = 1u << (t & 31);
                if (atomicAnd(w.touched + (t >> 5), ~bit) & bit) t1_apply_mark(d, f, g, w, S, b, dcap, t, acc, false, 0ull);
            }
        }
        {
            const unsigned wm = __reduce_max_sync(0xffffffffu, acc.maxc);
            const unsigned wsh = __reduce_or_sync(0xffffffffu, acc.shared ? 1u : 0u);
            if ((tid & 31) == 0) {
                if (wm) atomicMax(&S.maxc, wm);
                if (wsh) S.shared = 1;
            }
        }
        __syncthreads();
        const unsigned nedit = S.nedit, ndet = S.ndet;
        const bool ovf_edit = S.ovf_edit != 0;
        const bool ovf = ovf_edit || S.ovf_mark != 0;
        const unsigned ne = min(nedit, (unsigned)kT1Set);
        shared_or |= S.shared;
        detections += ndet;
        if (tid == 0) {
            hist[it] = nedit;
            if (trace) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                trace[2 * it] = t;
                trace[2 * it + 1] = S.nd[b ^ 1];
            }
        }
        unsigned long long exit = 0, pending = 0;
        if (nedit == 0) {
            exit = kTailConverged;
        } else if (ovf) {
            // a shared structure overflowed: the 1-rings of every edit go through
            // the global marking of the list-mode iteration (actbits + act[xl])
            for (unsigned i = tid; i < ne; i += kT1Threads) mark_ring(d, w, S.edits[i], xl);
            if (ovf_edit) {
                const unsigned long long n = __ldcg(&c->nelist);
                for (unsigned long long i = tid; i < n; i += kT1Threads) mark_ring(d, w, __ldcg(w.elist + i), xl);
            }
            __threadfence();
            __syncthreads();
            pending = __ldcg(&c->nact[xl]);
            exit = pending > w.act_cap ? kTailOverflow : kTailBudget;
        } else if (it + 1 >= budget) {
            const unsigned n1 = S.nd[b ^ 1];
            for (unsigned i = tid; i < n1; i += kT1Threads) {
                const uint32_t u = S.dirty[b ^ 1][i];
                w.act[xl][i] = u;
                atomicOr(w.actbits + (u >> 5), 1u << (u & 31));
            }
            pending = n1;
            exit = kTailBudget;
            if (tid == 0) c->nact[xl] = n1;
        }
        if (exit) {
            if (tid == 0) {
                if (S.maxc) atomicMax(&c->maxcount, (unsigned long long)S.maxc);
                ts->iterations = (unsigned long long)(it0 + it + 1);
                ts->exit = exit;
                ts->cur = (unsigned long long)xl;
                ts->pending = pending;
                ts->last_edits = nedit;
                ts->last_detect = ndet;
                ts->shared_or = shared_or;
                ts->detections = detections;
                ts->appended = 1ull;
                c->ndetect = ndet;   // the host reads the last iteration's counters
            }
            return;
        }
        __syncthreads();   // every thread has read nedit / ndet / the flags above
        if (tid == 0) {    // the new dirty list is dirty[b ^ 1]
            S.nd[b] = 0;
            S.nedit = S.ndet = S.shared = 0;
        }
        b ^= 1;
    }
}

}  // namespace pmsz
