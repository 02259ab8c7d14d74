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

enum : unsigned long long { kTailConverged = 1, kTailBits = 2, kTailOverflow = 3, kTailBudget = 4, kTailSort = 5 };

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
                                              unsigned long long* __restrict__ trace) {
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
