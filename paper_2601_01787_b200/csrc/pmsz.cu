// pmsz.cu -- B200 (sm_100a) correction loop of pMSz behind the C ABI of
// include/pmsz.h.  One plan = one correction domain (the whole grid for
// run_correction, one block's extended extent for the block-parallel engine).
//
// Device layout per plan (N = domain voxels):
//   g      f64[N]   caller-owned corrected field (read-only inside K1, K2 writes)
//   f      f32/f64  caller-owned original field (read by K0 and, sparsely, by K2)
//   code   u8[N]    packed f-scan: nmax rank | nmin rank << 4, 15 = extremum
//   prop   u64[N]   order-preserving proposal keys, all-ones when idle (the
//                   invariant is restored by K2, so no per-iteration memset)
//   work   u32[N]   targets of the current iteration
//   act    u32[2][cap] + actbits u32[N/32]  dirty-centre lists (incremental mode)
//   editbits u32[N/32]  ever-edited bitmap -> EditSet
//   counts u16[N]   per-vertex edit counts (max_vertex_edits)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <atomic>
#include <algorithm>
#include <thread>
#include <chrono>

#include "../../include/pmsz.h"
#include "common.cuh"
#include "sweep.cuh"
#include "gen.cuh"
#include "tiles.cuh"
#include "tail.cuh"
#include "gather.cuh"
#include "qsweep.cuh"
#include "prep.cuh"
#include "segment.cuh"
#include "hoststage.h"

using namespace pmsz;

namespace {

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

pmsz_status fail(pmsz_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(PMSZ_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
    } while (0)

#define LAUNCHED() (g_launches.fetch_add(1, std::memory_order_relaxed))

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

inline unsigned grid_for(long long n, int threads, int per_sm = 8) {
    long long b = (n + threads - 1) / threads;
    long long cap = (long long)num_sms() * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (unsigned)b;
}


// ---- standalone scan (topology.scan_neighbors) -----------------------------
__global__ void __launch_bounds__(256) k_scan_full(Dom d, const double* __restrict__ v, int64_t* nmax,
                                                   int64_t* nmin, uint8_t* ismax, uint8_t* ismin,
                                                   uint8_t* code) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t y = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    const int64_t z = blockIdx.z;
    if (x >= d.nx || y >= d.ny) return;
    const int64_t c = x + y * d.sy + z * d.sz;
    const Scan s = gather_scan(d, v, x, y, z);
    if (nmax) nmax[c] = c + rank_off(d, s.rmax);
    if (nmin) nmin[c] = c + rank_off(d, s.rmin);
    if (ismax) ismax[c] = s.is_max;
    if (ismin) ismin[c] = s.is_min;
    if (code) code[c] = scan_code(s);
}

// ---- bounds check (BoundsField.admits) ------------------------------------
template <typename FT>
__global__ void __launch_bounds__(256) k_bounds(int64_t n, const FT* __restrict__ f, const double* __restrict__ g,
                                                double xi, unsigned long long* count) {
    unsigned long long mine = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double fv = (double)f[i];
        const double gv = g[i];
        if (!(gv >= fv - xi && gv <= fv + xi)) ++mine;
    }
    mine = __reduce_add_sync(0xffffffffu, (unsigned)mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, mine);
}

// g < lower (local_converge with an explicit lower bound): the reference's
// dense apply would raise such a vertex (correction.py:239-241)
__global__ void __launch_bounds__(256) k_below(int64_t n, const double* __restrict__ lower,
                                               const double* __restrict__ g, unsigned long long* count) {
    unsigned mine = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (g[i] < lower[i]) ++mine;
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, (unsigned long long)mine);
}

// f64 -> f32 with an exactness count (the drop-in's f32 fast path: fields read
// from f32 files are promoted exactly, codec.py:86-87)
__global__ void __launch_bounds__(256) k_narrow(int64_t n, const double* __restrict__ v, float* __restrict__ out,
                                                unsigned long long* inexact) {
    unsigned mine = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = v[i];
        const float y = (float)x;
        out[i] = y;
        if (!((double)y == x)) ++mine;   // NaN counts as inexact: the f64 path reports it
    }
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(inexact, (unsigned long long)mine);
}

// ---- bitmap compaction (ascending id lists) ----------------------------------
// The bitmap is cut into at most kMaxChunks contiguous chunks of whole warps'
// words (one chunk per CTA).  k_chunk_count sums each chunk; k_chunk_scan
// (one CTA) turns the sums into exclusive offsets in place and writes the
// total; the list/write kernels then compact each chunk in rounds of 4 x 256
// words with a block-wide scan, so ids come out ascending.
constexpr int kCompactThreads = 256;
constexpr int kMaxChunks = 1024;

struct Chunks {
    int64_t nwords, chunk;   // words per chunk (multiple of 4 x kCompactThreads)
    int n;                   // number of chunks
};

inline Chunks make_chunks(int64_t nwords, int sms) {
    Chunks c;
    c.nwords = nwords;
    // six chunks per SM (measured: 16 or 27 per SM, i.e. shorter chains of
    // rounds per CTA, are 0.01 ms slower per step at 512^3)
    static const int per_sm = getenv("PMSZ_COMPACT_PER_SM") ? std::max(1, atoi(getenv("PMSZ_COMPACT_PER_SM"))) : 6;
    int64_t want = std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, (int64_t)sms * per_sm));
    int64_t per = (nwords + want - 1) / want;
    constexpr int64_t kRound = 4 * kCompactThreads;   // words per round of the list / write kernels
    per = std::max<int64_t>(kRound, (per + kRound - 1) / kRound * kRound);
    c.chunk = per;
    c.n = (int)std::max<int64_t>(1, (nwords + per - 1) / per);
    return c;
}

__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* warp_tot, unsigned& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
    }
    if (lane == 31) warp_tot[wid] = s;
    __syncthreads();
    unsigned before = 0;
    total = 0;
#pragma unroll
    for (int q = 0; q < kCompactThreads / 32; ++q) {
        const unsigned t = warp_tot[q];
        before += q < wid ? t : 0u;
        total += t;
    }
    __syncthreads();   // warp_tot is reused by the next round
    return before + s - v;
}

// Per-chunk set-bit counts and their exclusive scan in one launch: the last
// CTA to finish (a ticket in *done, reset by that CTA) scans the counts.
__global__ void __launch_bounds__(kCompactThreads) k_chunk_count_scan(const uint32_t* __restrict__ bits, Chunks c,
                                                                      unsigned long long* counts,
                                                                      unsigned long long* total, unsigned* done) {
    pdl_wait();   // (programmatic dependent launch)
    __shared__ unsigned long long ws[kCompactThreads / 32];
    __shared__ bool last;
    const int64_t w0 = (int64_t)blockIdx.x * c.chunk, w1 = min(w0 + c.chunk, c.nwords);
    unsigned t = 0;
    for (int64_t w = w0 + threadIdx.x; w < w1; w += kCompactThreads) t += __popc(__ldg(bits + w));
    t = __reduce_add_sync(0xffffffffu, t);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) ws[wid] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long sum = 0;
        for (int q = 0; q < kCompactThreads / 32; ++q) sum += ws[q];
        counts[blockIdx.x] = sum;
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // exclusive scan of counts[0 .. n), n <= kMaxChunks = kPer per thread
    constexpr int kPer = kMaxChunks / kCompactThreads;
    const int n = (int)gridDim.x;
    unsigned long long v[kPer], mine = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = kPer * threadIdx.x + k;
        v[k] = i < n ? __ldcg(counts + i) : 0ull;
        mine += v[k];
    }
    unsigned long long sc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, sc, o);
        if (lane >= o) sc += y;
    }
    __syncthreads();   // ws is reused
    if (lane == 31) ws[wid] = sc;
    __syncthreads();
    unsigned long long before = 0, all = 0;
#pragma unroll
    for (int q = 0; q < kCompactThreads / 32; ++q) {
        before += q < wid ? ws[q] : 0ull;
        all += ws[q];
    }
    unsigned long long pos = before + sc - mine;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = kPer * threadIdx.x + k;
        if (i < n) counts[i] = pos;
        pos += v[k];
    }
    if (threadIdx.x == 0) {
        if (total) *total = all;
        *done = 0u;
    }
}

// Four consecutive bitmap words w .. w + 3 of [.., w1) (one 16-byte load when whole).
__device__ __forceinline__ uint4 load_words4(const uint32_t* bits, int64_t w, int64_t w1) {
    if (w + 3 < w1 && (reinterpret_cast<uintptr_t>(bits + w) & 15) == 0)
        return *reinterpret_cast<const uint4*>(bits + w);
    uint4 v = make_uint4(0u, 0u, 0u, 0u);   // tail of the bitmap, or a caller's unaligned view
    if (w < w1) v.x = bits[w];
    if (w + 1 < w1) v.y = bits[w + 1];
    if (w + 2 < w1) v.z = bits[w + 2];
    if (w + 3 < w1) v.w = bits[w + 3];
    return v;
}

// Chunk of the bitmap -> ascending ids (bits cleared on the way when `clear`).
// A round covers 4 x 256 words: thread t owns the four consecutive words
// 4 t .. 4 t + 3 (one vector load), one block scan per round.  The round's
// ids are staged in shared memory at their scanned positions and written out
// by consecutive threads (coalesced), unless the round holds more than
// kStageIds of them (then each thread writes its own, as the bits come).
constexpr int kStageIds = 4096;

template <class Out>
__device__ __forceinline__ void compact_round(const uint4 v, int64_t w, unsigned long long pos0, uint32_t* stage,
                                              unsigned* wt, unsigned& total, Out&& out) {
    const unsigned before = block_exclusive_scan(__popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w), wt, total);
    const uint32_t m4[4] = {v.x, v.y, v.z, v.w};
    if (total <= (unsigned)kStageIds) {
        unsigned k = before;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t m = m4[q];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                stage[k++] = (uint32_t)((w + q) * 32 + b);   // ids < 2^32 (plan limit)
            }
        }
        __syncthreads();
        for (unsigned e = threadIdx.x; e < total; e += kCompactThreads) out(pos0 + e, (int64_t)stage[e]);
        __syncthreads();   // stage is reused by the next round
    } else {
        unsigned long long pos = pos0 + before;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t m = m4[q];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                out(pos++, (w + q) * 32 + b);
            }
        }
    }
}

template <typename IdT>
__global__ void __launch_bounds__(kCompactThreads) k_chunk_list(uint32_t* __restrict__ bits, Chunks c,
                                                                const unsigned long long* __restrict__ offs,
                                                                IdT* __restrict__ list, int clear) {
    pdl_wait();   // (programmatic dependent launch)
    __shared__ unsigned wt[kCompactThreads / 32];
    __shared__ uint32_t stage[kStageIds];
    const int64_t w0 = (int64_t)blockIdx.x * c.chunk, w1 = min(w0 + c.chunk, c.nwords);
    unsigned long long pos0 = offs[blockIdx.x];
    uint4 nxt = load_words4(bits, w0 + 4 * threadIdx.x, w1);
    for (int64_t base = w0; base < w1; base += 4 * kCompactThreads) {
        const int64_t w = base + 4 * threadIdx.x;
        const uint4 v = nxt;
        nxt = load_words4(bits, w + 4 * kCompactThreads, w1);   // next round in flight
        if (clear && (v.x | v.y | v.z | v.w)) {
            if (w + 3 < w1 && (reinterpret_cast<uintptr_t>(bits + w) & 15) == 0)
                *reinterpret_cast<uint4*>(bits + w) = make_uint4(0u, 0u, 0u, 0u);
            else
                for (int q = 0; q < 4 && w + q < w1; ++q) bits[w + q] = 0u;
        }
        unsigned total;
        compact_round(v, w, pos0, stage, wt, total,
                      [&](unsigned long long pos, int64_t id) { list[pos] = (IdT)id; });
        pos0 += total;
    }
}

// Export of the edit record: ids and the corrected values (EditSet.diff).
__global__ void __launch_bounds__(kCompactThreads) k_chunk_write(const uint32_t* __restrict__ bits, Chunks c,
                                                                 int64_t n, const unsigned long long* __restrict__ offs,
                                                                 const double* __restrict__ g, int64_t* ids,
                                                                 double* vals, int64_t cap) {
    pdl_wait();   // (programmatic dependent launch)
    __shared__ unsigned wt[kCompactThreads / 32];
    __shared__ uint32_t stage[kStageIds];
    const int64_t w0 = (int64_t)blockIdx.x * c.chunk, w1 = min(w0 + c.chunk, c.nwords);
    unsigned long long pos0 = offs[blockIdx.x];
    uint4 nxt = load_words4(bits, w0 + 4 * threadIdx.x, w1);
    for (int64_t base = w0; base < w1; base += 4 * kCompactThreads) {
        const int64_t w = base + 4 * threadIdx.x;
        const uint4 v = nxt;
        nxt = load_words4(bits, w + 4 * kCompactThreads, w1);
        unsigned total;
        compact_round(v, w, pos0, stage, wt, total, [&](unsigned long long pos, int64_t id) {
            if (id < n && (long long)pos < cap) {
                ids[pos] = id;
                vals[pos] = g[id];
            }
        });
        pos0 += total;
    }
}

// ---- ghost-box helpers -------------------------------------------------------
struct Box {
    int64_t nx, ny;
    int64_t lo[3], ext[3];
    uint64_t mxy, mx;   // div_magic(ext[0] * ext[1]), div_magic(ext[0]): 32-bit index decode
};

// Field offset of element i (x-fastest) of box b; boxes hold < 2^32 elements.
__device__ __forceinline__ int64_t box_off(const Box& b, int64_t i) {
    const uint32_t ii = (uint32_t)i;
    const uint32_t z = fast_div(ii, b.mxy);
    const uint32_t r = ii - z * (uint32_t)(b.ext[0] * b.ext[1]);
    const uint32_t y = fast_div(r, b.mx);
    const uint32_t x = r - y * (uint32_t)b.ext[0];
    return (b.lo[0] + x) + b.nx * ((b.lo[1] + y) + b.ny * (b.lo[2] + z));
}

__global__ void __launch_bounds__(256) k_box_pack(Box b, const double* __restrict__ src, double* __restrict__ buf) {
    pdl_wait();   // (programmatic dependent launch)
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        buf[i] = src[box_off(b, i)];
    }
}

template <bool kMin>
__global__ void __launch_bounds__(256) k_box_unpack(Box b, double* __restrict__ dst, const double* __restrict__ buf,
                                                    unsigned long long* changed) {
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    unsigned mine = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = box_off(b, i);
        const double cur = dst[o], in = buf[i];
        const double nv = kMin ? (in < cur ? in : cur) : in;
        if (nv != cur) {
            dst[o] = nv;
            ++mine;
        }
    }
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine && changed) atomicAdd(changed, (unsigned long long)mine);
}

// Vertices changed outside an iteration (ghost merges) dirty their 1-ring:
// into the pending list (bits == 0) or the pending edit bitmap (bits != 0).
__device__ __forceinline__ void mark_changed(const Dom& d, const Work& w, int64_t v, int cur, int bits) {
    if (bits) atomicOr(w.iteredit + (v >> 5), 1u << (v & 31));
    else mark_ring(d, w, v, cur);
}

__global__ void __launch_bounds__(256) k_box_mark(Dom d, Work w, Box b, const double* __restrict__ before,
                                                  const double* __restrict__ g, int cur, int bits) {
    pdl_wait();   // (programmatic dependent launch)
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = box_off(b, i);
        if (g[o] != before[i]) mark_changed(d, w, o, cur, bits);
    }
}

// Ghost merge: dst[box] = min(dst[box], buf); changed vertices dirty their
// 1-ring (list or edit-bitmap, by the plan's pending mode; none if kFull).
__global__ void __launch_bounds__(256) k_box_merge(Dom d, Work w, Box b, double* __restrict__ g,
                                                   const double* __restrict__ buf, int cur, int mode,
                                                   unsigned long long* changed) {
    pdl_wait();   // (programmatic dependent launch)
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    unsigned mine = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = box_off(b, i);
        const double cur_v = g[o], in = buf[i];
        if (in < cur_v) {
            g[o] = in;
            ++mine;
            if (mode == 1) mark_changed(d, w, o, cur, 1);        // masked: edit bitmap
            else if (mode == 2) mark_changed(d, w, o, cur, 0);   // list
        }
    }
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(changed, (unsigned long long)mine);
}

__global__ void __launch_bounds__(256) k_mark_ids(Dom d, Work w, const uint32_t* __restrict__ ids, int64_t n, int cur,
                                                  int bits) {
    pdl_wait();   // (programmatic dependent launch)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        mark_changed(d, w, ids[i], cur, bits);
}

// Closed-1-ring dilation of the per-iteration edit bitmap: centre c is dirty
// when c + delta_o was edited for some o in {0} u STENCIL.  Word-level funnel
// shifts over the linear id space; bits that wrap across a row or plane edge
// only add clean centres (a superset is exact).
struct RingDelta {
    int64_t d[15];
};

// The masked sweep re-evaluates exactly the dirty centres, so their detection
// bits are cleared here and set again by the sweep for those that still fire.
__global__ void __launch_bounds__(256) k_dilate(const uint32_t* __restrict__ e, uint32_t* __restrict__ out,
                                                uint32_t* __restrict__ det, const uint32_t* __restrict__ frag,
                                                int64_t nwords, RingDelta rd) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
         w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < 15; ++k) {
            const int64_t p = w * 32 + rd.d[k];       // source bit of output bit 0
            const int64_t q = p >> 5;                 // floor division (arithmetic shift)
            const int sh = (int)(p & 31);
            const uint32_t lo = (q >= 0 && q < nwords) ? __ldg(e + q) : 0u;
            const uint32_t hi = (q + 1 >= 0 && q + 1 < nwords) ? __ldg(e + q + 1) : 0u;
            acc |= __funnelshift_r(lo, hi, sh);
        }
        if (frag) acc &= __ldg(frag + w);   // robust centres are never evaluated
        out[w] = acc;
        if (acc) det[w] &= ~acc;
    }
}

// kMaskedQ: kMasked swept by the TMA queue sweep (dense dirty sets) instead of the gather
enum { kFull = 0, kMasked = 1, kList = 2, kMaskedList = 3, kMaskedQ = 4 };

template <typename FT>
__global__ void __launch_bounds__(256) k_box_extract(Box b, int64_t gny, const FT* __restrict__ src, FT* __restrict__ dst) {
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        Box bg = b;
        bg.ny = gny;
        dst[i] = src[box_off(bg, i)];
    }
}

// ---- cross-rank epoch barrier carrying the round sums (pmsz_rounds) --------
struct SigArgs {
    unsigned long long* sums[PMSZ_MAX_RANKS];    // each rank's sum slots [2][world][4]
    unsigned long long* flags[PMSZ_MAX_RANKS];   // each rank's arrival epochs [world]
    unsigned long long v[4];
    unsigned long long* out;                     // the 4 sums over ranks (mapped pinned memory)
    unsigned long long epoch;
    volatile unsigned long long* flag;           // then seq here (the host spins on it)
    unsigned long long seq;
    int world, rank;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Thread q publishes this rank's values into rank q's slot of this epoch's
// parity and raises this rank's epoch there; then waits for q's epoch here.
__global__ void __launch_bounds__(PMSZ_MAX_RANKS) k_signal(SigArgs a) {
    pdl_wait();   // (programmatic dependent launch)
    const int q = threadIdx.x;
    const int par = (int)(a.epoch & 1);
    if (q < a.world) {
        unsigned long long* slot = a.sums[q] + ((size_t)par * a.world + a.rank) * 4;
        slot[0] = a.v[0]; slot[1] = a.v[1]; slot[2] = a.v[2]; slot[3] = a.v[3];
        st_release_sys(a.flags[q] + a.rank, a.epoch);   // orders the slot stores before the epoch
        while (ld_acquire_sys(a.flags[a.rank] + q) < a.epoch) __nanosleep(64);
    }
    __syncthreads();
    if (q < 4) {
        unsigned long long t = 0;
        for (int r = 0; r < a.world; ++r) t += a.sums[a.rank][((size_t)par * a.world + r) * 4 + q];
        a.out[q] = t;
    }
    if (a.flag) {
        __threadfence_system();
        __syncthreads();
        if (q == 0) *a.flag = a.seq;
    }
}

// g_host[ids[i]] = vals[i] (the edit record onto the streamed-back fhat), on
// a few host threads: ids are ascending, so each thread writes one contiguous
// range of the field.
// The record arrives in nch chunks (event ev[c] = chunk c landed); thread t
// owns one contiguous share of the record and patches it chunk by chunk as
// the chunks land, so the patch overlaps the transfer.
void patch_host(double* g, const int64_t* ids, const double* vals, int64_t m, cudaEvent_t* ev, int nch) {
    // latency-bound (one cache line per write, ~30 values apart): every host
    // thread, at least 64 k writes each
    const int64_t per = 1 << 16;
    const int nt = (int)std::min<int64_t>(std::min(64u, std::max(1u, std::thread::hardware_concurrency())),
                                          std::max<int64_t>(1, (m + per - 1) / per));
    auto work = [&](int t) {
        const int64_t a = m * t / nt, b = m * (t + 1) / nt;
        constexpr int64_t kAhead = 32;   // read-for-ownership of the target lines, this far ahead
        int c = 0;
        for (int64_t i = a; i < b;) {
            while (m * (c + 1) / nch <= i) ++c;                 // chunk holding record entry i
            cudaEventSynchronize(ev[c]);
            const int64_t e = std::min<int64_t>(b, m * (c + 1) / nch);
            for (; i < e; ++i) {
                if (i + kAhead < e) __builtin_prefetch(g + ids[i + kAhead], 1, 0);
                g[ids[i]] = vals[i];
            }
        }
    };
    if (nt == 1) { work(0); return; }
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
}

}  // namespace

// ============================================================================
// Plan
// ============================================================================
struct pmsz_plan {
    pmsz_desc desc;
    Dom dom;
    int64_t n = 0, nwords = 0;
    Work w{};
    DevCounters* ctr = nullptr;
    DevCounters* hctr = nullptr;   // pinned mirror
    volatile unsigned long long* hflag = nullptr;   // pinned: the last k_publish sequence number
    unsigned long long sync_seq = 0;
    unsigned long long* block_counts = nullptr;
    Chunks ch{};              // bitmap compaction layout
    int64_t scratch_bytes = 0;
    int cur = 0;              // pending dirty list
    int next_mode = 0;        // kFull / kMasked / kList / kMaskedList for the next iteration
    int last_mode = 0;
    int64_t pending = 0;      // length of the pending dirty list (kList)
    int64_t ncore = 0;        // centres in the core box
    RingDelta ring_delta{};   // id offsets of the closed 1-ring (dilation)
    bool prepared = false;
    int64_t floor_viol = 0, upper_viol = 0;
    // block-round bookkeeping
    int64_t iterations = 0, edit_total = 0;
    int f32 = 0;
    // live kernel timing (pmsz_profile)
    bool prof_on = false;
    bool prof_light = false;   // only the full-domain classes (PMSZ_PROFILE_FULL_DOMAIN)
    std::vector<cudaEvent_t> prof_ev;   // pairs
    std::vector<int> prof_cls;          // class per recorded pair
    double prof_ms[PMSZ_K_COUNT] = {};
    long long prof_n[PMSZ_K_COUNT] = {};
    // device-resident tail (k_tail)
    bool tail_on = true;
    bool tail1_on = true;                 // small dirty sets in the one-CTA shared-memory tail (k_tail1)
    bool totals_ready = false;            // the last tail_step converged and counted residual / edits
    int64_t pre_residual = 0, pre_edits = 0;
    TailState* tail = nullptr;
    TailState* htail = nullptr;          // pinned mirror
    unsigned long long* thist = nullptr;  // per-iteration edits of one tail launch
    unsigned long long* hthist = nullptr; // pinned mirror
    int tail_blocks[2] = {0, 0};          // cooperative grid per FT (f64, f32)
    int64_t sort_min = 262144;            // longer dirty lists are kept in actbits only and rebuilt sorted
    int64_t dense_min = 0;                // dirty lists above this take the pipelined gather (kMaskedList)
    bool mark_deferred = false;           // a merge marked rings without reading the counters back
    bool bits_only = false;               // the pending dirty set is in actbits only (no list)
    int64_t full_div = 8;                 // a full sweep follows when 15 x edits > ncore / full_div
    const uint32_t* offsets_of = nullptr; // bitmap whose block offsets block_counts holds
    int64_t edits_cached = -1;            // popcount(editbits) since the last iteration, -1 = unknown
    bool gather_on = true;                // masked iterations as sorted gathers (gather.cuh)
    bool robust_on = true;                // K0 classifies robust centres (never evaluated afterwards)
    bool qsweep_on = true;                // tiled sweeps evaluate a per-plane queue of fragile centres (qsweep.cuh)
    bool qprep_on = true;                 // K0 as screen + queue (prep.cuh)
    bool fuse_on = true;                  // K0 also runs the first detection sweep (prep.cuh)
    bool qmask_ok = false;                // dense masked iterations can use the TMA queue sweep (kMaskedQ)
    bool k0_detected = false;             // detbits / ndetect of the first iteration come from K0
    uint32_t* frag = nullptr;             // fragile-centre bitmap written by K0
    int64_t hist_chunk = 0;               // thist / hthist entries: iterations per tail launch
    std::vector<int64_t> hist_all;        // edits_per_iteration of the last pmsz_run_correction
    // host-buffer entry point staging (pmsz_run_correction_host)
    uint32_t* frag_out() const { return robust_on ? frag : nullptr; }
    void* stage_f = nullptr;
    double* stage_g = nullptr;
    int64_t* stage_ids = nullptr;
    double* stage_vals = nullptr;
    int64_t stage_cap = 0;
    cudaStream_t copy_stream = nullptr;   // host-to-device slabs of pmsz_run_correction_host
    std::vector<cudaEvent_t> stage_ev;    // [0]: staging free; [1 + c]: slab c landed
    std::vector<int64_t> stage_z;         // slab boundaries in z (nslabs + 1)
    std::vector<cudaEvent_t> rec_ev;      // edit-record chunks back on the host
    bool stage_pending = false;           // the next K0 waits for the slabs, one launch per slab
    cudaStream_t d2h_stream = nullptr;    // corrected-field slabs back to the host (pmsz_run_correction_host)
    cudaEvent_t d2h_done = nullptr;
    int64_t* hrec_ids = nullptr;          // pinned bounce buffers of the edit record (field patch)
    double* hrec_vals = nullptr;
    int64_t hrec_cap = 0;
    int64_t hrec_count = -1;              // record entries held there after a host run (pmsz_edits_host)
    StageFeed* feed = nullptr;            // host staging thread of a pageable-input host run
    char* hring = nullptr;                // pinned staging ring (pageable inputs): hring_n x hring_chunk
    size_t hring_chunk = 0;
    int hring_n = 0;
    std::vector<cudaEvent_t> hring_ev;    // ring slot c free again
    unsigned long long* dsig = nullptr;   // pmsz_rounds: the summed round values (device) ...
    unsigned long long* hsig = nullptr;   // ... and their pinned mirror
};

namespace {

Dom make_dom(const pmsz_desc& d) {
    Dom o{};
    o.nx = d.nx; o.ny = d.ny; o.nz = d.nz;
    o.sy = d.nx; o.sz = d.nx * d.ny; o.n = d.nx * d.ny * d.nz;
    for (int a = 0; a < 3; ++a) {
        o.lo[a] = d.core_lo[a]; o.hi[a] = d.core_hi[a];
        o.shl[a] = d.shared_lo[a]; o.shh[a] = d.shared_hi[a];
    }
    o.xi = d.xi; o.tau = d.tau;
    o.lxi = (d.flags & PMSZ_FLAG_LOWER) ? 0.0 : d.xi;
    o.extrema_only = (d.flags & PMSZ_FLAG_EXTREMA_ONLY) ? 1 : 0;
    o.msy = div_magic((uint64_t)o.sy);
    o.msz = div_magic((uint64_t)o.sz);
    return o;
}

// ---- live kernel timing: an event pair around every launch of a plan --------
int prof_begin(pmsz_plan* p, cudaStream_t s, int cls) {
    if (!p->prof_on) return -1;
    if (p->prof_light && cls != PMSZ_K_PREP && cls != PMSZ_K_SWEEP_FULL && cls != PMSZ_K_VERIFY) return -1;
    const size_t k = p->prof_cls.size();
    while (p->prof_ev.size() < 2 * (k + 1)) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return -1;
        p->prof_ev.push_back(e);
    }
    cudaEventRecord(p->prof_ev[2 * k], s);
    return (int)k;
}

void prof_end(pmsz_plan* p, cudaStream_t s, int tok, int cls) {
    if (tok < 0) return;
    cudaEventRecord(p->prof_ev[2 * tok + 1], s);
    p->prof_cls.push_back(cls);
}

// Called once the stream is known to be idle.
void prof_flush(pmsz_plan* p) {
    for (size_t k = 0; k < p->prof_cls.size(); ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p->prof_ev[2 * k], p->prof_ev[2 * k + 1]) == cudaSuccess) {
            p->prof_ms[p->prof_cls[k]] += ms;
            p->prof_n[p->prof_cls[k]] += 1;
        }
    }
    p->prof_cls.clear();
}

struct ProfScope {
    pmsz_plan* p; cudaStream_t s; int tok; int cls;
    ProfScope(pmsz_plan* p_, cudaStream_t s_, int cls_) : p(p_), s(s_), tok(prof_begin(p_, s_, cls_)), cls(cls_) {}
    ~ProfScope() { prof_end(p, s, tok, cls); }
};

// The counters reach the host by a one-CTA kernel writing them into the
// pinned (mapped) mirror and then a sequence number into a pinned flag the
// host spins on: no copy-engine round trip and no stream synchronisation on
// the ~5 host decisions of a run (each cost the device ~25 us idle).  The
// kernel is the last operation of the stream, so the flag also means every
// earlier operation has completed.
// (tail: also the tail state and its per-iteration edit counts, k words of
// them where k = the state's iteration count, capped at hist_cap)
__global__ void k_publish(const DevCounters* __restrict__ c, DevCounters* h, volatile unsigned long long* flag,
                          unsigned long long seq, const unsigned long long* __restrict__ ts, unsigned long long* hts,
                          int ts_words, const unsigned long long* __restrict__ hist, unsigned long long* hhist,
                          long long hist_cap) {
    pdl_wait();   // (programmatic dependent launch)
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(c);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(h);
    for (int i = threadIdx.x; i < (int)(sizeof(DevCounters) / 8); i += blockDim.x) dst[i] = __ldcg(src + i);
    if (ts) {
        for (int i = threadIdx.x; i < ts_words; i += blockDim.x) hts[i] = __ldcg(ts + i);
        const long long k = min((long long)__ldcg(ts), hist_cap);   // TailState::iterations
        for (long long i = threadIdx.x; i < k; i += blockDim.x) hhist[i] = __ldcg(hist + i);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *flag = seq;
}

bool sync_by_kernel() {
    static const bool on = !(getenv("PMSZ_SYNC_KERNEL") && atoi(getenv("PMSZ_SYNC_KERNEL")) == 0);
    return on;
}

// Spin until the stream's last kernel has written `seq` into the plan's flag.
pmsz_status spin_flag(pmsz_plan* p, cudaStream_t s, unsigned long long seq) {
    CUDA_TRY(cudaGetLastError());
    for (unsigned long long i = 1;; ++i) {
        if (*p->hflag == seq) break;
        // short waits spin; long ones (a host run's K0 waiting for its input)
        // yield the core to the staging threads
        if (i < 4096) host_pause();
        else std::this_thread::yield();
        if ((i & 4095) == 0) {   // a failed stream would never set the flag
            const cudaError_t q = cudaStreamQuery(s);
            if (q != cudaSuccess && q != cudaErrorNotReady) {
                cudaGetLastError();
                return fail(PMSZ_ERR_CUDA, std::string("CUDA: ") + cudaGetErrorString(q));
            }
            if (q == cudaSuccess && *p->hflag != seq) return fail(PMSZ_ERR_CUDA, "counter publish lost");
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return PMSZ_OK;
}

pmsz_status sync_counters(pmsz_plan* p, cudaStream_t s) {
    if (sync_by_kernel() && p->hflag) {
        const unsigned long long seq = ++p->sync_seq;
        pdl_launch(k_publish, 1, 64, 0, s, p->ctr, p->hctr, p->hflag, seq, (const unsigned long long*)nullptr,
                   (unsigned long long*)nullptr, 0, (const unsigned long long*)nullptr, (unsigned long long*)nullptr, 0LL);
        const pmsz_status st = spin_flag(p, s, seq);
        if (st) return st;
        prof_flush(p);
        return PMSZ_OK;
    }
    CUDA_TRY(cudaMemcpyAsync(p->hctr, p->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    prof_flush(p);
    return PMSZ_OK;
}

// Reset the per-iteration counters (nwork, nedits, ndetect, shared_dirty, nact[nxt]).
pmsz_status reset_iter(pmsz_plan* p, cudaStream_t s, int nxt) {
    CUDA_TRY(cudaMemsetAsync(p->ctr, 0, offsetof(DevCounters, nact), s));
    CUDA_TRY(cudaMemsetAsync(&p->ctr->nact[nxt], 0, sizeof(unsigned long long), s));
    return PMSZ_OK;
}

// Set bits of a bitmap: per-block counts + one-block exclusive scan; the total
// lands in *dst on the device.
void launch_bits_total(pmsz_plan* p, const uint32_t* bits, unsigned long long* dst, cudaStream_t s) {
    p->offsets_of = bits;
    pdl_launch(k_chunk_count_scan, (unsigned)p->ch.n, kCompactThreads, 0, s, bits, p->ch, p->block_counts, dst,
               (unsigned*)(p->block_counts + kMaxChunks));
    LAUNCHED();
}

// A large pending dirty list is replaced by the ascending compaction of actbits
// (the same set; the bits are cleared on the way): neighbouring threads then
// gather neighbouring cache lines instead of one ring after another.
int sort_pending(pmsz_plan* p, cudaStream_t s) {
    if (p->pending <= p->sort_min && !p->bits_only) return 0;
    p->bits_only = false;
    ProfScope ps(p, s, PMSZ_K_COMPACT);
    launch_bits_total(p, p->w.actbits, &p->ctr->nact[p->cur], s);
    pdl_launch(k_chunk_list<uint32_t>, (unsigned)p->ch.n, kCompactThreads, 0, s, p->w.actbits, p->ch,
               (const unsigned long long*)p->block_counts, p->w.act[p->cur], 1);
    LAUNCHED();
    return 1;
}

template <typename FT>
pmsz_status launch_apply(pmsz_plan* p, const void* f, double* g, cudaStream_t s, int nxt, bool after_full,
                         int64_t bound) {
    if (after_full) {
        // touched bitmap -> ascending target list (load-balanced apply)
        ProfScope ps(p, s, PMSZ_K_COMPACT);
        launch_bits_total(p, p->w.touched, &p->ctr->nwork, s);
        pdl_launch(k_chunk_list<uint32_t>, (unsigned)p->ch.n, kCompactThreads, 0, s, p->w.touched, p->ch,
                   (const unsigned long long*)p->block_counts, p->w.work, 1);
        LAUNCHED();
    }
    ProfScope ps(p, s, PMSZ_K_APPLY);
    // one CTA per SM: fewer targets in flight keep the z-window of the sorted
    // target list (g, prop, f, counts) L2-resident -- 10 % faster than 8 / SM
    static const int apply_per_sm = getenv("PMSZ_APPLY_PER_SM") ? atoi(getenv("PMSZ_APPLY_PER_SM")) : 1;
    Work w = p->w;
    w.first_apply = p->iterations == 0 ? 1 : 0;   // nothing edited yet: no counts / editbits reads
    pdl_launch(k_apply_list<FT>, grid_for(bound, 256, apply_per_sm), 256, 0, s, p->dom, (const FT*)f, g, w, nxt);
    LAUNCHED();
    if (p->w.incremental) {   // list-mode ring marking (no-op when the edits went to the bitmap)
        pdl_launch(k_mark_list, grid_for(std::min<int64_t>(15 * bound, (int64_t)p->w.mark_limit), 256, 4), 256, 0, s,
                   p->dom, p->w, nxt, (unsigned long long)p->sort_min);
        LAUNCHED();
    }
    return PMSZ_OK;
}

// Form of the next iteration from the marking of the last one:
//   edits marked in the edit bitmap (many edits) -> masked sweep over its
//     dilation (or, with the old tiled scan, a full sweep when dense);
//   dirty list overflowed                        -> full sweep;
//   dirty list longer than dense_min             -> masked sweep over actbits;
//   otherwise                                    -> list (gather) sweep.
pmsz_status choose_next(pmsz_plan* p, cudaStream_t s, bool marked_bits, int64_t nedits, int nxt, int64_t nact,
                        bool appended, int64_t bound) {
    if (marked_bits) {
        if (15 * nedits > p->ncore / p->full_div) {
            if (p->qmask_ok) {
                p->next_mode = kMaskedQ;   // dense: masked queue sweep over the dilation
            } else {
                p->next_mode = kFull;
                CUDA_TRY(cudaMemsetAsync(p->w.iteredit, 0, p->nwords * 4, s));
            }
        } else {
            p->next_mode = kMasked;
        }
    } else if (!appended) {   // dirty set in actbits only; `bound` >= its size
        p->cur = nxt;
        p->pending = bound;
        p->bits_only = true;
        p->next_mode = (p->gather_on && bound > p->dense_min) ? kMaskedList : kList;
        if (p->next_mode == kList && bound > (int64_t)p->w.act_cap) p->next_mode = kFull;   // list would overflow
    } else if (nact > (int64_t)p->w.act_cap) {
        p->next_mode = kFull;
    } else {
        p->cur = nxt;
        p->pending = nact;
        p->bits_only = false;
        p->next_mode = (p->gather_on && nact > p->dense_min) ? kMaskedList : kList;
    }
    return PMSZ_OK;
}

// One Jacobi iteration: K1 in one of four forms, then K2.  Leaves the
// counters on the host and decides the form of the next iteration:
//   kFull       -- tiled sweep of every core centre (first iteration)
//   kMasked     -- the centres of the dilated edit bitmap of the previous
//                  iteration (exact by SURVEY H7), compacted to an ascending
//                  list and swept by the pipelined gather (gather.cuh)
//   kMaskedList -- the same over the marked dirty set (actbits) when the
//                  explicit list is long
//   kList       -- gather sweep over the explicit dirty-centre list (short)
pmsz_status iterate_once(pmsz_plan* p, const void* f, double* g, cudaStream_t s) {
    const int nxt = p->cur ^ 1;
    p->edits_cached = -1;
    const Dom& d = p->dom;
    const int mode = p->w.incremental ? p->next_mode : kFull;
    // the first full sweep ran inside K0 (detbits and ndetect are set; every
    // other per-iteration counter is still zero from reset_run_state)
    const bool predetected = mode == kFull && p->k0_detected;
    p->k0_detected = false;
    pmsz_status st = predetected ? PMSZ_OK : reset_iter(p, s, nxt);
    if (st) return st;
    const int64_t cx = d.hi[0] - d.lo[0], cy = d.hi[1] - d.lo[1], cz = d.hi[2] - d.lo[2];
    const bool nonempty = cx > 0 && cy > 0 && cz > 0;
    int64_t apply_bound = p->n;   // upper bound of the targets, sizes the apply grid
    const bool gather = p->gather_on && mode != kFull && mode != kMaskedQ;
    if (mode != kList) p->bits_only = false;   // actbits is consumed (compacted or cleared) below
    if (mode == kFull) {
        if (p->w.incremental) CUDA_TRY(cudaMemsetAsync(p->w.actbits, 0, p->nwords * 4, s));
        if (!predetected) CUDA_TRY(cudaMemsetAsync(p->w.detbits, 0, p->nwords * 4, s));
        p->w.track = 0;
        if (nonempty && !predetected) {
            ProfScope ps(p, s, PMSZ_K_SWEEP_FULL);
            // the TMA queue sweep runs the rules of its mismatches itself
            if (!(p->qsweep_on && launch_sweep_q<false>(d, g, p->w, s))) launch_sweep_full<false>(d, g, p->w, s);
            LAUNCHED();
        }
    } else if (mode == kMasked || mode == kMaskedList || mode == kMaskedQ) {
        p->w.track = 0;
        if (mode != kMaskedList) {   // dirty set = dilation of the previous iteration's edits
            ProfScope ps(p, s, PMSZ_K_OTHER);
            k_dilate<<<grid_for(p->nwords, 256, 8), 256, 0, s>>>(p->w.iteredit, p->w.actbits, p->w.detbits,
                                                               p->w.frag, p->nwords, p->ring_delta);
            LAUNCHED();
            CUDA_TRY(cudaMemsetAsync(p->w.iteredit, 0, p->nwords * 4, s));
        }                        // kMaskedList: the dirty set is actbits as marked (list dropped)
        if (gather) {
            // actbits -> ascending centre list (in `work`, bits cleared) -> pipelined gather sweep
            {
                ProfScope ps(p, s, PMSZ_K_COMPACT);
                launch_bits_total(p, p->w.actbits, &p->ctr->ndefer, s);
                pdl_launch(k_chunk_list<uint32_t>, (unsigned)p->ch.n, kCompactThreads, 0, s, p->w.actbits, p->ch,
                           (const unsigned long long*)p->block_counts, p->w.work, 1);
                LAUNCHED();
            }
            if (nonempty) {
                ProfScope ps(p, s, PMSZ_K_SWEEP_MASKED);
                // one thread per centre (k_sweep_list, 4 CTAs / SM) beats the
                // cp.async-pipelined k_gather on the fragile-filtered lists
                // (0.12 vs 0.25 ms at 512^3); PMSZ_LIST_SWEEP=0 selects k_gather
                static const int list_per_sm = getenv("PMSZ_LIST_SWEEP") ? atoi(getenv("PMSZ_LIST_SWEEP")) : 4;
                if (list_per_sm > 0)
                    pdl_launch(k_sweep_list, num_sms() * list_per_sm, 256, 0, s, d, g, p->w,
                               (const uint32_t*)p->w.work, (const unsigned long long*)&p->ctr->ndefer);
                else
                    k_gather<false><<<num_sms() * 2, kGWarps * 32, kGatherSmem, s>>>(d, g, p->w, p->w.work,
                                                                                     &p->ctr->ndefer);
                LAUNCHED();
            }
        } else {
            if (nonempty) {
                ProfScope ps(p, s, PMSZ_K_SWEEP_MASKED);
                if (!(p->qsweep_on && launch_sweep_q<false>(d, g, p->w, s, p->w.actbits)))
                    launch_sweep_full<false>(d, g, p->w, s, p->w.actbits);
                LAUNCHED();
            }
            CUDA_TRY(cudaMemsetAsync(p->w.actbits, 0, p->nwords * 4, s));
        }
    }
    if (mode != kList && nonempty && !gather) {
        // centres with a detection (bitmap set by the tiled sweep) -> list -> rules
        {
            ProfScope ps(p, s, PMSZ_K_COMPACT);
            launch_bits_total(p, p->w.detbits, &p->ctr->ndefer, s);
            pdl_launch(k_chunk_list<uint32_t>, (unsigned)p->ch.n, kCompactThreads, 0, s, p->w.detbits, p->ch,
                       (const unsigned long long*)p->block_counts, p->w.work, 0);
            LAUNCHED();
        }
        ProfScope ps(p, s, PMSZ_K_DEFER);
        // two CTAs per SM measured best (the same L2-window effect as the apply)
        static const int defer_per_sm = getenv("PMSZ_DEFER_PER_SM") ? atoi(getenv("PMSZ_DEFER_PER_SM")) : 2;
        pdl_launch(k_defer, grid_for(p->n, 256, defer_per_sm), 256, 0, s, d, g, p->w);
        LAUNCHED();
    }
    if (mode == kList) {
        const int sorted = sort_pending(p, s);
        ProfScope ps(p, s, PMSZ_K_SWEEP_SPARSE);
        p->w.track = 1;
        const int64_t m = std::min<int64_t>(p->pending, (int64_t)p->w.act_cap);
        pdl_launch(k_sweep_sparse, grid_for(m, 256, 8), 256, 0, s, d, g, p->w, p->cur, sorted);
        LAUNCHED();
        apply_bound = std::min<int64_t>(p->n, 15 * m + 32);
    }
    p->last_mode = mode;
    st = p->f32 ? launch_apply<float>(p, f, g, s, nxt, mode != kList, apply_bound)
                : launch_apply<double>(p, f, g, s, nxt, mode != kList, apply_bound);
    if (st) return st;
    CUDA_TRY(cudaGetLastError());
    st = sync_counters(p, s);
    if (st) return st;
    if (p->w.incremental) {
        const int64_t bound = 15 * (int64_t)p->hctr->nelist;
        st = choose_next(p, s, p->hctr->scratch[3] == kMarkBits, (int64_t)p->hctr->nedits, nxt,
                         (int64_t)p->hctr->nact[nxt], bound <= p->sort_min, bound);
        if (st) return st;
    }
    return PMSZ_OK;
}

// ---- device-resident tail ---------------------------------------------------
void fill_result(pmsz_plan* p, pmsz_result* r);

bool tail_ok(const pmsz_plan* p) {
    return p->tail_on && p->w.incremental && p->next_mode == kList && p->floor_viol == 0 &&
           p->w.edited_mask == nullptr;
}

template <typename FT>
pmsz_status launch_tail(pmsz_plan* p, const void* f, double* g, cudaStream_t s, long long budget, int sorted) {
    int& nb = p->tail_blocks[std::is_same<FT, float>::value ? 1 : 0];
    if (nb == 0) {
        int per = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tail<FT>, 256, 0));
        if (per < 1) return fail(PMSZ_ERR_CUDA, "k_tail cannot be resident");
        static const int cap = getenv("PMSZ_TAIL_PER_SM") ? std::max(1, atoi(getenv("PMSZ_TAIL_PER_SM"))) : 1;
        nb = std::min(per, cap) * num_sms();
        static const int nb_env = getenv("PMSZ_TAIL_BLOCKS") ? atoi(getenv("PMSZ_TAIL_BLOCKS")) : 0;
        if (nb_env > 0) nb = std::min(nb, nb_env);
    }
    unsigned long long sort_min = (unsigned long long)p->sort_min;
    unsigned long long dense_min = (unsigned long long)(p->gather_on ? p->dense_min : p->w.act_cap);
    unsigned long long* cc = p->block_counts;
    Dom d = p->dom;
    const FT* fp = (const FT*)f;
    Work w = p->w;
    int cur = p->cur;
    unsigned long long* h = p->thist;
    TailState* t = p->tail;
    // PMSZ_TAIL_TRACE=1: per-iteration device timestamps printed to stderr
    // (diagnostics only; synchronises after the launch)
    unsigned long long* tr = nullptr;
    static const bool trace = getenv("PMSZ_TAIL_TRACE") != nullptr;
    static unsigned long long* trace_buf = nullptr;
    if (trace) {
        if (!trace_buf) CUDA_TRY(cudaMalloc(&trace_buf, 2 * 8 * 4096));
        tr = trace_buf;
        CUDA_TRY(cudaMemsetAsync(tr, 0, 2 * 8 * 4096, s));
    }
    static const int64_t t1max = getenv("PMSZ_TAIL1_MAX") ? atoll(getenv("PMSZ_TAIL1_MAX")) : kT1Handover;
    unsigned long long small_max =
        p->tail1_on ? (unsigned long long)std::min<int64_t>(std::min<int64_t>(t1max, kT1Dirty), (int64_t)p->w.act_cap) : 0ull;
    void* args[] = {&d, &fp, &g, &w, &cur, &sorted, &sort_min, &dense_min, &cc, &budget, &h, &t, &tr, &small_max};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_tail<FT>, dim3(nb), dim3(256), args, 0, s));
    LAUNCHED();
    if (trace) {
        std::vector<unsigned long long> h2(2 * 4096);
        cudaMemcpyAsync(h2.data(), tr, h2.size() * 8, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "tail nb=%d cur=%d pending=%lld:", nb, cur, (long long)p->pending);
        for (int i = 0; i < 4000 && h2[2 * i]; ++i)
            fprintf(stderr, " %.1fus/%llu", (h2[2 * i] - (i ? h2[2 * i - 2] : h2[8190])) / 1e3, h2[2 * i + 1]);
        fprintf(stderr, "\n  phases S/A/M of the first iterations:");
        for (int i = 0; i < 4 && h2[2 * i]; ++i) {
            const unsigned long long t0 = i ? h2[2 * i - 2] : h2[8190];
            fprintf(stderr, " [%.1f %.1f %.1f]", (h2[8000 + 2 * i] - t0) / 1e3, (h2[8001 + 2 * i] - h2[8000 + 2 * i]) / 1e3,
                    (h2[2 * i] - h2[8001 + 2 * i]) / 1e3);
        }
        fprintf(stderr, "\n");
    }
    return PMSZ_OK;
}

// Small dirty sets: the one-CTA shared-memory tail (k_tail1, tail.cuh).
template <typename FT>
pmsz_status launch_tail1(pmsz_plan* p, const void* f, double* g, cudaStream_t s, long long budget, int chained) {
    static unsigned long long attr = 0;
    smem_attr_once(k_tail1<FT>, (int)kT1SmemBytes, attr);
    static const bool trace = getenv("PMSZ_TAIL_TRACE") != nullptr;
    static unsigned long long* trace_buf = nullptr;
    unsigned long long* tr = nullptr;
    if (trace) {
        if (!trace_buf) CUDA_TRY(cudaMalloc(&trace_buf, 2 * 8 * 4096));
        tr = trace_buf;
        CUDA_TRY(cudaMemsetAsync(tr, 0, 2 * 8 * 4096, s));
    }
    pdl_launch(k_tail1<FT>, 1, kT1Threads, kT1SmemBytes, s, p->dom, (const FT*)f, g, p->w, p->cur, budget, p->thist,
               p->tail, tr, chained);
    LAUNCHED();
    if (trace) {
        std::vector<unsigned long long> h2(2 * 4096);
        cudaMemcpyAsync(h2.data(), tr, h2.size() * 8, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "tail1 cur=%d pending=%lld:", p->cur, (long long)p->pending);
        for (int i = 0; i < 4000 && h2[2 * i]; ++i)
            fprintf(stderr, " %.1fus/%llu", (h2[2 * i] - (i ? h2[2 * i - 2] : h2[8190])) / 1e3, h2[2 * i + 1]);
        fprintf(stderr, "\n");
    }
    return PMSZ_OK;
}

// Run up to `budget` list-mode iterations in one k_tail launch and bring the
// plan state to where iterate_once would have left it.  Per-iteration edit
// counts land in p->hthist[0 .. *k).
pmsz_status tail_step(pmsz_plan* p, const void* f, double* g, cudaStream_t s, long long budget, int64_t* k,
                      bool* shared_any, bool totals = false) {
    p->totals_ready = false;
    p->edits_cached = -1;
    pmsz_status st = reset_iter(p, s, p->cur ^ 1);
    if (st) return st;
    static const int64_t t1max = getenv("PMSZ_TAIL1_MAX") ? atoll(getenv("PMSZ_TAIL1_MAX")) : kT1Handover;
    const bool micro = p->tail1_on && !p->bits_only && p->pending > 0 &&
                       p->pending <= std::min<int64_t>(std::min<int64_t>(t1max, kT1Dirty), (int64_t)p->w.act_cap);
    const int sorted = micro ? 0 : sort_pending(p, s);
    {
        ProfScope ps(p, s, PMSZ_K_TAIL);
        if (micro) {
            st = p->f32 ? launch_tail1<float>(p, f, g, s, budget, 0) : launch_tail1<double>(p, f, g, s, budget, 0);
        } else {
            st = p->f32 ? launch_tail<float>(p, f, g, s, budget, sorted) : launch_tail<double>(p, f, g, s, budget, sorted);
            // the grid tail hands a small dirty list straight to k_tail1 (kTailSmall)
            if (!st && p->tail1_on)
                st = p->f32 ? launch_tail1<float>(p, f, g, s, budget, 1) : launch_tail1<double>(p, f, g, s, budget, 1);
        }
        if (st) return st;
    }
    if (totals) {   // the run's closing counts, read with this synchronisation (used if the tail converged)
        ProfScope ps(p, s, PMSZ_K_COMPACT);
        launch_bits_total(p, p->w.detbits, &p->ctr->scratch[1], s);
        launch_bits_total(p, p->w.editbits, &p->ctr->scratch[2], s);
    }
    if (sync_by_kernel() && p->hflag) {   // state + history + counters in one publish
        const unsigned long long seq = ++p->sync_seq;
        k_publish<<<1, 128, 0, s>>>(p->ctr, p->hctr, p->hflag, seq, (const unsigned long long*)p->tail,
                                    (unsigned long long*)p->htail, (int)(sizeof(TailState) / 8), p->thist, p->hthist,
                                    budget);
        st = spin_flag(p, s, seq);
        if (st) return st;
        prof_flush(p);
    } else {
        CUDA_TRY(cudaMemcpyAsync(p->htail, p->tail, sizeof(TailState), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(p->hthist, p->thist, sizeof(unsigned long long) * budget, cudaMemcpyDeviceToHost, s));
        st = sync_counters(p, s);
        if (st) return st;
    }
    const TailState& ts = *p->htail;
    if (totals && ts.exit == kTailConverged) {
        p->totals_ready = true;
        p->pre_residual = (int64_t)p->hctr->scratch[1];
        p->pre_edits = (int64_t)p->hctr->scratch[2];
    }
    *k = (int64_t)ts.iterations;
    *shared_any = ts.shared_or != 0;
    p->iterations += *k;
    for (int64_t i = 0; i < *k; ++i) p->edit_total += (int64_t)p->hthist[i];
    p->last_mode = kList;
    if (ts.exit == kTailOverflow) {
        p->next_mode = kFull;
    } else {
        st = choose_next(p, s, ts.exit == kTailBits, (int64_t)ts.last_edits, (int)ts.cur, (int64_t)ts.pending,
                         ts.appended != 0, (int64_t)ts.pending);
        if (st) return st;
    }
    return PMSZ_OK;
}

void tail_result(pmsz_plan* p, pmsz_result* r, int64_t k) {
    if (!r) return;
    fill_result(p, r);
    r->last_edits = (int64_t)p->htail->last_edits;
    r->last_detections = (int64_t)p->htail->last_detect;
    r->shared_dirty = p->htail->shared_or ? 1 : 0;
    r->iterations = p->iterations;
    r->edit_count = p->edit_total;
    r->sparse_sweeps += k;
}

// The per-run resets in one launch (instead of a memset call each: the host
// side of those calls delayed K0 by ~40 us per run).  Buffers are cudaMalloc'd
// (16-byte aligned); the counters are reset by one thread, which then sets
// bound_first to all-ones.
struct ZeroList {
    void* p[8];
    unsigned long long bytes[8];
    int k;
};
__global__ void __launch_bounds__(256) k_zero_many(ZeroList z, DevCounters* ctr) {
    pdl_wait();   // (programmatic dependent launch)
    const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    if (t == 0) {
        unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
        for (size_t i = 0; i < sizeof(DevCounters) / 8; ++i) c[i] = 0ull;
        ctr->bound_first = ~0ull;
    }
    for (int b = 0; b < z.k; ++b) {
        uint4* q = reinterpret_cast<uint4*>(z.p[b]);
        const unsigned long long n16 = z.bytes[b] / 16;
        for (unsigned long long i = t; i < n16; i += stride) q[i] = make_uint4(0u, 0u, 0u, 0u);
        unsigned char* tail = reinterpret_cast<unsigned char*>(z.p[b]);
        for (unsigned long long i = n16 * 16 + t; i < z.bytes[b]; i += stride) tail[i] = 0;
    }
}

pmsz_status reset_run_state(pmsz_plan* p, cudaStream_t s, uint32_t* extra0 = nullptr, uint32_t* extra1 = nullptr) {
    p->edits_cached = -1;
    p->mark_deferred = false;
    ZeroList z{};
    auto add = [&](void* ptr, unsigned long long bytes) {
        if (ptr && bytes) { z.p[z.k] = ptr; z.bytes[z.k] = bytes; ++z.k; }
    };
    add(p->w.editbits, p->nwords * 4);
    add(p->w.counts, p->n * (p->w.counts32 ? 4 : 2));
    if (p->w.incremental) {
        add(p->w.actbits, p->nwords * 4);
        add(p->w.iteredit, p->nwords * 4);
    }
    add(extra0, p->nwords * 4);   // (prep: the fragile and detection bitmaps)
    add(extra1, p->nwords * 4);
    pdl_launch(k_zero_many, num_sms() * 4, 256, 0, s, z, p->ctr);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    p->cur = 0;
    p->next_mode = kFull;
    p->pending = 0;
    p->bits_only = false;
    p->iterations = 0;
    p->edit_total = 0;
    return PMSZ_OK;
}

// After an aborted run the proposal array may hold stale keys.
pmsz_status restore_prop(pmsz_plan* p, cudaStream_t s) {
    CUDA_TRY(cudaMemsetAsync(p->w.prop, 0xff, p->n * sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(p->w.touched, 0, p->nwords * 4, s));
    return PMSZ_OK;
}

// K0.  sync == false leaves the validation counters on the device: the caller
// reads them with the first iteration's counters (one synchronisation less)
// and must call prep_checks() before trusting anything else.
pmsz_status prep(pmsz_plan* p, const void* f, const double* fh, double* g, cudaStream_t s, bool sync = true) {
    // K0 also runs the first detection sweep (g = fhat) unless told otherwise;
    // the fragile and detection bitmaps are cleared with the run state
    uint32_t* det = p->fuse_on ? p->w.detbits : nullptr;
    pmsz_status st = reset_run_state(p, s, p->robust_on ? p->frag : nullptr, det);
    if (st) return st;
    {
        ProfScope ps(p, s, PMSZ_K_PREP);
        p->w.frag = p->robust_on ? p->frag : nullptr;
        bool queued = false;
        const size_t nsl = p->stage_pending ? p->stage_z.size() - 1 : 0;
        if (p->qprep_on && nsl > 0) {
            // input still arriving in z-slabs: K0 over slab c once slab c and
            // the first plane of slab c + 1 (its upper halo) have landed
            for (size_t c = 0; c < nsl; ++c) {
                const size_t j = std::min(c + 1, nsl - 1);
                if (p->feed && !p->feed->wait((int)j + 1)) break;   // staged on the host: enqueued yet?
                CUDA_TRY(cudaStreamWaitEvent(s, p->stage_ev[1 + j], 0));
                queued = p->f32 ? launch_prep_q<float>(p->dom, (const float*)f, fh, g, p->w.code, p->frag_out(), p->ctr,
                                                       det, s, p->stage_z[c], p->stage_z[c + 1], false)
                                : launch_prep_q<double>(p->dom, (const double*)f, fh, g, p->w.code, p->frag_out(),
                                                        p->ctr, det, s, p->stage_z[c], p->stage_z[c + 1], false);
                if (!queued) break;   // no tensor map for this field: nothing was launched
                if (c + 1 < nsl) LAUNCHED();
            }
        } else if (p->qprep_on) {
            queued = p->f32 ? launch_prep_q<float>(p->dom, (const float*)f, fh, g, p->w.code, p->frag_out(), p->ctr, det, s)
                            : launch_prep_q<double>(p->dom, (const double*)f, fh, g, p->w.code, p->frag_out(), p->ctr, det, s);
        }
        if (nsl > 0 && p->feed && !p->feed->wait((int)nsl)) {
            p->stage_pending = false;
            if (p->feed->inexact) return fail(PMSZ_ERR_INEXACT, "original is not exactly representable in float32");
            return fail(PMSZ_ERR_CUDA, std::string("host staging: ") + cudaGetErrorString(p->feed->err));
        }
        if (nsl > 0) CUDA_TRY(cudaStreamWaitEvent(s, p->stage_ev[nsl], 0));   // every slab is in
        p->stage_pending = false;
        p->k0_detected = queued && det != nullptr;
        if (!queued) {
            if (p->f32)
                launch_prep<float>(p->dom, (const float*)f, fh, g, p->w.code, p->frag_out(), p->ctr, s);
            else
                launch_prep<double>(p->dom, (const double*)f, fh, g, p->w.code, p->frag_out(), p->ctr, s);
        }
        LAUNCHED();
    }
    CUDA_TRY(cudaGetLastError());
    p->prepared = true;
    if (!sync) {
        p->floor_viol = p->upper_viol = 0;   // unknown until prep_checks()
        return PMSZ_OK;
    }
    st = sync_counters(p, s);
    if (st) return st;
    p->floor_viol = (int64_t)p->hctr->floor_viol;
    p->upper_viol = (int64_t)p->hctr->upper_viol;
    return PMSZ_OK;
}

// The K0 verdicts from the (already synchronised) host counters.
pmsz_status prep_checks(pmsz_plan* p) {
    p->floor_viol = (int64_t)p->hctr->floor_viol;
    p->upper_viol = (int64_t)p->hctr->upper_viol;
    if (p->hctr->nonfinite) return fail(PMSZ_ERR_NONFINITE, "field values must all be finite");
    if (p->hctr->bound_viol) return fail(PMSZ_ERR_BOUND, "error bound violated");
    return PMSZ_OK;
}

pmsz_status verify_sweep(pmsz_plan* p, const double* g, cudaStream_t s, int64_t kinds[6]) {
    CUDA_TRY(cudaMemsetAsync(&p->ctr->kinds[0], 0, sizeof(p->ctr->kinds), s));
    const Dom& d = p->dom;
    const int64_t cx = d.hi[0] - d.lo[0], cy = d.hi[1] - d.lo[1], cz = d.hi[2] - d.lo[2];
    if (cx > 0 && cy > 0 && cz > 0) {
        ProfScope ps(p, s, PMSZ_K_VERIFY);
        if (!(p->qsweep_on && launch_sweep_q<true>(d, g, p->w, s))) launch_sweep_full<true>(d, g, p->w, s);
        LAUNCHED();
    }
    CUDA_TRY(cudaGetLastError());
    pmsz_status st = sync_counters(p, s);
    if (st) return st;
    for (int k = 0; k < 6; ++k) kinds[k] = (int64_t)p->hctr->kinds[k];
    return PMSZ_OK;
}

pmsz_status count_bounds(pmsz_plan* p, const void* f, const double* g, cudaStream_t s, int64_t* out) {
    CUDA_TRY(cudaMemsetAsync(&p->ctr->scratch[1], 0, sizeof(unsigned long long), s));
    ProfScope* ps = new ProfScope(p, s, PMSZ_K_OTHER);
    if (p->f32)
        k_bounds<float><<<grid_for(p->n, 256), 256, 0, s>>>(p->n, (const float*)f, g, p->dom.xi, &p->ctr->scratch[1]);
    else
        k_bounds<double><<<grid_for(p->n, 256), 256, 0, s>>>(p->n, (const double*)f, g, p->dom.xi, &p->ctr->scratch[1]);
    delete ps;
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    pmsz_status st = sync_counters(p, s);
    if (st) return st;
    *out = (int64_t)p->hctr->scratch[1];
    return PMSZ_OK;
}

pmsz_status bits_total(pmsz_plan* p, const uint32_t* bits, cudaStream_t s, int64_t* count) {
    {
        ProfScope ps(p, s, PMSZ_K_COMPACT);
        launch_bits_total(p, bits, &p->ctr->scratch[2], s);
    }
    CUDA_TRY(cudaGetLastError());
    pmsz_status st = sync_counters(p, s);
    if (st) return st;
    *count = (int64_t)p->hctr->scratch[2];
    return PMSZ_OK;
}

pmsz_status edit_count(pmsz_plan* p, cudaStream_t s, int64_t* count) {
    if (p->edits_cached >= 0 && p->offsets_of == p->w.editbits) {   // offsets still in block_counts
        *count = p->edits_cached;
        return PMSZ_OK;
    }
    {
        ProfScope ps(p, s, PMSZ_K_COMPACT);
        launch_bits_total(p, p->w.editbits, &p->ctr->scratch[2], s);
    }
    CUDA_TRY(cudaGetLastError());
    pmsz_status st = sync_counters(p, s);
    if (st) return st;
    *count = (int64_t)p->hctr->scratch[2];
    p->edits_cached = *count;
    return PMSZ_OK;
}

// Residual detections and the edit count with one synchronisation; the edit
// bitmap's block offsets stay in block_counts for the export.
pmsz_status residual_and_edits(pmsz_plan* p, cudaStream_t s, int64_t* residual, int64_t* edits) {
    {
        ProfScope ps(p, s, PMSZ_K_COMPACT);
        launch_bits_total(p, p->w.detbits, &p->ctr->scratch[1], s);
        launch_bits_total(p, p->w.editbits, &p->ctr->scratch[2], s);
    }
    CUDA_TRY(cudaGetLastError());
    pmsz_status st = sync_counters(p, s);
    if (st) return st;
    *residual = (int64_t)p->hctr->scratch[1];
    *edits = (int64_t)p->hctr->scratch[2];
    p->edits_cached = *edits;
    return PMSZ_OK;
}

void fill_result(pmsz_plan* p, pmsz_result* r) {
    if (!r) return;
    r->bound_violations = (int64_t)p->hctr->bound_viol;
    r->bound_first_index = (int64_t)p->hctr->bound_first;
    r->floor_violations = p->floor_viol;
    r->nonfinite = (int64_t)p->hctr->nonfinite;
    r->fragile = p->robust_on ? (int64_t)p->hctr->nfragile : p->n;
    r->max_vertex_edits = (int64_t)p->hctr->maxcount;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* pmsz_last_error(void) { return g_last_error.c_str(); }
const char* pmsz_version(void) { return "pmsz-b200 0.1.0 (sm_100a)"; }
int64_t pmsz_launch_count(void) { return (int64_t)g_launches.load(); }

pmsz_status pmsz_plan_create(const pmsz_desc* desc, pmsz_plan** out) {
    if (!desc || !out) return fail(PMSZ_ERR_INVALID, "null argument");
    *out = nullptr;
    const pmsz_desc& d = *desc;
    if (d.nx < 1 || d.ny < 1 || d.nz < 1) return fail(PMSZ_ERR_INVALID, "dims must be positive");
    const int64_t n = d.nx * d.ny * d.nz;
    if (n >= (int64_t)0xffffffffll) return fail(PMSZ_ERR_INVALID, "domain too large for 32-bit ids");
    if (!(d.xi > 0) || !(d.tau > 0) || !(d.tau < 2 * d.xi))
        return fail(PMSZ_ERR_INVALID, "need xi > 0 and 0 < tau < 2 xi");
    const int64_t ext[3] = {d.nx, d.ny, d.nz};
    for (int a = 0; a < 3; ++a)
        if (d.core_lo[a] < 0 || d.core_hi[a] > ext[a] || d.core_lo[a] > d.core_hi[a])
            return fail(PMSZ_ERR_INVALID, "core box outside the domain");
    pmsz_plan* p = new pmsz_plan();
    p->desc = d;
    p->dom = make_dom(d);
    p->n = n;
    p->nwords = (n + 31) / 32;
    p->f32 = (d.flags & PMSZ_FLAG_F32_ORIGINAL) ? 1 : 0;
    p->w.incremental = (d.flags & PMSZ_FLAG_INCREMENTAL) ? 1 : 0;
    // a vertex is edited at most once per iteration: u16 counts hold any run of <= 65535 iterations
    p->w.counts32 = d.max_iterations > 65535 ? 1 : 0;
    if (d.flags & PMSZ_FLAG_LOWER) p->f32 = 0;   // the iteration operand is the f64 lower bound
    const int64_t ncore = (d.core_hi[0] - d.core_lo[0]) * (d.core_hi[1] - d.core_lo[1]) *
                          (d.core_hi[2] - d.core_lo[2]);
    p->w.act_cap = (unsigned long long)std::max<int64_t>(ncore / 4, 4096);
    // explicit dirty lists while their ring entries stay below ~6% of the core
    // box (gathers beat a tiled sweep there); larger dirty sets go through the
    // edit bitmap: a masked tiled sweep, or a plain full sweep when the dirty
    // set is so spread that every warp-step would be dirty anyway
    p->w.mark_limit = (unsigned long long)std::max<int64_t>(ncore / 16, 4096);
    p->ncore = ncore;
    p->w.nwords = p->nwords;
    {
        int k = 0;
        p->ring_delta.d[k++] = 0;
        for (int r = 0; r < 14; ++r) p->ring_delta.d[k++] = rank_off(p->dom, r);
    }
    p->ch = make_chunks(p->nwords, num_sms());
    auto alloc = [&](void** ptr, size_t bytes) -> bool {
        if (cudaMalloc(ptr, bytes) != cudaSuccess) return false;
        p->scratch_bytes += (int64_t)bytes;
        return true;
    };
    bool ok = alloc((void**)&p->w.prop, n * 8) && alloc((void**)&p->w.work, n * 4) &&
              alloc((void**)&p->w.editbits, p->nwords * 4) && alloc((void**)&p->w.counts, n * (p->w.counts32 ? 4 : 2)) &&
              alloc((void**)&p->w.touched, p->nwords * 4) && alloc((void**)&p->w.detbits, p->nwords * 4) &&
              alloc((void**)&p->w.code, n) && alloc((void**)&p->frag, p->nwords * 4) &&
              alloc((void**)&p->ctr, sizeof(DevCounters)) &&
              alloc((void**)&p->block_counts, (kMaxChunks + 1) * 8);   // + the count/scan ticket
    if (ok && p->w.incremental)
        ok = alloc((void**)&p->w.actbits, p->nwords * 4) && alloc((void**)&p->w.act[0], p->w.act_cap * 4) &&
             alloc((void**)&p->w.act[1], p->w.act_cap * 4) && alloc((void**)&p->w.iteredit, p->nwords * 4) &&
             alloc((void**)&p->w.elist, p->w.mark_limit * 4);
    // per-launch history of the device tail: a fixed chunk (the tail hands back
    // to the host after at most this many iterations), not the iteration cap
    const int64_t hist_n = std::min<int64_t>(std::max<int64_t>(d.max_iterations, 1), 4096);
    p->hist_chunk = hist_n;
    if (ok) ok = alloc((void**)&p->tail, sizeof(TailState)) && alloc((void**)&p->thist, hist_n * 8);
    if (ok) {
        unsigned long long* fl = nullptr;
        ok = cudaMallocHost((void**)&fl, 64) == cudaSuccess;
        if (ok) { *fl = 0; p->hflag = fl; }
    }
    if (ok) ok = cudaMallocHost((void**)&p->hctr, sizeof(DevCounters)) == cudaSuccess &&
                 cudaMallocHost((void**)&p->htail, sizeof(TailState)) == cudaSuccess &&
                 cudaMallocHost((void**)&p->hthist, hist_n * 8) == cudaSuccess;
    p->tail_on = (d.flags & PMSZ_FLAG_HOST_LOOP) == 0;
    // dirty lists above ~0.4 % of the core take the host-launched list sweep (4 CTAs / SM) rather than the
    // tail (1 CTA / SM): measured 3.73 -> 3.70 ms at 512^3 (ncore / 96: the first tail iteration swept 1.1 M)
    p->dense_min = std::max<int64_t>(ncore / 256, 65536);
    if (const char* e = getenv("PMSZ_SORT_MIN")) p->sort_min = atoll(e);
    if (const char* e = getenv("PMSZ_DENSE_MIN")) p->dense_min = atoll(e);
    if (const char* e = getenv("PMSZ_FULL_DIV")) p->full_div = std::max<int64_t>(1, atoll(e));
    if (const char* e = getenv("PMSZ_SWEEP")) p->gather_on = strcmp(e, "tiled") != 0;
    if (const char* e = getenv("PMSZ_ROBUST")) p->robust_on = atoi(e) != 0;
    if (d.flags & PMSZ_FLAG_NO_ROBUST) p->robust_on = false;
    if (const char* e = getenv("PMSZ_QSWEEP")) p->qsweep_on = atoi(e) != 0;
    if (const char* e = getenv("PMSZ_QPREP")) p->qprep_on = atoi(e) != 0;
    if (const char* e = getenv("PMSZ_FUSE")) p->fuse_on = atoi(e) != 0;
    if (const char* e = getenv("PMSZ_TAIL1")) p->tail1_on = atoi(e) != 0;
    // measured: the dense masked queue sweep (0.45 ms) plus the dilation (0.08 ms)
    // do not beat the plain queue sweep (0.49 ms) at 512^3, so it is opt-in
    p->qmask_ok = p->qsweep_on && p->gather_on && qsweep_masked_ok(p->dom) && getenv("PMSZ_QMASK") &&
                  atoi(getenv("PMSZ_QMASK")) != 0;
    if (cudaFuncSetAttribute(k_gather<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGatherSmem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(k_gather<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGatherSmem) !=
            cudaSuccess) {
        cudaGetLastError();
        pmsz_plan_destroy(p);
        return fail(PMSZ_ERR_CUDA, "k_gather shared memory configuration failed");
    }
    if (!ok) {
        cudaGetLastError();
        pmsz_plan_destroy(p);
        return fail(PMSZ_ERR_CUDA, "device allocation failed");
    }
    p->w.ctr = p->ctr;
    memset(p->hctr, 0, sizeof(DevCounters));
    if (cudaMemset(p->w.prop, 0xff, n * 8) != cudaSuccess || cudaMemset(p->ctr, 0, sizeof(DevCounters)) != cudaSuccess ||
        cudaMemset(p->w.touched, 0, p->nwords * 4) != cudaSuccess || cudaMemset(p->w.detbits, 0, p->nwords * 4) != cudaSuccess ||
        cudaMemset(p->block_counts, 0, (kMaxChunks + 1) * 8) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        pmsz_plan_destroy(p);
        return fail(PMSZ_ERR_CUDA, "plan initialisation failed");
    }
    *out = p;
    return PMSZ_OK;
}

void pmsz_plan_destroy(pmsz_plan* p) {
    if (!p) return;
    cudaFree(p->w.prop); cudaFree(p->w.work); cudaFree(p->w.touched); cudaFree(p->w.detbits); cudaFree(p->w.editbits); cudaFree(p->w.counts);
    cudaFree(p->w.code); cudaFree(p->frag); cudaFree(p->ctr); cudaFree(p->block_counts);
    cudaFree(p->w.actbits); cudaFree(p->w.act[0]); cudaFree(p->w.act[1]); cudaFree(p->w.iteredit);
    cudaFree(p->w.elist);
    if (p->hctr) cudaFreeHost(p->hctr);
    if (p->hflag) cudaFreeHost((void*)p->hflag);
    cudaFree(p->tail); cudaFree(p->thist);
    if (p->htail) cudaFreeHost(p->htail);
    if (p->hthist) cudaFreeHost(p->hthist);
    cudaFree(p->stage_f); cudaFree(p->stage_g); cudaFree(p->stage_ids); cudaFree(p->stage_vals);
    for (cudaEvent_t e : p->stage_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : p->rec_ev) cudaEventDestroy(e);
    cudaFree(p->dsig);
    if (p->d2h_stream) cudaStreamDestroy(p->d2h_stream);
    if (p->d2h_done) cudaEventDestroy(p->d2h_done);
    if (p->hrec_ids) cudaFreeHost(p->hrec_ids);
    if (p->hrec_vals) cudaFreeHost(p->hrec_vals);
    if (p->hring) cudaFreeHost(p->hring);
    for (cudaEvent_t e : p->hring_ev) cudaEventDestroy(e);
    if (p->hsig) cudaFreeHost(p->hsig);
    if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
    for (cudaEvent_t e : p->prof_ev) cudaEventDestroy(e);
    delete p;
}

pmsz_status pmsz_profile(pmsz_plan* p, int32_t enable) {
    if (!p) return fail(PMSZ_ERR_INVALID, "null plan");
    p->prof_on = enable != 0;
    p->prof_light = enable == PMSZ_PROFILE_FULL_DOMAIN;
    return PMSZ_OK;
}

pmsz_status pmsz_profile_read(pmsz_plan* p, double* ms, int64_t* launches, int32_t reset) {
    if (!p) return fail(PMSZ_ERR_INVALID, "null plan");
    if (!p->prof_cls.empty()) {
        CUDA_TRY(cudaEventSynchronize(p->prof_ev[2 * (p->prof_cls.size() - 1) + 1]));
        prof_flush(p);
    }
    for (int k = 0; k < PMSZ_K_COUNT; ++k) {
        if (ms) ms[k] = p->prof_ms[k];
        if (launches) launches[k] = p->prof_n[k];
        if (reset) { p->prof_ms[k] = 0; p->prof_n[k] = 0; }
    }
    return PMSZ_OK;
}

int64_t pmsz_plan_scratch_bytes(const pmsz_plan* p) { return p ? p->scratch_bytes : 0; }

pmsz_status pmsz_prepare(pmsz_plan* p, const void* f, const double* fh, double* g, pmsz_result* r, void* stream) {
    if (!p || !f || !fh || !g) return fail(PMSZ_ERR_INVALID, "null argument");
    cudaStream_t s = S(stream);
    pmsz_status st = prep(p, f, fh, g, s);
    if (st) return st;
    fill_result(p, r);
    if (p->hctr->nonfinite) return fail(PMSZ_ERR_NONFINITE, "field values must all be finite");
    if (p->hctr->bound_viol) return fail(PMSZ_ERR_BOUND, "error bound violated");
    return PMSZ_OK;
}

static pmsz_status flush_deferred_marks(pmsz_plan* p, cudaStream_t s);

pmsz_status pmsz_iterate(pmsz_plan* p, const void* f, double* g, uint8_t* edited_mask, pmsz_result* r,
                         void* stream) {
    if (!p || !p->prepared) return fail(PMSZ_ERR_INVALID, "plan not prepared");
    cudaStream_t s = S(stream);
    {
        const pmsz_status st0 = flush_deferred_marks(p, s);
        if (st0) return st0;
    }
    p->w.edited_mask = edited_mask;
    if (edited_mask) CUDA_TRY(cudaMemsetAsync(edited_mask, 0, p->n, s));
    pmsz_status st = iterate_once(p, f, g, s);
    p->w.edited_mask = nullptr;
    if (st) { restore_prop(p, s); return st; }
    if (p->floor_viol > 0 && p->hctr->ndetect > 0) {
        restore_prop(p, s);
        return fail(PMSZ_ERR_MONOTONE, "edit raised a value; monotonicity broken");
    }
    ++p->iterations;
    p->edit_total += (int64_t)p->hctr->nedits;
    if (r) {
        fill_result(p, r);
        r->last_edits = (int64_t)p->hctr->nedits;
        r->last_detections = (int64_t)p->hctr->ndetect;
        r->shared_dirty = (int64_t)p->hctr->shared_dirty;
        r->iterations = p->iterations;
        r->edit_count = p->edit_total;
        if (p->last_mode == kFull) ++r->full_sweeps;
        else if (p->last_mode == kMasked || p->last_mode == kMaskedList || p->last_mode == kMaskedQ) ++r->masked_sweeps;
        else ++r->sparse_sweeps;
    }
    return PMSZ_OK;
}

pmsz_status pmsz_block_round(pmsz_plan* p, const void* f, double* g, int32_t lockstep, int64_t* round_edits,
                             pmsz_result* r, void* stream) {
    if (!p || !p->prepared) return fail(PMSZ_ERR_INVALID, "plan not prepared");
    {
        const pmsz_status st0 = flush_deferred_marks(p, S(stream));
        if (st0) return st0;
    }
    int64_t total = 0;
    bool dirty = false;
    for (int64_t it = 0; it < p->desc.max_iterations; ++it) {
        if (!lockstep && tail_ok(p)) {
            int64_t k = 0;
            bool sh = false;
            pmsz_status st = tail_step(p, f, g, S(stream), std::min(p->desc.max_iterations - it, p->hist_chunk), &k, &sh);
            if (st) { restore_prop(p, S(stream)); return st; }
            tail_result(p, r, k);
            for (int64_t i = 0; i < k; ++i) total += (int64_t)p->hthist[i];
            dirty = dirty || sh;
            it += k - 1;
            if (p->htail->last_edits == 0) {
                if (round_edits) *round_edits = total;
                if (r) r->shared_dirty = dirty;
                return PMSZ_OK;
            }
            continue;
        }
        pmsz_status st = pmsz_iterate(p, f, g, nullptr, r, stream);
        if (st) return st;
        const int64_t e = (int64_t)p->hctr->nedits;
        total += e;
        dirty = dirty || p->hctr->shared_dirty;
        if (lockstep || e == 0) {
            if (round_edits) *round_edits = total;
            if (r) r->shared_dirty = dirty;
            return PMSZ_OK;
        }
    }
    return fail(PMSZ_ERR_CONVERGENCE, "block found no zero-edit iteration within the cap");
}

// Something may change g before the first iteration: K0's detections are stale.
static void drop_k0(pmsz_plan* p, cudaStream_t) { p->k0_detected = false; }

pmsz_status pmsz_mark_all_dirty(pmsz_plan* p, void* stream) {
    if (!p) return fail(PMSZ_ERR_INVALID, "null plan");
    drop_k0(p, S(stream));   // g may change before the first iteration: K0's detections are stale
    p->next_mode = kFull;
    return PMSZ_OK;
}

// After marking outside an iteration: refresh the pending list length, or
// fall back to a full sweep when the list overflowed.
static pmsz_status after_mark(pmsz_plan* p, cudaStream_t s) {
    p->mark_deferred = false;
    CUDA_TRY(cudaGetLastError());
    pmsz_status st = sync_counters(p, s);
    if (st) return st;
    if (p->next_mode == kList || p->next_mode == kMaskedList) {
        const int64_t nact = (int64_t)p->hctr->nact[p->cur];
        if (p->bits_only) {
            p->pending += nact;   // still a bound; the list is rebuilt from actbits
        } else if (nact > (int64_t)p->w.act_cap) {
            p->next_mode = kFull;
        } else {
            p->pending = nact;
            if (p->gather_on && nact > p->dense_min) p->next_mode = kMaskedList;
        }
    }
    return PMSZ_OK;
}

pmsz_status pmsz_mark_dirty_ids(pmsz_plan* p, const uint32_t* ids, int64_t count, void* stream) {
    if (!p) return fail(PMSZ_ERR_INVALID, "null plan");
    drop_k0(p, S(stream));   // g may change before the first iteration: K0's detections are stale
    if (!p->w.incremental || p->next_mode == kFull || count <= 0) return PMSZ_OK;
    cudaStream_t s = S(stream);
    pdl_launch(k_mark_ids, grid_for(count, 256), 256, 0, s, p->dom, p->w, ids, count, p->cur,
               p->next_mode == kMasked || p->next_mode == kMaskedQ);
    LAUNCHED();
    return after_mark(p, s);
}

pmsz_status pmsz_box_mark_changed(pmsz_plan* p, const int64_t lo[3], const int64_t hi[3], const double* before,
                                  const double* g, void* stream) {
    if (!p) return fail(PMSZ_ERR_INVALID, "null plan");
    drop_k0(p, S(stream));   // g may change before the first iteration: K0's detections are stale
    if (!p->w.incremental || p->next_mode == kFull) return PMSZ_OK;
    cudaStream_t s = S(stream);
    Box b{p->dom.nx, p->dom.ny, {lo[0], lo[1], lo[2]}, {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]}, 0, 0};
    b.mxy = div_magic((uint64_t)(b.ext[0] * b.ext[1]));
    b.mx = div_magic((uint64_t)b.ext[0]);
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    if (n <= 0) return PMSZ_OK;
    pdl_launch(k_box_mark, grid_for(n, 256), 256, 0, s, p->dom, p->w, b, before, g, p->cur,
               p->next_mode == kMasked || p->next_mode == kMaskedQ);
    LAUNCHED();
    return after_mark(p, s);
}

static bool make_box(int64_t nx, int64_t ny, int64_t nz, const int64_t lo[3], const int64_t hi[3], Box& b);

static pmsz_status flush_deferred_marks(pmsz_plan* p, cudaStream_t s) {
    return p->mark_deferred ? after_mark(p, s) : PMSZ_OK;
}

pmsz_status pmsz_box_merge_min(pmsz_plan* p, double* g, const int64_t lo[3], const int64_t hi[3], const double* buf,
                               int64_t* changed_out, void* stream) {
    if (!p || !g || !buf) return fail(PMSZ_ERR_INVALID, "null argument");
    drop_k0(p, S(stream));   // g may change before the first iteration: K0's detections are stale
    cudaStream_t s = S(stream);
    Box b;
    if (!make_box(p->dom.nx, p->dom.ny, p->dom.nz, lo, hi, b)) return fail(PMSZ_ERR_INVALID, "box outside the domain");
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    CUDA_TRY(cudaMemsetAsync(&p->ctr->changed, 0, sizeof(unsigned long long), s));
    if (n > 0) {
        const int mode = !p->w.incremental ? 0
                         : ((p->next_mode == kMasked || p->next_mode == kMaskedQ) ? 1
                            : ((p->next_mode == kList || p->next_mode == kMaskedList) ? 2 : 0));
        ProfScope ps(p, s, PMSZ_K_OTHER);
        pdl_launch(k_box_merge, grid_for(n, 256), 256, 0, s, p->dom, p->w, b, g, buf, p->cur, mode, &p->ctr->changed);
        LAUNCHED();
    }
    if (!changed_out) {   // the counters are read at the next iteration
        CUDA_TRY(cudaGetLastError());
        p->mark_deferred = true;
        return PMSZ_OK;
    }
    pmsz_status st = after_mark(p, s);
    if (st) return st;
    *changed_out = (int64_t)p->hctr->changed;
    return PMSZ_OK;
}

// One epoch of the cross-rank barrier; the four sums land in p->hsig.
static pmsz_status rounds_signal(pmsz_plan* p, pmsz_rounds_desc* rd, const unsigned long long v[4], cudaStream_t s) {
    SigArgs a{};
    for (int r = 0; r < rd->world; ++r) {
        a.sums[r] = (unsigned long long*)rd->bufs[r] + rd->sums_off;
        a.flags[r] = (unsigned long long*)rd->bufs[r] + rd->flags_off;
    }
    for (int k = 0; k < 4; ++k) a.v[k] = v[k];
    a.epoch = ++rd->epoch;
    a.world = rd->world;
    a.rank = rd->rank;
    if (sync_by_kernel() && p->hflag) {   // sums straight into the pinned mirror, then the flag
        a.out = p->hsig;
        a.flag = p->hflag;
        a.seq = ++p->sync_seq;
        pdl_launch(k_signal, 1, PMSZ_MAX_RANKS, 0, s, a);
        LAUNCHED();
        return spin_flag(p, s, a.seq);
    }
    a.out = p->dsig;
    k_signal<<<1, PMSZ_MAX_RANKS, 0, s>>>(a);
    LAUNCHED();
    CUDA_TRY(cudaMemcpyAsync(p->hsig, p->dsig, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return PMSZ_OK;
}

pmsz_status pmsz_rounds(pmsz_plan* p, const void* f, double* g, pmsz_rounds_desc* rd, int64_t* rounds_out,
                        int64_t* syncs_out, int64_t* totals, int64_t totals_cap, pmsz_result* r, void* stream) {
    if (!p || !f || !g || !rd) return fail(PMSZ_ERR_INVALID, "null argument");
    if (rd->world < 1 || rd->world > PMSZ_MAX_RANKS || rd->rank < 0 || rd->rank >= rd->world ||
        rd->nex < 0 || rd->nex > PMSZ_MAX_EXCHANGES)
        return fail(PMSZ_ERR_INVALID, "bad rounds descriptor");
    cudaStream_t s = S(stream);
    if (!p->dsig) {
        CUDA_TRY(cudaMalloc((void**)&p->dsig, 4 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMallocHost((void**)&p->hsig, 4 * sizeof(unsigned long long)));
    }
    Box boxes[PMSZ_MAX_EXCHANGES];
    for (int e = 0; e < rd->nex; ++e)
        if (!make_box(p->dom.nx, p->dom.ny, p->dom.nz, rd->ex_lo[e], rd->ex_hi[e], boxes[e]))
            return fail(PMSZ_ERR_INVALID, "exchange box outside the domain");
    const bool lockstep = rd->lockstep != 0;
    int64_t nr = 0, ns = 0;
    pmsz_result rr{};
    for (;;) {
        if (nr >= rd->cap) return fail(PMSZ_ERR_CONVERGENCE, "no terminal round within the cap");
        ++nr;
        int64_t e = 0;
        memset(&rr, 0, sizeof(rr));
        pmsz_status st = pmsz_block_round(p, f, g, rd->lockstep, &e, &rr, stream);
        if (st) return st;
        // this round's replicas into the parity area of the round
        const int64_t area = (int64_t)(++rd->rounds_total & 1) * rd->repl_doubles;
        double* mine = (double*)rd->bufs[rd->rank] + area;
        for (int x = 0; x < rd->nex; ++x) {
            const Box& b = boxes[x];
            const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
            if (n == 0) continue;
            pdl_launch(k_box_pack, grid_for(n, 256), 256, 0, s, b, (const double*)g, mine + rd->ex_off[x]);
            LAUNCHED();
        }
        const unsigned long long v[4] = {(unsigned long long)e, rr.shared_dirty ? 1ull : 0ull, 0ull, 0ull};
        st = rounds_signal(p, rd, v, s);
        if (st) return st;
        const int64_t round_edits = (int64_t)p->hsig[0];
        const bool any_dirty = p->hsig[1] != 0;
        if (totals && nr - 1 < totals_cap) totals[nr - 1] = round_edits;
        if (!lockstep && (round_edits == 0 || !any_dirty)) break;   // parallel.py:304-314
        // _merge_min (parallel.py:122-140) pairwise over the full overlaps
        int64_t changed = 0;
        for (int x = 0; x < rd->nex; ++x) {
            const double* theirs = (const double*)rd->bufs[rd->ex_peer[x]] + area + rd->ex_peer_off[x];
            int64_t c = 0;
            st = pmsz_box_merge_min(p, g, rd->ex_lo[x], rd->ex_hi[x], theirs, lockstep ? &c : nullptr, stream);
            if (st) return st;
            changed += c;
        }
        ++ns;
        if (lockstep) {   // parallel.py:321-322
            const unsigned long long w[4] = {(unsigned long long)changed, 0ull, 0ull, 0ull};
            st = rounds_signal(p, rd, w, s);
            if (st) return st;
            if (round_edits == 0 && p->hsig[0] == 0) break;
        }
    }
    if (rounds_out) *rounds_out = nr;
    if (syncs_out) *syncs_out = ns;
    if (r) *r = rr;
    return PMSZ_OK;
}

pmsz_status pmsz_residual(pmsz_plan* p, int64_t* count_out, void* stream) {
    if (!p || !count_out) return fail(PMSZ_ERR_INVALID, "null argument");
    return bits_total(p, p->w.detbits, S(stream), count_out);
}

pmsz_status pmsz_verify(pmsz_plan* p, const double* g, pmsz_result* r, void* stream) {
    if (!p || !p->prepared) return fail(PMSZ_ERR_INVALID, "plan not prepared");
    int64_t kinds[6];
    pmsz_status st = verify_sweep(p, g, S(stream), kinds);
    if (st) return st;
    if (r) {
        for (int k = 0; k < 6; ++k) r->residual[k] = kinds[k];
        ++r->full_sweeps;
    }
    return PMSZ_OK;
}

pmsz_status pmsz_floor_violations(pmsz_plan* p, const double* lower, const double* g, int64_t* out, void* stream) {
    if (!p || !lower || !g || !out) return fail(PMSZ_ERR_INVALID, "null argument");
    cudaStream_t s = S(stream);
    CUDA_TRY(cudaMemsetAsync(&p->ctr->scratch[1], 0, sizeof(unsigned long long), s));
    k_below<<<grid_for(p->n, 256), 256, 0, s>>>(p->n, lower, g, &p->ctr->scratch[1]);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    pmsz_status st = sync_counters(p, s);
    if (st) return st;
    *out = (int64_t)p->hctr->scratch[1];
    p->floor_viol = *out;   // arms the monotonicity check of pmsz_iterate (correction.py:240-241)
    return PMSZ_OK;
}

pmsz_status pmsz_history(const pmsz_plan* p, int64_t* out, int64_t cap, int64_t* count) {
    if (!p || !count) return fail(PMSZ_ERR_INVALID, "null argument");
    *count = (int64_t)p->hist_all.size();
    for (int64_t i = 0; out && i < cap && i < *count; ++i) out[i] = p->hist_all[i];
    return PMSZ_OK;
}

pmsz_status pmsz_bounds_violations(pmsz_plan* p, const void* f, const double* g, int64_t* out, void* stream) {
    if (!p || !out) return fail(PMSZ_ERR_INVALID, "null argument");
    return count_bounds(p, f, g, S(stream), out);
}

pmsz_status pmsz_run_correction(pmsz_plan* p, const void* f, const double* fh, double* g, int64_t* history,
                                int64_t history_cap, pmsz_result* r, void* stream) {
    if (!p || !f || !fh || !g) return fail(PMSZ_ERR_INVALID, "null argument");
    cudaStream_t s = S(stream);
    pmsz_result local{};
    if (!r) r = &local;
    memset(r, 0, sizeof(*r));
    p->hist_all.clear();
    // Out of place, K0's validation is read together with the first
    // iteration's counters (g is an output buffer, so running one iteration
    // on invalid input has no visible effect beyond the error).  In place
    // (g aliases fhat) it is checked before anything is written.
    const bool deferred = g != fh && p->desc.max_iterations > 0;
    pmsz_status st = deferred ? prep(p, f, fh, g, s, false) : pmsz_prepare(p, f, fh, g, r, stream);
    if (st) return st;
    bool converged = false;
    int64_t it = 0;
    if (deferred) {
        st = pmsz_iterate(p, f, g, nullptr, r, stream);
        if (st) return st;
        fill_result(p, r);
        st = prep_checks(p);
        if (st) { restore_prop(p, s); return st; }
        if (p->floor_viol > 0 && p->hctr->ndetect > 0) {   // correction.py:240-241
            restore_prop(p, s);
            return fail(PMSZ_ERR_MONOTONE, "edit raised a value; monotonicity broken");
        }
        const int64_t e = (int64_t)p->hctr->nedits;
        p->hist_all.push_back(e);
        if (history && history_cap > 0) history[0] = e;
        it = 1;
        if (e == 0) converged = true;
    }
    for (; !converged && it < p->desc.max_iterations; ++it) {
        if (tail_ok(p)) {
            int64_t k = 0;
            bool sh = false;
            st = tail_step(p, f, g, s, std::min(p->desc.max_iterations - it, p->hist_chunk), &k, &sh, true);
            if (st) { restore_prop(p, s); return st; }
            tail_result(p, r, k);
            for (int64_t i = 0; i < k; ++i) {
                p->hist_all.push_back((int64_t)p->hthist[i]);
                if (history && it + i < history_cap) history[it + i] = (int64_t)p->hthist[i];
            }
            it += k;
            if (p->htail->last_edits == 0) { converged = true; break; }
            --it;   // the loop increment
            continue;
        }
        st = pmsz_iterate(p, f, g, nullptr, r, stream);
        if (st) return st;
        const int64_t e = (int64_t)p->hctr->nedits;
        p->hist_all.push_back(e);
        if (history && it < history_cap) history[it] = e;
        if (e == 0) { converged = true; ++it; break; }
    }
    r->iterations = it;
    fill_result(p, r);
    if (!converged) {
        r->convergence_kind = PMSZ_CONV_CAP;
        restore_prop(p, s);
        return fail(PMSZ_ERR_CONVERGENCE, "no zero-edit iteration within the iteration cap");
    }
    // bounds.admits(g) (correction.py:422-423): only vertices whose fhat was
    // outside [L, U] can fail, so the dense check runs only if K0 saw one.
    if (p->floor_viol > 0 || p->upper_viol > 0) {
        int64_t bad = 0;
        st = count_bounds(p, f, g, s, &bad);
        if (st) return st;
        if (bad) {
            r->convergence_kind = PMSZ_CONV_BOUND;
            return fail(PMSZ_ERR_CONVERGENCE, "corrected field escaped the error bound");
        }
    }
    // re-scan + _kind_masks must be empty (correction.py:424-426).  Every
    // centre's detection status at its latest evaluation is kept in detbits
    // and a centre is re-evaluated whenever a vertex of its closed 1-ring
    // changes (or by a full sweep), so the popcount equals the detections of
    // a full re-scan of the final field.  The per-kind split is only computed
    // when something survived.
    int64_t residual = 0, count = 0;
    if (p->totals_ready && p->offsets_of == p->w.editbits) {   // counted by the converging tail_step
        residual = p->pre_residual;
        count = p->pre_edits;
        p->edits_cached = count;
    } else {
        st = residual_and_edits(p, s, &residual, &count);
        if (st) return st;
    }
    p->totals_ready = false;
    if (residual) {
        st = pmsz_verify(p, g, r, stream);
        if (st) return st;
        r->convergence_kind = PMSZ_CONV_RESIDUAL;
        return fail(PMSZ_ERR_CONVERGENCE, "distortions survived a zero-edit iteration");
    }
    r->edit_count = count;
    return PMSZ_OK;
}

pmsz_status pmsz_edits_export(pmsz_plan* p, const double* g, int64_t* ids, double* vals, int64_t cap,
                              int64_t* count_out, void* stream) {
    if (!p || !g) return fail(PMSZ_ERR_INVALID, "null argument");
    cudaStream_t s = S(stream);
    int64_t count = 0;
    pmsz_status st = edit_count(p, s, &count);
    if (st) return st;
    if (count_out) *count_out = count;
    if (ids && vals && cap > 0 && count > 0) {
        ProfScope ps(p, s, PMSZ_K_COMPACT);
        pdl_launch(k_chunk_write, (unsigned)p->ch.n, kCompactThreads, 0, s, (const uint32_t*)p->w.editbits, p->ch, p->n,
                   (const unsigned long long*)p->block_counts, g, ids,
                                                                   vals, cap);
        LAUNCHED();
        CUDA_TRY(cudaGetLastError());
    }
    return PMSZ_OK;
}

pmsz_status pmsz_run_correction_export(pmsz_plan* p, const void* f, const double* fh, double* g, int64_t* history,
                                       int64_t history_cap, pmsz_result* r, int64_t* ids, double* vals, int64_t cap,
                                       void* stream) {
    pmsz_status st = pmsz_run_correction(p, f, fh, g, history, history_cap, r, stream);
    if (st) return st;
    int64_t count = 0;
    st = pmsz_edits_export(p, g, ids, vals, cap, &count, stream);
    if (st == PMSZ_OK && r) r->edit_count = count;
    return st;
}

namespace {
// Staging thread of a host run with pageable buffers (hoststage.h): per z-slab,
// the f and fhat bytes go pageable -> pinned ring slot (all pool threads) ->
// device (copy_stream), chunk by chunk, so the memcpy of chunk k + 1 overlaps
// the DMA of chunk k; a pageable corrected field is filled from the fhat chunk
// in the same pass.  stage_ev[1 + c] is recorded and published per slab for
// K0's slab launches (prep()).
void feed_slabs(pmsz_plan* p, StageFeed* fd, int dev, const char* fsrc, bool f_pin, bool narrow, const double* hsrc,
                bool h_pin, char* fdst, double* hdst, double* gfill, double* gpinned, int64_t plane) {
    cudaError_t err = cudaSetDevice(dev);
    bool inexact = false;
    HostPool& pool = HostPool::get();
    const size_t fel = p->f32 ? 4 : 8, sel = narrow ? 8 : fel;
    static const int want = [] {
        const char* e = getenv("PMSZ_STAGE_THREADS");
        return e ? atoi(e) : 0;
    }();
    static const bool trace = getenv("PMSZ_E2E_TRACE") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double t_wait = 0, t_copy = 0, t_start = trace ? now() : 0.0;
    int k = 0;
    // dbytes device bytes from src (narrow: f64 source, f32 destination)
    auto stage = [&](char* dst, const char* src, size_t dbytes, bool nar, double* fill) -> cudaError_t {
        for (size_t o = 0; o < dbytes; o += p->hring_chunk) {
            if (fd->stop.load(std::memory_order_relaxed)) return cudaSuccess;
            const size_t len = std::min(p->hring_chunk, dbytes - o);
            const int r = k++ % p->hring_n;
            double ta = trace ? now() : 0.0;
            cudaError_t e = cudaEventSynchronize(p->hring_ev[r]);   // the slot's previous DMA is done
            if (e != cudaSuccess) return e;
            double tb = trace ? now() : 0.0;
            char* pin = p->hring + (size_t)r * p->hring_chunk;
            std::atomic<bool> bad{false};
            pool.run([&](int t, int nt) {
                size_t x0, x1;
                if (fill)
                    share_at((uintptr_t)fill + o, len, t, nt, (size_t)2 << 20, &x0, &x1);
                else
                    share(len, t, nt, &x0, &x1);
                if (nar) {   // NaN and overflow fail the round trip too: the f64 plan reports them
                    if (nt_narrow((float*)(pin + x0), (const double*)src + (o + x0) / 4, (x1 - x0) / 4))
                        bad.store(true, std::memory_order_relaxed);
                } else {
                    nt_copy(pin + x0, fill ? (char*)fill + o + x0 : nullptr, src + o + x0, x1 - x0);
                }
                host_sfence();   // the streaming stores are visible before the DMA is issued
            }, want);
            if (trace) {
                const double tc = now();
                t_wait += tb - ta;
                t_copy += tc - tb;
            }
            if (bad.load()) {
                inexact = true;
                fd->mark_inexact();
                return cudaSuccess;
            }
            e = cudaMemcpyAsync(dst + o, pin, len, cudaMemcpyHostToDevice, p->copy_stream);
            if (e == cudaSuccess) e = cudaEventRecord(p->hring_ev[r], p->copy_stream);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    };
    const int64_t nsl = (int64_t)p->stage_z.size() - 1;
    for (int64_t c = 0; c < nsl && err == cudaSuccess && !inexact && !fd->stop.load(); ++c) {
        const int64_t o = p->stage_z[c] * plane, m = (p->stage_z[c + 1] - p->stage_z[c]) * plane;
        if (f_pin)
            err = cudaMemcpyAsync(fdst + o * fel, fsrc + o * fel, m * fel, cudaMemcpyHostToDevice, p->copy_stream);
        else
            err = stage(fdst + o * fel, fsrc + o * sel, m * fel, narrow, nullptr);
        if (err != cudaSuccess || inexact) break;
        if (h_pin) {
            err = cudaMemcpyAsync(hdst + o, hsrc + o, m * 8, cudaMemcpyHostToDevice, p->copy_stream);
            if (gfill) pool_memcpy(gfill + o, hsrc + o, m * 8);
        } else {
            err = stage((char*)(hdst + o), (const char*)(hsrc + o), m * 8, false, gfill ? gfill + o : nullptr);
        }
        if (err == cudaSuccess) err = cudaEventRecord(p->stage_ev[1 + c], p->copy_stream);
        if (gpinned && err == cudaSuccess) {   // pinned field out: the slab streams back (see the caller)
            err = cudaStreamWaitEvent(p->d2h_stream, p->stage_ev[1 + c], 0);
            if (err == cudaSuccess)
                err = cudaMemcpyAsync(gpinned + o, hdst + o, m * 8, cudaMemcpyDeviceToHost, p->d2h_stream);
        }
        if (err != cudaSuccess) break;
        fd->publish((int)c + 1);
    }
    if (trace)
        fprintf(stderr, "stage: %d chunks of %zu MiB, %.2f ms (slot waits %.2f, host copies %.2f), %d threads\n", k,
                p->hring_chunk >> 20, now() - t_start, t_wait, t_copy, want > 0 ? std::min(want, pool.threads()) : pool.threads());
    fd->finish(err, inexact);
}
}  // namespace

pmsz_status pmsz_run_correction_host(pmsz_plan* p, const void* f_host, const double* fh_host, double* g_host,
                                     int64_t* ids_host, double* vals_host, int64_t edits_cap, int64_t* history,
                                     int64_t history_cap, pmsz_result* r, void* stream) {
    if (!p || !f_host || !fh_host) return fail(PMSZ_ERR_INVALID, "null argument");
    cudaStream_t s = S(stream);
    const size_t fbytes = p->n * (p->f32 ? 4 : 8), gbytes = p->n * 8;
    p->hrec_count = -1;
    // device staging owned by the plan (allocated on first use, reused: a
    // per-call allocation would remap ~12 bytes/voxel of device memory)
    auto grow = [&](void** ptr, size_t bytes) -> bool {
        if (*ptr) return true;
        if (cudaMalloc(ptr, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
        p->scratch_bytes += (int64_t)bytes;
        return true;
    };
    if (!grow(&p->stage_f, fbytes) || !grow((void**)&p->stage_g, gbytes))
        return fail(PMSZ_ERR_CUDA, "staging allocation failed");
    void* f = p->stage_f;
    double* g = p->stage_g;
    pmsz_status st = PMSZ_OK;
    // Input copy in z-slabs on a second stream; K0 runs slab by slab as the
    // data lands (prep), so only the last slab's K0 is exposed.
    const int64_t nz = p->dom.nz, plane = p->dom.nx * p->dom.ny;
    const int64_t nsl = (p->n >= (int64_t)1 << 22) ? std::min<int64_t>(nz, 16) : 1;
    if (!p->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    while ((int64_t)p->stage_ev.size() < nsl + 1) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p->stage_ev.push_back(e);
    }
    p->stage_z.assign(nsl + 1, 0);
    for (int64_t c = 0; c <= nsl; ++c) p->stage_z[c] = nz * c / nsl;
    CUDA_TRY(cudaEventRecord(p->stage_ev[0], s));   // earlier work on the staging buffers is done
    CUDA_TRY(cudaStreamWaitEvent(p->copy_stream, p->stage_ev[0], 0));
    const bool narrow = p->f32 && (p->desc.flags & PMSZ_FLAG_HOST_F64);
    const bool f_pin = !narrow && host_pinned(f_host), h_pin = host_pinned(fh_host);
    const bool g_pin = g_host && host_pinned(g_host);
    double* g_fill = (g_host && !g_pin) ? g_host : nullptr;   // pageable field out: filled from fhat on the host
    std::thread feeder;
    if (f_pin && h_pin && !g_fill) {
        const size_t fel = p->f32 ? 4 : 8;
        for (int64_t c = 0; c < nsl; ++c) {
            const int64_t o = p->stage_z[c] * plane, m = (p->stage_z[c + 1] - p->stage_z[c]) * plane;
            CUDA_TRY(cudaMemcpyAsync((char*)f + o * fel, (const char*)f_host + o * fel, m * fel, cudaMemcpyHostToDevice,
                                     p->copy_stream));
            CUDA_TRY(cudaMemcpyAsync(g + o, fh_host + o, m * 8, cudaMemcpyHostToDevice, p->copy_stream));
            CUDA_TRY(cudaEventRecord(p->stage_ev[1 + c], p->copy_stream));
        }
    } else {
        if (!f_pin || !h_pin) {
            static const size_t chunk = [] {
                const char* e = getenv("PMSZ_STAGE_CHUNK_MB");
                const long mb = e ? atol(e) : 32;
                return (size_t)std::max(1L, std::min(256L, mb)) << 20;
            }();
            if (p->hring_chunk != chunk) {
                if (p->hring) cudaFreeHost(p->hring);
                p->hring = nullptr;
                p->hring_chunk = 0;
                p->hring_n = 4;
                CUDA_TRY(cudaMallocHost((void**)&p->hring, chunk * p->hring_n));
                p->hring_chunk = chunk;
            }
            while ((int)p->hring_ev.size() < p->hring_n) {
                cudaEvent_t e;
                CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                p->hring_ev.push_back(e);
            }
        }
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        if (g_pin && !p->d2h_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->d2h_stream, cudaStreamNonBlocking));
        try {   // (no exception may cross the C ABI)
            p->feed = new StageFeed();
            feeder = std::thread(feed_slabs, p, p->feed, dev, (const char*)f_host, f_pin, narrow, fh_host, h_pin, (char*)f,
                                 g, g_fill, g_pin ? g_host : nullptr, plane);
        } catch (const std::exception& e) {
            delete p->feed;
            p->feed = nullptr;
            return fail(PMSZ_ERR_CUDA, std::string("host staging thread: ") + e.what());
        }
    }
    // Pinned field out: g equals fhat except at the edits, so the host copy
    // is streamed back slab by slab as soon as each fhat slab has landed --
    // the device-to-host direction of the link runs concurrently with the
    // host-to-device slabs -- and is patched with the edit record at the end.
    // (A slab may be read while the loop already edits it: every such vertex
    // is in the edit record and gets its final value from the patch.)
    auto finish_feed = [&]() -> pmsz_status {
        if (!feeder.joinable()) return PMSZ_OK;
        p->feed->stop = true;   // a run that failed early stops the staging
        feeder.join();
        const cudaError_t e = p->feed->err;
        delete p->feed;
        p->feed = nullptr;
        if (e != cudaSuccess) return fail(PMSZ_ERR_CUDA, std::string("host staging: ") + cudaGetErrorString(e));
        return PMSZ_OK;
    };
    if (g_pin) {
        if (!p->d2h_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->d2h_stream, cudaStreamNonBlocking));
        if (!p->d2h_done) CUDA_TRY(cudaEventCreateWithFlags(&p->d2h_done, cudaEventDisableTiming));
        for (int64_t c = 0; c < nsl && !feeder.joinable(); ++c) {   // (with a staging thread it issues these)
            const int64_t o = p->stage_z[c] * plane, m = (p->stage_z[c + 1] - p->stage_z[c]) * plane;
            CUDA_TRY(cudaStreamWaitEvent(p->d2h_stream, p->stage_ev[1 + c], 0));
            CUDA_TRY(cudaMemcpyAsync(g_host + o, g + o, m * 8, cudaMemcpyDeviceToHost, p->d2h_stream));
        }
    }
    static const bool etrace = getenv("PMSZ_E2E_TRACE") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double t0 = etrace ? now() : 0.0, t1 = 0, t2 = 0, t3 = 0;
    p->stage_pending = true;
    st = pmsz_run_correction(p, f, g, g, history, history_cap, r, stream);
    p->stage_pending = false;
    {
        const pmsz_status fs = finish_feed();
        if (st == PMSZ_OK) st = fs;
    }
    if (etrace) t1 = now();
    CUDA_TRY(cudaStreamWaitEvent(s, p->stage_ev[nsl], 0));   // (already waited by K0 unless it failed early)
    if (g_pin) {
        CUDA_TRY(cudaEventRecord(p->d2h_done, p->d2h_stream));
        CUDA_TRY(cudaStreamWaitEvent(s, p->d2h_done, 0));
    }
    if (etrace) {
        cudaStreamSynchronize(s);
        t2 = now();
    }
    if (st == PMSZ_OK && r && r->edit_count == 0) p->hrec_count = 0;
    if (st == PMSZ_OK && r && r->edit_count > 0 && (g_host || (ids_host && vals_host && edits_cap > 0))) {
        const int64_t count = r->edit_count;
        // the whole record when the field is patched from it, else what fits the caller's buffers
        const int64_t m = g_host ? count : std::min(edits_cap, count);
        if (m > p->stage_cap) {
            cudaFree(p->stage_ids);
            cudaFree(p->stage_vals);
            p->stage_ids = nullptr;
            p->stage_vals = nullptr;
            p->scratch_bytes -= p->stage_cap * 16;
            p->stage_cap = 0;
            const int64_t want = std::min<int64_t>(p->n, std::max<int64_t>(m, m + m / 4));
            if (!grow((void**)&p->stage_ids, want * 8) || !grow((void**)&p->stage_vals, want * 8))
                return fail(PMSZ_ERR_CUDA, "staging allocation failed");
            p->stage_cap = want;
        }
        st = pmsz_edits_export(p, g, p->stage_ids, p->stage_vals, m, nullptr, stream);
        if (st == PMSZ_OK) {
            // host destination of the full record: the caller's buffers when they
            // are pinned and hold it, else the plan's pinned bounce buffers
            const bool direct = ids_host && vals_host && edits_cap >= m && host_pinned(ids_host) && host_pinned(vals_host);
            int64_t* hid = ids_host;
            double* hval = vals_host;
            if (!direct) {
                if (p->hrec_cap < m) {
                    if (p->hrec_ids) cudaFreeHost(p->hrec_ids);
                    if (p->hrec_vals) cudaFreeHost(p->hrec_vals);
                    p->hrec_ids = nullptr;
                    p->hrec_vals = nullptr;
                    p->hrec_cap = 0;
                    CUDA_TRY(cudaMallocHost((void**)&p->hrec_ids, m * 8));
                    CUDA_TRY(cudaMallocHost((void**)&p->hrec_vals, m * 8));
                    p->hrec_cap = m;
                }
                hid = p->hrec_ids;
                hval = p->hrec_vals;
            }
            // the record comes back in a few chunks; the host patches chunk c of
            // the field while chunk c + 1 is still on the link
            const int nch = g_host ? (int)std::min<int64_t>(8, std::max<int64_t>(1, m >> 18)) : 1;
            while ((int)p->rec_ev.size() < nch) {
                cudaEvent_t e;
                CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                p->rec_ev.push_back(e);
            }
            for (int c = 0; c < nch; ++c) {
                const int64_t a = m * c / nch, b = m * (c + 1) / nch;
                CUDA_TRY(cudaMemcpyAsync(hid + a, p->stage_ids + a, (b - a) * 8, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaMemcpyAsync(hval + a, p->stage_vals + a, (b - a) * 8, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaEventRecord(p->rec_ev[c], s));
            }
            if (etrace) t3 = now();
            if (g_host) {
                patch_host(g_host, hid, hval, m, p->rec_ev.data(), nch);
            } else {
                CUDA_TRY(cudaEventSynchronize(p->rec_ev[nch - 1]));
            }
            if (!direct) {
                if (m == count) p->hrec_count = m;
                if (ids_host && vals_host && edits_cap > 0) {
                    const int64_t k = std::min(edits_cap, count);
                    pool_memcpy(ids_host, hid, k * 8);
                    pool_memcpy(vals_host, hval, k * 8);
                }
            }
        }
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    if (etrace)
        fprintf(stderr, "e2e: run %.2f ms, d2h field wait %.2f, export %.2f, record + patch + copy-out %.2f (total %.2f)\n", t1 - t0,
                t2 - t1, t3 - t2, now() - t3, now() - t0);
    return st;
}

pmsz_status pmsz_edits_host(pmsz_plan* p, int64_t* ids_host, double* vals_host, int64_t cap, int64_t* count_out) {
    if (!p) return fail(PMSZ_ERR_INVALID, "null argument");
    if (p->hrec_count < 0) return fail(PMSZ_ERR_INVALID, "the plan holds no edit record (see pmsz_run_correction_host)");
    if (count_out) *count_out = p->hrec_count;
    const int64_t k = std::min(cap, p->hrec_count);
    if (k > 0 && ids_host && vals_host) {
        pool_memcpy(ids_host, p->hrec_ids, k * 8);
        pool_memcpy(vals_host, p->hrec_vals, k * 8);
    }
    return PMSZ_OK;
}

// ---- host <-> device copies of pageable arrays ----------------------------
// The staging of pmsz_run_correction_host as a plain copy (the block-parallel
// drop-in, local_converge, ... move whole host fields too): one process-wide
// pinned ring, pool threads on the host side, streaming stores.
namespace {
struct CopyRing {
    std::mutex m;   // one copy at a time
    char* buf = nullptr;
    size_t chunk = 0;
    int n = 0;
    std::vector<cudaEvent_t> ev;
    cudaStream_t st = nullptr;
    int dev = -1;
};
CopyRing& copy_ring() {
    static CopyRing* r = new CopyRing();
    return *r;
}
// (under r.m) the ring on the current device
cudaError_t copy_ring_ready(CopyRing& r) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (r.buf && r.dev == dev) return cudaSuccess;
    if (r.buf) {   // another device: rebuild (events and streams belong to a device)
        cudaFreeHost(r.buf);
        for (cudaEvent_t x : r.ev) cudaEventDestroy(x);
        r.ev.clear();
        if (r.st) cudaStreamDestroy(r.st);
        r.buf = nullptr;
        r.st = nullptr;
    }
    r.chunk = (size_t)32 << 20;
    r.n = 4;
    if ((e = cudaMallocHost((void**)&r.buf, r.chunk * r.n)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking)) != cudaSuccess) return e;
    for (int i = 0; i < r.n; ++i) {
        cudaEvent_t x;
        if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
        r.ev.push_back(x);
    }
    r.dev = dev;
    return cudaSuccess;
}
}  // namespace

pmsz_status pmsz_host_to_device(void* dst_dev, const void* src_host, int64_t n, int32_t narrow_f64, int64_t* inexact,
                                void* stream) {
    if (inexact) *inexact = 0;
    if (n < 0 || (n > 0 && (!dst_dev || !src_host))) return fail(PMSZ_ERR_INVALID, "bad arguments");
    if (n == 0) return PMSZ_OK;
    cudaStream_t s = S(stream);
    const size_t dbytes = (size_t)n * (narrow_f64 ? 4 : 1);
    if (!narrow_f64 && host_pinned(src_host)) {
        CUDA_TRY(cudaMemcpyAsync(dst_dev, src_host, dbytes, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return PMSZ_OK;
    }
    CopyRing& r = copy_ring();
    std::lock_guard<std::mutex> lk(r.m);
    CUDA_TRY(copy_ring_ready(r));
    cudaEvent_t start;
    CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(start, s));                 // earlier work on dst is ordered first
    CUDA_TRY(cudaStreamWaitEvent(r.st, start, 0));
    cudaEventDestroy(start);
    HostPool& pool = HostPool::get();
    bool bad = false;
    int k = 0;
    for (size_t o = 0; o < dbytes && !bad; o += r.chunk, ++k) {
        const size_t len = std::min(r.chunk, dbytes - o);
        char* pin = r.buf + (size_t)(k % r.n) * r.chunk;
        CUDA_TRY(cudaEventSynchronize(r.ev[k % r.n]));
        std::atomic<bool> nb{false};
        pool.run([&](int t, int nt) {
            size_t a, b;
            share(len, t, nt, &a, &b);
            if (narrow_f64) {
                if (nt_narrow((float*)(pin + a), (const double*)src_host + (o + a) / 4, (b - a) / 4))
                    nb.store(true, std::memory_order_relaxed);
            } else {
                nt_copy(pin + a, nullptr, (const char*)src_host + o + a, b - a);
            }
            host_sfence();
        });
        if (nb.load()) bad = true;
        CUDA_TRY(cudaMemcpyAsync((char*)dst_dev + o, pin, len, cudaMemcpyHostToDevice, r.st));
        CUDA_TRY(cudaEventRecord(r.ev[k % r.n], r.st));
    }
    CUDA_TRY(cudaStreamSynchronize(r.st));
    if (inexact) *inexact = bad ? 1 : 0;
    return PMSZ_OK;
}

pmsz_status pmsz_device_to_host(void* dst_host, const void* src_dev, int64_t bytes, void* stream) {
    if (bytes < 0 || (bytes > 0 && (!dst_host || !src_dev))) return fail(PMSZ_ERR_INVALID, "bad arguments");
    if (bytes == 0) return PMSZ_OK;
    cudaStream_t s = S(stream);
    if (host_pinned(dst_host)) {
        CUDA_TRY(cudaMemcpyAsync(dst_host, src_dev, (size_t)bytes, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return PMSZ_OK;
    }
    CopyRing& r = copy_ring();
    std::lock_guard<std::mutex> lk(r.m);
    CUDA_TRY(copy_ring_ready(r));
    cudaEvent_t start;
    CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(start, s));                 // the producer of src is ordered first
    CUDA_TRY(cudaStreamWaitEvent(r.st, start, 0));
    cudaEventDestroy(start);
    HostPool& pool = HostPool::get();
    const size_t total = (size_t)bytes;
    const int64_t nch = (int64_t)((total + r.chunk - 1) / r.chunk);
    // DMA up to r.n chunks ahead of the host copy-out
    auto issue = [&](int64_t c) -> cudaError_t {
        const size_t o = (size_t)c * r.chunk, len = std::min(r.chunk, total - o);
        cudaError_t e = cudaMemcpyAsync(r.buf + (size_t)(c % r.n) * r.chunk, (const char*)src_dev + o, len,
                                        cudaMemcpyDeviceToHost, r.st);
        return e == cudaSuccess ? cudaEventRecord(r.ev[c % r.n], r.st) : e;
    };
    for (int64_t c = 0; c < std::min<int64_t>(nch, r.n); ++c) CUDA_TRY(issue(c));
    for (int64_t c = 0; c < nch; ++c) {
        const size_t o = (size_t)c * r.chunk, len = std::min(r.chunk, total - o);
        const char* pin = r.buf + (size_t)(c % r.n) * r.chunk;
        CUDA_TRY(cudaEventSynchronize(r.ev[c % r.n]));
        pool.run([&](int t, int nt) {
            size_t a, b;
            share_at((uintptr_t)dst_host + o, len, t, nt, (size_t)2 << 20, &a, &b);
            nt_copy((char*)dst_host + o + a, nullptr, pin + a, b - a);
            host_sfence();
        });
        if (c + r.n < nch) CUDA_TRY(issue(c + r.n));   // the slot is free again
    }
    return PMSZ_OK;
}

// ---- topology -------------------------------------------------------------
static Dom whole_dom(int64_t nx, int64_t ny, int64_t nz) {
    pmsz_desc d{};
    d.nx = nx; d.ny = ny; d.nz = nz;
    d.core_hi[0] = nx; d.core_hi[1] = ny; d.core_hi[2] = nz;
    d.xi = 1; d.tau = 0.5;
    return make_dom(d);
}

pmsz_status pmsz_scan_neighbors(int64_t nx, int64_t ny, int64_t nz, const double* v, int64_t* nmax, int64_t* nmin,
                                uint8_t* ismax, uint8_t* ismin, void* stream) {
    if (nx < 1 || ny < 1 || nz < 1 || !v) return fail(PMSZ_ERR_INVALID, "bad arguments");
    Dom d = whole_dom(nx, ny, nz);
    dim3 block(32, 8, 1), grid((unsigned)((nx + 31) / 32), (unsigned)((ny + 7) / 8), (unsigned)nz);
    k_scan_full<<<grid, block, 0, S(stream)>>>(d, v, nmax, nmin, ismax, ismin, nullptr);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

pmsz_status pmsz_scan_codes(int64_t nx, int64_t ny, int64_t nz, const double* v, uint8_t* code, void* stream) {
    if (nx < 1 || ny < 1 || nz < 1 || !v || !code) return fail(PMSZ_ERR_INVALID, "bad arguments");
    Dom d = whole_dom(nx, ny, nz);
    dim3 block(32, 8, 1), grid((unsigned)((nx + 31) / 32), (unsigned)((ny + 7) / 8), (unsigned)nz);
    k_scan_full<<<grid, block, 0, S(stream)>>>(d, v, nullptr, nullptr, nullptr, nullptr, code);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

// ---- ghost boxes ------------------------------------------------------------
static bool make_box(int64_t nx, int64_t ny, int64_t nz, const int64_t lo[3], const int64_t hi[3], Box& b) {
    const int64_t ext[3] = {nx, ny, nz};
    for (int a = 0; a < 3; ++a)
        if (lo[a] < 0 || hi[a] > ext[a] || lo[a] > hi[a]) return false;
    b = Box{nx, ny, {lo[0], lo[1], lo[2]}, {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]}, 0, 0};
    b.mxy = div_magic((uint64_t)(b.ext[0] * b.ext[1]));
    b.mx = div_magic((uint64_t)b.ext[0]);
    return true;
}

pmsz_status pmsz_box_pack(int64_t nx, int64_t ny, int64_t nz, const double* src, const int64_t lo[3],
                          const int64_t hi[3], double* buf, void* stream) {
    Box b;
    if (!make_box(nx, ny, nz, lo, hi, b)) return fail(PMSZ_ERR_INVALID, "box outside the domain");
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    if (n == 0) return PMSZ_OK;
    k_box_pack<<<grid_for(n, 256), 256, 0, S(stream)>>>(b, src, buf);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

pmsz_status pmsz_box_unpack_min(int64_t nx, int64_t ny, int64_t nz, double* dst, const int64_t lo[3],
                                const int64_t hi[3], const double* buf, unsigned long long* changed, void* stream) {
    Box b;
    if (!make_box(nx, ny, nz, lo, hi, b)) return fail(PMSZ_ERR_INVALID, "box outside the domain");
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    if (n == 0) return PMSZ_OK;
    k_box_unpack<true><<<grid_for(n, 256), 256, 0, S(stream)>>>(b, dst, buf, changed);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

pmsz_status pmsz_box_unpack_copy(int64_t nx, int64_t ny, int64_t nz, double* dst, const int64_t lo[3],
                                 const int64_t hi[3], const double* buf, unsigned long long* changed, void* stream) {
    Box b;
    if (!make_box(nx, ny, nz, lo, hi, b)) return fail(PMSZ_ERR_INVALID, "box outside the domain");
    const int64_t n = b.ext[0] * b.ext[1] * b.ext[2];
    if (n == 0) return PMSZ_OK;
    k_box_unpack<false><<<grid_for(n, 256), 256, 0, S(stream)>>>(b, dst, buf, changed);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

pmsz_status pmsz_box_extract(const int64_t gdims[3], const void* src, int32_t is_f32, const int64_t lo[3],
                             const int64_t ext[3], void* dst, void* stream) {
    int64_t hi[3] = {lo[0] + ext[0], lo[1] + ext[1], lo[2] + ext[2]};
    Box b;
    if (!make_box(gdims[0], gdims[1], gdims[2], lo, hi, b)) return fail(PMSZ_ERR_INVALID, "box outside the grid");
    const int64_t n = ext[0] * ext[1] * ext[2];
    if (n == 0) return PMSZ_OK;
    if (is_f32)
        k_box_extract<float><<<grid_for(n, 256), 256, 0, S(stream)>>>(b, gdims[1], (const float*)src, (float*)dst);
    else
        k_box_extract<double><<<grid_for(n, 256), 256, 0, S(stream)>>>(b, gdims[1], (const double*)src, (double*)dst);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

// ---- generators ---------------------------------------------------------------
pmsz_status pmsz_perlin(const int64_t gdims[3], const int64_t lo[3], const int64_t ext[3], const int32_t* perm512,
                        double frequency, int32_t octaves, double* out64, float* out32, void* stream) {
    if (!gdims || !lo || !ext || !perm512 || octaves < 1) return fail(PMSZ_ERR_INVALID, "bad arguments");
    cudaStream_t s = S(stream);
    PerlinArgs a{};
    for (int i = 0; i < 3; ++i) { a.gdims[i] = gdims[i]; a.lo[i] = lo[i]; a.ext[i] = ext[i]; }
    a.frequency = frequency;
    a.octaves = octaves;
    int* perm = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&perm, 512 * sizeof(int), s));
    CUDA_TRY(cudaMemcpyAsync(perm, perm512, 512 * sizeof(int), cudaMemcpyHostToDevice, s));
    const int64_t n = ext[0] * ext[1] * ext[2];
    k_perlin<<<grid_for(n, 256, 16), 256, 0, s>>>(a, perm, out64, out32);
    LAUNCHED();
    cudaFreeAsync(perm, s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));   // perm512 is a host buffer owned by the caller
    return PMSZ_OK;
}

pmsz_status pmsz_narrow_f32(const double* v, int64_t n, float* out, int64_t* inexact, void* stream) {
    if (!v || !out || n < 0 || !inexact) return fail(PMSZ_ERR_INVALID, "bad arguments");
    cudaStream_t s = S(stream);
    unsigned long long* k = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&k, 8, s));
    CUDA_TRY(cudaMemsetAsync(k, 0, 8, s));
    if (n > 0) {
        k_narrow<<<grid_for(n, 256, 16), 256, 0, s>>>(n, v, out, k);
        LAUNCHED();
    }
    unsigned long long h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, k, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    cudaFreeAsync(k, s);
    *inexact = (int64_t)h;
    return PMSZ_OK;
}

pmsz_status pmsz_minmax(const void* v, int32_t is_f32, int64_t n, double* mn, double* mx, void* stream) {
    if (!v || n < 1 || !mn || !mx) return fail(PMSZ_ERR_INVALID, "bad arguments");
    cudaStream_t s = S(stream);
    unsigned long long* k = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&k, 16, s));
    unsigned long long init[2] = {0xffffffffffffffffull, 0ull};
    CUDA_TRY(cudaMemcpyAsync(k, init, 16, cudaMemcpyHostToDevice, s));
    if (is_f32)
        k_minmax<float><<<grid_for(n, 256, 16), 256, 0, s>>>((const float*)v, n, k, k + 1);
    else
        k_minmax<double><<<grid_for(n, 256, 16), 256, 0, s>>>((const double*)v, n, k, k + 1);
    LAUNCHED();
    unsigned long long out[2];
    CUDA_TRY(cudaMemcpyAsync(out, k, 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    cudaFreeAsync(k, s);
    auto inv = [](unsigned long long key) {
        unsigned long long b = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
        double d;
        memcpy(&d, &b, 8);
        return d;
    };
    *mn = inv(out[0]);
    *mx = inv(out[1]);
    return PMSZ_OK;
}

pmsz_status pmsz_quantize(const void* f, int32_t is_f32, int64_t n, double origin, double xi, double* recon,
                          int64_t* max_code, void* stream) {
    return pmsz_quantize_codes(f, is_f32, n, origin, xi, recon, nullptr, max_code, stream);
}

pmsz_status pmsz_quantize_codes(const void* f, int32_t is_f32, int64_t n, double origin, double xi, double* recon,
                                uint64_t* codes, int64_t* max_code, void* stream) {
    if (!f || !recon || n < 1 || !(xi > 0)) return fail(PMSZ_ERR_INVALID, "bad arguments");
    cudaStream_t s = S(stream);
    unsigned long long* k = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&k, 16, s));
    CUDA_TRY(cudaMemsetAsync(k, 0, 16, s));
    const double two_xi = 2.0 * xi;
    if (is_f32)
        k_quantize<float><<<grid_for(n, 256, 16), 256, 0, s>>>((const float*)f, n, origin, xi, two_xi, recon, k, k + 1,
                                                               (unsigned long long*)codes);
    else
        k_quantize<double><<<grid_for(n, 256, 16), 256, 0, s>>>((const double*)f, n, origin, xi, two_xi, recon, k, k + 1,
                                                                (unsigned long long*)codes);
    LAUNCHED();
    unsigned long long out[2];
    CUDA_TRY(cudaMemcpyAsync(out, k, 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    cudaFreeAsync(k, s);
    if (max_code) *max_code = (int64_t)out[0];
    if (out[1]) return fail(PMSZ_ERR_INVALID, "quantizer failed to meet its own bound");
    return PMSZ_OK;
}

pmsz_status pmsz_bounded_noise(const void* f, int32_t is_f32, int64_t nx, int64_t ny, int64_t nz,
                               const int64_t gdims[3], const int64_t lo[3], double xi, uint64_t seed, double* out,
                               void* stream) {
    if (!f || !out || !(xi > 0)) return fail(PMSZ_ERR_INVALID, "bad arguments");
    cudaStream_t s = S(stream);
    const int64_t n = nx * ny * nz;
    if (is_f32)
        k_bounded_noise<float><<<grid_for(n, 256, 16), 256, 0, s>>>((const float*)f, nx, ny, nz, gdims[0], gdims[1],
                                                                   lo[0], lo[1], lo[2], xi, seed, out);
    else
        k_bounded_noise<double><<<grid_for(n, 256, 16), 256, 0, s>>>((const double*)f, nx, ny, nz, gdims[0],
                                                                    gdims[1], lo[0], lo[1], lo[2], xi, seed, out);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

// ---- segmentation / compare_plmss ----------------------
static pmsz_status full_codes(int64_t nx, int64_t ny, int64_t nz, const void* v, int32_t is_f32, uint16_t* fc,
                              cudaStream_t s) {
    Dom d = whole_dom(nx, ny, nz);
    dim3 block(32, 8, 1), grid((unsigned)((nx + 31) / 32), (unsigned)((ny + 7) / 8), (unsigned)nz);
    if (is_f32) k_full_code<float><<<grid, block, 0, s>>>(d, (const float*)v, fc);
    else k_full_code<double><<<grid, block, 0, s>>>(d, (const double*)v, fc);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

// Pointer jumping to the fixpoint; `flag` is one device counter.
static pmsz_status jump_to_roots(uint32_t* ptr, int64_t n, unsigned long long* flag, cudaStream_t s) {
    for (int pass = 0; pass < 64; ++pass) {
        unsigned long long h = 0;
        CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(h), s));
        k_jump<<<grid_for(n, 256, 16), 256, 0, s>>>(ptr, n, flag);
        LAUNCHED();
        CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (h == 0) return PMSZ_OK;
    }
    return fail(PMSZ_ERR_CUDA, "pointer jumping did not reach a fixpoint");
}

// up/down root pointers of one field into asc (down) / desc (up), u32 device arrays.
static pmsz_status segment_u32(int64_t nx, int64_t ny, int64_t nz, const void* v, int32_t is_f32, uint16_t* fc,
                               uint32_t* asc, uint32_t* desc, unsigned long long* flag, cudaStream_t s) {
    pmsz_status st = full_codes(nx, ny, nz, v, is_f32, fc, s);
    if (st) return st;
    Dom d = whole_dom(nx, ny, nz);
    k_seg_ptr<<<grid_for(d.n, 256, 16), 256, 0, s>>>(d, fc, desc, asc);
    LAUNCHED();
    st = jump_to_roots(desc, d.n, flag, s);
    if (st) return st;
    return jump_to_roots(asc, d.n, flag, s);
}

pmsz_status pmsz_segmentation(int64_t nx, int64_t ny, int64_t nz, const void* v, int32_t is_f32,
                              int64_t* asc_target, int64_t* desc_target, void* stream) {
    if (nx < 1 || ny < 1 || nz < 1 || !v || !asc_target || !desc_target) return fail(PMSZ_ERR_INVALID, "bad arguments");
    const int64_t n = nx * ny * nz;
    if (n >= (int64_t)0xffffffffll) return fail(PMSZ_ERR_INVALID, "domain too large for 32-bit ids");
    cudaStream_t s = S(stream);
    uint16_t* fc = nullptr;
    uint32_t *a = nullptr, *dd = nullptr;
    unsigned long long* flag = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&fc, n * 2, s));
    CUDA_TRY(cudaMallocAsync((void**)&a, n * 4, s));
    CUDA_TRY(cudaMallocAsync((void**)&dd, n * 4, s));
    CUDA_TRY(cudaMallocAsync((void**)&flag, 8, s));
    pmsz_status st = segment_u32(nx, ny, nz, v, is_f32, fc, a, dd, flag, s);
    if (st == PMSZ_OK) {
        k_widen<<<grid_for(n, 256, 16), 256, 0, s>>>(a, asc_target, n);
        LAUNCHED();
        k_widen<<<grid_for(n, 256, 16), 256, 0, s>>>(dd, desc_target, n);
        LAUNCHED();
    }
    cudaFreeAsync(fc, s); cudaFreeAsync(a, s); cudaFreeAsync(dd, s); cudaFreeAsync(flag, s);
    CUDA_TRY(cudaGetLastError());
    return st;
}

pmsz_status pmsz_compare_plmss(int64_t nx, int64_t ny, int64_t nz, const void* ref, int32_t ref_f32, const void* test,
                               int32_t test_f32, uint32_t* kind_bits, int64_t* counts, void* stream) {
    if (nx < 1 || ny < 1 || nz < 1 || !ref || !test || !counts) return fail(PMSZ_ERR_INVALID, "bad arguments");
    const int64_t n = nx * ny * nz;
    if (n >= (int64_t)0xffffffffll) return fail(PMSZ_ERR_INVALID, "domain too large for 32-bit ids");
    cudaStream_t s = S(stream);
    uint16_t *rc = nullptr, *tc = nullptr;
    uint32_t *ra = nullptr, *rd = nullptr, *ta = nullptr, *td = nullptr;
    unsigned long long* cnt = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&rc, n * 2, s));
    CUDA_TRY(cudaMallocAsync((void**)&tc, n * 2, s));
    CUDA_TRY(cudaMallocAsync((void**)&ra, n * 4, s));
    CUDA_TRY(cudaMallocAsync((void**)&rd, n * 4, s));
    CUDA_TRY(cudaMallocAsync((void**)&ta, n * 4, s));
    CUDA_TRY(cudaMallocAsync((void**)&td, n * 4, s));
    CUDA_TRY(cudaMallocAsync((void**)&cnt, 8 * 8, s));
    pmsz_status st = segment_u32(nx, ny, nz, ref, ref_f32, rc, ra, rd, cnt + 7, s);
    if (st == PMSZ_OK) st = segment_u32(nx, ny, nz, test, test_f32, tc, ta, td, cnt + 7, s);
    if (st == PMSZ_OK) {
        CUDA_TRY(cudaMemsetAsync(cnt, 0, 7 * 8, s));
        k_plmss<<<grid_for((n + 31) / 32 * 32, 256, 16), 256, 0, s>>>(n, rc, tc, ra, ta, rd, td, kind_bits,
                                                                       (n + 31) / 32, cnt);
        LAUNCHED();
        unsigned long long h[7];
        CUDA_TRY(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (int k = 0; k < 7; ++k) counts[k] = (int64_t)h[k];
    }
    cudaFreeAsync(rc, s); cudaFreeAsync(tc, s); cudaFreeAsync(ra, s); cudaFreeAsync(rd, s);
    cudaFreeAsync(ta, s); cudaFreeAsync(td, s); cudaFreeAsync(cnt, s);
    CUDA_TRY(cudaGetLastError());
    return st;
}

pmsz_status pmsz_bits_to_ids(const uint32_t* bits, int64_t nbits, int64_t* ids, int64_t cap, int64_t* count,
                             void* stream) {
    if (!bits || nbits < 0 || !count) return fail(PMSZ_ERR_INVALID, "bad arguments");
    cudaStream_t s = S(stream);
    const int64_t nwords = (nbits + 31) / 32;
    if (nwords == 0) {
        *count = 0;
        return PMSZ_OK;
    }
    const Chunks ch = make_chunks(nwords, num_sms());
    unsigned long long* bc = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&bc, (kMaxChunks + 2) * 8, s));
    CUDA_TRY(cudaMemsetAsync(bc + kMaxChunks, 0, 8, s));   // the ticket
    k_chunk_count_scan<<<(unsigned)ch.n, kCompactThreads, 0, s>>>(bits, ch, bc, bc + kMaxChunks + 1,
                                                                  (unsigned*)(bc + kMaxChunks));
    LAUNCHED();
    unsigned long long total = 0;
    CUDA_TRY(cudaMemcpyAsync(&total, bc + kMaxChunks + 1, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *count = (int64_t)total;
    if (ids && (int64_t)total <= cap && total > 0) {
        k_chunk_list<int64_t><<<(unsigned)ch.n, kCompactThreads, 0, s>>>(const_cast<uint32_t*>(bits), ch, bc, ids, 0);
        LAUNCHED();
    }
    cudaFreeAsync(bc, s);
    CUDA_TRY(cudaGetLastError());
    if (ids && (int64_t)total > cap) return fail(PMSZ_ERR_INVALID, "id buffer too small");
    return PMSZ_OK;
}

pmsz_status pmsz_gaussian_peaks(const int64_t gdims[3], const int64_t lo[3], const int64_t ext[3], uint64_t seed,
                                int32_t out_f32, void* out, void* stream) {
    if (!gdims || !lo || !ext || !out) return fail(PMSZ_ERR_INVALID, "null argument");
    for (int a = 0; a < 3; ++a)
        if (gdims[a] < 1 || ext[a] < 1 || lo[a] < 0 || lo[a] + ext[a] > gdims[a])
            return fail(PMSZ_ERR_INVALID, "sub-box outside the global grid");
    PeakArgs a{gdims[0], gdims[1], gdims[2], lo[0], lo[1], lo[2], ext[0], ext[1], ext[2], seed};
    const int64_t n = ext[0] * ext[1] * ext[2];
    cudaStream_t s = S(stream);
    if (out_f32) k_peaks<float><<<grid_for(n, 256, 16), 256, 0, s>>>(a, (float*)out);
    else k_peaks<double><<<grid_for(n, 256, 16), 256, 0, s>>>(a, (double*)out);
    LAUNCHED();
    CUDA_TRY(cudaGetLastError());
    return PMSZ_OK;
}

}  // extern "C"
