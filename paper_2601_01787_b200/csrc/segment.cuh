// segment.cuh -- steepest-path segmentation and compare_plmss on the device
// (topology.py:156-174,254-274).
//
//   full code  u16 per vertex: rmax | rmin << 4 | is_max << 8 | is_min << 9.
//              Unlike the 1-byte f-code it keeps the argmax / argmin rank of
//              extrema too, which the order-violation kinds of compare_plmss
//              read (topology.py:271-272 compare nmax of every non-maximum of
//              the reference, whatever the test field's flag).
//   pointers   up = is_max ? id : nmax, down = is_min ? id : nmin (u32 ids).
//   jumping    s[i] <- s[s[i]] in place, several hops per visit, until a pass
//              changes nothing: the fixpoint of topology.py:147-153 (in-place
//              updates only shorten paths towards the same root).
#pragma once
#include "common.cuh"

namespace pmsz {

template <typename T>
__global__ void __launch_bounds__(256) k_full_code(Dom d, const T* __restrict__ v, uint16_t* __restrict__ fc) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t y = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    const int64_t z = blockIdx.z;
    if (x >= d.nx || y >= d.ny) return;
    const int64_t c = x + y * d.sy + z * d.sz;
    double nv[14];
#pragma unroll
    for (int r = 0; r < 14; ++r) {
        const bool ok = in_dom(d, x + rank_dx(r), y + rank_dy(r), z + rank_dz(r));
        nv[r] = ok ? (double)__ldg(v + c + rank_off(d, r)) : nan64();
    }
    const Scan s = fold_scan((double)__ldg(v + c), nv);
    fc[c] = (uint16_t)(s.rmax | (s.rmin << 4) | ((s.is_max ? 1 : 0) << 8) | ((s.is_min ? 1 : 0) << 9));
}

__global__ void __launch_bounds__(256) k_seg_ptr(Dom d, const uint16_t* __restrict__ fc, uint32_t* __restrict__ up,
                                                 uint32_t* __restrict__ down) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = fc[c];
        up[c] = (k & 0x100u) ? (uint32_t)c : (uint32_t)(c + rank_off(d, (int)(k & 15u)));
        down[c] = (k & 0x200u) ? (uint32_t)c : (uint32_t)(c + rank_off(d, (int)((k >> 4) & 15u)));
    }
}

// One pass of in-place pointer jumping; *changed counts warps that moved a pointer.
__global__ void __launch_bounds__(256) k_jump(uint32_t* s, int64_t n, unsigned long long* changed) {
    bool moved = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t a = __ldcg(s + i);
        uint32_t b = __ldcg(s + a);
        if (b == a) continue;
#pragma unroll 1
        for (int hop = 0; hop < 8; ++hop) {
            const uint32_t c2 = __ldcg(s + b);
            if (c2 == b) break;
            b = c2;
        }
        s[i] = b;
        moved = true;
    }
    if (__any_sync(0xffffffffu, moved) && (threadIdx.x & 31) == 0) atomicAdd(changed, 1ull);
}

__global__ void __launch_bounds__(256) k_widen(const uint32_t* __restrict__ s, int64_t* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)s[i];
}

// compare_plmss kinds (topology.py:266-272) as six bitmaps + counts, and the
// label-pair disagreement count (topology.py:273).  Block-reduced counters.
__global__ void __launch_bounds__(256) k_plmss(int64_t n, const uint16_t* __restrict__ rc,
                                               const uint16_t* __restrict__ tc, const uint32_t* __restrict__ ra,
                                               const uint32_t* __restrict__ ta, const uint32_t* __restrict__ rd,
                                               const uint32_t* __restrict__ td, uint32_t* __restrict__ bits,
                                               int64_t nwords, unsigned long long* counts) {
    __shared__ unsigned long long part[8][7];
    unsigned long long cnt[7] = {0, 0, 0, 0, 0, 0, 0};
    const int lane = threadIdx.x & 31;
    // whole warps per 32-vertex word so the ballots are the bitmap words
    const int64_t nw = (n + 31) / 32;
    for (int64_t wd = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wd < nw;
         wd += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t i = wd * 32 + lane;
        bool k[6] = {false, false, false, false, false, false};
        bool wrong = false;
        if (i < n) {
            const uint32_t r = rc[i], t = tc[i];
            const bool rmax = r & 0x100u, rmin = r & 0x200u, tmax = t & 0x100u, tmin = t & 0x200u;
            k[0] = tmax && !rmax;
            k[1] = rmax && !tmax;
            k[2] = tmin && !rmin;
            k[3] = rmin && !tmin;
            k[4] = !rmax && ((t & 15u) != (r & 15u));
            k[5] = !rmin && (((t >> 4) & 15u) != ((r >> 4) & 15u));
            wrong = ra[i] != ta[i] || rd[i] != td[i];
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const unsigned m = __ballot_sync(0xffffffffu, k[q]);
            if (lane == 0) {
                if (bits) bits[q * nwords + wd] = m;
                cnt[q] += __popc(m);
            }
        }
        const unsigned mw = __ballot_sync(0xffffffffu, wrong);
        if (lane == 0) cnt[6] += __popc(mw);
    }
    const int wid = threadIdx.x >> 5;
    if (lane == 0)
        for (int q = 0; q < 7; ++q) part[wid][q] = cnt[q];
    __syncthreads();
    if (threadIdx.x < 7) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; ++w) t += part[w][threadIdx.x];
        if (t) atomicAdd(&counts[threadIdx.x], t);
    }
}

}  // namespace pmsz
