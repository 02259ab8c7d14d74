// gather.cuh -- K1 detect+propose over a SORTED list of dirty centres with
// the 15 stencil values of each centre fetched by cp.async into shared memory.
//
// A plain gather kernel (one centre per thread, 15 loads, fold, rules) is
// latency bound: each thread waits for its loads before it can issue the next
// centre's, and registers cap the warps per SM.  Here every warp runs a
// software pipeline over batches of 32 list entries (one centre per lane):
// the loads of kGP batches are in flight as asynchronous copies into the
// warp's shared buffers while the lanes fold the oldest batch, so the memory
// system sees ~kGP x 32 x 15 independent requests per warp without spending
// registers on them.  The list is ascending (compacted from a bitmap), so the
// 32 centres of a batch are neighbours and their copies share sectors.
//
// Arithmetic per centre is k_defer / sweep_sparse_range: fold_scan with NaN
// for missing neighbours, code_mismatch, the six rules; the detection bit of
// the centre is set on a mismatch and cleared otherwise.  Emit chooses how
// targets are recorded: EmitRed (touched bitmap, compacted afterwards) or
// EmitList (appended to the target list).
#pragma once
#include "tiles.cuh"

namespace pmsz {

constexpr int kGP = 3;          // batches in flight per warp
constexpr int kGWarps = 8;      // warps per CTA
constexpr int kGSlots = 17;     // 14 neighbours, centre, code word, detection word
constexpr int kGBuf = kGSlots * 32;   // doubles per batch buffer
constexpr size_t kGatherSmem = (size_t)kGWarps * kGP * kGBuf * sizeof(double);

template <bool kList>
__global__ void __launch_bounds__(kGWarps * 32, 2) k_gather(Dom d, const double* __restrict__ g, Work w,
                                                            const uint32_t* __restrict__ list,
                                                            const unsigned long long* __restrict__ count) {
    extern __shared__ __align__(16) double gsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* wb = gsm + (size_t)wid * kGP * kGBuf;
    const unsigned long long n = *count;
    const unsigned long long nb = (n + 31) / 32;
    const unsigned long long nwarps = (unsigned long long)gridDim.x * kGWarps;
    const unsigned long long first = (unsigned long long)blockIdx.x * kGWarps + wid;
    const double nanv = nan64();

    // issue the copies of batch b into buffer slot `buf`; the centre id is kept
    // in the code-word slot's upper half
    auto issue = [&](unsigned long long b, int buf) {
        double* B = wb + buf * kGBuf;
        const unsigned long long i = b * 32 + lane;
        if (b >= nb || i >= n) {
            reinterpret_cast<uint32_t*>(B + 15 * 32 + lane)[1] = 0xffffffffu;
            return;
        }
        const int64_t c = __ldcg(list + i);
        int64_t x, y, z;
        coords(d, c, x, y, z);
        // a dilated mask may reach past the core box (ghost layers of a block)
        if (!(x >= d.lo[0] && x < d.hi[0] && y >= d.lo[1] && y < d.hi[1] && z >= d.lo[2] && z < d.hi[2])) {
            reinterpret_cast<uint32_t*>(B + 15 * 32 + lane)[1] = 0xffffffffu;
            return;
        }
        const double* p0 = g + c;
        if (x > 0 && x + 1 < d.nx && y > 0 && y + 1 < d.ny && z > 0 && z + 1 < d.nz) {
            // interior: the 14 sources are 3 rows of plane z-1/z/z+1 around p0
            const double* dn = p0 - d.sz;
            const double* up = p0 + d.sz;
            const double* dnm = dn - d.sy;
            const double* ctm = p0 - d.sy;
            const double* ctp = p0 + d.sy;
            const double* upp = up + d.sy;
            cp_async8(B + 0 * 32 + lane, dnm - 1);   // (-1,-1,-1)
            cp_async8(B + 1 * 32 + lane, dnm);       // ( 0,-1,-1)
            cp_async8(B + 2 * 32 + lane, dn - 1);    // (-1, 0,-1)
            cp_async8(B + 3 * 32 + lane, dn);        // ( 0, 0,-1)
            cp_async8(B + 4 * 32 + lane, ctm - 1);   // (-1,-1, 0)
            cp_async8(B + 5 * 32 + lane, ctm);       // ( 0,-1, 0)
            cp_async8(B + 6 * 32 + lane, p0 - 1);    // (-1, 0, 0)
            cp_async8(B + 7 * 32 + lane, p0 + 1);    // ( 1, 0, 0)
            cp_async8(B + 8 * 32 + lane, ctp);       // ( 0, 1, 0)
            cp_async8(B + 9 * 32 + lane, ctp + 1);   // ( 1, 1, 0)
            cp_async8(B + 10 * 32 + lane, up);       // ( 0, 0, 1)
            cp_async8(B + 11 * 32 + lane, up + 1);   // ( 1, 0, 1)
            cp_async8(B + 12 * 32 + lane, upp);      // ( 0, 1, 1)
            cp_async8(B + 13 * 32 + lane, upp + 1);  // ( 1, 1, 1)
        } else {
#pragma unroll
            for (int r = 0; r < 14; ++r) {
                const bool ok = in_dom(d, x + rank_dx(r), y + rank_dy(r), z + rank_dz(r));
                if (ok) cp_async8(B + r * 32 + lane, p0 + rank_off(d, r));
                else B[r * 32 + lane] = nanv;
            }
        }
        cp_async8(B + 14 * 32 + lane, p0);
        uint32_t* cw = reinterpret_cast<uint32_t*>(B + 15 * 32 + lane);
        cp_async4(cw, reinterpret_cast<const uint32_t*>(w.code + (c & ~3ll)));
        cw[1] = (uint32_t)c;
        cp_async4(reinterpret_cast<uint32_t*>(B + 16 * 32 + lane), w.detbits + (c >> 5));
    };

#pragma unroll
    for (int q = 0; q < kGP; ++q) {
        issue(first + q * nwarps, q);
        cp_async_commit();
    }
    unsigned ndet = 0;
    int buf = 0;
    for (unsigned long long b = first; b < nb; b += nwarps) {
        cp_async_wait<kGP - 1>();
        __syncwarp();
        const double* B = wb + buf * kGBuf;
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(B + 15 * 32 + lane);
        const uint32_t cid = cw[1];
        if (cid != 0xffffffffu) {
            const int64_t c = cid;
            double nv[14];
#pragma unroll
            for (int r = 0; r < 14; ++r) nv[r] = B[r * 32 + lane];
            const Scan s = fold_scan(B[14 * 32 + lane], nv);
            const uint8_t fc = (uint8_t)(cw[0] >> (8 * (c & 3)));
            const uint32_t bit = 1u << (c & 31);
            const bool det_was = (reinterpret_cast<const uint32_t*>(B + 16 * 32 + lane)[0] & bit) != 0;
            if (code_mismatch(d, scan_code(s), fc)) {
                ++ndet;
                if (!det_was) atomicOr(w.detbits + (c >> 5), bit);
                if (kList) {
                    EmitList emit{w, {}, 0};
                    rules<false>(d, w, s, nv, fc, c, emit);
                    emit.flush();
                } else {
                    EmitRed emit{w};
                    rules<false>(d, w, s, nv, fc, c, emit);
                }
            } else if (det_was) {
                atomicAnd(w.detbits + (c >> 5), ~bit);
            }
        }
        __syncwarp();
        issue(b + kGP * nwarps, buf);
        cp_async_commit();
        buf = buf + 1 == kGP ? 0 : buf + 1;
    }
    cp_async_wait<0>();
    const unsigned t = __reduce_add_sync(0xffffffffu, ndet);
    if (t && lane == 0) atomicAdd(&w.ctr->ndetect, (unsigned long long)t);
}

}  // namespace pmsz
