// prep2.cuh -- K0 as a barrier-free producer / consumer pipeline with the
// first iteration's detection AND rules fused in.
//
// K0 (correction.py:52-60,118-122,404-405) validates the pair, copies
// g <- fhat and builds the f-code (field_scan(original)); the first Jacobi
// iteration (correction.py:232-242 with g = fhat) then detects every
// mismatching centre and proposes.  This kernel does all of it in one pass
// over f and fhat:
//
//   * a producer warp stages, per plane, the f tile (f32 or f64, halo
//     included) and the fhat tile (f64, halo included) by two TMA boxes into a
//     4-slot ring (full / empty mbarriers; no block barrier anywhere);
//   * each consumer warp owns 4 rows x 32 columns of the CTA's 32 x 32 column
//     and, per plane: finishes the robust SCREEN of its centres (top-2 /
//     bottom-2 of the closed ring, prep.cuh), validates and copies its 128
//     centres, writes the fragile bitmap word of each row, and queues its
//     fragile centres in a warp-private queue;
//   * the warp then evaluates its queue one centre per lane: the exact f-code
//     (balanced-tree fold on the staged f values), and -- for centres of the
//     core box -- the g-scan of fhat (balanced tree on the staged fhat ring),
//     the code comparison and, on a mismatch, the six rules
//     (correction.py:169-229) with proposals by RED.MIN into prop / touched.
//     The first iteration's tiled sweep, the detection-bit compaction and the
//     deferred rule kernel are all gone.
//
// Robust centres (prep.cuh) get f-code kRobust and are never evaluated.
// Cells outside the field are NaN (TMA fill), as in every tiled kernel.
#pragma once
#include "prep.cuh"

namespace pmsz {

constexpr int kP2Slots = 4;                      // planes k .. k+2 in use, k+3 in flight
constexpr int kP2Consumers = kQY / kQRowsPerThread;   // 8 warps x 4 rows
constexpr int kP2Threads = (kP2Consumers + 1) * 32;   // + the producer warp

template <typename FT>
struct P2Smem {
    using G = PrepGeo<FT>;
    FT plane[kP2Slots][G::kStride];
    double fh[kP2Slots][kQPlaneStride];
    uint16_t queue[kP2Consumers][kQRowsPerThread * 32];   // r * 32 + lane of this warp's fragile centres
    unsigned long long full[kP2Slots];
    unsigned long long empty[kP2Slots];
};

template <typename FT, bool kExtrema>
__global__ void __launch_bounds__(kP2Threads, 2)
k_prep2(Dom d, const __grid_constant__ CUtensorMap tf, const __grid_constant__ CUtensorMap th, PrepArgs a, Work w,
        int zchunk) {
    using G = PrepGeo<FT>;
    using V = FT;
    extern __shared__ __align__(1024) unsigned char p2raw[];
    P2Smem<FT>& S = *reinterpret_cast<P2Smem<FT>*>(p2raw);
    const int lane = threadIdx.x, wid = threadIdx.y;
    const int x0 = (int)blockIdx.x * kQX, y0 = (int)blockIdx.y * kQY;
    const int zb = a.z0 + (int)blockIdx.z * zchunk;
    const int K = min(zb + zchunk, a.z1) - zb;
    const unsigned full0 = smem_u32(&S.full[0]), empty0 = smem_u32(&S.empty[0]);
    if (wid == kP2Consumers && lane == 0) {
        for (int s = 0; s < kP2Slots; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, kP2Consumers);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (wid == kP2Consumers) {
        // ---- producer: plane index i = p - (zb - 1), i in [0, K + 1] ----
        if (lane == 0) {
            const int xs = (x0 - 1) & ~(G::kAlign - 1), xh = (x0 - 1) & ~1;   // 16-byte aligned box origins
            const unsigned pl0 = smem_u32(&S.plane[0][0]), fh0 = smem_u32(&S.fh[0][0]);
            for (int i = 0; i <= K + 1; ++i) {
                const int s = i & (kP2Slots - 1);
                if (i >= kP2Slots) mbar_wait(empty0 + 8 * s, (unsigned)((i / kP2Slots - 1) & 1));
                mbar_expect_tx(full0 + 8 * s, G::kPlane * (unsigned)sizeof(FT) + kQPlane * 8);
                tma_load_3d(pl0 + s * G::kStride * (unsigned)sizeof(FT), &tf, xs, y0 - 1, zb - 1 + i, full0 + 8 * s);
                tma_load_3d(fh0 + s * kQPlaneStride * 8, &th, xh, y0 - 1, zb - 1 + i, full0 + 8 * s);
            }
        }
        return;
    }
    // ---- consumers ----
    auto wait_plane = [&](int i) { mbar_wait(full0 + 8 * (i & (kP2Slots - 1)), (unsigned)((i / kP2Slots) & 1)); };
    const uint32_t sy = (uint32_t)d.sy, sz = (uint32_t)d.sz;
    const int xo = (x0 - 1) - ((x0 - 1) & ~(G::kAlign - 1));   // staged column of x0 - 1 (f)
    const int xho = (x0 - 1) - ((x0 - 1) & ~1);                // staged column of x0 - 1 (fhat)
    const int x = x0 + lane, yr = y0 + kQRowsPerThread * wid;
    const bool live_x = x < d.nx;
    bool live[kQRowsPerThread];
#pragma unroll
    for (int r = 0; r < kQRowsPerThread; ++r) live[r] = live_x && yr + r < d.ny;
    const uint32_t c0 = (uint32_t)x + (uint32_t)yr * sy + (uint32_t)zb * sz;   // row-0 centre at plane zb
    const int col = xo + lane;                 // staged column of x - 1
    const int row0 = kQRowsPerThread * wid;    // staged row of y_0 - 1
    const bool edge_xy = x0 == 0 || x0 + kQX >= d.nx || y0 == 0 || y0 + kQY >= d.ny;
    const bool core_xy = x0 >= a.core_lo[0] && x0 + kQX <= a.core_hi[0] && y0 >= a.core_lo[1] && y0 + kQY <= a.core_hi[1];
    uint16_t* q = S.queue[wid];
    const unsigned below = (1u << lane) - 1u;
    unsigned nfrag = 0, ndet = 0;

    // plane_groups of prep.cuh on this warp's rows of one staged f plane
    auto plane_groups = [&](const V* P, auto&& emit) {
        const V* row = P + row0 * G::kPX + col;
        V l = row[0], m = row[1], rr = row[2];
        P2<V> pl = p2(l, m), pr = p2(m, rr), pl1;
        V leaf_prev = rr;
#pragma unroll
        for (int j = 1; j < kQRowsPerThread + 2; ++j) {
            row += G::kPX;
            l = row[0]; m = row[1];
            const V rn = row[2];
            const P2<V> pln = p2(l, m), prn = p2(m, rn);
            if (j >= 2) emit(j - 2, box2(pl1, pl), box2(pr, prn), prn, leaf_prev);
            pl1 = pl; pl = pln;
            pr = prn;
            leaf_prev = rn;
        }
    };
    T2<V> lbprev[kQRowsPerThread], acc[kQRowsPerThread];
    wait_plane(0);
    wait_plane(1);
    plane_groups(S.plane[0], [&](int r, const T2<V>& lb, const T2<V>&, const P2<V>&, V) { lbprev[r] = lb; });
    plane_groups(S.plane[1], [&](int r, const T2<V>& lb, const T2<V>& rb, const P2<V>&, V) {
        acc[r] = lbprev[r];
        merge2(acc[r], lb);
        merge2(acc[r], rb);
        lbprev[r] = lb;
    });
    const V thr = (V)a.thr;
    for (int k = 0; k < K; ++k) {
        // centre plane zb + k: plane indices k (below), k + 1 (centre), k + 2 (above)
        wait_plane(k + 2);
        const int s0 = k & (kP2Slots - 1), s1 = (k + 1) & (kP2Slots - 1), s2 = (k + 2) & (kP2Slots - 1);
        const V* fct = S.plane[s1];
        const double* hct = S.fh[s1];
        const uint32_t cz = c0 + (uint32_t)k * sz;
        bool want[kQRowsPerThread];
        plane_groups(S.plane[s2], [&](int r, const T2<V>& lb, const T2<V>& rb, const P2<V>&, V) {
            merge2(acc[r], rb);   // U group: the ring of centre r is complete
            const bool robust = robust2(acc[r], thr, a.xi);
            want[r] = live[r] && !robust;
            if (live[r]) {
                const uint32_t c = cz + r * sy;
                // validation (correction.py:52-60), hazard H6, g <- fhat
                const double fv = (double)fct[(row0 + r + 1) * G::kPX + col + 1];
                const double hv = hct[(row0 + r + 1) * kQPX + xho + 1 + lane];
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
                if (a.g != nullptr) a.g[c] = hv;
                if (robust) a.code[c] = kRobust;
            }
            // partial ring of the same column at the next plane
            acc[r] = lbprev[r];
            merge2(acc[r], lb);
            merge2(acc[r], rb);
            lbprev[r] = lb;
        });
        // fragile bitmap and the warp's queue
        unsigned bal[kQRowsPerThread], n = 0;
#pragma unroll
        for (int r = 0; r < kQRowsPerThread; ++r) {
            bal[r] = __ballot_sync(0xffffffffu, want[r]);
            if (want[r]) q[n + __popc(bal[r] & below)] = (uint16_t)(r * 32 + lane);
            n += __popc(bal[r]);
        }
        if (a.frag_direct) {
            // one word per row: lane r stores row r's ballot
            if (lane < kQRowsPerThread && yr + lane < d.ny) {
                unsigned b = bal[0];
#pragma unroll
                for (int r = 1; r < kQRowsPerThread; ++r) b = lane == r ? bal[r] : b;
                a.frag[(cz - (uint32_t)lane + (uint32_t)lane * sy) >> 5] = b;
            }
        } else if (lane == 0) {
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
        nfrag += lane == 0 ? n : 0u;
        __syncwarp();
        // the queue, one centre per lane: exact f-code; in the core box also
        // the first detection (g = fhat) and, on a mismatch, the rules
        const int zc = zb + k;
        const bool edge = edge_xy || zc == 0 || zc + 1 >= d.nz;
        const bool core_z = zc >= a.core_lo[2] && zc < a.core_hi[2];
        const V* dn = S.plane[s0];
        const V* up = S.plane[s2];
        for (unsigned e = lane; e < n; e += 32) {
            const int ent = q[e];
            const int r = ent >> 5, lx = ent & 31;
            const int cell = (row0 + r + 1) * G::kPX + xo + 1 + lx;
            V nv[14];
            nv[0] = dn[cell - G::kPX - 1]; nv[1] = dn[cell - G::kPX]; nv[2] = dn[cell - 1]; nv[3] = dn[cell];
            nv[4] = fct[cell - G::kPX - 1]; nv[5] = fct[cell - G::kPX]; nv[6] = fct[cell - 1]; nv[7] = fct[cell + 1];
            nv[8] = fct[cell + G::kPX]; nv[9] = fct[cell + G::kPX + 1];
            nv[10] = up[cell]; nv[11] = up[cell + 1]; nv[12] = up[cell + G::kPX]; nv[13] = up[cell + G::kPX + 1];
            const uint8_t fc = edge ? fold_code<V>(fct[cell], nv) : tree_code<V>(fct[cell], nv);
            const uint32_t c = cz + (uint32_t)r * sy + (uint32_t)lx - (uint32_t)lane;
            a.code[c] = fc;
            if (a.det == nullptr || !core_z) continue;
            const int gx = x0 + lx, gy = yr + r;
            if (!core_xy && !(gx >= a.core_lo[0] && gx < a.core_hi[0] && gy >= a.core_lo[1] && gy < a.core_hi[1]))
                continue;
            double hv[14], hc;
            ring_from_smem(S.fh[s0], hct, S.fh[s2], (row0 + r + 1) * kQPX + xho + 1 + lx, hv, hc);
            const Scan sc = edge ? fold_scan(hc, hv) : tree_scan(hc, hv);
            const uint8_t gc = scan_code(sc);
            const bool mismatch = kExtrema ? (((gc & 15) == kExtremum) != ((fc & 15) == kExtremum) ||
                                              ((gc >> 4) == kExtremum) != ((fc >> 4) == kExtremum))
                                           : gc != fc;
            if (mismatch) {
                atomicOr(a.det + (c >> 5), 1u << (c & 31));
                ++ndet;
                EmitRed emit{w};
                rules<false>(d, w, sc, hv, fc, (int64_t)c, emit);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * s0);   // plane index k is no longer needed
    }
    const unsigned nfr = __reduce_add_sync(0xffffffffu, nfrag);
    const unsigned nd = __reduce_add_sync(0xffffffffu, ndet);
    if (lane == 0) {
        if (nd) atomicAdd(&a.ctr->ndetect, (unsigned long long)nd);
        if (nfr) atomicAdd(&a.ctr->nfragile, (unsigned long long)nfr);
    }
}

// Launch the fused K0 over z planes [z0, z1) of the domain (every centre of the
// ext extent gets its f-code, parallel.py:212; only core centres are
// detected).  Returns false when the fields cannot be described by tensor
// maps or the robust classification is off (the caller takes prep.cuh).
template <typename FT>
inline bool launch_prep2(const Dom& d, const FT* f, const double* fh, double* g, uint8_t* code, uint32_t* frag,
                         DevCounters* ctr, uint32_t* det, const Work& w, cudaStream_t s, int64_t z0 = 0,
                         int64_t z1 = -1) {
    using G = PrepGeo<FT>;
    if (!frag || !det) return false;
    if (z1 < 0) z1 = d.nz;
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
    Dom all = d;   // rank offsets / strides of the whole ext domain (rules propose anywhere in it)
    const int64_t tiles = ((d.nx + kQX - 1) / kQX) * ((d.ny + kQY - 1) / kQY);
    const int64_t want = (148 * 2 * 6 + tiles - 1) / tiles;
    int64_t chunks = std::max<int64_t>((nzr + 23) / 24, std::min<int64_t>(want, nzr / 16));
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, nzr));
    int zchunk = (int)std::max<int64_t>(1, (nzr + chunks - 1) / chunks);
    static const int zc_env = getenv("PMSZ_PREP_ZCHUNK") ? atoi(getenv("PMSZ_PREP_ZCHUNK")) : 0;
    if (zc_env > 0) zchunk = (int)std::min<int64_t>(zc_env, nzr);
    chunks = (nzr + zchunk - 1) / zchunk;
    const dim3 grid((unsigned)((d.nx + kQX - 1) / kQX), (unsigned)((d.ny + kQY - 1) / kQY), (unsigned)chunks);
    const dim3 block(32, kP2Consumers + 1, 1);
    const size_t smem = sizeof(P2Smem<FT>);
    if (d.extrema_only) {
        cudaFuncSetAttribute(k_prep2<FT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_prep2<FT, true><<<grid, block, smem, s>>>(all, tf, th, a, w, zchunk);
    } else {
        cudaFuncSetAttribute(k_prep2<FT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_prep2<FT, false><<<grid, block, smem, s>>>(all, tf, th, a, w, zchunk);
    }
    return true;
}

}  // namespace pmsz
