// rules1.cuh -- the first Jacobi iteration after K0 as ONE tiled pass.
//
// K0 leaves, for g = fhat, the detection bit of every mismatching centre.  The
// rest of iteration 1 (correction.py:207-242) is the rules of those centres
// (~2.5 % of the field at 512^3), the min-merge of their proposals and the
// clamped apply -- as separate passes a detection-bit compaction, k_defer
// (15 gathers and 2 global atomics per proposal), a target compaction and
// k_apply_list (378 B of DRAM per target).  Here a CTA owns a 32 x 32 column
// and marches its z chunk with fhat planes staged by TMA with a 2-voxel halo:
//
//   per centre plane zc: its detected centres of the 1-halo region (from the
//   detection bits) are queued per warp and their rules run one per lane on
//   the staged ring; proposals to targets inside the CTA's own box are
//   min-merged in a 3-plane shared ring (atomicMin on the order keys, exactly
//   np.minimum.at) -- every proposing centre of such a target lies in the
//   1-halo, so the merged value is complete once centre plane zc has run for
//   target plane zc - 1;
//   then target plane zc - 1 is applied from the staged fhat value and f:
//   g' = max(min(fhat, p), f - xi) is written to g (K0 already copied fhat
//   there), and the ever-edited and per-iteration edit bits are stored one
//   word per row.
//
// Jacobi semantics hold because the rules read fhat while the edits go to g
// (out-of-place runs only).  No global proposal array, no work lists, no
// atomics on global memory apart from the counters.
#pragma once
#include "sweep.cuh"
#include "tma.cuh"

namespace pmsz {

constexpr int kR1X = 32, kR1Y = 32;                         // core tile
constexpr int kR1PX = kR1X + 4, kR1PY = kR1Y + 4;           // staged fhat plane: x0-2 .. x0+33, y0-2 .. y0+33
constexpr int kR1Plane = kR1PX * kR1PY;
constexpr int kR1PlaneStride = ((kR1Plane * 8 + 127) / 128) * 128 / 8;
constexpr int kR1Slots = 5;                                  // planes k .. k+2 in use, 2 in flight
constexpr int kR1Warps = 8;
constexpr int kR1Halo = kR1Y + 2;                            // 34 rows / columns of candidate centres
constexpr int kR1QCap = ((kR1Halo + kR1Warps - 1) / kR1Warps) * kR1Halo;   // rows w, w+8, ... of the halo region

struct R1Smem {
    double plane[kR1Slots][kR1PlaneStride];
    unsigned long long prop[3][kR1X * kR1Y];   // merged proposal keys of target planes (z % 3)
    uint16_t queue[kR1Warps][kR1QCap];         // (row << 6) | column in the 34 x 34 halo region
    unsigned long long full[kR1Slots];
    unsigned edits, maxc, shared;
};

struct R1Args {
    double* g;                    // out: corrected field (holds fhat already)
    const void* f;                // original (f32 or f64)
    const uint8_t* code;
    const uint32_t* det;          // detection bits of K0 (g = fhat)
    uint32_t* editbits;
    uint32_t* iteredit;
    DevCounters* ctr;
    int words_direct;             // nx % 32 == 0: a tile row is exactly one bitmap word
};

// Proposals of a queued centre: kept when the target lies in the CTA's box.
struct EmitR1 {
    const Dom& d;
    R1Smem& S;
    int x0, y0, zb, ze;
    __device__ __forceinline__ void operator()(int64_t t, double val) {
        int64_t tx, ty, tz;
        coords(d, t, tx, ty, tz);
        const int lx = (int)(tx - x0), ly = (int)(ty - y0);
        if (lx < 0 || lx >= kR1X || ly < 0 || ly >= kR1Y || tz < zb || tz >= ze) return;   // a neighbour's target
        atomicMin(&S.prop[(int)(tz % 3)][ly * kR1X + lx], okey(val));
    }
};

template <typename FT>
__global__ void __launch_bounds__(kR1Warps * 32, 2) k_rules1(Dom d, const __grid_constant__ CUtensorMap th, R1Args a,
                                                             int zchunk) {
    extern __shared__ __align__(1024) unsigned char r1raw[];
    R1Smem& S = *reinterpret_cast<R1Smem*>(r1raw);
    const int lane = threadIdx.x, wid = threadIdx.y, tid = wid * 32 + lane;
    const int x0 = (int)blockIdx.x * kR1X, y0 = (int)blockIdx.y * kR1Y;
    const int zb = (int)blockIdx.z * zchunk;
    const int ze = (int)min((int64_t)zb + zchunk, d.nz);
    const int K = ze - zb;
    const unsigned full0 = smem_u32(&S.full[0]), pl0 = smem_u32(&S.plane[0][0]);
    // staged plane index i <-> z = zb - 2 + i, i in [0, K + 3]
    auto issue = [&](int i) {
        const int s = i % kR1Slots;
        mbar_expect_tx(full0 + 8 * s, kR1Plane * 8);
        tma_load_3d(pl0 + s * kR1PlaneStride * 8, &th, x0 - 2, y0 - 2, zb - 2 + i, full0 + 8 * s);
    };
    auto wait_plane = [&](int i) { mbar_wait(full0 + 8 * (i % kR1Slots), (unsigned)((i / kR1Slots) & 1)); };
    for (int i = tid; i < 3 * kR1X * kR1Y; i += kR1Warps * 32) (&S.prop[0][0])[i] = kNoProposal;
    if (tid == 0) {
        for (int s = 0; s < kR1Slots; ++s) mbar_init(full0 + 8 * s, 1);
        mbar_fence_init();
        S.edits = S.maxc = S.shared = 0;
        for (int i = 0; i <= min(3, K + 3); ++i) issue(i);
    }
    __syncthreads();
    const uint32_t sy = (uint32_t)d.sy, sz = (uint32_t)d.sz;
    uint16_t* q = S.queue[wid];
    const unsigned below = (1u << lane) - 1u;
    unsigned myedits = 0;
    bool myshared = false;
    EmitR1 emit{d, S, x0, y0, zb, ze};
    for (int k = 0; k <= K + 1; ++k) {
        const int zc = zb - 1 + k;   // centre plane of this step: staged planes k, k + 1, k + 2
        wait_plane(k);
        wait_plane(k + 1);
        wait_plane(k + 2);
        // ---- the detected centres of the 34 x 34 halo region of plane zc ----
        unsigned n = 0;
        if (zc >= d.lo[2] && zc < d.hi[2]) {
            for (int ry = wid; ry < kR1Halo; ry += kR1Warps) {
                const int y = y0 - 1 + ry;
                const bool yok = y >= 0 && y < d.ny;
#pragma unroll
                for (int pass = 0; pass < 2; ++pass) {
                    const int cx = pass * 32 + lane;
                    const int x = x0 - 1 + cx;
                    bool hit = false;
                    if (yok && cx < kR1Halo && x >= 0 && x < d.nx) {
                        const uint32_t c = (uint32_t)x + (uint32_t)y * sy + (uint32_t)zc * sz;
                        hit = (__ldg(a.det + (c >> 5)) >> (c & 31)) & 1u;
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (hit) q[n + __popc(bal & below)] = (uint16_t)((ry << 6) | cx);
                    n += __popc(bal);
                }
            }
        }
        __syncwarp();
        // ---- their rules, one centre per lane, on the staged fhat ring ----
        const double* dn = S.plane[k % kR1Slots];
        const double* ct = S.plane[(k + 1) % kR1Slots];
        const double* up = S.plane[(k + 2) % kR1Slots];
        for (unsigned e = lane; e < n; e += 32) {
            const int ent = q[e];
            const int ry = ent >> 6, cx = ent & 63;
            const int x = x0 - 1 + cx, y = y0 - 1 + ry;
            const int64_t c = (int64_t)x + (int64_t)y * d.sy + (int64_t)zc * d.sz;
            double nv[14], vc;
            ring_from_smem(dn, ct, up, (ry + 1) * kR1PX + cx + 1, nv, vc);
            const bool interior = x > 0 && x + 1 < d.nx && y > 0 && y + 1 < d.ny && zc > 0 && zc + 1 < d.nz;
            const Scan s = interior ? tree_scan(vc, nv) : fold_scan(vc, nv);   // NaN = outside the field
            rules<false>(d, Work{}, s, nv, __ldg(a.code + c), c, emit);
        }
        __syncthreads();   // every proposal to target plane zc - 1 is merged
        // ---- apply target plane q = zc - 1 (staged plane k) ----
        const int qz = zc - 1;
        if (qz >= zb && qz < ze) {
            unsigned long long* pr = S.prop[qz % 3];
            const double* tp = S.plane[k % kR1Slots];
            const int x = x0 + lane;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int ly = wid * 4 + r, y = y0 + ly;
                const unsigned long long key = pr[ly * kR1X + lane];
                pr[ly * kR1X + lane] = kNoProposal;
                bool ed = false;
                const int64_t t = (int64_t)x + (int64_t)y * d.sy + (int64_t)qz * d.sz;
                if (key != kNoProposal && x < d.nx && y < d.ny) {
                    const double gt = tp[(ly + 2) * kR1PX + lane + 2];
                    const double fv = sizeof(FT) == 4 ? (double)__ldg((const float*)a.f + t) : __ldg((const double*)a.f + t);
                    const double p = okey_inv(key);
                    const double m = (p < gt) ? p : gt;                 // np.minimum(g, prop)
                    const double nvv = (m < fv - d.lxi) ? fv - d.lxi : m;   // np.maximum(., lower)
                    if (nvv != gt) {
                        a.g[t] = nvv;
                        ed = true;
                        myshared = myshared || in_shared(d, x, y, qz);
                    }
                }
                const unsigned bal = __ballot_sync(0xffffffffu, ed);
                myedits += ed ? 1u : 0u;
                if (bal) {
                    if (a.words_direct) {   // the row's word is this CTA's alone (zeroed for the run)
                        if (lane == 0) {
                            const uint32_t w0 = (uint32_t)((t - lane) >> 5);
                            a.editbits[w0] = bal;
                            if (a.iteredit) a.iteredit[w0] = bal;
                        }
                    } else if (ed) {
                        atomicOr(a.editbits + (t >> 5), 1u << (t & 31));
                        if (a.iteredit) atomicOr(a.iteredit + (t >> 5), 1u << (t & 31));
                    }
                }
            }
        }
        __syncthreads();   // the ring slot of plane zc - 1 is free again; staged plane k is done
        if (tid == 0 && k + 4 <= K + 3) issue(k + 4);
    }
    const unsigned we = __reduce_add_sync(0xffffffffu, myedits);
    const unsigned ws = __reduce_or_sync(0xffffffffu, myshared ? 1u : 0u);
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        a.ctr->scratch[3] = (unsigned long long)kMarkBits;   // the next iteration's dirty set: iteredit
    if (lane == 0) {
        if (we) atomicAdd(&a.ctr->nedits, (unsigned long long)we);
        if (we) atomicMax(&a.ctr->maxcount, 1ull);   // every edit of the first iteration is a first edit
        if (ws) atomicOr(&a.ctr->shared_dirty, 1ull);
    }
}

// Launch over the whole domain (targets anywhere in the ext extent; centres
// are the core box, whose detection bits K0 set).  False when a tensor map of
// fhat cannot be built (the caller takes the compaction + k_defer + apply path).
template <typename FT>
inline bool launch_rules1(const Dom& d, const double* fh, double* g, const FT* f, const uint8_t* code,
                          const uint32_t* det, uint32_t* editbits, uint32_t* iteredit, DevCounters* ctr,
                          cudaStream_t s) {
    CUtensorMap th;
    if (!tma_field_map(&th, fh, false, d.nx, d.ny, d.nz, kR1PX, kR1PY)) return false;
    R1Args a{g, f, code, det, editbits, iteredit, ctr, (d.nx % 32) == 0 ? 1 : 0};
    const int64_t tiles = ((d.nx + kR1X - 1) / kR1X) * ((d.ny + kR1Y - 1) / kR1Y);
    const int64_t want = (148 * 2 * 4 + tiles - 1) / tiles;
    int64_t chunks = std::max<int64_t>((d.nz + 31) / 32, std::min<int64_t>(want, d.nz / 8));
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, d.nz));
    const int zchunk = (int)std::max<int64_t>(1, (d.nz + chunks - 1) / chunks);
    chunks = (d.nz + zchunk - 1) / zchunk;
    const dim3 grid((unsigned)((d.nx + kR1X - 1) / kR1X), (unsigned)((d.ny + kR1Y - 1) / kR1Y), (unsigned)chunks);
    const size_t smem = sizeof(R1Smem);
    static bool attr = false;
    if (!attr) attr = cudaFuncSetAttribute(k_rules1<FT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
    k_rules1<FT><<<grid, dim3(32, kR1Warps, 1), smem, s>>>(d, th, a, zchunk);
    return true;
}

}  // namespace pmsz
