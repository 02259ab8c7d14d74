// tiles.cuh -- launch of the full-domain detection sweep (K1 / K4).
#pragma once
#include "sweep.cuh"

namespace pmsz {

template <bool kCount>
inline void launch_sweep_full(const Dom& d, const double* g, const Work& w, cudaStream_t s) {
    const int64_t cx = d.hi[0] - d.lo[0], cy = d.hi[1] - d.lo[1], cz = d.hi[2] - d.lo[2];
    dim3 block(32, 8, 1);
    dim3 grid((unsigned)((cx + 31) / 32), (unsigned)((cy + 7) / 8), (unsigned)cz);
    k_sweep_gather<kCount><<<grid, block, 0, s>>>(d, g, w);
}

}  // namespace pmsz
