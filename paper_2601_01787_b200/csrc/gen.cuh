// gen.cuh -- input generation and small utility kernels.
//
// perlin   : synth.perlin (synth.py:33-100), bit-exact.  The library is built
//            with --fmad=false so no a+b*c is contracted and every
//            expression below evaluates in the same order as the NumPy code.
// quantize : quantizer.quantize (quantizer.py:122-154) incl. the ulp repair.
// noise    : the seeded bounded-noise stand-in of BASELINE config 1 (new; the
//            oracle's C restatement uses the identical counter hash).
#pragma once
#include "common.cuh"

namespace pmsz {

__device__ __forceinline__ double p_fade(double t) {
    return t * t * t * (t * (t * 6.0 - 15.0) + 10.0);
}
__device__ __forceinline__ double p_grad(int h, double x, double y, double z) {
    h &= 15;
    const double u = h < 8 ? x : y;
    const double v = h < 4 ? y : ((h == 12 || h == 14) ? x : z);
    return ((h & 1) == 0 ? u : -u) + ((h & 2) == 0 ? v : -v);
}
__device__ __forceinline__ double p_lerp(double a, double b, double t) { return a + t * (b - a); }

__device__ double p_noise3(double px, double py, double pz, const int* __restrict__ perm) {
    const double fx0 = floor(px), fy0 = floor(py), fz0 = floor(pz);
    const long long xi0 = (long long)fx0, yi0 = (long long)fy0, zi0 = (long long)fz0;
    const double xf = px - (double)xi0, yf = py - (double)yi0, zf = pz - (double)zi0;
    const int xi = (int)(xi0 & 255), yi = (int)(yi0 & 255), zi = (int)(zi0 & 255);
    const double u = p_fade(xf), v = p_fade(yf), w = p_fade(zf);
    const int pa = perm[xi] + yi, pb = perm[xi + 1] + yi;
    const int paa = perm[pa] + zi, pab = perm[pa + 1] + zi;
    const int pba = perm[pb] + zi, pbb = perm[pb + 1] + zi;
    double x1 = p_lerp(p_grad(perm[paa], xf, yf, zf), p_grad(perm[pba], xf - 1, yf, zf), u);
    double x2 = p_lerp(p_grad(perm[pab], xf, yf - 1, zf), p_grad(perm[pbb], xf - 1, yf - 1, zf), u);
    const double y1 = p_lerp(x1, x2, v);
    x1 = p_lerp(p_grad(perm[paa + 1], xf, yf, zf - 1), p_grad(perm[pba + 1], xf - 1, yf, zf - 1), u);
    x2 = p_lerp(p_grad(perm[pab + 1], xf, yf - 1, zf - 1),
                p_grad(perm[pbb + 1], xf - 1, yf - 1, zf - 1), u);
    const double y2 = p_lerp(x1, x2, v);
    return p_lerp(y1, y2, w);
}

struct PerlinArgs {
    int64_t gdims[3], lo[3], ext[3];
    double scale[3];   // freq/n per octave-0 axis is recomputed per octave
    double frequency;
    int octaves;
};

__global__ void __launch_bounds__(256) k_perlin(PerlinArgs a, const int* __restrict__ perm_g,
                                               double* __restrict__ out64, float* __restrict__ out32) {
    __shared__ int perm[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) perm[i] = perm_g[i];
    __syncthreads();
    const int64_t n = a.ext[0] * a.ext[1] * a.ext[2];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lz = i / (a.ext[0] * a.ext[1]);
        const int64_t r = i - lz * a.ext[0] * a.ext[1];
        const int64_t ly = r / a.ext[0];
        const int64_t lx = r - ly * a.ext[0];
        const double xx = (double)(a.lo[0] + lx), yy = (double)(a.lo[1] + ly), zz = (double)(a.lo[2] + lz);
        double total = 0.0, amp_sum = 0.0;
        double pw = 1.0, amp = 1.0;   // 2.0**o, 0.5**o (exact powers)
        for (int o = 0; o < a.octaves; ++o) {
            const double freq = a.frequency * pw;
            const double px = xx * (freq / (double)a.gdims[0]);
            const double py = yy * (freq / (double)a.gdims[1]);
            const double pz = a.gdims[2] > 1 ? zz * (freq / (double)a.gdims[2]) : 0.0;
            total = total + amp * p_noise3(px, py, pz, perm);
            amp_sum = amp_sum + amp;
            pw = pw * 2.0;
            amp = amp * 0.5;
        }
        const double v = total / amp_sum;
        if (out64) out64[i] = v;
        if (out32) out32[i] = __double2float_rn(v);
    }
}

template <typename FT>
__global__ void __launch_bounds__(256) k_minmax(const FT* __restrict__ v, int64_t n,
                                               unsigned long long* mn_key, unsigned long long* mx_key) {
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = (double)v[i];
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
    }
    // -0.0 and +0.0: keep the reference's float(min) semantics irrelevant here
    // because only hi-lo and origin=min are used; +0.0 canonicalised.
    lo = lo + 0.0; hi = hi + 0.0;
    unsigned long long klo = okey(lo), khi = okey(hi);
    for (int o = 16; o; o >>= 1) {
        klo = min(klo, __shfl_xor_sync(0xffffffffu, klo, o));
        khi = max(khi, __shfl_xor_sync(0xffffffffu, khi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mn_key, klo);
        atomicMax(mx_key, khi);
    }
}

template <typename FT>
__global__ void __launch_bounds__(256) k_quantize(const FT* __restrict__ f, int64_t n, double origin,
                                                 double xi, double two_xi, double* __restrict__ recon,
                                                 unsigned long long* maxcode, unsigned long long* fails,
                                                 unsigned long long* __restrict__ codes) {
    unsigned long long my_max = 0, my_fail = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double fv = (double)f[i];
        long long code = (long long)rint((fv - origin) / two_xi);       // quantizer.py:136
        double r = origin + (double)code * two_xi;                      // quantizer.py:119
        code += (fv - r > xi) ? 1 : 0;                                  // quantizer.py:139-140
        code -= (r - fv > xi) ? 1 : 0;
        r = origin + (double)code * two_xi;
        if (fabs(fv - r) > xi || code < 0) ++my_fail;                   // quantizer.py:142-145
        recon[i] = r;
        if (codes) codes[i] = (unsigned long long)code;                  // QuantizedPayload.codes
        my_max = max(my_max, (unsigned long long)(code < 0 ? 0 : code));
    }
    for (int o = 16; o; o >>= 1) {
        my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
        my_fail += __shfl_xor_sync(0xffffffffu, my_fail, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(maxcode, my_max);
        if (my_fail) atomicAdd(fails, my_fail);
    }
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t id) {
    uint64_t z = seed + (id + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename FT>
__global__ void __launch_bounds__(256) k_bounded_noise(const FT* __restrict__ f, int64_t nx, int64_t ny,
                                                      int64_t nz, int64_t gnx, int64_t gny, int64_t lox,
                                                      int64_t loy, int64_t loz, double xi, uint64_t seed,
                                                      double* __restrict__ out) {
    const int64_t n = nx * ny * nz;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / (nx * ny), r = i - z * nx * ny, y = r / nx, x = r - y * nx;
        const int64_t gid = (lox + x) + gnx * ((loy + y) + gny * (loz + z));
        const double u = (double)(mix64(seed, (uint64_t)gid) >> 11) * 0x1.0p-53;   // [0,1)
        const double s = u * 2.0 - 1.0;                                           // [-1,1)
        const double fv = (double)f[i];
        const double lo = fv - xi, hi = fv + xi;
        double v = fv + xi * s;
        v = v < lo ? lo : v;
        v = v > hi ? hi : v;
        if (fabs(fv - v) > xi || v < lo) v = fv;   // re-validate
        out[i] = v;
    }
}

// ---- HEDM-like Gaussian-peak stack (BASELINE config 5) ----------
// Not in the reference: a stack of detector frames (z) with sparse Gaussian
// diffraction spots over a faint hash-noise background.  The domain is cut
// into cells of (64, 64, 32) voxels; a cell holds one peak with probability
// 0.6, of amplitude A in [0.2, 1), widths sx, sy in [1, 3), sz in [0.7, 2)
// and a centre kept >= 4 sigma from the cell faces, truncated at 4 sigma:
//   v = bg + A * exp(-(dx^2/(2 sx^2) + dy^2/(2 sy^2) + dz^2/(2 sz^2)))
// All arithmetic is +, -, *, / in a fixed order plus det_exp (Cody-Waite
// reduction + degree-11 Horner + ldexp), so the oracle (C, no contraction)
// and this kernel (--fmad=false) produce identical bits.
struct PeakArgs {
    int64_t gnx, gny, gnz;        // global dims
    int64_t lox, loy, loz;        // sub-box origin
    int64_t nx, ny, nz;           // sub-box extents
    uint64_t seed;
};
constexpr int64_t kPeakCX = 64, kPeakCY = 64, kPeakCZ = 32;

__host__ __device__ __forceinline__ double det_exp(double x) {
    if (x < -700.0) return 0.0;
    const double kf = floor(x * 1.4426950408889634 + 0.5);
    const double r = (x - kf * 0.6931471803691238) - kf * 1.9082149292705877e-10;
    double p = 2.505210838544172e-08;
    p = p * r + 2.755731922398589e-07;
    p = p * r + 2.7557319223985893e-06;
    p = p * r + 2.48015873015873e-05;
    p = p * r + 0.0001984126984126984;
    p = p * r + 0.001388888888888889;
    p = p * r + 0.008333333333333333;
    p = p * r + 0.041666666666666664;
    p = p * r + 0.16666666666666666;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    return ldexp(p, (int)kf);
}

__host__ __device__ __forceinline__ double peak_u(uint64_t seed, uint64_t cell, int k) {
    return (double)(mix64(seed ^ 0x5EEDC0DEULL, cell * 8ull + (uint64_t)k) >> 11) * 0x1.0p-53;
}

__host__ __device__ __forceinline__ double peak_value(const PeakArgs& a, int64_t x, int64_t y, int64_t z) {
    const int64_t ncx = (a.gnx + kPeakCX - 1) / kPeakCX, ncy = (a.gny + kPeakCY - 1) / kPeakCY;
    const int64_t cx = x / kPeakCX, cy = y / kPeakCY, cz = z / kPeakCZ;
    const uint64_t cell = (uint64_t)(cx + ncx * (cy + ncy * cz));
    const uint64_t gid = (uint64_t)(x + a.gnx * (y + a.gny * z));
    const double bg = 0.02 * ((double)(mix64(a.seed, gid) >> 11) * 0x1.0p-53);
    if (!(peak_u(a.seed, cell, 0) < 0.6)) return bg;
    const double amp = 0.2 + 0.8 * peak_u(a.seed, cell, 1);
    const double sx = 1.0 + 2.0 * peak_u(a.seed, cell, 2);
    const double sy = 1.0 + 2.0 * peak_u(a.seed, cell, 3);
    const double sz = 0.7 + 1.3 * peak_u(a.seed, cell, 4);
    const double px = (double)(cx * kPeakCX) + 12.0 + peak_u(a.seed, cell, 5) * (double)(kPeakCX - 24);
    const double py = (double)(cy * kPeakCY) + 12.0 + peak_u(a.seed, cell, 6) * (double)(kPeakCY - 24);
    const double pz = (double)(cz * kPeakCZ) + 8.0 + peak_u(a.seed, cell, 7) * (double)(kPeakCZ - 16);
    const double dx = (double)x - px, dy = (double)y - py, dz = (double)z - pz;
    if (fabs(dx) > 4.0 * sx || fabs(dy) > 4.0 * sy || fabs(dz) > 4.0 * sz) return bg;
    const double q = (dx * dx) / (2.0 * sx * sx) + (dy * dy) / (2.0 * sy * sy) + (dz * dz) / (2.0 * sz * sz);
    return bg + amp * det_exp(-q);
}

template <typename OT>
__global__ void __launch_bounds__(256) k_peaks(PeakArgs a, OT* __restrict__ out) {
    const int64_t n = a.nx * a.ny * a.nz;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / (a.nx * a.ny), r = i - z * a.nx * a.ny, y = r / a.nx, x = r - y * a.nx;
        out[i] = (OT)peak_value(a, a.lox + x, a.loy + y, a.loz + z);
    }
}

}  // namespace pmsz
