/*
 * pmsz_oracle.c -- CPU ORACLE for the pMSz correction loop.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product.
 *
 * A plain-C restatement of the reference package topocorrect
 * (/root/reference/pkg/src/topocorrect, Python/NumPy).  Each function cites
 * the file:line it follows.  It is written in the reference's definition
 * form -- explicit (value, id) comparisons over the canonical STENCIL, dense
 * proposal arrays, dense Jacobi apply -- and shares no code or tie-break
 * shortcut with the GPU kernels (which use the rank-ordered form of SURVEY H2).
 *
 * Parity is pinned against the reference itself: tests/golden/make_golden.py
 * imports the reference in the build container and commits its outputs
 * (scan results, per-iteration g, run_correction results, run_parallel stats,
 * the golden edits-file hash) as fixtures under tests/golden/.
 *
 * Floating point: compiled with -O2 -ffp-contract=off (no FMA, no
 * reassociation), so perlin/quantize reproduce NumPy's elementwise IEEE
 * arithmetic bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* grid.py:24-32 -- canonical Freudenthal stencil (dx, dy, dz). */
static const int STENCIL[14][3] = {
    {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
    {1, 1, 0}, {-1, -1, 0}, {0, 1, 1}, {0, -1, -1}, {1, 0, 1}, {-1, 0, -1},
    {1, 1, 1}, {-1, -1, -1}};

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_BOUND = 2, ORC_MONOTONE = 3, ORC_CONVERGENCE = 4 };
enum { ORC_CONV_CAP = 1, ORC_CONV_BOUND = 2, ORC_CONV_RESIDUAL = 3, ORC_CONV_SEGMENTATION = 4 };

int orc_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* grid.py:111-118 -- strict total order: (value, id) lexicographic. */
static inline int precedes(const double* v, int64_t i, int64_t j) {
    return v[i] < v[j] || (v[i] == v[j] && i < j);
}

/* In-grid neighbour of (x,y,z) along stencil entry s, or -1. */
static inline int64_t nbr(int64_t nx, int64_t ny, int64_t nz, int64_t x, int64_t y, int64_t z, int s) {
    const int64_t px = x + STENCIL[s][0], py = y + STENCIL[s][1], pz = z + STENCIL[s][2];
    if (px < 0 || px >= nx || py < 0 || py >= ny || pz < 0 || pz >= nz) return -1;
    return px + nx * (py + ny * pz);
}

/* topology.py:47-86 (scan_neighbors); definition form of topology.py:93-121. */
void orc_scan(const double* v, int64_t nx, int64_t ny, int64_t nz, int64_t* nmax, int64_t* nmin,
              uint8_t* is_max, uint8_t* is_min) {
    const int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
        const int64_t x = c % nx, y = (c / nx) % ny, z = c / (nx * ny);
        int64_t hi = -1, lo = -1;
        for (int s = 0; s < 14; ++s) {
            const int64_t j = nbr(nx, ny, nz, x, y, z, s);
            if (j < 0) continue;
            if (hi < 0 || precedes(v, hi, j)) hi = j;
            if (lo < 0 || precedes(v, j, lo)) lo = j;
        }
        nmax[c] = hi;
        nmin[c] = lo;
        is_max[c] = (uint8_t)precedes(v, hi, c);   /* topology.py:79 */
        is_min[c] = (uint8_t)precedes(v, c, lo);   /* topology.py:80 */
    }
}

/* Atomic min of a double cell (proposal merge = np.minimum.at, correction.py:213-229). */
static inline void prop_min(double* prop, int64_t t, double val) {
#ifdef _OPENMP
    double cur;
    __atomic_load(&prop[t], &cur, __ATOMIC_RELAXED);
    while (val < cur) {
        if (__atomic_compare_exchange(&prop[t], &cur, &val, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) break;
    }
#else
    if (val < prop[t]) prop[t] = val;
#endif
}

typedef struct {
    int64_t *nmax, *nmin;
    uint8_t *is_max, *is_min;
} orc_scan_t;

/* _push_above_anchor (correction.py:183-204): g[a]-tau at every neighbour j of c
 * whose (g, id) key exceeds the anchor's. */
static void push_above(double* prop, const double* g, int64_t nx, int64_t ny, int64_t nz, int64_t c,
                       int64_t a, double tau) {
    const int64_t x = c % nx, y = (c / nx) % ny, z = c / (nx * ny);
    const double val = g[a] - tau;
    for (int s = 0; s < 14; ++s) {
        const int64_t j = nbr(nx, ny, nz, x, y, z, s);
        if (j < 0) continue;
        if (g[j] > g[a] || (g[j] == g[a] && j > a)) prop_min(prop, j, val);
    }
}

/* _kind_masks (correction.py:169-180) for one centre; bit k = DistortionKind rank k. */
static inline int kinds_of(const orc_scan_t* fs, const orc_scan_t* gs, int64_t c, int extrema_only) {
    int m = 0;
    if (gs->is_max[c] && !fs->is_max[c]) m |= 1;
    if (fs->is_max[c] && !gs->is_max[c]) m |= 2;
    if (gs->is_min[c] && !fs->is_min[c]) m |= 4;
    if (fs->is_min[c] && !gs->is_min[c]) m |= 8;
    if (!extrema_only) {
        if (!fs->is_max[c] && gs->nmax[c] != fs->nmax[c]) m |= 16;
        if (!fs->is_min[c] && gs->nmin[c] != fs->nmin[c]) m |= 32;
    }
    return m;
}

/*
 * _iterate_array (correction.py:232-242) incl. _proposal_array (:207-229).
 * g is updated in place; edited (optional) receives new_g != g; returns the
 * edit count, or -1 if the monotonicity assertion (:240-241) fires.
 * center_mask (optional) restricts detections to core centres (parallel.py).
 * kinds_out (optional) receives per-kind detection counts of this snapshot.
 */
int64_t orc_iterate(int64_t nx, int64_t ny, int64_t nz, const int64_t* f_nmax, const int64_t* f_nmin,
                    const uint8_t* f_ismax, const uint8_t* f_ismin, double* g, const double* lower,
                    double tau, const uint8_t* center_mask, uint8_t* edited, int extrema_only,
                    int64_t* kinds_out) {
    const int64_t n = nx * ny * nz;
    orc_scan_t fs = {(int64_t*)f_nmax, (int64_t*)f_nmin, (uint8_t*)f_ismax, (uint8_t*)f_ismin};
    orc_scan_t gs;
    gs.nmax = (int64_t*)malloc(n * sizeof(int64_t));
    gs.nmin = (int64_t*)malloc(n * sizeof(int64_t));
    gs.is_max = (uint8_t*)malloc(n);
    gs.is_min = (uint8_t*)malloc(n);
    orc_scan(g, nx, ny, nz, gs.nmax, gs.nmin, gs.is_max, gs.is_min);
    int64_t kinds[6] = {0, 0, 0, 0, 0, 0};
    int64_t any = 0;
#pragma omp parallel for reduction(+ : any) schedule(static)
    for (int64_t c = 0; c < n; ++c) {
        if (center_mask && !center_mask[c]) continue;
        if (kinds_of(&fs, &gs, c, extrema_only)) any += 1;
    }
    if (kinds_out) {
        for (int64_t c = 0; c < n; ++c) {
            if (center_mask && !center_mask[c]) continue;
            const int m = kinds_of(&fs, &gs, c, extrema_only);
            for (int k = 0; k < 6; ++k)
                if (m & (1 << k)) ++kinds[k];
        }
        memcpy(kinds_out, kinds, sizeof(kinds));
    }
    if (edited) memset(edited, 0, n);
    if (!any) { /* correction.py:236-237 early return */
        free(gs.nmax); free(gs.nmin); free(gs.is_max); free(gs.is_min);
        return 0;
    }
    double* prop = (double*)malloc(n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) prop[i] = INFINITY;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t c = 0; c < n; ++c) {
        if (center_mask && !center_mask[c]) continue;
        const int m = kinds_of(&fs, &gs, c, extrema_only);
        if (!m) continue;
        if (m & 1) prop_min(prop, c, g[fs.nmax[c]] - tau);              /* FALSE_MAXIMUM */
        if (m & 2) push_above(prop, g, nx, ny, nz, c, c, tau);           /* MISSING_MAXIMUM */
        if (m & 4) prop_min(prop, fs.nmin[c], g[c] - tau);              /* FALSE_MINIMUM */
        if (m & 8) prop_min(prop, c, g[gs.nmin[c]] - tau);              /* MISSING_MINIMUM */
        if (m & 16) push_above(prop, g, nx, ny, nz, c, fs.nmax[c], tau); /* ASC_ORDER */
        if (m & 32) prop_min(prop, fs.nmin[c], g[gs.nmin[c]] - tau);    /* DESC_ORDER */
    }
    int64_t edits = 0, raised = 0;
#pragma omp parallel for reduction(+ : edits, raised) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double m1 = g[i] < prop[i] ? g[i] : prop[i];     /* np.minimum(g, prop) */
        const double nv = m1 > lower[i] ? m1 : lower[i];       /* np.maximum(., lower) */
        if (nv > g[i]) raised += 1;
        if (nv != g[i]) {
            edits += 1;
            if (edited) edited[i] = 1;
        }
        prop[i] = nv;   /* reuse prop as new_g */
    }
    if (!raised) memcpy(g, prop, n * sizeof(double));
    free(prop);
    free(gs.nmax); free(gs.nmin); free(gs.is_max); free(gs.is_min);
    return raised ? -1 : edits;
}

/* Per-kind detection counts of g against the f-scan (the post-loop check,
 * correction.py:424-426).  Returns the total. */
int64_t orc_residual(int64_t nx, int64_t ny, int64_t nz, const int64_t* f_nmax, const int64_t* f_nmin,
                     const uint8_t* f_ismax, const uint8_t* f_ismin, const double* g, int extrema_only,
                     int64_t* kinds_out) {
    const int64_t n = nx * ny * nz;
    orc_scan_t fs = {(int64_t*)f_nmax, (int64_t*)f_nmin, (uint8_t*)f_ismax, (uint8_t*)f_ismin};
    orc_scan_t gs;
    gs.nmax = (int64_t*)malloc(n * sizeof(int64_t));
    gs.nmin = (int64_t*)malloc(n * sizeof(int64_t));
    gs.is_max = (uint8_t*)malloc(n);
    gs.is_min = (uint8_t*)malloc(n);
    orc_scan(g, nx, ny, nz, gs.nmax, gs.nmin, gs.is_max, gs.is_min);
    int64_t kinds[6] = {0, 0, 0, 0, 0, 0}, total = 0;
    for (int64_t c = 0; c < n; ++c) {
        const int m = kinds_of(&fs, &gs, c, extrema_only);
        for (int k = 0; k < 6; ++k)
            if (m & (1 << k)) { ++kinds[k]; ++total; }
    }
    if (kinds_out) memcpy(kinds_out, kinds, sizeof(kinds));
    free(gs.nmax); free(gs.nmin); free(gs.is_max); free(gs.is_min);
    return total;
}

/* _pointer_fixpoint + compute_segmentation (topology.py:156-174). */
void orc_segmentation(const double* v, int64_t nx, int64_t ny, int64_t nz, int64_t* asc_target,
                      int64_t* desc_target) {
    const int64_t n = nx * ny * nz;
    int64_t* nmax = (int64_t*)malloc(n * sizeof(int64_t));
    int64_t* nmin = (int64_t*)malloc(n * sizeof(int64_t));
    uint8_t* ismax = (uint8_t*)malloc(n);
    uint8_t* ismin = (uint8_t*)malloc(n);
    int64_t* tmp = (int64_t*)malloc(n * sizeof(int64_t));
    orc_scan(v, nx, ny, nz, nmax, nmin, ismax, ismin);
    for (int64_t i = 0; i < n; ++i) {
        desc_target[i] = ismax[i] ? i : nmax[i];   /* up */
        asc_target[i] = ismin[i] ? i : nmin[i];    /* down */
    }
    int64_t* arrs[2] = {asc_target, desc_target};
    for (int k = 0; k < 2; ++k) {
        int64_t* s = arrs[k];
        for (;;) {
            int64_t changed = 0;
#pragma omp parallel for reduction(+ : changed) schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                tmp[i] = s[s[i]];
                changed += tmp[i] != s[i];
            }
            memcpy(s, tmp, n * sizeof(int64_t));
            if (!changed) break;
        }
    }
    free(nmax); free(nmin); free(ismax); free(ismin); free(tmp);
}

/*
 * run_correction (correction.py:391-436) without the Python result objects.
 * g_out receives the corrected field; history receives edits_per_iteration.
 * Returns ORC_* status; on ORC_BOUND, *bound_first / *bound_count are set; on
 * ORC_CONVERGENCE, *conv_kind says which check failed.
 */
int orc_run_correction(int64_t nx, int64_t ny, int64_t nz, const double* f, const double* fh, double xi,
                       double tau, int64_t max_iter, int extrema_only, double* g_out, int64_t* history,
                       int64_t hist_cap, int64_t* iterations, int64_t* max_vertex_edits,
                       int64_t* bound_first, int64_t* bound_count, int64_t* conv_kind, int check_segmentation) {
    const int64_t n = nx * ny * nz;
    *iterations = 0;
    *max_vertex_edits = 0;
    *conv_kind = 0;
    /* validate_error_bound (correction.py:52-60) */
    int64_t first = -1, count = 0;
    for (int64_t i = 0; i < n; ++i)
        if (fabs(f[i] - fh[i]) > xi) {
            if (first < 0) first = i;
            ++count;
        }
    if (count) {
        *bound_first = first;
        *bound_count = count;
        return ORC_BOUND;
    }
    /* BoundsField.from_field (correction.py:118-122) */
    double* lower = (double*)malloc(n * sizeof(double));
    double* upper = (double*)malloc(n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        lower[i] = f[i] - xi;
        upper[i] = f[i] + xi;
    }
    int64_t* fnmax = (int64_t*)malloc(n * sizeof(int64_t));
    int64_t* fnmin = (int64_t*)malloc(n * sizeof(int64_t));
    uint8_t* fismax = (uint8_t*)malloc(n);
    uint8_t* fismin = (uint8_t*)malloc(n);
    orc_scan(f, nx, ny, nz, fnmax, fnmin, fismax, fismin);
    memcpy(g_out, fh, n * sizeof(double));
    int64_t* counts = (int64_t*)calloc(n, sizeof(int64_t));
    uint8_t* edited = (uint8_t*)malloc(n);
    int status = ORC_OK, converged = 0;
    int64_t it = 0;
    for (; it < max_iter; ++it) {
        const int64_t e = orc_iterate(nx, ny, nz, fnmax, fnmin, fismax, fismin, g_out, lower, tau, NULL,
                                      edited, extrema_only, NULL);
        if (e < 0) {
            status = ORC_MONOTONE;
            break;
        }
        if (history && it < hist_cap) history[it] = e;
        if (e == 0) {
            converged = 1;
            ++it;
            break;
        }
        for (int64_t i = 0; i < n; ++i) counts[i] += edited[i];
    }
    *iterations = it;
    for (int64_t i = 0; i < n; ++i)
        if (counts[i] > *max_vertex_edits) *max_vertex_edits = counts[i];
    if (status == ORC_OK && !converged) {
        status = ORC_CONVERGENCE;
        *conv_kind = ORC_CONV_CAP;
    }
    if (status == ORC_OK) { /* bounds.admits (correction.py:422-423) */
        for (int64_t i = 0; i < n; ++i)
            if (!(g_out[i] >= lower[i] && g_out[i] <= upper[i])) {
                status = ORC_CONVERGENCE;
                *conv_kind = ORC_CONV_BOUND;
                break;
            }
    }
    if (status == ORC_OK) { /* correction.py:424-426 */
        if (orc_residual(nx, ny, nz, fnmax, fnmin, fismax, fismin, g_out, extrema_only, NULL)) {
            status = ORC_CONVERGENCE;
            *conv_kind = ORC_CONV_RESIDUAL;
        }
    }
    if (status == ORC_OK && check_segmentation && !extrema_only) { /* compare_plmss (correction.py:427-429) */
        int64_t* a1 = (int64_t*)malloc(n * sizeof(int64_t));
        int64_t* d1 = (int64_t*)malloc(n * sizeof(int64_t));
        int64_t* a2 = (int64_t*)malloc(n * sizeof(int64_t));
        int64_t* d2 = (int64_t*)malloc(n * sizeof(int64_t));
        orc_segmentation(f, nx, ny, nz, a1, d1);
        orc_segmentation(g_out, nx, ny, nz, a2, d2);
        for (int64_t i = 0; i < n; ++i)
            if (a1[i] != a2[i] || d1[i] != d2[i]) {
                status = ORC_CONVERGENCE;
                *conv_kind = ORC_CONV_SEGMENTATION;
                break;
            }
        free(a1); free(d1); free(a2); free(d2);
    }
    free(lower); free(upper); free(fnmax); free(fnmin); free(fismax); free(fismin);
    free(counts); free(edited);
    return status;
}

/* ---- synthetic inputs ------------------------------------------------------ */
/* synth.py:40-52 */
static double fade(double t) { return t * t * t * (t * (t * 6.0 - 15.0) + 10.0); }
static double grad(int64_t h, double x, double y, double z) {
    h = h & 15;
    const double u = h < 8 ? x : y;
    const double v = h < 4 ? y : ((h == 12 || h == 14) ? x : z);
    return ((h & 1) == 0 ? u : -u) + ((h & 2) == 0 ? v : -v);
}
static double lerp(double a, double b, double t) { return a + t * (b - a); }

/* synth.py:55-80 */
static double noise3(double px, double py, double pz, const int32_t* perm) {
    const int64_t xi0 = (int64_t)floor(px), yi0 = (int64_t)floor(py), zi0 = (int64_t)floor(pz);
    const double xf = px - (double)xi0, yf = py - (double)yi0, zf = pz - (double)zi0;
    const int64_t xi = xi0 & 255, yi = yi0 & 255, zi = zi0 & 255;
    const double u = fade(xf), v = fade(yf), w = fade(zf);
    const int64_t pa = perm[xi] + yi, pb = perm[xi + 1] + yi;
    const int64_t paa = perm[pa] + zi, pab = perm[pa + 1] + zi;
    const int64_t pba = perm[pb] + zi, pbb = perm[pb + 1] + zi;
    double x1 = lerp(grad(perm[paa], xf, yf, zf), grad(perm[pba], xf - 1, yf, zf), u);
    double x2 = lerp(grad(perm[pab], xf, yf - 1, zf), grad(perm[pbb], xf - 1, yf - 1, zf), u);
    const double y1 = lerp(x1, x2, v);
    x1 = lerp(grad(perm[paa + 1], xf, yf, zf - 1), grad(perm[pba + 1], xf - 1, yf, zf - 1), u);
    x2 = lerp(grad(perm[pab + 1], xf, yf - 1, zf - 1), grad(perm[pbb + 1], xf - 1, yf - 1, zf - 1), u);
    const double y2 = lerp(x1, x2, v);
    return lerp(y1, y2, w);
}

/* synth.py:83-100, restricted to the sub-box [lo, lo+ext) of the global grid. */
void orc_perlin(const int64_t* gdims, const int64_t* lo, const int64_t* ext, const int32_t* perm512,
                double frequency, int32_t octaves, double* out) {
    const int64_t n = ext[0] * ext[1] * ext[2];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t lz = i / (ext[0] * ext[1]), r = i - lz * ext[0] * ext[1];
        const int64_t ly = r / ext[0], lx = r - ly * ext[0];
        const double xx = (double)(lo[0] + lx), yy = (double)(lo[1] + ly), zz = (double)(lo[2] + lz);
        double total = 0.0, amp_sum = 0.0;
        for (int o = 0; o < octaves; ++o) {
            const double freq = frequency * ldexp(1.0, o);
            const double amp = ldexp(1.0, -o);
            const double px = xx * (freq / (double)gdims[0]);
            const double py = yy * (freq / (double)gdims[1]);
            const double pz = gdims[2] > 1 ? zz * (freq / (double)gdims[2]) : 0.0;
            total = total + amp * noise3(px, py, pz, perm512);
            amp_sum = amp_sum + amp;
        }
        out[i] = total / amp_sum;
    }
}

/* quantize (quantizer.py:122-154); returns 0, or -1 if the self-check fails.
 * origin = min(f) unless use_origin (a sub-box of a larger field passes the
 * whole field's minimum so the sample equals the slice of the whole). */
int orc_quantize(const double* f, int64_t n, double xi, double origin_in, int use_origin, double* recon) {
    double origin = f[0];
    for (int64_t i = 1; i < n; ++i)
        if (f[i] < origin) origin = f[i];
    if (use_origin) origin = origin_in;
    const double two_xi = 2.0 * xi;
    int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int64_t code = (int64_t)nearbyint((f[i] - origin) / two_xi);
        double r = origin + (double)code * two_xi;
        code += (f[i] - r > xi) ? 1 : 0;
        code -= (r - f[i] > xi) ? 1 : 0;
        r = origin + (double)code * two_xi;
        if (fabs(f[i] - r) > xi || code < 0) bad |= 1;
        recon[i] = r;
    }
    return bad ? -1 : 0;
}

/* Seeded bounded noise of BASELINE config 1 (no reference counterpart):
 * fhat = clamp(f + xi*s, f - xi, f + xi), s in [-1,1) from a splitmix64 hash of
 * (seed, global id); re-validated so |f - fhat| <= xi and fhat >= f - xi (H6). */
static uint64_t mix64(uint64_t seed, uint64_t id) {
    uint64_t z = seed + (id + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void orc_bounded_noise(const double* f, int64_t nx, int64_t ny, int64_t nz, const int64_t* gdims,
                       const int64_t* lo, double xi, uint64_t seed, double* out) {
    const int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t z = i / (nx * ny), r = i - z * nx * ny, y = r / nx, x = r - y * nx;
        const int64_t gid = (lo[0] + x) + gdims[0] * ((lo[1] + y) + gdims[1] * (lo[2] + z));
        const double u = (double)(mix64(seed, (uint64_t)gid) >> 11) * 0x1.0p-53;
        const double s = u * 2.0 - 1.0;
        const double fv = f[i], lo_b = fv - xi, hi_b = fv + xi;
        double v = fv + xi * s;
        v = v < lo_b ? lo_b : v;
        v = v > hi_b ? hi_b : v;
        if (fabs(fv - v) > xi || v < lo_b) v = fv;
        out[i] = v;
    }
}

/* ---- HEDM-like Gaussian-peak stack (BASELINE config 5) ---------
 * The generator is new (the reference has none); this is its CPU definition,
 * written operation by operation like gen.cuh's peak_value so both produce
 * the same bits (no contraction here, --fmad=false there). */
static double det_exp(double x) {
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

static double peak_u(uint64_t seed, uint64_t cell, int k) {
    return (double)(mix64(seed ^ 0x5EEDC0DEULL, cell * 8ull + (uint64_t)k) >> 11) * 0x1.0p-53;
}

static double peak_value(const int64_t* gd, uint64_t seed, int64_t x, int64_t y, int64_t z) {
    const int64_t CX = 64, CY = 64, CZ = 32;
    const int64_t ncx = (gd[0] + CX - 1) / CX, ncy = (gd[1] + CY - 1) / CY;
    const int64_t cx = x / CX, cy = y / CY, cz = z / CZ;
    const uint64_t cell = (uint64_t)(cx + ncx * (cy + ncy * cz));
    const uint64_t gid = (uint64_t)(x + gd[0] * (y + gd[1] * z));
    const double bg = 0.02 * ((double)(mix64(seed, gid) >> 11) * 0x1.0p-53);
    if (!(peak_u(seed, cell, 0) < 0.6)) return bg;
    const double amp = 0.2 + 0.8 * peak_u(seed, cell, 1);
    const double sx = 1.0 + 2.0 * peak_u(seed, cell, 2);
    const double sy = 1.0 + 2.0 * peak_u(seed, cell, 3);
    const double sz = 0.7 + 1.3 * peak_u(seed, cell, 4);
    const double px = (double)(cx * CX) + 12.0 + peak_u(seed, cell, 5) * (double)(CX - 24);
    const double py = (double)(cy * CY) + 12.0 + peak_u(seed, cell, 6) * (double)(CY - 24);
    const double pz = (double)(cz * CZ) + 8.0 + peak_u(seed, cell, 7) * (double)(CZ - 16);
    const double dx = (double)x - px, dy = (double)y - py, dz = (double)z - pz;
    if (fabs(dx) > 4.0 * sx || fabs(dy) > 4.0 * sy || fabs(dz) > 4.0 * sz) return bg;
    const double q = (dx * dx) / (2.0 * sx * sx) + (dy * dy) / (2.0 * sy * sy) + (dz * dz) / (2.0 * sz * sz);
    return bg + amp * det_exp(-q);
}

void orc_peaks(const int64_t* gdims, const int64_t* lo, const int64_t* ext, uint64_t seed, double* out) {
    const int64_t n = ext[0] * ext[1] * ext[2];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t z = i / (ext[0] * ext[1]), r = i - z * ext[0] * ext[1], y = r / ext[0], x = r - y * ext[0];
        out[i] = peak_value(gdims, seed, lo[0] + x, lo[1] + y, lo[2] + z);
    }
}
