/*
 * pmsz.h -- C ABI of the B200-native pMSz correction loop.
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json: the
 * reference package `topocorrect` (Python/NumPy, /root/reference/pkg) exposes
 * the path as Python functions, not as an FFI, so every entry point below is
 * the C-level equivalent of one reference function, cited by file:line
 * (paths relative to /root/reference/pkg/src/topocorrect/).  The Python
 * mirror in paper_2601_01787_b200/ binds these symbols with ctypes (see
 * INTEGRATION.md for the stub a maintainer would add on the reference side).
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch types.  Pointers suffixed _dev
 *    are CUDA device pointers, _host are host pointers.  `stream` is a
 *    cudaStream_t passed as void*.  NULL stream = legacy default stream.
 *  - Fields are flat, x fastest: id = x + nx*(y + ny*z) (grid.py:9-13,85-89).
 *  - Values are f64 (grid.py:57).  The original field f may be passed as f32
 *    when the caller knows it is f32-exact (codec.py:86-87 promotion is exact).
 *  - Every function returns a pmsz_status; details of the last error on the
 *    calling thread are available from pmsz_last_error().
 */
#ifndef PMSZ_H
#define PMSZ_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PMSZ_OK = 0,
    PMSZ_ERR_INVALID = 1,      /* ValueError: dims/config/grid (correction.py:54-55,77-91) */
    PMSZ_ERR_BOUND = 2,        /* BoundViolationError (correction.py:33-45,52-60) */
    PMSZ_ERR_MONOTONE = 3,     /* AssertionError "edit raised a value" (correction.py:240-241) */
    PMSZ_ERR_CONVERGENCE = 4,  /* ConvergenceError (correction.py:48-49,417-429) */
    PMSZ_ERR_CUDA = 5,         /* CUDA runtime failure */
    PMSZ_ERR_NONFINITE = 6,    /* ValueError "field values must all be finite" (grid.py:62-63) */
    PMSZ_ERR_INEXACT = 7       /* PMSZ_FLAG_HOST_F64: the f64 original did not narrow exactly to
                                  float32 -- no error in the reference; rerun with an f64 plan */
} pmsz_status;

/* ConvergenceError sub-kinds, reported in pmsz_result.convergence_kind. */
enum {
    PMSZ_CONV_NONE = 0,
    PMSZ_CONV_CAP = 1,       /* "no zero-edit iteration within cap"        correction.py:417-419 */
    PMSZ_CONV_BOUND = 2,     /* "corrected field escaped the error bound"  correction.py:422-423 */
    PMSZ_CONV_RESIDUAL = 3   /* "distortions survived a zero-edit iteration" correction.py:424-426 */
};

/* Plan flags. */
enum {
    PMSZ_FLAG_INCREMENTAL = 1,   /* dirty-ring sweeps after the first (exact) */
    PMSZ_FLAG_EXTREMA_ONLY = 2,  /* drop the two order kinds (BASELINE config 5) */
    PMSZ_FLAG_F32_ORIGINAL = 4,  /* f is passed as float32 (exact promotion) */
    PMSZ_FLAG_HOST_LOOP = 8,     /* no device-resident tail: every iteration is launched
                                    and synchronised from the host (A/B and tests) */
    PMSZ_FLAG_NO_ROBUST = 16,    /* evaluate every centre: required when g may leave
                                    [f - xi, f + xi] (local_converge on arbitrary inputs) */
    PMSZ_FLAG_LOWER = 32,        /* pmsz_iterate / pmsz_block_round receive the f64 lower
                                    bound L itself in place of f (local_converge's lower_ext,
                                    parallel.py:150-172): the apply clamps to L, not f - xi */
    PMSZ_FLAG_HOST_F64 = 64      /* with PMSZ_FLAG_F32_ORIGINAL: pmsz_run_correction_host gets an
                                    f64 host original and narrows it while staging; returns
                                    PMSZ_ERR_INEXACT (before any iteration) when a value does
                                    not round-trip (the reference's ScalarField is always f64,
                                    grid.py:57; fields read from f32 files narrow exactly) */
};

/* Distortion kinds, in the reference declaration order (correction.py:133-139). */
enum {
    PMSZ_KIND_FALSE_MAX = 0, PMSZ_KIND_MISSING_MAX = 1,
    PMSZ_KIND_FALSE_MIN = 2, PMSZ_KIND_MISSING_MIN = 3,
    PMSZ_KIND_ASC_ORDER = 4, PMSZ_KIND_DESC_ORDER = 5
};

/*
 * One correction domain: the whole grid (run_correction) or one block's
 * extended extent (parallel.py:43-82).  Centers are restricted to the core
 * box [core_lo, core_hi) given in the domain's own coordinates
 * (the reference's `center_mask`, correction.py:169-180, parallel.py:73-77).
 * shared_lo/shared_hi give, per axis, the width (0 or 2) of the band at the
 * low/high face whose vertices are replicated in a neighbouring block
 * (`_replicated_mask_zyx`, parallel.py:228-234); edits there raise
 * shared_dirty (parallel.py:249-250).
 */
typedef struct {
    int64_t nx, ny, nz;
    int64_t core_lo[3];
    int64_t core_hi[3];
    int32_t shared_lo[3];
    int32_t shared_hi[3];
    double xi;                 /* CorrectionConfig.xi_abs (correction.py:63-96) */
    double tau;                /* CorrectionConfig.tau */
    int64_t max_iterations;    /* CorrectionConfig.max_outer_iterations */
    int32_t flags;             /* PMSZ_FLAG_* */
    int32_t reserved;
} pmsz_desc;

typedef struct pmsz_plan pmsz_plan;

/* Counters of one run / one iteration (all on the host after the call). */
typedef struct {
    int64_t iterations;            /* CorrectionResult.iterations */
    int64_t edit_count;            /* |EditSet| */
    int64_t max_vertex_edits;      /* CorrectionResult.max_vertex_edits */
    int64_t bound_violations;      /* BoundViolationError.offenders */
    int64_t bound_first_index;     /* BoundViolationError.index */
    int64_t floor_violations;      /* fhat < f - xi (hazard H6) */
    int64_t nonfinite;             /* non-finite inputs */
    int64_t residual[6];           /* detections left by the final sweep, per kind */
    int64_t convergence_kind;      /* PMSZ_CONV_* */
    int64_t full_sweeps;           /* full-grid detection sweeps executed (incl. verify) */
    int64_t sparse_sweeps;         /* dirty-ring sweeps executed */
    int64_t shared_dirty;          /* block mode: an edit touched a replicated vertex */
    int64_t last_edits;            /* edits of the last iteration */
    int64_t last_detections;       /* centres with a detection in the last iteration */
    int64_t masked_sweeps;         /* tiled sweeps restricted to a dilated dirty bitmap */
    int64_t fragile;               /* centres K0 found not robust (the only ones ever evaluated) */
} pmsz_result;

/* Error string of the last failing call on this thread. */
const char* pmsz_last_error(void);
/* Library version string. */
const char* pmsz_version(void);
/* Number of kernel launches issued by this library since load (evidence for bench). */
int64_t pmsz_launch_count(void);

/* Kernel classes for pmsz_profile_read. */
enum {
    PMSZ_K_PREP = 0, PMSZ_K_SWEEP_FULL = 1, PMSZ_K_SWEEP_SPARSE = 2, PMSZ_K_APPLY = 3,
    PMSZ_K_VERIFY = 4, PMSZ_K_COMPACT = 5, PMSZ_K_OTHER = 6, PMSZ_K_SWEEP_MASKED = 7, PMSZ_K_DEFER = 8,
    PMSZ_K_TAIL = 9,   /* persistent list-mode iterations (one cooperative launch) */
    PMSZ_K_COUNT = 10
};

/* ---- plans -------------------------------------------------------------- */
pmsz_status pmsz_plan_create(const pmsz_desc* desc, pmsz_plan** out);
void pmsz_plan_destroy(pmsz_plan* plan);
/* Device bytes of scratch owned by the plan. */
int64_t pmsz_plan_scratch_bytes(const pmsz_plan* plan);
/* Time every kernel launch of this plan with CUDA events on its stream
 * (enable != 0; enable == PMSZ_PROFILE_FULL_DOMAIN: only the full-domain
 * classes PREP / SWEEP_FULL / VERIFY, whose events cost nothing measurable --
 * timing all ~40 launches of a step adds ~0.15 ms at 512^3).
 * pmsz_profile_read returns the accumulated device time (ms) and launch count
 * per kernel class (arrays of PMSZ_K_COUNT) and optionally resets. */
#define PMSZ_PROFILE_FULL_DOMAIN 2
pmsz_status pmsz_profile(pmsz_plan* plan, int32_t enable);
pmsz_status pmsz_profile_read(pmsz_plan* plan, double* ms, int64_t* launches, int32_t reset);

/*
 * run_correction (correction.py:391-436) on device-resident buffers.
 * f_dev: original (f64, or f32 with PMSZ_FLAG_F32_ORIGINAL); fhat_dev: f64;
 * g_dev: f64 output (the corrected field; may alias fhat_dev for in-place).
 * history_host: receives edits_per_iteration (capacity history_cap).
 * Returns PMSZ_OK or the reference's failure (bound / monotone / convergence).
 * The edit set is read afterwards with pmsz_edits_export.
 */
pmsz_status pmsz_run_correction(pmsz_plan* plan, const void* f_dev, const double* fhat_dev,
                                double* g_dev, int64_t* history_host, int64_t history_cap,
                                pmsz_result* result, void* stream);

/* pmsz_run_correction followed by pmsz_edits_export into device buffers of
 * capacity cap (the first min(cap, count) edits) with no return to the caller
 * in between; result->edit_count is the full count. */
pmsz_status pmsz_run_correction_export(pmsz_plan* plan, const void* f_dev, const double* fhat_dev,
                                       double* g_dev, int64_t* history_host, int64_t history_cap,
                                       pmsz_result* result, int64_t* ids_dev, double* vals_dev,
                                       int64_t cap, void* stream);

/*
 * The same call with HOST buffers (the end-to-end drop-in): copies f and fhat
 * in, runs, and writes the corrected field and the edit set back to the host.
 * g_host may be NULL (edit set only); ids_host/vals_host receive the first
 * min(edits_cap, edit_count) edits (EditSet.diff, correction.py:363-369) --
 * result->edit_count is always the full count, so a caller detects a
 * truncated record by edit_count > edits_cap.  history_host receives up to
 * history_cap entries (pmsz_history has all of them).  The device staging
 * (12 or 16 bytes per voxel plus the edit record) is owned by the plan,
 * allocated on the first call and reused.  The host-to-device copy runs in
 * z-slabs on a second stream and K0 starts on each slab as soon as it (and
 * its upper neighbour plane) has landed.
 * Any buffer may be pageable (plain malloc / numpy memory): pageable inputs
 * are staged through a pinned ring by host threads while the previous chunk
 * is on the link; a pageable g_host is filled from fhat_host on the host and
 * patched with the edit record (no device-to-host copy of the field).  With
 * g_host given and no (pinned, large enough) ids/vals buffers the whole
 * record stays in the plan's pinned buffers for pmsz_edits_host.
 */
pmsz_status pmsz_run_correction_host(pmsz_plan* plan, const void* f_host, const double* fhat_host,
                                     double* g_host, int64_t* ids_host, double* vals_host,
                                     int64_t edits_cap, int64_t* history_host, int64_t history_cap,
                                     pmsz_result* result, void* stream);

/* The edit record of the last pmsz_run_correction_host call when the plan
 * kept it (see there): the first min(cap, count) entries into host buffers;
 * *count_out = the full count.  PMSZ_ERR_INVALID when no record is held. */
pmsz_status pmsz_edits_host(pmsz_plan* plan, int64_t* ids_host, double* vals_host, int64_t cap,
                            int64_t* count_out);

/* Ascending ids where g != fhat and the corrected values (EditSet.diff). */
pmsz_status pmsz_edits_export(pmsz_plan* plan, const double* g_dev, int64_t* ids_dev,
                              double* vals_dev, int64_t cap, int64_t* count_out, void* stream);

/* ---- stepwise interface (block-parallel engine, parallel.py:150-255) ---- */
/* K0: validate the pair, build the f-code, g <- fhat (correction.py:52-60,118-122,404-405). */
pmsz_status pmsz_prepare(pmsz_plan* plan, const void* f_dev, const double* fhat_dev,
                         double* g_dev, pmsz_result* result, void* stream);
/* One Jacobi iteration (_iterate_array, correction.py:232-242) over the core box.
 * Returns edits / detections / shared_dirty in result->last_*.
 * edited_mask_dev (optional, u8 per vertex) receives the iteration's edited mask. */
pmsz_status pmsz_iterate(pmsz_plan* plan, const void* f_dev, double* g_dev,
                         uint8_t* edited_mask_dev, pmsz_result* result, void* stream);
/* Iterate to a local fixpoint (local_converge / relaxed _block_round, parallel.py:150-172,237-255);
 * lockstep != 0 runs exactly one iteration.  iterations/edit totals are accumulated into result. */
pmsz_status pmsz_block_round(pmsz_plan* plan, const void* f_dev, double* g_dev, int32_t lockstep,
                             int64_t* round_edits, pmsz_result* result, void* stream);
/* Mark the whole core box dirty again (after a ghost merge changed replicas). */
pmsz_status pmsz_mark_all_dirty(pmsz_plan* plan, void* stream);
/* Mark the dirty 1-ring of the given ext-local vertex ids (after a ghost merge). */
pmsz_status pmsz_mark_dirty_ids(pmsz_plan* plan, const uint32_t* ids_dev, int64_t count, void* stream);
/* Final full detection sweep; per-kind residuals into result->residual (correction.py:424-426). */
pmsz_status pmsz_verify(pmsz_plan* plan, const double* g_dev, pmsz_result* result, void* stream);
/* Vertices with g < lower (f64, e.g. local_converge's lower_ext): the reference's
 * monotonicity assertion fires at the first iteration with a detection when this is
 * non-zero (correction.py:239-241).  The count is recorded in the plan (PMSZ_FLAG_LOWER). */
pmsz_status pmsz_floor_violations(pmsz_plan* plan, const double* lower_dev, const double* g_dev,
                                  int64_t* count_out, void* stream);
/* Full per-iteration edit history of the plan's last run (edits_per_iteration,
 * correction.py:411-416); *count receives its length, out up to cap entries. */
pmsz_status pmsz_history(const pmsz_plan* plan, int64_t* out, int64_t cap, int64_t* count);
/* Dense bounds check L <= g <= U (BoundsField.admits, correction.py:124-125); count out. */
pmsz_status pmsz_bounds_violations(pmsz_plan* plan, const void* f_dev, const double* g_dev,
                                   int64_t* count_out, void* stream);

/* ---- multi-GPU round loop (run_parallel, parallel.py:258-367, one block per rank) ---- */
#define PMSZ_MAX_RANKS 64
#define PMSZ_MAX_EXCHANGES 26
/*
 * The reference's relaxed / lockstep round loop (parallel.py:289-322) of ONE
 * rank, driven from C with every exchange over NVLink peer memory: each rank
 * owns a buffer that every other rank can address (torch symmetric memory;
 * `bufs` holds all of them as device pointers valid in this process).
 * Buffer layout (per rank, identical offsets everywhere): two parity areas of
 * repl_doubles f64 each for the packed overlap replicas (this rank's overlap
 * with every peer, one box per exchange), then u64 sum slots [2][world][4] at
 * sums_off, then u64 arrival epochs [world] at flags_off (zero at creation).
 * A round: pmsz_block_round; pack the replicas into the round's parity area;
 * publish {edits, shared_dirty} into every peer's slot and raise this rank's
 * epoch there (release, system scope); wait until every peer's epoch arrived
 * (acquire); sum; terminate exactly as parallel.py:304-322; else min-merge
 * every peer's replica straight out of its buffer (pmsz_box_merge_min).
 * Parity areas and epoch-parity sum slots make a second barrier unnecessary.
 * epoch and rounds_total persist across calls on the same buffers.
 */
typedef struct {
    int32_t world, rank;
    int32_t nex;                     /* exchanges of this rank (its overlaps with other blocks) */
    int32_t lockstep;
    int64_t cap;                     /* CorrectionConfig.max_outer_iterations (rounds) */
    int64_t repl_doubles;            /* one parity area (doubles) */
    int64_t sums_off;                /* u64 offset of the sum slots in every buffer */
    int64_t flags_off;               /* u64 offset of the arrival epochs in every buffer */
    uint64_t epoch;                  /* in: last epoch used on these buffers; out: updated */
    uint64_t rounds_total;           /* in/out: rounds run on these buffers (replica parity) */
    void* bufs[PMSZ_MAX_RANKS];
    int32_t ex_peer[PMSZ_MAX_EXCHANGES];
    int64_t ex_lo[PMSZ_MAX_EXCHANGES][3];     /* overlap box in this rank's ext coordinates */
    int64_t ex_hi[PMSZ_MAX_EXCHANGES][3];
    int64_t ex_off[PMSZ_MAX_EXCHANGES];       /* this rank's replica of the box in its buffer (doubles) */
    int64_t ex_peer_off[PMSZ_MAX_EXCHANGES];  /* the peer's replica of the same box in the peer's buffer */
} pmsz_rounds_desc;
/* rounds / syncs (ParallelStats), totals[k] = edits of round k summed over ranks
 * (edits_per_iteration of run_parallel); result = this block's last pmsz_block_round. */
pmsz_status pmsz_rounds(pmsz_plan* plan, const void* f_dev, double* g_dev, pmsz_rounds_desc* rd, int64_t* rounds,
                        int64_t* syncs, int64_t* totals, int64_t totals_cap, pmsz_result* result, void* stream);

/* ---- topology kernels ---------------------------------------------------- */
/* scan_neighbors (topology.py:47-86): ids of the (value,id)-largest/smallest neighbour
 * and extremum flags.  Outputs are device arrays of n entries. */
pmsz_status pmsz_scan_neighbors(int64_t nx, int64_t ny, int64_t nz, const double* values_dev,
                                int64_t* nmax_dev, int64_t* nmin_dev, uint8_t* is_max_dev,
                                uint8_t* is_min_dev, void* stream);
/* Packed 1-byte code per vertex: low nibble nmax direction rank (15 = maximum),
 * high nibble nmin direction rank (15 = minimum). */
pmsz_status pmsz_scan_codes(int64_t nx, int64_t ny, int64_t nz, const double* values_dev,
                            uint8_t* code_dev, void* stream);

/* ---- segmentation and distortion report (topology.py:156-174, 254-274) ---- */
/* compute_segmentation(field): asc_target = minimum reached by the descending
 * steepest path, desc_target = maximum reached by the ascending path (int64
 * vertex ids, device arrays of nx*ny*nz).  v is f64, or f32 with is_f32. */
pmsz_status pmsz_segmentation(int64_t nx, int64_t ny, int64_t nz, const void* values_dev, int32_t is_f32,
                              int64_t* asc_target_dev, int64_t* desc_target_dev, void* stream);
/* compare_plmss(reference, test): counts[7] (host) = sizes of fp_max, fn_max,
 * fp_min, fn_min, asc_order_violations, desc_order_violations, then
 * wrong_label_count.  kind_bits (device, may be NULL) receives the six vertex
 * sets as bitmaps of ceil(n/32) words each, in that order. */
pmsz_status pmsz_compare_plmss(int64_t nx, int64_t ny, int64_t nz, const void* reference_dev, int32_t ref_f32,
                               const void* test_dev, int32_t test_f32, uint32_t* kind_bits_dev,
                               int64_t* counts, void* stream);
/* Ascending ids of the set bits of a device bitmap (np.flatnonzero); *count
 * always receives the number of set bits; ids is written when it fits cap. */
pmsz_status pmsz_bits_to_ids(const uint32_t* bits_dev, int64_t nbits, int64_t* ids_dev, int64_t cap,
                             int64_t* count, void* stream);

/* ---- ghost exchange helpers (_merge_min, parallel.py:122-140) ------------ */
/* Pack a sub-box [lo, hi) of a domain array into a contiguous buffer. */
pmsz_status pmsz_box_pack(int64_t nx, int64_t ny, int64_t nz, const double* src_dev,
                          const int64_t lo[3], const int64_t hi[3], double* buf_dev, void* stream);
/* dst[box] = min(dst[box], buf); counts changed vertices into *changed_dev (u64, device). */
pmsz_status pmsz_box_unpack_min(int64_t nx, int64_t ny, int64_t nz, double* dst_dev,
                                const int64_t lo[3], const int64_t hi[3], const double* buf_dev,
                                unsigned long long* changed_dev, void* stream);
/* dst[box] = buf (owner broadcast); counts changed vertices. */
pmsz_status pmsz_box_unpack_copy(int64_t nx, int64_t ny, int64_t nz, double* dst_dev,
                                 const int64_t lo[3], const int64_t hi[3], const double* buf_dev,
                                 unsigned long long* changed_dev, void* stream);
/* Ghost merge of a received replica box (_merge_min, parallel.py:122-140):
 * g[box] = min(g[box], buf) and every vertex that changed dirties its 1-ring
 * for the next incremental sweep of the plan.  *changed_out = changed vertices;
 * changed_out == NULL: no host synchronisation -- the plan reads the marking
 * counters at its next iteration (pmsz_iterate / pmsz_block_round). */
pmsz_status pmsz_box_merge_min(pmsz_plan* plan, double* g_dev, const int64_t lo[3], const int64_t hi[3],
                               const double* buf_dev, int64_t* changed_out, void* stream);
/* Detections left at the latest evaluation of every core centre (the
 * incremental equivalent of the final re-scan, correction.py:424-426). */
pmsz_status pmsz_residual(pmsz_plan* plan, int64_t* count_out, void* stream);
/* After a merge: mark the 1-ring of every vertex of box [lo,hi) whose value differs
 * from `before` as dirty for the next incremental sweep. */
pmsz_status pmsz_box_mark_changed(pmsz_plan* plan, const int64_t lo[3], const int64_t hi[3],
                                  const double* before_buf_dev, const double* g_dev, void* stream);

/* ---- synthetic inputs (synth.py, quantizer.py) --------------------------- */
/* Fractal Perlin noise of a sub-box [lo, lo+ext) of the global grid gdims, bit-exact with
 * synth.perlin (synth.py:55-100).  perm512: the 512-entry table of synth._permutation. */
pmsz_status pmsz_perlin(const int64_t gdims[3], const int64_t lo[3], const int64_t ext[3],
                        const int32_t* perm512_host, double frequency, int32_t octaves,
                        double* out_f64_dev, float* out_f32_dev, void* stream);
/* out = (float)v; *inexact (host) = values that do not survive the round trip
 * (f32 fields promoted to f64 survive it exactly, codec.py:86-87; the drop-in
 * then runs the f32 K0). */
pmsz_status pmsz_narrow_f32(const double* v_dev, int64_t n, float* out_dev, int64_t* inexact, void* stream);
/* Synchronous copies between a HOST array (pageable or pinned) and device
 * memory, for callers that hold whole fields in plain host memory (the
 * drop-in's numpy arrays): pageable memory is staged through a process-wide
 * pinned ring by host threads with streaming stores (see
 * pmsz_run_correction_host).  pmsz_host_to_device copies n bytes, or with
 * narrow_f64 != 0 converts n f64 host values to f32 on the device side of the
 * ring; *inexact = 1 when some value did not survive the round trip.  Both
 * order themselves after the work already queued on `stream` and return when
 * the copy is complete. */
pmsz_status pmsz_host_to_device(void* dst_dev, const void* src_host, int64_t n, int32_t narrow_f64,
                                int64_t* inexact, void* stream);
pmsz_status pmsz_device_to_host(void* dst_host, const void* src_dev, int64_t bytes, void* stream);
/* min / max of n values (f32 or f64); result on the host. */
pmsz_status pmsz_minmax(const void* values_dev, int32_t is_f32, int64_t n, double* mn, double* mx,
                        void* stream);
/* quantize (quantizer.py:122-154): recon = origin + code*(2 xi) with the ulp repair. */
pmsz_status pmsz_quantize(const void* f_dev, int32_t is_f32, int64_t n, double origin, double xi,
                          double* recon_dev, int64_t* max_code_out, void* stream);
/* The same with the integer codes of the payload (QuantizedPayload.codes,
 * quantizer.py:146-153) into codes_dev (u64[n]). */
pmsz_status pmsz_quantize_codes(const void* f_dev, int32_t is_f32, int64_t n, double origin, double xi,
                                double* recon_dev, uint64_t* codes_dev, int64_t* max_code_out, void* stream);
/* Seeded bounded noise fhat = clamp(f + xi*u, f - xi, f + xi), u in [-1,1) from a
 * counter hash of (seed, global id); ids are global so blocks agree. */
pmsz_status pmsz_bounded_noise(const void* f_dev, int32_t is_f32, int64_t nx, int64_t ny,
                               int64_t nz, const int64_t gdims[3], const int64_t lo[3],
                               double xi, uint64_t seed, double* out_dev, void* stream);
/* HEDM-like Gaussian-peak stack (BASELINE config 5; not in the reference):
 * sparse Gaussian spots in (64,64,32)-voxel cells over a faint hash-noise
 * background, for the sub-box [lo, lo+ext) of a global grid; f64 or f32
 * output.  Bit-identical to the oracle's orc_peaks (det_exp, no FMA). */
pmsz_status pmsz_gaussian_peaks(const int64_t gdims[3], const int64_t lo[3], const int64_t ext[3], uint64_t seed,
                                int32_t out_f32, void* out_dev, void* stream);
/* Copy a sub-box of a global device array into a contiguous domain array (f64 or f32). */
pmsz_status pmsz_box_extract(const int64_t gdims[3], const void* src_dev, int32_t is_f32,
                             const int64_t lo[3], const int64_t ext[3], void* dst_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PMSZ_H */
