"""Generate the golden fixtures that pin the oracle (and the GPU path) to the
REFERENCE ITSELF.

Run in the build container, where the reference is importable read-only:

    python tests/golden/make_golden.py

It imports topocorrect from /root/reference/pkg/src, runs the reference's own
entry points (scan_neighbors, _iterate_array, run_correction, run_parallel,
perlin, quantize, codec.encode_edits) on seeded inputs, and writes
tests/golden/golden.json + tests/golden/golden.npz.  Nothing on the GPU box
reads /root/reference: the tests read only these committed files.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parent.parent))

import topocorrect as tc  # noqa: E402
from topocorrect import codec  # noqa: E402
from topocorrect.correction import BoundsField, _iterate_array  # noqa: E402
from topocorrect.topology import field_scan  # noqa: E402

from oracle import oracle as orc  # noqa: E402  (only for the bounded-noise input recipe)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def f32_perlin(dims, seed, freq=4.0, octaves=3):
    f = tc.perlin(tc.NoiseSpec(dims=dims, seed=seed, frequency=freq, octaves=octaves))
    return f.with_values(f.values.astype(np.float32).astype(np.float64))


def main():
    meta: dict = {"generator": "tests/golden/make_golden.py", "reference": "topocorrect " + tc.__version__}
    arrays: dict[str, np.ndarray] = {}

    # ---- scans on random fields (topology.py:47-86; test_topology.py:56-71 styles)
    rng = np.random.default_rng(20261018)
    scans = []
    shapes = [(5, 4, 3), (6, 6, 6), (7, 3, 2), (2, 9, 7), (9, 2, 5), (3, 3, 1), (8, 5, 1), (1, 6, 5),
              (6, 1, 4), (2, 2, 2), (4, 7, 1), (11, 4, 3)]
    for i, dims in enumerate(shapes):
        for style in ("uniform", "plateau", "coarse"):
            n = int(np.prod(dims))
            if style == "uniform":
                v = rng.standard_normal(n)
            elif style == "plateau":
                v = rng.integers(0, 4, size=n).astype(np.float64)
            else:
                v = np.round(rng.standard_normal(n), 1)
            s = tc.scan_neighbors(v, dims)
            key = f"scan_{i}_{style}"
            arrays[key + "_v"] = v
            arrays[key + "_nmax"] = s.nmax
            arrays[key + "_nmin"] = s.nmin
            arrays[key + "_ismax"] = s.is_max
            arrays[key + "_ismin"] = s.is_min
            scans.append({"key": key, "dims": list(dims)})
    meta["scans"] = scans

    # ---- Perlin / quantize pins
    perl = []
    for dims, seed, freq, octv in [((16, 16, 16), 42, 4.0, 3), ((12, 10, 3), 9, 3.0, 2), ((32, 32), 1, 4.0, 3),
                                   ((20, 17, 9), 7, 4.0, 3), ((64, 64, 64), 0, 4.0, 3), ((33, 5, 7), 123456789, 2.5, 4)]:
        f = tc.perlin(tc.NoiseSpec(dims=dims, seed=seed, frequency=freq, octaves=octv))
        xi = tc.relative_to_absolute(f, 1e-3)
        payload, recon = tc.quantize(f, xi)
        perl.append({"dims": list(dims), "seed": seed, "frequency": freq, "octaves": octv,
                     "sha256": sha(f.values), "xi_rel_1e-3": xi, "quantized_sha256": sha(recon.values),
                     "f32_sha256": sha(f.values.astype(np.float32)),
                     "payload": {"origin": payload.origin, "bit_width": payload.bit_width,
                                 "payload_bytes": payload.payload_bytes, "codes_sha256": sha(payload.codes)}})
    meta["perlin"] = perl

    # ---- _iterate_array trajectories (test_correction.py:215-235)
    iters = []
    for seed, rel in [(0, 1e-1), (1, 1e-2), (2, 1e-3), (3, 1e-1)]:
        f = tc.perlin(tc.NoiseSpec(dims=(8, 8, 8), seed=seed))
        xi = tc.relative_to_absolute(f, rel)
        _, recon = tc.quantize(f, xi)
        cfg = tc.CorrectionConfig(xi_abs=xi)
        lower = BoundsField.from_field(f, xi).lower
        fs = field_scan(f)
        g = recon.values
        traj = []
        for _ in range(cfg.max_outer_iterations):
            g, ed = _iterate_array(f.dims, fs, g, lower, cfg.tau)
            traj.append({"edits": int(ed.sum()), "g_sha256": sha(g), "edited_sha256": sha(ed)})
            if not ed.any():
                break
        iters.append({"seed": seed, "rel": rel, "xi": xi, "tau": cfg.tau, "trajectory": traj})
    meta["iterate"] = iters

    # ---- run_correction cases
    def record(name, f, fh, cfg, recipe):
        res = tc.run_correction(f, fh, cfg)
        arrays[name + "_ids"] = res.edits.ids
        arrays[name + "_vals"] = res.edits.values
        return {"name": name, "dims": list(f.dims), "xi": cfg.xi_abs, "tau": cfg.tau,
                "cap": cfg.max_outer_iterations, "recipe": recipe,
                "f_sha256": sha(f.values), "fhat_sha256": sha(fh.values),
                "iterations": res.iterations, "edits_per_iteration": list(res.edits_per_iteration),
                "max_vertex_edits": res.max_vertex_edits, "edit_count": res.edits.count,
                "corrected_sha256": sha(res.corrected.values)}

    runs = []
    perlin_cases = [
        ("golden8", (8, 8, 8), 42, 1e-1, False),
        ("p8_s0_1e-1", (8, 8, 8), 0, 1e-1, False),
        ("p16_s4_1e-3", (16, 16, 16), 4, 1e-3, False),
        ("p12x12x6_s5_1e-2", (12, 12, 6), 5, 1e-2, False),
        ("p32_s12_1e-2", (32, 32, 32), 12, 1e-2, False),
        ("p32_s13_1e-1", (32, 32, 32), 13, 1e-1, False),
        ("p2d_64_s3_1e-2", (64, 64), 3, 1e-2, False),
        ("p2d_96_s1_1e-3", (96, 96), 1, 1e-3, False),
        ("thin_2x9x7", (2, 9, 7), 2, 1e-1, False),
        ("thin_9x2x5", (9, 2, 5), 3, 1e-1, False),
        ("odd_21x13x11", (21, 13, 11), 6, 1e-2, True),
        ("cfg1_64_q_1e-3", (64, 64, 64), 0, 1e-3, True),
        ("p48_s7_1e-4", (48, 48, 48), 7, 1e-4, True),
    ]
    for name, dims, seed, rel, f32 in perlin_cases:
        f = f32_perlin(dims, seed) if f32 else tc.perlin(tc.NoiseSpec(dims=dims, seed=seed))
        xi = tc.relative_to_absolute(f, rel)
        _, recon = tc.quantize(f, xi)
        cfg = tc.CorrectionConfig(xi_abs=xi)
        runs.append(record(name, f, recon, cfg, {"kind": "perlin_quantize", "dims": list(dims), "seed": seed,
                                                 "rel": rel, "f32": f32}))
        if name == "golden8":
            blob = codec.encode_edits(tc.run_correction(f, recon, cfg).edits, xi, cfg.tau)
            meta["golden_edits_sha256"] = hashlib.sha256(blob).hexdigest()
    # BASELINE config 1: 64^3 f32 Perlin, rel 1e-3, bounded noise (seed 0)
    f = f32_perlin((64, 64, 64), 0)
    xi = tc.relative_to_absolute(f, 1e-3)
    fh = f.with_values(orc.bounded_noise(f.values, f.dims, xi, 0))
    runs.append(record("cfg1_64_noise_1e-3", f, fh, tc.CorrectionConfig(xi_abs=xi),
                       {"kind": "perlin_noise", "dims": [64, 64, 64], "seed": 0, "rel": 1e-3, "f32": True,
                        "noise_seed": 0}))
    # tie-heavy random fields (plateau/coarse), bounded-noise on a 0.01 lattice
    for i, dims in enumerate([(6, 6, 6), (9, 7, 5), (12, 12, 1), (5, 11, 4)]):
        r = np.random.default_rng(100 + i)
        n = int(np.prod(dims))
        fv = np.round(r.standard_normal(n), 1)
        xi = 0.05
        fhv = np.clip(np.round(fv + r.uniform(-xi, xi, n), 2), fv - xi, fv + xi)
        fhv = np.where(np.abs(fv - fhv) > xi, fv, fhv)
        arrays[f"tie_{i}_f"] = fv
        arrays[f"tie_{i}_fhat"] = fhv
        f = tc.ScalarField(dims, fv)
        runs.append(record(f"tie_{i}", f, f.with_values(fhv), tc.CorrectionConfig(xi_abs=xi, tau=0.01),
                           {"kind": "stored", "key": f"tie_{i}"}))
    meta["runs"] = runs

    # ---- failure modes
    f = tc.perlin(tc.NoiseSpec(dims=(8, 8), seed=7))
    bad = f.values.copy()
    bad[5] += 0.5
    bad[17] -= 0.9
    bad[40] += 1.0
    arrays["bound_f"] = f.values
    arrays["bound_fhat"] = bad
    try:
        tc.run_correction(f, f.with_values(bad), tc.CorrectionConfig(xi_abs=0.1))
        raise SystemExit("expected BoundViolationError")
    except tc.BoundViolationError as e:
        meta["bound_violation"] = {"dims": [8, 8, 1], "xi": 0.1, "index": e.index, "offenders": e.offenders}
    g8 = tc.perlin(tc.NoiseSpec(dims=(8, 8, 8), seed=42))
    x8 = tc.relative_to_absolute(g8, 1e-1)
    try:
        tc.run_correction(g8, tc.quantize(g8, x8)[1], tc.CorrectionConfig(xi_abs=x8, max_outer_iterations=3))
        raise SystemExit("expected ConvergenceError")
    except tc.ConvergenceError as e:
        meta["cap_error"] = {"cap": 3, "message": str(e)}

    # ---- run_parallel (parallel.py:258-367)
    par = []
    pcases = [((16, 16, 16), 14, 1e-2, (2, 1, 1)), ((16, 16, 16), 14, 1e-2, (2, 2, 1)),
              ((16, 16, 16), 14, 1e-2, (2, 2, 2)), ((24, 24, 24), 3, 1e-1, (2, 2, 2)),
              ((24, 24, 24), 3, 1e-1, (4, 2, 2)), ((30, 30, 30), 5, 1e-1, (3, 3, 3)),
              ((32, 32), 16, 1e-2, (2, 2, 1)), ((30, 20), 2, 1e-1, (3, 2, 1)),
              ((16, 16, 24), 9, 1e-2, (1, 1, 4))]
    for dims, seed, rel, grid in pcases:
        f = tc.perlin(tc.NoiseSpec(dims=dims, seed=seed))
        xi = tc.relative_to_absolute(f, rel)
        _, recon = tc.quantize(f, xi)
        cfg = tc.CorrectionConfig(xi_abs=xi)
        for strat in (tc.SyncStrategy.LOCKSTEP, tc.SyncStrategy.RELAXED):
            res, st = tc.run_parallel(f, recon, cfg, grid, strat)
            d = st.to_dict()
            d.pop("timings")
            name = f"par_{'x'.join(map(str, dims))}_{seed}_{'x'.join(map(str, grid))}_{strat.value}"
            arrays[name + "_ids"] = res.edits.ids
            arrays[name + "_vals"] = res.edits.values
            par.append({"name": name, "dims": list(f.dims), "seed": seed, "rel": rel, "grid": list(grid),
                        "strategy": strat.value, "xi": xi, "tau": cfg.tau, "stats": d,
                        "iterations": res.iterations, "edits_per_iteration": list(res.edits_per_iteration),
                        "max_vertex_edits": res.max_vertex_edits, "corrected_sha256": sha(res.corrected.values)})
    meta["parallel"] = par

    # ---- segmentation + compare_plmss (topology.py:156-174,254-274; test_codec.py:15-26)
    segs = []
    gf = tc.perlin(tc.NoiseSpec(dims=(8, 8, 8), seed=42))
    lab = tc.compute_segmentation(gf)
    meta["golden_labels"] = {
        "asc_file_sha256": hashlib.sha256(codec.write_labels(gf.dims, lab.asc_target)).hexdigest(),
        "desc_file_sha256": hashlib.sha256(codec.write_labels(gf.dims, lab.desc_target)).hexdigest(),
        "field_file_sha256": hashlib.sha256(codec.write_field(gf)).hexdigest(),
        "field_f32_file_sha256": hashlib.sha256(codec.write_field(gf, precision="f32")).hexdigest(),
    }
    for i, (dims, style) in enumerate([((8, 8, 8), "perlin"), ((9, 7, 5), "plateau"), ((16, 12, 1), "uniform"),
                                      ((6, 6, 6), "ramp"), ((13, 11, 7), "coarse"), ((24, 20, 16), "perlin")]):
        n = int(np.prod(dims))
        if style == "perlin":
            v = tc.perlin(tc.NoiseSpec(dims=dims, seed=i + 3)).values
        elif style == "plateau":
            v = rng.integers(0, 3, size=n).astype(np.float64)
        elif style == "uniform":
            v = rng.standard_normal(n)
        elif style == "ramp":
            v = np.arange(n, dtype=np.float64) * 0.5
        else:
            v = np.round(rng.standard_normal(n), 1)
        f = tc.ScalarField(dims, v)
        lab = tc.compute_segmentation(f)
        key = f"seg_{i}"
        arrays[key + "_v"] = v
        arrays[key + "_asc"] = lab.asc_target
        arrays[key + "_desc"] = lab.desc_target
        # a perturbed copy for compare_plmss: noise plus a few forced ties
        w = v + np.round(rng.standard_normal(n) * 0.3, 1)
        w[rng.integers(0, n, size=max(1, n // 10))] = float(np.median(v))
        t = tc.ScalarField(dims, w)
        rep = tc.compare_plmss(f, t)
        arrays[key + "_w"] = w
        segs.append({"key": key, "dims": list(dims), "style": style, "report": rep.to_dict()})
    meta["segmentation"] = segs

    # ---- extrema-only mode: the reference's own _iterate_array with
    # its _kind_masks wrapped so the two order masks are always empty, iterated
    # to a zero-edit pass.  Inputs: the (new) Gaussian-peak stack, stored, and
    # a Perlin field; fhat from the reference quantizer.
    import topocorrect.correction as tcc
    orig_masks = tcc._kind_masks

    def extrema_masks(f_scan, g_scan, center_mask=None):
        m = orig_masks(f_scan, g_scan, center_mask)
        z = np.zeros_like(m[0])
        return (m[0], m[1], m[2], m[3], z, z)

    ext = []
    for name, dims, rel in [("peaks", (64, 64, 32), 1e-3), ("peaks_fine", (64, 64, 32), 1e-4),
                            ("perlin", (20, 18, 16), 1e-2)]:
        if name.startswith("peaks"):
            f = tc.ScalarField(dims, orc.peaks(dims, 7))   # regenerated by the tests, pinned by f_sha256
        else:
            f = tc.perlin(tc.NoiseSpec(dims=dims, seed=11))
        xi = tc.relative_to_absolute(f, rel)
        _, fh = tc.quantize(f, xi)
        cfg = tc.CorrectionConfig(xi_abs=xi)
        f_scan = field_scan(f)
        lower = BoundsField.from_field(f, xi).lower
        g = fh.values.copy()
        counts = np.zeros(g.size, np.int64)
        hist = []
        tcc._kind_masks = extrema_masks
        try:
            for _ in range(cfg.max_outer_iterations):
                g, ed = _iterate_array(f.dims, f_scan, g, lower, cfg.tau)
                counts += ed
                hist.append(int(ed.sum()))
                if not ed.any():
                    break
        finally:
            tcc._kind_masks = orig_masks
        rs, ts = field_scan(f), tc.scan_neighbors(g, f.dims)
        ext.append({"name": name, "dims": list(dims), "rel": rel, "xi": xi, "tau": cfg.tau,
                    "edits_per_iteration": hist, "max_vertex_edits": int(counts.max()),
                    "corrected_sha256": sha(g), "fhat_sha256": sha(fh.values), "f_sha256": sha(f.values),
                    "extrema_clean": bool(np.array_equal(rs.is_max, ts.is_max) and np.array_equal(rs.is_min, ts.is_min)),
                    "order_violations_left": int(np.count_nonzero(~rs.is_max & (ts.nmax != rs.nmax)))})
    meta["extrema_only"] = ext

    (OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "golden.npz", **arrays)
    print("wrote", OUT / "golden.json", OUT / "golden.npz",
          sum(a.nbytes for a in arrays.values()) // 1024, "KiB raw")


if __name__ == "__main__":
    main()
