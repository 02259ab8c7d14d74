"""Pin the BENCHMARK-SIZE results to the REFERENCE ITSELF.

Run once in the build container (the reference is importable read-only there;
it never travels to the GPU box):

    python tests/golden/make_golden_large.py            # 256^3 cases + 512^3 (~1 h, ~40 GB RSS)
    python tests/golden/make_golden_large.py --skip-512  # 256^3 cases only (~6 min)

For each case it runs the reference's own public entry points
(`topocorrect.run_correction`, `correction.py:391-436`, and
`topocorrect.run_parallel`, `parallel.py:258-367`) on the benchmark inputs --
`perlin(NoiseSpec(dims, seed))` cast to f32 and promoted to f64 (what
`codec.read_field` does for f32 files, `codec.py:86-87`),
`xi = relative_to_absolute(f, rel)`, `fhat = quantize(f, xi)[1]`,
`CorrectionConfig(xi_abs=xi)` -- and records SHA-256 digests of the f32 input,
of fhat, of the corrected field and of the edit record (ids int64 / values
f64), plus `edits_per_iteration` / `max_vertex_edits` / `ParallelStats`.
Output: tests/golden/golden_large.json (digests only, a few KiB).  The GPU
tests (`tests/test_gpu_large.py`) regenerate the same inputs ON THE DEVICE and
compare digests; bench.py compares its corrected-field digest too.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden_large.json"
sys.path.insert(0, str(REF))

import topocorrect as tc  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def inputs(n: int, seed: int, rel: float):
    t = time.time()
    f = tc.perlin(tc.NoiseSpec(dims=(n, n, n), seed=seed))
    f32 = f.values.astype(np.float32)
    del f
    f = tc.ScalarField((n, n, n), f32.astype(np.float64))
    xi = tc.relative_to_absolute(f, rel)
    _, fh = tc.quantize(f, xi)
    rec = {"dims": [n, n, n], "seed": seed, "rel": rel, "xi": xi, "tau": tc.CorrectionConfig(xi_abs=xi).tau,
           "f32_sha256": sha(f32), "fhat_sha256": sha(fh.values), "inputs_seconds": round(time.time() - t, 1)}
    return f, fh, rec


def result_record(res) -> dict:
    return {"iterations": res.iterations, "edits_per_iteration": list(res.edits_per_iteration),
            "max_vertex_edits": res.max_vertex_edits, "edit_count": res.edits.count,
            "corrected_sha256": sha(res.corrected.values), "ids_sha256": sha(res.edits.ids.astype(np.int64)),
            "vals_sha256": sha(res.edits.values.astype(np.float64))}


def save(meta):
    OUT.write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", OUT, flush=True)


def main():
    skip512 = "--skip-512" in sys.argv
    meta = json.loads(OUT.read_text()) if OUT.exists() else {}
    meta["generator"] = "tests/golden/make_golden_large.py"
    meta["reference"] = "topocorrect " + tc.__version__

    # ---- 256^3: serial + run_parallel (lockstep == serial, relaxed per grid)
    if "c256" not in meta:
        f, fh, rec = inputs(256, 0, 1e-4)
        cfg = tc.CorrectionConfig(xi_abs=rec["xi"])
        t = time.time()
        rec["serial"] = result_record(tc.run_correction(f, fh, cfg))
        rec["serial"]["seconds"] = round(time.time() - t, 1)
        par = []
        for grid, strat in [((2, 2, 2), tc.SyncStrategy.RELAXED), ((1, 1, 2), tc.SyncStrategy.RELAXED),
                            ((1, 1, 4), tc.SyncStrategy.RELAXED), ((2, 2, 2), tc.SyncStrategy.LOCKSTEP)]:
            t = time.time()
            res, st = tc.run_parallel(f, fh, cfg, grid, strat, workers=8)
            d = st.to_dict()
            d.pop("timings")
            r = result_record(res)
            r.update({"grid": list(grid), "strategy": strat.value, "stats": d, "seconds": round(time.time() - t, 1)})
            par.append(r)
            print("256^3", grid, strat.value, r["iterations"], d["rounds"], d["syncs"], flush=True)
        rec["parallel"] = par
        meta["c256"] = rec
        save(meta)
        del f, fh

    # ---- 512^3: BASELINE config 2 (perlin seed 0, f32, rel 1e-4, quantizer)
    if not skip512 and "c512" not in meta:
        f, fh, rec = inputs(512, 0, 1e-4)
        print("512^3 inputs", rec, flush=True)
        cfg = tc.CorrectionConfig(xi_abs=rec["xi"])
        t = time.time()
        rec["serial"] = result_record(tc.run_correction(f, fh, cfg))
        rec["serial"]["seconds"] = round(time.time() - t, 1)
        meta["c512"] = rec
        save(meta)


if __name__ == "__main__":
    main()
