"""Small device correction vs the oracle (debug aid): python tools/small_run.py nx ny nz [rel]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2601_01787_b200 as pm
from oracle import oracle as orc
dims = tuple(int(v) for v in sys.argv[1:4])
rel = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-3
f = orc.perlin(dims, seed=1)
xi = orc.relative_to_absolute(f, rel)
fh = orc.quantize(f, xi)
res = pm.run_correction(pm.ScalarField(dims, f), pm.ScalarField(dims, fh), pm.CorrectionConfig(xi_abs=xi))
ref = orc.run_correction(dims, f, fh, xi)
ok = np.array_equal(res.corrected.values, ref.corrected) and res.edits_per_iteration == ref.edits_per_iteration
print("dims", dims, "iterations", res.iterations, "ok", ok)
sys.exit(0 if ok else 1)
