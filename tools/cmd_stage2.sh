#!/bin/bash
# host staging: fresh vs pre-touched output field, chunk sizes (pageable drop-in path, 512^3)
mkdir -p gpurun_out
cat > /tmp/st2.py <<'P'
import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2601_01787_b200 as pm
from paper_2601_01787_b200 import inputs as gen
from paper_2601_01787_b200.correction import _plan_for
dims = (512,) * 3
f32 = gen.perlin_device(gen.NoiseSpec(dims, 0), f32=True)
lo, hi = gen.minmax_device(f32)
xi = gen.relative_to_absolute_range(lo, hi, 1e-4)
fh = gen.quantize_device(f32, xi, lo, hi)
f = f32.double().cpu().numpy(); fhn = fh.cpu().numpy()
cfg = pm.CorrectionConfig(xi_abs=xi)
plan = _plan_for(dims, cfg, incremental=True, extrema_only=False, f32_original=True, host_f64=True)
g = np.empty(f.size)
plan.run_host(f, fhn, g)
for mode in ("fresh", "touched", "nofill"):
    ts = []
    for _ in range(3):
        g = np.empty(f.size) if mode == "fresh" else (g if mode == "touched" else None)
        t0 = time.perf_counter(); plan.run_host(f, fhn, g); ts.append(time.perf_counter() - t0)
    print(mode, "ms", [round(t * 1e3, 1) for t in ts], flush=True)
P
for ch in 16 32 64; do
  echo "== chunk $ch MiB"
  PMSZ_E2E_TRACE=1 PMSZ_STAGE_CHUNK_MB=$ch timeout 300 python /tmp/st2.py 2>&1 | grep -v Warn | grep -v "^e2e"
done
