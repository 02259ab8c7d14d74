#!/bin/bash
# host staging sweep of the drop-in path (pageable numpy buffers) at 512^3
mkdir -p gpurun_out
cat > /tmp/st.py <<'P'
import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2601_01787_b200 as pm
from paper_2601_01787_b200 import inputs as gen
dims = (512,) * 3
f32 = gen.perlin_device(gen.NoiseSpec(dims, 0), f32=True)
lo, hi = gen.minmax_device(f32)
xi = gen.relative_to_absolute_range(lo, hi, 1e-4)
fh = gen.quantize_device(f32, xi, lo, hi)
f = pm.ScalarField(dims, f32.double().cpu().numpy()); fhat = pm.ScalarField(dims, fh.cpu().numpy())
cfg = pm.CorrectionConfig(xi_abs=xi)
r = pm.run_correction(f, fhat, cfg)
ts = []
for _ in range(4):
    t0 = time.perf_counter(); r = pm.run_correction(f, fhat, cfg); ts.append(time.perf_counter() - t0)
print("dropin ms", [round(t * 1e3, 1) for t in ts], flush=True)
P
for ch in 8 16 32 64; do for th in 8 16; do
  echo "== chunk $ch MiB threads $th"
  PMSZ_E2E_TRACE=1 PMSZ_STAGE_CHUNK_MB=$ch PMSZ_STAGE_THREADS=$th timeout 300 python /tmp/st.py 2>&1 | grep -v Warn | tail -4
done; done
