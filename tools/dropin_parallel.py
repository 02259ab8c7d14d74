"""Wall-clock of the reference-facing drop-ins at 512^3 on pageable ScalarFields:
run_correction and run_parallel (relaxed and lockstep block grids)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2601_01787_b200 as pm
from paper_2601_01787_b200 import inputs as gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
f32 = gen.perlin_device(gen.NoiseSpec(dims, 0), f32=True)
lo, hi = gen.minmax_device(f32)
xi = gen.relative_to_absolute_range(lo, hi, 1e-4)
fh = gen.quantize_device(f32, xi, lo, hi)
f = pm.ScalarField(dims, f32.double().cpu().numpy())
fhat = pm.ScalarField(dims, fh.cpu().numpy())
cfg = pm.CorrectionConfig(xi_abs=xi)


def t(label, fn, reps=3):
    r = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{label:48s} " + " ".join(f"{x:7.1f}" for x in ts) + " ms", flush=True)
    return r


t("run_correction", lambda: pm.run_correction(f, fhat, cfg))
t("run_parallel (1,1,2) relaxed", lambda: pm.run_parallel(f, fhat, cfg, (1, 1, 2)))
t("run_parallel (2,2,2) relaxed", lambda: pm.run_parallel(f, fhat, cfg, (2, 2, 2)))
t("run_parallel (1,1,2) lockstep", lambda: pm.run_parallel(f, fhat, cfg, (1, 1, 2), pm.SyncStrategy.LOCKSTEP), reps=1)
