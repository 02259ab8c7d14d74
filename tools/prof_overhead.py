"""Step time of the 512^3 bench workload with the per-kernel event profiling on and off.
usage: python tools/prof_overhead.py [size] [steps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2601_01787_b200 as pm
from paper_2601_01787_b200 import inputs as gen
from paper_2601_01787_b200.engine import DomainPlan, DomainSpec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dims = (n, n, n)
f32 = gen.perlin_device(gen.NoiseSpec(dims, 0), f32=True)
lo, hi = gen.minmax_device(f32)
xi = gen.relative_to_absolute_range(lo, hi, 1e-4)
fh = gen.quantize_device(f32, xi, lo, hi)
cfg = pm.CorrectionConfig(xi_abs=xi)
plan = DomainPlan(DomainSpec.whole(dims), xi, cfg.tau, cfg.max_outer_iterations, incremental=True, f32_original=True)
g = torch.empty_like(fh)
for _ in range(3):
    pm.run_correction_device(f32, fh, dims, cfg, out=g, plan=plan)
for rep in range(3):
    for on in (False, True):
        plan.profile(on)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            pm.run_correction_device(f32, fh, dims, cfg, out=g, plan=plan)
        e1.record()
        torch.cuda.synchronize()
        print(f"profile={on}: {e0.elapsed_time(e1) / steps:.3f} ms/step")
        plan.profile_read(reset=True)
