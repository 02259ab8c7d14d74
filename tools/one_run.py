"""One device-resident correction of the bench workload (for ncu captures).
usage: python tools/one_run.py [size] [runs] [--full-sweeps] [--host-loop]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2601_01787_b200 as pm
from paper_2601_01787_b200 import inputs as gen
from paper_2601_01787_b200.engine import DomainPlan, DomainSpec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
full = "--full-sweeps" in sys.argv
host_loop = "--host-loop" in sys.argv
dims = (n, n, n)
f32 = gen.perlin_device(gen.NoiseSpec(dims, 0), f32=True)
lo, hi = gen.minmax_device(f32)
xi = gen.relative_to_absolute_range(lo, hi, 1e-4)
fh = gen.quantize_device(f32, xi, lo, hi)
cfg = pm.CorrectionConfig(xi_abs=xi)
plan = DomainPlan(DomainSpec.whole(dims), xi, cfg.tau, cfg.max_outer_iterations, incremental=not full,
                  f32_original=True, host_loop=host_loop)
g = torch.empty_like(fh)
for _ in range(runs):
    r = pm.run_correction_device(f32, fh, dims, cfg, out=g, plan=plan)
torch.cuda.synchronize()
print("iterations", r.iterations, "edits", r.edit_ids.numel(), r.edits_per_iteration[:4])
