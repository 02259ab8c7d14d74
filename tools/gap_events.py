"""Host-induced GPU gaps at the end of run_correction_device (512^3): CUDA
events recorded right after plan.run returns and right before the export
launch measure how long the GPU waits on the host there."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2601_01787_b200 as pm
from paper_2601_01787_b200 import inputs as gen
from paper_2601_01787_b200.correction import _plan_for
from paper_2601_01787_b200.engine import raise_for

dims = (512,) * 3
f32 = gen.perlin_device(gen.NoiseSpec(dims, 0), f32=True)
lo, hi = gen.minmax_device(f32)
xi = gen.relative_to_absolute_range(lo, hi, 1e-4)
fh = gen.quantize_device(f32, xi, lo, hi)
cfg = pm.CorrectionConfig(xi_abs=xi)
out = torch.empty_like(fh)
plan = _plan_for(dims, cfg, incremental=True, extrema_only=False, f32_original=True)
for _ in range(3):
    pm.run_correction_device(f32, fh, dims, cfg, out=out, plan=plan)
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(5):
    e0, e1, e2, e3 = E(), E(), E(), E()
    e0.record()
    st, res, hist = plan.run(f32, fh, out)
    e1.record()
    raise_for(st, res, None, None, cfg.xi_abs, f_dev=f32, fhat_dev=fh)
    e2.record()
    ids, vals = plan.export_edits(out)
    e3.record()
    torch.cuda.synchronize()
    print(f"run {e0.elapsed_time(e1):.3f} ms   host gap after run {e1.elapsed_time(e2)*1e3:.1f} us   export {e2.elapsed_time(e3)*1e3:.1f} us")
