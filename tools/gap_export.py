"""Where the host time between the end of the loop and the edit export goes
(512^3): CUDA events between the host steps of DomainPlan.export_edits."""
import sys, time, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2601_01787_b200 as pm
from paper_2601_01787_b200 import inputs as gen, _native as N
from paper_2601_01787_b200.correction import _plan_for

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
for rep in range(4):
    ev = [E() for _ in range(5)]
    h = []
    st, res, hist = plan.run(f32, fh, out)
    ev[0].record(); h.append(time.perf_counter())
    cnt = ctypes.c_int64()
    N.check(plan.lib.pmsz_edits_export(plan.handle, N.ptr(out), None, None, 0, ctypes.byref(cnt), N.stream_handle()), "x")
    ev[1].record(); h.append(time.perf_counter())
    m = int(cnt.value)
    ids = torch.empty(m, dtype=torch.int64, device=out.device)
    vals = torch.empty(m, dtype=torch.float64, device=out.device)
    ev[2].record(); h.append(time.perf_counter())
    N.check(plan.lib.pmsz_edits_export(plan.handle, N.ptr(out), N.ptr(ids), N.ptr(vals), m, ctypes.byref(cnt),
                                       N.stream_handle()), "x")
    ev[3].record(); h.append(time.perf_counter())
    torch.cuda.synchronize()
    print("gpu: count %.1f us, alloc %.1f us, export %.1f us | host: count %.1f, alloc %.1f, export launch %.1f us" % (
        ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3, ev[2].elapsed_time(ev[3]) * 1e3,
        (h[1] - h[0]) * 1e6, (h[2] - h[1]) * 1e6, (h[3] - h[2]) * 1e6))
