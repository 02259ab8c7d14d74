"""GPU idle gaps inside one 512^3 correction step: CUPTI kernel/memcpy/memset
timestamps through torch.profiler (the library's own kernels included), sorted
by start; prints every gap above 3 us with the surrounding operations."""
import json, sys, os
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
cfg = pm.CorrectionConfig(xi_abs=xi)
out = torch.empty_like(fh)
for _ in range(3):
    pm.run_correction_device(f32, fh, dims, cfg, out=out)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pm.run_correction_device(f32, fh, dims, cfg, out=out)
    torch.cuda.synchronize()
path = "gpurun_out/gap_trace.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
busy = sum(e["dur"] for e in gpu)
span = gpu[-1]["ts"] + gpu[-1]["dur"] - t0
print(f"ops {len(gpu)}  span {span:.1f} us  busy {busy:.1f} us  idle {span - busy:.1f} us")
prev_end = None
for i, e in enumerate(gpu):
    if prev_end is not None:
        gap = e["ts"] - prev_end
        if gap > 3:
            print(f"  gap {gap:7.1f} us before {e['name'][:60]}  (after {gpu[i-1]['name'][:50]})")
    prev_end = max(prev_end or 0, e["ts"] + e["dur"])
