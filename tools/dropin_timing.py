"""Break down the host-side cost of the drop-in run_correction(ScalarField) at 512^3."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
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
dev = torch.device("cuda", 0)


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) / reps * 1e3:9.1f} ms", flush=True)
    return r


t("run_correction (drop-in)", lambda: pm.run_correction(f, fhat, cfg))
t("H2D pageable from_numpy().to()", lambda: torch.from_numpy(f.values).to(dev))
g = torch.from_numpy(fhat.values).to(dev)
t("D2H g.cpu()", lambda: g.cpu())
t("D2H into np.empty", lambda: torch.from_numpy(np.empty(g.numel())).copy_(g))
t("pinned alloc 1 GB", lambda: torch.empty(g.numel(), dtype=torch.float64, pin_memory=True))
pin = torch.empty(g.numel(), dtype=torch.float64, pin_memory=True)
t("D2H into pinned", lambda: pin.copy_(g))
t("ScalarField(host array)", lambda: pm.ScalarField(dims, pin.numpy()))
t("np.isfinite.all", lambda: np.isfinite(fhat.values).all())
t("np copy", lambda: np.array(fhat.values, copy=True))
