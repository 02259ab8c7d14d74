#!/usr/bin/env python
"""bench.py -- pMSz correction loop on B200: corrected voxels/s and % of the
HBM roofline (BASELINE.json metric).

Workload (N=1, BASELINE config 2): Perlin 512^3 (seed 0, frequency 4,
3 octaves) cast to float32, rel. error bound 1e-4, decompressed field from the
deterministic bounded-error quantizer (quantizer.quantize), full correction to
zero residual mismatches.  One step = one complete run_correction on the
device: K0 prepare -> K1/K2 iterations to the zero-edit fixpoint -> K4 verify
-> K5 edit export.  Inputs (1.5 GB) exceed the 126 MB L2.

N>1 (torchrun): weak scaling, 512^3 per rank, z-slab decomposition of a
512 x 512 x 512N field with NCCL ghost exchange (dist.py), relaxed sync.

--impl reference: the reference algorithm's CPU path (the C oracle port of
topocorrect, all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "corrected voxels/sec (512^3 per GPU, rel 1e-4)"
UNIT = "voxels/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", type=int, default=512, help="edge of the per-GPU cube")
    ap.add_argument("--rel", type=float, default=1e-4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dropin", action="store_true", help="skip the drop-in run_correction(ScalarField) timing")
    ap.add_argument("--f64-original", action="store_true",
                    help="pass the original field as f64 (the K0 variant for fields that are not f32-exact)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-z", type=int, default=64, help="z-planes of the CPU baseline sample")
    ap.add_argument("--full-sweeps", action="store_true", help="disable incremental dirty-ring sweeps")
    ap.add_argument("--strategy", default="relaxed", choices=["relaxed", "lockstep"])
    ap.add_argument("--workload", default="perlin", choices=["perlin", "strong", "hedm"],
                    help="perlin: configs 2/3 (default); strong: config 4; hedm: config 5 (extrema-only)")
    ap.add_argument("--decomp", default="slab", choices=["slab", "block"], help="strong scaling layout")
    ap.add_argument("--weak-layout", default="tile", choices=["tile", "mirror", "continuous"],
                    help="weak scaling: every GPU's core is the 1-GPU cube (tile, default), the cube or its "
                         "z-mirror (mirror: duplicates the interface planes), or the next stretch of the Perlin "
                         "function (continuous)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def ncu_traffic(kernel: str, workload: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/*_ncu_traffic.json), when it was taken on this workload."""
    best = None
    for p in sorted((ROOT / "profiles").glob("*_ncu_traffic.json")):
        try:
            d = json.loads(p.read_text())
        except Exception:
            continue
        if d.get("workload") == workload and kernel in d:
            best = (d[kernel]["traffic_bytes"], p.name)
    return best


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "fallback": True}


# ---------------------------------------------------------------------------
def _oracle_slab(kind: str, gdims, seed: int, z0: int, zs: int, norm=None) -> np.ndarray:
    """z-planes [z0, z0+zs) of the workload's f32 field, generated by the oracle
    (`norm`: the Perlin normalisation extents when they differ from gdims)."""
    from oracle import oracle as orc
    ext = (gdims[0], gdims[1], zs)
    if kind == "hedm":
        v = orc.peaks(gdims, seed, lo=(0, 0, z0), ext=ext)
    else:
        v = orc.perlin(norm or gdims, seed, lo=(0, 0, z0), ext=ext)
    return v.astype(np.float32).astype(np.float64)


def cpu_sample_inputs(kind: str, gdims, zs: int, rel: float, seed: int, xi=None, origin=None, norm=None,
                      stat_planes=None):
    """Bounded CPU sample of the workload: the first `zs` z-planes of the same
    field (global coordinates).  xi and the quantizer origin belong to the
    whole field: passed in when the GPU already has them, else computed from
    the oracle field slab by slab over the first `stat_planes` planes (all by
    default)."""
    from oracle import oracle as orc
    if xi is None:
        lo, hi = np.inf, -np.inf
        nzs = gdims[2] if stat_planes is None else min(stat_planes, gdims[2])
        for z0 in range(0, nzs, 32):
            v = _oracle_slab(kind, gdims, seed, z0, min(32, nzs - z0), norm)
            lo, hi = min(lo, float(v.min())), max(hi, float(v.max()))
        xi = rel * (hi - lo) if hi > lo else rel * abs(hi)
        origin = lo
    f = _oracle_slab(kind, gdims, seed, 0, zs, norm)
    fh = orc.quantize(f, xi, origin=origin)
    return f, fh, xi, (gdims[0], gdims[1], zs)


def time_cpu_oracle(f, fh, xi, dims, threads: int, reps: int = 1, extrema_only: bool = False) -> tuple[float, dict]:
    from oracle import oracle as orc
    used = orc.set_threads(threads)
    times = []
    r = None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = orc.run_correction(dims, f, fh, xi, check_segmentation=not extrema_only, extrema_only=extrema_only)
        times.append(time.perf_counter() - t0)
    n = dims[0] * dims[1] * dims[2]
    assert r.status == orc.ORC_OK, r
    return n / statistics.median(times), {"threads": used, "iterations": r.iterations,
                                          "seconds": statistics.median(times)}


def run_reference_arm(args):
    """--impl reference: the reference algorithm (C oracle port) on the host."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2601_01787_b200.dist import workload
    from oracle import oracle as orc
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    wl = workload(args, max(world, 1))
    threads = os.cpu_count() or 1
    # weak scaling: xi from the first GPU's block (every block has its statistics)
    f, fh, xi, dims = cpu_sample_inputs(args.workload, wl["gdims"], args.cpu_sample_z, args.rel, args.seed,
                                        norm=wl.get("norm"),
                                        stat_planes=args.size if wl["scaling"] == "weak" else None)
    orc.set_threads(threads)
    eo = wl["extrema_only"]
    n = dims[0] * dims[1] * dims[2]
    for _ in range(args.warmup):
        orc.run_correction(dims, f, fh, xi, check_segmentation=not eo, extrema_only=eo)
    t0 = time.perf_counter()
    iters = 0
    for _ in range(args.steps):
        r = orc.run_correction(dims, f, fh, xi, check_segmentation=not eo, extrema_only=eo)
        assert r.status == orc.ORC_OK
        iters = r.iterations
    dt = (time.perf_counter() - t0) / args.steps
    value = n / dt
    sample = (f"{dims[0]}x{dims[1]}x{dims[2]} z-slab of the {wl['label']} field (seed {args.seed}, f32), "
              f"rel {args.rel}, quantizer; full run_correction"
              f"{' (extrema-only)' if eo else ' incl. compare_plmss post-check'}; {iters} iterations")
    line = {"metric": wl["metric"] or METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f64", "data": f"synthetic ({wl['data']}, seeded)",
            "impl": "reference",
            "config": {"workload": wl["label"], "sample": sample, "cpu_threads": threads},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_ours_single(args):
    import torch
    import paper_2601_01787_b200 as pm
    from paper_2601_01787_b200 import _native as N
    from paper_2601_01787_b200 import inputs as gen
    from paper_2601_01787_b200.engine import DomainPlan, DomainSpec

    from paper_2601_01787_b200.dist import workload
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    wl = workload(args, 1)
    dims = wl["gdims"]
    nvox = dims[0] * dims[1] * dims[2]
    f32 = wl["make"]((0, 0, 0), dims, dev)
    lo, hi = gen.minmax_device(f32)
    xi = gen.relative_to_absolute_range(lo, hi, args.rel)
    fh = gen.quantize_device(f32, xi, lo, hi)
    cfg = pm.CorrectionConfig(xi_abs=xi)
    if args.f64_original:   # the same values, handed over as f64 (f64 K0)
        f32 = f32.double()
    plan = DomainPlan(DomainSpec.whole(dims), cfg.xi_abs, cfg.tau, cfg.max_outer_iterations,
                      incremental=not args.full_sweeps, f32_original=not args.f64_original,
                      extrema_only=wl["extrema_only"])
    g = torch.empty_like(fh)
    stream = torch.cuda.current_stream()

    def step():
        return pm.run_correction_device(f32, fh, dims, cfg, out=g, plan=plan, extrema_only=wl["extrema_only"])

    for _ in range(max(args.warmup, 3)):
        res = step()
    torch.cuda.synchronize()
    # events around the full-domain launches only: timing all ~40 launches of
    # a step costs ~0.15 ms (tools/prof_overhead.py); the breakdown of the
    # other kernel classes comes from a separate profiled pass below
    plan.profile(True, full_domain_only=True)
    plan.profile_read(reset=True)
    launches0 = N.launch_count()
    clocks = ClockSampler(0)
    clocks.start()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res = step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    launches = N.launch_count() - launches0
    prof = plan.profile_read(reset=True)
    plan.profile(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof_all = plan.profile_read(reset=True)
    plan.profile(False)
    value = nvox / (ms / 1e3)

    # roofline of the dominant kernels (algorithmic bytes per launch / event time)
    peaks = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    per_voxel = {"sweep_full": 9, "verify": 9, "prep": f32.element_size() + 8 + 8 + 1}   # full-domain kernels only
    kernels = {}
    for name, (kms, cnt) in prof.items():
        if name not in per_voxel:
            kms, cnt = prof_all[name]
        if cnt == 0:
            continue
        entry = {"ms_total_per_step": kms / args.steps, "launches_per_step": cnt / args.steps,
                 "ms_per_launch": kms / cnt}
        if name in per_voxel:
            gbs = per_voxel[name] * nvox / (kms / cnt / 1e3) / 1e9
            entry.update({"bytes_per_launch": per_voxel[name] * nvox, "achieved_gbs": gbs, "frac": gbs / peak})
        kernels[name] = entry
    # the roofline object describes the full-domain kernel with the largest
    # share of the step (K0 since it absorbed the first detection sweep)
    dominant = max((k for k in kernels if k in per_voxel), key=lambda k: kernels[k]["ms_total_per_step"])
    dk = kernels[dominant]
    what = {"prep": "K0 k_prep_q (validation, g <- fhat, robust screen; exact f-codes and the first detection "
                    "sweep for the fragile centres)",
            "sweep_full": "K1 k_qsweep_tma (full detection sweep over the fragile centres)",
            "verify": "K4 count sweep"}
    roofline = {"bound": "hbm", "kernel": what.get(dominant, dominant),
                "achieved": dk["achieved_gbs"], "peak": peak, "unit": "GB/s", "frac": dk["achieved_gbs"] / peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if not peaks.get("fallback")
                else "fallback 6650 GB/s", "traffic": None,
                "traffic_source": None,
                "bytes_per_voxel": per_voxel[dominant], "per_kernel": kernels,
                "per_kernel_source": "prep / sweep_full / verify: events in the timed region; other classes: "
                                     "a second, fully event-timed pass of the same steps"}

    tr = ncu_traffic(dominant, wl["label"])
    if tr is not None:
        roofline["traffic"] = tr[0]
        roofline["traffic_source"] = f"profiles/{tr[1]} (dram__bytes_read+write per launch, ncu --set full)"

    # correctness evidence of the timed run
    check = {"iterations": res.iterations, "edits_per_iteration": list(res.edits_per_iteration),
             "edit_count": int(res.edit_ids.numel()), "max_vertex_edits": res.max_vertex_edits,
             "full_sweeps": res.full_sweeps, "masked_sweeps": res.masked_sweeps,
             "fragile_fraction": round(res.fragile / float(nvox), 4) if res.fragile >= 0 else None,
             "sparse_sweeps": res.sparse_sweeps}
    # zero residual, checked independently of the loop's detection bookkeeping:
    # a full K4 count sweep of the final field (correction.py:424-426) and the
    # dense bound check (BoundsField.admits, :422-423), after the timed region
    kinds = plan.verify(res.corrected)
    check["residual"] = int(sum(kinds))
    check["residual_per_kind"] = kinds
    check["bound_violations"] = plan.bounds_violations(f32, res.corrected)
    check["residual_check"] = "full K4 count sweep + dense bound check of the final field, after the timed region"

    line = {"metric": wl["metric"] or METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic ({wl['data']} seed {args.seed} f32 + quantizer, generated on device)",
            "config": {"workload": wl["label"], "dims": list(dims), "rel": args.rel,
                       "voxels": nvox, "xi_abs": xi, "tau": cfg.tau, "extrema_only": wl["extrema_only"],
                       "mode": "full sweeps" if args.full_sweeps else "incremental dirty-ring sweeps",
                       "l2": f"inputs {nvox * 12 / 1e9:.1f} GB > 126 MB L2 (no flush needed)",
                       "parallelism": "single GPU"},
            "roofline": roofline, "clocks": clk, "gpu_launches": launches, "result": check}

    # bit-exact pin against the reference's own 512^3 result (tests/golden/
    # make_golden_large.py): corrected field, edit record, schedule
    line["result"].update(reference_pin(args, wl, f32, fh, res))
    if not args.no_e2e:
        line["e2e"] = e2e_host(args, plan, f32, fh, dims, nvox, res)
    if not args.no_dropin and not wl["extrema_only"]:
        line["dropin"] = dropin_api(args, f32, fh, dims, cfg, res)
    if not args.no_cpu_baseline:
        f, fhs, xic, sdims = cpu_sample_inputs(args.workload, dims, args.cpu_sample_z, args.rel, args.seed,
                                               xi=xi, origin=lo, norm=wl.get("norm"))
        threads = os.cpu_count() or 1
        v, info = time_cpu_oracle(f, fhs, xic, sdims, threads, extrema_only=wl["extrema_only"])
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": info["threads"], "kind": "port",
                                "sample": f"{sdims[0]}x{sdims[1]}x{sdims[2]} z-slab of the same field, "
                                          f"run_correction{' (extrema-only)' if wl['extrema_only'] else ' incl. compare_plmss'}, "
                                          f"{info['iterations']} iterations, {info['seconds']:.1f} s"}
    print(json.dumps(line), flush=True)
    return 0


def _sha(t) -> str:
    import hashlib
    import torch
    a = t.detach().cpu() if isinstance(t, torch.Tensor) else t
    return hashlib.sha256(np.ascontiguousarray(a.numpy() if hasattr(a, "numpy") else a).tobytes()).hexdigest()


def reference_pin(args, wl, f32, fh, res) -> dict:
    """Digests of this run against the reference's result on the same inputs
    (tests/golden/golden_large.json, generated by the reference itself)."""
    p = ROOT / "tests" / "golden" / "golden_large.json"
    key = {256: "c256", 512: "c512"}.get(args.size)
    out = {"corrected_sha256": _sha(res.corrected), "ids_sha256": _sha(res.edit_ids),
           "vals_sha256": _sha(res.edit_values)}
    if not p.exists() or key is None or args.workload != "perlin" or args.seed != 0 or args.rel != 1e-4:
        out["reference_pin"] = "no reference digest for this workload"
        return out
    ref = json.loads(p.read_text()).get(key)
    if ref is None or "serial" not in ref:
        out["reference_pin"] = "no reference digest for this workload"
        return out
    s = ref["serial"]
    inputs_ok = _sha(f32.float()) == ref["f32_sha256"] and _sha(fh) == ref["fhat_sha256"]
    match = (inputs_ok and out["corrected_sha256"] == s["corrected_sha256"] and out["ids_sha256"] == s["ids_sha256"]
             and out["vals_sha256"] == s["vals_sha256"] and list(res.edits_per_iteration) == s["edits_per_iteration"]
             and res.max_vertex_edits == s["max_vertex_edits"])
    out["reference_pin"] = {"source": f"tests/golden/golden_large.json[{key}] (reference run_correction, "
                                      f"{s.get('seconds', '?')} s on the build host)",
                            "inputs_match": inputs_ok, "bit_exact": bool(match)}
    return out


def dropin_api(args, f32, fh, dims, cfg, dev_res) -> dict:
    """The reference-facing Python API on host data: run_correction(ScalarField,
    ScalarField, CorrectionConfig) -> CorrectionResult (correction.py:391-436),
    i.e. what a topocorrect user calls.  Timed per call (wall clock: host f64
    arrays in, host corrected ScalarField + EditSet out), with the device path
    plus the copies it implies beside it for comparison."""
    import torch
    import paper_2601_01787_b200 as pm
    f = pm.ScalarField(dims, f32.double().cpu().numpy())
    fhat = pm.ScalarField(dims, fh.cpu().numpy())
    steps = max(2, min(args.steps, 3))
    pm.run_correction(f, fhat, cfg)   # warm-up (plan creation)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        r = pm.run_correction(f, fhat, cfg)
    dt = (time.perf_counter() - t0) / steps
    ok = (list(r.edits_per_iteration) == list(dev_res.edits_per_iteration) and r.edits.count == dev_res.edit_ids.numel()
          and _sha(r.corrected.values) == _sha(dev_res.corrected) and _sha(r.edits.ids) == _sha(dev_res.edit_ids)
          and _sha(r.edits.values) == _sha(dev_res.edit_values))
    if not ok:
        raise SystemExit("drop-in run_correction differs from the device-resident run")
    n = dims[0] * dims[1] * dims[2]
    return {"ms_per_call": dt * 1e3, "voxels_per_s": n / dt, "calls": steps, "matches_device": ok,
            "path": "paper_2601_01787_b200.run_correction(ScalarField f64 x2, CorrectionConfig) -> CorrectionResult "
                    "(pageable host f64 in, corrected ScalarField + EditSet out): pmsz_run_correction_host staging "
                    "the numpy arrays through a pinned ring, f64 original narrowed to f32 while staged, field "
                    "filled from fhat on the host and patched with the edit record",
            "ids_sha256": _sha(r.edits.ids), "values_sha256": _sha(r.edits.values)}


def e2e_host(args, plan, f32, fh, dims, nvox, dev_res) -> dict:
    """Same metric through the C ABI with HOST buffers: pinned f32 original and
    f64 decompressed in, corrected field + edit record (ids + values) out,
    copies inside the timed region (pmsz_run_correction_host).  The outputs of
    the last timed call are checked against the device-resident run."""
    import ctypes
    import torch
    from paper_2601_01787_b200 import _native as N
    L = N.lib()
    fh_host = torch.empty(nvox, dtype=torch.float64, pin_memory=True)
    f_host = torch.empty(nvox, dtype=f32.dtype, pin_memory=True)
    fh_host.copy_(fh)
    f_host.copy_(f32)
    cap = nvox // 8
    ids = torch.empty(cap, dtype=torch.int64, pin_memory=True)
    vals = torch.empty(cap, dtype=torch.float64, pin_memory=True)
    g_host = torch.empty(nvox, dtype=torch.float64, pin_memory=True)
    hist = (ctypes.c_int64 * plan.max_iterations)()
    res = N.PmszResult()
    stream = torch.cuda.current_stream()

    def call():
        st = L.pmsz_run_correction_host(plan.handle, N.ptr(f_host), N.ptr(fh_host), N.ptr(g_host), N.ptr(ids), N.ptr(vals),
                                        cap, hist, plan.max_iterations, ctypes.byref(res),
                                        N.stream_handle(stream))
        N.check(st, "pmsz_run_correction_host")

    for _ in range(2):
        call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        call()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.steps
    edits = int(res.edit_count)
    m = min(edits, cap)
    check = {"edit_count": edits, "matches_device": bool(
        edits == int(dev_res.edit_ids.numel()) and edits <= cap
        and _sha(ids[:m]) == _sha(dev_res.edit_ids) and _sha(vals[:m]) == _sha(dev_res.edit_values)
        and _sha(g_host) == _sha(dev_res.corrected)
        and list(hist[:int(res.iterations)]) == list(dev_res.edits_per_iteration))}
    if not check["matches_device"]:
        raise SystemExit("e2e host path differs from the device-resident run")
    return {"value": nvox / dt, "unit": UNIT, "h2d_bytes_per_step": nvox * (4 + 8),
            "d2h_bytes_per_step": nvox * 8 + edits * 16 + 8 * int(res.iterations), "ms_per_step": dt * 1e3,
            "path": "pmsz_run_correction_host (pinned host f32 f + f64 fhat in; corrected f64 field + edit "
                    "ids/values out; input copied in z-slabs overlapped with K0, the field streamed back slab by "
                    "slab concurrently and patched with the edit record)",
            "check": check}


def main():
    # The image sets NCCL_DEBUG=VERSION, which prints a banner on stdout at the
    # first communicator; the contract is one JSON line on stdout (an explicit
    # INFO / TRACE setting is kept, its output sent to stderr)
    if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference_arm(args)
    if world > 1 or args.gpus > 1:
        from paper_2601_01787_b200 import dist
        return dist.bench_main(args, METRIC, UNIT, ClockSampler, measured_peaks, cpu_sample_inputs,
                               time_cpu_oracle)
    return run_ours_single(args)


if __name__ == "__main__":
    sys.exit(main())
