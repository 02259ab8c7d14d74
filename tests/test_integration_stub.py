"""The reference-side ctypes stub of INTEGRATION.md, executed verbatim against
the reference's golden runs (the host-buffer C-ABI entry
pmsz_run_correction_host had no test)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stub():
    from paper_2601_01787_b200 import _native as N
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n(# topocorrect/_gpu.py.*?)```", text, re.S).group(1)
    os.environ["PMSZ_LIB"] = str(N.LIB_PATH)
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def _field(dims, v):
    import paper_2601_01787_b200 as pm
    return pm.ScalarField(dims, v)


@pytest.mark.parametrize("name", ["cfg1_64_q_1e-3", "cfg1_64_noise_1e-3", "p32_s12_1e-2", "golden8", "tie_1",
                                  "p2d_96_s1_1e-3", "odd_21x13x11"])
def test_stub_matches_reference(stub, golden, name):
    import paper_2601_01787_b200 as pm
    meta, arrays = golden
    run = next(r for r in meta["runs"] if r["name"] == name)
    f, fh, dims = golden_inputs(run, arrays)
    cfg = pm.CorrectionConfig(xi_abs=run["xi"], tau=run["tau"], max_outer_iterations=run["cap"])
    st, g, ids, vals, hist, res = stub["run_correction_gpu"](_field(dims, f), _field(dims, fh), cfg)
    assert st == 0
    import hashlib
    assert hashlib.sha256(g.tobytes()).hexdigest() == run["corrected_sha256"], name
    assert np.array_equal(ids, arrays[name + "_ids"]) and np.array_equal(vals, arrays[name + "_vals"]), name
    assert hist.tolist() == run["edits_per_iteration"], name
    assert res.iterations == run["iterations"] and res.max_vertex_edits == run["max_vertex_edits"]
    assert res.edit_count == run["edit_count"]


def test_stub_reports_bound_violation(stub, golden):
    import paper_2601_01787_b200 as pm
    meta, arrays = golden
    bv = meta["bound_violation"]
    dims = tuple(bv["dims"])
    st, *_, res = stub["run_correction_gpu"](_field(dims, arrays["bound_f"]), _field(dims, arrays["bound_fhat"]),
                                             pm.CorrectionConfig(xi_abs=bv["xi"]))
    assert st == 2
    assert (res.bound_first_index, res.bound_violations) == (bv["index"], bv["offenders"])


def test_host_entry_truncated_record_and_corrected_field(golden):
    """pmsz_run_correction_host directly: f32 original, edits_cap below the edit
    count (the full count still comes back), g_host NULL and non-NULL."""
    import ctypes
    import torch
    import paper_2601_01787_b200 as pm
    from paper_2601_01787_b200 import _native as N
    from paper_2601_01787_b200.engine import DomainPlan, DomainSpec
    meta, arrays = golden
    run = next(r for r in meta["runs"] if r["name"] == "cfg1_64_q_1e-3")
    f, fh, dims = golden_inputs(run, arrays)
    cfg = pm.CorrectionConfig(xi_abs=run["xi"])
    plan = DomainPlan(DomainSpec.whole(dims), cfg.xi_abs, cfg.tau, cfg.max_outer_iterations, f32_original=True)
    L = N.lib()
    f32 = np.ascontiguousarray(f.astype(np.float32))
    fh = np.ascontiguousarray(fh)
    n = f32.size
    cap = run["edit_count"] // 3
    ids = np.zeros(n, np.int64)
    vals = np.zeros(n)
    hist = (ctypes.c_int64 * 64)()
    for g in (None, np.empty(n)):
        res = N.PmszResult()
        st = L.pmsz_run_correction_host(plan.handle, f32.ctypes.data, fh.ctypes.data,
                                        None if g is None else g.ctypes.data, ids.ctypes.data, vals.ctypes.data,
                                        cap, hist, 64, ctypes.byref(res), N.stream_handle(torch.cuda.current_stream()))
        assert st == 0
        assert res.edit_count == run["edit_count"] > cap
        assert np.array_equal(ids[:cap], arrays["cfg1_64_q_1e-3_ids"][:cap])
        assert np.array_equal(vals[:cap], arrays["cfg1_64_q_1e-3_vals"][:cap])
        assert not ids[cap:].any()
        assert list(hist[:res.iterations]) == run["edits_per_iteration"]
        if g is not None:
            import hashlib
            assert hashlib.sha256(g.tobytes()).hexdigest() == run["corrected_sha256"]
    plan.close()


@pytest.mark.parametrize("dims", [(256, 128, 129), (192, 160, 144)])
def test_host_entry_slab_pipeline_matches_device(dims):
    """pmsz_run_correction_host above the slab threshold (>= 4 M voxels): the
    input arrives in 16 z-slabs (nz not a multiple of 16), K0 runs per slab,
    the corrected field streams back concurrently and is patched with the
    edit record -- all equal to the device-resident run."""
    import ctypes
    import torch
    import paper_2601_01787_b200 as pm
    from paper_2601_01787_b200 import _native as N
    from paper_2601_01787_b200 import inputs as gen
    from paper_2601_01787_b200.engine import DomainPlan, DomainSpec
    f32 = gen.perlin_device(gen.NoiseSpec(dims, 3), f32=True)
    xi = gen.relative_to_absolute_device(f32, 1e-4)
    fh = gen.quantize_device(f32, xi)
    cfg = pm.CorrectionConfig(xi_abs=xi)
    ref = pm.run_correction_device(f32, fh, dims, cfg)
    n = f32.numel()
    fh_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    f_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    fh_h.copy_(fh)
    f_h.copy_(f32)
    g_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    ids = torch.zeros(n // 4, dtype=torch.int64, pin_memory=True)
    vals = torch.zeros(n // 4, dtype=torch.float64, pin_memory=True)
    plan = DomainPlan(DomainSpec.whole(dims), cfg.xi_abs, cfg.tau, cfg.max_outer_iterations, f32_original=True)
    hist = (ctypes.c_int64 * 256)()
    for _ in range(2):   # twice: the plan's staging is reused
        res = N.PmszResult()
        st = N.lib().pmsz_run_correction_host(plan.handle, N.ptr(f_h), N.ptr(fh_h), N.ptr(g_h), N.ptr(ids),
                                              N.ptr(vals), ids.numel(), hist, 256, ctypes.byref(res),
                                              N.stream_handle(torch.cuda.current_stream()))
        assert st == 0
        m = int(res.edit_count)
        assert m == ref.edit_ids.numel() and list(hist[:res.iterations]) == list(ref.edits_per_iteration)
        assert torch.equal(g_h, ref.corrected.cpu())
        assert torch.equal(ids[:m], ref.edit_ids.cpu()) and torch.equal(vals[:m], ref.edit_values.cpu())
    plan.close()


def _slab_case(dims, seed=3):
    import paper_2601_01787_b200 as pm
    from paper_2601_01787_b200 import inputs as gen
    f32 = gen.perlin_device(gen.NoiseSpec(dims, seed), f32=True)
    xi = gen.relative_to_absolute_device(f32, 1e-4)
    fh = gen.quantize_device(f32, xi)
    cfg = pm.CorrectionConfig(xi_abs=xi)
    return f32, fh, cfg


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["pageable", "narrow", "mixed"])
def test_host_entry_pageable_buffers(mode):
    """pmsz_run_correction_host on pageable (numpy) buffers: the inputs are
    staged through the plan's pinned ring by host threads, the corrected field
    is filled from fhat on the host and patched; 'narrow' hands an f64
    original to an f32 plan (PMSZ_FLAG_HOST_F64); 'mixed' has pinned f / g and
    a pageable fhat and truncated pageable record buffers."""
    import ctypes
    import torch
    import paper_2601_01787_b200 as pm
    from paper_2601_01787_b200 import _native as N
    from paper_2601_01787_b200.engine import DomainPlan, DomainSpec
    dims = (256, 128, 129)
    f32, fh, cfg = _slab_case(dims)
    ref = pm.run_correction_device(f32, fh, dims, cfg)
    n = f32.numel()
    ref_g = ref.corrected.cpu().numpy()
    plan = DomainPlan(DomainSpec.whole(dims), cfg.xi_abs, cfg.tau, cfg.max_outer_iterations, f32_original=True,
                      host_f64=(mode == "narrow"))
    for _ in range(2):   # twice: the ring and the record bounce are reused
        if mode == "mixed":
            f_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
            f_h.copy_(f32)
            g_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
            fh_h = fh.cpu().numpy()
            cap = ref.edit_ids.numel() // 3
            ids = np.zeros(cap, dtype=np.int64)
            vals = np.zeros(cap, dtype=np.float64)
            hist = (ctypes.c_int64 * 256)()
            res = N.PmszResult()
            st = N.lib().pmsz_run_correction_host(plan.handle, N.ptr(f_h), fh_h.ctypes.data, N.ptr(g_h),
                                                  ids.ctypes.data, vals.ctypes.data, cap, hist, 256,
                                                  ctypes.byref(res), None)
            assert st == 0 and int(res.edit_count) == ref.edit_ids.numel()
            assert np.array_equal(g_h.numpy(), ref_g)
            assert np.array_equal(ids, ref.edit_ids[:cap].cpu().numpy())
            assert np.array_equal(vals, ref.edit_values[:cap].cpu().numpy())
            continue
        f_h = f32.cpu().numpy() if mode == "pageable" else f32.double().cpu().numpy()
        fh_h = fh.cpu().numpy()
        g_h = np.empty(n, dtype=np.float64)
        st, res, hist, ids, vals = plan.run_host(f_h, fh_h, g_h)
        assert st == 0
        assert list(hist) == list(ref.edits_per_iteration)
        assert np.array_equal(g_h, ref_g)
        assert np.array_equal(ids, ref.edit_ids.cpu().numpy())
        assert np.array_equal(vals, ref.edit_values.cpu().numpy())
    plan.close()


@pytest.mark.gpu
@pytest.mark.parametrize("where", ["first", "last"])
def test_host_f64_inexact_original(where):
    """PMSZ_FLAG_HOST_F64 with an original that does not narrow exactly: the
    staging thread reports it before K0 has seen the slab, the call returns
    PMSZ_ERR_INEXACT with no iteration run, and the drop-in reruns on an f64
    plan -- equal to the device f64 run."""
    import torch
    import paper_2601_01787_b200 as pm
    from paper_2601_01787_b200 import _native as N
    from paper_2601_01787_b200.engine import DomainPlan, DomainSpec
    dims = (256, 128, 129)
    f32, fh, cfg = _slab_case(dims, seed=5)
    f64 = f32.double()
    i = 7 if where == "first" else f64.numel() - 300
    f64[i] = f64[i] + abs(float(f64[i])) * 2.0 ** -40 + 1e-300   # no longer an f32 value, same order
    plan = DomainPlan(DomainSpec.whole(dims), cfg.xi_abs, cfg.tau, cfg.max_outer_iterations, f32_original=True,
                      host_f64=True)
    st, res, hist, ids, vals = plan.run_host(f64.cpu().numpy(), fh.cpu().numpy(), np.empty(f64.numel()))
    assert st == N.PMSZ_ERR_INEXACT and res.iterations == 0
    plan.close()
    ref = pm.run_correction_device(f64, fh, dims, cfg)
    out = pm.run_correction(pm.ScalarField(dims, f64.cpu().numpy()), pm.ScalarField(dims, fh.cpu().numpy()), cfg)
    assert np.array_equal(out.corrected.values, ref.corrected.cpu().numpy())
    assert np.array_equal(out.edits.ids, ref.edit_ids.cpu().numpy())
    assert np.array_equal(out.edits.values, ref.edit_values.cpu().numpy())
    assert out.edits_per_iteration == ref.edits_per_iteration
    assert out.max_vertex_edits == ref.max_vertex_edits


@pytest.mark.gpu
def test_dropin_at_slab_size_matches_device():
    """The drop-in run_correction(ScalarField, ...) above the slab threshold
    (narrowed f32 original, pageable arrays) equals the device run."""
    import paper_2601_01787_b200 as pm
    dims = (192, 160, 144)
    f32, fh, cfg = _slab_case(dims, seed=9)
    ref = pm.run_correction_device(f32, fh, dims, cfg)
    out = pm.run_correction(pm.ScalarField(dims, f32.double().cpu().numpy()),
                            pm.ScalarField(dims, fh.cpu().numpy()), cfg)
    assert np.array_equal(out.corrected.values, ref.corrected.cpu().numpy())
    assert np.array_equal(out.edits.ids, ref.edit_ids.cpu().numpy())
    assert np.array_equal(out.edits.values, ref.edit_values.cpu().numpy())
    assert np.all(np.diff(out.edits.ids) > 0)
    assert out.iterations == ref.iterations and out.edits_per_iteration == ref.edits_per_iteration
    # recycled output arrays (HostFieldCache): a held result is never overwritten,
    # a dropped one is reused
    ref_g = ref.corrected.cpu().numpy()
    held = out.corrected.values[::7]           # a view keeps the array alive
    base = id(out.corrected.values.base)     # (an id: a reference would keep it busy)
    del out
    f = pm.ScalarField(dims, f32.double().cpu().numpy())
    fhat = pm.ScalarField(dims, fh.cpu().numpy())
    from paper_2601_01787_b200.engine import HOST_FIELDS
    second = pm.run_correction(f, fhat, cfg)
    assert id(second.corrected.values.base) != base
    del held
    third = pm.run_correction(f, fhat, cfg)
    if HOST_FIELDS.enabled:   # (PMSZ_HOST_CACHE=0: fresh arrays)
        assert id(third.corrected.values.base) == base
    for r in (second, third):
        assert np.array_equal(r.corrected.values, ref_g)
        assert np.array_equal(r.edits.ids, ref.edit_ids.cpu().numpy())


@pytest.mark.parametrize("n", [1, 1000, (32 << 20) // 8 + 3, 3 * (32 << 20) // 8 + 77])
def test_staged_host_device_copies(n):
    """pmsz_host_to_device / pmsz_device_to_host on pageable numpy arrays
    (pinned ring, host threads, streaming stores): exact bytes both ways for
    sizes around the 32 MiB ring chunk, and the f64 -> f32 narrowing reports
    a value that does not survive the round trip."""
    import ctypes
    import torch
    from paper_2601_01787_b200 import _native as N
    rng = np.random.default_rng(n)
    src = rng.standard_normal(n)
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    N.check(N.lib().pmsz_host_to_device(N.ptr(dev), src.ctypes.data, src.nbytes, 0, None, None), "h2d")
    assert np.array_equal(dev.cpu().numpy(), src)
    back = np.empty(n)
    N.check(N.lib().pmsz_device_to_host(back.ctypes.data, N.ptr(dev), back.nbytes, None), "d2h")
    assert np.array_equal(back, src)
    exact = src.astype(np.float32).astype(np.float64)
    d32 = torch.empty(n, dtype=torch.float32, device="cuda")
    bad = ctypes.c_int64(-1)
    N.check(N.lib().pmsz_host_to_device(N.ptr(d32), exact.ctypes.data, n, 1, ctypes.byref(bad), None), "narrow")
    assert bad.value == 0 and np.array_equal(d32.cpu().numpy(), exact.astype(np.float32))
    exact[n // 2] += 2.0 ** -40 * (1 + abs(exact[n // 2]))
    N.check(N.lib().pmsz_host_to_device(N.ptr(d32), exact.ctypes.data, n, 1, ctypes.byref(bad), None), "narrow")
    assert bad.value == 1


def test_run_parallel_dropin_staged_matches_device():
    """run_parallel(ScalarField, ...) above the staging threshold: the original
    is narrowed while staged, the result comes back through the staged copy
    into a recycled array -- equal to the single-domain device run (lockstep)
    and bit-identical across two calls."""
    import paper_2601_01787_b200 as pm
    dims = (128, 96, 130)
    f32, fh, cfg = _slab_case(dims, seed=11)
    ref = pm.run_correction_device(f32, fh, dims, cfg)
    f = pm.ScalarField(dims, f32.double().cpu().numpy())
    fhat = pm.ScalarField(dims, fh.cpu().numpy())
    a, sa = pm.run_parallel(f, fhat, cfg, (1, 2, 2), pm.SyncStrategy.LOCKSTEP)
    b, sb = pm.run_parallel(f, fhat, cfg, (1, 2, 2), pm.SyncStrategy.LOCKSTEP)
    assert np.array_equal(a.corrected.values, ref.corrected.cpu().numpy())
    assert np.array_equal(a.edits.ids, ref.edit_ids.cpu().numpy())
    assert np.array_equal(a.edits.values, ref.edit_values.cpu().numpy())
    assert np.array_equal(b.corrected.values, a.corrected.values) and sa.rounds == sb.rounds


@pytest.mark.parametrize("dims", [(2048, 1024, 3), (3000, 2000, 1), (1024, 64, 65)])
def test_dropin_staging_odd_slab_layouts(dims):
    """The staged host path where the z-slabs are single planes (nz = 3),
    where there is one plane (2-D: one slab), and with a chunk size that does
    not divide the slabs -- equal to the device run."""
    import paper_2601_01787_b200 as pm
    f32, fh, cfg = _slab_case(dims, seed=13)
    ref = pm.run_correction_device(f32, fh, dims, cfg)
    out = pm.run_correction(pm.ScalarField(dims, f32.double().cpu().numpy()),
                            pm.ScalarField(dims, fh.cpu().numpy()), cfg)
    assert np.array_equal(out.corrected.values, ref.corrected.cpu().numpy())
    assert np.array_equal(out.edits.ids, ref.edit_ids.cpu().numpy())
    assert out.edits_per_iteration == ref.edits_per_iteration
