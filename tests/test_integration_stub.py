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
