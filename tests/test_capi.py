"""The C-ABI library loads without a GPU and exports every symbol the header
declares (CPU)."""

import re
import subprocess

import pytest

from paper_2601_01787_b200 import _native as N


def declared_symbols():
    text = N.HEADER_PATH.read_text()
    return sorted(set(re.findall(r"\b(pmsz_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libpath():
    if not N.LIB_PATH.exists():
        import __graft_entry__ as g
        g.build_native()
    return N.LIB_PATH


def test_header_and_binding_agree():
    assert set(declared_symbols()) == set(N.SIGNATURES)


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", str(libpath)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (pmsz_[a-z0-9_]+)$", out, re.M))
    missing = set(declared_symbols()) - exported
    assert not missing, missing


def test_library_loads_and_binds_without_gpu(libpath):
    lib = N.load(libpath)
    assert lib.pmsz_version().startswith(b"pmsz-b200")
    assert lib.pmsz_launch_count() >= 0


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", str(libpath)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_structs_match_header_layout():
    import ctypes
    # pmsz_desc: 3 + 3 + 3 int64, 3 + 3 int32, 2 double, int64, 2 int32
    assert ctypes.sizeof(N.PmszDesc) == 9 * 8 + 6 * 4 + 2 * 8 + 8 + 2 * 4
    assert ctypes.sizeof(N.PmszResult) == 21 * 8


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        N.lib()


def _desc(N, dims, xi=0.1, tau=0.01, core=None, cap=10, flags=1):
    d = N.PmszDesc()
    d.nx, d.ny, d.nz = dims
    lo, hi = core if core is not None else ((0, 0, 0), dims)
    for a in range(3):
        d.core_lo[a], d.core_hi[a] = lo[a], hi[a]
    d.xi, d.tau, d.max_iterations, d.flags = xi, tau, cap, flags
    return d


@pytest.mark.parametrize("kw", [
    dict(dims=(0, 4, 4)),                                   # empty extent
    dict(dims=(4, 4, 4), xi=0.0),                           # xi must be positive
    dict(dims=(4, 4, 4), xi=0.1, tau=0.2),                  # tau < 2 xi (correction.py:77-91)
    dict(dims=(4, 4, 4), tau=0.0),
    dict(dims=(4, 4, 4), core=((0, 0, 0), (5, 4, 4))),      # core box outside the domain
    dict(dims=(4, 4, 4), core=((3, 0, 0), (2, 4, 4))),      # inverted core box
    dict(dims=(65536, 65536, 2)),                           # ids must fit 32 bits
])
def test_plan_create_rejects_invalid_descriptors_without_touching_the_device(libpath, kw):
    """Argument validation happens before any CUDA call, so it is testable here;
    the status maps to ValueError in engine.DomainPlan."""
    import ctypes
    lib = N.load(libpath)
    h = ctypes.c_void_p()
    st = lib.pmsz_plan_create(ctypes.byref(_desc(N, **kw)), ctypes.byref(h))
    assert st == N.PMSZ_ERR_INVALID and not h.value
    assert lib.pmsz_last_error()


def test_null_arguments_are_rejected(libpath):
    import ctypes
    lib = N.load(libpath)
    assert lib.pmsz_plan_create(None, None) == N.PMSZ_ERR_INVALID
    assert lib.pmsz_run_correction(None, None, None, None, None, 0, None, None) == N.PMSZ_ERR_INVALID
    assert lib.pmsz_edits_export(None, None, None, None, 0, None, None) == N.PMSZ_ERR_INVALID
    cnt = ctypes.c_int64(-1)
    assert lib.pmsz_bits_to_ids(None, 10, None, 0, ctypes.byref(cnt), None) == N.PMSZ_ERR_INVALID
    assert lib.pmsz_segmentation(0, 1, 1, None, 0, None, None, None) == N.PMSZ_ERR_INVALID
    g3 = (ctypes.c_int64 * 3)(4, 4, 4)
    lo = (ctypes.c_int64 * 3)(2, 0, 0)
    ext = (ctypes.c_int64 * 3)(4, 4, 4)
    assert lib.pmsz_gaussian_peaks(g3, lo, ext, 0, 0, ctypes.c_void_p(1), None) == N.PMSZ_ERR_INVALID
