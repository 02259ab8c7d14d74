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
    assert ctypes.sizeof(N.PmszResult) == 20 * 8


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        N.lib()
