"""sync_ghosts / local_converge (parallel.py:143-172) against goldens generated
by the reference itself (tests/golden/make_golden_api.py): the oracle on CPU,
the device implementation of the drop-in on the GPU."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as orc


@pytest.fixture(scope="module")
def api_golden():
    meta = json.loads((GOLDEN / "golden_api.json").read_text())
    arrays = dict(np.load(GOLDEN / "golden_api.npz"))
    return meta, arrays


def _block(pm, e):
    return pm.Block(tuple(e["block_index"]), tuple(e["core_start"]), tuple(e["core_stop"]),
                    tuple(e["ext_start"]), tuple(e["ext_stop"]))


def test_oracle_sync_ghosts_matches_reference(api_golden):
    meta, arrays = api_golden
    for case in meta["sync_ghosts"]:
        k = case["key"]
        arrs = [arrays[f"{k}_in{i}"].copy() for i in range(case["blocks"])]
        assert orc.sync_ghosts(case["dims"], case["grid"], arrs) == case["changed"], k
        for i, a in enumerate(arrs):
            assert np.array_equal(a, arrays[f"{k}_out{i}"]), (k, i)
        assert orc.sync_ghosts(case["dims"], case["grid"], arrs) == case["changed_again"], k


def test_oracle_local_converge_matches_reference(api_golden):
    meta, arrays = api_golden
    for e in meta["local_converge"]:
        k = e["key"]
        args = (e["core_start"], e["core_stop"], e["ext_start"], e["ext_stop"], arrays[k + "_f"],
                arrays[k + "_g"], arrays[k + "_lower"], e["tau"], e["cap"])
        if e["error"] == "AssertionError":
            with pytest.raises(AssertionError):
                orc.local_converge(*args)
        elif e["error"] == "ConvergenceError":
            with pytest.raises(RuntimeError):
                orc.local_converge(*args)
        else:
            g, it, ed = orc.local_converge(*args)
            assert np.array_equal(g, arrays[k + "_out"]), k
            assert (it, ed) == (e["iterations"], e["edits"]), k


@pytest.mark.gpu
def test_sync_ghosts_matches_reference(api_golden):
    import torch
    import paper_2601_01787_b200 as pm
    meta, arrays = api_golden
    for case in meta["sync_ghosts"]:
        k = case["key"]
        decomp = pm.decompose(case["dims"], case["grid"])
        arrs = [arrays[f"{k}_in{i}"].copy() for i in range(case["blocks"])]
        assert pm.sync_ghosts(decomp, arrs) == case["changed"], k
        for i, a in enumerate(arrs):
            assert np.array_equal(a, arrays[f"{k}_out{i}"]), (k, i)
        assert pm.sync_ghosts(decomp, arrs) == case["changed_again"], k
        # device tensors are merged in place
        dev = [torch.from_numpy(arrays[f"{k}_in{i}"]).cuda() for i in range(case["blocks"])]
        assert pm.sync_ghosts(decomp, dev) == case["changed"], k
        for i, t in enumerate(dev):
            assert np.array_equal(t.cpu().numpy(), arrays[f"{k}_out{i}"]), (k, i)
    with pytest.raises(ValueError):
        pm.sync_ghosts(pm.decompose((4, 1, 1), (2, 1, 1)), [np.zeros(3)])


@pytest.mark.gpu
def test_local_converge_matches_reference(api_golden):
    import paper_2601_01787_b200 as pm
    meta, arrays = api_golden
    for e in meta["local_converge"]:
        k = e["key"]
        cfg = pm.CorrectionConfig(xi_abs=e["xi"], tau=e["tau"], max_outer_iterations=e["cap"])
        args = (_block(pm, e), arrays[k + "_f"], arrays[k + "_g"], arrays[k + "_lower"], cfg)
        if e["error"] == "AssertionError":
            with pytest.raises(AssertionError):
                pm.local_converge(*args)
        elif e["error"] == "ConvergenceError":
            with pytest.raises(pm.ConvergenceError):
                pm.local_converge(*args)
        else:
            g0 = arrays[k + "_g"].copy()
            g, it, ed = pm.local_converge(*args)
            assert np.array_equal(g, arrays[k + "_out"]), k
            assert (it, ed) == (e["iterations"], e["edits"]), k
            assert np.array_equal(arrays[k + "_g"], g0)   # the input is not modified


def test_oracle_h6_outcome_matches_reference():
    meta = json.loads((GOLDEN / "golden_api.json").read_text())["h6"]
    fh = np.load(GOLDEN / "golden_api.npz")["h6_fhat"]
    dims = tuple(meta["dims"])
    f = orc.perlin(dims, meta["seed"])
    assert meta["outcome"] == "AssertionError"
    assert orc.run_correction(dims, f, fh, meta["xi"]).status == orc.ORC_MONOTONE


@pytest.mark.gpu
@pytest.mark.parametrize("cap", [70000, 10 ** 9])
def test_huge_iteration_cap(golden, cap):
    """a legal but huge max_outer_iterations must not size device or
    pinned buffers (history chunks, u32 edit counts past 65535 iterations)."""
    import hashlib
    import paper_2601_01787_b200 as pm
    from conftest import golden_inputs
    meta, arrays = golden
    run = next(r for r in meta["runs"] if r["name"] == "golden8")
    f, fh, dims = golden_inputs(run, arrays)
    res = pm.run_correction(pm.ScalarField(dims, f), pm.ScalarField(dims, fh),
                            pm.CorrectionConfig(xi_abs=run["xi"], max_outer_iterations=cap))
    assert list(res.edits_per_iteration) == run["edits_per_iteration"]
    assert res.max_vertex_edits == run["max_vertex_edits"]
    assert hashlib.sha256(res.corrected.values.tobytes()).hexdigest() == run["corrected_sha256"]
