"""Pin the CPU oracle to the reference's own outputs (tests/golden, generated
by make_golden.py from /root/reference).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import golden_inputs
from oracle import oracle as orc
from paper_2601_01787_b200 import codec
from paper_2601_01787_b200.correction import EditSet


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_scan_matches_reference(golden):
    meta, arrays = golden
    for case in meta["scans"]:
        k = case["key"]
        s = orc.scan(arrays[k + "_v"], case["dims"])
        assert np.array_equal(s.nmax, arrays[k + "_nmax"]), k
        assert np.array_equal(s.nmin, arrays[k + "_nmin"]), k
        assert np.array_equal(s.is_max, arrays[k + "_ismax"]), k
        assert np.array_equal(s.is_min, arrays[k + "_ismin"]), k


def test_perlin_and_quantize_match_reference(golden):
    meta, _ = golden
    for p in meta["perlin"]:
        f = orc.perlin(p["dims"], p["seed"], p["frequency"], p["octaves"])
        assert sha(f) == p["sha256"], p
        assert sha(f.astype(np.float32)) == p["f32_sha256"]
        xi = orc.relative_to_absolute(f, 1e-3)
        assert xi == p["xi_rel_1e-3"]
        assert sha(orc.quantize(f, xi)) == p["quantized_sha256"]


def test_perlin_sub_box_is_a_slice_of_the_whole():
    dims = (20, 17, 9)
    whole = orc.perlin(dims, 7).reshape(9, 17, 20)
    part = orc.perlin(dims, 7, lo=(3, 5, 2), ext=(10, 6, 4)).reshape(4, 6, 10)
    assert np.array_equal(part, whole[2:6, 5:11, 3:13])


def test_iterate_trajectory_matches_reference(golden):
    meta, _ = golden
    for case in meta["iterate"]:
        dims = (8, 8, 8)
        f = orc.perlin(dims, case["seed"])
        fh = orc.quantize(f, case["xi"])
        fs = orc.scan(f, dims)
        g = fh
        for step in case["trajectory"]:
            g, ed = orc.iterate(dims, fs, g, f - case["xi"], case["tau"])
            assert int(ed.sum()) == step["edits"]
            assert sha(g) == step["g_sha256"]
            assert sha(ed) == step["edited_sha256"]


def test_run_correction_matches_reference(golden):
    meta, arrays = golden
    for run in meta["runs"]:
        f, fh, dims = golden_inputs(run, arrays)
        assert sha(f) == run["f_sha256"] and sha(fh) == run["fhat_sha256"], run["name"]
        r = orc.run_correction(dims, f, fh, run["xi"], run["tau"], run["cap"])
        assert r.status == orc.ORC_OK, run["name"]
        assert r.iterations == run["iterations"]
        assert list(r.edits_per_iteration) == run["edits_per_iteration"]
        assert r.max_vertex_edits == run["max_vertex_edits"]
        assert sha(r.corrected) == run["corrected_sha256"], run["name"]
        ids = np.flatnonzero(r.corrected != fh)
        assert np.array_equal(ids, arrays[run["name"] + "_ids"])
        assert np.array_equal(r.corrected[ids], arrays[run["name"] + "_vals"])


def test_failure_modes_match_reference(golden):
    meta, arrays = golden
    bv = meta["bound_violation"]
    r = orc.run_correction((8, 8, 1), arrays["bound_f"], arrays["bound_fhat"], bv["xi"])
    assert r.status == orc.ORC_BOUND
    assert (r.bound_first, r.bound_count) == (bv["index"], bv["offenders"])
    f = orc.perlin((8, 8, 8), 42)
    xi = orc.relative_to_absolute(f, 1e-1)
    r = orc.run_correction((8, 8, 8), f, orc.quantize(f, xi), xi, max_iter=meta["cap_error"]["cap"])
    assert r.status == orc.ORC_CONVERGENCE and r.conv_kind == 1


def test_golden_edits_file_hash(golden):
    meta, arrays = golden
    run = next(r for r in meta["runs"] if r["name"] == "golden8")
    edits = EditSet(arrays["golden8_ids"], arrays["golden8_vals"], 512)
    blob = codec.encode_edits(edits, run["xi"], run["tau"])
    assert hashlib.sha256(blob).hexdigest() == meta["golden_edits_sha256"]
    back, xi, tau = codec.decode_edits_meta(blob)
    assert np.array_equal(back.ids, edits.ids) and np.array_equal(back.values, edits.values)
    assert (xi, tau) == (run["xi"], run["tau"])


def test_edits_codec_large_ids_round_trip():
    rng = np.random.default_rng(0)
    ids = np.unique(rng.integers(0, 2**40, 5000))
    e = EditSet(ids, rng.standard_normal(ids.size), 2**41)
    back = codec.decode_edits(codec.encode_edits(e, 0.1, 0.001))
    assert np.array_equal(back.ids, e.ids) and np.array_equal(back.values, e.values)
    with pytest.raises(codec.FormatError):
        codec.decode_edits(codec.encode_edits(e, 0.1, 0.001)[:-1] + b"\x00")


@pytest.mark.parametrize("idx", range(18))
def test_run_parallel_matches_reference(golden, idx):
    meta, arrays = golden
    case = meta["parallel"][idx]
    dims = tuple(case["dims"])
    f = orc.perlin(dims, case["seed"])
    fh = orc.quantize(f, case["xi"])
    g, st = orc.run_parallel(dims, f, fh, case["xi"], tuple(case["grid"]), case["strategy"] == "lockstep")
    ref = case["stats"]
    assert st["rounds"] == ref["rounds"] and st["syncs"] == ref["syncs"]
    assert list(st["per_block_iterations"]) == ref["per_block_iterations"]
    assert list(st["per_block_edit_totals"]) == ref["per_block_edit_totals"]
    assert list(st["per_block_max_vertex_edits"]) == ref["per_block_max_vertex_edits"]
    assert list(st["edits_per_iteration"]) == case["edits_per_iteration"]
    assert sha(g) == case["corrected_sha256"], case["name"]


def test_bounded_noise_respects_bound_and_floor():
    dims = (16, 12, 8)
    f = orc.perlin(dims, 3).astype(np.float32).astype(np.float64)
    xi = orc.relative_to_absolute(f, 1e-3)
    fh = orc.bounded_noise(f, dims, xi, 11)
    assert np.all(np.abs(f - fh) <= xi)
    assert np.all(fh >= f - xi)
    assert not np.array_equal(fh, f)
    part = orc.bounded_noise(f.reshape(8, 12, 16)[2:5, 1:7, 4:9].reshape(-1), (5, 6, 3), xi, 11,
                             gdims=dims, lo=(4, 1, 2))
    assert np.array_equal(part, fh.reshape(8, 12, 16)[2:5, 1:7, 4:9].reshape(-1))


# --- segmentation / compare_plmss / field + label files ------------------------
def test_oracle_segmentation_matches_reference(golden):
    meta, arrays = golden
    for case in meta["segmentation"]:
        k = case["key"]
        a, d = orc.segmentation(arrays[k + "_v"], case["dims"])
        assert np.array_equal(a, arrays[k + "_asc"]), k
        assert np.array_equal(d, arrays[k + "_desc"]), k


def test_oracle_compare_plmss_matches_reference(golden):
    meta, arrays = golden
    for case in meta["segmentation"]:
        k = case["key"]
        rep = orc.compare_plmss(arrays[k + "_v"], arrays[k + "_w"], case["dims"])
        ref = case["report"]
        for name in ("fp_max", "fn_max", "fp_min", "fn_min", "asc_order_violations", "desc_order_violations"):
            assert rep[name].tolist() == ref[name], (k, name)
        assert rep["wrong_label_count"] == ref["wrong_label_count"], k


def test_golden_field_and_label_files(golden):
    """test_codec.py:15-26,228-235: the reference's golden field / label file
    hashes, reproduced through this codec from the oracle's Perlin and
    segmentation."""
    import paper_2601_01787_b200 as pm
    meta, _ = golden
    g = meta["golden_labels"]
    f = pm.ScalarField((8, 8, 8), orc.perlin((8, 8, 8), 42))
    assert hashlib.sha256(codec.write_field(f)).hexdigest() == g["field_file_sha256"]
    assert hashlib.sha256(codec.write_field(f, precision="f32")).hexdigest() == g["field_f32_file_sha256"]
    a, d = orc.segmentation(f.values, f.dims)
    assert hashlib.sha256(codec.write_labels(f.dims, a)).hexdigest() == g["asc_file_sha256"]
    assert hashlib.sha256(codec.write_labels(f.dims, d)).hexdigest() == g["desc_file_sha256"]


def test_field_and_label_codec_round_trips():
    import paper_2601_01787_b200 as pm
    f = pm.ScalarField((6, 5, 4), orc.perlin((6, 5, 4), 0))
    back = codec.read_field(codec.write_field(f))
    assert back.dims == f.dims and np.array_equal(back.values, f.values)
    b32 = codec.read_field(codec.write_field(f, precision="f32"))
    assert np.array_equal(b32.values, f.values.astype(np.float32).astype(np.float64))
    f2 = pm.ScalarField((4, 3), orc.perlin((4, 3, 1), 3))
    data2 = codec.write_field(f2, precision="f32")
    assert data2[8] == 2 and codec.read_field(data2).dims == (4, 3, 1)
    a, _ = orc.segmentation(f.values, f.dims)
    dims, lab = codec.read_labels(codec.write_labels(f.dims, a))
    assert dims == f.dims and np.array_equal(lab, a)
    with pytest.raises(codec.FormatError):
        codec.read_labels(codec.write_field(f))
    with pytest.raises(codec.FormatError):
        codec.read_field(codec.write_labels(f.dims, a))
    with pytest.raises(ValueError):
        codec.write_labels((2, 2, 1), np.array([0, 1, 2]))
    with pytest.raises(ValueError):
        codec.write_labels((2, 2, 1), np.array([0, 1, 2, 4]))
    with pytest.raises(codec.FormatError):
        codec.read_field(codec.write_field(f) + b"\x00")


# --- extrema-only mode ------------------------------------------------
def test_oracle_extrema_only_matches_reference_iteration(golden):
    """orc_run_correction(extrema_only) == the reference's _iterate_array with
    the order masks zeroed, iterated to a zero-edit pass."""
    meta, _ = golden
    for case in meta["extrema_only"]:
        dims = tuple(case["dims"])
        f = orc.peaks(dims, 7) if case["name"].startswith("peaks") else orc.perlin(dims, 11)
        assert hashlib.sha256(f.tobytes()).hexdigest() == case["f_sha256"]
        fh = orc.quantize(f, case["xi"])
        assert hashlib.sha256(fh.tobytes()).hexdigest() == case["fhat_sha256"]
        r = orc.run_correction(dims, f, fh, case["xi"], extrema_only=True, check_segmentation=False)
        assert r.status == orc.ORC_OK, case["name"]
        assert list(r.edits_per_iteration) == case["edits_per_iteration"], case["name"]
        assert r.max_vertex_edits == case["max_vertex_edits"]
        assert hashlib.sha256(r.corrected.tobytes()).hexdigest() == case["corrected_sha256"]
        assert case["extrema_clean"] and case["order_violations_left"] > 0


def test_peak_stack_properties():
    v = orc.peaks((128, 128, 64), 3)
    assert v.min() >= 0.0 and v.max() < 1.02
    assert 0.0005 < (v > 0.05).mean() < 0.01          # sparse spots
    sub = orc.peaks((128, 128, 64), 3, lo=(5, 70, 9), ext=(40, 30, 20))
    assert np.array_equal(sub.reshape(20, 30, 40), v.reshape(64, 128, 128)[9:29, 70:100, 5:45])
