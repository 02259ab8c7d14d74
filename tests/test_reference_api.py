"""The reference's public names beyond run_correction / run_parallel: the
record route (detect_distortions, propose_corrections, correction_iteration,
Distortion, DistortionKind -- correction.py:133-160,245-325), the per-vertex
helpers (topology.py:93-122,177-194) and the synthetic generators
(synth.py:108-121).  The 3 x 3 known-answer cases are the reference suite's
(test_correction.py:15-43); the rest holds the device paths against the
host record route, as the reference holds its two routes together."""

import numpy as np
import pytest

import paper_2601_01787_b200 as pm
from oracle import oracle as orc
from paper_2601_01787_b200.records import apply_proposals

pytestmark = pytest.mark.gpu

K = pm.DistortionKind
# a different neighbour dips below the centre's original steepest-descent one
DESC = ([0.15, 0.10, 0.40, 0.50, 0.60, 0.70, 0.90, 0.80, 0.95],
        [0.08, 0.10, 0.40, 0.50, 0.60, 0.70, 0.90, 0.80, 0.95], 0.1, 0.1)
# a spurious neighbour overtakes the centre's original largest one
ASC = ([0.02, 0.08, 0.12, 0.00, 0.20, 0.30, 0.05, 0.10, 0.25],
       [0.02, 0.08, 0.12, 0.00, 0.20, 0.30, 0.05, 0.10, 0.40], 0.3, 0.05)


def _pair(case):
    f, g, xi, tau = case
    return pm.ScalarField((3, 3), f), pm.ScalarField((3, 3), g), xi, tau


def test_detect_records_known_answers():
    f, g, _, _ = _pair(DESC)
    recs = pm.detect_distortions(f, g)
    assert [(r.kind, r.center) for r in recs] == [(K.FALSE_MINIMUM, 0), (K.MISSING_MINIMUM, 1), (K.DESC_ORDER, 4)]
    assert (recs[-1].anchor, recs[-1].targets) == (0, (1,))
    f, g, _, _ = _pair(ASC)
    recs = pm.detect_distortions(f, g)
    assert [(r.kind, r.center) for r in recs] == [(K.ASC_ORDER, 4), (K.MISSING_MAXIMUM, 5), (K.FALSE_MAXIMUM, 8)]
    assert (recs[0].anchor, recs[0].targets) == (5, (8,))
    spike = pm.ScalarField((3, 3), np.arange(9.0))
    g = spike.values.copy()
    g[4] = 100.0
    kinds = {(r.kind, r.center) for r in pm.detect_distortions(spike, spike.with_values(g))}
    assert (K.FALSE_MAXIMUM, 4) in kinds and (K.MISSING_MAXIMUM, 8) in kinds
    assert pm.detect_distortions(spike, spike) == []
    with pytest.raises(ValueError):
        pm.detect_distortions(spike, pm.ScalarField((4, 3), np.zeros(12)))


def test_propose_and_iterate_known_answers():
    g = pm.ScalarField((2, 2), [0.5, 0.9, 0.2, 0.8])
    recs = [pm.Distortion(K.FALSE_MAXIMUM, 1, 0, (1,)), pm.Distortion(K.DESC_ORDER, 3, 2, (1,))]
    assert pm.propose_corrections(g, 0.1, recs) == {1: pytest.approx(0.2 - 0.1)}
    f, g, xi, tau = _pair(DESC)
    assert pm.propose_corrections(g, tau, pm.detect_distortions(f, g)) == {1: pytest.approx(0.08 - tau)}
    g1, e = pm.correction_iteration(f, g, pm.compute_bounds(f, xi), tau)
    assert e == 1 and g1.values[1] == 0.0 and np.flatnonzero(g1.values != g.values).tolist() == [1]
    f, g, xi, tau = _pair(ASC)
    g1, e = pm.correction_iteration(f, g, pm.compute_bounds(f, xi), tau)
    assert e == 1 and g1.values[8] == pytest.approx(0.30 - tau) and np.all(g1.values <= g.values)


@pytest.mark.parametrize("seed,rel", [(0, 1e-1), (1, 1e-2), (2, 1e-3), (3, 1e-1)])
def test_device_iteration_equals_record_route(seed, rel):
    """correction_iteration (device array engine) == the host record route
    (detect -> propose -> apply_edit) at every iteration to the fixpoint."""
    dims = (10, 9, 8) if seed % 2 else (12, 11, 1)
    f = pm.ScalarField(dims, orc.perlin(dims, seed))
    xi = pm.relative_to_absolute(f, rel)
    _, g = pm.quantize(f, xi)
    bounds = pm.compute_bounds(f, xi)
    tau = pm.CorrectionConfig(xi_abs=xi).tau
    for _ in range(200):
        ref, ref_e = apply_proposals(g, pm.propose_corrections(g, tau, pm.detect_distortions(f, g)), bounds.lower)
        dev, dev_e = pm.correction_iteration(f, g, bounds, tau)
        assert dev_e == ref_e and np.array_equal(dev.values, ref.values)
        g = dev
        if dev_e == 0:
            break
    else:
        pytest.fail("no fixpoint")


def test_iteration_below_the_floor_clamps_like_the_record_route():
    f = pm.ScalarField((6, 5, 4), orc.perlin((6, 5, 4), 9))
    xi = pm.relative_to_absolute(f, 1e-1)
    bounds = pm.compute_bounds(f, xi)
    low = f.values - 2 * xi            # below the floor everywhere
    g = pm.ScalarField(f.dims, low)
    tau = xi / 1024
    ref = apply_proposals(g, pm.propose_corrections(g, tau, pm.detect_distortions(f, g)), bounds.lower)
    dev = pm.correction_iteration(f, g, bounds, tau)
    assert dev[1] == ref[1] and np.array_equal(dev[0].values, ref[0].values)


def test_per_vertex_helpers_and_generators():
    f = pm.ScalarField((7, 6, 5), orc.perlin((7, 6, 5), 4))
    s = pm.field_scan(f)
    for v in range(0, f.vertex_count, 7):
        assert pm.extreme_neighbor(f, v, "ascending") == s.nmax[v]
        assert pm.extreme_neighbor(f, v, "descending") == s.nmin[v]
        assert pm.is_maximum(f, v) == bool(s.is_max[v]) and pm.is_minimum(f, v) == bool(s.is_min[v])
    with pytest.raises(ValueError):
        pm.extreme_neighbor(f, 0, "sideways")
    a, b = pm.compute_segmentation_naive(f), pm.compute_segmentation(f)
    assert np.array_equal(a.asc_target, b.asc_target) and np.array_equal(a.desc_target, b.desc_target)
    r = pm.ramp((4, 3, 2))
    assert r.values[1 + 4 * 1 + 12 * 1] == 1.0 + 2.0 + 4.0 and pm.find_extrema(r).maxima == {23}
    c = pm.constant((3, 3), 2.5)
    assert c.dims == (3, 3, 1) and np.all(c.values == 2.5)
    assert issubclass(pm.PayloadFormatError, ValueError)
