"""Host-side logic of the drop-in API (CPU): types, validation, decomposition,
shared bands."""

import numpy as np
import pytest

import paper_2601_01787_b200 as pm
from oracle import oracle as orc


def test_scalar_field_validation():
    f = pm.ScalarField((3, 2), np.arange(6.0))
    assert f.dims == (3, 2, 1) and f.is_2d and not f.values.flags.writeable
    with pytest.raises(ValueError):
        pm.ScalarField((3, 1, 1), np.zeros(3))
    with pytest.raises(ValueError):
        pm.ScalarField((2, 2), [0.0, np.nan, 1.0, 2.0])
    with pytest.raises(ValueError):
        pm.ScalarField((2, 2), np.zeros(5))


def test_config_defaults_and_validation():
    c = pm.CorrectionConfig(xi_abs=1.0)
    assert c.tau == 1.0 / 1024 and c.max_outer_iterations == 10 * 2048
    assert c.per_vertex_edit_budget == 2049
    for bad in (dict(xi_abs=0.0), dict(xi_abs=1.0, tau=2.0), dict(xi_abs=1.0, tau=0.0),
                dict(xi_abs=1.0, max_outer_iterations=0)):
        with pytest.raises(ValueError):
            pm.CorrectionConfig(**bad)


def test_rank_offsets_are_ascending_ids():
    for nx, ny in ((2, 2), (3, 5), (7, 4)):
        deltas = [dx + nx * (dy + ny * dz) for dx, dy, dz in pm.RANK_OFFSETS]
        assert deltas == sorted(deltas)
    assert pm.RANK_OFFSETS[6] == (-1, 0, 0) and pm.RANK_OFFSETS[7] == (1, 0, 0)


def test_neighbors_and_precedes():
    assert sorted(pm.neighbors((3, 3, 3), 13)) == sorted(
        13 + dx + 3 * (dy + 3 * dz) for dx, dy, dz in pm.STENCIL)
    f = pm.ScalarField((2, 2), [1.0, 1.0, 0.0, 2.0])
    assert pm.precedes(f, 0, 1) and not pm.precedes(f, 1, 0) and pm.precedes(f, 2, 0)


@pytest.mark.parametrize("dims,grid", [((8, 8, 1), (2, 2, 1)), ((7, 5, 1), (3, 2, 1)), ((6, 6, 6), (2, 2, 2)),
                                       ((9, 4, 5), (4, 2, 2)), ((5, 5, 5), (1, 1, 1)), ((16, 16, 24), (1, 1, 4))])
def test_decompose_matches_oracle(dims, grid):
    d = pm.decompose(dims, grid)
    ref = orc.decompose(dims, grid)
    assert [(b.index, b.core_start, b.core_stop, b.ext_start, b.ext_stop) for b in d.blocks] == ref


def test_decompose_rejects_bad_grids():
    with pytest.raises(ValueError):
        pm.decompose((4, 4, 1), (5, 1, 1))
    with pytest.raises(ValueError):
        pm.decompose((4, 4, 1), (0, 1, 1))
    with pytest.raises(ValueError):
        pm.decompose((4, 4), (1, 1, 1))


@pytest.mark.parametrize("dims,grid", [((12, 10, 9), (2, 2, 2)), ((9, 4, 5), (4, 2, 2)), ((30, 20, 1), (3, 2, 1)),
                                       ((16, 16, 24), (1, 1, 4)), ((24, 24, 24), (3, 3, 3))])
def test_shared_bands_equal_replication_multiplicity(dims, grid):
    """block_domain's shared bands mark exactly the vertices held by more than
    one extended block (_replicated_mask_zyx, parallel.py:228-234)."""
    d = pm.decompose(dims, grid)
    nx, ny, nz = d.dims
    mult = np.zeros((nz, ny, nx), dtype=np.int32)
    for b in d.blocks:
        mult[b.ext_slices_zyx()] += 1
    for b in d.blocks:
        spec = pm.block_domain(b, d.dims)
        ex, ey, ez = spec.dims
        z, y, x = np.meshgrid(np.arange(ez), np.arange(ey), np.arange(ex), indexing="ij")
        band = ((x < spec.shared_lo[0]) | (x >= ex - spec.shared_hi[0]) | (y < spec.shared_lo[1])
                | (y >= ey - spec.shared_hi[1]) | (z < spec.shared_lo[2]) | (z >= ez - spec.shared_hi[2]))
        assert np.array_equal(band, mult[b.ext_slices_zyx()] > 1), b.index
        assert spec.core_hi[0] - spec.core_lo[0] == b.core_stop[0] - b.core_start[0]


def test_edit_set_rules():
    e = pm.EditSet([1, 4, 9], [0.1, 0.2, 0.3], 10)
    assert e.count == 3 and e.ratio == 0.3
    with pytest.raises(ValueError):
        pm.EditSet([4, 1], [0.0, 0.0], 10)
    with pytest.raises(ValueError):
        pm.EditSet([10], [0.0], 10)
    f = pm.ScalarField((5, 2), np.zeros(10))
    g = e.apply_to(f)
    assert pm.EditSet.diff(f, g).ids.tolist() == [1, 4, 9]


def test_apply_edit_rule():
    assert pm.apply_edit(0.1, -0.5, 0.0) == 0.0
    assert pm.apply_edit(0.2, 0.9, 0.0) == 0.2
    assert pm.apply_edit(0.4, 0.25, -10.0) == 0.25


def test_host_field_cache_reuses_only_unreferenced_arrays():
    """HostFieldCache (the drop-in's recycled output arrays): an array is
    reused only when no array, view or memoryview of it is alive, and at most
    max_idle spare arrays are kept."""
    import numpy as np
    from paper_2601_01787_b200.engine import HostFieldCache
    c = HostFieldCache(max_idle=2)
    c.enabled = True
    a = c.take(16)
    v = a[3:9]
    m = memoryview(a)
    del a
    b = c.take(16)
    assert b is not v.base                   # the view still holds the first array
    del v
    assert c.take(16) is not b and len(c.arrays) == 3   # the memoryview still holds it
    m.release()
    del m
    first = c.arrays[0]
    del first
    again = c.take(16)
    assert again is c.arrays[-1]
    arrs = [c.take(8) for _ in range(5)]
    del arrs
    keep = c.take(32)
    idle = sum(1 for i in range(len(c.arrays)) if c._idle(i))
    assert idle <= 2
    c.clear()
    assert all(not c._idle(i) for i in range(len(c.arrays)))
    assert keep.size == 32
    assert isinstance(np.asarray(keep), np.ndarray)
