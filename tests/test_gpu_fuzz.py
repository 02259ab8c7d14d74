"""Seeded random cases against the CPU oracle: field styles the reference's
own helpers use (tests/helpers.py random_field: uniform, plateau -- few
distinct levels, so index tie-breaking carries the order -- and coarse),
Perlin fields, quantized or bounded-noise decompressed fields, relative
bounds from 1e-1 to 1e-4, odd / 2-D / thin shapes (the non-TMA fallbacks),
f32-exact and f64 originals, extrema-only.  Every case runs through the
device API and, where the reference has it, the drop-in (host staging), and
must equal the oracle bit for bit: corrected field, edits per iteration,
max per-vertex edits."""

import numpy as np
import pytest
import torch

import paper_2601_01787_b200 as pm
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

SHAPES = [(37, 23, 11), (64, 48, 40), (96, 7, 33), (50, 50, 1), (128, 96, 1), (5, 300, 3), (80, 72, 66),
          (33, 64, 64), (2, 40, 40), (129, 31, 17)]
STYLES = ["perlin", "uniform", "plateau", "coarse"]
RELS = [1e-1, 1e-2, 1e-3, 1e-4]


def _case(seed):
    rng = np.random.default_rng(seed)
    dims = SHAPES[seed % len(SHAPES)]
    style = STYLES[(seed // 2) % len(STYLES)]
    rel = RELS[rng.integers(len(RELS))]
    n = dims[0] * dims[1] * dims[2]
    if style == "perlin":
        f = orc.perlin(dims, int(rng.integers(1 << 30)))
    elif style == "uniform":
        f = rng.standard_normal(n)
    elif style == "plateau":
        f = rng.integers(0, 4, size=n).astype(np.float64)
    else:
        f = np.round(rng.standard_normal(n), 1)
    if rng.random() < 0.5:
        f = f.astype(np.float32).astype(np.float64)   # an f32 file, promoted
    xi = orc.relative_to_absolute(f, rel)
    noise = rng.random() < 0.4 or style == "plateau"   # (quantizing integer levels is exact: no edits)
    fh = orc.bounded_noise(f, dims, xi, int(rng.integers(1 << 30))) if noise else orc.quantize(f, xi)
    extrema = rng.random() < 0.25
    return dims, f, fh, xi, extrema, f"{style} {dims} rel={rel} {'noise' if noise else 'quant'}"


@pytest.mark.parametrize("seed", range(32))
def test_random_case_matches_oracle(seed):
    dims, f, fh, xi, extrema, label = _case(seed)
    ref = orc.run_correction(dims, f, fh, xi, extrema_only=extrema, check_segmentation=False)
    cfg = pm.CorrectionConfig(xi_abs=xi)
    if ref.status != orc.ORC_OK:
        pytest.skip(f"oracle status {ref.status} ({label})")
    fd = torch.from_numpy(f).cuda()
    fhd = torch.from_numpy(fh).cuda()
    out = pm.run_correction_device(fd, fhd, dims, cfg, extrema_only=extrema)
    assert out.edits_per_iteration == ref.edits_per_iteration, label
    assert out.max_vertex_edits == ref.max_vertex_edits, label
    assert np.array_equal(out.corrected.cpu().numpy(), ref.corrected), label
    ids = np.flatnonzero(ref.corrected != fh)
    assert np.array_equal(out.edit_ids.cpu().numpy(), ids), label
    if extrema:
        return   # (the reference API has no extrema-only switch)
    res = pm.run_correction(pm.ScalarField(dims, f), pm.ScalarField(dims, fh), cfg)
    assert res.edits_per_iteration == ref.edits_per_iteration, label
    assert np.array_equal(res.corrected.values, ref.corrected), label
    assert np.array_equal(res.edits.ids, ids), label
    assert np.array_equal(res.edits.values, ref.corrected[ids]), label
