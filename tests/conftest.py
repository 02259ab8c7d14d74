import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large-size parity (minutes)")


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN / "golden.json").read_text())
    arrays = dict(np.load(GOLDEN / "golden.npz"))
    return meta, arrays


def golden_inputs(run, arrays):
    """Rebuild (f, fhat, dims) of a golden run from its recipe with the oracle's
    generators (pinned to the reference by the Perlin/quantize hashes)."""
    from oracle import oracle as orc
    rec = run["recipe"]
    dims = tuple(run["dims"])
    if rec["kind"] == "stored":
        return arrays[rec["key"] + "_f"], arrays[rec["key"] + "_fhat"], dims
    f = orc.perlin(dims, rec["seed"])
    if rec.get("f32"):
        f = f.astype(np.float32).astype(np.float64)
    if rec["kind"] == "perlin_quantize":
        fh = orc.quantize(f, run["xi"])
    else:
        fh = orc.bounded_noise(f, dims, run["xi"], rec["noise_seed"])
    return f, fh, dims
