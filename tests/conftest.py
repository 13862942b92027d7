import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

CASES = ["pml2d", "wedge2d", "sponge2d", "fe9_2d", "pml3d", "pml3d_s", "nx2d"]
SOLVED = ["pml2d", "wedge2d", "sponge2d", "pml3d_s", "nx2d"]
# NX groupings stored in nx2d.npz: make_nx_cells(8, n) for n = 1..4 and a hand grouping
NX_KEYS = ["nx1", "nx2", "nx3", "nx4", "nxc"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhsweep.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have = torch.cuda.is_available()
    except Exception:
        have = False
    if have:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_case(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def c1_anchors():
    return json.loads((GOLDEN / "c1_anchors.json").read_text())


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def crand(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
