"""The 2.5-D blocked 27-point kernel (k_stencil27, hs_stencil.cu) in every
mode on an odd shape: several i0 runs (n0 > 16, plane hand-off between runs)
and partial x/y tiles, against the oracle (1e-13), and bitwise against the
flat kernel (HS_STENCIL27_FLAT=1 in a subprocess: the switch is read once
per process)."""

import itertools
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, crand, rel

pytestmark = pytest.mark.gpu

SHAPE = (37, 19, 45)
OMEGA = 0.6


def _problem():
    rng = np.random.default_rng(2727)
    offs = list(itertools.product((-1, 0, 1), repeat=3))
    coeffs = {o: crand(rng, SHAPE) * (0.1 if o != (0, 0, 0) else 1.0) for o in offs}
    coeffs[(0, 0, 0)] = coeffs[(0, 0, 0)] + 8.0
    return offs, coeffs, crand(rng, SHAPE), crand(rng, SHAPE)


def _device_outputs():
    """every mode's output through the C ABI (flat arrays, one dict)"""
    import torch
    from paper_1412_0464_b200.device import DeviceStencil, to_device
    offs, coeffs, x, f = _problem()
    op = DeviceStencil(SHAPE, offs, np.stack([coeffs[o].ravel() for o in offs]))
    out = {"apply": op.apply(x).ravel(), "residual": op.residual(f, x).cpu().numpy()}
    xt, _ = to_device(x, op.n)
    ft, _ = to_device(f, op.n)
    for steps in (1, 2, 3):
        u = xt.clone()
        op.jacobi(u, ft, OMEGA, steps)
        out[f"jacobi{steps}"] = u.cpu().numpy()
        z = torch.zeros_like(xt)
        op.jacobi(z, ft, OMEGA, steps, u_is_zero=True)
        out[f"jacobi0_{steps}"] = z.cpu().numpy()
    return out


def test_stencil27_modes_vs_oracle():
    from oracle import tgsp_oracle as orc
    offs, coeffs, x, f = _problem()
    op = orc.Op.from_dict(coeffs)
    got = _device_outputs()
    assert rel(got["apply"], op.apply(x)) < 1e-13
    assert rel(got["residual"], f - op.apply(x)) < 1e-13
    for steps in (1, 2, 3):
        assert rel(got[f"jacobi{steps}"], orc.jacobi(op, x, f, OMEGA, steps)) < 1e-13, steps
        assert rel(got[f"jacobi0_{steps}"],
                   orc.jacobi(op, np.zeros(SHAPE, complex), f, OMEGA, steps)) < 1e-13, steps


def test_stencil27_blocked_bitwise_equals_flat(tmp_path):
    blocked = _device_outputs()
    dump = tmp_path / "flat.npz"
    code = ("import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r); "
            "import test_stencil27 as t; np.savez(%r, **t._device_outputs())"
            % (str(ROOT), str(ROOT / "tests"), str(dump)))
    env = dict(os.environ, HS_STENCIL27_FLAT="1")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=str(ROOT), timeout=300)
    with np.load(dump) as z:
        for k, v in blocked.items():
            assert np.array_equal(v, z[k]), k
