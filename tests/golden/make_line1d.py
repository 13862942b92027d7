"""Golden vectors of the 1-D line and of general-matrix factorisations,
computed by running the REFERENCE (build container only):

    python tests/golden/make_line1d.py      # writes tests/golden/line1d.npz

* the robin line (robin_level_1d, reference sweepdd.py:90) for the line
  known-answer cases of test_sweepdd.py:194-210 / test_acceptance.py:52-71:
  partition geometry, the reference's prec_x / prec_ud outputs for a seeded
  right-hand side, and its dense forward/backward transmission matrices;
* factorize() of scipy matrices (sparselin.py:40-68): SuperLU solves of a
  2-D fine operator's CSR, a random banded matrix and the hand-solved
  tridiagonal system.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

REF = os.environ.get("HELMSWEEP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import helmsweep as hs  # noqa: E402  (the reference)
from helmsweep.mesh import PML, AbsorbingLayerSpec  # noqa: E402
from helmsweep.sweepdd import build_partition  # noqa: E402

OUT = Path(__file__).resolve().parent / "line1d.npz"
LINES = [("a", 240, 6, False), ("b", 240, 6, True), ("c", 2000, 16, False), ("d", 400, 8, False)]


def crand(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def main():
    out = {}
    rng = np.random.default_rng(77)
    for key, n, J, tr in LINES:
        h = 1.0 / n
        k = 2 * np.pi * (n / 10.0)
        level = hs.robin_level_1d(k, h, n)
        part = build_partition(level, J=J, tilde_right=tr)
        f = crand(rng, part.shape)
        out[f"{key}_meta"] = np.array([n, J, int(tr)])
        out[f"{key}_k"] = np.array(k)
        out[f"{key}_beta"] = part.beta
        out[f"{key}_beta_tilde"] = part.beta_tilde
        out[f"{key}_lohi"] = np.array([[s.pt_lo, s.pt_hi] for s in part.subs])
        out[f"{key}_f"] = f
        out[f"{key}_ux"] = hs.prec_x(part, f)
        out[f"{key}_uud"] = hs.prec_ud(part, f)
        out[f"{key}_tfwd2"] = hs.extract_transmission(part, 2, "forward").dense()
        out[f"{key}_tbwd1"] = hs.extract_transmission(part, 1, "backward").dense()
        for o, c in level.op.coeffs.items():
            out[f"{key}_op{o[0]:+d}"] = c
    # factorize(scipy matrix)
    mesh = hs.build_mesh(2, 16, 1.0 / 16, AbsorbingLayerSpec(PML, 4, 20.0))
    model = hs.WaveModel.constant(mesh, 2 * np.pi * 16 / 8.0)
    a = hs.to_csr(hs.assemble_fine(mesh, model)).tocsr()
    b = crand(rng, a.shape[0])
    out["fine_indptr"], out["fine_indices"], out["fine_data"] = a.indptr, a.indices, a.data
    out["fine_b"] = b
    out["fine_x"] = hs.factorize(a).solve(b)
    n = 300
    band = sp.diags([crand(rng, n - abs(d)) for d in range(-7, 8)], list(range(-7, 8)),
                    format="csr") + sp.eye(n) * 12.0
    band = band.tocsr()
    bb = crand(rng, (n, 3))
    out["band_indptr"], out["band_indices"], out["band_data"] = band.indptr, band.indices, band.data
    out["band_b"] = bb
    out["band_x"] = hs.solve_factored(hs.factorize(band), bb)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({len(out)} arrays)")


if __name__ == "__main__":
    main()
