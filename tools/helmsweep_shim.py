"""pytest plugin: run the REFERENCE's own test files against this package.

    python -m pytest -p tools.helmsweep_shim baseline/reftests/test_sweepdd.py ...

(see tools/run_reference_tests.sh, which copies the reference's tests into
the git-ignored ``baseline/reftests/``; nothing of the reference is tracked
here).  ``helmsweep`` and its hot-path submodules (mesh, discretize,
sparselin, sweepdd, twogrid, krylov) are aliased to ``paper_1412_0464_b200``,
so every solve, sweep, factorisation and GMRES the tests run goes through
this package's CUDA path.  The reference's analysis module ``oracles.py``
(closed-form 1-D / strip solutions the tests compare against) and its CLI
(``wedge_velocity`` in the tests' conftest) are out of this build's scope
(SURVEY section 2); they are loaded from the reference install
``baseline/_ref`` as submodules of the alias, so their own imports resolve
to this package too.
"""

from __future__ import annotations

import importlib
import importlib.util
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_1412_0464_b200 as pkg  # noqa: E402

sys.modules["helmsweep"] = pkg
for _sub in ("mesh", "discretize", "sparselin", "sweepdd", "twogrid", "krylov"):
    sys.modules[f"helmsweep.{_sub}"] = importlib.import_module(f"paper_1412_0464_b200.{_sub}")

_REF = ROOT / "baseline" / "_ref" / "helmsweep"
for _sub in ("oracles", "cli"):
    _spec = importlib.util.spec_from_file_location(f"helmsweep.{_sub}", _REF / f"{_sub}.py")
    _mod = importlib.util.module_from_spec(_spec)
    _mod.__package__ = "helmsweep"
    sys.modules[f"helmsweep.{_sub}"] = _mod
    _spec.loader.exec_module(_mod)
    setattr(pkg, _sub, _mod)

# names the reference re-exports from oracles.py (its __init__.py)
for _name in ("RobinProblem1D", "StripMode", "dispersion_error", "dtn_closure_factor",
              "phase_speed_error_std_1d", "reflection_coeffs", "solve_1d_analytic",
              "solve_strip_fourier"):
    setattr(pkg, _name, getattr(sys.modules["helmsweep.oracles"], _name))
