"""``rbfdeform`` -> ``paper_2004_04817_b200`` alias for the drop-in conformance run.

Staged as ``build/conformance/rbfdeform/__init__.py`` by tools/conformance/stage.py.
The reference's own unit tests (``/root/reference/pkg/tests``; SURVEY.md §4, §7.2
step 6) import ``rbfdeform`` and its submodules; this package answers every import
on the hot path with this repository's modules:

    rbfdeform, rbfdeform.core, .selection, .errors, .estimator, .metrics, .meshio,
    .cli, .deformers
        -> paper_2004_04817_b200 (and its submodules of the same names)

Reference code outside the hot path is used only as test fixtures (the desk-wing
mesh generator the reference's conftest builds its cases with, and the
surface-cell quality metrics test_metrics.py imports): ``rbfdeform.synthetic`` is
the reference's own file, and ``cell_quality`` / ``quality_report`` come from the
reference's metrics.py, both copied next to this shim at staging time (not
committed) and bound to this repository's ``errors`` / ``meshio`` / ``core``. The
CLI's ``make-wing`` and quality sections are registered with them
(``cli.MAKE_WING`` / ``cli.QUALITY_REPORT``).
"""

import sys

import paper_2004_04817_b200 as _P
from paper_2004_04817_b200 import *  # noqa: F401,F403
from paper_2004_04817_b200 import cli, core, deformers, errors, estimator, meshio, metrics, selection  # noqa: F401

for _name in ("cli", "core", "deformers", "errors", "estimator", "meshio", "metrics", "selection"):
    sys.modules[f"{__name__}.{_name}"] = getattr(_P, _name)

from . import synthetic  # noqa: E402  (reference test fixture)


def _with_cell_quality(ours):
    """metrics: this repository's boundary metrics (the §8(f) row) plus the
    reference's own surface-cell quality functions (``cell_quality``,
    ``quality_report``: mesh analytics outside the hot path),
    taken from the staged reference metrics.py with its package imports bound
    to this repository's modules."""
    import contextlib
    import types
    from pathlib import Path

    src = (Path(__file__).with_name("_ref_metrics.py")).read_text()
    body = "\n".join(ln for ln in src.splitlines() if not ln.startswith("from ."))
    ns = dict(vars(ours))
    ns.update(SupportSet=core.SupportSet, assemble_phi=core.assemble_phi,
              _single_threaded_blas=contextlib.nullcontext, DegenerateCellError=errors.DegenerateCellError,
              EmptySupportSetError=errors.EmptySupportSetError, __name__="rbfdeform._ref_metrics")
    exec(compile(body, "rbfdeform/_ref_metrics.py", "exec"), ns)
    mod = types.ModuleType(f"{__name__}.metrics", ours.__doc__)
    mod.__dict__.update(vars(ours))
    for name in ("cell_quality", "quality_report", "QualityReport", "QUALITY_BIN_WIDTH"):
        if name in ns:
            setattr(mod, name, ns[name])
    return mod


metrics = _with_cell_quality(_P.metrics)
sys.modules[f"{__name__}.metrics"] = metrics
cell_quality, quality_report = metrics.cell_quality, metrics.quality_report
QualityReport = metrics.QualityReport
from paper_2004_04817_b200.deformers import (  # noqa: E402,F401
    BendTwistParams, SpanSineParams, bend_twist, prescribe, span_sine)
from .synthetic import swept_wing_case, swept_wing_surface  # noqa: E402,F401

cli.QUALITY_REPORT = quality_report
cli.MAKE_WING = swept_wing_case

BACKEND = "paper_2004_04817_b200 (sm_100a)"
