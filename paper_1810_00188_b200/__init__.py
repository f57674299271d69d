"""B200-native ERMC solver — drop-in for the reference's `ermc` Python package.

`import paper_1810_00188_b200 as ermc` exposes the same names as the
reference's `_ermc` module on the solve path (proj/python/bindings.cpp):
CartesianGrid, TemperatureField, BoundarySpec, Wall, AxisKind, NarrowBand,
QuadratureSet, LineSpectrum, SpectralModel, SolveConfig, SolutionField, the
table builders, KTAB1/TFLD1/QRF1 I/O and `solve` — which runs every cell and
ray on the GPU through the C-ABI in include/ermc_b200.h.

The compiled extension is required: importing without it raises ImportError
(there is no CPU fallback). Run `python paper_1810_00188_b200/build.py` or
`__graft_entry__.build()` first.
"""
from __future__ import annotations

from pathlib import Path

_HERE = Path(__file__).resolve().parent

try:
    from . import _ermc  # noqa: F401
    from ._ermc import *  # noqa: F401,F403
    from ._ermc import __doc__ as _core_doc  # noqa: F401
except ModuleNotFoundError as exc:  # pragma: no cover - only when unbuilt
    raise ImportError(
        "paper_1810_00188_b200: the compiled extension (_ermc / libermc_b200.so) "
        "is missing; build it with `python paper_1810_00188_b200/build.py`. "
        "There is no CPU fallback."
    ) from exc

__version__ = "0.1.0"
LIB_PATH = _HERE / "libermc_b200.so"
