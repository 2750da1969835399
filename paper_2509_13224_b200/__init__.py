"""B200-native TT-IGA hot path (arXiv 2509.13224), mirroring the reference ``ttiga`` API.

Every numerical step (basis/geometry evaluation, TT-cross fiber sampling,
quadrature contraction, TT arithmetic and rounding, AMEn) runs on sm_100a
kernels in ``libttiga_b200.so`` (C ABI: ``include/ttiga_b200.h``); host Python
only orchestrates. There is no CPU fallback: calls raise ``NativeUnavailable``
without the library or a CUDA device.
"""

from ._lib import NativeError, NativeUnavailable, load_library

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing the package must not need a GPU (CPU-side tests load the library only)
    if name in ("SolveConfig", "SolutionReport", "solve_poisson"):
        from . import driver
        return getattr(driver, name)
    raise AttributeError(name)


__all__ = ["SolveConfig", "SolutionReport", "solve_poisson", "NativeError", "NativeUnavailable", "load_library",
           "__version__"]
