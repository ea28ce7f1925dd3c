"""B200-native XCT reconstruction hot path (Petascale XCT, arXiv 2009.07226).

Drop-in for the reference package's operator API (``xct.geometry``,
``xct.pipeline``, ``xct.solver``): Siddon system-matrix construction,
staged FP32/FP16-storage SpMM projection and back projection, and CGLS --
all on sm_100a kernels in ``libxct_b200.so`` behind a C ABI
(``include/xct_b200.h``).  There is no CPU fallback.
"""

from . import (cli, dataio, engine, geometry, hilbert, matrixstore, parallel,  # noqa: F401
               pipeline, solver)

__version__ = "0.1.0"
__all__ = ["cli", "dataio", "engine", "geometry", "hilbert", "matrixstore", "parallel",
           "pipeline", "solver"]
