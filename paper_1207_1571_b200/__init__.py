"""B200-native PISO/SIMPLE finite-volume engine (arXiv 1207.1571).

Drop-in for the hot path of the reference package ``fvflow``: the modules
``mesh``, ``sparse``, ``linsolve``, ``fvm``, ``coupling``, ``config``,
``cases``, ``fileio`` (mesh files) and ``report`` (profiles) expose the
reference's names, dataclasses and exceptions, while all numerical work runs in libfvb.so (hand-written FP64 CUDA for sm_100a,
C ABI in include/fvb.h).  Importing the package loads libfvb.so and fails
loudly if it has not been built; there is no CPU fallback.
"""

from . import _lib  # noqa: F401  (loads libfvb.so or raises ImportError)
from . import cases, config, coupling, fileio, fvm, linsolve, mesh, report, sparse  # noqa: F401

__version__ = "0.1.0"
