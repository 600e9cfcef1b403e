"""Exception classes of the reference API (one per reference module).

mesh.MeshError (mesh.py:27), sparse.SparseError (sparse.py:25),
linsolve.SolverError (linsolve.py:24), fvm.FvmError (fvm.py:30),
coupling.CouplingError (coupling.py:64), config.ConfigError (config.py:19),
fileio.MeshFileError (fileio.py:27), report.ProfileError (report.py:23).
"""


class MeshError(Exception):
    """Topological or geometric defect in a mesh."""


class SparseError(Exception):
    pass


class SolverError(Exception):
    pass


class FvmError(Exception):
    pass


class CouplingError(Exception):
    pass


class ConfigError(Exception):
    pass


class MeshFileError(Exception):
    """Malformed mesh file; message carries the line number."""


class ProfileError(Exception):
    pass


class DeviceError(RuntimeError):
    """CUDA/driver failure inside libfvb (no CPU fallback exists)."""
