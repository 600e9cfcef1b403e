"""pytest plugin for the drop-in conformance run (tools/ref_conformance.py):
makes `import fvflow.<module>` resolve to this package's module of the same
name, so the reference's own test files run unmodified against libfvb.  This
is exactly the switch INTEGRATION.md shows a maintainer adding to
fvflow/__init__.py.  Loaded with `pytest -p fvflow_alias` before any test
module (and the reference's conftest.py) is imported."""
import importlib
import sys
import types

import paper_1207_1571_b200 as _pkg

MODULES = ("mesh", "sparse", "linsolve", "fvm", "coupling", "config", "cases", "fileio", "report")

_alias = types.ModuleType("fvflow")
_alias.__path__ = []  # a package: `fvflow.x` submodules come from sys.modules
_alias.__file__ = _pkg.__file__
sys.modules["fvflow"] = _alias
for _m in MODULES:
    _mod = importlib.import_module(f"paper_1207_1571_b200.{_m}")
    sys.modules[f"fvflow.{_m}"] = _mod
    setattr(_alias, _m, _mod)
