"""Case configuration dataclasses (reference: config.py:23-76).

Only the in-memory configuration the coupled loop consumes is restated;
the INI reader/writer of the reference is host I/O outside the hot path
(SURVEY.md §2 row 7).  Defaults are the reference's.
"""

from dataclasses import dataclass, field

from .errors import ConfigError

__all__ = ["ConfigError", "BoundarySpec", "SampleLine", "CaseConfig", "validate_config"]


@dataclass
class BoundarySpec:
    """Per-patch textual conditions: u and p tagged tuples (config.py:23-32)."""

    u: tuple
    p: tuple


@dataclass
class SampleLine:
    name: str
    p0: tuple
    p1: tuple
    n: int


@dataclass
class CaseConfig:
    nu: float = 1e-6
    rho: float = 1000.0
    convection: str = "upwind"
    nonorth_correction: bool = True
    limiter: float = 1.0
    cg_tol: float = 1e-10
    bicgstab_tol: float = 1e-8
    max_iters: int = 2000
    algorithm: str = "simple"
    alpha_u: float = 0.7
    alpha_p: float = 0.3
    n_correctors: int = 2
    n_nonorth_correctors: int = 0
    dt: float = 1e-3
    end_time: float = 1.0
    outer_tol: float = 1e-5
    max_outer: int = 2000
    pressure_ref_cell: int = 0
    pressure_ref_value: float = 0.0
    write_interval: int = 0
    samples: list = field(default_factory=list)
    boundary: dict = field(default_factory=dict)


POSITIVE_KEYS = ("nu", "rho", "cg_tol", "bicgstab_tol", "max_iters", "dt", "end_time",
                 "outer_tol")


def validate_config(cfg):
    """Value checks of config.py:140-156."""
    for key in POSITIVE_KEYS:
        if getattr(cfg, key) <= 0:
            raise ConfigError(f"{key} must be positive")
    if cfg.convection not in ("upwind", "linear"):
        raise ConfigError(f"convection must be upwind or linear, got {cfg.convection!r}")
    if cfg.algorithm not in ("simple", "piso"):
        raise ConfigError(f"algorithm must be simple or piso, got {cfg.algorithm!r}")
    if not 0.0 < cfg.alpha_u <= 1.0 or not 0.0 < cfg.alpha_p <= 1.0:
        raise ConfigError("relaxation factors must lie in (0, 1]")
    if cfg.n_correctors < 1:
        raise ConfigError("n_correctors must be at least 1")
    if cfg.n_nonorth_correctors < 0 or cfg.write_interval < 0 or cfg.max_outer < 0:
        raise ConfigError("counts must be non-negative")
    if not 0.0 <= cfg.limiter <= 1.0:
        raise ConfigError("limiter must lie in [0, 1]")
