"""The five BASELINE.json configurations as parity cases,
at sizes the numpy oracle (pinned to the reference's golden vectors)
finishes in seconds.  Fields are compared normwise (north_star: U, p, phi
within 1e-8 relative L2), iteration counts per solve (CG +-1, BiCGStab +-2,
the round-off-driven uz solves of one-cell-thick meshes excluded as
SURVEY.md §7 prescribes), and continuity (test_coupling.py:50 bound).
"""

import numpy as np
import pytest

from golden_io import rel
from oracle import fvoracle as O
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import (
    CouplingConfig, continuity_error, init_state, piso_time_step, simple_outer_iteration)
from paper_1207_1571_b200.team import DecomposedRun

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-8


def _check_logs(mine, ref, two_d=False):
    assert [(r[0], r[1], r[2]) for r in mine] == [(r[0], r[1], r[2]) for r in ref]
    for a, b in zip(mine, ref):
        if two_d and a[1] == "uz":
            continue
        assert abs(a[3] - b[3]) <= (1 if a[0] == "cg" else 2), (a, b)


def _fields(st):
    return st.u.values, st.p.values, st.flux


def _oracle_fields(run):
    return run.u.values, run.p.values, run.flux


def test_c1_cavity2d_20x20_100_steps():
    """C1: icoFoam cavity 20x20x1, Re 10, dt 0.005, end 0.5 s (100 PISO steps)."""
    case = cases.box_mesh(20, 20, 1, 0.1, 0.1, 0.01,
                          [("movingWall", "wall", ["y+"]),
                           ("fixedWalls", "wall", ["x-", "x+", "y-"]),
                           ("frontAndBack", "empty", ["z-", "z+"])])
    from paper_1207_1571_b200.cases import Case
    from paper_1207_1571_b200.config import BoundarySpec, CaseConfig

    cc = CaseConfig()
    cc.nu, cc.algorithm, cc.dt, cc.end_time = 0.01, "piso", 0.005, 0.5
    cc.boundary = {
        "movingWall": BoundarySpec(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
        "fixedWalls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
        "frontAndBack": BoundarySpec(u=("empty",), p=("empty",)),
    }
    c = Case("cavity2d", case, cc)
    cfg = CouplingConfig.from_case_config(cc)
    st = init_state(c, cfg)
    run = O.Run(c.mesh, cc)
    for _ in range(100):
        piso_time_step(st, cfg)
        run.piso_step()
    for a, b in zip(_fields(st), _oracle_fields(run)):
        assert rel(a, b) < FIELD_TOL
    _check_logs(st.residual_log, run.log, two_d=True)
    assert continuity_error(st) <= 1e-8 * np.abs(st.flux).max()


def test_c2_cavity32_piso():
    """C2 shape (gen_cavity PISO, Co = 1) at 32^3, reference defaults."""
    n = 32
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    run = O.Run(case.mesh, case.config)
    for _ in range(2):
        piso_time_step(st, cfg)
        run.piso_step()
        for a, b in zip(_fields(st), _oracle_fields(run)):
            assert rel(a, b) < FIELD_TOL
    _check_logs(st.residual_log, run.log)


def test_c3_backward_step_simple():
    """C3: backward-facing step (Re_h 200) steady SIMPLE, nh = 8."""
    case = cases.gen_backward_step(8)
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    run = O.Run(case.mesh, case.config)
    for _ in range(25):
        simple_outer_iteration(st, cfg)
        run.simple_sweep()
    for a, b in zip(_fields(st), _oracle_fields(run)):
        assert rel(a, b) < FIELD_TOL
    _check_logs(st.residual_log, run.log, two_d=True)
    assert continuity_error(st) <= 1e-8 * np.abs(st.flux).max()


def test_c4_perturbed_renumbered_cavity():
    """C4 recipe: perturbed + renumbered hex cavity, non-orthogonal
    correction with one extra corrector, at 16^3."""
    case = cases.perturbed_cavity(16)
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    run = O.Run(case.mesh, case.config)
    for _ in range(2):
        piso_time_step(st, cfg)
        run.piso_step()
        for a, b in zip(_fields(st), _oracle_fields(run)):
            assert rel(a, b) < FIELD_TOL
    _check_logs(st.residual_log, run.log)


def test_c4_perturbed_renumbered_cavity_rcm_order_vs_oracle():
    """C4 recipe at 41^3 (68,921 cells): large enough that CG runs in the
    solver's internal RCM order (no stencil codes on a renumbered mesh).
    One step against the oracle at tight solver tolerances (the dot-product
    grouping differs from the oracle's either way)."""
    import ctypes as C
    from paper_1207_1571_b200 import _lib

    case = cases.perturbed_cavity(41)
    case.config.cg_tol, case.config.bicgstab_tol, case.config.max_iters = 1e-13, 1e-11, 20000
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    run = O.Run(case.mesh, case.config)
    piso_time_step(st, cfg)
    run.piso_step()
    rcm = C.c_int64()
    _lib.check(_lib.lib.fvb_pattern_codes(st._ctx.h, None, None, None, C.byref(rcm)))
    assert rcm.value == 2 * cfg.n_correctors + 1  # CG solves + the momentum batch
    for a, b in zip(_fields(st), _oracle_fields(run)):
        assert rel(a, b) < FIELD_TOL
    for a, b in zip(st.residual_log, run.log):
        # at tightened tolerances the counts follow the rounding of the dot
        # products (the same bound as the full-size decomposed test)
        tol = 2 if a[0] == "cg" else max(3, int(0.1 * b[3]))
        assert a[0] == b[0] and abs(a[3] - b[3]) <= tol, (a, b)


@pytest.mark.parametrize("nparts", [2, 4])
def test_c5_decomposed_cavity_vs_oracle(nparts):
    """C5 shape: gen_cavity split into z-slabs, against the oracle."""
    n = 24
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    cfg = CouplingConfig.from_case_config(case.config)
    team = DecomposedRun(case, cfg, nparts)
    run = O.Run(case.mesh, case.config)
    for _ in range(2):
        team.piso_time_step(cfg)
        run.piso_step()
    u, p, flux = team.gather()
    for a, b in zip((u, p, flux), _oracle_fields(run)):
        assert rel(a, b) < FIELD_TOL
    _check_logs(team.residual_log, run.log)
    team.close()
