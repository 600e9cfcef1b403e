"""BASELINE.json configurations at their full sizes, through size-independent
properties (the oracle needs minutes per step there): discrete continuity of
the corrected flux (test_coupling.py:50 bound), bitwise determinism of a
repeated run, agreement of a decomposed run with the single-domain one, and
the CG iteration counts the reference itself reported for the 128^3 cavity
(1494 + 1510 CG iterations in PISO step 2)."""

import numpy as np
import pytest

from golden_io import rel
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import (
    CouplingConfig, continuity_error, init_state, piso_time_step, simple_outer_iteration)
from paper_1207_1571_b200.team import DecomposedRun

pytestmark = pytest.mark.gpu


def _cavity(n):
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    return case, CouplingConfig.from_case_config(case.config)


def test_c2_cavity128_two_steps():
    case, cfg = _cavity(128)
    st = init_state(case, cfg)
    for _ in range(2):
        piso_time_step(st, cfg)
        assert continuity_error(st) <= 1e-8 * np.abs(st.flux).max()
    cg = [r[3] for r in st.residual_log if r[0] == "cg"]
    # reference step 2: 1494 + 1510; the dot-product order
    # differs from OpenBLAS, so allow the parity rule's +-1 plus the
    # measured CPU-vs-CPU spread at this size
    assert abs(cg[2] - 1494) <= 3 and abs(cg[3] - 1510) <= 3, cg
    u1, p1, f1 = st.u.values.copy(), st.p.values.copy(), st.flux.copy()
    st2 = init_state(case, cfg)
    for _ in range(2):
        piso_time_step(st2, cfg)
    assert np.array_equal(st2.u.values, u1) and np.array_equal(st2.p.values, p1)
    assert np.array_equal(st2.flux, f1)
    assert st2.residual_log == st.residual_log


def test_c2_cavity128_decomposed_matches_single():
    # fields judged at tightened tolerances (SURVEY.md §7 hard part 1: at
    # default tolerances the rounding floor at 128^3 is ~1e-7 between any two
    # dot-product orders, CPU vs CPU included)
    case, cfg = _cavity(128)
    case.config.cg_tol, case.config.bicgstab_tol, case.config.max_iters = 1e-13, 1e-10, 20000
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    piso_time_step(st, cfg)
    run = DecomposedRun(case, cfg, 2)
    run.piso_time_step(cfg)
    u, p, flux = run.gather()
    assert rel(u, st.u.values) < 1e-8 and rel(p, st.p.values) < 1e-8
    assert rel(flux, st.flux) < 1e-8
    for a, b in zip(run.residual_log, st.residual_log):
        # at tightened tolerances BiCGStab counts follow the rounding of the
        # dot products (+-3 between two CPU orderings at 64^3);
        # counts are judged at default tolerances elsewhere
        tol = 2 if a[0] == "cg" else max(3, int(0.1 * b[3]))
        assert abs(a[3] - b[3]) <= tol, (a, b)
    assert run.continuity_error() <= 1e-8 * np.abs(flux).max()
    run.close()


def test_c4_perturbed_cavity_2m_cells():
    case = cases.perturbed_cavity(126)
    assert case.mesh.n_cells == 2000376
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    piso_time_step(st, cfg)
    assert continuity_error(st) <= 1e-8 * np.abs(st.flux).max()
    assert all(r[5] <= cfg.pressure.tolerance for r in st.residual_log if r[0] == "cg")
    # n_nonorth_correctors = 1: two CG solves per corrector
    assert sum(1 for r in st.residual_log if r[0] == "cg") == 2 * cfg.n_correctors


def test_c3_backward_step_nh32_simple():
    case = cases.gen_backward_step(32)
    cfg = CouplingConfig.from_case_config(case.config)
    cfg.pressure.max_iters = cfg.momentum.max_iters = 20000
    st = init_state(case, cfg)
    res = [simple_outer_iteration(st, cfg) for _ in range(10)]
    assert continuity_error(st) <= 1e-8 * np.abs(st.flux).max()
    assert res[-1][0] < res[0][0] or res[-1][1] < 1.0
