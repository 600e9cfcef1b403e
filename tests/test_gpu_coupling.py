"""The device PISO step and SIMPLE sweep against the reference's coupled
loop (§8(c) items 4-5): golden runs of the real reference, the oracle at
larger sizes, loop invariants (continuity, determinism, fixed points)."""

import numpy as np
import pytest

from golden_io import CASES, golden_case, rel
from oracle import fvoracle as O
from paper_1207_1571_b200 import cases, coupling
from paper_1207_1571_b200.coupling import (
    CouplingConfig,
    continuity_error,
    init_state,
    piso_time_step,
    run_case,
    simple_outer_iteration,
)

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-8  # north_star: converged per-step U, p, phi within 1e-8 relative L2


def step(state, cfg):
    if cfg.algorithm == "piso":
        return piso_time_step(state, cfg)
    return simple_outer_iteration(state, cfg)


@pytest.mark.parametrize("name", CASES)
def test_free_running_steps_match_reference(name):
    case, g = golden_case(name)
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    assert rel(st.flux, g["init_flux"]) <= 1e-15
    assert np.array_equal(st.u.boundary, g["init_ub"])
    for s in range(int(g["steps"])):
        nlog = len(st.residual_log)
        r = step(st, cfg)
        assert np.allclose(r, g[f"s{s}_ret"], rtol=1e-5, atol=1e-12), (s, r, g[f"s{s}_ret"])
        assert rel(st.u.values, g[f"s{s}_u"]) < FIELD_TOL, s
        assert rel(st.p.values, g[f"s{s}_p"]) < FIELD_TOL, s
        assert rel(st.flux, g[f"s{s}_flux"]) < FIELD_TOL, s
        rows = st.residual_log[nlog:]
        names = [f"{a}:{b}" for a, b, *_ in rows]
        assert names == [str(x) for x in g[f"s{s}_log_names"]]
        ref = g[f"s{s}_log"]
        two_d = case.mesh.n_cells in (48, 260, 400)
        for (solver, fld, outer, it, r0, r1), rr in zip(rows, ref):
            assert outer == rr[0]
            if two_d and fld == "uz":
                continue  # round-off-driven solve on one-cell-thick meshes
            assert abs(it - rr[1]) <= (1 if solver == "cg" else 2), (s, solver, fld, it, rr[1])
            assert abs(r0 - rr[2]) <= 1e-9 * max(abs(rr[2]), 1e-300) + 1e-14
        assert continuity_error(st) <= max(1e-8 * np.abs(st.flux).max(), 1e-16)


def test_deterministic_bitwise():
    a = run_case(_short(cases.gen_cavity(6)))
    b = run_case(_short(cases.gen_cavity(6)))
    assert (a.u.values == b.u.values).all() and (a.p.values == b.p.values).all()
    assert (a.flux == b.flux).all() and a.cum_iters == b.cum_iters


def _short(case):
    case.config.max_outer = 5
    return case


def test_zero_state_fixed_point():
    case = cases.gen_cavity(4)
    from paper_1207_1571_b200.config import BoundarySpec

    case.config.boundary["lid"] = BoundarySpec(u=("no_slip",), p=("zero_gradient",))
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    ru, rp = simple_outer_iteration(st, cfg)
    assert np.abs(st.u.values).max() == 0.0 and np.abs(st.p.values).max() == 0.0
    assert np.abs(st.flux).max() == 0.0 and ru == 0.0 and rp == 0.0


def test_simple_cavity8_converges_like_reference():
    st = run_case(cases.gen_cavity(8))
    assert st.converged and st.outer < 2000
    assert continuity_error(st) < 1e-8 * np.abs(st.flux).max()
    top = st.geom.cell_centroid[:, 1] > 0.1 * (7.5 / 8)
    assert st.u.values[top, 0].mean() > 0.1
    cg_sum = sum(r[3] for r in st.residual_log if r[0] == "cg")
    assert st.cum_iters["cg"] == cg_sum


def test_host_assignment_is_uploaded():
    case = cases.gen_channel(8, 4)
    case.config.dt = 0.01
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    c = st.geom.cell_centroid
    st.u.values = 2.0 * np.stack([c[:, 1], -c[:, 0], np.zeros(len(c))], axis=1)
    st.flux = coupling._plain_flux(st.u, st.geom)
    run = O.Run(case.mesh, case.config)
    run.u.values = 2.0 * np.stack([c[:, 1], -c[:, 0], np.zeros(len(c))], axis=1)
    run.flux = run._plain_flux()
    assert rel(st.flux, run.flux) < 1e-15
    piso_time_step(st, cfg)
    run.piso_step()
    assert rel(st.u.values, run.u.values) < 1e-8


@pytest.mark.slow
@pytest.mark.parametrize("n,steps", [(24, 2)])
def test_piso_cavity_vs_oracle_tight(n, steps):
    """Tight solver tolerances (SURVEY §7 protocol): fields within 1e-8."""
    case = cases.gen_cavity(n)
    cc = case.config
    cc.algorithm, cc.dt, cc.cg_tol, cc.bicgstab_tol, cc.max_iters = "piso", 0.1 / n, 1e-13, 1e-10, 20000
    cfg = CouplingConfig.from_case_config(cc)
    st = init_state(case, cfg)
    run = O.Run(case.mesh, cc)
    for _ in range(steps):
        piso_time_step(st, cfg)
        run.piso_step()
        assert rel(st.u.values, run.u.values) < FIELD_TOL
        assert rel(st.p.values, run.p.values) < FIELD_TOL
        assert rel(st.flux, run.flux) < FIELD_TOL
    mine = [r[3] for r in st.residual_log if r[0] == "cg"]
    ref = [r[3] for r in run.log if r[0] == "cg"]
    assert max(abs(a - b) for a, b in zip(mine, ref)) <= 2


@pytest.mark.parametrize("maker,algo", [(lambda: cases.gen_cavity(12), "piso"),
                                        (lambda: cases.gen_backward_step(4), "simple")])
def test_one_step_reseeded_from_oracle_state(maker, algo):
    """the oracle runs a few steps, its state (u, p,
    flux, outer, t) is loaded into the device state, and one more step on
    each side must agree (fields 1e-8, iteration counts CG +-1 / BiCGStab +-2)."""
    case = maker()
    cc = case.config
    cc.algorithm = algo
    if algo == "piso":
        cc.dt = 0.1 / 12
    run = O.Run(case.mesh, cc)
    for _ in range(4):
        run.piso_step() if algo == "piso" else run.simple_sweep()
    cfg = CouplingConfig.from_case_config(cc)
    st = init_state(case, cfg)
    st.u.values = run.u.values.copy()
    st.p.values = run.p.values.copy()
    st.u.boundary = run.u.boundary.copy()
    st.p.boundary = run.p.boundary.copy()
    st.flux = run.flux.copy()
    st.outer, st.t = run.outer, run.t
    nlog = len(run.log)
    if algo == "piso":
        piso_time_step(st, cfg)
        run.piso_step()
    else:
        st._res_scale = dict(run._scale)
        simple_outer_iteration(st, cfg)
        run.simple_sweep()
    for a, b in ((st.u.values, run.u.values), (st.p.values, run.p.values), (st.flux, run.flux)):
        assert rel(a, b) < FIELD_TOL
    for a, b in zip(st.residual_log, run.log[nlog:]):
        assert a[:3] == b[:3]
        if a[1] == "uz" and case.mesh.n_cells in (1040,):
            continue  # one-cell-thick mesh: round-off-driven uz solve
        assert abs(a[3] - b[3]) <= (1 if a[0] == "cg" else 2), (a, b)


def _cavity_2d():
    """C1 (BASELINE configs[0]): 2D lid-driven cavity 20x20x1, PISO dt 0.005."""
    from paper_1207_1571_b200.cases import Case
    from paper_1207_1571_b200.config import BoundarySpec, CaseConfig

    m = cases.box_mesh(20, 20, 1, 0.1, 0.1, 0.01,
                       [("movingWall", "wall", ["y+"]), ("fixedWalls", "wall", ["x-", "x+", "y-"]),
                        ("frontAndBack", "empty", ["z-", "z+"])])
    cc = CaseConfig()
    cc.nu, cc.algorithm, cc.dt, cc.end_time = 0.01, "piso", 0.005, 0.5
    cc.boundary = {"movingWall": BoundarySpec(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
                   "fixedWalls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
                   "frontAndBack": BoundarySpec(u=("empty",), p=("empty",))}
    return Case("c1", m, cc)


def _bfs_simple():
    case = cases.gen_backward_step(4)
    case.config.algorithm = "simple"
    return case


@pytest.mark.parametrize("maker", [_cavity_2d, _bfs_simple, lambda: cases.gen_cavity(10)])
def test_step_graph_replay_is_bitwise(maker):
    """The step's assembly segments run as captured CUDA graphs (fvb_api.cu
    step_segment) from the second step on: fields, residual logs, operator
    call counts and the number of kernels launched must be exactly those of
    launching every kernel directly (FVB_STEP_NO_GRAPHS)."""
    from paper_1207_1571_b200 import _lib

    def run(flags):
        case = maker()
        cfg = CouplingConfig.from_case_config(case.config)
        st = init_state(case, cfg)
        _lib.check(_lib.lib.fvb_set_solver_options(st._ctx.h, flags))
        l0 = _lib.lib.fvb_launch_count()
        for _ in range(5):
            step(st, cfg)
        return st, _lib.lib.fvb_launch_count() - l0

    a, la = run(0)
    b, lb = run(_lib.STEP_NO_GRAPHS)
    assert np.array_equal(a.u.values, b.u.values) and np.array_equal(a.p.values, b.p.values)
    assert np.array_equal(a.flux, b.flux)
    assert a.residual_log == b.residual_log
    assert {k: v[1] for k, v in a.ops.items()} == {k: v[1] for k, v in b.ops.items()}
    assert la == lb > 0
    assert all(a.wall[k] > 0.0 for k in ("momentum_assembly", "pressure_assembly", "correction"))
