"""The numpy oracle (oracle/fvoracle.py) against the golden vectors that the
REAL reference produced (oracle/make_golden.py).  This pins the oracle
before any CUDA result is compared with it."""

import os

import numpy as np
import pytest

from golden_io import CASES, GOLDEN, golden_case, rel
from oracle import fvoracle as O


@pytest.mark.parametrize("name", CASES)
def test_oracle_geometry_and_pattern_bitwise(name):
    case, g = golden_case(name)
    m = O.mesh_arrays(case.mesh)
    geo = O.geometry(m)
    for k, v in geo.items():
        assert np.array_equal(v, g["geom_" + k]), k
    P = O.mesh_pattern(m)
    for k in ("I", "J", "diag_slot", "ell_twin_crs", "crs_row_ptr", "crs_col", "crs_twin_in_ell",
              "crs_twin_pos", "diag_addr", "face_addr"):
        assert np.array_equal(P[k], g["pat_" + k]), k
    assert P["k"] == int(g["pat_k"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_operators(name):
    case, g = golden_case(name)
    m = O.mesh_arrays(case.mesh)
    geo = O.geometry(m)
    P = O.mesh_pattern(m)
    ub = {n: O.bc_kind(s.u) for n, s in case.config.boundary.items()}
    pb = {n: O.bc_kind(s.p) for n, s in case.config.boundary.items()}
    u = O.BField(m, ub, g["in_u"].copy())
    p = O.BField(m, pb, g["in_p"].copy())
    O.apply_bcs(u, geo, float(g["in_t"]))
    O.apply_bcs(p, geo, float(g["in_t"]))
    assert np.array_equal(u.boundary, g["op_ub"]) and np.array_equal(p.boundary, g["op_pb"])
    assert np.array_equal(O.face_values(u, geo), g["op_interp_u"])
    assert np.array_equal(O.face_values(p, geo), g["op_interp_p"])
    assert np.array_equal(O.face_values_raw(m, geo, g["in_raw"]), g["op_interp_raw"])
    assert np.array_equal(O.gradient(u, geo), g["op_grad_u"])
    assert np.array_equal(O.gradient(p, geo), g["op_grad_p"])
    assert np.array_equal(O.divergence(m, g["in_flux"]), g["op_div"])
    A = O.Matrix(P)
    rhs = np.zeros((m["nc"], 3))
    O.ddt(A, rhs, g["in_old"], 0.01, geo)
    assert np.array_equal(A.V, g["op_ddt_V"]) and np.array_equal(rhs, g["op_ddt_rhs"])
    O.convection(A, rhs, g["in_flux"], u, geo)
    assert np.array_equal(A.V, g["op_conv_V"]) and np.array_equal(rhs, g["op_conv_rhs"])
    coef, corr = O.laplacian(A, rhs, 0.013, u, geo, coeff=-1.0)
    assert np.array_equal(A.V, g["op_lapv_V"]) and np.array_equal(rhs, g["op_lapv_rhs"])
    assert np.array_equal(coef, g["op_lapv_coef"]) and np.array_equal(corr, g["op_lapv_corr"])
    assert np.array_equal(O.laplacian_flux(coef, corr, u), g["op_lapv_flux"])
    assert np.array_equal(O.spmv(A, g["in_x"]), g["op_smvp"])
    As = O.Matrix(P)
    rs = np.zeros(m["nc"])
    O.convection(As, rs, g["in_flux"], p, geo, scheme="linear", coeff=0.7)
    assert np.array_equal(As.V, g["op_convlin_V"]) and np.array_equal(rs, g["op_convlin_rhs"])
    Ap = O.Matrix(P)
    rp = np.zeros(m["nc"])
    coef, corr = O.laplacian(Ap, rp, g["in_gamma"], p, geo, coeff=-1.0)
    assert np.array_equal(Ap.V, g["op_lapp_V"]) and np.array_equal(rp, g["op_lapp_rhs"])
    assert np.array_equal(O.laplacian_flux(coef, corr, p), g["op_lapp_flux"])
    Ap.V[0, P["diag_slot"][0]] *= 2.0
    x, rep = O.pcg(Ap, g["in_b"], np.zeros(m["nc"]), 1e-10, max_iters=5000)
    ref = g["sol_cg_rep"]
    assert abs(rep[0] - ref[0]) <= 1 and rel(x, g["sol_cg_x"]) < 1e-9
    x, rep = O.pbicgstab(A, g["in_b"], np.zeros(m["nc"]), 1e-10, max_iters=5000)
    ref = g["sol_bi_rep"]
    assert abs(rep[0] - ref[0]) <= 1 and rel(x, g["sol_bi_x"]) < 1e-8


@pytest.mark.parametrize("name", CASES)
def test_oracle_coupled_steps(name):
    case, g = golden_case(name)
    run = O.Run(case.mesh, case.config)
    assert np.array_equal(run.flux, g["init_flux"])
    for s in range(int(g["steps"])):
        r = run.piso_step() if case.config.algorithm == "piso" else run.simple_sweep()
        assert np.allclose(r, g[f"s{s}_ret"], rtol=1e-6, atol=1e-14)
        assert rel(run.u.values, g[f"s{s}_u"]) < 1e-9
        assert rel(run.p.values, g[f"s{s}_p"]) < 1e-9
        assert rel(run.flux, g[f"s{s}_flux"]) < 1e-9
        log = g[f"s{s}_log"]
        mine = np.array([r[3] for r in run.log[-len(log):]])
        assert np.abs(mine - log[:, 1]).max() <= 1


@pytest.mark.parametrize("name", CASES)
def test_oracle_rhie_chow_vs_reference(name):
    """oracle.rhie_chow against the real reference's rhie_chow_flux
    (fvm.py:499-538; tests/golden/rhie.npz, oracle/make_golden_rhie.py)."""
    case, g = golden_case(name)
    with np.load(os.path.join(GOLDEN, "rhie.npz")) as z:
        a_diag, want = z[f"{name}_a_diag"], z[f"{name}_flux"]
    m = O.mesh_arrays(case.mesh)
    geo = O.geometry(m)
    ub = {n: O.bc_kind(s.u) for n, s in case.config.boundary.items()}
    pb = {n: O.bc_kind(s.p) for n, s in case.config.boundary.items()}
    u = O.BField(m, ub, g["in_u"].copy())
    p = O.BField(m, pb, g["in_p"].copy())
    O.apply_bcs(u, geo, float(g["in_t"]))
    O.apply_bcs(p, geo, float(g["in_t"]))
    got = O.rhie_chow(u, p, a_diag, geo)
    assert np.array_equal(got, want), rel(got, want)
    bad = a_diag.copy()
    bad[3] = 0.0
    with pytest.raises(O.OracleError, match="cell 3"):
        O.rhie_chow(u, p, bad, geo)
