"""Single-operator parity on the device: every FV
kernel and the SpMV against the real reference's outputs (golden fixtures)
and the oracle.  Bar: 1e-12 relative (north_star); most are bitwise."""

import numpy as np
import pytest

from golden_io import CASES, golden_case, rel
from paper_1207_1571_b200 import fvm, mesh as pmesh, sparse

pytestmark = pytest.mark.gpu
TOL = 1e-12


def setup(name):
    case, g = golden_case(name)
    geo = pmesh.compute_geometry(case.mesh)
    pat = sparse.build_pattern(case.mesh)
    ub = {n: fvm.bc_from_tuple(s.u) for n, s in case.config.boundary.items()}
    pb = {n: fvm.bc_from_tuple(s.p) for n, s in case.config.boundary.items()}
    u = fvm.make_vector("u", case.mesh, ub)
    p = fvm.make_scalar("p", case.mesh, pb)
    u.values = g["in_u"].copy()
    p.values = g["in_p"].copy()
    return case, g, geo, pat, u, p


def close(a, b, tol=TOL):
    assert np.shape(a) == np.shape(b)
    assert rel(a, b) <= tol, rel(a, b)


@pytest.mark.parametrize("name", CASES)
def test_bcs_interp_gradient_divergence(name):
    case, g, geo, pat, u, p = setup(name)
    t = float(g["in_t"])
    fvm.apply_bcs(u, geo, t)
    fvm.apply_bcs(p, geo, t)
    assert np.array_equal(u.boundary, g["op_ub"])
    assert np.array_equal(p.boundary, g["op_pb"])
    assert np.array_equal(fvm.interpolate_to_faces(u, geo), g["op_interp_u"])
    assert np.array_equal(fvm.interpolate_to_faces(p, geo), g["op_interp_p"])
    assert np.array_equal(fvm.interpolate_cell_values(case.mesh, geo, g["in_raw"]),
                          g["op_interp_raw"])
    assert np.array_equal(fvm.gauss_gradient(u, geo), g["op_grad_u"])
    assert np.array_equal(fvm.gauss_gradient(p, geo), g["op_grad_p"])
    assert np.array_equal(fvm.face_divergence(case.mesh, g["in_flux"]), g["op_div"])


@pytest.mark.parametrize("name", CASES)
def test_assembly_operators(name):
    case, g, geo, pat, u, p = setup(name)
    t = float(g["in_t"])
    fvm.apply_bcs(u, geo, t)
    fvm.apply_bcs(p, geo, t)
    scheme = fvm.SchemeConfig()
    sysv = fvm.LinearSystem.zeros(pat, "vector")
    fvm.ddt_euler(sysv, u, g["in_old"], 0.01, geo)
    assert np.array_equal(sysv.A.V, g["op_ddt_V"]) and np.array_equal(sysv.rhs, g["op_ddt_rhs"])
    fvm.divergence_convection(sysv, g["in_flux"], u, scheme, geom=geo)
    close(sysv.A.V, g["op_conv_V"])
    close(sysv.rhs, g["op_conv_rhs"])
    fd = fvm.laplacian(sysv, 0.013, u, geo, scheme, coeff=-1.0)
    close(sysv.A.V, g["op_lapv_V"])
    close(sysv.rhs, g["op_lapv_rhs"])
    close(fd.coef, g["op_lapv_coef"])
    close(fd.corr, g["op_lapv_corr"])
    close(fvm.laplacian_face_flux(fd, u), g["op_lapv_flux"])
    y = sparse.smvp(sysv.A, g["in_x"])
    assert np.array_equal(y, sparse.smvp(sysv.A, g["in_x"]))
    close(y, g["op_smvp"])
    syss = fvm.LinearSystem.zeros(pat)
    fvm.divergence_convection(syss, g["in_flux"], p, fvm.SchemeConfig(convection="linear"),
                              geom=geo, coeff=0.7)
    close(syss.A.V, g["op_convlin_V"])
    close(syss.rhs, g["op_convlin_rhs"])
    sysp = fvm.LinearSystem.zeros(pat)
    fd = fvm.laplacian(sysp, g["in_gamma"], p, geo, scheme, coeff=-1.0)
    close(sysp.A.V, g["op_lapp_V"])
    close(sysp.rhs, g["op_lapp_rhs"])
    close(fd.coef, g["op_lapp_coef"])
    close(fd.corr, g["op_lapp_corr"])
    close(fvm.laplacian_face_flux(fd, p), g["op_lapp_flux"])


@pytest.mark.parametrize("name", CASES)
def test_operators_bitwise_where_reference_order_is_known(name):
    # the device replays np.add.at order and numpy's einsum order: on the
    # reference's own inputs the assembled systems come out bit-identical
    case, g, geo, pat, u, p = setup(name)
    fvm.apply_bcs(u, geo, float(g["in_t"]))
    sysv = fvm.LinearSystem.zeros(pat, "vector")
    fvm.ddt_euler(sysv, u, g["in_old"], 0.01, geo)
    fvm.divergence_convection(sysv, g["in_flux"], u, fvm.SchemeConfig(), geom=geo)
    fd = fvm.laplacian(sysv, 0.013, u, geo, fvm.SchemeConfig(), coeff=-1.0)
    assert np.array_equal(sysv.A.V, g["op_lapv_V"])
    assert np.array_equal(sysv.rhs, g["op_lapv_rhs"])
    assert np.array_equal(fd.corr, g["op_lapv_corr"])
    assert np.array_equal(sparse.smvp(sysv.A, g["in_x"]), g["op_smvp"])


def test_smvp_random_hybrid_with_crs_vs_dense():
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(3, 60))
        iu, ju = np.triu_indices(n, 1)
        mask = rng.random(len(iu)) < rng.uniform(0.05, 0.4)
        pairs = np.stack([iu[mask], ju[mask]], axis=1)
        p = sparse.pattern_from_pairs(n, pairs, int(rng.integers(1, 9)))
        A = sparse.HybridMatrix.zeros(p)
        A.V[p.I >= 0] = rng.normal(size=int((p.I >= 0).sum()))
        A.crs_val[:] = rng.normal(size=p.nnz_crs)
        x = rng.normal(size=n)
        y = sparse.smvp(A, x)
        d = A.to_dense() @ x
        scale = np.abs(A.to_dense()) @ np.abs(x)
        assert np.all(np.abs(y - d) <= 1e-13 * scale + 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_rhie_chow_flux_bitwise(name):
    """fvm.rhie_chow_flux (fvb_op_rhie_chow: device gradient + face kernel)
    against the real reference's rhie_chow_flux (fvm.py:499-538) on the
    golden meshes: 2D empties, pressure-pinned outlets, perturbed cells."""
    import os
    from golden_io import GOLDEN
    from paper_1207_1571_b200.errors import FvmError

    case, g, geo, pat, u, p = setup(name)
    t = float(g["in_t"])
    fvm.apply_bcs(u, geo, t)
    fvm.apply_bcs(p, geo, t)
    with np.load(os.path.join(GOLDEN, "rhie.npz")) as z:
        a_diag, want = z[f"{name}_a_diag"], z[f"{name}_flux"]
    got = fvm.rhie_chow_flux(u, p, a_diag, geo)
    assert np.array_equal(got, want), rel(got, want)
    bad = a_diag.copy()
    bad[5] = 0.0
    with pytest.raises(FvmError, match="zero momentum diagonal at cell 5"):
        fvm.rhie_chow_flux(u, p, bad, geo)
