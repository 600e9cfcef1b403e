"""Device CG / BiCGStab against the reference's solver semantics
(linsolve.py:102-282): golden solves, dense oracles, error contract."""

import numpy as np
import pytest

from golden_io import CASES, golden_case, rel
from paper_1207_1571_b200 import fvm, linsolve, mesh as pmesh, sparse
from paper_1207_1571_b200.errors import SolverError
from paper_1207_1571_b200.linsolve import SolveConfig, bicgstab, bicgstab_batched, cg

pytestmark = pytest.mark.gpu


def hybrid_from_dense(dense):
    n = len(dense)
    struct = (dense != 0) | (dense.T != 0)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if struct[i, j]]
    p = sparse.pattern_from_pairs(n, pairs, n)
    A = sparse.HybridMatrix.zeros(p)
    for i in range(n):
        for j in range(n):
            if i == j or struct[i, j]:
                sparse.coeff_accumulate(A, p.address(i, j), dense[i, j], add=False)
    return A


def random_spd(rng, n):
    dense = np.zeros((n, n))
    iu, ju = np.triu_indices(n, 1)
    mask = rng.random(len(iu)) < 0.2
    dense[iu[mask], ju[mask]] = rng.normal(size=mask.sum())
    dense += dense.T
    dense[np.diag_indices(n)] = np.abs(dense).sum(axis=1) + rng.uniform(0.5, 2.0, n)
    return dense


@pytest.mark.parametrize("name", CASES)
def test_golden_solves(name):
    case, g = golden_case(name)
    pat = sparse.build_pattern(case.mesh)
    n = case.mesh.n_cells
    A = sparse.HybridMatrix.zeros(pat)
    A.V[:] = g["sol_cg_V"]
    x, rep = cg(A, g["in_b"], np.zeros(n), SolveConfig(tolerance=1e-10, max_iters=5000))
    ref = g["sol_cg_rep"]
    assert rep.converged and abs(rep.iterations - ref[0]) <= 1
    assert abs(rep.initial_residual - ref[1]) <= 1e-12 * ref[1]
    assert rel(x, g["sol_cg_x"]) < 1e-8
    M = sparse.HybridMatrix.zeros(pat)
    M.V[:] = g["op_lapv_V"]
    x, rep = bicgstab(M, g["in_b"], np.zeros(n), SolveConfig(tolerance=1e-10, max_iters=5000))
    ref = g["sol_bi_rep"]
    # BiCGStab counts on a random rhs at 1e-10 move with rounding (SURVEY §7
    # hard part 1 measured +-3 between two CPU orderings)
    assert rep.converged and abs(rep.iterations - ref[0]) <= max(3, 0.05 * ref[0])
    assert rel(x, g["sol_bi_x"]) < 1e-8


def test_cg_identity_and_2x2():
    p = sparse.pattern_from_pairs(6, [], 1)
    A = sparse.HybridMatrix.zeros(p)
    A.V[:, 0] = 1.0
    b = np.arange(1.0, 7.0)
    x, rep = cg(A, b, np.zeros(6), SolveConfig(tolerance=1e-12))
    assert np.allclose(x, b, atol=1e-14) and rep.iterations <= 1 and rep.converged
    A = hybrid_from_dense(np.array([[4.0, 1.0], [1.0, 3.0]]))
    x0 = np.array([0.3, 0.4])
    keep = x0.copy()
    x, rep = cg(A, np.array([1.0, 2.0]), x0, SolveConfig(tolerance=1e-13))
    assert np.allclose(x, [1 / 11, 7 / 11], atol=1e-10) and rep.iterations <= 2
    assert (x0 == keep).all()


def test_cg_random_spd_vs_dense():
    rng = np.random.default_rng(77)
    for _ in range(30):
        n = int(rng.integers(2, 51))
        dense = random_spd(rng, n)
        A = hybrid_from_dense(dense)
        b = rng.normal(size=n)
        x, rep = cg(A, b, np.zeros(n), SolveConfig(tolerance=1e-11, max_iters=2 * n))
        assert rep.converged and rep.iterations <= 2 * n
        assert np.allclose(x, np.linalg.solve(dense, b), rtol=1e-8, atol=1e-9)


def test_bicgstab_nonsymmetric_vs_dense_and_batched():
    rng = np.random.default_rng(5)
    for _ in range(10):
        n = int(rng.integers(3, 40))
        dense = random_spd(rng, n)
        dense += np.triu(rng.normal(scale=0.3, size=(n, n)) * (dense != 0), 1)
        A = hybrid_from_dense(dense)
        B = rng.normal(size=(n, 3))
        cfg = SolveConfig(tolerance=1e-11, max_iters=500)
        xs = []
        for c in range(3):
            x, rep = bicgstab(A, B[:, c], np.zeros(n), cfg)
            assert rep.converged
            assert np.allclose(x, np.linalg.solve(dense, B[:, c]), rtol=1e-7, atol=1e-9)
            xs.append((x, rep))
        X, reps = bicgstab_batched(A, B, np.zeros((n, 3)), cfg)
        for c in range(3):
            assert np.array_equal(X[:, c], xs[c][0])
            assert reps[c].iterations == xs[c][1].iterations


def test_error_contract():
    A = hybrid_from_dense(np.array([[0.0, 1.0], [1.0, 3.0]]))
    with pytest.raises(SolverError, match="row 0"):
        cg(A, np.ones(2), np.zeros(2), SolveConfig())
    A = hybrid_from_dense(np.array([[-1.0, 0.0], [0.0, -2.0]]))
    with pytest.raises(SolverError, match="not positive definite at iteration 1"):
        cg(A, np.ones(2), np.zeros(2), SolveConfig())
    dense = np.array([[4.0, 1.0], [1.0, 3.0]])
    A = hybrid_from_dense(dense)
    x, rep = cg(A, np.zeros(2), np.zeros(2), SolveConfig())
    assert rep.iterations == 0 and rep.converged and rep.initial_residual == 0.0
    x, rep = cg(random_spd_hybrid(40), np.ones(40), np.zeros(40),
                SolveConfig(tolerance=1e-30, max_iters=3))
    assert rep.iterations == 3 and not rep.converged


def random_spd_hybrid(n):
    return hybrid_from_dense(random_spd(np.random.default_rng(1), n))


def test_stage_times_from_device_timers():
    """record_stages fills the reference's six StageTimer buckets
    (linsolve.py:18-79) from the persistent kernel's device timers."""
    from paper_1207_1571_b200.linsolve import STAGES

    case, g = golden_case("cav6")
    pat = sparse.build_pattern(case.mesh)
    n = case.mesh.n_cells
    A = sparse.HybridMatrix.zeros(pat)
    A.V[:] = g["sol_cg_V"]
    x, rep = cg(A, g["in_b"], np.zeros(n), SolveConfig(tolerance=1e-10, max_iters=5000,
                                                       record_stages=True))
    st = rep.stage_times
    assert set(st) == set(STAGES)
    assert st["smvp"] > 0 and st["daxpy"] > 0 and st["reduction"] > 0
    assert sum(st.values()) <= rep.wall_time * 1.000001 + 1e-9
    x, rep = cg(A, g["in_b"], np.zeros(n), SolveConfig(tolerance=1e-10, max_iters=5000))
    assert rep.stage_times == {}


def _box_operator(n, crs_tail, rng):
    from paper_1207_1571_b200 import cases
    mesh = cases.box_mesh(n, n, n, 1.0, 1.0, 1.0, [("all", "wall", ["x-", "x+", "y-", "y+", "z-", "z+"])])
    ni = mesh.n_internal
    pairs = np.stack([np.asarray(mesh.owner[:ni]), np.asarray(mesh.neighbour)], axis=1)
    N = mesh.n_cells
    if crs_tail:
        # random long-range couplings on ~2% of the rows with K capped at 7:
        # the overflow entries go to the CRS tail and those rows escape the
        # stencil codes
        a = rng.choice(N, size=max(1, N // 50), replace=False)
        b = rng.integers(0, N, size=a.size)
        extra = np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1)
        pairs = np.unique(np.concatenate([pairs, extra[extra[:, 0] != extra[:, 1]]]), axis=0)
    p = sparse.pattern_from_pairs(N, pairs, 7)
    A = sparse.HybridMatrix.zeros(p)
    rows = np.arange(N)[:, None]
    A.V[:] = np.where(p.I >= 0, np.where(p.I > rows, -0.6, -1.4) * rng.uniform(0.5, 1.5, p.I.shape), 0.0)
    A.V[np.arange(N), p.diag_slot] = 0.0
    dense_rows = [np.repeat(np.arange(N), p.k)[p.I.ravel() >= 0]]
    dense_cols = [p.I.ravel()[p.I.ravel() >= 0]]
    vals = [A.V.ravel()[p.I.ravel() >= 0]]
    if p.nnz_crs:
        A.crs_val[:] = -0.3 * rng.uniform(0.5, 1.5, p.nnz_crs)
        crow = np.repeat(np.arange(N), np.diff(p.crs_row_ptr))
        dense_rows.append(crow)
        dense_cols.append(np.asarray(p.crs_col))
        vals.append(A.crs_val)
        tail = np.bincount(crow, weights=A.crs_val, minlength=N)
    else:
        tail = np.zeros(N)
    diag = -A.V.sum(axis=1) - tail + 0.5
    A.V[np.arange(N), p.diag_slot] = diag
    import scipy.sparse as sp
    M = sp.csr_matrix((np.concatenate(vals), (np.concatenate(dense_rows), np.concatenate(dense_cols))),
                      shape=(N, N))
    M = M + sp.diags(diag)
    return p, A, M


@pytest.mark.parametrize("n,crs_tail", [(8, False), (20, False), (20, True), (5, True)])
def test_bicgstab_batch_kernel_on_box_operators(n, crs_tail):
    # the persistent BiCGStab kernels on 7-point rows (one block for small
    # systems, the whole grid otherwise; CRS tail when rows overflow K):
    # the 3-component batch against a direct solve, and each component
    # against the single-vector solver (same arithmetic per component)
    import scipy.sparse.linalg as spla
    rng = np.random.default_rng(11 + n)
    p, A, M = _box_operator(n, crs_tail, rng)
    assert p.k == 7 and (p.nnz_crs > 0) == crs_tail
    N = p.n
    B = rng.normal(size=(N, 3))
    cfg = SolveConfig(tolerance=1e-12, max_iters=2000)
    X, reps = bicgstab_batched(A, B, np.zeros((N, 3)), cfg)
    for c in range(3):
        assert reps[c].converged, reps[c]
        ref = spla.spsolve(M.tocsc(), B[:, c])
        assert rel(X[:, c], ref) < 1e-9
        x1, r1 = bicgstab(A, B[:, c], np.zeros(N), cfg)
        assert abs(r1.iterations - reps[c].iterations) <= 1
        assert rel(X[:, c], x1) < 1e-9


@pytest.mark.parametrize("mode", ["", "crs"])
def test_stencil_codes_cg_bitwise_equals_explicit_indices(mode):
    # pass A on 1-byte stencil codes reads exactly the columns of the
    # explicit index array: same iterates, bit for bit ("explicit" sets
    # FVB_SOLVER_EXPLICIT_INDEX); "crs": escaped rows + CRS tail
    import json, os, subprocess, sys
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
    out = {}
    for var in ("codes", "explicit"):
        res = subprocess.run([sys.executable, os.path.join(root, "tools", "cg_micro.py"), "24", "60",
                              mode or "box", var], capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr
        out[var] = json.loads(res.stdout.strip().splitlines()[-1])
    if mode:
        assert out["codes"]["escaped"] > 0 and out["codes"]["nnz_crs"] > 0
    else:
        assert out["codes"]["codes"] == 27 and out["codes"]["escaped"] == 0
    assert out["explicit"]["codes"] == 0 and out["codes"]["defer_x"] == 1
    assert out["codes"]["x_sha"] == out["explicit"]["x_sha"]
    assert out["codes"]["res"] == out["explicit"]["res"]


def test_stencil_code_dictionary():
    import ctypes as C
    from paper_1207_1571_b200 import _lib, cases
    from paper_1207_1571_b200.device import context_for

    def codes_of(pat):
        ctx = context_for(None, None, pat)
        nc, ne = C.c_int(), C.c_int64()
        _lib.check(_lib.lib.fvb_pattern_codes(ctx.h, C.byref(nc), C.byref(ne), None, None))
        return nc.value, ne.value

    box = cases.box_mesh(10, 9, 8, 1.0, 1.0, 1.0, [("all", "wall", ["x-", "x+", "y-", "y+", "z-", "z+"])])
    assert codes_of(sparse.build_pattern(box)) == (27, 0)
    # a random renumbering leaves no common offset tuples: codes off
    perm = np.random.default_rng(3).permutation(box.n_cells)
    ni = box.n_internal
    pairs = np.stack([perm[np.asarray(box.owner[:ni])], perm[np.asarray(box.neighbour)]], axis=1)
    pairs = np.sort(pairs, axis=1)
    assert codes_of(sparse.pattern_from_pairs(box.n_cells, pairs, 16)) == (0, 0)


@pytest.mark.parametrize("mode", ["", "crs"])
def test_stencil_codes_bicgstab_bitwise_equals_explicit_indices(mode):
    # batched BiCGStab SpMV sweeps on stencil codes ("explicit" sets
    # FVB_SOLVER_EXPLICIT_INDEX); "crs" adds rows that overflow K (escaped
    # rows and a CRS tail)
    import json, os, subprocess, sys
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
    out = {}
    for var in ("codes", "explicit"):
        res = subprocess.run([sys.executable, os.path.join(root, "tools", "bi_micro.py"), "20", "30",
                              mode or "box", var], capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr
        out[var] = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["codes"]["codes"] > 0 and out["explicit"]["codes"] == 0
    assert out["codes"]["x_sha"] == out["explicit"]["x_sha"]
    assert out["codes"]["iters"] == out["explicit"]["iters"]
    assert out["codes"]["res"] == out["explicit"]["res"]


def test_rcm_ordered_cg_on_renumbered_box():
    # a randomly renumbered box has no stencil codes; CG then runs in the
    # solver's reverse Cuthill-McKee order (>= 65536 rows).  Same row
    # products, only the dot-product grouping moves: residual and iterate
    # agree with the original-order solve ("norcm" sets FVB_SOLVER_NO_RCM)
    # to rounding
    import json, os, subprocess, sys
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
    out = {}
    for var in ("rcm", "norcm"):
        res = subprocess.run([sys.executable, os.path.join(root, "tools", "cg_micro.py"), "48", "80", "perm",
                              var], capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, res.stderr
        out[var] = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["rcm"]["codes"] == 0 and out["rcm"]["rcm_solves"] == 3
    assert out["norcm"]["rcm_solves"] == 0
    assert abs(out["rcm"]["res"] - out["norcm"]["res"]) <= 1e-9 * out["norcm"]["res"]


def test_rcm_ordered_bicgstab_single_and_batched():
    # renumbered 42^3 box (74,088 rows, no stencil codes): BiCGStab runs in
    # the RCM order for one and for three right-hand sides; the batch equals
    # the single solves component by component, and the residual is small
    import scipy.sparse as sp
    from paper_1207_1571_b200 import cases

    n = 42
    box = cases.box_mesh(n, n, n, 1.0, 1.0, 1.0, [("all", "wall", ["x-", "x+", "y-", "y+", "z-", "z+"])])
    ni = box.n_internal
    perm = np.random.default_rng(6).permutation(box.n_cells)
    pairs = np.sort(np.stack([perm[np.asarray(box.owner[:ni])], perm[np.asarray(box.neighbour)]], axis=1), axis=1)
    p = sparse.pattern_from_pairs(box.n_cells, pairs, 16)
    N = p.n
    assert p.k == 7 and p.nnz_crs == 0
    A = sparse.HybridMatrix.zeros(p)
    rows = np.arange(N)[:, None]
    A.V[:] = np.where(p.I >= 0, np.where(p.I > rows, -0.7, -1.3), 0.0)
    A.V[np.arange(N), p.diag_slot] = 0.0
    A.V[np.arange(N), p.diag_slot] = -A.V.sum(axis=1) + 0.3
    mask = p.I.ravel() >= 0
    M = sp.csr_matrix((A.V.ravel()[mask], (np.repeat(np.arange(N), p.k)[mask], p.I.ravel()[mask])),
                      shape=(N, N))
    B = np.random.default_rng(7).normal(size=(N, 3))
    cfg = SolveConfig(tolerance=1e-10, max_iters=2000)
    import ctypes as C
    from paper_1207_1571_b200 import _lib
    from paper_1207_1571_b200.device import context_for
    ctx = context_for(None, None, p)
    r0, r1c = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib.fvb_pattern_codes(ctx.h, None, None, None, C.byref(r0)))
    X, reps = bicgstab_batched(A, B, np.zeros((N, 3)), cfg)
    for c in range(3):
        x1, r1 = bicgstab(A, B[:, c], np.zeros(N), cfg)
        assert r1.converged and reps[c].converged
        assert np.array_equal(X[:, c], x1) and r1.iterations == reps[c].iterations
        assert np.linalg.norm(B[:, c] - M @ x1) <= 1e-8 * np.linalg.norm(B[:, c])
    _lib.check(_lib.lib.fvb_pattern_codes(ctx.h, None, None, None, C.byref(r1c)))
    assert r1c.value - r0.value == 4  # one batch + three single solves


@pytest.mark.parametrize("n", [7, 20])
def test_small_system_paths_match_grid_path(n):
    # n=7 (343 rows): one block with the work vectors in shared memory;
    # n=20 (8000 rows): one 16-CTA thread-block cluster (DSMEM reductions).
    # Both against the plain block / grid path (FVB_SOLVER_NO_CLUSTER): same
    # row arithmetic, only the grouping of the dot products differs.
    from paper_1207_1571_b200 import _lib
    from paper_1207_1571_b200.device import context_for

    rng = np.random.default_rng(40 + n)
    p, A, M = _box_operator(n, False, rng)
    N = p.n
    b = rng.normal(size=N)
    B = rng.normal(size=(N, 3))
    # SPD copy for CG: symmetric part made diagonally dominant
    S = sparse.HybridMatrix.zeros(p)
    rows = np.arange(N)[:, None]
    S.V[:] = np.where(p.I >= 0, -1.0, 0.0)
    S.V[np.arange(N), p.diag_slot] = (p.I >= 0).sum(axis=1) - 1 + 0.05
    cfg = SolveConfig(tolerance=1e-11, max_iters=5000)
    ctx = context_for(None, None, p)
    out = {}
    for mode, flags in (("small", 0), ("grid", _lib.SOLVER_NO_CLUSTER)):
        _lib.check(_lib.lib.fvb_set_solver_options(ctx.h, flags))
        try:
            out[mode] = (cg(S, b, np.zeros(N), cfg), bicgstab_batched(A, B, np.zeros((N, 3)), cfg))
        finally:
            _lib.check(_lib.lib.fvb_set_solver_options(ctx.h, 0))
    (xs, rs), (Xs, Rs) = out["small"]
    (xg, rg), (Xg, Rg) = out["grid"]
    assert rs.converged and rg.converged and abs(rs.iterations - rg.iterations) <= 1
    assert rel(xs, xg) < 1e-9
    for c in range(3):
        assert Rs[c].converged and abs(Rs[c].iterations - Rg[c].iterations) <= 2
        assert rel(Xs[:, c], Xg[:, c]) < 1e-8
        assert np.linalg.norm(B[:, c] - M @ Xs[:, c]) <= 1e-9 * np.linalg.norm(B[:, c])
    # deterministic: a repeat of the small-path solves is bitwise equal
    x2, r2 = cg(S, b, np.zeros(N), cfg)
    X2, R2 = bicgstab_batched(A, B, np.zeros((N, 3)), cfg)
    assert np.array_equal(x2, xs) and np.array_equal(X2, Xs)
