"""Native (C++) setup path against the reference: the box-mesh generator,
compute_geometry and the hybrid pattern must be bit-identical (§8 a1-a3)."""

import numpy as np
import pytest

from golden_io import CASES, golden_case, load
from oracle import fvoracle as O
from paper_1207_1571_b200 import cases, mesh as pmesh, sparse
from paper_1207_1571_b200.errors import MeshError, SparseError


@pytest.mark.parametrize("name", CASES)
def test_geometry_bitwise(name):
    case, g = golden_case(name)
    geo = pmesh.compute_geometry(case.mesh)
    for k in geo.__dataclass_fields__:
        assert np.array_equal(getattr(geo, k), g["geom_" + k]), k


@pytest.mark.parametrize("name", CASES)
def test_pattern_bitwise(name):
    case, g = golden_case(name)
    p = sparse.build_pattern(case.mesh)
    for k in ("I", "J", "diag_slot", "ell_twin_crs", "crs_row_ptr", "crs_col", "crs_twin_in_ell",
              "crs_twin_pos", "diag_addr", "face_addr"):
        assert np.array_equal(getattr(p, k), g["pat_" + k]), k
    assert p.k == int(g["pat_k"])
    p.check_invariants()


@pytest.mark.parametrize("name,make", [
    ("cav6", lambda: cases.gen_cavity(6)),
    ("chan", lambda: cases.gen_channel(12, 4)),
    ("duct", lambda: cases.gen_skewed_duct(8, 6, 30.0)),
])
def test_generators_match_reference_meshes(name, make):
    g = load(name)
    m = make().mesh
    for k in ("points", "face_points", "face_offsets", "owner", "neighbour"):
        assert np.array_equal(getattr(m, k), g[k]), k
        assert getattr(m, k).dtype == g[k].dtype
    assert [p.name for p in m.patches] == [str(s) for s in g["patch_names"]]
    assert [p.start for p in m.patches] == g["patch_start"].tolist()


def test_box_counts_and_c3_c4_generators():
    m = cases.gen_cavity(7).mesh
    assert (m.n_cells, m.n_faces) == cases.box_counts(7, 7, 7)
    bfs = cases.gen_backward_step(4).mesh  # 1,040 cells, 4,308 faces
    assert (bfs.n_cells, bfs.n_faces) == (1040, 4308)
    geo = pmesh.compute_geometry(bfs)
    assert pmesh.closedness_error(bfs, geo) < 1e-18
    pc = cases.perturbed_cavity(8).mesh
    geo = pmesh.compute_geometry(pc)
    assert geo.max_nonorth_deg < 80.0 and geo.max_nonorth_deg > 5.0
    assert abs(geo.cell_volume.sum() - 1e-3) < 1e-15
    assert sparse.build_pattern(pc).k == 7


def test_pattern_random_with_crs_spill_matches_oracle():
    rng = np.random.default_rng(3)
    spilled = 0
    for trial in range(40):
        n = int(rng.integers(2, 40))
        iu, ju = np.triu_indices(n, 1)
        mask = rng.random(len(iu)) < rng.uniform(0.05, 0.5)
        pairs = np.stack([iu[mask], ju[mask]], axis=1)
        if not len(pairs):
            continue
        kcap = int(rng.integers(1, 8))
        p = sparse.pattern_from_pairs(n, pairs, kcap)
        q = O.pattern(n, pairs, kcap)
        for k in ("I", "J", "diag_slot", "ell_twin_crs", "crs_row_ptr", "crs_col",
                  "crs_twin_in_ell", "crs_twin_pos", "face_addr"):
            assert np.array_equal(getattr(p, k), q[k]), (trial, k)
        spilled += p.nnz_crs > 0
        p.check_invariants()
    assert spilled >= 10


def test_ring_fixture():
    g = load("fixtures")
    p = sparse.build_pattern_from_example()
    assert np.array_equal(p.I, g["ring_I"]) and np.array_equal(p.J, g["ring_J"])
    assert np.array_equal(p.diag_slot, g["ring_diag_slot"])


def test_errors():
    with pytest.raises(SparseError, match="k_cap"):
        sparse.pattern_from_pairs(3, [(0, 1)], 0)
    with pytest.raises(SparseError, match="self-pair"):
        sparse.pattern_from_pairs(3, [(1, 1)], 4)
    m = cases.gen_cavity(2).mesh
    m.points = m.points.copy()
    m.points[:, 0] = 0.0  # flatten: every x-normal face degenerates
    with pytest.raises(MeshError, match="degenerate"):
        pmesh.compute_geometry(m)


def test_face_triangles_close_the_volume():
    """mesh._face_triangles (reference mesh.py:154-170): the fan triangles of
    a warped hexahedron reproduce the native geometry's cell volume through
    the divergence identity (the reference's test_mesh.py check)."""
    from paper_1207_1571_b200.mesh import Mesh, Patch

    corners = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                        [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]], dtype=float)
    loops = [[0, 3, 2, 1], [4, 5, 6, 7], [0, 4, 7, 3], [1, 2, 6, 5], [0, 1, 5, 4], [3, 7, 6, 2]]
    rng = np.random.default_rng(3)
    for _ in range(10):
        pts = corners + rng.uniform(-0.15, 0.15, size=(8, 3))
        m = Mesh(points=pts, face_points=np.concatenate(loops).astype(np.int64),
                 face_offsets=np.arange(0, 25, 4, dtype=np.int64), owner=np.zeros(6, dtype=np.int64),
                 neighbour=np.zeros(0, dtype=np.int64), patches=[Patch("walls", "wall", 0, 6)],
                 n_cells=1)
        m.validate()
        geo = pmesh.compute_geometry(m)
        a, b, seed, face = pmesh._face_triangles(m)
        assert a.shape == b.shape == seed.shape == (24, 3) and list(face) == sorted(face)
        tri_s = 0.5 * np.cross(b - a, seed - a)
        vol = np.einsum("ij,ij->i", (a + b + seed) / 3.0, tri_s).sum() / 3.0
        assert geo.cell_volume[0] == pytest.approx(vol, rel=1e-12)


def test_jacobi_apply():
    """linsolve.jacobi_apply (reference linsolve.py:82-87): r / D, and the
    solvers' zero-diagonal message."""
    from paper_1207_1571_b200.linsolve import SolverError, jacobi_apply

    d = np.array([2.0, 4.0, 0.5])
    r = np.array([1.0, -2.0, 3.0])
    assert np.array_equal(jacobi_apply(d, r), r / d)
    with pytest.raises(SolverError, match="zero diagonal at row 1"):
        jacobi_apply(np.array([1.0, 0.0, 0.0]), np.ones(3))
