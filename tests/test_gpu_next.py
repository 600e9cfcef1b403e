"""SURVEY.md §8(f) next rows on the device: the transposed product through
the paper's J twin table (stmvp, sparse.py:308-334) against the REAL
reference's outputs, and the profile report built from device timers."""

import os

import numpy as np
import pytest

from golden_io import GOLDEN, golden_case, load
from paper_1207_1571_b200 import cases, report, sparse
from paper_1207_1571_b200.coupling import CouplingConfig, run_case

pytestmark = pytest.mark.gpu
NZ = np.load(os.path.join(GOLDEN, "next.npz"))


@pytest.mark.parametrize("name", ["cav6", "pcav5", "bfs2", "duct"])
def test_stmvp_bitwise_vs_reference(name):
    case, g = golden_case(name)
    pat = sparse.build_pattern(case.mesh)
    A = sparse.HybridMatrix.zeros(pat)
    A.V[:] = g["op_conv_V"]
    y = sparse.stmvp(A, g["in_x"])
    assert np.array_equal(y, NZ[f"{name}_stmvp"])
    dense = A.to_dense()
    ref = dense.T @ g["in_x"]
    assert np.abs(y - ref).max() <= 1e-13 * (np.abs(dense.T) @ np.abs(g["in_x"])).max()


@pytest.mark.parametrize("t", range(6))
def test_stmvp_with_crs_spill(t):
    n = int(NZ[f"rnd{t}_n"])
    pat = sparse.pattern_from_pairs(n, NZ[f"rnd{t}_pairs"], int(NZ[f"rnd{t}_kcap"]))
    A = sparse.HybridMatrix.zeros(pat)
    A.V[:] = NZ[f"rnd{t}_V"]
    A.crs_val[:] = NZ[f"rnd{t}_crs"]
    x = NZ[f"rnd{t}_x"]
    y = sparse.stmvp(A, x)
    ref = NZ[f"rnd{t}_stmvp"]
    scale = (np.abs(A.to_dense().T) @ np.abs(x)).max()
    assert np.abs(y - ref).max() <= 1e-13 * scale
    assert np.abs(sparse.smvp(A, x) - NZ[f"rnd{t}_smvp"]).max() <= 1e-13 * scale


def test_profile_report_from_device_timers():
    case = cases.gen_cavity(8)
    cc = case.config
    cc.algorithm, cc.dt, cc.end_time = "piso", 0.1 / 8, 3 * 0.1 / 8
    st = run_case(case, record_stages=True)
    assert st.outer == 3
    for name in ("ddt", "convection", "laplacian", "gradient", "divergence"):
        sec, calls = st.ops[name]
        assert sec > 0 and calls > 0, name
    assert st.ops["ddt"][1] == 3 and st.ops["laplacian"][1] == 3 + 3 * cc.n_correctors
    prof = report.collect_profile(st)
    h, rows = report.solver_share_table(prof)
    assert abs(sum(r[2] for r in rows) - 100.0) < 1e-9
    h, rows = report.cg_stage_table(prof)
    assert dict((r[0], r[1]) for r in rows)["smvp"] > 0
    h, rows = report.assembly_norm_table(prof)
    assert all(np.isfinite(r[4]) and r[4] > 0 for r in rows)
    text = report.format_tables(prof)
    assert "cg kernel breakdown" in text and "assembly cost per operator" in text
