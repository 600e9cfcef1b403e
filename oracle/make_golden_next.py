"""Golden vectors for the SURVEY.md §8(f) "next" rows, from the REAL reference
(test infrastructure; run in the build container where /root/reference exists):

    python oracle/make_golden_next.py

  * stmvp (sparse.py:308-334) on the golden momentum matrices and on random
    structurally-symmetric patterns with CRS spill (test_sparse.py:85-113);
  * pack_q / unpack_q (sparse.py:337-363) in both modes;
  * write_mesh text (fileio.py:50-65) for three meshes and the read_mesh
    MeshFileError message (fileio.py:106-185) for a set of malformed files;
  * collect_profile / table outputs (report.py:33-134) on a synthetic run.

Output: tests/golden/next.npz and tests/golden/next.json (small).
"""

import json
import os
import sys
import tempfile
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
REF = "/root/reference/pkg/src"


def _stub_matplotlib():
    mpl = types.ModuleType("matplotlib")
    mpl.use = lambda *a, **k: None
    plt = types.ModuleType("matplotlib.pyplot")
    mpl.pyplot = plt
    sys.modules["matplotlib"] = mpl
    sys.modules["matplotlib.pyplot"] = plt


def main():
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _stub_matplotlib()
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import fvflow.cases as rcases
    import fvflow.fileio as rfile
    import fvflow.mesh as rmesh
    import fvflow.report as rreport
    import fvflow.sparse as rs

    npz, js = {}, {}
    # ---------------------------------------------------------------- stmvp
    from golden_io import load

    for name in ("cav6", "pcav5", "bfs2", "duct"):
        g = load(name)
        m = rmesh.Mesh(points=g["points"], face_points=g["face_points"],
                       face_offsets=g["face_offsets"], owner=g["owner"], neighbour=g["neighbour"],
                       patches=[rmesh.Patch(str(a), str(b), int(c), int(d)) for a, b, c, d in
                                zip(g["patch_names"], g["patch_kinds"], g["patch_start"],
                                    g["patch_count"])], n_cells=int(g["n_cells"]))
        pat = rs.build_pattern(m)
        A = rs.HybridMatrix.zeros(pat)
        A.V[:] = g["op_conv_V"]          # convection makes it non-symmetric
        npz[f"{name}_stmvp"] = rs.stmvp(A, g["in_x"])
        for mode in ("by_N", "by_K"):
            npz[f"{name}_q_{mode}"] = rs.pack_q(pat, mode)
    rng = np.random.default_rng(1207)
    for t in range(6):
        n = int(rng.integers(5, 40))
        iu, ju = np.triu_indices(n, 1)
        mask = rng.random(len(iu)) < 0.3
        pairs = np.stack([iu[mask], ju[mask]], axis=1)
        pat = rs.pattern_from_pairs(n, pairs, k_cap=int(rng.integers(2, 5)))
        A = rs.HybridMatrix.zeros(pat)
        A.V[:] = rng.normal(size=A.V.shape) * (pat.I >= 0)
        A.crs_val[:] = rng.normal(size=A.crs_val.shape)
        x = rng.normal(size=n)
        npz[f"rnd{t}_n"] = np.int64(n)
        npz[f"rnd{t}_pairs"] = pairs
        npz[f"rnd{t}_kcap"] = np.int64(pat.k if pat.nnz_crs == 0 else pat.k)
        npz[f"rnd{t}_V"] = A.V
        npz[f"rnd{t}_crs"] = A.crs_val
        npz[f"rnd{t}_x"] = x
        npz[f"rnd{t}_stmvp"] = rs.stmvp(A, x)
        npz[f"rnd{t}_smvp"] = rs.smvp(A, x)
        npz[f"rnd{t}_nnz_crs"] = np.int64(pat.nnz_crs)
        for mode in ("by_N", "by_K"):
            npz[f"rnd{t}_q_{mode}"] = rs.pack_q(pat, mode)
    # --------------------------------------------------------------- mesh I/O
    tmp = tempfile.mkdtemp()
    texts = {}
    meshes = {"cav3": rcases.gen_cavity(3).mesh, "chan": rcases.gen_channel(6, 3).mesh,
              "duct": rcases.gen_skewed_duct(4, 3, 30.0).mesh}
    for k, m in meshes.items():
        p = os.path.join(tmp, k + ".msh")
        rfile.write_mesh(m, p)
        texts[k] = open(p).read()
    js["mesh_text"] = texts
    base = texts["cav3"]
    lines = base.splitlines()
    bad = {}

    def mutate(name, text):
        bad[name] = text

    mutate("bad_header", "POINTS eight\n")
    mutate("short_points", "POINTS 4\n0 0 0\n1 0 0\n")
    mutate("coords", base.replace(lines[1], "0 0", 1))
    mutate("nonnumeric", base.replace(lines[2], "0 x 0", 1))
    i_f = lines.index(next(l for l in lines if l.startswith("FACES")))
    mutate("face_count", base.replace(lines[i_f + 1], "5 " + lines[i_f + 1][2:], 1))
    mutate("face_small", "\n".join(lines[:i_f + 1] + ["2 0 1"] + lines[i_f + 2:]) + "\n")
    mutate("face_point", "\n".join(lines[:i_f + 1] + ["4 0 1 2 999"] + lines[i_f + 2:]) + "\n")
    mutate("face_int", "\n".join(lines[:i_f + 1] + ["4 0 1 2 3.5"] + lines[i_f + 2:]) + "\n")
    i_o = lines.index(next(l for l in lines if l.startswith("OWNER")))
    mutate("owner_count", "\n".join(lines[:i_o] + ["OWNER 7"] + lines[i_o + 1:]) + "\n")
    mutate("owner_two", "\n".join(lines[:i_o + 1] + ["0 1"] + lines[i_o + 2:]) + "\n")
    mutate("owner_int", "\n".join(lines[:i_o + 1] + ["zero"] + lines[i_o + 2:]) + "\n")
    i_n = lines.index(next(l for l in lines if l.startswith("NEIGHBOUR")))
    mutate("nbr_exceeds", "\n".join(lines[:i_n] + ["NEIGHBOUR 100000"] + lines[i_n + 1:]) + "\n")
    mutate("nbr_truncated", "\n".join(lines[:i_n + 1] + lines[i_n + 2:]) + "\n")
    i_p = lines.index(next(l for l in lines if l.startswith("PATCHES")))
    mutate("patch_fields", "\n".join(lines[:i_p + 1] + ["lid wall 54"] + lines[i_p + 2:]) + "\n")
    mutate("patch_int", "\n".join(lines[:i_p + 1] + ["lid wall 54 nine"] + lines[i_p + 2:]) + "\n")
    mutate("negative", "POINTS -1\n")
    mutate("comments_ok", "# header comment\n\n" + base.replace("\n", "  # trailing\n", 3))
    mutate("validate", base.replace("walls wall 63 45", "walls wall 63 44"))
    mutate("quote", "POINTS 'x\n")
    errors = {}
    for k, text in bad.items():
        p = os.path.join(tmp, k + ".msh")
        with open(p, "w") as f:
            f.write(text)
        try:
            m = rfile.read_mesh(p)
            errors[k] = ["ok", int(m.n_cells), int(m.n_faces)]
        except Exception as e:  # noqa: BLE001 - record the class and the text
            errors[k] = [type(e).__name__, str(e)]
    js["bad_files"] = bad
    js["bad_errors"] = errors
    # ---------------------------------------------------------------- report
    st = types.SimpleNamespace(
        wall={"total": 12.5, "momentum_assembly": 0.8, "momentum_solve": 1.9,
              "pressure_assembly": 0.7, "pressure_solve": 8.1, "correction": 0.4},
        residual_log=[("bicgstab", "ux", 1, 12, 1.0, 1e-9), ("bicgstab", "uy", 1, 11, 1.0, 1e-9),
                      ("bicgstab", "uz", 1, 0, 0.0, 0.0), ("cg", "p", 1, 140, 1.0, 1e-11),
                      ("cg", "p", 1, 133, 0.3, 1e-11)],
        stage_times={"cg": {"smvp": 5.1, "daxpy": 1.2, "dot": 0.2, "reduction": 0.3,
                            "precond": 0.4, "other": 0.9},
                     "bicgstab": {"smvp": 1.1, "daxpy": 0.5, "dot": 0.1, "reduction": 0.1,
                                  "precond": 0.05, "other": 0.05}},
        ops={"ddt": [0.01, 1], "convection": [0.05, 1], "laplacian": [0.3, 3],
             "gradient": [0.2, 5], "divergence": [0.02, 2]},
        cum_iters={"cg": 273, "bicgstab": 23}, outer=1, converged=True)
    prof = rreport.collect_profile(st)
    js["profile"] = prof
    js["tables"] = {
        "solver_share": rreport.solver_share_table(prof),
        "cg_stage": rreport.cg_stage_table(prof),
        "assembly_norm": rreport.assembly_norm_table(prof),
    }
    js["format_tables"] = rreport.format_tables(prof)
    np.savez_compressed(os.path.join(OUT, "next.npz"), **npz)
    with open(os.path.join(OUT, "next.json"), "w") as f:
        json.dump(js, f, indent=0, sort_keys=True, default=lambda o: o.tolist())
    print("next.npz", os.path.getsize(os.path.join(OUT, "next.npz")) // 1024, "KiB;",
          "next.json", os.path.getsize(os.path.join(OUT, "next.json")) // 1024, "KiB")
    print({k: v[0] for k, v in errors.items()})


if __name__ == "__main__":
    main()
