"""Golden vectors for rhie_chow_flux (fvm.py:499-538) from the REAL reference
(test infrastructure; run in the build container where /root/reference
exists):

    python oracle/make_golden_rhie.py

For every golden case mesh (tests/golden/<case>.npz: its mesh, BCs and the
seeded u / p inputs), the reference applies its BCs at the case's input time
and evaluates rhie_chow_flux with a seeded positive momentum diagonal.  The
cases cover u-empty faces (cav6, cav20, bfs2: 2D), pressure-pinned outlets
with zero-gradient u (chan, duct, bfs2) and perturbed, non-orthogonal cells
(pcav5).  Output: tests/golden/rhie.npz (small).
"""

import ast
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden", "rhie.npz")
REF = "/root/reference/pkg/src"
CASES = ("cav6", "chan", "duct", "pcav5", "bfs2", "cav20")


def a_diag_for(n, seed):
    return np.random.default_rng(seed).uniform(0.5, 3.0, n)


def main():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import fvflow.fvm as rf
    import fvflow.mesh as rmesh
    from golden_io import load

    out = {}
    for k, name in enumerate(CASES):
        g = load(name)
        m = rmesh.Mesh(points=g["points"], face_points=g["face_points"],
                       face_offsets=g["face_offsets"], owner=g["owner"], neighbour=g["neighbour"],
                       patches=[rmesh.Patch(str(a), str(b), int(c), int(d)) for a, b, c, d in
                                zip(g["patch_names"], g["patch_kinds"], g["patch_start"],
                                    g["patch_count"])], n_cells=int(g["n_cells"]))
        geo = rmesh.compute_geometry(m)
        bu = {str(n): rf.bc_from_tuple(ast.literal_eval(str(s))) for n, s in zip(g["bc_patches"], g["bc_u"])}
        bp = {str(n): rf.bc_from_tuple(ast.literal_eval(str(s))) for n, s in zip(g["bc_patches"], g["bc_p"])}
        u = rf.make_vector("u", m, bu)
        p = rf.make_scalar("p", m, bp)
        u.values = g["in_u"].copy()
        p.values = g["in_p"].copy()
        t = float(g["in_t"])
        rf.apply_bcs(u, geo, t)
        rf.apply_bcs(p, geo, t)
        a = a_diag_for(m.n_cells, 100 + k)
        out[f"{name}_a_diag"] = a
        out[f"{name}_flux"] = rf.rhie_chow_flux(u, p, a, geo)
    np.savez_compressed(OUT, **out)
    print(OUT, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
