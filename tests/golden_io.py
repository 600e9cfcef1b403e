"""Load the golden fixtures (tests/golden/*.npz, made by oracle/make_golden.py
from the real reference) into this package's mesh / case objects."""

import ast
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ("cav6", "chan", "duct", "pcav5", "bfs2", "cav20")


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_mesh(g):
    from paper_1207_1571_b200.mesh import Mesh, Patch

    patches = [Patch(str(n), str(k), int(s), int(c)) for n, k, s, c in
               zip(g["patch_names"], g["patch_kinds"], g["patch_start"], g["patch_count"])]
    m = Mesh(points=g["points"].copy(), face_points=g["face_points"].copy(),
             face_offsets=g["face_offsets"].copy(), owner=g["owner"].copy(),
             neighbour=g["neighbour"].copy(), patches=patches, n_cells=int(g["n_cells"]))
    m.validate()
    return m


def golden_config(g):
    from paper_1207_1571_b200.config import BoundarySpec, CaseConfig

    cc = CaseConfig()
    for k in g:
        if k.startswith("cfg_"):
            v = g[k].item()
            setattr(cc, k[4:], v)
    cc.boundary = {str(n): BoundarySpec(u=ast.literal_eval(str(u)), p=ast.literal_eval(str(p)))
                   for n, u, p in zip(g["bc_patches"], g["bc_u"], g["bc_p"])}
    return cc


def golden_case(name):
    from paper_1207_1571_b200.cases import Case

    g = load(name)
    return Case(name, golden_mesh(g), golden_config(g)), g


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
