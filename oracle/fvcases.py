"""CPU ORACLE — test infrastructure only, never product code.

Cavity-case generator for the oracle, so that the CPU baseline of bench.py
(its `--impl reference` arm when the reference package is not installed, and
its `cpu_baseline` leg) can build the benchmark mesh without importing the
product package.  Restates fvflow's `box_mesh` (cases.py:30-128), its
`CaseConfig` defaults (config.py:44-76) and `gen_cavity` (cases.py:164-181):
same points, same canonical face order (internal faces by (owner,
neighbour), boundary faces grouped per patch in patch_sides order, each side
walked with its first free index outermost), same quad loops (counter-
clockwise seen from the owner, so S points owner -> neighbour / outward).
Pinned against the reference's own cavity mesh in tests/golden/cav6.npz
(tests/test_oracle_golden.py).
"""

from types import SimpleNamespace

import numpy as np

# CaseConfig defaults (config.py:44-76), hot-path fields only
CASE_DEFAULTS = dict(nu=1e-6, rho=1000.0, convection="upwind", nonorth_correction=True,
                     limiter=1.0, cg_tol=1e-10, bicgstab_tol=1e-8, max_iters=2000,
                     algorithm="simple", alpha_u=0.7, alpha_p=0.3, n_correctors=2,
                     n_nonorth_correctors=0, dt=1e-3, end_time=1.0, outer_tol=1e-5,
                     max_outer=2000, pressure_ref_cell=0, pressure_ref_value=0.0)


def case_config(**kw):
    d = dict(CASE_DEFAULTS)
    d.update(kw)
    d.setdefault("boundary", {})
    return SimpleNamespace(**d)


def box_mesh(nx, ny, nz, lx, ly, lz, patch_sides):
    """Hexahedral box mesh in the reference's canonical order (cases.py:30-128)."""
    sx, sy = nx + 1, (nx + 1) * (ny + 1)
    x = np.linspace(0.0, lx, nx + 1)
    y = np.linspace(0.0, ly, ny + 1)
    z = np.linspace(0.0, lz, nz + 1)
    # point id = i + (nx+1)(j + (ny+1)k): x fastest, z slowest
    pts = np.empty(((nz + 1) * (ny + 1) * (nx + 1), 3))
    pts[:, 0] = np.tile(x, (ny + 1) * (nz + 1))
    pts[:, 1] = np.tile(np.repeat(y, nx + 1), nz + 1)
    pts[:, 2] = np.repeat(z, (nx + 1) * (ny + 1))

    def P(i, j, k):
        return i + sx * j + sy * k

    # internal faces: every cell's +x, +y, +z neighbour.  With cell id
    # c = i + nx(j + ny k) the three neighbours are c+1 < c+nx < c+nx*ny,
    # so ordering by (cell, direction) is the (owner, neighbour) order.
    k3, j3, i3 = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i3, j3, k3 = i3.ravel(), j3.ravel(), k3.ravel()
    cell = i3 + nx * (j3 + ny * k3)
    parts = []
    for d, ok, step in ((0, i3 < nx - 1, 1), (1, j3 < ny - 1, nx), (2, k3 < nz - 1, nx * ny)):
        i, j, k, c = i3[ok], j3[ok], k3[ok], cell[ok]
        if d == 0:
            q = (P(i + 1, j, k), P(i + 1, j + 1, k), P(i + 1, j + 1, k + 1), P(i + 1, j, k + 1))
        elif d == 1:
            q = (P(i, j + 1, k), P(i, j + 1, k + 1), P(i + 1, j + 1, k + 1), P(i + 1, j + 1, k))
        else:
            q = (P(i, j, k + 1), P(i + 1, j, k + 1), P(i + 1, j + 1, k + 1), P(i, j + 1, k + 1))
        parts.append((3 * c + d, np.stack(q, axis=1), c, c + step))
    key = np.concatenate([p[0] for p in parts])
    order = np.argsort(key, kind="stable")
    quads = [np.concatenate([p[1] for p in parts])[order]]
    owner = [np.concatenate([p[2] for p in parts])[order]]
    nbr = np.concatenate([p[3] for p in parts])[order]

    def side(s):
        # first free index outermost (meshgrid "ij" order of the reference)
        if s[0] == "x":
            a, b = np.meshgrid(np.arange(ny), np.arange(nz), indexing="ij")
            j, k = a.ravel(), b.ravel()
            if s == "x-":
                return np.stack((P(0, j, k), P(0, j, k + 1), P(0, j + 1, k + 1), P(0, j + 1, k)), 1), \
                    nx * (j + ny * k)
            return np.stack((P(nx, j, k), P(nx, j + 1, k), P(nx, j + 1, k + 1), P(nx, j, k + 1)), 1), \
                nx - 1 + nx * (j + ny * k)
        if s[0] == "y":
            a, b = np.meshgrid(np.arange(nx), np.arange(nz), indexing="ij")
            i, k = a.ravel(), b.ravel()
            if s == "y-":
                return np.stack((P(i, 0, k), P(i + 1, 0, k), P(i + 1, 0, k + 1), P(i, 0, k + 1)), 1), \
                    i + nx * ny * k
            return np.stack((P(i, ny, k), P(i, ny, k + 1), P(i + 1, ny, k + 1), P(i + 1, ny, k)), 1), \
                i + nx * (ny - 1 + ny * k)
        a, b = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
        i, j = a.ravel(), b.ravel()
        if s == "z-":
            return np.stack((P(i, j, 0), P(i, j + 1, 0), P(i + 1, j + 1, 0), P(i + 1, j, 0)), 1), \
                i + nx * j
        return np.stack((P(i, j, nz), P(i + 1, j, nz), P(i + 1, j + 1, nz), P(i, j + 1, nz)), 1), \
            i + nx * (j + ny * (nz - 1))

    patches, start, used = [], len(nbr), []
    for name, kind, sides in patch_sides:
        count = 0
        for s in sides:
            if s in used:
                raise ValueError(f"side {s} assigned to two patches")
            used.append(s)
            q, o = side(s)
            quads.append(q)
            owner.append(o)
            count += len(o)
        patches.append(SimpleNamespace(name=name, kind=kind, start=start, count=count))
        start += count
    if sorted(used) != sorted(["x-", "x+", "y-", "y+", "z-", "z+"]):
        raise ValueError("patch sides must cover the six box sides")
    own = np.concatenate(owner).astype(np.int64)
    return SimpleNamespace(points=pts, face_points=np.concatenate(quads).ravel().astype(np.int64),
                           face_offsets=4 * np.arange(len(own) + 1, dtype=np.int64), owner=own,
                           neighbour=nbr.astype(np.int64), patches=patches, n_cells=nx * ny * nz)


def cavity(n, algorithm="piso", dt=None, **kw):
    """gen_cavity(n) (cases.py:164-181): 0.1 m cube, lid y+ at (1,0,0), nu 0.01.
    Returns (mesh, config); dt defaults to 0.1/n (Co = 1, the C2/C5 setting)."""
    mesh = box_mesh(n, n, n, 0.1, 0.1, 0.1,
                    [("lid", "wall", ["y+"]), ("walls", "wall", ["x-", "x+", "y-", "z-", "z+"])])
    cc = case_config(nu=0.01, algorithm=algorithm, dt=0.1 / n if dt is None else dt, **kw)
    cc.boundary = {
        "lid": SimpleNamespace(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
        "walls": SimpleNamespace(u=("no_slip",), p=("zero_gradient",)),
    }
    return mesh, cc
