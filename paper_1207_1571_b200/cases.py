"""Synthetic cases for the benchmark and the parity tests (reference: cases.py).

``box_mesh`` emits the reference's canonical hexahedral box numbering —
point (i, j, k) -> i + (nx+1)(j + (ny+1)k), cell (i, j, k) -> i + nx(j + ny k),
internal faces ordered by (owner, neighbour), boundary faces grouped per
patch in side order — so a mesh built here is array-identical to
fvflow.cases.box_mesh (checked by tests/test_cases.py against golden
fixtures).  Two generators the reference lacks implement SURVEY.md
Appendix B: the masked-box backward-facing step (config C3) and the
perturbed + renumbered cavity (config C4).
"""

from dataclasses import dataclass

import numpy as np

from .config import BoundarySpec, CaseConfig
from .mesh import Mesh, Patch

SIDES = ("x-", "x+", "y-", "y+", "z-", "z+")

__all__ = ["box_counts", "box_mesh", "Case", "gen_cavity", "gen_channel", "gen_skewed_duct",
           "gen_backward_step", "perturbed_cavity", "GENERATORS"]


def box_counts(nx, ny, nz):
    """(cells, faces) of an nx x ny x nz box (cases.py:22-27)."""
    cells = nx * ny * nz
    internal = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
    return cells, internal + 2 * (ny * nz + nx * nz + nx * ny)


def _side(nx, ny, nz, side):
    """Outward quads and owner cells of one box side (reference orientation)."""
    px, pxy = nx + 1, (nx + 1) * (ny + 1)
    axis, hi = "xyz".index(side[0]), side[1] == "+"
    if axis == 0:
        a, b = np.meshgrid(np.arange(ny), np.arange(nz), indexing="ij")
        j, k = a.ravel(), b.ravel()
        i = np.full_like(j, nx if hi else 0)
        base = i + px * j + pxy * k
        if hi:
            quad = [base, base + px, base + px + pxy, base + pxy]
        else:
            quad = [base, base + pxy, base + px + pxy, base + px]
        own = (nx - 1 if hi else 0) + nx * (j + ny * k)
    elif axis == 1:
        a, b = np.meshgrid(np.arange(nx), np.arange(nz), indexing="ij")
        i, k = a.ravel(), b.ravel()
        j = ny if hi else 0
        base = i + px * j + pxy * k
        if hi:
            quad = [base, base + pxy, base + 1 + pxy, base + 1]
        else:
            quad = [base, base + 1, base + 1 + pxy, base + pxy]
        own = i + nx * ((ny - 1 if hi else 0) + ny * k)
    else:
        a, b = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
        i, j = a.ravel(), b.ravel()
        k = nz if hi else 0
        base = i + px * j + pxy * k
        if hi:
            quad = [base, base + 1, base + 1 + px, base + px]
        else:
            quad = [base, base + px, base + 1 + px, base + 1]
        own = i + nx * (j + ny * (nz - 1 if hi else 0))
    return np.stack(quad, axis=1), own


def box_mesh(nx, ny, nz, lx, ly, lz, patch_sides, shear_xy=0.0) -> Mesh:
    """Hexahedral box [0,lx]x[0,ly]x[0,lz] (cases.py:30-161)."""
    xs = np.linspace(0.0, lx, nx + 1)
    ys = np.linspace(0.0, ly, ny + 1)
    zs = np.linspace(0.0, lz, nz + 1)
    npt = (nx + 1) * (ny + 1) * (nz + 1)
    pid = np.arange(npt)
    pi, pj, pk = pid % (nx + 1), (pid // (nx + 1)) % (ny + 1), pid // ((nx + 1) * (ny + 1))
    pts = np.stack([xs[pi], ys[pj], zs[pk]], axis=1)
    if shear_xy:
        pts[:, 0] += shear_xy * pts[:, 1]
    px, pxy = nx + 1, (nx + 1) * (ny + 1)
    # internal faces in (owner, neighbour) order: per owner cell the x-, y-,
    # then z-neighbour (their neighbour indices ascend in that order)
    c = np.arange(nx * ny * nz)
    ci, cj, ck = c % nx, (c // nx) % ny, c // (nx * ny)
    base = ci + px * cj + pxy * ck  # point (i, j, k) of the cell's low corner
    has = np.stack([ci < nx - 1, cj < ny - 1, ck < nz - 1], axis=1)
    quads_dir = [
        np.stack([base + 1, base + 1 + px, base + 1 + px + pxy, base + 1 + pxy], axis=1),
        np.stack([base + px, base + px + pxy, base + 1 + px + pxy, base + 1 + px], axis=1),
        np.stack([base + pxy, base + 1 + pxy, base + 1 + px + pxy, base + px + pxy], axis=1),
    ]
    step = np.array([1, nx, nx * ny])
    sel = has.ravel()
    own_i = np.repeat(c, 3)[sel]
    nbr_i = (c[:, None] + step[None, :]).ravel()[sel]
    q_i = np.stack(quads_dir, axis=1).reshape(-1, 4)[sel]
    bq, bo, patches = [], [], []
    start = len(own_i)
    seen = set()
    for name, kind, sides in patch_sides:
        cnt = 0
        for s in sides:
            if s in seen:
                raise ValueError(f"side {s} assigned to two patches")
            seen.add(s)
            q, o = _side(nx, ny, nz, s)
            bq.append(q)
            bo.append(o)
            cnt += len(o)
        patches.append(Patch(name=name, kind=kind, start=start, count=cnt))
        start += cnt
    if seen != set(SIDES):
        raise ValueError(f"sides not covered by patches: {sorted(set(SIDES) - seen)}")
    quads = np.concatenate([q_i] + bq)
    owners = np.concatenate([own_i] + bo)
    mesh = Mesh(points=pts, face_points=quads.ravel().astype(np.int64),
                face_offsets=4 * np.arange(len(owners) + 1, dtype=np.int64),
                owner=owners.astype(np.int64), neighbour=nbr_i.astype(np.int64),
                patches=patches, n_cells=nx * ny * nz)
    mesh.validate()
    return mesh


@dataclass
class Case:
    name: str
    mesh: Mesh
    config: CaseConfig


def gen_cavity(n) -> Case:
    """Lid-driven cubic cavity, 0.1 m, lid (y+) at 1 m/s, Re 10 (cases.py:173-190)."""
    mesh = box_mesh(n, n, n, 0.1, 0.1, 0.1,
                    [("lid", "wall", ["y+"]), ("walls", "wall", ["x-", "x+", "y-", "z-", "z+"])])
    cfg = CaseConfig()
    cfg.nu = 0.01
    cfg.algorithm = "simple"
    cfg.boundary = {
        "lid": BoundarySpec(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
        "walls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
    }
    return Case(name=f"cavity{n}", mesh=mesh, config=cfg)


_CHANNEL_PATCHES = [("inlet", "inlet", ["x-"]), ("outlet", "outlet", ["x+"]),
                    ("walls", "wall", ["y-", "y+"]), ("frontAndBack", "empty", ["z-", "z+"])]


def gen_channel(nx, ny, length=0.16, height=0.02) -> Case:
    """2D channel with a sine-pulsed inlet, PISO preset (cases.py:193-223)."""
    mesh = box_mesh(nx, ny, 1, length, height, height / ny, _CHANNEL_PATCHES)
    cfg = CaseConfig()
    cfg.nu = 3.3e-6
    cfg.algorithm = "piso"
    cfg.dt = 1e-4
    cfg.end_time = 0.5
    cfg.boundary = {
        "inlet": BoundarySpec(u=("sine_inlet", 0.01, 0.5), p=("zero_gradient",)),
        "outlet": BoundarySpec(u=("zero_gradient",), p=("fixed_value", 0.0)),
        "walls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
        "frontAndBack": BoundarySpec(u=("empty",), p=("empty",)),
    }
    return Case(name=f"channel{nx}x{ny}", mesh=mesh, config=cfg)


def gen_skewed_duct(nx, ny, skew_deg, length=1.0, height=1.0) -> Case:
    """Sheared duct, x-normal faces skew_deg non-orthogonal (cases.py:226-253)."""
    if not 0.0 <= skew_deg <= 45.0:
        raise ValueError("skew_deg must be in [0, 45]")
    mesh = box_mesh(nx, ny, 1, length, height, height / ny, _CHANNEL_PATCHES,
                    shear_xy=np.tan(np.radians(skew_deg)))
    cfg = CaseConfig()
    cfg.nu = 3e-6
    cfg.algorithm = "simple"
    cfg.n_nonorth_correctors = 1
    cfg.boundary = {
        "inlet": BoundarySpec(u=("mass_flow", 9.975e-4, 1000.0), p=("zero_gradient",)),
        "outlet": BoundarySpec(u=("zero_gradient",), p=("fixed_value", 0.0)),
        "walls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
        "frontAndBack": BoundarySpec(u=("empty",), p=("empty",)),
    }
    return Case(name=f"duct{nx}x{ny}s{skew_deg:g}", mesh=mesh, config=cfg)


def _assemble(pts, quads, own, nbr, nc, groups):
    """Mesh from internal faces (sorted here) + ordered boundary groups."""
    ni = len(nbr)
    order = np.lexsort((nbr, own[:ni]))
    q_i, o_i, n_i = quads[:ni][order], own[:ni][order], nbr[order]
    bq, bo, patches = [], [], []
    start = ni
    for name, kind, q, o in groups:
        bq.append(q)
        bo.append(o)
        patches.append(Patch(name=name, kind=kind, start=start, count=len(o)))
        start += len(o)
    fq = np.concatenate([q_i] + bq)
    fo = np.concatenate([o_i] + bo)
    mesh = Mesh(points=pts, face_points=fq.ravel().astype(np.int64),
                face_offsets=4 * np.arange(len(fo) + 1, dtype=np.int64),
                owner=fo.astype(np.int64), neighbour=n_i.astype(np.int64),
                patches=patches, n_cells=nc)
    mesh.validate()
    return mesh


def perturbed_cavity(n, seed=1207, amp=0.2) -> Case:
    """Config C4: gen_cavity(n) with interior points
    shifted by U(-amp h, amp h)^3, cells renumbered by a random permutation,
    internal faces re-oriented owner < neighbour and re-sorted."""
    base = gen_cavity(n)
    m = base.mesh
    h = 0.1 / n
    rng = np.random.default_rng(seed)
    pts = m.points.copy()
    on_face = ((np.abs(pts) < 1e-12) | (np.abs(pts - 0.1) < 1e-12)).any(axis=1)
    inner = np.nonzero(~on_face)[0]
    pts[inner] += rng.uniform(-amp * h, amp * h, size=(len(inner), 3))
    perm = rng.permutation(m.n_cells)
    ni = m.n_internal
    quads = m.face_points.reshape(-1, 4).copy()
    own = perm[m.owner]
    nbr = perm[m.neighbour]
    swap = own[:ni] > nbr
    lo = np.where(swap, nbr, own[:ni])
    hi = np.where(swap, own[:ni], nbr)
    qi = quads[:ni]
    qi[swap] = qi[swap][:, ::-1]
    own_all = np.concatenate([lo, own[ni:]])
    allq = np.concatenate([qi, quads[ni:]])
    groups = []
    for p in m.patches:
        sl = slice(p.start, p.start + p.count)
        groups.append((p.name, p.kind, allq[sl], own_all[sl]))
    mesh = _assemble(pts, allq, own_all, hi, m.n_cells, groups)
    cfg = base.config
    cfg.algorithm = "piso"
    cfg.dt = 0.1 / n
    cfg.n_nonorth_correctors = 1
    return Case(name=f"pcavity{n}", mesh=mesh, config=cfg)


def gen_backward_step(nh, U=1.0) -> Case:
    """Config C3: laminar backward-facing step, Re_h 200.

    Step height h = 0.01 m = nh cells; inlet height h, outlet height 2h,
    upstream 5h, downstream 30h; one cell thick with empty front/back.
    """
    nx, ny = 35 * nh, 2 * nh
    box = box_mesh(nx, ny, 1, 0.35, 0.02, 0.01 / nh,
                   [("all", "wall", list(SIDES))])
    nc0 = box.n_cells
    ci, cj = np.arange(nc0) % nx, (np.arange(nc0) // nx) % ny
    keep = ~((ci < 5 * nh) & (cj < nh))
    new_id = np.full(nc0, -1, dtype=np.int64)
    new_id[keep] = np.arange(keep.sum())
    quads = box.face_points.reshape(-1, 4)
    ni0 = box.n_internal
    own0 = box.owner
    nbr0 = np.concatenate([box.neighbour, np.full(box.n_faces - ni0, -1)])
    ko = keep[own0]
    kn = np.where(nbr0 >= 0, keep[np.maximum(nbr0, 0)], False)
    internal = ko & kn
    bnd_from_own = ko & ~kn
    bnd_from_nbr = ~ko & kn
    iq = quads[internal]
    io, inb = new_id[own0[internal]], new_id[nbr0[internal]]
    bsel = np.nonzero(bnd_from_own | bnd_from_nbr)[0]
    bq = quads[bsel].copy()
    flip = bnd_from_nbr[bsel]
    bq[flip] = bq[flip][:, ::-1]
    bo = np.where(flip, new_id[np.maximum(nbr0[bsel], 0)], new_id[own0[bsel]])
    ctr = box.points[bq].mean(axis=1)
    dz = 0.01 / nh
    is_fb = (np.abs(ctr[:, 2]) < 1e-12) | (np.abs(ctr[:, 2] - dz) < 1e-12)
    is_in = ~is_fb & (np.abs(ctr[:, 0]) < 1e-12)
    is_out = ~is_fb & (np.abs(ctr[:, 0] - 0.35) < 1e-12)
    is_wall = ~(is_fb | is_in | is_out)
    groups = [(nm, kd, bq[msk], bo[msk]) for nm, kd, msk in (
        ("inlet", "inlet", is_in), ("outlet", "outlet", is_out), ("walls", "wall", is_wall),
        ("frontAndBack", "empty", is_fb))]
    allq = np.concatenate([iq, bq])
    allo = np.concatenate([io, bo])
    mesh = _assemble(box.points, allq, allo, inb, int(keep.sum()), groups)
    cfg = CaseConfig()
    cfg.nu = U * 0.01 / 200.0
    cfg.algorithm = "simple"
    cfg.boundary = {
        "inlet": BoundarySpec(u=("fixed_value", (U, 0.0, 0.0)), p=("zero_gradient",)),
        "outlet": BoundarySpec(u=("zero_gradient",), p=("fixed_value", 0.0)),
        "walls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
        "frontAndBack": BoundarySpec(u=("empty",), p=("empty",)),
    }
    return Case(name=f"bfs{nh}", mesh=mesh, config=cfg)


GENERATORS = {
    "cavity": gen_cavity,
    "channel": gen_channel,
    "skewed-duct": gen_skewed_duct,
    "backward-step": gen_backward_step,
    "perturbed-cavity": perturbed_cavity,
}
