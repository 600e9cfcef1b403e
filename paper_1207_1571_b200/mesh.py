"""Face-addressed polyhedral mesh and its geometry (reference: mesh.py).

Same data model as the reference: owner/neighbour face addressing,
internal faces first with owner < neighbour, boundary faces grouped in
contiguous patches.  ``compute_geometry`` runs the native builder in
libfvb (fvb_geometry), which replays the reference's numpy arithmetic
operation by operation, so every metric array is bit-identical to
fvflow.mesh.compute_geometry (mesh.py:173-278).
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import MeshError

PATCH_KINDS = ("wall", "inlet", "outlet", "empty")
MAX_NONORTHOGONALITY_DEG = 80.0  # mesh.py:24

__all__ = [
    "PATCH_KINDS", "MAX_NONORTHOGONALITY_DEG", "MeshError", "Patch", "Mesh",
    "MeshGeometry", "compute_geometry", "cell_face_adjacency", "cell_neighbour_counts",
    "max_neighbours", "closedness_error",
]


@dataclass
class Patch:
    """Contiguous run of boundary faces sharing a physical role (mesh.py:30-42)."""

    name: str
    kind: str
    start: int
    count: int

    @property
    def faces(self):
        return np.arange(self.start, self.start + self.count)


@dataclass
class Mesh:
    """Polyhedral mesh in owner/neighbour face addressing (mesh.py:45-128)."""

    points: np.ndarray
    face_points: np.ndarray
    face_offsets: np.ndarray
    owner: np.ndarray
    neighbour: np.ndarray
    patches: list = field(default_factory=list)
    n_cells: int = 0

    @property
    def n_faces(self):
        return len(self.owner)

    @property
    def n_internal(self):
        return len(self.neighbour)

    @property
    def n_boundary(self):
        return self.n_faces - self.n_internal

    @property
    def n_points(self):
        return len(self.points)

    def patch_by_name(self, name):
        for p in self.patches:
            if p.name == name:
                return p
        raise KeyError(f"no patch named {name!r}")

    def face_patch_ids(self):
        ids = np.full(self.n_faces, -1, dtype=np.int64)
        for i, p in enumerate(self.patches):
            ids[p.start:p.start + p.count] = i
        return ids

    def validate(self):
        """Structural invariants; MeshError on the first failure (mesh.py:90-128)."""
        nf, ni, nc = self.n_faces, self.n_internal, self.n_cells
        off = np.asarray(self.face_offsets)
        if len(off) != nf + 1:
            raise MeshError("face_offsets length does not match face count")
        counts = np.diff(off)
        if counts.min(initial=3) < 3:
            raise MeshError(f"face {int(np.argmax(counts < 3))} has fewer than 3 points")
        fp = np.asarray(self.face_points)
        if fp.min(initial=0) < 0 or (nf and fp.max() >= self.n_points):
            raise MeshError("face point index out of range")
        own = np.asarray(self.owner)
        if own.min(initial=0) < 0 or (nf and own.max() >= nc):
            raise MeshError("owner cell index out of range")
        if ni:
            nbr = np.asarray(self.neighbour)
            if nbr.min() < 0 or nbr.max() >= nc:
                raise MeshError("neighbour cell index out of range")
            bad = ~(own[:ni] < nbr)
            if bad.any():
                raise MeshError(f"internal face {int(np.argmax(bad))}: owner must be < neighbour")
        covered = np.zeros(nf - ni, dtype=bool)
        for p in self.patches:
            if p.kind not in PATCH_KINDS:
                raise MeshError(f"patch {p.name!r} has unknown kind {p.kind!r}")
            if p.start < ni or p.start + p.count > nf:
                raise MeshError(f"patch {p.name!r} extends outside boundary faces")
            seg = covered[p.start - ni:p.start - ni + p.count]
            if seg.any():
                raise MeshError(f"patch {p.name!r} overlaps another patch")
            seg[:] = True
        if not covered.all():
            raise MeshError("boundary faces not fully covered by patches")
        touched = np.zeros(nc, dtype=bool)
        touched[own] = True
        touched[np.asarray(self.neighbour)] = True
        if not touched.all():
            raise MeshError(f"cell {int(np.argmax(~touched))} has no faces")


@dataclass
class MeshGeometry:
    """Metric quantities per face or cell (mesh.py:131-151)."""

    cell_volume: np.ndarray
    cell_centroid: np.ndarray
    face_area: np.ndarray
    face_area_mag: np.ndarray
    face_centroid: np.ndarray
    d: np.ndarray
    d_mag: np.ndarray
    weight: np.ndarray
    nonorth_deg: np.ndarray
    d_boundary: np.ndarray
    d_boundary_mag: np.ndarray

    @property
    def max_nonorth_deg(self):
        return float(self.nonorth_deg.max()) if len(self.nonorth_deg) else 0.0


def _face_triangles(mesh):
    """The fan triangles fvb_geometry integrates over (reference helper
    mesh.py:154-170): for every loop edge (p_k, p_k+1) of a face, the
    triangle (p_k, p_k+1, seed) with seed the mean of the face's points.
    Returns (a, b, seed per triangle, face per triangle)."""
    off = np.asarray(mesh.face_offsets, dtype=np.int64)
    fp = np.asarray(mesh.face_points, dtype=np.int64)
    npts = off[1:] - off[:-1]
    tri_face = np.repeat(np.arange(len(npts)), npts)
    k = np.arange(len(fp)) - off[tri_face]        # position of the edge in its loop
    succ = off[tri_face] + (k + 1) % npts[tri_face]
    pts = np.asarray(mesh.points, dtype=float)
    seeds = np.add.reduceat(pts[fp], off[:-1], axis=0) / npts[:, None]
    return pts[fp], pts[fp[succ]], seeds[tri_face], tri_face


def compute_geometry(mesh, check=True) -> MeshGeometry:
    """Native fan-triangle / tet-decomposition metrics (fvb_geometry).

    Raises MeshError for zero-area faces, non-positive volumes, inverted
    internal faces and (check=True) faces beyond 80 deg non-orthogonality.
    """
    nf, ni, nc = mesh.n_faces, mesh.n_internal, mesh.n_cells
    nb = nf - ni
    pts = _lib.f64(mesh.points)
    off = _lib.i64(mesh.face_offsets)
    fp = _lib.i64(mesh.face_points)
    own = _lib.i64(mesh.owner)
    nbr = _lib.i64(mesh.neighbour)
    vol = np.empty(nc)
    cc = np.empty((nc, 3))
    sf = np.empty((nf, 3))
    smag = np.empty(nf)
    fc = np.empty((nf, 3))
    d = np.empty((ni, 3))
    dmag = np.empty(ni)
    w = np.empty(ni)
    cosang = np.empty(ni)
    db = np.empty((nb, 3))
    dbmag = np.empty(nb)
    P = _lib.ptr
    rc = _lib.lib.fvb_geometry(
        len(pts), P(pts), nf, P(off, _lib.i64p), P(fp, _lib.i64p), nc, ni,
        P(own, _lib.i64p), P(nbr, _lib.i64p), int(bool(check)), P(vol), P(cc), P(sf),
        P(smag), P(fc), P(d), P(dmag), P(w), P(cosang), P(db), P(dbmag))
    _lib.check(rc, MeshError)
    # numpy's own arccos/degrees for the reported angle (mesh.py:254-255)
    nonorth = np.degrees(np.arccos(cosang))
    if check and ni and nonorth.max() > MAX_NONORTHOGONALITY_DEG:
        bad = int(np.argmax(nonorth))
        raise MeshError(
            f"internal face {bad} is {nonorth[bad]:.1f} deg non-orthogonal "
            f"(limit {MAX_NONORTHOGONALITY_DEG:g})"
        )
    return MeshGeometry(cell_volume=vol, cell_centroid=cc, face_area=sf, face_area_mag=smag,
                        face_centroid=fc, d=d, d_mag=dmag, weight=w, nonorth_deg=nonorth,
                        d_boundary=db, d_boundary_mag=dbmag)


def _cell_face_incidence(mesh):
    """(cell, face, sign, other) of every cell-face incidence, vectorised:
    internal faces twice (owner +1 / neighbour -1), boundary faces once with
    other = -(patch index + 1)."""
    ni, nf = mesh.n_internal, mesh.n_faces
    own = np.asarray(mesh.owner, dtype=np.int64)
    nbr = np.asarray(mesh.neighbour, dtype=np.int64)
    faces = np.arange(nf, dtype=np.int64)
    cell = np.concatenate([own[:ni], nbr, own[ni:]])
    face = np.concatenate([faces[:ni], faces[:ni], faces[ni:]])
    sign = np.concatenate([np.ones(ni, np.int64), -np.ones(ni, np.int64),
                           np.ones(nf - ni, np.int64)])
    other = np.concatenate([nbr, own[:ni], -(np.asarray(mesh.face_patch_ids()[ni:]) + 1)])
    return cell, face, sign, other


def cell_face_adjacency(mesh):
    """Per-cell lists of (face, sign, other) in ascending face order
    (reference mesh.py:281-300); host utility, off the hot path."""
    cell, face, sign, other = _cell_face_incidence(mesh)
    order = np.lexsort((face, cell))
    bounds = np.cumsum(np.bincount(cell, minlength=mesh.n_cells))[:-1]
    rows = zip(face[order].tolist(), sign[order].tolist(), other[order].tolist())
    flat = list(rows)
    out, start = [], 0
    for end in list(bounds) + [len(flat)]:
        out.append(flat[start:end])
        start = end
    return out


def cell_neighbour_counts(mesh):
    """Internal faces per cell (reference mesh.py:303-309)."""
    ni = mesh.n_internal
    both = np.concatenate([np.asarray(mesh.owner[:ni]), np.asarray(mesh.neighbour)])
    return np.bincount(both, minlength=mesh.n_cells)


def max_neighbours(mesh):
    return int(cell_neighbour_counts(mesh).max(initial=0))


def closedness_error(mesh, geom):
    """Largest |sum of outward area vectors| over the cells (reference
    mesh.py:317-327): per component, owner sums minus neighbour sums."""
    ni = mesh.n_internal
    S = np.asarray(geom.face_area)
    acc = np.stack([np.bincount(mesh.owner, weights=S[:, d], minlength=mesh.n_cells)
                    - np.bincount(mesh.neighbour, weights=S[:ni, d], minlength=mesh.n_cells)
                    for d in range(3)], axis=1)
    return float(np.sqrt((acc * acc).sum(axis=1)).max(initial=0.0))
