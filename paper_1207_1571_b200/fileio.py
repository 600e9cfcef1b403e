"""Mesh file I/O in the reference's ASCII format (reference: fileio.py:50-185).

Parsing and writing run natively in libfvb (csrc/meshio.cpp): the same five
sections, comment and blank-line rules, line-numbered MeshFileError texts
and "%.17g" floats, so a file written here is byte-identical to one written
by fvflow and a write/read cycle is exact.  The VTK writer, line sampling
and CSV helpers of the reference are host post-processing outside the hot
path and are not rebuilt.
"""

import ctypes as C
import os

import numpy as np

from . import _lib
from .errors import MeshFileError
from .mesh import Mesh, Patch

__all__ = ["MeshFileError", "read_mesh", "write_mesh"]


def write_mesh(mesh, path):
    """Write `mesh` to `path` (fileio.py:50-65)."""
    P = _lib.ptr
    pts = _lib.f64(mesh.points).reshape(-1, 3)
    off = _lib.i64(mesh.face_offsets)
    fp = _lib.i64(mesh.face_points)
    own = _lib.i64(mesh.owner)
    nbr = _lib.i64(mesh.neighbour)
    names = (C.c_char_p * max(len(mesh.patches), 1))(*[p.name.encode() for p in mesh.patches])
    kinds = (C.c_char_p * max(len(mesh.patches), 1))(*[p.kind.encode() for p in mesh.patches])
    start = _lib.i64([p.start for p in mesh.patches])
    count = _lib.i64([p.count for p in mesh.patches])
    _lib.check(_lib.lib.fvb_mesh_write(
        os.fsencode(path), len(pts), P(pts), mesh.n_faces, P(off, _lib.i64p), P(fp, _lib.i64p),
        P(own, _lib.i64p), mesh.n_internal, P(nbr, _lib.i64p), len(mesh.patches), names, kinds,
        P(start, _lib.i64p), P(count, _lib.i64p)))


def read_mesh(path) -> Mesh:
    """Parse a mesh file and validate it (fileio.py:106-185)."""
    h = C.c_void_p()
    counts = np.zeros(5, dtype=np.int64)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_mesh_read(os.fsencode(path), C.byref(h), P(counts, _lib.i64p)))
    try:
        n_points, n_faces, n_fp, n_internal, n_patches = (int(c) for c in counts)
        points = np.empty((n_points, 3))
        off = np.empty(n_faces + 1, dtype=np.int64)
        fp = np.empty(n_fp, dtype=np.int64)
        owner = np.empty(n_faces, dtype=np.int64)
        nbr = np.empty(n_internal, dtype=np.int64)
        ps = np.empty(max(n_patches, 1), dtype=np.int64)
        pc = np.empty(max(n_patches, 1), dtype=np.int64)
        names = C.create_string_buffer(256 * max(n_patches, 1))
        kinds = C.create_string_buffer(256 * max(n_patches, 1))
        _lib.check(_lib.lib.fvb_mesh_read_take(
            h, P(points), P(off, _lib.i64p), P(fp, _lib.i64p), P(owner, _lib.i64p),
            P(nbr, _lib.i64p), P(ps, _lib.i64p), P(pc, _lib.i64p), names, kinds))
    finally:
        _lib.lib.fvb_mesh_read_free(h)
    raw_n, raw_k = names.raw, kinds.raw
    patches = [Patch(name=raw_n[256 * i:256 * (i + 1)].split(b"\0", 1)[0].decode(),
                     kind=raw_k[256 * i:256 * (i + 1)].split(b"\0", 1)[0].decode(),
                     start=int(ps[i]), count=int(pc[i])) for i in range(n_patches)]
    n_cells = int(owner.max()) + 1 if n_faces else 0
    if n_internal and int(nbr.max()) + 1 > n_cells:
        n_cells = int(nbr.max()) + 1
    mesh = Mesh(points=points, face_points=fp, face_offsets=off, owner=owner, neighbour=nbr,
                patches=patches, n_cells=n_cells)
    mesh.validate()
    return mesh
