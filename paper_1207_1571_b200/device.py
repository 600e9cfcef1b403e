"""Device contexts: one libfvb context holds a mesh, its geometry-derived
face tables, a sparsity pattern and the boundary tables resident in HBM.

Contexts for the operator-level API are cached on the mesh (or pattern)
object so repeated operator calls upload the mesh once; the coupled loop
(coupling.RunState) owns a dedicated context that also holds the fields.
"""

import ctypes as C
import os

import numpy as np

from . import _lib
from .errors import FvmError

__all__ = ["DeviceContext", "context_for", "device_index", "bc_table"]


def device_index():
    """CUDA device for new contexts: FVB_DEVICE, else LOCAL_RANK, else 0."""
    return int(os.environ.get("FVB_DEVICE", os.environ.get("LOCAL_RANK", "0")))


class DeviceContext:
    def __init__(self, device=None):
        self.device = device_index() if device is None else int(device)
        h = C.c_void_p()
        _lib.check(_lib.lib.fvb_ctx_create(self.device, C.byref(h)))
        self.h = h
        self.mesh = None
        self.pattern = None
        self.n = 0
        self.nf = self.ni = self.nb = 0
        self.k = 0
        self.nnz_crs = 0
        self.bc_key = [None, None]

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            _lib.lib.fvb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_bytes(self):
        return int(_lib.lib.fvb_ctx_device_bytes(self.h))

    def upload_mesh(self, mesh, geom):
        P = _lib.ptr
        own = _lib.i64(mesh.owner)
        nbr = _lib.i64(mesh.neighbour)
        sf = _lib.f64(geom.face_area)
        smag = _lib.f64(geom.face_area_mag)
        vol = _lib.f64(geom.cell_volume)
        w = _lib.f64(geom.weight)
        d = _lib.f64(geom.d).reshape(-1, 3)
        db = _lib.f64(geom.d_boundary).reshape(-1, 3)
        _lib.check(_lib.lib.fvb_upload_mesh(
            self.h, mesh.n_cells, mesh.n_faces, mesh.n_internal, P(own, _lib.i64p),
            P(nbr, _lib.i64p), P(sf), P(smag), P(vol), P(w), P(d), P(db)))
        self.mesh = mesh
        self.n = mesh.n_cells
        self.nf, self.ni = mesh.n_faces, mesh.n_internal
        self.nb = self.nf - self.ni

    def upload_pattern(self, pattern, faces=True):
        P = _lib.ptr
        I = _lib.i64(pattern.I)
        ds = _lib.i64(pattern.diag_slot)
        fa = _lib.i64(pattern.face_addr) if faces else None
        nfp = len(pattern.face_addr) if faces else 0
        rp = _lib.i64(pattern.crs_row_ptr)
        cc = _lib.i64(pattern.crs_col)
        _lib.check(_lib.lib.fvb_upload_pattern(
            self.h, pattern.n, pattern.k, P(I, _lib.i64p), P(ds, _lib.i64p),
            P(fa, _lib.i64p) if faces else None, nfp, pattern.nnz_crs,
            P(rp, _lib.i64p), P(cc, _lib.i64p)))
        self.pattern = pattern
        if not self.n:
            self.n = pattern.n
        self.k = pattern.k
        self.nnz_crs = pattern.nnz_crs

    def set_bcs(self, field, kinds, patch, fixed, n_patches):
        P = _lib.ptr
        kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
        patch = np.ascontiguousarray(patch, dtype=np.int32)
        fixed = _lib.f64(fixed)
        _lib.check(_lib.lib.fvb_set_bcs(self.h, field, P(kinds, _lib.u8p), P(patch, _lib.i32p),
                                        P(fixed), n_patches))


def bc_table(field, geom, t=0.0, with_speeds=True):
    """Per-boundary-face kind/patch/fixed tables + per-patch speeds at t.

    with_speeds=False skips the speeds (a subdomain's tables: the mass-flow
    area is the whole patch's and comes from the global geometry).

    Encodes the reference's condition classes (fvm.py:37-105) for libfvb;
    the per-patch normal speed of timed / mass-flow inlets is evaluated on
    the host with numpy exactly as apply_bcs does (fvm.py:183-193).
    """
    from . import fvm

    mesh = field.mesh
    ni, nb = mesh.n_internal, mesh.n_boundary
    ncomp = 3 if field.rank == "vector" else 1
    kinds = np.zeros(nb, dtype=np.uint8)
    patch = np.zeros(nb, dtype=np.int32)
    fixed = np.zeros((nb, ncomp)) if ncomp == 3 else np.zeros(nb)
    speeds = np.zeros(max(len(mesh.patches), 1))
    for pi, p in enumerate(mesh.patches):
        bc = field.bcs[p.name]
        sl = slice(p.start - ni, p.start - ni + p.count)
        patch[sl] = pi
        if isinstance(bc, (fvm.FixedValue, fvm.FixedPressure)):
            kinds[sl] = _lib.BC_FIXED
            fixed[sl] = bc.value
        elif isinstance(bc, fvm.NoSlip):
            kinds[sl] = _lib.BC_NO_SLIP
        elif isinstance(bc, fvm.FixedValueTimed):
            kinds[sl] = _lib.BC_SINE
            speeds[pi] = bc.u0 * np.sin(fvm.TWO_PI * bc.freq * t)
        elif isinstance(bc, fvm.FixedMassFlow):
            kinds[sl] = _lib.BC_MASS_FLOW
            if not with_speeds:
                continue
            faces = slice(p.start, p.start + p.count)
            area = float(geom.face_area_mag[faces].sum())
            if area <= 0.0:
                raise FvmError(f"mass-flow patch {p.name!r} has zero area")
            speeds[pi] = bc.rate / (bc.rho * area)
        elif isinstance(bc, fvm.ZeroGradient):
            kinds[sl] = _lib.BC_ZERO_GRADIENT
        elif isinstance(bc, fvm.Empty):
            kinds[sl] = _lib.BC_EMPTY
        else:
            raise FvmError(f"unhandled boundary condition {type(bc).__name__}")
    fixed_soa = np.ascontiguousarray(fixed.T) if ncomp == 3 else fixed
    return kinds, patch, fixed_soa, speeds


def _cache(obj):
    d = obj.__dict__.get("_fvb_contexts")
    if d is None:
        d = {}
        obj.__dict__["_fvb_contexts"] = d
    return d


def context_for(mesh=None, geom=None, pattern=None):
    """Cached operator context for (mesh, geom, pattern)."""
    owner = mesh if mesh is not None else pattern
    key = (id(geom), id(pattern), device_index())
    cache = _cache(owner)
    ctx = cache.get(key)
    if ctx is None:
        ctx = DeviceContext()
        if mesh is not None:
            ctx.upload_mesh(mesh, geom)
        if pattern is not None:
            ctx.upload_pattern(pattern, faces=mesh is not None)
        ctx._keep = (geom, pattern)
        cache[key] = ctx
    return ctx


def set_field_bcs(ctx, field, geom, t=0.0):
    """Install a field's BC tables into slot 0 (vector) / 1 (scalar)."""
    slot = 0 if field.rank == "vector" else 1
    kinds, patch, fixed, speeds = bc_table(field, geom, t)
    ctx.set_bcs(slot, kinds, patch, fixed, len(field.mesh.patches))
    return slot, speeds
