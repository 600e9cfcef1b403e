"""Finite-volume fields, boundary conditions and discrete operators
(reference: fvm.py), executed by the libfvb kernels.

Same convention as the reference: an operator adds coeff*M into the
system matrix and coeff*s into the right-hand side for a term discretised
as M*phi - s; the Laplacian uses the over-relaxed split S = a d + k with a
deferred explicit correction gamma k.(grad phi)_f.  The device kernels
replay the reference's accumulation order per matrix row (owner faces
ascending, then neighbour faces, then boundary faces), including its
vector-rhs quirk where a cell with several value-BC faces keeps only the
highest-index face's Dirichlet/convection source (fvm.py:378, 473).
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import context_for, set_field_bcs
from .errors import FvmError

TWO_PI = 2.0 * np.pi

__all__ = [
    "FvmError", "BoundaryCondition", "FixedValue", "FixedValueTimed", "ZeroGradient", "NoSlip",
    "FixedMassFlow", "FixedPressure", "Empty", "bc_from_tuple", "is_value_bc", "SchemeConfig",
    "Field", "make_scalar", "make_vector", "apply_bcs", "interpolate_to_faces",
    "interpolate_cell_values", "face_divergence", "gauss_gradient", "LinearSystem",
    "LaplacianFaceData", "laplacian", "laplacian_face_flux", "divergence_convection",
    "ddt_euler", "rhie_chow_flux", "TWO_PI",
]


class BoundaryCondition:
    pass


@dataclass
class FixedValue(BoundaryCondition):
    value: object


@dataclass
class FixedValueTimed(BoundaryCondition):
    """Inflow along the inward normal at speed u0 sin(2 pi freq t)."""

    u0: float
    freq: float


@dataclass
class ZeroGradient(BoundaryCondition):
    pass


@dataclass
class NoSlip(BoundaryCondition):
    pass


@dataclass
class FixedMassFlow(BoundaryCondition):
    rate: float
    rho: float


@dataclass
class FixedPressure(BoundaryCondition):
    value: float


@dataclass
class Empty(BoundaryCondition):
    pass


def _fixed_value(a):
    return FixedValue(value=np.asarray(a[0]) if len(a) == 1 else float(a[0]))


_TAGS = {
    "fixed_value": _fixed_value,
    "sine_inlet": lambda a: FixedValueTimed(u0=float(a[0]), freq=float(a[1])),
    "mass_flow": lambda a: FixedMassFlow(rate=float(a[0]), rho=float(a[1])),
    "no_slip": lambda a: NoSlip(),
    "zero_gradient": lambda a: ZeroGradient(),
    "empty": lambda a: Empty(),
}


def bc_from_tuple(spec):
    """Condition from a config tuple such as ("fixed_value", (1, 0, 0)) (fvm.py:92-100)."""
    tag, args = spec[0], spec[1:]
    if tag not in _TAGS:
        raise FvmError(f"unknown boundary condition tag {tag!r}")
    bc = _TAGS[tag](args)
    if isinstance(bc, FixedMassFlow) and bc.rho <= 0:
        raise FvmError("mass-flow condition needs rho > 0")
    return bc


def is_value_bc(bc):
    return isinstance(bc, (FixedValue, FixedValueTimed, NoSlip, FixedMassFlow, FixedPressure))


@dataclass
class SchemeConfig:
    convection: str = "upwind"
    nonorth_correction: bool = True
    limiter: float = 1.0

    def __post_init__(self):
        if self.convection not in ("upwind", "linear"):
            raise FvmError(f"unknown convection scheme {self.convection!r}")
        if not 0.0 <= self.limiter <= 1.0:
            raise FvmError("limiter must lie in [0, 1]")


@dataclass
class Field:
    """Cell-centred unknown with one condition per patch (fvm.py:125-158)."""

    name: str
    mesh: object
    values: np.ndarray
    bcs: dict
    boundary: np.ndarray = None
    face_flux: np.ndarray = None

    def __post_init__(self):
        names = {p.name for p in self.mesh.patches}
        if set(self.bcs) != names:
            missing = names - set(self.bcs)
            extra = set(self.bcs) - names
            raise FvmError(f"field {self.name!r}: boundary coverage mismatch "
                           f"(missing {sorted(missing)}, unknown {sorted(extra)})")
        if len(self.values) != self.mesh.n_cells:
            raise FvmError(f"field {self.name!r}: cell value count mismatch")
        if self.boundary is None:
            self.boundary = np.zeros((self.mesh.n_boundary,) + np.shape(self.values)[1:])

    @property
    def rank(self):
        return "vector" if np.ndim(self.values) == 2 else "scalar"


def make_scalar(name, mesh, bcs, init=0.0):
    return Field(name, mesh, np.full(mesh.n_cells, float(init)), dict(bcs))


def make_vector(name, mesh, bcs, init=(0.0, 0.0, 0.0)):
    return Field(name, mesh, np.tile(np.asarray(init, dtype=float), (mesh.n_cells, 1)), dict(bcs))


# ------------------------------------------------------------- plumbing

def _soa(a, ncomp):
    a = np.asarray(a, dtype=float)
    return np.ascontiguousarray(a.T) if ncomp == 3 else np.ascontiguousarray(a)


def _aos(a, ncomp, m):
    return np.ascontiguousarray(a.reshape(ncomp, m).T) if ncomp == 3 else a


def _ncomp(field):
    return 3 if field.rank == "vector" else 1


def _mesh_ctx(mesh, geom=None, pattern=None):
    if geom is None:
        cache = mesh.__dict__.get("_fvb_contexts") or {}
        for ctx in cache.values():
            if ctx.mesh is not None and (pattern is None or ctx.pattern is pattern):
                return ctx, ctx._keep[0]
        from .mesh import compute_geometry

        geom = mesh.__dict__.get("_fvb_geom") or compute_geometry(mesh, check=False)
        mesh.__dict__["_fvb_geom"] = geom
    return context_for(mesh, geom, pattern), geom


def _boundary_masks(field):
    """(value, zero-gradient, empty) masks over boundary faces (fvm.py:200-217)."""
    mesh = field.mesh
    ni, nb = mesh.n_internal, mesh.n_boundary
    value = np.zeros(nb, dtype=bool)
    zerog = np.zeros(nb, dtype=bool)
    empty = np.zeros(nb, dtype=bool)
    for p in mesh.patches:
        bc = field.bcs[p.name]
        sl = slice(p.start - ni, p.start - ni + p.count)
        if isinstance(bc, Empty):
            empty[sl] = True
        elif is_value_bc(bc):
            value[sl] = True
        else:
            zerog[sl] = True
    return value, zerog, empty


# ------------------------------------------------------------ operators

def apply_bcs(field, geom, t=0.0):
    """Refresh boundary face values at time t (fvm.py:170-197) on the device."""
    ctx, geom = _mesh_ctx(field.mesh, geom)
    slot, speeds = set_field_bcs(ctx, field, geom, t)
    nc = _ncomp(field)
    vals = _soa(field.values, nc)
    out = np.empty(nc * field.mesh.n_boundary)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_apply_bcs(ctx.h, slot, P(vals), P(_lib.f64(speeds)), P(out)),
               FvmError)
    field.boundary = _aos(out, nc, field.mesh.n_boundary)


def interpolate_to_faces(field, geom):
    """Linear interpolation; value-BC faces take the BC value, others the owner (fvm.py:220-239)."""
    ctx, geom = _mesh_ctx(field.mesh, geom)
    slot, _ = set_field_bcs(ctx, field, geom)
    nc = _ncomp(field)
    vals = _soa(field.values, nc)
    bnd = _soa(field.boundary, nc)
    out = np.empty(nc * field.mesh.n_faces)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_interpolate(ctx.h, slot, nc, P(vals), P(bnd), P(out)), FvmError)
    return _aos(out, nc, field.mesh.n_faces)


def interpolate_cell_values(mesh, geom, values):
    """Interpolation of a raw cell array, owner copy on boundary (fvm.py:242-247)."""
    ctx, geom = _mesh_ctx(mesh, geom)
    vals = _lib.f64(values)
    out = np.empty(mesh.n_faces)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_interpolate(ctx.h, -1, 1, P(vals), None, P(out)), FvmError)
    return out


def face_divergence(mesh, face_flux):
    """Per-cell signed sum of face fluxes (fvm.py:250-255)."""
    ctx, _ = _mesh_ctx(mesh)
    fl = _lib.f64(face_flux)
    out = np.empty(mesh.n_cells)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_divergence(ctx.h, P(fl), P(out)), FvmError)
    return out


def gauss_gradient(field, geom):
    """Gauss gradient: (n, 3) for scalars, (n, 3, 3) with grad[c,i,d] = du_i/dx_d (fvm.py:258-275)."""
    ctx, geom = _mesh_ctx(field.mesh, geom)
    slot, _ = set_field_bcs(ctx, field, geom)
    nc = _ncomp(field)
    n = field.mesh.n_cells
    vals = _soa(field.values, nc)
    bnd = _soa(field.boundary, nc)
    out = np.empty(nc * 3 * n)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_gradient(ctx.h, slot, nc, P(vals), P(bnd), P(out)), FvmError)
    g = out.reshape(nc, 3, n).transpose(2, 0, 1)
    return np.ascontiguousarray(g[:, 0, :] if nc == 1 else g)


@dataclass
class LinearSystem:
    """A x = rhs under assembly; rhs is (n,) or (n, 3) (fvm.py:281-295)."""

    A: object
    rhs: np.ndarray

    @classmethod
    def zeros(cls, pattern, rank="scalar"):
        from .sparse import HybridMatrix

        shape = (pattern.n,) if rank == "scalar" else (pattern.n, 3)
        return cls(A=HybridMatrix.zeros(pattern), rhs=np.zeros(shape))

    @property
    def pattern(self):
        return self.A.pattern


@dataclass
class LaplacianFaceData:
    """Per-face coef = gamma |S|^2/(S.d) and frozen explicit correction (fvm.py:320-332)."""

    coef: np.ndarray
    corr: np.ndarray


def _face_gamma(gamma, n_faces):
    g = np.asarray(gamma, dtype=float)
    if g.ndim == 0:
        return float(g), None
    if g.shape != (n_faces,):
        raise FvmError("gamma must be a scalar or a per-face array")
    return 0.0, np.ascontiguousarray(g)


def _sys_arrays(sys, nc):
    V = np.ascontiguousarray(sys.A.V, dtype=float)
    crs = np.ascontiguousarray(sys.A.crs_val, dtype=float)
    rhs = _soa(sys.rhs, nc).copy()
    return V, crs, rhs


def _sys_store(sys, V, crs, rhs, nc):
    sys.A.V[...] = V
    sys.A.crs_val[...] = crs
    sys.rhs[...] = _aos(rhs, nc, sys.pattern.n)


def laplacian(sys, gamma, field, geom, scheme, coeff=1.0):
    """Add coeff*laplacian(gamma, phi) to the system (fvm.py:335-408); returns face data."""
    mesh = field.mesh
    gs, gf = _face_gamma(gamma, mesh.n_faces)
    if geom is not None:
        # the reference validates the geometry object it is handed
        # (fvm.py:353-354, 369-371), which may differ from the context's
        # device copy (a caller can edit it): same checks, same messages
        zero = np.flatnonzero(np.asarray(geom.d_mag) == 0.0)
        if zero.size:
            raise FvmError(f"coincident centroids at internal face {int(zero[0])}")
        value_m, _, _ = _boundary_masks(field)
        bad = np.flatnonzero(value_m & (np.asarray(geom.d_boundary_mag) == 0.0))
        if bad.size:
            raise FvmError(f"coincident centroids at boundary face {int(bad[0]) + mesh.n_internal}")
    ctx, geom = _mesh_ctx(mesh, geom, sys.pattern)
    slot, _ = set_field_bcs(ctx, field, geom)
    nc = _ncomp(field)
    V, crs, rhs = _sys_arrays(sys, nc)
    vals = _soa(field.values, nc)
    bnd = _soa(field.boundary, nc)
    coef = np.empty(mesh.n_faces)
    corr = np.empty(nc * mesh.n_faces)
    P = _lib.ptr
    rc = _lib.lib.fvb_op_laplacian(
        ctx.h, slot, nc, P(V), P(crs), P(rhs), gs, P(gf) if gf is not None else None, P(vals),
        P(bnd), int(bool(scheme.nonorth_correction)), float(scheme.limiter), float(coeff),
        P(coef), P(corr))
    _lib.check(rc, FvmError)
    _sys_store(sys, V, crs, rhs, nc)
    return LaplacianFaceData(coef=coef, corr=_aos(corr, nc, mesh.n_faces))


def laplacian_face_flux(fdata, field):
    """Face fluxes of a recorded unit-coeff Laplacian (fvm.py:411-429)."""
    mesh = field.mesh
    ctx, geom = _mesh_ctx(mesh)
    slot, _ = set_field_bcs(ctx, field, geom)
    nc = _ncomp(field)
    coef = _lib.f64(fdata.coef)
    corr = _soa(fdata.corr, nc)
    vals = _soa(field.values, nc)
    bnd = _soa(field.boundary, nc)
    out = np.empty(nc * mesh.n_faces)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_laplacian_flux(ctx.h, slot, nc, P(coef), P(corr), P(vals),
                                              P(bnd), P(out)), FvmError)
    return _aos(out, nc, mesh.n_faces)


def divergence_convection(sys, flux, field, scheme, geom=None, coeff=1.0):
    """Add coeff*div(flux, phi), implicit in phi (fvm.py:432-482)."""
    mesh = field.mesh
    if flux is None or len(flux) != mesh.n_faces:
        raise FvmError("divergence needs a flux value for every face")
    if scheme.convection != "upwind" and geom is None:
        raise FvmError("linear convection needs the mesh geometry")
    ctx, geom = _mesh_ctx(mesh, geom, sys.pattern)
    slot, _ = set_field_bcs(ctx, field, geom)
    nc = _ncomp(field)
    V, crs, rhs = _sys_arrays(sys, nc)
    fl = _lib.f64(flux)
    bnd = _soa(field.boundary, nc)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_convection(ctx.h, slot, nc, P(V), P(crs), P(rhs), P(fl), P(bnd),
                                          0 if scheme.convection == "upwind" else 1,
                                          float(coeff)), FvmError)
    _sys_store(sys, V, crs, rhs, nc)


def ddt_euler(sys, field, old_values, dt, geom, coeff=1.0):
    """Implicit Euler: V/dt on the diagonal, V phi_old/dt as source (fvm.py:485-496)."""
    if dt <= 0.0:
        raise FvmError("dt must be positive")
    mesh = field.mesh
    ctx, geom = _mesh_ctx(mesh, geom, sys.pattern)
    nc = _ncomp(field)
    V, crs, rhs = _sys_arrays(sys, nc)
    old = _soa(old_values, nc)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_ddt(ctx.h, nc, P(V), P(rhs), P(old), float(dt), float(coeff)),
               FvmError)
    sys.A.V[...] = V
    sys.rhs[...] = _aos(rhs, nc, sys.pattern.n)


def rhie_chow_flux(u, p_field, a_diag, geom):
    """Face volume fluxes with Rhie-Chow pressure smoothing (fvm.py:499-538):
    S . u_f, less D_f a_f [(p_N - p_O) - (grad p)_f . d] on internal faces
    (D = V / a_diag interpolated to the face) and on boundary faces where p
    is pinned and u is not; 0 where u is empty.  One gradient and one face
    kernel on the device (fvb_op_rhie_chow)."""
    mesh = u.mesh
    ctx, geom = _mesh_ctx(mesh, geom)
    set_field_bcs(ctx, u, geom)
    set_field_bcs(ctx, p_field, geom)
    a = _lib.f64(a_diag)
    out = np.empty(mesh.n_faces)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_rhie_chow(
        ctx.h, P(_soa(u.values, 3)), P(_soa(u.boundary, 3)), P(_lib.f64(p_field.values)),
        P(_lib.f64(p_field.boundary)), P(a), P(_soa(geom.d, 3)), P(_soa(geom.d_boundary, 3)),
        P(out)), FvmError)
    return out
