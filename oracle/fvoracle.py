"""CPU ORACLE — test infrastructure only, never product code.

A numpy restatement of the hot path of the reference package `fvflow`
(/root/reference/pkg/src/fvflow), i.e. arXiv 1207.1571's PISO/SIMPLE loop:
face-addressed mesh geometry, the hybrid ELL+CRS pattern, SpMV, Jacobi-PCG,
Jacobi-PBiCGStab, the finite-volume operators and the coupled step.  Every
function cites the reference file:line whose arithmetic it restates.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module, and only as the checker.  It is pinned against golden
vectors produced by the real reference (tests/golden/, made by
oracle/make_golden.py) in tests/test_oracle_golden.py.

The oracle works on plain arrays.  A mesh is any object exposing the
reference Mesh attributes (points, face_points, face_offsets, owner,
neighbour, patches[name, kind, start, count], n_cells); a case config is any
object exposing the reference CaseConfig attributes (config.py:44-76).

Arithmetic order follows the reference wherever numpy fixes it
(np.add.at = sequential in index order; einsum over 3 = (s0+s2)+s1;
SpMV over K<=7 = (sum of even slots)+(sum of odd slots)); dot products use
numpy's own ``@`` exactly as the reference does.
"""

import math
import time

import numpy as np

RES_FLOOR = 1e-30  # linsolve.py:20
TINY = 1e-300  # linsolve.py:21
VALUE_KINDS = ("fixed_value", "sine_inlet", "mass_flow", "no_slip", "fixed_pressure")


class OracleError(Exception):
    pass


# ------------------------------------------------------------------ mesh


def mesh_arrays(mesh):
    """Normalise any reference-shaped mesh into a dict of int64/f64 arrays."""
    own = np.asarray(mesh.owner, dtype=np.int64)
    nbr = np.asarray(mesh.neighbour, dtype=np.int64)
    return dict(
        points=np.asarray(mesh.points, dtype=float),
        fp=np.asarray(mesh.face_points, dtype=np.int64),
        off=np.asarray(mesh.face_offsets, dtype=np.int64),
        own=own,
        nbr=nbr,
        nc=int(mesh.n_cells),
        nf=len(own),
        ni=len(nbr),
        patches=[(p.name, p.kind, int(p.start), int(p.count)) for p in mesh.patches],
    )


def _dot3(a, b):
    # einsum("ij,ij->i") over 3 columns sums as (s0 + s2) + s1 (numpy SIMD order)
    return (a[:, 0] * b[:, 0] + a[:, 2] * b[:, 2]) + a[:, 1] * b[:, 1]


def _norm3(a):
    return np.sqrt((a[:, 0] * a[:, 0] + a[:, 1] * a[:, 1]) + a[:, 2] * a[:, 2])


def _cross(a, b):
    return np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
                     a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                     a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)


def geometry(m):
    """Fan-triangle / tet-decomposition metrics (mesh.py:154-278)."""
    pts, fp, off = m["points"], m["fp"], m["off"]
    nf, ni, nc, own, nbr = m["nf"], m["ni"], m["nc"], m["own"], m["nbr"]
    cnt = np.diff(off)
    # face seed: mean of the loop points (mesh.py:161)
    seed = np.add.reduceat(pts[fp], off[:-1], axis=0) / cnt[:, None]
    nxt = np.arange(len(fp)) + 1
    nxt[off[1:] - 1] = off[:-1]
    tri = np.repeat(np.arange(nf), cnt)
    a, b, s = pts[fp], pts[fp[nxt]], seed[tri]
    tsf = 0.5 * _cross(b - a, s - a)  # mesh.py:190
    tarea = _norm3(tsf)
    tctr = (a + b + s) / 3.0
    sf = np.zeros((nf, 3))
    np.add.at(sf, tri, tsf)
    asum = np.bincount(tri, weights=tarea, minlength=nf)
    if (asum < 1e-30).any():
        raise OracleError(f"face {int(np.argmax(asum < 1e-30))} is degenerate (zero area)")
    fc = np.zeros((nf, 3))
    for k in range(3):
        np.add.at(fc[:, k], tri, tarea * tctr[:, k])
    fc /= asum[:, None]
    smag = _norm3(sf)
    # cell seed: mean of its face centroids (mesh.py:207-213)
    nfc = np.bincount(own, minlength=nc) + np.bincount(nbr, minlength=nc)
    cs = np.zeros((nc, 3))
    np.add.at(cs, own, fc)
    np.add.at(cs, nbr, fc[:ni])
    cs /= nfc[:, None]
    vol = np.zeros(nc)
    cc = np.zeros((nc, 3))
    itri = tri < ni
    for apex, sel, sign in ((own[tri], slice(None), 1.0), (nbr[tri[itri]], itri, -1.0)):
        d = cs[apex]
        aa, bb, ss = a[sel] - d, b[sel] - d, s[sel] - d
        v = _dot3(aa, _cross(bb, ss)) / 6.0  # mesh.py:219
        if sign < 0:
            v = -v
        c = (a[sel] + b[sel] + s[sel] + d) / 4.0
        np.add.at(vol, apex, v)
        for k in range(3):
            np.add.at(cc[:, k], apex, v * c[:, k])
    if (vol <= 0.0).any():
        raise OracleError(f"cell {int(np.argmax(vol <= 0.0))} has non-positive volume")
    cc /= vol[:, None]
    d = cc[nbr] - cc[own[:ni]]
    dmag = _norm3(d)
    sd = _dot3(sf[:ni], d)
    if (sd <= 0.0).any():
        raise OracleError("internal face area vector points away from neighbour")
    w = _dot3(sf[:ni], cc[nbr] - fc[:ni]) / sd  # mesh.py:253
    cosang = sd / np.maximum(dmag * smag[:ni], 1e-300)
    nonorth = np.degrees(np.arccos(np.clip(cosang, -1.0, 1.0)))
    db = fc[ni:] - cc[own[ni:]]
    return dict(cell_volume=vol, cell_centroid=cc, face_area=sf, face_area_mag=smag,
                face_centroid=fc, d=d, d_mag=dmag, weight=w, nonorth_deg=nonorth,
                d_boundary=db, d_boundary_mag=_norm3(db))


# --------------------------------------------------------------- pattern


def pattern(n, pairs, k_cap=16, face_pairs=None):
    """Hybrid ELL(I,J)+CRS pattern with flat addresses (sparse.py:111-209)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    lo, hi = pairs.min(axis=1), pairs.max(axis=1)
    if (lo == hi).any():
        raise OracleError("self-pair in adjacency")
    u = np.unique(lo * n + hi)
    lo, hi = u // n, u % n
    ar = np.arange(n, dtype=np.int64)
    row = np.concatenate([lo, hi, ar])
    col = np.concatenate([hi, lo, ar])
    key = row * n + col
    o = np.argsort(key, kind="stable")
    row, col, key = row[o], col[o], key[o]
    cnt = np.bincount(row, minlength=n)
    k = int(min(cnt.max(), k_cap))
    start = np.concatenate([[0], np.cumsum(cnt)])
    ell = np.ones(len(row), dtype=bool)
    for i in np.nonzero(cnt > k)[0]:
        seg = np.arange(start[i], start[i + 1])
        offd = seg[col[seg] != i]
        ell[offd[k - 1:]] = False  # keep the k-1 lowest off-diagonal columns
    # slot of each kept entry within its row, CRS position of the rest
    kept_before = np.concatenate([[0], np.cumsum(ell)])
    slot = np.cumsum(ell) - 1 - kept_before[start[row]]
    cpos = np.cumsum(~ell) - 1
    addr = np.where(ell, row * k + slot, n * k + cpos)
    twin = addr[np.searchsorted(key, col * n + row)]
    I = np.full((n, k), -1, dtype=np.int64)
    J = np.full((n, k), -1, dtype=np.int64)
    tcrs = np.full((n, k), -1, dtype=np.int64)
    er, es, ec, et = row[ell], slot[ell], col[ell], twin[ell]
    I[er, es] = ec
    inell = et < n * k
    J[er[inell], es[inell]] = et[inell] % k
    tcrs[er[~inell], es[~inell]] = et[~inell] - n * k
    dslot = slot[row == col]
    crow, ccol = row[~ell], col[~ell]
    cptr = np.concatenate([[0], np.cumsum(np.bincount(crow, minlength=n))])
    ct = twin[~ell]
    if face_pairs is None:
        face_pairs = np.stack([lo, hi], axis=1)
    face_pairs = np.asarray(face_pairs, dtype=np.int64).reshape(-1, 2)
    flo, fhi = face_pairs.min(axis=1), face_pairs.max(axis=1)
    fa = np.stack([addr[np.searchsorted(key, flo * n + fhi)],
                   addr[np.searchsorted(key, fhi * n + flo)]], axis=1)
    return dict(n=n, k=k, I=I, J=J, diag_slot=dslot.astype(np.int64), ell_twin_crs=tcrs,
                crs_row_ptr=cptr.astype(np.int64), crs_col=ccol,
                crs_twin_in_ell=ct < n * k, crs_twin_row=ccol.copy(),
                crs_twin_pos=np.where(ct < n * k, ct % k, ct - n * k).astype(np.int64),
                diag_addr=ar * k + dslot, face_addr=fa)


def mesh_pattern(m, k_cap=16):
    """Cell-connectivity pattern of a mesh (sparse.py:212-220)."""
    pairs = np.stack([m["own"][: m["ni"]], m["nbr"]], axis=1)
    return pattern(m["nc"], pairs, k_cap, face_pairs=pairs)


class Matrix:
    """Value store over a pattern: V (n,k) + CRS values (sparse.py:233-258)."""

    def __init__(self, P):
        self.P = P
        self.V = np.zeros((P["n"], P["k"]))
        self.crs = np.zeros(len(P["crs_col"]))

    def add(self, addr, vals):
        addr = np.asarray(addr)
        vals = np.broadcast_to(np.asarray(vals, dtype=float), addr.shape)
        split = self.P["n"] * self.P["k"]
        e = addr < split
        np.add.at(self.V.reshape(-1), addr[e], vals[e])
        np.add.at(self.crs, addr[~e] - split, vals[~e])

    def diag(self):
        return self.V[np.arange(self.P["n"]), self.P["diag_slot"]].copy()

    def copy(self):
        c = Matrix(self.P)
        c.V[:] = self.V
        c.crs[:] = self.crs
        return c


def spmv(A, x):
    """y = A x; ELL part summed (even slots)+(odd slots) (sparse.py:296-305)."""
    P = A.P
    g = x[np.maximum(P["I"], 0)]
    y = np.einsum("nk,nk->n", A.V, g)
    if len(P["crs_col"]):
        crow = np.repeat(np.arange(P["n"]), np.diff(P["crs_row_ptr"]))
        y = y + np.bincount(crow, weights=A.crs * x[P["crs_col"]], minlength=P["n"])
    return y


# --------------------------------------------------------------- solvers


def _inv_diag(A):
    d = A.diag()
    if (d == 0.0).any():
        raise OracleError(f"singular preconditioner: zero diagonal at row {int(np.argmax(d == 0.0))}")
    return 1.0 / d


def pcg(A, b, x0, tol, abs_tol=0.0, max_iters=1000):
    """Jacobi-PCG (linsolve.py:102-172). Returns x, (iters, res0, res, converged)."""
    inv = _inv_diag(A)
    x = np.array(x0, dtype=float)
    r = b - spmv(A, x)
    bn = max(float(np.linalg.norm(b)), RES_FLOOR)
    res = float(np.linalg.norm(r)) / bn
    res0, it = res, 0
    done = res <= tol or res * bn <= abs_tol
    if not done:
        z = r * inv
        p = z.copy()
        rz = float(r @ z)
        while it < max_iters:
            it += 1
            q = spmv(A, p)
            pq = float(p @ q)
            if pq <= 0.0 or not math.isfinite(pq):
                raise OracleError(f"cg: matrix not positive definite at iteration {it}")
            al = rz / pq
            x += al * p
            r -= al * q
            res = float(np.linalg.norm(r)) / bn
            if not math.isfinite(res):
                raise OracleError(f"cg: residual diverged at iteration {it}")
            if res <= tol or res * bn <= abs_tol:
                done = True
                break
            z = r * inv
            rzn = float(r @ z)
            be = rzn / rz
            rz = rzn
            p *= be
            p += z
    return x, (it, res0, res, done)


def pbicgstab(A, b, x0, tol, abs_tol=0.0, max_iters=1000):
    """Jacobi-PBiCGStab with shadow restart (linsolve.py:175-282)."""
    inv = _inv_diag(A)
    x = np.array(x0, dtype=float)
    r = b - spmv(A, x)
    bn = max(float(np.linalg.norm(b)), RES_FLOOR)
    res = float(np.linalg.norm(r)) / bn
    res0, it = res, 0
    done = res <= tol or res * bn <= abs_tol
    rh = r.copy()
    rho = al = om = 1.0
    v = np.zeros(len(b))
    p = np.zeros(len(b))
    while not done and it < max_iters:
        it += 1
        rn = float(rh @ r)
        restart = abs(rn) < TINY
        if restart:
            rh = r.copy()
            rn = float(rh @ r)
            if rn < TINY:
                raise OracleError(f"bicgstab: rho breakdown at iteration {it}")
        if it == 1 or restart:
            p[:] = r
        else:
            be = (rn / rho) * (al / om)
            p -= om * v
            p *= be
            p += r
        rho = rn
        ph = p * inv
        v = spmv(A, ph)
        rv = float(rh @ v)
        if abs(rv) < TINY:
            raise OracleError(f"bicgstab: breakdown (r_hat . v = 0) at iteration {it}")
        al = rho / rv
        s = r - al * v
        sn = float(np.linalg.norm(s))
        if sn / bn <= tol or sn <= abs_tol:
            x += al * ph
            res = sn / bn
            done = True
            break
        sh = s * inv
        t = spmv(A, sh)
        tt = float(t @ t)
        ts = float(t @ s)
        if tt == 0.0:
            raise OracleError(f"bicgstab: omega breakdown at iteration {it}")
        om = ts / tt
        if abs(om) < TINY:
            raise OracleError(f"bicgstab: omega breakdown at iteration {it}")
        x += al * ph
        x += om * sh
        r = s - om * t
        res = float(np.linalg.norm(r)) / bn
        if not math.isfinite(res):
            raise OracleError(f"bicgstab: residual diverged at iteration {it}")
        if res <= tol or res * bn <= abs_tol:
            done = True
    return x, (it, res0, res, done)


# ------------------------------------------------------------ boundaries


def bc_kind(spec):
    """Normalise a reference BC tuple (fvm.py:79-86) to (kind, params)."""
    tag = spec[0]
    if tag == "fixed_value":
        a = spec[1:]
        return ("fixed_value", np.asarray(a[0], dtype=float) if len(a) == 1 else float(a[0]))
    if tag == "sine_inlet":
        return ("sine_inlet", (float(spec[1]), float(spec[2])))
    if tag == "mass_flow":
        return ("mass_flow", (float(spec[1]), float(spec[2])))
    if tag in ("no_slip", "zero_gradient", "empty"):
        return (tag, None)
    raise OracleError(f"unknown boundary condition tag {tag!r}")


class BField:
    """Cell values + boundary-face values + per-patch conditions (fvm.py:125-167)."""

    def __init__(self, m, bcs, values):
        self.m = m
        self.bcs = bcs  # patch name -> (kind, params)
        self.values = values
        self.boundary = np.zeros((m["nf"] - m["ni"],) + values.shape[1:])

    @property
    def vector(self):
        return self.values.ndim == 2

    def masks(self):
        """(value, zero-gradient, empty) masks over boundary faces (fvm.py:200-217)."""
        nb = self.m["nf"] - self.m["ni"]
        val, zg, em = (np.zeros(nb, bool) for _ in range(3))
        for name, _kind, start, cnt in self.m["patches"]:
            sl = slice(start - self.m["ni"], start - self.m["ni"] + cnt)
            k = self.bcs[name][0]
            (em if k == "empty" else val if k in VALUE_KINDS else zg)[sl] = True
        return val, zg, em


def apply_bcs(f, g, t=0.0):
    """Refresh boundary values at time t (fvm.py:170-197)."""
    m, ni = f.m, f.m["ni"]
    for name, _kind, start, cnt in m["patches"]:
        kind, par = f.bcs[name]
        sl = slice(start - ni, start - ni + cnt)
        faces = slice(start, start + cnt)
        if kind == "fixed_value":
            f.boundary[sl] = par
        elif kind == "no_slip":
            f.boundary[sl] = 0.0
        elif kind == "sine_inlet":
            speed = par[0] * np.sin(2.0 * np.pi * par[1] * t)
            nh = g["face_area"][faces] / g["face_area_mag"][faces, None]
            f.boundary[sl] = -speed * nh
        elif kind == "mass_flow":
            area = float(g["face_area_mag"][faces].sum())
            speed = par[0] / (par[1] * area)
            nh = g["face_area"][faces] / g["face_area_mag"][faces, None]
            f.boundary[sl] = -speed * nh
        else:  # zero_gradient, empty
            f.boundary[sl] = f.values[m["own"][faces]]


# ------------------------------------------------------------- operators


def face_values(f, g):
    """Linear interpolation, BC values on value faces, owner elsewhere (fvm.py:220-239)."""
    m, ni = f.m, f.m["ni"]
    w = g["weight"][:, None] if f.vector else g["weight"]
    vals = f.values
    inner = w * vals[m["own"][:ni]] + (1.0 - w) * vals[m["nbr"]]
    val, _, _ = f.masks()
    bsel = val[:, None] if f.vector else val
    return np.concatenate([inner, np.where(bsel, f.boundary, vals[m["own"][ni:]])])


def face_values_raw(m, g, vals):
    """Interpolation of a raw cell array, owner copy on boundary (fvm.py:242-247)."""
    ni = m["ni"]
    w = g["weight"]
    return np.concatenate([w * vals[m["own"][:ni]] + (1.0 - w) * vals[m["nbr"]], vals[m["own"][ni:]]])


def divergence(m, flux):
    """Per-cell signed face-flux sum (fvm.py:250-255)."""
    div = np.zeros(m["nc"])
    np.add.at(div, m["own"], flux)
    np.add.at(div, m["nbr"], -flux[: m["ni"]])
    return div


def gradient(f, g):
    """Gauss gradient, grad[c,i,d] = d u_i/d x_d for vectors (fvm.py:258-275)."""
    m, ni = f.m, f.m["ni"]
    fv = face_values(f, g)
    S = g["face_area"]
    con = fv[:, :, None] * S[:, None, :] if f.vector else fv[:, None] * S
    gr = np.zeros((m["nc"],) + con.shape[1:])
    np.add.at(gr, m["own"], con)
    np.add.at(gr, m["nbr"], -con[:ni])
    return gr / g["cell_volume"].reshape((-1,) + (1,) * (gr.ndim - 1))


def rhie_chow(u, p, a_diag, g):
    """Rhie-Chow face fluxes (fvm.py:499-538): S.u_f, less D_f a_f
    [(p_N - p_O) - (grad p)_f . d] on internal faces, the owner's D and d_b
    on boundary faces where p is pinned and u is not, 0 on u-empty faces."""
    m, ni = u.m, u.m["ni"]
    if (a_diag == 0.0).any():
        raise OracleError(f"zero momentum diagonal at cell {int(np.argmax(a_diag == 0.0))}")
    own, nbr = m["own"], m["nbr"]
    flux = _dot3(face_values(u, g), g["face_area"])
    dc = g["cell_volume"] / a_diag
    w = g["weight"]
    df = w * dc[own[:ni]] + (1.0 - w) * dc[nbr]
    a, _ = split_coeffs(g["face_area"][:ni], g["d"])
    gp = gradient(p, g)
    gpf = w[:, None] * gp[own[:ni]] + (1.0 - w[:, None]) * gp[nbr]
    flux[:ni] -= df * a * ((p.values[nbr] - p.values[own[:ni]]) - _dot3(gpf, g["d"]))
    uval, _, uem = u.masks()
    pval, _, _ = p.masks()
    sel = np.flatnonzero(pval & ~uval & ~uem)
    if sel.size:
        fb = ni + sel
        ob = own[fb]
        ab, _ = split_coeffs(g["face_area"][fb], g["d_boundary"][sel])
        flux[fb] -= dc[ob] * ab * ((p.boundary[sel] - p.values[ob]) - _dot3(gp[ob], g["d_boundary"][sel]))
    flux[ni:][uem] = 0.0
    return flux


def split_coeffs(S, d):
    """Over-relaxed split a = |S|^2/(S.d), k = S - a d (fvm.py:307-317)."""
    a = _dot3(S, S) / _dot3(S, d)
    return a, S - a[:, None] * d


def laplacian(A, rhs, gamma, f, g, nonorth=True, limiter=1.0, coeff=1.0):
    """coeff * laplacian(gamma, phi) into (A, rhs); returns (coef, corr) per face
    (fvm.py:335-408), including the vector-rhs last-write-wins of fvm.py:378-379."""
    m, ni, nf = f.m, f.m["ni"], f.m["nf"]
    P = A.P
    gam = np.full(nf, float(gamma)) if np.ndim(gamma) == 0 else np.asarray(gamma, dtype=float)
    coef = np.zeros(nf)
    corr = np.zeros((nf, 3) if f.vector else nf)
    if (g["d_mag"] == 0.0).any():
        raise OracleError(f"coincident centroids at internal face {int(np.argmax(g['d_mag'] == 0.0))}")
    a, k = split_coeffs(g["face_area"][:ni], g["d"])
    w = coeff * gam[:ni] * a
    coef[:ni] = gam[:ni] * a
    A.add(P["face_addr"][:, 0], w)
    A.add(P["face_addr"][:, 1], w)
    A.add(P["diag_addr"][m["own"][:ni]], -w)
    A.add(P["diag_addr"][m["nbr"]], -w)
    val, _, _ = f.masks()
    bsel = np.nonzero(val)[0]
    bf = bsel + ni
    ob = m["own"][bf]
    if len(bsel):
        ab, kb = split_coeffs(g["face_area"][bf], g["d_boundary"][bsel])
        wb = coeff * gam[bf] * ab
        coef[bf] = gam[bf] * ab
        A.add(P["diag_addr"][ob], -wb)
        if f.vector:
            rhs[ob] -= wb[:, None] * f.boundary[bsel]  # fancy-index: last write wins
        else:
            np.add.at(rhs, ob, -wb * f.boundary[bsel])
    if nonorth and limiter > 0.0:
        gr = gradient(f, g)
        wr = g["weight"].reshape((-1,) + (1,) * (gr.ndim - 1))
        gf = wr * gr[m["own"][:ni]] + (1.0 - wr) * gr[m["nbr"]]
        if f.vector:
            c = _dot3_rows(gf, k) * (gam[:ni] * limiter)[:, None]
        else:
            c = _dot3(k, gf) * gam[:ni] * limiter
        np.add.at(rhs, m["own"][:ni], -coeff * c)
        np.add.at(rhs, m["nbr"], coeff * c)
        corr[:ni] = c
        if len(bsel):
            gb = gr[ob]
            if f.vector:
                cb = _dot3_rows(gb, kb) * (gam[bf] * limiter)[:, None]
            else:
                cb = _dot3(kb, gb) * gam[bf] * limiter
            np.add.at(rhs, ob, -coeff * cb)
            corr[bf] = cb
    return coef, corr


def _dot3_rows(G, k):
    # einsum("fij,fj->fi"): per row i, (G_i0 k0 + G_i2 k2) + G_i1 k1
    return (G[:, :, 0] * k[:, None, 0] + G[:, :, 2] * k[:, None, 2]) + G[:, :, 1] * k[:, None, 1]


def laplacian_flux(coef, corr, f):
    """Face fluxes of a recorded unit-coeff laplacian (fvm.py:411-429)."""
    m, ni = f.m, f.m["ni"]
    v = f.values
    val, _, _ = f.masks()
    ob = m["own"][ni:]
    if f.vector:
        bv = np.where(val[:, None], f.boundary, v[ob])
        dphi = np.concatenate([v[m["nbr"]] - v[m["own"][:ni]], bv - v[ob]])
        return coef[:, None] * dphi + corr
    bv = np.where(val, f.boundary, v[ob])
    dphi = np.concatenate([v[m["nbr"]] - v[m["own"][:ni]], bv - v[ob]])
    return coef * dphi + corr


def convection(A, rhs, flux, f, g, scheme="upwind", coeff=1.0):
    """coeff * div(flux, phi), implicit (fvm.py:432-482)."""
    m, ni = f.m, f.m["ni"]
    P = A.P
    fi = flux[:ni]
    wo = (fi >= 0.0).astype(float) if scheme == "upwind" else g["weight"]
    co = coeff * fi * wo
    cn = coeff * fi * (1.0 - wo)
    A.add(P["diag_addr"][m["own"][:ni]], co)
    A.add(P["face_addr"][:, 0], cn)
    A.add(P["face_addr"][:, 1], -co)
    A.add(P["diag_addr"][m["nbr"]], -cn)
    val, zg, _ = f.masks()
    fb = flux[ni:]
    ob = m["own"][ni:]
    vs = np.nonzero(val)[0]
    if len(vs):
        c = coeff * fb[vs]
        if f.vector:
            rhs[ob[vs]] -= c[:, None] * f.boundary[vs]  # last write wins
        else:
            np.add.at(rhs, ob[vs], -c * f.boundary[vs])
    zs = np.nonzero(zg)[0]
    if len(zs):
        A.add(P["diag_addr"][ob[zs]], coeff * np.maximum(fb[zs], 0.0))


def ddt(A, rhs, old, dt, g, coeff=1.0):
    """Implicit Euler V/dt (fvm.py:485-496)."""
    vdt = coeff * g["cell_volume"] / dt
    A.add(A.P["diag_addr"], vdt)
    rhs += vdt[:, None] * old if old.ndim == 2 else vdt * old


# --------------------------------------------------------------- coupling


class Run:
    """Coupled PISO/SIMPLE state (coupling.py:132-423), array-level restatement."""

    def __init__(self, mesh, cc, pattern_override=None, geom_override=None, iter_caps=None):
        # iter_caps = (cg, bicgstab) per-solve iteration caps (bench.py's bounded
        # CPU samples); None = cc.max_iters for both, as the reference
        self.caps = iter_caps or (cc.max_iters, cc.max_iters)
        self.wall = {}  # coupling.py's RunState.wall sections (coupling.py:230-343)
        self.m = m = mesh_arrays(mesh)
        self.g = geom_override if geom_override is not None else geometry(m)
        self.P = pattern_override if pattern_override is not None else mesh_pattern(m)
        self.cc = cc
        ub = {n: bc_kind(s.u) for n, s in cc.boundary.items()}
        pb = {n: bc_kind(s.p) for n, s in cc.boundary.items()}
        self.u = BField(m, ub, np.zeros((m["nc"], 3)))
        self.p = BField(m, pb, np.zeros(m["nc"]))
        apply_bcs(self.u, self.g, 0.0)
        apply_bcs(self.p, self.g, 0.0)
        self.pin = not any(k[0] in VALUE_KINDS for k in pb.values())
        self.flux = self._plain_flux()
        self.t = 0.0
        self.outer = 0
        self.log = []
        self.cum = {"cg": 0, "bicgstab": 0}
        self._scale = {}

    # coupling.py:206-213
    def _plain_flux(self):
        fl = _dot3(face_values(self.u, self.g), self.g["face_area"])
        _, _, em = self.u.masks()
        fl[self.m["ni"]:][em] = 0.0
        return fl

    def _tick(self, section, t0):
        self.wall[section] = self.wall.get(section, 0.0) + time.perf_counter() - t0
        return time.perf_counter()

    def _record(self, solver, name, rep):
        self.cum[solver] += rep[0]
        self.log.append((solver, name, self.outer, rep[0], rep[1], rep[2]))

    # coupling.py:216-231
    def momentum_matrix(self, u_old=None):
        cc = self.cc
        t0 = time.perf_counter()
        A = Matrix(self.P)
        rhs = np.zeros((self.m["nc"], 3))
        if u_old is not None:
            ddt(A, rhs, u_old, cc.dt, self.g)
        convection(A, rhs, self.flux, self.u, self.g, cc.convection)
        laplacian(A, rhs, cc.nu, self.u, self.g, cc.nonorth_correction, cc.limiter, coeff=-1.0)
        self._tick("momentum_assembly", t0)
        return A, rhs

    # coupling.py:234-279
    def solve_momentum(self, A, b0, relax):
        cc = self.cc
        t0 = time.perf_counter()
        dg = A.diag()
        gp = gradient(self.p, self.g)
        rhs = b0 - self.g["cell_volume"][:, None] * gp
        As = A
        if relax and cc.alpha_u < 1.0:
            As = A.copy()
            sc = dg / cc.alpha_u
            As.V[np.arange(self.m["nc"]), self.P["diag_slot"]] = sc
            rhs = rhs + (sc - dg)[:, None] * self.u.values
        bn = np.linalg.norm(rhs, axis=0)
        bs = max(float(bn.max()), 1e-30)
        worst = 0.0
        for c, name in enumerate(("ux", "uy", "uz")):
            x, rep = pbicgstab(As, rhs[:, c], self.u.values[:, c], cc.bicgstab_tol,
                               max_iters=self.caps[1])
            self.u.values[:, c] = x
            self._record("bicgstab", name, rep)
            worst = max(worst, rep[1] * float(bn[c]) / bs)
        self._tick("momentum_solve", t0)
        return dg, worst

    # coupling.py:282-344
    def pressure_correct(self, A, b0, dg, relax_p):
        cc, m, g = self.cc, self.m, self.g
        u, p = self.u, self.p
        t0 = time.perf_counter()
        au = np.stack([spmv(A, u.values[:, c]) for c in range(3)], axis=1)
        hv = u.values + (b0 - au) / dg[:, None]
        hb = BField(m, u.bcs, hv)
        hb.boundary = u.boundary
        ph = _dot3(face_values(hb, g), g["face_area"])
        _, _, em = u.masks()
        ph[m["ni"]:][em] = 0.0
        divh = divergence(m, ph)
        rau = g["cell_volume"] / dg
        rauf = face_values_raw(m, g, rau)
        p_before = p.values.copy()
        first = None
        coef = corr = None
        for _ in range(cc.n_nonorth_correctors + 1):
            Ap = Matrix(self.P)
            rl = np.zeros(m["nc"])
            coef, corr = laplacian(Ap, rl, rauf, p, g, cc.nonorth_correction, cc.limiter, coeff=-1.0)
            rhs = rl - divh
            if self.pin:
                ref = cc.pressure_ref_cell
                ds = self.P["diag_slot"][ref]
                dref = Ap.V[ref, ds]
                rhs[ref] += dref * cc.pressure_ref_value
                Ap.V[ref, ds] = 2.0 * dref
            t0 = self._tick("pressure_assembly", t0)
            x, rep = pcg(Ap, rhs, p.values, cc.cg_tol, max_iters=self.caps[0])
            t0 = self._tick("pressure_solve", t0)
            self._record("cg", "p", rep)
            if first is None:
                first = rep[1]
            p.values = x
        self.flux = ph - laplacian_flux(coef, corr, p)
        if relax_p and cc.alpha_p < 1.0:
            p.values = p_before + cc.alpha_p * (p.values - p_before)
        apply_bcs(p, g, self.t)
        gp = gradient(p, g)
        u.values = hv - rau[:, None] * gp
        apply_bcs(u, g, self.t)
        self._tick("correction", t0)
        return first

    def normalized(self, slot, res):
        seen = max(self._scale.get(slot, 0.0), res)
        self._scale[slot] = seen
        return res / max(seen, 1e-30)

    # coupling.py:347-353
    def simple_sweep(self):
        self.outer += 1
        A, b0 = self.momentum_matrix()
        dg, mr = self.solve_momentum(A, b0, relax=True)
        pr = self.pressure_correct(A, b0, dg, relax_p=True)
        return self.normalized("u", mr), self.normalized("p", pr)

    # coupling.py:356-370
    def piso_step(self):
        self.outer += 1
        self.t = self.outer * self.cc.dt
        apply_bcs(self.u, self.g, self.t)
        apply_bcs(self.p, self.g, self.t)
        old = self.u.values.copy()
        A, b0 = self.momentum_matrix(old)
        dg, mr = self.solve_momentum(A, b0, relax=False)
        pr = None
        for _ in range(self.cc.n_correctors):
            r = self.pressure_correct(A, b0, dg, relax_p=False)
            if pr is None:
                pr = r
        return mr, pr

    # coupling.py:373-375
    def continuity(self):
        return float(np.abs(divergence(self.m, self.flux)).max())
