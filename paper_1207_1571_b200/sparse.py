"""Hybrid ELL(V, I, J) + CRS sparse format of the paper (reference: sparse.py).

The pattern is built natively (fvb_pattern_plan_*) with the reference's
exact integer semantics: entries sorted by (row, col), K = min(max row
count, k_cap), the diagonal pinned in ELL and the highest-column
off-diagonals of over-long rows spilled to CRS, flat addresses
row*K + slot / N*K + pos, J = slot of the transposed twin
(sparse.py:111-209).  On the device the ELL block is stored slot-major
(V[s*N + i], int32 I) so a warp reads each slot coalesced.

smvp runs the libfvb kernel, which sums a row exactly like numpy's einsum
for K <= 7 (even slots, odd slots, then their sum) and is therefore
bit-identical to fvflow.sparse.smvp on hex/quad meshes.
"""

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import context_for
from .errors import SparseError

__all__ = [
    "SparseError", "SparsityPattern", "pattern_from_pairs", "build_pattern",
    "build_pattern_from_example", "HybridMatrix", "coeff_accumulate", "diagonal", "smvp",
    "stmvp", "pack_q", "unpack_q", "format_debug",
]


@dataclass
class SparsityPattern:
    """Integer layout shared by all matrices on one mesh (sparse.py:29-108)."""

    n: int
    k: int
    I: np.ndarray
    J: np.ndarray
    diag_slot: np.ndarray
    ell_twin_crs: np.ndarray
    crs_row_ptr: np.ndarray
    crs_col: np.ndarray
    crs_twin_in_ell: np.ndarray
    crs_twin_row: np.ndarray
    crs_twin_pos: np.ndarray
    diag_addr: np.ndarray
    face_addr: np.ndarray

    @property
    def nnz_crs(self):
        return len(self.crs_col)

    @property
    def crs_row(self):
        return np.repeat(np.arange(self.n), np.diff(self.crs_row_ptr))

    def address(self, i, j):
        """Flat address of entry (i, j); SparseError if absent."""
        hits = np.nonzero(self.I[i] == j)[0]
        if len(hits):
            return i * self.k + int(hits[0])
        lo, hi = self.crs_row_ptr[i], self.crs_row_ptr[i + 1]
        hits = lo + np.nonzero(self.crs_col[lo:hi] == j)[0]
        if len(hits):
            return self.n * self.k + int(hits[0])
        raise SparseError(f"entry ({i}, {j}) not in pattern")

    def check_invariants(self):
        """Vectorised check of the structural invariants (sparse.py:66-108)."""
        n, k = self.n, self.k
        I, J = self.I, self.J
        real = I >= 0
        # real entries first, strictly increasing, diagonal where claimed
        assert (real[:, :-1] | ~real[:, 1:]).all(), "sentinel before entry"
        inc = (I[:, 1:] > I[:, :-1]) | ~real[:, 1:]
        assert inc.all(), "columns not increasing"
        assert (I[np.arange(n), self.diag_slot] == np.arange(n)).all(), "diagonal misplaced"
        assert ((J == -1) | real).all() and ((self.ell_twin_crs == -1) | real).all()
        r, s = np.nonzero(real & (J >= 0))
        assert (I[I[r, s], J[r, s]] == r).all(), "J inconsistent"
        r, s = np.nonzero(real & (J < 0))
        pos = self.ell_twin_crs[r, s]
        assert (pos >= 0).all(), "missing CRS twin ref"
        if len(pos):
            assert (self.crs_col[pos] == r).all()
            assert (self.crs_row[pos] == I[r, s]).all(), "CRS twin in wrong row"
        crow = self.crs_row
        assert (crow != self.crs_col).all(), "diagonal must not overflow to CRS"
        assert (self.crs_twin_row == self.crs_col).all()
        te = self.crs_twin_in_ell
        if te.any():
            assert (I[self.crs_col[te], self.crs_twin_pos[te]] == crow[te]).all()
        if (~te).any():
            q = self.crs_twin_pos[~te]
            assert (self.crs_col[q] == crow[~te]).all() and (crow[q] == self.crs_col[~te]).all()
        rows = np.concatenate([np.nonzero(real)[0], crow])
        cols = np.concatenate([I[real], self.crs_col])
        key = rows * n + cols
        assert len(np.unique(key)) == len(key), "duplicate coordinates"
        twin = np.isin(cols * n + rows, key)
        assert twin.all(), "entry lacks structural twin"


def pattern_from_pairs(n, pairs, k_cap, face_pairs=None) -> SparsityPattern:
    """Native pattern build with the reference's semantics (sparse.py:111-209)."""
    if k_cap < 1:
        raise SparseError("k_cap must be at least 1")
    pairs = _lib.i64(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
    P = _lib.ptr
    plan = C.c_void_p()
    k = C.c_int64()
    nnz = C.c_int64()
    _lib.check(_lib.lib.fvb_pattern_plan_create(n, len(pairs), P(pairs, _lib.i64p), k_cap,
                                                C.byref(plan), C.byref(k), C.byref(nnz)),
               SparseError)
    try:
        k, nnz = k.value, nnz.value
        if face_pairs is None:
            lo = pairs.min(axis=1) if len(pairs) else np.zeros(0, np.int64)
            hi = pairs.max(axis=1) if len(pairs) else np.zeros(0, np.int64)
            u = np.unique(lo * n + hi)
            face_pairs = np.stack([u // n, u % n], axis=1) if len(u) else np.zeros((0, 2), np.int64)
        fpairs = _lib.i64(np.asarray(face_pairs, dtype=np.int64).reshape(-1, 2))
        I = np.empty((n, k), np.int64)
        J = np.empty((n, k), np.int64)
        ds = np.empty(n, np.int64)
        tcrs = np.empty((n, k), np.int64)
        rp = np.empty(n + 1, np.int64)
        ccol = np.empty(nnz, np.int64)
        cin = np.empty(nnz, np.uint8)
        cpos = np.empty(nnz, np.int64)
        fa = np.empty((len(fpairs), 2), np.int64)
        _lib.check(_lib.lib.fvb_pattern_plan_fill(
            plan, len(fpairs), P(fpairs, _lib.i64p), P(I, _lib.i64p), P(J, _lib.i64p),
            P(ds, _lib.i64p), P(tcrs, _lib.i64p), P(rp, _lib.i64p), P(ccol, _lib.i64p),
            P(cin, _lib.u8p), P(cpos, _lib.i64p), P(fa, _lib.i64p)), SparseError)
    finally:
        _lib.lib.fvb_pattern_plan_destroy(plan)
    return SparsityPattern(n=n, k=k, I=I, J=J, diag_slot=ds, ell_twin_crs=tcrs, crs_row_ptr=rp,
                           crs_col=ccol, crs_twin_in_ell=cin.astype(bool), crs_twin_row=ccol.copy(),
                           crs_twin_pos=cpos, diag_addr=np.arange(n, dtype=np.int64) * k + ds,
                           face_addr=fa)


def build_pattern(mesh, k_cap=16) -> SparsityPattern:
    """Cell-connectivity pattern: diagonal + internal faces (sparse.py:212-220)."""
    ni = mesh.n_internal
    pairs = np.stack([np.asarray(mesh.owner[:ni]), np.asarray(mesh.neighbour)], axis=1)
    return pattern_from_pairs(mesh.n_cells, pairs, k_cap, face_pairs=pairs)


def build_pattern_from_example() -> SparsityPattern:
    """4x4 ring fixture, K = 3 (sparse.py:223-230)."""
    return pattern_from_pairs(4, [(0, 1), (1, 2), (2, 3), (0, 3)], 3)


@dataclass
class HybridMatrix:
    """Values over a pattern: V (n, k) with 0.0 at padding, plus CRS values."""

    pattern: SparsityPattern
    V: np.ndarray
    crs_val: np.ndarray

    @classmethod
    def zeros(cls, pattern):
        return cls(pattern=pattern, V=np.zeros((pattern.n, pattern.k)),
                   crs_val=np.zeros(pattern.nnz_crs))

    def clear(self):
        self.V[:] = 0.0
        self.crs_val[:] = 0.0

    def add_at(self, addr, values):
        """Host-side accumulate at flat addresses (test/setup utility)."""
        addr = np.asarray(addr)
        values = np.broadcast_to(np.asarray(values, dtype=float), addr.shape)
        split = self.pattern.n * self.pattern.k
        e = addr < split
        np.add.at(self.V.reshape(-1), addr[e], values[e])
        np.add.at(self.crs_val, addr[~e] - split, values[~e])

    def to_dense(self):
        """Dense copy (debugging and small-case tests only)."""
        p = self.pattern
        out = np.zeros((p.n, p.n))
        live = p.I >= 0
        out[np.nonzero(live)[0], p.I[live]] = self.V[live]
        if p.nnz_crs:
            out[p.crs_row, p.crs_col] = self.crs_val
        return out


def _slot_of(p, addr):
    """(value array, index) behind a flat address: ELL slots first, then the
    CRS tail (the address space of sparse.py:158)."""
    addr = int(addr)
    ell = p.n * p.k
    if 0 <= addr < ell:
        i, s = divmod(addr, p.k)
        if p.I[i, s] < 0:
            raise SparseError(f"address {addr} points at a padding sentinel")
        return "V", (i, s)
    if ell <= addr < ell + p.nnz_crs:
        return "crs_val", addr - ell
    raise SparseError(f"address {addr} outside pattern")


def coeff_accumulate(A, addr, value, add=True):
    """Checked single-entry add (or set, add=False) (sparse.py:269-288)."""
    name, at = _slot_of(A.pattern, addr)
    arr = getattr(A, name)
    arr[at] = arr[at] + value if add else value


def diagonal(A):
    p = A.pattern
    return A.V[np.arange(p.n), p.diag_slot].copy()


def _ctx(A, mesh=None, geom=None):
    return context_for(mesh, geom, A.pattern)


def smvp(A, x):
    """y = A x on the device (fvb_op_smvp; reference sparse.py:296-305)."""
    p = A.pattern
    if len(x) != p.n:
        raise SparseError(f"dimension mismatch: {len(x)} != {p.n}")
    ctx = _ctx(A)
    V = _lib.f64(A.V)
    crs = _lib.f64(A.crs_val)
    xx = _lib.f64(x)
    y = np.empty(p.n)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_op_smvp(ctx.h, P(V), P(crs), P(xx), P(y)))
    return y


def stmvp(A, x):
    """y = A^T x without forming the transpose (fvb_op_stmvp; reference
    sparse.py:308-334): scanning row i, the value of the twin (c, i) of every
    stored (i, c) is gathered through J or the CRS back-references — the
    paper's column-access path (§3.1).  Same summation order as the
    reference (einsum over the slots, then the CRS tail)."""
    p = A.pattern
    if len(x) != p.n:
        raise SparseError(f"dimension mismatch: {len(x)} != {p.n}")
    ctx = _ctx(A)
    P = _lib.ptr
    V = _lib.f64(A.V)
    crs = _lib.f64(A.crs_val) if p.nnz_crs else np.zeros(1)
    J = _lib.i64(p.J)
    tw = _lib.i64(p.ell_twin_crs)
    ce = np.ascontiguousarray(p.crs_twin_in_ell, dtype=np.uint8)
    cr = _lib.i64(p.crs_twin_row)
    cp = _lib.i64(p.crs_twin_pos)
    xx = _lib.f64(x)
    y = np.empty(p.n)
    _lib.check(_lib.lib.fvb_op_stmvp(ctx.h, P(V), P(crs), P(J, _lib.i64p), P(tw, _lib.i64p),
                                     P(ce, _lib.u8p), P(cr, _lib.i64p), P(cp, _lib.i64p),
                                     P(xx), P(y)))
    return y


_Q_MODES = {"by_N": 0, "by_K": 1}


def pack_q(pattern, mode="by_N"):
    """Fuse I and J into one integer array Q (reference sparse.py:337-351):
    by_N: Q = N*I + J, by_K: Q = K*I + J; padding -> -1, twin in CRS -> -2 - I."""
    if mode not in _Q_MODES:
        raise SparseError(f"unknown mode {mode!r}")
    p = pattern
    I = _lib.i64(p.I)
    J = _lib.i64(p.J)
    q = np.empty(I.shape, dtype=np.int64)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_pack_q(p.n, p.k, P(I, _lib.i64p), P(J, _lib.i64p), _Q_MODES[mode],
                                   P(q, _lib.i64p)), SparseError)
    return q


def unpack_q(q, n, k, mode="by_N"):
    """Inverse of pack_q: (I, J) exactly, sentinels included (sparse.py:354-363)."""
    if mode not in _Q_MODES:
        raise SparseError(f"unknown mode {mode!r}")
    q = _lib.i64(q)
    I = np.empty(q.shape, dtype=np.int64)
    J = np.empty(q.shape, dtype=np.int64)
    P = _lib.ptr
    _lib.check(_lib.lib.fvb_unpack_q(n, k, q.size, P(q, _lib.i64p), _Q_MODES[mode],
                                     P(I, _lib.i64p), P(J, _lib.i64p)), SparseError)
    return I, J


def format_debug(A):
    """Text dump of a small matrix: dense rows, then I, J, V and the CRS
    tail (reference sparse.py:366-383 content)."""
    p = A.pattern
    if p.n > 16:
        raise SparseError("debug dump limited to n <= 16")
    dense = A.to_dense()
    parts = [f"hybrid {p.n}x{p.n}, K={p.k}, crs entries: {p.nnz_crs}"]
    parts += ["  [" + " ".join(format(v, "10.4g") for v in row) + "]" for row in dense]
    for label, arr in (("I", p.I), ("J", p.J)):
        parts.append(f"{label} = {arr.tolist()}")
    parts.append("V = %s" % np.round(A.V, 6).tolist())
    if p.nnz_crs:
        parts.append("CRS rows %s cols %s vals %s" % (p.crs_row.tolist(), p.crs_col.tolist(),
                                                      np.round(A.crs_val, 6).tolist()))
    return "\n".join(parts)
