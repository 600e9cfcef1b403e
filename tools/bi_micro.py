"""BiCGStab kernel microbenchmark: fixed-iteration batched (3-component)
Jacobi-BiCGStab on a convection-diffusion-like nonsymmetric matrix (K = 7)
through fvb_op_bicgstab_batched; prints device time per batched iteration
and the algorithmic HBM rate (600 B per row per batched iteration).
Usage: python tools/bi_micro.py N ITERS [crs] [explicit]
"crs" adds long-range couplings that spill into the CRS tail; "explicit"
makes the SpMV sweeps read int32 indices instead of stencil codes
(fvb_set_solver_options)."""
import ctypes as C, hashlib, json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
if os.environ.get("FVB_PKG_ROOT"):  # A/B of diagnostic builds (tools/build_variant.py)
    sys.path.insert(0, os.environ["FVB_PKG_ROOT"])
import numpy as np
from paper_1207_1571_b200 import _lib, cases, sparse
from paper_1207_1571_b200.device import context_for

n = int(sys.argv[1]); iters = int(sys.argv[2])
opts = (1 if "explicit" in sys.argv[3:] else 0) | (4 if "nocluster" in sys.argv[3:] else 0)
mesh = cases.box_mesh(n, n, n, 1.0, 1.0, 1.0, [("all", "wall", ["x-", "x+", "y-", "y+", "z-", "z+"])])
crs_mode = "crs" in sys.argv[3:]
if crs_mode:
    # extra long-range couplings on ~2% of the rows with K capped at 7: the
    # overflow entries go to the CRS tail
    ni = mesh.n_internal
    pairs = np.stack([np.asarray(mesh.owner[:ni]), np.asarray(mesh.neighbour)], axis=1)
    rng = np.random.default_rng(1)
    a = rng.choice(mesh.n_cells, size=max(1, mesh.n_cells // 50), replace=False)
    bb = rng.integers(0, mesh.n_cells, size=a.size)  # random partners: distinct offset tuples
    extra = np.stack([np.minimum(a, bb), np.maximum(a, bb)], axis=1)
    extra = extra[extra[:, 0] != extra[:, 1]]
    pairs = np.unique(np.concatenate([pairs, extra]), axis=0)
    pat = sparse.pattern_from_pairs(mesh.n_cells, pairs, 7)
else:
    pat = sparse.build_pattern(mesh)
N, K = pat.n, pat.k
rows = np.arange(N)[:, None]
V = np.where(pat.I >= 0, np.where(pat.I > rows, -0.6, -1.4), 0.0)
V[np.arange(N), pat.diag_slot] = 0.0
crs = np.full(max(pat.nnz_crs, 1), -0.3)
tail = np.zeros(N)
if pat.nnz_crs:
    tail = np.bincount(np.repeat(np.arange(N), np.diff(pat.crs_row_ptr)), weights=crs[:pat.nnz_crs],
                       minlength=N)
V[np.arange(N), pat.diag_slot] = -V.sum(axis=1) - tail + 0.05
b = np.random.default_rng(0).normal(size=3 * N)
x = np.empty(3 * N)
ctx = context_for(None, None, pat)
if opts:  # (absent from builds older than the options API)
    _lib.check(_lib.lib.fvb_set_solver_options(ctx.h, opts))
reps = (_lib.SolveReportC * 3)()
P = _lib.ptr
res = []
for rpt in range(3):
    rc = _lib.lib.fvb_op_bicgstab_batched(ctx.h, 3, P(_lib.f64(V)), P(crs), P(b), P(np.zeros(3 * N)),
                                          P(x), 1e-300, 0.0, iters, reps)
    _lib.check(rc)
    r = reps[0]
    res.append((r.wall_time, r.t_smvp, r.t_daxpy, r.t_reduction))
t, ts, ta, tr = min(res)
codes, nesc, defer = C.c_int(), C.c_int64(), C.c_int()
_lib.check(_lib.lib.fvb_pattern_codes(ctx.h, C.byref(codes), C.byref(nesc), C.byref(defer), None))
use_codes = codes.value > 0
# the two SpMV passes read 1-byte stencil codes instead of K int32 indices
row_bytes = 600.0 - (2 * (4 * K - 1) if use_codes else 0)
it = reps[0].iterations
print(json.dumps({"options": opts, "res_full": [reps[c].final_residual for c in range(3)], "n": n, "k": int(K),
                  "nnz_crs": int(pat.nnz_crs),
                  "iters": [reps[c].iterations for c in range(3)],
                  "err": [reps[c].error_kind for c in range(3)] if hasattr(reps[0], "error_kind") else None,
                  "us_per_iter": 1e6 * t / it, "us_spmv": 1e6 * ts / it, "us_update": 1e6 * ta / it,
                  "us_reduce": 1e6 * tr / it, "alg_gbs": row_bytes * N * it / t / 1e9, "codes": codes.value if use_codes else 0,
                  "res": [reps[c].final_residual for c in range(3)],
                  "x_sha": hashlib.sha256(x.tobytes()).hexdigest()[:16]}))
