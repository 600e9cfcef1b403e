"""CG kernel microbenchmark: fixed-iteration Jacobi-PCG on a cavity
Laplacian-like SPD matrix (K = 7) through fvb_op_cg; prints device time per
iteration and the algorithmic HBM rate (N(12K+96) bytes per iteration).
Usage: python tools/cg_micro.py N ITERS [crs|perm] [explicit] [norcm] [nocluster] [grid=B]
"crs" adds long-range couplings: CRS tail + escaped stencil-code rows; "perm"
randomly renumbers the box: no stencil codes, RCM-ordered solve; "explicit"
and "norcm" set the context's solver format options (fvb_set_solver_options:
explicit int32 indices instead of stencil codes / mesh order instead of RCM)."""
import ctypes as C, hashlib, json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
if os.environ.get("FVB_PKG_ROOT"):  # A/B of diagnostic builds (tools/build_variant.py)
    sys.path.insert(0, os.environ["FVB_PKG_ROOT"])
import numpy as np
from paper_1207_1571_b200 import _lib, cases, sparse
from paper_1207_1571_b200.device import context_for

n = int(sys.argv[1]); iters = int(sys.argv[2])
opts = (1 if "explicit" in sys.argv[3:] else 0) | (2 if "norcm" in sys.argv[3:] else 0) | \
    (4 if "nocluster" in sys.argv[3:] else 0)
t0 = time.time()
mesh = cases.box_mesh(n, n, n, 1.0, 1.0, 1.0, [("all", "wall", ["x-", "x+", "y-", "y+", "z-", "z+"])])
if len(sys.argv) > 3 and sys.argv[3] == "perm":
    # randomly renumbered box: no stencil codes, the solver's RCM order applies
    ni = mesh.n_internal
    perm = np.random.default_rng(2).permutation(mesh.n_cells)
    pairs = np.stack([perm[np.asarray(mesh.owner[:ni])], perm[np.asarray(mesh.neighbour)]], axis=1)
    pat = sparse.pattern_from_pairs(mesh.n_cells, np.sort(pairs, axis=1), 16)
elif len(sys.argv) > 3 and sys.argv[3] == "crs":
    # symmetric long-range couplings on ~2% of the rows with K capped at 7:
    # overflow entries go to the CRS tail, those rows escape the stencil codes
    ni = mesh.n_internal
    pairs = np.stack([np.asarray(mesh.owner[:ni]), np.asarray(mesh.neighbour)], axis=1)
    rng = np.random.default_rng(1)
    a = rng.choice(mesh.n_cells, size=max(1, mesh.n_cells // 50), replace=False)
    bb = rng.integers(0, mesh.n_cells, size=a.size)  # random partners: distinct offset tuples
    extra = np.stack([np.minimum(a, bb), np.maximum(a, bb)], axis=1)
    pairs = np.unique(np.concatenate([pairs, extra[extra[:, 0] != extra[:, 1]]]), axis=0)
    pat = sparse.pattern_from_pairs(mesh.n_cells, pairs, 7)
else:
    pat = sparse.build_pattern(mesh)
N, K = pat.n, pat.k
V = np.where(pat.I >= 0, -1.0, 0.0)
ncrs = np.diff(pat.crs_row_ptr) if pat.nnz_crs else np.zeros(N, dtype=np.int64)
V[np.arange(N), pat.diag_slot] = (pat.I >= 0).sum(axis=1) - 1 + ncrs + 0.01
b = np.random.default_rng(0).normal(size=N)
x = np.empty(N)
ctx = context_for(None, None, pat)
grid = [int(a[5:]) for a in sys.argv[3:] if a.startswith("grid=")]
if opts or grid:  # (absent from builds older than the options API)
    _lib.check(_lib.lib.fvb_set_solver_options(ctx.h, opts))
if grid:
    _lib.check(_lib.lib.fvb_set_solver_grid(ctx.h, grid[0]))
rep = _lib.SolveReportC()
P = _lib.ptr
crs = np.full(max(pat.nnz_crs, 1), -1.0)
setup = time.time() - t0
rcm0 = C.c_int64()
_lib.check(_lib.lib.fvb_pattern_codes(ctx.h, None, None, None, C.byref(rcm0)))
res = []
for rpt in range(3):
    rc = _lib.lib.fvb_op_cg(ctx.h, P(_lib.f64(V)), P(crs), P(b), P(np.zeros(N)), P(x), 1e-300, 0.0,
                            iters, C.byref(rep))
    _lib.check(rc)
    res.append((rep.wall_time, rep.t_smvp, rep.t_daxpy, rep.t_reduction))
t, ta, tb, tr = min(res)
codes, nesc, defer = C.c_int(), C.c_int64(), C.c_int()
rcm1 = C.c_int64()
_lib.check(_lib.lib.fvb_pattern_codes(ctx.h, C.byref(codes), C.byref(nesc), C.byref(defer), C.byref(rcm1)))
# 1-byte stencil codes replace the K int32 indices when the pattern compresses
use_codes = codes.value > 0
# deferred x update (large systems): pass B no longer re-reads p
bytes_it = N * ((8 * K + 1 if use_codes else 12 * K) + (88 if defer.value else 96))
setup_b = N * (12 * K + 80)
print(json.dumps({"options": opts, "grid": grid[0] if grid else 0, "n": n, "iters": rep.iterations,
                  "us_per_iter": 1e6 * t / iters,
                  "us_passA": 1e6 * ta / iters, "us_passB": 1e6 * tb / iters,
                  "us_reduce2x": 1e6 * tr / iters,
                  "alg_gbs": (setup_b + iters * bytes_it) / t / 1e9, "setup_s": round(setup, 1),
                  "codes": codes.value if use_codes else 0, "defer_x": defer.value, "rcm_solves": rcm1.value - rcm0.value, "escaped": nesc.value if use_codes else 0,
                  "nnz_crs": int(pat.nnz_crs), "res": rep.final_residual,
                  "x_sha": hashlib.sha256(x.tobytes()).hexdigest()[:16]}))
