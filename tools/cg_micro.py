"""CG kernel microbenchmark: fixed-iteration Jacobi-PCG on a cavity
Laplacian-like SPD matrix (K = 7) through fvb_op_cg; prints device time per
iteration and the algorithmic HBM rate (N(12K+96) bytes per iteration).
Usage: python tools/cg_micro.py N ITERS  (FVB_CG_VARIANT selects the kernel)"""
import ctypes as C, hashlib, json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1207_1571_b200 import _lib, cases, sparse
from paper_1207_1571_b200.device import context_for

n = int(sys.argv[1]); iters = int(sys.argv[2])
t0 = time.time()
mesh = cases.box_mesh(n, n, n, 1.0, 1.0, 1.0, [("all", "wall", ["x-", "x+", "y-", "y+", "z-", "z+"])])
pat = sparse.build_pattern(mesh)
N, K = pat.n, pat.k
V = np.where(pat.I >= 0, -1.0, 0.0)
V[np.arange(N), pat.diag_slot] = (pat.I >= 0).sum(axis=1) - 1 + 0.01
b = np.random.default_rng(0).normal(size=N)
x = np.empty(N)
ctx = context_for(None, None, pat)
rep = _lib.SolveReportC()
P = _lib.ptr
crs = np.zeros(max(pat.nnz_crs, 1))
setup = time.time() - t0
res = []
for rpt in range(3):
    rc = _lib.lib.fvb_op_cg(ctx.h, P(_lib.f64(V)), P(crs), P(b), P(np.zeros(N)), P(x), 1e-300, 0.0,
                            iters, C.byref(rep))
    _lib.check(rc)
    res.append((rep.wall_time, rep.t_smvp, rep.t_daxpy, rep.t_reduction))
t, ta, tb, tr = min(res)
codes, nesc = C.c_int(), C.c_int64()
_lib.check(_lib.lib.fvb_pattern_codes(ctx.h, C.byref(codes), C.byref(nesc)))
# 1-byte stencil codes replace the K int32 indices when the pattern compresses
use_codes = codes.value and os.environ.get("FVB_CG_VARIANT", "-1") == "-1"
bytes_it = N * ((8 * K + 1 + 96) if use_codes else (12 * K + 96))
setup_b = N * (12 * K + 80)
print(json.dumps({"variant": os.environ.get("FVB_CG_VARIANT", "-1"), "n": n, "iters": rep.iterations,
                  "us_per_iter": 1e6 * t / iters,
                  "us_passA": 1e6 * ta / iters, "us_passB": 1e6 * tb / iters,
                  "us_reduce2x": 1e6 * tr / iters,
                  "alg_gbs": (setup_b + iters * bytes_it) / t / 1e9, "setup_s": round(setup, 1),
                  "codes": codes.value if use_codes else 0, "res": rep.final_residual,
                  "x_sha": hashlib.sha256(x.tobytes()).hexdigest()[:16]}))
