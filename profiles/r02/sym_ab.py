"""A/B of the pressure CG on the symmetric half storage (cg_pass_a_sym)
against the full matrix (FVB_SOLVER_NO_SYM): gen_cavity(N) PISO, W warm-up
steps then S timed steps on each side from the same state, device ms per
step and CG us per iteration, and whether the two give bitwise the same
fields and residual logs.   Usage: python tools/sym_ab.py N [S] [W]"""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
if os.environ.get("FVB_PKG_ROOT"):
    sys.path.insert(0, os.environ["FVB_PKG_ROOT"])
import numpy as np
from paper_1207_1571_b200 import _lib, cases
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step

n = int(sys.argv[1])
S = int(sys.argv[2]) if len(sys.argv) > 2 else 3
W = int(sys.argv[3]) if len(sys.argv) > 3 else 1


def run(flags):
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    if n > 128:
        case.config.max_iters = 5000
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    _lib.check(_lib.lib.fvb_set_solver_options(st._ctx.h, flags))
    for _ in range(W):
        piso_time_step(st, cfg)
    t0 = time.perf_counter()
    cg_t = cg_it = 0
    n0 = len(st.residual_log)
    for _ in range(S):
        piso_time_step(st, cfg)
        cg_t += sum(w for s, it, w in st._last_solves if s == "cg")
        cg_it += sum(it for s, it, w in st._last_solves if s == "cg")
    wall = (time.perf_counter() - t0) / S
    return st, {"ms_per_step": 1e3 * wall, "cg_us_per_iter": 1e6 * cg_t / max(cg_it, 1),
                "cg_iters": cg_it}, st.residual_log[n0:]


a, ra, la = run(0)
b, rb, lb = run(_lib.SOLVER_NO_SYM)
same = (np.array_equal(a.u.values, b.u.values) and np.array_equal(a.p.values, b.p.values)
        and np.array_equal(a.flux, b.flux) and la == lb)
print(json.dumps({"n": n, "sym": ra, "full": rb, "bitwise_equal": bool(same)}), flush=True)
