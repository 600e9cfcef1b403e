"""Debug harness: one decomposed run vs the single-domain run, step by step."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from golden_io import golden_case, rel
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step, simple_outer_iteration
from paper_1207_1571_b200.team import DecomposedRun

name = sys.argv[1]; nparts = int(sys.argv[2])
case, g = golden_case(name)
cfg = CouplingConfig.from_case_config(case.config)
st = init_state(case, cfg)
t0 = time.time()
run = DecomposedRun(case, cfg, nparts)
print(name, nparts, "init", time.time() - t0, flush=True)
u, p, f = run.gather()
print(" init rel u p flux", rel(u, st.u.values), rel(p, st.p.values), rel(f, st.flux), flush=True)
for s in range(int(g["steps"])):
    if cfg.algorithm == "piso":
        piso_time_step(st, cfg)
    else:
        simple_outer_iteration(st, cfg)
    try:
        if cfg.algorithm == "piso":
            run.piso_time_step(cfg)
        else:
            run.simple_outer_iteration(cfg)
    except Exception as e:
        print(" step", s, "FAILED", type(e).__name__, e, flush=True)
        print(" team log", run.residual_log[-6:])
        print(" single log", st.residual_log[-6:])
        break
    u, p, f = run.gather()
    print(" step", s, "rel u p flux", rel(u, st.u.values), rel(p, st.p.values), rel(f, st.flux), flush=True)
    print("   team  ", [(r[0], r[1], r[3]) for r in run.residual_log[-8:]])
    print("   single", [(r[0], r[1], r[3]) for r in st.residual_log[-8:]], flush=True)
run.close()
