"""Small PISO / SIMPLE runs for compute-sanitizer (memcheck / initcheck):
gen_cavity(n) PISO and the perturbed renumbered cavity(n) PISO for each n
given (n >= 24: multi-block solver grids; n >= 41: the RCM-ordered solves),
BFS nh=4 SIMPLE.  Usage: compute-sanitizer --tool initcheck python
tools/sanitize_run.py 16 24 41"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import (CouplingConfig, init_state, piso_time_step,
                                           simple_outer_iteration)

sizes = [int(a) for a in sys.argv[1:]] or [16]
runs = []
for n in sizes:
    runs += [(f"cavity{n}", cases.gen_cavity(n), True), (f"c4_{n}", cases.perturbed_cavity(n), True)]
runs.append(("bfs4", cases.gen_backward_step(4), False))
for name, case, piso in runs:
    if piso:
        case.config.algorithm = "piso"
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    for _ in range(2):
        piso_time_step(st, cfg) if piso else simple_outer_iteration(st, cfg)
    print(name, "ok", [r[3] for r in st.residual_log][:6], flush=True)
