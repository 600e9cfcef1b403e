"""Decomposition overhead on ONE device: gen_cavity(n) PISO with the mesh
split into P co-resident ranks (each rank's persistent grids on 1/P of the
SMs), device time per step and per CG iteration against P = 1.  With all
ranks on one B200 the per-rank bandwidth is 1/P of the device, so the ideal
is equal step time for every P; the difference is the cost of the team
machinery (halo stores, peer-mailbox reductions, halo syncs) without the
NVLink latency of a real multi-GPU run.
Usage: python tools/team_bench.py N P [P ...] [sys]   (sys: force the
system-scope kernels of a multi-GPU team; FVB_TEAM_SCOPE=sys does the same)"""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import CouplingConfig
from paper_1207_1571_b200.team import DecomposedRun

n = int(sys.argv[1])
scope = "sys" if ("sys" in sys.argv[2:] or os.environ.get("FVB_TEAM_SCOPE") == "sys") else None
for P in [int(x) for x in sys.argv[2:] if x != "sys"]:
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    cfg = CouplingConfig.from_case_config(case.config)
    run = DecomposedRun(case, cfg, P, scope=scope)
    for _ in range(2):
        run.piso_time_step(cfg)
    t0 = time.perf_counter()
    steps = 3
    cg_t = 0.0
    cg_it = 0
    for _ in range(steps):
        run.piso_time_step(cfg)
        cg_t += sum(w for s, it, w in run.last_solves if s == "cg")
        cg_it += sum(it for s, it, w in run.last_solves if s == "cg")
    wall = (time.perf_counter() - t0) / steps
    print(json.dumps({"n": n, "ranks_on_one_gpu": P, "wall_s_per_step": wall,
                      "cg_us_per_iter": 1e6 * cg_t / cg_it, "cg_iters_per_step": cg_it / steps}),
          flush=True)
    run.close()
