"""Determinism stress of the decomposed path (the flat all-to-all team
reduction, round 2): gen_cavity(N) PISO split into P co-resident ranks on
one device, S steps from a fresh DecomposedRun, repeated R times; every run
must give bitwise the same u, p, flux and per-solve iteration counts as run
0 (the reduction order is fixed by construction, so a difference would be a
race in the team barrier).
Usage: python tools/team_stress.py N P S R"""
import hashlib, json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import CouplingConfig
from paper_1207_1571_b200.team import DecomposedRun

n, P, S, R = (int(x) for x in sys.argv[1:5])
ref = None
bad = 0
for k in range(R):
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    cfg = CouplingConfig.from_case_config(case.config)
    run = DecomposedRun(case, cfg, P)
    its = []
    for _ in range(S):
        run.piso_time_step(cfg)
        its.append([(s, it) for s, it, _ in run.last_solves])
    u, p, flux = run.gather()
    run.close()
    h = hashlib.sha1(u.tobytes() + p.tobytes() + flux.tobytes()).hexdigest()
    rec = {"run": k, "sha1": h, "iters": its}
    if ref is None:
        ref = rec
    elif rec["sha1"] != ref["sha1"] or rec["iters"] != ref["iters"]:
        bad += 1
        print(json.dumps({"mismatch": rec}), flush=True)
print(json.dumps({"n": n, "ranks": P, "steps": S, "runs": R, "mismatches": bad,
                  "sha1": ref["sha1"], "iters_run0": ref["iters"]}), flush=True)
