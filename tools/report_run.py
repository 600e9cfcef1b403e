"""The paper's profile views (Fig. 4/5, Table 3; reference report.py) from a
device run: gen_cavity(N) PISO with solver stage timers on, then the
report's tables (text) and figures (SVG + CSV) written to OUT_DIR.
Usage: python tools/report_run.py N STEPS OUT_DIR"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1207_1571_b200 import cases, report
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step

n, steps, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
case = cases.gen_cavity(n)
case.config.algorithm, case.config.dt = "piso", 0.1 / n
cfg = CouplingConfig.from_case_config(case.config, record_stages=True)
st = init_state(case, cfg)
t0 = time.perf_counter()
for _ in range(steps):
    piso_time_step(st, cfg)
st.add_wall("total", time.perf_counter() - t0)
prof = report.collect_profile(st)
os.makedirs(out, exist_ok=True)
report.write_profile(prof, os.path.join(out, "profile.json"))
with open(os.path.join(out, "tables.txt"), "w") as f:
    f.write(report.format_tables(prof))
paths = report.render_figures(prof, st.residual_log, out)
print(report.format_tables(prof))
print([str(p) for p in paths])
