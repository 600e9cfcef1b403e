"""Quick device timing probe: PISO steps on gen_cavity(n)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1207_1571_b200 import cases  # noqa: E402
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.time()
case = cases.gen_cavity(n)
cc = case.config
cc.algorithm, cc.dt = "piso", 0.1 / n
cfg = CouplingConfig.from_case_config(cc)
st = init_state(case, cfg)
print(f"n={n} cells={case.mesh.n_cells} setup {time.time() - t0:.2f}s dev bytes {st._ctx.device_bytes / 1e9:.2f} GB")
N = case.mesh.n_cells
for s in range(steps):
    nlog = len(st.residual_log)
    t = time.time()
    piso_time_step(st, cfg)
    dt = time.time() - t
    rows = st.residual_log[nlog:]
    print(f"step {s + 1}: {dt * 1e3:.1f} ms wall; solves " + ", ".join(f"{r[1]}:{r[3]}" for r in rows))
    print("   wall", {k: round(v * 1e3, 2) for k, v in st.wall.items()})
