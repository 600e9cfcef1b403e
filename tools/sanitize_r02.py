"""compute-sanitizer workload for the round-2 additions (diagnostic, not
the product): C1 PISO steps (single-block solvers, the split momentum batch,
step-graph capture and replay), a C3 nh=8 SIMPLE sweep (one-cluster
solvers), rhie_chow_flux, and a decomposed 2-rank step (flat team
reduction).  Run as: compute-sanitizer --tool memcheck python tools/sanitize_r02.py
(the decomposed step cannot complete under the sanitizer: it serialises the
co-resident ranks' kernels, which spin-wait for each other inside the
kernels, so the 20 s team watchdog fires — profiles/r02_memcheck.log)"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1207_1571_b200 import cases, fvm, mesh as pmesh
from paper_1207_1571_b200.cases import Case
from paper_1207_1571_b200.config import BoundarySpec, CaseConfig
from paper_1207_1571_b200.coupling import (CouplingConfig, init_state, piso_time_step,
                                           simple_outer_iteration)
from paper_1207_1571_b200.team import DecomposedRun

m = cases.box_mesh(20, 20, 1, 0.1, 0.1, 0.01, [("movingWall", "wall", ["y+"]), ("fixedWalls", "wall", ["x-", "x+", "y-"]), ("frontAndBack", "empty", ["z-", "z+"])])
cc = CaseConfig(); cc.nu, cc.algorithm, cc.dt, cc.end_time = 0.01, "piso", 0.005, 0.5
cc.boundary = {"movingWall": BoundarySpec(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
               "fixedWalls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
               "frontAndBack": BoundarySpec(u=("empty",), p=("empty",))}
cfg = CouplingConfig.from_case_config(cc)
st = init_state(Case("c1", m, cc), cfg)
for _ in range(3):
    piso_time_step(st, cfg)
print("c1 ok", st.residual_log[-1][:4], flush=True)

case = cases.gen_backward_step(8)
cfg3 = CouplingConfig.from_case_config(case.config)
s3 = init_state(case, cfg3)
for _ in range(2):
    simple_outer_iteration(s3, cfg3)
print("c3 ok", s3.residual_log[-1][:4], flush=True)

geo = pmesh.compute_geometry(st.u.mesh)
flux = fvm.rhie_chow_flux(st.u, st.p, np.full(st.u.mesh.n_cells, 2.0), geo)
print("rhie_chow ok", float(np.abs(flux).max()), flush=True)

case = cases.gen_cavity(12)
case.config.algorithm, case.config.dt = "piso", 0.1 / 12
cfgt = CouplingConfig.from_case_config(case.config)
run = DecomposedRun(case, cfgt, 2)
for _ in range(2):
    run.piso_time_step(cfgt)
run.close()
print("team ok", flush=True)
