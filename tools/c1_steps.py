"""C1 (2D cavity 20x20x1, PISO dt 0.005) for profiling: N steps through the
public API after a warm-up step.  Usage: python tools/c1_steps.py [N]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1207_1571_b200 import _lib, cases
from paper_1207_1571_b200.cases import Case
from paper_1207_1571_b200.config import BoundarySpec, CaseConfig
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step

m = cases.box_mesh(20, 20, 1, 0.1, 0.1, 0.01, [("movingWall", "wall", ["y+"]), ("fixedWalls", "wall", ["x-", "x+", "y-"]), ("frontAndBack", "empty", ["z-", "z+"])])
cc = CaseConfig(); cc.nu, cc.algorithm, cc.dt, cc.end_time = 0.01, "piso", 0.005, 0.5
cc.boundary = {"movingWall": BoundarySpec(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
               "fixedWalls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
               "frontAndBack": BoundarySpec(u=("empty",), p=("empty",))}
cfg = CouplingConfig.from_case_config(cc)
st = init_state(Case("c1", m, cc), cfg)
piso_time_step(st, cfg)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
l0 = _lib.lib.fvb_launch_count()
for _ in range(n):
    piso_time_step(st, cfg)
print("launches per step", (_lib.lib.fvb_launch_count() - l0) / n, "solves", st.residual_log[-5:])
