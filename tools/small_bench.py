"""Small-mesh timing (BASELINE configs[0] C1: 2D cavity 20x20, 100 PISO
steps; and C3 BFS nh=16 SIMPLE): wall seconds per step on the device path."""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
if os.environ.get("FVB_PKG_ROOT"):  # A/B of diagnostic builds (tools/build_variant.py)
    sys.path.insert(0, os.environ["FVB_PKG_ROOT"])
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.cases import Case
from paper_1207_1571_b200.config import BoundarySpec, CaseConfig
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step, simple_outer_iteration

m = cases.box_mesh(20, 20, 1, 0.1, 0.1, 0.01, [("movingWall", "wall", ["y+"]), ("fixedWalls", "wall", ["x-", "x+", "y-"]), ("frontAndBack", "empty", ["z-", "z+"])])
cc = CaseConfig(); cc.nu, cc.algorithm, cc.dt, cc.end_time = 0.01, "piso", 0.005, 0.5
cc.boundary = {"movingWall": BoundarySpec(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
               "fixedWalls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
               "frontAndBack": BoundarySpec(u=("empty",), p=("empty",))}
case = Case("c1", m, cc)
cfg = CouplingConfig.from_case_config(cc)
st = init_state(case, cfg)
from paper_1207_1571_b200 import _lib
FLAGS = _lib.STEP_NO_GRAPHS if "--no-graphs" in sys.argv else 0  # A/B: direct launches
_lib.check(_lib.lib.fvb_set_solver_options(st._ctx.h, FLAGS))
piso_time_step(st, cfg)
import ctypes as C
from paper_1207_1571_b200 import _lib
h = st._ctx.h
t0 = time.perf_counter()
ccall = 0.0
l0 = _lib.lib.fvb_launch_count()
_lib.check(_lib.lib.fvb_timer_start(h))
for _ in range(99):
    piso_time_step(st, cfg)
    ccall += st._last_step_s
dev = C.c_double()
_lib.check(_lib.lib.fvb_timer_stop(h, C.byref(dev)))
dt = (time.perf_counter() - t0) / 99
launches = _lib.lib.fvb_launch_count() - l0
# wall per step, of which inside the C call (host launches + syncs), and the
# device time between the first and last event of the 99 steps
print(json.dumps({"case": "C1 cavity 20x20x1 PISO", "ms_per_step": 1e3 * dt,
                  "c_call_ms_per_step": 1e3 * ccall / 99, "device_span_ms_per_step": dev.value / 99,
                  "cg_iters_per_step": st.cum_iters["cg"] / 100, "reference_ms_per_step": 7.4,
                  "wall_sections_ms_per_step": {k: round(1e3 * v / 100, 4) for k, v in st.wall.items()},
                  "launches_per_step": launches / 99}))
case = cases.gen_backward_step(16)
cfg = CouplingConfig.from_case_config(case.config)
st = init_state(case, cfg)
_lib.check(_lib.lib.fvb_set_solver_options(st._ctx.h, FLAGS))
simple_outer_iteration(st, cfg)
t0 = time.perf_counter()
for _ in range(20):
    simple_outer_iteration(st, cfg)
dt = (time.perf_counter() - t0) / 20
print(json.dumps({"case": "C3 BFS nh=16 SIMPLE", "ms_per_sweep": 1e3 * dt,
                  "cg_iters_per_sweep": st.cum_iters["cg"] / 21, "reference_ms_per_sweep": 689}))
