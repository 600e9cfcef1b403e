"""C4 timing: PISO on the perturbed + randomly renumbered 126^3 cavity
(2,000,376 cells, BASELINE configs[3]); the renumbering leaves no common
column-offset tuples, so the solvers run on explicit indices and CG in the
solver's internal RCM order ("norcm": original order, FVB_SOLVER_NO_RCM).
Device ms per step (CUDA events) and CG iterations.
Usage: python tools/c4_bench.py [norcm]"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1207_1571_b200 import _lib, cases
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step

case = cases.perturbed_cavity(126)
cfg = CouplingConfig.from_case_config(case.config)
st = init_state(case, cfg)
h = st._ctx.h
if "norcm" in sys.argv[1:]:
    _lib.check(_lib.lib.fvb_set_solver_options(h, _lib.SOLVER_NO_RCM))
for _ in range(2):
    piso_time_step(st, cfg)
nc, ne, rcm = C.c_int(), C.c_int64(), C.c_int64()
_lib.check(_lib.lib.fvb_pattern_codes(h, C.byref(nc), C.byref(ne), None, C.byref(rcm)))
steps = 3
n0 = len(st.residual_log)
_lib.check(_lib.lib.fvb_sync(h))
_lib.check(_lib.lib.fvb_timer_start(h))
for _ in range(steps):
    piso_time_step(st, cfg)
ms = C.c_double()
_lib.check(_lib.lib.fvb_timer_stop(h, C.byref(ms)))
cg = [r[3] for r in st.residual_log[n0:] if r[0] == "cg"]
print(json.dumps({"workload": "C4 perturbed_cavity(126)", "cells": case.mesh.n_cells,
                  "ms_per_step": ms.value / steps, "cg_iters_per_step": sum(cg) / steps,
                  "stencil_codes": nc.value, "escaped_rows": ne.value,
                  "solves_in_rcm_order": rcm.value}))
