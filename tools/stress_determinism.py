"""Determinism stress: the solvers and FV kernels are
deterministic by construction (fixed reduction order, no atomics), so any
run-to-run difference would expose a memory-ordering race in the persistent
kernels' grid barrier.

    python tools/stress_determinism.py [--edge 128] [--fresh 20] [--reseed 200]
                                       [--big 256] [--out profiles/r02_stress.jsonl]

* reseed: one context, the two PISO steps of tests/test_gpu_fullsize.py::
  test_c2_cavity128_two_steps re-run R times from the same initial state;
* fresh: the same two steps from a fresh init_state (new context, new
  allocations) F times;
* big: two fresh runs of two PISO steps on gen_cavity(BIG), compared bitwise.

Every run logs its per-launch device results (solver, field, iterations,
initial and final residual of every solve) and a SHA-1 of u, p, flux; all
are compared bitwise with run 0.  One JSON line per run, then a summary.
"""

import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
if os.environ.get("FVB_PKG_ROOT"):  # A/B of diagnostic builds (tools/build_variant.py)
    sys.path.insert(0, os.environ["FVB_PKG_ROOT"])

from paper_1207_1571_b200 import cases  # noqa: E402
from paper_1207_1571_b200.coupling import (CouplingConfig, continuity_error,  # noqa: E402
                                           init_state, piso_time_step)


def cavity(n):
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    if n > 128:
        case.config.max_iters = 5000
    return case, CouplingConfig.from_case_config(case.config)


def digest(st):
    h = hashlib.sha1()
    for a in (st.u.values, st.p.values, st.flux):
        h.update(a.tobytes())
    return h.hexdigest()


def two_steps(st, cfg):
    n0 = len(st.residual_log)
    for _ in range(2):
        piso_time_step(st, cfg)
    return [list(r[:4]) + [float(r[4]).hex(), float(r[5]).hex()] for r in st.residual_log[n0:]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edge", type=int, default=128)
    ap.add_argument("--fresh", type=int, default=20)
    ap.add_argument("--reseed", type=int, default=200)
    ap.add_argument("--big", type=int, default=256)
    ap.add_argument("--out", default="profiles/r02_stress.jsonl")
    ap.add_argument("--step2", type=int, default=0,
                    help="R repeats of PISO step 2 alone from the saved step-1 state")
    a = ap.parse_args()
    out = open(a.out, "w")
    fails = []

    def emit(kind, i, log, dg, extra=None):
        rec = {"kind": kind, "run": i, "digest": dg, "log": log}
        rec.update(extra or {})
        out.write(json.dumps(rec) + "\n")
        out.flush()

    case, cfg = cavity(a.edge)
    if a.step2:
        st = init_state(case, cfg)
        piso_time_step(st, cfg)
        s1 = (st.u.values.copy(), st.p.values.copy(), st.flux.copy(), st.u.boundary.copy(),
              st.p.boundary.copy(), st.outer, st.t)
        ref = None
        t0 = time.time()
        for i in range(a.step2):
            st.u.values, st.p.values, st.flux = s1[0], s1[1], s1[2]
            st.u.boundary, st.p.boundary = s1[3], s1[4]
            st.outer, st.t = s1[5], s1[6]
            n0 = len(st.residual_log)
            piso_time_step(st, cfg)
            log = [list(r[:4]) + [float(r[4]).hex(), float(r[5]).hex()]
                   for r in st.residual_log[n0:]]
            dg = digest(st)
            emit("step2", i, log, dg)
            if ref is None:
                ref = (log, dg)
            elif (log, dg) != ref:
                fails.append(("step2", i))
                print(f"  step2 {i}: MISMATCH {[r[3] for r in log]}", flush=True)
        print(f"step2 x{a.step2}: {time.time() - t0:.1f} s, mismatches {len(fails)}", flush=True)
        out.write(json.dumps({"summary": True, "step2": a.step2, "mismatches": fails}) + "\n")
        out.close()
        sys.exit(1 if fails else 0)
    t0 = time.time()
    st = init_state(case, cfg)
    u0, p0, f0 = st.u.values.copy(), st.p.values.copy(), st.flux.copy()
    ub0, pb0 = st.u.boundary.copy(), st.p.boundary.copy()
    ref_log = two_steps(st, cfg)
    ref_dg = digest(st)
    cont = continuity_error(st)
    emit("reseed", 0, ref_log, ref_dg, {"continuity": cont})
    print(f"edge {a.edge}: reference run {time.time() - t0:.1f} s, cg "
          f"{[r[3] for r in ref_log if r[0] == 'cg']}", flush=True)
    t0 = time.time()
    for i in range(1, a.reseed + 1):
        st.u.values, st.p.values, st.flux = u0, p0, f0
        st.u.boundary, st.p.boundary = ub0, pb0
        st.outer, st.t = 0, 0.0
        log = two_steps(st, cfg)
        dg = digest(st)
        emit("reseed", i, log, dg)
        if log != ref_log or dg != ref_dg:
            fails.append(("reseed", i))
            print(f"  reseed {i}: MISMATCH", flush=True)
    print(f"reseed x{a.reseed}: {time.time() - t0:.1f} s, mismatches "
          f"{sum(1 for f in fails if f[0] == 'reseed')}", flush=True)
    del st
    t0 = time.time()
    for i in range(a.fresh):
        s2 = init_state(case, cfg)
        log = two_steps(s2, cfg)
        dg = digest(s2)
        emit("fresh", i, log, dg)
        if log != ref_log or dg != ref_dg:
            fails.append(("fresh", i))
            print(f"  fresh {i}: MISMATCH", flush=True)
        del s2
    print(f"fresh x{a.fresh}: {time.time() - t0:.1f} s, mismatches "
          f"{sum(1 for f in fails if f[0] == 'fresh')}", flush=True)
    big = None
    if a.big:
        caseb, cfgb = cavity(a.big)
        runs = []
        for i in range(2):
            t0 = time.time()
            sb = init_state(caseb, cfgb)
            log = two_steps(sb, cfgb)
            dg = digest(sb)
            emit(f"big{a.big}", i, log, dg)
            runs.append((log, dg))
            print(f"big {a.big} run {i}: {time.time() - t0:.1f} s cg "
                  f"{[r[3] for r in log if r[0] == 'cg']}", flush=True)
            del sb
        big = runs[0] == runs[1]
        if not big:
            fails.append((f"big{a.big}", 1))
    summary = {"summary": True, "edge": a.edge, "reseed": a.reseed, "fresh": a.fresh,
               "big": a.big, "big_bitwise_equal": big, "mismatches": fails}
    out.write(json.dumps(summary) + "\n")
    out.close()
    print(json.dumps(summary))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
