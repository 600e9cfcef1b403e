"""Benchmark: FP64 PISO time steps of the 3D lid-driven cavity on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c5] [--n CELLS_PER_EDGE]

Workload (BASELINE.json configs[1], "C2"): gen_cavity(128) (2,097,152 hex
cells, K = 7), PISO with the reference defaults (cg_tol 1e-10,
bicgstab_tol 1e-8, max_iters 2000, 2 correctors), dt = 0.1/128 (Co = 1),
from rest; W warm-up steps, then K timed steps.  The working set (matrix,
pattern, Krylov vectors: ~1.4 GB) is larger than the 126 MB L2, so no
flush is needed between steps.

One JSON line on rank 0:
  value        cell-updates/s = cells / (device ms per step), device-resident
  e2e          same metric through the C ABI with pinned HOST buffers: each
               step uploads u, p, flux and downloads them again
  roofline     the dominant kernel (persistent Jacobi-PCG, k_cg): algorithmic
               bytes per launch N(12K+80) + iters*N(12K+96)
               over its CUDA-event duration, against MEASURED_PEAKS hbm_gbs
  cpu_baseline the reference fvflow (baseline/_ref, unmodified) on a bounded
               sample of the same step, extrapolated with the step's counts
--impl reference prints the reference arm's line (CPU, no GPU work).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

HBM_FALLBACK = 6650.0  # B200_PROFILING.md fallback, only if MEASURED_PEAKS.json is absent
REF_DIR = os.path.join(HERE, "baseline", "_ref")
# reference iteration counts of gen_cavity(128) PISO step 2 measured on the
# reference itself: CG 1494 + 1510, BiCGStab 65 + 62 + 66
REF_COUNTS_C2 = {"cg": 3004, "cg_solves": 2, "bicgstab": 193, "bicgstab_solves": 3}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c5"])
    ap.add_argument("--n", type=int, default=0, help="override cells per edge")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cg-sample", type=int, default=20)
    return ap.parse_args()


def workload(args):
    n = args.n or (128 if args.config == "c2" else 256)
    return n


def peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, v in zip(names, r[3:7]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_case(n):
    from paper_1207_1571_b200 import cases

    case = cases.gen_cavity(n)
    cc = case.config
    cc.algorithm = "piso"
    cc.dt = 0.1 / n
    if n > 128:
        cc.max_iters = 5000  # the 2000 cap binds at 256^3
    return case


# ------------------------------------------------------------ reference arm
def _ref_modules():
    if not os.path.isdir(os.path.join(REF_DIR, "fvflow")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import fvflow.coupling as rc
    import fvflow.fvm as rf
    import fvflow.linsolve as rl
    import fvflow.mesh as rm
    import fvflow.sparse as rs
    from fvflow.config import BoundarySpec, CaseConfig

    return rc, rf, rl, rm, rs, BoundarySpec, CaseConfig


class RefSampler:
    """Bounded samples of the reference's own piso_time_step on the same
    workload.  The reference objects are built from this package's setup
    arrays, which are bit-identical to the reference's own compute_geometry
    / build_pattern (tests/test_native_setup.py) — that skips its 30-50 s
    numpy setup.  Each sample is one reference step with CG capped at cg_cap
    and BiCGStab at bi_cap iterations per solve: assembly and correction
    are timed in full, solver time per iteration is scaled to the full
    step's iteration counts."""

    def __init__(self, case, seed=None, cg_cap=20, bi_cap=10):
        mods = _ref_modules()
        self.ok = mods is not None
        if not self.ok:
            return
        rc, rf, rl, rm, rs, BoundarySpec, CaseConfig = mods
        from paper_1207_1571_b200 import mesh as pmesh, sparse as psparse

        self.rc, self.rs = rc, rs
        m = case.mesh
        rmesh = rm.Mesh(points=m.points, face_points=m.face_points, face_offsets=m.face_offsets,
                        owner=m.owner, neighbour=m.neighbour,
                        patches=[rm.Patch(p.name, p.kind, p.start, p.count) for p in m.patches],
                        n_cells=m.n_cells)
        g = pmesh.compute_geometry(m)
        geom = rm.MeshGeometry(**{k: getattr(g, k) for k in g.__dataclass_fields__})
        pp = psparse.build_pattern(m)
        self.pat = rs.SparsityPattern(**{k: getattr(pp, k) for k in pp.__dataclass_fields__})
        cc = CaseConfig(**{k: getattr(case.config, k) for k in case.config.__dataclass_fields__
                           if k not in ("boundary", "samples")})
        cc.boundary = {k: BoundarySpec(u=v.u, p=v.p) for k, v in case.config.boundary.items()}
        self.cfg = rc.CouplingConfig.from_case_config(cc)
        self.cfg.pressure.max_iters = cg_cap
        self.cfg.momentum.max_iters = bi_cap
        ub = {k: rf.bc_from_tuple(s.u) for k, s in cc.boundary.items()}
        pb = {k: rf.bc_from_tuple(s.p) for k, s in cc.boundary.items()}
        u = rf.make_vector("u", rmesh, ub)
        p = rf.make_scalar("p", rmesh, pb)
        if seed is not None:
            u.values = seed["u"].copy()
            p.values = seed["p"].copy()
        rf.apply_bcs(u, geom, 0.0)
        rf.apply_bcs(p, geom, 0.0)
        flux = seed["flux"].copy() if seed is not None else rc._plain_flux(u, geom)
        self.state = rc.RunState(mesh=rmesh, geom=geom, pattern=self.pat, u=u, p=p, flux=flux,
                                 pin_pressure=True)
        self.start = (u.values.copy(), p.values.copy(), flux.copy(),
                      seed["outer"] if seed is not None else 0)
        self.n = m.n_cells

    def sample(self, counts):
        rc, rs, st = self.rc, self.rs, self.state
        st.u.values = self.start[0].copy()
        st.p.values = self.start[1].copy()
        st.flux = self.start[2].copy()
        st.outer = self.start[3]
        st.wall, st.residual_log = {}, []
        A = rs.HybridMatrix.zeros(self.pat)
        A.V[:] = 1.0
        t = time.perf_counter()
        rs.smvp(A, np.ones(self.n))
        t_smvp = time.perf_counter() - t
        t0 = time.perf_counter()
        rc.piso_time_step(st, self.cfg)
        t_sample = time.perf_counter() - t0
        w = st.wall
        cg_rows = [r for r in st.residual_log if r[0] == "cg"]
        bi_rows = [r for r in st.residual_log if r[0] == "bicgstab"]
        cg_it = sum(r[3] for r in cg_rows)
        bi_it = sum(r[3] for r in bi_rows)
        t_cg_iter = max(w.get("pressure_solve", 0.0) - len(cg_rows) * t_smvp, 0.0) / max(cg_it, 1)
        t_bi_iter = max(w.get("momentum_solve", 0.0) - len(bi_rows) * t_smvp, 0.0) / max(bi_it, 1)
        fixed = (w.get("momentum_assembly", 0.0) + w.get("pressure_assembly", 0.0)
                 + w.get("correction", 0.0))
        t_step = (fixed + counts["cg_solves"] * t_smvp + counts["cg"] * t_cg_iter
                  + counts["bicgstab_solves"] * t_smvp + counts["bicgstab"] * t_bi_iter)
        return {"s_per_step": t_step, "sample_s": t_sample, "t_cg_iter_s": t_cg_iter,
                "t_bicgstab_iter_s": t_bi_iter, "t_smvp_s": t_smvp,
                "assembly_correction_s": fixed,
                "sampled_iters": {"cg": cg_it, "bicgstab": bi_it}, "counts": counts,
                "threads": os.environ.get("OPENBLAS_NUM_THREADS", "default")}


def reference_sample(case, counts, seed=None, cg_cap=20, bi_cap=10):
    s = RefSampler(case, seed, cg_cap, bi_cap)
    return s.sample(counts) if s.ok else None


def run_reference(args):
    n = workload(args)
    case = make_case(n)
    N = case.mesh.n_cells
    counts = dict(REF_COUNTS_C2)
    if n != 128:  # scale counts like the CG iteration growth (~2x per doubling)
        f = n / 128
        counts = {"cg": int(3004 * f), "cg_solves": 2, "bicgstab": int(193 * f),
                  "bicgstab_solves": 3}
    times = []
    detail = None
    sampler = RefSampler(case, cg_cap=args.cg_sample)
    if not sampler.ok:
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref/fvflow not installed"}))
        return
    # warm-up: the CPU code has nothing to JIT; W SpMV calls touch the data
    A = sampler.rs.HybridMatrix.zeros(sampler.pat)
    for _ in range(args.warmup):
        sampler.rs.smvp(A, np.ones(sampler.n))
    for _ in range(args.steps):
        d = sampler.sample(counts)
        times.append(d["s_per_step"])
        detail = d
    ms = 1e3 * statistics.mean(times)
    value = N / (ms / 1e3)
    sample = (f"reference fvflow piso_time_step on gen_cavity({n}); CG capped at "
              f"{args.cg_sample} and BiCGStab at 10 iterations per solve, assembly and "
              f"correction timed in full; per-iteration costs scaled to the reference's own "
              f"step-2 counts (CG {counts['cg']}, BiCGStab {counts['bicgstab']}, SURVEY.md §6)")
    cores = os.cpu_count()
    out = {
        "metric": "cell-updates/s (FP64 PISO time step)", "impl": "reference",
        "value": value, "unit": "cell-updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_cavity mesh, from rest)",
        "config": {"workload": f"C2 gen_cavity({n}) PISO dt=0.1/{n}", "cells": N,
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "detail": detail,
    }
    print(json.dumps(out))


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import ctypes as C

    from paper_1207_1571_b200 import _lib
    from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        raise SystemExit("multi-GPU domain decomposition is not wired into bench.py yet")
    n = workload(args)
    t_setup = time.perf_counter()
    case = make_case(n)
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    t_setup = time.perf_counter() - t_setup
    mesh = case.mesh
    N, F = mesh.n_cells, mesh.n_faces
    K = st.pattern.k
    h = st._ctx.h
    for _ in range(args.warmup):
        piso_time_step(st, cfg)
    # seed for the CPU reference sample: the state the timed steps start from
    seed = None
    if not args.no_cpu_baseline:
        seed = {"u": st.u.values.copy(), "p": st.p.values.copy(), "flux": st.flux.copy(),
                "outer": st.outer}
        st._dev.host_dirty.clear()
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    nlog = len(st.residual_log)
    l0 = _lib.lib.fvb_launch_count()
    _lib.check(_lib.lib.fvb_sync(h))
    _lib.check(_lib.lib.fvb_timer_start(h))
    kernel_rows = []
    for _ in range(args.steps):
        piso_time_step(st, cfg)
        kernel_rows.extend(st._last_solves)
    ms = C.c_double()
    _lib.check(_lib.lib.fvb_timer_stop(h, C.byref(ms)))
    launches = _lib.lib.fvb_launch_count() - l0
    clk = clocks.stop()
    ms_step = ms.value / args.steps
    rows = st.residual_log[nlog:]
    cg_iters = [r[3] for r in rows if r[0] == "cg"]
    bi_iters = [r[3] for r in rows if r[0] == "bicgstab"]
    # dominant kernel: persistent PCG (k_cg)
    cg_k = [(it, ks) for (solver, it, ks) in kernel_rows if solver == "cg"]
    b_setup = N * (12 * K + 80)
    b_iter = N * (12 * K + 96)
    cg_bytes = sum(b_setup + it * b_iter for it, _ in cg_k)
    cg_time = sum(ks for _, ks in cg_k)
    peak, peak_kind = peaks()
    achieved = cg_bytes / cg_time / 1e9 if cg_time > 0 else 0.0
    traffic = None
    prof = os.path.join(HERE, "profiles", "ncu_k_cg_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            pj = json.load(f)
        traffic = pj.get("bytes_per_launch")
    # whole-step algorithmic bytes: solves + ~3.2 kB/cell FV work
    bi_max = []
    per = 3
    for i in range(0, len(bi_iters), per):
        bi_max.append(max(bi_iters[i:i + per]))
    step_bytes = (cg_bytes + sum(bi_iters) * 160 * N + sum(bi_max) * 24 * K * N
                  + len(bi_max) * 3 * N * (12 * K + 56) + args.steps * 3200 * N)
    step_gbs = step_bytes / (ms.value / 1e3) / 1e9
    # ---------------------------------------------------------------- e2e
    u_h = np.ascontiguousarray(st.u.values.T).reshape(-1).copy()
    p_h = st.p.values.copy()
    f_h = st.flux.copy()
    st._dev.host_dirty.clear()
    bufs = (u_h, p_h, f_h)
    for b in bufs:
        _lib.check(_lib.lib.fvb_host_register(b.ctypes.data, b.nbytes))
    P = _lib.ptr
    scfg_state = st
    _lib.check(_lib.lib.fvb_sync(h))
    _lib.check(_lib.lib.fvb_timer_start(h))
    for _ in range(args.steps):
        _lib.check(_lib.lib.fvb_set_state(h, P(u_h), P(p_h), P(f_h), None, None))
        piso_time_step(scfg_state, cfg)
        _lib.check(_lib.lib.fvb_get_state(h, P(u_h), P(p_h), P(f_h), None, None))
    e2e_ms = C.c_double()
    _lib.check(_lib.lib.fvb_timer_stop(h, C.byref(e2e_ms)))
    for b in bufs:
        _lib.lib.fvb_host_unregister(b.ctypes.data)
    e2e_step = e2e_ms.value / args.steps
    io_bytes = sum(b.nbytes for b in bufs)
    # ------------------------------------------------------- cpu baseline
    cpu = None
    if seed is not None:
        counts = {"cg": statistics.mean(cg_iters) * 2 if cg_iters else 0,
                  "cg_solves": 2,
                  "bicgstab": sum(bi_iters) / max(args.steps, 1),
                  "bicgstab_solves": 3}
        d = reference_sample(case, counts, seed=seed, cg_cap=args.cg_sample)
        if d is not None:
            cpu = {"value": N / d["s_per_step"], "unit": "cell-updates/s",
                   "cores": os.cpu_count(), "kind": "reference",
                   "sample": (f"unmodified reference fvflow (baseline/_ref) piso_time_step from "
                              f"the same state as the timed steps, CG capped at "
                              f"{args.cg_sample} and BiCGStab at 10 iterations; assembly and "
                              f"correction timed in full, per-iteration solver cost scaled to "
                              f"this run's mean counts (CG {counts['cg']:.0f}, BiCGStab "
                              f"{counts['bicgstab']:.0f} per step); OpenBLAS default threads; "
                              f"{d['sample_s']:.1f} s of CPU work"),
                   "s_per_step": d["s_per_step"]}
    out = {
        "metric": "cell-updates/s (FP64 PISO time step)",
        "value": N / (ms_step / 1e3),
        "unit": "cell-updates/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (gen_cavity mesh, PISO from rest; steps W+1..W+K timed)",
        "config": {"workload": f"C2 gen_cavity({n}) PISO dt=0.1/{n} (Co=1), reference defaults",
                   "cells": N, "faces": F, "K": K, "parallelism": "single",
                   "l2": "inputs larger than L2 (device working set "
                         f"{st._ctx.device_bytes / 1e9:.2f} GB > 126 MB L2)",
                   "setup_s": round(t_setup, 2)},
        "e2e": {"value": N / (e2e_step / 1e3), "unit": "cell-updates/s",
                "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes,
                "ms_per_step": e2e_step},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": "k_cg (persistent PCG)",
                     "peak_kind": peak_kind,
                     "bytes_model": f"N*(12K+80) + iters*N*(12K+96), K={K}",
                     "launches": len(cg_k), "mean_iters": cg_bytes and
                     sum(it for it, _ in cg_k) / max(len(cg_k), 1)},
        "step_hbm": {"achieved_gbs": step_gbs, "frac": step_gbs / peak,
                     "bytes_per_step": step_bytes / args.steps},
        "iterations_per_step": {"cg": sum(cg_iters) / args.steps,
                                "bicgstab": sum(bi_iters) / args.steps},
        "gpu_launches": int(launches),
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))


def main():
    args = parse()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank == 0:
            run_reference(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
