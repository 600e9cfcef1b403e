"""Parity at the BASELINE configurations' NAMED sizes against the real
reference (fixtures tests/golden/full_*.npz, made by oracle/make_golden_full.py
from /root/reference's own run_case / piso_time_step).

* C2 gen_cavity(128), PISO steps 1-2: fields (u, p, phi on a seeded
  32768-cell / 32768-face sample, plus full-field norms) within 1e-8
  relative L2 at cg_tol 1e-13 / bicgstab_tol 1e-10 (SURVEY.md §7 hard part
  1 protocol (i)); iteration counts at the reference defaults, CG +-1 and
  BiCGStab +-2 per solve (protocol (ii)).
* C3 backward-facing step nh = 16 (16,640 cells), SIMPLE run to convergence
  by run_case: number of sweeps, converged fields, continuity; per-solve
  counts over the first sweeps (uz of the one-cell-thick mesh excluded, as
  SURVEY.md §7 prescribes: its rhs is round-off).
* C4 perturbed + randomly renumbered 126^3 cavity (2,000,376 cells; the
  device solvers run in RCM order): one PISO step's fields at tight
  tolerances, two steps' counts at defaults.

Counts at default tolerances are judged around the spread of the
reference's OWN counts under 1-ulp reorderings of its arithmetic (OpenBLAS
thread count, SpMV summation order; tests/golden/floor_*.json from
oracle/noise_floor.py), as SURVEY.md §7 hard part 1 prescribes: e.g. the
step-1 ux BiCGStab solve of C2 takes 67, 69 or 70 iterations in the
reference depending on that order alone.
"""

import os

import numpy as np
import pytest

from golden_io import rel
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import (CouplingConfig, continuity_error, init_state,
                                           piso_time_step, run_case)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIELD_TOL = 1e-8
TIGHT = dict(cg_tol=1e-13, bicgstab_tol=1e-10, max_iters=20000)


def _gold(name):
    return np.load(os.path.join(GOLD, f"full_{name}.npz"))


def _log_rows(names, log):
    return [(str(nm).split(":")[0], str(nm).split(":")[1], int(r[0]), int(r[1]))
            for nm, r in zip(names, log)]


def _check_counts(mine, ref, skip_uz=False, spread=None):
    """CG +-1, BiCGStab +-2 per solve, same solve sequence.  spread: per
    solve (lo, hi) of the reference's own counts under 1-ulp reorderings
    (tests/golden/floor_*.json, oracle/noise_floor.py; SURVEY.md §7 hard part
    1: counts are judged next to the CPU-vs-CPU floor): the bound then
    applies around [lo, hi] instead of the single golden count, and is at
    least hi - lo (C4's step-1 ux solve takes 68, 72 or 73 iterations in
    the reference depending on the summation order alone)."""
    assert [(a[0], a[1], a[2]) for a in mine] == [(b[0], b[1], b[2]) for b in ref]
    bad = []
    for j, (a, b) in enumerate(zip(mine, ref)):
        if skip_uz and a[1] == "uz":
            continue
        lo, hi = spread[j] if spread else (b[3], b[3])
        # the parity rule, widened to the reference's own spread for a solve
        # whose count moves by more than that under a 1-ulp reordering (the
        # device order is one more such reordering)
        tol = max(1 if a[0] == "cg" else 2, hi - lo)
        if not (lo - tol <= a[3] <= hi + tol):
            bad.append((a, b, (lo, hi)))
    assert not bad, bad


def _floor_spread(case, step, ref):
    """(lo, hi) per solve of step `step` over the golden run and every
    committed reference floor run of `case`."""
    import glob
    import json

    counts = [[r[3]] for r in ref]
    for path in sorted(glob.glob(os.path.join(GOLD, f"floor_{case}_*.json"))):
        with open(path) as f:
            steps = json.load(f)["steps"]
        if step < len(steps):
            for j, row in enumerate(steps[step]):
                counts[j].append(int(row[2]))
    return [(min(c), max(c)) for c in counts]


def _cavity(n, tight):
    case = cases.gen_cavity(n)
    case.config.algorithm, case.config.dt = "piso", 0.1 / n
    if tight:
        for k, v in TIGHT.items():
            setattr(case.config, k, v)
    return case


def _steps(case, g):
    cfg = CouplingConfig.from_case_config(case.config)
    st = init_state(case, cfg)
    ci, fi = g["sample_cells"], g["sample_faces"]
    out = []
    for s in range(int(g["steps"])):
        n0 = len(st.residual_log)
        piso_time_step(st, cfg)
        u, p, f = st.u.values, st.p.values, st.flux
        err = {"u": rel(u[ci], g[f"s{s}_u"]), "p": rel(p[ci], g[f"s{s}_p"]),
               "flux": rel(f[fi], g[f"s{s}_flux"]),
               "norm_u": float(np.max(np.abs(np.linalg.norm(u, axis=0) / g[f"s{s}_norm_u"] - 1))),
               "norm_p": abs(np.linalg.norm(p) / float(g[f"s{s}_norm_p"]) - 1),
               "norm_flux": abs(np.linalg.norm(f) / float(g[f"s{s}_norm_flux"]) - 1)}
        rows = [(r[0], r[1], 0, r[3]) for r in st.residual_log[n0:]]
        ref = [(a, b, 0, n) for a, b, _, n in _log_rows(g[f"s{s}_log_names"], g[f"s{s}_log"])]
        out.append((err, rows, ref, continuity_error(st), np.abs(f).max()))
    return out


def _fields_ok(results):
    for s, (err, _rows, _ref, cont, fmax) in enumerate(results):
        assert max(err.values()) < FIELD_TOL, (s, err)
        assert cont <= 1e-8 * fmax


@pytest.mark.slow
def test_c2_cavity128_fields_tight_tolerances():
    g = _gold("c2_tight")
    res = _steps(_cavity(128, True), g)
    _fields_ok(res)
    for _err, rows, ref, _c, _m in res:
        # counts at tightened tolerances follow the dot-product rounding
        # (BiCGStab +-3 between two CPU orderings at 64^3)
        for a, b in zip(rows, ref):
            assert abs(a[3] - b[3]) <= (2 if a[0] == "cg" else max(3, b[3] // 10)), (a, b)


@pytest.mark.slow
def test_c2_cavity128_iteration_counts_defaults():
    g = _gold("c2_default")
    for s, (_err, rows, ref, cont, fmax) in enumerate(_steps(_cavity(128, False), g)):
        _check_counts(rows, ref, spread=_floor_spread("c2", s, ref))
        assert cont <= 1e-8 * fmax


def _c4(tight):
    case = cases.perturbed_cavity(126)
    if tight:
        for k, v in TIGHT.items():
            setattr(case.config, k, v)
    return case


@pytest.mark.slow
def test_c4_perturbed_126_fields_tight_tolerances_rcm():
    g = _gold("c4_tight")
    res = _steps(_c4(True), g)
    _fields_ok(res)


@pytest.mark.slow
def test_c4_perturbed_126_iteration_counts_defaults_rcm():
    g = _gold("c4_default")
    for s, (_err, rows, ref, cont, fmax) in enumerate(_steps(_c4(False), g)):
        _check_counts(rows, ref, spread=_floor_spread("c4", s, ref))
        assert cont <= 1e-8 * fmax


def test_c3_backward_step_nh16_simple_to_convergence():
    g = _gold("c3_nh16")
    case = cases.gen_backward_step(16)
    st = run_case(case)
    assert st.converged and bool(g["converged"])
    ref = _log_rows(g["log_names"], g["log"])
    mine = [(r[0], r[1], r[2], r[3]) for r in st.residual_log]
    # the first sweeps solve identical systems up to rounding: counts per
    # solve within the parity rule (uz of the one-cell-thick mesh excluded)
    n_early = 4 * 20
    _check_counts(mine[:n_early], ref[:n_early], skip_uz=True)
    # the converged state: same number of sweeps to outer_tol, fields within
    # the field tolerance, continuity at the reference's level
    assert abs(st.outer - int(g["sweeps"])) <= 1, (st.outer, int(g["sweeps"]))
    errs = {"u": rel(st.u.values[:, :2], g["u"][:, :2]), "p": rel(st.p.values, g["p"]),
            "flux": rel(st.flux, g["flux"])}
    assert max(errs.values()) < FIELD_TOL, errs
    assert continuity_error(st) <= 1e-8 * np.abs(st.flux).max()


@pytest.mark.slow
def test_reseeded_one_step_64_vs_oracle():
    """SURVEY.md §7 hard part 1 protocol (iii): one PISO step of gen_cavity(64)
    from the same seeded non-trivial state on the device and in the oracle
    (oracle/fvoracle.py, pinned to the reference), at tightened tolerances."""
    from oracle import fvoracle as O
    from paper_1207_1571_b200.mesh import compute_geometry

    n = 64
    case = _cavity(n, True)
    cfg = CouplingConfig.from_case_config(case.config)
    geo = compute_geometry(case.mesh)
    x, y, z = (geo.cell_centroid[:, k] / 0.1 for k in range(3))
    rng = np.random.default_rng(1207)
    ph = rng.uniform(0, 2 * np.pi, size=6)
    u0 = np.stack([0.3 * np.sin(np.pi * x + ph[0]) * np.cos(np.pi * y) * np.sin(np.pi * z + ph[1]),
                   0.2 * np.cos(np.pi * x) * np.sin(np.pi * y + ph[2]) * np.sin(np.pi * z),
                   0.1 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.cos(np.pi * z + ph[3])], axis=1)
    p0 = 0.05 * np.cos(np.pi * x + ph[4]) * np.cos(np.pi * y + ph[5]) * np.cos(np.pi * z)
    run = O.Run(case.mesh, case.config)
    run.u.values[:] = u0
    run.p.values[:] = p0
    O.apply_bcs(run.u, run.g, cfg.dt)
    O.apply_bcs(run.p, run.g, cfg.dt)
    flux0 = run._plain_flux()
    run.flux = flux0.copy()
    run.outer = 1
    st = init_state(case, cfg)
    st.u.values, st.p.values, st.flux = u0, p0, flux0
    st.outer, st.t = 1, cfg.dt
    piso_time_step(st, cfg)
    run.piso_step()
    errs = {"u": rel(st.u.values, run.u.values), "p": rel(st.p.values, run.p.values),
            "flux": rel(st.flux, run.flux)}
    assert max(errs.values()) < FIELD_TOL, errs
    for a, b in zip(st.residual_log, run.log):
        assert (a[0], a[1]) == (b[0], b[1])
        assert abs(a[3] - b[3]) <= (2 if a[0] == "cg" else max(3, b[3] // 10)), (a, b)
