"""Golden fixtures at the BASELINE configs' NAMED sizes, from the REAL reference
(test infrastructure; run in the build container, where /root/reference exists):

    python oracle/make_golden_full.py CASE [CASE ...]

CASE is one of
  c2_tight    gen_cavity(128) PISO dt 0.1/128, PISO steps 1-2 at cg_tol 1e-13,
              bicgstab_tol 1e-10, max_iters 20000 (fields: SURVEY.md §7 hard
              part 1 protocol (i))
  c2_default  the same two steps at the reference defaults (iteration
              counts: protocol (ii))
  c3_nh16     backward-facing step nh = 16 (16,640 cells) SIMPLE run to
              convergence by run_case (outer_tol 1e-5; 589 sweeps)
  c4_tight    perturbed + renumbered cavity 126^3 (2,000,376 cells), one PISO
              step at cg_tol 1e-13 / bicgstab_tol 1e-10 / max_iters 20000
  c4_default  PISO steps 1-2 at the reference defaults (iteration counts on
              the randomly renumbered mesh, where the device solvers run in
              RCM order; step 2 has non-trivial uy/uz solves)

Full 128^3 / 126^3 fields are ~120 MB per step, too big to commit, so each
step stores: full-field L2 norms (per u component, p, flux), a seeded
sample of 32768 cells (u, p) and 32768 faces (flux), the complete residual
log and the continuity error.  c3_nh16 stores its full final fields.
The C3/C4 meshes come from this repo's generators (the reference has none)
and are handed to the reference as reference Mesh objects, which validates
them (mesh.py:90-128); everything after that is the reference's own code.
Outputs: tests/golden/full_<case>.npz.  Wall time (1 thread): c2_* ~15-25
min, c3 ~7 min, c4_* ~10-20 min.
"""

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
REF = "/root/reference/pkg/src"
NSAMPLE = 32768
TIGHT = dict(cg_tol=1e-13, bicgstab_tol=1e-10, max_iters=20000)


def _ref():
    sys.path.insert(0, REF)
    import fvflow.cases as rcases
    import fvflow.coupling as rcoup
    import fvflow.mesh as rmesh
    from fvflow.config import BoundarySpec, CaseConfig

    return rcases, rcoup, rmesh, BoundarySpec, CaseConfig


def _from_repo(R, mc):
    """Repo-generated Case -> reference Case (mesh validated by the reference)."""
    rcases, _, rmesh, BoundarySpec, CaseConfig = R
    m = mc.mesh
    rm = rmesh.Mesh(points=m.points, face_points=m.face_points, face_offsets=m.face_offsets,
                    owner=m.owner, neighbour=m.neighbour,
                    patches=[rmesh.Patch(p.name, p.kind, p.start, p.count) for p in m.patches],
                    n_cells=m.n_cells)
    rm.validate()
    cc = CaseConfig(**{k: getattr(mc.config, k) for k in mc.config.__dataclass_fields__
                       if k not in ("boundary", "samples")})
    cc.boundary = {k: BoundarySpec(u=v.u, p=v.p) for k, v in mc.config.boundary.items()}
    return rcases.Case(mc.name, rm, cc)


def make(R, name):
    rcases = R[0]
    if name.startswith("c2"):
        c = rcases.gen_cavity(128)
        c.config.algorithm, c.config.dt = "piso", 0.1 / 128
        steps = 2
    elif name == "c3_nh16":
        sys.path.insert(0, REPO)
        from paper_1207_1571_b200 import cases as mycases

        return _from_repo(R, mycases.gen_backward_step(16)), None
    else:
        sys.path.insert(0, REPO)
        from paper_1207_1571_b200 import cases as mycases

        c = _from_repo(R, mycases.perturbed_cavity(126))
        steps = 2 if name == "c4_default" else 1
    if name.endswith("tight"):
        for k, v in TIGHT.items():
            setattr(c.config, k, v)
    return c, steps


def sample_idx(n, seed):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(NSAMPLE, n), replace=False))


def log_arrays(rows):
    return (np.array([f"{a}:{b}" for a, b, *_ in rows]),
            np.array([[c, d, e, f] for _, _, c, d, e, f in rows], dtype=float))


def run(name):
    R = _ref()
    rcoup = R[1]
    t0 = time.perf_counter()
    case, steps = make(R, name)
    cc = case.config
    out = {"cfg_cg_tol": np.float64(cc.cg_tol), "cfg_bicgstab_tol": np.float64(cc.bicgstab_tol),
           "cfg_max_iters": np.int64(cc.max_iters), "n_cells": np.int64(case.mesh.n_cells),
           "n_faces": np.int64(case.mesh.n_faces),
           "blas_threads": np.array(os.environ.get("OPENBLAS_NUM_THREADS", ""))}
    if steps is None:  # C3: run_case to convergence, full fields
        st = rcoup.run_case(case)
        out.update(u=st.u.values, p=st.p.values, flux=st.flux, sweeps=np.int64(st.outer),
                   converged=np.bool_(st.converged),
                   cont=np.float64(rcoup.continuity_error(st)))
        out["log_names"], out["log"] = log_arrays(st.residual_log)
    else:
        cfg = rcoup.CouplingConfig.from_case_config(cc)
        st = rcoup.init_state(case, cfg)
        ci = sample_idx(case.mesh.n_cells, 1207)
        fi = sample_idx(case.mesh.n_faces, 1208)
        out.update(sample_cells=ci, sample_faces=fi, steps=np.int64(steps))
        for s in range(steps):
            n0 = len(st.residual_log)
            ts = time.perf_counter()
            r = rcoup.piso_time_step(st, cfg)
            out[f"s{s}_wall"] = np.float64(time.perf_counter() - ts)
            out[f"s{s}_ret"] = np.array(r, dtype=float)
            u, p, f = st.u.values, st.p.values, st.flux
            out[f"s{s}_norm_u"] = np.linalg.norm(u, axis=0)
            out[f"s{s}_norm_p"] = np.float64(np.linalg.norm(p))
            out[f"s{s}_norm_flux"] = np.float64(np.linalg.norm(f))
            out[f"s{s}_u"] = u[ci]
            out[f"s{s}_p"] = p[ci]
            out[f"s{s}_flux"] = f[fi]
            out[f"s{s}_log_names"], out[f"s{s}_log"] = log_arrays(st.residual_log[n0:])
            out[f"s{s}_cont"] = np.float64(rcoup.continuity_error(st))
            print(f"{name} step {s + 1}: {time.perf_counter() - ts:.1f} s, log "
                  f"{[(a, b, d) for a, b, _, d, *_ in st.residual_log[n0:]]}", flush=True)
    out["wall_total"] = np.float64(time.perf_counter() - t0)
    path = os.path.join(OUT, f"full_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {case.mesh.n_cells} cells -> {path} ({out['wall_total']:.0f} s)", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        run(nm)
