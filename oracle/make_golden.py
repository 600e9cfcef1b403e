"""Generate golden vectors from the REAL reference (test infrastructure).

Run in the build container, where /root/reference exists:

    python oracle/make_golden.py

It imports fvflow from /root/reference/pkg/src (with a 2-line matplotlib
stub so nothing else is needed), runs the reference's own functions on
small seeded inputs and stores inputs + outputs as compressed .npz files
under tests/golden/.  Those fixtures pin both the numpy oracle
(oracle/fvoracle.py) and the CUDA path; they travel to the GPU box, the
reference does not.

Cases (all small enough for seconds of CPU):
  cav6   gen_cavity(6) PISO, dt 0.1/6, 3 steps           (config C2 shape)
  chan   gen_channel(12, 4) PISO, sine inlet, 3 steps   (empty + outlet p)
  duct   gen_skewed_duct(8, 6, 30) SIMPLE, 3 sweeps      (non-orthogonal)
  pcav5  perturbed + renumbered cavity 5^3 PISO, 2 steps (config C4 recipe)
  bfs2   backward-facing step nh=2 SIMPLE, 3 sweeps      (config C3 recipe)
  cav20  2D cavity 20x20x1 PISO, dt 0.005, 5 steps       (config C1)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
REF = "/root/reference/pkg/src"


def _import_reference():
    sys.path.insert(0, REF)
    import fvflow.cases as rcases
    import fvflow.coupling as rcoup
    import fvflow.fvm as rfvm
    import fvflow.linsolve as rlin
    import fvflow.mesh as rmesh
    import fvflow.sparse as rsparse
    from fvflow.config import BoundarySpec, CaseConfig

    return rcases, rcoup, rfvm, rlin, rmesh, rsparse, BoundarySpec, CaseConfig


def mesh_dict(m):
    return dict(points=m.points, face_points=m.face_points, face_offsets=m.face_offsets,
                owner=m.owner, neighbour=m.neighbour, n_cells=np.int64(m.n_cells),
                patch_names=np.array([p.name for p in m.patches]),
                patch_kinds=np.array([p.kind for p in m.patches]),
                patch_start=np.array([p.start for p in m.patches], dtype=np.int64),
                patch_count=np.array([p.count for p in m.patches], dtype=np.int64))


def config_dict(cc):
    out = {}
    for k in ("nu", "convection", "nonorth_correction", "limiter", "cg_tol", "bicgstab_tol",
              "max_iters", "algorithm", "alpha_u", "alpha_p", "n_correctors",
              "n_nonorth_correctors", "dt", "end_time", "outer_tol", "max_outer",
              "pressure_ref_cell", "pressure_ref_value"):
        out["cfg_" + k] = np.array(getattr(cc, k))
    names = sorted(cc.boundary)
    out["bc_patches"] = np.array(names)
    out["bc_u"] = np.array([repr(cc.boundary[n].u) for n in names])
    out["bc_p"] = np.array([repr(cc.boundary[n].p) for n in names])
    return out


def make_case(R, name):
    rcases = R[0]
    BoundarySpec, CaseConfig = R[6], R[7]
    if name == "cav6":
        c = rcases.gen_cavity(6)
        c.config.algorithm, c.config.dt = "piso", 0.1 / 6
        return c, 3
    if name == "chan":
        c = rcases.gen_channel(12, 4)
        c.config.dt = 0.05
        return c, 3
    if name == "duct":
        return rcases.gen_skewed_duct(8, 6, 30.0), 3
    if name == "cav20":
        m = rcases.box_mesh(20, 20, 1, 0.1, 0.1, 0.01, [
            ("movingWall", "wall", ["y+"]), ("fixedWalls", "wall", ["x-", "x+", "y-"]),
            ("frontAndBack", "empty", ["z-", "z+"])])
        cc = CaseConfig()
        cc.nu, cc.algorithm, cc.dt, cc.end_time = 0.01, "piso", 0.005, 0.5
        cc.boundary = {
            "movingWall": BoundarySpec(u=("fixed_value", (1.0, 0.0, 0.0)), p=("zero_gradient",)),
            "fixedWalls": BoundarySpec(u=("no_slip",), p=("zero_gradient",)),
            "frontAndBack": BoundarySpec(u=("empty",), p=("empty",)),
        }
        return rcases.Case("cav20", m, cc), 5
    # C3 / C4: meshes from this repo's generators (the reference has none),
    # converted to reference objects and solved by the reference
    sys.path.insert(0, REPO)
    from paper_1207_1571_b200 import cases as mycases

    rmesh = R[4]
    mc = mycases.perturbed_cavity(5) if name == "pcav5" else mycases.gen_backward_step(2)
    m = mc.mesh
    rm = rmesh.Mesh(points=m.points, face_points=m.face_points, face_offsets=m.face_offsets,
                    owner=m.owner, neighbour=m.neighbour,
                    patches=[rmesh.Patch(p.name, p.kind, p.start, p.count) for p in m.patches],
                    n_cells=m.n_cells)
    rm.validate()
    cc = CaseConfig(**{k: getattr(mc.config, k) for k in mc.config.__dataclass_fields__
                       if k not in ("boundary", "samples")})
    cc.boundary = {k: BoundarySpec(u=v.u, p=v.p) for k, v in mc.config.boundary.items()}
    return rcases.Case(mc.name, rm, cc), (2 if name == "pcav5" else 3)


def operators(R, case, rng):
    """Single-operator outputs of the reference on seeded random fields."""
    _, rcoup, rfvm, rlin, rmesh, rsparse = R[:6]
    m = case.mesh
    g = rmesh.compute_geometry(m)
    pat = rsparse.build_pattern(m)
    n, nf, ni = m.n_cells, m.n_faces, m.n_internal
    out = {}
    for k in g.__dataclass_fields__:
        out["geom_" + k] = getattr(g, k)
    for k in ("I", "J", "diag_slot", "ell_twin_crs", "crs_row_ptr", "crs_col", "crs_twin_in_ell",
              "crs_twin_pos", "diag_addr", "face_addr"):
        out["pat_" + k] = getattr(pat, k)
    out["pat_k"] = np.int64(pat.k)
    ub = {nm: rfvm.bc_from_tuple(bs.u) for nm, bs in case.config.boundary.items()}
    pb = {nm: rfvm.bc_from_tuple(bs.p) for nm, bs in case.config.boundary.items()}
    u = rfvm.make_vector("u", m, ub)
    p = rfvm.make_scalar("p", m, pb)
    u.values = rng.normal(size=(n, 3))
    p.values = rng.normal(size=n)
    t = 0.37
    rfvm.apply_bcs(u, g, t)
    rfvm.apply_bcs(p, g, t)
    out.update(in_u=u.values, in_p=p.values, in_t=np.float64(t), op_ub=u.boundary,
               op_pb=p.boundary)
    flux = rng.normal(size=nf)
    flux[ni:][rfvm._boundary_masks(u)[2]] = 0.0
    out["in_flux"] = flux
    out["op_interp_u"] = rfvm.interpolate_to_faces(u, g)
    out["op_interp_p"] = rfvm.interpolate_to_faces(p, g)
    rv = rng.uniform(0.5, 2.0, size=n)
    out["in_raw"] = rv
    out["op_interp_raw"] = rfvm.interpolate_cell_values(m, g, rv)
    out["op_grad_u"] = rfvm.gauss_gradient(u, g)
    out["op_grad_p"] = rfvm.gauss_gradient(p, g)
    out["op_div"] = rfvm.face_divergence(m, flux)
    scheme = rfvm.SchemeConfig()
    # momentum-like vector system: ddt + convection + laplacian(coeff -1)
    sysv = rfvm.LinearSystem.zeros(pat, "vector")
    old = rng.normal(size=(n, 3))
    out["in_old"] = old
    rfvm.ddt_euler(sysv, u, old, 0.01, g)
    out["op_ddt_V"], out["op_ddt_rhs"] = sysv.A.V.copy(), sysv.rhs.copy()
    rfvm.divergence_convection(sysv, flux, u, scheme, geom=g)
    out["op_conv_V"], out["op_conv_rhs"] = sysv.A.V.copy(), sysv.rhs.copy()
    fd = rfvm.laplacian(sysv, 0.013, u, g, scheme, coeff=-1.0)
    out["op_lapv_V"], out["op_lapv_rhs"] = sysv.A.V.copy(), sysv.rhs.copy()
    out["op_lapv_coef"], out["op_lapv_corr"] = fd.coef, fd.corr
    out["op_lapv_flux"] = rfvm.laplacian_face_flux(fd, u)
    # linear-scheme convection on a fresh scalar system
    syss = rfvm.LinearSystem.zeros(pat)
    rfvm.divergence_convection(syss, flux, p, rfvm.SchemeConfig(convection="linear"), geom=g,
                               coeff=0.7)
    out["op_convlin_V"], out["op_convlin_rhs"] = syss.A.V.copy(), syss.rhs.copy()
    # pressure-like scalar laplacian with per-face gamma
    gam = rng.uniform(0.5, 2.0, size=nf)
    out["in_gamma"] = gam
    sysp = rfvm.LinearSystem.zeros(pat)
    fd = rfvm.laplacian(sysp, gam, p, g, scheme, coeff=-1.0)
    out["op_lapp_V"], out["op_lapp_rhs"] = sysp.A.V.copy(), sysp.rhs.copy()
    out["op_lapp_coef"], out["op_lapp_corr"] = fd.coef, fd.corr
    out["op_lapp_flux"] = rfvm.laplacian_face_flux(fd, p)
    # SpMV on the assembled momentum matrix
    x = rng.normal(size=n)
    out["in_x"] = x
    out["op_smvp"] = rsparse.smvp(sysv.A, x)
    # solves: CG on the (pinned) pressure system, BiCGStab on momentum
    A = sysp.A
    A.V[0, pat.diag_slot[0]] *= 2.0
    b = rng.normal(size=n)
    out["in_b"] = b
    xc, rep = rlin.cg(A, b, np.zeros(n), rlin.SolveConfig(tolerance=1e-10, max_iters=5000))
    out["sol_cg_x"] = xc
    out["sol_cg_rep"] = np.array([rep.iterations, rep.initial_residual, rep.final_residual,
                                  rep.converged])
    out["sol_cg_V"] = A.V.copy()
    xb, rep = rlin.bicgstab(sysv.A, b, np.zeros(n), rlin.SolveConfig(tolerance=1e-10,
                                                                      max_iters=5000))
    out["sol_bi_x"] = xb
    out["sol_bi_rep"] = np.array([rep.iterations, rep.initial_residual, rep.final_residual,
                                  rep.converged])
    return out


def coupled(R, case, steps):
    rcoup = R[1]
    cfg = rcoup.CouplingConfig.from_case_config(case.config)
    st = rcoup.init_state(case, cfg)
    out = {"init_u": st.u.values.copy(), "init_p": st.p.values.copy(),
           "init_flux": st.flux.copy(), "init_ub": st.u.boundary.copy(),
           "init_pb": st.p.boundary.copy()}
    for s in range(steps):
        nlog = len(st.residual_log)
        if cfg.algorithm == "piso":
            r = rcoup.piso_time_step(st, cfg)
        else:
            r = rcoup.simple_outer_iteration(st, cfg)
        out[f"s{s}_ret"] = np.array(r, dtype=float)
        out[f"s{s}_u"] = st.u.values.copy()
        out[f"s{s}_p"] = st.p.values.copy()
        out[f"s{s}_flux"] = st.flux.copy()
        out[f"s{s}_ub"] = st.u.boundary.copy()
        out[f"s{s}_pb"] = st.p.boundary.copy()
        rows = st.residual_log[nlog:]
        out[f"s{s}_log_names"] = np.array([f"{a}:{b}" for a, b, *_ in rows])
        out[f"s{s}_log"] = np.array([[c, d, e, f] for _, _, c, d, e, f in rows], dtype=float)
        out[f"s{s}_cont"] = np.float64(rcoup.continuity_error(st))
    out["steps"] = np.int64(steps)
    return out


def main():
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    R = _import_reference()
    os.makedirs(OUT, exist_ok=True)
    for name in ("cav6", "chan", "duct", "pcav5", "bfs2", "cav20"):
        case, steps = make_case(R, name)
        rng = np.random.default_rng(abs(hash(name)) % 2**32 if False else
                                    sum(map(ord, name)) + 1207)
        data = {}
        data.update(mesh_dict(case.mesh))
        data.update(config_dict(case.config))
        data.update(operators(R, case, rng))
        data.update(coupled(R, case, steps))
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{name}: cells {case.mesh.n_cells} faces {case.mesh.n_faces} -> {path} "
              f"({os.path.getsize(path) // 1024} KiB)")
    # paper fixture + 2x2 CG known answer (test_sparse.py:45-53, test_linsolve.py:82-86)
    rsparse, rlin = R[5], R[3]
    pp = rsparse.build_pattern_from_example()
    A = rsparse.HybridMatrix.zeros(pp)
    A.V[:] = np.arange(1, 13, dtype=float).reshape(4, 3)
    np.savez_compressed(os.path.join(OUT, "fixtures.npz"), ring_I=pp.I, ring_J=pp.J,
                        ring_diag_slot=pp.diag_slot, ring_smvp=rsparse.smvp(A, np.ones(4)))


if __name__ == "__main__":
    main()
