"""BiCGStab iteration counts of the step-1 momentum solve (cavity from rest)
on the device and in the oracle, on the identical oracle-assembled system
(diagnostic for the default-tolerance count checks of
tests/test_gpu_golden_full.py).

    python tools/bicgstab_diag.py N [N ...]     (N = cavity edge, or c4 for the
                                                 perturbed + renumbered 126^3 mesh)

For each N: gen_cavity(N) PISO dt 0.1/N; the oracle assembles the step-1
momentum matrix and rhs (ddt + convection + Laplacian, pressure gradient);
ux is solved by oracle.pbicgstab and by linsolve.bicgstab / the batched
device solve, at the reference default tolerance 1e-8 and at 1e-10.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from oracle import fvoracle as O  # noqa: E402
from paper_1207_1571_b200 import cases, sparse  # noqa: E402
from paper_1207_1571_b200.linsolve import SolveConfig, bicgstab, bicgstab_batched  # noqa: E402


def main():
    for arg in sys.argv[1:]:
        if arg == "c4":
            case = cases.perturbed_cavity(126)
            cc = case.config
            n = arg
        else:
            n = int(arg)
            case = cases.gen_cavity(n)
            cc = case.config
            cc.algorithm, cc.dt = "piso", 0.1 / n
        run = O.Run(case.mesh, cc)
        run.outer, run.t = 1, cc.dt
        O.apply_bcs(run.u, run.g, run.t)
        O.apply_bcs(run.p, run.g, run.t)
        A, b0 = run.momentum_matrix(run.u.values.copy())
        gp = O.gradient(run.p, run.g)
        rhs = b0 - run.g["cell_volume"][:, None] * gp
        pat = sparse.build_pattern(case.mesh)
        H = sparse.HybridMatrix.zeros(pat)
        H.V[:] = A.V
        out = {"n": n}
        for tol in (1e-8, 1e-10):
            x0 = run.u.values.copy()
            _, rep = O.pbicgstab(A, rhs[:, 0], x0[:, 0], tol, max_iters=5000)
            xd, rd = bicgstab(H, rhs[:, 0], x0[:, 0], SolveConfig(tolerance=tol, max_iters=5000))
            Xb, rb = bicgstab_batched(H, rhs, x0, SolveConfig(tolerance=tol, max_iters=5000))
            from paper_1207_1571_b200 import _lib
            from paper_1207_1571_b200.device import context_for
            ctx = context_for(None, None, pat)
            _lib.check(_lib.lib.fvb_set_solver_options(ctx.h, _lib.SOLVER_NO_RCM))
            xn, rn = bicgstab(H, rhs[:, 0], x0[:, 0], SolveConfig(tolerance=tol, max_iters=5000))
            _lib.check(_lib.lib.fvb_set_solver_options(ctx.h, 0))
            out[f"tol{tol:g}"] = {"oracle": [rep[0], rep[2]], "device": [rd.iterations, rd.final_residual],
                                  "device_batched_ux": [rb[0].iterations, rb[0].final_residual],
                                  "device_mesh_order": [rn.iterations, rn.final_residual]}
        if os.environ.get("BIDIAG_CURVE"):
            # residual after k iterations, device vs oracle (same system, x0)
            lo, hi = (int(v) for v in os.environ["BIDIAG_CURVE"].split(":"))
            curve = []
            for k in range(lo, hi + 1):
                x0 = run.u.values.copy()
                _, rep = O.pbicgstab(A, rhs[:, 0], x0[:, 0], 1e-300, max_iters=k)
                _, rd = bicgstab(H, rhs[:, 0], x0[:, 0], SolveConfig(tolerance=1e-300, max_iters=k))
                curve.append([k, rep[2], rd.final_residual])
            out["curve_k_oracle_device"] = curve
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
