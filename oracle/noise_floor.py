"""CPU-vs-CPU rounding floor of the reference itself (SURVEY.md §7 hard part
1, Appendix B "Noise floor"; test infrastructure): runs the real reference's
PISO steps of gen_cavity(N) or the C4 mesh with a 1-ulp perturbation of the
arithmetic order and prints the per-solve iteration counts, to set next to
the golden run (tests/golden/full_*.npz) when judging the device counts.

    python oracle/noise_floor.py c2|c4 MODE [steps]

MODE "seqspmv": smvp summed slot by slot (y = V0 x0; y += Vk xk) instead of
numpy's einsum grouping; MODE "blasT": OpenBLAS with T threads (ddot split
differently) instead of 1.  Output: tests/golden/floor_<case>_<mode>.json.
"""
import json
import os
import sys

MODE = sys.argv[2]
os.environ["OPENBLAS_NUM_THREADS"] = MODE[4:] if MODE.startswith("blas") else "1"

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden_full as M  # noqa: E402


def main():
    name, steps = sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 2
    R = M._ref()
    rcoup = R[1]
    import fvflow.linsolve as rl
    import fvflow.sparse as rs

    if MODE == "seqspmv":
        def smvp(A, x):
            p = A.pattern
            g = x[np.maximum(p.I, 0)]
            y = A.V[:, 0] * g[:, 0]
            for k in range(1, p.k):
                y = y + A.V[:, k] * g[:, k]
            if p.nnz_crs:
                y = y + np.bincount(p.crs_row, weights=A.crs_val * x[p.crs_col], minlength=p.n)
            return y
        for mod in (rl, rcoup, rs):
            if hasattr(mod, "smvp"):
                mod.smvp = smvp
    case, _ = M.make(R, f"{name}_default")
    cfg = rcoup.CouplingConfig.from_case_config(case.config)
    st = rcoup.init_state(case, cfg)
    out = []
    for s in range(steps):
        n0 = len(st.residual_log)
        rcoup.piso_time_step(st, cfg)
        out.append([[a, b, int(d)] for a, b, _, d, *_ in st.residual_log[n0:]])
        print(name, MODE, "step", s + 1, out[-1], flush=True)
    with open(os.path.join(M.OUT, f"floor_{name}_{MODE}.json"), "w") as f:
        json.dump({"case": name, "mode": MODE, "steps": out}, f)


if __name__ == "__main__":
    main()
