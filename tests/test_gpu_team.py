"""Domain-decomposed runs on the device.

P ranks share one B200 here (one libfvb context and host thread per rank,
each persistent solver grid on 1/P of the SMs); the kernels, halo stores
and peer-mailbox reductions are the ones a multi-GPU run uses.  A team of
one must be bitwise the single-domain run; a team of P must match it
under the parity rules (fields to the CPU-vs-CPU noise floor, CG
iterations +-1, BiCGStab +-2) and match the reference's golden steps.
"""

import numpy as np
import pytest

from golden_io import golden_case, rel
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import (
    CouplingConfig, continuity_error, init_state, piso_time_step, simple_outer_iteration)
from paper_1207_1571_b200.team import DecomposedRun

pytestmark = pytest.mark.gpu


def _single(case, cfg, steps):
    st = init_state(case, cfg)
    for _ in range(steps):
        if cfg.algorithm == "piso":
            piso_time_step(st, cfg)
        else:
            simple_outer_iteration(st, cfg)
    return st


def _team(case, cfg, steps, nparts, scope=None):
    run = DecomposedRun(case, cfg, nparts, scope=scope)
    for _ in range(steps):
        if cfg.algorithm == "piso":
            run.piso_time_step(cfg)
        else:
            run.simple_outer_iteration(cfg)
    return run


def test_team_of_one_is_bitwise_single_domain():
    case = cases.gen_cavity(8)
    case.config.algorithm, case.config.dt = "piso", 0.1 / 8
    cfg = CouplingConfig.from_case_config(case.config)
    st = _single(case, cfg, 2)
    run = _team(case, cfg, 2, 1)
    u, p, flux = run.gather()
    assert np.array_equal(u, st.u.values)
    assert np.array_equal(p, st.p.values)
    assert np.array_equal(flux, st.flux)
    assert run.residual_log == st.residual_log
    run.close()


@pytest.mark.parametrize("name,nparts", [("cav6", 2), ("cav6", 3), ("pcav5", 2), ("pcav5", 4),
                                         ("bfs2", 2), ("chan", 2), ("duct", 3), ("cav20", 2)])
def test_team_matches_single_domain_and_reference(name, nparts):
    case, g = golden_case(name)
    cfg = CouplingConfig.from_case_config(case.config)
    steps = int(g["steps"])
    st = _single(case, cfg, steps)
    run = _team(case, cfg, steps, nparts)
    u, p, flux = run.gather()
    for a, b in ((u, st.u.values), (p, st.p.values), (flux, st.flux)):
        assert rel(a, b) < 1e-9
    s = steps - 1
    assert rel(u, g[f"s{s}_u"]) < 1e-8
    assert rel(p, g[f"s{s}_p"]) < 1e-8
    assert rel(flux, g[f"s{s}_flux"]) < 1e-8
    two_d = case.mesh.n_cells in (48, 260, 400)
    assert len(run.residual_log) == len(st.residual_log)
    for a, b in zip(run.residual_log, st.residual_log):
        assert a[:3] == b[:3]
        if two_d and a[1] == "uz":
            continue
        assert abs(a[3] - b[3]) <= (1 if a[0] == "cg" else 2), (a, b)
    assert run.continuity_error() <= max(1e-8 * np.abs(flux).max(), 1e-16)
    run.close()


def test_team_cavity24_four_ranks():
    case = cases.gen_cavity(24)
    case.config.algorithm, case.config.dt = "piso", 0.1 / 24
    cfg = CouplingConfig.from_case_config(case.config)
    st = _single(case, cfg, 2)
    run = _team(case, cfg, 2, 4)
    u, p, flux = run.gather()
    assert rel(u, st.u.values) < 1e-9 and rel(p, st.p.values) < 1e-9 and rel(flux, st.flux) < 1e-9
    for a, b in zip(run.residual_log, st.residual_log):
        assert abs(a[3] - b[3]) <= (1 if a[0] == "cg" else 2), (a, b)
    assert continuity_error(st) <= 1e-8 * np.abs(st.flux).max()
    run.close()


def test_ipc_team_two_processes_one_device():
    """The one-process-per-GPU path (RankRun: CUDA IPC pool mappings,
    torch.distributed plumbing) with both ranks on this device."""
    import os
    import socket
    import subprocess
    import sys

    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, FVB_DEVICE="0", FVB_SM_SHARE="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(here, "tools", "ipc_team_check.py"), "4"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300, cwd=here)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("IPC team of 2")]
    assert line, out.stdout[-2000:]
    import re

    rels = [float(x) for x in re.findall(r"(?:u|p|flux) ([0-9.e+-]+)", line[0])]
    assert len(rels) == 3 and max(rels) < 1e-9, line[0]
    team, single = re.findall(r"\[([0-9, ]+)\]", line[0])
    ta = [int(x) for x in team.split(",")]
    sa = [int(x) for x in single.split(",")]
    assert len(ta) == len(sa) and all(abs(a - b) <= 1 for a, b in zip(ta, sa)), line[0]


@pytest.mark.parametrize("nparts", [2, 4])
def test_team_system_scope_kernels(nparts):
    # the kernels a team over several GPUs uses (system-scope release fences
    # and acquires, the SYS instantiations), forced on one device with
    # scope="sys": same results as the single-domain run under the parity
    # rules
    case = cases.gen_cavity(12)
    case.config.algorithm, case.config.dt = "piso", 0.1 / 12
    case.config.cg_tol, case.config.bicgstab_tol, case.config.max_iters = 1e-13, 1e-10, 20000
    cfg = CouplingConfig.from_case_config(case.config)
    st = _single(case, cfg, 2)
    run = _team(case, cfg, 2, nparts, scope="sys")
    u, p, flux = run.gather()
    assert rel(u, st.u.values) < 1e-9 and rel(p, st.p.values) < 1e-9 and rel(flux, st.flux) < 1e-9
    for a, b in zip(run.residual_log, st.residual_log):
        assert abs(a[3] - b[3]) <= (2 if a[0] == "cg" else 3), (a, b)
    assert run.continuity_error() <= 1e-8 * np.abs(flux).max()
    run.close()
