"""Two processes, one IPC-joined team (RankRun), checked against the
single-domain run.  Launch: torchrun --nproc-per-node 2 tools/ipc_team_check.py N
(on one GPU set FVB_DEVICE=0 FVB_SM_SHARE=2)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch.distributed as dist
from paper_1207_1571_b200 import cases
from paper_1207_1571_b200.coupling import CouplingConfig, init_state, piso_time_step
from paper_1207_1571_b200.team import RankRun

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
def allgather(obj):
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out
case = cases.gen_cavity(n)
case.config.algorithm, case.config.dt = "piso", 0.1 / n
cfg = CouplingConfig.from_case_config(case.config)
dev = int(os.environ.get("FVB_DEVICE", os.environ.get("LOCAL_RANK", "0")))
t0 = time.time()
run = RankRun(case, cfg, rank, world, dev, allgather)
for _ in range(2):
    run.piso_time_step(cfg)
ul, pl, fl = run.local_state()
sd = run.member.sd
parts = allgather((sd.l2g[:sd.n_rows], ul[:sd.n_rows], pl[:sd.n_rows], sd.faces, fl))
if rank == 0:
    N, F = case.mesh.n_cells, case.mesh.n_faces
    u = np.empty((N, 3)); p = np.empty(N); f = np.empty(F)
    for rows, a, b, faces, c in parts:
        u[rows] = a; p[rows] = b; f[faces] = c
    st = init_state(case, cfg)
    for _ in range(2):
        piso_time_step(st, cfg)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    print(f"IPC team of {world}: rel u {rel(u, st.u.values):.3e} p {rel(p, st.p.values):.3e} "
          f"flux {rel(f, st.flux):.3e}; iters team {[r[3] for r in run.residual_log]} "
          f"single {[r[3] for r in st.residual_log]}; {time.time() - t0:.1f} s", flush=True)
run.close()
dist.destroy_process_group()
