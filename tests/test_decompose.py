"""Domain decomposition bookkeeping on CPU.

Each subdomain must reproduce, for its owned rows, exactly the global
rows: the same faces in the same order, the same ELL columns in the same
slot order, the same face -> coefficient addresses; and the halo send
tables must deliver every ghost its owner's value.  The world-size-2 test
runs the halo exchange and a distributed SpMV over torch.distributed
(gloo) and checks it bitwise against the global SpMV.
"""

import os
import socket

import numpy as np
import pytest

from golden_io import golden_case
from paper_1207_1571_b200 import cases, sparse
from paper_1207_1571_b200.decompose import build_subdomains, slab_partition


def _meshes():
    yield "cav6", cases.gen_cavity(6).mesh
    yield "pcav5", golden_case("pcav5")[0].mesh
    yield "bfs2", golden_case("bfs2")[0].mesh
    yield "chan", golden_case("chan")[0].mesh


def _row_faces(own, nbr, nc):
    """Reference per-cell face order: owned faces ascending, then neighbour faces."""
    lists = [[] for _ in range(nc)]
    for f, o in enumerate(own):
        lists[o].append(f)
    for f, n in enumerate(nbr):
        lists[n].append(~f)
    return lists


def spmv_ref_order(V, I, x):
    """numpy-einsum row order for K <= 7: even slots, odd slots, then sum."""
    K = I.shape[1]
    g = x[np.maximum(I, 0)] * V
    ev = g[:, 0].copy()
    for s in range(2, K, 2):
        ev = ev + g[:, s]
    if K == 1:
        return ev
    od = g[:, 1].copy()
    for s in range(3, K, 2):
        od = od + g[:, s]
    return ev + od


@pytest.mark.parametrize("nparts", [1, 2, 3, 4])
def test_subdomains_reproduce_global_rows(nparts):
    for name, mesh in _meshes():
        pat = sparse.build_pattern(mesh)
        sds = build_subdomains(mesh, pat, nparts)
        part, _ = slab_partition(mesh.n_cells, nparts)
        owned = np.concatenate([sd.l2g[:sd.n_rows] for sd in sds])
        assert np.array_equal(np.sort(owned), np.arange(mesh.n_cells)), name
        glob = _row_faces(mesh.owner, mesh.neighbour, mesh.n_cells)
        K = pat.k
        for sd in sds:
            assert len(np.unique(sd.l2g)) == sd.n_cells
            assert (part[sd.l2g[:sd.n_rows]] == sd.rank).all()
            assert (part[sd.l2g[sd.n_rows:]] != sd.rank).all()
            assert (sd.ghost_rank == part[sd.l2g[sd.n_rows:]]).all()
            assert np.array_equal(sd.faces, np.sort(sd.faces))
            loc = _row_faces(sd.owner, sd.neighbour, sd.n_cells)
            for i in range(sd.n_rows):
                g = sd.l2g[i]
                mapped = [int(sd.faces[f]) if f >= 0 else ~int(sd.faces[~f]) for f in loc[i]]
                assert mapped == glob[g], (name, sd.rank, i)
            # ELL rows: same slots, columns mapped through l2g
            Ig = pat.I[sd.l2g[:sd.n_rows]]
            back = np.where(sd.I >= 0, sd.l2g[np.maximum(sd.I, 0)], -1)
            assert np.array_equal(back, Ig)
            assert np.array_equal(sd.diag_slot, pat.diag_slot[sd.l2g[:sd.n_rows]])
            # face_addr: local flat address -> the global one
            fa = pat.face_addr[sd.faces[:sd.n_internal]]
            for side in range(2):
                a = sd.face_addr[:, side]
                ok = a >= 0
                grow = sd.l2g[a[ok] // K]
                assert np.array_equal(grow * K + a[ok] % K, fa[ok, side])
                # a missing side is exactly a row owned elsewhere
                gr = fa[~ok, side] // K
                assert (part[gr] != sd.rank).all()
            # boundary faces keep their patch
            for gp, lp in zip(mesh.patches, sd.patches):
                lf = sd.faces[lp.start:lp.start + lp.count]
                assert ((lf >= gp.start) & (lf < gp.start + gp.count)).all()


def _halo_exchange_local(sds, vals_per_rank):
    """Apply every rank's send table to the other ranks' local vectors."""
    for sd, v in zip(sds, vals_per_rank):
        for t in range(sd.n_rows - sd.n_inner):
            row = sd.n_inner + t
            for e in range(sd.send_ptr[t], sd.send_ptr[t + 1]):
                vals_per_rank[sd.send_rank[e]][sd.send_dst[e]] = v[row]


@pytest.mark.parametrize("nparts", [2, 3, 5])
def test_halo_tables_fill_every_ghost(nparts):
    for name, mesh in _meshes():
        pat = sparse.build_pattern(mesh)
        sds = build_subdomains(mesh, pat, nparts)
        x = np.random.default_rng(3).normal(size=mesh.n_cells)
        vals = []
        for sd in sds:
            v = np.full(sd.n_cells, np.nan)
            v[:sd.n_rows] = x[sd.l2g[:sd.n_rows]]
            vals.append(v)
        _halo_exchange_local(sds, vals)
        V = np.random.default_rng(4).normal(size=pat.I.shape) * (pat.I >= 0)
        y = spmv_ref_order(V, pat.I, x)
        for sd, v in zip(sds, vals):
            assert np.array_equal(v, x[sd.l2g]), (name, sd.rank)
            yl = spmv_ref_order(V[sd.l2g[:sd.n_rows]], sd.I, v)
            assert np.array_equal(yl, y[sd.l2g[:sd.n_rows]])  # bitwise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = golden_case("pcav5")[0].mesh
        pat = sparse.build_pattern(mesh)
        part, _ = slab_partition(mesh.n_cells, world)
        from paper_1207_1571_b200.decompose import build_subdomain

        sd = build_subdomain(mesh, pat, part, rank)
        x = np.random.default_rng(11).normal(size=mesh.n_cells)
        V = np.random.default_rng(12).normal(size=pat.I.shape) * (pat.I >= 0)
        v = np.zeros(sd.n_cells)
        v[:sd.n_rows] = x[sd.l2g[:sd.n_rows]]
        # pack per destination rank in send-table order, exchange counts then values
        out = {}
        for t in range(sd.n_rows - sd.n_inner):
            row = sd.n_inner + t
            for e in range(sd.send_ptr[t], sd.send_ptr[t + 1]):
                out.setdefault(int(sd.send_rank[e]), []).append((int(sd.send_dst[e]), v[row]))
        peer = 1 - rank
        mine = out.get(peer, [])
        n_out = torch.tensor([len(mine)], dtype=torch.int64)
        n_in = torch.zeros(1, dtype=torch.int64)
        reqs = [dist.isend(n_out, peer), dist.irecv(n_in, peer)]
        for r in reqs:
            r.wait()
        buf_out = torch.tensor([[d, val] for d, val in mine], dtype=torch.float64).reshape(-1, 2)
        buf_in = torch.zeros((int(n_in.item()), 2), dtype=torch.float64)
        reqs = [dist.isend(buf_out, peer), dist.irecv(buf_in, peer)]
        for r in reqs:
            r.wait()
        for d, val in buf_in.numpy():
            v[int(d)] = val
        ok_halo = bool(np.array_equal(v, x[sd.l2g]))
        yl = spmv_ref_order(V[sd.l2g[:sd.n_rows]], sd.I, v)
        y = spmv_ref_order(V, pat.I, x)
        ok_spmv = bool(np.array_equal(yl, y[sd.l2g[:sd.n_rows]]))
        # a global dot as the device team does it: per-rank sums combined in rank order
        part_sum = torch.tensor([float(yl @ yl)], dtype=torch.float64)
        allp = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, part_sum)
        tot = sum(float(a.item()) for a in allp)
        ok_dot = abs(tot - float(y @ y)) <= 1e-12 * float(y @ y)
        q.put((rank, ok_halo, ok_spmv, ok_dot))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_and_spmv():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    for rank, ok_halo, ok_spmv, ok_dot in res:
        assert ok_halo and ok_spmv and ok_dot, (rank, ok_halo, ok_spmv, ok_dot)
