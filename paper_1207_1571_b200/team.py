"""Domain-decomposed PISO/SIMPLE runs.

One libfvb context per rank holds that rank's subdomain (decompose.py);
the contexts are joined into a *team* by handing every rank the device
address of every other rank's cell pool, so the solver kernels store halo
values straight into the neighbours' ghost slots and combine their
reduction partials through peer mailboxes — no host round trip and no
separate collective launch inside a Krylov iteration.

Two ways to form a team:

* ``DecomposedRun(case, cfg, nparts)`` — all ranks in this process, one
  host thread per rank (ctypes releases the GIL).  Ranks may share one
  device: their persistent kernels then take 1/nparts of the SMs each so
  they are co-resident.  Used by the parity tests on a single B200.
* ``RankRun(case, cfg, rank, size, device, allgather)`` — one process per
  GPU (torchrun); the pools travel as CUDA IPC handles through
  ``allgather`` (e.g. torch.distributed.all_gather_object).

Both keep the reference's bookkeeping (outer, t, cum_iters, residual_log)
and gather u, p, flux back into global order on request.
"""

import ctypes as C
import os
import socket
import threading

import numpy as np

from . import _lib
from .coupling import _FIELD_NAMES, _OP_NAMES, _step_cfg
from .decompose import _Topology, build_subdomain, local_geometry, slab_partition
from .device import DeviceContext, bc_table, device_index
from .errors import CouplingError
from .fvm import bc_from_tuple, is_value_bc, make_scalar, make_vector
from .linsolve import SolveReport
from .mesh import compute_geometry
from .sparse import build_pattern

__all__ = ["DecomposedRun", "RankRun"]


class _Member:
    """One rank: its subdomain uploaded to a context of its own."""

    def __init__(self, sd, geom, ni_global, device, share):
        self.sd = sd
        self.ctx = DeviceContext(device)
        if share > 1:
            _lib.check(_lib.lib.fvb_set_sm_share(self.ctx.h, share))
        g = local_geometry(geom, sd, ni_global)
        P = _lib.ptr
        own = _lib.i64(sd.owner)
        nbr = _lib.i64(sd.neighbour)
        _lib.check(_lib.lib.fvb_upload_mesh_part(
            self.ctx.h, sd.n_cells, sd.n_rows, sd.n_faces, sd.n_internal,
            P(own, _lib.i64p), P(nbr, _lib.i64p), P(_lib.f64(g["face_area"])),
            P(_lib.f64(g["face_area_mag"])), P(_lib.f64(g["cell_volume"])),
            P(_lib.f64(g["weight"])), P(_lib.f64(g["d"]).reshape(-1, 3)),
            P(_lib.f64(g["d_boundary"]).reshape(-1, 3))))
        I = _lib.i64(sd.I)
        ds = _lib.i64(sd.diag_slot)
        fa = _lib.i64(sd.face_addr)
        rp = _lib.i64(sd.crs_row_ptr)
        cc = _lib.i64(sd.crs_col)
        _lib.check(_lib.lib.fvb_upload_pattern(
            self.ctx.h, sd.n_rows, sd.k, P(I, _lib.i64p), P(ds, _lib.i64p), P(fa, _lib.i64p),
            sd.n_internal, len(cc), P(rp, _lib.i64p), P(cc, _lib.i64p)))
        self.local_mesh = sd.local_mesh()

    def export(self):
        base = C.c_void_p()
        nc = C.c_int64()
        handle = (C.c_uint8 * 64)()
        _lib.check(_lib.lib.fvb_team_export(self.ctx.h, C.byref(base), C.byref(nc), handle))
        return base.value, nc.value, bytes(handle)

    def attach(self, bases, ncs):
        sd = self.sd
        arr = (C.c_void_p * len(bases))(*bases)
        ncs = _lib.i64(ncs)
        sp, sr, sdst = _lib.i64(sd.send_ptr), _lib.i64(sd.send_rank), _lib.i64(sd.send_dst)
        P = _lib.ptr
        return _lib.lib.fvb_team_attach(self.ctx.h, sd.rank, sd.nparts, arr, P(ncs, _lib.i64p),
                                        sd.n_inner, P(sp, _lib.i64p), P(sr, _lib.i64p),
                                        P(sdst, _lib.i64p))

    def set_bcs(self, u_field, p_field, geom):
        """BC tables of the local boundary faces (patch order of the global mesh)."""
        lm = self.local_mesh
        for slot, fld in ((0, u_field), (1, p_field)):
            loc = _LocalField(fld, lm)
            kinds, patch, fixed, _ = bc_table(loc, geom, 0.0, with_speeds=False)
            self.ctx.set_bcs(slot, kinds, patch, fixed, len(lm.patches))

    def set_state(self, u, p, flux):
        """Upload global arrays restricted to this subdomain (ghosts included)."""
        sd = self.sd
        ul = np.ascontiguousarray(np.asarray(u)[sd.l2g].T)
        pl = np.ascontiguousarray(np.asarray(p)[sd.l2g])
        fl = np.ascontiguousarray(np.asarray(flux)[sd.faces]) if flux is not None else None
        P = _lib.ptr
        _lib.check(_lib.lib.fvb_set_state(self.ctx.h, P(_lib.f64(ul)), P(_lib.f64(pl)),
                                          P(fl) if fl is not None else None, None, None))

    def get_state(self):
        sd = self.sd
        u = np.empty(3 * sd.n_cells)
        p = np.empty(sd.n_cells)
        fl = np.empty(sd.n_faces)
        P = _lib.ptr
        _lib.check(_lib.lib.fvb_get_state(self.ctx.h, P(u), P(p), P(fl), None, None))
        return u.reshape(3, sd.n_cells).T, p, fl


class _LocalField:
    """Duck-typed Field for bc_table: global BCs on the local patches."""

    def __init__(self, field, local_mesh):
        self.mesh = local_mesh
        self.bcs = field.bcs
        self.rank = field.rank


def _scope(same_device, scope=None):
    """System-scope ordering unless every rank shares one device; `scope`
    ("sys" / "gpu") forces one (DecomposedRun: the system-scope kernels a
    multi-GPU team runs, exercised on one device by tests and
    tools/team_bench.py)."""
    if scope is not None:
        if scope not in ("sys", "gpu"):
            raise ValueError(f"scope must be 'sys' or 'gpu', not {scope!r}")
        return 1 if scope == "sys" else 0
    return 0 if same_device else 1


def _speeds(u_field, geom, t):
    """Per-patch normal speeds of timed / mass-flow inlets, from the GLOBAL
    geometry (the mass-flow area is the whole patch's, fvm.py:187-193)."""
    return _lib.f64(bc_table(u_field, geom, t)[3])


class _TeamRunBase:
    """Bookkeeping shared by the in-process and the one-process-per-GPU team."""

    def _init_common(self, case, cfg):
        mesh = case.mesh
        self.case, self.cfg = case, cfg
        self.mesh = mesh
        missing = [p.name for p in mesh.patches if p.name not in case.config.boundary]
        if missing:
            raise CouplingError(f"no boundary conditions for patches {missing}")
        self.u_bcs = {n: bc_from_tuple(bs.u) for n, bs in case.config.boundary.items()}
        self.p_bcs = {n: bc_from_tuple(bs.p) for n, bs in case.config.boundary.items()}
        self.u_field = make_vector("u", mesh, self.u_bcs)
        self.p_field = make_scalar("p", mesh, self.p_bcs)
        self.pin_pressure = not any(is_value_bc(bc) for bc in self.p_bcs.values())
        if self.pin_pressure and not 0 <= cfg.pressure_ref_cell < mesh.n_cells:
            raise CouplingError(
                f"pressure reference cell {cfg.pressure_ref_cell} outside 0..{mesh.n_cells - 1}")
        self.outer = 0
        self.t = 0.0
        self.converged = False
        self.cum_iters = {"cg": 0, "bicgstab": 0}
        self.residual_log = []
        self.wall = {}
        self.ops = {}
        self._res_scale = {}
        self.last_solves = []

    def _cfg_for(self, member, cfg):
        s = _step_cfg(self, cfg)
        ref = member.sd.local_index(cfg.pressure_ref_cell) if self.pin_pressure else -1
        s.pin_pressure = int(ref >= 0)
        s.pressure_ref_cell = max(ref, 0)
        return s

    def _record(self, rep, cfg):
        self.last_solves = []
        for k in range(rep.n_solves):
            r = rep.rep[k]
            solver = "cg" if rep.solver[k] == 0 else "bicgstab"
            self.last_solves.append((solver, int(r.iterations), float(r.wall_time)))
            self.cum_iters[solver] += int(r.iterations)
            self.residual_log.append((solver, _FIELD_NAMES[rep.field[k]], self.outer,
                                      int(r.iterations), float(r.initial_residual),
                                      float(r.final_residual)))
        for key in ("momentum_assembly", "momentum_solve", "pressure_assembly",
                    "pressure_solve", "correction"):
            self.wall[key] = self.wall.get(key, 0.0) + float(getattr(rep, "t_" + key))
        for i, name in enumerate(_OP_NAMES):
            if rep.op_calls[i]:
                rec = self.ops.setdefault(name, [0.0, 0])
                rec[0] += float(rep.op_seconds[i])
                rec[1] += int(rep.op_calls[i])

    def normalized(self, slot, res):
        seen = max(self._res_scale.get(slot, 0.0), res)
        self._res_scale[slot] = seen
        return res / max(seen, 1e-30)


class DecomposedRun(_TeamRunBase):
    """All ranks of a decomposition in this process (one thread per rank)."""

    def __init__(self, case, cfg, nparts, devices=None, part=None, scope=None):
        self._init_common(case, cfg)
        mesh = case.mesh
        self.geom = compute_geometry(mesh)
        self.pattern = build_pattern(mesh)
        if part is None:
            part, _ = slab_partition(mesh.n_cells, nparts)
        topo = _Topology(mesh, self.pattern, part)
        self.nparts = topo.nparts
        if devices is None:
            devices = [device_index()] * self.nparts
        share = max(devices.count(d) for d in set(devices))
        if share > 4:
            # ranks sharing one device spin-wait on each other inside kernels;
            # beyond 4 per device the scheduler can starve a waiting rank
            raise ValueError(f"{share} ranks on one device (at most 4 are supported; "
                             "use one device per rank for larger teams)")
        self.members = []
        for r in range(self.nparts):
            sd = build_subdomain(mesh, self.pattern, part, r, topo)
            self.members.append(_Member(sd, self.geom, mesh.n_internal, devices[r], share))
        ex = [m.export() for m in self.members]
        bases = [e[0] for e in ex]
        ncs = [e[1] for e in ex]
        same_device = len(set(devices)) == 1
        scope = _scope(same_device, scope)
        for m in self.members:  # allocations + copies: no team sync inside
            _lib.check(m.attach(bases, ncs))
            _lib.check(_lib.lib.fvb_team_set_scope(m.ctx.h, scope))
        self._parallel(lambda m: _lib.lib.fvb_team_check(m.ctx.h))
        for m in self.members:
            m.set_bcs(self.u_field, self.p_field, self.geom)
        # initial state: u = 0, p = 0, BCs at t = 0, flux = S.u_f (coupling.py:182-213)
        n = mesh.n_cells
        zero_u, zero_p = np.zeros((n, 3)), np.zeros(n)
        sp = _speeds(self.u_field, self.geom, 0.0)
        for m in self.members:
            m.set_state(zero_u, zero_p, None)
            _lib.check(_lib.lib.fvb_state_apply_bcs(m.ctx.h, _lib.ptr(sp)))
            _lib.check(_lib.lib.fvb_plain_flux(m.ctx.h), CouplingError)

    def _parallel(self, fn):
        """fn(member) on every rank at once (team syncs need all ranks in
        flight); libfvb's error text is thread-local, so it is read in the
        worker thread."""
        rcs = [0] * len(self.members)
        msgs = [""] * len(self.members)
        errs = [None] * len(self.members)

        def run(i, m):
            try:
                rc = fn(m)
                if isinstance(rc, int) and rc != 0:
                    rcs[i] = rc
                    msgs[i] = _lib.last_error()
            except Exception as e:  # noqa: BLE001 - re-raised below
                errs[i] = e

        th = [threading.Thread(target=run, args=(i, m)) for i, m in enumerate(self.members)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        for rc, msg in zip(rcs, msgs):
            if rc != 0:
                cls = CouplingError if rc == _lib.E_COUPLING else _lib._ERR.get(rc, RuntimeError)
                raise cls(msg.replace("{outer}", str(self.outer)))
        return rcs

    def _step(self, cfg, piso):
        sp = _speeds(self.u_field, self.geom, self.t)
        fn = _lib.lib.fvb_piso_step if piso else _lib.lib.fvb_simple_sweep
        reps = [_lib.StepReportC() for _ in self.members]
        cfgs = {id(m): self._cfg_for(m, cfg) for m in self.members}
        rep_of = {id(m): r for m, r in zip(self.members, reps)}

        def go(m):
            return fn(m.ctx.h, C.byref(cfgs[id(m)]), _lib.ptr(sp), C.byref(rep_of[id(m)]))

        try:
            self._parallel(go)
        finally:
            self._record(reps[0], cfg)
        return float(reps[0].mom_res), float(reps[0].p_res)

    def piso_time_step(self, cfg):
        self.outer += 1
        self.t = self.outer * cfg.dt
        return self._step(cfg, True)

    def simple_outer_iteration(self, cfg):
        self.outer += 1
        ru, rp = self._step(cfg, False)
        return self.normalized("u", ru), self.normalized("p", rp)

    def gather(self):
        """Global u (N,3), p (N), flux (F) assembled from the owned rows and
        local faces of every rank."""
        n, nf = self.mesh.n_cells, self.mesh.n_faces
        u = np.empty((n, 3))
        p = np.empty(n)
        flux = np.empty(nf)
        for m in self.members:
            ul, pl, fl = m.get_state()
            rows = m.sd.l2g[:m.sd.n_rows]
            u[rows] = ul[:m.sd.n_rows]
            p[rows] = pl[:m.sd.n_rows]
            flux[m.sd.faces] = fl
        return u, p, flux

    def continuity_error(self):
        out = {id(m): C.c_double() for m in self.members}
        self._parallel(lambda m: _lib.lib.fvb_continuity_error(m.ctx.h, C.byref(out[id(m)])))
        return float(out[id(self.members[0])].value)

    def close(self):
        for m in self.members:
            m.ctx.close()


class RankRun(_TeamRunBase):
    """One rank of a decomposition with one process per GPU.

    ``allgather(obj) -> list`` exchanges small Python objects between the
    ranks (torch.distributed.all_gather_object under torchrun).  Every rank
    builds the global setup deterministically and keeps only its own
    subdomain; pools are shared through CUDA IPC handles.
    """

    def __init__(self, case, cfg, rank, size, device, allgather, geom=None, pattern=None):
        self._init_common(case, cfg)
        mesh = case.mesh
        self.geom = geom if geom is not None else compute_geometry(mesh)
        self.pattern = pattern if pattern is not None else build_pattern(mesh)
        part, _ = slab_partition(mesh.n_cells, size)
        self.rank, self.nparts = rank, size
        sd = build_subdomain(mesh, self.pattern, part, rank)
        # FVB_SM_SHARE > 1: several ranks (processes) share one device (tests)
        share = int(os.environ.get("FVB_SM_SHARE", "1"))
        self.member = _Member(sd, self.geom, mesh.n_internal, device, share)
        base, nc, handle = self.member.export()
        infos = allgather((os.getpid(), device, base, nc, handle, socket.gethostname()))
        self._opened = []
        bases = []
        for q, (pid, dev, b, ncq, h, _host) in enumerate(infos):
            if q == rank:
                bases.append(base)
            elif pid == os.getpid():
                bases.append(b)
            else:
                ptr = C.c_void_p()
                buf = (C.c_uint8 * 64).from_buffer_copy(h)
                _lib.check(_lib.lib.fvb_ipc_open(buf, C.byref(ptr)))
                self._opened.append(ptr.value)
                bases.append(ptr.value)
        _lib.check(self.member.attach(bases, [i[3] for i in infos]))
        same_device = len({(i[5], i[1]) for i in infos}) == 1
        # evidence for the multi-GPU bench line: where each rank runs and how
        # it reaches its peers' pools
        peer_ok = []
        for q, (_pid, dev, *_rest) in enumerate(infos):
            ok = C.c_int()
            _lib.check(_lib.lib.fvb_device_can_access_peer(device, dev, C.byref(ok)))
            peer_ok.append(int(ok.value))
        self.diag = {"rank": rank, "pid": os.getpid(), "device": device,
                     "host": socket.gethostname(), "ipc_mapped": len(self._opened),
                     "same_process_peers": sum(1 for q, i in enumerate(infos)
                                               if q != rank and i[0] == os.getpid()),
                     "peer_devices": [i[1] for i in infos], "can_access_peer": peer_ok,
                     "rows": int(sd.n_rows), "scope": "gpu" if same_device else "sys"}
        _lib.check(_lib.lib.fvb_team_set_scope(self.member.ctx.h, _scope(same_device)))
        _lib.check(_lib.lib.fvb_team_check(self.member.ctx.h))
        self.member.set_bcs(self.u_field, self.p_field, self.geom)
        n = mesh.n_cells
        sp = _speeds(self.u_field, self.geom, 0.0)
        self.member.set_state(np.zeros((n, 3)), np.zeros(n), None)
        h = self.member.ctx.h
        _lib.check(_lib.lib.fvb_state_apply_bcs(h, _lib.ptr(sp)))
        _lib.check(_lib.lib.fvb_plain_flux(h), CouplingError)

    @property
    def ctx(self):
        return self.member.ctx

    def _step(self, cfg, piso):
        sp = _speeds(self.u_field, self.geom, self.t)
        fn = _lib.lib.fvb_piso_step if piso else _lib.lib.fvb_simple_sweep
        rep = _lib.StepReportC()
        scfg = self._cfg_for(self.member, cfg)
        rc = fn(self.member.ctx.h, C.byref(scfg), _lib.ptr(sp), C.byref(rep))
        self._record(rep, cfg)
        if rc != 0:
            msg = _lib.last_error().replace("{outer}", str(self.outer))
            if rc == _lib.E_COUPLING:
                raise CouplingError(msg)
            raise _lib._ERR.get(rc, RuntimeError)(msg)
        return float(rep.mom_res), float(rep.p_res)

    def piso_time_step(self, cfg):
        self.outer += 1
        self.t = self.outer * cfg.dt
        return self._step(cfg, True)

    def simple_outer_iteration(self, cfg):
        self.outer += 1
        ru, rp = self._step(cfg, False)
        return self.normalized("u", ru), self.normalized("p", rp)

    def local_state(self):
        return self.member.get_state()

    def close(self):
        for p in self._opened:
            _lib.lib.fvb_ipc_close(p)
        self._opened = []
        self.member.ctx.close()
