"""ctypes binding of libfvb.so (include/fvb.h).

The shared library is the only compute path of this package: importing
this module loads it and raises ImportError if it has not been built
(run ``python -c "import __graft_entry__ as g; g.build()"`` or
``python paper_1207_1571_b200/build.py``).  There is no CPU fallback.
"""

import ctypes as C
import os

import numpy as np

from .errors import (
    CouplingError,
    DeviceError,
    FvmError,
    MeshError,
    MeshFileError,
    SolverError,
    SparseError,
)

# Load every kernel when the CUDA context is created.  With lazy loading
# the first launch of a kernel may wait for the device to drain; ranks of a
# decomposition that share one device spin-wait on each other inside
# kernels, so a lazily loaded kernel of one rank could stall behind the
# other rank's waiting kernel until the watchdog fires.  (Takes effect if
# CUDA has not been initialised in this process yet.)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfvb.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python paper_1207_1571_b200/build.py); there is no CPU fallback"
    )
lib = C.CDLL(LIB_PATH)

BC_ZERO_GRADIENT, BC_EMPTY, BC_FIXED, BC_NO_SLIP, BC_SINE, BC_MASS_FLOW = range(6)

E_ARG, E_MESH, E_SPARSE, E_SOLVER, E_FVM, E_COUPLING, E_CUDA, E_TIMEOUT, E_MESHFILE, E_IO = range(
    -1, -11, -1)
_ERR = {
    E_ARG: ValueError,
    E_MESH: MeshError,
    E_SPARSE: SparseError,
    E_SOLVER: SolverError,
    E_FVM: FvmError,
    E_COUPLING: CouplingError,
    E_CUDA: DeviceError,
    E_TIMEOUT: DeviceError,
    E_MESHFILE: MeshFileError,
    E_IO: OSError,
}

dp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("initial_residual", C.c_double),
        ("final_residual", C.c_double),
        ("wall_time", C.c_double),
        ("error_iteration", C.c_int32),
        ("error_kind", C.c_int32),
        ("t_smvp", C.c_double),
        ("t_daxpy", C.c_double),
        ("t_reduction", C.c_double),
    ]


class StepCfgC(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32),
        ("scheme", C.c_int32),
        ("nonorth_correction", C.c_int32),
        ("n_correctors", C.c_int32),
        ("n_nonorth_correctors", C.c_int32),
        ("pin_pressure", C.c_int32),
        ("pressure_ref_cell", C.c_int32),
        ("mom_max_iters", C.c_int32),
        ("p_max_iters", C.c_int32),
        ("record_stages", C.c_int32),
        ("nu", C.c_double),
        ("alpha_u", C.c_double),
        ("alpha_p", C.c_double),
        ("dt", C.c_double),
        ("t", C.c_double),
        ("limiter", C.c_double),
        ("mom_tol", C.c_double),
        ("mom_abs_tol", C.c_double),
        ("p_tol", C.c_double),
        ("p_abs_tol", C.c_double),
        ("pressure_ref_value", C.c_double),
    ]


MAX_SOLVES = 64


class StepReportC(C.Structure):
    _fields_ = [
        ("n_solves", C.c_int32),
        ("solver", C.c_int32 * MAX_SOLVES),
        ("field", C.c_int32 * MAX_SOLVES),
        ("rep", SolveReportC * MAX_SOLVES),
        ("mom_res", C.c_double),
        ("p_res", C.c_double),
        ("t_momentum_assembly", C.c_double),
        ("t_momentum_solve", C.c_double),
        ("t_pressure_assembly", C.c_double),
        ("t_pressure_solve", C.c_double),
        ("t_correction", C.c_double),
        ("failed_solve", C.c_int32),
        ("op_seconds", C.c_double * 5),
        ("op_calls", C.c_int32 * 5),
    ]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


I = C.c_int
I64 = C.c_int64
D = C.c_double
_sig("fvb_version", I)
_sig("fvb_last_error", C.c_char_p)
_sig("fvb_device_count", I)
_sig("fvb_geometry", I, I64, dp, I64, i64p, i64p, I64, I64, i64p, i64p, I,
     dp, dp, dp, dp, dp, dp, dp, dp, dp, dp, dp)
_sig("fvb_pattern_plan_create", I, I64, I64, i64p, I64, C.POINTER(vp), i64p, i64p)
_sig("fvb_pattern_plan_fill", I, vp, I64, i64p, i64p, i64p, i64p, i64p, i64p, i64p,
     u8p, i64p, i64p)
_sig("fvb_pattern_plan_destroy", None, vp)
_sig("fvb_mesh_read", I, C.c_char_p, C.POINTER(vp), i64p)
_sig("fvb_mesh_read_take", I, vp, dp, i64p, i64p, i64p, i64p, i64p, i64p, C.c_char_p, C.c_char_p)
_sig("fvb_mesh_read_free", None, vp)
_sig("fvb_mesh_write", I, C.c_char_p, I64, dp, I64, i64p, i64p, i64p, I64, i64p, I64,
     C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), i64p, i64p)
_sig("fvb_ctx_create", I, I, C.POINTER(vp))
_sig("fvb_ctx_destroy", I, vp)
_sig("fvb_ctx_device_bytes", I64, vp)
_sig("fvb_upload_mesh", I, vp, I64, I64, I64, i64p, i64p, dp, dp, dp, dp, dp, dp)
_sig("fvb_upload_mesh_part", I, vp, I64, I64, I64, I64, i64p, i64p, dp, dp, dp, dp, dp, dp)
_sig("fvb_upload_pattern", I, vp, I64, I64, i64p, i64p, i64p, I64, I64, i64p, i64p)
_sig("fvb_team_export", I, vp, C.POINTER(vp), i64p, u8p)
_sig("fvb_ipc_open", I, u8p, C.POINTER(vp))
_sig("fvb_ipc_close", I, vp)
_sig("fvb_team_attach", I, vp, I, I, C.POINTER(vp), i64p, I64, i64p, i64p, i64p)
_sig("fvb_team_check", I, vp)
_sig("fvb_team_set_scope", I, vp, I)
_sig("fvb_team_allreduce", I, vp, dp, I, I)
_sig("fvb_set_sm_share", I, vp, I)
_sig("fvb_set_bcs", I, vp, I, u8p, i32p, dp, I)
_sig("fvb_set_state", I, vp, dp, dp, dp, dp, dp)
_sig("fvb_get_state", I, vp, dp, dp, dp, dp, dp)
_sig("fvb_op_smvp", I, vp, dp, dp, dp, dp)
_sig("fvb_op_stmvp", I, vp, dp, dp, i64p, i64p, u8p, i64p, i64p, dp, dp)
_sig("fvb_pack_q", I, I64, I64, i64p, i64p, I, i64p)
_sig("fvb_unpack_q", I, I64, I64, I64, i64p, I, i64p, i64p)
_sig("fvb_op_cg", I, vp, dp, dp, dp, dp, dp, D, D, I, C.POINTER(SolveReportC))
_sig("fvb_op_bicgstab", I, vp, dp, dp, dp, dp, dp, D, D, I, C.POINTER(SolveReportC))
_sig("fvb_op_bicgstab_batched", I, vp, I, dp, dp, dp, dp, dp, D, D, I, C.POINTER(SolveReportC))
_sig("fvb_op_apply_bcs", I, vp, I, dp, dp, dp)
_sig("fvb_op_interpolate", I, vp, I, I, dp, dp, dp)
_sig("fvb_op_gradient", I, vp, I, I, dp, dp, dp)
_sig("fvb_op_divergence", I, vp, dp, dp)
_sig("fvb_op_laplacian", I, vp, I, I, dp, dp, dp, D, dp, dp, dp, I, D, D, dp, dp)
_sig("fvb_op_laplacian_flux", I, vp, I, I, dp, dp, dp, dp, dp)
_sig("fvb_op_convection", I, vp, I, I, dp, dp, dp, dp, dp, I, D)
_sig("fvb_op_ddt", I, vp, I, dp, dp, dp, D, D)
_sig("fvb_piso_step", I, vp, C.POINTER(StepCfgC), dp, C.POINTER(StepReportC))
_sig("fvb_simple_sweep", I, vp, C.POINTER(StepCfgC), dp, C.POINTER(StepReportC))
_sig("fvb_plain_flux", I, vp)
_sig("fvb_state_apply_bcs", I, vp, dp)
_sig("fvb_op_face_flux", I, vp, dp, dp, dp)
_sig("fvb_op_rhie_chow", I, vp, dp, dp, dp, dp, dp, dp, dp, dp)
_sig("fvb_continuity_error", I, vp, dp)
_sig("fvb_sync", I, vp)
_sig("fvb_set_solver_options", I, vp, C.c_int)
_sig("fvb_set_solver_grid", I, vp, C.c_int)
_sig("fvb_device_can_access_peer", I, C.c_int, C.c_int, C.POINTER(C.c_int))
SOLVER_EXPLICIT_INDEX, SOLVER_NO_RCM, SOLVER_NO_CLUSTER, STEP_NO_GRAPHS = 1, 2, 4, 8
_sig("fvb_pattern_codes", I, vp, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int),
     C.POINTER(C.c_int64))
_sig("fvb_launch_count", C.c_ulonglong)
_sig("fvb_host_register", I, vp, I64)
_sig("fvb_host_unregister", I, vp)
_sig("fvb_timer_start", I, vp)
_sig("fvb_timer_stop", I, vp, dp)

EXPORTS = [
    "fvb_version", "fvb_last_error", "fvb_device_count", "fvb_geometry",
    "fvb_pattern_plan_create", "fvb_pattern_plan_fill", "fvb_pattern_plan_destroy",
    "fvb_ctx_create", "fvb_ctx_destroy", "fvb_ctx_device_bytes", "fvb_upload_mesh",
    "fvb_upload_mesh_part", "fvb_team_export", "fvb_ipc_open", "fvb_ipc_close",
    "fvb_team_attach", "fvb_team_check", "fvb_team_set_scope", "fvb_team_allreduce", "fvb_set_sm_share",
    "fvb_upload_pattern", "fvb_set_bcs", "fvb_set_state", "fvb_get_state", "fvb_op_smvp",
    "fvb_op_stmvp", "fvb_pack_q", "fvb_unpack_q",
    "fvb_mesh_read", "fvb_mesh_read_take", "fvb_mesh_read_free", "fvb_mesh_write",
    "fvb_op_cg", "fvb_op_bicgstab", "fvb_op_bicgstab_batched", "fvb_op_apply_bcs",
    "fvb_op_interpolate", "fvb_op_gradient", "fvb_op_divergence", "fvb_op_laplacian",
    "fvb_op_laplacian_flux", "fvb_op_convection", "fvb_op_ddt", "fvb_piso_step",
    "fvb_simple_sweep", "fvb_plain_flux", "fvb_state_apply_bcs", "fvb_op_face_flux", "fvb_op_rhie_chow", "fvb_continuity_error", "fvb_sync", "fvb_timer_start", "fvb_timer_stop",
    "fvb_launch_count", "fvb_pattern_codes", "fvb_set_solver_options", "fvb_set_solver_grid", "fvb_device_can_access_peer", "fvb_host_register", "fvb_host_unregister",
]


def last_error():
    return lib.fvb_last_error().decode()


def check(rc, exc=None):
    """Raise the reference exception class mapped from a libfvb status."""
    if rc == 0:
        return
    cls = exc or _ERR.get(rc, RuntimeError)
    raise cls(last_error())


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def ptr(a, kind=dp):
    if a is None:
        return None
    return a.ctypes.data_as(kind)
