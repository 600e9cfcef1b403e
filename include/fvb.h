/*
 * fvb.h — C ABI of libfvb.so, the B200-native (sm_100a, FP64) PISO/SIMPLE
 * engine that replaces the numpy hot path of the reference package fvflow
 * (arXiv 1207.1571 restated in /root/reference/pkg/src/fvflow).
 *
 * The reference is pure Python: its "plugin API" is its function surface.
 * Each entry point below names the reference function it replaces
 * (file:line relative to /root/reference/pkg/src/fvflow).  The Python
 * package paper_1207_1571_b200 binds these with ctypes and presents the
 * reference's own names, dataclasses and exceptions on top.
 *
 * Conventions
 *   - plain C types only; host pointers are caller-owned numpy buffers;
 *     device memory is owned by the context for its lifetime;
 *   - every function returns 0 on success or a negative FVB_E* code;
 *     fvb_last_error() returns the message of the last failure on the
 *     calling thread (text mirrors the reference's exception messages);
 *   - cell-vector data crosses the ABI component-major (SoA):
 *     v[c*n + i] is component c of cell i; gradients g[(c*3+d)*n + i];
 *   - integer mesh/pattern arrays cross as int64 (the reference dtype).
 */
#ifndef FVB_H
#define FVB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes (mapped 1:1 onto the reference's exception classes) */
#define FVB_OK 0
#define FVB_E_ARG -1        /* ValueError / bad sizes                          */
#define FVB_E_MESH -2       /* mesh.MeshError            (mesh.py:27)          */
#define FVB_E_SPARSE -3     /* sparse.SparseError        (sparse.py:25)        */
#define FVB_E_SOLVER -4     /* linsolve.SolverError      (linsolve.py:24)      */
#define FVB_E_FVM -5        /* fvm.FvmError              (fvm.py:30)           */
#define FVB_E_COUPLING -6   /* coupling.CouplingError    (coupling.py:64)      */
#define FVB_E_CUDA -7       /* device / driver failure                          */
#define FVB_E_TIMEOUT -8    /* device watchdog fired inside a persistent kernel */
#define FVB_E_MESHFILE -9   /* fileio.MeshFileError      (fileio.py:27)        */
#define FVB_E_IO -10        /* OSError opening / writing a file                 */

/* boundary-condition kinds per boundary face (fvm.py:37-105) */
#define FVB_BC_ZERO_GRADIENT 0
#define FVB_BC_EMPTY 1
#define FVB_BC_FIXED 2      /* FixedValue / FixedPressure: per-face values    */
#define FVB_BC_NO_SLIP 3
#define FVB_BC_SINE 4       /* FixedValueTimed: -u0 sin(2 pi f t) n_hat        */
#define FVB_BC_MASS_FLOW 5  /* FixedMassFlow: -rate/(rho A) n_hat              */

typedef struct fvb_ctx fvb_ctx;

int fvb_version(void);
const char* fvb_last_error(void);
/* cudaDeviceCanAccessPeer (bench/team diagnostics: every rank of a
 * multi-GPU team stores into its peers' pools over NVLink). */
int fvb_device_can_access_peer(int device, int peer, int* ok);
int fvb_device_count(void);

/* ------------------------------------------------------------------ setup
 * Host-side native builders (no GPU needed). */

/* compute_geometry (mesh.py:173-278), bitwise the reference's arithmetic.
 * Outputs are caller-allocated: vol[nc], cc[3nc], sf[3nf], smag[nf],
 * fc[3nf], d[3ni], dmag[ni], w[ni], nonorth[ni], db[3nb], dbmag[nb]
 * (row-major (.,3) like the reference arrays).  check=1 enforces the 80 deg
 * non-orthogonality limit (mesh.py:256-261). */
int fvb_geometry(int64_t n_points, const double* points, int64_t n_faces,
                 const int64_t* face_offsets, const int64_t* face_points,
                 int64_t n_cells, int64_t n_internal, const int64_t* owner,
                 const int64_t* neighbour, int check, double* vol, double* cc,
                 double* sf, double* smag, double* fc, double* d, double* dmag,
                 double* w, double* nonorth, double* db, double* dbmag);

/* pattern_from_pairs (sparse.py:111-209), bit-exact integers.  Phase 1
 * returns sizes (k, nnz_crs); phase 2 fills caller-allocated arrays. */
typedef struct fvb_pattern_plan fvb_pattern_plan;
int fvb_pattern_plan_create(int64_t n, int64_t n_pairs, const int64_t* pairs,
                            int64_t k_cap, fvb_pattern_plan** out,
                            int64_t* k_out, int64_t* nnz_crs_out);
int fvb_pattern_plan_fill(fvb_pattern_plan* plan, int64_t n_face_pairs,
                          const int64_t* face_pairs, int64_t* I, int64_t* J,
                          int64_t* diag_slot, int64_t* ell_twin_crs,
                          int64_t* crs_row_ptr, int64_t* crs_col,
                          uint8_t* crs_twin_in_ell, int64_t* crs_twin_pos,
                          int64_t* face_addr);
void fvb_pattern_plan_destroy(fvb_pattern_plan* plan);

/* Mesh file I/O (fileio.py:50-185): the reference's ASCII format, read
 * with its exact line-numbered MeshFileError messages and written with
 * "%.17g" so files are byte-identical to fvflow's.  Read is two-phase:
 * fvb_mesh_read parses and returns counts[5] = {n_points, n_faces,
 * n_face_points, n_internal, n_patches}; fvb_mesh_read_take copies into
 * caller arrays (names/kinds: n_patches x 256 chars) and keeps the handle
 * valid until fvb_mesh_read_free. */
typedef struct fvb_meshfile fvb_meshfile;
int fvb_mesh_read(const char* path, fvb_meshfile** out, int64_t* counts);
int fvb_mesh_read_take(fvb_meshfile* mf, double* points, int64_t* face_offsets,
                       int64_t* face_points, int64_t* owner, int64_t* neighbour,
                       int64_t* patch_start, int64_t* patch_count, char* patch_names,
                       char* patch_kinds);
void fvb_mesh_read_free(fvb_meshfile* mf);
int fvb_mesh_write(const char* path, int64_t n_points, const double* points,
                   int64_t n_faces, const int64_t* face_offsets,
                   const int64_t* face_points, const int64_t* owner,
                   int64_t n_internal, const int64_t* neighbour, int64_t n_patches,
                   const char* const* names, const char* const* kinds,
                   const int64_t* start, const int64_t* count);

/* ---------------------------------------------------------------- context */
int fvb_ctx_create(int device, fvb_ctx** out);
int fvb_ctx_destroy(fvb_ctx* ctx);
/* bytes of device memory held by the context */
int64_t fvb_ctx_device_bytes(fvb_ctx* ctx);

/* Upload mesh addressing + geometry once (init_state, coupling.py:182-203).
 * sf is (nf,3) row-major, d (ni,3), db (nb,3). */
int fvb_upload_mesh(fvb_ctx* ctx, int64_t n_cells, int64_t n_faces,
                    int64_t n_internal, const int64_t* owner,
                    const int64_t* neighbour, const double* sf,
                    const double* smag, const double* vol, const double* w,
                    const double* d, const double* db);

/* Domain-decomposed variant: the local mesh of one rank
 * holds n_rows owned cells followed by n_cells - n_rows ghost cells (cells
 * of other ranks adjacent to an owned cell).  Faces are the local faces
 * (every face with an owned side) in ascending global order, internal
 * faces first; processor faces are internal faces with a ghost side.
 * Only owned rows are assembled and solved; ghost values arrive by halo
 * exchange.  fvb_upload_mesh(...) == fvb_upload_mesh_part(n_rows=n_cells). */
int fvb_upload_mesh_part(fvb_ctx* ctx, int64_t n_cells, int64_t n_rows,
                         int64_t n_faces, int64_t n_internal,
                         const int64_t* owner, const int64_t* neighbour,
                         const double* sf, const double* smag, const double* vol,
                         const double* w, const double* d, const double* db);

/* Upload the hybrid pattern once (build_pattern, sparse.py:212-220).
 * n = owned rows; columns may address ghost cells (< n_cells); a negative
 * face_addr entry marks a side whose row lives on another rank. */
int fvb_upload_pattern(fvb_ctx* ctx, int64_t n, int64_t k, const int64_t* I,
                       const int64_t* diag_slot, const int64_t* face_addr,
                       int64_t n_face_pairs, int64_t nnz_crs,
                       const int64_t* crs_row_ptr, const int64_t* crs_col);

/* Boundary conditions of field 0 (u, vector) or 1 (p, scalar), per boundary
 * face: kind[nb], patch[nb]; fixed values fixed[ncomp*nb] (SoA). */
int fvb_set_bcs(fvb_ctx* ctx, int field, const uint8_t* kind,
                const int32_t* patch, const double* fixed, int n_patches);

/* ---------------------------------------------------------- device state
 * Fields of the coupled state: u[3n] SoA, p[n], flux[nf], ub[3nb], pb[nb]. */
int fvb_set_state(fvb_ctx* ctx, const double* u, const double* p,
                  const double* flux, const double* ub, const double* pb);
int fvb_get_state(fvb_ctx* ctx, double* u, double* p, double* flux,
                  double* ub, double* pb);

/* ------------------------------------------------------------- operators
 * Single-operator entry points (host buffers in/out), for parity tests
 * and for the reference's operator-level API.  A "system" is V[n*k]
 * row-major (reference layout), crs[nnz], rhs[ncomp*n] SoA. */

/* smvp (sparse.py:296-305) */
int fvb_op_smvp(fvb_ctx* ctx, const double* V, const double* crs,
                const double* x, double* y);
/* stmvp (sparse.py:308-334): y = A^T x without forming the transpose,
 * twins through J (row-major (n,k) ELL twin slots), ell_twin_crs (CRS
 * position of an ELL entry's twin) and the CRS back-references */
int fvb_op_stmvp(fvb_ctx* ctx, const double* V, const double* crs, const int64_t* J,
                 const int64_t* ell_twin_crs, const uint8_t* crs_twin_in_ell,
                 const int64_t* crs_twin_row, const int64_t* crs_twin_pos,
                 const double* x, double* y);
/* pack_q / unpack_q (sparse.py:337-363), host-side: mode 0 by_N, 1 by_K;
 * I, J, q are (n*k) row-major; unpack_q decodes m entries */
int fvb_pack_q(int64_t n, int64_t k, const int64_t* I, const int64_t* J, int mode,
               int64_t* q);
int fvb_unpack_q(int64_t n, int64_t k, int64_t m, const int64_t* q, int mode,
                 int64_t* I, int64_t* J);
/* cg (linsolve.py:102-172) / bicgstab (linsolve.py:175-282) */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double initial_residual;
  double final_residual;
  double wall_time;   /* device time, seconds                        */
  int32_t error_iteration; /* >0 when the solve raised at that iteration */
  int32_t error_kind;      /* 0 none, see fvb.cu solver error table      */
  /* device stage timers of the persistent kernel (seconds; StageTimer
   * buckets of linsolve.py:18-79): SpMV passes (with the fused p-update /
   * preconditioner), vector-update passes (with the fused z = r/D and the
   * per-thread dot partials), and the grid/team reductions */
  double t_smvp, t_daxpy, t_reduction;
} fvb_solve_report;
int fvb_op_cg(fvb_ctx* ctx, const double* V, const double* crs,
              const double* b, const double* x0, double* x, double tol,
              double abs_tol, int max_iters, fvb_solve_report* rep);
int fvb_op_bicgstab(fvb_ctx* ctx, const double* V, const double* crs,
                    const double* b, const double* x0, double* x, double tol,
                    double abs_tol, int max_iters, fvb_solve_report* rep);
/* batched: ncomp right-hand sides against one matrix (coupling.py:267-275) */
int fvb_op_bicgstab_batched(fvb_ctx* ctx, int ncomp, const double* V,
                            const double* crs, const double* b,
                            const double* x0, double* x, double tol,
                            double abs_tol, int max_iters,
                            fvb_solve_report* reps);

/* apply_bcs (fvm.py:170-197): boundary[ncomp*nb] from values + kinds;
 * speeds[n_patches] = the per-patch normal speed for SINE/MASS_FLOW. */
int fvb_op_apply_bcs(fvb_ctx* ctx, int field, const double* values,
                     const double* speeds, double* boundary);
/* interpolate_to_faces (fvm.py:220-239) for field 0/1 BC masks, or raw
 * owner-copy interpolation (fvm.py:242-247) when field < 0. */
int fvb_op_interpolate(fvb_ctx* ctx, int field, int ncomp,
                       const double* values, const double* boundary,
                       double* face_values);
/* gauss_gradient (fvm.py:258-275): grad[(c*3+d)*n + i] */
int fvb_op_gradient(fvb_ctx* ctx, int field, int ncomp, const double* values,
                    const double* boundary, double* grad);
/* face_divergence (fvm.py:250-255) */
int fvb_op_divergence(fvb_ctx* ctx, const double* flux, double* div);
/* laplacian (fvm.py:335-408): accumulates into V/crs/rhs in place and
 * writes coef[nf], corr[ncomp*nf].  gamma: scalar if gamma_faces==NULL. */
int fvb_op_laplacian(fvb_ctx* ctx, int field, int ncomp, double* V,
                     double* crs, double* rhs, double gamma,
                     const double* gamma_faces, const double* values,
                     const double* boundary, int nonorth, double limiter,
                     double coeff, double* coef, double* corr);
/* laplacian_face_flux (fvm.py:411-429) */
int fvb_op_laplacian_flux(fvb_ctx* ctx, int field, int ncomp,
                          const double* coef, const double* corr,
                          const double* values, const double* boundary,
                          double* flux_out);
/* divergence_convection (fvm.py:432-482); scheme 0 upwind, 1 linear */
int fvb_op_convection(fvb_ctx* ctx, int field, int ncomp, double* V,
                      double* crs, double* rhs, const double* flux,
                      const double* boundary, int scheme, double coeff);
/* ddt_euler (fvm.py:485-496) */
int fvb_op_ddt(fvb_ctx* ctx, int ncomp, double* V, double* rhs,
               const double* old_values, double dt, double coeff);

/* ------------------------------------------------------------ the loop */
typedef struct {
  int32_t algorithm;          /* 0 simple, 1 piso (coupling.py:68-99)   */
  int32_t scheme;             /* 0 upwind, 1 linear                     */
  int32_t nonorth_correction;
  int32_t n_correctors;
  int32_t n_nonorth_correctors;
  int32_t pin_pressure;
  int32_t pressure_ref_cell;
  int32_t mom_max_iters;
  int32_t p_max_iters;
  int32_t record_stages;
  double nu, alpha_u, alpha_p, dt, t, limiter;
  double mom_tol, mom_abs_tol, p_tol, p_abs_tol;
  double pressure_ref_value;
} fvb_step_cfg;

#define FVB_MAX_SOLVES 64
typedef struct {
  int32_t n_solves;                 /* rows appended to residual_log     */
  int32_t solver[FVB_MAX_SOLVES];   /* 0 cg, 1 bicgstab                  */
  int32_t field[FVB_MAX_SOLVES];    /* 0 ux 1 uy 2 uz 3 p                */
  fvb_solve_report rep[FVB_MAX_SOLVES];
  double mom_res;                   /* largest normalized initial residual */
  double p_res;                     /* first pressure initial residual     */
  /* device-timed sections (seconds), RunState.wall keys (coupling.py:163) */
  double t_momentum_assembly, t_momentum_solve, t_pressure_assembly,
      t_pressure_solve, t_correction;
  int32_t failed_solve;             /* index of the solve that raised, -1 */
  /* per-operator device times and call counts, RunState.ops keys
   * (coupling.py:166, 223-229, 252, 299, 313, 340), in the order
   * ddt, convection, laplacian, gradient, divergence; a laplacian includes
   * its non-orthogonal-correction gradient as in the reference */
  double op_seconds[5];
  int32_t op_calls[5];
} fvb_step_report;

/* piso_time_step (coupling.py:356-370) with speeds[] for time-dependent
 * BCs at cfg.t; simple_outer_iteration (coupling.py:347-353). */
int fvb_piso_step(fvb_ctx* ctx, const fvb_step_cfg* cfg,
                  const double* u_speeds, fvb_step_report* rep);
int fvb_simple_sweep(fvb_ctx* ctx, const fvb_step_cfg* cfg,
                     const double* u_speeds, fvb_step_report* rep);
/* apply_bcs(u, t) and apply_bcs(p, t) on the resident state
 * (fvm.py:170-197 as called by coupling.py:193-194, 360-361) */
int fvb_state_apply_bcs(fvb_ctx* ctx, const double* u_speeds);
/* S . u_f of a vector field under the u-table BC masks, 0 on empty faces
 * (coupling.py:206-213; the _plain_flux helper) */
int fvb_op_face_flux(fvb_ctx* ctx, const double* values, const double* boundary,
                     double* flux_out);
/* rhie_chow_flux (fvm.py:499-538): face fluxes S.u_f with the pressure-
 * gradient smoothing D_f a_f [(p_N - p_O) - (grad p)_f . d] on internal
 * faces and on boundary faces where p is value-pinned and u is not; 0 on
 * u-empty faces.  u / ub SoA (3 x n_cells / 3 x n_boundary), p / pb, the
 * momentum diagonal a_diag [n_cells] (FVB_E_FVM "zero momentum diagonal at
 * cell N"), d SoA [3 x n_internal], d_boundary SoA [3 x n_boundary].  BC
 * tables of the u (0) and p (1) fields must be set. */
int fvb_op_rhie_chow(fvb_ctx* ctx, const double* u, const double* ub, const double* p,
                     const double* pb, const double* a_diag, const double* d,
                     const double* d_boundary, double* flux_out);
/* plain flux S.u_f with 0 on empty faces (coupling.py:206-213) */
int fvb_plain_flux(fvb_ctx* ctx);
/* continuity_error (coupling.py:373-375) */
int fvb_continuity_error(fvb_ctx* ctx, double* out);
/* ------------------------------------------------------------- team
 * Ranks of one domain decomposition share their cell pools: kernels store
 * halo values straight into the neighbours' ghost slots (NVLink P2P) and
 * combine reduction partials through peer mailboxes, inside the persistent
 * Krylov kernels.  Across processes the pools travel as CUDA IPC handles
 * (64 bytes, exchanged by the caller, e.g. torch.distributed); ranks in one
 * process pass the raw pool pointers.  There is no reference counterpart:
 * fvflow is single-process. */
/* pool base (device pointer), local cell count and IPC handle of a context */
int fvb_team_export(fvb_ctx* ctx, void** pool_base, int64_t* n_cells,
                    uint8_t* ipc_handle /* 64 bytes */);
int fvb_ipc_open(const uint8_t* ipc_handle, void** pool_base);
int fvb_ipc_close(void* pool_base);
/* attach this context as `rank` of `size`: pool_bases[q] / n_cells[q] of
 * every rank (own included); owned rows >= n_inner send their values to
 * (send_rank[e], ghost index send_dst[e]) for e in
 * send_ptr[row-n_inner] .. send_ptr[row-n_inner+1] */
int fvb_team_attach(fvb_ctx* ctx, int rank, int size, void* const* pool_bases,
                    const int64_t* n_cells, int64_t n_inner,
                    const int64_t* send_ptr, const int64_t* send_rank,
                    const int64_t* send_dst);
/* memory-ordering scope of the team's halo stores and reductions: 1 (the
 * default after attach) when ranks sit on different devices, 0 when every
 * rank shares this device (gpu-scope fences suffice) */
int fvb_team_set_scope(fvb_ctx* ctx, int system_scope);
/* after every rank attached: make the mesh checks that raise inside a step
 * (coincident centroids, fvm.py:349-370) raise on every rank (team sync) */
int fvb_team_check(fvb_ctx* ctx);
/* deterministic allreduce of m <= 16 doubles over the team (op 0 sum,
 * 1 max, 2 min); a no-op without a team */
int fvb_team_allreduce(fvb_ctx* ctx, double* vals, int m, int op);
/* several teams sharing one device (tests): persistent grids use 1/share
 * of the SMs so every rank's solver kernel is co-resident */
int fvb_set_sm_share(fvb_ctx* ctx, int share);

/* solver data-format options of a context (no reference counterpart: the
 * reference has one format).  Both give the same iterates: stencil codes
 * read exactly the columns of the explicit indices (bitwise), and the RCM
 * order keeps every row's products (only the dot-product grouping moves).
 * Used by the format-equivalence tests and tools/cg_micro.py. */
#define FVB_SOLVER_EXPLICIT_INDEX 1 /* SpMV passes read int32 indices, not stencil codes */
#define FVB_SOLVER_NO_RCM 2         /* solve in the mesh order on renumbered meshes */
#define FVB_SOLVER_NO_CLUSTER 4     /* small systems on the plain grid / block path (no one-cluster or shared-memory solver) */
#define FVB_STEP_NO_GRAPHS 8        /* launch the step's assembly kernels one by one instead of replaying their CUDA graphs */
int fvb_set_solver_options(fvb_ctx* ctx, int flags);

/* grid of the persistent solver kernels (no reference counterpart): at most
 * max_blocks cooperative blocks; 0 = automatic (one block per SM on large
 * systems, fewer on small ones, where the grid barriers dominate).  Changes
 * only the grouping of the dot-product partial sums. */
int fvb_set_solver_grid(fvb_ctx* ctx, int max_blocks);

/* solver data formats of the uploaded pattern (no reference counterpart;
 * bench/roofline evidence): n_codes distinct column-offset tuples of the
 * stencil-code compression (0 = off or FVB_SOLVER_EXPLICIT_INDEX set:
 * the solvers read the explicit indices), n_escape rows outside the dictionary, cg_defer_x = 1 when CG
 * folds x += alpha p into the next SpMV pass, rcm_solves = CG and BiCGStab
 * solves (a batch counts once) run so far in the solvers' internal reverse
 * Cuthill-McKee order (patterns without stencil codes, e.g. randomly
 * renumbered meshes).  Any pointer may be NULL. */
int fvb_pattern_codes(fvb_ctx* ctx, int* n_codes, int64_t* n_escape, int* cg_defer_x,
                      int64_t* rcm_solves);

/* number of kernels libfvb has launched in this process (bench evidence) */
unsigned long long fvb_launch_count(void);
/* page-lock caller-owned host buffers (pinned H2D/D2H for the e2e path) */
int fvb_host_register(void* ptr, int64_t bytes);
int fvb_host_unregister(void* ptr);
/* device timer on the context stream (CUDA events): start, then stop
 * (synchronises) returning elapsed milliseconds */
int fvb_timer_start(fvb_ctx* ctx);
int fvb_timer_stop(fvb_ctx* ctx, double* ms);
/* synchronise the context stream */
int fvb_sync(fvb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FVB_H */
