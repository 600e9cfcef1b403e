// libfvb C ABI: context lifetime, one-time uploads of the mesh, pattern and
// boundary tables, single-operator entry points (host buffers in/out) and
// the device-resident PISO step / SIMPLE sweep (coupling.py:216-370).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "fvb_internal.cuh"

static thread_local std::string g_last_error;
std::atomic<unsigned long long> fvb::g_launches{0};

void fvb_set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

using namespace fvb;

namespace fvb {
// One allocation: the team comm area followed by kPoolSlots cell vectors.
// Without a team the context is its own rank 0 of size 1.
int ensure_pool(Ctx* c) {
  if (c->pool) return FVB_OK;
  const size_t bytes = kCommBytes + sizeof(double) * size_t(kPoolSlots) * size_t(c->nc);
  char* p = nullptr;
  FVB_TRY(dalloc(c, &p, bytes));
  FVB_CUDA(cudaMemset(p, 0, bytes));
  c->pool = p;
  c->cells = reinterpret_cast<double*>(p + kCommBytes);
  c->u = c->slot(S_U);
  c->p = c->slot(S_P);
  c->scratch = c->slot(S_SCR);
  TeamView& T = c->team;
  T = TeamView{};
  T.rank = 0;
  T.size = 1;
  T.sys = 0;
  T.comm = reinterpret_cast<Comm*>(p);
  T.peer_comm[0] = T.comm;
  T.peer_cells[0] = c->cells;
  T.peer_nc[0] = c->nc;
  T.n_inner = c->nr;
  return FVB_OK;
}
}  // namespace fvb


namespace {

constexpr int kThreads = 256;

// temporary device buffer for the operator entry points
struct Tmp {
  void* p = nullptr;
  ~Tmp() {
    if (p) cudaFree(p);
  }
};

template <typename T>
int tmp_upload(Ctx* c, Tmp& t, const T* host, size_t n, T** out) {
  FVB_CUDA(cudaMalloc(&t.p, (n ? n : 1) * sizeof(T)));
  if (host && n) FVB_CUDA(cudaMemcpyAsync(t.p, host, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  *out = static_cast<T*>(t.p);
  return FVB_OK;
}

template <typename T>
int tmp_zero(Ctx* c, Tmp& t, size_t n, T** out) {
  FVB_CUDA(cudaMalloc(&t.p, (n ? n : 1) * sizeof(T)));
  FVB_CUDA(cudaMemsetAsync(t.p, 0, (n ? n : 1) * sizeof(T), c->stream));
  *out = static_cast<T*>(t.p);
  return FVB_OK;
}

template <typename T>
int d2h(Ctx* c, T* host, const T* dev, size_t n) {
  if (n) FVB_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  return FVB_OK;
}

template <typename T>
int h2d(Ctx* c, T* dev, const T* host, size_t n) {
  if (n) FVB_CUDA(cudaMemcpyAsync(dev, host, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return FVB_OK;
}

int sync(Ctx* c) {
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  return FVB_OK;
}

// row-major (n,k) <-> slot-major [k*n]
std::vector<double> to_slot_major(const double* V, int n, int k) {
  std::vector<double> o(size_t(n) * k);
  for (int i = 0; i < n; ++i)
    for (int s = 0; s < k; ++s) o[size_t(s) * n + i] = V[size_t(i) * k + s];
  return o;
}
void from_slot_major(const std::vector<double>& o, double* V, int n, int k) {
  for (int i = 0; i < n; ++i)
    for (int s = 0; s < k; ++s) V[size_t(i) * k + s] = o[size_t(s) * n + i];
}

struct DevMatrix {
  Tmp tv, tc;
  MatView m{nullptr, nullptr};
};

int upload_matrix(Ctx* c, DevMatrix& M, const double* V, const double* crs) {
  std::vector<double> sm = to_slot_major(V, c->nr, c->k);
  double* dv;
  double* dc;
  FVB_TRY(tmp_upload(c, M.tv, sm.data(), sm.size(), &dv));
  FVB_TRY(tmp_upload(c, M.tc, crs, size_t(c->nnz_crs), &dc));
  M.m = MatView{dv, dc};
  return sync(c);
}

int download_matrix(Ctx* c, DevMatrix& M, double* V, double* crs) {
  std::vector<double> sm(size_t(c->nr) * c->k);
  FVB_TRY(d2h(c, sm.data(), M.m.V, sm.size()));
  if (crs) FVB_TRY(d2h(c, crs, M.m.crs, size_t(c->nnz_crs)));
  FVB_TRY(sync(c));
  from_slot_major(sm, V, c->nr, c->k);
  return FVB_OK;
}

int need_mesh(Ctx* c) {
  if (!c->have_mesh) {
    fvb_set_error("no mesh uploaded to this context");
    return FVB_E_ARG;
  }
  return FVB_OK;
}
int need_pattern(Ctx* c) {
  if (!c->have_pattern) {
    fvb_set_error("no pattern uploaded to this context");
    return FVB_E_ARG;
  }
  return FVB_OK;
}
int need_bc(Ctx* c, int field) {
  if (field < 0 || field > 1 || !c->have_bc[field]) {
    fvb_set_error("boundary conditions of field %d not set", field);
    return FVB_E_ARG;
  }
  return FVB_OK;
}

// ---------------------------------------------------------------- kernels
// Row kernels loop over the nr owned rows; V has slot stride nr, cell
// vectors have component stride nv (= nc, owned rows + ghosts).
__global__ void k_get_diag(int n, const int* ds, const double* V, double* diag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    diag[i] = V[size_t(ds[i]) * n + i];
}

__global__ void k_set_diag(int n, const int* ds, double* V, const double* diag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    V[size_t(ds[i]) * n + i] = diag[i];
}

// rhs = b0 - V grad p   (coupling.py:253); SIMPLE implicit relaxation
// (coupling.py:254-258): V[diag] = diag/alpha, rhs += (scaled - diag) u
__global__ void k_mom_rhs(int n, size_t nv, const double* b0, const double* vol,
                          const double* gp, const double* diag, const double* u, double* rhs,
                          double* V, const int* ds, int relax, double alpha_u) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double v = vol[i];
    double scaled = 0.0;
    if (relax) {
      scaled = diag[i] / alpha_u;
      V[size_t(ds[i]) * n + i] = scaled;
    }
    for (int c = 0; c < 3; ++c) {
      double r = b0[c * nv + i] - v * gp[c * nv + i];
      if (relax) r = r + (scaled - diag[i]) * u[c * nv + i];
      rhs[c * nv + i] = r;
    }
  }
}

// per-block sum of squares of up to 3 vectors (partials, fixed order)
__global__ void k_sumsq(int n, size_t nv, int ncomp, const double* x, double* partials) {
  __shared__ double red[32 * 3];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int c = 0; c < ncomp; ++c) {
      const double v = x[c * nv + i];
      acc[c] += v * v;
    }
  block_reduce<3>(acc, red);
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) partials[size_t(c) * gridDim.x + blockIdx.x] = acc[c];
}

__global__ void k_absmax(int n, const double* x, double* partials) {
  __shared__ double red[32];
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) partials[blockIdx.x] = m;
  }
}

// HbyA = u + (b0 - A u)/a_P  (coupling.py:290-291); rAU = V/a_P (301)
__global__ void k_hbya(int n, size_t nv, const double* u, const double* b0, const double* au,
                       const double* diag, const double* vol, double* hv, double* rau) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d = diag[i];
    for (int c = 0; c < 3; ++c) {
      const size_t k = c * nv + i;
      hv[k] = u[k] + (b0[k] - au[k]) / d;
    }
    rau[i] = vol[i] / d;
  }
}

// rhs = rhs_L - div(phiHbyA); pin the reference cell (coupling.py:314-319)
__global__ void k_p_rhs(int n, const double* rl, const double* divh, double* rhs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    rhs[i] = rl[i] - divh[i];
}
__global__ void k_pin(int n, const int* ds, double* V, double* rhs, int ref, double pref) {
  const double dref = V[size_t(ds[ref]) * n + ref];
  rhs[ref] += dref * pref;
  V[size_t(ds[ref]) * n + ref] = 2.0 * dref;
}

// flux = phiHbyA - laplacian_face_flux (coupling.py:334)
__global__ void k_flux_corr(int nf, const double* phih, const double* lf, double* flux) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x)
    flux[f] = phih[f] - lf[f];
}

// p = p_before + alpha_p (p - p_before)  (coupling.py:335-336)
__global__ void k_relax_p(int n, double* p, const double* pb, double a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = pb[i] + a * (p[i] - pb[i]);
}

// u = HbyA - rAU grad p  (coupling.py:341)
__global__ void k_u_corr(int n, size_t nv, const double* hv, const double* rau, const double* gp,
                         double* u) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int c = 0; c < 3; ++c) u[c * nv + i] = hv[c * nv + i] - rau[i] * gp[c * nv + i];
}

// ----------------------------------------------------------- step state
// Cell vectors of the step live in pool slots (Slot enum); matrices and
// face arrays are plain allocations owned by the context.
struct StepWork {
  double*& Vm; double*& crsm; double*& Vp; double*& crsp; double*& phih; double*& rauf;
  double*& coef; double*& corr; double*& lf;
};

StepWork work_of(Ctx* c) {
  return StepWork{c->Vm, c->crsm, c->Vp, c->crsp, c->phih, c->rauf, c->coef, c->corr, c->lf};
}

int ensure_work(Ctx* c) {
  if (c->work_ready || !c->have_mesh || !c->have_pattern) return FVB_OK;
  const size_t nf = c->nf, kn = size_t(c->k) * c->nr, nz = size_t(c->nnz_crs);
  FVB_TRY(dalloc(c, &c->Vm, kn));
  FVB_TRY(dalloc(c, &c->crsm, nz));
  FVB_TRY(dalloc(c, &c->Vp, kn));
  FVB_TRY(dalloc(c, &c->crsp, nz));
  FVB_TRY(dalloc(c, &c->phih, nf));
  FVB_TRY(dalloc(c, &c->rauf, nf));
  FVB_TRY(dalloc(c, &c->coef, nf));
  FVB_TRY(dalloc(c, &c->corr, nf));
  FVB_TRY(dalloc(c, &c->lf, nf));
  FVB_TRY(dalloc(c, &c->u_save, 3 * size_t(c->nc)));
  c->work_ready = true;
  return FVB_OK;
}

void fill_report(fvb_solve_report& r, const SolveOut& o) {
  r.iterations = o.iterations;
  r.converged = o.converged;
  r.initial_residual = o.res0;
  r.final_residual = o.res;
  r.wall_time = o.kernel_ms * 1e-3;
  r.error_iteration = o.error_iteration;
  r.error_kind = o.error_kind;
  r.t_smvp = o.t_smvp;
  r.t_daxpy = o.t_daxpy;
  r.t_reduction = o.t_red;
}

int log_solve(fvb_step_report* rep, int solver, int field, const SolveOut& o) {
  if (rep->n_solves >= FVB_MAX_SOLVES) {
    fvb_set_error("too many solves in one step");
    return FVB_E_ARG;
  }
  const int k = rep->n_solves++;
  rep->solver[k] = solver;
  rep->field[k] = field;
  fill_report(rep->rep[k], o);
  return FVB_OK;
}

float ev_ms(Ctx* c, int a, int b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]);
  return ms;
}

// Event record that becomes a timing node when the stream is being
// captured into a step graph (a plain record otherwise).
void rec(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &st);
  if (st == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}

// RunState.ops timing: an event pair around each operator of the step
enum OpId { OP_DDT = 0, OP_CONV = 1, OP_LAP = 2, OP_GRAD = 3, OP_DIV = 4 };

int op_begin(Ctx* c, int op) {
  if (c->n_op >= Ctx::kOpEvents / 2) return -1;
  const int k = c->n_op++;
  c->op_id[k] = op;
  rec(c->opev[2 * k], c->stream);
  return k;
}
void op_end(Ctx* c, int k) {
  if (k >= 0) rec(c->opev[2 * k + 1], c->stream);
}
void op_collect(Ctx* c, fvb_step_report* rep) {
  for (int k = 0; k < c->n_op; ++k) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->opev[2 * k], c->opev[2 * k + 1]);
    rep->op_seconds[c->op_id[k]] += 1e-3 * ms;
    rep->op_calls[c->op_id[k]] += 1;
  }
  c->n_op = 0;
}

uint64_t fnv1a(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// One assembly segment of a step: the kernels, memsets and timing events
// between two solver readbacks (host syncs).  The first time a segment
// instance runs under a step configuration it is captured into a CUDA graph;
// later steps replay the graph, one launch instead of 5-15 kernel launches,
// memsets and event records (the small configs are launch-bound: C1 has 52
// launches per step).  Kernel arguments are device pointers that never move
// after the context's allocations and configuration scalars that are part
// of the key, so a replay launches exactly the kernels a direct run would,
// with the same arguments (same results, bitwise).  The host bookkeeping of
// the segment (operator-timer ids, launch count) is recorded at capture and
// re-applied on replay.  Decomposed contexts (their halo syncs talk to the
// peers) and FVB_STEP_NO_GRAPHS run the body directly.
template <class F>
int step_segment(Ctx* c, const fvb_step_cfg* cfg, int id, int a, int b, F&& body) {
  if (c->teamed() || (c->solver_flags & FVB_STEP_NO_GRAPHS)) return body();
  if (c->seg_allocs != c->allocs.size()) {  // new allocations: pointers may have moved
    for (auto& kv : c->segs) cudaGraphExecDestroy(kv.second.exec);
    c->segs.clear();
    c->seg_allocs = c->allocs.size();
  }
  // the key: segment instance, operator-timer position, options, and the
  // step configuration without the time (no kernel reads cfg->t)
  fvb_step_cfg kc = *cfg;
  kc.t = 0.0;
  const int key_ints[5] = {id, a, b, c->n_op, c->solver_flags};
  const uint64_t key = fnv1a(&kc, sizeof kc, fnv1a(key_ints, sizeof key_ints));
  auto it = c->segs.find(key);
  if (it != c->segs.end()) {
    const Ctx::Seg& sg = it->second;
    for (int op : sg.ops) c->op_id[c->n_op++] = op;
    g_launches.fetch_add(sg.launches, std::memory_order_relaxed);
    FVB_CUDA(cudaGraphLaunch(sg.exec, c->stream));
    return FVB_OK;
  }
  if (c->segs.size() >= 64) {  // the configuration keeps changing: start over
    for (auto& kv : c->segs) cudaGraphExecDestroy(kv.second.exec);
    c->segs.clear();
  }
  const int n_op0 = c->n_op;
  const unsigned long long l0 = g_launches.load(std::memory_order_relaxed);
  FVB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const int rc = body();
  cudaGraph_t g = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(c->stream, &g);
  if (rc != FVB_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  FVB_CUDA(ec);
  Ctx::Seg sg;
  const cudaError_t ei = cudaGraphInstantiate(&sg.exec, g, 0);
  cudaGraphDestroy(g);
  FVB_CUDA(ei);
  sg.ops.assign(c->op_id + n_op0, c->op_id + c->n_op);
  sg.launches = g_launches.load(std::memory_order_relaxed) - l0;
  FVB_CUDA(cudaGraphLaunch(sg.exec, c->stream));
  c->segs.emplace(key, std::move(sg));
  return FVB_OK;
}

enum SegId { SEG_MOM_ASM = 1, SEG_MOM_RHS = 2, SEG_P_PRE = 3, SEG_P_ASM = 4, SEG_P_CORR = 5 };

// _momentum_matrix (coupling.py:216-231)
int momentum_matrix(Ctx* c, const fvb_step_cfg* cfg, bool with_ddt) {
  StepWork w = work_of(c);
  const size_t n = c->nr;
  double* b0 = c->slot(S_B0);
  double* gu = c->slot(S_GU);
  MatView Am{w.Vm, w.crsm};
  FVB_CUDA(cudaMemsetAsync(w.Vm, 0, sizeof(double) * c->k * n, c->stream));
  if (c->nnz_crs) FVB_CUDA(cudaMemsetAsync(w.crsm, 0, sizeof(double) * c->nnz_crs, c->stream));
  FVB_CUDA(cudaMemsetAsync(b0, 0, sizeof(double) * 3 * size_t(c->nc), c->stream));
  if (with_ddt) {
    const int t = op_begin(c, OP_DDT);
    FVB_TRY(op_ddt(c, 3, Am, b0, c->u, cfg->dt, 1.0));
    op_end(c, t);
  }
  int t = op_begin(c, OP_CONV);
  FVB_TRY(op_convection(c, 0, 3, Am, b0, c->flux, c->ub, cfg->scheme, 1.0));
  op_end(c, t);
  t = op_begin(c, OP_LAP);
  const bool corr = cfg->nonorth_correction && cfg->limiter > 0.0;
  if (corr) {
    FVB_TRY(op_gradient(c, 0, 3, c->u, c->ub, gu));
    FVB_TRY(team_halo(c, S_GU, 9));  // face-interpolated gradient on processor faces
  }
  FVB_TRY(op_laplacian(c, 0, 3, Am, b0, cfg->nu, nullptr, c->u, c->ub, gu,
                       cfg->nonorth_correction, cfg->limiter, -1.0, nullptr, nullptr));
  op_end(c, t);
  return FVB_OK;
}

// _solve_momentum (coupling.py:234-279); returns worst normalised residual
int solve_momentum(Ctx* c, const fvb_step_cfg* cfg, bool relax, fvb_step_report* rep) {
  StepWork w = work_of(c);
  const int n = c->nr;
  const size_t nv = c->nc;
  const int g = grid_for(n, kThreads);
  double* diag = c->slot(S_DIAG);
  double* gp = c->slot(S_GP);
  double* rhs = c->slot(S_RHS);
  const bool relaxing = relax && cfg->alpha_u < 1.0;
  // ||b_c|| of the three solve right-hand sides: block partials on the
  // device, read back with the solve's results (one host sync for both)
  const int sblocks = 2 * c->num_sms;
  double* spart = c->partials + kStepPartials;
  FVB_TRY(step_segment(c, cfg, SEG_MOM_RHS, relaxing, 0, [&] {
    { k_get_diag<<<g, kThreads, 0, c->stream>>>(n, c->diag_slot, w.Vm, diag); fvb::note_launch(); }
    const int tg = op_begin(c, OP_GRAD);
    FVB_TRY(op_gradient(c, 1, 1, c->p, c->pb, gp));
    op_end(c, tg);
    { k_mom_rhs<<<g, kThreads, 0, c->stream>>>(n, nv, c->slot(S_B0), c->vol, gp, diag, c->u, rhs,
                                             w.Vm, c->diag_slot, relaxing, cfg->alpha_u); fvb::note_launch(); }
    FVB_CUDA(cudaGetLastError());
    { k_sumsq<<<sblocks, kThreads, 0, c->stream>>>(c->nr, nv, 3, rhs, spart); fvb::note_launch(); }
    FVB_CUDA(cudaGetLastError());
    rec(c->ev[2], c->stream);
    // the batched solve updates the three components in place; the reference
    // solves them one by one and raises before assigning a failed one
    // (coupling.py:259-277), so keep u to restore the unsolved components
    FVB_CUDA(cudaMemcpyAsync(c->u_save, c->u, sizeof(double) * 3 * nv, cudaMemcpyDeviceToDevice,
                             c->stream));
    return FVB_OK;
  }));
  std::vector<double> hpart(3 * size_t(sblocks));
  const Readback rb{spart, hpart.data(), 3 * sblocks};
  const double* b[3] = {rhs, rhs + nv, rhs + 2 * nv};
  double* x[3] = {c->u, c->u + nv, c->u + 2 * nv};
  SolveOut out[3];
  FVB_TRY(bicgstab_solve(c, MatView{w.Vm, w.crsm}, 3, b, x, cfg->mom_tol, cfg->mom_abs_tol,
                         cfg->mom_max_iters, out, &rb));
  FVB_CUDA(cudaEventRecord(c->ev[3], c->stream));
  double bn2[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k)
    for (int q = 0; q < sblocks; ++q) bn2[k] += hpart[size_t(k) * sblocks + q];
  FVB_TRY(team_allreduce(c, bn2, 3, RED_SUM));
  double bn[3], bscale = 0.0;
  for (int k = 0; k < 3; ++k) {
    bn[k] = std::sqrt(bn2[k]);
    bscale = std::max(bscale, bn[k]);
  }
  bscale = std::max(bscale, 1e-30);
  static const char* names[3] = {"ux", "uy", "uz"};
  double worst = 0.0;
  for (int k = 0; k < 3; ++k) {
    if (out[k].error_kind != SE_NONE) {
      rep->failed_solve = rep->n_solves;
      FVB_CUDA(cudaMemcpyAsync(c->u + k * nv, c->u_save + k * nv, sizeof(double) * (3 - k) * nv,
                               cudaMemcpyDeviceToDevice, c->stream));
      FVB_CUDA(cudaStreamSynchronize(c->stream));
      std::string msg = solve_error_text("bicgstab", out[k], out[k].error_iteration);
      fvb_set_error("momentum solve for %s failed at outer {outer}: %s", names[k], msg.c_str());
      return out[k].error_kind == SE_TIMEOUT ? FVB_E_TIMEOUT : FVB_E_COUPLING;
    }
    FVB_TRY(log_solve(rep, 1, k, out[k]));
    worst = std::max(worst, out[k].res0 * bn[k] / bscale);
  }
  if (relaxing) {
    { k_set_diag<<<g, kThreads, 0, c->stream>>>(n, c->diag_slot, w.Vm, diag); fvb::note_launch(); }
    FVB_CUDA(cudaGetLastError());
  }
  FVB_TRY(team_halo(c, S_U, 3));  // A u of the correctors gathers ghost u
  rep->mom_res = worst;
  return FVB_OK;
}

// _pressure_correct (coupling.py:282-344)
int pressure_correct(Ctx* c, const fvb_step_cfg* cfg, bool relax_p, fvb_step_report* rep,
                     double* first_res, double* t_asm, double* t_solve, double* t_corr,
                     int corr_index) {
  StepWork w = work_of(c);
  const int n = c->nr;
  const size_t nv = c->nc;
  const int g = grid_for(n, kThreads);
  double* hv = c->slot(S_HV);
  double* rau = c->slot(S_RAU);
  double* au = c->slot(S_AU);
  double* gp = c->slot(S_GP);
  double* divh = c->slot(S_DIVH);
  double* rl = c->slot(S_RL);
  double* rp = c->slot(S_RP);
  double* pbefore = c->slot(S_PBEFORE);
  FVB_TRY(step_segment(c, cfg, SEG_P_PRE, relax_p, 0, [&] {
    rec(c->ev[4], c->stream);
    MatView Am{w.Vm, w.crsm};
    for (int k = 0; k < 3; ++k) FVB_TRY(smvp(c, Am, c->u + k * nv, au + k * nv));
    { k_hbya<<<g, kThreads, 0, c->stream>>>(n, nv, c->u, c->slot(S_B0), au, c->slot(S_DIAG), c->vol,
                                          hv, rau); fvb::note_launch(); }
    FVB_CUDA(cudaGetLastError());
    FVB_TRY(team_halo(c, S_HV, 4));  // HbyA and rAU on processor faces
    FVB_TRY(op_face_flux(c, 3, hv, c->ub, 0, w.phih));
    const int td = op_begin(c, OP_DIV);
    FVB_TRY(op_divergence(c, w.phih, divh));
    op_end(c, td);
    FVB_TRY(op_interp(c, -1, 1, rau, nullptr, w.rauf));
    if (relax_p) FVB_CUDA(cudaMemcpyAsync(pbefore, c->p, sizeof(double) * nv, cudaMemcpyDeviceToDevice, c->stream));
    rec(c->ev[5], c->stream);
    return FVB_OK;
  }));
  float asm_ms = 0.f, solve_ms = 0.f;
  const bool corr = cfg->nonorth_correction && cfg->limiter > 0.0;
  MatView Ap{w.Vp, w.crsp};
  for (int it = 0; it <= cfg->n_nonorth_correctors; ++it) {
    FVB_TRY(step_segment(c, cfg, SEG_P_ASM, it, 0, [&] {
      rec(c->ev[6], c->stream);
      FVB_CUDA(cudaMemsetAsync(w.Vp, 0, sizeof(double) * c->k * size_t(n), c->stream));
      if (c->nnz_crs) FVB_CUDA(cudaMemsetAsync(w.crsp, 0, sizeof(double) * c->nnz_crs, c->stream));
      FVB_CUDA(cudaMemsetAsync(rl, 0, sizeof(double) * nv, c->stream));
      const int tl = op_begin(c, OP_LAP);
      if (corr) {
        FVB_TRY(op_gradient(c, 1, 1, c->p, c->pb, gp));
        FVB_TRY(team_halo(c, S_GP, 3));
      }
      FVB_TRY(op_laplacian(c, 1, 1, Ap, rl, 0.0, w.rauf, c->p, c->pb, gp,
                           cfg->nonorth_correction, cfg->limiter, -1.0, w.coef, w.corr));
      op_end(c, tl);
      { k_p_rhs<<<g, kThreads, 0, c->stream>>>(n, rl, divh, rp); fvb::note_launch(); }
      if (cfg->pin_pressure)
        { k_pin<<<1, 1, 0, c->stream>>>(n, c->diag_slot, w.Vp, rp, cfg->pressure_ref_cell,
                                      cfg->pressure_ref_value); fvb::note_launch(); }
      FVB_CUDA(cudaGetLastError());
      rec(c->ev[7], c->stream);
      return FVB_OK;
    }));
    SolveOut o;
    FVB_TRY(cg_solve(c, Ap, rp, c->p, cfg->p_tol, cfg->p_abs_tol, cfg->p_max_iters, &o));
    asm_ms += ev_ms(c, 6, 7);
    FVB_CUDA(cudaEventRecord(c->ev[6], c->stream));
    FVB_CUDA(cudaEventSynchronize(c->ev[6]));
    solve_ms += ev_ms(c, 7, 6);
    if (o.error_kind != SE_NONE) {
      rep->failed_solve = rep->n_solves;
      std::string msg = solve_error_text("cg", o, o.error_iteration);
      fvb_set_error("pressure solve failed at outer {outer}: %s", msg.c_str());
      return o.error_kind == SE_TIMEOUT ? FVB_E_TIMEOUT : FVB_E_COUPLING;
    }
    FVB_TRY(log_solve(rep, 0, 3, o));
    if (*first_res < 0) *first_res = o.res0;
    FVB_TRY(team_halo(c, S_P, 1));  // unrelaxed p on processor faces
  }
  // the correction tail is timed by an event pair read at the end of the
  // step (no host sync here: the next corrector's launches queue behind it)
  const bool defer = corr_index < Ctx::kTailPairs;
  cudaEvent_t e0 = defer ? c->cev[2 * corr_index] : c->ev[6];
  cudaEvent_t e1 = defer ? c->cev[2 * corr_index + 1] : c->ev[7];
  FVB_TRY(step_segment(c, cfg, SEG_P_CORR, corr_index, relax_p, [&] {
    rec(e0, c->stream);
    FVB_TRY(op_lap_flux(c, 1, 1, w.coef, w.corr, c->p, c->pb, w.lf));
    { k_flux_corr<<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(c->nf, w.phih, w.lf, c->flux); fvb::note_launch(); }
    if (relax_p && cfg->alpha_p < 1.0) {
      // the neighbours may still be reading the unrelaxed ghost p (their
      // laplacian_face_flux): sync before overwriting it (write-after-read)
      FVB_TRY(team_halo(c, S_P, 0));
      { k_relax_p<<<g, kThreads, 0, c->stream>>>(n, c->p, pbefore, cfg->alpha_p); fvb::note_launch(); }
      FVB_TRY(team_halo(c, S_P, 1));
    }
    FVB_CUDA(cudaGetLastError());
    FVB_TRY(op_apply_bcs(c, 1, 1, c->p, c->pb));
    const int tg = op_begin(c, OP_GRAD);
    FVB_TRY(op_gradient(c, 1, 1, c->p, c->pb, gp));
    op_end(c, tg);
    { k_u_corr<<<g, kThreads, 0, c->stream>>>(n, nv, hv, rau, gp, c->u); fvb::note_launch(); }
    FVB_CUDA(cudaGetLastError());
    FVB_TRY(team_halo(c, S_U, 3));
    FVB_TRY(op_apply_bcs(c, 0, 3, c->u, c->ub));
    rec(e1, c->stream);
    return FVB_OK;
  }));
  *t_asm += (ev_ms(c, 4, 5) + asm_ms) * 1e-3;  // complete: the CG readback synced
  *t_solve += solve_ms * 1e-3;
  if (defer) {
    c->n_tail = corr_index + 1;
  } else {
    FVB_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FVB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *t_corr += ms * 1e-3;
  }
  return FVB_OK;
}

int run_step(Ctx* c, const fvb_step_cfg* cfg, const double* speeds, fvb_step_report* rep,
             bool piso) {
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_pattern(c));
  FVB_TRY(need_bc(c, 0));
  FVB_TRY(need_bc(c, 1));
  FVB_TRY(ensure_work(c));
  memset(rep, 0, sizeof(*rep));
  c->n_op = 0;
  rep->failed_solve = -1;
  rep->p_res = -1.0;
  if (c->n_patches[0] && speeds)
    FVB_TRY(h2d(c, c->bc_speed[0], speeds, size_t(c->n_patches[0])));
  FVB_TRY(step_segment(c, cfg, SEG_MOM_ASM, piso, 0, [&] {
    rec(c->ev[0], c->stream);
    if (piso) {  // piso_time_step applies BCs at the new time first (coupling.py:360-361)
      FVB_TRY(op_apply_bcs(c, 0, 3, c->u, c->ub));
      FVB_TRY(op_apply_bcs(c, 1, 1, c->p, c->pb));
    }
    FVB_TRY(momentum_matrix(c, cfg, piso));
    rec(c->ev[1], c->stream);
    return FVB_OK;
  }));
  FVB_TRY(solve_momentum(c, cfg, !piso, rep));
  FVB_CUDA(cudaEventSynchronize(c->ev[3]));
  rep->t_momentum_assembly = ev_ms(c, 0, 1) * 1e-3;
  rep->t_momentum_solve = ev_ms(c, 2, 3) * 1e-3;
  double first = -1.0;
  const int ncorr = piso ? cfg->n_correctors : 1;
  c->n_tail = 0;
  for (int k = 0; k < ncorr; ++k)
    FVB_TRY(pressure_correct(c, cfg, !piso, rep, &first, &rep->t_pressure_assembly,
                             &rep->t_pressure_solve, &rep->t_correction, k));
  rep->p_res = first;
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < c->n_tail; ++k) {
    float ms = 0.f;
    FVB_CUDA(cudaEventElapsedTime(&ms, c->cev[2 * k], c->cev[2 * k + 1]));
    rep->t_correction += ms * 1e-3;
  }
  op_collect(c, rep);
  if (c->teamed()) {
    unsigned err = 0;
    FVB_CUDA(cudaMemcpyAsync(&err, c->sync + 3, sizeof err, cudaMemcpyDeviceToHost, c->stream));
    FVB_CUDA(cudaStreamSynchronize(c->stream));
    if (err) return team_timeout_error(c);
  }
  return FVB_OK;
}

}  // namespace

// ================================================================ C ABI
extern "C" {

int fvb_version(void) { return 100; }
const char* fvb_last_error(void) { return g_last_error.c_str(); }
int fvb_device_can_access_peer(int device, int peer, int* ok) {
  *ok = 0;
  if (device == peer) {
    *ok = 1;
    return FVB_OK;
  }
  FVB_CUDA(cudaDeviceCanAccessPeer(ok, device, peer));
  return FVB_OK;
}

int fvb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int fvb_ctx_create(int device, fvb_ctx** out) {
  auto* h = new fvb_ctx();
  Ctx* c = &h->c;
  c->dev = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    fvb_set_error("cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
    delete h;
    return FVB_E_CUDA;
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    fvb_set_error("stream creation failed");
    delete h;
    return FVB_E_CUDA;
  }
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  for (auto& ev : c->tev) cudaEventCreate(&ev);
  for (auto& ev : c->kev) cudaEventCreate(&ev);
  for (auto& ev : c->opev) cudaEventCreate(&ev);
  for (auto& ev : c->cev) cudaEventCreate(&ev);
  int rc = dalloc(c, &c->sync, 64);
  if (!rc) rc = dalloc(c, &c->partials, 16 * 4096 + 256);
  if (!rc) rc = dalloc(c, &c->ipart, 64);
  if (rc) {
    fvb_ctx_destroy(h);
    return rc;
  }
  cudaMemset(c->sync, 0, 64 * sizeof(unsigned));
  *out = h;
  return FVB_OK;
}

int fvb_ctx_destroy(fvb_ctx* h) {
  if (!h) return FVB_OK;
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& kv : c->segs) cudaGraphExecDestroy(kv.second.exec);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : c->tev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : c->kev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : c->opev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : c->cev)
    if (ev) cudaEventDestroy(ev);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete h;
  return FVB_OK;
}

int64_t fvb_ctx_device_bytes(fvb_ctx* h) { return h ? h->c.bytes : 0; }

int fvb_upload_mesh_part(fvb_ctx* h, int64_t n_cells, int64_t n_rows, int64_t n_faces,
                         int64_t n_internal, const int64_t* owner, const int64_t* neighbour,
                         const double* sf, const double* smag, const double* vol, const double* w,
                         const double* d, const double* db) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  if (c->have_mesh) {
    fvb_set_error("mesh already uploaded");
    return FVB_E_ARG;
  }
  if (n_cells <= 0 || n_rows <= 0 || n_rows > n_cells || n_faces < n_internal ||
      n_faces >= (int64_t(1) << 31) || n_cells >= (int64_t(1) << 31)) {
    fvb_set_error("mesh sizes out of range");
    return FVB_E_ARG;
  }
  if (c->have_pattern && n_rows != c->nr) {
    fvb_set_error("mesh rows %lld do not match the pattern rows %d", (long long)n_rows, c->nr);
    return FVB_E_MESH;
  }
  c->nc = int(n_cells);
  c->nr = int(n_rows);
  c->nf = int(n_faces);
  c->ni = int(n_internal);
  c->nb = c->nf - c->ni;
  const size_t nc = c->nc, nr = c->nr, nf = c->nf, ni = c->ni, nb = c->nb;
  std::vector<int> own(nf), nbr(ni);
  for (size_t f = 0; f < nf; ++f) {
    if (owner[f] < 0 || owner[f] >= n_cells) {
      fvb_set_error("owner cell index out of range");
      return FVB_E_MESH;
    }
    own[f] = int(owner[f]);
  }
  for (size_t f = 0; f < ni; ++f) {
    if (neighbour[f] < 0 || neighbour[f] >= n_cells) {
      fvb_set_error("neighbour cell index out of range");
      return FVB_E_MESH;
    }
    nbr[f] = int(neighbour[f]);
  }
  for (size_t f = ni; f < nf; ++f)
    if (size_t(own[f]) >= nr) {
      fvb_set_error("boundary face %zu is owned by a ghost cell", f);
      return FVB_E_MESH;
    }
  // per-row face list: owned faces ascending, then neighbour faces ascending
  // (ghost cells get no list: their rows belong to another rank)
  std::vector<int> nown(nr, 0), nnb(nr, 0);
  for (size_t f = 0; f < nf; ++f)
    if (size_t(own[f]) < nr) nown[own[f]]++;
  for (size_t f = 0; f < ni; ++f)
    if (size_t(nbr[f]) < nr) nnb[nbr[f]]++;
  std::vector<int> ptr(nr + 1, 0);
  for (size_t i = 0; i < nr; ++i) {
    const int64_t next = int64_t(ptr[i]) + nown[i] + nnb[i];
    if (next >= (int64_t(1) << 31)) {
      fvb_set_error("face list too long");
      return FVB_E_ARG;
    }
    ptr[i + 1] = int(next);
  }
  std::vector<int> cf(ptr[nr]);
  std::vector<int> po(nr), pn(nr);
  for (size_t i = 0; i < nr; ++i) {
    po[i] = ptr[i];
    pn[i] = ptr[i] + nown[i];
  }
  for (size_t f = 0; f < nf; ++f)
    if (size_t(own[f]) < nr) cf[po[own[f]]++] = int(f);
  for (size_t f = 0; f < ni; ++f)
    if (size_t(nbr[f]) < nr) cf[pn[nbr[f]]++] = ~int(f);
  // SoA geometry
  std::vector<double> tmp(std::max(nf, nc));
  auto up3 = [&](const double* src, size_t m, double** o0, double** o1, double** o2) -> int {
    double* outs[3];
    for (int k = 0; k < 3; ++k) {
      FVB_TRY(dalloc(c, &outs[k], m));
      for (size_t i = 0; i < m; ++i) tmp[i] = src[3 * i + k];
      if (m) FVB_CUDA(cudaMemcpy(outs[k], tmp.data(), m * sizeof(double), cudaMemcpyHostToDevice));
    }
    *o0 = outs[0];
    *o1 = outs[1];
    *o2 = outs[2];
    return FVB_OK;
  };
  auto up1 = [&](const auto* src, size_t m, auto** o) -> int {
    FVB_TRY(dalloc(c, o, m));
    if (m) FVB_CUDA(cudaMemcpy(*o, src, m * sizeof(**o), cudaMemcpyHostToDevice));
    return FVB_OK;
  };
  FVB_TRY(up1(own.data(), nf, &c->own));
  FVB_TRY(up1(nbr.data(), ni, &c->nbr));
  FVB_TRY(up1(ptr.data(), nr + 1, &c->cf_ptr));
  FVB_TRY(up1(cf.data(), cf.size(), &c->cf));
  FVB_TRY(up3(sf, nf, &c->sx, &c->sy, &c->sz));
  FVB_TRY(up1(smag, nf, &c->smag));
  FVB_TRY(up1(vol, nc, &c->vol));
  FVB_TRY(up1(w, ni, &c->w));
  double *dx, *dy, *dz, *dbx, *dby, *dbz;
  FVB_TRY(up3(d, ni, &dx, &dy, &dz));
  FVB_TRY(up3(db, nb, &dbx, &dby, &dbz));
  FVB_TRY(dalloc(c, &c->a, nf));
  FVB_TRY(dalloc(c, &c->kx, nf));
  FVB_TRY(dalloc(c, &c->ky, nf));
  FVB_TRY(dalloc(c, &c->kz, nf));
  FVB_TRY(op_precompute_geometry(c, dx, dy, dz, dbx, dby, dbz));
  // coincident-centroid checks of fvm.py:349-350 / 368-370 (norms as mesh.py)
  c->first_zero_dmag = -1;
  for (size_t f = 0; f < ni; ++f) {
    const double m = std::sqrt((d[3 * f] * d[3 * f] + d[3 * f + 1] * d[3 * f + 1]) +
                               d[3 * f + 2] * d[3 * f + 2]);
    if (m == 0.0) {
      c->first_zero_dmag = int(f);
      break;
    }
  }
  c->dbmag_host.resize(nb);
  for (size_t j = 0; j < nb; ++j)
    c->dbmag_host[j] = std::sqrt((db[3 * j] * db[3 * j] + db[3 * j + 1] * db[3 * j + 1]) +
                                 db[3 * j + 2] * db[3 * j + 2]);
  // coupled state: u, p in the cell pool; face / boundary arrays apart
  FVB_TRY(ensure_pool(c));
  FVB_TRY(dalloc(c, &c->flux, nf));
  FVB_TRY(dalloc(c, &c->ub, 3 * nb));
  FVB_TRY(dalloc(c, &c->pb, nb));
  FVB_CUDA(cudaMemset(c->flux, 0, (nf ? nf : 1) * sizeof(double)));
  FVB_CUDA(cudaMemset(c->ub, 0, 3 * (nb ? nb : 1) * sizeof(double)));
  FVB_CUDA(cudaMemset(c->pb, 0, (nb ? nb : 1) * sizeof(double)));
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  // the temporaries dx.. stay in the allocation list (freed with the context)
  c->have_mesh = true;
  return ensure_work(c);
}

int fvb_upload_mesh(fvb_ctx* h, int64_t n_cells, int64_t n_faces, int64_t n_internal,
                    const int64_t* owner, const int64_t* neighbour, const double* sf,
                    const double* smag, const double* vol, const double* w, const double* d,
                    const double* db) {
  return fvb_upload_mesh_part(h, n_cells, n_cells, n_faces, n_internal, owner, neighbour, sf,
                              smag, vol, w, d, db);
}

namespace fvb {
// Stencil-code compression of the column indices (PatternView::code): the
// solvers' SpMV passes read one byte per row instead of K int32 indices
// when the rows' column-offset tuples (col - row per slot) fall into at
// most kMaxCodes distinct patterns — every row of a structured hex mesh
// does (27 tuples: interior, faces, edges, corners).  Rows outside the
// dictionary are coded kEscapeCode and read their explicit indices; with
// more than 1/16 of the rows escaping the codes are not used at all.  The
// columns, and hence every product and sum, are exactly those of I.
static int build_stencil_codes(Ctx* c, const std::vector<int>& Is, size_t nn, size_t kk) {
  std::vector<uint8_t> code(nn, uint8_t(kEscapeCode));
  std::vector<int> tab;
  std::unordered_map<uint64_t, std::vector<int>> dict;  // hash -> codes
  size_t escapes = 0;
  std::vector<int> off(kk);
  for (size_t i = 0; i < nn; ++i) {
    uint64_t h = 1469598103934665603ull;
    for (size_t s = 0; s < kk; ++s) {
      const int col = Is[s * nn + i];
      off[s] = col < 0 ? kPadOffset : col - int(i);
      h = (h ^ uint32_t(off[s])) * 1099511628211ull;
    }
    int found = -1;
    auto it = dict.find(h);
    if (it != dict.end())
      for (int q : it->second)
        if (std::equal(off.begin(), off.end(), tab.begin() + size_t(q) * kk)) {
          found = q;
          break;
        }
    if (found < 0 && int(tab.size() / kk) < kMaxCodes) {
      found = int(tab.size() / kk);
      tab.insert(tab.end(), off.begin(), off.end());
      dict[h].push_back(found);
    }
    if (found < 0) {
      if (++escapes > nn / 16) return FVB_OK;  // not worth it: plain I
    } else {
      code[i] = uint8_t(found);
    }
  }
  FVB_TRY(dalloc(c, &c->scode, nn));
  FVB_CUDA(cudaMemcpy(c->scode, code.data(), nn, cudaMemcpyHostToDevice));
  FVB_TRY(dalloc(c, &c->stab, tab.size()));
  FVB_CUDA(cudaMemcpy(c->stab, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice));
  c->n_scode = int(tab.size() / kk);
  c->n_sescape = int64_t(escapes);
  return FVB_OK;
}
}  // namespace fvb

namespace fvb {
// Reverse Cuthill-McKee order of the pattern's row graph (CG on meshes whose
// numbering leaves no stencil codes, e.g. a randomly renumbered mesh): BFS
// from a minimum-degree row of every component, neighbours by ascending
// degree, reversed.  Only the solver's internal order changes: every row
// keeps its slots in the same order (same products, same sums); only the
// grouping of the dot products over rows moves.
static int build_rcm(Ctx* c, const std::vector<int>& Is, const std::vector<int>& ds, size_t nn,
                     size_t kk) {
  std::vector<int> deg(nn, 0);
  for (size_t i = 0; i < nn; ++i)
    for (size_t s = 0; s < kk; ++s) {
      const int col = Is[s * nn + i];
      if (col >= 0 && size_t(col) != i) deg[i]++;
    }
  std::vector<int> order;
  order.reserve(nn);
  std::vector<char> seen(nn, 0);
  std::vector<int> by_deg(nn);
  for (size_t i = 0; i < nn; ++i) by_deg[i] = int(i);
  std::stable_sort(by_deg.begin(), by_deg.end(), [&](int a, int b) { return deg[a] < deg[b]; });
  std::vector<int> nb;
  for (int start : by_deg) {
    if (seen[start]) continue;
    seen[start] = 1;
    size_t head = order.size();
    order.push_back(start);
    while (head < order.size()) {
      const int i = order[head++];
      nb.clear();
      for (size_t s = 0; s < kk; ++s) {
        const int col = Is[s * nn + size_t(i)];
        if (col >= 0 && col != i && !seen[col]) {
          seen[col] = 1;
          nb.push_back(col);
        }
      }
      std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
      order.insert(order.end(), nb.begin(), nb.end());
    }
  }
  std::reverse(order.begin(), order.end());  // perm[new] = old
  std::vector<int> iperm(nn);
  for (size_t r = 0; r < nn; ++r) iperm[size_t(order[r])] = int(r);
  std::vector<int> Ip(nn * kk), dsp(nn);
  for (size_t r = 0; r < nn; ++r) {
    const size_t o = size_t(order[r]);
    dsp[r] = ds[o];
    for (size_t s = 0; s < kk; ++s) {
      const int col = Is[s * nn + o];
      Ip[s * nn + r] = col < 0 ? -1 : iperm[size_t(col)];
    }
  }
  auto up = [&](const std::vector<int>& v, int** o) -> int {
    FVB_TRY(dalloc(c, o, v.size()));
    FVB_CUDA(cudaMemcpy(*o, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    return FVB_OK;
  };
  FVB_TRY(up(order, &c->rcm_perm));
  FVB_TRY(up(Ip, &c->rcm_I));
  FVB_TRY(up(dsp, &c->rcm_ds));
  return FVB_OK;
}
}  // namespace fvb

int fvb_upload_pattern(fvb_ctx* h, int64_t n, int64_t k, const int64_t* I,
                       const int64_t* diag_slot, const int64_t* face_addr, int64_t n_face_pairs,
                       int64_t nnz_crs, const int64_t* crs_row_ptr, const int64_t* crs_col) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  if (c->have_pattern) {
    fvb_set_error("pattern already uploaded");
    return FVB_E_ARG;
  }
  if (c->have_mesh && n != c->nr) {
    fvb_set_error("pattern size %lld does not match mesh rows %d", (long long)n, c->nr);
    return FVB_E_SPARSE;
  }
  if (k < 1 || k > kMaxK) {
    fvb_set_error("pattern width K=%lld outside 1..%d", (long long)k, kMaxK);
    return FVB_E_SPARSE;
  }
  if (n <= 0 || n * k >= (int64_t(1) << 31)) {
    fvb_set_error("pattern too large");
    return FVB_E_SPARSE;
  }
  if (!c->have_mesh) c->nc = c->nr = int(n);
  c->k = int(k);
  c->nnz_crs = int(nnz_crs);
  const size_t nn = size_t(n), kk = size_t(k), nk = nn * kk;
  std::vector<int> Is(nk), sf(nk, -1), ds(nn);
  for (size_t i = 0; i < nn; ++i) {
    ds[i] = int(diag_slot[i]);
    for (size_t s = 0; s < kk; ++s) {
      const int64_t col = I[i * kk + s];
      if (col >= c->nc) {
        fvb_set_error("pattern column %lld outside the %d local cells", (long long)col, c->nc);
        return FVB_E_SPARSE;
      }
      Is[s * nn + i] = int(col);
    }
  }
  std::vector<int> cptr(nn + 1, 0), ccol(nnz_crs), cface(nnz_crs, -1);
  if (nnz_crs) {
    for (size_t i = 0; i <= nn; ++i) cptr[i] = int(crs_row_ptr[i]);
    for (int64_t q = 0; q < nnz_crs; ++q) ccol[q] = int(crs_col[q]);
  }
  if (c->have_mesh && face_addr) {
    if (n_face_pairs != c->ni) {
      fvb_set_error("face_addr rows %lld != internal faces %d", (long long)n_face_pairs, c->ni);
      return FVB_E_SPARSE;
    }
    const int64_t split = int64_t(nk);
    for (int64_t f = 0; f < n_face_pairs; ++f) {
      for (int side = 0; side < 2; ++side) {
        const int64_t a = face_addr[2 * f + side];
        if (a < 0) continue;  // the row of that side belongs to another rank
        int* slot;
        if (a < split) {
          slot = &sf[size_t(a % k) * nn + size_t(a / k)];
        } else {
          slot = &cface[size_t(a - split)];
        }
        if (*slot >= 0) {
          fvb_set_error("faces %d and %lld join the same pair of cells; the device path "
                        "needs one face per cell pair", *slot, (long long)f);
          return FVB_E_SPARSE;
        }
        *slot = int(f);
      }
    }
  }
  auto up = [&](const std::vector<int>& v, int** o) -> int {
    FVB_TRY(dalloc(c, o, v.size()));
    if (!v.empty()) FVB_CUDA(cudaMemcpy(*o, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    return FVB_OK;
  };
  FVB_TRY(up(Is, &c->I));
  if (kk <= 16) FVB_TRY(build_stencil_codes(c, Is, nn, kk));
  // no stencil codes on a large single-domain 7-point pattern without CRS
  // tail: CG runs in RCM order (cg_solve)
  if (!c->scode && kk == 7 && nnz_crs == 0 && c->nc == c->nr && nn >= 65536)
    FVB_TRY(build_rcm(c, Is, ds, nn, kk));
  FVB_TRY(up(ds, &c->diag_slot));
  FVB_TRY(up(sf, &c->slot_face));
  if (nnz_crs) {
    FVB_TRY(up(cptr, &c->crs_ptr));
    FVB_TRY(up(ccol, &c->crs_col));
    FVB_TRY(up(cface, &c->crs_face));
  }
  FVB_TRY(ensure_pool(c));
  c->have_pattern = true;
  return ensure_work(c);
}

int fvb_set_bcs(fvb_ctx* h, int field, const uint8_t* kind, const int32_t* patch,
                const double* fixed, int n_patches) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  if (field < 0 || field > 1) {
    fvb_set_error("field must be 0 (u) or 1 (p)");
    return FVB_E_ARG;
  }
  const int ncomp = field == 0 ? 3 : 1;
  const size_t nb = c->nb;
  if (!c->have_bc[field]) {
    FVB_TRY(dalloc(c, &c->bc_kind[field], nb));
    FVB_TRY(dalloc(c, &c->bc_patch[field], nb));
    FVB_TRY(dalloc(c, &c->bc_fixed[field], ncomp * nb));
    FVB_TRY(dalloc(c, &c->bc_speed[field], size_t(std::max(n_patches, 1)) + 64));
  }
  if (n_patches > 64 + std::max(c->n_patches[field], 1) && c->have_bc[field]) {
    fvb_set_error("patch count changed");
    return FVB_E_ARG;
  }
  c->n_patches[field] = n_patches;
  if (nb) {
    FVB_CUDA(cudaMemcpy(c->bc_kind[field], kind, nb, cudaMemcpyHostToDevice));
    FVB_CUDA(cudaMemcpy(c->bc_patch[field], patch, nb * sizeof(int), cudaMemcpyHostToDevice));
    FVB_CUDA(cudaMemcpy(c->bc_fixed[field], fixed, ncomp * nb * sizeof(double), cudaMemcpyHostToDevice));
  }
  c->first_zero_dbmag_value[field] = -1;
  for (size_t j = 0; j < nb; ++j)
    if (bc_is_value(kind[j]) && c->dbmag_host[j] == 0.0) {
      c->first_zero_dbmag_value[field] = int(c->ni + j);
      break;
    }
  c->have_bc[field] = true;
  return FVB_OK;
}

int fvb_set_state(fvb_ctx* h, const double* u, const double* p, const double* flux,
                  const double* ub, const double* pb) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  if (u) FVB_TRY(h2d(c, c->u, u, 3 * size_t(c->nc)));
  if (p) FVB_TRY(h2d(c, c->p, p, size_t(c->nc)));
  if (flux) FVB_TRY(h2d(c, c->flux, flux, size_t(c->nf)));
  if (ub) FVB_TRY(h2d(c, c->ub, ub, 3 * size_t(c->nb)));
  if (pb) FVB_TRY(h2d(c, c->pb, pb, size_t(c->nb)));
  return sync(c);
}

int fvb_get_state(fvb_ctx* h, double* u, double* p, double* flux, double* ub, double* pb) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  if (u) FVB_TRY(d2h(c, u, c->u, 3 * size_t(c->nc)));
  if (p) FVB_TRY(d2h(c, p, c->p, size_t(c->nc)));
  if (flux) FVB_TRY(d2h(c, flux, c->flux, size_t(c->nf)));
  if (ub) FVB_TRY(d2h(c, ub, c->ub, 3 * size_t(c->nb)));
  if (pb) FVB_TRY(d2h(c, pb, c->pb, size_t(c->nb)));
  return sync(c);
}

// ----------------------------------------------------------- operators
int fvb_op_smvp(fvb_ctx* h, const double* V, const double* crs, const double* x, double* y) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_pattern(c));
  DevMatrix M;
  FVB_TRY(upload_matrix(c, M, V, crs));
  Tmp tx, ty;
  double *dx, *dy;
  FVB_TRY(tmp_upload(c, tx, x, c->nc, &dx));
  FVB_TRY(tmp_zero(c, ty, c->nc, &dy));
  FVB_TRY(smvp(c, M.m, dx, dy));
  FVB_TRY(d2h(c, y, dy, c->nc));
  return sync(c);
}

int fvb_op_stmvp(fvb_ctx* h, const double* V, const double* crs, const int64_t* J,
                 const int64_t* ell_twin_crs, const uint8_t* crs_twin_in_ell,
                 const int64_t* crs_twin_row, const int64_t* crs_twin_pos, const double* x,
                 double* y) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_pattern(c));
  const size_t n = c->nr, k = c->k, nz = c->nnz_crs;
  // twin tables to slot-major int32 (J is a slot, ell_twin_crs a CRS position)
  std::vector<int> js(n * k), tc(n * k), cr(nz), cp(nz);
  std::vector<uint8_t> ce(nz);
  for (size_t i = 0; i < n; ++i)
    for (size_t s = 0; s < k; ++s) {
      js[s * n + i] = int(J[i * k + s]);
      tc[s * n + i] = ell_twin_crs ? int(ell_twin_crs[i * k + s]) : -1;
    }
  for (size_t q = 0; q < nz; ++q) {
    ce[q] = crs_twin_in_ell[q];
    cr[q] = int(crs_twin_row[q]);
    cp[q] = int(crs_twin_pos[q]);
  }
  DevMatrix M;
  FVB_TRY(upload_matrix(c, M, V, crs));
  Tmp t1, t2, t3, t4, t5, tx, ty;
  int *dj, *dtc, *dcr, *dcp;
  uint8_t* dce;
  double *dx, *dy;
  FVB_TRY(tmp_upload(c, t1, js.data(), js.size(), &dj));
  FVB_TRY(tmp_upload(c, t2, tc.data(), tc.size(), &dtc));
  FVB_TRY(tmp_upload(c, t3, ce.data(), ce.size(), &dce));
  FVB_TRY(tmp_upload(c, t4, cr.data(), cr.size(), &dcr));
  FVB_TRY(tmp_upload(c, t5, cp.data(), cp.size(), &dcp));
  FVB_TRY(tmp_upload(c, tx, x, size_t(c->nc), &dx));
  FVB_TRY(tmp_zero(c, ty, n, &dy));
  FVB_TRY(stmvp(c, M.m, dj, dtc, dce, dcr, dcp, dx, dy));
  FVB_TRY(d2h(c, y, dy, n));
  return sync(c);
}

static int solve_common(fvb_ctx* h, bool use_cg, int ncomp, const double* V, const double* crs,
                        const double* b, const double* x0, double* x, double tol, double abs_tol,
                        int max_iters, fvb_solve_report* reps) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_pattern(c));
  const size_t n = c->nc;
  DevMatrix M;
  FVB_TRY(upload_matrix(c, M, V, crs));
  Tmp tb, tx;
  double *db, *dx;
  FVB_TRY(tmp_upload(c, tb, b, ncomp * n, &db));
  FVB_TRY(tmp_upload(c, tx, x0, ncomp * n, &dx));
  FVB_CUDA(cudaEventRecord(c->ev[0], c->stream));
  SolveOut out[3];
  if (use_cg) {
    FVB_TRY(cg_solve(c, M.m, db, dx, tol, abs_tol, max_iters, out));
  } else {
    const double* bb[3] = {db, db + n, db + 2 * n};
    double* xx[3] = {dx, dx + n, dx + 2 * n};
    FVB_TRY(bicgstab_solve(c, M.m, ncomp, bb, xx, tol, abs_tol, max_iters, out));
  }
  FVB_CUDA(cudaEventRecord(c->ev[1], c->stream));
  FVB_TRY(d2h(c, x, dx, ncomp * n));
  FVB_TRY(sync(c));
  for (int k = 0; k < ncomp; ++k) fill_report(reps[k], out[k]);
  for (int k = 0; k < ncomp; ++k) {
    if (out[k].error_kind != SE_NONE) {
      std::string msg = solve_error_text(use_cg ? "cg" : "bicgstab", out[k], out[k].error_iteration);
      fvb_set_error("%s", msg.c_str());
      return out[k].error_kind == SE_TIMEOUT ? FVB_E_TIMEOUT : FVB_E_SOLVER;
    }
  }
  return FVB_OK;
}

int fvb_op_cg(fvb_ctx* h, const double* V, const double* crs, const double* b, const double* x0,
              double* x, double tol, double abs_tol, int max_iters, fvb_solve_report* rep) {
  return solve_common(h, true, 1, V, crs, b, x0, x, tol, abs_tol, max_iters, rep);
}

int fvb_op_bicgstab(fvb_ctx* h, const double* V, const double* crs, const double* b,
                    const double* x0, double* x, double tol, double abs_tol, int max_iters,
                    fvb_solve_report* rep) {
  return solve_common(h, false, 1, V, crs, b, x0, x, tol, abs_tol, max_iters, rep);
}

int fvb_op_bicgstab_batched(fvb_ctx* h, int ncomp, const double* V, const double* crs,
                            const double* b, const double* x0, double* x, double tol,
                            double abs_tol, int max_iters, fvb_solve_report* reps) {
  if (ncomp != 1 && ncomp != 3) {
    fvb_set_error("ncomp must be 1 or 3");
    return FVB_E_ARG;
  }
  return solve_common(h, false, ncomp, V, crs, b, x0, x, tol, abs_tol, max_iters, reps);
}

int fvb_op_apply_bcs(fvb_ctx* h, int field, const double* values, const double* speeds,
                     double* boundary) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_bc(c, field));
  const int ncomp = field == 0 ? 3 : 1;
  if (speeds && c->n_patches[field]) FVB_TRY(h2d(c, c->bc_speed[field], speeds, size_t(c->n_patches[field])));
  Tmp tv, tb;
  double *dv, *db;
  FVB_TRY(tmp_upload(c, tv, values, ncomp * size_t(c->nc), &dv));
  FVB_TRY(tmp_zero(c, tb, ncomp * size_t(c->nb), &db));
  FVB_TRY(op_apply_bcs(c, field, ncomp, dv, db));
  FVB_TRY(d2h(c, boundary, db, ncomp * size_t(c->nb)));
  return sync(c);
}

int fvb_op_interpolate(fvb_ctx* h, int field, int ncomp, const double* values,
                       const double* boundary, double* face_values) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  if (field >= 0) FVB_TRY(need_bc(c, field));
  Tmp tv, tb, tf;
  double *dv, *db = nullptr, *df;
  FVB_TRY(tmp_upload(c, tv, values, ncomp * size_t(c->nc), &dv));
  FVB_TRY(tmp_upload(c, tb, boundary, boundary ? ncomp * size_t(c->nb) : 0, &db));
  FVB_TRY(tmp_zero(c, tf, ncomp * size_t(c->nf), &df));
  FVB_TRY(op_interp(c, field, ncomp, dv, db, df));
  FVB_TRY(d2h(c, face_values, df, ncomp * size_t(c->nf)));
  return sync(c);
}

int fvb_op_gradient(fvb_ctx* h, int field, int ncomp, const double* values,
                    const double* boundary, double* grad) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_bc(c, field));
  Tmp tv, tb, tg;
  double *dv, *db, *dg;
  FVB_TRY(tmp_upload(c, tv, values, ncomp * size_t(c->nc), &dv));
  FVB_TRY(tmp_upload(c, tb, boundary, ncomp * size_t(c->nb), &db));
  FVB_TRY(tmp_zero(c, tg, 3 * ncomp * size_t(c->nc), &dg));
  FVB_TRY(op_gradient(c, field, ncomp, dv, db, dg));
  FVB_TRY(d2h(c, grad, dg, 3 * ncomp * size_t(c->nc)));
  return sync(c);
}

int fvb_op_divergence(fvb_ctx* h, const double* flux, double* div) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  Tmp tf, td;
  double *df, *dd;
  FVB_TRY(tmp_upload(c, tf, flux, size_t(c->nf), &df));
  FVB_TRY(tmp_zero(c, td, size_t(c->nc), &dd));
  FVB_TRY(op_divergence(c, df, dd));
  FVB_TRY(d2h(c, div, dd, size_t(c->nc)));
  return sync(c);
}

int fvb_op_laplacian(fvb_ctx* h, int field, int ncomp, double* V, double* crs, double* rhs,
                     double gamma, const double* gamma_faces, const double* values,
                     const double* boundary, int nonorth, double limiter, double coeff,
                     double* coef, double* corr) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_pattern(c));
  FVB_TRY(need_bc(c, field));
  DevMatrix M;
  FVB_TRY(upload_matrix(c, M, V, crs));
  Tmp tr, tg, tv, tb, tgr, tco, tcr;
  double *dr, *dg = nullptr, *dv, *db, *dgr, *dco, *dcr;
  const size_t n = c->nc, nf = c->nf, nb = c->nb;
  FVB_TRY(tmp_upload(c, tr, rhs, ncomp * n, &dr));
  if (gamma_faces) FVB_TRY(tmp_upload(c, tg, gamma_faces, nf, &dg));
  FVB_TRY(tmp_upload(c, tv, values, ncomp * n, &dv));
  FVB_TRY(tmp_upload(c, tb, boundary, ncomp * nb, &db));
  FVB_TRY(tmp_zero(c, tgr, 3 * ncomp * n, &dgr));
  FVB_TRY(tmp_zero(c, tco, nf, &dco));
  FVB_TRY(tmp_zero(c, tcr, ncomp * nf, &dcr));
  if (nonorth && limiter > 0.0) FVB_TRY(op_gradient(c, field, ncomp, dv, db, dgr));
  FVB_TRY(op_laplacian(c, field, ncomp, M.m, dr, gamma, dg, dv, db, dgr, nonorth, limiter, coeff,
                       dco, dcr));
  FVB_TRY(download_matrix(c, M, V, crs));
  FVB_TRY(d2h(c, rhs, dr, ncomp * n));
  if (coef) FVB_TRY(d2h(c, coef, dco, nf));
  if (corr) FVB_TRY(d2h(c, corr, dcr, ncomp * nf));
  return sync(c);
}

int fvb_op_laplacian_flux(fvb_ctx* h, int field, int ncomp, const double* coef,
                          const double* corr, const double* values, const double* boundary,
                          double* flux_out) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_bc(c, field));
  const size_t n = c->nc, nf = c->nf, nb = c->nb;
  Tmp t1, t2, t3, t4, t5;
  double *dco, *dcr, *dv, *db, *dout;
  FVB_TRY(tmp_upload(c, t1, coef, nf, &dco));
  FVB_TRY(tmp_upload(c, t2, corr, ncomp * nf, &dcr));
  FVB_TRY(tmp_upload(c, t3, values, ncomp * n, &dv));
  FVB_TRY(tmp_upload(c, t4, boundary, ncomp * nb, &db));
  FVB_TRY(tmp_zero(c, t5, ncomp * nf, &dout));
  FVB_TRY(op_lap_flux(c, field, ncomp, dco, dcr, dv, db, dout));
  FVB_TRY(d2h(c, flux_out, dout, ncomp * nf));
  return sync(c);
}

int fvb_op_convection(fvb_ctx* h, int field, int ncomp, double* V, double* crs, double* rhs,
                      const double* flux, const double* boundary, int scheme, double coeff) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_pattern(c));
  FVB_TRY(need_bc(c, field));
  DevMatrix M;
  FVB_TRY(upload_matrix(c, M, V, crs));
  const size_t n = c->nc, nf = c->nf, nb = c->nb;
  Tmp t1, t2, t3;
  double *dr, *df, *db;
  FVB_TRY(tmp_upload(c, t1, rhs, ncomp * n, &dr));
  FVB_TRY(tmp_upload(c, t2, flux, nf, &df));
  FVB_TRY(tmp_upload(c, t3, boundary, ncomp * nb, &db));
  FVB_TRY(op_convection(c, field, ncomp, M.m, dr, df, db, scheme, coeff));
  FVB_TRY(download_matrix(c, M, V, crs));
  FVB_TRY(d2h(c, rhs, dr, ncomp * n));
  return sync(c);
}

int fvb_op_ddt(fvb_ctx* h, int ncomp, double* V, double* rhs, const double* old_values, double dt,
               double coeff) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_pattern(c));
  if (!(dt > 0.0)) {
    fvb_set_error("dt must be positive");
    return FVB_E_FVM;
  }
  std::vector<double> zero_crs(size_t(std::max(c->nnz_crs, 1)), 0.0);
  DevMatrix M;
  FVB_TRY(upload_matrix(c, M, V, zero_crs.data()));
  const size_t n = c->nc;
  Tmp t1, t2;
  double *dr, *dold;
  FVB_TRY(tmp_upload(c, t1, rhs, ncomp * n, &dr));
  FVB_TRY(tmp_upload(c, t2, old_values, ncomp * n, &dold));
  FVB_TRY(op_ddt(c, ncomp, M.m, dr, dold, dt, coeff));
  FVB_TRY(download_matrix(c, M, V, nullptr));
  FVB_TRY(d2h(c, rhs, dr, ncomp * n));
  return sync(c);
}

int fvb_state_apply_bcs(fvb_ctx* h, const double* u_speeds) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_bc(c, 0));
  FVB_TRY(need_bc(c, 1));
  if (c->n_patches[0] && u_speeds)
    FVB_TRY(h2d(c, c->bc_speed[0], u_speeds, size_t(c->n_patches[0])));
  FVB_TRY(op_apply_bcs(c, 0, 3, c->u, c->ub));
  FVB_TRY(op_apply_bcs(c, 1, 1, c->p, c->pb));
  return sync(c);
}

int fvb_op_face_flux(fvb_ctx* h, const double* values, const double* boundary,
                     double* flux_out) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_bc(c, 0));
  Tmp tv, tb, tf;
  double *dv, *db, *df;
  FVB_TRY(tmp_upload(c, tv, values, 3 * size_t(c->nc), &dv));
  FVB_TRY(tmp_upload(c, tb, boundary, 3 * size_t(c->nb), &db));
  FVB_TRY(tmp_zero(c, tf, size_t(c->nf), &df));
  FVB_TRY(op_face_flux(c, 3, dv, db, 0, df));
  FVB_TRY(d2h(c, flux_out, df, size_t(c->nf)));
  return sync(c);
}

int fvb_op_rhie_chow(fvb_ctx* h, const double* u, const double* ub, const double* p,
                     const double* pb, const double* a_diag, const double* d, const double* d_boundary,
                     double* flux_out) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_bc(c, 0));
  FVB_TRY(need_bc(c, 1));
  for (int i = 0; i < c->nr; ++i)
    if (a_diag[i] == 0.0) {
      fvb_set_error("zero momentum diagonal at cell %d", i);
      return FVB_E_FVM;
    }
  Tmp tu, tub, tp, tpb, ta, td, tdb, tg, tf;
  double *du, *dub, *dp, *dpb, *da, *dd, *ddb, *dg, *df;
  FVB_TRY(tmp_upload(c, tu, u, 3 * size_t(c->nc), &du));
  FVB_TRY(tmp_upload(c, tub, ub, 3 * size_t(c->nb), &dub));
  FVB_TRY(tmp_upload(c, tp, p, size_t(c->nc), &dp));
  FVB_TRY(tmp_upload(c, tpb, pb, size_t(c->nb), &dpb));
  FVB_TRY(tmp_upload(c, ta, a_diag, size_t(c->nc), &da));
  FVB_TRY(tmp_upload(c, td, d, 3 * size_t(c->ni), &dd));
  FVB_TRY(tmp_upload(c, tdb, d_boundary, 3 * size_t(c->nb), &ddb));
  FVB_TRY(tmp_zero(c, tg, 3 * size_t(c->nc), &dg));
  FVB_TRY(tmp_zero(c, tf, size_t(c->nf), &df));
  FVB_TRY(op_gradient(c, 1, 1, dp, dpb, dg));
  FVB_TRY(op_rhie_chow(c, du, dub, dp, dpb, da, dg, dd, ddb, df));
  FVB_TRY(d2h(c, flux_out, df, size_t(c->nf)));
  return sync(c);
}

int fvb_plain_flux(fvb_ctx* h) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  FVB_TRY(need_bc(c, 0));
  FVB_TRY(op_face_flux(c, 3, c->u, c->ub, 0, c->flux));
  return sync(c);
}

int fvb_continuity_error(fvb_ctx* h, double* out) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_TRY(need_mesh(c));
  double* div = c->slot(S_SCR);
  FVB_TRY(op_divergence(c, c->flux, div));
  const int blocks = 2 * c->num_sms;
  { k_absmax<<<blocks, kThreads, 0, c->stream>>>(c->nr, div, c->partials); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  std::vector<double> hm(blocks);
  FVB_TRY(d2h(c, hm.data(), c->partials, size_t(blocks)));
  FVB_TRY(sync(c));
  double m = 0.0;
  for (double v : hm) m = std::max(m, v);
  FVB_TRY(team_allreduce(c, &m, 1, RED_MAX));
  *out = m;
  return FVB_OK;
}

// ------------------------------------------------------------------ team
int fvb_team_export(fvb_ctx* h, void** pool_base, int64_t* n_cells, uint8_t* ipc_handle) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  if (!c->pool) {
    fvb_set_error("team export needs an uploaded mesh");
    return FVB_E_ARG;
  }
  if (pool_base) *pool_base = c->pool;
  if (n_cells) *n_cells = c->nc;
  if (ipc_handle) {
    cudaIpcMemHandle_t hd;
    FVB_CUDA(cudaIpcGetMemHandle(&hd, c->pool));
    memcpy(ipc_handle, &hd, sizeof hd);
  }
  return FVB_OK;
}

int fvb_ipc_open(const uint8_t* ipc_handle, void** base) {
  cudaIpcMemHandle_t hd;
  memcpy(&hd, ipc_handle, sizeof hd);
  FVB_CUDA(cudaIpcOpenMemHandle(base, hd, cudaIpcMemLazyEnablePeerAccess));
  return FVB_OK;
}

int fvb_ipc_close(void* base) {
  FVB_CUDA(cudaIpcCloseMemHandle(base));
  return FVB_OK;
}

int fvb_team_attach(fvb_ctx* h, int rank, int size, void* const* pool_bases,
                    const int64_t* n_cells, int64_t n_inner, const int64_t* send_ptr,
                    const int64_t* send_rank, const int64_t* send_dst) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  if (!c->pool || !c->have_mesh) {
    fvb_set_error("team attach needs an uploaded mesh");
    return FVB_E_ARG;
  }
  if (size < 1 || size > kMaxTeam || rank < 0 || rank >= size) {
    fvb_set_error("team rank %d of size %d outside 1..%d", rank, size, kMaxTeam);
    return FVB_E_ARG;
  }
  if (n_inner < 0 || n_inner > c->nr) {
    fvb_set_error("n_inner %lld outside 0..%d", (long long)n_inner, c->nr);
    return FVB_E_ARG;
  }
  if (pool_bases[rank] != c->pool) {
    fvb_set_error("pool_bases[rank] is not this context's pool");
    return FVB_E_ARG;
  }
  // peers on other devices (an in-process team over several GPUs, or IPC
  // mappings): kernels store halos and mailbox words straight into their
  // pools, so this device needs peer access to each of them
  for (int q = 0; q < size; ++q) {
    if (q == rank) continue;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, pool_bases[q]) != cudaSuccess) {
      cudaGetLastError();
      fvb_set_error("team rank %d: pool_bases[%d] is not a device pointer", rank, q);
      return FVB_E_ARG;
    }
    if (at.type != cudaMemoryTypeDevice || at.device == c->dev) continue;
    int ok = 0;
    FVB_CUDA(cudaDeviceCanAccessPeer(&ok, c->dev, at.device));
    if (!ok) {
      fvb_set_error("team rank %d: device %d cannot access peer device %d (rank %d)", rank,
                    c->dev, at.device, q);
      return FVB_E_ARG;
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
      cudaGetLastError();
    else
      FVB_CUDA(e);
  }
  TeamView& T = c->team;
  T.rank = rank;
  T.size = size;
  T.comm = reinterpret_cast<Comm*>(c->pool);
  for (int q = 0; q < kMaxTeam; ++q) {
    T.peer_comm[q] = nullptr;
    T.peer_cells[q] = nullptr;
    T.peer_nc[q] = 0;
  }
  for (int q = 0; q < size; ++q) {
    char* b = static_cast<char*>(pool_bases[q]);
    T.peer_comm[q] = reinterpret_cast<Comm*>(b);
    T.peer_cells[q] = reinterpret_cast<double*>(b + kCommBytes);
    T.peer_nc[q] = int(n_cells[q]);
  }
  T.n_inner = int(n_inner);
  T.sys = 1;  // until fvb_team_set_scope says all ranks share this device
  const int nsr = c->nr - int(n_inner);
  const int64_t ns = nsr > 0 ? send_ptr[nsr] : 0;
  std::vector<int> sp(size_t(nsr) + 1), sr(static_cast<size_t>(ns)), sd(static_cast<size_t>(ns));
  for (int t = 0; t <= nsr; ++t) sp[t] = int(send_ptr[t]);
  for (int64_t e = 0; e < ns; ++e) {
    if (send_rank[e] < 0 || send_rank[e] >= size || send_rank[e] == rank ||
        send_dst[e] < 0 || send_dst[e] >= n_cells[send_rank[e]]) {
      fvb_set_error("halo send %lld targets rank %lld cell %lld", (long long)e,
                    (long long)send_rank[e], (long long)send_dst[e]);
      return FVB_E_ARG;
    }
    sr[e] = int(send_rank[e]);
    sd[e] = int(send_dst[e]);
  }
  auto up = [&](const std::vector<int>& v, int** o) -> int {
    FVB_TRY(dalloc(c, o, v.size()));
    if (!v.empty()) FVB_CUDA(cudaMemcpy(*o, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    return FVB_OK;
  };
  FVB_TRY(up(sp, &c->send_ptr));
  FVB_TRY(up(sr, &c->send_rank));
  FVB_TRY(up(sd, &c->send_dst));
  T.send_ptr = c->send_ptr;
  T.send_rank = c->send_rank;
  T.send_dst = c->send_dst;
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  // No team sync here: allocations and copies above must not overlap a
  // peer's spinning sync kernel.  fvb_team_check (called by every rank
  // after all ranks attached) makes the mesh checks team-consistent.
  return FVB_OK;
}

int fvb_team_check(fvb_ctx* h) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  // mesh checks that raise inside a step must raise on every rank
  double flags[3] = {double(c->first_zero_dmag >= 0), double(c->first_zero_dbmag_value[0] >= 0),
                     double(c->first_zero_dbmag_value[1] >= 0)};
  FVB_TRY(team_allreduce(c, flags, 3, RED_MAX));
  if (flags[0] > 0 && c->first_zero_dmag < 0) c->first_zero_dmag = 0x7ffffffe;
  for (int f = 0; f < 2; ++f)
    if (flags[1 + f] > 0 && c->first_zero_dbmag_value[f] < 0) c->first_zero_dbmag_value[f] = 0x7ffffffe;
  return FVB_OK;
}

int fvb_team_set_scope(fvb_ctx* h, int system_scope) {
  h->c.team.sys = system_scope ? 1 : 0;
  return FVB_OK;
}

int fvb_team_allreduce(fvb_ctx* h, double* vals, int m, int op) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  return team_allreduce(c, vals, m, op);
}

int fvb_set_sm_share(fvb_ctx* h, int share) {
  if (share < 1) {
    fvb_set_error("sm share must be >= 1");
    return FVB_E_ARG;
  }
  h->c.sm_share = share;
  return FVB_OK;
}

int fvb_piso_step(fvb_ctx* h, const fvb_step_cfg* cfg, const double* u_speeds,
                  fvb_step_report* rep) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  return run_step(c, cfg, u_speeds, rep, true);
}

int fvb_simple_sweep(fvb_ctx* h, const fvb_step_cfg* cfg, const double* u_speeds,
                     fvb_step_report* rep) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  return run_step(c, cfg, u_speeds, rep, false);
}

int fvb_set_solver_options(fvb_ctx* h, int flags) {
  if (flags & ~(FVB_SOLVER_EXPLICIT_INDEX | FVB_SOLVER_NO_RCM | FVB_SOLVER_NO_CLUSTER |
                FVB_STEP_NO_GRAPHS)) {
    fvb_set_error("unknown solver option bits 0x%x", flags);
    return FVB_E_ARG;
  }
  h->c.solver_flags = flags;
  return FVB_OK;
}

int fvb_set_solver_grid(fvb_ctx* h, int max_blocks) {
  if (max_blocks < 0) {
    fvb_set_error("max_blocks %d < 0", max_blocks);
    return FVB_E_ARG;
  }
  h->c.solver_max_blocks = max_blocks;
  return FVB_OK;
}

int fvb_pattern_codes(fvb_ctx* h, int* n_codes, int64_t* n_escape, int* cg_defer_x,
                      int64_t* rcm_solves) {
  Ctx* c = &h->c;
  const bool sc = uses_codes(c);
  if (n_codes) *n_codes = sc ? c->n_scode : 0;
  if (n_escape) *n_escape = sc ? c->n_sescape : 0;
  if (cg_defer_x) *cg_defer_x = cg_defers_x(c) ? 1 : 0;
  if (rcm_solves) *rcm_solves = c->cg_rcm_solves + c->bi_rcm_solves;
  return FVB_OK;
}

unsigned long long fvb_launch_count(void) { return g_launches.load(); }

int fvb_host_register(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return FVB_OK;
  FVB_CUDA(cudaHostRegister(ptr, size_t(bytes), cudaHostRegisterDefault));
  return FVB_OK;
}

int fvb_host_unregister(void* ptr) {
  if (!ptr) return FVB_OK;
  FVB_CUDA(cudaHostUnregister(ptr));
  return FVB_OK;
}

int fvb_timer_start(fvb_ctx* h) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_CUDA(cudaEventRecord(c->tev[0], c->stream));
  return FVB_OK;
}

int fvb_timer_stop(fvb_ctx* h, double* ms) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  FVB_CUDA(cudaEventRecord(c->tev[1], c->stream));
  FVB_CUDA(cudaEventSynchronize(c->tev[1]));
  float f = 0.f;
  FVB_CUDA(cudaEventElapsedTime(&f, c->tev[0], c->tev[1]));
  *ms = f;
  return FVB_OK;
}

int fvb_sync(fvb_ctx* h) {
  Ctx* c = &h->c;
  cudaSetDevice(c->dev);
  return sync(c);
}

}  // extern "C"
