// Jacobi-preconditioned CG and BiCGStab as persistent, cooperatively
// launched kernels (linsolve.py:102-282 restated for sm_100a).
//
// One launch runs a whole solve: rows are strided over the co-resident
// grid, every global sync point is one team_reduce (grid barrier + peer
// mailbox exchange when the mesh is decomposed), and the dot products are
// deterministic (fixed per-thread order -> warp-shuffle tree -> fixed block
// order -> fixed rank order), so every block of every rank holds identical
// scalars and takes identical branches: the reference's stopping rules
// (check on entry, break right after the residual test, breakdown checks)
// run on the device with no host round trip per iteration.
//
// CG is fused into two passes per iteration: pass A
// rebuilds p = z + beta p on the fly for every gathered column while it
// forms q = A p and p.q; pass B updates x and r, stores z = r / D and forms
// ||r||^2 and r.z.  Rows on a processor boundary store their fresh p (pass
// A) and z (pass B) straight into the neighbour ranks' ghost slots; the
// reduction that closes the pass orders those stores.
#include "fvb_solvers_common.cuh"

namespace fvb {

namespace {

struct CgParams {
  PatternView P;
  TeamView T;
  const double* V;
  const double* crs;
  const double* inv;
  const double* b;
  double* x;
  double* r;
  double* z;
  double* pa;
  double* pb;
  double* q;
  int slot_z, slot_pa, slot_pb;  // pool slots (halo targets)
  double tol, abs_tol;
  int max_iters;
  unsigned* sync;
  double* partials;
  double* result;  // [iters, converged, res0, res, err_kind, err_iter]
  const int* zero_flag;  // single domain: k_inv_diag's first zero row (INT_MAX - row), or null
  const double* Vp;      // matrix values read by the SpMV passes (== V, or a shared copy)
  const uint8_t* codep;  // stencil codes read by the SpMV passes (== P.code, or a shared copy)
};


// Pass A with the column indices (the gather's address chain) prefetched
// DEPTH rows ahead; the values V of the current row are loaded in-iteration
// (they are off the critical path) with evict-first, so the gathered vectors
// keep L1/L2.  Same arithmetic and order as ell_row.
// load the index ring of the first DEPTH rows of a sweep
template <int KT, int DEPTH>
__device__ __forceinline__ void icols_ring_load(const PatternView& P, int (&cq)[DEPTH][KT], int i,
                                                int end, int step) {
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) {
    const int r = i + d * step;
    if (r < end) {
#pragma unroll
      for (int s = 0; s < KT; ++s) cq[d][s] = __ldcs(P.I + size_t(s) * P.n + r);
    }
  }
}

template <int KT, int DEPTH, bool TEAM>
__device__ __forceinline__ double cg_pass_a_icols(const CgParams& A, const double* __restrict__ z,
                                                  const double* __restrict__ po,
                                                  double* __restrict__ pnew, double beta,
                                                  bool first, int slot_new, int i, int end,
                                                  int step, int (&cq)[DEPTH][KT],
                                                  double* __restrict__ xd = nullptr,
                                                  double alpha_prev = 0.0) {
  const PatternView& P = A.P;
  const TeamView& T = A.T;
  const int n = P.n;
  const int* __restrict__ I = P.I;
  const double* __restrict__ V = A.V;
  const bool team = TEAM && T.size > 1;
  double acc = 0.0;
  icols_ring_load<KT, DEPTH>(P, cq, i, end, step);
  auto g = [&](int col) { return first ? z[col] : po[col] * beta + z[col]; };
  while (i < end) {
    double vi[KT];
#pragma unroll
    for (int s = 0; s < KT; ++s) vi[s] = __ldcs(V + size_t(s) * n + i);
    int ci[KT];
#pragma unroll
    for (int s = 0; s < KT; ++s) ci[s] = cq[0][s];
#pragma unroll
    for (int d = 0; d + 1 < DEPTH; ++d)
#pragma unroll
      for (int s = 0; s < KT; ++s) cq[d][s] = cq[d + 1][s];
    const int nx = i + DEPTH * step;
    if (nx < end) {
#pragma unroll
      for (int s = 0; s < KT; ++s) cq[DEPTH - 1][s] = __ldcs(I + size_t(s) * n + nx);
    }
    double pr[KT];
#pragma unroll
    for (int s = 0; s < KT; ++s) pr[s] = vi[s] * g(ci[s] < 0 ? 0 : ci[s]);
    double ev = pr[0];
#pragma unroll
    for (int s = 2; s < KT; s += 2) ev = ev + pr[s];
    double y = ev;
    if (KT > 1) {
      double od = pr[1];
#pragma unroll
      for (int s = 3; s < KT; s += 2) od = od + pr[s];
      y = ev + od;
    }
    const double qi = crs_tail(P, A.crs, i, y, g);
    const double pi = g(i);
    pnew[i] = pi;
    A.q[i] = qi;
    if (team && i >= T.n_inner) halo_send(T, i, slot_new, pi);
    acc += pi * qi;
    // deferred x += alpha p of the previous iteration (po is that p)
    if (xd && !first) xd[i] = __ldcs(xd + i) + alpha_prev * po[i];
    i += step;
  }
  return acc;
}

// Pass A over stencil-coded rows (PatternView::code): the ring carries
// each row's one-byte code DEPTH rows ahead and the column offsets come
// from the shared-memory copy of the code table; rows coded kEscapeCode
// load their explicit indices.  Columns, products and order as
// cg_pass_a_icols.
template <int KT, int DEPTH, bool TEAM, bool SMEM = false>
__device__ __forceinline__ double cg_pass_a_codes(const CgParams& A, const double* __restrict__ z,
                                                  const double* __restrict__ po,
                                                  double* __restrict__ pnew, double beta,
                                                  bool first, int slot_new, int i, int end,
                                                  int step, const int* __restrict__ s_tab,
                                                  double* __restrict__ xd, double alpha_prev) {
  const PatternView& P = A.P;
  const TeamView& T = A.T;
  const int n = P.n;
  const int* __restrict__ I = P.I;
  const uint8_t* __restrict__ code = A.codep;
  const double* __restrict__ V = A.Vp;
  const bool team = TEAM && T.size > 1;
  double acc = 0.0;
  int cq[DEPTH];
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) {
    const int r = i + d * step;
    cq[d] = r < end ? int(ldst<SMEM>(code + r)) : 0;
  }
#ifdef FVB_DIAG_GATHER_CG  // diagnostic build: gathers bypass L1
  auto g = [&](int col) { return first ? __ldcg(z + col) : __ldcg(po + col) * beta + __ldcg(z + col); };
#else
  auto g = [&](int col) { return first ? z[col] : po[col] * beta + z[col]; };
#endif
  while (i < end) {
    double vi[KT];
#pragma unroll
    for (int s = 0; s < KT; ++s) vi[s] = ldst<SMEM>(V + size_t(s) * n + i);
    const int cd = cq[0];
#pragma unroll
    for (int d = 0; d + 1 < DEPTH; ++d) cq[d] = cq[d + 1];
    const int nx = i + DEPTH * step;
    if (nx < end) cq[DEPTH - 1] = int(ldst<SMEM>(code + nx));
    int ci[KT];
    if (cd != kEscapeCode) {
      const int* so = s_tab + cd * KT;
#pragma unroll
      for (int s = 0; s < KT; ++s) {
        const int o = so[s];
        ci[s] = o == kPadOffset ? 0 : i + o;
      }
    } else {
#pragma unroll
      for (int s = 0; s < KT; ++s) {
        const int c = __ldcs(I + size_t(s) * n + i);
        ci[s] = c < 0 ? 0 : c;
      }
    }
    double pr[KT];
    if constexpr (!TEAM) {
      // issue every gather of the row before the first use (memory-level
      // parallelism: the compiler otherwise interleaves load-use pairs);
      // the team kernel has no registers to spare for it
      double zg[KT], pg[KT];
#pragma unroll
      for (int s = 0; s < KT; ++s) zg[s] = z[ci[s]];
      if (!first) {
#pragma unroll
        for (int s = 0; s < KT; ++s) pg[s] = po[ci[s]];
      }
#pragma unroll
      for (int s = 0; s < KT; ++s) pr[s] = vi[s] * (first ? zg[s] : pg[s] * beta + zg[s]);
    } else {
#pragma unroll
      for (int s = 0; s < KT; ++s) pr[s] = vi[s] * g(ci[s]);
    }
    double ev = pr[0];
#pragma unroll
    for (int s = 2; s < KT; s += 2) ev = ev + pr[s];
    double y = ev;
    if (KT > 1) {
      double od = pr[1];
#pragma unroll
      for (int s = 3; s < KT; s += 2) od = od + pr[s];
      y = ev + od;
    }
    const double qi = crs_tail(P, A.crs, i, y, g);
    const double pi = g(i);
    pnew[i] = pi;
    A.q[i] = qi;
    if (team && i >= T.n_inner) halo_send(T, i, slot_new, pi);
    acc += pi * qi;
    // deferred x += alpha p of the previous iteration (po is that p)
    if (xd && !first) xd[i] = __ldcs(xd + i) + alpha_prev * po[i];
    i += step;
  }
  return acc;
}

// KT > 0: fixed K, pass A with the index ring (cg_pass_a_icols) or, SC,
// the stencil-code ring (cg_pass_a_codes), pass B on row pairs with 16-byte
// L2-only loads; KT = 0: generic K, plain row loops.  Rows are grid-strided
// over every thread (team_rows).
template <int KT, int THREADS, int MINB, int SC = 0, int DF = 0, bool TEAM = false,
          bool CLUSTER = false, bool SMEM = false, bool SYS = false>
__device__ __forceinline__ void cg_body(const CgParams& A) {
  __shared__ double red[32 * 3 + 3];
  // SC: stencil-coded pass A (PatternView::code) with the code table here
  __shared__ int s_tab[SC ? kMaxCodes * (KT > 0 ? KT : 1) : 1];
  if (SC) {
    for (int j = threadIdx.x; j < A.P.ncode * KT; j += blockDim.x) s_tab[j] = A.P.stab[j];
    __syncthreads();
  }
  if (zero_diag_exit(A.zero_flag, A.result, 1)) return;
  constexpr bool PB2 = KT > 0 && !SMEM;  // 16-byte global loads: not on shared memory
  const PatternView& P = A.P;
  const TeamView& T = A.T;
  const int nrows = P.n;
  unsigned rnd = 0;  // reduction round of this launch (team_reduce)
  const RowRange R = team_rows(T, nrows);
  const int row0 = R.begin, n = R.end, G = R.step;
  const bool sends = TEAM && R.sends;
  const int tid = row0;
  const bool team = TEAM && T.size > 1;
  const double* __restrict__ inv = A.inv;
  const bool vec_ok = PB2 && ((reinterpret_cast<uintptr_t>(A.pb) | reinterpret_cast<uintptr_t>(A.pa) |
                               reinterpret_cast<uintptr_t>(A.x) | reinterpret_cast<uintptr_t>(A.r) |
                               reinterpret_cast<uintptr_t>(A.q) | reinterpret_cast<uintptr_t>(A.z) |
                               reinterpret_cast<uintptr_t>(inv)) & 15u) == 0;

  // setup: r = b - A x0, z = r / D, ||b||, ||r||, r.z  (linsolve.py:106-127)
  double s3[3] = {0.0, 0.0, 0.0};
  {
    const double* x = A.x;
    for (int i = tid; i < n; i += G) {
      auto g = [&](int col) { return x[col]; };
      const double ax = crs_tail(P, A.crs, i, ell_row<KT>(A.V, P.I, nrows, P.k, i, g), g);
      const double bi = A.b[i];
      const double ri = bi - ax;
      const double zi = ri * inv[i];
      A.r[i] = ri;
      A.z[i] = zi;
      if (team && i >= T.n_inner) halo_send(T, i, A.slot_z, zi);
      s3[0] += bi * bi;
      s3[1] += ri * ri;
      s3[2] += ri * zi;
    }
  }
  if (!team_reduce<3, true, TEAM, CLUSTER, SYS>(T, A.sync, A.partials, s3, red, rnd, sends)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) A.result[4] = SE_TIMEOUT;
    return;
  }
  const double bnorm = fmax(sqrt(s3[0]), kResFloor);
  double res = sqrt(s3[1]) / bnorm;
  const double res0 = res;
  double rz = s3[2];
  int it = 0;
  bool conv = res <= A.tol || res * bnorm <= A.abs_tol;
  int err = SE_NONE;
  double beta = 0.0;
  double* pold = A.pa;
  double* pnew = A.pb;
  int slot_new = A.slot_pb;
  bool first = true;
  uint64_t t_spmv = 0, t_axpy = 0, t_red = 0, tk = 0;
  const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
  constexpr int KR = KT > 0 ? KT : 1;
  constexpr int DR = 2;  // rows of column indices in flight ahead of use
  // DEFER (DF): x += alpha p of iteration k runs in pass A of iteration
  // k + 1 (which holds that p as its old p), or in a final sweep — pass B
  // then streams r, q, 1/D and z only; same expression x + alpha p per row
  constexpr bool DEFER = DF && KT > 0;
  double alpha_prev = 0.0;
  const double* p_pend = nullptr;  // p whose x update is still pending
  int ring[DR][KR];
  while (!conv && it < A.max_iters) {
    ++it;
    if (timer) tk = global_ns();
    // pass A: p <- z + beta p (gathered columns), q = A p, p.q
    double pq[1] = {0.0};
    {
      const double* __restrict__ z = A.z;
      const double* __restrict__ po = pold;
      if (SC && KT > 0) {
        pq[0] = cg_pass_a_codes<KR, DR, TEAM, SMEM>(A, z, po, pnew, beta, first, slot_new, tid, n, G, s_tab,
                                        DEFER ? A.x : nullptr, alpha_prev);
      } else if (KT > 0) {
        pq[0] = cg_pass_a_icols<KR, DR, TEAM>(A, z, po, pnew, beta, first, slot_new, tid, n, G, ring,
                                        DEFER ? A.x : nullptr, alpha_prev);
      } else {
        for (int i = tid; i < n; i += G) {
          auto g = [&](int col) { return first ? z[col] : po[col] * beta + z[col]; };
          const double qi = crs_tail(P, A.crs, i, ell_row<KT>(A.V, P.I, nrows, P.k, i, g), g);
          const double pi = g(i);
          pnew[i] = pi;
          A.q[i] = qi;
          if (team && i >= T.n_inner) halo_send(T, i, slot_new, pi);
          pq[0] += pi * qi;
        }
      }
    }
    if (DEFER) p_pend = nullptr;  // pass A applied the previous update
    if (timer) { const uint64_t t = global_ns(); t_spmv += t - tk; tk = t; }
    if (!team_reduce<1, true, TEAM, CLUSTER, SYS>(T, A.sync, A.partials, pq, red, rnd, sends)) { err = SE_TIMEOUT; break; }
    if (timer) { const uint64_t t = global_ns(); t_red += t - tk; tk = t; }
    if (pq[0] <= 0.0 || !isfinite(pq[0])) { err = SE_CG_NOT_SPD; break; }
    const double alpha = rz / pq[0];
    // pass B: x += alpha p (DEFER: in the next pass A, or the final sweep),
    // r -= alpha q, z = r / D, ||r||^2, r.z
    double s2[2] = {0.0, 0.0};
    int i_scalar = tid;
    if (PB2 && vec_ok) {
      // two consecutive rows per thread with 16-byte loads/stores
      const int npair = n >> 1;
      for (int j = tid; j < npair; j += G) {
        const int i = 2 * j;
        if (!DEFER) {
          const double2 pv = __ldcg(reinterpret_cast<const double2*>(pnew + i));
          const double2 xv = __ldcg(reinterpret_cast<const double2*>(A.x + i));
          double2 xo;
          xo.x = xv.x + alpha * pv.x;
          xo.y = xv.y + alpha * pv.y;
          *reinterpret_cast<double2*>(A.x + i) = xo;
        }
        const double2 rv = __ldcg(reinterpret_cast<const double2*>(A.r + i));
        const double2 qv = __ldcg(reinterpret_cast<const double2*>(A.q + i));
        const double2 iv = __ldcg(reinterpret_cast<const double2*>(inv + i));
        double2 ro, zo;
        ro.x = rv.x - alpha * qv.x;
        ro.y = rv.y - alpha * qv.y;
        zo.x = ro.x * iv.x;
        zo.y = ro.y * iv.y;
        *reinterpret_cast<double2*>(A.r + i) = ro;
        *reinterpret_cast<double2*>(A.z + i) = zo;
        if (team && i + 1 >= T.n_inner) {
          if (i >= T.n_inner) halo_send(T, i, A.slot_z, zo.x);
          halo_send(T, i + 1, A.slot_z, zo.y);
        }
        s2[0] += ro.x * ro.x;
        s2[1] += ro.x * zo.x;
        s2[0] += ro.y * ro.y;
        s2[1] += ro.y * zo.y;
      }
      i_scalar = 2 * npair + tid;  // odd tail row
    }
    for (int i = i_scalar; i < n; i += G) {
      if (!DEFER) A.x[i] = A.x[i] + alpha * pnew[i];
      const double ri = A.r[i] - alpha * A.q[i];
      const double zi = ri * inv[i];
      A.r[i] = ri;
      A.z[i] = zi;
      if (team && i >= T.n_inner) halo_send(T, i, A.slot_z, zi);
      s2[0] += ri * ri;
      s2[1] += ri * zi;
    }
    if (timer) { const uint64_t t = global_ns(); t_axpy += t - tk; tk = t; }
    if (DEFER) {
      p_pend = pnew;
      alpha_prev = alpha;
    }
    if (!team_reduce<2, true, TEAM, CLUSTER, SYS>(T, A.sync, A.partials, s2, red, rnd, sends)) { err = SE_TIMEOUT; break; }
    if (timer) t_red += global_ns() - tk;
    res = sqrt(s2[0]) / bnorm;
    if (!isfinite(res)) { err = SE_DIVERGED; break; }
    if (res <= A.tol || res * bnorm <= A.abs_tol) { conv = true; break; }
    beta = s2[1] / rz;
    rz = s2[1];
    double* t = pold; pold = pnew; pnew = t;
    slot_new = (slot_new == A.slot_pb) ? A.slot_pa : A.slot_pb;
    first = false;
  }
  if (DEFER && p_pend && err != SE_TIMEOUT) {
    // the last iteration's x += alpha p (own rows only: no barrier needed)
    for (int i = tid; i < n; i += G) A.x[i] = A.x[i] + alpha_prev * p_pend[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.result[0] = it;
    A.result[1] = conv ? 1.0 : 0.0;
    A.result[2] = res0;
    A.result[3] = res;
    A.result[4] = err;
    A.result[5] = err ? it : 0;
    A.result[6] = 1e-9 * double(t_spmv);
    A.result[7] = 1e-9 * double(t_axpy);
    A.result[8] = 1e-9 * double(t_red);
  }
}

// Persistent CG kernel.  SMEM (single-block systems, one block): the work
// vectors r, z, the two p buffers, q and 1/D live in dynamic shared memory
// for the whole solve, so the gathers of pass A are shared-memory loads
// (x, b and the matrix stay in global memory: own-row or streamed accesses).
template <int KT, int THREADS, int MINB, int SC = 0, int DF = 0, bool TEAM = false,
          bool CLUSTER = false, bool SMEM = false, bool SYS = false>
__global__ void __launch_bounds__(THREADS, MINB) k_cg(CgParams A) {
  if constexpr (SMEM) {
    extern __shared__ double dyn[];
    const int n = A.P.n;
    CgParams B = A;
    B.r = dyn;
    B.z = dyn + n;
    B.pa = dyn + 2 * n;
    B.pb = dyn + 3 * n;
    B.q = dyn + 4 * n;
    double* inv = dyn + 5 * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) inv[i] = A.inv[i];
    B.inv = inv;
    if constexpr (SC != 0 && KT > 0) {
      // the matrix and its stencil codes too (read every pass)
      double* vs = dyn + 6 * n;
      for (int e = threadIdx.x; e < KT * n; e += blockDim.x) vs[e] = A.V[e];
      uint8_t* cs = reinterpret_cast<uint8_t*>(vs + KT * n);
      for (int i = threadIdx.x; i < n; i += blockDim.x) cs[i] = A.P.code[i];
      B.Vp = vs;
      B.codep = cs;
    }
    __syncthreads();
    cg_body<KT, THREADS, MINB, SC, DF, TEAM, CLUSTER, true>(B);
  } else {
    cg_body<KT, THREADS, MINB, SC, DF, TEAM, CLUSTER, false, SYS>(A);
  }
}

}  // namespace

std::string solve_error_text(const char* solver, const SolveOut& o, int zero_row) {
  char buf[256];
  switch (o.error_kind) {
    case SE_ZERO_DIAG:
      snprintf(buf, sizeof buf, "singular preconditioner: zero diagonal at row %d", zero_row);
      break;
    case SE_CG_NOT_SPD:
      snprintf(buf, sizeof buf, "cg: matrix not positive definite at iteration %d", o.error_iteration);
      break;
    case SE_DIVERGED:
      snprintf(buf, sizeof buf, "%s: residual diverged at iteration %d", solver, o.error_iteration);
      break;
    case SE_RHO:
      snprintf(buf, sizeof buf, "bicgstab: rho breakdown at iteration %d", o.error_iteration);
      break;
    case SE_RV:
      snprintf(buf, sizeof buf, "bicgstab: breakdown (r_hat . v = 0) at iteration %d",
               o.error_iteration);
      break;
    case SE_OMEGA:
      snprintf(buf, sizeof buf, "bicgstab: omega breakdown at iteration %d", o.error_iteration);
      break;
    case SE_TIMEOUT:
      snprintf(buf, sizeof buf, "%s: device watchdog fired (grid barrier timeout)", solver);
      break;
    default:
      snprintf(buf, sizeof buf, "%s: ok", solver);
  }
  return buf;
}


// Work vectors are pool slots S_SCR.. (so the ghost entries can be written
// by the neighbour ranks).
// RCM-ordered CG (Ctx::rcm_*): gather the system into the permuted order
// (matrix slots, b, x0, 1/D), and scatter x back after the solve.
template <int KT>
__global__ void k_rcm_gather(int n, const int* __restrict__ perm, const double* __restrict__ V,
                             const double* __restrict__ b, const double* __restrict__ x,
                             const double* __restrict__ inv, double* __restrict__ Vp,
                             double* __restrict__ bp, double* __restrict__ xp,
                             double* __restrict__ invp) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int o = perm[r];
#pragma unroll
    for (int s = 0; s < KT; ++s) Vp[size_t(s) * n + r] = V[size_t(s) * n + o];
    bp[r] = b[o];
    xp[r] = x[o];
    invp[r] = inv[o];
  }
}
__global__ void k_rcm_scatter(int n, const int* __restrict__ perm, const double* __restrict__ xp,
                              double* __restrict__ x) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    x[perm[r]] = xp[r];
}


// k_cg instantiation for the context: K (5, 7 or generic), stencil codes,
// deferred x update on 7-point rows, team or single domain
template <bool TEAM, bool SYS = false>
static int cg_launch(Ctx* c, CgParams& prm, bool sc) {
  if (!TEAM && (c->k == 7 || c->k == 5) && c->nr <= kSingleBlockRowsPerThread * 1024 &&
      smem_cg_bytes(c->nr, c->k) <= kSmemSolverMax && !(c->solver_flags & FVB_SOLVER_NO_CLUSTER)) {
    const size_t bytes = smem_cg_bytes(c->nr, c->k);
    if (c->k == 7)
      return sc ? smem_launch(c, k_cg<7, 1024, 1, 1, 1, false, false, true>, prm, 1024, bytes)
                : smem_launch(c, k_cg<7, 1024, 1, 0, 1, false, false, true>, prm, 1024, bytes);
    return sc ? smem_launch(c, k_cg<5, 1024, 1, 1, 0, false, false, true>, prm, 1024, bytes)
              : smem_launch(c, k_cg<5, 1024, 1, 0, 0, false, false, true>, prm, 1024, bytes);
  }
  // one-cluster CG: 512 threads per CTA (about 2 rows per thread on the
  // cluster's range): cheaper block barriers in the two reductions per
  // iteration than with 1024 — 5.5 vs 6.6 us per iteration at 13.8k rows,
  // 7.7 vs 8.2 at 32.8k, 8.9 vs 10.6 at 39.3k; 256 is slower again
  // (profiles/r02_small.md)
#ifndef FVB_DIAG_CLUSTER_THREADS  // diagnostic builds: threads per cluster CTA
#define FVB_DIAG_CLUSTER_THREADS 512
#endif
  constexpr int CLT = FVB_DIAG_CLUSTER_THREADS;
  if (!TEAM && (c->k == 7 || c->k == 5)) {
    const int want = cluster_want(c, CLT);
    const int nb = want ? (c->k == 7 ? cluster_blocks(c, k_cg<7, CLT, 1, 1, 1, false, true>, CLT, want)
                                     : cluster_blocks(c, k_cg<5, CLT, 1, 1, 0, false, true>, CLT, want))
                        : 0;
    if (nb >= 2) {
      if (c->k == 7)
        return sc ? cluster_launch(c, k_cg<7, CLT, 1, 1, 1, false, true>, prm, CLT, nb)
                  : cluster_launch(c, k_cg<7, CLT, 1, 0, 1, false, true>, prm, CLT, nb);
      return sc ? cluster_launch(c, k_cg<5, CLT, 1, 1, 0, false, true>, prm, CLT, nb)
                : cluster_launch(c, k_cg<5, CLT, 1, 0, 0, false, true>, prm, CLT, nb);
    }
  }
#ifdef FVB_DIAG_GRID_THREADS  // diagnostic builds: threads per block of the single-domain grid
  if (!TEAM && (c->k == 5 || c->k == 7)) {
    constexpr int GT = FVB_DIAG_GRID_THREADS;
    if (c->k == 5)
      return sc ? coop_launch(c, k_cg<5, GT, 1, 1, 0>, prm, GT, 1)
                : coop_launch(c, k_cg<5, GT, 1, 0, 0>, prm, GT, 1);
    return sc ? coop_launch(c, k_cg<7, GT, 1, 1, 1>, prm, GT, 1)
              : coop_launch(c, k_cg<7, GT, 1, 0, 1>, prm, GT, 1);
  }
#endif
  switch (c->k) {
    case 5:
      if (sc) return coop_launch(c, k_cg<5, 1024, 1, 1, 0, TEAM, false, false, SYS>, prm, 1024, 1);
      return coop_launch(c, k_cg<5, 1024, 1, 0, 0, TEAM, false, false, SYS>, prm, 1024, 1);
    case 7:  // x update folded into pass A (cg_defers_x)
      if (sc) return coop_launch(c, k_cg<7, 1024, 1, 1, 1, TEAM, false, false, SYS>, prm, 1024, 1);
      return coop_launch(c, k_cg<7, 1024, 1, 0, 1, TEAM, false, false, SYS>, prm, 1024, 1);
    default: return coop_launch(c, k_cg<0, 512, 2, 0, 0, TEAM, false, false, SYS>, prm);
  }
}

bool uses_codes(const Ctx* c) {
  return c->scode != nullptr && !(c->solver_flags & FVB_SOLVER_EXPLICIT_INDEX);
}
bool uses_rcm(const Ctx* c) {
  return c->rcm_perm && !c->teamed() && c->k == 7 && !(c->solver_flags & FVB_SOLVER_NO_RCM);
}

// x += alpha p folded into the next pass A on 7-point rows: 426.6 -> 398.4
// us per iteration at 16.8M rows, even at 2.1M (57.3 vs 56.9 us, one call;
// profiles/r01_cg_variants.md)
bool cg_defers_x(const Ctx* c) { return c->k == 7; }

int cg_solve(Ctx* c, MatView A, const double* b, double* x, double tol, double abs_tol,
             int max_iters, SolveOut* out, const Readback* extra) {
  double* inv = c->slot(S_SCR + 0);
  double* r = c->slot(S_SCR + 1);
  double* z = c->slot(S_SCR + 2);
  double* pa = c->slot(S_SCR + 3);
  double* pb = c->slot(S_SCR + 4);
  double* q = c->slot(S_SCR + 5);
  double* result = c->partials + 16 * 4096;
  int zero_row = 0x7fffffff;
  FVB_TRY(prepare_diag(c, A, inv, &zero_row));
  *out = SolveOut{0, 0, SE_NONE, 0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (zero_row != 0x7fffffff) {
    out->error_kind = SE_ZERO_DIAG;
    out->error_iteration = zero_row;
    return FVB_OK;
  }
  CgParams prm{c->pattern(), c->team, A.V, A.crs, inv, b, x, r, z, pa, pb, q,
               S_SCR + 2, S_SCR + 3, S_SCR + 4, tol, abs_tol, max_iters,
               c->sync, c->partials, result, c->teamed() ? nullptr : c->ipart, A.V, c->scode};
  // RCM order (patterns without stencil codes, one domain, 7-point rows):
  // the solve runs on a permuted copy of the system
  const bool rcm = uses_rcm(c);
  double* xp = c->slot(S_SCR + 6);
  if (rcm) {
    if (!c->rcm_V) FVB_TRY(dalloc(c, &c->rcm_V, size_t(c->k) * size_t(c->nr)));
    double* bp = c->slot(S_SCR + 7);
    double* invp = c->slot(S_SCR + 8);
    k_rcm_gather<7><<<grid_for(c->nr, 256), 256, 0, c->stream>>>(c->nr, c->rcm_perm, A.V, b, x, inv,
                                                                c->rcm_V, bp, xp, invp);
    note_launch();
    FVB_CUDA(cudaGetLastError());
    prm.P.I = c->rcm_I;
    prm.P.diag_slot = c->rcm_ds;
    prm.P.slot_face = nullptr;
    prm.V = prm.Vp = c->rcm_V;
    prm.b = bp;
    prm.x = xp;
    prm.inv = invp;
    c->cg_rcm_solves++;
  }
  FVB_CUDA(cudaEventRecord(c->kev[0], c->stream));
  // one 1024-thread block per SM; pass A on 1-byte stencil codes when the
  // pattern has them, else on the explicit index ring (tuning history:
  // profiles/r01_cg_variants.md)
  const bool sc = uses_codes(c);
  if (c->teamed() && c->team.sys)
    FVB_TRY((cg_launch<true, true>(c, prm, sc)));
  else if (c->teamed())
    FVB_TRY((cg_launch<true, false>(c, prm, sc)));
  else
    FVB_TRY(cg_launch<false>(c, prm, sc));
  if (rcm) {
    k_rcm_scatter<<<grid_for(c->nr, 256), 256, 0, c->stream>>>(c->nr, c->rcm_perm, xp, x);
    note_launch();
    FVB_CUDA(cudaGetLastError());
  }
  FVB_CUDA(cudaEventRecord(c->kev[1], c->stream));
  double h[9];
  unsigned team_err = 0;
  FVB_CUDA(cudaMemcpyAsync(h, result, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  if (extra && extra->n)
    FVB_CUDA(cudaMemcpyAsync(extra->host, extra->dev, sizeof(double) * extra->n,
                             cudaMemcpyDeviceToHost, c->stream));
  FVB_CUDA(cudaMemcpyAsync(&team_err, c->sync + 3, sizeof team_err, cudaMemcpyDeviceToHost, c->stream));
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  if (team_err) h[4] = SE_TIMEOUT;
  out->iterations = int(h[0]);
  out->converged = int(h[1]);
  out->res0 = h[2];
  out->res = h[3];
  out->error_kind = int(h[4]);
  out->error_iteration = int(h[5]);
  out->t_smvp = h[6];
  out->t_daxpy = h[7];
  out->t_red = h[8];
  float kms = 0.f;
  FVB_CUDA(cudaEventElapsedTime(&kms, c->kev[0], c->kev[1]));
  out->kernel_ms = kms;
  return FVB_OK;
}


}  // namespace fvb
