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
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "fvb_internal.cuh"

namespace fvb {

namespace {

constexpr int kSolverThreads = 512;
constexpr double kResFloor = 1e-30;   // linsolve.py:20
constexpr double kTiny = 1e-300;      // linsolve.py:21

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

// A zero diagonal (found by the k_inv_diag launch before the solve) ends
// the solve before its first pass, with the reference's error and row; every
// block reads the same flag, so no block enters a barrier alone.
__device__ __forceinline__ bool zero_diag_exit(const int* flag, double* result, int ncomp) {
  if (!flag) return false;
  const int v = *flag;
  if (v == 0) return false;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int c = 0; c < ncomp; ++c)
      for (int k = 0; k < 6; ++k) result[6 * c + k] = 0.0;
    result[4] = SE_ZERO_DIAG;
    result[5] = double(0x7fffffff - v);
    for (int k = 6 * ncomp; k < 6 * ncomp + 3; ++k) result[k] = 0.0;
  }
  return true;
}

// Streamed (read-once) load: evict-first from global memory, or a plain
// load when the SMEM solver variants staged the array in shared memory.
template <bool SMEM, typename T>
__device__ __forceinline__ T ldst(const T* p) {
  if constexpr (SMEM) return *p;
  else return __ldcs(p);
}

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

// ------------------------------------------------------------ BiCGStab
// y_c = A x_c for NC vectors sharing one pass over V and I.
template <int KT, int NC, typename G>
__device__ __forceinline__ void ell_rows_multi(const PatternView& P, const double* __restrict__ V,
                                               const double* crs, int i, const bool* act,
                                               G gather, double* y) {
  const int n = P.n, K = KT > 0 ? KT : P.k;
  double ev[NC], od[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) ev[c] = od[c] = 0.0;
#pragma unroll
  for (int s = 0; s < (KT > 0 ? KT : K); s += 2) {
    int col = __ldg(P.I + size_t(s) * n + i);
    col = col < 0 ? 0 : col;
    const double v = __ldg(V + size_t(s) * n + i);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (act[c]) {
        const double pr = v * gather(c, col);
        ev[c] = s == 0 ? pr : ev[c] + pr;
      }
  }
#pragma unroll
  for (int s = 1; s < (KT > 0 ? KT : K); s += 2) {
    int col = __ldg(P.I + size_t(s) * n + i);
    col = col < 0 ? 0 : col;
    const double v = __ldg(V + size_t(s) * n + i);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (act[c]) {
        const double pr = v * gather(c, col);
        od[c] = s == 1 ? pr : od[c] + pr;
      }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    if (!act[c]) continue;
    double yy = K > 1 ? ev[c] + od[c] : ev[c];
    if (P.nnz_crs) {
      double tl = 0.0;
      for (int q = P.crs_ptr[i]; q < P.crs_ptr[i + 1]; ++q) tl += crs[q] * gather(c, P.crs_col[q]);
      yy = yy + tl;
    }
    y[c] = yy;
  }
}

// Row sweep computing y_c = (A x_c)_i for the active components with the
// column indices prefetched two rows ahead (the gather's address chain; see
// cg_pass_a_icols) and evict-first matrix loads; body(i, y) consumes a row.
// Same products and summation order as ell_rows_multi.
// SC: stencil-coded rows (PatternView::code, table in shared memory s_tab):
// the ring carries one code per row instead of KT indices.
template <int KT, int NC, bool SC = false, bool SMEM = false, typename Gt, typename Bt>
__device__ __forceinline__ void spmv_sweep(const PatternView& P, const double* __restrict__ V,
                                           const double* crs, int i, int end, int step,
                                           const bool* act, Gt gather, Bt body,
                                           const int* s_tab = nullptr,
                                           const uint8_t* __restrict__ code = nullptr) {
  const int n = P.n;
  constexpr int KC = SC ? 1 : KT;  // ring entries per row
  int c0[KC], c1[KC];
  auto ring_load = [&](int (&cq)[KC], int r) {
    if (SC) {
      cq[0] = int(ldst<SMEM>(code + r));
    } else {
#pragma unroll
      for (int s = 0; s < KC; ++s) cq[s] = __ldcs(P.I + size_t(s) * n + r);
    }
  };
  if (i < end) ring_load(c0, i);
  if (i + step < end) ring_load(c1, i + step);
  while (i < end) {
    double v[KT];
    int ci[KT];
#pragma unroll
    for (int s = 0; s < KT; ++s) v[s] = ldst<SMEM>(V + size_t(s) * n + i);
    if (SC) {
      const int cd = c0[0];
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
          const int c = __ldcs(P.I + size_t(s) * n + i);
          ci[s] = c < 0 ? 0 : c;
        }
      }
    } else {
#pragma unroll
      for (int s = 0; s < KT; ++s) ci[s] = c0[s] < 0 ? 0 : c0[s];
    }
#pragma unroll
    for (int s = 0; s < KC; ++s) c0[s] = c1[s];
    const int nx = i + 2 * step;
    if (nx < end) ring_load(c1, nx);
    double y[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (!act[c]) continue;
      double ev = v[0] * gather(c, ci[0]);
#pragma unroll
      for (int s = 2; s < KT; s += 2) ev = ev + v[s] * gather(c, ci[s]);
      double yy = ev;
      if (KT > 1) {
        double od = v[1] * gather(c, ci[1]);
#pragma unroll
        for (int s = 3; s < KT; s += 2) od = od + v[s] * gather(c, ci[s]);
        yy = ev + od;
      }
      if (P.nnz_crs) {
        double tl = 0.0;
        for (int q = P.crs_ptr[i]; q < P.crs_ptr[i + 1]; ++q) tl += crs[q] * gather(c, P.crs_col[q]);
        yy = yy + tl;
      }
      y[c] = yy;
    }
    body(i, y);
    i += step;
  }
}

struct CompState {
  int it, done, err, err_it, sconv, restart, copy, live;
  double bn, res0, res, rho, alpha, omega, beta, rr, rhr;
};

// ------------------------------------------------------ BiCGStab, 3 passes
// Jacobi-PBiCGStab (linsolve.py:175-282) with the reference's five vector
// passes fused into three: p_hat and s_hat are never
// stored — every SpMV rebuilds them for the gathered columns from r, p, v
// and 1/D with the reference's rounding (p_hat = p / D as linsolve.py
// computes it), and the update pass rebuilds them for the own row.  Three reductions per iteration: r_hat.v;
// ||s||^2, t.t, t.s (t is formed speculatively and dropped when s already
// converged); ||r||^2, r_hat.r.  p and v are double-buffered because pass 1
// gathers the previous ones while writing the new ones.  Decomposed runs
// send the new p and v (pass 1) and r (pass 3) of processor-boundary rows,
// and 1/D and r once at setup.
template <int NC>
struct Bi3Params {
  PatternView P;
  TeamView T;
  const double* V;
  const double* crs;
  double* inv;
  const double* b[NC];
  double* x[NC];
  double* r[NC];
  double* rh[NC];
  double* p[2][NC];
  double* v[2][NC];
  double* t[NC];
  int slot_inv, slot_r[NC], slot_p[2][NC], slot_v[2][NC];
  double tol, abs_tol;
  int max_iters;
  unsigned* sync;
  double* partials;
  double* result;
  const int* zero_flag;  // as CgParams::zero_flag
  const double* Vp;      // as CgParams::Vp / codep
  const uint8_t* codep;
};

// resident 512-thread blocks per SM of the BiCGStab kernel (64 registers)
#ifndef FVB_BI_MINB
#define FVB_BI_MINB 2
#endif

template <int KT, int NC, bool SC = false, bool TEAM = false, bool CLUSTER = false,
          bool SMEM = false, bool SYS = false>
__device__ __forceinline__ void bicgstab3_body(const Bi3Params<NC>& A) {
  __shared__ double red[32 * 3 * NC + 3 * NC];  // team_reduce<3 NC> in pass 2
  __shared__ CompState S[NC];
  // SC: stencil-coded SpMV sweeps (PatternView::code) with the code table here
  __shared__ int s_tab[SC ? kMaxCodes * (KT > 0 ? KT : 1) : 1];
  if (SC) {
    for (int j = threadIdx.x; j < A.P.ncode * KT; j += blockDim.x) s_tab[j] = A.P.stab[j];
    __syncthreads();
  }
  if (zero_diag_exit(A.zero_flag, A.result, NC)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) A.result[18] = A.result[19] = A.result[20] = 0.0;
    return;
  }
  const PatternView& P = A.P;
  const TeamView& T = A.T;
  const RowRange R = team_rows(T, P.n);
  const int n = R.end;       // rows of this block: tid, tid + G, ... < n
  const int G = R.step;
  const int tid = R.begin;
  const bool sends = TEAM && R.sends;
  unsigned rnd = 0;  // reduction round of this launch (team_reduce)
  const bool team = TEAM && T.size > 1;
  const double* __restrict__ inv = A.inv;
  bool act[NC];
  bool timeout = false;
  constexpr int KR = KT > 0 ? KT : 1;
  uintptr_t al_or = reinterpret_cast<uintptr_t>(inv);
#pragma unroll
  for (int c = 0; c < NC; ++c)
    al_or |= reinterpret_cast<uintptr_t>(A.x[c]) | reinterpret_cast<uintptr_t>(A.r[c]) |
             reinterpret_cast<uintptr_t>(A.rh[c]) | reinterpret_cast<uintptr_t>(A.t[c]) |
             reinterpret_cast<uintptr_t>(A.p[0][c]) | reinterpret_cast<uintptr_t>(A.p[1][c]) |
             reinterpret_cast<uintptr_t>(A.v[0][c]) | reinterpret_cast<uintptr_t>(A.v[1][c]);
  const bool vec_ok = !SMEM && (al_or & 15u) == 0;  // 16-byte global loads

  // setup (linsolve.py:180-196): r = b - A x0, r_hat = r, ||b||, ||r||
  double sums[2 * NC];
  {
#pragma unroll
    for (int m = 0; m < 2 * NC; ++m) sums[m] = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) act[c] = true;
    for (int i = tid; i < n; i += G) {
      double ax[NC];
      auto g = [&](int c, int col) { return A.x[c][col]; };
      ell_rows_multi<KT, NC>(P, A.V, A.crs, i, act, g, ax);
      const bool snd = team && i >= T.n_inner;
      if (snd) halo_send(T, i, A.slot_inv, inv[i]);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double bi = A.b[c][i];
        const double ri = bi - ax[c];
        A.r[c][i] = ri;
        A.rh[c][i] = ri;
        if (snd) halo_send(T, i, A.slot_r[c], ri);
        sums[2 * c] += bi * bi;
        sums[2 * c + 1] += ri * ri;
      }
    }
  }
  if (!team_reduce<2 * NC, false, TEAM, CLUSTER, SYS>(T, A.sync, A.partials, sums, red, rnd, sends)) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int c = 0; c < NC; ++c) A.result[6 * c + 4] = SE_TIMEOUT;
    return;
  }
  if (threadIdx.x == 0) {
    for (int c = 0; c < NC; ++c) {
      CompState& q = S[c];
      q.it = 0; q.err = SE_NONE; q.err_it = 0; q.sconv = 0; q.restart = 0; q.copy = 0; q.live = 0;
      q.bn = fmax(sqrt(sums[2 * c]), kResFloor);
      q.res = sqrt(sums[2 * c + 1]) / q.bn;
      q.res0 = q.res;
      q.rr = sums[2 * c + 1];
      q.rhr = q.rr;
      q.done = q.res <= A.tol || q.res * q.bn <= A.abs_tol;
      q.rho = q.alpha = q.omega = 1.0;
      q.beta = 0.0;
    }
  }
  __syncthreads();

  uint64_t t_spmv = 0, t_axpy = 0, t_red = 0, tk = 0;
  const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
  // p (own rows), v, and d = p - omega v stored by pass 3 for the next pass 1,
  // so pass 1 gathers r and d only (the reference's p = r + beta (p - omega v)
  // with the inner difference rounded once, as it is there)
  double* const* Pp = A.p[0];
  double* const* Pv = A.v[0];
  double* const* Pd = A.p[1];
  while (!timeout) {
    if (timer) tk = global_ns();
    if (threadIdx.x == 0) {
      for (int c = 0; c < NC; ++c) {
        CompState& q = S[c];
        q.sconv = 0;
        q.live = 0;
        if (q.done || q.err || q.it >= A.max_iters) continue;
        q.it++;
        double rho_new = q.it == 1 ? q.rr : q.rhr;
        q.restart = fabs(rho_new) < kTiny;
        if (q.restart) {
          rho_new = q.rr;  // r_hat := r, so r_hat.r = ||r||^2
          if (rho_new < kTiny) { q.err = SE_RHO; q.err_it = q.it; continue; }
        }
        q.copy = (q.it == 1 || q.restart);
        if (!q.copy) q.beta = (rho_new / q.rho) * (q.alpha / q.omega);
        q.rho = rho_new;
        q.live = 1;
      }
    }
    __syncthreads();
    bool any = false;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      act[c] = S[c].live != 0;
      any = any || act[c];
    }
    if (!any) break;
    // pass 1: p = r | r + beta (p - omega v); v = A (p / D) rebuilt per
    // gathered column; r_hat.v
    {
      double rv[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) rv[c] = 0.0;
      bool cp[NC];
      double be[NC], om[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        cp[c] = S[c].copy != 0;
        be[c] = S[c].beta;
        om[c] = S[c].omega;
      }
      auto pval = [&](int c, int col) {
        const double ri = A.r[c][col];
        if (cp[c]) return ri;
        return Pd[c][col] * be[c] + ri;
      };
      auto g = [&](int c, int col) { return pval(c, col) * inv[col]; };
      auto body = [&](int i, const double* y) {
        const bool snd = team && i >= T.n_inner;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (!act[c]) continue;
          const double pi = pval(c, i);
          Pp[c][i] = pi;
          Pv[c][i] = y[c];
          double rhi;
          if (S[c].restart) {
            rhi = A.r[c][i];
            A.rh[c][i] = rhi;
          } else {
            rhi = A.rh[c][i];
          }
          if (snd) {
            halo_send(T, i, A.slot_v[0][c], y[c]);
          }
          rv[c] += rhi * y[c];
        }
      };
      if (KT > 0) {
        spmv_sweep<KR, NC, SC, SMEM>(P, A.Vp, A.crs, tid, n, G, act, g, body, s_tab, A.codep);
      } else {
        for (int i = tid; i < n; i += G) {
          double y[NC];
          ell_rows_multi<KT, NC>(P, A.V, A.crs, i, act, g, y);
          body(i, y);
        }
      }
      if (timer) { const uint64_t t_ = global_ns(); t_spmv += t_ - tk; tk = t_; }
      if (!team_reduce<NC, false, TEAM, CLUSTER, SYS>(T, A.sync, A.partials, rv, red, rnd, sends)) { timeout = true; break; }
      if (timer) { const uint64_t t_ = global_ns(); t_red += t_ - tk; tk = t_; }
      if (threadIdx.x == 0)
        for (int c = 0; c < NC; ++c) {
          if (!act[c]) continue;
          if (fabs(rv[c]) < kTiny) { S[c].err = SE_RV; S[c].err_it = S[c].it; continue; }
          S[c].alpha = S[c].rho / rv[c];
        }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < NC; ++c) act[c] = act[c] && !S[c].err;
    }
    // pass 2: s = r - alpha v, t = A (s / D) rebuilt per gathered column;
    // ||s||^2, t.t, t.s
    {
      double st[3 * NC];
#pragma unroll
      for (int m = 0; m < 3 * NC; ++m) st[m] = 0.0;
      double al[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) al[c] = S[c].alpha;
      auto sval = [&](int c, int col) { return A.r[c][col] - al[c] * Pv[c][col]; };
      auto g = [&](int c, int col) { return sval(c, col) * inv[col]; };
      auto body = [&](int i, const double* y) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (!act[c]) continue;
          const double si = sval(c, i);
          A.t[c][i] = y[c];
          st[3 * c] += si * si;
          st[3 * c + 1] += y[c] * y[c];
          st[3 * c + 2] += y[c] * si;
        }
      };
      bool any_a = false;
#pragma unroll
      for (int c = 0; c < NC; ++c) any_a = any_a || act[c];
      if (KT > 0 && any_a) {
        spmv_sweep<KR, NC, SC, SMEM>(P, A.Vp, A.crs, tid, n, G, act, g, body, s_tab, A.codep);
      } else {
        for (int i = tid; i < n; i += G) {
          double y[NC];
          ell_rows_multi<KT, NC>(P, A.V, A.crs, i, act, g, y);
          body(i, y);
        }
      }
      if (timer) { const uint64_t t_ = global_ns(); t_spmv += t_ - tk; tk = t_; }
      if (!team_reduce<3 * NC, false, TEAM, CLUSTER, SYS>(T, A.sync, A.partials, st, red, rnd, sends)) { timeout = true; break; }
      if (timer) { const uint64_t t_ = global_ns(); t_red += t_ - tk; tk = t_; }
      if (threadIdx.x == 0)
        for (int c = 0; c < NC; ++c) {
          if (!act[c]) continue;
          const double sn = sqrt(st[3 * c]);
          if (sn / S[c].bn <= A.tol || sn <= A.abs_tol) {  // linsolve.py:234-245
            S[c].sconv = 1;
            S[c].res = sn / S[c].bn;
            continue;
          }
          const double tt = st[3 * c + 1], ts = st[3 * c + 2];
          if (tt == 0.0) { S[c].err = SE_OMEGA; S[c].err_it = S[c].it; continue; }
          S[c].omega = ts / tt;
          if (fabs(S[c].omega) < kTiny) { S[c].err = SE_OMEGA; S[c].err_it = S[c].it; }
        }
      __syncthreads();
    }
    // pass 3: x += alpha p_hat (+ omega s_hat); r = s - omega t; ||r||^2, r_hat.r
    {
      double rr[2 * NC];
#pragma unroll
      for (int m = 0; m < 2 * NC; ++m) rr[m] = 0.0;
      bool xa[NC], full[NC];
      double al[NC], om[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        // s-converged components take x += alpha p_hat only; erred ones nothing
        xa[c] = act[c] && (S[c].sconv || !S[c].err);
        full[c] = act[c] && !S[c].sconv && !S[c].err;
        al[c] = S[c].alpha;
        om[c] = S[c].omega;
      }
      int i_scalar = tid;
      if (vec_ok) {
        // row pairs, 16-byte L2-only loads and 16-byte stores (as CG pass B)
        const int npair = n >> 1;
        for (int j = tid; j < npair; j += G) {
          const int i = 2 * j;
          const double2 iv = __ldcg(reinterpret_cast<const double2*>(inv + i));
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            if (!xa[c]) continue;
            const double2 pv = __ldcg(reinterpret_cast<const double2*>(Pp[c] + i));
            const double2 xv = __ldcg(reinterpret_cast<const double2*>(A.x[c] + i));
            double2 xo;
            xo.x = xv.x + al[c] * (pv.x * iv.x);
            xo.y = xv.y + al[c] * (pv.y * iv.y);
            if (full[c]) {
              const double2 rv = __ldcg(reinterpret_cast<const double2*>(A.r[c] + i));
              const double2 vv = __ldcg(reinterpret_cast<const double2*>(Pv[c] + i));
              const double2 tv = __ldcg(reinterpret_cast<const double2*>(A.t[c] + i));
              const double2 hv = __ldcg(reinterpret_cast<const double2*>(A.rh[c] + i));
              const double s0 = rv.x - al[c] * vv.x, s1 = rv.y - al[c] * vv.y;
              xo.x = xo.x + om[c] * (s0 * iv.x);
              xo.y = xo.y + om[c] * (s1 * iv.y);
              const double r0 = s0 - om[c] * tv.x, r1 = s1 - om[c] * tv.y;
              const double d0 = pv.x - om[c] * vv.x, d1 = pv.y - om[c] * vv.y;
              *reinterpret_cast<double2*>(A.r[c] + i) = make_double2(r0, r1);
              *reinterpret_cast<double2*>(Pd[c] + i) = make_double2(d0, d1);
              if (team && i + 1 >= T.n_inner) {
                if (i >= T.n_inner) {
                  halo_send(T, i, A.slot_r[c], r0);
                  halo_send(T, i, A.slot_p[1][c], d0);
                }
                halo_send(T, i + 1, A.slot_r[c], r1);
                halo_send(T, i + 1, A.slot_p[1][c], d1);
              }
              rr[2 * c] += r0 * r0;
              rr[2 * c + 1] += hv.x * r0;
              rr[2 * c] += r1 * r1;
              rr[2 * c + 1] += hv.y * r1;
            }
            *reinterpret_cast<double2*>(A.x[c] + i) = xo;
          }
        }
        i_scalar = 2 * npair + tid;
      }
      for (int i = i_scalar; i < n; i += G) {
        const double iv = inv[i];
        const bool snd = team && i >= T.n_inner;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (!xa[c]) continue;
          const double pi = Pp[c][i];
          const double phi = pi * iv;
          double xi = A.x[c][i] + al[c] * phi;
          if (full[c]) {
            const double vi = Pv[c][i];
            const double si = A.r[c][i] - al[c] * vi;
            const double shi = si * iv;
            xi = xi + om[c] * shi;
            const double ri = si - om[c] * A.t[c][i];
            const double di = pi - om[c] * vi;
            A.r[c][i] = ri;
            Pd[c][i] = di;
            if (snd) {
              halo_send(T, i, A.slot_r[c], ri);
              halo_send(T, i, A.slot_p[1][c], di);
            }
            rr[2 * c] += ri * ri;
            rr[2 * c + 1] += A.rh[c][i] * ri;
          }
          A.x[c][i] = xi;
        }
      }
      if (timer) { const uint64_t t_ = global_ns(); t_axpy += t_ - tk; tk = t_; }
      if (!team_reduce<2 * NC, false, TEAM, CLUSTER, SYS>(T, A.sync, A.partials, rr, red, rnd, sends)) { timeout = true; break; }
      if (timer) { const uint64_t t_ = global_ns(); t_red += t_ - tk; tk = t_; }
      if (threadIdx.x == 0)
        for (int c = 0; c < NC; ++c) {
          if (!act[c]) continue;
          if (S[c].sconv) { S[c].done = 1; continue; }
          if (!full[c]) continue;
          S[c].rr = rr[2 * c];
          S[c].rhr = rr[2 * c + 1];
          S[c].res = sqrt(rr[2 * c]) / S[c].bn;
          if (!isfinite(S[c].res)) { S[c].err = SE_DIVERGED; S[c].err_it = S[c].it; continue; }
          if (S[c].res <= A.tol || S[c].res * S[c].bn <= A.abs_tol) S[c].done = 1;
        }
      __syncthreads();
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int c = 0; c < NC; ++c) {
      A.result[6 * c + 0] = S[c].it;
      A.result[6 * c + 1] = S[c].done ? 1.0 : 0.0;
      A.result[6 * c + 2] = S[c].res0;
      A.result[6 * c + 3] = S[c].res;
      A.result[6 * c + 4] = timeout ? SE_TIMEOUT : S[c].err;
      A.result[6 * c + 5] = S[c].err_it;
    }
    A.result[18] = 1e-9 * double(t_spmv);
    A.result[19] = 1e-9 * double(t_axpy);
    A.result[20] = 1e-9 * double(t_red);
  }
}

// Persistent batched BiCGStab.  SMEM (single-block systems): r, r_hat, the
// p / d and v buffers, t and 1/D live in dynamic shared memory for the
// solve (x and b stay in global memory).
template <int KT, int NC, bool SC = false, bool TEAM = false, bool CLUSTER = false,
          bool SMEM = false, bool SYS = false>
__global__ void __launch_bounds__(kSolverThreads, FVB_BI_MINB) k_bicgstab3(Bi3Params<NC> A) {
  if constexpr (SMEM) {
    extern __shared__ double dyn[];
    const int n = A.P.n;
    Bi3Params<NC> B = A;
    double* q = dyn;
    for (int c = 0; c < NC; ++c) {
      B.r[c] = q; q += n;
      B.rh[c] = q; q += n;
      B.p[0][c] = q; q += n;
      B.p[1][c] = q; q += n;
      B.v[0][c] = q; q += n;
      B.v[1][c] = q; q += n;
      B.t[c] = q; q += n;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) q[i] = A.inv[i];
    B.inv = q;
    q += n;
    if constexpr (KT > 0) {
      // the matrix and its stencil codes too (read by both SpMV passes)
      for (int e = threadIdx.x; e < KT * n; e += blockDim.x) q[e] = A.V[e];
      B.Vp = q;
      if constexpr (SC) {
        uint8_t* cs = reinterpret_cast<uint8_t*>(q + KT * n);
        for (int i = threadIdx.x; i < n; i += blockDim.x) cs[i] = A.P.code[i];
        B.codep = cs;
      }
    }
    __syncthreads();
    bicgstab3_body<KT, NC, SC, TEAM, CLUSTER, true>(B);
  } else {
    bicgstab3_body<KT, NC, SC, TEAM, CLUSTER, false, SYS>(A);
  }
}

// dynamic shared memory of the SMEM solver kernels for n rows (0 = too large)
inline size_t smem_cg_bytes(int n, int k) {
  return size_t(6 + k) * n * sizeof(double) + size_t(n) + 16;
}
inline size_t smem_bi_bytes(int n, int nc, int k) {
  return size_t(7 * nc + 1 + k) * n * sizeof(double) + size_t(n) + 16;
}
constexpr size_t kSmemSolverMax = 200 * 1024;

template <typename K, typename Args>
int smem_launch(Ctx* c, K kernel, Args& args, int threads, size_t bytes) {
  FVB_CUDA(cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(bytes)));
  FVB_CUDA(cudaMemsetAsync(c->sync, 0, 3 * sizeof(unsigned), c->stream));
  // one row per thread: fewer warps make the block barriers of the tiny
  // solves cheaper (rounded to whole warps pairs, at most `threads`)
  const int t = std::min(threads, std::max(64, (c->nr + 63) / 64 * 64));
  void* params[] = {&args};
  fvb::note_launch();
  FVB_CUDA(cudaLaunchKernel((const void*)kernel, dim3(1), dim3(t), params, bytes, c->stream));
  return FVB_OK;
}

template <typename K>
int coop_blocks(Ctx* c, K kernel, int threads, int max_per_sm, int* blocks) {
  int per_sm = 0;
  FVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0));
  if (per_sm < 1) {
    fvb_set_error("solver kernel cannot be resident");
    return FVB_E_CUDA;
  }
  if (per_sm > max_per_sm) per_sm = max_per_sm;
  // ranks sharing one device (tests): each takes 1/share of the SMs, with
  // `share` SMs left over for the other ranks' one-block sync kernels
  const int share = c->sm_share > 0 ? c->sm_share : 1;
  int b = share > 1 ? per_sm * (c->num_sms - share) / share : per_sm * c->num_sms;
  // small systems: one block (block barriers instead of grid barriers) while
  // a block holds at most two rows per thread (larger ones up to
  // kClusterMaxRows run as one cluster, cluster_want)
  if (!c->teamed() && c->nr <= kSingleBlockRowsPerThread * threads) b = 1;
  if (c->solver_max_blocks > 0 && b > c->solver_max_blocks) b = c->solver_max_blocks;
  if (b > int(kStepPartials / (2 * kRedStride))) b = int(kStepPartials / (2 * kRedStride));
  *blocks = b < 1 ? 1 : b;
  return FVB_OK;
}

template <typename K, typename Args>
int coop_launch(Ctx* c, K kernel, Args& args, int threads = kSolverThreads, int max_per_sm = 2) {
  int blocks = 0;
  FVB_TRY(coop_blocks(c, kernel, threads, max_per_sm, &blocks));
  // words 0-2: arrivals, generation, abort; word 3 (team error) is sticky
  FVB_CUDA(cudaMemsetAsync(c->sync, 0, 3 * sizeof(unsigned), c->stream));
  void* params[] = {&args};
  fvb::note_launch();
  if (c->sm_share > 1) {
    // several ranks share this device: each grid is sized to 1/share of the
    // resident capacity, so the ranks' grids are co-resident together; a
    // plain launch avoids relying on concurrent cooperative launches
    FVB_CUDA(cudaLaunchKernel((const void*)kernel, dim3(blocks), dim3(threads), params, 0,
                              c->stream));
  } else {
    FVB_CUDA(cudaLaunchCooperativeKernel((const void*)kernel, dim3(blocks), dim3(threads),
                                         params, 0, c->stream));
  }
  return FVB_OK;
}

// Small single-domain systems: the persistent solver runs as ONE thread-
// block cluster of `blocks` CTAs (cluster_reduce instead of grid barriers).
// The cluster size (<= 16, non-portable above 8) is what the device can
// co-schedule for this kernel; 0 means no cluster launch is possible.
template <typename K>
int cluster_blocks(Ctx* c, K kernel, int threads, int want) {
  int& cmax = c->cluster_max[threads >= 1024 ? 1 : 0];
  if (cmax < 0) {
    cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxPotentialClusterSize(&n, (const void*)kernel, &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
    cmax = n > 16 ? 16 : n;
  }
  return want <= cmax ? want : cmax;
}

template <typename K, typename Args>
int cluster_launch(Ctx* c, K kernel, Args& args, int threads, int blocks) {
  FVB_CUDA(cudaFuncSetAttribute((const void*)kernel,
                                cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(blocks);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  fvb::note_launch();
  FVB_CUDA(cudaLaunchKernelEx(&cfg, kernel, args));
  return FVB_OK;
}

// cluster size for a single-domain solve of nr rows with `threads`-thread
// CTAs: the largest cluster the device co-schedules (16), none when the system is
// large (the full grid wins above ~40k rows, tools/cg_micro.py) or fits one
// block (block barriers), or the context asks for the grid path
inline int cluster_want(const Ctx* c, int threads) {
  if (c->teamed() || (c->solver_flags & FVB_SOLVER_NO_CLUSTER) || c->sm_share > 1) return 0;
  if (c->nr <= kSingleBlockRowsPerThread * threads || c->nr > kClusterMaxRows) return 0;
  if (c->solver_max_blocks > 0) return 0;  // an explicit grid cap wins
  (void)threads;
  return 16;  // as many SMs as one cluster can hold (cluster_blocks clamps)
}

// Inverse diagonal of the owned rows, and the first zero-diagonal row into
// c->ipart[0] (INT_MAX - row; 0 = none).  A team reads it back now, so a zero
// diagonal anywhere is reported on every rank before any rank enters the
// solve; a single domain leaves it to the solver kernel (zero_diag_exit), so
// the solve needs no host round trip before its launch.  zero_row: INT_MAX,
// or the row when the team found one.
int prepare_diag(Ctx* c, MatView A, double* inv, int* zero_row) {
  int* dz = c->ipart;
  *zero_row = 0x7fffffff;
  FVB_CUDA(cudaMemsetAsync(dz, 0, sizeof(int), c->stream));
  FVB_TRY(launch_inv_diag(c, A.V, inv, dz));
  if (c->teamed()) {
    int v = 0;
    FVB_CUDA(cudaMemcpyAsync(&v, dz, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    FVB_CUDA(cudaStreamSynchronize(c->stream));
    double m = double(v ? 0x7fffffff - v : 0x7fffffff);
    FVB_TRY(team_allreduce(c, &m, 1, RED_MIN));
    *zero_row = int(m);
  }
  return FVB_OK;
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

// RCM-ordered BiCGStab batch: the same gather / scatter for up to three
// right-hand sides and solutions.
struct RcmVecs {
  const double* b[3];
  double* x[3];
  double* bp[3];
  double* xp[3];
};
template <int KT>
__global__ void k_rcm_gather_multi(int n, int ncomp, const int* __restrict__ perm,
                                   const double* __restrict__ V, const double* __restrict__ inv,
                                   double* __restrict__ Vp, double* __restrict__ invp, RcmVecs R) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int o = perm[r];
#pragma unroll
    for (int s = 0; s < KT; ++s) Vp[size_t(s) * n + r] = V[size_t(s) * n + o];
    invp[r] = inv[o];
    for (int k = 0; k < ncomp; ++k) {
      R.bp[k][r] = R.b[k][o];
      R.xp[k][r] = R.x[k][o];
    }
  }
}
__global__ void k_rcm_scatter_multi(int n, int ncomp, const int* __restrict__ perm, RcmVecs R) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    for (int k = 0; k < ncomp; ++k) R.x[k][perm[r]] = R.xp[k][r];
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
  if (!TEAM && (c->k == 7 || c->k == 5)) {
    const int want = cluster_want(c, 1024);
    const int nb = want ? (c->k == 7 ? cluster_blocks(c, k_cg<7, 1024, 1, 1, 1, false, true>, 1024, want)
                                     : cluster_blocks(c, k_cg<5, 1024, 1, 1, 0, false, true>, 1024, want))
                        : 0;
    if (nb >= 2) {
      if (c->k == 7)
        return sc ? cluster_launch(c, k_cg<7, 1024, 1, 1, 1, false, true>, prm, 1024, nb)
                  : cluster_launch(c, k_cg<7, 1024, 1, 0, 1, false, true>, prm, 1024, nb);
      return sc ? cluster_launch(c, k_cg<5, 1024, 1, 1, 0, false, true>, prm, 1024, nb)
                : cluster_launch(c, k_cg<5, 1024, 1, 0, 0, false, true>, prm, 1024, nb);
    }
  }
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

template <int NC>
static int bicg3_launch(Ctx* c, MatView A, const double* const* b, double* const* x, double tol,
                        double abs_tol, int max_iters, double* inv, double* result,
                        const PatternView* pov = nullptr) {
  Bi3Params<NC> prm;
  prm.P = pov ? *pov : c->pattern();
  prm.T = c->team;
  prm.V = A.V;
  prm.crs = A.crs;
  prm.inv = inv;
  prm.slot_inv = S_SCR + 0;
  int s = S_SCR + 1;
  for (int k = 0; k < NC; ++k) {
    prm.b[k] = b[k];
    prm.x[k] = x[k];
    prm.slot_r[k] = s;
    prm.r[k] = c->slot(s++);
    prm.rh[k] = c->slot(s++);
    for (int q = 0; q < 2; ++q) {
      prm.slot_p[q][k] = s;
      prm.p[q][k] = c->slot(s++);
      prm.slot_v[q][k] = s;
      prm.v[q][k] = c->slot(s++);
    }
    prm.t[k] = c->slot(s++);
  }
  prm.tol = tol;
  prm.abs_tol = abs_tol;
  prm.max_iters = max_iters;
  prm.sync = c->sync;
  prm.partials = c->partials;
  prm.result = result;
  prm.zero_flag = c->teamed() ? nullptr : c->ipart;
  prm.Vp = A.V;
  prm.codep = prm.P.code;
  // stencil-coded SpMV sweeps when the pattern has codes (unless the
  // context asks for the explicit indices, FVB_SOLVER_EXPLICIT_INDEX)
  const bool sc = uses_codes(c);
  if (c->teamed() && c->team.sys) {
    switch (c->k) {
      case 5: return sc ? coop_launch(c, k_bicgstab3<5, NC, true, true, false, false, true>, prm, kSolverThreads, FVB_BI_MINB)
                        : coop_launch(c, k_bicgstab3<5, NC, false, true, false, false, true>, prm, kSolverThreads, FVB_BI_MINB);
      case 7: return sc ? coop_launch(c, k_bicgstab3<7, NC, true, true, false, false, true>, prm, kSolverThreads, FVB_BI_MINB)
                        : coop_launch(c, k_bicgstab3<7, NC, false, true, false, false, true>, prm, kSolverThreads, FVB_BI_MINB);
      default: return coop_launch(c, k_bicgstab3<0, NC, false, true, false, false, true>, prm, kSolverThreads, FVB_BI_MINB);
    }
  }
  if (c->teamed()) {
    switch (c->k) {
      case 5: return sc ? coop_launch(c, k_bicgstab3<5, NC, true, true>, prm, kSolverThreads, FVB_BI_MINB)
                        : coop_launch(c, k_bicgstab3<5, NC, false, true>, prm, kSolverThreads, FVB_BI_MINB);
      case 7: return sc ? coop_launch(c, k_bicgstab3<7, NC, true, true>, prm, kSolverThreads, FVB_BI_MINB)
                        : coop_launch(c, k_bicgstab3<7, NC, false, true>, prm, kSolverThreads, FVB_BI_MINB);
      default: return coop_launch(c, k_bicgstab3<0, NC, false, true>, prm, kSolverThreads, FVB_BI_MINB);
    }
  }
  if ((c->k == 7 || c->k == 5) && !pov && c->nr <= kSingleBlockRowsPerThread * kSolverThreads &&
      smem_bi_bytes(c->nr, NC, c->k) <= kSmemSolverMax && !(c->solver_flags & FVB_SOLVER_NO_CLUSTER)) {
    const size_t bytes = smem_bi_bytes(c->nr, NC, c->k);
    if (c->k == 7)
      return sc ? smem_launch(c, k_bicgstab3<7, NC, true, false, false, true>, prm, kSolverThreads, bytes)
                : smem_launch(c, k_bicgstab3<7, NC, false, false, false, true>, prm, kSolverThreads, bytes);
    return sc ? smem_launch(c, k_bicgstab3<5, NC, true, false, false, true>, prm, kSolverThreads, bytes)
              : smem_launch(c, k_bicgstab3<5, NC, false, false, false, true>, prm, kSolverThreads, bytes);
  }
  if (c->k == 7 || c->k == 5) {
    const int want = cluster_want(c, kSolverThreads);
    const int nb = want ? (c->k == 7
                               ? cluster_blocks(c, k_bicgstab3<7, NC, true, false, true>,
                                                kSolverThreads, want)
                               : cluster_blocks(c, k_bicgstab3<5, NC, true, false, true>,
                                                kSolverThreads, want))
                        : 0;
    if (nb >= 2) {
      if (c->k == 7)
        return sc ? cluster_launch(c, k_bicgstab3<7, NC, true, false, true>, prm, kSolverThreads, nb)
                  : cluster_launch(c, k_bicgstab3<7, NC, false, false, true>, prm, kSolverThreads, nb);
      return sc ? cluster_launch(c, k_bicgstab3<5, NC, true, false, true>, prm, kSolverThreads, nb)
                : cluster_launch(c, k_bicgstab3<5, NC, false, false, true>, prm, kSolverThreads, nb);
    }
  }
  switch (c->k) {
    case 5: return sc ? coop_launch(c, k_bicgstab3<5, NC, true>, prm, kSolverThreads, FVB_BI_MINB)
                      : coop_launch(c, k_bicgstab3<5, NC>, prm, kSolverThreads, FVB_BI_MINB);
    case 7: return sc ? coop_launch(c, k_bicgstab3<7, NC, true>, prm, kSolverThreads, FVB_BI_MINB)
                      : coop_launch(c, k_bicgstab3<7, NC>, prm, kSolverThreads, FVB_BI_MINB);
    default: return coop_launch(c, k_bicgstab3<0, NC>, prm, kSolverThreads, FVB_BI_MINB);
  }
}

int bicgstab_solve(Ctx* c, MatView A, int ncomp, const double* const* b, double* const* x,
                   double tol, double abs_tol, int max_iters, SolveOut* out,
                   const Readback* extra) {
  double* inv = c->slot(S_SCR + 0);
  double* result = c->partials + 16 * 4096;
  int zero_row = 0x7fffffff;
  FVB_TRY(prepare_diag(c, A, inv, &zero_row));
  for (int k = 0; k < ncomp; ++k) out[k] = SolveOut{0, 0, SE_NONE, 0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (zero_row != 0x7fffffff) {
    out[0].error_kind = SE_ZERO_DIAG;
    out[0].error_iteration = zero_row;
    return FVB_OK;
  }
  if (ncomp != 1 && ncomp != 3) {
    fvb_set_error("bicgstab batch supports 1 or 3 components");
    return FVB_E_ARG;
  }
  FVB_CUDA(cudaEventRecord(c->kev[0], c->stream));
  if (uses_rcm(c)) {
    // renumbered mesh without stencil codes: solve in the RCM order (as CG)
    if (!c->rcm_V) FVB_TRY(dalloc(c, &c->rcm_V, size_t(c->k) * size_t(c->nr)));
    if (!c->rcm_vec) FVB_TRY(dalloc(c, &c->rcm_vec, size_t(7) * size_t(c->nr)));
    RcmVecs R{};
    double* bpp[3];
    double* xpp[3];
    for (int k = 0; k < ncomp; ++k) {
      R.b[k] = b[k];
      R.x[k] = x[k];
      R.bp[k] = bpp[k] = c->rcm_vec + size_t(2 * k) * c->nr;
      R.xp[k] = xpp[k] = c->rcm_vec + size_t(2 * k + 1) * c->nr;
    }
    double* invp = c->rcm_vec + size_t(6) * c->nr;
    k_rcm_gather_multi<7><<<grid_for(c->nr, 256), 256, 0, c->stream>>>(
        c->nr, ncomp, c->rcm_perm, A.V, inv, c->rcm_V, invp, R);
    note_launch();
    FVB_CUDA(cudaGetLastError());
    PatternView P = c->pattern();
    P.I = c->rcm_I;
    P.diag_slot = c->rcm_ds;
    P.slot_face = nullptr;
    const MatView Ap{c->rcm_V, A.crs};
    if (ncomp == 1)
      FVB_TRY(bicg3_launch<1>(c, Ap, bpp, xpp, tol, abs_tol, max_iters, invp, result, &P));
    else
      FVB_TRY(bicg3_launch<3>(c, Ap, bpp, xpp, tol, abs_tol, max_iters, invp, result, &P));
    k_rcm_scatter_multi<<<grid_for(c->nr, 256), 256, 0, c->stream>>>(c->nr, ncomp, c->rcm_perm, R);
    note_launch();
    FVB_CUDA(cudaGetLastError());
    c->bi_rcm_solves++;
  } else {
    if (ncomp == 1)
      FVB_TRY(bicg3_launch<1>(c, A, b, x, tol, abs_tol, max_iters, inv, result));
    else
      FVB_TRY(bicg3_launch<3>(c, A, b, x, tol, abs_tol, max_iters, inv, result));
  }
  FVB_CUDA(cudaEventRecord(c->kev[1], c->stream));
  double h[21];
  unsigned team_err = 0;
  FVB_CUDA(cudaMemcpyAsync(h, result, sizeof(double) * 21, cudaMemcpyDeviceToHost, c->stream));
  if (extra && extra->n)
    FVB_CUDA(cudaMemcpyAsync(extra->host, extra->dev, sizeof(double) * extra->n,
                             cudaMemcpyDeviceToHost, c->stream));
  FVB_CUDA(cudaMemcpyAsync(&team_err, c->sync + 3, sizeof team_err, cudaMemcpyDeviceToHost, c->stream));
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  if (team_err)
    for (int k = 0; k < ncomp; ++k) h[6 * k + 4] = SE_TIMEOUT;
  for (int k = 0; k < ncomp; ++k) {
    out[k].iterations = int(h[6 * k]);
    out[k].converged = int(h[6 * k + 1]);
    out[k].res0 = h[6 * k + 2];
    out[k].res = h[6 * k + 3];
    out[k].error_kind = int(h[6 * k + 4]);
    out[k].error_iteration = int(h[6 * k + 5]);
    out[k].t_smvp = h[18];
    out[k].t_daxpy = h[19];
    out[k].t_red = h[20];
  }
  float kms = 0.f;
  FVB_CUDA(cudaEventElapsedTime(&kms, c->kev[0], c->kev[1]));
  for (int k = 0; k < ncomp; ++k) out[k].kernel_ms = kms;
  return FVB_OK;
}

}  // namespace fvb
