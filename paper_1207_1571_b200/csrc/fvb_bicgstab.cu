// Jacobi-preconditioned BiCGStab (linsolve.py:175-282) as a persistent,
// cooperatively launched kernel batching the three momentum components
// against one matrix read; see fvb_cg.cu for the shared design (one launch
// per solve, deterministic reductions, stopping rules on the device).
#include "fvb_solvers_common.cuh"

namespace fvb {

namespace {

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
constexpr int kBiBlocksPerSM = 2;

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
  // (a single-block solver owns every row, also when it is one of several
  // independent solves of the launch, k_bicgstab_split)
  const RowRange R = SMEM ? RowRange{int(threadIdx.x), P.n, int(blockDim.x), false}
                          : team_rows(T, P.n);
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
  if (!team_reduce<2 * NC, false, TEAM, CLUSTER, SYS, SMEM>(T, A.sync, A.partials, sums, red, rnd, sends)) {
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
      if (!team_reduce<NC, false, TEAM, CLUSTER, SYS, SMEM>(T, A.sync, A.partials, rv, red, rnd, sends)) { timeout = true; break; }
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
      if (!team_reduce<3 * NC, false, TEAM, CLUSTER, SYS, SMEM>(T, A.sync, A.partials, st, red, rnd, sends)) { timeout = true; break; }
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
      if (!team_reduce<2 * NC, false, TEAM, CLUSTER, SYS, SMEM>(T, A.sync, A.partials, rr, red, rnd, sends)) { timeout = true; break; }
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
  if (threadIdx.x == 0 && (SMEM || blockIdx.x == 0)) {
    for (int c = 0; c < NC; ++c) {
      A.result[6 * c + 0] = S[c].it;
      A.result[6 * c + 1] = S[c].done ? 1.0 : 0.0;
      A.result[6 * c + 2] = S[c].res0;
      A.result[6 * c + 3] = S[c].res;
      A.result[6 * c + 4] = timeout ? SE_TIMEOUT : S[c].err;
      A.result[6 * c + 5] = S[c].err_it;
    }
    if (blockIdx.x == 0) {
      A.result[18] = 1e-9 * double(t_spmv);
      A.result[19] = 1e-9 * double(t_axpy);
      A.result[20] = 1e-9 * double(t_red);
    }
  }
}

// Shared-memory staging of a single-block solve: r, r_hat, the p / d and v
// buffers, t and 1/D (and the matrix with its stencil codes) move to dynamic
// shared memory for the solve; x and b stay in global memory.
template <int KT, int NC, bool SC>
__device__ __forceinline__ void smem_stage(Bi3Params<NC>& B, double* dyn) {
  const int n = B.P.n;
  const double* inv = B.inv;
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
  for (int i = threadIdx.x; i < n; i += blockDim.x) q[i] = inv[i];
  B.inv = q;
  q += n;
  if constexpr (KT > 0) {
    // the matrix and its stencil codes too (read by both SpMV passes)
    for (int e = threadIdx.x; e < KT * n; e += blockDim.x) q[e] = B.V[e];
    B.Vp = q;
    if constexpr (SC) {
      uint8_t* cs = reinterpret_cast<uint8_t*>(q + KT * n);
      for (int i = threadIdx.x; i < n; i += blockDim.x) cs[i] = B.P.code[i];
      B.codep = cs;
    }
  }
  __syncthreads();
}

// Persistent batched BiCGStab.  SMEM (single-block systems): r, r_hat, the
// p / d and v buffers, t and 1/D live in dynamic shared memory for the
// solve (x and b stay in global memory).
template <int KT, int NC, bool SC = false, bool TEAM = false, bool CLUSTER = false,
          bool SMEM = false, bool SYS = false>
__global__ void __launch_bounds__(kSolverThreads, kBiBlocksPerSM) k_bicgstab3(Bi3Params<NC> A) {
  if constexpr (SMEM) {
    extern __shared__ double dyn[];
    Bi3Params<NC> B = A;
    smem_stage<KT, NC, SC>(B, dyn);
    bicgstab3_body<KT, NC, SC, TEAM, CLUSTER, true>(B);
  } else {
    bicgstab3_body<KT, NC, SC, TEAM, CLUSTER, false, SYS>(A);
  }
}

// The three momentum components as three independent single-block solves
// of one launch (block c solves component c; small systems whose batch fits
// in shared memory, C1): a third of the rows' work per thread and a third of
// the values per reduction, on three SMs instead of one (C1 momentum solve
// 260 -> 146 us per step, profiles/r02_small.md).  Each block runs the
// batched kernel's arithmetic for its component (the components of a batch
// never interact: per-component scalars, reductions over M values sum each
// value separately), so the iterates are those of the batched kernel.
template <int KT, bool SC>
__global__ void __launch_bounds__(kSolverThreads, kBiBlocksPerSM) k_bicgstab_split(Bi3Params<3> A) {
  if (A.zero_flag && *A.zero_flag) {  // the batched kernel's zero-diagonal result, once
    if (blockIdx.x == 0) zero_diag_exit(A.zero_flag, A.result, 3);
    return;
  }
  const int c = blockIdx.x;
  Bi3Params<1> B;
  B.P = A.P;
  B.T = A.T;
  B.V = A.V;
  B.crs = A.crs;
  B.inv = A.inv;
  B.b[0] = A.b[c];
  B.x[0] = A.x[c];
  B.tol = A.tol;
  B.abs_tol = A.abs_tol;
  B.max_iters = A.max_iters;
  B.sync = A.sync;
  B.partials = A.partials;
  B.result = A.result + 6 * c;
  B.zero_flag = nullptr;
  B.Vp = A.Vp;
  B.codep = A.codep;
  extern __shared__ double dyn[];
  smem_stage<KT, 1, SC>(B, dyn);
  bicgstab3_body<KT, 1, SC, false, false, true>(B);
}

}  // namespace

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
      case 5: return sc ? coop_launch(c, k_bicgstab3<5, NC, true, true, false, false, true>, prm, kSolverThreads, kBiBlocksPerSM)
                        : coop_launch(c, k_bicgstab3<5, NC, false, true, false, false, true>, prm, kSolverThreads, kBiBlocksPerSM);
      case 7: return sc ? coop_launch(c, k_bicgstab3<7, NC, true, true, false, false, true>, prm, kSolverThreads, kBiBlocksPerSM)
                        : coop_launch(c, k_bicgstab3<7, NC, false, true, false, false, true>, prm, kSolverThreads, kBiBlocksPerSM);
      default: return coop_launch(c, k_bicgstab3<0, NC, false, true, false, false, true>, prm, kSolverThreads, kBiBlocksPerSM);
    }
  }
  if (c->teamed()) {
    switch (c->k) {
      case 5: return sc ? coop_launch(c, k_bicgstab3<5, NC, true, true>, prm, kSolverThreads, kBiBlocksPerSM)
                        : coop_launch(c, k_bicgstab3<5, NC, false, true>, prm, kSolverThreads, kBiBlocksPerSM);
      case 7: return sc ? coop_launch(c, k_bicgstab3<7, NC, true, true>, prm, kSolverThreads, kBiBlocksPerSM)
                        : coop_launch(c, k_bicgstab3<7, NC, false, true>, prm, kSolverThreads, kBiBlocksPerSM);
      default: return coop_launch(c, k_bicgstab3<0, NC, false, true>, prm, kSolverThreads, kBiBlocksPerSM);
    }
  }
  if ((c->k == 7 || c->k == 5) && !pov && c->nr <= kSingleBlockRowsPerThread * kSolverThreads &&
      smem_bi_bytes(c->nr, NC, c->k) <= kSmemSolverMax && !(c->solver_flags & FVB_SOLVER_NO_CLUSTER)) {
    if constexpr (NC == 3) {
      // one block per component (k_bicgstab_split)
      const size_t b1 = smem_bi_bytes(c->nr, 1, c->k);
      if (c->k == 7)
        return sc ? smem_launch(c, k_bicgstab_split<7, true>, prm, kSolverThreads, b1, 3)
                  : smem_launch(c, k_bicgstab_split<7, false>, prm, kSolverThreads, b1, 3);
      return sc ? smem_launch(c, k_bicgstab_split<5, true>, prm, kSolverThreads, b1, 3)
                : smem_launch(c, k_bicgstab_split<5, false>, prm, kSolverThreads, b1, 3);
    } else {
      const size_t bytes = smem_bi_bytes(c->nr, NC, c->k);
      if (c->k == 7)
        return sc ? smem_launch(c, k_bicgstab3<7, NC, true, false, false, true>, prm, kSolverThreads, bytes)
                  : smem_launch(c, k_bicgstab3<7, NC, false, false, false, true>, prm, kSolverThreads, bytes);
      return sc ? smem_launch(c, k_bicgstab3<5, NC, true, false, false, true>, prm, kSolverThreads, bytes)
                : smem_launch(c, k_bicgstab3<5, NC, false, false, false, true>, prm, kSolverThreads, bytes);
    }
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
    case 5: return sc ? coop_launch(c, k_bicgstab3<5, NC, true>, prm, kSolverThreads, kBiBlocksPerSM)
                      : coop_launch(c, k_bicgstab3<5, NC>, prm, kSolverThreads, kBiBlocksPerSM);
    case 7: return sc ? coop_launch(c, k_bicgstab3<7, NC, true>, prm, kSolverThreads, kBiBlocksPerSM)
                      : coop_launch(c, k_bicgstab3<7, NC>, prm, kSolverThreads, kBiBlocksPerSM);
    default: return coop_launch(c, k_bicgstab3<0, NC>, prm, kSolverThreads, kBiBlocksPerSM);
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
