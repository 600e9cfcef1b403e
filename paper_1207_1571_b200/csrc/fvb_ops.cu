// Finite-volume operator kernels (fvm.py restated for sm_100a, FP64).
//
// Assembly is cell-centric: one thread owns one matrix row and walks the
// cell's face list (owned faces ascending, then neighbour faces ascending)
// so every np.add.at accumulation of the reference is replayed in the same
// order with no atomics — deterministic and bitwise faithful.  Face-centric
// kernels (interpolation, fluxes, face data) write coalesced per-face
// arrays.  Per-face data gathered by both adjacent cells is recomputed in
// each (cheap FP64 ALU work; the kernels are bandwidth bound).
#include "fvb_internal.cuh"

namespace fvb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double face_value(const MeshView& M, const BcView& B,
                                             bool raw, int f, const double* __restrict__ v,
                                             const double* __restrict__ bnd) {
  // interpolate_to_faces / interpolate_cell_values (fvm.py:220-247)
  if (f < M.ni) {
    const double w = M.w[f];
    return w * v[M.own[f]] + (1.0 - w) * v[M.nbr[f]];
  }
  const int j = f - M.ni;
  if (!raw && bc_is_value(B.kind[j])) return bnd[j];
  return v[M.own[f]];
}

// ------------------------------------------------------------ geometry
__global__ void k_precompute(MeshView M, double* a, double* kx, double* ky, double* kz,
                             const double* dx, const double* dy, const double* dz,
                             const double* dbx, const double* dby, const double* dbz) {
  // _overrelaxed_split (fvm.py:307-317) is pure geometry: computed once
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M.nf; f += gridDim.x * blockDim.x) {
    double d0, d1, d2;
    if (f < M.ni) {
      d0 = dx[f]; d1 = dy[f]; d2 = dz[f];
    } else {
      const int j = f - M.ni;
      d0 = dbx[j]; d1 = dby[j]; d2 = dbz[j];
    }
    const double s0 = M.sx[f], s1 = M.sy[f], s2 = M.sz[f];
    const double ss = (s0 * s0 + s2 * s2) + s1 * s1;
    const double sd = (s0 * d0 + s2 * d2) + s1 * d1;
    const double af = ss / sd;
    a[f] = af;
    kx[f] = s0 - af * d0;
    ky[f] = s1 - af * d1;
    kz[f] = s2 - af * d2;
  }
}

// ------------------------------------------------------------ boundaries
__global__ void k_apply_bcs(MeshView M, BcView B, int ncomp, const double* __restrict__ vals,
                            double* __restrict__ bnd) {
  // apply_bcs (fvm.py:170-197)
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < M.nb; j += gridDim.x * blockDim.x) {
    const int f = M.ni + j;
    const uint8_t k = B.kind[j];
    for (int c = 0; c < ncomp; ++c) {
      double out;
      if (k == FVB_BC_FIXED) {
        out = B.fixed[size_t(c) * M.nb + j];
      } else if (k == FVB_BC_NO_SLIP) {
        out = 0.0;
      } else if (k == FVB_BC_SINE || k == FVB_BC_MASS_FLOW) {
        const double s = c == 0 ? M.sx[f] : (c == 1 ? M.sy[f] : M.sz[f]);
        const double nh = s / M.smag[f];
        out = (-B.speeds[B.patch[j]]) * nh;
      } else {
        out = vals[size_t(c) * M.nc + M.own[f]];
      }
      bnd[size_t(c) * M.nb + j] = out;
    }
  }
}

__global__ void k_interp(MeshView M, BcView B, bool raw, int ncomp, const double* vals,
                         const double* bnd, double* fv) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M.nf; f += gridDim.x * blockDim.x)
    for (int c = 0; c < ncomp; ++c)
      fv[size_t(c) * M.nf + f] = face_value(M, B, raw, f, vals + size_t(c) * M.nc,
                                            bnd + size_t(c) * M.nb);
}

// ------------------------------------------------------------ gradient
template <int NC>
__global__ void k_gradient(MeshView M, BcView B, const double* __restrict__ vals,
                           const double* __restrict__ bnd, double* __restrict__ grad) {
  // gauss_gradient (fvm.py:258-275): owner faces then neighbour faces, / V
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < M.nr; c += gridDim.x * blockDim.x) {
    double g[NC][3];
#pragma unroll
    for (int i = 0; i < NC; ++i) g[i][0] = g[i][1] = g[i][2] = 0.0;
    const int e1 = M.cf_ptr[c + 1];
    for (int e = M.cf_ptr[c]; e < e1; ++e) {
      const int code = M.cf[e];
      const bool own = code >= 0;
      const int f = own ? code : ~code;
      const double S[3] = {M.sx[f], M.sy[f], M.sz[f]};
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const double fv = face_value(M, B, false, f, vals + size_t(i) * M.nc, bnd + size_t(i) * M.nb);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double con = fv * S[d];
          g[i][d] = own ? g[i][d] + con : g[i][d] + (-con);
        }
      }
    }
    const double V = M.vol[c];
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int d = 0; d < 3; ++d) grad[size_t(i * 3 + d) * M.nc + c] = g[i][d] / V;
  }
}

__global__ void k_divergence(MeshView M, const double* __restrict__ flux, double* __restrict__ div) {
  // face_divergence (fvm.py:250-255)
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < M.nr; c += gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int e1 = M.cf_ptr[c + 1];
    for (int e = M.cf_ptr[c]; e < e1; ++e) {
      const int code = M.cf[e];
      acc = code >= 0 ? acc + flux[code] : acc + (-flux[~code]);
    }
    div[c] = acc;
  }
}

// ------------------------------------------------------------ laplacian
struct LapArgs {
  double gs;            // scalar gamma
  const double* gf;     // per-face gamma or nullptr
  double coeff;
  int nonorth;          // correction active (scheme on and limiter > 0)
  double lim;
};

__device__ __forceinline__ double gam(const LapArgs& L, int f) { return L.gf ? L.gf[f] : L.gs; }

// explicit non-orthogonal correction of one component (fvm.py:383-407)
template <int NC>
__device__ __forceinline__ double lap_corr(const MeshView& M, const LapArgs& L,
                                           const double* __restrict__ grad, int comp, int f) {
  const double k0 = M.kx[f], k1 = M.ky[f], k2 = M.kz[f];
  const double g = gam(L, f);
  const size_t n = M.nc;
  if (f < M.ni) {
    const int o = M.own[f], nb = M.nbr[f];
    const double w = M.w[f];
    double gf[3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
      gf[d] = w * grad[(comp * 3 + d) * n + o] + (1.0 - w) * grad[(comp * 3 + d) * n + nb];
    if (NC == 1) return (((k0 * gf[0] + k2 * gf[2]) + k1 * gf[1]) * g) * L.lim;
    return ((gf[0] * k0 + gf[2] * k2) + gf[1] * k1) * (g * L.lim);
  }
  const int o = M.own[f];
  const double g0 = grad[(comp * 3 + 0) * n + o], g1 = grad[(comp * 3 + 1) * n + o],
               g2 = grad[(comp * 3 + 2) * n + o];
  if (NC == 1) return (((k0 * g0 + k2 * g2) + k1 * g1) * g) * L.lim;
  return ((g0 * k0 + g2 * k2) + g1 * k1) * (g * L.lim);
}

template <int NC>
__global__ void k_laplacian_rows(MeshView M, PatternView P, BcView B, LapArgs L, MatView A,
                                 double* __restrict__ rhs, const double* __restrict__ bnd,
                                 const double* __restrict__ grad) {
  // laplacian (fvm.py:335-408), one matrix row per thread
  const int n = P.n;            // rows = slot stride of V
  const size_t nv = M.nc;       // component stride of cell vectors
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int e0 = M.cf_ptr[c], e1 = M.cf_ptr[c + 1];
    const int ds = P.diag_slot[c];
    double d = A.V[size_t(ds) * n + c];
    for (int e = e0; e < e1; ++e) {  // diag_addr[owner] -= w, internal, ascending
      const int code = M.cf[e];
      if (code >= 0 && code < M.ni) d = d + (-((L.coeff * gam(L, code)) * M.a[code]));
    }
    for (int e = e0; e < e1; ++e) {  // diag_addr[neighbour] -= w
      const int code = M.cf[e];
      if (code < 0) { const int f = ~code; d = d + (-((L.coeff * gam(L, f)) * M.a[f])); }
    }
    int last_value = -1;
    for (int e = e0; e < e1; ++e) {  // value-pinned boundary faces -= w_b
      const int f = M.cf[e];
      if (f >= M.ni && bc_is_value(B.kind[f - M.ni])) {
        d = d + (-((L.coeff * gam(L, f)) * M.a[f]));
        last_value = f;
      }
    }
    A.V[size_t(ds) * n + c] = d;
    for (int s = 0; s < P.k; ++s) {  // both face_addr slots += w
      if (s == ds) continue;
      const int f = P.slot_face[size_t(s) * n + c];
      if (f >= 0) A.V[size_t(s) * n + c] += (L.coeff * gam(L, f)) * M.a[f];
    }
    if (P.nnz_crs) {
      for (int q = P.crs_ptr[c]; q < P.crs_ptr[c + 1]; ++q) {
        const int f = P.crs_face[q];
        A.crs[q] += (L.coeff * gam(L, f)) * M.a[f];
      }
    }
    // right-hand side
    double r[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) r[i] = rhs[size_t(i) * nv + c];
    if (NC == 3) {
      // vector branch: fancy-index "-=", the highest-index face wins (fvm.py:378-379)
      if (last_value >= 0) {
        const double wb = (L.coeff * gam(L, last_value)) * M.a[last_value];
        const int j = last_value - M.ni;
#pragma unroll
        for (int i = 0; i < NC; ++i) r[i] = r[i] - wb * bnd[size_t(i) * M.nb + j];
      }
    } else {
      for (int e = e0; e < e1; ++e) {  // np.add.at, ascending (fvm.py:381)
        const int f = M.cf[e];
        if (f >= M.ni && bc_is_value(B.kind[f - M.ni])) {
          const double wb = (L.coeff * gam(L, f)) * M.a[f];
          r[0] = r[0] + (-wb) * bnd[f - M.ni];
        }
      }
    }
    if (L.nonorth) {
      const double mc = -L.coeff;
      for (int e = e0; e < e1; ++e) {  // owner rows of internal faces
        const int code = M.cf[e];
        if (code >= 0 && code < M.ni) {
#pragma unroll
          for (int i = 0; i < NC; ++i) r[i] = r[i] + mc * lap_corr<NC>(M, L, grad, i, code);
        }
      }
      for (int e = e0; e < e1; ++e) {  // neighbour rows
        const int code = M.cf[e];
        if (code < 0) {
#pragma unroll
          for (int i = 0; i < NC; ++i) r[i] = r[i] + L.coeff * lap_corr<NC>(M, L, grad, i, ~code);
        }
      }
      for (int e = e0; e < e1; ++e) {  // value-pinned boundary faces
        const int f = M.cf[e];
        if (f >= M.ni && bc_is_value(B.kind[f - M.ni])) {
#pragma unroll
          for (int i = 0; i < NC; ++i) r[i] = r[i] + mc * lap_corr<NC>(M, L, grad, i, f);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) rhs[size_t(i) * nv + c] = r[i];
  }
}

template <int NC>
__global__ void k_laplacian_faces(MeshView M, BcView B, LapArgs L, const double* __restrict__ grad,
                                  double* __restrict__ coef, double* __restrict__ corr) {
  // LaplacianFaceData (fvm.py:320-332): coef = gamma a, corr frozen
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M.nf; f += gridDim.x * blockDim.x) {
    const bool active = f < M.ni || bc_is_value(B.kind[f - M.ni]);
    coef[f] = active ? gam(L, f) * M.a[f] : 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i)
      corr[size_t(i) * M.nf + f] = (active && L.nonorth) ? lap_corr<NC>(M, L, grad, i, f) : 0.0;
  }
}

__global__ void k_lap_flux(MeshView M, BcView B, int ncomp, const double* __restrict__ coef,
                           const double* __restrict__ corr, const double* __restrict__ vals,
                           const double* __restrict__ bnd, double* __restrict__ out) {
  // laplacian_face_flux (fvm.py:411-429)
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M.nf; f += gridDim.x * blockDim.x) {
    for (int i = 0; i < ncomp; ++i) {
      const double* v = vals + size_t(i) * M.nc;
      double dphi;
      if (f < M.ni) {
        dphi = v[M.nbr[f]] - v[M.own[f]];
      } else {
        const int j = f - M.ni;
        const double vo = v[M.own[f]];
        const double bv = bc_is_value(B.kind[j]) ? bnd[size_t(i) * M.nb + j] : vo;
        dphi = bv - vo;
      }
      out[size_t(i) * M.nf + f] = coef[f] * dphi + corr[size_t(i) * M.nf + f];
    }
  }
}

// ------------------------------------------------------------ convection
template <int NC>
__global__ void k_convection_rows(MeshView M, PatternView P, BcView B, MatView A,
                                  double* __restrict__ rhs, const double* __restrict__ flux,
                                  const double* __restrict__ bnd, int linear, double coeff) {
  // divergence_convection (fvm.py:432-482), one matrix row per thread
  const int n = P.n;            // rows = slot stride of V
  const size_t nv = M.nc;       // component stride of cell vectors
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int e0 = M.cf_ptr[c], e1 = M.cf_ptr[c + 1];
    const int ds = P.diag_slot[c];
    double d = A.V[size_t(ds) * n + c];
    for (int e = e0; e < e1; ++e) {  // diag(owner) += coeff F w_own
      const int code = M.cf[e];
      if (code >= 0 && code < M.ni) {
        const double F = flux[code];
        const double wo = linear ? M.w[code] : (F >= 0.0 ? 1.0 : 0.0);
        d = d + (coeff * F) * wo;
      }
    }
    for (int e = e0; e < e1; ++e) {  // diag(neighbour) -= coeff F (1 - w_own)
      const int code = M.cf[e];
      if (code < 0) {
        const int f = ~code;
        const double F = flux[f];
        const double wo = linear ? M.w[f] : (F >= 0.0 ? 1.0 : 0.0);
        d = d + (-((coeff * F) * (1.0 - wo)));
      }
    }
    int last_value = -1;
    for (int e = e0; e < e1; ++e) {  // zero-gradient outflow, implicit
      const int f = M.cf[e];
      if (f >= M.ni) {
        const uint8_t k = B.kind[f - M.ni];
        if (k == FVB_BC_ZERO_GRADIENT) {
          const double F = flux[f];
          const double mx = (F >= 0.0 || F != F) ? F : 0.0;
          d = d + coeff * mx;
        } else if (bc_is_value(k)) {
          last_value = f;
        }
      }
    }
    A.V[size_t(ds) * n + c] = d;
    for (int s = 0; s < P.k; ++s) {
      if (s == ds) continue;
      const int f = P.slot_face[size_t(s) * n + c];
      if (f < 0) continue;
      const double F = flux[f];
      const double wo = linear ? M.w[f] : (F >= 0.0 ? 1.0 : 0.0);
      if (M.own[f] == c)
        A.V[size_t(s) * n + c] += (coeff * F) * (1.0 - wo);
      else
        A.V[size_t(s) * n + c] += -((coeff * F) * wo);
    }
    if (P.nnz_crs) {
      for (int q = P.crs_ptr[c]; q < P.crs_ptr[c + 1]; ++q) {
        const int f = P.crs_face[q];
        const double F = flux[f];
        const double wo = linear ? M.w[f] : (F >= 0.0 ? 1.0 : 0.0);
        A.crs[q] += (M.own[f] == c) ? (coeff * F) * (1.0 - wo) : -((coeff * F) * wo);
      }
    }
    if (NC == 3) {
      if (last_value >= 0) {  // vector branch: highest-index value face wins (fvm.py:473)
        const double cb = coeff * flux[last_value];
        const int j = last_value - M.ni;
#pragma unroll
        for (int i = 0; i < NC; ++i)
          rhs[size_t(i) * nv + c] = rhs[size_t(i) * nv + c] - cb * bnd[size_t(i) * M.nb + j];
      }
    } else {
      double r = rhs[c];
      for (int e = e0; e < e1; ++e) {
        const int f = M.cf[e];
        if (f >= M.ni && bc_is_value(B.kind[f - M.ni])) {
          const double cb = coeff * flux[f];
          r = r + (-cb) * bnd[f - M.ni];
        }
      }
      rhs[c] = r;
    }
  }
}

__global__ void k_ddt(int nv, PatternView P, MatView A, int ncomp, double* __restrict__ rhs,
                      const double* __restrict__ old, const double* __restrict__ vol, double dt,
                      double coeff) {
  // ddt_euler (fvm.py:485-496); rows P.n, cell vectors strided by nv
  const int n = P.n;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double vdt = (coeff * vol[c]) / dt;
    const int ds = P.diag_slot[c];
    A.V[size_t(ds) * n + c] += vdt;
    for (int i = 0; i < ncomp; ++i) rhs[size_t(i) * nv + c] += vdt * old[size_t(i) * nv + c];
  }
}

__global__ void k_face_flux(MeshView M, BcView B, const double* __restrict__ vals,
                            const double* __restrict__ bnd, double* __restrict__ flux) {
  // S . u_f, zero on empty faces (coupling.py:206-213, 292-296)
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M.nf; f += gridDim.x * blockDim.x) {
    if (f >= M.ni && B.kind[f - M.ni] == FVB_BC_EMPTY) {
      flux[f] = 0.0;
      continue;
    }
    const double f0 = face_value(M, B, false, f, vals, bnd);
    const double f1 = face_value(M, B, false, f, vals + M.nc, bnd + M.nb);
    const double f2 = face_value(M, B, false, f, vals + 2 * size_t(M.nc), bnd + 2 * size_t(M.nb));
    flux[f] = (f0 * M.sx[f] + f2 * M.sz[f]) + f1 * M.sy[f];
  }
}

// rhie_chow_flux (fvm.py:499-538): F = S . u_f, minus on internal faces
// D_f a_f [(p_N - p_O) - (grad p)_f . d] with D = V / a_diag interpolated
// linearly, and on boundary faces where p is pinned but u is not the same
// with the owner's D and d_b; 0 on faces where u is empty.  Dot products in
// the reference's einsum order (x + z) + y, as k_face_flux.
__global__ void k_rhie_chow(MeshView M, BcView Bu, BcView Bp, const double* __restrict__ u,
                            const double* __restrict__ ub, const double* __restrict__ p,
                            const double* __restrict__ pb, const double* __restrict__ adiag,
                            const double* __restrict__ gp, const double* __restrict__ d,
                            const double* __restrict__ db, double* __restrict__ flux) {
  const size_t nc = size_t(M.nc), ni = size_t(M.ni), nb = size_t(M.nb);
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M.nf; f += gridDim.x * blockDim.x) {
    const int j = f - M.ni;
    if (f >= M.ni && Bu.kind[j] == FVB_BC_EMPTY) {
      flux[f] = 0.0;
      continue;
    }
    const double f0 = face_value(M, Bu, false, f, u, ub);
    const double f1 = face_value(M, Bu, false, f, u + nc, ub + nb);
    const double f2 = face_value(M, Bu, false, f, u + 2 * nc, ub + 2 * nb);
    double F = (f0 * M.sx[f] + f2 * M.sz[f]) + f1 * M.sy[f];
    const int o = M.own[f];
    const double d_o = M.vol[o] / adiag[o];
    if (f < M.ni) {
      const int q = M.nbr[f];
      const double w = M.w[f], w1 = 1.0 - w;
      const double d_f = w * d_o + w1 * (M.vol[q] / adiag[q]);
      const double g0 = w * gp[o] + w1 * gp[q];
      const double g1 = w * gp[nc + o] + w1 * gp[nc + q];
      const double g2 = w * gp[2 * nc + o] + w1 * gp[2 * nc + q];
      const double gd = (g0 * d[f] + g2 * d[2 * ni + f]) + g1 * d[ni + f];
      F -= (d_f * M.a[f]) * ((p[q] - p[o]) - gd);
    } else if (bc_is_value(Bp.kind[j]) && !bc_is_value(Bu.kind[j])) {
      const double gd = (gp[o] * db[j] + gp[2 * nc + o] * db[2 * nb + j]) + gp[nc + o] * db[nb + j];
      F -= (d_o * M.a[f]) * ((pb[j] - p[o]) - gd);
    }
    flux[f] = F;
  }
}

__global__ void k_inv_diag(int n, const int* __restrict__ ds, const double* __restrict__ V,
                           double* __restrict__ inv, int* first_zero) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d = V[size_t(ds[i]) * n + i];
    // first zero-diagonal row, encoded INT_MAX - row (0 = none; max = first)
    if (d == 0.0) atomicMax(first_zero, 0x7fffffff - i);
    inv[i] = 1.0 / d;
  }
}

template <int KT>
__global__ void k_smvp(PatternView P, const double* __restrict__ V, const double* __restrict__ crs,
                       const double* __restrict__ x, double* __restrict__ y) {
  const int n = P.n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    auto g = [&](int col) { return x[col]; };
    double r = ell_row<KT>(V, P.I, n, P.k, i, g);
    y[i] = crs_tail(P, crs, i, r, g);
  }
}

// stmvp (sparse.py:308-334): y = A^T x scanning row i, the value of the
// transposed twin (c, i) of every stored (i, c) gathered through J (ELL
// twin slot, slot-major V) or ell_twin_crs; padding contributes 0.  Same
// einsum order as the SpMV; the CRS tail accumulates sequentially.
template <int KT>
__global__ void k_stmvp(PatternView P, const double* __restrict__ V, const double* __restrict__ crs,
                        const int* __restrict__ J, const int* __restrict__ twin_crs,
                        const uint8_t* __restrict__ ct_in_ell, const int* __restrict__ ct_row,
                        const int* __restrict__ ct_pos, const double* __restrict__ x,
                        double* __restrict__ y) {
  const int n = P.n;
  const int K = KT > 0 ? KT : P.k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    auto term = [&](int s) {
      const int c = P.I[size_t(s) * n + i];
      const int col = c < 0 ? 0 : c;
      const int js = J[size_t(s) * n + i];
      double tv = V[size_t(js < 0 ? 0 : js) * n + col];
      if (P.nnz_crs && js < 0) {
        const int q = twin_crs[size_t(s) * n + i];
        tv = crs[q < 0 ? 0 : q];
      }
      if (c < 0) tv = 0.0;
      return tv * x[col];
    };
    double ev = term(0);
    for (int s = 2; s < K; s += 2) ev = ev + term(s);
    double yy = ev;
    if (K > 1) {
      double od = term(1);
      for (int s = 3; s < K; s += 2) od = od + term(s);
      yy = ev + od;
    }
    if (P.nnz_crs) {
      double t = 0.0;
      for (int q = P.crs_ptr[i]; q < P.crs_ptr[i + 1]; ++q) {
        const int pos = ct_pos[q];
        const double tv = ct_in_ell[q] ? V[size_t(pos < P.k - 1 ? pos : P.k - 1) * n + ct_row[q]]
                                       : crs[pos < P.nnz_crs - 1 ? pos : P.nnz_crs - 1];
        t += tv * x[P.crs_col[q]];
      }
      yy = yy + t;
    }
    y[i] = yy;
  }
}

}  // namespace

// ------------------------------------------------------------ launchers
int op_precompute_geometry(Ctx* c, const double* dx, const double* dy, const double* dz,
                           const double* dbx, const double* dby, const double* dbz) {
  { k_precompute<<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(
      c->mesh(), c->a, c->kx, c->ky, c->kz, dx, dy, dz, dbx, dby, dbz); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_apply_bcs(Ctx* c, int field, int ncomp, const double* vals, double* bnd) {
  if (c->nb == 0) return FVB_OK;
  { k_apply_bcs<<<grid_for(c->nb, kThreads), kThreads, 0, c->stream>>>(c->mesh(), c->bc(field), ncomp,
                                                                     vals, bnd); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_interp(Ctx* c, int field, int ncomp, const double* vals, const double* bnd, double* fv) {
  BcView B = field >= 0 ? c->bc(field) : BcView{nullptr, nullptr, nullptr, nullptr};
  { k_interp<<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(c->mesh(), B, field < 0, ncomp,
                                                                   vals, bnd, fv); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_gradient(Ctx* c, int field, int ncomp, const double* vals, const double* bnd,
                double* grad) {
  if (ncomp == 1)
    { k_gradient<1><<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(c->mesh(), c->bc(field),
                                                                         vals, bnd, grad); fvb::note_launch(); }
  else
    { k_gradient<3><<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(c->mesh(), c->bc(field),
                                                                         vals, bnd, grad); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_divergence(Ctx* c, const double* flux, double* div) {
  { k_divergence<<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(c->mesh(), flux, div); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_laplacian(Ctx* c, int field, int ncomp, MatView A, double* rhs, double gamma,
                 const double* gamma_faces, const double* vals, const double* bnd,
                 const double* grad, int nonorth, double limiter, double coeff, double* coef,
                 double* corr) {
  (void)vals;
  if (c->first_zero_dmag >= 0) {
    fvb_set_error("coincident centroids at internal face %d", c->first_zero_dmag);
    return FVB_E_FVM;
  }
  if (c->first_zero_dbmag_value[field] >= 0) {
    fvb_set_error("coincident centroids at boundary face %d", c->first_zero_dbmag_value[field]);
    return FVB_E_FVM;
  }
  LapArgs L{gamma, gamma_faces, coeff, nonorth && limiter > 0.0, limiter};
  if (ncomp == 1) {
    { k_laplacian_rows<1><<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(
        c->mesh(), c->pattern(), c->bc(field), L, A, rhs, bnd, grad); fvb::note_launch(); }
    if (coef)
      { k_laplacian_faces<1><<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(
          c->mesh(), c->bc(field), L, grad, coef, corr); fvb::note_launch(); }
  } else {
    { k_laplacian_rows<3><<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(
        c->mesh(), c->pattern(), c->bc(field), L, A, rhs, bnd, grad); fvb::note_launch(); }
    if (coef)
      { k_laplacian_faces<3><<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(
          c->mesh(), c->bc(field), L, grad, coef, corr); fvb::note_launch(); }
  }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_lap_flux(Ctx* c, int field, int ncomp, const double* coef, const double* corr,
                const double* vals, const double* bnd, double* out) {
  { k_lap_flux<<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(c->mesh(), c->bc(field), ncomp,
                                                                    coef, corr, vals, bnd, out); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_convection(Ctx* c, int field, int ncomp, MatView A, double* rhs, const double* flux,
                  const double* bnd, int scheme, double coeff) {
  if (ncomp == 1)
    { k_convection_rows<1><<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(
        c->mesh(), c->pattern(), c->bc(field), A, rhs, flux, bnd, scheme, coeff); fvb::note_launch(); }
  else
    { k_convection_rows<3><<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(
        c->mesh(), c->pattern(), c->bc(field), A, rhs, flux, bnd, scheme, coeff); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_ddt(Ctx* c, int ncomp, MatView A, double* rhs, const double* old, double dt,
           double coeff) {
  { k_ddt<<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(c->nc, c->pattern(), A, ncomp, rhs,
                                                               old, c->vol, dt, coeff); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_face_flux(Ctx* c, int ncomp_field, const double* vals, const double* bnd,
                 int field_for_mask, double* flux) {
  (void)ncomp_field;
  { k_face_flux<<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(c->mesh(), c->bc(field_for_mask),
                                                                     vals, bnd, flux); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int op_rhie_chow(Ctx* c, const double* u, const double* ub, const double* p, const double* pb,
                 const double* adiag, const double* gp, const double* d, const double* db,
                 double* flux) {
  { k_rhie_chow<<<grid_for(c->nf, kThreads), kThreads, 0, c->stream>>>(
        c->mesh(), c->bc(0), c->bc(1), u, ub, p, pb, adiag, gp, d, db, flux); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int launch_inv_diag(Ctx* c, const double* V, double* inv, int* first_zero) {
  { k_inv_diag<<<grid_for(c->nr, kThreads), kThreads, 0, c->stream>>>(c->nr, c->diag_slot, V, inv,
                                                                     first_zero); fvb::note_launch(); }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int smvp(Ctx* c, MatView A, const double* x, double* y) {
  PatternView P = c->pattern();
  const int g = grid_for(c->nr, kThreads);
  switch (c->k) {
    case 5: { k_smvp<5><<<g, kThreads, 0, c->stream>>>(P, A.V, A.crs, x, y); fvb::note_launch(); } break;
    case 7: { k_smvp<7><<<g, kThreads, 0, c->stream>>>(P, A.V, A.crs, x, y); fvb::note_launch(); } break;
    default: { k_smvp<0><<<g, kThreads, 0, c->stream>>>(P, A.V, A.crs, x, y); fvb::note_launch(); } break;
  }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int stmvp(Ctx* c, MatView A, const int* J, const int* twin_crs, const uint8_t* ct_in_ell,
          const int* ct_row, const int* ct_pos, const double* x, double* y) {
  PatternView P = c->pattern();
  const int g = grid_for(c->nr, kThreads);
  switch (c->k) {
    case 7: { k_stmvp<7><<<g, kThreads, 0, c->stream>>>(P, A.V, A.crs, J, twin_crs, ct_in_ell, ct_row, ct_pos, x, y); fvb::note_launch(); } break;
    default: { k_stmvp<0><<<g, kThreads, 0, c->stream>>>(P, A.V, A.crs, J, twin_crs, ct_in_ell, ct_row, ct_pos, x, y); fvb::note_launch(); } break;
  }
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

}  // namespace fvb
