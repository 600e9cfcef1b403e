// libfvb internals: device-resident mesh/pattern/state, shared kernels'
// helpers, deterministic reductions and the grid barrier used by the
// persistent Krylov kernels.  FP64 throughout; compiled with -fmad=false so
// every a*b+c rounds twice, exactly like the numpy reference.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/fvb.h"
#include "common.h"

#define FVB_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      fvb_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),      \
                    __FILE__, __LINE__, cudaGetErrorString(e_));             \
      return FVB_E_CUDA;                                                     \
    }                                                                        \
  } while (0)

#define FVB_TRY(call)         \
  do {                        \
    int rc_ = (call);         \
    if (rc_ != FVB_OK) return rc_; \
  } while (0)

namespace fvb {

constexpr int kMaxK = 1 << 20;  // K is a runtime bound on the generic path

// host-side count of kernel launches issued by libfvb (fvb_launch_count)
extern unsigned long long g_launches;
inline void note_launch() { ++g_launches; }

// ------------------------------------------------------------ device views
// Face numbering follows the reference: internal faces [0, ni), boundary
// faces [ni, nf); boundary arrays are indexed j = f - ni.
struct MeshView {
  int nc, nf, ni, nb;
  const int* own;     // [nf]
  const int* nbr;     // [ni]
  const double* sx;   // area vector S, SoA [nf]
  const double* sy;
  const double* sz;
  const double* smag; // |S| [nf]
  const double* vol;  // [nc]
  const double* w;    // owner interpolation weight [ni]
  const double* a;    // |S|^2/(S.d) [nf]: internal with d, boundary with d_b
  const double* kx;   // S - a d      [nf]
  const double* ky;
  const double* kz;
  const int* cf_ptr;  // per-cell face list [nc+1]
  const int* cf;      // f for owned faces, ~f for neighbour faces
};

struct PatternView {
  int n, k, nnz_crs;
  const int* I;          // slot-major [k*n], -1 padding
  const int* diag_slot;  // [n]
  const int* slot_face;  // slot-major [k*n]: internal face of the entry, -1
  const int* crs_ptr;    // [n+1] (nullptr when nnz_crs == 0)
  const int* crs_col;
  const int* crs_face;
};

struct BcView {
  const uint8_t* kind;   // [nb]
  const int* patch;      // [nb]
  const double* fixed;   // [ncomp*nb]
  const double* speeds;  // [n_patches]
};

__host__ __device__ inline bool bc_is_value(uint8_t k) { return k >= FVB_BC_FIXED; }

// A matrix over the pattern: slot-major values + CRS values.
struct MatView {
  double* V;    // [k*n]
  double* crs;  // [nnz_crs]
};

// --------------------------------------------------------------- context
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
};

struct Ctx {
  int dev = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8];
  cudaEvent_t tev[2];
  cudaEvent_t kev[2];
  int64_t bytes = 0;
  bool have_mesh = false, have_pattern = false;
  bool have_bc[2] = {false, false};
  int nc = 0, nf = 0, ni = 0, nb = 0, k = 0, nnz_crs = 0;
  int first_zero_dmag = -1;          // coincident-centroid internal face
  int first_zero_dbmag_value[2] = {-1, -1};
  std::vector<double> dbmag_host;    // boundary |d_b| (for BC checks)
  int n_patches[2] = {0, 0};
  // mesh
  int *own = nullptr, *nbr = nullptr, *cf_ptr = nullptr, *cf = nullptr;
  double *sx = nullptr, *sy = nullptr, *sz = nullptr, *smag = nullptr;
  double *vol = nullptr, *w = nullptr, *a = nullptr, *kx = nullptr,
         *ky = nullptr, *kz = nullptr;
  // pattern
  int *I = nullptr, *diag_slot = nullptr, *slot_face = nullptr;
  int *crs_ptr = nullptr, *crs_col = nullptr, *crs_face = nullptr;
  // boundary conditions: 0 = u (3 comps), 1 = p
  uint8_t* bc_kind[2] = {nullptr, nullptr};
  int* bc_patch[2] = {nullptr, nullptr};
  double* bc_fixed[2] = {nullptr, nullptr};
  double* bc_speed[2] = {nullptr, nullptr};
  // coupled state (SoA)
  double *u = nullptr, *p = nullptr, *flux = nullptr, *ub = nullptr, *pb = nullptr;
  // work
  std::vector<void*> allocs;
  double* scratch = nullptr;  // general work pool
  size_t scratch_n = 0;
  unsigned* sync = nullptr;   // grid barrier words + error slots
  double* partials = nullptr;
  int* ipart = nullptr;
  double* host_pinned = nullptr;  // small pinned staging buffer

  MeshView mesh() const {
    return MeshView{nc, nf, ni, nb, own, nbr, sx, sy, sz, smag, vol, w, a, kx, ky, kz, cf_ptr, cf};
  }
  PatternView pattern() const {
    return PatternView{nc, k, nnz_crs, I, diag_slot, slot_face, crs_ptr, crs_col, crs_face};
  }
  BcView bc(int field) const {
    return BcView{bc_kind[field], bc_patch[field], bc_fixed[field], bc_speed[field]};
  }
};

template <typename T>
int dalloc(Ctx* c, T** out, size_t n) {
  void* p = nullptr;
  size_t bytes = (n ? n : 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    fvb_set_error("cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
    return FVB_E_CUDA;
  }
  c->allocs.push_back(p);
  c->bytes += int64_t(bytes);
  *out = static_cast<T*>(p);
  return FVB_OK;
}

// ------------------------------------------------------- kernel helpers
inline int grid_for(int64_t n, int threads, int cap = 148 * 32) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return int(b);
}

// Reference SpMV order for one row (sparse.py:302, numpy einsum): products
// of even slots summed left to right, odd slots likewise, then even + odd.
// Gather functor G(col) returns x[col]; padding slots gather x[0] (V = 0).
template <int KT, typename G>
__device__ __forceinline__ double ell_row(const double* __restrict__ V,
                                          const int* __restrict__ I, int n,
                                          int kdyn, int i, G gather) {
  const int K = KT > 0 ? KT : kdyn;
  double ev = 0.0, od = 0.0;
#pragma unroll
  for (int s = 0; s < (KT > 0 ? KT : K); s += 2) {
    if (KT == 0 && s >= K) break;
    int col = __ldg(I + size_t(s) * n + i);
    double v = __ldg(V + size_t(s) * n + i);
    double pr = v * gather(col < 0 ? 0 : col);
    ev = (s == 0) ? pr : ev + pr;
  }
#pragma unroll
  for (int s = 1; s < (KT > 0 ? KT : K); s += 2) {
    if (KT == 0 && s >= K) break;
    int col = __ldg(I + size_t(s) * n + i);
    double v = __ldg(V + size_t(s) * n + i);
    double pr = v * gather(col < 0 ? 0 : col);
    od = (s == 1) ? pr : od + pr;
  }
  return K > 1 ? ev + od : ev;
}

// CRS tail of a row (np.bincount: sequential from 0), then y + tail.
template <typename G>
__device__ __forceinline__ double crs_tail(const PatternView& P, const double* crs,
                                           int i, double y, G gather) {
  if (P.nnz_crs == 0) return y;
  int s = P.crs_ptr[i], e = P.crs_ptr[i + 1];
  double t = 0.0;
  for (int q = s; q < e; ++q) t += crs[q] * gather(P.crs_col[q]);
  return y + t;
}

// Deterministic block reduction of M doubles; result valid in thread 0.
template <int M>
__device__ __forceinline__ void block_reduce(double (&v)[M], double* smem /*[32*M]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int m = 0; m < M; ++m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[m] += __shfl_down_sync(0xffffffffu, v[m], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int m = 0; m < M; ++m) smem[warp * M + m] = v[m];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double x = lane < nw ? smem[lane * M + m] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      v[m] = x;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid-wide barrier for co-resident (cooperatively launched) grids.
// sync[0] = arrival count, sync[1] = generation, sync[2] = abort flag.
// A watchdog turns a would-be hang into FVB_E_TIMEOUT instead of a dead GPU.
__device__ __forceinline__ bool grid_barrier(unsigned* sync, unsigned nblocks) {
  __syncthreads();
  __shared__ int s_abort;
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = sync + 1;
    volatile unsigned* vabort = sync + 2;
    unsigned gen = *vgen;
    __threadfence();
    unsigned arrived = atomicAdd(sync, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(sync, 0u);
      __threadfence();
      atomicAdd(sync + 1, 1u);
    } else {
      uint64_t t0 = global_ns();
      while (*vgen == gen) {
        if (*vabort) break;
        __nanosleep(20);
        if (global_ns() - t0 > 20000000000ull) {  // 20 s watchdog
          atomicExch(sync + 2, 1u);
          break;
        }
      }
    }
    __threadfence();
    s_abort = *vabort;
  }
  __syncthreads();
  return s_abort == 0;
}

// After a barrier: every block sums the per-block partials of M scalars in
// the same fixed order, so all blocks hold bit-identical results.
template <int M>
__device__ __forceinline__ void grid_sum(const double* partials, int nblocks,
                                         double (&out)[M], double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double x = 0.0;
      for (int b = lane; b < nblocks; b += 32) x += __ldcg(partials + size_t(m) * nblocks + b);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      if (lane == 0) smem[m] = x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < M; ++m) out[m] = smem[m];
  __syncthreads();
}

template <int M>
__device__ __forceinline__ void publish_partials(double (&v)[M], double* partials,
                                                 double* smem) {
  block_reduce<M>(v, smem);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int m = 0; m < M; ++m) partials[size_t(m) * gridDim.x + blockIdx.x] = v[m];
  }
}

// ------------------------------------------------------------ launchers
// (implemented in fvb_ops.cu / fvb_solvers.cu)
int launch_inv_diag(Ctx* c, const double* V, double* inv, int* first_zero);
int smvp(Ctx* c, MatView A, const double* x, double* y);

struct SolveOut {
  int iterations, converged, error_kind, error_iteration;
  double res0, res;
  double kernel_ms;  // device time of the persistent solver kernel alone
};
enum SolveErr {
  SE_NONE = 0,
  SE_ZERO_DIAG = 1,
  SE_CG_NOT_SPD = 2,
  SE_DIVERGED = 3,
  SE_RHO = 4,
  SE_RV = 5,
  SE_OMEGA = 6,
  SE_TIMEOUT = 7,
};
// x must hold x0 on entry; returns solution in x.
int cg_solve(Ctx* c, MatView A, const double* b, double* x, double tol,
             double abs_tol, int max_iters, SolveOut* out);
int bicgstab_solve(Ctx* c, MatView A, int ncomp, const double* const* b,
                   double* const* x, double tol, double abs_tol, int max_iters,
                   SolveOut* out);
std::string solve_error_text(const char* solver, const SolveOut& o, int zero_row);

// FV operators on device buffers (fvb_ops.cu)
int op_apply_bcs(Ctx* c, int field, int ncomp, const double* vals, double* bnd);
int op_interp(Ctx* c, int field, int ncomp, const double* vals, const double* bnd,
              double* fv);
int op_gradient(Ctx* c, int field, int ncomp, const double* vals, const double* bnd,
                double* grad);
int op_divergence(Ctx* c, const double* flux, double* div);
int op_laplacian(Ctx* c, int field, int ncomp, MatView A, double* rhs, double gamma,
                 const double* gamma_faces, const double* vals, const double* bnd,
                 const double* grad, int nonorth, double limiter, double coeff,
                 double* coef, double* corr);
int op_lap_flux(Ctx* c, int field, int ncomp, const double* coef, const double* corr,
                const double* vals, const double* bnd, double* out);
int op_convection(Ctx* c, int field, int ncomp, MatView A, double* rhs,
                  const double* flux, const double* bnd, int scheme, double coeff);
int op_ddt(Ctx* c, int ncomp, MatView A, double* rhs, const double* old, double dt,
           double coeff);
int op_face_flux(Ctx* c, int ncomp_field, const double* vals, const double* bnd,
                 int field_for_mask, double* flux);
int op_precompute_geometry(Ctx* c, const double* dx, const double* dy,
                           const double* dz, const double* dbx, const double* dby,
                           const double* dbz);

}  // namespace fvb

struct fvb_ctx {
  fvb::Ctx c;
};
