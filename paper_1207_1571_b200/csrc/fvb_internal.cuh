// libfvb internals: device-resident mesh/pattern/state, shared kernel
// helpers, deterministic reductions, and the team (domain-decomposition)
// layer: every cell vector lives in one per-context "cell pool" whose
// base address is shared with the other ranks of the team (CUDA IPC across
// processes, plain pointers inside one process), so kernels store halo
// values straight into a neighbour's ghost slots over NVLink and exchange
// reduction partials through peer mailboxes.  FP64 throughout; compiled
// with -fmad=false so every a*b+c rounds twice, exactly like the numpy
// reference.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include <atomic>
#include <string>
#include <unordered_map>
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
constexpr int kMaxTeam = 8;     // ranks of one domain decomposition (one node)
constexpr int kMailM = 16;      // doubles per mailbox message

// host-side count of kernel launches issued by libfvb (fvb_launch_count);
// ranks of an in-process team launch from several host threads
extern std::atomic<unsigned long long> g_launches;
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ------------------------------------------------------------ cell pool
// Slot map of the per-context cell pool.  Every slot is one cell vector of
// nc doubles (owned rows first, then ghost cells); multi-component fields
// occupy consecutive slots, so component c of a field is base + c*nc.
enum Slot : int {
  S_U = 0,        // u, 3 slots
  S_P = 3,        // p
  S_HV = 4,       // HbyA, 3
  S_RAU = 7,      // rAU
  S_GU = 8,       // grad u, 9
  S_GP = 17,      // grad p, 3
  S_AU = 20,      // A u, 3
  S_B0 = 23,      // momentum rhs b0, 3
  S_RHS = 26,     // momentum solve rhs, 3
  S_DIAG = 29,    // momentum diagonal
  S_DIVH = 30,    // div(phiHbyA)
  S_RL = 31,      // pressure Laplacian rhs
  S_RP = 32,      // pressure solve rhs
  S_PBEFORE = 33, // p before the SIMPLE correction
  S_SCR = 34,     // solver scratch
  kScrSlots = 26, // BiCGStab x3: inv + 8 vectors per component + spare
  kPoolSlots = S_SCR + kScrSlots,
};

// Team comm area at the head of the pool (shared with the peers).
struct Comm {
  unsigned long long seq[kMaxTeam];              // written by peers: last epoch seen
  unsigned long long epoch;                      // local: team syncs completed
  unsigned long long pad[7];
  double mail[2][kMaxTeam][kMailM];              // [epoch parity][sender][payload]
  // solver reductions of a decomposed mesh (team_reduce): arrivals of every
  // rank's blocks (written by the peers), rounds this rank completed
  unsigned long long tr_arrive;
  unsigned long long tr_round;  // reductions this rank completed (all launches)
  unsigned long long tr_base;   // block arrivals those reductions took (grids differ per kernel)
};
// team-partials buffer of the solver reductions, after the comm struct:
// [round parity][sender rank][value][sender block], written by the peers
constexpr unsigned long long kReduceTimeoutMark = 0xFEEDFACE00000000ull;  // Comm::pad[6]
constexpr int kTeamGridMax = 512;  // blocks of a team solver grid (coop_blocks caps)
constexpr size_t kTeamPartOffset = 4096;
constexpr size_t kTeamPartBytes = size_t(2) * kMaxTeam * 16 * kTeamGridMax * sizeof(double);
constexpr size_t kCommBytes = kTeamPartOffset + kTeamPartBytes;
static_assert(sizeof(Comm) <= kTeamPartOffset, "comm area");
__host__ __device__ inline double* team_part(Comm* c) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(c) + kTeamPartOffset);
}
__host__ __device__ inline size_t team_part_index(int par, int rank, int m, int block) {
  return ((size_t(par) * kMaxTeam + size_t(rank)) * 16 + size_t(m)) * kTeamGridMax + size_t(block);
}

// Device view of the team: who the peers are and where their pools are.
struct TeamView {
  int rank, size;             // size 1 = no decomposition
  int sys;                    // 1: ranks on several devices (system-scope ordering)
  Comm* comm;                 // local comm area
  Comm* peer_comm[kMaxTeam];  // every rank's comm area (own included)
  double* peer_cells[kMaxTeam];  // every rank's slot 0 base
  int peer_nc[kMaxTeam];      // every rank's slot stride
  // halo sends: owned rows >= n_inner send their values; row i sends
  // entries send_ptr[i-n_inner] .. send_ptr[i-n_inner+1] to
  // (send_rank[e], ghost index send_dst[e])
  int n_inner;
  const int* send_ptr;
  const int* send_rank;
  const int* send_dst;
};

// Row ownership of one block in the persistent solvers: rows are
// grid-strided over every thread (a sweep front that keeps the +-n^2
// neighbours of the rows in flight L2-resident).  In a team every block may
// hold send rows, so every arrival is ordered at the team's scope.  (Giving
// the send rows their own few blocks, so only those arrive at system scope,
// measured 40% slower per CG iteration on one device: profiles/r01_team.md.)
struct RowRange {
  int begin, end, step;
  bool sends;
};
__device__ __forceinline__ RowRange team_rows(const TeamView& T, int nrows) {
  return RowRange{int(blockIdx.x) * int(blockDim.x) + int(threadIdx.x), nrows,
                  int(gridDim.x) * int(blockDim.x), T.size > 1 && nrows > T.n_inner};
}

// Store value v of row i (pool slot `slot`) into the ghost copies held by
// the ranks that need it.
__device__ __forceinline__ void halo_send(const TeamView& T, int i, int slot, double v) {
  const int t = i - T.n_inner;
  const int e1 = T.send_ptr[t + 1];
  for (int e = T.send_ptr[t]; e < e1; ++e) {
    const int q = T.send_rank[e];
    T.peer_cells[q][size_t(slot) * T.peer_nc[q] + T.send_dst[e]] = v;
  }
}

// ------------------------------------------------------------ device views
// Face numbering follows the reference: internal faces [0, ni), boundary
// faces [ni, nf); boundary arrays are indexed j = f - ni.  Row loops run
// over the nr owned cells; vectors hold nc = nr + ghosts entries.
struct MeshView {
  int nc, nr, nf, ni, nb;
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
  const int* cf_ptr;  // per-row face list [nr+1]
  const int* cf;      // f for owned faces, ~f for neighbour faces
};

struct PatternView {
  int n, k, nnz_crs;     // n = rows (slot stride of V and I)
  const int* I;          // slot-major [k*n], -1 padding, columns < nc
  const int* diag_slot;  // [n]
  const int* slot_face;  // slot-major [k*n]: internal face of the entry, -1
  const int* crs_ptr;    // [n+1] (nullptr when nnz_crs == 0)
  const int* crs_col;
  const int* crs_face;
  // Stencil codes (nullptr when off): row i's column offsets are
  // stab[code[i]*k + s] (col = i + offset; kPadOffset = padding, column 0),
  // code kEscapeCode = read I.  Built at upload when few distinct offset
  // tuples cover the rows (structured and block-structured meshes).
  const uint8_t* code;
  const int* stab;
  int ncode;
};
constexpr int kMaxCodes = 255;      // distinct offset tuples per pattern
constexpr int kEscapeCode = 255;    // row outside the dictionary: explicit I
constexpr int kPadOffset = INT_MIN; // padding slot (column 0, value 0)

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
struct Ctx {
  int dev = 0;
  int num_sms = 148;
  int sm_share = 1;                 // teams sharing one device (tests): grid / sm_share
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8] = {};
  cudaEvent_t tev[2];
  cudaEvent_t kev[2];
  // correction-tail event pairs of one step's correctors, read after the
  // step's final sync (pressure_correct)
  static constexpr int kTailPairs = 8;
  cudaEvent_t cev[2 * kTailPairs] = {};
  int n_tail = 0;
  // per-operator timing of one step (RunState.ops): event pairs + op ids
  static constexpr int kOpEvents = 96;
  cudaEvent_t opev[kOpEvents];
  int op_id[kOpEvents / 2];
  int n_op = 0;
  // CUDA graphs of the step's assembly segments (step_segment, fvb_api.cu):
  // captured on first use per segment instance and step configuration,
  // replayed afterwards; dropped when the context allocates (new pointers)
  struct Seg {
    cudaGraphExec_t exec = nullptr;
    std::vector<int> ops;            // operator-timer ids the segment records
    unsigned long long launches = 0; // kernel launches it holds
  };
  std::unordered_map<uint64_t, Seg> segs;
  size_t seg_allocs = 0;             // allocs.size() the graphs were captured under
  int64_t bytes = 0;
  bool have_mesh = false, have_pattern = false;
  bool have_bc[2] = {false, false};
  int nc = 0, nr = 0, nf = 0, ni = 0, nb = 0, k = 0, nnz_crs = 0;
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
  uint8_t* scode = nullptr;  // stencil codes (PatternView::code), or nullptr
  int* stab = nullptr;
  int n_scode = 0;
  int64_t n_sescape = 0;     // rows coded kEscapeCode
  // bandwidth-reducing (reverse Cuthill-McKee) order for CG on patterns
  // without stencil codes: rcm_perm[new] = old row, permuted slot-major
  // columns and diagonal slots; the per-solve permuted matrix in rcm_V
  int* rcm_perm = nullptr;
  int* rcm_I = nullptr;
  int* rcm_ds = nullptr;
  double* rcm_V = nullptr;
  double* rcm_vec = nullptr;  // BiCGStab: b', x' per component + 1/D'
  int64_t cg_rcm_solves = 0;
  int solver_flags = 0;      // FVB_SOLVER_* (fvb_set_solver_options)
  int solver_max_blocks = 0; // persistent solver grid cap (fvb_set_solver_grid; 0 = auto)
  int cluster_max[2] = {-1, -1};  // largest solver cluster, 512 / 1024 threads (-1 = not queried)
  int64_t bi_rcm_solves = 0;
  int *crs_ptr = nullptr, *crs_col = nullptr, *crs_face = nullptr;
  // boundary conditions: 0 = u (3 comps), 1 = p
  uint8_t* bc_kind[2] = {nullptr, nullptr};
  int* bc_patch[2] = {nullptr, nullptr};
  double* bc_fixed[2] = {nullptr, nullptr};
  double* bc_speed[2] = {nullptr, nullptr};
  // cell pool (comm area + kPoolSlots vectors of nc doubles)
  char* pool = nullptr;
  double* cells = nullptr;           // slot 0
  // coupled state on the device (faces/boundary arrays outside the pool)
  double *u = nullptr, *p = nullptr, *flux = nullptr, *ub = nullptr, *pb = nullptr;
  // team
  TeamView team{};
  int* send_ptr = nullptr;
  int* send_rank = nullptr;
  int* send_dst = nullptr;
  // step work (allocated once, at upload time: never inside a step, where a
  // peer rank may be spinning in a team sync)
  bool work_ready = false;
  double *Vm = nullptr, *crsm = nullptr, *Vp = nullptr, *crsp = nullptr, *phih = nullptr,
         *rauf = nullptr, *coef = nullptr, *corr = nullptr, *lf = nullptr;
  double* u_save = nullptr;  // u before the batched momentum solve (error rollback)
  // work
  std::vector<void*> allocs;
  double* scratch = nullptr;  // solver scratch (pool slots S_SCR..)
  unsigned* sync = nullptr;   // grid barrier words + broadcast slots
  double* partials = nullptr;
  int* ipart = nullptr;

  double* slot(int s) const { return cells + size_t(s) * nc; }
  int slot_of(const double* q) const {
    if (!cells || q < cells) return -1;
    const size_t off = size_t(q - cells);
    if (off % size_t(nc)) return -1;
    const size_t s = off / size_t(nc);
    return s < size_t(kPoolSlots) ? int(s) : -1;
  }
  MeshView mesh() const {
    return MeshView{nc, nr, nf, ni, nb, own, nbr, sx, sy, sz, smag, vol, w, a, kx, ky, kz,
                    cf_ptr, cf};
  }
  PatternView pattern() const {
    return PatternView{nr, k, nnz_crs, I, diag_slot, slot_face, crs_ptr, crs_col, crs_face,
                       scode, stab, n_scode};
  }
  BcView bc(int field) const {
    return BcView{bc_kind[field], bc_patch[field], bc_fixed[field], bc_speed[field]};
  }
  bool teamed() const { return team.size > 1; }
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

// create the cell pool once nc is known (mesh or pattern upload)
int ensure_pool(Ctx* c);

// Regions of Ctx::partials (16*4096 + 256 doubles): grid-reduction partials
// from 0 (at most 2 x 9 x 2 x 148 doubles), step-level block partials read
// back with a solve's results, solver results, team allreduce staging.
constexpr size_t kStepPartials = 32768;
// single-domain systems up to this many rows solve on one thread-block
// cluster (cluster_reduce), larger ones on the full persistent grid
constexpr int kClusterMaxRows = 40000;
// ... and systems of at most this many rows per thread of one block run on a
// single block (block barriers; tools/cg_micro.py: CG at 3375 rows 9.4 us
// per iteration on one block against ~7 on a 16-CTA cluster)
constexpr int kSingleBlockRowsPerThread = 2;
constexpr size_t kResults = 16 * 4096;

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
    int col = __ldg(I + size_t(s) * n + i);
    double v = __ldg(V + size_t(s) * n + i);
    double pr = v * gather(col < 0 ? 0 : col);
    ev = (s == 0) ? pr : ev + pr;
  }
#pragma unroll
  for (int s = 1; s < (KT > 0 ? KT : K); s += 2) {
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

// block_reduce without the trailing barrier (result in thread 0): for the
// single-block and cluster reductions, whose next barrier already orders
// the reuse of smem
template <int M>
__device__ __forceinline__ void block_reduce_lean(double (&v)[M], double* smem /*[32*M]*/) {
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
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr uint64_t kWatchdogNs = 20000000000ull;  // 20 s: a hang becomes FVB_E_TIMEOUT

enum ReduceOp { RED_SUM = 0, RED_MAX = 1, RED_MIN = 2 };

// Exchange M doubles with every rank of the team and combine them in rank
// order (identical on every rank).  Called by ONE thread.  Returns false
// when the watchdog fired.  Epoch parity double-buffers the mailboxes: a
// rank can run at most one sync ahead of the slowest reader.
template <int M>
__device__ bool team_exchange(const TeamView& T, double (&v)[M], int op) {
  Comm* me = T.comm;
  volatile unsigned long long* vep = &me->epoch;  // written by other blocks' SMs
  const unsigned long long ep = *vep + 1;
  *vep = ep;
  const int par = int(ep & 1ull);
  // This rank's halo stores are already ordered before this thread (the
  // blocks' sys-scope acq_rel arrivals, or the fence.sys that ends every
  // halo-push thread); one fence then orders the payloads before the flags.
  for (int q = 0; q < T.size; ++q) {
    Comm* pc = T.peer_comm[q];
#pragma unroll
    for (int m = 0; m < M; ++m) pc->mail[par][T.rank][m] = v[m];
  }
  if (T.sys) __threadfence_system(); else __threadfence();
  for (int q = 0; q < T.size; ++q)
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&T.peer_comm[q]->seq[T.rank]),
                 "l"(ep)
                 : "memory");
  const uint64_t t0 = global_ns();
  for (int q = 0; q < T.size; ++q) {
    for (;;) {
      unsigned long long sq;
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(sq) : "l"(&me->seq[q]) : "memory");
      if (sq >= ep) break;
      if (global_ns() - t0 > kWatchdogNs) {
        // diagnostics for the host: the epoch waited for and every flag seen
        me->pad[0] = ep;
        for (int k = 0; k < T.size && k < 6; ++k) me->pad[1 + k] = me->seq[k];
        return false;
      }
    }
  }
  // relaxed reads that observed every flag + fence = acquire (the
  // mailboxes and the peers' halo stores below are current)
  if (T.sys)
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const volatile double* box = &me->mail[par][0][m];
    double acc = box[0];
    for (int q = 1; q < T.size; ++q) {
      const double x = box[q * kMailM];
      acc = op == RED_SUM ? acc + x : (op == RED_MAX ? fmax(acc, x) : fmin(acc, x));
    }
    v[m] = acc;
  }
  return true;
}

// Scoped atomics / loads of the single-device grid barrier: arrival is a
// release add on a monotonic counter, waiters poll relaxed and finish with
// a fence (an acquire pattern that also invalidates this SM's L1).
__device__ __forceinline__ void red_release_add(unsigned* p, bool sys) {
  if (sys)
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
  else
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid(+team)-wide deterministic sum of M doubles for co-resident
// (cooperatively launched) grids.  v holds each thread's partial sums on
// entry and the global sums on exit, bit-identical in every thread of every
// block of every rank: every block sums all block partials itself in a
// fixed order (lane-strided over blocks, then a shuffle tree; per rank and
// then in rank order when the mesh is decomposed).  sync words: [0]
// arrivals (single device), [2] abort flag.  The barrier also orders every
// halo store issued before it.  Returns false on watchdog.
// Partials of consecutive reductions alternate between two buffers of
// kRedStride x gridDim.x doubles.  The buffer stride must not depend on M:
// with a stride of M x gridDim.x, a fast block writing the partials of
// reduction k+1 (M = 2) overlapped the upper half of reduction k's buffer
// (M = 1) while a slow block could still be reading it — a rare wrong
// p.q in one block (profiles/r02_stress.md).
constexpr size_t kRedStride = 16;

// Lane-strided sums of G block partials of M values (value m of block b at
// base[m * ms + b]) in the order of the plain loop
//   for (b = lane; b < G; b += 32) x[m] += base[m * ms + b],
// with the loads of a lane issued together instead of one L2 round trip per
// value and per block stride: on 148 blocks a reduction took 3.6 us with the
// plain loop, 2.1 us with every load issued first and 2.4 us with the
// value-inner form (tools/probe/barrier_probe.cu, profiles/r02_barrier_probe.md).
// Out-of-range lanes load a valid partial and skip the add (same sums,
// bitwise, as the plain loop).
template <int M, int NB>
__device__ __forceinline__ void lane_sums_fixed(const double* __restrict__ base, size_t ms, int G,
                                                int lane, double (&x)[M]) {
  double xs[M][NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const int b = min(lane + 32 * k, G - 1);
#pragma unroll
    for (int m = 0; m < M; ++m) xs[m][k] = __ldcg(base + size_t(m) * ms + b);
  }
#pragma unroll
  for (int m = 0; m < M; ++m) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < NB; ++k) a = lane + 32 * k < G ? a + xs[m][k] : a;
    x[m] = a;
  }
}
template <int M>
__device__ __forceinline__ void lane_sums(const double* __restrict__ base, size_t ms, int G,
                                          int lane, double (&x)[M]) {
  const int nb = (G + 31) >> 5;
#ifdef FVB_DIAG_LANE_SUMS_FIXED  // diagnostic builds: every load of a lane issued first
  if (M <= 3 && nb <= 5) {
    lane_sums_fixed<M, 5>(base, ms, G, lane, x);
    return;
  }
#endif
#pragma unroll
  for (int m = 0; m < M; ++m) x[m] = 0.0;
  for (int k = 0; k < nb; ++k) {  // value-inner: the M loads of one stride together
    const int b = lane + 32 * k;
    if (b < G) {
#pragma unroll
      for (int m = 0; m < M; ++m) x[m] += __ldcg(base + size_t(m) * ms + b);
    }
  }
}

// Reduction of a kernel launched as ONE thread-block cluster (small single-
// domain systems, CLUSTER kernels): each CTA publishes its block sum in its
// own shared memory, one hardware cluster barrier (release/acquire, which
// also invalidates L1 for the vectors the next pass gathers), and every CTA
// sums the CTAs' values over distributed shared memory in rank order — no
// global-memory atomics or polling (~1 us less per barrier than the grid
// path on 16 SMs).  Buffers alternate by round parity, as the grid path.
template <int M>
__device__ __forceinline__ void cluster_reduce(double (&v)[M], double* smem, unsigned& rnd) {
  __shared__ double s_cl[2][kRedStride];
  block_reduce_lean<M>(v, smem);
  double* mine = s_cl[rnd & 1u];
  ++rnd;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int m = 0; m < M; ++m) mine[m] = v[m];
  }
  cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
  cl.sync();
  // remote loads in parallel (one value per thread), then the rank-order sum
  const unsigned nb = cl.num_blocks();
  __shared__ double s_all[16 * kRedStride];
  if (threadIdx.x < nb * unsigned(M)) {
    const unsigned b = threadIdx.x / unsigned(M), m = threadIdx.x % unsigned(M);
    s_all[b * M + m] = cl.map_shared_rank(mine, b)[m];
  }
  __syncthreads();
  if (threadIdx.x < unsigned(M)) {
    double acc = 0.0;
    for (unsigned b = 0; b < nb; ++b) acc += s_all[b * M + threadIdx.x];
    smem[32 * M + threadIdx.x] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < M; ++m) v[m] = smem[32 * M + m];
  // (no trailing barrier: the next reduction's cluster barrier orders the
  // reuse of smem and s_all)
}

// Per-block copies of the rank's round and arrival counts at the launch's
// first team reduction.  Namespace scope, not inside team_reduce: each
// instantiation (M = 1, 2, 3, ...) of a function-scope __shared__ variable
// would be a different variable.
static __shared__ unsigned long long s_team_round0;
static __shared__ unsigned long long s_team_arrive0;

// TEAM = false: the kernel instantiation for a single domain, which
// compiles the team path away (it costs registers in the solver loops).
// CLUSTER: the kernel runs as one thread-block cluster (cluster_reduce).
// SYS: a team over several devices (compile-time, so the single-device and
// co-resident team kernels carry no system-scope code).
// OOL: unused since the team path stopped going through the mailboxes
// (kept so the call sites read the same).
// BLOCK: the kernel is a single-block solver (a block may be one of several
// independent solves of a launch), whose block barrier is the grid barrier.
template <int M, bool OOL = false, bool TEAM = true, bool CLUSTER = false, bool SYS = false,
          bool BLOCK = false>
__device__ __forceinline__ bool team_reduce(const TeamView& T, unsigned* sync,
                                            double* partials, double (&v)[M],
                                            double* smem /*[32*M+M]*/, unsigned& rnd,
                                            bool sends = true) {
  if (CLUSTER) {
    cluster_reduce<M>(v, smem, rnd);
    return true;
  }
  static_assert(M <= int(kRedStride), "team_reduce: at most kRedStride values");
  __shared__ int s_ok;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef FVB_DIAG_FENCE  // diagnostic build (tools/build_variant.py): every thread fences
  __threadfence();
#endif
  // (TEAM kernels are launched for decomposed meshes only: no single-device
  // path in them)
  if (!TEAM) {
    // One device: a monotonic arrival counter, no last-arriver hand-off.
    // Every block publishes its partials, arrives with a release add and
    // waits until all gridDim.x blocks of round rnd arrived, then sums the
    // partials itself in the fixed order (identical in every block).
    // Partials are double-buffered by round parity: a block writes round
    // r+2 only after passing round r+1, i.e. after every block finished
    // reading round r.
    (void)sends;
    if (BLOCK || gridDim.x == 1) {
      // small systems run on a single block: the block barrier is the grid
      // barrier (two barriers per reduction: the next reduction's first one
      // orders the reuse of the broadcast slot; a one-barrier variant in
      // which every warp sums the warp partials itself measured slower,
      // profiles/r02_small.md)
      block_reduce_lean<M>(v, smem);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m) smem[32 * M + m] = v[m];
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < M; ++m) v[m] = smem[32 * M + m];
      ++rnd;
      return true;
    }
    block_reduce<M>(v, smem);
    const unsigned r = rnd++;
    double* part = partials + size_t(r & 1u) * kRedStride * gridDim.x;
    volatile unsigned* vabort = sync + 2;
    if (threadIdx.x == 0) {
#pragma unroll
      for (int m = 0; m < M; ++m) part[size_t(m) * gridDim.x + blockIdx.x] = v[m];
      red_release_add(sync, false);
      const unsigned target = (r + 1u) * gridDim.x;
      const uint64_t t0 = global_ns();
      int spins = 0;
      while (ld_relaxed_gpu(sync) < target) {
        if (*vabort) break;
        if (++spins > 64) __nanosleep(32);
        if ((spins & 1023) == 0 && global_ns() - t0 > kWatchdogNs) {
          atomicExch(sync + 2, 1u);
          break;
        }
      }
      // acquire before anyone reads partials or vectors of other blocks:
      // the relaxed load that observed every arrival + fence.acq_rel is an
      // acquire pattern (and invalidates this SM's L1).  (An ld.acquire
      // whose value is unused is dropped by ptxas down to its L1
      // invalidate, which is what round 1 had.)
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      s_ok = *vabort == 0;
    }
    __syncthreads();
    if (M > 1) {
      // several values: one warp per value, in parallel
      if (warp < M) {
        const int G = int(gridDim.x);
        const double* pm = part + size_t(warp) * gridDim.x;
        double x = 0.0;
        for (int b = lane; b < G; b += 32) x += __ldcg(pm + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) smem[32 * M + warp] = x;
      }
    } else if (warp == 0) {
      double xs[M];
      lane_sums<M>(part, gridDim.x, int(gridDim.x), lane, xs);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double x = xs[m];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) smem[32 * M + m] = x;
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = smem[32 * M + m];
    const bool ok = s_ok != 0;
    __syncthreads();
#ifdef FVB_DIAG_FENCE
    __threadfence();
#endif
    return ok;
  }
  // Decomposed mesh (TEAM kernels): flat all-to-all arrival, no last
  // arriver, no mailbox round trip, no broadcast.  Thread 0 of every block
  // stores the block's partial sums into EVERY rank's team-partials buffer
  // (peer memory: NVLink across devices) and then arrives once on every
  // rank's 64-bit arrival counter after one release fence at the team's
  // scope (system scope across devices: the fence also orders the block's
  // halo stores of the pass, observed by thread 0 through the block barrier).  Each
  // block then waits on its OWN rank's counter for the P x G arrivals of
  // this round and sums the partials itself: per rank, lane-strided over
  // that rank's blocks and a shuffle tree, then the ranks in order — the same
  // sum the per-rank last arriver + rank-order mailbox combine formed, on
  // every block of every rank.  Rounds and arrivals are counted across
  // launches (the rank's completed rounds and the arrivals they took live in
  // its comm area: the CG and BiCGStab grids differ in size), so a fast
  // peer's arrivals for the next launch are never lost to a counter reset; buffers
  // alternate by round parity (a block writes round k+2 only after round
  // k+1 completed everywhere, i.e. after every block read round k).  Every
  // rank of a team runs the same grid size (same device type, same share).
  (void)sends;  // every block of a team holds send rows (grid-strided rows)
  unsigned long long& s_base = s_team_round0;
  unsigned long long& s_abase = s_team_arrive0;
  block_reduce<M>(v, smem);
  volatile unsigned* vabort = sync + 2;
  Comm* me = T.comm;
  const unsigned r = rnd++;
  if (threadIdx.x == 0) {
    if (r == 0) {  // rounds and arrivals of the earlier launches
      s_base = me->tr_round;
      s_abase = me->tr_base;
    }
    const unsigned long long round = s_base + r;
    const unsigned long long per_round = (unsigned long long)(T.size) * gridDim.x;
    const int par = int(round & 1ull);
#pragma unroll 1
    for (int q = 0; q < T.size; ++q) {
      double* part = team_part(T.peer_comm[q]) + team_part_index(par, T.rank, 0, blockIdx.x);
#pragma unroll
      for (int m = 0; m < M; ++m) part[size_t(m) * kTeamGridMax] = v[m];
    }
    // one release fence, then relaxed arrivals (a release pattern for every
    // counter: one system-scope fence per block and reduction instead of P)
    if (SYS)
      asm volatile("fence.acq_rel.sys;" ::: "memory");
    else
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll 1
    for (int q = 0; q < T.size; ++q) {
      unsigned long long* ctr = &T.peer_comm[q]->tr_arrive;
      if (SYS)
        asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
      else
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    }
    const unsigned long long target = s_abase + (r + 1ull) * per_round;
    const uint64_t t0 = global_ns();
    int spins = 0;
    for (;;) {
      unsigned long long seen;
      if (SYS)
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(seen) : "l"(&me->tr_arrive) : "memory");
      else
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(&me->tr_arrive) : "memory");
      if (seen >= target) break;
      if (*vabort) break;
      if (++spins > 64) __nanosleep(32);
      if ((spins & 1023) == 0 && global_ns() - t0 > kWatchdogNs) {
        // diagnostics for the host (team_timeout_error): the round waited
        // for and the arrivals seen
        me->pad[0] = target;
        me->pad[1] = seen;
        me->pad[6] = kReduceTimeoutMark;
        atomicExch(sync + 2, 1u);
        break;
      }
    }
    // acquire: one acquire load of the counter whose value is used (ptxas
    // keeps it; the partials and the peers' halo stores are then current,
    // L1 invalidated) instead of a full fence after the relaxed polls
    {
      unsigned long long seen2;
      if (SYS)
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(seen2) : "l"(&me->tr_arrive) : "memory");
      else
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen2) : "l"(&me->tr_arrive) : "memory");
      if (seen2 < target) atomicExch(sync + 2, 1u);  // cannot happen: counters only grow
    }
    s_ok = *vabort == 0;
    // block 0 records the round for the next launch (every block read the
    // base before its first arrival, and round r completed only after
    // every block arrived)
    if (blockIdx.x == 0) {
      me->tr_round = round + 1ull;
      me->tr_base = target;
    }
  }
  __syncthreads();
  if (warp < M) {
    // one warp per value (in parallel): per rank lane-strided over that
    // rank's blocks and a shuffle tree, then the ranks in order
    const int par = int((s_base + r) & 1ull);
    const double* part = team_part(me);
    const int G = int(gridDim.x);
    double acc = 0.0;
    for (int q = 0; q < T.size; ++q) {
      const double* pq = part + team_part_index(par, q, warp, 0);
      double x = 0.0;
      for (int b = lane; b < G; b += 32) x += __ldcg(pq + b);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      acc = q == 0 ? x : acc + x;  // rank order, as the mailbox combine
    }
    if (lane == 0) smem[32 * M + warp] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < M; ++m) v[m] = smem[32 * M + m];
  const bool ok = s_ok != 0;
  __syncthreads();
  return ok;
}

// ------------------------------------------------------------ launchers
// (implemented in fvb_ops.cu / fvb_cg.cu / fvb_bicgstab.cu / fvb_team.cu)
int launch_inv_diag(Ctx* c, const double* V, double* inv, int* first_zero);
int smvp(Ctx* c, MatView A, const double* x, double* y);
int stmvp(Ctx* c, MatView A, const int* J, const int* twin_crs, const uint8_t* ct_in_ell,
          const int* ct_row, const int* ct_pos, const double* x, double* y);

struct SolveOut {
  int iterations, converged, error_kind, error_iteration;
  double res0, res;
  double kernel_ms;  // device time of the persistent solver kernel alone
  double t_smvp, t_daxpy, t_red;  // device stage timers (s), block 0's view
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
// Extra device -> host copy folded into a solve's result readback (one
// stream sync for both).
struct Readback {
  const double* dev;
  double* host;
  int n;
};
// x must hold x0 on entry (ghost entries current); returns solution in x.
int cg_solve(Ctx* c, MatView A, const double* b, double* x, double tol,
             double abs_tol, int max_iters, SolveOut* out, const Readback* extra = nullptr);
// true when cg_solve folds x += alpha p into the next pass A (7-point rows)
bool cg_defers_x(const Ctx* c);
// the solvers read stencil codes / run in RCM order (format options)
bool uses_codes(const Ctx* c);
bool uses_rcm(const Ctx* c);
int bicgstab_solve(Ctx* c, MatView A, int ncomp, const double* const* b,
                   double* const* x, double tol, double abs_tol, int max_iters,
                   SolveOut* out, const Readback* extra = nullptr);
std::string solve_error_text(const char* solver, const SolveOut& o, int zero_row);

// team collectives (fvb_team.cu): halo exchange of consecutive pool slots
// and a small allreduce; both are no-ops for a context without a team.
int team_halo(Ctx* c, int first_slot, int nslots);
int team_allreduce(Ctx* c, double* host_vals, int m, int op);
int team_timeout_error(Ctx* c);  // sets the diagnostic error text, returns FVB_E_TIMEOUT

// FV operators on device buffers (fvb_ops.cu); multi-component vectors use
// component stride nc (the pool layout).
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
int op_rhie_chow(Ctx* c, const double* u, const double* ub, const double* p, const double* pb,
                 const double* adiag, const double* gp, const double* d, const double* db,
                 double* flux);
int op_precompute_geometry(Ctx* c, const double* dx, const double* dy,
                           const double* dz, const double* dbx, const double* dby,
                           const double* dbz);

}  // namespace fvb

struct fvb_ctx {
  fvb::Ctx c;
};
