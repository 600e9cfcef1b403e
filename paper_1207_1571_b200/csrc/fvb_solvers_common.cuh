// Shared by the persistent Krylov solver units (fvb_cg.cu, fvb_bicgstab.cu):
// solver constants, the zero-diagonal exit, streamed loads and the launch
// helpers (cooperative grid, one thread-block cluster, one shared-memory
// block).  Split from one unit so the two solvers' many kernel
// instantiations compile in parallel.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "fvb_internal.cuh"

namespace fvb {

namespace {

constexpr int kSolverThreads = 512;
constexpr double kResFloor = 1e-30;   // linsolve.py:20
constexpr double kTiny = 1e-300;      // linsolve.py:21


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


// dynamic shared memory of the SMEM solver kernels for n rows (0 = too large)
inline size_t smem_cg_bytes(int n, int k) {
  return size_t(6 + k) * n * sizeof(double) + size_t(n) + 16;
}
inline size_t smem_bi_bytes(int n, int nc, int k) {
  return size_t(7 * nc + 1 + k) * n * sizeof(double) + size_t(n) + 16;
}
constexpr size_t kSmemSolverMax = 200 * 1024;

template <typename K, typename Args>
int smem_launch(Ctx* c, K kernel, Args& args, int threads, size_t bytes, int blocks = 1) {
  FVB_CUDA(cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(bytes)));
  FVB_CUDA(cudaMemsetAsync(c->sync, 0, 3 * sizeof(unsigned), c->stream));
  // one row per thread: fewer warps make the block barriers of the tiny
  // solves cheaper (rounded to whole warps pairs, at most `threads`)
#ifndef FVB_DIAG_SMEM_ROWS  // diagnostic builds: rows per thread
#define FVB_DIAG_SMEM_ROWS 1
#endif
  const int t = std::min(threads, std::max(64, (c->nr / FVB_DIAG_SMEM_ROWS + 63) / 64 * 64));
  void* params[] = {&args};
  fvb::note_launch();
  FVB_CUDA(cudaLaunchKernel((const void*)kernel, dim3(blocks), dim3(t), params, bytes, c->stream));
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
  if (c->teamed() && b > kTeamGridMax) b = kTeamGridMax;  // team-partials buffer (team_reduce)
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
#ifdef FVB_DIAG_CLUSTER  // diagnostic builds: cluster size
  return FVB_DIAG_CLUSTER;
#endif
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

}  // namespace fvb
