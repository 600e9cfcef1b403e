// Grid-reduction latency probe (diagnostic, not the product): one
// cooperatively launched grid of one 1024-thread block per SM runs R
// reductions of M = 2 doubles per thread, with the single-device barrier
// forms below; prints microseconds per reduction.
//   A  every block polls a monotonic counter, then sums all block partials
//      (the product's team_reduce single-device path)
//   B  A without the nanosleep back-off in the poll
//   C  A on clusters of 2 CTAs: the pair combines over DSMEM first, one
//      arrival and one partial per pair
//   D  last arriver sums and publishes; the others poll a generation word
//   E  A without the block reduction (thread 0's own value is the partial)
//   F  E without the partial sums (the barrier alone)
//   H  A with every partial load of both values issued before the sums
//   I  A with the partial loads k-outer / value-inner over a fixed 16-step
//      lane stride (predicated), accumulated in the same order
//   J  I with one warp per value (warp m sums value m)
//   G  per-block round tags instead of one counter: each block stores its
//      partials and then its tag (release); warp 0 of every block polls the
//      tags lane-strided, fences, and sums the partials (no atomics)
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int M = 2;
__device__ __forceinline__ void block_reduce(double (&v)[M], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int m = 0; m < M; ++m)
    for (int o = 16; o > 0; o >>= 1) v[m] += __shfl_down_sync(0xffffffffu, v[m], o);
  if (lane == 0)
    for (int m = 0; m < M; ++m) sm[warp * M + m] = v[m];
  __syncthreads();
  if (warp == 0)
    for (int m = 0; m < M; ++m) {
      double x = lane < nw ? sm[lane * M + m] : 0.0;
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      v[m] = x;
    }
  __syncthreads();
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int VAR>
__global__ void __launch_bounds__(1024, 1) k_probe(int rounds, unsigned* ctr, double* part, double* out) {
  __shared__ double sm[32 * M + M];
  __shared__ double s_pair[2][M];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int G = gridDim.x, me = blockIdx.x;
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    double v[M] = {1.0 + threadIdx.x, 2.0};
    if (VAR < 4) block_reduce(v, sm);
    if (VAR == 2) {
      cg::cluster_group cl = cg::this_cluster();
      if (threadIdx.x == 0)
        for (int m = 0; m < M; ++m) s_pair[r & 1][m] = v[m];
      cl.sync();
      if (threadIdx.x == 0 && cl.block_rank() == 0)
        for (int m = 0; m < M; ++m) v[m] += cl.map_shared_rank(&s_pair[r & 1][0], 1)[m];
      G = gridDim.x / 2;
      me = blockIdx.x / 2;
    }
    double* pp = part + size_t(r & 1) * 16 * 2048;
    if (VAR == 3) {
      __shared__ int s_last;
      __shared__ unsigned s_gen;
      if (threadIdx.x == 0) {
        s_gen = ld_relaxed(ctr + 1);
        for (int m = 0; m < M; ++m) pp[m * G + me] = v[m];
        unsigned o;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(o) : "l"(ctr) : "memory");
        s_last = o == unsigned(G) - 1;
      }
      __syncthreads();
      if (s_last) {
        if (warp == 0) {
          for (int m = 0; m < M; ++m) {
            double x = 0.0;
            for (int b = lane; b < G; b += 32) x += __ldcg(pp + m * G + b);
            for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
            if (lane == 0) __stcg(out + 8 + m, x);
          }
          if (lane == 0) {
            ctr[0] = 0;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + 1) : "memory");
          }
        }
      } else if (threadIdx.x == 0) {
        while (ld_relaxed(ctr + 1) == s_gen) {}
      }
      if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int m = 0; m < M; ++m) sm[32 * M + m] = __ldcg(out + 8 + m);
      }
      __syncthreads();
      acc += sm[32 * M];
      __syncthreads();
      continue;
    }
    if (VAR == 6) {
      unsigned* tag = ctr + 64;  // [blocks]
      if (threadIdx.x == 0) {
        for (int m = 0; m < M; ++m) pp[m * G + me] = v[m];
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(tag + me), "r"(unsigned(r + 1)) : "memory");
      }
      if (warp == 0) {
        for (int b = lane; b < G; b += 32)
          while (ld_relaxed(tag + b) < unsigned(r + 1)) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int m = 0; m < M; ++m) {
          double x = 0.0;
          for (int b = lane; b < G; b += 32) x += __ldcg(pp + m * G + b);
          for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
          if (lane == 0) sm[32 * M + m] = x;
        }
      }
      __syncthreads();
      acc += sm[32 * M];
      __syncthreads();
      continue;
    }
    const bool writer = VAR != 2 || cg::this_cluster().block_rank() == 0;
    if (threadIdx.x == 0) {
      if (writer) {
        for (int m = 0; m < M; ++m) pp[m * G + me] = v[m];
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      }
      const unsigned target = unsigned(r + 1) * unsigned(G);
      int spins = 0;
      while (ld_relaxed(ctr) < target) {
        if (VAR != 1 && ++spins > 64) __nanosleep(32);
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    if (VAR == 7 && warp == 0) {
      constexpr int NB = 5;  // ceil(148 / 32)
      double xs[M][NB];
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          const int b = lane + 32 * k;
          xs[m][k] = b < G ? __ldcg(pp + m * G + b) : 0.0;
        }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double x = 0.0;
#pragma unroll
        for (int k = 0; k < NB; ++k) x += xs[m][k];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) sm[32 * M + m] = x;
      }
    } else if (VAR == 8 && warp == 0) {
      double xm[M];
#pragma unroll
      for (int m = 0; m < M; ++m) xm[m] = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int b = lane + 32 * k;
        if (b < G) {
#pragma unroll
          for (int m = 0; m < M; ++m) xm[m] += __ldcg(pp + m * G + b);
        }
      }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double x = xm[m];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) sm[32 * M + m] = x;
      }
    } else if (VAR == 9) {
      if (warp < M) {
        double x = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int b = lane + 32 * k;
          if (b < G) x += __ldcg(pp + warp * G + b);
        }
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) sm[32 * M + warp] = x;
      }
    } else if (VAR != 5 && warp == 0)
      for (int m = 0; m < M; ++m) {
        double x = 0.0;
        for (int b = lane; b < G; b += 32) x += __ldcg(pp + m * G + b);
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) sm[32 * M + m] = x;
      }
    __syncthreads();
    acc += sm[32 * M];
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

template <int VAR>
float run(int blocks, int rounds, unsigned* ctr, double* part, double* out) {
  cudaMemset(ctr, 0, 64 * 4 + 4 * 4096);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(1024);
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  ++na;
  if (VAR == 2) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_probe<VAR>, rounds, ctr, part, out);
  cudaEventRecord(e1);
  cudaError_t e2 = cudaEventSynchronize(e1);
  float ms = -1.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (e != cudaSuccess || e2 != cudaSuccess)
    printf("  variant %d: %s / %s\n", VAR, cudaGetErrorString(e), cudaGetErrorString(e2));
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* ctr;
  double *part, *out;
  cudaMalloc(&ctr, 64 * 4 + 4 * 4096);
  cudaMalloc(&part, sizeof(double) * 2 * 16 * 2048);
  cudaMalloc(&out, 64 * sizeof(double));
  const int R = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    printf("blocks %d rounds %d (us per reduction): A %.3f  B %.3f  C %.3f  D %.3f  E %.3f  F %.3f  G %.3f  H %.3f  I %.3f  J %.3f\n", sms, R,
           1e3f * run<0>(sms, R, ctr, part, out) / R, 1e3f * run<1>(sms, R, ctr, part, out) / R,
           1e3f * run<2>(sms & ~1, R, ctr, part, out) / R, 1e3f * run<3>(sms, R, ctr, part, out) / R,
           1e3f * run<4>(sms, R, ctr, part, out) / R, 1e3f * run<5>(sms, R, ctr, part, out) / R,
           1e3f * run<6>(sms, R, ctr, part, out) / R, 1e3f * run<7>(sms, R, ctr, part, out) / R,
           1e3f * run<8>(sms, R, ctr, part, out) / R, 1e3f * run<9>(sms, R, ctr, part, out) / R);
  }
  return 0;
}
