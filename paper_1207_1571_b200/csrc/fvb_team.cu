// Team collectives outside the persistent solvers: halo exchange of cell
// vectors (owned boundary rows -> neighbour ghost slots, stored directly
// into the peer's cell pool over NVLink) and a small deterministic
// allreduce through the peer mailboxes.  The domain decomposition itself
// (which rows send where) is built on the host (decompose.py) and handed
// over by fvb_team_attach.
#include <cstddef>

#include "fvb_internal.cuh"

namespace fvb {

namespace {

constexpr int kThreads = 256;

// One thread per (send row, slot): push the owned value into every ghost
// copy, then fence at system scope so the stores are performed before the
// team sync that follows on the stream.
__global__ void k_halo_push(TeamView T, int nr, int first_slot, int nslots,
                            const double* __restrict__ cells, int nc) {
  const int nsend = nr - T.n_inner;
  const int total = nsend * nslots;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int row = T.n_inner + t % nsend;
    const int s = first_slot + t / nsend;
    halo_send(T, row, s, cells[size_t(s) * nc + row]);
  }
  __threadfence_system();
}

// One thread: exchange up to kMailM doubles with every rank and combine in
// rank order.  err (device word) is set when the watchdog fires.
__global__ void k_team_sync(TeamView T, double* vals, int m, int op, unsigned* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double v[kMailM];
#pragma unroll
  for (int k = 0; k < kMailM; ++k) v[k] = k < m ? vals[k] : 0.0;
  if (!team_exchange<kMailM>(T, v, op)) {
    atomicExch(err, 1u);
    return;
  }
  for (int k = 0; k < m; ++k) vals[k] = v[k];
}

}  // namespace

int team_timeout_error(Ctx* c) {
  unsigned long long d[8] = {0};
  cudaMemcpy(d, reinterpret_cast<const char*>(c->pool) + offsetof(Comm, pad), 7 * sizeof(d[0]),
             cudaMemcpyDeviceToHost);
  unsigned long long seq[kMaxTeam] = {0};
  cudaMemcpy(seq, c->pool, sizeof seq, cudaMemcpyDeviceToHost);
  char peers[256] = {0};
  int o = 0;
  for (int q = 0; q < c->team.size && q < kMaxTeam; ++q)
    o += snprintf(peers + o, sizeof peers - o, "%s%llu", q ? "," : "", seq[q]);
  if (d[6] == kReduceTimeoutMark)
    fvb_set_error("team solver reduction timed out (rank %d of %d): a peer did not arrive "
                  "(waited for %llu block arrivals, saw %llu)", c->team.rank, c->team.size, d[0], d[1]);
  else
    fvb_set_error("team sync timed out (rank %d of %d): a peer did not arrive (waited for epoch "
                  "%llu; peer epochs now %s)", c->team.rank, c->team.size, d[0], peers);
  return FVB_E_TIMEOUT;
}

int team_halo(Ctx* c, int first_slot, int nslots) {
  if (!c->teamed()) return FVB_OK;
  const int nsend = c->nr - c->team.n_inner;
  if (nsend > 0 && nslots > 0) {
    k_halo_push<<<grid_for(int64_t(nsend) * nslots, kThreads), kThreads, 0, c->stream>>>(
        c->team, c->nr, first_slot, nslots, c->cells, c->nc);
    note_launch();
    FVB_CUDA(cudaGetLastError());
  }
  // zero-payload sync: every rank's pushes are complete before anyone reads
  double* dv = c->partials + 16 * 4096 + 64;
  k_team_sync<<<1, 32, 0, c->stream>>>(c->team, dv, 0, RED_SUM, c->sync + 3);
  note_launch();
  FVB_CUDA(cudaGetLastError());
  return FVB_OK;
}

int team_allreduce(Ctx* c, double* host_vals, int m, int op) {
  if (!c->teamed()) return FVB_OK;
  if (m < 1 || m > kMailM) {
    fvb_set_error("team allreduce of %d values (max %d)", m, kMailM);
    return FVB_E_ARG;
  }
  double* dv = c->partials + 16 * 4096 + 64;
  FVB_CUDA(cudaMemcpyAsync(dv, host_vals, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
  k_team_sync<<<1, 32, 0, c->stream>>>(c->team, dv, m, op, c->sync + 3);
  note_launch();
  FVB_CUDA(cudaGetLastError());
  unsigned err = 0;
  FVB_CUDA(cudaMemcpyAsync(host_vals, dv, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
  FVB_CUDA(cudaMemcpyAsync(&err, c->sync + 3, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  FVB_CUDA(cudaStreamSynchronize(c->stream));
  if (err) return team_timeout_error(c);
  return FVB_OK;
}

}  // namespace fvb
