// f2v_shard.cu -- the vertex-partitioned multi-GPU run.
//
// One process per GPU.  Every GPU holds a full replica of Z (Zold + Znew,
// the epoch kernel's double buffer) and runs the dataflow epoch kernel over
// the positions of its own rows; the kernel's finalise stores each new row
// into the local Znew AND into every peer's Znew through CUDA IPC mappings
// over NVLink (f2v_epoch.cuh finalize), so the all-gather of updated rows is
// fused into the update epilogue, row by row, overlapped with the compute.
// Readers on any GPU poll the row's sentinel in their local replica exactly as
// on one GPU.  The only synchronisation outside the kernel is two device-side
// barriers per epoch over a small IPC-shared control block: after the sentinel
// fill (no peer may store a row into a replica before it is reset) and after
// the kernel (every replica complete; first failure and loss exchanged).
#include <cstring>

#include "f2v_epoch.cuh"

namespace f2v {

struct ShardCtl {
  unsigned long long barrier;                // arrivals (every rank adds 1 per barrier)
  unsigned long long bad[ep::kMaxShards];    // first failing combined position per rank
  double loss[ep::kMaxShards];               // epoch loss partial per rank
  unsigned int timeout;                      // set when a barrier waited > 60 s
};

struct CtlPtrs {
  ShardCtl* p[ep::kMaxShards];  // p[rank] = the local block
};

namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void barrier_kernel(CtlPtrs peers, uint32_t world, uint32_t rank,
                               unsigned long long target) {
  __threadfence_system();  // this GPU's row stores are visible before the arrival
  for (uint32_t g = 0; g < world; ++g) atomicAdd_system(&peers.p[g]->barrier, 1ull);
  ShardCtl* me = peers.p[rank];
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  while (ld_acquire_sys(&me->barrier) < target) {
    __nanosleep(200);
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
    if (now - t0 > 60000000000ull) {  // a peer is gone: report instead of hanging
      me->timeout = 1u;
      break;
    }
  }
}

__global__ void publish_kernel(CtlPtrs peers, uint32_t world, uint32_t rank,
                               unsigned long long bad, double loss) {
  for (uint32_t g = 0; g < world; ++g) {
    peers.p[g]->bad[rank] = bad;
    peers.p[g]->loss[rank] = loss;
  }
  __threadfence_system();
}

CtlPtrs ctl_ptrs(const Ctx& c) {
  CtlPtrs p{};
  for (uint32_t g = 0; g < c.world; ++g)
    p.p[g] = int32_t(g) == c.rank ? c.ctl.as<ShardCtl>() : static_cast<ShardCtl*>(c.peer_ctl[g]);
  return p;
}

}  // namespace

void k_shard_barrier(Ctx& c) {
  ++c.barriers;
  barrier_kernel<<<1, 1, 0, c.stream>>>(ctl_ptrs(c), c.world, uint32_t(c.rank),
                                        c.barriers * c.world);
  F2V_LAUNCHED(c.stream, "barrier_kernel");
  ++c.launches;
  unsigned int to = 0;
  F2V_CUDA(cudaMemcpyAsync(&to, &c.ctl.as<ShardCtl>()->timeout, sizeof(to),
                           cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  if (to) fail(F2V_ECUDA, "shard barrier timed out (a peer GPU stopped)");
}

void k_shard_publish(Ctx& c, uint64_t bad, double loss) {
  publish_kernel<<<1, 1, 0, c.stream>>>(ctl_ptrs(c), c.world, uint32_t(c.rank), bad, loss);
  F2V_LAUNCHED(c.stream, "publish_kernel");
  ++c.launches;
}

void k_shard_collect(Ctx& c, uint64_t& bad, double& loss) {
  ShardCtl h;
  F2V_CUDA(cudaMemcpyAsync(&h, c.ctl.p, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  bad = ~0ull;
  loss = 0.0;
  for (uint32_t g = 0; g < c.world; ++g) {  // rank order: the same sum on every rank
    bad = std::min<uint64_t>(bad, h.bad[g]);
    loss += h.loss[g];
  }
}

size_t shard_ctl_bytes() { return sizeof(ShardCtl); }

// rows of Z by id (the per-step all-gather driver's pack / unpack, dist.py)
__global__ void rows_kernel(float* __restrict__ z, const uint32_t* __restrict__ ids, uint32_t b,
                            uint32_t d, float* __restrict__ rows, int to_z) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= uint64_t(b) * d) return;
  const uint64_t i = t / d, k = t % d;
  float* zr = z + size_t(ids[i]) * d + k;
  if (to_z) *zr = rows[t];
  else rows[t] = *zr;
}

void k_rows(Ctx& c, uint32_t b, float* rows_dev, bool to_z) {
  const uint64_t tot = uint64_t(b) * c.d;
  if (!tot) return;
  rows_kernel<<<uint32_t((tot + 255) / 256), 256, 0, c.stream>>>(c.zcur(), c.ids.as<uint32_t>(), b,
                                                                c.d, rows_dev, to_z ? 1 : 0);
  F2V_LAUNCHED(c.stream, "rows_kernel");
  ++c.launches;
}

}  // namespace f2v
