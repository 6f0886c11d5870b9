// f2v_walk.cu -- walk mode (rForce2Vec; SampleMode::walk(k), sampling.hpp:12-20)
// on the device.
//
// In walk mode the context of a batch vertex u is a k-step random walk from u
// (gen_walk, sampling.cpp:27-41: one below() per step, a dead end restarts at
// u, an isolated u has no walk), drawn on its batch's stream
// (seed, {0x33, epoch, batch}) BEFORE the batch's negatives
// (build_minibatch, sampling.cpp:43-61).  Every non-isolated vertex draws
// exactly k numbers, so vertex i of a batch starts at draw k * (non-isolated
// vertices before it in the batch): the walks of an epoch are generated in
// parallel, one thread per vertex, straight into a "context CSR" (row u = the
// walk of u, k entries; static layout), and the unchanged dataflow epoch
// kernel runs on that CSR instead of the graph's.  The graph CSR is parked in
// Ctx::grow / gcol while a walk context is active.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <utility>

#include "f2v_epoch.cuh"

namespace f2v {
namespace {

struct ShardBounds {
  uint32_t lo[ep::kMaxShards + 1];
};

// flag[p] = the vertex at combined position p has a walk (degree > 0)
__global__ void walkable_kernel(const uint32_t* __restrict__ perm,
                                const uint64_t* __restrict__ grow, uint32_t* __restrict__ flag,
                                uint32_t n) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  flag[p] = p < n && grow[perm[p] + 1] > grow[perm[p]] ? 1u : 0u;
}

__global__ void walk_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ state,
                            const uint32_t* __restrict__ wpos, const uint32_t* __restrict__ poff,
                            const uint64_t* __restrict__ grow, const uint32_t* __restrict__ gcol,
                            const uint64_t* __restrict__ crow, uint32_t* __restrict__ ccol,
                            uint32_t n, ShardBounds sb, uint32_t G, uint32_t k, uint64_t seed,
                            uint32_t epoch) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t u = perm[p];
  const uint64_t d0 = grow[u + 1] - grow[u];
  if (d0 == 0) return;  // isolated start: empty walk
  const uint32_t t = state[u] >> 1;
  const uint32_t g = ep::shard_of(u, sb.lo, G);
  const uint64_t s0 = G == 1 ? rng_keyed3(seed, kStreamSampling, epoch, t)
                             : rng_keyed4(seed, kStreamSampling, epoch, t, g);
  const uint64_t base = uint64_t(k) * (wpos[p] - wpos[poff[uint64_t(t) * G + g]]);
  uint32_t* out = ccol + crow[u];
  uint32_t w = u;
  for (uint32_t i = 0; i < k; ++i) {
    uint64_t dw = grow[w + 1] - grow[w];
    if (dw == 0) {  // dead end: restart
      w = u;
      dw = d0;
    }
    const uint32_t next = gcol[grow[w] + rng_below(rng_draw(s0, base + i), dw)];
    out[i] = next;
    w = next;
  }
}

}  // namespace

// Make the context CSR the one-hop graph (k = 0) or the k-step walk layout.
void k_set_context(Ctx& c, uint32_t k) {
  if (k == c.walk_k) return;
  if (c.walk_k) {  // back to the graph
    std::swap(c.rowptr, c.grow);
    std::swap(c.col, c.gcol);
    std::swap(c.h_rowptr, c.h_growptr);
    c.nnz = c.gnnz;
    c.grow.release();
    c.gcol.release();
    c.h_growptr.clear();
    c.walk_k = 0;
  }
  if (k) {
    std::swap(c.rowptr, c.grow);
    std::swap(c.col, c.gcol);
    std::swap(c.h_rowptr, c.h_growptr);
    c.gnnz = c.nnz;
    c.h_rowptr.assign(size_t(c.n) + 1, 0);
    for (uint32_t u = 0; u < c.n; ++u)
      c.h_rowptr[u + 1] = c.h_rowptr[u] + (c.h_growptr[u + 1] > c.h_growptr[u] ? k : 0);
    c.nnz = c.h_rowptr[c.n];
    c.rowptr.ensure(sizeof(uint64_t) * (size_t(c.n) + 1));
    c.col.ensure(sizeof(uint32_t) * std::max<uint64_t>(c.nnz, 1));
    F2V_CUDA(cudaMemcpyAsync(c.rowptr.p, c.h_rowptr.data(), sizeof(uint64_t) * (c.n + 1),
                             cudaMemcpyHostToDevice, c.stream));
    c.walk_k = k;
  }
  k_prepare_graph(c);  // chunk layout of the new context
}

// The walks of every batch of this epoch (after k_epoch_perm) into the
// context CSR, and the per-position walk counts the negatives need.
void k_epoch_walks(Ctx& c, uint32_t epoch, uint64_t seed) {
  const uint32_t n = c.n;
  c.wflag.ensure(sizeof(uint32_t) * (size_t(n) + 1));
  c.wpos.ensure(sizeof(uint32_t) * (size_t(n) + 1));
  walkable_kernel<<<(n + 1 + 255) / 256, 256, 0, c.stream>>>(
      c.perm.as<uint32_t>(), c.grow.as<uint64_t>(), c.wflag.as<uint32_t>(), n);
  F2V_LAUNCHED(c.stream, "walkable_kernel");
  size_t tmp = 0;
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.wflag.as<uint32_t>(),
                                         c.wpos.as<uint32_t>(), n + 1, c.stream));
  c.scan_tmp.ensure(tmp);
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp, c.wflag.as<uint32_t>(),
                                         c.wpos.as<uint32_t>(), n + 1, c.stream));
  ShardBounds bounds{};
  for (uint32_t g = 0; g <= c.shards; ++g) bounds.lo[g] = c.sh_lo[g];
  walk_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(
      c.perm.as<uint32_t>(), c.state.as<uint32_t>(), c.wpos.as<uint32_t>(),
      c.poff.as<uint32_t>(), c.grow.as<uint64_t>(), c.gcol.as<uint32_t>(),
      c.rowptr.as<uint64_t>(), c.col.as<uint32_t>(), n, bounds, c.shards, c.walk_k, seed, epoch);
  F2V_LAUNCHED(c.stream, "walk_kernel");
  c.launches += 3;
}

}  // namespace f2v
