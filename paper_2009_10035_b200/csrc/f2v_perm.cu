// f2v_perm.cu -- partition_epoch's Fisher-Yates shuffle (sampling.cpp:7-19)
// on the device, bit-identical to the sequential reference.
//
// The reference performs, for m = n-1 down to 1, swap(A[m], A[J_m]) with
// J_m = below(m + 1) from draw number n-1-m of the keyed SplitMix stream
// (seed, {0x22, epoch}).  Every J_m is known up front (counter-based stream),
// so the swaps can run as "deterministic reservations" (Shun, Gu, Blelloch,
// Fineman, Gibbons, SODA'15): in each round every pending step m reserves
// both positions it touches with priority m (an atomicMax of a round-stamped
// key); a step whose reservations both survive commits its swap.  A step
// commits only when every earlier (larger-m) step touching its positions has
// committed, and steps committing in one round touch disjoint positions, so
// each swap sees exactly the array state the sequential loop gives it.  The
// dependence depth is O(log n) w.h.p.; the rounds run inside one cooperative
// kernel with a grid barrier between the reserve and commit phases.
#include <cooperative_groups.h>

#include <algorithm>

#include "f2v_internal.h"
#include "f2v_rng.h"

namespace cg = cooperative_groups;

namespace f2v {
namespace {

struct ShuffleArgs {
  uint32_t* A;                 // the permutation, initialised to iota
  unsigned long long* R;       // reservations, zeroed
  uint32_t* list[2];           // pending step lists (ping-pong)
  uint32_t* count;             // [0], [1]: pending counts; [2] rounds used
  uint32_t n;
  uint64_t s0;                 // keyed stream state
};

__device__ __forceinline__ uint32_t target(const ShuffleArgs& a, uint32_t m) {
  return uint32_t(rng_below(rng_draw(a.s0, uint64_t(a.n) - 1 - m), uint64_t(m) + 1));
}

__global__ void shuffle_kernel(ShuffleArgs a) {
  cg::grid_group grid = cg::this_grid();
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  // init: A = iota, R = 0, all steps m in [1, n) pending
  for (uint64_t i = tid; i < a.n; i += stride) {
    __stcg(a.A + i, uint32_t(i));
    __stcg(a.R + i, 0ull);
    if (i >= 1) __stcg(a.list[0] + i - 1, uint32_t(i));
  }
  if (tid == 0) {
    a.count[0] = a.n > 0 ? a.n - 1 : 0;
    a.count[1] = 0;
  }
  grid.sync();
  uint32_t round = 1;
  int cur = 0;
  while (true) {
    const uint32_t pending = __ldcg(a.count + cur);
    if (pending == 0) break;
    const unsigned long long stamp = (unsigned long long)round << 32;
    for (uint64_t t = tid; t < pending; t += stride) {  // reserve
      const uint32_t m = __ldcg(a.list[cur] + t);
      const uint32_t J = target(a, m);
      atomicMax(a.R + m, stamp | m);
      if (J != m) atomicMax(a.R + J, stamp | m);
    }
    if (tid == 0) a.count[cur ^ 1] = 0;
    grid.sync();
    for (uint64_t t = tid; t < pending; t += stride) {  // commit or defer
      const uint32_t m = __ldcg(a.list[cur] + t);
      const uint32_t J = target(a, m);
      const unsigned long long key = stamp | m;
      if (__ldcg(a.R + m) == key && __ldcg(a.R + J) == key) {
        const uint32_t x = __ldcg(a.A + m);
        __stcg(a.A + m, __ldcg(a.A + J));
        __stcg(a.A + J, x);
      } else {
        __stcg(a.list[cur ^ 1] + atomicAdd(a.count + (cur ^ 1), 1u), m);
      }
    }
    grid.sync();
    cur ^= 1;
    ++round;
  }
  if (tid == 0) a.count[2] = round - 1;
}

}  // namespace

// perm_out (device, n entries) = partition_epoch(n, b, Rng::keyed(seed, {0x22, epoch})).perm
void k_device_partition(Ctx& c, uint32_t n, uint64_t seed, uint32_t epoch, uint32_t* perm_out) {
  c.shufR.ensure(sizeof(unsigned long long) * std::max<uint32_t>(n, 1));
  c.shufL.ensure(sizeof(uint32_t) * 2 * std::max<uint32_t>(n, 1));
  c.shufC.ensure(sizeof(uint32_t) * 4);
  ShuffleArgs a;
  a.A = perm_out;
  a.R = c.shufR.as<unsigned long long>();
  a.list[0] = c.shufL.as<uint32_t>();
  a.list[1] = c.shufL.as<uint32_t>() + std::max<uint32_t>(n, 1);
  a.count = c.shufC.as<uint32_t>();
  a.n = n;
  a.s0 = rng_keyed2(seed, kStreamPartition, epoch);
  int per_sm = 0;
  F2V_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, shuffle_kernel, 256, 0));
  const int blocks = std::max(1, per_sm) * c.num_sms;
  void* args[] = {&a};
  F2V_CUDA(cudaLaunchCooperativeKernel((void*)shuffle_kernel, blocks, 256, args, 0, c.stream));
  F2V_LAUNCHED(c.stream, "shuffle_kernel");
  ++c.launches;
}

}  // namespace f2v
