// f2v_perm.cu -- partition_epoch's Fisher-Yates shuffle (sampling.cpp:7-19)
// on the device, bit-identical to the sequential reference.
//
// The reference performs, for m = n-1 down to 1, swap(A[m], A[J_m]) with
// J_m = below(m + 1) from draw number n-1-m of the keyed SplitMix stream
// (seed, {0x22, epoch}).  Every J_m is known up front (counter-based stream),
// so the final array has a closed form:
//   position m is final right after step m, so A[m] = V(J_m, m), the value at
//   position J_m just before step m.  That position was last written by the
//   smallest step m' > m with J_m' = J_m (which moved in W(m'), the value at
//   position m' just before step m'), or never (value J_m).  Likewise
//   W(m) = W(next(m)) with next(m) = the smallest step m'' > m targeting m,
//   and W(m) = m when there is none.
// Steps are grouped by target with a stable radix sort of (J_m, m); the W
// chains (strictly increasing step indices, expected length ~ln n) are
// followed to their roots.  O(n log n) work, a handful of passes.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "f2v_internal.h"
#include "f2v_rng.h"

namespace f2v {
namespace {

constexpr uint32_t kNone = 0xffffffffu;

__global__ void targets_kernel(uint32_t* __restrict__ key, uint32_t* __restrict__ val, uint32_t n,
                               uint64_t s0) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // step m = i + 1
  if (i + 1 >= n) return;
  const uint32_t m = i + 1;
  key[i] = uint32_t(rng_below(rng_draw(s0, uint64_t(n) - 1 - m), uint64_t(m) + 1));
  val[i] = m;
}

// sorted (J, m): successor of m inside its target group, first step of each group
__global__ void groups_kernel(const uint32_t* __restrict__ ks, const uint32_t* __restrict__ vs,
                              uint32_t N, uint32_t* __restrict__ succ,
                              uint32_t* __restrict__ first) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const uint32_t key = ks[k], m = vs[k];
  succ[m] = (k + 1 < N && ks[k + 1] == key) ? vs[k + 1] : kNone;
  if (k == 0 || ks[k - 1] != key) first[key] = m;
}

// next(m): the smallest step > m targeting m (root: itself)
__global__ void next_kernel(const uint32_t* __restrict__ succ, const uint32_t* __restrict__ first,
                            uint32_t* __restrict__ ptr, uint32_t n) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  if (m == 0) {
    ptr[0] = 0;
    return;
  }
  uint32_t f = first[m];
  if (f == m) f = succ[m];  // J_m == m: skip the self-target
  ptr[m] = f == kNone ? m : f;
}

// W(m): follow next() to the chain's root (chains are short: E[length] ~ ln n)
__global__ void root_kernel(const uint32_t* __restrict__ ptr, uint32_t* __restrict__ W,
                            uint32_t n) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  uint32_t x = m, y = ptr[m];
  while (y != x) {
    x = y;
    y = ptr[x];
  }
  W[m] = x;
}

__global__ void final_kernel(const uint32_t* __restrict__ succ, const uint32_t* __restrict__ first,
                             const uint32_t* __restrict__ W, uint32_t* __restrict__ A, uint32_t n,
                             uint64_t s0) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  if (m == 0) {
    const uint32_t f = first[0];
    A[0] = f == kNone ? 0u : W[f];
    return;
  }
  const uint32_t s = succ[m];
  A[m] = s != kNone ? W[s]
                    : uint32_t(rng_below(rng_draw(s0, uint64_t(n) - 1 - m), uint64_t(m) + 1));
}

}  // namespace

// perm_out (device, n entries) = partition_epoch(n, b, Rng::keyed(seed, {0x22, epoch})).perm
void k_device_partition(Ctx& c, uint32_t n, uint64_t seed, uint32_t epoch, uint32_t* perm_out) {
  k_device_partition_keyed(c, n, rng_keyed2(seed, kStreamPartition, epoch), perm_out);
}

// the same shuffle of n elements from a stream whose initial state is s0
void k_device_partition_keyed(Ctx& c, uint32_t n, uint64_t s0, uint32_t* perm_out) {
  if (n == 0) return;
  const uint32_t N = n - 1;  // steps m = 1 .. n-1
  const size_t nn = std::max<uint32_t>(n, 1);
  c.shufL.ensure(sizeof(uint32_t) * nn * 8);
  uint32_t* key = c.shufL.as<uint32_t>();
  uint32_t* val = key + nn;
  uint32_t* ks = val + nn;
  uint32_t* vs = ks + nn;
  uint32_t* succ = vs + nn;
  uint32_t* first = succ + nn;
  uint32_t* p0 = first + nn;
  uint32_t* p1 = p0 + nn;
  const uint32_t g = (n + 255) / 256;
  F2V_CUDA(cudaMemsetAsync(first, 0xff, sizeof(uint32_t) * n, c.stream));
  if (N) {
    targets_kernel<<<g, 256, 0, c.stream>>>(key, val, n, s0);
    F2V_LAUNCHED(c.stream, "targets_kernel");
    int bits = 1;
    while (bits < 32 && (uint64_t(1) << bits) < n) ++bits;
    size_t tmp = 0;
    F2V_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, ks, val, vs, N, 0, bits,
                                             c.stream));
    c.shufR.ensure(tmp);
    F2V_CUDA(cub::DeviceRadixSort::SortPairs(c.shufR.p, tmp, key, ks, val, vs, N, 0, bits,
                                             c.stream));
    groups_kernel<<<(N + 255) / 256, 256, 0, c.stream>>>(ks, vs, N, succ, first);
    F2V_LAUNCHED(c.stream, "groups_kernel");
  }
  next_kernel<<<g, 256, 0, c.stream>>>(succ, first, p0, n);
  F2V_LAUNCHED(c.stream, "next_kernel");
  root_kernel<<<g, 256, 0, c.stream>>>(p0, p1, n);
  F2V_LAUNCHED(c.stream, "root_kernel");
  final_kernel<<<g, 256, 0, c.stream>>>(succ, first, p1, perm_out, n, s0);
  F2V_LAUNCHED(c.stream, "final_kernel");
  c.launches += 6;
}

}  // namespace f2v
