// f2v_csr.cu -- CsrGraph::from_edges (csr_graph.cpp:57-97) on the device
// (SURVEY.md section 8(f) row 2): the canonical CSR of an edge list -- drop
// self-loops (counted), optionally add every reversed arc, sort, unique, count
// per row, prefix -- byte-identical to the reference's, for the multi-billion-
// arc configs whose host build takes minutes (C5: 2.1B arcs).
//
//   1. emit:  one 64-bit key (u << 32 | v) per arc (two when symmetrising);
//             a self-loop emits the key ~0 (sorts last, removed at the end);
//   2. CUB radix sort of the keys over the bits the ids need;
//   3. CUB unique (the reference's std::unique): the duplicate count;
//   4. row offsets from the sorted keys by boundary detection (no atomics):
//      the thread at the first arc of row u writes rowptr[r] for the empty
//      rows before it and for u itself; col = the low 32 bits.
// An arc with an endpoint >= n raises RangeError, as the reference does after
// its dedup (the loop test comes first in both).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>

#include "f2v_internal.h"

namespace f2v {
namespace {

constexpr uint64_t kLoopKey = ~0ull;

__global__ void emit_arcs_kernel(const uint32_t* __restrict__ pairs, uint64_t m, uint32_t n,
                                 int sym, uint64_t* __restrict__ keys,
                                 unsigned long long* __restrict__ stats /* loops, range */) {
  unsigned long long loops = 0, range = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    uint64_t k0 = (uint64_t(u) << 32) | v, k1 = (uint64_t(v) << 32) | u;
    if (u == v) {
      ++loops;
      k0 = k1 = kLoopKey;
    } else if (u >= n || v >= n) {
      ++range;
    }
    if (sym) {
      keys[2 * i] = k0;
      keys[2 * i + 1] = k1;
    } else {
      keys[i] = k0;
    }
  }
  if (loops) atomicAdd(stats, loops);
  if (range) atomicAdd(stats + 1, range);
}

// rowptr[r] for r in (row(i-1), row(i)] at each row start i, and the tail
__global__ void row_offsets_kernel(const uint64_t* __restrict__ keys, uint64_t nnz, uint32_t n,
                                   uint64_t* __restrict__ rowptr, uint32_t* __restrict__ col) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= nnz;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t u = i < nnz ? keys[i] >> 32 : uint64_t(n);  // row n = "after the last"
    const uint64_t up = i ? keys[i - 1] >> 32 : ~0ull;         // ~0: before row 0
    if (i < nnz) col[i] = uint32_t(keys[i]);
    if (i == 0 || u != up)
      for (uint64_t r = (i == 0 ? 0 : up + 1); r <= u && r <= n; ++r) rowptr[r] = i;
  }
}

int bits_for(uint32_t n) {
  int b = 1;
  while (b < 32 && (uint64_t(1) << b) < uint64_t(n)) ++b;
  return b;
}

}  // namespace

// The CSR of pairs[0..2m) on the device: row offsets / column indices left in
// rowptr_dev / col_dev (sized by the callee), counts on the host.
void device_csr_from_edges(cudaStream_t st, int num_sms, const uint32_t* pairs_host, uint64_t m,
                           uint32_t n, bool symmetrize, DeviceBuf& rowptr_dev, DeviceBuf& col_dev,
                           uint64_t* nnz_out, uint64_t* dups_out, uint64_t* loops_out) {
  const uint64_t total = symmetrize ? 2 * m : m;
  DeviceBuf pairs, keys, alt, tmp, stats;
  pairs.ensure(sizeof(uint32_t) * std::max<uint64_t>(2 * m, 2));
  keys.ensure(sizeof(uint64_t) * std::max<uint64_t>(total, 1));
  alt.ensure(sizeof(uint64_t) * std::max<uint64_t>(total, 1));
  stats.ensure(64);
  F2V_CUDA(cudaMemsetAsync(stats.p, 0, 64, st));
  if (m)
    F2V_CUDA(cudaMemcpyAsync(pairs.p, pairs_host, sizeof(uint32_t) * 2 * m, cudaMemcpyHostToDevice,
                             st));
  const uint32_t grid = uint32_t(std::max<uint64_t>(
      1, std::min<uint64_t>((m + 255) / 256, uint64_t(num_sms) * 16)));
  emit_arcs_kernel<<<grid, 256, 0, st>>>(pairs.as<uint32_t>(), m, n, symmetrize ? 1 : 0,
                                         keys.as<uint64_t>(), stats.as<unsigned long long>());
  F2V_LAUNCHED(st, "emit_arcs_kernel");
  pairs.release();
  // sort over the id bits (the loop key ~0 has every bit set: still last)
  const int bits = 32 + bits_for(n);
  size_t tb = 0;
  F2V_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<uint64_t>(), alt.as<uint64_t>(),
                                          total, 0, bits, st));
  tmp.ensure(tb);
  F2V_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.as<uint64_t>(), alt.as<uint64_t>(),
                                          total, 0, bits, st));
  // unique (std::unique, csr_graph.cpp:75-77) back into keys
  int64_t* nsel = reinterpret_cast<int64_t*>(stats.as<uint8_t>() + 16);
  size_t tb2 = 0;
  F2V_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, alt.as<uint64_t>(), keys.as<uint64_t>(), nsel,
                                     int64_t(total), st));
  tmp.ensure(tb2);
  F2V_CUDA(cub::DeviceSelect::Unique(tmp.p, tb2, alt.as<uint64_t>(), keys.as<uint64_t>(), nsel,
                                     int64_t(total), st));
  unsigned long long host[4] = {0, 0, 0, 0};
  F2V_CUDA(cudaMemcpyAsync(host, stats.p, 32, cudaMemcpyDeviceToHost, st));
  F2V_CUDA(cudaStreamSynchronize(st));
  const uint64_t loops = host[0], range = host[1];
  uint64_t uniq = uint64_t(int64_t(host[2]));
  if (range) fail(F2V_ERANGE, "edge endpoint out of range");  // csr_graph.cpp:87
  const uint64_t loop_keys = loops * (symmetrize ? 2 : 1);
  const uint64_t before = total - loop_keys;  // arcs after erase_if + symmetrise
  const uint64_t nnz = uniq - (loops ? 1 : 0);  // the one surviving loop key
  uint64_t dups = before - nnz;
  if (symmetrize) dups /= 2;  // csr_graph.cpp:80
  alt.release();
  rowptr_dev.ensure(sizeof(uint64_t) * (uint64_t(n) + 1));
  col_dev.ensure(sizeof(uint32_t) * std::max<uint64_t>(nnz, 1));
  const uint32_t grid2 = uint32_t(std::max<uint64_t>(
      1, std::min<uint64_t>((nnz + 1 + 255) / 256, uint64_t(num_sms) * 16)));
  row_offsets_kernel<<<grid2, 256, 0, st>>>(keys.as<uint64_t>(), nnz, n,
                                            rowptr_dev.as<uint64_t>(), col_dev.as<uint32_t>());
  F2V_LAUNCHED(st, "row_offsets_kernel");
  F2V_CUDA(cudaStreamSynchronize(st));
  if (nnz_out) *nnz_out = nnz;
  if (dups_out) *dups_out = dups;
  if (loops_out) *loops_out = loops;
}

}  // namespace f2v
