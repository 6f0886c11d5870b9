// f2v_epoch.cu -- one device-resident epoch of train() (trainer.cpp:211-249):
// every batch's grad_minibatch + batch_loss + apply_update in ONE persistent
// dataflow kernel on sm_100a, with the reference's exact sequential-batch
// snapshot semantics and no grid-wide barrier between batches.
//
// Semantics.  Z is double-buffered: Zold = the
// epoch-start state, Znew = written exactly once per row.  A vertex u of
// batch j must see row v as of the end of batch j-1, i.e. Znew[v] iff
// batch(v) < j, else Zold[v].  state[v] = batch(v) << 1 | written.
//
// Schedule.  Each vertex's work is split into
//   E items (one per C-arc chunk of its CSR row): arcs to rows that are either
//     in batches >= j (Zold, no dependency) or "past" (batch < j - W, final long
//     ago).  The remaining "window" arcs (j - W <= batch(v) < j) are compacted
//     into a per-chunk list.  A vertex with no window arcs and no window
//     negatives is finalised right here.
//   L items (one per G chunks): the window arcs, oldest first, then the
//     most recent (age <= R) last, waiting on each row's written bit; combine
//     with the E partial + the shared negatives; finalise.
// Items are claimed in a static order where the E items of batch t sit next to
// the L items of batch t - A (lookahead A < W): the bandwidth-heavy E work
// runs A batches ahead of the latency-critical L chain, and every wait points
// at an item claimed earlier (deadlock-free on any number of resident CTAs).
// Partials of split rows are combined in a fixed order by the last arrival
// (no float atomics): results are bitwise reproducible run to run.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "f2v_internal.h"
#include "f2v_pair.cuh"
#include "f2v_rng.h"

namespace f2v {

__global__ void sum_kernel(const double* __restrict__ v, uint64_t m, double* out);

namespace {

using namespace dev;

constexpr uint32_t kLBit = 0x80000000u;
constexpr int kU = 4;  // rows in flight per warp per accumulate step

struct EpochArgs {
  const uint64_t* rowptr;
  const uint32_t* col;
  const float* zold;
  float* znew;
  const uint32_t* perm;
  uint32_t* state;
  const uint32_t* negs;
  const uint32_t* negwin;
  const uint2* items;
  uint32_t nitems;
  uint32_t* next;
  const uint32_t* cbase;
  const uint32_t* lbase;
  const uint32_t* lpo;
  double* epart;
  double* eloss;
  uint32_t* wcnt;
  uint32_t* wl;
  double* lpart;
  double* lloss;
  uint32_t* ecnt;
  uint32_t* lcnt;
  uint32_t* vflag;
  double* ploss;
  unsigned long long* bad;
  uint32_t n, d, b, s;
  uint32_t C, G, A, W, R;
  float eta;
  ForceParams fp;
};

__device__ __forceinline__ uint32_t wait_written(const uint32_t* state, uint32_t v, uint32_t st) {
  while (!(st & 1u)) {
    __nanosleep(32);
    st = ld_relaxed(state + v);
  }
  return st;
}

__device__ __forceinline__ uint32_t lanemask_lt(int lane) { return (1u << lane) - 1u; }

// Compact the lanes with `keep` (in lane order) into lanes 0..cnt-1.
__device__ __forceinline__ uint32_t compact(uint32_t* sh, int lane, bool keep, uint32_t val,
                                            int& cnt) {
  const uint32_t m = __ballot_sync(kFull, keep);
  if (keep) sh[__popc(m & lanemask_lt(lane))] = val;
  __syncwarp();
  cnt = __popc(m);
  const uint32_t out = lane < cnt ? sh[lane] : 0u;
  __syncwarp();
  return out;
}

// The shared negatives of batch j, in sample order (sampling.cpp:59).
template <int K, bool VEC, bool MON>
__device__ __forceinline__ void do_negatives(const EpochArgs& a, uint32_t j, int lane,
                                             const double (&uu)[K], double (&acc)[K],
                                             double& lsum) {
  for (uint32_t k0 = 0; k0 < a.s; k0 += 32) {
    const int cnt = int(umin32(32, a.s - k0));
    uint32_t pk = 0;
    if (lane < cnt) {
      const uint32_t w = a.negs[size_t(j) * a.s + k0 + lane];
      uint32_t st = ld_relaxed(a.state + w);
      if ((st >> 1) < j) {
        wait_written(a.state, w, st);
        pk = w | kNewBit;
      } else {
        pk = w;
      }
    }
    accumulate_rows<K, VEC, kU, MON, false>(a.fp, pk, cnt, lane, a.d, a.zold, a.znew, uu, acc,
                                            lsum);
  }
}

// g = float(acc) (trainer.cpp:140-145); z_u -= eta*g in fp32 (trainer.cpp:173);
// publish row u of Znew.
template <int K, bool VEC, bool MON>
__device__ __forceinline__ void finalize(const EpochArgs& a, uint32_t p, uint32_t u, int lane,
                                         const float (&zu)[K], const double (&acc)[K],
                                         double lsum) {
  using L = Lay<K, VEC>;
  bool bad = false;
  float nz[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float g = __double2float_rn(acc[k]);
    if (L::valid(lane, k, a.d) && !isfinite(g)) bad = true;
    nz[k] = __fsub_rn(zu[k], __fmul_rn(a.eta, g));
  }
  L::store(a.znew + size_t(u) * a.d, lane, a.d, nz);
  const bool any_bad = __any_sync(kFull, bad);
  if (MON && lane == 0) a.ploss[p] = lsum;
  __threadfence();
  __syncwarp();
  if (lane == 0) {
    if (any_bad) atomicMin(a.bad, (unsigned long long)p);
    atomicOr(a.state + u, 1u);
  }
}

template <int K, bool VEC, bool MON>
__device__ void do_E(const EpochArgs& a, uint32_t p, uint32_t c, int lane, uint32_t* sh) {
  using L = Lay<K, VEC>;
  const uint32_t u = a.perm[p];
  const uint32_t j = p / a.b;
  const uint64_t r0 = a.rowptr[u], r1 = a.rowptr[u + 1];
  const uint32_t cb = a.cbase[u];
  const uint32_t nch = a.cbase[u + 1] - cb;
  const uint32_t cs = cb + c;
  const uint64_t e0 = r0 + uint64_t(c) * a.C;
  const uint64_t e1 = umin64(e0 + a.C, r1);
  float zu[K];
  L::load(a.zold + size_t(u) * a.d, lane, a.d, zu, false);
  double uu[K], acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { uu[k] = zu[k]; acc[k] = 0.0; }
  double lsum = 0.0;
  uint32_t wc = 0;
  for (uint64_t e = e0; e < e1; e += 32) {
    const int cnt = int(umin64(32, e1 - e));
    uint32_t v = 0, pk = 0;
    bool use = false, win = false;
    if (lane < cnt) {
      v = a.col[e + lane];
      uint32_t st = ld_relaxed(a.state + v);
      const uint32_t bv = st >> 1;
      if (bv >= j) {
        use = true;
        pk = v;
      } else if (bv + a.W < j) {  // past: final long ago (rarely waits)
        wait_written(a.state, v, st);
        use = true;
        pk = v | kNewBit;
      } else {
        win = true;
      }
    }
    const uint32_t wm = __ballot_sync(kFull, win);
    if (win) a.wl[e0 + wc + __popc(wm & lanemask_lt(lane))] = v;
    wc += __popc(wm);
    int cu;
    const uint32_t pkc = compact(sh, lane, use, pk, cu);
    accumulate_rows<K, VEC, kU, MON, true>(a.fp, pkc, cu, lane, a.d, a.zold, a.znew, uu, acc,
                                           lsum);
  }
  const bool negwin = a.negwin[j] != 0;
  if (nch == 1) {
    if (wc == 0 && !negwin) {  // nothing depends on the window: finalise now
      do_negatives<K, VEC, MON>(a, j, lane, uu, acc, lsum);
      finalize<K, VEC, MON>(a, p, u, lane, zu, acc, lsum);
      if (lane == 0) st_relaxed(a.vflag + u, 2u);
    } else {
      L::store_acc(a.epart + size_t(cs) * a.d, lane, a.d, acc);
      if (lane == 0) {
        if (MON) __stcg(a.eloss + cs, lsum);
        __stcg(a.wcnt + cs, wc);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_relaxed(a.vflag + u, 1u);
    }
    return;
  }
  // hub chunk: publish the partial; the last E arrival combines in chunk order
  L::store_acc(a.epart + size_t(cs) * a.d, lane, a.d, acc);
  if (lane == 0) {
    if (MON) __stcg(a.eloss + cs, lsum);
    __stcg(a.wcnt + cs, wc);
  }
  __threadfence();
  __syncwarp();
  uint32_t last = 0;
  if (lane == 0) last = atomicAdd(a.ecnt + u, 1u) == nch - 1 ? 1u : 0u;
  if (!__shfl_sync(kFull, last, 0)) return;
  __threadfence();
  L::load_acc(a.epart + size_t(cb) * a.d, lane, a.d, acc);
  lsum = MON ? __ldcg(a.eloss + cb) : 0.0;
  uint32_t anyw = __ldcg(a.wcnt + cb);
#pragma unroll 4
  for (uint32_t q = 1; q < nch; ++q) {
    L::add_acc(a.epart + size_t(cb + q) * a.d, lane, a.d, acc);
    if (MON) lsum = __dadd_rn(lsum, __ldcg(a.eloss + cb + q));
    anyw += __ldcg(a.wcnt + cb + q);
  }
  if (lane == 0) a.ecnt[u] = 0;
  if (anyw == 0 && !negwin) {
    do_negatives<K, VEC, MON>(a, j, lane, uu, acc, lsum);
    finalize<K, VEC, MON>(a, p, u, lane, zu, acc, lsum);
    if (lane == 0) st_relaxed(a.vflag + u, 2u);
  } else {
    L::store_acc(a.epart + size_t(cb) * a.d, lane, a.d, acc);  // the E total
    if (MON && lane == 0) __stcg(a.eloss + cb, lsum);
    __threadfence();
    __syncwarp();
    if (lane == 0) st_relaxed(a.vflag + u, 1u);
  }
}

// Window arcs of chunks [c0, c1) of u: pass 0 = age > R, pass 1 = age <= R.
template <int K, bool VEC, bool MON>
__device__ __forceinline__ void window_pass(const EpochArgs& a, uint32_t u, uint32_t j,
                                            uint32_t c0, uint32_t c1, int pass, int lane,
                                            uint32_t* sh, const double (&uu)[K],
                                            double (&acc)[K], double& lsum) {
  const uint64_t r0 = a.rowptr[u];
  const uint32_t cb = a.cbase[u];
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t m = __ldcg(a.wcnt + cb + c);
    const uint64_t base = r0 + uint64_t(c) * a.C;
    for (uint32_t k0 = 0; k0 < m; k0 += 32) {
      const int cnt = int(umin32(32, m - k0));
      bool use = false;
      uint32_t pk = 0;
      if (lane < cnt) {
        const uint32_t v = __ldcg(a.wl + base + k0 + lane);
        uint32_t st = ld_relaxed(a.state + v);
        const uint32_t age = j - (st >> 1);
        use = pass == 0 ? age > a.R : age <= a.R;
        if (use) {
          wait_written(a.state, v, st);
          pk = v | kNewBit;
        }
      }
      int cu;
      const uint32_t pkc = compact(sh, lane, use, pk, cu);
      accumulate_rows<K, VEC, kU, MON, true>(a.fp, pkc, cu, lane, a.d, a.zold, a.znew, uu, acc,
                                             lsum);
    }
  }
}

template <int K, bool VEC, bool MON>
__device__ void do_L(const EpochArgs& a, uint32_t p, uint32_t cl, int lane, uint32_t* sh) {
  using L = Lay<K, VEC>;
  const uint32_t u = a.perm[p];
  const uint32_t j = p / a.b;
  const uint32_t cb = a.cbase[u];
  const uint32_t nch = a.cbase[u + 1] - cb;
  const uint32_t nchL = a.lbase[u + 1] - a.lbase[u];
  uint32_t f = ld_relaxed(a.vflag + u);
  while (f == 0) {  // the E work of u (claimed A batches earlier) is not done yet
    __nanosleep(64);
    f = ld_relaxed(a.vflag + u);
  }
  if (f == 2) {  // finalised by its E item
    if (nchL == 1) {
      if (lane == 0) a.vflag[u] = 0;
    } else if (lane == 0 && atomicAdd(a.lcnt + u, 1u) == nchL - 1) {
      a.lcnt[u] = 0;
      a.vflag[u] = 0;
    }
    return;
  }
  float zu[K];
  L::load(a.zold + size_t(u) * a.d, lane, a.d, zu, false);
  double uu[K], acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { uu[k] = zu[k]; acc[k] = 0.0; }
  double lsum = 0.0;
  const uint32_t c0 = cl * a.G, c1 = umin32(nch, c0 + a.G);
  if (nchL == 1) {  // E total + old window arcs + negatives + recent arcs
    L::load_acc(a.epart + size_t(cb) * a.d, lane, a.d, acc);
    if (MON) lsum = __ldcg(a.eloss + cb);
    window_pass<K, VEC, MON>(a, u, j, c0, c1, 0, lane, sh, uu, acc, lsum);
    do_negatives<K, VEC, MON>(a, j, lane, uu, acc, lsum);
    window_pass<K, VEC, MON>(a, u, j, c0, c1, 1, lane, sh, uu, acc, lsum);
    finalize<K, VEC, MON>(a, p, u, lane, zu, acc, lsum);
    if (lane == 0) a.vflag[u] = 0;
    return;
  }
  window_pass<K, VEC, MON>(a, u, j, c0, c1, 0, lane, sh, uu, acc, lsum);
  window_pass<K, VEC, MON>(a, u, j, c0, c1, 1, lane, sh, uu, acc, lsum);
  const uint32_t slot = a.lpo[u] + cl;
  L::store_acc(a.lpart + size_t(slot) * a.d, lane, a.d, acc);
  if (MON && lane == 0) __stcg(a.lloss + slot, lsum);
  __threadfence();
  __syncwarp();
  uint32_t last = 0;
  if (lane == 0) last = atomicAdd(a.lcnt + u, 1u) == nchL - 1 ? 1u : 0u;
  if (!__shfl_sync(kFull, last, 0)) return;
  __threadfence();
  L::load_acc(a.epart + size_t(cb) * a.d, lane, a.d, acc);
  lsum = MON ? __ldcg(a.eloss + cb) : 0.0;
  const uint32_t lp = a.lpo[u];
#pragma unroll 4
  for (uint32_t q = 0; q < nchL; ++q) {
    L::add_acc(a.lpart + size_t(lp + q) * a.d, lane, a.d, acc);
    if (MON) lsum = __dadd_rn(lsum, __ldcg(a.lloss + lp + q));
  }
  do_negatives<K, VEC, MON>(a, j, lane, uu, acc, lsum);
  finalize<K, VEC, MON>(a, p, u, lane, zu, acc, lsum);
  if (lane == 0) {
    a.lcnt[u] = 0;
    a.vflag[u] = 0;
  }
}

template <int K, bool VEC, bool MON>
__global__ void __launch_bounds__(256) epoch_kernel(EpochArgs a) {
  __shared__ uint32_t shc[8][32];
  const int lane = threadIdx.x & 31;
  uint32_t* sh = shc[threadIdx.x >> 5];
  uint32_t it = 0;
  if (lane == 0) it = atomicAdd(a.next, 1u);
  it = __shfl_sync(kFull, it, 0);
  while (it < a.nitems) {
    uint32_t nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.next, 1u);  // claim ahead: hides the atomic's latency
    const uint2 item = a.items[it];
    if (item.y & kLBit) do_L<K, VEC, MON>(a, item.x, item.y & ~kLBit, lane, sh);
    else do_E<K, VEC, MON>(a, item.x, item.y, lane, sh);
    it = __shfl_sync(kFull, nxt, 0);
  }
}

// ------------------------------------------------------ per-epoch prep
__global__ void state_kernel(const uint32_t* __restrict__ perm, uint32_t* __restrict__ state,
                             uint32_t n, uint32_t b, const uint32_t* __restrict__ cbase,
                             const uint32_t* __restrict__ lbase, uint32_t* __restrict__ nE,
                             uint32_t* __restrict__ nL) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  if (p == n) {
    nE[n] = 0;
    nL[n] = 0;
    return;
  }
  const uint32_t u = perm[p];
  state[u] = (p / b) << 1;
  nE[p] = cbase[u + 1] - cbase[u];
  nL[p] = lbase[u + 1] - lbase[u];
}

__device__ __forceinline__ uint32_t batch_count(const uint32_t* P, uint32_t t, uint32_t b,
                                                uint32_t n) {
  const uint64_t lo = uint64_t(t) * b, hi = umin64(lo + b, n);
  return P[hi] - P[lo];
}

__global__ void slot_kernel(const uint32_t* __restrict__ EP, const uint32_t* __restrict__ LP,
                            uint32_t* __restrict__ sz, uint32_t nb, uint32_t A, uint32_t b,
                            uint32_t n) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nb + A) return;
  uint32_t v = 0;
  if (t < nb) v += batch_count(EP, t, b, n);
  if (t >= A && t - A < nb) v += batch_count(LP, t - A, b, n);
  sz[t] = v;
}

__global__ void emit_kernel(const uint32_t* __restrict__ EP, const uint32_t* __restrict__ LP,
                            const uint32_t* __restrict__ SS, uint2* __restrict__ items,
                            uint32_t n, uint32_t b, uint32_t nb, uint32_t A) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t j = p / b;
  const uint64_t j0 = uint64_t(j) * b;
  const uint32_t eo = SS[j] + (EP[p] - EP[j0]);
  for (uint32_t c = 0, ne = EP[p + 1] - EP[p]; c < ne; ++c) items[eo + c] = make_uint2(p, c);
  const uint32_t t = j + A;
  const uint32_t lo = SS[t] + (t < nb ? batch_count(EP, t, b, n) : 0u) + (LP[p] - LP[j0]);
  for (uint32_t c = 0, nl = LP[p + 1] - LP[p]; c < nl; ++c)
    items[lo + c] = make_uint2(p, c | kLBit);
}

__global__ void negs_kernel(uint32_t* __restrict__ out, uint32_t* __restrict__ negwin,
                            const uint32_t* __restrict__ state, uint64_t nb, uint32_t s,
                            uint32_t n, uint64_t seed, uint32_t epoch, int sampler, uint32_t W) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  uint32_t win = 0;
  for (uint32_t k = 0; k < s; ++k) {
    const uint32_t w = sampler == F2V_SAMPLER_PHILOX ? philox_negative(seed, epoch, j, 0, k, n)
                                                     : splitmix_negative(seed, epoch, j, 0, 1, k, n);
    out[j * s + k] = w;
    const uint32_t bw = state[w] >> 1;
    if (bw < j && uint64_t(bw) + W >= j) win = 1;
  }
  negwin[j] = win;
}

// On a NumericalError at batch jb: rows of batches >= jb go back to Zold so
// Znew is the state after the last complete batch (trainer.cpp:149-152).
__global__ void restore_kernel(const uint32_t* __restrict__ state, const float* __restrict__ zold,
                               float* __restrict__ znew, uint32_t n, uint32_t d, uint64_t jb) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= uint64_t(n) * d) return;
  const uint32_t v = uint32_t(t / d);
  if ((state[v] >> 1) >= jb) znew[t] = zold[t];
}

template <int K, bool VEC, bool MON>
void launch_epoch_t(Ctx& c, const EpochArgs& a) {
  auto kern = epoch_kernel<K, VEC, MON>;
  int per_sm = 0;
  F2V_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
  if (per_sm < 1) per_sm = 1;
  uint32_t blocks = uint32_t(per_sm) * uint32_t(c.num_sms);
  const uint32_t need = uint32_t((uint64_t(a.nitems) * 32 + 255) / 256);
  blocks = std::max(1u, std::min(blocks, need));
  kern<<<blocks, 256, 0, c.stream>>>(a);
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
}

template <bool MON>
void launch_epoch(Ctx& c, const EpochArgs& a) {
  const uint32_t d = a.d;
  if (d == 128) launch_epoch_t<4, true, MON>(c, a);
  else if (d == 256) launch_epoch_t<8, true, MON>(c, a);
  else if (d == 64) launch_epoch_t<2, true, MON>(c, a);
  else if (d == 32) launch_epoch_t<1, true, MON>(c, a);
  else if (d <= 32) launch_epoch_t<1, false, MON>(c, a);
  else if (d <= 64) launch_epoch_t<2, false, MON>(c, a);
  else if (d <= 128) launch_epoch_t<4, false, MON>(c, a);
  else if (d <= 256) launch_epoch_t<8, false, MON>(c, a);
  else if (d <= 512) launch_epoch_t<16, false, MON>(c, a);
  else launch_epoch_t<32, false, MON>(c, a);
}

uint32_t env_u32(const char* name, uint32_t dflt) {
  if (const char* e = std::getenv(name)) {
    const long v = std::atol(e);
    if (v >= 0) return uint32_t(v);
  }
  return dflt;
}

}  // namespace

void load_tuning(EpochTuning& t) {
  t.chunk = std::max(1u, env_u32("F2V_CHUNK", t.chunk));
  t.lgroup = std::max(1u, env_u32("F2V_LGROUP", t.lgroup));
  t.lookahead = std::max(1u, env_u32("F2V_LOOKAHEAD", t.lookahead));
  t.window = std::max(t.lookahead + 1, env_u32("F2V_WINDOW", t.window));
  t.recent = env_u32("F2V_RECENT", t.recent);
}

// Static per-graph chunk / L-group layout (depends on chunk and lgroup only).
void k_prepare_graph(Ctx& c) {
  const uint32_t C = c.tune.chunk, G = c.tune.lgroup;
  std::vector<uint32_t> cbase(size_t(c.n) + 1), lbase(size_t(c.n) + 1), lpo(c.n ? c.n : 1, 0u);
  uint64_t chunks = 0, lgroups = 0, lslots = 0;
  for (uint32_t u = 0; u < c.n; ++u) {
    const uint64_t deg = c.h_rowptr[u + 1] - c.h_rowptr[u];
    const uint64_t nch = deg ? (deg + C - 1) / C : 1;
    const uint64_t nl = (nch + G - 1) / G;
    cbase[u] = uint32_t(chunks);
    lbase[u] = uint32_t(lgroups);
    if (nl > 1) {
      lpo[u] = uint32_t(lslots);
      lslots += nl;
    }
    chunks += nch;
    lgroups += nl;
    if (chunks >= (1ull << 31) || lgroups >= (1ull << 31))
      fail(F2V_EUSAGE, "graph too large for the chunk bookkeeping (raise F2V_CHUNK)");
  }
  cbase[c.n] = uint32_t(chunks);
  lbase[c.n] = uint32_t(lgroups);
  c.chunks = chunks;
  c.lgroups = lgroups;
  c.lslots = lslots;
  c.prepared_chunk = C;
  c.prepared_lgroup = G;
  c.cbase.ensure(sizeof(uint32_t) * (size_t(c.n) + 1));
  c.lbase.ensure(sizeof(uint32_t) * (size_t(c.n) + 1));
  c.lpo.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  c.ecnt.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  c.lcnt.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  c.vflag.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  F2V_CUDA(cudaMemcpyAsync(c.cbase.p, cbase.data(), sizeof(uint32_t) * (c.n + 1),
                           cudaMemcpyHostToDevice, c.stream));
  F2V_CUDA(cudaMemcpyAsync(c.lbase.p, lbase.data(), sizeof(uint32_t) * (c.n + 1),
                           cudaMemcpyHostToDevice, c.stream));
  if (c.n) {
    F2V_CUDA(cudaMemcpyAsync(c.lpo.p, lpo.data(), sizeof(uint32_t) * c.n,
                             cudaMemcpyHostToDevice, c.stream));
    F2V_CUDA(cudaMemsetAsync(c.ecnt.p, 0, sizeof(uint32_t) * c.n, c.stream));
    F2V_CUDA(cudaMemsetAsync(c.lcnt.p, 0, sizeof(uint32_t) * c.n, c.stream));
    F2V_CUDA(cudaMemsetAsync(c.vflag.p, 0, sizeof(uint32_t) * c.n, c.stream));
  }
  F2V_CUDA(cudaStreamSynchronize(c.stream));
}

// Per-epoch preparation: perm (already in c.perm) -> state, the ordered work
// items, the negatives of every batch and their window flags.
void k_epoch_begin(Ctx& c, uint32_t b, uint32_t s, uint32_t epoch, uint64_t seed, int sampler) {
  const uint32_t n = c.n;
  const uint32_t nb = uint32_t((uint64_t(n) + b - 1) / b);
  const uint32_t A = c.tune.lookahead;
  if (c.prepared_chunk != c.tune.chunk || c.prepared_lgroup != c.tune.lgroup)
    k_prepare_graph(c);
  c.state.ensure(sizeof(uint32_t) * n);
  c.nE.ensure(sizeof(uint32_t) * (n + 1));
  c.nL.ensure(sizeof(uint32_t) * (n + 1));
  c.EP.ensure(sizeof(uint32_t) * (n + 1));
  c.LP.ensure(sizeof(uint32_t) * (n + 1));
  c.sz.ensure(sizeof(uint32_t) * (size_t(nb) + A + 1));
  c.SS.ensure(sizeof(uint32_t) * (size_t(nb) + A + 1));
  c.items.ensure(sizeof(uint2) * std::max<uint64_t>(c.chunks + c.lgroups, 1));
  c.negs_all.ensure(sizeof(uint32_t) * std::max<uint64_t>(uint64_t(nb) * s, 1));
  c.negwin.ensure(sizeof(uint32_t) * std::max<uint32_t>(nb, 1));
  c.epart.ensure(sizeof(double) * std::max<uint64_t>(c.chunks * c.d, 1));
  c.eloss.ensure(sizeof(double) * std::max<uint64_t>(c.chunks, 1));
  c.wcnt.ensure(sizeof(uint32_t) * std::max<uint64_t>(c.chunks, 1));
  c.wl.ensure(sizeof(uint32_t) * std::max<uint64_t>(c.nnz, 1));
  c.lpart.ensure(sizeof(double) * std::max<uint64_t>(c.lslots * c.d, 1));
  c.lloss.ensure(sizeof(double) * std::max<uint64_t>(c.lslots, 1));
  c.ploss.ensure(sizeof(double) * std::max<uint32_t>(n, 1));
  c.counters.ensure(64);
  state_kernel<<<(n + 1 + 255) / 256, 256, 0, c.stream>>>(
      c.perm.as<uint32_t>(), c.state.as<uint32_t>(), n, b, c.cbase.as<uint32_t>(),
      c.lbase.as<uint32_t>(), c.nE.as<uint32_t>(), c.nL.as<uint32_t>());
  F2V_CUDA(cudaGetLastError());
  size_t tmp = 0, tmp2 = 0;
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.nE.as<uint32_t>(), c.EP.as<uint32_t>(),
                                         n + 1, c.stream));
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, c.sz.as<uint32_t>(),
                                         c.SS.as<uint32_t>(), nb + A + 1, c.stream));
  c.scan_tmp.ensure(std::max(tmp, tmp2));
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp, c.nE.as<uint32_t>(),
                                         c.EP.as<uint32_t>(), n + 1, c.stream));
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp, c.nL.as<uint32_t>(),
                                         c.LP.as<uint32_t>(), n + 1, c.stream));
  slot_kernel<<<(nb + A + 1 + 255) / 256, 256, 0, c.stream>>>(
      c.EP.as<uint32_t>(), c.LP.as<uint32_t>(), c.sz.as<uint32_t>(), nb, A, b, n);
  F2V_CUDA(cudaGetLastError());
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp2, c.sz.as<uint32_t>(),
                                         c.SS.as<uint32_t>(), nb + A + 1, c.stream));
  emit_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(c.EP.as<uint32_t>(), c.LP.as<uint32_t>(),
                                                     c.SS.as<uint32_t>(), c.items.as<uint2>(), n,
                                                     b, nb, A);
  F2V_CUDA(cudaGetLastError());
  negs_kernel<<<(nb + 255) / 256, 256, 0, c.stream>>>(
      c.negs_all.as<uint32_t>(), c.negwin.as<uint32_t>(), c.state.as<uint32_t>(), nb, s, n, seed,
      epoch, sampler, c.tune.window);
  F2V_CUDA(cudaGetLastError());
  c.launches += 8;
}

EpochResult k_epoch_run(Ctx& c, uint32_t b, uint32_t s, float eta, const ForceParams& fp,
                        bool monitor) {
  const int nxt = 1 - c.cur;
  c.z[nxt].ensure(sizeof(float) * size_t(c.n) * c.d);
  uint32_t* ctr = c.counters.as<uint32_t>();  // [0] next item, [2..3] bad (u64), [4..5] loss
  F2V_CUDA(cudaMemsetAsync(ctr, 0, 8, c.stream));
  F2V_CUDA(cudaMemsetAsync(ctr + 2, 0xff, 8, c.stream));
  EpochArgs a;
  a.rowptr = c.rowptr.as<uint64_t>();
  a.col = c.col.as<uint32_t>();
  a.zold = c.z[c.cur].as<float>();
  a.znew = c.z[nxt].as<float>();
  a.perm = c.perm.as<uint32_t>();
  a.state = c.state.as<uint32_t>();
  a.negs = c.negs_all.as<uint32_t>();
  a.negwin = c.negwin.as<uint32_t>();
  a.items = c.items.as<uint2>();
  a.nitems = uint32_t(c.chunks + c.lgroups);
  a.next = ctr;
  a.cbase = c.cbase.as<uint32_t>();
  a.lbase = c.lbase.as<uint32_t>();
  a.lpo = c.lpo.as<uint32_t>();
  a.epart = c.epart.as<double>();
  a.eloss = c.eloss.as<double>();
  a.wcnt = c.wcnt.as<uint32_t>();
  a.wl = c.wl.as<uint32_t>();
  a.lpart = c.lpart.as<double>();
  a.lloss = c.lloss.as<double>();
  a.ecnt = c.ecnt.as<uint32_t>();
  a.lcnt = c.lcnt.as<uint32_t>();
  a.vflag = c.vflag.as<uint32_t>();
  a.ploss = c.ploss.as<double>();
  a.bad = reinterpret_cast<unsigned long long*>(ctr + 2);
  a.n = c.n;
  a.d = c.d;
  a.b = b;
  a.s = s;
  a.C = c.tune.chunk;
  a.G = c.tune.lgroup;
  a.A = c.tune.lookahead;
  a.W = c.tune.window;
  a.R = c.tune.recent;
  a.eta = eta;
  a.fp = fp;
  if (!c.ev_kernel.size()) {
    c.ev_kernel.resize(2);
    F2V_CUDA(cudaEventCreate(&c.ev_kernel[0]));
    F2V_CUDA(cudaEventCreate(&c.ev_kernel[1]));
  }
  F2V_CUDA(cudaEventRecord(c.ev_kernel[0], c.stream));
  if (monitor) launch_epoch<true>(c, a);
  else launch_epoch<false>(c, a);
  F2V_CUDA(cudaEventRecord(c.ev_kernel[1], c.stream));
  if (monitor) {
    sum_kernel<<<1, 1024, 0, c.stream>>>(c.ploss.as<double>(), c.n,
                                         reinterpret_cast<double*>(ctr + 4));
    F2V_CUDA(cudaGetLastError());
    ++c.launches;
  }
  uint64_t host[3];
  F2V_CUDA(cudaMemcpyAsync(host, ctr, 24, cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  float kms = 0.f;
  F2V_CUDA(cudaEventElapsedTime(&kms, c.ev_kernel[0], c.ev_kernel[1]));
  c.timing[1] += kms;
  c.timing[2] += 1;
  EpochResult r{host[1], 0.0};
  if (monitor) std::memcpy(&r.loss, &host[2], sizeof(double));
  c.cur = nxt;  // Znew becomes the current embedding
  return r;
}

void k_epoch_restore(Ctx& c, uint32_t b, uint64_t bad_batch) {
  (void)b;
  const uint64_t total = uint64_t(c.n) * c.d;
  restore_kernel<<<uint32_t((total + 255) / 256), 256, 0, c.stream>>>(
      c.state.as<uint32_t>(), c.z[1 - c.cur].as<float>(), c.zcur(), c.n, c.d, bad_batch);
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
  F2V_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace f2v
