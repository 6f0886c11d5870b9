// f2v_kernels.cu -- hand-written sm_100a kernels for Force2Vec's minibatch SGD
// step (the fused SDDMM+SpMM gradient + update of trainer.cpp:108-190).
//
// Layout: Z is row-major f32[n x d]; one warp owns
// one batch row; lane L holds K columns of every row it touches (VEC layout:
// columns [L*K, L*K+K), one 16-byte load per lane for d = 128), so a neighbour
// row is one fully coalesced 512-byte gather.  Dot products / distances are
// fp64 (warp butterfly), the per-pair term and the per-vertex accumulator are
// fp64 exactly as force_kernels.cpp:30-77 / trainer.cpp:124-138 compute them,
// the gradient is rounded to fp32 once (trainer.cpp:142) and the update is
// fp32 multiply-then-subtract (trainer.cpp:173).  This file is compiled with
// --fmad=false so nvcc cannot contract the reference's separate roundings.
//
// Two entry points:
//  * the per-step operators (grad_minibatch / apply_update / batch_loss), one
//    launch each, operating in place on Z (snapshot by construction);
//  * the device-resident epoch: a persistent DATAFLOW kernel over all batches
//    of an epoch.  Z is double-buffered (Zold = epoch start, Znew = written
//    once per row); batch j reads row v from Znew iff batch(v) < j, waiting on
//    v's per-row "written" bit, else from Zold -- exactly the sequential
//    batch-after-batch snapshot semantics of train() (trainer.cpp:220-236),
//    without a grid-wide barrier between batches.  Hubs are split into
//    chunks of <= `chunk` arcs whose fp64 partials are combined in a fixed
//    order by the last-arriving chunk (deterministic, no float atomics).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "f2v_internal.h"
#include "f2v_rng.h"

namespace f2v {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kNewBit = 0x80000000u;

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int m = 16; m; m >>= 1) x = __dadd_rn(x, __shfl_xor_sync(kFull, x, m));
  return x;
}

// force_kernels.hpp:25-29
__device__ __forceinline__ double stable_sigmoid(double x) {
  if (x >= 0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
  const double e = exp(x);
  return __ddiv_rn(e, __dadd_rn(1.0, e));
}

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- row I/O
// K columns per lane. VEC: columns lane*K..lane*K+K-1 (d == 32*K exactly,
// vector loads). !VEC: columns k*32+lane, masked by d (any d <= 32*K).
template <int K, bool VEC>
struct Lay {
  __device__ static __forceinline__ uint32_t col(int lane, int k) {
    return VEC ? uint32_t(lane * K + k) : uint32_t(k * 32 + lane);
  }
  __device__ static __forceinline__ bool valid(int lane, int k, uint32_t d) {
    return VEC ? true : (uint32_t(k * 32 + lane) < d);
  }
  // coherent = row may have been written during this launch (L2 path)
  __device__ static __forceinline__ void load(const float* row, int lane, uint32_t d,
                                              float (&v)[K], bool coherent) {
    if constexpr (VEC && K % 4 == 0) {
#pragma unroll
      for (int q = 0; q < K / 4; ++q) {
        const float4* p = reinterpret_cast<const float4*>(row + lane * K) + q;
        const float4 t = coherent ? __ldcg(p) : __ldg(p);
        v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
      }
    } else if constexpr (VEC && K == 2) {
      const float2* p = reinterpret_cast<const float2*>(row + lane * 2);
      const float2 t = coherent ? __ldcg(p) : __ldg(p);
      v[0] = t.x; v[1] = t.y;
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t c = col(lane, k);
        v[k] = (VEC || c < d) ? (coherent ? __ldcg(row + c) : __ldg(row + c)) : 0.0f;
      }
    }
  }
  __device__ static __forceinline__ void store(float* row, int lane, uint32_t d,
                                               const float (&v)[K]) {
    if constexpr (VEC && K % 4 == 0) {
#pragma unroll
      for (int q = 0; q < K / 4; ++q)
        __stcg(reinterpret_cast<float4*>(row + lane * K) + q,
               make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (valid(lane, k, d)) __stcg(row + col(lane, k), v[k]);
    }
  }
};

// ------------------------------------------------------- per-pair terms
// The reduction a pair needs: <u,o> (sigmoid) or ||u-o||^2 (distance kinds),
// plus ||o||^2 for the clamped sigmoid repulsion (force_kernels.cpp:95).
template <int K>
__device__ __forceinline__ double partial_sim(const ForceParams& fp, const double (&uu)[K],
                                              const float (&v)[K]) {
  double s = 0.0;
  if (fp.kind == F2V_SIGMOID) {
#pragma unroll
    for (int k = 0; k < K; ++k) s = __dadd_rn(s, __dmul_rn(uu[k], double(v[k])));
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double t = __dsub_rn(uu[k], double(v[k]));
      s = __dadd_rn(s, __dmul_rn(t, t));
    }
  }
  return s;
}
template <int K>
__device__ __forceinline__ double partial_norm2(const float (&v)[K]) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) s = __dadd_rn(s, __dmul_rn(double(v[k]), double(v[k])));
  return s;
}

// Scalar part of one pair: out_j = coef * o_j              (sigmoid)
//                          out_j = coef * (u_j - o_j) * inv (distance kinds)
//                          out   = (coef, 0, ..., 0)       (fallback)
// followed by  out_j *= scale  when clamped (force_kernels.cpp:69-77).
struct Term {
  double coef, inv, scale;
  bool dist, fallback, clamped;
  double loss;
};

template <bool MON>
__device__ __forceinline__ Term pair_term(const ForceParams& fp, bool attractive, double red,
                                          double nw2) {
  Term t{};
  t.scale = 1.0;
  if (fp.kind == F2V_SIGMOID) {  // force_kernels.cpp:79-97
    const double x = red;
    const double sg = stable_sigmoid(x);
    t.coef = attractive ? __dsub_rn(sg, 1.0) : sg;
    if (!attractive && fp.has_cap) {
      const double m = __dmul_rn(t.coef, sqrt(nw2));
      t.clamped = !(m <= fp.cap || m == 0.0);
      if (t.clamped) t.scale = __ddiv_rn(fp.cap, m);
    }
    if (MON) {  // force_kernels.cpp:213-219
      if (attractive)
        t.loss = x >= 0 ? log1p(exp(-x)) : __dadd_rn(-x, log1p(exp(x)));
      else
        t.loss = x >= 0 ? __dadd_rn(x, log1p(exp(-x))) : log1p(exp(x));
    }
    return t;
  }
  t.dist = true;
  const double r_raw = sqrt(red);  // distance(), force_kernels.cpp:36-43
  double scalar;
  bool clamp_it = false;
  if (fp.kind == F2V_TDIST) {
    if (attractive) {  // 99-107
      scalar = __ddiv_rn(__dmul_rn(2.0, r_raw), __dadd_rn(1.0, __dmul_rn(r_raw, r_raw)));
    } else {  // 109-119
      const double tt = dmax(r_raw, fp.eps);
      scalar = __ddiv_rn(-2.0, __dmul_rn(tt, __dadd_rn(1.0, __dmul_rn(tt, tt))));
      clamp_it = true;
    }
    if (MON) {  // force_kernels.cpp:221-227
      const double t2 = __dmul_rn(r_raw, r_raw);
      if (attractive) {
        t.loss = log1p(t2);
      } else {
        const double tc = dmax(t2, __dmul_rn(fp.eps, fp.eps));
        t.loss = -log(__ddiv_rn(tc, __dadd_rn(1.0, tc)));
      }
    }
  } else {  // table-II kinds, force_kernels.cpp:121-147
    if (attractive) {
      scalar = fp.kind == F2V_FR ? __dmul_rn(r_raw, r_raw)
                                 : (fp.kind == F2V_FA ? r_raw : log1p(r_raw));
    } else {
      scalar = __ddiv_rn(-1.0, dmax(r_raw, fp.eps));
      clamp_it = true;
    }
  }
  t.coef = scalar;
  t.fallback = r_raw < fp.eps;  // scaled_unit_diff, force_kernels.cpp:54-65
  t.inv = __ddiv_rn(1.0, r_raw);
  if (clamp_it && fp.has_cap) {
    const double m = fabs(scalar);
    t.clamped = !(m <= fp.cap || m == 0.0);
    if (t.clamped) t.scale = __ddiv_rn(fp.cap, m);
  }
  return t;
}

template <int K, bool VEC>
__device__ __forceinline__ void accumulate(const Term& t, int lane, const double (&uu)[K],
                                           const float (&v)[K], double (&acc)[K]) {
  if (!t.dist) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double o = __dmul_rn(t.coef, double(v[k]));
      if (t.clamped) o = __dmul_rn(o, t.scale);
      acc[k] = __dadd_rn(acc[k], o);
    }
    return;
  }
  if (t.fallback) {
    if (lane == 0) {  // column 0 lives on lane 0, k = 0 in both layouts
      double o = t.coef;
      if (t.clamped) o = __dmul_rn(o, t.scale);
      acc[0] = __dadd_rn(acc[0], o);
    }
    // the other columns add +0.0 (or +0.0*scale): acc + 0.0 == acc except -0.0
    const double zero = t.clamped ? __dmul_rn(0.0, t.scale) : 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane != 0 || k != 0) acc[k] = __dadd_rn(acc[k], zero);
    return;
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double diff = __dsub_rn(uu[k], double(v[k]));
    double o = __dmul_rn(__dmul_rn(t.coef, diff), t.inv);
    if (t.clamped) o = __dmul_rn(o, t.scale);
    acc[k] = __dadd_rn(acc[k], o);
  }
}

// Accumulate the pairs of `cnt` (<= 32) other-rows whose packed ids sit one per
// lane (bit 31 = read the coherent Znew buffer), in lane order, U at a time.
template <int K, bool VEC, int U, bool MON>
__device__ __forceinline__ void accumulate_rows(const ForceParams& fp, bool attractive,
                                                uint32_t packed, int cnt, int lane, uint32_t d,
                                                const float* __restrict__ zold,
                                                const float* __restrict__ znew,
                                                const double (&uu)[K], double (&acc)[K],
                                                double& lsum) {
  using L = Lay<K, VEC>;
  for (int k0 = 0; k0 < cnt; k0 += U) {
    float v[U][K];
    uint32_t pk[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      pk[i] = __shfl_sync(kFull, packed, (k0 + i) & 31);
      if (k0 + i < cnt) {
        const bool coh = (pk[i] & kNewBit) != 0;
        const float* base = coh ? znew : zold;
        L::load(base + size_t(pk[i] & ~kNewBit) * d, lane, d, v[i], coh);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) v[i][k] = 0.0f;
      }
    }
    double red[U], nw[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      red[i] = partial_sim<K>(fp, uu, v[i]);
      nw[i] = (!attractive && fp.kind == F2V_SIGMOID) ? partial_norm2<K>(v[i]) : 0.0;
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) {
#pragma unroll
      for (int i = 0; i < U; ++i) {
        red[i] = __dadd_rn(red[i], __shfl_xor_sync(kFull, red[i], m));
        if (!attractive && fp.kind == F2V_SIGMOID)
          nw[i] = __dadd_rn(nw[i], __shfl_xor_sync(kFull, nw[i], m));
      }
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      if (k0 + i < cnt) {
        const Term t = pair_term<MON>(fp, attractive, red[i], nw[i]);
        accumulate<K, VEC>(t, lane, uu, v[i], acc);
        if (MON) lsum = __dadd_rn(lsum, t.loss);
      }
    }
  }
}

// ============================================================ per-step path
struct StepArgs {
  const uint64_t* rowptr;
  const uint32_t* col;
  const float* z;
  const uint32_t* ids;
  const uint32_t* negs;
  float* grads;
  double* vloss;
  unsigned long long* bad;
  uint32_t b, s, d;
  ForceParams fp;
};

// grad_minibatch (trainer.cpp:108-165): one warp per batch row.
template <int K, bool VEC, bool MON>
__global__ void __launch_bounds__(256) grad_step_kernel(StepArgs a) {
  using L = Lay<K, VEC>;
  const int lane = threadIdx.x & 31;
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= a.b) return;
  const uint32_t u = a.ids[i];
  float zu[K];
  L::load(a.z + size_t(u) * a.d, lane, a.d, zu, false);
  double uu[K], acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { uu[k] = zu[k]; acc[k] = 0.0; }
  double lsum = 0.0;
  const uint64_t r0 = a.rowptr[u], r1 = a.rowptr[u + 1];
  for (uint64_t e = r0; e < r1; e += 32) {
    const int cnt = int(umin64(32, r1 - e));
    const uint32_t v = lane < cnt ? a.col[e + lane] : 0u;
    accumulate_rows<K, VEC, 4, MON>(a.fp, true, v, cnt, lane, a.d, a.z, a.z, uu, acc, lsum);
  }
  for (uint32_t k0 = 0; k0 < a.s; k0 += 32) {
    const int cnt = int(umin32(32, a.s - k0));
    const uint32_t w = lane < cnt ? a.negs[k0 + lane] : 0u;
    accumulate_rows<K, VEC, 4, MON>(a.fp, false, w, cnt, lane, a.d, a.z, a.z, uu, acc, lsum);
  }
  float g[K];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    g[k] = __double2float_rn(acc[k]);
    if (L::valid(lane, k, a.d) && !isfinite(g[k])) bad = true;
  }
  L::store(a.grads + size_t(i) * a.d, lane, a.d, g);
  if (__any_sync(kFull, bad) && lane == 0) atomicMin(a.bad, (unsigned long long)i);
  if (MON && lane == 0) a.vloss[i] = lsum;
}

// apply_update (trainer.cpp:167-175), distinct ids: one thread per element.
__global__ void apply_kernel(float* __restrict__ z, const uint32_t* __restrict__ ids,
                             const float* __restrict__ g, uint32_t b, uint32_t d, float eta) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= uint64_t(b) * d) return;
  const uint32_t i = uint32_t(t / d), c = uint32_t(t % d);
  float* p = z + size_t(ids[i]) * d + c;
  *p = __fsub_rn(*p, __fmul_rn(eta, g[t]));
}

// apply_update with repeated ids: rows in batch order per column.
__global__ void apply_seq_kernel(float* __restrict__ z, const uint32_t* __restrict__ ids,
                                 const float* __restrict__ g, uint32_t b, uint32_t d, float eta) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  for (uint32_t i = 0; i < b; ++i) {
    float* p = z + size_t(ids[i]) * d + c;
    *p = __fsub_rn(*p, __fmul_rn(eta, g[size_t(i) * d + c]));
  }
}

// deterministic fixed-order sum of v[0..m): per-thread strided sequential
// sums, then a fixed tree (one block).
__global__ void sum_kernel(const double* __restrict__ v, uint64_t m, double* out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (uint64_t k = threadIdx.x; k < m; k += blockDim.x) s = __dadd_rn(s, v[k]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w; w >>= 1) {
    if (int(threadIdx.x) < w) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// U(lo, hi) from a SplitMix stream (test_trainer.cpp:18-23 / trainer.cpp:62-72)
__global__ void uniform_kernel(float* z, uint64_t total, uint64_t s0, double lo, double hi) {
  const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= total) return;
  const double u = rng_uniform(rng_draw(s0, k));
  z[k] = __double2float_rn(__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u)));
}

// ============================================================ epoch path
struct EpochArgs {
  const uint64_t* rowptr;
  const uint32_t* col;
  const float* zold;
  float* znew;
  const uint32_t* perm;
  uint32_t* state;  // (batch(v) << 1) | written
  const uint32_t* negs;
  const uint2* items;
  uint32_t nitems;
  uint32_t* next;
  double* partials;
  double* partial_loss;
  const uint32_t* part_off;
  uint32_t* chunk_cnt;
  double* ploss;
  unsigned long long* bad;
  uint32_t n, d, b, s, chunk;
  float eta;
  ForceParams fp;
};

// batch j of the row of v: Zold if batch(v) >= j, else Znew once written.
__device__ __forceinline__ uint32_t resolve(uint32_t* state, uint32_t v, uint32_t j) {
  uint32_t st = ld_acquire(state + v);
  if ((st >> 1) >= j) return v;
  while (!(st & 1u)) {
    __nanosleep(64);
    st = ld_acquire(state + v);
  }
  return v | kNewBit;
}

template <int K, bool VEC, bool MON>
__global__ void __launch_bounds__(256) epoch_kernel(EpochArgs a) {
  using L = Lay<K, VEC>;
  const int lane = threadIdx.x & 31;
  uint32_t it = 0;
  if (lane == 0) it = atomicAdd(a.next, 1u);
  it = __shfl_sync(kFull, it, 0);
  while (it < a.nitems) {
    uint32_t nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.next, 1u);  // claim ahead: hides the atomic's latency
    const uint2 item = a.items[it];
    const uint32_t p = item.x, c = item.y;
    const uint32_t u = a.perm[p];
    const uint32_t j = p / a.b;
    const uint64_t r0 = a.rowptr[u], r1 = a.rowptr[u + 1];
    const uint64_t deg = r1 - r0;
    const uint32_t nch = deg ? uint32_t((deg + a.chunk - 1) / a.chunk) : 1u;
    const uint64_t e0 = r0 + uint64_t(c) * a.chunk;
    const uint64_t e1 = umin64(e0 + a.chunk, r1);

    float zu[K];
    L::load(a.zold + size_t(u) * a.d, lane, a.d, zu, false);
    double uu[K], acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { uu[k] = zu[k]; acc[k] = 0.0; }
    double lsum = 0.0;

    for (uint64_t e = e0; e < e1; e += 32) {
      const int cnt = int(umin64(32, e1 - e));
      uint32_t pk = 0;
      if (lane < cnt) pk = resolve(a.state, a.col[e + lane], j);
      accumulate_rows<K, VEC, 4, MON>(a.fp, true, pk, cnt, lane, a.d, a.zold, a.znew, uu, acc,
                                      lsum);
    }

    bool finish = true;
    if (nch > 1) {  // hub split: publish the partial, last arrival combines
      const size_t slot = size_t(a.part_off[u]) + c;
      double* P = a.partials + slot * a.d;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (L::valid(lane, k, a.d)) __stcg(P + L::col(lane, k), acc[k]);
      if (MON && lane == 0) __stcg(a.partial_loss + slot, lsum);
      __threadfence();
      __syncwarp();
      uint32_t last = 0;
      if (lane == 0) last = (atomicAdd(a.chunk_cnt + u, 1u) == nch - 1) ? 1u : 0u;
      finish = __shfl_sync(kFull, last, 0) != 0;
      if (finish) {
        __threadfence();
        const double* P0 = a.partials + size_t(a.part_off[u]) * a.d;
#pragma unroll
        for (int k = 0; k < K; ++k)
          acc[k] = L::valid(lane, k, a.d) ? __ldcg(P0 + L::col(lane, k)) : 0.0;
        if (MON) lsum = __ldcg(a.partial_loss + a.part_off[u]);
        for (uint32_t cc = 1; cc < nch; ++cc) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (L::valid(lane, k, a.d))
              acc[k] = __dadd_rn(acc[k], __ldcg(P0 + size_t(cc) * a.d + L::col(lane, k)));
          if (MON) lsum = __dadd_rn(lsum, __ldcg(a.partial_loss + a.part_off[u] + cc));
        }
        if (lane == 0) a.chunk_cnt[u] = 0;  // self-reset for the next epoch
      }
    }

    if (finish) {
      // shared negatives of batch j (sampling.cpp:59), after the context
      for (uint32_t k0 = 0; k0 < a.s; k0 += 32) {
        const int cnt = int(umin32(32, a.s - k0));
        uint32_t pk = 0;
        if (lane < cnt) pk = resolve(a.state, a.negs[size_t(j) * a.s + k0 + lane], j);
        accumulate_rows<K, VEC, 4, MON>(a.fp, false, pk, cnt, lane, a.d, a.zold, a.znew, uu,
                                        acc, lsum);
      }
      // g = float(acc) (trainer.cpp:140-145); z -= eta*g (trainer.cpp:173)
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
        atomicOr(a.state + u, 1u);  // publish: row u of Znew is final
      }
    }
    it = __shfl_sync(kFull, nxt, 0);
  }
}

__global__ void state_kernel(const uint32_t* __restrict__ perm, uint32_t* __restrict__ state,
                             uint32_t n, uint32_t b, uint64_t* __restrict__ cnt,
                             const uint64_t* __restrict__ rowptr, uint32_t chunk) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  if (p == n) { cnt[n] = 0; return; }
  const uint32_t u = perm[p];
  state[u] = (p / b) << 1;
  const uint64_t deg = rowptr[u + 1] - rowptr[u];
  cnt[p] = deg ? (deg + chunk - 1) / chunk : 1;
}

__global__ void items_kernel(const uint64_t* __restrict__ cnt, const uint64_t* __restrict__ off,
                             uint2* __restrict__ items, uint32_t n) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t o = off[p];
  for (uint32_t c = 0; c < cnt[p]; ++c) items[o + c] = make_uint2(p, c);
}

__global__ void negs_kernel(uint32_t* __restrict__ out, uint64_t nb, uint32_t s, uint32_t n,
                            uint64_t seed, uint32_t epoch, int sampler) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nb * s) return;
  const uint64_t j = t / s;
  const uint32_t k = uint32_t(t % s);
  out[t] = sampler == F2V_SAMPLER_PHILOX ? philox_negative(seed, epoch, j, 0, k, n)
                                         : splitmix_negative(seed, epoch, j, 0, 1, k, n);
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

// ------------------------------------------------------------ dispatch
template <bool MON>
void launch_step(Ctx& c, const StepArgs& a, uint32_t blocks) {
  const uint32_t d = a.d;
  cudaStream_t st = c.stream;
  if (d == 128) grad_step_kernel<4, true, MON><<<blocks, 256, 0, st>>>(a);
  else if (d == 256) grad_step_kernel<8, true, MON><<<blocks, 256, 0, st>>>(a);
  else if (d == 64) grad_step_kernel<2, true, MON><<<blocks, 256, 0, st>>>(a);
  else if (d == 32) grad_step_kernel<1, true, MON><<<blocks, 256, 0, st>>>(a);
  else if (d <= 32) grad_step_kernel<1, false, MON><<<blocks, 256, 0, st>>>(a);
  else if (d <= 64) grad_step_kernel<2, false, MON><<<blocks, 256, 0, st>>>(a);
  else if (d <= 128) grad_step_kernel<4, false, MON><<<blocks, 256, 0, st>>>(a);
  else if (d <= 256) grad_step_kernel<8, false, MON><<<blocks, 256, 0, st>>>(a);
  else if (d <= 512) grad_step_kernel<16, false, MON><<<blocks, 256, 0, st>>>(a);
  else grad_step_kernel<32, false, MON><<<blocks, 256, 0, st>>>(a);
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
}

template <int K, bool VEC, bool MON>
void launch_epoch_t(Ctx& c, const EpochArgs& a) {
  auto kern = epoch_kernel<K, VEC, MON>;
  int per_sm = 0;
  F2V_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, int(c.tune.threads), 0));
  if (per_sm < 1) per_sm = 1;
  const uint32_t warps_needed = a.nitems;
  uint32_t blocks = uint32_t(per_sm) * uint32_t(c.num_sms);
  const uint32_t need = (warps_needed * 32 + c.tune.threads - 1) / c.tune.threads;
  blocks = std::max(1u, std::min(blocks, need));
  kern<<<blocks, c.tune.threads, 0, c.stream>>>(a);
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

}  // namespace

// ====================================================== host-side launchers
ForceParams make_params(const f2v_force_model& m) {
  ForceParams p;
  p.kind = m.kind;
  p.has_cap = m.repulsion_cap > 0 ? 1 : 0;
  p.eps = double(m.epsilon);
  p.cap = double(m.repulsion_cap);
  return p;
}

void k_grad_minibatch(Ctx& c, uint32_t b, uint32_t s, const ForceParams& fp, bool want_loss) {
  StepArgs a;
  a.rowptr = c.rowptr.as<uint64_t>();
  a.col = c.col.as<uint32_t>();
  a.z = c.zcur();
  a.ids = c.ids.as<uint32_t>();
  a.negs = c.negs.as<uint32_t>();
  a.grads = c.grads.as<float>();
  a.vloss = c.vloss.as<double>();
  a.bad = c.bad.as<unsigned long long>();
  a.b = b;
  a.s = s;
  a.d = c.d;
  a.fp = fp;
  F2V_CUDA(cudaMemsetAsync(a.bad, 0xff, sizeof(unsigned long long), c.stream));
  if (b == 0) return;
  const uint32_t blocks = (b * 32 + 255) / 256;
  if (want_loss) launch_step<true>(c, a, blocks);
  else launch_step<false>(c, a, blocks);
}

void k_apply_update(Ctx& c, uint32_t b, float eta, bool unique_ids) {
  if (b == 0) return;
  if (unique_ids) {
    const uint64_t total = uint64_t(b) * c.d;
    apply_kernel<<<uint32_t((total + 255) / 256), 256, 0, c.stream>>>(
        c.zcur(), c.ids.as<uint32_t>(), c.grads.as<float>(), b, c.d, eta);
  } else {
    apply_seq_kernel<<<(c.d + 127) / 128, 128, 0, c.stream>>>(c.zcur(), c.ids.as<uint32_t>(),
                                                               c.grads.as<float>(), b, c.d, eta);
  }
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
}

double k_batch_loss_sum(Ctx& c, uint32_t b) {
  c.scratch.ensure(sizeof(double));
  sum_kernel<<<1, 1024, 0, c.stream>>>(c.vloss.as<double>(), b, c.scratch.as<double>());
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
  double out = 0.0;
  F2V_CUDA(cudaMemcpyAsync(&out, c.scratch.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  return out;
}

void k_uniform_embedding(Ctx& c, uint64_t seed, float lo, float hi, int keyed_init) {
  const uint64_t total = uint64_t(c.n) * c.d;
  uint64_t s0;
  double dlo, dhi;
  if (keyed_init) {  // init_embedding: keyed (seed,{0x11}), U(-0.5/d, 0.5/d)
    s0 = rng_keyed1(seed, kStreamInit);
    const double half = 0.5 / double(c.d);
    dlo = -half;
    dhi = half;
  } else {  // random_embedding: Rng(seed, 0), U(lo, hi)
    s0 = rng_init(seed, 0);
    dlo = lo;
    dhi = hi;
  }
  if (total == 0) return;
  uniform_kernel<<<uint32_t((total + 255) / 256), 256, 0, c.stream>>>(c.zcur(), total, s0, dlo,
                                                                     dhi);
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
}

// Static per-graph hub-splitting layout: partial slots for multi-chunk rows.
void k_prepare_graph(Ctx& c) {
  const uint32_t C = c.tune.chunk;
  std::vector<uint32_t> off(c.n, 0u);
  uint64_t slots = 0, items = 0;
  for (uint32_t u = 0; u < c.n; ++u) {
    const uint64_t deg = c.h_rowptr[u + 1] - c.h_rowptr[u];
    const uint64_t nch = deg ? (deg + C - 1) / C : 1;
    items += nch;
    if (nch > 1) {
      off[u] = uint32_t(slots);
      slots += nch;
    }
  }
  if (slots >= (1ull << 32)) fail(F2V_EUSAGE, "graph too large for hub-split bookkeeping");
  c.part_slots = slots;
  c.max_items = items;
  c.part_chunk = C;
  c.part_off.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  c.chunk_cnt.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  if (c.n) {
    F2V_CUDA(cudaMemcpyAsync(c.part_off.p, off.data(), sizeof(uint32_t) * c.n,
                             cudaMemcpyHostToDevice, c.stream));
    F2V_CUDA(cudaMemsetAsync(c.chunk_cnt.p, 0, sizeof(uint32_t) * c.n, c.stream));
  }
  F2V_CUDA(cudaStreamSynchronize(c.stream));
}

// Per-epoch preparation: perm (already in c.perm) -> state, work items,
// negatives of every batch.
void k_epoch_begin(Ctx& c, uint32_t b, uint32_t s, uint32_t epoch, uint64_t seed, int sampler) {
  const uint32_t n = c.n;
  const uint64_t nb = (uint64_t(n) + b - 1) / b;
  if (c.part_chunk != c.tune.chunk) k_prepare_graph(c);
  c.state.ensure(sizeof(uint32_t) * n);
  c.cnt.ensure(sizeof(uint64_t) * (n + 1));
  c.off.ensure(sizeof(uint64_t) * (n + 1));
  c.items.ensure(sizeof(uint2) * std::max<uint64_t>(c.max_items, 1));
  c.negs_all.ensure(sizeof(uint32_t) * std::max<uint64_t>(nb * s, 1));
  c.partials.ensure(sizeof(double) * std::max<uint64_t>(c.part_slots * c.d, 1));
  c.partial_loss.ensure(sizeof(double) * std::max<uint64_t>(c.part_slots, 1));
  c.ploss.ensure(sizeof(double) * std::max<uint32_t>(n, 1));
  c.counters.ensure(64);
  state_kernel<<<(n + 1 + 255) / 256, 256, 0, c.stream>>>(
      c.perm.as<uint32_t>(), c.state.as<uint32_t>(), n, b, c.cnt.as<uint64_t>(),
      c.rowptr.as<uint64_t>(), c.tune.chunk);
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
  size_t tmp = 0;
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.cnt.as<uint64_t>(),
                                         c.off.as<uint64_t>(), n + 1, c.stream));
  c.scan_tmp.ensure(tmp);
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp, c.cnt.as<uint64_t>(),
                                         c.off.as<uint64_t>(), n + 1, c.stream));
  ++c.launches;
  items_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(c.cnt.as<uint64_t>(), c.off.as<uint64_t>(),
                                                     c.items.as<uint2>(), n);
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
  const uint64_t tot = nb * s;
  negs_kernel<<<uint32_t((tot + 255) / 256), 256, 0, c.stream>>>(c.negs_all.as<uint32_t>(), nb, s,
                                                                n, seed, epoch, sampler);
  F2V_CUDA(cudaGetLastError());
  ++c.launches;
}

EpochResult k_epoch_run(Ctx& c, uint32_t b, uint32_t s, float eta, const ForceParams& fp,
                        bool monitor) {
  const int nxt = 1 - c.cur;
  c.z[nxt].ensure(sizeof(float) * size_t(c.n) * c.d);
  uint32_t* ctr = c.counters.as<uint32_t>();  // [0] next item, [2..3] bad (u64)
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
  a.items = c.items.as<uint2>();
  a.nitems = uint32_t(c.max_items);
  a.next = ctr;
  a.partials = c.partials.as<double>();
  a.partial_loss = c.partial_loss.as<double>();
  a.part_off = c.part_off.as<uint32_t>();
  a.chunk_cnt = c.chunk_cnt.as<uint32_t>();
  a.ploss = c.ploss.as<double>();
  a.bad = reinterpret_cast<unsigned long long*>(ctr + 2);
  a.n = c.n;
  a.d = c.d;
  a.b = b;
  a.s = s;
  a.chunk = c.tune.chunk;
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
  EpochResult r{~0ull, 0.0};
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
  r.bad_pos = host[1];
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
