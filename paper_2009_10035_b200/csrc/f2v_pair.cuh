// f2v_pair.cuh -- the per-pair force math of force_kernels.cpp:30-169 and the
// warp-level row accumulation shared by the step and epoch kernels.
//
// Layout: Z is row-major f32[n x d]; one warp owns
// one batch row; lane L holds K columns of every row it touches (VEC layout:
// columns [L*K, L*K+K), one 16-byte load per lane for d = 128), so a
// neighbour row is one fully coalesced 512-byte gather.  Dot products /
// distances are fp64 (warp butterfly), the per-pair term and the per-vertex
// accumulator are fp64 exactly as force_kernels.cpp:30-77 and
// trainer.cpp:124-138 compute them; every multiply and add is an explicit
// __d*_rn so the separate roundings of the reference survive (the files are
// also compiled with --fmad=false).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "f2v_internal.h"

namespace f2v {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

constexpr uint32_t kNewBit = 0x80000000u;

// Znew rows hold this NaN bit pattern until their final value is stored: a
// reader polls the row itself instead of a separate flag (one L2 round trip,
// no fence on the writer).  Finalised values are never this NaN.
constexpr uint32_t kSentinel = 0xffc0ffeeu;
#ifndef F2V_POLL_MAX_NS
#define F2V_POLL_MAX_NS 256
#endif

// STEP = 2 for rows written and read as 16-byte vectors (VEC, K % 4 == 0):
// aligned 8-byte halves are accessed atomically (the assumption NCCL's LL
// protocol also makes), so one float per half decides it.  Scalar layouts
// check every float.
template <int K, int STEP = 1>
__device__ __forceinline__ bool has_sentinel(const float (&v)[K]) {
  bool b = false;
#pragma unroll
  for (int k = 0; k < K; k += STEP) b |= __float_as_uint(v[k]) == kSentinel;
  return b;
}

// A row poll gives up after kPollLimit iterations (>= 2^28 x 32..256 ns of
// back-off: about a minute) and raises *stall (the row keeps its sentinel NaN);
// the host then reports F2V_ECUDA (a stalled or dead peer GPU) instead of the
// device trapping or hanging.  An iteration count, not %globaltimer: the poll
// loop is on the batch chain and inlined at every row-block site, and a clock
// read per iteration (or an out-of-line poll) cost config 2 10-80%.
constexpr uint32_t kPollLimit = 1u << 28;
static __device__ __noinline__ void poll_stalled(uint32_t* stall) {
  if (stall) atomicExch(stall, 1u);
}

// Relaxed (no L1 invalidation) global loads/stores for cross-warp flags; the
// data they guard is always read through L2 (ld.cg) after the flag is seen.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// force_kernels.hpp:25-29: x >= 0 -> 1 / (1 + e^-x), else e^x / (1 + e^x).
// Both branches are n / (1 + e) with e = exp(-|x|) (the same exp argument and
// the same two roundings), so one exp and one division serve both: the hot
// EXACT row function is instruction-fetch sensitive.
__device__ __forceinline__ double stable_sigmoid(double x) {
  const double e = exp(-fabs(x));
  return __ddiv_rn(x >= 0 ? 1.0 : e, __dadd_rn(1.0, e));
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
  // a Znew row: re-load until no lane sees the sentinel (warp-uniform loop).
  // A row that never arrives (a peer GPU stalled or died mid-epoch) gives up
  // after kPollDeadlineNs of wall time and raises *stall: the host reports
  // F2V_ECUDA instead of the device hanging or trapping.
  __device__ static __forceinline__ void poll(const float* row, int lane, uint32_t d,
                                              float (&v)[K], uint32_t* stall) {
    // exponential back-off (32 ns .. F2V_POLL_MAX_NS): spinning warps would
    // otherwise take issue slots from the warps streaming rows on the same SM
    uint32_t ns = 32, it = 0;
    while (__any_sync(kFull, it < kPollLimit && has_sentinel<K, (VEC && K % 4 == 0) ? 2 : 1>(v))) {
      __nanosleep(ns);
      ns = ns < F2V_POLL_MAX_NS ? 2 * ns : ns;
      load(row, lane, d, v, true);
      if (++it == kPollLimit) poll_stalled(stall);  // give up (the loop ends for every lane)
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
  // fp64 accumulator rows (hub partials): plain coalesced L2 stores / loads
  __device__ static __forceinline__ void store_acc(double* row, int lane, uint32_t d,
                                                   const double (&a)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (valid(lane, k, d)) __stcg(row + col(lane, k), a[k]);
  }
  __device__ static __forceinline__ void load_acc(const double* row, int lane, uint32_t d,
                                                  double (&a)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = valid(lane, k, d) ? __ldcg(row + col(lane, k)) : 0.0;
  }
  __device__ static __forceinline__ void add_acc(const double* row, int lane, uint32_t d,
                                                 double (&a)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (valid(lane, k, d)) a[k] = __dadd_rn(a[k], __ldcg(row + col(lane, k)));
  }
};

// ------------------------------------------------ TMA row ring (F2V_ROW_TMA)
// Each warp owns kRingStages x 8 row slots of 512 bytes in dynamic shared
// memory plus one mbarrier per stage.  A block of up to 8 neighbour rows is
// fetched by bulk async copies (cp.async.bulk global -> shared, completion
// counted in bytes on the stage's mbarrier; one row per lane 0..7), so the
// next block's gathers are in flight -- without registers -- while this
// block's pair math runs.  The copies read L2 like ld.cg; Znew rows still go
// through the sentinel check (and the poll on direct loads).
// Same-box A/B measurements (C3 epoch kernel):
//   EXACT, 1 stage (the next block streams into shared memory while this one
//   is reduced from registers), 2 CTAs/SM: 58.8 -> 56.3 ms  <- the default
//   EXACT, 2 stages: 62.6 ms at 2 CTAs/SM, 75.6 ms at 3 (the carve-out halves L1)
//   FAST, 2 stages: C3 30.6 -> 30.4 ms, C2 8.35 -> 9.03 ms (the bulk copies
//   bypass L1, where R-MAT's hub rows hit) -- FAST keeps register gathers.
#ifndef F2V_ROW_TMA_EXACT
#define F2V_ROW_TMA_EXACT 1
#endif
#ifndef F2V_ROW_TMA_FAST
#define F2V_ROW_TMA_FAST 0
#endif
#ifndef F2V_RING_STAGES
#define F2V_RING_STAGES 1  // 1: the next block streams in while this one is reduced from registers
#endif
constexpr int kRingStages = F2V_RING_STAGES;
constexpr uint32_t kRowBytes = 512;  // d = 128 rows (the ring serves the VEC K = 4 layouts)
constexpr uint32_t kRingWarpBytes = 128 + kRingStages * 8 * kRowBytes;  // barriers + slots

// EXACT d = 128 (rows_exact128): per warp, kXStages x 8 row slots filled by
// cp.async, the transposed-reduction scratch (8 pairs x 32 lane partials,
// row stride kXRedStride doubles: conflict-free 16-byte reads) and the 8
// pairs' coefficients.
#ifndef F2V_EXACT_V3
#define F2V_EXACT_V3 1
#endif

#ifndef F2V_XSTAGES
#define F2V_XSTAGES 1
#endif
constexpr uint32_t kXStages = F2V_XSTAGES;
constexpr uint32_t kXRedStride = 40;
constexpr uint32_t kXRedOff = kXStages * 8 * kRowBytes;
constexpr uint32_t kXCoefOff = kXRedOff + 8 * kXRedStride * 8;
constexpr uint32_t kXWarpBytes = kXCoefOff + 384;

// dynamic shared memory per warp of a kernel instantiated for this row layout
// (0 = none); kernels launch with kWarps x this and call ring_init
template <int K, bool VEC, bool FAST>
__host__ __device__ constexpr uint32_t warp_smem_bytes() {
  if (K == 1 && !VEC && !FAST) return 4 * 32 * 8;  // rows_lowd_exact's transpose block
  if (!(K == 4 && VEC)) return 0;
  if (FAST) return F2V_ROW_TMA_FAST ? kRingWarpBytes : 0;
  if (F2V_EXACT_V3) return kXWarpBytes;
  return F2V_ROW_TMA_EXACT ? kRingWarpBytes : 0;
}
template <int K, bool VEC, bool FAST>
__host__ __device__ constexpr bool uses_ring() {  // the TMA ring (mbarriers to initialise)
  return warp_smem_bytes<K, VEC, FAST>() == kRingWarpBytes;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
extern __shared__ __align__(128) uint8_t f2v_dsmem[];
// this warp's ring: [0, 8 S) mbarriers, [64] phase bits, slots from 128
__device__ __forceinline__ uint8_t* ring_base() {
  return f2v_dsmem + (threadIdx.x >> 5) * kRingWarpBytes;
}
__device__ __forceinline__ uint8_t* xstage_base() {
  return f2v_dsmem + (threadIdx.x >> 5) * kXWarpBytes;
}
#ifndef F2V_EXACT_LOAD
// rows_exact128 row fetch: 0 cp.async.cg staging (L2; the default), 1 cp.async.ca (through
// L1), 2 direct register loads.  Same-box A/B, C3 / C2 kernel ms: 35.0 / 16.9, 37.4 / 17.4,
// 39.6 / 17.1.
#define F2V_EXACT_LOAD 0
#endif
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
#if F2V_EXACT_LOAD == 1
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ring_init(int lane) {
  uint8_t* b = ring_base();
  if (lane == 0) {
    for (int s = 0; s < kRingStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b + 8 * s)));
    *reinterpret_cast<uint32_t*>(b + 64) = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}
// fetch rows (packed ids of rows k0..k0+7 of the call; nr <= 8 valid) into stage st
__device__ __forceinline__ void ring_issue(int st, uint32_t packed, int k0, int nr, int lane,
                                           const float* zold, const float* znew) {
  uint8_t* b = ring_base();
  const uint32_t bar = smem_addr(b + 8 * st);
  const uint32_t pk = __shfl_sync(kFull, packed, (k0 + (lane & 7)) & 31);
  if (lane == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(uint32_t(nr) * kRowBytes)
                 : "memory");
  if (lane < nr) {
    const float* src = ((pk & kNewBit) ? znew : zold) + size_t(pk & ~kNewBit) * (kRowBytes / 4);
    const uint32_t dst = smem_addr(b + 128 + (st * 8 + lane) * kRowBytes);
    // the slot's previous rows were read through the generic proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(kRowBytes), "r"(bar)
        : "memory");
  }
}
__device__ __forceinline__ void ring_wait(int st, uint32_t& ph) {
  const uint32_t bar = smem_addr(ring_base() + 8 * st);
  const uint32_t par = (ph >> st) & 1u;
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(par)
      : "memory");
  ph ^= 1u << st;
}
// row i of stage st into registers (lane holds columns 4 lane .. 4 lane + 3)
__device__ __forceinline__ void ring_read(int st, int i, int lane, float (&v)[4]) {
  const float4 t =
      *reinterpret_cast<const float4*>(ring_base() + 128 + (st * 8 + i) * kRowBytes + 16 * lane);
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}

// ------------------------------------------------------- per-pair terms
// Scalar part of one pair: out_j = coef * o_j              (sigmoid)
//                          out_j = coef * (u_j - o_j) * inv (distance kinds)
//                          out   = (coef, 0, ..., 0)       (coincident fallback)
// followed by  out_j *= scale  when clamped (force_kernels.cpp:69-77).
struct Term {
  double coef, inv, scale, r;  // r = the distance (distance kinds)
  bool dist, fallback, clamped;
  double loss;
};

// red = <u,o> (sigmoid) or ||u-o||^2 (distance kinds); nw2 = ||o||^2 for the
// clamped sigmoid repulsion (force_kernels.cpp:95).
template <bool MON>
__device__ __forceinline__ Term pair_term(int kind, const ForceParams& fp, bool attractive,
                                          double red, double nw2) {
  Term t{};
  t.scale = 1.0;
  if (kind == F2V_SIGMOID) {  // force_kernels.cpp:79-97
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
  if (kind == F2V_TDIST) {
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
      scalar = kind == F2V_FR ? __dmul_rn(r_raw, r_raw)
                              : (kind == F2V_FA ? r_raw : log1p(r_raw));
    } else {
      scalar = __ddiv_rn(-1.0, dmax(r_raw, fp.eps));
      clamp_it = true;
    }
  }
  t.coef = scalar;
  t.r = r_raw;
  t.fallback = r_raw < fp.eps;  // scaled_unit_diff, force_kernels.cpp:54-65
  t.inv = __ddiv_rn(1.0, r_raw);
  if (clamp_it && fp.has_cap) {
    const double m = fabs(scalar);
    t.clamped = !(m <= fp.cap || m == 0.0);
    if (t.clamped) t.scale = __ddiv_rn(fp.cap, m);
  }
  return t;
}

// The fp64 quotient x / t correctly rounded from inv = RN(1 / t): q = RN(x inv),
// the exact residual x - q t (one fma), one correction fma (Markstein's
// theorem: the result is RN(x / t) barring over/underflow).  Three fp64 ops
// instead of a ~20-instruction division per column; checked against __ddiv_rn
// (tests/test_gpu_parity.py::test_exact_quotient).
__device__ __forceinline__ double div_by(double x, double t, double inv) {
  const double q = __dmul_rn(x, inv);
  const double r = __fma_rn(-q, t, x);
  return __fma_rn(r, inv, q);
}

// acc += out(term) with the reference's rounding sequence.  w = the other
// row (sigmoid) or u - other (distance kinds), both exact in fp64.
template <int K>
__device__ __forceinline__ void accumulate(const Term& t, int lane, const double (&w)[K],
                                           double (&acc)[K]) {
  if (!t.dist) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double o = __dmul_rn(t.coef, w[k]);
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
    double o = div_by(__dmul_rn(t.coef, w[k]), t.r, t.inv);  // (c w) / t
    if (t.clamped) o = __dmul_rn(o, t.scale);
    acc[k] = __dadd_rn(acc[k], o);
  }
}

// Accumulate the pairs of `cnt` (<= 32) other-rows whose packed ids sit one per
// lane (bit 31 = read the coherent Znew buffer), in lane order, U at a time.
// EXACT: everything fp64 in the reference's operation order (bitwise parity
// in practice).  KIND < 0 = force kind chosen at run time.
// lsum is a per-lane loss partial: the caller warp-sums it.
template <int KIND, int K, bool VEC, int U, bool MON, bool ATT>
__device__ __forceinline__ void rows_exact(const ForceParams& fp, uint32_t packed, int cnt,
                                           int lane, uint32_t d, const float* __restrict__ zold,
                                           const float* __restrict__ znew, const float (&zu)[K],
                                           double (&acc)[K], double& lsum) {
  using L = Lay<K, VEC>;
  const int kind = KIND >= 0 ? KIND : fp.kind;
  const bool sig = kind == F2V_SIGMOID;
  double uu[K];
#pragma unroll
  for (int k = 0; k < K; ++k) uu[k] = zu[k];
  for (int k0 = 0; k0 < cnt; k0 += U) {
    float v[U][K];
    uint32_t pks[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t pk = __shfl_sync(kFull, packed, (k0 + i) & 31);
      pks[i] = pk;
      if (k0 + i < cnt) {
        const bool coh = (pk & kNewBit) != 0;
        L::load((coh ? znew : zold) + size_t(pk & ~kNewBit) * d, lane, d, v[i], coh);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) v[i][k] = 0.0f;
      }
    }
#pragma unroll
    for (int i = 0; i < U; ++i)  // Znew rows not yet final: poll
      if (k0 + i < cnt && (pks[i] & kNewBit))
        L::poll(znew + size_t(pks[i] & ~kNewBit) * d, lane, d, v[i], fp.stall);
    double w[U][K], red[U], nw[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      double s = 0.0, q = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double o = double(v[i][k]);
        if (sig) {
          w[i][k] = o;
          s = __dadd_rn(s, __dmul_rn(uu[k], o));
          if (!ATT) q = __dadd_rn(q, __dmul_rn(o, o));
        } else {
          w[i][k] = __dsub_rn(uu[k], o);
          s = __dadd_rn(s, __dmul_rn(w[i][k], w[i][k]));
        }
      }
      red[i] = s;
      nw[i] = q;
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) {
#pragma unroll
      for (int i = 0; i < U; ++i) {
        red[i] = __dadd_rn(red[i], __shfl_xor_sync(kFull, red[i], m));
        if (!ATT && sig) nw[i] = __dadd_rn(nw[i], __shfl_xor_sync(kFull, nw[i], m));
      }
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      if (k0 + i < cnt) {
        const Term t = pair_term<MON>(kind, fp, ATT, red[i], nw[i]);
        accumulate<K>(t, lane, w[i], acc);
        if (MON && lane == 0) lsum = __dadd_rn(lsum, t.loss);
      }
    }
  }
}

// ------------------------------------------------------------ FAST mode
// fp32 per-pair math (dot / distance, coefficient, axpy) with fp64
// accumulation: every block of 8 pairs is summed in fp32 registers and then
// added into the fp64 accumulator, so rounding error does not grow with the
// degree (fp32 dot + fp64 accumulate stays within
// ~3e-7 row-relative of the reference).  The 8 partial reductions of a block
// are reduced "transposed": 4+2+1 exchange rounds leave each 4-lane group with
// one pair's total, so the scalar force term of 8 pairs is evaluated once, in
// parallel, and broadcast back.
struct FastTerm {
  float q;     // out_j = q * w_j   (w = o for sigmoid, u - o otherwise)
  float fb;    // coincident fallback: out = (fb, 0, ..., 0), q = 0
  float loss;
};

template <int KIND, bool ATT, bool MON>
__device__ __forceinline__ FastTerm fast_term(const ForceParams& fp, float red, float nw2) {
  FastTerm t{0.f, 0.f, 0.f};
  const float eps = float(fp.eps), cap = float(fp.cap);
  if (KIND == F2V_SIGMOID) {  // force_kernels.cpp:79-97, 213-219
    const float x = red;
    const float e = __expf(-fabsf(x));
    const float inv = __fdividef(1.0f, 1.0f + e);
    if (ATT) {
      t.q = x >= 0.f ? -e * inv : -inv;  // sigma(x) - 1
      if (MON) t.loss = x >= 0.f ? log1pf(e) : -x + log1pf(e);
    } else {
      const float sg = x >= 0.f ? inv : e * inv;
      t.q = sg;
      if (fp.has_cap) {
        const float m = sg * sqrtf(nw2);
        if (!(m <= cap || m == 0.f)) t.q = sg * __fdividef(cap, m);
      }
      if (MON) t.loss = x >= 0.f ? x + log1pf(e) : log1pf(e);
    }
    return t;
  }
  const float s = red;
  if (KIND == F2V_TDIST && ATT) {  // force_kernels.cpp:99-107: (2t/(1+t^2)) (u-v)/t
    if (s < eps * eps) t.fb = 2.0f * sqrtf(s) / (1.0f + s);
    else t.q = __fdividef(2.0f, 1.0f + s);
    if (MON) t.loss = log1pf(s);
    return t;
  }
  const float r = sqrtf(s);
  float scalar;
  if (KIND == F2V_TDIST) {  // repulsive, force_kernels.cpp:109-119
    const float tt = fmaxf(r, eps);
    scalar = __fdividef(-2.0f, tt * (1.0f + tt * tt));
    if (MON) {
      const float tc = fmaxf(s, eps * eps);
      t.loss = -logf(__fdividef(tc, 1.0f + tc));
    }
  } else if (ATT) {  // table-II attraction, force_kernels.cpp:121-134
    scalar = KIND == F2V_FR ? s : (KIND == F2V_FA ? r : log1pf(r));
  } else {
    scalar = __fdividef(-1.0f, fmaxf(r, eps));
  }
  if (!ATT && fp.has_cap) {
    const float m = fabsf(scalar);
    if (!(m <= cap || m == 0.f)) scalar *= __fdividef(cap, m);
  }
  if (r < eps) t.fb = scalar;
  else t.q = __fdividef(scalar, r);
  return t;
}

// Transposed reduction of 8 per-lane partials: returns, on every lane, the
// warp total of partial number pair_of_lane(lane).
__device__ __forceinline__ float reduce8(float (&p)[8], int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool hi = lane & 16;
    const float send = hi ? p[i] : p[i + 4];
    const float keep = hi ? p[i + 4] : p[i];
    p[i] = keep + __shfl_xor_sync(kFull, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 8;
    const float send = hi ? p[i] : p[i + 2];
    const float keep = hi ? p[i + 2] : p[i];
    p[i] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  {
    const bool hi = lane & 4;
    const float send = hi ? p[0] : p[1];
    const float keep = hi ? p[1] : p[0];
    p[0] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  p[0] += __shfl_xor_sync(kFull, p[0], 2);
  p[0] += __shfl_xor_sync(kFull, p[0], 1);
  return p[0];
}
__device__ __forceinline__ int pair_of_lane(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}
__device__ __forceinline__ int lane_of_pair(int i) {
  return (((i >> 2) & 1) << 4) | (((i >> 1) & 1) << 3) | ((i & 1) << 2);
}

// One block of 8 loaded rows w (pairs k0..k0+7 of the call): transposed
// reduction, force term, fp32 axpy of the block, fp64 accumulate.
template <int KIND, int K, bool MON, bool ATT>
__device__ __forceinline__ void fast_block(const ForceParams& fp, int k0, int cnt, int lane,
                                           const float (&zu)[K], float (&w)[8][K],
                                           double (&acc)[K], double& lsum) {
  constexpr bool SIG = KIND == F2V_SIGMOID;
  const int pi = pair_of_lane(lane);
  float part[8], nrm[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float s = 0.f, q = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (SIG) {
        s = fmaf(zu[k], w[i][k], s);
        if (!ATT) q = fmaf(w[i][k], w[i][k], q);
      } else {
        w[i][k] = zu[k] - w[i][k];
        s = fmaf(w[i][k], w[i][k], s);
      }
    }
    part[i] = s;
    nrm[i] = q;
  }
  const float red = reduce8(part, lane);
  const float nr = (SIG && !ATT) ? reduce8(nrm, lane) : 0.f;
  const FastTerm t = fast_term<KIND, ATT, MON>(fp, red, nr);
  if (MON && (lane & 3) == 0 && k0 + pi < cnt) lsum = __dadd_rn(lsum, double(t.loss));
  float a32[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a32[k] = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float qi = __shfl_sync(kFull, t.q, lane_of_pair(i));
    const float fbi = SIG ? 0.f : __shfl_sync(kFull, t.fb, lane_of_pair(i));
    if (k0 + i < cnt) {
#pragma unroll
      for (int k = 0; k < K; ++k) a32[k] = fmaf(qi, w[i][k], a32[k]);
      if (!SIG && lane == 0) a32[0] += fbi;
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = __dadd_rn(acc[k], double(a32[k]));
}

// FAST, d = 128 (round 2): the same numerics as rows_fast / fast_block, with the
// per-row overheads the EXACT rewrite removed (profiles/r2_c3_fast_v2: 75 warp
// instructions per pair):
//  * no per-row predication: rows past the end repeat the last valid row with
//    a zero coefficient (the fp32 block sum starts at +0.0, so adding +-0.0
//    leaves it unchanged);
//  * every row is a plain cached 16-byte load through a per-lane row pointer
//    (two shuffles + one 64-bit add per row; no Zold / Znew flag per row): a
//    Znew row is written exactly once per launch, so the only stale line L1
//    can hold is one that still carries the sentinel, which the test below
//    catches;
//  * the sentinel test is the dot: a row that still holds the sentinel NaN
//    gives a NaN reduction, and only then are the block's Znew rows polled
//    through L2 and the dots recomputed.
// Measured and rejected on top of it (same-box A/B, C3 / C2 kernel ms; the
// default is 25.4 / 7.2): the next block staged in shared memory by cp.async.ca
// 25.3 / 7.7; the next block's gathers issued into a second register block
// before this block's math 29.0 / 11.8; 4 CTAs/SM at 64 registers 34.0 / 13.8;
// forcing the 3-CTA build 28.0 / 11.1 (the occupancy autotune picks 2 CTAs/SM on
// both graphs).  Every variant that puts more gathers in flight per SM loses:
// with power-law degrees L1 serves a large share of the row reads, and on a
// near-regular graph of the same size (tools/skew_probe.py) the kernel is
// slower (30.1 ms), not faster.
#ifndef F2V_FAST_V3
#define F2V_FAST_V3 1
#endif

template <int KIND, bool MON, bool ATT>
__device__ __forceinline__ void rows_fast128(const ForceParams& fp, uint32_t packed, int cnt,
                                             int lane, const float* __restrict__ zold,
                                             const float* __restrict__ znew,
                                             const float (&zu)[4], double (&acc)[4],
                                             double& lsum) {
  constexpr int K = 4;
  constexpr uint32_t d = 128;
  using L = Lay<K, true>;
  constexpr bool SIG = KIND == F2V_SIGMOID;
  if (cnt <= 0) return;
  const int pi = pair_of_lane(lane);
  const uint32_t pkc = __shfl_sync(kFull, packed, min(lane, cnt - 1));
  const char* mine = reinterpret_cast<const char*>(((pkc & kNewBit) ? znew : zold) +
                                                   size_t(pkc & ~kNewBit) * d);
  auto load_block = [&](int k0, float (&w)[8][K]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const char* src = reinterpret_cast<const char*>(
          __shfl_sync(kFull, reinterpret_cast<unsigned long long>(mine), (k0 + i) & 31));
      const float4 t = *reinterpret_cast<const float4*>(src + 16 * lane);
      w[i][0] = t.x; w[i][1] = t.y; w[i][2] = t.z; w[i][3] = t.w;
    }
  };
  auto compute_block = [&](int k0, float (&w)[8][K]) {
    float red, nr = 0.f;
    bool polled = false;
    for (;;) {
      float part[8], nrm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float s = 0.f, q = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (SIG) {
            s = fmaf(zu[k], w[i][k], s);
            if (!ATT) q = fmaf(w[i][k], w[i][k], q);
          } else {
            const float df = zu[k] - w[i][k];
            s = fmaf(df, df, s);
          }
        }
        part[i] = s;
        nrm[i] = q;
      }
      red = reduce8(part, lane);
      if (SIG && !ATT) nr = reduce8(nrm, lane);
      // a Znew row not yet final still holds the sentinel NaN -> NaN here
      if (polled || !__any_sync(kFull, red != red)) break;
      polled = true;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t pk = __shfl_sync(kFull, packed, min(k0 + i, cnt - 1));
        if (pk & kNewBit) {
          L::load(znew + size_t(pk & ~kNewBit) * d, lane, d, w[i], true);
          L::poll(znew + size_t(pk & ~kNewBit) * d, lane, d, w[i], fp.stall);
        }
      }
    }
    FastTerm t = fast_term<KIND, ATT, MON>(fp, red, nr);
    const bool valid = k0 + pi < cnt;
    if (MON && (lane & 3) == 0 && valid) lsum = __dadd_rn(lsum, double(t.loss));
    if (!valid) t.q = t.fb = 0.f;  // rows past the end: a zero coefficient on a finite row
    float a32[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a32[k] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float qi = __shfl_sync(kFull, t.q, lane_of_pair(i));
      if (SIG) {
#pragma unroll
        for (int k = 0; k < K; ++k) a32[k] = fmaf(qi, w[i][k], a32[k]);
      } else {
        const float fbi = __shfl_sync(kFull, t.fb, lane_of_pair(i));
#pragma unroll
        for (int k = 0; k < K; ++k) a32[k] = fmaf(qi, zu[k] - w[i][k], a32[k]);
        if (lane == 0) a32[0] += fbi;
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = __dadd_rn(acc[k], double(a32[k]));
  };
  for (int k0 = 0; k0 < cnt; k0 += 8) {
    float w[8][K];
    load_block(k0, w);
    compute_block(k0, w);
  }
}

#ifndef F2V_EXACT_REUSE
#define F2V_EXACT_REUSE 0  // EXACT: keep the block's rows converted to fp64 for the accumulate
#endif

#ifndef F2V_EXACT_PIPE
#define F2V_EXACT_PIPE 0  // EXACT: gather the next 8-row block during this one's math
#endif

#ifndef F2V_FAST_INFLIGHT
#define F2V_FAST_INFLIGHT 8  // row gathers in flight per warp (8; 16 measured slower)
#endif

// The rows of one call are gathered NB = F2V_FAST_INFLIGHT at a time (all
// loads issued before any block is reduced: 16 x 512 B in flight per warp),
// then reduced 8 at a time in order.
template <int KIND, int K, bool MON, bool ATT>
__device__ __forceinline__ void rows_fast(const ForceParams& fp, uint32_t packed, int cnt,
                                          int lane, uint32_t d, const float* __restrict__ zold,
                                          const float* __restrict__ znew, const float (&zu)[K],
                                          double (&acc)[K], double& lsum) {
  using L = Lay<K, true>;
  constexpr int NB = F2V_FAST_INFLIGHT;
  d = 32 * K;  // VEC layout: a compile-time row stride
#if F2V_ROW_TMA_FAST
  if constexpr (K == 4) {
    const int nblk = (cnt + 7) / 8;
    uint32_t* phw = reinterpret_cast<uint32_t*>(ring_base() + 64);
    uint32_t ph = *phw;
    for (int b = 0; b < nblk && b < kRingStages; ++b)
      ring_issue(b, packed, 8 * b, min(8, cnt - 8 * b), lane, zold, znew);
    for (int b = 0; b < nblk; ++b) {
      const int st = b % kRingStages, k0 = 8 * b;
      ring_wait(st, ph);
      float w[8][K];
      uint32_t pks[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        pks[i] = __shfl_sync(kFull, packed, (k0 + i) & 31);
        if (k0 + i < cnt) ring_read(st, i, lane, w[i]);
        else w[i][0] = w[i][1] = w[i][2] = w[i][3] = 0.0f;
      }
      __syncwarp();  // every lane has its rows: the stage takes the block after next
      if (b + kRingStages < nblk)
        ring_issue(st, packed, k0 + 8 * kRingStages, min(8, cnt - k0 - 8 * kRingStages), lane,
                   zold, znew);
      bool pend = false;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (k0 + i < cnt && (pks[i] & kNewBit)) pend |= has_sentinel<K, 2>(w[i]);
      if (__any_sync(kFull, pend)) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (k0 + i < cnt && (pks[i] & kNewBit))
            L::poll(znew + size_t(pks[i] & ~kNewBit) * d, lane, d, w[i], fp.stall);
      }
      fast_block<KIND, K, MON, ATT>(fp, k0, cnt, lane, zu, w, acc, lsum);
    }
    *phw = ph;
    return;
  }
#endif
  for (int k0 = 0; k0 < cnt; k0 += NB) {
    float w[NB / 8][8][K];
    uint32_t pks[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const uint32_t pk = __shfl_sync(kFull, packed, (k0 + i) & 31);
      pks[i] = pk;
      if (k0 + i < cnt) {
        const bool coh = (pk & kNewBit) != 0;
        L::load((coh ? znew : zold) + size_t(pk & ~kNewBit) * d, lane, d, w[i / 8][i % 8], coh);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) w[i / 8][i % 8][k] = 0.0f;
      }
    }
#pragma unroll
    for (int h = 0; h < NB / 8; ++h) {
      if (k0 + 8 * h >= cnt) break;
      // Znew rows not yet final: one vote for the block, then poll row by row
      bool pend = false;
#pragma unroll
      for (int i = 8 * h; i < 8 * h + 8; ++i)
        if (k0 + i < cnt && (pks[i] & kNewBit))
          pend |= has_sentinel<K, (K % 4 == 0) ? 2 : 1>(w[h][i % 8]);
      if (__any_sync(kFull, pend)) {
#pragma unroll
        for (int i = 8 * h; i < 8 * h + 8; ++i)
          if (k0 + i < cnt && (pks[i] & kNewBit))
            L::poll(znew + size_t(pks[i] & ~kNewBit) * d, lane, d, w[h][i % 8], fp.stall);
      }
      fast_block<KIND, K, MON, ATT>(fp, k0 + 8 * h, cnt, lane, zu, w[h], acc, lsum);
    }
  }
}

// ------------------------------------------------------- EXACT, transposed
// EXACT (fp64 in the reference's operation order) for the VEC layouts, 8
// pairs at a time: per-lane fp64 partial dots as in rows_exact, then a
// transposed fp64 reduction (4+2+1 exchange rounds leave each 4-lane group
// one pair's total), so the fp64 force term (exp / div / sqrt) of 8 pairs is
// evaluated once, in parallel, instead of redundantly on all 32 lanes; its
// coefficients are broadcast and every lane accumulates its columns pair by
// pair in the reference's order (accumulate<K>).  Only the cross-lane order
// of the dot reduction differs from rows_exact (both are fp64 trees).
__device__ __forceinline__ double reduce8d(double (&p)[8], int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool hi = lane & 16;
    const double send = hi ? p[i] : p[i + 4];
    const double keep = hi ? p[i + 4] : p[i];
    p[i] = __dadd_rn(keep, __shfl_xor_sync(kFull, send, 16));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 8;
    const double send = hi ? p[i] : p[i + 2];
    const double keep = hi ? p[i + 2] : p[i];
    p[i] = __dadd_rn(keep, __shfl_xor_sync(kFull, send, 8));
  }
  {
    const bool hi = lane & 4;
    const double send = hi ? p[0] : p[1];
    const double keep = hi ? p[1] : p[0];
    p[0] = __dadd_rn(keep, __shfl_xor_sync(kFull, send, 4));
  }
  p[0] = __dadd_rn(p[0], __shfl_xor_sync(kFull, p[0], 2));
  p[0] = __dadd_rn(p[0], __shfl_xor_sync(kFull, p[0], 1));
  return p[0];
}

// ------------------------------------------------- EXACT, d = 128 (round 2)
// The same arithmetic as rows_exact8 (fp64 in the reference's operation
// order, per-lane partial dots, a transposed reduction so each pair's force
// term is evaluated once per 4-lane group), restructured after the ncu
// capture profiles/r2_c3_exact_v3 (108 warp instructions per pair, 120 register
// moves and 56 sentinel compares per 8-row block, a warp-serialised 9-
// instruction loop per TMA row copy):
//  * the next block's 8 rows stream into shared memory with cp.async.cg (one
//    16-byte copy per lane per row, L2-coherent like ld.cg, no uniform-register
//    hand-off), waited on per block;
//  * no per-row predication: rows past the end of the call repeat the last
//    valid row with a zero coefficient (acc + 0.0 == acc: an accumulator that
//    starts at +0.0 never becomes -0.0 under round-to-nearest);
//  * the sentinel test is the dot itself: a row that still holds the sentinel
//    NaN gives a NaN reduction, and only then are the block's Znew rows polled
//    and the dots recomputed (a genuine NaN polls once and goes on);
//  * the 8 x 32 lane partials are transposed through shared memory (8 stores,
//    4 16-byte loads, 7 adds, two shuffle rounds) instead of a select-and-
//    shuffle network, and the 8 pairs' coefficients go back through shared
//    memory as broadcast loads instead of 16+ shuffles.
// Measured and rejected (same-box A/B, C3 kernel): two cp.async stages 36.1 ->
// 40.8 ms (the second stage's shared memory costs L1); 3 CTAs/SM at 80
// registers 53 ms (spills); issuing the first block of the row queue's NEXT
// call during this call's last block (cross-call prefetch) 35.3 -> 42.1 ms.
struct XCoef {
  double c[8], sc[8], tr[8], inv[8];
  int fl[8];
};
static_assert(sizeof(XCoef) <= 384, "coefficient block");


// sum over the 32 lanes of partial number pi = lane >> 2, on every lane:
// 8 x 32 partials through shared memory (conflict-free), then two rounds
__device__ __forceinline__ double reduce8x(double (&part)[8], double* red, int lane) {
#pragma unroll
  for (int i = 0; i < 8; ++i) red[i * kXRedStride + lane] = part[i];
  __syncwarp();
  const double2* rp =
      reinterpret_cast<const double2*>(red + (lane >> 2) * kXRedStride + (lane & 3) * 2);
  double2 t[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) t[q] = rp[q * 4];
  double s = __dadd_rn(__dadd_rn(__dadd_rn(t[0].x, t[0].y), __dadd_rn(t[1].x, t[1].y)),
                       __dadd_rn(__dadd_rn(t[2].x, t[2].y), __dadd_rn(t[3].x, t[3].y)));
  s = __dadd_rn(s, __shfl_xor_sync(kFull, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(kFull, s, 2));
  return s;
}

template <int KIND, bool MON, bool ATT>
__device__ __forceinline__ void rows_exact128(const ForceParams& fp, uint32_t packed, int cnt,
                                              int lane, const float* __restrict__ zold,
                                              const float* __restrict__ znew,
                                              const float (&zu)[4], double (&acc_io)[4],
                                              double& lsum_io) {
  static_assert(KIND >= 0, "compiled per force kind");
  constexpr int K = 4;
  constexpr uint32_t d = 128;
  using L = Lay<K, true>;
  constexpr bool SIG = KIND == F2V_SIGMOID;
  constexpr bool SCALED = !ATT;  // repulsive kinds may be clamped (a second multiply)
  if (cnt <= 0) return;
  uint8_t* base = xstage_base();
  const uint32_t slots = smem_addr(base) + 16 * lane;
  const float4* slotp = reinterpret_cast<const float4*>(base) + lane;
  double* red = reinterpret_cast<double*>(base + kXRedOff);
  XCoef* cf = reinterpret_cast<XCoef*>(base + kXCoefOff);
  const int pi = lane >> 2;
  double uu[K], acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uu[k] = zu[k];
    acc[k] = acc_io[k];
  }
  double lsum = lsum_io;
  // this lane's 16 bytes of the row whose id lane min(lane, cnt - 1) holds
  const uint32_t pkc = __shfl_sync(kFull, packed, min(lane, cnt - 1));
  const char* mine = reinterpret_cast<const char*>(((pkc & kNewBit) ? znew : zold) +
                                                   size_t(pkc & ~kNewBit) * d);
#if F2V_EXACT_LOAD != 2
  // blocks are issued strictly in order: the pointers rotate by 8 lanes per
  // block, so row i of the block being issued always sits in lane i (shuffles
  // with constant lanes, no per-row index arithmetic)
  unsigned long long rot = reinterpret_cast<unsigned long long>(mine);
  const int rot_src = (lane + 8) & 31;
  auto issue = [&](int, int st) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const char* src = reinterpret_cast<const char*>(__shfl_sync(kFull, rot, i));
      cp_async16(slots + (st * 8 + i) * kRowBytes, src + 16 * lane);
    }
    cp_async_commit();
    rot = __shfl_sync(kFull, rot, rot_src);
  };
#endif
  const int nblk = (cnt + 7) >> 3;
#if F2V_EXACT_LOAD != 2
#pragma unroll
  for (int b = 0; b < int(kXStages); ++b)
    if (b < nblk) issue(8 * b, b);
#endif
  for (int b = 0; b < nblk; ++b) {
    const int k0 = 8 * b, st = kXStages == 1 ? 0 : b % int(kXStages);
    float v[8][K];
#if F2V_EXACT_LOAD == 2
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const char* src = reinterpret_cast<const char*>(
          __shfl_sync(kFull, reinterpret_cast<unsigned long long>(mine), (k0 + i) & 31));
      const float4 t = *reinterpret_cast<const float4*>(src + 16 * lane);
      v[i][0] = t.x; v[i][1] = t.y; v[i][2] = t.z; v[i][3] = t.w;
    }
#else
    if (kXStages == 1 || b + int(kXStages) > nblk) cp_async_wait<0>();
    else cp_async_wait<int(kXStages) - 1>();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 t = slotp[(st * 8 + i) * (kRowBytes / 16)];
      v[i][0] = t.x; v[i][1] = t.y; v[i][2] = t.z; v[i][3] = t.w;
    }
    if (b + int(kXStages) < nblk) issue(k0 + 8 * int(kXStages), st);
#endif
    double w[8][K], red_p, nrm_p = 0.0;
    bool polled = false;
    for (;;) {
      // per-lane fp64 partial dot / distance of the 8 pairs.  Sigmoid: the
      // products of two floats are exact in fp64, so fma(u, o, s) rounds exactly
      // like the reference's separate multiply and add (force_kernels.cpp:30-34).
      double part[8], nrm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double s = 0.0, q = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double o = double(v[i][k]);
          if (SIG) {
            w[i][k] = o;
            s = __fma_rn(uu[k], o, s);
            if (!ATT) q = __fma_rn(o, o, q);
          } else {  // distance(): diff * diff may be inexact -> separate roundings
            w[i][k] = __dsub_rn(uu[k], o);
            s = __dadd_rn(s, __dmul_rn(w[i][k], w[i][k]));
          }
        }
        part[i] = s;
        nrm[i] = q;
      }
      red_p = reduce8x(part, red, lane);
      if (SIG && !ATT) {
        __syncwarp();
        nrm_p = reduce8x(nrm, red, lane);
      }
      // a Znew row not yet final still holds the sentinel NaN -> NaN here
      if (polled || !__any_sync(kFull, red_p != red_p)) break;
      polled = true;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t pk = __shfl_sync(kFull, packed, min(k0 + i, cnt - 1));
        if (pk & kNewBit) L::poll(znew + size_t(pk & ~kNewBit) * d, lane, d, v[i], fp.stall);
      }
      __syncwarp();
    }
    Term t = pair_term<MON>(KIND, fp, ATT, red_p, nrm_p);  // pair pi, once per 4-lane group
    const bool valid = k0 + pi < cnt;
    if (MON && (lane & 3) == 0 && valid) lsum = __dadd_rn(lsum, t.loss);
    if ((lane & 3) == 0) {  // rows past the end: a zero coefficient on a finite row
      cf->c[pi] = valid ? t.coef : 0.0;
      if (SCALED) cf->sc[pi] = t.clamped ? t.scale : 1.0;
      if (!SIG) {
        cf->tr[pi] = valid ? t.r : 1.0;
        cf->inv[pi] = valid ? t.inv : 1.0;
      }
      if (SCALED || !SIG)
        cf->fl[pi] = valid ? ((t.fallback ? 1 : 0) | (t.clamped ? 2 : 0)) : 0;
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double c = cf->c[i];
      const int f = (SCALED || !SIG) ? cf->fl[i] : 0;
      if (SIG) {  // out_j = c z_j (x scale): scale_into + clamp_magnitude
        if (SCALED && (f & 2)) {
          const double si = cf->sc[i];
#pragma unroll
          for (int k = 0; k < K; ++k)
            acc[k] = __dadd_rn(acc[k], __dmul_rn(__dmul_rn(c, w[i][k]), si));
        } else {
#pragma unroll
          for (int k = 0; k < K; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(c, w[i][k]));
        }
      } else {
        const double si = SCALED ? cf->sc[i] : 1.0;
        if (f & 1) {  // coincident: out = (c, 0, ..., 0) (scaled_unit_diff)
          if (lane == 0) {
            double o = c;
            if (f & 2) o = __dmul_rn(o, si);
            acc[0] = __dadd_rn(acc[0], o);
          }
          const double zero = (f & 2) ? __dmul_rn(0.0, si) : 0.0;
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (lane != 0 || k != 0) acc[k] = __dadd_rn(acc[k], zero);
        } else {  // out_j = (c (u_j - o_j)) / t (force_kernels.cpp:63-64)
          const double tr = cf->tr[i], inv = cf->inv[i];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            double o = div_by(__dmul_rn(c, w[i][k]), tr, inv);
            if (SCALED && (f & 2)) o = __dmul_rn(o, si);
            acc[k] = __dadd_rn(acc[k], o);
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) acc_io[k] = acc[k];
  lsum_io = lsum;
}

template <int KIND, int K, bool MON, bool ATT>
__device__ __forceinline__ void rows_exact8(const ForceParams& fp, uint32_t packed, int cnt,
                                            int lane, uint32_t d, const float* __restrict__ zold,
                                            const float* __restrict__ znew, const float (&zu)[K],
                                            double (&acc_io)[K], double& lsum_io) {
  static_assert(KIND >= 0, "the EXACT vector path is compiled per force kind");
  using L = Lay<K, true>;
  constexpr bool SIG = KIND == F2V_SIGMOID;
  // what a pair's term needs beyond its coefficient
  constexpr bool SCALED = !ATT;       // repulsive kinds may be clamped (a second multiply)
  const int pi = pair_of_lane(lane);
  d = 32 * K;  // VEC layout: a compile-time row stride
  // the caller's accumulators live in its stack frame (Rows::run is out of
  // line): work on register copies, written back once
  double uu[K], acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uu[k] = zu[k];
    acc[k] = acc_io[k];
  }
  double lsum = lsum_io;
  // one block = 8 rows: gather (one 16-byte load per lane per row), then
  // the fp64 pair math of the block
  auto load_block = [&](int k0, float (&v)[8][K], uint32_t (&pks)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t pk = __shfl_sync(kFull, packed, (k0 + i) & 31);
      pks[i] = pk;
      if (k0 + i < cnt) {
        const bool coh = (pk & kNewBit) != 0;
        L::load((coh ? znew : zold) + size_t(pk & ~kNewBit) * d, lane, d, v[i], coh);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) v[i][k] = 0.0f;
      }
    }
  };
  auto compute_block = [&](int k0, float (&v)[8][K], const uint32_t (&pks)[8]) {
    {  // Znew rows not yet final: one vote for the block, then poll row by row
      bool pend = false;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (k0 + i < cnt && (pks[i] & kNewBit))
          pend |= has_sentinel<K, (K % 4 == 0) ? 2 : 1>(v[i]);
      if (__any_sync(kFull, pend)) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (k0 + i < cnt && (pks[i] & kNewBit))
            L::poll(znew + size_t(pks[i] & ~kNewBit) * d, lane, d, v[i], fp.stall);
      }
    }
    // per-lane fp64 partial dot / distance of the 8 pairs.  Sigmoid: the
    // products of two floats are exact in fp64, so fma(u, o, s) rounds exactly
    // like the reference's separate multiply and add (force_kernels.cpp:30-34).
    double part[8], nrm[8];
#if F2V_EXACT_REUSE
    double ov[8][K];  // the converted rows, reused by the accumulate (one F2F per element)
#endif
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = 0.0, q = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double o = double(v[i][k]);
#if F2V_EXACT_REUSE
        ov[i][k] = o;
#endif
        if (SIG) {
          s = __fma_rn(uu[k], o, s);
          if (!ATT) q = __fma_rn(o, o, q);
        } else {  // distance(): diff * diff may be inexact -> separate roundings
          const double w = __dsub_rn(uu[k], o);
          s = __dadd_rn(s, __dmul_rn(w, w));
        }
      }
      part[i] = s;
      nrm[i] = q;
    }
    const double red = reduce8d(part, lane);
    const double nr = (SIG && !ATT) ? reduce8d(nrm, lane) : 0.0;
    const Term t = pair_term<MON>(KIND, fp, ATT, red, nr);  // pair pi, once per 4-lane group
    if (MON && (lane & 3) == 0 && k0 + pi < cnt) lsum = __dadd_rn(lsum, t.loss);
    // what each lane broadcasts: the coefficient, the clamp scale (1.0 when
    // not clamped, applied only when clamped), the distance and 1/distance
    const double sc = t.clamped ? t.scale : 1.0;
    const int fl = (t.fallback ? 1 : 0) | (t.clamped ? 2 : 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int src = lane_of_pair(i);
      const double c = __shfl_sync(kFull, t.coef, src);
      const int f = (SCALED || !SIG) ? __shfl_sync(kFull, fl, src) : 0;
      const double si = SCALED ? __shfl_sync(kFull, sc, src) : 1.0;
      if (k0 + i >= cnt) continue;
      if (SIG) {  // out_j = c z_j (x scale): scale_into + clamp_magnitude
#pragma unroll
        for (int k = 0; k < K; ++k) {
#if F2V_EXACT_REUSE
          double o = __dmul_rn(c, ov[i][k]);
#else
          double o = __dmul_rn(c, double(v[i][k]));
#endif
          if (SCALED && (f & 2)) o = __dmul_rn(o, si);
          acc[k] = __dadd_rn(acc[k], o);
        }
      } else {
        const double tr = __shfl_sync(kFull, t.r, src);
        const double inv = __shfl_sync(kFull, t.inv, src);
        if (f & 1) {  // coincident: out = (c, 0, ..., 0) (scaled_unit_diff)
          if (lane == 0) {
            double o = c;
            if (f & 2) o = __dmul_rn(o, si);
            acc[0] = __dadd_rn(acc[0], o);
          }
          const double zero = (f & 2) ? __dmul_rn(0.0, si) : 0.0;
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (lane != 0 || k != 0) acc[k] = __dadd_rn(acc[k], zero);
        } else {  // out_j = (c (u_j - o_j)) / t (force_kernels.cpp:63-64)
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const double w = __dsub_rn(uu[k], double(v[i][k]));
            double o = div_by(__dmul_rn(c, w), tr, inv);
            if (SCALED && (f & 2)) o = __dmul_rn(o, si);
            acc[k] = __dadd_rn(acc[k], o);
          }
        }
      }
    }
    };
#if F2V_ROW_TMA_EXACT
  if constexpr (K == 4) {  // the next block's rows stream into the shared-memory ring
    const int nblk = (cnt + 7) / 8;
    uint32_t* phw = reinterpret_cast<uint32_t*>(ring_base() + 64);
    uint32_t ph = *phw;
    for (int b = 0; b < nblk && b < kRingStages; ++b)
      ring_issue(b, packed, 8 * b, min(8, cnt - 8 * b), lane, zold, znew);
    for (int b = 0; b < nblk; ++b) {
      const int st = b % kRingStages, k0 = 8 * b;
      ring_wait(st, ph);
      float v[8][K];
      uint32_t pks[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        pks[i] = __shfl_sync(kFull, packed, (k0 + i) & 31);
        if (k0 + i < cnt) ring_read(st, i, lane, v[i]);
        else v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0.0f;
      }
      __syncwarp();
      if (b + kRingStages < nblk)
        ring_issue(st, packed, k0 + 8 * kRingStages, min(8, cnt - k0 - 8 * kRingStages), lane,
                   zold, znew);
      compute_block(k0, v, pks);
    }
    *phw = ph;
#pragma unroll
    for (int k = 0; k < K; ++k) acc_io[k] = acc[k];
    lsum_io = lsum;
    return;
  } else
#endif
#if F2V_EXACT_PIPE
  // software pipeline: the next block's gathers are in flight while this
  // block's fp64 math runs (two register blocks, no dynamic indexing)
  float va[8][K], vb[8][K];
  uint32_t pa[8], pb[8];
  load_block(0, va, pa);
  for (int k0 = 0; k0 < cnt; k0 += 16) {
    if (k0 + 8 < cnt) load_block(k0 + 8, vb, pb);
    compute_block(k0, va, pa);
    if (k0 + 8 >= cnt) break;
    if (k0 + 16 < cnt) load_block(k0 + 16, va, pa);
    compute_block(k0 + 8, vb, pb);
  }
#else
  for (int k0 = 0; k0 < cnt; k0 += 8) {
    float v[8][K];
    uint32_t pks[8];
    load_block(k0, v, pks);
    compute_block(k0, v, pks);
  }
#endif
#pragma unroll
  for (int k = 0; k < K; ++k) acc_io[k] = acc[k];
  lsum_io = lsum;
}

// ------------------------------------------------------- FAST low-d
// d <= kLowD (the 2-D layout config): rows are too narrow to fill a warp, so
// each lane owns one PAIR of the call -- its row (d floats) is one 8/16-byte
// load, the dot / distance and the force term are lane-local fp32 -- and the
// warp sums the d contribution columns of up to 32 pairs with a butterfly,
// flushed into the fp64 accumulators (lane c owns column c, the masked
// layout Lay<1, false>).  Same FAST numerics as rows_fast: fp32 pair math,
// fp32 block sums, fp64 accumulation.
constexpr int kLowD = 4;

template <int KIND, bool MON, bool ATT>
__device__ __forceinline__ void rows_lowd(const ForceParams& fp, uint32_t packed, int cnt,
                                          int lane, uint32_t d, const float* __restrict__ zold,
                                          const float* __restrict__ znew, const float (&zu1)[1],
                                          double (&acc1)[1], double& lsum) {
  constexpr bool SIG = KIND == F2V_SIGMOID;
  float zu[kLowD];
#pragma unroll
  for (int c = 0; c < kLowD; ++c) zu[c] = __shfl_sync(kFull, zu1[0], c);  // lane c = column c
  const bool mine = lane < cnt;
  const uint32_t pk = packed;
  const float* row = ((pk & kNewBit) ? znew : zold) + size_t(pk & ~kNewBit) * d;
  float w[kLowD];
  auto load = [&]() {
#pragma unroll
    for (int c = 0; c < kLowD; ++c)
      w[c] = (mine && c < int(d)) ? ((pk & kNewBit) ? __ldcg(row + c) : __ldg(row + c)) : 0.0f;
  };
  load();
  // Znew rows not yet final: re-load until no lane sees the sentinel
  auto pending = [&]() {
    bool b = false;
#pragma unroll
    for (int c = 0; c < kLowD; ++c) b |= __float_as_uint(w[c]) == kSentinel;
    return b && mine && (pk & kNewBit);
  };
  uint32_t ns = 32, it = 0;
  while (__any_sync(kFull, it < kPollLimit && pending())) {
    __nanosleep(ns);
    ns = ns < F2V_POLL_MAX_NS ? 2 * ns : ns;
    if (pending()) load();
    if (++it == kPollLimit) poll_stalled(fp.stall);  // give up (the loop ends for every lane)
  }
  float red = 0.f, nrm = 0.f;
#pragma unroll
  for (int c = 0; c < kLowD; ++c) {
    if (SIG) {
      red = fmaf(zu[c], w[c], red);
      if (!ATT) nrm = fmaf(w[c], w[c], nrm);
    } else {
      w[c] = zu[c] - w[c];
      red = fmaf(w[c], w[c], red);
    }
  }
  const FastTerm t = fast_term<KIND, ATT, MON>(fp, red, nrm);
  if (MON && mine) lsum = __dadd_rn(lsum, double(t.loss));
  float col[kLowD];
#pragma unroll
  for (int c = 0; c < kLowD; ++c) col[c] = mine ? t.q * w[c] : 0.f;
  if (!SIG && mine) col[0] += t.fb;
#pragma unroll
  for (int m = 16; m; m >>= 1)
#pragma unroll
    for (int c = 0; c < kLowD; ++c) col[c] += __shfl_xor_sync(kFull, col[c], m);
  float mycol = 0.f;
#pragma unroll
  for (int c = 0; c < kLowD; ++c)
    if (lane == c) mycol = col[c];
  if (lane < int(d)) acc1[0] = __dadd_rn(acc1[0], double(mycol));
}

// ------------------------------------------------------- EXACT low-d
// d <= kLowD at the reference's arithmetic (config 4 with precision = exact):
// the generic masked layout would spend a whole warp butterfly on two columns.
// Here each lane owns one PAIR: its row is one 8/16-byte load, the fp64 dot /
// distance runs over the columns sequentially -- exactly the reference's
// order (force_kernels.cpp:30-43), not a tree -- and the fp64 force term is
// lane-local.  The per-column accumulate has to stay in pair order
// (trainer.cpp:129-138): the 32 x d contributions are transposed through a
// 1 KB per-warp shared-memory block and lane c adds column c's in order (pairs
// past the end contribute +0.0: acc + 0.0 == acc, see rows_exact128).
constexpr uint32_t kLowdWarpBytes = kLowD * 32 * sizeof(double);
__device__ __forceinline__ double* lowd_base() {
  return reinterpret_cast<double*>(f2v_dsmem + (threadIdx.x >> 5) * kLowdWarpBytes);
}

template <int KIND, bool MON, bool ATT>
__device__ __forceinline__ void rows_lowd_exact(const ForceParams& fp, uint32_t packed, int cnt,
                                                int lane, uint32_t d,
                                                const float* __restrict__ zold,
                                                const float* __restrict__ znew,
                                                const float (&zu1)[1], double (&acc1)[1],
                                                double& lsum) {
  static_assert(KIND >= 0, "compiled per force kind");
  constexpr bool SIG = KIND == F2V_SIGMOID;
  double zu[kLowD];
#pragma unroll
  for (int c = 0; c < kLowD; ++c) zu[c] = double(__shfl_sync(kFull, zu1[0], c));  // lane c = column c
  const bool mine = lane < cnt;
  const uint32_t pk = packed;
  const float* row = ((pk & kNewBit) ? znew : zold) + size_t(pk & ~kNewBit) * d;
  float w[kLowD];
  auto load = [&]() {
#pragma unroll
    for (int c = 0; c < kLowD; ++c)
      w[c] = (mine && c < int(d)) ? ((pk & kNewBit) ? __ldcg(row + c) : __ldg(row + c)) : 0.0f;
  };
  load();
  auto pending = [&]() {
    bool b = false;
#pragma unroll
    for (int c = 0; c < kLowD; ++c) b |= __float_as_uint(w[c]) == kSentinel;
    return b && mine && (pk & kNewBit);
  };
  uint32_t ns = 32, it = 0;
  while (__any_sync(kFull, it < kPollLimit && pending())) {
    __nanosleep(ns);
    ns = ns < F2V_POLL_MAX_NS ? 2 * ns : ns;
    if (pending()) load();
    if (++it == kPollLimit) poll_stalled(fp.stall);
  }
  double x[kLowD], red = 0.0, nrm = 0.0;  // x = the other row (sigmoid) or u - other
#pragma unroll
  for (int c = 0; c < kLowD; ++c) {
    const double o = double(w[c]);
    if (SIG) {
      x[c] = o;
      if (c < int(d)) {
        red = __dadd_rn(red, __dmul_rn(zu[c], o));
        if (!ATT) nrm = __dadd_rn(nrm, __dmul_rn(o, o));
      }
    } else {
      x[c] = __dsub_rn(zu[c], o);
      if (c < int(d)) red = __dadd_rn(red, __dmul_rn(x[c], x[c]));
    }
  }
  const Term t = pair_term<MON>(KIND, fp, ATT, red, nrm);
  if (MON && mine) lsum = __dadd_rn(lsum, t.loss);
  double* buf = lowd_base();
#pragma unroll
  for (int c = 0; c < kLowD; ++c) {
    double o;
    if (!t.dist) {
      o = __dmul_rn(t.coef, x[c]);
    } else if (t.fallback) {  // coincident: out = (coef, 0, ..., 0) (scaled_unit_diff)
      o = c == 0 ? t.coef : 0.0;
    } else {
      o = div_by(__dmul_rn(t.coef, x[c]), t.r, t.inv);
    }
    if (t.clamped) o = __dmul_rn(o, t.scale);
    buf[c * 32 + lane] = (mine && c < int(d)) ? o : 0.0;
  }
  __syncwarp();
  if (lane < int(d)) {
    double a = acc1[0];
    const double* colp = buf + lane * 32;
    for (int i = 0; i < cnt; ++i) a = __dadd_rn(a, colp[i]);
    acc1[0] = a;
  }
  __syncwarp();
}

// The row-accumulation policy the epoch kernel is instantiated with.  run is
// out of line (one copy per (kind, attractive): the kernel is instruction-
// fetch sensitive); run_inl is the same body inlined at a hot call site.
template <int KIND, int K, bool VEC, bool MON, bool FAST>
struct Rows {
  template <bool ATT>
  __device__ static __forceinline__ void run_inl(const ForceParams& fp, uint32_t packed, int cnt,
                                                 int lane, uint32_t d, const float* zold,
                                                 const float* znew, const float (&zu)[K],
                                                 double (&acc)[K], double& lsum) {
    if constexpr (FAST && K == 1 && !VEC)
      rows_lowd<KIND, MON, ATT>(fp, packed, cnt, lane, d, zold, znew, zu, acc, lsum);
    else if constexpr (FAST && K == 4 && KIND >= 0 && F2V_FAST_V3 != 0 && F2V_ROW_TMA_FAST == 0)
      rows_fast128<KIND, MON, ATT>(fp, packed, cnt, lane, zold, znew, zu, acc, lsum);
    else if constexpr (FAST)
      rows_fast<KIND, K, MON, ATT>(fp, packed, cnt, lane, d, zold, znew, zu, acc, lsum);
    else if constexpr (VEC && KIND >= 0 && K == 4 && F2V_EXACT_V3 != 0)
      rows_exact128<KIND, MON, ATT>(fp, packed, cnt, lane, zold, znew, zu, acc, lsum);
    else if constexpr (!VEC && K == 1 && KIND >= 0) {
      if (d <= uint32_t(kLowD))
        rows_lowd_exact<KIND, MON, ATT>(fp, packed, cnt, lane, d, zold, znew, zu, acc, lsum);
      else
        rows_exact<KIND, K, VEC, 4, MON, ATT>(fp, packed, cnt, lane, d, zold, znew, zu, acc,
                                              lsum);
    }
    else if constexpr (VEC && KIND >= 0)
      rows_exact8<KIND, K, MON, ATT>(fp, packed, cnt, lane, d, zold, znew, zu, acc, lsum);
    else
      rows_exact<KIND, K, VEC, 4, MON, ATT>(fp, packed, cnt, lane, d, zold, znew, zu, acc,
                                            lsum);
  }
  // (fp by reference: by value measured C2 +10%, C3 EXACT +4% -- more
  // spills around the calls outweigh the local reads of the parameter block)
  template <bool ATT>
  __device__ static __noinline__ void run(const ForceParams& fp, uint32_t packed, int cnt,
                                          int lane, uint32_t d, const float* zold,
                                          const float* znew, const float (&zu)[K],
                                          double (&acc)[K], double& lsum) {
    run_inl<ATT>(fp, packed, cnt, lane, d, zold, znew, zu, acc, lsum);
  }
};

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int m = 16; m; m >>= 1) x = __dadd_rn(x, __shfl_xor_sync(kFull, x, m));
  return x;
}

}  // namespace dev
}  // namespace f2v
