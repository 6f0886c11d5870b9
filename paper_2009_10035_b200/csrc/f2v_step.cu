// f2v_step.cu -- the per-step operators of the reference seam on sm_100a:
// grad_minibatch (trainer.cpp:108-165), apply_update (167-175), batch_loss
// (177-190), plus the embedding initialisers (trainer.cpp:62-72,
// test_trainer.cpp:18-23) and a deterministic fixed-order fp64 sum.
// Each operates in place on the current Z; a grad launch never writes Z, so
// every read sees the pre-batch snapshot by construction.
#include "f2v_internal.h"
#include "f2v_pair.cuh"
#include "f2v_rng.h"

namespace f2v {
namespace {

using namespace dev;

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

// grad_minibatch: one warp per batch row, context arcs in CSR order then the
// shared negatives in sample order (trainer.cpp:129-138).
template <int K, bool VEC, bool MON>
__global__ void __launch_bounds__(256) grad_step_kernel(StepArgs a) {
  using L = Lay<K, VEC>;
  const int lane = threadIdx.x & 31;
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= a.b) return;
  const uint32_t u = a.ids[i];
  float zu[K];
  L::load(a.z + size_t(u) * a.d, lane, a.d, zu, false);
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  double lsum = 0.0;
  const uint64_t r0 = a.rowptr[u], r1 = a.rowptr[u + 1];
  for (uint64_t e = r0; e < r1; e += 32) {
    const int cnt = int(umin64(32, r1 - e));
    const uint32_t v = lane < cnt ? a.col[e + lane] : 0u;
    rows_exact<-1, K, VEC, 4, MON, true>(a.fp, v, cnt, lane, a.d, a.z, a.z, zu, acc, lsum);
  }
  for (uint32_t k0 = 0; k0 < a.s; k0 += 32) {
    const int cnt = int(umin32(32, a.s - k0));
    const uint32_t w = lane < cnt ? a.negs[k0 + lane] : 0u;
    rows_exact<-1, K, VEC, 4, MON, false>(a.fp, w, cnt, lane, a.d, a.z, a.z, zu, acc, lsum);
  }
  float g[K];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    g[k] = __double2float_rn(acc[k]);  // trainer.cpp:142
    if (L::valid(lane, k, a.d) && !isfinite(g[k])) bad = true;
  }
  L::store(a.grads + size_t(i) * a.d, lane, a.d, g);
  if (__any_sync(kFull, bad) && lane == 0) atomicMin(a.bad, (unsigned long long)i);
  if (MON) {
    const double tot = warp_sum_d(lsum);
    if (lane == 0) a.vloss[i] = tot;
  }
}

// apply_update, distinct ids: one thread per element (fp32 mul then sub).
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

// U(lo, hi) from a SplitMix stream, one draw per element in row-major order.
__global__ void uniform_kernel(float* z, uint64_t total, uint64_t s0, double lo, double hi) {
  const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= total) return;
  const double u = rng_uniform(rng_draw(s0, k));
  z[k] = __double2float_rn(__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u)));
}

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
  F2V_LAUNCHED(c.stream, "kernel");
  ++c.launches;
}

}  // namespace

// deterministic fixed-order sum of v[0..m): per-thread strided sequential
// sums, then a fixed tree (one block of 1024 threads).
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

ForceParams make_params(const f2v_force_model& m) {
  ForceParams p;
  p.kind = m.kind;
  p.has_cap = m.has_repulsion_cap ? 1 : 0;  // std::optional<float> (force_kernels.cpp:72)
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
  F2V_LAUNCHED(c.stream, "apply_seq_kernel");
  ++c.launches;
}

double k_batch_loss_sum(Ctx& c, uint32_t b) {
  c.scratch.ensure(sizeof(double));
  sum_kernel<<<1, 1024, 0, c.stream>>>(c.vloss.as<double>(), b, c.scratch.as<double>());
  F2V_LAUNCHED(c.stream, "sum_kernel");
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
  F2V_LAUNCHED(c.stream, "uniform_kernel");
  ++c.launches;
}

}  // namespace f2v
