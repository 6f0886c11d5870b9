// f2v_eval.cu -- SURVEY.md section 8(f) row 4: the evaluation step after
// training (proj/core/src/evaluation.cpp) on the device: k-means with
// k-means++ seeding and the modularity sweep (evaluation.cpp:323-473), binary
// logistic regression by full-batch gradient descent (evaluation.cpp:87-137)
// and the link-prediction / node-classification scoring built on it.
//
// Parity rule.  Every fp64 reduction whose order the reference fixes is
// reproduced in that order, so clusterings are bit-identical to the
// reference's (k-means has no transcendental):
//   * a distance / a logit is one thread's sequential loop over the columns
//     (sq_distance, evaluation.cpp:325-333; probability, :87-91), separate
//     multiply and add (the library is compiled with --fmad=false);
//   * sums over the points (inertia, the k-means++ total and its cumulative
//     scan, centroid sums, logistic-regression gradients) are sequential in
//     point order: one thread per output column walks the points in index
//     order (columns in parallel), scalar sums are one thread's loop with the
//     loads batched ahead of the dependent adds.
// The parallelism is over points (distances, logits) and over columns,
// clusters and one-vs-rest classes (sums); points are stored transposed
// (d x n) where a thread walks a row's columns, so those loads coalesce.
// Logistic regression calls exp (sigmoid): the device's is within 1 ulp of
// glibc's, so weights agree to ~1e-13 relative rather than bitwise.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <limits>

#include "f2v_internal.h"
#include "f2v_rng.h"

namespace f2v {
namespace ev {
namespace {

constexpr int kTB = 128;

inline unsigned grid_for(uint64_t n, int tb = kTB) {
  return unsigned(std::max<uint64_t>(1, (n + tb - 1) / tb));
}

// ---------------------------------------------------------------- layout
// xt[j * n + i] = x[row(i) * d + j]: a 32 x 32 shared-memory tile transpose;
// rows gathered through ids when given (features of a vertex subset).
__global__ void transpose_kernel(const float* __restrict__ x, const uint32_t* __restrict__ ids,
                                 uint64_t n, uint32_t d, float* __restrict__ xt) {
  __shared__ float tile[32][33];
  const uint64_t i0 = uint64_t(blockIdx.x) * 32;
  const uint32_t j0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const uint64_t i = i0 + r;
    const uint32_t j = j0 + threadIdx.x;
    if (i < n && j < d) tile[r][threadIdx.x] = x[size_t(ids ? ids[i] : i) * d + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const uint32_t j = j0 + r;
    const uint64_t i = i0 + threadIdx.x;
    if (i < n && j < d) xt[size_t(j) * n + i] = tile[threadIdx.x][r];
  }
}

// rows of x by id (row-major): the one-vs-rest training features
__global__ void gather_rows_kernel(const float* __restrict__ x, const uint32_t* __restrict__ ids,
                                   uint64_t n, uint32_t d, float* __restrict__ out) {
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n * d;
       t += uint64_t(gridDim.x) * blockDim.x)
    out[t] = x[size_t(ids[t / d]) * d + t % d];
}

// hadamard(z_u, z_v) (evaluation.cpp:17-23): fp32 products, row-major
__global__ void hadamard_kernel(const float* __restrict__ z, const uint32_t* __restrict__ pairs,
                                uint64_t m, uint32_t d, float* __restrict__ out) {
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < m * d;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = t / d;
    const uint32_t j = uint32_t(t % d);
    out[t] = __fmul_rn(z[size_t(pairs[3 * i]) * d + j], z[size_t(pairs[3 * i + 1]) * d + j]);
  }
}

// ---------------------------------------------------------------- k-means
// sq_distance (evaluation.cpp:325-333) of point i to centroid row c
__device__ __forceinline__ double sq_dist(const float* __restrict__ zt, uint64_t n, uint64_t i,
                                          const double* __restrict__ cen, uint32_t d) {
  double s = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    const double diff = __dsub_rn(double(zt[size_t(j) * n + i]), __ldg(cen + j));
    s = __dadd_rn(s, __dmul_rn(diff, diff));
  }
  return s;
}

// k-means++ round (evaluation.cpp:352-357): dist2[i] = min(dist2[i], |z_i - c|^2)
__global__ void seed_dist_kernel(const float* __restrict__ zt, uint64_t n, uint32_t d,
                                 const double* __restrict__ cen, double* __restrict__ dist2) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d2 = sq_dist(zt, n, i, cen, d);
  const double cur = dist2[i];
  dist2[i] = d2 < cur ? d2 : cur;  // std::min(dist2[i], d2)
}

// s += v[0..n) in index order: the loads of a block of 8 are independent, the
// adds are the reference's dependent chain
__device__ __forceinline__ double seq_sum(const double* __restrict__ v, uint64_t n, double s) {
  uint64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    double t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = v[i + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dadd_rn(s, t[q]);
  }
  for (; i < n; ++i) s = __dadd_rn(s, v[i]);
  return s;
}

// The draw of a k-means++ centre (evaluation.cpp:358-371) and its copy into
// centroid row c.  raw = the stream's next() value: uniform() * total when
// total > 0, else below(n) -- both consume exactly that one draw.
__global__ void seed_pick_kernel(const float* __restrict__ z, uint64_t n, uint32_t d,
                                 const double* __restrict__ dist2, uint64_t raw, int first,
                                 double* __restrict__ cen_row) {
  __shared__ uint64_t chosen_s;
  if (threadIdx.x == 0) {
    uint64_t chosen = 0;
    if (first) {
      chosen = rng_below(raw, n);
    } else {
      const double total = seq_sum(dist2, n, 0.0);
      if (total > 0) {
        double target = __dmul_rn(rng_uniform(raw), total);
        for (uint64_t i = 0; i < n; i += 8) {
          double t[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) t[q] = i + q < n ? dist2[i + q] : 0.0;
          bool hit = false;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (!hit && i + q < n) {
              target = __dsub_rn(target, t[q]);
              if (target <= 0) {
                chosen = i + q;
                hit = true;
              }
            }
          }
          if (hit) break;
        }
      } else {
        chosen = rng_below(raw, n);
      }
    }
    chosen_s = chosen;
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x)
    cen_row[j] = double(z[size_t(chosen_s) * d + j]);
}

// the assignment step (evaluation.cpp:381-392): first nearest centroid
__global__ void assign_kernel(const float* __restrict__ zt, uint64_t n, uint32_t d,
                              const double* __restrict__ cen, int k, int32_t* __restrict__ assign,
                              double* __restrict__ best_out, uint32_t* __restrict__ changed) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int best = 0;
  double best_d2 = std::numeric_limits<double>::infinity();
  for (int c = 0; c < k; ++c) {
    const double d2 = sq_dist(zt, n, i, cen + size_t(c) * d, d);
    if (d2 < best_d2) {
      best_d2 = d2;
      best = c;
    }
  }
  if (assign[i] != best) {
    assign[i] = best;
    *changed = 1u;
  }
  best_out[i] = best_d2;
}

// out[0] = sum of v in index order (the inertia, evaluation.cpp:391)
__global__ void seq_sum_kernel(const double* __restrict__ v, uint64_t n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = seq_sum(v, n, 0.0);
}

__global__ void fill_kernel(double* v, uint64_t n, double x) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = x;
}

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = uint32_t(i);
}

// off[c] = first position of cluster c in the sorted keys (c = 0..k)
__global__ void cluster_offsets_kernel(const uint32_t* __restrict__ keys, uint64_t n, int k,
                                       uint64_t* __restrict__ off) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > k) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (keys[mid] < uint32_t(c)) lo = mid + 1;
    else hi = mid;
  }
  off[c] = lo;
}

// The update step (evaluation.cpp:396-407): one CTA per cluster, one thread per
// column, members in point order.  Empty clusters keep their row and raise
// *any_empty (the host re-seeds them, evaluation.cpp:408-419).
__global__ void centroid_kernel(const float* __restrict__ z, uint32_t d,
                                const uint32_t* __restrict__ members,
                                const uint64_t* __restrict__ off, double* __restrict__ cen,
                                uint32_t* __restrict__ any_empty) {
  const int c = blockIdx.x;
  const uint64_t b = off[c], e = off[c + 1];
  if (b == e) {
    if (threadIdx.x == 0) *any_empty = 1u;
    return;
  }
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    uint64_t t = b;
    for (; t + 4 <= e; t += 4) {
      float v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = z[size_t(members[t + q]) * d + j];
#pragma unroll
      for (int q = 0; q < 4; ++q) s = __dadd_rn(s, double(v[q]));
    }
    for (; t < e; ++t) s = __dadd_rn(s, double(z[size_t(members[t]) * d + j]));
    cen[size_t(c) * d + j] = __ddiv_rn(s, double(e - b));  // sums / sizes[c]
  }
}

// distance of every point to the centroid of its own cluster, where clusters
// below `split` read cen_new and the others cen_old: the half-updated centroid
// array the reference's in-place loop sees at an empty cluster
__global__ void own_dist_kernel(const float* __restrict__ zt, uint64_t n, uint32_t d,
                                const int32_t* __restrict__ assign,
                                const double* __restrict__ cen_new,
                                const double* __restrict__ cen_old, int split,
                                double* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = assign[i];
  out[i] = sq_dist(zt, n, i, (a < split ? cen_new : cen_old) + size_t(a) * d, d);
}

// first index of the maximum (evaluation.cpp:411-416: strict >, from -1) and the
// copy of that point into centroid row cen_row.  One CTA.
__global__ void farthest_kernel(const float* __restrict__ z, uint64_t n, uint32_t d,
                                const double* __restrict__ v, double* __restrict__ cen_row) {
  __shared__ double sv[1024];
  __shared__ uint64_t si[1024];
  double bv = -1.0;
  uint64_t bi = 0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
    if (v[i] > bv) {
      bv = v[i];
      bi = i;
    }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s; s >>= 1) {
    if (int(threadIdx.x) < s) {
      const double ov = sv[threadIdx.x + s];
      const uint64_t oi = si[threadIdx.x + s];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  // a maximum that never beat -1.0 keeps the reference's index 0
  const uint64_t far = sv[0] > -1.0 ? si[0] : 0;
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x)
    cen_row[j] = double(z[size_t(far) * d + j]);
}

// modularity tallies (evaluation.cpp:441-449): integers, any order
__global__ void modularity_kernel(const uint64_t* __restrict__ rowptr,
                                  const uint32_t* __restrict__ col, uint32_t n,
                                  const int32_t* __restrict__ assign,
                                  unsigned long long* __restrict__ intra,
                                  unsigned long long* __restrict__ degsum) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u = w; u < n; u += nw) {
    const int cu = assign[u];
    const uint64_t b = rowptr[u], e = rowptr[u + 1];
    unsigned long long in = 0;
    for (uint64_t t = b + lane; t < e; t += 32) in += assign[col[t]] == cu ? 1u : 0u;
    for (int m = 16; m; m >>= 1) in += __shfl_xor_sync(0xffffffffu, in, m);
    if (lane == 0) {
      if (in) atomicAdd(intra + cu, in);
      if (e > b) atomicAdd(degsum + cu, (unsigned long long)(e - b));
    }
  }
}

// ------------------------------------------------------- logistic regression
// stable_sigmoid (force_kernels.hpp:25-29)
__device__ __forceinline__ double sigmoid(double x) {
  if (x >= 0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
  const double e = exp(x);
  return __ddiv_rn(e, __dadd_rn(1.0, e));
}

// LogRegModel::probability (evaluation.cpp:87-91) of row i for model m:
// s = bias, then s += w_j * x_j in column order
__device__ __forceinline__ double logit_prob(const float* __restrict__ xt, uint64_t n, uint64_t i,
                                             const double* __restrict__ w, uint32_t d) {
  double s = __ldg(w + d);
  for (uint32_t j = 0; j < d; ++j)
    s = __dadd_rn(s, __dmul_rn(__ldg(w + j), double(xt[size_t(j) * n + i])));
  return sigmoid(s);
}

// err[m][i] = p_m(x_i) - target_m(i) (evaluation.cpp:108); targets are
// bit m of a row's class mask when cls != nullptr... kept simple: tgt[m*n + i]
__global__ void logreg_err_kernel(const float* __restrict__ xt, uint64_t n, uint32_t d,
                                  const double* __restrict__ w, const uint8_t* __restrict__ tgt,
                                  double* __restrict__ err) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t m = blockIdx.y;
  if (i >= n) return;
  const double p = logit_prob(xt, n, i, w + size_t(m) * (d + 1), d);
  err[size_t(m) * n + i] = __dsub_rn(p, double(tgt[size_t(m) * n + i]));
}

// The gradient and the weight update of one iteration (evaluation.cpp:104-116):
// one CTA per model, one thread per weight, rows in order:
// grad_j += err_i * x_ij; w_j -= lr (grad_j / n + l2 w_j); the bias is not
// regularised and is updated as (lr * grad_d) * inv_n.
__global__ void logreg_step_kernel(const float* __restrict__ x, uint64_t n, uint32_t d,
                                   const double* __restrict__ err, double* __restrict__ w,
                                   double lr, double l2) {
  const uint32_t m = blockIdx.x;
  const double* e = err + size_t(m) * n;
  double* wm = w + size_t(m) * (d + 1);
  const double inv_n = __ddiv_rn(1.0, double(n));
  for (uint32_t j = threadIdx.x; j <= d; j += blockDim.x) {
    double g = 0.0;
    if (j < d) {
      uint64_t i = 0;
      for (; i + 8 <= n; i += 8) {
        float xv[8];
        double ev[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          xv[q] = x[size_t(i + q) * d + j];
          ev[q] = e[i + q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) g = __dadd_rn(g, __dmul_rn(ev[q], double(xv[q])));
      }
      for (; i < n; ++i) g = __dadd_rn(g, __dmul_rn(e[i], double(x[size_t(i) * d + j])));
      wm[j] = __dsub_rn(wm[j], __dmul_rn(lr, __dadd_rn(__dmul_rn(g, inv_n), __dmul_rn(l2, wm[j]))));
    } else {
      g = seq_sum(e, n, 0.0);
      wm[d] = __dsub_rn(wm[d], __dmul_rn(__dmul_rn(lr, g), inv_n));
    }
  }
}

// The same step with the rows streamed through shared memory: tiles of R rows
// (contiguous R x d floats) and their R errors are copied in by cp.async, double
// buffered, while the previous tile is accumulated -- the per-row cost drops
// from a global-load latency (~175 ns/row measured) to the dependent fp64 add.
// Same sums in the same order as logreg_step_kernel.
__global__ void logreg_step_tiled_kernel(const float* __restrict__ x, uint64_t n, uint32_t d,
                                         const double* __restrict__ err, double* __restrict__ w,
                                         double lr, double l2, uint32_t R) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t m = blockIdx.x, j = threadIdx.x;
  const double* e = err + size_t(m) * n;
  double* wm = w + size_t(m) * (d + 1);
  const size_t tile_bytes = size_t(R) * d * sizeof(float);
  float* tile[2] = {reinterpret_cast<float*>(smem), reinterpret_cast<float*>(smem + tile_bytes)};
  double* et[2] = {reinterpret_cast<double*>(smem + 2 * tile_bytes),
                   reinterpret_cast<double*>(smem + 2 * tile_bytes) + R};
  const uint64_t ntiles = (n + R - 1) / R;
  auto load = [&](uint64_t t, int b) {
    const uint64_t r0 = t * R;
    const uint32_t rows = uint32_t(min(uint64_t(R), n - r0));
    const size_t bytes = size_t(rows) * d * sizeof(float);
    const char* src = reinterpret_cast<const char*>(x + r0 * d);
    if (bytes % 16 == 0) {
      const uint32_t dst = uint32_t(__cvta_generic_to_shared(tile[b]));
      for (size_t off = size_t(threadIdx.x) * 16; off < bytes; off += size_t(blockDim.x) * 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + uint32_t(off)),
                     "l"(src + off)
                     : "memory");
    } else {  // a ragged last tile
      for (size_t q = threadIdx.x; q < size_t(rows) * d; q += blockDim.x)
        tile[b][q] = x[r0 * d + q];
    }
    for (uint32_t r = threadIdx.x; r < rows; r += blockDim.x) et[b][r] = e[r0 + r];
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double g = 0.0;
  if (ntiles) load(0, 0);
  for (uint64_t t = 0; t < ntiles; ++t) {
    const int b = int(t & 1);
    if (t + 1 < ntiles) {
      load(t + 1, b ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint32_t rows = uint32_t(min(uint64_t(R), n - t * R));
    if (j < d) {
      const float* col = tile[b] + j;
#pragma unroll 4
      for (uint32_t r = 0; r < rows; ++r)
        g = __dadd_rn(g, __dmul_rn(et[b][r], double(col[size_t(r) * d])));
    } else if (j == d) {
#pragma unroll 4
      for (uint32_t r = 0; r < rows; ++r) g = __dadd_rn(g, et[b][r]);
    }
    __syncthreads();  // the buffer is refilled two tiles on
  }
  const double inv_n = __ddiv_rn(1.0, double(n));
  if (j < d)
    wm[j] = __dsub_rn(wm[j], __dmul_rn(lr, __dadd_rn(__dmul_rn(g, inv_n), __dmul_rn(l2, wm[j]))));
  else if (j == d)
    wm[d] = __dsub_rn(wm[d], __dmul_rn(__dmul_rn(lr, g), inv_n));
}

// prob[i * M + m] = p_m(x_i) (test rows; row-major over models for the host ranking)
__global__ void logreg_prob_kernel(const float* __restrict__ xt, uint64_t n, uint32_t d,
                                   const double* __restrict__ w, uint32_t M,
                                   double* __restrict__ prob) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t m = blockIdx.y;
  if (i >= n) return;
  prob[i * M + m] = logit_prob(xt, n, i, w + size_t(m) * (d + 1), d);
}

// per-row loss term of logreg_loss (evaluation.cpp:141-147)
__global__ void logreg_loss_kernel(const float* __restrict__ xt, uint64_t n, uint32_t d,
                                   const double* __restrict__ w, const uint8_t* __restrict__ tgt,
                                   double* __restrict__ term) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double p = logit_prob(xt, n, i, w, d);
  const double eps = 1e-15;
  const double a = tgt[i] ? p : __dsub_rn(1.0, p);
  term[i] = log(a < eps ? eps : a);  // std::max(., eps)
}

// loss -= term_i in row order
__global__ void seq_neg_sum_kernel(const double* __restrict__ v, uint64_t n, double* out) {
  if (threadIdx.x || blockIdx.x) return;
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s = __dsub_rn(s, v[i]);
  out[0] = s;
}

// link-prediction test pass (evaluation.cpp:165-171): predicted = p >= 0.5
__global__ void link_correct_kernel(const float* __restrict__ ft, uint64_t m, uint32_t d,
                                    const double* __restrict__ w,
                                    const uint32_t* __restrict__ pairs,
                                    unsigned long long* __restrict__ correct) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool ok = false;
  if (i < m) ok = (logit_prob(ft, m, i, w, d) >= 0.5) == (pairs[3 * i + 2] != 0);
  const unsigned b = __ballot_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(correct, (unsigned long long)__popc(b));
}

void transpose(Ctx& c, const float* x, const uint32_t* ids, uint64_t n, uint32_t d, float* xt) {
  if (!n) return;
  dim3 grid(unsigned((n + 31) / 32), (d + 31) / 32), block(32, 8);
  transpose_kernel<<<grid, block, 0, c.stream>>>(x, ids, n, d, xt);
  F2V_LAUNCHED(c.stream, "transpose_kernel");
  ++c.launches;
}

}  // namespace

// ------------------------------------------------------------------ k-means
struct KmeansWork {
  DeviceBuf zt, cen, cen_new, dist2, assign, keys, keys2, idx, idx2, off, sorttmp, flags;
  size_t sort_bytes = 0;
  ~KmeansWork() {
    for (DeviceBuf* b : {&zt, &cen, &cen_new, &dist2, &assign, &keys, &keys2, &idx, &idx2, &off,
                         &sorttmp, &flags})
      b->release();
  }
};

// members of each cluster in point order + the cluster offsets, then the
// centroid update into `out` (rows of empty clusters untouched)
static void update_centroids(Ctx& c, KmeansWork& w, const float* z, uint64_t n, uint32_t d, int k,
                             const int32_t* assign, double* out, uint32_t* any_empty) {
  int bits = 1;
  while ((1ll << bits) < k) ++bits;
  iota_kernel<<<grid_for(n), kTB, 0, c.stream>>>(w.idx.as<uint32_t>(), n);
  F2V_LAUNCHED(c.stream, "iota_kernel");
  F2V_CUDA(cub::DeviceRadixSort::SortPairs(
      w.sorttmp.p, w.sort_bytes, reinterpret_cast<const uint32_t*>(assign), w.keys2.as<uint32_t>(),
      w.idx.as<uint32_t>(), w.idx2.as<uint32_t>(), n, 0, bits, c.stream));
  cluster_offsets_kernel<<<grid_for(uint64_t(k) + 1), kTB, 0, c.stream>>>(
      w.keys2.as<uint32_t>(), n, k, w.off.as<uint64_t>());
  F2V_LAUNCHED(c.stream, "cluster_offsets_kernel");
  centroid_kernel<<<k, std::min<uint32_t>(1024, std::max<uint32_t>(32, (d + 31) / 32 * 32)), 0,
                    c.stream>>>(z, d, w.idx2.as<uint32_t>(), w.off.as<uint64_t>(), out, any_empty);
  F2V_LAUNCHED(c.stream, "centroid_kernel");
  c.launches += 4;
}

static void kmeans_alloc(Ctx& c, KmeansWork& w, const float* z, uint64_t n, uint32_t d, int k) {
  w.zt.ensure(sizeof(float) * n * d);
  w.cen.ensure(sizeof(double) * size_t(k) * d);
  w.cen_new.ensure(sizeof(double) * size_t(k) * d);
  w.dist2.ensure(sizeof(double) * n);
  w.assign.ensure(sizeof(int32_t) * n);
  w.keys2.ensure(sizeof(uint32_t) * n);
  w.idx.ensure(sizeof(uint32_t) * n);
  w.idx2.ensure(sizeof(uint32_t) * n);
  w.off.ensure(sizeof(uint64_t) * (size_t(k) + 1));
  w.flags.ensure(64);
  size_t bytes = 0;
  F2V_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, n, 0, 32, c.stream));
  w.sorttmp.ensure(bytes);
  w.sort_bytes = bytes;
  transpose(c, z, nullptr, n, d, w.zt.as<float>());
}

// lloyd_once (evaluation.cpp:340-424): assignment left in w.assign, returns the inertia
static double lloyd_once(Ctx& c, KmeansWork& w, const float* z, uint64_t n, uint32_t d, int k,
                         uint64_t& rng, int max_iters) {
  const float* zt = w.zt.as<float>();
  double* cen = w.cen.as<double>();
  double* dist2 = w.dist2.as<double>();
  int32_t* assign = w.assign.as<int32_t>();
  // flags: [0] changed, [1] any_empty (u32), inertia at byte 8
  uint32_t* flags = w.flags.as<uint32_t>();
  double* inertia_dev = reinterpret_cast<double*>(w.flags.as<uint8_t>() + 8);
  auto next = [&]() {
    rng += kGamma;
    return mix64(rng);
  };
  {  // k-means++ seeding, queued without a host round trip
    fill_kernel<<<grid_for(n), kTB, 0, c.stream>>>(dist2, n,
                                                   std::numeric_limits<double>::infinity());
    F2V_LAUNCHED(c.stream, "fill_kernel");
    seed_pick_kernel<<<1, kTB, 0, c.stream>>>(z, n, d, dist2, next(), 1, cen);
    F2V_LAUNCHED(c.stream, "seed_pick_kernel");
    ++c.launches;
    for (int cc = 1; cc < k; ++cc) {
      seed_dist_kernel<<<grid_for(n), kTB, 0, c.stream>>>(zt, n, d, cen + size_t(cc - 1) * d,
                                                          dist2);
      F2V_LAUNCHED(c.stream, "seed_dist_kernel");
      seed_pick_kernel<<<1, kTB, 0, c.stream>>>(z, n, d, dist2, next(), 0, cen + size_t(cc) * d);
      F2V_LAUNCHED(c.stream, "seed_pick_kernel");
      c.launches += 2;
    }
  }
  F2V_CUDA(cudaMemsetAsync(assign, 0xff, sizeof(int32_t) * n, c.stream));  // -1
  double inertia = std::numeric_limits<double>::infinity();
  for (int it = 0; it < max_iters; ++it) {
    F2V_CUDA(cudaMemsetAsync(flags, 0, 8, c.stream));
    assign_kernel<<<grid_for(n), kTB, 0, c.stream>>>(zt, n, d, cen, k, assign, dist2, flags);
    F2V_LAUNCHED(c.stream, "assign_kernel");
    seq_sum_kernel<<<1, 32, 0, c.stream>>>(dist2, n, inertia_dev);
    F2V_LAUNCHED(c.stream, "seq_sum_kernel");
    c.launches += 2;
    // the update is queued before the host learns whether this was the last
    // iteration: it changes only the centroids, which are not an output
    F2V_CUDA(cudaMemcpyAsync(w.cen_new.p, cen, sizeof(double) * size_t(k) * d,
                             cudaMemcpyDeviceToDevice, c.stream));
    update_centroids(c, w, z, n, d, k, assign, w.cen_new.as<double>(), flags + 1);
    struct {
      uint32_t changed, any_empty;
      double inertia;
    } h;
    F2V_CUDA(cudaMemcpyAsync(&h, flags, 16, cudaMemcpyDeviceToHost, c.stream));
    F2V_CUDA(cudaStreamSynchronize(c.stream));
    inertia = h.inertia;
    if (!h.changed && it > 0) break;
    if (h.any_empty) {
      // re-seed each empty cluster, in cluster order, at the point farthest
      // from its own centroid in the half-updated array (evaluation.cpp:408-419)
      std::vector<uint64_t> off(size_t(k) + 1);
      F2V_CUDA(cudaMemcpy(off.data(), w.off.p, sizeof(uint64_t) * off.size(),
                          cudaMemcpyDeviceToHost));
      for (int cc = 0; cc < k; ++cc) {
        if (off[cc] != off[cc + 1]) continue;
        own_dist_kernel<<<grid_for(n), kTB, 0, c.stream>>>(zt, n, d, assign,
                                                           w.cen_new.as<double>(), cen, cc, dist2);
        F2V_LAUNCHED(c.stream, "own_dist_kernel");
        farthest_kernel<<<1, 1024, 0, c.stream>>>(z, n, d, dist2,
                                                  w.cen_new.as<double>() + size_t(cc) * d);
        F2V_LAUNCHED(c.stream, "farthest_kernel");
        c.launches += 2;
      }
    }
    std::swap(w.cen, w.cen_new);
    cen = w.cen.as<double>();
  }
  return inertia;
}

// kmeans (evaluation.cpp:428-438): best of `restarts` by inertia (first best)
double kmeans(Ctx& c, const float* z, uint64_t n, uint32_t d, int k, uint64_t& rng, int restarts,
              int max_iters, int32_t* assign_host) {
  if (k < 1 || uint64_t(k) > n) fail(F2V_EUSAGE, "kmeans: k must be in [1, n]");
  KmeansWork w;
  kmeans_alloc(c, w, z, n, d, k);
  DeviceBuf best;
  best.ensure(sizeof(int32_t) * n);
  double best_inertia = std::numeric_limits<double>::infinity();
  bool have = false;
  for (int r = 0; r < restarts; ++r) {
    const double inertia = lloyd_once(c, w, z, n, d, k, rng, max_iters);
    if (inertia < best_inertia) {
      best_inertia = inertia;
      have = true;
      F2V_CUDA(cudaMemcpyAsync(best.p, w.assign.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice,
                               c.stream));
    }
  }
  // no restart (or only non-finite inertias): the reference returns an empty assignment
  if (have)
    F2V_CUDA(cudaMemcpyAsync(assign_host, best.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                             c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  best.release();
  if (!have) fail(F2V_ENUMERICAL, "kmeans: no restart produced a finite inertia");
  return best_inertia;
}

// kmeans_inertia (evaluation.cpp:440-458)
double kmeans_inertia(Ctx& c, const float* z, uint64_t n, uint32_t d, int k,
                      const int32_t* assign_host) {
  for (uint64_t i = 0; i < n; ++i)
    if (assign_host[i] < 0 || assign_host[i] >= k) fail(F2V_ERANGE, "cluster id out of range");
  KmeansWork w;
  kmeans_alloc(c, w, z, n, d, k);
  F2V_CUDA(cudaMemcpyAsync(w.assign.p, assign_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                           c.stream));
  F2V_CUDA(cudaMemsetAsync(w.cen.p, 0, sizeof(double) * size_t(k) * d, c.stream));
  F2V_CUDA(cudaMemsetAsync(w.flags.p, 0, 16, c.stream));
  update_centroids(c, w, z, n, d, k, w.assign.as<int32_t>(), w.cen.as<double>(),
                   w.flags.as<uint32_t>() + 1);
  own_dist_kernel<<<grid_for(n), kTB, 0, c.stream>>>(w.zt.as<float>(), n, d,
                                                     w.assign.as<int32_t>(), w.cen.as<double>(),
                                                     w.cen.as<double>(), 0, w.dist2.as<double>());
  F2V_LAUNCHED(c.stream, "own_dist_kernel");
  double* out = reinterpret_cast<double*>(w.flags.as<uint8_t>() + 8);
  seq_sum_kernel<<<1, 32, 0, c.stream>>>(w.dist2.as<double>(), n, out);
  F2V_LAUNCHED(c.stream, "seq_sum_kernel");
  c.launches += 2;
  double inertia = 0.0;
  F2V_CUDA(cudaMemcpyAsync(&inertia, out, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  return inertia;
}

// modularity (evaluation.cpp:460-483) of the context's graph
double modularity(Ctx& c, int k, const int32_t* assign_host) {
  if (c.nnz == 0) fail(F2V_EUSAGE, "modularity undefined for m = 0");
  for (uint32_t i = 0; i < c.n; ++i)
    if (assign_host[i] < 0 || assign_host[i] >= k) fail(F2V_ERANGE, "cluster id out of range");
  DeviceBuf a, t;
  a.ensure(sizeof(int32_t) * c.n);
  t.ensure(sizeof(unsigned long long) * 2 * size_t(k));
  F2V_CUDA(cudaMemcpyAsync(a.p, assign_host, sizeof(int32_t) * c.n, cudaMemcpyHostToDevice,
                           c.stream));
  F2V_CUDA(cudaMemsetAsync(t.p, 0, sizeof(unsigned long long) * 2 * size_t(k), c.stream));
  modularity_kernel<<<unsigned(std::min<uint64_t>((uint64_t(c.n) + 3) / 4, uint64_t(c.num_sms) * 16)),
                      kTB, 0, c.stream>>>(c.rowptr.as<uint64_t>(), c.col.as<uint32_t>(), c.n,
                                          a.as<int32_t>(), t.as<unsigned long long>(),
                                          t.as<unsigned long long>() + k);
  F2V_LAUNCHED(c.stream, "modularity_kernel");
  ++c.launches;
  std::vector<unsigned long long> h(2 * size_t(k));
  F2V_CUDA(cudaMemcpyAsync(h.data(), t.p, sizeof(unsigned long long) * h.size(),
                           cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  a.release();
  t.release();
  const double m = double(c.nnz) / 2.0;
  double q = 0.0;
  for (int cl = 0; cl < k; ++cl) {
    const double l_c = double(h[cl]) / 2.0;
    const double d_c = double(h[size_t(k) + cl]);
    const volatile double a1 = l_c / m;  // separate roundings, as the reference's build
    const volatile double b1 = d_c / (2.0 * m);
    const volatile double b2 = b1 * b1;
    const volatile double t1 = a1 - b2;
    q = q + t1;
  }
  return q;
}

// ------------------------------------------------------- logistic regression
struct LogRegWork {
  DeviceBuf x, xt, w, err, tgt;
  ~LogRegWork() {
    for (DeviceBuf* b : {&x, &xt, &w, &err, &tgt}) b->release();
  }
};

// fit M one-vs-rest models (evaluation.cpp:93-121) on device features x
// (row-major) / xt (transposed); tgt_host = u8[M * n]; weights_out = f64[M * (d+1)]
static void fit_models(Ctx& c, LogRegWork& w, uint64_t n, uint32_t d, uint32_t M,
                       const uint8_t* tgt_host, double lr, int iters, double l2,
                       double* weights_out) {
  w.w.ensure(sizeof(double) * size_t(M) * (d + 1));
  w.err.ensure(sizeof(double) * size_t(M) * n);
  w.tgt.ensure(size_t(M) * n);
  F2V_CUDA(cudaMemcpyAsync(w.tgt.p, tgt_host, size_t(M) * n, cudaMemcpyHostToDevice, c.stream));
  F2V_CUDA(cudaMemsetAsync(w.w.p, 0, sizeof(double) * size_t(M) * (d + 1), c.stream));
  const uint32_t tb = std::min<uint32_t>(1024, (d + 1 + 31) / 32 * 32);
  // rows per shared-memory tile of the tiled step: two tiles + their errors in <= 160 KB
  uint32_t R = 64;
  while (R >= 8 && 2 * (size_t(R) * d * sizeof(float) + R * sizeof(double)) > 160 * 1024) R /= 2;
  const bool tiled = R >= 8 && d + 1 <= 1024;
  const size_t tsmem = 2 * (size_t(R) * d * sizeof(float) + R * sizeof(double));
  if (tiled)
    F2V_CUDA(cudaFuncSetAttribute(logreg_step_tiled_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(tsmem)));
  for (int it = 0; it < iters; ++it) {
    logreg_err_kernel<<<dim3(grid_for(n), M), kTB, 0, c.stream>>>(
        w.xt.as<float>(), n, d, w.w.as<double>(), w.tgt.as<uint8_t>(), w.err.as<double>());
    F2V_LAUNCHED(c.stream, "logreg_err_kernel");
    if (tiled)
      logreg_step_tiled_kernel<<<M, tb, tsmem, c.stream>>>(w.x.as<float>(), n, d,
                                                           w.err.as<double>(), w.w.as<double>(),
                                                           lr, l2, R);
    else
      logreg_step_kernel<<<M, tb, 0, c.stream>>>(w.x.as<float>(), n, d, w.err.as<double>(),
                                                 w.w.as<double>(), lr, l2);
    F2V_LAUNCHED(c.stream, "logreg_step_kernel");
    c.launches += 2;
  }
  F2V_CUDA(cudaMemcpyAsync(weights_out, w.w.p, sizeof(double) * size_t(M) * (d + 1),
                           cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  for (size_t t = 0; t < size_t(M) * (d + 1); ++t)
    if (!std::isfinite(weights_out[t])) fail(F2V_ENUMERICAL, "fit_logreg: non-finite weights");
}

static void check_targets(const int32_t* targets, uint64_t n, std::vector<uint8_t>& t8) {
  t8.resize(n);
  uint64_t ones = 0;
  for (uint64_t i = 0; i < n; ++i) {
    t8[i] = uint8_t(targets[i]);
    ones += targets[i] == 1;  // std::count(targets, 1)
  }
  if (ones == 0 || ones == n) fail(F2V_EERROR, "fit_logreg: degenerate single-class input");
}

// fit_logreg (evaluation.cpp:93-121) on host features (row-major f32[n * d])
void fit_logreg(Ctx& c, const float* x_host, uint64_t n, uint32_t d, const int32_t* targets,
                double lr, int iters, double l2, double* weights_out) {
  std::vector<uint8_t> t8;
  check_targets(targets, n, t8);
  LogRegWork w;
  w.x.ensure(sizeof(float) * n * d);
  w.xt.ensure(sizeof(float) * n * d);
  F2V_CUDA(cudaMemcpyAsync(w.x.p, x_host, sizeof(float) * n * d, cudaMemcpyHostToDevice,
                           c.stream));
  transpose(c, w.x.as<float>(), nullptr, n, d, w.xt.as<float>());
  fit_models(c, w, n, d, 1, t8.data(), lr, iters, l2, weights_out);
}

// logreg_loss (evaluation.cpp:139-153)
double logreg_loss(Ctx& c, const double* weights, const float* x_host, uint64_t n, uint32_t d,
                   const int32_t* targets, double l2) {
  LogRegWork w;
  w.x.ensure(sizeof(float) * n * d);
  w.xt.ensure(sizeof(float) * n * d);
  w.w.ensure(sizeof(double) * (d + 1));
  w.err.ensure(sizeof(double) * (n + 1));
  w.tgt.ensure(n);
  std::vector<uint8_t> t8(n);
  for (uint64_t i = 0; i < n; ++i) t8[i] = targets[i] ? 1 : 0;
  F2V_CUDA(cudaMemcpyAsync(w.x.p, x_host, sizeof(float) * n * d, cudaMemcpyHostToDevice,
                           c.stream));
  F2V_CUDA(cudaMemcpyAsync(w.w.p, weights, sizeof(double) * (d + 1), cudaMemcpyHostToDevice,
                           c.stream));
  F2V_CUDA(cudaMemcpyAsync(w.tgt.p, t8.data(), n, cudaMemcpyHostToDevice, c.stream));
  transpose(c, w.x.as<float>(), nullptr, n, d, w.xt.as<float>());
  logreg_loss_kernel<<<grid_for(n), kTB, 0, c.stream>>>(w.xt.as<float>(), n, d, w.w.as<double>(),
                                                        w.tgt.as<uint8_t>(), w.err.as<double>());
  F2V_LAUNCHED(c.stream, "logreg_loss_kernel");
  seq_neg_sum_kernel<<<1, 32, 0, c.stream>>>(w.err.as<double>(), n, w.err.as<double>() + n);
  F2V_LAUNCHED(c.stream, "seq_neg_sum_kernel");
  c.launches += 2;
  double loss = 0.0;
  F2V_CUDA(cudaMemcpyAsync(&loss, w.err.as<double>() + n, sizeof(double), cudaMemcpyDeviceToHost,
                           c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  const volatile double mean = loss / double(n);
  double reg = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    const volatile double sq = weights[j] * weights[j];
    reg = reg + sq;
  }
  const volatile double half = 0.5 * l2;
  const volatile double r = half * reg;
  return mean + r;
}

// link_prediction_accuracy (evaluation.cpp:155-173): pairs = u32[3 * m] (u, v, is_edge)
double link_accuracy(Ctx& c, const float* z, uint32_t d, const uint32_t* train_pairs,
                     uint64_t ntrain, const uint32_t* test_pairs, uint64_t ntest, double lr,
                     int iters, double l2, double* weights_out) {
  for (uint64_t i = 0; i < ntrain; ++i)
    if (train_pairs[3 * i] >= c.n || train_pairs[3 * i + 1] >= c.n)
      fail(F2V_ERANGE, "vertex id out of range");
  for (uint64_t i = 0; i < ntest; ++i)
    if (test_pairs[3 * i] >= c.n || test_pairs[3 * i + 1] >= c.n)
      fail(F2V_ERANGE, "vertex id out of range");
  std::vector<uint8_t> t8(ntrain);
  uint64_t ones = 0;
  for (uint64_t i = 0; i < ntrain; ++i) ones += (t8[i] = train_pairs[3 * i + 2] ? 1 : 0);
  if (ones == 0 || ones == ntrain)
    fail(F2V_EERROR, "fit_logreg: degenerate single-class input");
  LogRegWork w;
  DeviceBuf pairs;
  const uint64_t mmax = std::max(ntrain, ntest);
  pairs.ensure(sizeof(uint32_t) * 3 * mmax);
  w.x.ensure(sizeof(float) * mmax * d);
  w.xt.ensure(sizeof(float) * mmax * d);
  F2V_CUDA(cudaMemcpyAsync(pairs.p, train_pairs, sizeof(uint32_t) * 3 * ntrain,
                           cudaMemcpyHostToDevice, c.stream));
  hadamard_kernel<<<unsigned(std::min<uint64_t>(grid_for(ntrain * d), 1u << 20)), kTB, 0,
                    c.stream>>>(z, pairs.as<uint32_t>(), ntrain, d, w.x.as<float>());
  F2V_LAUNCHED(c.stream, "hadamard_kernel");
  ++c.launches;
  transpose(c, w.x.as<float>(), nullptr, ntrain, d, w.xt.as<float>());
  std::vector<double> wts(d + 1);
  fit_models(c, w, ntrain, d, 1, t8.data(), lr, iters, l2, wts.data());
  if (weights_out) std::copy(wts.begin(), wts.end(), weights_out);
  // test pass
  DeviceBuf cnt;
  cnt.ensure(sizeof(unsigned long long));
  F2V_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), c.stream));
  F2V_CUDA(cudaMemcpyAsync(pairs.p, test_pairs, sizeof(uint32_t) * 3 * ntest,
                           cudaMemcpyHostToDevice, c.stream));
  if (ntest) {
    hadamard_kernel<<<unsigned(std::min<uint64_t>(grid_for(ntest * d), 1u << 20)), kTB, 0,
                      c.stream>>>(z, pairs.as<uint32_t>(), ntest, d, w.x.as<float>());
    F2V_LAUNCHED(c.stream, "hadamard_kernel");
    transpose(c, w.x.as<float>(), nullptr, ntest, d, w.xt.as<float>());
    link_correct_kernel<<<grid_for(ntest), kTB, 0, c.stream>>>(
        w.xt.as<float>(), ntest, d, w.w.as<double>(), pairs.as<uint32_t>(),
        cnt.as<unsigned long long>());
    F2V_LAUNCHED(c.stream, "link_correct_kernel");
    c.launches += 2;
  }
  unsigned long long correct = 0;
  F2V_CUDA(cudaMemcpyAsync(&correct, cnt.p, sizeof(correct), cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  pairs.release();
  cnt.release();
  return double(correct) / double(ntest);
}

// The one-vs-rest core of node_classification (evaluation.cpp:262-281): fit M
// models on the rows train_ids of z (tgt = u8[M * ntrain]) and return the
// probabilities of the rows test_ids, prob_out = f64[ntest * M]
void one_vs_rest(Ctx& c, const float* z, uint32_t d, const uint32_t* train_ids, uint64_t ntrain,
                 const uint32_t* test_ids, uint64_t ntest, uint32_t M, const uint8_t* tgt,
                 double lr, int iters, double l2, double* weights_out, double* prob_out) {
  for (uint32_t m = 0; m < M; ++m) {
    uint64_t ones = 0;
    for (uint64_t i = 0; i < ntrain; ++i) ones += tgt[size_t(m) * ntrain + i];
    if (ones == 0 || ones == ntrain)
      fail(F2V_EERROR, "fit_logreg: degenerate single-class input");
  }
  LogRegWork w;
  DeviceBuf ids, prob;
  ids.ensure(sizeof(uint32_t) * std::max(ntrain, ntest));
  w.x.ensure(sizeof(float) * ntrain * d);
  w.xt.ensure(sizeof(float) * std::max(ntrain, ntest) * d);
  F2V_CUDA(cudaMemcpyAsync(ids.p, train_ids, sizeof(uint32_t) * ntrain, cudaMemcpyHostToDevice,
                           c.stream));
  gather_rows_kernel<<<unsigned(std::min<uint64_t>(grid_for(ntrain * d), 1u << 20)), kTB, 0,
                       c.stream>>>(z, ids.as<uint32_t>(), ntrain, d, w.x.as<float>());
  F2V_LAUNCHED(c.stream, "gather_rows_kernel");
  ++c.launches;
  transpose(c, z, ids.as<uint32_t>(), ntrain, d, w.xt.as<float>());
  std::vector<double> wts(size_t(M) * (d + 1));
  fit_models(c, w, ntrain, d, M, tgt, lr, iters, l2, wts.data());
  if (weights_out) std::copy(wts.begin(), wts.end(), weights_out);
  prob.ensure(sizeof(double) * ntest * M);
  F2V_CUDA(cudaMemcpyAsync(ids.p, test_ids, sizeof(uint32_t) * ntest, cudaMemcpyHostToDevice,
                           c.stream));
  transpose(c, z, ids.as<uint32_t>(), ntest, d, w.xt.as<float>());
  logreg_prob_kernel<<<dim3(grid_for(ntest), M), kTB, 0, c.stream>>>(
      w.xt.as<float>(), ntest, d, w.w.as<double>(), M, prob.as<double>());
  F2V_LAUNCHED(c.stream, "logreg_prob_kernel");
  ++c.launches;
  F2V_CUDA(cudaMemcpyAsync(prob_out, prob.p, sizeof(double) * ntest * M, cudaMemcpyDeviceToHost,
                           c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  ids.release();
  prob.release();
}

}  // namespace ev
}  // namespace f2v
