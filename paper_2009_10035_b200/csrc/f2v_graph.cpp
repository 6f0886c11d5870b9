// f2v_graph.cpp -- host-side data formats either side of the device step:
// the canonical CSR builder (CsrGraph::from_edges, csr_graph.cpp:57-97),
// Fisher-Yates partition_epoch (sampling.cpp:7-19), host negatives, and the
// BASELINE configs' synthetic graph generators.  Multithreaded C++; the CSR
// it builds is byte-identical to the reference's (tests/test_graph_host.py).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "f2v_internal.h"
#include "f2v_rng.h"

namespace f2v {

static unsigned host_threads() {
  static const unsigned t = [] {
    if (const char* e = std::getenv("F2V_HOST_THREADS")) {
      const int v = std::atoi(e);
      if (v > 0) return unsigned(v);
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? std::min(h, 64u) : 4u;
  }();
  return t;
}

// run fn(lo, hi) over [0, total) split into `threads` contiguous ranges
static void parallel_for(uint64_t total, const std::function<void(uint64_t, uint64_t)>& fn,
                         unsigned threads = 0) {
  if (!threads) threads = host_threads();
  if (total < 4096 || threads <= 1) {
    fn(0, total);
    return;
  }
  threads = unsigned(std::min<uint64_t>(threads, total));
  std::vector<std::thread> ts;
  ts.reserve(threads);
  for (unsigned t = 0; t < threads; ++t) {
    const uint64_t lo = total * t / threads, hi = total * (t + 1) / threads;
    ts.emplace_back([&, lo, hi] { fn(lo, hi); });
  }
  for (auto& t : ts) t.join();
}

// run fn(t, lo, hi) with exactly `threads` workers (t = worker index)
static void parallel_for_t(uint64_t total,
                           const std::function<void(unsigned, uint64_t, uint64_t)>& fn,
                           unsigned threads) {
  std::vector<std::thread> ts;
  for (unsigned t = 0; t < threads; ++t) {
    const uint64_t lo = total * t / threads, hi = total * (t + 1) / threads;
    ts.emplace_back([&, t, lo, hi] { fn(t, lo, hi); });
  }
  for (auto& t : ts) t.join();
}

// ------------------------------------------------ CsrGraph::from_edges
// csr_graph.cpp:57-97: drop self-loops (counted), optionally append reversed
// arcs, sort, unique, count, prefix.  Here: counting sort by source with
// atomic cursors, per-row sort + unique, compaction -- the canonical CSR of
// the same arc set, hence byte-identical.
void csr_from_edges(const uint32_t* pairs, uint64_t m, uint32_t n, bool symmetrize,
                    uint64_t* rowptr, uint32_t* col_out, uint64_t* nnz_out, uint64_t* dups_out,
                    uint64_t* loops_out) {
  std::atomic<uint64_t> loops{0};
  std::atomic<bool> range_err{false};
  std::vector<std::atomic<uint32_t>> deg(size_t(n) + 1);
  parallel_for(n + 1, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) deg[i].store(0, std::memory_order_relaxed);
  });
  parallel_for(m, [&](uint64_t lo, uint64_t hi) {
    uint64_t lp = 0;
    bool bad = false;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
      if (u == v) { ++lp; continue; }
      if (u >= n || v >= n) { bad = true; continue; }
      deg[u].fetch_add(1, std::memory_order_relaxed);
      if (symmetrize) deg[v].fetch_add(1, std::memory_order_relaxed);
    }
    loops += lp;
    if (bad) range_err = true;
  });
  if (range_err) fail(F2V_ERANGE, "edge endpoint out of range");
  // raw offsets (with duplicates)
  std::vector<uint64_t> raw(size_t(n) + 1, 0);
  for (uint32_t u = 0; u < n; ++u) raw[u + 1] = raw[u] + deg[u].load(std::memory_order_relaxed);
  const uint64_t total = raw[n];
  std::vector<uint32_t> tmp(std::max<uint64_t>(total, 1));
  std::vector<std::atomic<uint64_t>> cursor(n);
  parallel_for(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t u = lo; u < hi; ++u) cursor[u].store(raw[u], std::memory_order_relaxed);
  });
  parallel_for(m, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
      if (u == v) continue;
      tmp[cursor[u].fetch_add(1, std::memory_order_relaxed)] = v;
      if (symmetrize) tmp[cursor[v].fetch_add(1, std::memory_order_relaxed)] = u;
    }
  });
  // per-row sort + unique
  std::vector<uint64_t> ucount(size_t(n) + 1, 0);
  parallel_for(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t u = lo; u < hi; ++u) {
      uint32_t* b = tmp.data() + raw[u];
      uint32_t* e = tmp.data() + raw[u + 1];
      std::sort(b, e);
      ucount[u + 1] = uint64_t(std::unique(b, e) - b);
    }
  });
  rowptr[0] = 0;
  for (uint32_t u = 0; u < n; ++u) rowptr[u + 1] = rowptr[u] + ucount[u + 1];
  parallel_for(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t u = lo; u < hi; ++u)
      std::memcpy(col_out + rowptr[u], tmp.data() + raw[u], sizeof(uint32_t) * ucount[u + 1]);
  });
  const uint64_t nnz = rowptr[n];
  uint64_t dups = total - nnz;
  if (symmetrize) dups /= 2;  // csr_graph.cpp:80
  if (nnz_out) *nnz_out = nnz;
  if (dups_out) *dups_out = dups;
  if (loops_out) *loops_out = loops.load();
}

// ------------------------------------------------ partition_epoch (Fisher-Yates)
void partition_epoch(uint32_t n, uint32_t b, uint64_t state, uint32_t* perm) {
  if (b == 0 || b > n) fail(F2V_EUSAGE, "batch size must be in [1, n]");  // sampling.cpp:8
  for (uint32_t i = 0; i < n; ++i) perm[i] = i;
  uint64_t k = 0;
  for (uint32_t i = n; i > 1; --i, ++k) {
    const uint32_t j = uint32_t(rng_below(rng_draw(state, k), i));
    std::swap(perm[i - 1], perm[j]);
  }
}

// ------------------------------------------------ generators
// sbm_graph of tests/support/test_graphs.hpp:67-78 (the reference's own C1
// generator): sequential Bernoulli draws from Rng(seed, 0).
std::vector<uint32_t> gen_sbm(uint32_t n, int blocks, double p_in, double p_out, uint64_t seed) {
  if (blocks < 1 || uint32_t(blocks) > n) fail(F2V_EUSAGE, "sbm: bad block count");
  std::vector<uint32_t> e;
  const uint64_t s0 = rng_init(seed, 0);
  uint64_t k = 0;
  const uint32_t bs = n / uint32_t(blocks);
  for (uint32_t u = 0; u < n; ++u)
    for (uint32_t v = u + 1; v < n; ++v) {
      const bool same = u / bs == v / bs;
      if (rng_uniform(rng_draw(s0, k++)) < (same ? p_in : p_out)) {
        e.push_back(u);
        e.push_back(v);
      }
    }
  return e;
}

// R-MAT (Chakrabarti et al. 2004): edge i picks one quadrant per level with
// probabilities (a, b, c, 1-a-b-c); draw (i*scale + level) of the keyed
// stream (seed, {'RMAT'}), so the list is identical for any thread count.
std::vector<uint32_t> gen_rmat(uint32_t scale, uint32_t ef, double a, double b, double c,
                               uint64_t seed) {
  if (scale < 1 || scale > 31) fail(F2V_EUSAGE, "rmat: scale must be in [1, 31]");
  const uint64_t m = uint64_t(ef) << scale;
  std::vector<uint32_t> e(2 * m);
  const uint64_t s0 = rng_keyed1(seed, 0x524d4154ull);
  const double ab = a + b, abc = a + b + c;
  parallel_for(m, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      uint32_t u = 0, v = 0;
      for (uint32_t l = 0; l < scale; ++l) {
        const double r = rng_uniform(rng_draw(s0, i * scale + l));
        const uint32_t bit = 1u << (scale - 1 - l);
        if (r < a) {
        } else if (r < ab) {
          v |= bit;
        } else if (r < abc) {
          u |= bit;
        } else {
          u |= bit;
          v |= bit;
        }
      }
      e[2 * i] = u;
      e[2 * i + 1] = v;
    }
  });
  return e;
}

// Chung-Lu with power-law expected degrees: w_i = min_deg * (1-U)^(-1/(g-1)),
// clipped to max_deg and rescaled to mean_deg (three clip/rescale passes);
// n*mean_deg/2 edges whose endpoints are drawn independently with
// probability proportional to w (inverse CDF).  Stream (seed, {'CHLU'}).
std::vector<uint32_t> gen_chung_lu(uint32_t n, double expo, double min_deg, double max_deg,
                                   double mean_deg, uint64_t seed) {
  if (n < 2 || !(expo > 1.0)) fail(F2V_EUSAGE, "chung_lu: need n >= 2 and exponent > 1");
  std::vector<double> w(n);
  const uint64_t s0 = rng_keyed1(seed, 0x43484c55ull);
  parallel_for(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i)
      w[i] = min_deg * std::pow(1.0 - rng_uniform(rng_draw(s0, i)), -1.0 / (expo - 1.0));
  });
  for (int pass = 0; pass < 3; ++pass) {
    double sum = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
      w[i] = std::min(w[i], max_deg);
      sum += w[i];
    }
    const double f = mean_deg * n / sum;
    for (uint32_t i = 0; i < n; ++i) w[i] *= f;
  }
  for (uint32_t i = 0; i < n; ++i) w[i] = std::min(w[i], max_deg);
  std::vector<double> cdf(size_t(n) + 1, 0.0);
  for (uint32_t i = 0; i < n; ++i) cdf[i + 1] = cdf[i] + w[i];
  const double tot = cdf[n];
  const uint64_t m = uint64_t(double(n) * mean_deg / 2.0);
  std::vector<uint32_t> e(2 * m);
  const uint64_t s1 = rng_keyed2(seed, 0x43484c55ull, 1);
  parallel_for(m, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i)
      for (int side = 0; side < 2; ++side) {
        const double r = rng_uniform(rng_draw(s1, 2 * i + side)) * tot;
        uint32_t idx = uint32_t(std::upper_bound(cdf.begin() + 1, cdf.end(), r) - cdf.begin() - 1);
        if (idx >= n) idx = n - 1;
        e[2 * i + side] = idx;
      }
  });
  return e;
}

// Random geometric graph: n points U([0,1)^2) (draws 2i, 2i+1 of (seed,
// {'RGG'})), an edge for every pair closer than r with
// pi r^2 n = mean_deg; grid-bucket search, pairs emitted as (i, j), i < j.
std::vector<uint32_t> gen_rgg(uint32_t n, double mean_deg, uint64_t seed) {
  if (n < 2) fail(F2V_EUSAGE, "rgg: need n >= 2");
  const double r = std::sqrt(mean_deg / (M_PI * double(n)));
  const uint64_t s0 = rng_keyed1(seed, 0x524747ull);
  std::vector<double> x(n), y(n);
  for (uint32_t i = 0; i < n; ++i) {
    x[i] = rng_uniform(rng_draw(s0, 2ull * i));
    y[i] = rng_uniform(rng_draw(s0, 2ull * i + 1));
  }
  const uint32_t G = std::max<uint32_t>(1, uint32_t(1.0 / r));
  std::vector<uint32_t> cell_cnt(size_t(G) * G + 1, 0), cell_of(n);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t cx = std::min<uint32_t>(G - 1, uint32_t(x[i] * G));
    const uint32_t cy = std::min<uint32_t>(G - 1, uint32_t(y[i] * G));
    cell_of[i] = cy * G + cx;
    ++cell_cnt[cell_of[i] + 1];
  }
  for (size_t c = 0; c < size_t(G) * G; ++c) cell_cnt[c + 1] += cell_cnt[c];
  std::vector<uint32_t> members(n), fill(cell_cnt.begin(), cell_cnt.end() - 1);
  for (uint32_t i = 0; i < n; ++i) members[fill[cell_of[i]]++] = i;
  const unsigned T = host_threads();
  std::vector<std::vector<uint32_t>> parts(T);
  const double r2 = r * r;
  parallel_for_t(n, [&](unsigned t, uint64_t lo, uint64_t hi) {
    auto& out = parts[t];
    for (uint64_t ii = lo; ii < hi; ++ii) {
      const uint32_t i = uint32_t(ii);
      const int cx = int(cell_of[i] % G), cy = int(cell_of[i] / G);
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int nx = cx + dx, ny = cy + dy;
          if (nx < 0 || ny < 0 || nx >= int(G) || ny >= int(G)) continue;
          const uint32_t c = uint32_t(ny) * G + uint32_t(nx);
          for (uint32_t q = cell_cnt[c]; q < cell_cnt[c + 1]; ++q) {
            const uint32_t j = members[q];
            if (j <= i) continue;
            const double ddx = x[i] - x[j], ddy = y[i] - y[j];
            if (ddx * ddx + ddy * ddy < r2) {
              out.push_back(i);
              out.push_back(j);
            }
          }
        }
    }
  }, T);
  std::vector<uint32_t> e;
  size_t tot = 0;
  for (auto& p : parts) tot += p.size();
  e.reserve(tot);
  for (auto& p : parts) e.insert(e.end(), p.begin(), p.end());
  return e;
}

}  // namespace f2v
