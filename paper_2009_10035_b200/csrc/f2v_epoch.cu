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
// Work split.  Arcs (u, v) of a batch-j vertex fall in three classes:
//   early   batch(v) >= j        -> Zold, no dependency;
//   past    batch(v) <  j - W    -> Znew, final long before u's turn;
//   window  j - W <= batch(v) < j -> Znew, on the dependency chain.
// E items (one per C-arc chunk, bandwidth-heavy) take early + past arcs and
// compact the window arcs into a per-chunk list.  A per-epoch pre-scan marks
// the vertices that have window arcs or window negatives ("needs L"); every
// other vertex is finalised by its E item.  L items (one per G chunks of a
// needs-L vertex, latency-critical) take the E partial, the window arcs with
// age > R, the shared negatives, then the most recent window arcs, waiting
// on each row's written bit, and finalise.
//
// Warp roles.  Every CTA has E warps and L warps with their own claim
// counters over statically ordered (batch-major) item lists.  Each list is
// claimed in order and every wait points at an item that is lower in the
// global (batch, E-before-L) order, so the lowest unfinished item is always
// claimed and runnable: deadlock-free on any number of resident CTAs.
// Partials of split rows are combined in a fixed order by the last arrival
// (no float atomics): results are bitwise reproducible run to run.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "f2v_epoch.cuh"

namespace f2v {

__global__ void sum_kernel(const double* __restrict__ v, uint64_t m, double* out);

namespace {

using namespace dev;

// ------------------------------------------------------ per-epoch prep
__global__ void state_kernel(const uint32_t* __restrict__ perm, uint32_t* __restrict__ state,
                             uint32_t n, uint32_t b, const uint32_t* __restrict__ cbase,
                             uint32_t* __restrict__ nE, uint32_t* __restrict__ wtot) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  if (p == n) {
    nE[n] = 0;
    return;
  }
  const uint32_t u = perm[p];
  state[u] = (p / b) << 1;
  nE[p] = cbase[u + 1] - cbase[u];
  wtot[u] = 0;
}

// One thread per arc: mark the vertices that have a window arc (batch(v) in
// [batch(u) - W, batch(u))).  src[] is the static arc -> source map.
__global__ void window_scan_kernel(const uint32_t* __restrict__ src,
                                   const uint32_t* __restrict__ col,
                                   const uint32_t* __restrict__ state, uint32_t* __restrict__ wtot,
                                   uint64_t nnz, uint32_t W, uint32_t Re) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const uint32_t u = __ldg(src + e), v = __ldg(col + e);
  const uint32_t j = __ldg(state + u) >> 1, bv = __ldg(state + v) >> 1;
  if (bv < j && bv + W >= j) atomicOr(wtot + u, bv + Re >= j ? 3u : 1u);  // bit1: engine-recent
}

// src[e] = the row of arc e (static per graph)
__global__ void src_kernel(const uint64_t* __restrict__ rowptr, uint32_t* __restrict__ src,
                           uint32_t n) {
  const uint32_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (u >= n) return;
  for (uint64_t e = rowptr[u] + lane; e < rowptr[u + 1]; e += 32) src[e] = u;
}

__global__ void needs_kernel(const uint32_t* __restrict__ perm, uint32_t n, uint32_t b,
                             const uint32_t* __restrict__ wtot, const uint32_t* __restrict__ negwin,
                             const uint32_t* __restrict__ lbase, uint32_t* __restrict__ needs,
                             uint32_t* __restrict__ nL, uint32_t* __restrict__ nEng, int nodep) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  if (p == n) {
    nL[n] = 0;
    nEng[n] = 0;
    return;
  }
  const uint32_t u = perm[p];
  const uint32_t nw = negwin[p / b];
  uint32_t nd = ((wtot[u] | nw) & 1u) && !nodep ? 1u : 0u;
  if (nd && (wtot[u] & 2u) && lbase[u + 1] - lbase[u] == 1) nd |= 2u;  // the chain engine's
  needs[u] = nd;
  nL[p] = nd ? lbase[u + 1] - lbase[u] : 0u;
  nEng[p] = (nd & 2u) ? 1u : 0u;
}

__global__ void emit_kernel(const uint32_t* __restrict__ P, const uint32_t* __restrict__ cnt,
                            uint2* __restrict__ items, uint32_t n) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t o = P[p];
  for (uint32_t c = 0, m = P[p + 1] - o; c < m; ++c) items[o + c] = make_uint2(p, c);
  (void)cnt;
}

// engine positions (batch-major) and each engine vertex's slot in its batch
__global__ void engine_emit_kernel(const uint32_t* __restrict__ ecum,
                                   const uint32_t* __restrict__ nEng,
                                   const uint32_t* __restrict__ perm,
                                   const uint32_t* __restrict__ cbase, uint4* __restrict__ erec,
                                   uint32_t* __restrict__ eslot, uint32_t* __restrict__ eidx,
                                   uint32_t n, uint32_t b) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n || !nEng[p]) return;
  const uint32_t u = perm[p], i = ecum[p];
  erec[i] = make_uint4(u, cbase[u], p, 0u);
  eslot[u] = i - ecum[uint64_t(p / b) * b];
  eidx[u] = i;
}

__global__ void negs_kernel(uint32_t* __restrict__ out, uint32_t* __restrict__ negwin,
                            const uint32_t* __restrict__ state, uint64_t nb, uint32_t s,
                            uint32_t n, uint64_t seed, uint32_t epoch, int sampler, uint32_t W,
                            uint32_t Re) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  uint32_t win = 0;
  for (uint32_t k = 0; k < s; ++k) {
    const uint32_t w = sampler == F2V_SAMPLER_PHILOX ? philox_negative(seed, epoch, j, 0, k, n)
                                                     : splitmix_negative(seed, epoch, j, 0, 1, k, n);
    out[j * s + k] = w;
    const uint32_t bw = state[w] >> 1;
    if (bw < j && uint64_t(bw) + W >= j) win |= uint64_t(bw) + Re >= j ? 3u : 1u;
  }
  negwin[j] = win;
}

// Znew := the sentinel NaN everywhere (rows become readable once stored).
__global__ void sentinel_kernel(uint4* __restrict__ z, uint64_t n16) {
  const uint4 s = make_uint4(kSentinel, kSentinel, kSentinel, kSentinel);
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += uint64_t(gridDim.x) * blockDim.x)
    __stcg(z + i, s);
}

__global__ void sentinel_tail_kernel(float* __restrict__ z, uint64_t from, uint64_t to) {
  const uint64_t i = from + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < to) z[i] = __uint_as_float(kSentinel);
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
  t.window = std::max(1u, env_u32("F2V_WINDOW", t.window));
  t.recent = env_u32("F2V_RECENT", t.recent);
  t.lwarps = std::min(uint32_t(ep::kWarps - 1), std::max(1u, env_u32("F2V_LWARPS", t.lwarps)));
  if (const char* e = std::getenv("F2V_PRECISION")) t.fast = std::strcmp(e, "exact") != 0;
  t.erecent = env_u32("F2V_ERECENT", t.erecent);
  if (t.erecent >= t.window) t.erecent = t.window - 1;
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
  c.src.ensure(sizeof(uint32_t) * std::max<uint64_t>(c.nnz, 1));
  c.ecnt.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  c.lcnt.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  c.vflag.ensure(sizeof(uint32_t) * std::max<uint32_t>(c.n, 1));
  F2V_CUDA(cudaMemcpyAsync(c.cbase.p, cbase.data(), sizeof(uint32_t) * (c.n + 1),
                           cudaMemcpyHostToDevice, c.stream));
  F2V_CUDA(cudaMemcpyAsync(c.lbase.p, lbase.data(), sizeof(uint32_t) * (c.n + 1),
                           cudaMemcpyHostToDevice, c.stream));
  if (c.n) {
    src_kernel<<<uint32_t((uint64_t(c.n) * 32 + 255) / 256), 256, 0, c.stream>>>(
        c.rowptr.as<uint64_t>(), c.src.as<uint32_t>(), c.n);
    F2V_LAUNCHED(c.stream, "src_kernel");
  }
  if (c.n) {
    F2V_CUDA(cudaMemcpyAsync(c.lpo.p, lpo.data(), sizeof(uint32_t) * c.n,
                             cudaMemcpyHostToDevice, c.stream));
    F2V_CUDA(cudaMemsetAsync(c.ecnt.p, 0, sizeof(uint32_t) * c.n, c.stream));
    F2V_CUDA(cudaMemsetAsync(c.lcnt.p, 0, sizeof(uint32_t) * c.n, c.stream));
    F2V_CUDA(cudaMemsetAsync(c.vflag.p, 0, sizeof(uint32_t) * c.n, c.stream));
  }
  F2V_CUDA(cudaStreamSynchronize(c.stream));
}

// Per-epoch preparation: perm (already in c.perm) -> state, the negatives of
// every batch + window flags, the window pre-scan, the two ordered item lists.
void k_epoch_begin(Ctx& c, uint32_t b, uint32_t s, uint32_t epoch, uint64_t seed, int sampler) {
  const uint32_t n = c.n;
  const uint32_t nb = uint32_t((uint64_t(n) + b - 1) / b);
  if (c.prepared_chunk != c.tune.chunk || c.prepared_lgroup != c.tune.lgroup)
    k_prepare_graph(c);
  c.state.ensure(sizeof(uint32_t) * n);
  c.nE.ensure(sizeof(uint32_t) * (n + 1));
  c.nL.ensure(sizeof(uint32_t) * (n + 1));
  c.EP.ensure(sizeof(uint32_t) * (n + 1));
  c.LP.ensure(sizeof(uint32_t) * (n + 1));
  c.wtot.ensure(sizeof(uint32_t) * std::max<uint32_t>(n, 1));
  c.needs.ensure(sizeof(uint32_t) * std::max<uint32_t>(n, 1));
  c.items.ensure(sizeof(uint2) * std::max<uint64_t>(c.chunks, 1));
  c.litems.ensure(sizeof(uint2) * std::max<uint64_t>(c.lgroups, 1));
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
  const uint32_t W = c.tune.window;
  // effective engine window: 0 when the engine cannot run for this layout
  uint32_t Re = c.tune.erecent;
  {
    const size_t stage = 2 * size_t(ep::kEngineWarps) * ep::kStage *
                         ((size_t(c.d) * 12 + ep::kRefStride * 4 + 15) / 16 * 16);
    const size_t budget = 210u * 1024u > stage ? 210u * 1024u - stage : 0;
    c.eff_maxe = Re ? uint32_t(std::min<size_t>(64, budget / (size_t(Re + 1) * c.d * 4))) : 0u;
    if (Re && (!c.tune.fast || c.eff_maxe < 4 || n >= kIdMask ||
               (c.d != 64 && c.d != 128 && c.d != 256)))
      Re = 0;
    c.eff_re = Re;
  }
  c.nEng.ensure(sizeof(uint32_t) * (n + 1));
  c.ecum.ensure(sizeof(uint32_t) * (n + 1));
  c.epos.ensure(sizeof(uint4) * std::max<uint32_t>(n, 1));
  c.eslot.ensure(sizeof(uint32_t) * std::max<uint32_t>(n, 1));
  c.eidx.ensure(sizeof(uint32_t) * std::max<uint32_t>(n, 1));
  c.rcnt.ensure(sizeof(uint32_t) * ep::kRefStride * std::max<uint32_t>(n, 1));
  state_kernel<<<(n + 1 + 255) / 256, 256, 0, c.stream>>>(c.perm.as<uint32_t>(),
                                                         c.state.as<uint32_t>(), n, b,
                                                         c.cbase.as<uint32_t>(),
                                                         c.nE.as<uint32_t>(), c.wtot.as<uint32_t>());
  F2V_LAUNCHED(c.stream, "state_kernel");
  negs_kernel<<<(nb + 255) / 256, 256, 0, c.stream>>>(
      c.negs_all.as<uint32_t>(), c.negwin.as<uint32_t>(), c.state.as<uint32_t>(), nb, s, n, seed,
      epoch, sampler, W, Re);
  F2V_LAUNCHED(c.stream, "negs_kernel");
  if (c.nnz)
    window_scan_kernel<<<uint32_t((c.nnz + 255) / 256), 256, 0, c.stream>>>(
        c.src.as<uint32_t>(), c.col.as<uint32_t>(), c.state.as<uint32_t>(),
        c.wtot.as<uint32_t>(), c.nnz, W, Re);
  F2V_LAUNCHED(c.stream, "window_scan_kernel");
  needs_kernel<<<(n + 1 + 255) / 256, 256, 0, c.stream>>>(
      c.perm.as<uint32_t>(), n, b, c.wtot.as<uint32_t>(), c.negwin.as<uint32_t>(),
      c.lbase.as<uint32_t>(), c.needs.as<uint32_t>(), c.nL.as<uint32_t>(), c.nEng.as<uint32_t>(),
      std::getenv("F2V_DEBUG_NODEP") ? 1 : 0);
  F2V_LAUNCHED(c.stream, "needs_kernel");
  size_t tmp = 0;
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.nE.as<uint32_t>(), c.EP.as<uint32_t>(),
                                         n + 1, c.stream));
  c.scan_tmp.ensure(tmp);
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp, c.nE.as<uint32_t>(),
                                         c.EP.as<uint32_t>(), n + 1, c.stream));
  F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp, c.nL.as<uint32_t>(),
                                         c.LP.as<uint32_t>(), n + 1, c.stream));
  emit_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(c.EP.as<uint32_t>(), c.nE.as<uint32_t>(),
                                                     c.items.as<uint2>(), n);
  F2V_LAUNCHED(c.stream, "emit_kernel");
  emit_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(c.LP.as<uint32_t>(), c.nL.as<uint32_t>(),
                                                     c.litems.as<uint2>(), n);
  F2V_LAUNCHED(c.stream, "emit_kernel");
  if (Re) {
    F2V_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.p, tmp, c.nEng.as<uint32_t>(),
                                           c.ecum.as<uint32_t>(), n + 1, c.stream));
    engine_emit_kernel<<<(n + 255) / 256, 256, 0, c.stream>>>(
        c.ecum.as<uint32_t>(), c.nEng.as<uint32_t>(), c.perm.as<uint32_t>(),
        c.cbase.as<uint32_t>(), c.epos.as<uint4>(), c.eslot.as<uint32_t>(),
        c.eidx.as<uint32_t>(), n, b);
    F2V_LAUNCHED(c.stream, "engine_emit_kernel");
  }
  // number of L items (device value, read back asynchronously with the run)
  F2V_CUDA(cudaMemcpyAsync(c.counters.as<uint32_t>() + 8, c.LP.as<uint32_t>() + n,
                           sizeof(uint32_t), cudaMemcpyDeviceToDevice, c.stream));
  c.launches += 9;
}

EpochResult k_epoch_run(Ctx& c, uint32_t b, uint32_t s, float eta, const ForceParams& fp,
                        bool monitor) {
  const int nxt = 1 - c.cur;
  c.z[nxt].ensure(sizeof(float) * size_t(c.n) * c.d);
  uint32_t* ctr = c.counters.as<uint32_t>();  // [0..1] claims, [2..3] bad, [4..5] loss, [8] nL
  F2V_CUDA(cudaMemsetAsync(ctr, 0, 8, c.stream));
  F2V_CUDA(cudaMemsetAsync(ctr + 2, 0xff, 8, c.stream));
  {  // Znew := sentinel (cudaMalloc'd buffers are 256-byte aligned)
    const uint64_t total = uint64_t(c.n) * c.d, n16 = total / 4;
    sentinel_kernel<<<uint32_t(std::min<uint64_t>((n16 + 255) / 256, 4u * c.num_sms * 8)), 256, 0,
                      c.stream>>>(c.z[nxt].as<uint4>(), n16);
    F2V_LAUNCHED(c.stream, "sentinel_kernel");
    if (total % 4)
      sentinel_tail_kernel<<<1, 4, 0, c.stream>>>(c.z[nxt].as<float>(), n16 * 4, total);
    c.launches += 1;
  }
  ep::EpochArgs a;
  a.rowptr = c.rowptr.as<uint64_t>();
  a.col = c.col.as<uint32_t>();
  a.zold = c.z[c.cur].as<float>();
  a.znew = c.z[nxt].as<float>();
  a.perm = c.perm.as<uint32_t>();
  a.state = c.state.as<uint32_t>();
  a.negs = c.negs_all.as<uint32_t>();
  a.negwin = c.negwin.as<uint32_t>();
  a.eitems = c.items.as<uint2>();
  a.litems = c.litems.as<uint2>();
  a.n_eitems = uint32_t(c.chunks);
  a.n_litems = ctr + 8;
  a.next = ctr;
  a.cbase = c.cbase.as<uint32_t>();
  a.lbase = c.lbase.as<uint32_t>();
  a.lpo = c.lpo.as<uint32_t>();
  a.needs = c.needs.as<uint32_t>();
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
  a.W = c.tune.window;
  a.R = c.tune.recent;
  a.lwarps = c.tune.lwarps;
  a.rl = c.rcnt.as<uint32_t>();
  a.erec = c.epos.as<uint4>();
  a.ecum = c.ecum.as<uint32_t>();
  a.eslot = c.eslot.as<uint32_t>();
  a.eidx = c.eidx.as<uint32_t>();
  a.Re = c.eff_re;  // decided by the prep (0: no engine this epoch)
  a.maxe = c.eff_maxe;
  a.eta = eta;
  a.fp = fp;
  a.nodep = std::getenv("F2V_DEBUG_NODEP") ? 1 : 0;
  a.nnz = c.nnz;
  a.chunks = c.chunks;
  a.lslots = c.lslots;
  a.trace = nullptr;
  a.ltrace = nullptr;
  a.etrace = nullptr;
  if (std::getenv("F2V_TRACE")) {
    const uint32_t nbt = (c.n + b - 1) / b;
    c.trace.ensure(sizeof(unsigned long long) * (5ull * std::max<uint32_t>(c.n, 1) + 3ull * nbt + 2));
    a.trace = c.trace.as<unsigned long long>();
    a.ltrace = a.trace + c.n;
    a.etrace = a.ltrace + 4ull * c.n;
    F2V_CUDA(cudaMemsetAsync(a.ltrace, 0,
                             sizeof(unsigned long long) * (4ull * c.n + 3ull * nbt + 2), c.stream));
  }
  if (!c.ev_kernel.size()) {
    c.ev_kernel.resize(2);
    F2V_CUDA(cudaEventCreate(&c.ev_kernel[0]));
    F2V_CUDA(cudaEventCreate(&c.ev_kernel[1]));
  }
  F2V_CUDA(cudaEventRecord(c.ev_kernel[0], c.stream));
  ep::launch_epoch(c, a, monitor, c.tune.fast != 0);
  F2V_CUDA(cudaEventRecord(c.ev_kernel[1], c.stream));
  if (monitor) {
    sum_kernel<<<1, 1024, 0, c.stream>>>(c.ploss.as<double>(), c.n,
                                         reinterpret_cast<double*>(ctr + 4));
    F2V_LAUNCHED(c.stream, "sum_kernel");
    ++c.launches;
  }
  uint64_t host[5];
  F2V_CUDA(cudaMemcpyAsync(host, ctr, 40, cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  float kms = 0.f;
  F2V_CUDA(cudaEventElapsedTime(&kms, c.ev_kernel[0], c.ev_kernel[1]));
  c.timing[1] += kms;
  c.timing[2] += 1;
  c.last_litems = uint32_t(host[4]);
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
  F2V_LAUNCHED(c.stream, "restore_kernel");
  ++c.launches;
  F2V_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace f2v
