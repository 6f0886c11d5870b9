// f2v_epoch.cuh -- the persistent dataflow epoch kernel (see f2v_epoch.cu for
// the schedule).  Instantiated per (force kind, row layout, loss monitoring,
// precision, register budget) in the f2v_epoch_i_*.cu translation units.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "f2v_internal.h"
#include "f2v_pair.cuh"
#include "f2v_rng.h"

namespace f2v {
namespace ep {

using namespace dev;

constexpr int kWarps = 8;       // warps per CTA
// Register budgets of the epoch kernel (template MINB = resident CTAs per SM
// it is compiled for): 2 (128 registers, no spills; best when the batch chain
// dominates) or 3 (80 registers, more gathers in flight; best when bandwidth
// does).  FAST d = 128 builds both and the driver picks per graph by timing
// (Ctx::occ_ms); results are identical.
constexpr int kQ = 64;          // per-warp compaction queue (entries)
constexpr int kRq = 64;         // per-warp parking lot for the most recent window arcs
constexpr int kMaxShards = 8;   // vertex shards (GPUs) of one run

// An E work item with its vertex already resolved by the prep (emit_e_kernel),
// so a warp's first dependent load is the chunk's column indices.
struct alignas(16) EItem {
  uint32_t p, u, cb, c;  // position, vertex, first chunk slot of u, chunk of u
  uint64_t e0;           // first arc of the chunk
  uint32_t cnt, nch;     // arcs in the chunk, chunks of u
};

struct EpochArgs {
  const uint64_t* rowptr;
  const uint32_t* col;
  const float* zold;
  float* znew;
  const uint32_t* perm;
  uint32_t* state;
  const uint32_t* negs;
  const uint32_t* negwin;
  const EItem* eitems;
  const uint2* litems;
  uint32_t n_eitems;                 // host upper bound (grid sizing)
  const uint32_t* n_eitems_dev;      // device count (written by the prep)
  const uint32_t* n_litems;  // device count (written by the prep)
  uint32_t* next;  // [0] E claims, [1] L claims
  const uint32_t* cbase;
  const uint32_t* lbase;
  const uint32_t* lpo;
  const uint32_t* needs;  // per vertex: window arcs/negatives exist
  double* epart;            // fp64 partial rows, compact: slots pslot[p] .. of position p
  const uint32_t* pslot;    // per position: first partial slot (hub chunks / needs-L vertices)
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
  uint32_t C, G, W, R, lwarps;
  // vertex-partitioned shards: step j of a vertex = state >> 1,
  // its negatives = set j * shards + shard(u); finalised rows are also stored
  // into the peers' Znew replicas (NVLink P2P) when npeers > 0
  uint32_t shards, npeers;
  uint32_t shard_lo[kMaxShards + 1];  // shard g owns rows [shard_lo[g], shard_lo[g+1])
  float* peer_znew[kMaxShards];
  // replica emulation (tests, F2V_EMULATE_REPLICAS): one launch runs every
  // shard, but shard g's items read and write replica rep_znew[g] and store
  // each finished row into every other replica -- the G-GPU data flow
  // (store_peers, sentinel polls on peer-written rows) inside one kernel
  uint32_t emul;
  float* rep_znew[kMaxShards];
  float eta;
  ForceParams fp;
  uint64_t nnz, chunks, lslots;  // bounds, used by F2V_DEVICE_CHECKS builds
  const uint32_t* stop;         // back-to-back epochs: an earlier epoch failed -> no work
  int nodep;                    // DEBUG (F2V_DEBUG_NODEP): every row read from Zold, no waits
  unsigned long long* trace;    // DEBUG (F2V_TRACE): per position finalise time (ns)
  unsigned long long* ltrace;   // DEBUG (F2V_TRACE): per position L-item stage times (4 x ns)
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

#ifdef F2V_DEVICE_CHECKS
#define DCHECK(cond, ...)                                                      \
  do {                                                                         \
    if (!(cond)) {                                                             \
      printf("F2V_DEVICE_CHECK %s:%d " #cond " | ", __FILE__, __LINE__);      \
      printf(__VA_ARGS__);                                                     \
      printf("\n");                                                           \
      __trap();                                                                \
    }                                                                          \
  } while (0)
#else
#define DCHECK(cond, ...) \
  do {                    \
  } while (0)
#endif

// Debug instrumentation (F2V_DEBUG_NODEP, F2V_TRACE) is compiled in only for
// debug builds (F2V_NVCC_EXTRA=-DF2V_DEBUG_BUILD): the epoch kernel is
// instruction-fetch sensitive, so release builds carry none of it.
#ifdef F2V_DEBUG_BUILD
#define F2V_NODEP(a) ((a).nodep)
#define F2V_STAMP(ptr, idx) \
  do {                      \
    if (ptr) (ptr)[idx] = globaltimer(); \
  } while (0)
#else
#define F2V_NODEP(a) false
#define F2V_STAMP(ptr, idx) \
  do {                      \
  } while (0)
#endif

__device__ __forceinline__ uint32_t lanemask_lt(int lane) { return (1u << lane) - 1u; }

// shard g owns rows [lo[g], lo[g+1]) (orc_shard_layout; G <= kMaxShards)
// (not unrolled: an unrolled scan over the kernel-parameter array cost ~700
// instructions and ~90 local loads in the epoch kernel, which is instruction-
// fetch sensitive; it runs only for G > 1)
__device__ __forceinline__ uint32_t shard_of(uint32_t u, const uint32_t* lo, uint32_t G) {
  uint32_t g = 0;
#pragma unroll 1
  for (uint32_t i = 1; i < G; ++i) g += u >= lo[i] ? 1u : 0u;
  return g;
}
// index of the negative set of a vertex of step j: one set per (step, shard)
__device__ __forceinline__ uint32_t neg_set(const EpochArgs& a, uint32_t u, uint32_t j) {
  return a.shards == 1 ? j : j * a.shards + shard_of(u, a.shard_lo, a.shards);
}

// the Znew replica the items of vertex u read and publish into
// (EMUL: the replica-emulation instantiation, f2v_epoch_i_emul.cu; the
// production kernels carry none of it -- it cost C2 ~7% as a run-time branch)
template <bool EMUL>
__device__ __forceinline__ float* znew_of(const EpochArgs& a, uint32_t u) {
  if constexpr (EMUL) return a.rep_znew[shard_of(u, a.shard_lo, a.shards)];
  (void)u;
  return a.znew;
}

// Per-warp FIFO of packed row ids (bit 31 = Znew) in shared memory; rows
// are accumulated 32 at a time in push order (= the deterministic pair order).
// E items: the next groups' column ids / states in flight while this group's
// rows are reduced (the col -> state -> row chain is three dependent loads per
// arc).  Same-box A/B, C3 kernel: EXACT 36.1 -> 35.2 ms; FAST 27.3 -> 25.4 ms
// with the round-2 row function (it was a loss, 28.9 -> 29.5 ms, while the old
// 80-register row function spilled the prefetched words); C2 neutral.
#ifndef F2V_E_PREFETCH_EXACT
#define F2V_E_PREFETCH_EXACT 1
#endif
#ifndef F2V_E_PREFETCH_FAST
#define F2V_E_PREFETCH_FAST 1
#endif

#ifndef F2V_INLINE_E
#define F2V_INLINE_E 0  // E items: the row function inlined at their queue (1) or called (0)
#endif

template <int KIND, int K, bool VEC, bool MON, bool FAST, bool ATT, bool EMUL, bool INL = false>
struct RowQueue {
  uint32_t* buf;
  int n;
  const float* zn;  // the Znew replica of the item (EMUL; else a.znew, reloaded per call)
  __device__ __forceinline__ void push(const EpochArgs& a, int lane, bool keep, uint32_t val,
                                       const float (&zu)[K], double (&acc)[K], double& lsum) {
    const uint32_t m = __ballot_sync(kFull, keep);
    if (keep) buf[n + __popc(m & lanemask_lt(lane))] = val;
    __syncwarp();
    n += __popc(m);
    if (n >= 32) {
      const uint32_t pk = buf[lane];
      const uint32_t rest = lane + 32 < n ? buf[lane + 32] : 0u;
      __syncwarp();
      buf[lane] = rest;
      __syncwarp();
      n -= 32;
      if constexpr (INL)
        Rows<KIND, K, VEC, MON, FAST>::template run_inl<ATT>(a.fp, pk, 32, lane, a.d, a.zold,
                                                             EMUL ? zn : a.znew, zu, acc, lsum);
      else
        Rows<KIND, K, VEC, MON, FAST>::template run<ATT>(a.fp, pk, 32, lane, a.d, a.zold,
                                                         EMUL ? zn : a.znew, zu, acc, lsum);
    }
  }
  __device__ __forceinline__ void flush(const EpochArgs& a, int lane, const float (&zu)[K],
                                        double (&acc)[K], double& lsum) {
    if (n == 0) return;
    const uint32_t pk = lane < n ? buf[lane] : 0u;
    __syncwarp();
    const int cnt = n;
    n = 0;
    if constexpr (INL)
      Rows<KIND, K, VEC, MON, FAST>::template run_inl<ATT>(a.fp, pk, cnt, lane, a.d, a.zold,
                                                           EMUL ? zn : a.znew, zu, acc, lsum);
    else
      Rows<KIND, K, VEC, MON, FAST>::template run<ATT>(a.fp, pk, cnt, lane, a.d, a.zold,
                                                       EMUL ? zn : a.znew, zu, acc, lsum);
  }
};

// The shared negatives of batch j, in sample order (sampling.cpp:59).
template <int KIND, int K, bool VEC, bool MON, bool FAST, bool EMUL>
__device__ __forceinline__ void do_negatives(const EpochArgs& a, const float* zn, uint32_t j,
                                             uint32_t q, int lane, const float (&zu)[K],
                                             double (&acc)[K], double& lsum) {
  for (uint32_t k0 = 0; k0 < a.s; k0 += 32) {
    const int cnt = int(umin32(32, a.s - k0));
    uint32_t pk = 0;
    if (lane < cnt) {
      const uint32_t w = a.negs[size_t(q) * a.s + k0 + lane];
      const uint32_t st = ld_relaxed(a.state + w);
      if ((st >> 1) < j && !F2V_NODEP(a)) {
        pk = w | kNewBit;  // Znew row: the row loads poll its sentinel
      } else {
        pk = w;
      }
    }
    Rows<KIND, K, VEC, MON, FAST>::template run<false>(a.fp, pk, cnt, lane, a.d, a.zold,
                                                       EMUL ? zn : a.znew, zu, acc, lsum);
  }
}

// the row into every peer GPU's Znew replica (multi-GPU shards), out of line
template <int K, bool VEC>
__device__ __noinline__ void store_peers(const EpochArgs& a, const float* zn, uint32_t u, int lane,
                                         const float (&nz)[K]) {
  if (a.emul) {  // every other emulated replica
    for (uint32_t g = 0; g < a.shards; ++g)
      if (a.rep_znew[g] != zn) Lay<K, VEC>::store(a.rep_znew[g] + size_t(u) * a.d, lane, a.d, nz);
    return;
  }
  for (uint32_t g = 0; g < a.npeers; ++g)
    Lay<K, VEC>::store(a.peer_znew[g] + size_t(u) * a.d, lane, a.d, nz);
}

// g = float(acc) (trainer.cpp:140-145); z_u -= eta*g in fp32 (trainer.cpp:173);
// publish row u of Znew.
template <int K, bool VEC, bool MON, bool EMUL>
__device__ __forceinline__ void finalize(const EpochArgs& a, float* zn, uint32_t p, uint32_t u,
                                         int lane, const float (&zu)[K], const double (&acc)[K],
                                         double lsum) {
  using L = Lay<K, VEC>;
  bool bad = false;
  float nz[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float g = __double2float_rn(acc[k]);
    if (L::valid(lane, k, a.d) && !isfinite(g)) bad = true;
    nz[k] = __fsub_rn(zu[k], __fmul_rn(a.eta, g));
    if (nz[k] != nz[k]) nz[k] = __int_as_float(0x7fffffff);  // never the sentinel NaN
  }
  L::store((EMUL ? zn : a.znew) + size_t(u) * a.d, lane, a.d, nz);  // publishes the row
  if (EMUL || a.npeers) store_peers<K, VEC>(a, zn, u, lane, nz);  // peers' replicas (NVLink)
  const bool any_bad = __any_sync(kFull, bad);
  if (MON) {
    const double tot = warp_sum_d(lsum);
    if (lane == 0) a.ploss[p] = tot;
  }
  if (lane == 0) {
    if (any_bad) atomicMin(a.bad, (unsigned long long)p);
    F2V_STAMP(a.trace, p);
  }
}

template <int KIND, int K, bool VEC, bool MON, bool FAST, bool EMUL>
__device__ void do_E(const EpochArgs& a, const EItem& item, int lane, uint32_t* qbuf) {
  using L = Lay<K, VEC>;
  const uint32_t p = item.p, u = item.u, cb = item.cb, c = item.c, nch = item.nch;
  DCHECK(p < a.n && u < a.n, "E p=%u u=%u n=%u", p, u, a.n);
  const uint32_t j = __ldg(a.state + u) >> 1;
  const uint32_t needs_w = __ldg(a.needs + u);  // static during the launch; used at the end
  const uint32_t cs = cb + c;
  const uint32_t ps = __ldg(a.pslot + p);  // partial slots of u (used when nch > 1 or needs-L)
  DCHECK(c < nch && cs < a.chunks, "E c=%u nch=%u cs=%u chunks=%llu", c, nch, cs,
         (unsigned long long)a.chunks);
  const uint64_t e0 = item.e0;
  const uint64_t e1 = e0 + item.cnt;
  float zu[K];
  L::load(a.zold + size_t(u) * a.d, lane, a.d, zu, false);
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  double lsum = 0.0;
  uint32_t wc = 0;
  float* zn = znew_of<EMUL>(a, u);
  RowQueue<KIND, K, VEC, MON, FAST, true, EMUL, F2V_INLINE_E != 0> q{qbuf, 0, zn};
  // Software pipeline over the chunk's 32-arc groups: while group i's rows
  // are gathered and reduced, group i+1's states and group i+2's column ids
  // are already in flight (the col -> state -> row chain is three dependent
  // loads per arc).
  constexpr bool PRE = FAST ? F2V_E_PREFETCH_FAST != 0 : F2V_E_PREFETCH_EXACT != 0;
  uint32_t v_cur = 0, v_nx = 0, st_cur = 0;
  if constexpr (PRE) {
    v_cur = e0 + lane < e1 ? __ldg(a.col + e0 + lane) : 0u;            // this group's ids
    v_nx = e0 + 32 + lane < e1 ? __ldg(a.col + e0 + 32 + lane) : 0u;  // the next's
    st_cur = e0 + lane < e1 ? ld_relaxed(a.state + v_cur) : 0u;       // this group's states
  }
  for (uint64_t e = e0; e < e1; e += 32) {
    const int cnt = int(umin64(32, e1 - e));
    uint32_t v, st;
    if constexpr (PRE) {
      v = v_cur;
      st = st_cur;
      // issue the next group's states and the group after's column ids
      st_cur = e + 32 + lane < e1 ? ld_relaxed(a.state + v_nx) : 0u;
      v_cur = v_nx;
      v_nx = e + 64 + lane < e1 ? __ldg(a.col + e + 64 + lane) : 0u;
    } else {
      v = lane < cnt ? a.col[e + lane] : 0u;
      st = lane < cnt ? ld_relaxed(a.state + v) : 0u;
    }
    uint32_t pk = 0;
    bool use = false, win = false;
    if (lane < cnt) {
      DCHECK(e + lane < a.nnz, "E arc %llu nnz %llu", (unsigned long long)(e + lane),
             (unsigned long long)a.nnz);
      DCHECK(v < a.n, "E v=%u", v);
      const uint32_t bv = st >> 1;
      if (bv >= j || F2V_NODEP(a)) {
        use = true;
        pk = v;
      } else if (bv + a.W < j) {  // past: final long ago (the row load rarely polls)
        use = true;
        pk = v | kNewBit;
      } else {
        win = true;
      }
    }
    const uint32_t wm = __ballot_sync(kFull, win);
    DCHECK(!win || e0 + wc + __popc(wm & lanemask_lt(lane)) < e1, "E wl overflow");
    if (win) a.wl[e0 + wc + __popc(wm & lanemask_lt(lane))] = v;
    wc += __popc(wm);
    q.push(a, lane, use, pk, zu, acc, lsum);
  }
  q.flush(a, lane, zu, acc, lsum);
  const bool needs = needs_w != 0;
  if (nch == 1) {
    if (!needs) {
      do_negatives<KIND, K, VEC, MON, FAST, EMUL>(a, zn, j, neg_set(a, u, j), lane, zu, acc, lsum);
      finalize<K, VEC, MON, EMUL>(a, zn, p, u, lane, zu, acc, lsum);
    } else {
      L::store_acc(a.epart + size_t(ps) * a.d, lane, a.d, acc);
      const double ls = MON ? warp_sum_d(lsum) : 0.0;
      if (lane == 0) {
        if (MON) __stcg(a.eloss + cs, ls);
        __stcg(a.wcnt + cs, wc);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_relaxed(a.vflag + u, 1u);
    }
    return;
  }
  // hub chunk: publish the partial; the last E arrival combines in chunk order
  L::store_acc(a.epart + size_t(ps + c) * a.d, lane, a.d, acc);
  {
    const double ls = MON ? warp_sum_d(lsum) : 0.0;
    if (lane == 0) {
      if (MON) __stcg(a.eloss + cs, ls);
      __stcg(a.wcnt + cs, wc);
    }
  }
  __threadfence();
  __syncwarp();
  uint32_t last = 0;
  if (lane == 0) last = atomicAdd(a.ecnt + u, 1u) == nch - 1 ? 1u : 0u;
  if (!__shfl_sync(kFull, last, 0)) return;
  __threadfence();
  L::load_acc(a.epart + size_t(ps) * a.d, lane, a.d, acc);
  lsum = (MON && lane == 0) ? __ldcg(a.eloss + cb) : 0.0;
#pragma unroll 4
  for (uint32_t qq = 1; qq < nch; ++qq) {
    L::add_acc(a.epart + size_t(ps + qq) * a.d, lane, a.d, acc);
    if (MON && lane == 0) lsum = __dadd_rn(lsum, __ldcg(a.eloss + cb + qq));
  }
  if (lane == 0) a.ecnt[u] = 0;
  if (!needs) {
    do_negatives<KIND, K, VEC, MON, FAST, EMUL>(a, zn, j, neg_set(a, u, j), lane, zu, acc, lsum);
    finalize<K, VEC, MON, EMUL>(a, zn, p, u, lane, zu, acc, lsum);
  } else {
    L::store_acc(a.epart + size_t(ps) * a.d, lane, a.d, acc);  // the E total
    if (MON && lane == 0) __stcg(a.eloss + cb, lsum);  // lane 0 holds the whole sum here
    __threadfence();
    __syncwarp();
    if (lane == 0) st_relaxed(a.vflag + u, 1u);
  }
}

// Take the parked recent window arcs in order, waiting on each row.
template <int KIND, int K, bool VEC, bool MON, bool FAST, bool EMUL>
__device__ __forceinline__ void recent_pass(const EpochArgs& a, const float* zn, int lane,
                                            uint32_t* rbuf, int& nr, const float (&zu)[K],
                                            double (&acc)[K], double& lsum) {
  for (int t0 = 0; t0 < nr; t0 += 32) {
    const int cnt = min(32, nr - t0);
    uint32_t pk = 0;
    if (lane < cnt) {
      const uint32_t v = rbuf[t0 + lane];
      pk = v | kNewBit;
    }
    Rows<KIND, K, VEC, MON, FAST>::template run<true>(a.fp, pk, cnt, lane, a.d, a.zold,
                                                      EMUL ? zn : a.znew, zu, acc, lsum);
  }
  __syncwarp();
  nr = 0;
}

// Window arcs of chunks [c0, c1) of u.  All chunk counts are fetched at once
// and the lists walked as one flattened sequence: arcs older than R batches go
// straight into the row queue; the most recent ones are parked in rbuf and
// taken last (recent_pass) so the dependency tail of the item is short.  The
// order is a function of the data only (deterministic).
template <int KIND, int K, bool VEC, bool MON, bool FAST, bool EMUL>
__device__ __forceinline__ void window_collect(const EpochArgs& a, const float* zn, uint32_t u,
                                               uint32_t j, uint32_t c0, uint32_t c1, int lane,
                                               uint32_t* qbuf, uint32_t* rbuf, int& nr,
                                               const float (&zu)[K], double (&acc)[K],
                                               double& lsum) {
  const uint64_t r0 = a.rowptr[u];
  const uint32_t cb = a.cbase[u];
  RowQueue<KIND, K, VEC, MON, FAST, true, EMUL> q{qbuf, 0, zn};
  for (uint32_t cc = c0; cc < c1; cc += 32) {
    const uint32_t nc = umin32(32, c1 - cc);
    const uint32_t mine = lane < int(nc) ? __ldcg(a.wcnt + cb + cc + lane) : 0u;
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t excl = incl - mine;
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
      const uint32_t t = t0 + lane;
      // chunk of flattened position t: the last chunk whose exclusive start <= t
      uint32_t ci = 0, off = 0;
      for (uint32_t i = 0; i < nc; ++i) {  // shuffles outside any lane-divergent branch
        const uint32_t e = __shfl_sync(kFull, excl, i);
        const uint32_t m = __shfl_sync(kFull, mine, i);
        if (e <= t && m > 0) {
          ci = i;
          off = e;
        }
      }
      bool old = false, recent = false;
      uint32_t v = 0, st = 0;
      if (t < total) {
        DCHECK(cc + ci < c1 && t - off < a.C && r0 + uint64_t(cc + ci) * a.C + (t - off) < a.nnz,
               "L wl t=%u off=%u ci=%u cc=%u c1=%u", t, off, ci, cc, c1);
        v = __ldcg(a.wl + r0 + uint64_t(cc + ci) * a.C + (t - off));
        DCHECK(v < a.n, "L wl v=%u", v);
        st = ld_relaxed(a.state + v);
        const uint32_t age = j - (st >> 1);
        old = age > a.R;
        recent = !old;
      }
      const uint32_t rm = __ballot_sync(kFull, recent);
      q.push(a, lane, old, v | kNewBit, zu, acc, lsum);
      // park the recent ones (processed in place if the parking lot is full)
      if (nr + __popc(rm) > kRq) {
        q.flush(a, lane, zu, acc, lsum);
        recent_pass<KIND, K, VEC, MON, FAST, EMUL>(a, zn, lane, rbuf, nr, zu, acc, lsum);
      }
      if (recent) rbuf[nr + __popc(rm & lanemask_lt(lane))] = v;
      __syncwarp();
      nr += __popc(rm);
    }
  }
  q.flush(a, lane, zu, acc, lsum);
}

template <int KIND, int K, bool VEC, bool MON, bool FAST, bool EMUL>
__device__ void do_L(const EpochArgs& a, uint32_t p, uint32_t cl, int lane, uint32_t* qbuf,
                     uint32_t* rbuf) {
  using L = Lay<K, VEC>;
  DCHECK(p < a.n, "L p=%u", p);
  const uint32_t u = a.perm[p];
  DCHECK(u < a.n, "L u=%u", u);
  const uint32_t j = __ldg(a.state + u) >> 1;
  const uint32_t cb = a.cbase[u];
  const uint32_t nch = a.cbase[u + 1] - cb;
  const uint32_t nchL = a.lbase[u + 1] - a.lbase[u];
#ifdef F2V_DEBUG_BUILD
  unsigned long long* lt = (a.ltrace && cl == 0) ? a.ltrace + 4ull * p : nullptr;
#endif
  if (lane == 0) F2V_STAMP(lt, 0);
  float* zn = znew_of<EMUL>(a, u);
  float zu[K];
  L::load(a.zold + size_t(u) * a.d, lane, a.d, zu, false);
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  double lsum = 0.0;
  // the E work of u must be complete (its partial and window lists)
  uint32_t f = ld_relaxed(a.vflag + u);
  while (f == 0) {
    __nanosleep(64);
    f = ld_relaxed(a.vflag + u);
  }
  if (lane == 0) F2V_STAMP(lt, 1);
  const uint32_t c0 = cl * a.G, c1 = umin32(nch, c0 + a.G);
  const uint32_t ps = __ldg(a.pslot + p);  // the E total of u lives in partial slot ps
  if (nchL == 1) {
    L::load_acc(a.epart + size_t(ps) * a.d, lane, a.d, acc);
    if (MON && lane == 0) lsum = __ldcg(a.eloss + cb);
    int nr = 0;
    // E total + old window arcs + negatives + recent arcs
    window_collect<KIND, K, VEC, MON, FAST, EMUL>(a, zn, u, j, c0, c1, lane, qbuf, rbuf, nr, zu, acc,
                                            lsum);
    do_negatives<KIND, K, VEC, MON, FAST, EMUL>(a, zn, j, neg_set(a, u, j), lane, zu, acc, lsum);
    if (lane == 0) F2V_STAMP(lt, 2);
    recent_pass<KIND, K, VEC, MON, FAST, EMUL>(a, zn, lane, rbuf, nr, zu, acc, lsum);
    if (lane == 0) F2V_STAMP(lt, 3);
    finalize<K, VEC, MON, EMUL>(a, zn, p, u, lane, zu, acc, lsum);
    if (lane == 0) a.vflag[u] = 0;
    return;
  }
  int nr = 0;
  window_collect<KIND, K, VEC, MON, FAST, EMUL>(a, zn, u, j, c0, c1, lane, qbuf, rbuf, nr, zu, acc,
                                          lsum);
  recent_pass<KIND, K, VEC, MON, FAST, EMUL>(a, zn, lane, rbuf, nr, zu, acc, lsum);
  const uint32_t slot = a.lpo[u] + cl;
  DCHECK(slot < a.lslots, "L slot=%u lslots=%llu cl=%u nchL=%u", slot,
         (unsigned long long)a.lslots, cl, nchL);
  L::store_acc(a.lpart + size_t(slot) * a.d, lane, a.d, acc);
  {
    const double ls = MON ? warp_sum_d(lsum) : 0.0;
    if (MON && lane == 0) __stcg(a.lloss + slot, ls);
  }
  __threadfence();
  __syncwarp();
  uint32_t last = 0;
  if (lane == 0) last = atomicAdd(a.lcnt + u, 1u) == nchL - 1 ? 1u : 0u;
  if (!__shfl_sync(kFull, last, 0)) return;
  __threadfence();
  L::load_acc(a.epart + size_t(ps) * a.d, lane, a.d, acc);
  lsum = (MON && lane == 0) ? __ldcg(a.eloss + cb) : 0.0;
  const uint32_t lp = a.lpo[u];
#pragma unroll 4
  for (uint32_t qq = 0; qq < nchL; ++qq) {
    L::add_acc(a.lpart + size_t(lp + qq) * a.d, lane, a.d, acc);
    if (MON && lane == 0) lsum = __dadd_rn(lsum, __ldcg(a.lloss + lp + qq));
  }
  do_negatives<KIND, K, VEC, MON, FAST, EMUL>(a, zn, j, neg_set(a, u, j), lane, zu, acc, lsum);
  if (lane == 0) a.lcnt[u] = 0;
  finalize<K, VEC, MON, EMUL>(a, zn, p, u, lane, zu, acc, lsum);
  if (lane == 0) a.vflag[u] = 0;
}

template <int KIND, int K, bool VEC, bool MON, bool FAST, int MINB, bool EMUL = false>
__global__ void __launch_bounds__(kWarps * 32, MINB) epoch_kernel(EpochArgs a) {
  __shared__ uint32_t qs[kWarps][kQ];
  __shared__ uint32_t rs[kWarps][kRq];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  uint32_t* qbuf = qs[w];
  uint32_t* rbuf = rs[w];
  if (uses_ring<K, VEC, FAST>()) ring_init(lane);
  const bool lrole = w >= kWarps - int(a.lwarps);
  if (a.stop && ld_relaxed(a.stop)) return;  // an earlier epoch of this call failed
  uint32_t* counter = a.next + (lrole ? 1 : 0);
  const uint32_t total = lrole ? *a.n_litems : *a.n_eitems_dev;
  uint32_t it = 0;
  if (lane == 0) it = atomicAdd(counter, 1u);
  it = __shfl_sync(kFull, it, 0);
  while (it < total) {
    DCHECK(it < (lrole ? a.chunks + a.lslots + a.n : a.chunks), "item %u", it);
    uint32_t nxt = 0;
    if (lane == 0) nxt = atomicAdd(counter, 1u);  // claim ahead: hides the atomic's latency
    if (lrole) {
      const uint2 item = a.litems[it];
      do_L<KIND, K, VEC, MON, FAST, EMUL>(a, item.x, item.y, lane, qbuf, rbuf);
    } else {
      do_E<KIND, K, VEC, MON, FAST, EMUL>(a, a.eitems[it], lane, qbuf);
    }
    it = __shfl_sync(kFull, nxt, 0);
  }
}

// Launch one epoch kernel instantiation as a persistent grid.
template <int KIND, int K, bool VEC, bool MON, bool FAST, int MINB, bool EMUL = false>
void launch_one(Ctx& c, const EpochArgs& a) {
  auto kern = epoch_kernel<KIND, K, VEC, MON, FAST, MINB, EMUL>;
  const size_t dsmem = size_t(kWarps) * warp_smem_bytes<K, VEC, FAST>();
  if (dsmem) F2V_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(dsmem)));
  if (c.dry_launch) {  // load the function only (CUDA lazy loading) -- no launch
    cudaFuncAttributes fa;
    F2V_CUDA(cudaFuncGetAttributes(&fa, kern));
    return;
  }
  int per_sm = 0;
  F2V_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, dsmem));
  if (c.tune.ctas && int(c.tune.ctas) < per_sm) per_sm = int(c.tune.ctas);
  if (per_sm < 1) per_sm = 1;
  uint32_t blocks = uint32_t(per_sm) * uint32_t(c.num_sms);
  const uint64_t ew = kWarps - a.lwarps;
  const uint32_t need = uint32_t(std::max<uint64_t>((a.n_eitems + ew - 1) / ew, 1));
  blocks = std::max(1u, std::min(blocks, need));
  kern<<<blocks, kWarps * 32, dsmem, c.stream>>>(a);
  F2V_LAUNCHED(c.stream, "kern");
  ++c.launches;
}

#ifndef F2V_EXACT_MINB
// EXACT d = 128 register budget (resident 8-warp CTAs per SM).  Register
// gathers: 3 (80 registers, 24 warps/SM) measured 57.7 ms on C3 against 65.1
// ms at 2 (128); with the TMA row ring (F2V_ROW_TMA_EXACT) 2 is better: 56.3
// ms against 66.5 ms at 3 with one ring stage (the ring's shared memory
// costs resident L1)
#define F2V_EXACT_MINB ((F2V_EXACT_V3 || F2V_ROW_TMA_EXACT) ? 2 : 3)
#endif

#ifndef F2V_FAST_MINB_HI
#define F2V_FAST_MINB_HI 3  // FAST d = 128: the occupancy autotune's high-occupancy build
#endif

template <int KIND, int K, bool VEC, bool FAST>
void launch_mon(Ctx& c, const EpochArgs& a, bool mon) {
  if constexpr (!FAST && K == 4 && VEC) {
    if (mon) launch_one<KIND, K, VEC, true, FAST, F2V_EXACT_MINB>(c, a);
    else launch_one<KIND, K, VEC, false, FAST, F2V_EXACT_MINB>(c, a);
  } else if constexpr (FAST && K == 1 && !VEC) {
    // the low-d lane-per-pair path (config 4) is latency-bound: 3 CTAs/SM
    // (80 registers); at 2 the compiler takes 116 and C4 ran 2.2 -> 3.4 ms
    if (mon) launch_one<KIND, K, VEC, true, FAST, 3>(c, a);
    else launch_one<KIND, K, VEC, false, FAST, 3>(c, a);
  } else {
    if constexpr (FAST && K == 4) {
      if (c.occ_use == 3) {
        if (mon) launch_one<KIND, K, VEC, true, FAST, F2V_FAST_MINB_HI>(c, a);
        else launch_one<KIND, K, VEC, false, FAST, F2V_FAST_MINB_HI>(c, a);
        return;
      }
    }
    if (mon) launch_one<KIND, K, VEC, true, FAST, 2>(c, a);
    else launch_one<KIND, K, VEC, false, FAST, 2>(c, a);
  }
}

template <int K, bool VEC, bool FAST>
void launch_kind(Ctx& c, const EpochArgs& a, bool mon) {
  switch (a.fp.kind) {
    case F2V_SIGMOID: launch_mon<F2V_SIGMOID, K, VEC, FAST>(c, a, mon); break;
    case F2V_TDIST: launch_mon<F2V_TDIST, K, VEC, FAST>(c, a, mon); break;
    case F2V_FR: launch_mon<F2V_FR, K, VEC, FAST>(c, a, mon); break;
    case F2V_FA: launch_mon<F2V_FA, K, VEC, FAST>(c, a, mon); break;
    default: launch_mon<F2V_LINLOG, K, VEC, FAST>(c, a, mon); break;
  }
}

// instantiation translation units (f2v_epoch_i_*.cu, compiled in parallel)
void launch_fast_k4(Ctx& c, const EpochArgs& a, bool mon);
void launch_fast_k2(Ctx& c, const EpochArgs& a, bool mon);
void launch_fast_k8(Ctx& c, const EpochArgs& a, bool mon);
void launch_fast_lowd(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_vec_k1(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_vec_k2(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_vec_k4(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_vec_k8(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_any_k1(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_any_k2(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_any_k4(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_any_k8(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_any_k16(Ctx& c, const EpochArgs& a, bool mon);
void launch_exact_any_k32(Ctx& c, const EpochArgs& a, bool mon);
void launch_emul(Ctx& c, const EpochArgs& a, bool mon, bool fast);  // f2v_epoch_i_emul.cu

// d = 64/128/256 and d <= 4 (lane-per-pair, rows_lowd) run FAST when asked;
// everything else runs EXACT.
inline void launch_epoch(Ctx& c, const EpochArgs& a, bool mon, bool fast) {
  const uint32_t d = a.d;
  if (a.emul) {
    launch_emul(c, a, mon, fast);
    return;
  }
  if (fast && d == 128) launch_fast_k4(c, a, mon);
  else if (fast && d == 64) launch_fast_k2(c, a, mon);
  else if (fast && d == 256) launch_fast_k8(c, a, mon);
  else if (fast && d <= uint32_t(kLowD)) launch_fast_lowd(c, a, mon);
  else if (d == 128) launch_exact_vec_k4(c, a, mon);
  else if (d == 64) launch_exact_vec_k2(c, a, mon);
  else if (d == 256) launch_exact_vec_k8(c, a, mon);
  else if (d == 32) launch_exact_vec_k1(c, a, mon);
  else if (d < 32) launch_exact_any_k1(c, a, mon);
  else if (d < 64) launch_exact_any_k2(c, a, mon);
  else if (d < 128) launch_exact_any_k4(c, a, mon);
  else if (d < 256) launch_exact_any_k8(c, a, mon);
  else if (d <= 512) launch_exact_any_k16(c, a, mon);
  else if (d <= 1024) launch_exact_any_k32(c, a, mon);
  else fail(F2V_EUNSUPPORTED, "dim > 1024 is not supported by the device kernels");
}

}  // namespace ep
}  // namespace f2v

