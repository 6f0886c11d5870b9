// f2v_nccl.cu -- the per-step all-gather baseline of the G-shard schedule
// (SURVEY.md section 8(e) "implementation ladder (1)"), device-resident in the
// library: per step every rank computes its local batch's gradient on its
// full replica of Z, writes the updated rows (z_u - eta g_u, trainer.cpp:173)
// with their ids and a failure index into a pack, and an ncclAllGather over
// NVLink exchanges the packs; a vote kernel takes the first failure in
// (rank, batch index) order (trainer.cpp:149-152: no rank applies a failing
// step) and a scatter kernel writes every rank's rows into the local replica.
// No host staging and no host sync inside an epoch.  Same semantics, same
// numbers as the fused NVLink epoch kernel (f2v_epoch.cuh) and orc_train(G);
// it is the baseline the fused path is measured against.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the one already in the
// process -- torch's bundled NCCL, which the Python wrapper imports first --
// else the system one, RTLD_LOCAL), so the library has no link-time NCCL
// dependency; only <nccl.h>'s types are used.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "f2v_epoch.cuh"

namespace f2v {
namespace {

using namespace dev;

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // an NCCL already in the process first (torch's bundled one, whose newer
    // symbols torch needs), else the system library -- RTLD_LOCAL either way,
    // so this library never changes what other code resolves
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
      if (a.h) break;
    }
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      if (a.h) break;
      a.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    }
    if (!a.h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.h, "ncclGetUniqueId"));
    a.comm_init_rank =
        reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.h, "ncclCommInitRank"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.h, "ncclAllGather"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
    return a;
  }();
  if (!api.h || !api.get_unique_id || !api.comm_init_rank || !api.all_gather)
    fail(F2V_ECUDA, "NCCL (libnccl.so.2) is not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(F2V_ECUDA, std::string("NCCL error: ") +
                        (nccl().error_string ? nccl().error_string(r) : "?") + " at " + what);
}

// One rank's pack: header, ids[bmax], rows[bmax x d], per-row losses[bmax]
// (each section 16-byte aligned).
struct PackHdr {
  uint32_t count;   // rows of this rank's batch at this step
  uint32_t fail;    // first non-finite row in batch order, or ~0
  double loss;      // batch_loss partial (monitoring)
};

struct PackLayout {
  size_t ids, rows, loss, bytes;
  PackLayout(uint32_t bmax, uint32_t d) {
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    ids = 16;
    rows = ids + al(sizeof(uint32_t) * bmax);
    loss = rows + al(sizeof(float) * size_t(bmax) * d);
    bytes = (loss + sizeof(double) * bmax + 255) & ~size_t(255);
  }
};

struct AgArgs {
  const uint64_t* rowptr;
  const uint32_t* col;
  float* z;                 // the replica (read: snapshot; written only by the scatter)
  const uint32_t* perm;     // combined step-major order (k_epoch_perm)
  const uint32_t* negs;     // negative sets of every (step, shard)
  uint8_t* send;            // this rank's pack
  const uint8_t* recv;      // every rank's pack (rank order)
  uint32_t* stop;           // [0] stopped, [1] step, [2] rank, [3] index, [4] vertex
  double* loss;             // epoch loss, summed in (step, rank) order
  uint32_t p0, cnt;         // this rank's batch at this step: positions [p0, p0 + cnt)
  uint32_t q;               // its negative set
  uint32_t step, world, bmax, d, s;
  size_t pack_bytes, ids_off, rows_off, loss_off;
  float eta;
  ForceParams fp;
};

// The local batch: one warp per row; fp64 (EXACT, the reference's order) or
// FAST pair math as in the epoch kernel; new rows into the send pack.
template <int KIND, int K, bool VEC, bool MON, bool FAST>
__global__ void __launch_bounds__(256) ag_step_kernel(AgArgs a) {
  using L = Lay<K, VEC>;
  PackHdr* hdr = reinterpret_cast<PackHdr*>(a.send);
  uint32_t* ids = reinterpret_cast<uint32_t*>(a.send + a.ids_off);
  float* rows = reinterpret_cast<float*>(a.send + a.rows_off);
  double* vloss = reinterpret_cast<double*>(a.send + a.loss_off);
  const bool stopped = ld_relaxed(a.stop) != 0;
  const uint32_t cnt = stopped ? 0u : a.cnt;
  // hdr->fail was reset to ~0 by the previous step's vote (or the epoch start)
  if (blockIdx.x == 0 && threadIdx.x == 0) hdr->count = cnt;
  const int lane = threadIdx.x & 31;
  if (uses_ring<K, VEC, FAST>()) ring_init(lane);
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= cnt) return;
  const uint32_t u = a.perm[a.p0 + i];
  float zu[K];
  L::load(a.z + size_t(u) * a.d, lane, a.d, zu, true);
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  double lsum = 0.0;
  const uint64_t r0 = a.rowptr[u], r1 = a.rowptr[u + 1];
  for (uint64_t e = r0; e < r1; e += 32) {  // context arcs in CSR order (trainer.cpp:129-133)
    const int c = int(umin64(32, r1 - e));
    const uint32_t v = lane < c ? a.col[e + lane] : 0u;
    Rows<KIND, K, VEC, MON, FAST>::template run<true>(a.fp, v, c, lane, a.d, a.z, a.z, zu, acc,
                                                      lsum);
  }
  for (uint32_t k0 = 0; k0 < a.s; k0 += 32) {  // then the negatives (134-138)
    const int c = int(umin32(32, a.s - k0));
    const uint32_t w = lane < c ? a.negs[size_t(a.q) * a.s + k0 + lane] : 0u;
    Rows<KIND, K, VEC, MON, FAST>::template run<false>(a.fp, w, c, lane, a.d, a.z, a.z, zu, acc,
                                                       lsum);
  }
  bool bad = false;
  float nz[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float g = __double2float_rn(acc[k]);  // trainer.cpp:142
    if (L::valid(lane, k, a.d) && !isfinite(g)) bad = true;
    nz[k] = __fsub_rn(zu[k], __fmul_rn(a.eta, g));  // trainer.cpp:173
  }
  L::store(rows + size_t(i) * a.d, lane, a.d, nz);
  if (lane == 0) ids[i] = u;
  if (__any_sync(kFull, bad) && lane == 0) atomicMin(&hdr->fail, i);
  if (MON) {
    const double tot = warp_sum_d(lsum);
    if (lane == 0) vloss[i] = tot;
  }
}

// The step's vote (first failure in (rank, index) order), the loss partials
// in rank order, and the stop flag -- one thread.
template <bool MON>
__global__ void ag_vote_kernel(AgArgs a) {
  if (threadIdx.x || blockIdx.x) return;
  reinterpret_cast<PackHdr*>(a.send)->fail = ~0u;  // the send pack is free again: next step
  if (a.stop[0]) return;
  for (uint32_t r = 0; r < a.world; ++r) {
    const uint8_t* p = a.recv + size_t(r) * a.pack_bytes;
    const PackHdr* h = reinterpret_cast<const PackHdr*>(p);
    if (h->fail != ~0u) {
      a.stop[0] = 1;
      a.stop[1] = a.step;
      a.stop[2] = r;
      a.stop[3] = h->fail;
      a.stop[4] = reinterpret_cast<const uint32_t*>(p + a.ids_off)[h->fail];
      return;
    }
  }
  if (MON) {  // batch_loss of every rank's batch, summed in (step, rank) order
    for (uint32_t r = 0; r < a.world; ++r) {
      const uint8_t* p = a.recv + size_t(r) * a.pack_bytes;
      const uint32_t cnt = reinterpret_cast<const PackHdr*>(p)->count;
      const double* vl = reinterpret_cast<const double*>(p + a.loss_off);
      double s = 0.0;
      for (uint32_t i = 0; i < cnt; ++i) s = __dadd_rn(s, vl[i]);
      *a.loss = __dadd_rn(*a.loss, s);
    }
  }
}

// every rank's new rows into the local replica (after a passing vote)
__global__ void ag_scatter_kernel(AgArgs a) {
  if (ld_relaxed(a.stop) != 0) return;
  const uint64_t per = uint64_t(a.bmax) * a.d;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < per * a.world;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = uint32_t(t / per), i = uint32_t((t % per) / a.d), c = uint32_t(t % a.d);
    const uint8_t* p = a.recv + size_t(r) * a.pack_bytes;
    if (i >= reinterpret_cast<const PackHdr*>(p)->count) continue;
    const uint32_t u = reinterpret_cast<const uint32_t*>(p + a.ids_off)[i];
    a.z[size_t(u) * a.d + c] = reinterpret_cast<const float*>(p + a.rows_off)[size_t(i) * a.d + c];
  }
}

template <int KIND, int K, bool VEC, bool FAST>
void launch_ag_step(const AgArgs& a, bool mon, cudaStream_t st) {
  const uint32_t blocks = std::max(1u, (a.cnt * 32 + 255) / 256);
  const size_t dsmem = 8 * size_t(warp_smem_bytes<K, VEC, FAST>());
  auto k1 = ag_step_kernel<KIND, K, VEC, true, FAST>;
  auto k0 = ag_step_kernel<KIND, K, VEC, false, FAST>;
  if (dsmem) {
    F2V_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dsmem)));
    F2V_CUDA(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dsmem)));
  }
  if (mon) k1<<<blocks, 256, dsmem, st>>>(a);
  else k0<<<blocks, 256, dsmem, st>>>(a);
}

// d = 128 (the bench row width) per force kind, FAST or EXACT; any other d
// runs the run-time-kind EXACT path
void launch_step_any(const AgArgs& a, bool mon, bool fast, cudaStream_t st) {
  if (a.d == 128) {
    switch (a.fp.kind) {
#define F2V_AG_KIND(KD)                                          \
  case KD:                                                      \
    if (fast) launch_ag_step<KD, 4, true, true>(a, mon, st);    \
    else launch_ag_step<KD, 4, true, false>(a, mon, st);        \
    return;
      F2V_AG_KIND(F2V_SIGMOID)
      F2V_AG_KIND(F2V_TDIST)
      F2V_AG_KIND(F2V_FR)
      F2V_AG_KIND(F2V_FA)
      F2V_AG_KIND(F2V_LINLOG)
#undef F2V_AG_KIND
      default: break;
    }
  }
  if (a.d <= 32) launch_ag_step<-1, 1, false, false>(a, mon, st);
  else if (a.d <= 64) launch_ag_step<-1, 2, false, false>(a, mon, st);
  else if (a.d <= 128) launch_ag_step<-1, 4, false, false>(a, mon, st);
  else if (a.d <= 256) launch_ag_step<-1, 8, false, false>(a, mon, st);
  else fail(F2V_EUNSUPPORTED, "the all-gather baseline supports dim <= 256");
}

}  // namespace

// host API (f2v_capi.cpp)
void nccl_unique_id(uint8_t* out) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

void k_nccl_init(Ctx& c, const uint8_t* id_bytes, uint32_t rank, uint32_t world) {
  if (world < 1 || world > uint32_t(ep::kMaxShards)) fail(F2V_EUSAGE, "world must be in [1, 8]");
  if (rank >= world) fail(F2V_EUSAGE, "rank out of range");
  if (c.nccl_comm) fail(F2V_EUSAGE, "context already has an NCCL communicator");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t comm = nullptr;
  nccl_check(nccl().comm_init_rank(&comm, int(world), id, int(rank)), "ncclCommInitRank");
  c.nccl_comm = comm;
  c.nccl_rank = rank;
  c.nccl_world = world;
}

void k_nccl_destroy(Ctx& c) {
  if (c.nccl_comm && nccl().comm_destroy)
    nccl().comm_destroy(static_cast<ncclComm_t>(c.nccl_comm));
  c.nccl_comm = nullptr;
}

// One epoch of the G-shard schedule with a per-step all-gather (after
// k_epoch_perm and k_epoch_negatives).  Returns the first failure (or
// step = ~0) and the epoch loss.
AgResult k_allgather_epoch(Ctx& c, uint32_t s, float eta, const ForceParams& fp, bool monitor,
                           bool fast) {
  const uint32_t G = c.shards, r = c.nccl_rank;
  uint32_t bmax = 0;
  for (uint32_t g = 0; g < G; ++g) bmax = std::max(bmax, c.sh_bs[g]);
  const PackLayout lay(bmax, c.d);
  const size_t pack_bytes = lay.bytes;
  c.ag_send.ensure(pack_bytes);
  c.ag_recv.ensure(pack_bytes * G);
  c.ag_state.ensure(64);
  uint32_t* stop = c.ag_state.as<uint32_t>();
  double* loss = reinterpret_cast<double*>(c.ag_state.as<uint8_t>() + 32);
  F2V_CUDA(cudaMemsetAsync(c.ag_state.p, 0, 64, c.stream));
  F2V_CUDA(cudaMemsetAsync(c.ag_send.p, 0xff, sizeof(PackHdr), c.stream));  // fail = ~0
  AgArgs a{};
  a.rowptr = c.rowptr.as<uint64_t>();
  a.col = c.col.as<uint32_t>();
  a.z = c.zcur();
  a.perm = c.perm.as<uint32_t>();
  a.negs = c.negs_all.as<uint32_t>();
  a.send = c.ag_send.as<uint8_t>();
  a.recv = c.ag_recv.as<uint8_t>();
  a.stop = stop;
  a.loss = loss;
  a.world = G;
  a.bmax = bmax;
  a.d = c.d;
  a.s = s;
  a.pack_bytes = pack_bytes;
  a.ids_off = lay.ids;
  a.rows_off = lay.rows;
  a.loss_off = lay.loss;
  a.eta = eta;
  a.fp = fp;
  ncclComm_t comm = static_cast<ncclComm_t>(c.nccl_comm);
  const uint32_t scatter_blocks =
      uint32_t(std::min<uint64_t>(4ull * c.num_sms, (uint64_t(bmax) * c.d * G + 255) / 256));
  for (uint32_t t = 0; t < c.steps; ++t) {
    a.step = t;
    a.q = t * G + r;
    a.p0 = c.h_poff[size_t(t) * G + r];
    a.cnt = c.h_poff[size_t(t) * G + r + 1] - a.p0;
    launch_step_any(a, monitor, fast, c.stream);
    F2V_LAUNCHED(c.stream, "ag_step_kernel");
    nccl_check(nccl().all_gather(a.send, c.ag_recv.p, pack_bytes, ncclUint8, comm, c.stream),
               "ncclAllGather");
    if (monitor) ag_vote_kernel<true><<<1, 32, 0, c.stream>>>(a);
    else ag_vote_kernel<false><<<1, 32, 0, c.stream>>>(a);
    F2V_LAUNCHED(c.stream, "ag_vote_kernel");
    ag_scatter_kernel<<<scatter_blocks, 256, 0, c.stream>>>(a);
    F2V_LAUNCHED(c.stream, "ag_scatter_kernel");
    c.launches += 3;
  }
  uint32_t host[16];
  F2V_CUDA(cudaMemcpyAsync(host, c.ag_state.p, 64, cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  AgResult res;
  res.failed = host[0] != 0;
  res.step = host[1];
  res.rank = host[2];
  res.index = host[3];
  res.vertex = host[4];
  std::memcpy(&res.loss, host + 8, sizeof(double));
  return res;
}

}  // namespace f2v
