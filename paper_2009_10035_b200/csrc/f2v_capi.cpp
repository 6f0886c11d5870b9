// f2v_capi.cpp -- the extern "C" boundary (include/force2vec_b200.h) and the
// host-side training driver above the device kernels.  Mirrors the reference
// API: train() (trainer.cpp:192-251), grad_minibatch / apply_update /
// batch_loss (trainer.hpp:93-104), error taxonomy (errors.hpp:8-40).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "f2v_internal.h"
#include "f2v_rng.h"

namespace f2v {

void csr_from_edges(const uint32_t* pairs, uint64_t m, uint32_t n, bool symmetrize,
                    uint64_t* rowptr, uint32_t* col_out, uint64_t* nnz_out, uint64_t* dups_out,
                    uint64_t* loops_out);
void partition_epoch(uint32_t n, uint32_t b, uint64_t state, uint32_t* perm);
std::vector<uint32_t> gen_sbm(uint32_t n, int blocks, double p_in, double p_out, uint64_t seed);
std::vector<uint32_t> gen_rmat(uint32_t scale, uint32_t ef, double a, double b, double c,
                               uint64_t seed);
std::vector<uint32_t> gen_chung_lu(uint32_t n, double expo, double min_deg, double max_deg,
                                   double mean_deg, uint64_t seed);
std::vector<uint32_t> gen_rgg(uint32_t n, double mean_deg, uint64_t seed);

void fail(int32_t code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(F2V_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
}

void launch_check(cudaStream_t s, const char* what) {
  cuda_check(cudaGetLastError(), what);
  static const bool sync = std::getenv("F2V_SYNC_DEBUG") != nullptr;
  if (sync) cuda_check(cudaStreamSynchronize(s), what);
}

void DeviceBuf::ensure(size_t want) {
  if (want <= bytes && p) return;
  release();
  F2V_CUDA(cudaMalloc(&p, std::max<size_t>(want, 16)));
  bytes = std::max<size_t>(want, 16);
}

void DeviceBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

static thread_local std::string g_global_err;

int32_t guard(Ctx* c, const std::function<void()>& fn) {
  try {
    fn();
    if (c) c->err.clear();
    return F2V_OK;
  } catch (const Error& e) {
    if (c) c->err = e.msg;
    g_global_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host out of memory";
    g_global_err = "host out of memory";
    return F2V_ECUDA;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    g_global_err = e.what();
    return F2V_ECUDA;
  }
}

static void need_graph(const Ctx& c) {
  if (!c.rowptr.p) fail(F2V_EUSAGE, "no graph uploaded");
}
static void need_embedding(const Ctx& c) {
  if (!c.z[c.cur].p || c.d == 0) fail(F2V_EUSAGE, "no embedding set");
}

static void validate_model(const f2v_force_model& m) {
  if (m.kind < F2V_SIGMOID || m.kind > F2V_LINLOG) fail(F2V_EUSAGE, "unknown force model");
}

// Stage ids/negatives of one minibatch on the device (RangeError like
// CsrGraph::neighbors, csr_graph.hpp:40-43).
static bool stage_batch(Ctx& c, const uint32_t* ids, uint32_t b, const uint32_t* negs,
                        uint32_t s) {
  for (uint32_t i = 0; i < b; ++i)
    if (ids[i] >= c.n) fail(F2V_ERANGE, "vertex id out of range");
  for (uint32_t k = 0; k < s; ++k)
    if (negs[k] >= c.n) fail(F2V_ERANGE, "vertex id out of range");
  c.ids.ensure(sizeof(uint32_t) * std::max<uint32_t>(b, 1));
  c.negs.ensure(sizeof(uint32_t) * std::max<uint32_t>(s, 1));
  c.grads.ensure(sizeof(float) * std::max<size_t>(size_t(b) * c.d, 1));
  c.vloss.ensure(sizeof(double) * std::max<uint32_t>(b, 1));
  c.bad.ensure(sizeof(unsigned long long));
  if (b)
    F2V_CUDA(cudaMemcpyAsync(c.ids.p, ids, sizeof(uint32_t) * b, cudaMemcpyHostToDevice,
                             c.stream));
  if (s)
    F2V_CUDA(cudaMemcpyAsync(c.negs.p, negs, sizeof(uint32_t) * s, cudaMemcpyHostToDevice,
                             c.stream));
  std::vector<uint32_t> sorted(ids, ids + b);
  std::sort(sorted.begin(), sorted.end());
  return std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
}

static uint64_t read_bad(Ctx& c) {
  uint64_t bad = 0;
  F2V_CUDA(cudaMemcpyAsync(&bad, c.bad.p, sizeof(bad), cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
  return bad;
}

static uint64_t degree_sum(const Ctx& c, const uint32_t* ids, uint32_t b) {
  uint64_t s = 0;
  for (uint32_t i = 0; i < b; ++i) s += c.h_rowptr[ids[i] + 1] - c.h_rowptr[ids[i]];
  return s;
}

// -------------------------------------------------------- train() driver
// trainer.cpp:192-251 on the device.  Per epoch: eta (212-214), the
// Fisher-Yates partition (216-217, computed on the host one epoch ahead while
// the GPU runs), then one dataflow launch covering every batch's
// grad_minibatch + batch_loss + apply_update (220-236).
static void train_epochs_impl(Ctx& c, const f2v_train_config& cfg, double* loss_out,
                              f2v_counters* counters, f2v_failure* failure);
static void train_allgather_impl(Ctx& c, const f2v_train_config& cfg, double* loss_out,
                                 f2v_counters* counters, f2v_failure* failure);

// Timing wrapper: CUDA events on the context stream around the whole call.
static void train_epochs(Ctx& c, const f2v_train_config& cfg, double* loss_out,
                         f2v_counters* counters, f2v_failure* failure, bool allgather = false) {
  if (!c.ev_begin) {
    F2V_CUDA(cudaEventCreate(&c.ev_begin));
    F2V_CUDA(cudaEventCreate(&c.ev_end));
  }
  for (double& t : c.timing) t = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  F2V_CUDA(cudaEventRecord(c.ev_begin, c.stream));
  if (allgather) train_allgather_impl(c, cfg, loss_out, counters, failure);
  else train_epochs_impl(c, cfg, loss_out, counters, failure);
  F2V_CUDA(cudaEventRecord(c.ev_end, c.stream));
  F2V_CUDA(cudaEventSynchronize(c.ev_end));
  float ms = 0.f;
  F2V_CUDA(cudaEventElapsedTime(&ms, c.ev_begin, c.ev_end));
  c.timing[0] = ms;
  c.timing[3] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

static void train_epochs_impl(Ctx& c, const f2v_train_config& cfg, double* loss_out,
                              f2v_counters* counters, f2v_failure* failure) {
  need_graph(c);
  if (cfg.dim < 1) fail(F2V_EUSAGE, "dim must be >= 1");  // trainer.cpp:13-22
  if (cfg.batch < 1) fail(F2V_EUSAGE, "batch must be >= 1");
  if (cfg.negatives < 1) fail(F2V_EUSAGE, "negatives must be >= 1");
  if (!(cfg.lr > 0)) fail(F2V_EUSAGE, "lr must be > 0");
  if (cfg.epochs < 1) fail(F2V_EUSAGE, "epochs must be >= 1");
  if (cfg.first_epoch >= cfg.epochs) fail(F2V_EUSAGE, "first_epoch must be < epochs");
  const uint32_t end_epoch =
      cfg.run_epochs ? std::min(cfg.epochs, cfg.first_epoch + cfg.run_epochs) : cfg.epochs;
  validate_model(cfg.model);
  if (cfg.monitor_loss && cfg.model.kind != F2V_SIGMOID && cfg.model.kind != F2V_TDIST)
    fail(F2V_EUNSUPPORTED, "loss monitoring requires the sigmoid or tdist model");  // trainer.cpp:195-197
  if (cfg.sampler != F2V_SAMPLER_SPLITMIX && cfg.sampler != F2V_SAMPLER_PHILOX)
    fail(F2V_EUSAGE, "unknown sampler");
  if (c.n >= 0x80000000u) fail(F2V_EUSAGE, "n must be < 2^31");
  if (cfg.precision != F2V_PRECISION_FAST && cfg.precision != F2V_PRECISION_EXACT)
    fail(F2V_EUSAGE, "unknown precision");
  if (cfg.walk_length > 1024) fail(F2V_EUSAGE, "walk length must be <= 1024");
  const char* penv = std::getenv("F2V_PRECISION");  // test/debug override
  c.tune.fast = penv ? (std::strcmp(penv, "exact") != 0) : cfg.precision == F2V_PRECISION_FAST;
  if (cfg.init == 1) {
    c.d = cfg.dim;
    c.cur = 0;
    c.z[0].ensure(sizeof(float) * size_t(c.n) * c.d);
    k_uniform_embedding(c, cfg.seed, 0.f, 0.f, 1);
  } else {
    need_embedding(c);
    if (c.d != cfg.dim) fail(F2V_ERANGE, "embedding dim does not match cfg.dim");
  }
  const uint32_t n = c.n;
  const uint32_t s = cfg.negatives;
  const ForceParams fp = make_params(cfg.model);
  // G vertex shards: one process per GPU when the
  // context is attached to peers, else every shard in this process
  uint32_t G = cfg.shards ? cfg.shards : 1;
  if (c.world > 1) {
    if (!cfg.shards) G = c.world;
    if (G != c.world) fail(F2V_EUSAGE, "cfg.shards must equal the number of attached GPUs");
  }
  k_shard_layout(c, cfg.batch, G, s);  // batch clamped per shard (trainer.cpp:200)
  k_set_context(c, cfg.walk_length);  // SampleMode: one-hop CSR or k-step walks
  // a batch range of one epoch: steps [t0, t1) from the current Z
  c.ranged = cfg.run_batches > 0;
  if (c.ranged) {
    if (end_epoch != cfg.first_epoch + 1) fail(F2V_EUSAGE, "a batch range needs run_epochs == 1");
    if (cfg.walk_length) fail(F2V_EUSAGE, "batch ranges are one-hop only");
    if (c.shard_ready) fail(F2V_EUSAGE, "batch ranges need a single-process context");
    if (cfg.first_batch >= c.steps) fail(F2V_EUSAGE, "first_batch beyond the epoch's steps");
    c.range_t0 = cfg.first_batch;
    c.range_t1 = uint32_t(std::min<uint64_t>(c.steps, uint64_t(cfg.first_batch) + cfg.run_batches));
    c.range_p0 = c.h_poff[size_t(c.range_t0) * G];
    c.range_p1 = c.h_poff[size_t(c.range_t1) * G];
  }
  struct RangeReset {  // the context runs whole epochs again after this call
    Ctx& c;
    ~RangeReset() { c.ranged = false; }
  } range_reset{c};
  // Several epochs run back to back with no host round trip (the outcome of
  // each stays on the device); single-epoch calls, batch ranges, attached
  // multi-GPU contexts and the replica emulation keep the per-epoch sync.
  const uint32_t nep = end_epoch - cfg.first_epoch;
  const bool async = nep > 1 && !c.ranged && !c.shard_ready &&
                     std::getenv("F2V_EMULATE_REPLICAS") == nullptr &&
                     std::getenv("F2V_SYNC_EPOCHS") == nullptr;
  std::vector<int> znew_of_epoch;
  if (async) k_async_begin(c, nep);
  uint64_t attr = 0, rep = 0;
  for (uint32_t e = cfg.first_epoch; e < end_epoch; ++e) {
    float eta = cfg.lr;
    if (cfg.lr_decay) eta = cfg.lr * (1.0f - float(e) / float(cfg.epochs));
    // partition_epoch (trainer.cpp:216-217) as a device Fisher-Yates per shard
    k_epoch_perm(c, e, cfg.seed);
    if (c.walk_k) k_epoch_walks(c, e, cfg.seed);  // build_minibatch's walks (sampling.cpp:50-58)
    k_epoch_begin(c, s, e, cfg.seed, cfg.sampler);
    const EpochResult r =
        k_epoch_run(c, s, eta, fp, cfg.monitor_loss != 0, async ? int(e - cfg.first_epoch) : -1);
    if (async) {
      znew_of_epoch.push_back(c.cur);
      continue;
    }
    if (r.bad_pos != ~0ull) {
      // the step of the failing position (combined step-major order)
      const uint64_t T = c.steps;
      uint64_t jb = 0;
      while (jb + 1 < T && c.h_poff[(jb + 1) * G] <= r.bad_pos) ++jb;
      k_epoch_restore(c, jb);
      uint32_t v = 0;
      F2V_CUDA(cudaMemcpy(&v, c.perm.as<uint32_t>() + r.bad_pos, sizeof(v),
                          cudaMemcpyDeviceToHost));
      if (failure) {
        failure->epoch = e;
        failure->batch = jb;
        failure->vertex = v;
      }
      fail(F2V_ENUMERICAL, "non-finite gradient for vertex " + std::to_string(v) + " (epoch " +
                               std::to_string(e) + ", batch " + std::to_string(jb) + ")");
    }
    if (cfg.monitor_loss && loss_out) loss_out[e - cfg.first_epoch] = r.loss;
    if (c.ranged) {
      // rows outside the range keep their given values (state "after every step")
      k_epoch_restore(c, c.range_t1);
      std::vector<uint32_t> ids(c.range_p1 - c.range_p0);
      if (!ids.empty())
        F2V_CUDA(cudaMemcpy(ids.data(), c.perm.as<uint32_t>() + c.range_p0,
                            sizeof(uint32_t) * ids.size(), cudaMemcpyDeviceToHost));
      attr += degree_sum(c, ids.data(), uint32_t(ids.size()));
      rep += uint64_t(ids.size()) * s;
      continue;
    }
    attr += c.nnz;            // one-hop: every arc once per epoch (trainer.cpp:154-160)
    rep += uint64_t(n) * s;   // b*s per batch (trainer.cpp:161-162)
  }
  if (async) {
    const AsyncOutcome o = k_async_finish(c, nep, cfg.monitor_loss ? loss_out : nullptr);
    const uint32_t done = (o.failed || o.stalled) ? o.slot : nep;
    attr += c.nnz * done;  // one-hop: every arc once per epoch (trainer.cpp:154-160)
    rep += uint64_t(n) * s * done;
    if (counters) {
      counters->attractive_evals += attr;
      counters->repulsive_evals += rep;
    }
    if (o.stalled)
      fail(F2V_ECUDA, "a Znew row never arrived within the 60 s poll deadline; the epoch was "
                      "abandoned");
    if (o.failed) {  // Z = the failed epoch's buffer, restored on the device
      c.cur = znew_of_epoch[o.slot];
      const uint32_t e = cfg.first_epoch + o.slot;
      if (failure) {
        failure->epoch = e;
        failure->batch = o.step;
        failure->vertex = o.vertex;
      }
      fail(F2V_ENUMERICAL, "non-finite gradient for vertex " + std::to_string(o.vertex) +
                               " (epoch " + std::to_string(e) + ", batch " +
                               std::to_string(o.step) + ")");
    }
    return;
  }
  if (counters) {
    counters->attractive_evals += attr;
    counters->repulsive_evals += rep;
  }
}

// The same epochs with the per-step all-gather baseline (f2v_nccl.cu): each
// process runs its shard's batch of every step and exchanges the updated rows
// with ncclAllGather; same semantics and results as the fused path.
static void train_allgather_impl(Ctx& c, const f2v_train_config& cfg, double* loss_out,
                                 f2v_counters* counters, f2v_failure* failure) {
  need_graph(c);
  if (!c.nccl_comm) fail(F2V_EUSAGE, "f2v_nccl_init first");
  if (c.shard_ready) fail(F2V_EUSAGE, "an IPC-attached context runs the fused path");
  if (cfg.dim < 1) fail(F2V_EUSAGE, "dim must be >= 1");
  if (cfg.batch < 1) fail(F2V_EUSAGE, "batch must be >= 1");
  if (cfg.negatives < 1) fail(F2V_EUSAGE, "negatives must be >= 1");
  if (!(cfg.lr > 0)) fail(F2V_EUSAGE, "lr must be > 0");
  if (cfg.epochs < 1) fail(F2V_EUSAGE, "epochs must be >= 1");
  if (cfg.first_epoch >= cfg.epochs) fail(F2V_EUSAGE, "first_epoch must be < epochs");
  if (cfg.walk_length || cfg.run_batches)
    fail(F2V_EUNSUPPORTED, "the all-gather baseline runs one-hop whole epochs");
  validate_model(cfg.model);
  if (cfg.monitor_loss && cfg.model.kind != F2V_SIGMOID && cfg.model.kind != F2V_TDIST)
    fail(F2V_EUNSUPPORTED, "loss monitoring requires the sigmoid or tdist model");
  if (cfg.sampler != F2V_SAMPLER_SPLITMIX && cfg.sampler != F2V_SAMPLER_PHILOX)
    fail(F2V_EUSAGE, "unknown sampler");
  if (cfg.precision != F2V_PRECISION_FAST && cfg.precision != F2V_PRECISION_EXACT)
    fail(F2V_EUSAGE, "unknown precision");
  const uint32_t G = c.nccl_world;
  if (cfg.shards && cfg.shards != G) fail(F2V_EUSAGE, "cfg.shards must equal the NCCL world");
  if (cfg.init == 1) {
    c.d = cfg.dim;
    c.cur = 0;
    c.z[0].ensure(sizeof(float) * size_t(c.n) * c.d);
    k_uniform_embedding(c, cfg.seed, 0.f, 0.f, 1);
  } else {
    need_embedding(c);
    if (c.d != cfg.dim) fail(F2V_ERANGE, "embedding dim does not match cfg.dim");
  }
  const uint32_t end_epoch =
      cfg.run_epochs ? std::min(cfg.epochs, cfg.first_epoch + cfg.run_epochs) : cfg.epochs;
  const uint32_t s = cfg.negatives;
  const ForceParams fp = make_params(cfg.model);
  k_shard_layout(c, cfg.batch, G, s);
  k_set_context(c, 0);
  uint64_t attr = 0, rep = 0;
  for (uint32_t e = cfg.first_epoch; e < end_epoch; ++e) {
    float eta = cfg.lr;
    if (cfg.lr_decay) eta = cfg.lr * (1.0f - float(e) / float(cfg.epochs));
    k_epoch_perm(c, e, cfg.seed);  // every shard's partition_epoch, combined order
    k_epoch_negatives(c, s, e, cfg.seed, cfg.sampler);
    const AgResult r = k_allgather_epoch(c, s, eta, fp, cfg.monitor_loss != 0,
                                         cfg.precision == F2V_PRECISION_FAST);
    if (r.failed) {  // no rank applied the failing step (trainer.cpp:149-152)
      if (failure) {
        failure->epoch = e;
        failure->batch = r.step;
        failure->vertex = r.vertex;
      }
      fail(F2V_ENUMERICAL, "non-finite gradient for vertex " + std::to_string(r.vertex) +
                               " (epoch " + std::to_string(e) + ", batch " +
                               std::to_string(r.step) + ")");
    }
    if (cfg.monitor_loss && loss_out) loss_out[e - cfg.first_epoch] = r.loss;
    attr += c.nnz;
    rep += uint64_t(c.n) * s;
  }
  if (counters) {
    counters->attractive_evals += attr;
    counters->repulsive_evals += rep;
  }
}

}  // namespace f2v

using namespace f2v;

extern "C" {

f2v_ctx* f2v_create(int32_t device) {
  f2v_ctx* h = nullptr;
  const int32_t rc = guard(nullptr, [&] {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      fail(F2V_ECUDA, "no CUDA device available (there is no CPU fallback)");
    if (device < 0 || device >= count) fail(F2V_EUSAGE, "device ordinal out of range");
    F2V_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    F2V_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      fail(F2V_ECUDA, std::string("device ") + prop.name + " is not sm_100 (Blackwell)");
    h = new f2v_ctx();
    h->c.device = device;
    h->c.num_sms = prop.multiProcessorCount;
    F2V_CUDA(cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking));
    load_tuning(h->c.tune);
  });
  if (rc != F2V_OK) {
    delete h;
    return nullptr;
  }
  return h;
}

void f2v_destroy(f2v_ctx* h) {
  if (!h) return;
  cudaSetDevice(h->c.device);
  Ctx& c = h->c;
  for (DeviceBuf* b :
       {&c.rowptr, &c.col, &c.cbase, &c.lbase, &c.lpo, &c.ecnt, &c.lcnt, &c.vflag,
        &c.z[0], &c.z[1], &c.grads, &c.ids, &c.negs, &c.vloss, &c.bad, &c.scratch, &c.perm,
        &c.state, &c.negs_all, &c.negwin, &c.items, &c.litems, &c.nE, &c.nL, &c.EP, &c.LP,
        &c.wtot, &c.needs, &c.scan_tmp, &c.epart, &c.eloss, &c.wcnt, &c.wl, &c.lpart, &c.lloss,
        &c.ploss, &c.counters, &c.trace, &c.shufR, &c.shufL, &c.poff, &c.lperm, &c.grow, &c.gcol, &c.wflag, &c.wpos,
        &c.pcnt, &c.pslot})
    b->release();
  for (uint32_t g = 0; g < 8; ++g)  // peers' replicas mapped by f2v_shard_attach
    for (int i = 0; i < 3; ++i)
      if (c.peer_base[g][i]) cudaIpcCloseMemHandle(c.peer_base[g][i]);
  c.ctl.release();
  for (DeviceBuf& r : c.rep) r.release();
  for (DeviceBuf* b : {&c.ag_send, &c.ag_recv, &c.ag_state}) b->release();
  try {
    k_nccl_destroy(c);
  } catch (...) {
  }
  for (cudaEvent_t e : c.ev_kernel) cudaEventDestroy(e);
  for (cudaEvent_t e : c.ev_async) cudaEventDestroy(e);
  c.runst.release();
  if (c.ev_begin) cudaEventDestroy(c.ev_begin);
  if (c.ev_end) cudaEventDestroy(c.ev_end);
  if (c.stream) cudaStreamDestroy(c.stream);
  delete h;
}

const char* f2v_last_error(const f2v_ctx* h) { return h ? h->c.err.c_str() : ""; }

// DEBUG helper (not in the public header): per-position finalise timestamps
// of the last epoch (F2V_TRACE) and the L-item count.
int32_t f2v_debug_trace(f2v_ctx* h, uint64_t* out, uint32_t* litems) {
  if (!h || !h->c.trace.p) return F2V_EUSAGE;
  if (litems) *litems = h->c.last_litems;
  return cudaMemcpy(out, h->c.trace.p, h->c.trace.bytes, cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? F2V_OK
             : F2V_ECUDA;
}

int32_t f2v_last_timing(const f2v_ctx* h, double* out4) {
  if (!h) return F2V_EUSAGE;
  for (int i = 0; i < 4; ++i) out4[i] = h->c.timing[i];
  return F2V_OK;
}
const char* f2v_global_error(void) { return g_global_err.c_str(); }

uint64_t f2v_kernel_launches(const f2v_ctx* h, int32_t reset) {
  if (!h) return 0;
  const uint64_t v = h->c.launches;
  if (reset) const_cast<f2v_ctx*>(h)->c.launches = 0;
  return v;
}

int32_t f2v_upload_graph(f2v_ctx* h, uint32_t n, const uint64_t* row_offsets,
                         const uint32_t* col_indices, uint64_t nnz) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    F2V_CUDA(cudaSetDevice(c.device));
    if (row_offsets[0] != 0 || row_offsets[n] != nnz)
      fail(F2V_ERANGE, "row_offsets inconsistent with nnz");
    if (c.walk_k) {  // drop a walk context of the previous graph
      c.grow.release();
      c.gcol.release();
      c.h_growptr.clear();
      c.walk_k = 0;
    }
    c.n = n;
    c.nnz = nnz;
    ++c.graph_gen;  // shard layouts depend on the degrees
    c.h_rowptr.assign(row_offsets, row_offsets + n + 1);
    c.rowptr.ensure(sizeof(uint64_t) * (n + 1));
    c.col.ensure(sizeof(uint32_t) * std::max<uint64_t>(nnz, 1));
    F2V_CUDA(cudaMemcpyAsync(c.rowptr.p, row_offsets, sizeof(uint64_t) * (n + 1),
                             cudaMemcpyHostToDevice, c.stream));
    if (nnz)
      F2V_CUDA(cudaMemcpyAsync(c.col.p, col_indices, sizeof(uint32_t) * nnz,
                               cudaMemcpyHostToDevice, c.stream));
    k_prepare_graph(c);
  });
}

int32_t f2v_build_graph(f2v_ctx* h, const uint32_t* pairs, uint64_t m, uint32_t n,
                        int32_t symmetrize, uint64_t* nnz_out, uint64_t* dups_out,
                        uint64_t* loops_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    F2V_CUDA(cudaSetDevice(c.device));
    if (c.walk_k) {  // drop a walk context of the previous graph
      c.grow.release();
      c.gcol.release();
      c.h_growptr.clear();
      c.walk_k = 0;
    }
    uint64_t nnz = 0;
    device_csr_from_edges(c.stream, c.num_sms, pairs, m, n, symmetrize != 0, c.rowptr, c.col,
                          &nnz, dups_out, loops_out);
    c.n = n;
    c.nnz = nnz;
    ++c.graph_gen;
    c.h_rowptr.resize(size_t(n) + 1);
    F2V_CUDA(cudaMemcpyAsync(c.h_rowptr.data(), c.rowptr.p, sizeof(uint64_t) * (size_t(n) + 1),
                             cudaMemcpyDeviceToHost, c.stream));
    F2V_CUDA(cudaStreamSynchronize(c.stream));
    if (nnz_out) *nnz_out = nnz;
    k_prepare_graph(c);
  });
}

int32_t f2v_get_graph(f2v_ctx* h, uint64_t* row_offsets_out, uint32_t* col_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_graph(c);
    if (c.walk_k) fail(F2V_EUSAGE, "a walk context is active");
    F2V_CUDA(cudaSetDevice(c.device));
    F2V_CUDA(cudaMemcpyAsync(row_offsets_out, c.rowptr.p, sizeof(uint64_t) * (size_t(c.n) + 1),
                             cudaMemcpyDeviceToHost, c.stream));
    if (c.nnz)
      F2V_CUDA(cudaMemcpyAsync(col_out, c.col.p, sizeof(uint32_t) * c.nnz, cudaMemcpyDeviceToHost,
                               c.stream));
    F2V_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int32_t f2v_set_embedding(f2v_ctx* h, const float* z, uint32_t n, uint32_t d) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    F2V_CUDA(cudaSetDevice(c.device));
    if (c.rowptr.p && n != c.n) fail(F2V_ERANGE, "embedding rows do not match the graph");
    if (d < 1) fail(F2V_EUSAGE, "dim must be >= 1");
    c.n = n;
    c.d = d;
    c.cur = 0;
    c.z[0].ensure(sizeof(float) * size_t(n) * d);
    F2V_CUDA(cudaMemcpyAsync(c.z[0].p, z, sizeof(float) * size_t(n) * d, cudaMemcpyHostToDevice,
                             c.stream));
    F2V_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int32_t f2v_get_embedding(f2v_ctx* h, float* z) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_embedding(c);
    F2V_CUDA(cudaSetDevice(c.device));
    F2V_CUDA(cudaMemcpyAsync(z, c.zcur(), sizeof(float) * size_t(c.n) * c.d,
                             cudaMemcpyDeviceToHost, c.stream));
    F2V_CUDA(cudaStreamSynchronize(c.stream));
  });
}

static int32_t device_init(f2v_ctx* h, uint32_t n, uint32_t d, uint64_t seed, float lo, float hi,
                           int keyed) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    F2V_CUDA(cudaSetDevice(c.device));
    if (n < 1 || d < 1) fail(F2V_EUSAGE, "init_embedding: n and d must be >= 1");
    if (c.rowptr.p && n != c.n) fail(F2V_ERANGE, "embedding rows do not match the graph");
    c.n = n;
    c.d = d;
    c.cur = 0;
    c.z[0].ensure(sizeof(float) * size_t(n) * d);
    k_uniform_embedding(c, seed, lo, hi, keyed);
    F2V_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int32_t f2v_init_embedding(f2v_ctx* h, uint32_t n, uint32_t d, uint64_t seed) {
  return device_init(h, n, d, seed, 0.f, 0.f, 1);
}

int32_t f2v_uniform_embedding(f2v_ctx* h, uint32_t n, uint32_t d, uint64_t seed, float lo,
                              float hi) {
  return device_init(h, n, d, seed, lo, hi, 0);
}

int32_t f2v_grad_minibatch(f2v_ctx* h, const uint32_t* ids, uint32_t b, const uint32_t* negs,
                           uint32_t s, f2v_force_model model, float* grads_out,
                           f2v_counters* counters, uint32_t* bad_vertex) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_graph(c);
    k_set_context(c, 0);  // per-step operators take one-hop minibatches
    need_embedding(c);
    validate_model(model);
    F2V_CUDA(cudaSetDevice(c.device));
    stage_batch(c, ids, b, negs, s);
    k_grad_minibatch(c, b, s, make_params(model), false);
    c.staged_b = b;
    const uint64_t bad = read_bad(c);
    if (grads_out && b) {
      F2V_CUDA(cudaMemcpyAsync(grads_out, c.grads.p, sizeof(float) * size_t(b) * c.d,
                               cudaMemcpyDeviceToHost, c.stream));
      F2V_CUDA(cudaStreamSynchronize(c.stream));
    }
    if (bad != ~0ull) {
      if (bad_vertex) *bad_vertex = ids[bad];
      fail(F2V_ENUMERICAL, "non-finite gradient for vertex " + std::to_string(ids[bad]));
    }
    if (counters) {
      counters->attractive_evals += degree_sum(c, ids, b);
      counters->repulsive_evals += uint64_t(b) * s;
    }
  });
}

int32_t f2v_apply_update(f2v_ctx* h, const uint32_t* ids, uint32_t b, const float* grads,
                         float eta) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_embedding(c);
    F2V_CUDA(cudaSetDevice(c.device));
    if (!grads && b != c.staged_b) fail(F2V_EUSAGE, "no staged gradient of this batch size");
    for (uint32_t i = 0; i < b; ++i)
      if (ids[i] >= c.n) fail(F2V_ERANGE, "vertex id out of range");
    c.ids.ensure(sizeof(uint32_t) * std::max<uint32_t>(b, 1));
    c.grads.ensure(sizeof(float) * std::max<size_t>(size_t(b) * c.d, 1));
    F2V_CUDA(cudaMemcpyAsync(c.ids.p, ids, sizeof(uint32_t) * b, cudaMemcpyHostToDevice,
                             c.stream));
    if (grads)
      F2V_CUDA(cudaMemcpyAsync(c.grads.p, grads, sizeof(float) * size_t(b) * c.d,
                               cudaMemcpyHostToDevice, c.stream));
    std::vector<uint32_t> sorted(ids, ids + b);
    std::sort(sorted.begin(), sorted.end());
    const bool uniq = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    k_apply_update(c, b, eta, uniq);
    F2V_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int32_t f2v_batch_loss(f2v_ctx* h, const uint32_t* ids, uint32_t b, const uint32_t* negs,
                       uint32_t s, f2v_force_model model, double* loss_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_graph(c);
    k_set_context(c, 0);  // per-step operators take one-hop minibatches
    need_embedding(c);
    validate_model(model);
    if (model.kind != F2V_SIGMOID && model.kind != F2V_TDIST)
      fail(F2V_EUNSUPPORTED, "pair_loss is defined for sigmoid and tdist only");
    F2V_CUDA(cudaSetDevice(c.device));
    stage_batch(c, ids, b, negs, s);
    k_grad_minibatch(c, b, s, make_params(model), true);
    c.staged_b = 0;  // the staged gradient is not a requested one
    *loss_out = b ? k_batch_loss_sum(c, b) : 0.0;
  });
}

int32_t f2v_step(f2v_ctx* h, const uint32_t* ids, uint32_t b, const uint32_t* negs, uint32_t s,
                 f2v_force_model model, float eta, double* loss_out, f2v_counters* counters,
                 uint32_t* bad_vertex) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_graph(c);
    k_set_context(c, 0);  // per-step operators take one-hop minibatches
    need_embedding(c);
    validate_model(model);
    const bool mon = loss_out != nullptr;
    if (mon && model.kind != F2V_SIGMOID && model.kind != F2V_TDIST)
      fail(F2V_EUNSUPPORTED, "pair_loss is defined for sigmoid and tdist only");
    F2V_CUDA(cudaSetDevice(c.device));
    const bool uniq = stage_batch(c, ids, b, negs, s);
    k_grad_minibatch(c, b, s, make_params(model), mon);
    const uint64_t bad = read_bad(c);
    if (bad != ~0ull) {  // thrown before apply_update: Z untouched (trainer.cpp:149-152)
      if (bad_vertex) *bad_vertex = ids[bad];
      fail(F2V_ENUMERICAL, "non-finite gradient for vertex " + std::to_string(ids[bad]));
    }
    if (mon) *loss_out = b ? k_batch_loss_sum(c, b) : 0.0;
    k_apply_update(c, b, eta, uniq);
    c.staged_b = b;
    F2V_CUDA(cudaStreamSynchronize(c.stream));
    if (counters) {
      counters->attractive_evals += degree_sum(c, ids, b);
      counters->repulsive_evals += uint64_t(b) * s;
    }
  });
}

int32_t f2v_train_epochs(f2v_ctx* h, const f2v_train_config* cfg, double* loss_out,
                         f2v_counters* counters, f2v_failure* failure) {
  return guard(&h->c, [&] {
    F2V_CUDA(cudaSetDevice(h->c.device));
    train_epochs(h->c, *cfg, loss_out, counters, failure);
  });
}

int32_t f2v_train(int32_t device, uint32_t n, const uint64_t* row_offsets,
                  const uint32_t* col_indices, uint64_t nnz, float* z_inout,
                  const f2v_train_config* cfg, double* loss_out, f2v_counters* counters,
                  f2v_failure* failure) {
  f2v_ctx* h = f2v_create(device);
  if (!h) return F2V_ECUDA;
  int32_t rc = f2v_upload_graph(h, n, row_offsets, col_indices, nnz);
  if (rc == F2V_OK && cfg->init != 1) rc = f2v_set_embedding(h, z_inout, n, cfg->dim);
  if (rc == F2V_OK) {
    rc = f2v_train_epochs(h, cfg, loss_out, counters, failure);
    // Z after the last complete batch, also on F2V_ENUMERICAL
    if (rc == F2V_OK || rc == F2V_ENUMERICAL) {
      const int32_t rc2 = f2v_get_embedding(h, z_inout);
      if (rc == F2V_OK) rc = rc2;
    }
  }
  if (rc != F2V_OK) g_global_err = h->c.err;
  f2v_destroy(h);
  return rc;
}

int32_t f2v_nccl_unique_id(uint8_t* out) {
  return guard(nullptr, [&] { nccl_unique_id(out); });
}

int32_t f2v_nccl_init(f2v_ctx* h, const uint8_t* unique_id, uint32_t rank, uint32_t world) {
  return guard(&h->c, [&] {
    F2V_CUDA(cudaSetDevice(h->c.device));
    k_nccl_init(h->c, unique_id, rank, world);
  });
}

int32_t f2v_train_epochs_allgather(f2v_ctx* h, const f2v_train_config* cfg, double* loss_out,
                                   f2v_counters* counters, f2v_failure* failure) {
  return guard(&h->c, [&] {
    F2V_CUDA(cudaSetDevice(h->c.device));
    train_epochs(h->c, *cfg, loss_out, counters, failure, true);
  });
}

int32_t f2v_csr_from_edges(const uint32_t* pairs, uint64_t m, uint32_t n, int32_t symmetrize,
                           uint64_t* row_offsets_out, uint32_t* col_out, uint64_t* nnz_out,
                           uint64_t* duplicates_dropped, uint64_t* self_loops_dropped) {
  return guard(nullptr, [&] {
    csr_from_edges(pairs, m, n, symmetrize != 0, row_offsets_out, col_out, nnz_out,
                   duplicates_dropped, self_loops_dropped);
  });
}

int32_t f2v_partition_epoch(uint32_t n, uint32_t b, uint64_t seed, uint32_t epoch,
                            uint32_t* perm_out) {
  return guard(nullptr, [&] {
    partition_epoch(n, b, rng_keyed2(seed, kStreamPartition, epoch), perm_out);
  });
}

int32_t f2v_device_partition_epoch(f2v_ctx* h, uint32_t n, uint32_t b, uint64_t seed,
                                   uint32_t epoch, uint32_t* perm_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    F2V_CUDA(cudaSetDevice(c.device));
    if (b == 0 || b > n) fail(F2V_EUSAGE, "batch size must be in [1, n]");
    DeviceBuf out;
    out.ensure(sizeof(uint32_t) * n);
    k_device_partition(c, n, seed, epoch, out.as<uint32_t>());
    F2V_CUDA(cudaMemcpyAsync(perm_out, out.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost,
                             c.stream));
    F2V_CUDA(cudaStreamSynchronize(c.stream));
    out.release();
  });
}

int32_t f2v_negatives(int32_t sampler, uint64_t seed, uint32_t epoch, uint64_t batch,
                      uint32_t shard, uint32_t num_shards, uint32_t n, uint32_t s,
                      uint32_t* out) {
  return guard(nullptr, [&] {
    if (n < 1) fail(F2V_EUSAGE, "n must be >= 1");
    for (uint32_t k = 0; k < s; ++k)
      out[k] = sampler == F2V_SAMPLER_PHILOX
                   ? philox_negative(seed, epoch, batch, shard, k, n)
                   : splitmix_negative(seed, epoch, batch, shard, std::max(1u, num_shards), k, n);
  });
}

static int32_t emit(std::vector<uint32_t>&& e, uint32_t** pairs_out, uint64_t* m_out) {
  uint32_t* p = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<size_t>(e.size(), 2)));
  if (!p) return F2V_ECUDA;
  std::memcpy(p, e.data(), sizeof(uint32_t) * e.size());
  *pairs_out = p;
  *m_out = e.size() / 2;
  return F2V_OK;
}

int32_t f2v_gen_sbm(uint32_t n, int32_t blocks, double p_in, double p_out, uint64_t seed,
                    uint32_t** pairs_out, uint64_t* m_out) {
  int32_t rc2 = F2V_OK;
  const int32_t rc = guard(nullptr, [&] {
    rc2 = emit(gen_sbm(n, blocks, p_in, p_out, seed), pairs_out, m_out);
  });
  return rc ? rc : rc2;
}

int32_t f2v_gen_rmat(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                     uint32_t** pairs_out, uint64_t* m_out) {
  int32_t rc2 = F2V_OK;
  const int32_t rc = guard(nullptr, [&] {
    rc2 = emit(gen_rmat(scale, ef, a, b, c, seed), pairs_out, m_out);
  });
  return rc ? rc : rc2;
}

int32_t f2v_gen_chung_lu(uint32_t n, double expo, double min_deg, double max_deg,
                         double mean_deg, uint64_t seed, uint32_t** pairs_out, uint64_t* m_out) {
  int32_t rc2 = F2V_OK;
  const int32_t rc = guard(nullptr, [&] {
    rc2 = emit(gen_chung_lu(n, expo, min_deg, max_deg, mean_deg, seed), pairs_out, m_out);
  });
  return rc ? rc : rc2;
}

int32_t f2v_gen_rgg(uint32_t n, double mean_deg, uint64_t seed, uint32_t** pairs_out,
                    uint64_t* m_out) {
  int32_t rc2 = F2V_OK;
  const int32_t rc = guard(nullptr, [&] {
    rc2 = emit(gen_rgg(n, mean_deg, seed), pairs_out, m_out);
  });
  return rc ? rc : rc2;
}

void f2v_free(void* p) { std::free(p); }

// ------------------------------------------ multi-GPU shards (f2v_shard.cu)
int32_t f2v_shard_layout(uint32_t n, const uint64_t* row_offsets, uint32_t negatives,
                         uint32_t batch, uint32_t shards, uint32_t* lo_out, uint32_t* batch_out,
                         uint32_t* poff_out, uint32_t* steps_out) {
  return guard(nullptr, [&] {
    std::vector<uint32_t> lo, bs, nb, poff;
    uint32_t T = 0;
    shard_layout(row_offsets, n, negatives, batch, shards, lo, bs, nb, poff, T);
    if (steps_out) *steps_out = T;
    if (lo_out) std::memcpy(lo_out, lo.data(), sizeof(uint32_t) * lo.size());
    if (batch_out) std::memcpy(batch_out, bs.data(), sizeof(uint32_t) * bs.size());
    if (poff_out) std::memcpy(poff_out, poff.data(), sizeof(uint32_t) * poff.size());
  });
}

int32_t f2v_partition_shard(uint32_t n, uint32_t b, uint64_t seed, uint32_t epoch,
                            uint32_t shard, uint32_t shards, uint32_t* perm_out) {
  return guard(nullptr, [&] {
    if (shards < 1 || shard >= shards) fail(F2V_EUSAGE, "shard out of range");
    const uint64_t st = shards == 1 ? rng_keyed2(seed, kStreamPartition, epoch)
                                    : rng_keyed3(seed, kStreamPartition, epoch, shard);
    partition_epoch(n, b, st, perm_out);
  });
}

static void rows_io(Ctx& c, const uint32_t* ids, uint32_t b, float* host, bool to_z) {
  need_embedding(c);
  F2V_CUDA(cudaSetDevice(c.device));
  for (uint32_t i = 0; i < b; ++i)
    if (ids[i] >= c.n) fail(F2V_ERANGE, "vertex id out of range");
  c.ids.ensure(sizeof(uint32_t) * std::max<uint32_t>(b, 1));
  c.scratch.ensure(sizeof(float) * std::max<size_t>(size_t(b) * c.d, 8));
  const size_t bytes = sizeof(float) * size_t(b) * c.d;
  if (b)
    F2V_CUDA(cudaMemcpyAsync(c.ids.p, ids, sizeof(uint32_t) * b, cudaMemcpyHostToDevice,
                             c.stream));
  if (to_z && b)
    F2V_CUDA(cudaMemcpyAsync(c.scratch.p, host, bytes, cudaMemcpyHostToDevice, c.stream));
  k_rows(c, b, c.scratch.as<float>(), to_z);
  if (!to_z && b)
    F2V_CUDA(cudaMemcpyAsync(host, c.scratch.p, bytes, cudaMemcpyDeviceToHost, c.stream));
  F2V_CUDA(cudaStreamSynchronize(c.stream));
}

int32_t f2v_get_rows(f2v_ctx* h, const uint32_t* ids, uint32_t b, float* rows_out) {
  return guard(&h->c, [&] { rows_io(h->c, ids, b, rows_out, false); });
}

int32_t f2v_set_rows(f2v_ctx* h, const uint32_t* ids, uint32_t b, const float* rows) {
  return guard(&h->c, [&] { rows_io(h->c, ids, b, const_cast<float*>(rows), true); });
}

int32_t f2v_shard_handle_bytes(void) { return int32_t(3 * sizeof(cudaIpcMemHandle_t)); }

int32_t f2v_shard_init(f2v_ctx* h, uint32_t rank, uint32_t world) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    F2V_CUDA(cudaSetDevice(c.device));
    if (world < 1 || world > 8) fail(F2V_EUSAGE, "world must be in [1, 8]");
    if (rank >= world) fail(F2V_EUSAGE, "rank out of range");
    if (!c.rowptr.p) fail(F2V_EUSAGE, "upload the graph before f2v_shard_init");
    if (!c.z[c.cur].p || !c.d) fail(F2V_EUSAGE, "set the embedding before f2v_shard_init");
    if (c.n < world) fail(F2V_EUSAGE, "fewer vertices than shards");
    if (c.rank >= 0) fail(F2V_EUSAGE, "context already sharded");
    // both replica buffers exist from now on and never move (peers map them)
    const size_t zb = sizeof(float) * size_t(c.n) * c.d;
    c.z[0].ensure(zb);
    c.z[1].ensure(zb);
    c.ctl.ensure(shard_ctl_bytes());
    F2V_CUDA(cudaMemsetAsync(c.ctl.p, 0, shard_ctl_bytes(), c.stream));
    F2V_CUDA(cudaStreamSynchronize(c.stream));
    c.rank = int32_t(rank);
    c.world = world;
    c.barriers = 0;
    c.layout_key[2] = 0;  // re-plan the layout with the ownership
  });
}

int32_t f2v_shard_export(f2v_ctx* h, uint8_t* out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    if (c.rank < 0) fail(F2V_EUSAGE, "f2v_shard_init first");
    F2V_CUDA(cudaSetDevice(c.device));
    void* bufs[3] = {c.z[0].p, c.z[1].p, c.ctl.p};
    for (int i = 0; i < 3; ++i) {
      cudaIpcMemHandle_t hd;
      F2V_CUDA(cudaIpcGetMemHandle(&hd, bufs[i]));
      std::memcpy(out + i * sizeof(hd), &hd, sizeof(hd));
    }
  });
}

int32_t f2v_shard_attach(f2v_ctx* h, const uint8_t* all) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    if (c.rank < 0) fail(F2V_EUSAGE, "f2v_shard_init first");
    if (c.shard_ready) fail(F2V_EUSAGE, "context already attached");
    F2V_CUDA(cudaSetDevice(c.device));
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    for (uint32_t g = 0; g < c.world; ++g) {
      if (int32_t(g) == c.rank) {
        c.peer_z[g][0] = c.z[0].as<float>();
        c.peer_z[g][1] = c.z[1].as<float>();
        c.peer_ctl[g] = c.ctl.p;
        continue;
      }
      for (int i = 0; i < 3; ++i) {
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, all + (size_t(g) * 3 + i) * hb, hb);
        void* p = nullptr;
        F2V_CUDA(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
        c.peer_base[g][i] = p;
      }
      c.peer_z[g][0] = static_cast<float*>(c.peer_base[g][0]);
      c.peer_z[g][1] = static_cast<float*>(c.peer_base[g][1]);
      c.peer_ctl[g] = c.peer_base[g][2];
    }
    c.shard_ready = true;
  });
}

}  // extern "C"
