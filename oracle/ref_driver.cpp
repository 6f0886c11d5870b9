// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" driver over the UNMODIFIED reference library
// (/root/reference/proj/core/src/*.cpp, compiled in place by oracle/Makefile
// into oracle/_ref/libf2vref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline / --impl reference) may load it.
//
// It exposes the reference's own public API (rng.hpp, sampling.hpp,
// trainer.hpp, force_kernels.hpp, csr_graph.hpp) through plain pointers so
// the golden-fixture generator and the CPU-baseline timer can drive it:
//   * Rng / Rng::keyed / next / below / uniform      rng.hpp:12-53
//   * partition_epoch / build_minibatch               sampling.cpp:7-61
//   * CsrGraph::from_edges                            csr_graph.cpp:57-97
//   * pair_grad (double overload) / pair_loss         force_kernels.cpp:199-231
//   * grad_minibatch / apply_update / batch_loss      trainer.cpp:108-190
//   * the train() loop of trainer.cpp:192-251 with an injected initial Z and
//     (optionally) injected negatives, as SURVEY.md §8(c) prescribes.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "force2vec/csr_graph.hpp"
#include "force2vec/force_kernels.hpp"
#include "force2vec/rng.hpp"
#include "force2vec/sampling.hpp"
#include "force2vec/trainer.hpp"
#include "support/test_graphs.hpp"

using namespace force2vec;

namespace {
thread_local std::string g_err;

ForceModel make_model(int kind, float eps, float cap) {
  ForceModel m;
  m.kind = static_cast<ForceKind>(kind);
  m.epsilon = eps;
  // NaN = std::nullopt; any other value is a cap (0 zeroes the repulsion)
  if (!std::isnan(cap)) m.repulsion_cap = cap; else m.repulsion_cap.reset();
  return m;
}

int classify(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const UsageError*>(&e)) return 1;
  if (dynamic_cast<const IoError*>(&e)) return 2;
  if (dynamic_cast<const FormatError*>(&e)) return 3;
  if (dynamic_cast<const RangeError*>(&e)) return 3;
  if (dynamic_cast<const NumericalError*>(&e)) return 4;
  if (dynamic_cast<const UnsupportedError*>(&e)) return 6;
  return 7;
}

// Builds an EmbeddingMatrix view copy from a flat host array.
EmbeddingMatrix to_matrix(const float* z, std::uint32_t n, std::uint32_t d) {
  EmbeddingMatrix m(n, d);
  std::memcpy(m.data().data(), z, sizeof(float) * std::size_t(n) * d);
  return m;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- rng.hpp --------------------------------------------------------------
void ref_rng_keyed_draws(std::uint64_t seed, const std::uint64_t* key, int nkey,
                         std::uint64_t count, std::uint64_t* out) {
  Rng r = Rng::keyed(seed, {});
  // Rng::keyed takes an initializer_list; replicate for runtime-length keys by
  // folding one element at a time through the same public entry point is not
  // possible, so dispatch on the small lengths the tests use.
  switch (nkey) {
    case 0: r = Rng::keyed(seed, {}); break;
    case 1: r = Rng::keyed(seed, {key[0]}); break;
    case 2: r = Rng::keyed(seed, {key[0], key[1]}); break;
    case 3: r = Rng::keyed(seed, {key[0], key[1], key[2]}); break;
    case 4: r = Rng::keyed(seed, {key[0], key[1], key[2], key[3]}); break;
    default: r = Rng::keyed(seed, {key[0], key[1], key[2], key[3], key[4]}); break;
  }
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r.next();
}

void ref_rng_draws(std::uint64_t seed, std::uint64_t stream, std::uint64_t count,
                   std::uint64_t* out) {
  Rng r(seed, stream);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r.next();
}

void ref_rng_below(std::uint64_t seed, std::uint64_t stream, std::uint64_t n,
                   std::uint64_t count, std::uint64_t* out) {
  Rng r(seed, stream);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r.below(n);
}

// random_embedding of test_trainer.cpp:18-23: U(-1,1) from Rng(seed, 0).
void ref_random_embedding(std::uint32_t n, std::uint32_t d, std::uint64_t seed,
                          float* out) {
  Rng rng(seed, 0);
  for (std::size_t i = 0; i < std::size_t(n) * d; ++i)
    out[i] = static_cast<float>(rng.uniform(-1.0, 1.0));
}

// init_embedding (trainer.cpp:62-72) keyed as train() does (trainer.cpp:203-206).
int ref_init_embedding(std::uint32_t n, std::uint32_t d, std::uint64_t seed,
                       float* out) {
  try {
    Rng rng = Rng::keyed(seed, {0x11});
    EmbeddingMatrix z = init_embedding(n, d, rng);
    std::memcpy(out, z.data().data(), sizeof(float) * std::size_t(n) * d);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// ---- sampling.cpp ---------------------------------------------------------
// perm for train()'s epoch `epoch` (trainer.cpp:216-217).
int ref_partition_epoch(std::uint32_t n, std::uint32_t b, std::uint64_t seed,
                        std::uint32_t epoch, std::uint32_t* perm_out) {
  try {
    Rng rng = Rng::keyed(seed, {0x22, epoch});
    EpochPartition part = partition_epoch(n, b, rng);
    std::memcpy(perm_out, part.perm.data(), sizeof(std::uint32_t) * n);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// Generic-stream variant used by the sampling tests (Rng(seed, stream)).
int ref_partition_stream(std::uint32_t n, std::uint32_t b, std::uint64_t seed,
                         std::uint64_t stream, std::uint32_t* perm_out) {
  try {
    Rng rng(seed, stream);
    EpochPartition part = partition_epoch(n, b, rng);
    std::memcpy(perm_out, part.perm.data(), sizeof(std::uint32_t) * n);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// ---- csr_graph.cpp --------------------------------------------------------
void* ref_graph_from_edges(const std::uint32_t* pairs, std::uint64_t m,
                           std::uint32_t n, int symmetrize,
                           std::uint64_t* dups, std::uint64_t* loops) {
  try {
    std::vector<std::pair<VertexId, VertexId>> e(m);
    for (std::uint64_t i = 0; i < m; ++i) e[i] = {pairs[2 * i], pairs[2 * i + 1]};
    return new CsrGraph(CsrGraph::from_edges(std::move(e), n, symmetrize != 0, dups, loops));
  } catch (const std::exception& e) { classify(e); return nullptr; }
}

// A CSR already canonical (sorted, unique, loop-free) is reproduced exactly by
// from_edges(symmetrize=false) of its own arc list.
void* ref_graph_from_csr(std::uint32_t n, const std::uint64_t* rowptr,
                         const std::uint32_t* col) {
  try {
    std::vector<std::pair<VertexId, VertexId>> e(rowptr[n]);
    for (std::uint32_t u = 0; u < n; ++u)
      for (std::uint64_t k = rowptr[u]; k < rowptr[u + 1]; ++k) e[k] = {u, col[k]};
    return new CsrGraph(CsrGraph::from_edges(std::move(e), n, false));
  } catch (const std::exception& e) { classify(e); return nullptr; }
}

void* ref_sbm_graph(std::uint32_t n, int blocks, double p_in, double p_out,
                    std::uint64_t seed) {
  Rng rng(seed, 0);
  return new CsrGraph(f2v_test::sbm_graph(n, blocks, p_in, p_out, rng));
}

void* ref_random_graph(std::uint32_t n, double p, std::uint64_t seed) {
  Rng rng(seed, 0);
  return new CsrGraph(f2v_test::random_graph(n, p, rng));
}

void ref_graph_free(void* g) { delete static_cast<CsrGraph*>(g); }
std::uint32_t ref_graph_n(void* g) { return static_cast<CsrGraph*>(g)->num_vertices(); }
std::uint64_t ref_graph_nnz(void* g) { return static_cast<CsrGraph*>(g)->num_edges(); }
void ref_graph_export(void* gp, std::uint64_t* rowptr, std::uint32_t* col) {
  const CsrGraph& g = *static_cast<CsrGraph*>(gp);
  std::memcpy(rowptr, g.row_offsets().data(), sizeof(std::uint64_t) * (g.num_vertices() + 1));
  if (g.num_edges())
    std::memcpy(col, g.col_indices().data(), sizeof(std::uint32_t) * g.num_edges());
}

// ---- force_kernels.cpp ----------------------------------------------------
int ref_pair_grad(int kind, float eps, float cap, const float* zu, const float* zo,
                  std::uint32_t d, int attractive, double* out) {
  try {
    pair_grad(make_model(kind, eps, cap), std::span<const float>(zu, d),
              std::span<const float>(zo, d), attractive != 0, std::span<double>(out, d));
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_pair_grad_f32(int kind, float eps, float cap, const float* zu, const float* zo,
                      std::uint32_t d, int attractive, float* out) {
  try {
    pair_grad(make_model(kind, eps, cap), std::span<const float>(zu, d),
              std::span<const float>(zo, d), attractive != 0, std::span<float>(out, d));
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_pair_loss(int kind, float eps, float cap, const float* zu, const float* zo,
                  std::uint32_t d, int attractive, double* out) {
  try {
    *out = pair_loss(make_model(kind, eps, cap), std::span<const float>(zu, d),
                     std::span<const float>(zo, d), attractive != 0);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

double ref_stable_sigmoid(double x) { return stable_sigmoid(x); }

// ---- trainer.cpp ----------------------------------------------------------
// grad_minibatch over an explicit (ids, negatives) one-hop minibatch.
int ref_grad_minibatch(void* gp, const float* z, std::uint32_t n, std::uint32_t d,
                       const std::uint32_t* ids, std::uint32_t b,
                       const std::uint32_t* negs, std::uint32_t s, int kind,
                       float eps, float cap, std::uint32_t workers, float* grads_out,
                       std::uint64_t* counters /*[2] accumulated*/) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    const EmbeddingMatrix zm = to_matrix(z, n, d);
    Minibatch mb;
    mb.vertices.assign(ids, ids + b);
    mb.negatives.assign(negs, negs + s);
    mb.mode = SampleMode::one_hop();
    mb.graph = &g;
    BatchSchedule sched = make_schedule(g, mb.vertices, workers, true);
    GradBuffer grads;
    TrainCounters tc;
    grad_minibatch(g, zm, mb, make_model(kind, eps, cap), sched, grads, &tc);
    std::memcpy(grads_out, grads.data.data(), sizeof(float) * std::size_t(b) * d);
    if (counters) { counters[0] += tc.attractive_evals; counters[1] += tc.repulsive_evals; }
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_apply_update(float* z, std::uint32_t n, std::uint32_t d,
                     const std::uint32_t* ids, std::uint32_t b, const float* grads,
                     float eta) {
  EmbeddingMatrix zm = to_matrix(z, n, d);
  GradBuffer gb(b, d);
  std::memcpy(gb.data.data(), grads, sizeof(float) * std::size_t(b) * d);
  apply_update(zm, std::span<const VertexId>(ids, b), gb, eta);
  std::memcpy(z, zm.data().data(), sizeof(float) * std::size_t(n) * d);
  return 0;
}

int ref_batch_loss(void* gp, const float* z, std::uint32_t n, std::uint32_t d,
                   const std::uint32_t* ids, std::uint32_t b,
                   const std::uint32_t* negs, std::uint32_t s, int kind, float eps,
                   float cap, double* out) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    const EmbeddingMatrix zm = to_matrix(z, n, d);
    Minibatch mb;
    mb.vertices.assign(ids, ids + b);
    mb.negatives.assign(negs, negs + s);
    mb.mode = SampleMode::one_hop();
    mb.graph = &g;
    *out = batch_loss(zm, mb, make_model(kind, eps, cap));
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// Negatives that train() draws for (epoch, batch) (trainer.cpp:222-224).
int ref_batch_negatives(void* gp, std::uint64_t seed, std::uint32_t epoch,
                        std::uint64_t bi, std::uint32_t s, std::uint32_t* out) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    Rng batch_rng = Rng::keyed(seed, {0x33, epoch, bi});
    const VertexId first = 0;
    Minibatch mb = build_minibatch(g, std::span<const VertexId>(&first, 1),
                                   SampleMode::one_hop(), s, batch_rng);
    std::memcpy(out, mb.negatives.data(), sizeof(std::uint32_t) * s);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// The train() loop of trainer.cpp:192-251 with an injected initial Z.
// negs_in == nullptr: negatives from build_minibatch on the reference stream
// (seed, {0x33, epoch, batch}); otherwise negs_in[(epoch*nb + batch)*s + k].
// perm_in == nullptr: partition_epoch on (seed, {0x22, epoch}); otherwise
// perm_in[epoch*n + p].  loss_out (nullable) gets one entry per epoch.
// step_cb (nullable) is called after each apply_update with (epoch, batch).
typedef void (*ref_step_cb)(std::uint32_t epoch, std::uint64_t batch, const float* z,
                            void* user);
int ref_train_mode(void* gp, float* z, std::uint32_t d, std::uint32_t batch,
                   std::uint32_t s, float lr, std::uint32_t epochs, int kind, float eps,
                   float cap, std::uint64_t seed, std::uint32_t workers, int lr_decay,
                   int monitor, std::uint32_t walk_k, const std::uint32_t* perm_in,
                   const std::uint32_t* negs_in, double* loss_out, std::uint64_t* counters,
                   ref_step_cb cb, void* user, std::uint32_t* fail_info);

int ref_train(void* gp, float* z, std::uint32_t d, std::uint32_t batch,
              std::uint32_t s, float lr, std::uint32_t epochs, int kind, float eps,
              float cap, std::uint64_t seed, std::uint32_t workers, int lr_decay,
              int monitor, const std::uint32_t* perm_in, const std::uint32_t* negs_in,
              double* loss_out, std::uint64_t* counters, ref_step_cb cb, void* user,
              std::uint32_t* fail_info /*[3]: epoch, batch, vertex*/) {
  return ref_train_mode(gp, z, d, batch, s, lr, epochs, kind, eps, cap, seed, workers, lr_decay,
                        monitor, 0, perm_in, negs_in, loss_out, counters, cb, user, fail_info);
}

// ref_train with the reference's SampleMode: walk_k > 0 = SampleMode::walk(k)
// (build_minibatch draws the walks, then the negatives; injected negs_in
// replace only the negatives).
int ref_train_mode(void* gp, float* z, std::uint32_t d, std::uint32_t batch,
                   std::uint32_t s, float lr, std::uint32_t epochs, int kind, float eps,
                   float cap, std::uint64_t seed, std::uint32_t workers, int lr_decay,
                   int monitor, std::uint32_t walk_k, const std::uint32_t* perm_in,
                   const std::uint32_t* negs_in, double* loss_out, std::uint64_t* counters,
                   ref_step_cb cb, void* user, std::uint32_t* fail_info) {
  const CsrGraph& g = *static_cast<CsrGraph*>(gp);
  const VertexId n = g.num_vertices();
  std::uint32_t cur_epoch = 0;
  std::size_t cur_batch = 0;
  try {
    if (epochs < 1 || batch < 1 || s < 1 || !(lr > 0) || workers < 1)
      throw UsageError("invalid config");
    const VertexId b = std::min<VertexId>(batch, n);
    EmbeddingMatrix zm = to_matrix(z, n, d);
    const ForceModel model = make_model(kind, eps, cap);
    GradBuffer grads(b, d);
    TrainCounters tc;
    const std::size_t nb = (n + b - 1) / b;
    for (std::uint32_t epoch = 0; epoch < epochs; ++epoch) {
      cur_epoch = epoch;
      float eta = lr;
      if (lr_decay) eta = lr * (1.0f - float(epoch) / float(epochs));
      EpochPartition part;
      if (perm_in) {
        part.batch_size = b;
        part.perm.assign(perm_in + std::size_t(epoch) * n, perm_in + std::size_t(epoch + 1) * n);
      } else {
        Rng part_rng = Rng::keyed(seed, {0x22, epoch});
        part = partition_epoch(n, b, part_rng);
      }
      double epoch_loss = 0.0;
      for (std::size_t bi = 0; bi < part.num_batches(); ++bi) {
        cur_batch = bi;
        const auto ids = part.batch(bi);
        Minibatch mb;
        const SampleMode mode = walk_k ? SampleMode::walk(walk_k) : SampleMode::one_hop();
        if (negs_in && !walk_k) {
          mb.vertices.assign(ids.begin(), ids.end());
          const std::uint32_t* p = negs_in + (std::size_t(epoch) * nb + bi) * s;
          mb.negatives.assign(p, p + s);
          mb.mode = SampleMode::one_hop();
          mb.graph = &g;
        } else {
          Rng batch_rng = Rng::keyed(seed, {0x33, epoch, bi});
          mb = build_minibatch(g, ids, mode, s, batch_rng);
          if (negs_in) {
            const std::uint32_t* p = negs_in + (std::size_t(epoch) * nb + bi) * s;
            mb.negatives.assign(p, p + s);
          }
        }
        BatchSchedule sched = make_schedule(g, ids, workers, true);
        grad_minibatch(g, zm, mb, model, sched, grads, &tc);
        if (monitor) epoch_loss += batch_loss(zm, mb, model);
        apply_update(zm, ids, grads, eta);
        if (cb) cb(epoch, bi, zm.data().data(), user);
      }
      if (monitor && loss_out) loss_out[epoch] = epoch_loss;
    }
    std::memcpy(z, zm.data().data(), sizeof(float) * std::size_t(n) * d);
    if (counters) { counters[0] = tc.attractive_evals; counters[1] = tc.repulsive_evals; }
    return 0;
  } catch (const std::exception& e) {
    if (fail_info) { fail_info[0] = cur_epoch; fail_info[1] = std::uint32_t(cur_batch); }
    return classify(e);
  }
}

// build_minibatch in walk mode for one batch: the walks (ctx_offsets / ctx_ids,
// sampling.cpp:27-41,50-58) and then the negatives on (seed,{0x33,epoch,bi}).
int ref_walk_minibatch(void* gp, const std::uint32_t* ids, std::uint32_t b, std::uint32_t k,
                       std::uint32_t s, std::uint64_t seed, std::uint32_t epoch,
                       std::uint64_t bi, std::uint64_t* offs_out, std::uint32_t* ctx_out,
                       std::uint32_t* negs_out) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    Rng rng = Rng::keyed(seed, {0x33, epoch, bi});
    Minibatch mb = build_minibatch(g, std::span<const VertexId>(ids, b), SampleMode::walk(k), s,
                                   rng);
    for (std::size_t i = 0; i <= b; ++i) offs_out[i] = mb.ctx_offsets[i];
    std::memcpy(ctx_out, mb.ctx_ids.data(), sizeof(std::uint32_t) * mb.ctx_ids.size());
    std::memcpy(negs_out, mb.negatives.data(), sizeof(std::uint32_t) * s);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// The unmodified train() (init U(-0.5/d, 0.5/d), its own streams).
int ref_train_stock(void* gp, std::uint32_t d, std::uint32_t batch, std::uint32_t s,
                    float lr, std::uint32_t epochs, int kind, std::uint64_t seed,
                    std::uint32_t workers, int monitor, float* z_out, double* loss_out) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    TrainConfig cfg;
    cfg.dim = d; cfg.batch = batch; cfg.negatives = s; cfg.lr = lr; cfg.epochs = epochs;
    cfg.model = ForceModel{static_cast<ForceKind>(kind)};
    cfg.seed = seed; cfg.workers = workers; cfg.monitor_loss = monitor != 0;
    TrainResult r = train(g, cfg);
    std::memcpy(z_out, r.embedding.data().data(), sizeof(float) * r.embedding.data().size());
    if (monitor && loss_out)
      for (std::size_t i = 0; i < r.epoch_loss.size(); ++i) loss_out[i] = r.epoch_loss[i];
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// CPU baseline timer: the timed region of train() (trainer.cpp:210-236) --
// partition_epoch + build_minibatch + make_schedule + grad_minibatch +
// apply_update -- for the first `max_batches` batches of epoch 0, monitoring
// off.  negs_in == nullptr: build_minibatch's own negatives; otherwise batch
// bi's s negatives are negs_in[bi*s ..] (the BASELINE configs' Philox stream,
// injected into the Minibatch exactly as ref_train does).  Returns seconds;
// pairs_out = attractive + repulsive evaluations.
double ref_time_batches(void* gp, float* z, std::uint32_t d, std::uint32_t batch,
                        std::uint32_t s, float lr, int kind, std::uint64_t seed,
                        std::uint32_t workers, std::uint64_t max_batches,
                        const std::uint32_t* negs_in, std::uint64_t* pairs_out) {
  const CsrGraph& g = *static_cast<CsrGraph*>(gp);
  const VertexId n = g.num_vertices();
  const VertexId b = std::min<VertexId>(batch, n);
  EmbeddingMatrix zm(n, d);
  std::memcpy(zm.data().data(), z, sizeof(float) * std::size_t(n) * d);
  const ForceModel model{static_cast<ForceKind>(kind)};
  GradBuffer grads(b, d);
  TrainCounters tc;
  const auto t0 = std::chrono::steady_clock::now();
  Rng part_rng = Rng::keyed(seed, {0x22, 0});
  EpochPartition part = partition_epoch(n, b, part_rng);
  const std::size_t nb = std::min<std::size_t>(part.num_batches(), max_batches);
  for (std::size_t bi = 0; bi < nb; ++bi) {
    const auto ids = part.batch(bi);
    Rng batch_rng = Rng::keyed(seed, {0x33, 0u, bi});
    Minibatch mb = build_minibatch(g, ids, SampleMode::one_hop(), s, batch_rng);
    if (negs_in) mb.negatives.assign(negs_in + bi * s, negs_in + (bi + 1) * s);
    BatchSchedule sched = make_schedule(g, ids, workers, true);
    grad_minibatch(g, zm, mb, model, sched, grads, &tc);
    apply_update(zm, ids, grads, lr);
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (pairs_out) *pairs_out = tc.attractive_evals + tc.repulsive_evals;
  return std::chrono::duration<double>(t1 - t0).count();
}

unsigned ref_hardware_threads() { return std::thread::hardware_concurrency(); }

}  // extern "C"
