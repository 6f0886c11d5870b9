// integration/trainer_b200.cpp -- the reference-side binding a maintainer
// adds to proj/core: force2vec::train()'s signature and types
// (trainer.hpp:15-57, 115-116) forwarded to the B200 C-ABI
// (include/force2vec_b200.h).  Compiled against the reference's own headers
// and linked with libf2v_b200.so by tests/test_integration_cpu.py (CPU: the
// C-ABI reports F2V_ECUDA, surfaced as force2vec::Error) and run against the
// reference's own train() on the GPU (tests/test_gpu_integration.py).
#include <chrono>
#include <cmath>
#include <limits>
#include <string>

#include "force2vec/errors.hpp"
#include "force2vec/trainer.hpp"
#include "force2vec_b200.h"

namespace force2vec {

TrainResult train_b200(const CsrGraph& g, const TrainConfig& cfg, const ProgressFn& progress,
                       int device) {
  cfg.validate();  // trainer.cpp:13-22: same UsageErrors before any device work
  f2v_train_config c{};
  c.dim = cfg.dim;
  c.batch = cfg.batch;
  c.negatives = cfg.negatives;
  c.lr = cfg.lr;
  c.epochs = cfg.epochs;
  c.model.kind = static_cast<int32_t>(cfg.model.kind);
  c.model.epsilon = cfg.model.epsilon;
  c.model.has_repulsion_cap = cfg.model.repulsion_cap.has_value() ? 1 : 0;
  c.model.repulsion_cap = cfg.model.repulsion_cap.value_or(0.0f);
  c.seed = cfg.seed;
  c.lr_decay = cfg.lr_decay == TrainConfig::LrDecay::LinearToZero ? 1 : 0;
  c.monitor_loss = cfg.monitor_loss ? 1 : 0;
  c.sampler = F2V_SAMPLER_SPLITMIX;   // the reference's own negative stream
  c.precision = F2V_PRECISION_EXACT;  // the reference's fp64 arithmetic
  c.walk_length = cfg.mode.kind == SampleMode::Kind::Walk ? cfg.mode.walk_length : 0;
  TrainResult r;
  r.embedding = EmbeddingMatrix(g.num_vertices(), cfg.dim);
  f2v_ctx* ctx = f2v_create(device);
  if (!ctx) throw Error(f2v_global_error());
  auto check = [&](int32_t rc) {
    if (rc == F2V_OK) return;
    const std::string msg = f2v_last_error(ctx);
    f2v_destroy(ctx);
    switch (rc) {  // errors.hpp:8-40
      case F2V_EUSAGE: throw UsageError(msg);
      case F2V_ERANGE: throw RangeError(msg);
      case F2V_ENUMERICAL: throw NumericalError(msg);
      case F2V_EUNSUPPORTED: throw UnsupportedError(msg);
      default: throw Error(msg);
    }
  };
  check(f2v_upload_graph(ctx, g.num_vertices(), g.row_offsets().data(), g.col_indices().data(),
                         g.num_edges()));
  f2v_counters ctr{};
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t e = 0; e < cfg.epochs; ++e) {  // one call per epoch: progress callbacks
    c.first_epoch = e;
    c.run_epochs = 1;
    c.init = e == 0 ? 1 : 0;  // init_embedding exactly as train() does (trainer.cpp:203-206)
    double loss = 0;
    f2v_failure fail{};
    check(f2v_train_epochs(ctx, &c, &loss, &ctr, &fail));
    if (cfg.monitor_loss) r.epoch_loss.push_back(loss);
    if (progress)
      progress(e, cfg.monitor_loss ? loss : std::numeric_limits<double>::quiet_NaN(),
               std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                   .count());
  }
  check(f2v_get_embedding(ctx, r.embedding.data().data()));
  r.counters.attractive_evals = ctr.attractive_evals;
  r.counters.repulsive_evals = ctr.repulsive_evals;
  f2v_destroy(ctx);
  return r;
}

}  // namespace force2vec
