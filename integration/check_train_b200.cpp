// integration/check_train_b200.cpp -- test driver for the reference-side
// binding (trainer_b200.cpp): runs force2vec::train_b200 and the reference's
// own force2vec::train on the same graph and config, prints
//   OK <max |dz|> <bit-equal fraction> <loss_b200> <loss_ref>
// or, when the device path throws, ERROR <exception type> <message> (exit 3).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "force2vec/errors.hpp"
#include "force2vec/trainer.hpp"

namespace force2vec {
TrainResult train_b200(const CsrGraph& g, const TrainConfig& cfg, const ProgressFn& progress,
                       int device);
}

using namespace force2vec;

int main(int argc, char** argv) {
  const unsigned n = argc > 1 ? unsigned(std::atoi(argv[1])) : 2000;
  // a small planted graph: ring + chords from the reference's own Rng
  std::vector<std::pair<VertexId, VertexId>> e;
  Rng rng(7, 0);
  for (VertexId u = 0; u < n; ++u) {
    e.push_back({u, (u + 1) % n});
    for (int k = 0; k < 6; ++k) e.push_back({u, VertexId(rng.below(n))});
  }
  const CsrGraph g = CsrGraph::from_edges(std::move(e), n, true);
  TrainConfig cfg;
  cfg.dim = 32;
  cfg.batch = 128;
  cfg.negatives = 5;
  cfg.epochs = 3;
  cfg.seed = 11;
  cfg.model.kind = argc > 2 ? parse_force_kind(argv[2]) : ForceKind::Sigmoid;
  // pair_loss exists for sigmoid / tdist only (force_kernels.cpp:211-231)
  const bool lossy = cfg.model.kind == ForceKind::Sigmoid || cfg.model.kind == ForceKind::TDist;
  cfg.monitor_loss = lossy;
  TrainResult mine;
  try {
    mine = train_b200(g, cfg, {}, 0);
  } catch (const NumericalError& ex) {
    std::printf("ERROR NumericalError %s\n", ex.what());
    return 3;
  } catch (const Error& ex) {
    std::printf("ERROR Error %s\n", ex.what());
    return 3;
  }
  const TrainResult ref = train(g, cfg);
  double worst = 0;
  size_t same = 0;
  const auto& a = mine.embedding.data();
  const auto& b = ref.embedding.data();
  for (size_t i = 0; i < a.size(); ++i) {
    worst = std::max(worst, std::fabs(double(a[i]) - double(b[i])));
    same += a[i] == b[i];
  }
  std::printf("OK %.3e %.6f %.17g %.17g %llu %llu\n", worst, double(same) / double(a.size()),
              lossy ? mine.epoch_loss.back() : 0.0, lossy ? ref.epoch_loss.back() : 0.0,
              (unsigned long long)mine.counters.attractive_evals,
              (unsigned long long)ref.counters.attractive_evals);
  if (!lossy) {  // monitoring: UnsupportedError with the same message on both sides
    cfg.monitor_loss = true;
    std::string m1 = "-", m2 = "-";
    try {
      train_b200(g, cfg, {}, 0);
    } catch (const UnsupportedError& ex) {
      m1 = ex.what();
    } catch (const std::exception&) {
    }
    try {
      train(g, cfg);
    } catch (const UnsupportedError& ex) {
      m2 = ex.what();
    } catch (const std::exception&) {
    }
    std::printf("UNSUPPORTED %d %d\n", m1 != "-", int(m1 == m2));
  }
  return 0;
}
