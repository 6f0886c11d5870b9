// oracle/ref_eval.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" access to the UNMODIFIED reference's evaluation and embedding
// I/O (proj/core/src/evaluation.cpp, embedding_io.cpp, compiled in place by
// oracle/Makefile into oracle/_ref/libf2vref.so), for the golden fixtures of
// SURVEY.md section 8(f) row 4 (oracle/make_golden_eval.py) and the parity
// tests that run where the reference tree is present.
//   * write_embedding / read_embedding / write_layout_tsv  embedding_io.cpp:24-124
//   * kmeans / kmeans_inertia / modularity / sweep          evaluation.cpp:323-497
//   * fit_logreg / logreg_loss                              evaluation.cpp:87-153
//   * build_link_dataset / link_prediction_accuracy         evaluation.cpp:36-85,155-173
//   * node_classification                                   evaluation.cpp:217-321
// The Rng is passed as its state word (rng.hpp:52: the class's only member).
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "force2vec/csr_graph.hpp"
#include "force2vec/embedding_io.hpp"
#include "force2vec/evaluation.hpp"
#include "force2vec/rng.hpp"
#include "force2vec/trainer.hpp"

using namespace force2vec;

namespace {
// libstdc++ is linked statically into libf2vref.so: its stream/locale state is
// initialised only if some translation unit constructs ios_base::Init
std::ios_base::Init g_ios_init;
thread_local std::string g_err;

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

static_assert(sizeof(Rng) == sizeof(std::uint64_t), "Rng is its state word");
Rng rng_from(std::uint64_t state) {
  Rng r(0, 0);
  std::memcpy(&r, &state, sizeof(state));
  return r;
}
std::uint64_t rng_state(const Rng& r) {
  std::uint64_t s;
  std::memcpy(&s, &r, sizeof(s));
  return s;
}

EmbeddingMatrix to_matrix(const float* z, std::uint32_t n, std::uint32_t d) {
  EmbeddingMatrix m(n, d);
  std::memcpy(m.data().data(), z, sizeof(float) * std::size_t(n) * d);
  return m;
}

LabeledNodes to_labels(std::uint32_t n, const std::uint64_t* off, const std::int32_t* ids,
                       int num_classes) {
  LabeledNodes l;
  l.labels.resize(n);
  l.num_classes = num_classes;
  for (std::uint32_t u = 0; u < n; ++u) {
    l.labels[u].assign(ids + off[u], ids + off[u + 1]);
    if (l.labels[u].size() > 1) l.multi_label = true;
  }
  return l;
}

FeatureMatrix to_features(const float* x, std::uint64_t rows, std::uint32_t cols) {
  FeatureMatrix f(rows, cols);
  std::memcpy(f.data.data(), x, sizeof(float) * rows * cols);
  return f;
}
}  // namespace

extern "C" {

const char* ref_eval_last_error() { return g_err.c_str(); }

std::uint64_t ref_rng_state(std::uint64_t seed, std::uint64_t stream) {
  return rng_state(Rng(seed, stream));
}

// ---- embedding_io.cpp ------------------------------------------------------
int ref_write_embedding(const char* path, const float* z, std::uint32_t n, std::uint32_t d) {
  try {
    std::ofstream out(path, std::ios::binary);
    write_embedding(out, to_matrix(z, n, d));
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// reads the header first (n_out, d_out), then z when non-null
int ref_read_embedding(const char* path, float* z, std::uint32_t* n_out, std::uint32_t* d_out) {
  try {
    std::ifstream in(path, std::ios::binary);
    const EmbeddingMatrix m = read_embedding(in);
    *n_out = m.rows();
    *d_out = m.dim();
    if (z) std::memcpy(z, m.data().data(), sizeof(float) * std::size_t(m.rows()) * m.dim());
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_write_layout_tsv(const char* path, const float* z, std::uint32_t n, std::uint32_t d,
                         const std::int32_t* first_label) {
  try {
    std::ofstream out(path, std::ios::binary);
    LabeledNodes l;
    if (first_label) {
      l.labels.resize(n);
      for (std::uint32_t u = 0; u < n; ++u)
        if (first_label[u] >= 0) l.labels[u].push_back(first_label[u]);
    }
    write_layout_tsv(out, to_matrix(z, n, d), first_label ? &l : nullptr);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_write_layout_svg(const char* path, const float* z, std::uint32_t n, std::uint32_t d,
                         const std::int32_t* first_label) {
  try {
    std::ofstream out(path, std::ios::binary);
    LabeledNodes l;
    if (first_label) {
      l.labels.resize(n);
      for (std::uint32_t u = 0; u < n; ++u)
        if (first_label[u] >= 0) l.labels[u].push_back(first_label[u]);
    }
    write_layout_svg(out, to_matrix(z, n, d), first_label ? &l : nullptr);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// load_labels: CSR over vertices into caller buffers (ids sized >= the line count)
int ref_load_labels(const char* path, std::uint32_t n, std::uint64_t* off, std::int32_t* ids,
                    int* num_classes, int* multi) {
  try {
    std::ifstream in(path, std::ios::binary);
    const LabeledNodes l = load_labels(in, n);
    off[0] = 0;
    std::uint64_t k = 0;
    for (std::uint32_t u = 0; u < n; ++u) {
      for (int c : l.labels[u]) ids[k++] = c;
      off[u + 1] = k;
    }
    *num_classes = l.num_classes;
    *multi = l.multi_label ? 1 : 0;
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// ---- evaluation.cpp: clustering -------------------------------------------
int ref_kmeans(const float* z, std::uint32_t n, std::uint32_t d, int k, std::uint64_t* state,
               int restarts, int max_iters, std::int32_t* assign_out, double* inertia_out) {
  try {
    Rng rng = rng_from(*state);
    const EmbeddingMatrix m = to_matrix(z, n, d);
    const Clustering c = kmeans(m, k, rng, restarts, max_iters);
    *state = rng_state(rng);
    for (std::size_t i = 0; i < c.assignment.size(); ++i) assign_out[i] = c.assignment[i];
    if (inertia_out) *inertia_out = c.assignment.empty() ? 0.0 : kmeans_inertia(m, c);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_kmeans_inertia(const float* z, std::uint32_t n, std::uint32_t d, int k,
                       const std::int32_t* assign, double* out) {
  try {
    Clustering c;
    c.k = k;
    c.assignment.assign(assign, assign + n);
    *out = kmeans_inertia(to_matrix(z, n, d), c);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_modularity(void* gp, int k, const std::int32_t* assign, std::uint32_t len, double* out) {
  try {
    Clustering c;
    c.k = k;
    c.assignment.assign(assign, assign + len);
    *out = modularity(*static_cast<CsrGraph*>(gp), c);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_best_modularity_sweep(void* gp, const float* z, std::uint32_t n, std::uint32_t d,
                              std::uint64_t* state, int kmax, int* k_out, double* q_out) {
  try {
    Rng rng = rng_from(*state);
    const SweepResult r =
        best_modularity_sweep(*static_cast<CsrGraph*>(gp), to_matrix(z, n, d), rng, kmax);
    *state = rng_state(rng);
    *k_out = r.k;
    *q_out = r.q;
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// ---- evaluation.cpp: logistic regression ----------------------------------
int ref_fit_logreg(const float* x, std::uint64_t rows, std::uint32_t cols,
                   const std::int32_t* targets, double lr, int iters, double l2, double* w_out) {
  try {
    LogRegConfig cfg{lr, iters, l2};
    const std::vector<int> t(targets, targets + rows);
    const LogRegModel m = fit_logreg(to_features(x, rows, cols), t, cfg);
    std::memcpy(w_out, m.weights.data(), sizeof(double) * (cols + 1));
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_logreg_loss(const double* w, const float* x, std::uint64_t rows, std::uint32_t cols,
                    const std::int32_t* targets, double l2, double* out) {
  try {
    LogRegModel m;
    m.weights.assign(w, w + cols + 1);
    const std::vector<int> t(targets, targets + rows);
    *out = logreg_loss(m, to_features(x, rows, cols), t, l2);
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

// pairs as u32 triples (u, v, is_edge); buffers sized by ref_link_dataset_size
static LinkDataset g_ds;
int ref_build_link_dataset(void* gp, std::uint64_t* state, std::uint64_t* ntrain,
                           std::uint64_t* ntest) {
  try {
    Rng rng = rng_from(*state);
    g_ds = build_link_dataset(*static_cast<CsrGraph*>(gp), rng);
    *state = rng_state(rng);
    *ntrain = g_ds.train.size();
    *ntest = g_ds.test.size();
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}
void ref_link_dataset_export(std::uint32_t* train, std::uint32_t* test) {
  for (std::size_t i = 0; i < g_ds.train.size(); ++i) {
    train[3 * i] = g_ds.train[i].u;
    train[3 * i + 1] = g_ds.train[i].v;
    train[3 * i + 2] = g_ds.train[i].is_edge;
  }
  for (std::size_t i = 0; i < g_ds.test.size(); ++i) {
    test[3 * i] = g_ds.test[i].u;
    test[3 * i + 1] = g_ds.test[i].v;
    test[3 * i + 2] = g_ds.test[i].is_edge;
  }
}

int ref_link_prediction_accuracy(const float* z, std::uint32_t n, std::uint32_t d,
                                 const std::uint32_t* train, std::uint64_t ntrain,
                                 const std::uint32_t* test, std::uint64_t ntest, double lr,
                                 int iters, double l2, double* out) {
  try {
    LinkDataset ds;
    for (std::uint64_t i = 0; i < ntrain; ++i)
      ds.train.push_back({train[3 * i], train[3 * i + 1], train[3 * i + 2] != 0});
    for (std::uint64_t i = 0; i < ntest; ++i)
      ds.test.push_back({test[3 * i], test[3 * i + 1], test[3 * i + 2] != 0});
    *out = link_prediction_accuracy(to_matrix(z, n, d), ds, LogRegConfig{lr, iters, l2});
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

int ref_node_classification(const float* z, std::uint32_t n, std::uint32_t d,
                            const std::uint64_t* off, const std::int32_t* ids, int num_classes,
                            double train_fraction, std::uint64_t* state, double lr, int iters,
                            double l2, double* micro, double* macro) {
  try {
    Rng rng = rng_from(*state);
    const F1Scores s = node_classification(to_matrix(z, n, d), to_labels(n, off, ids, num_classes),
                                           train_fraction, rng, LogRegConfig{lr, iters, l2});
    *state = rng_state(rng);
    *micro = s.micro;
    *macro = s.macro;
    return 0;
  } catch (const std::exception& e) { return classify(e); }
}

}  // extern "C"
