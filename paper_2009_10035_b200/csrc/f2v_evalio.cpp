// f2v_evalio.cpp -- SURVEY.md section 8(f) row 4, host side: embedding text
// I/O (proj/core/src/embedding_io.cpp:24-124), the link-prediction dataset
// (evaluation.cpp:36-85), the node-classification and modularity-sweep drivers
// (evaluation.cpp:217-321, 485-497) above the device kernels of f2v_eval.cu,
// and their extern "C" entry points (include/force2vec_b200.h).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "f2v_internal.h"
#include "f2v_rng.h"

namespace f2v {
namespace {

// the reference's Rng (rng.hpp:26-42) over a caller-held state word
struct Stream {
  uint64_t& s;
  uint64_t next() {
    s += kGamma;
    return mix64(s);
  }
  uint64_t below(uint64_t n) { return rng_below(next(), n); }
};

template <class T>
void shuffle(std::vector<T>& v, Stream& rng) {  // evaluation.cpp:29-32
  for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[rng.below(i)]);
}

bool is_space(char c) {  // std::isspace in the "C" locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

void append_float(std::string& buf, float v) {  // shortest round-trip decimal
  char tmp[32];
  const auto r = std::to_chars(tmp, tmp + sizeof(tmp), v);
  buf.append(tmp, r.ptr);
}

// Rows [r0, r1) of the body, "id f_1 ... f_d\n" each (embedding_io.cpp:28-37)
void format_rows(const float* z, uint32_t d, uint64_t r0, uint64_t r1, std::string& out) {
  out.clear();
  out.reserve((r1 - r0) * (size_t(d) * 13 + 12));
  char tmp[24];
  for (uint64_t u = r0; u < r1; ++u) {
    const auto r = std::to_chars(tmp, tmp + sizeof(tmp), u);
    out.append(tmp, r.ptr);
    const float* row = z + u * d;
    for (uint32_t j = 0; j < d; ++j) {
      out.push_back(' ');
      append_float(out, row[j]);
    }
    out.push_back('\n');
  }
}

void write_embedding(const char* path, const float* z, uint32_t n, uint32_t d) {
  File fp(path, "wb");
  if (!fp.f) fail(F2V_EIO, std::string("cannot open ") + path + " for writing");
  std::string head = std::to_string(n) + ' ' + std::to_string(d) + '\n';
  bool ok = std::fwrite(head.data(), 1, head.size(), fp.f) == head.size();
  // row blocks are formatted by a wave of threads and written in order
  const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const uint64_t block = 2048;
  std::vector<std::string> bufs(T);
  for (uint64_t r0 = 0; r0 < n && ok; r0 += block * T) {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) {
      const uint64_t a = r0 + block * t, b = std::min<uint64_t>(n, a + block);
      if (a >= n) break;
      th.emplace_back([&, a, b, t] { format_rows(z, d, a, b, bufs[t]); });
    }
    for (size_t t = 0; t < th.size(); ++t) {
      th[t].join();
      ok = ok && std::fwrite(bufs[t].data(), 1, bufs[t].size(), fp.f) == bufs[t].size();
    }
  }
  if (!ok || std::fflush(fp.f) != 0) fail(F2V_EIO, "failed writing embedding");
}

std::vector<char> slurp(const char* path) {
  File fp(path, "rb");
  if (!fp.f) fail(F2V_EIO, std::string("cannot open ") + path);
  std::vector<char> buf;
  char tmp[1 << 16];
  size_t got;
  while ((got = std::fread(tmp, 1, sizeof(tmp), fp.f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  return buf;
}

// read_embedding (embedding_io.cpp:42-100): the same acceptance rules and the
// same messages, parsed from one in-memory buffer.
void read_embedding(const char* path, std::vector<float>& z, uint64_t& n, uint64_t& d) {
  const std::vector<char> buf = slurp(path);
  const char* cur = buf.data();
  const char* const eof = buf.data() + buf.size();
  // one std::getline: [cur, nl), '\r' stripped; false at end of input
  auto next_line = [&](const char*& p, const char*& end) {
    if (cur == eof) return false;
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', size_t(eof - cur)));
    p = cur;
    end = nl ? nl : eof;
    cur = nl ? nl + 1 : eof;
    if (end > p && end[-1] == '\r') --end;
    return true;
  };
  auto skip_space = [](const char*& p, const char* end) {
    while (p < end && is_space(*p)) ++p;
  };
  const char *p, *end;
  if (!next_line(p, end)) fail(F2V_ERANGE, "missing embedding header");
  {
    n = d = 0;
    const auto r1 = std::from_chars(p, end, n);
    p = r1.ptr;
    skip_space(p, end);
    const auto r2 = std::from_chars(p, end, d);
    if (r1.ec != std::errc() || r2.ec != std::errc() || n == 0 || d == 0 ||
        n > 0xffffffffull || d > 0xffffffffull)
      fail(F2V_ERANGE, "bad embedding header at line 1");
  }
  z.assign(size_t(n) * d, 0.0f);
  std::vector<bool> filled(n, false);
  uint64_t rows_read = 0, line_no = 1;
  while (next_line(p, end)) {
    ++line_no;
    const char* q = p;
    skip_space(q, end);
    if (q == end) continue;  // blank
    if (rows_read == n) fail(F2V_ERANGE, "extra body line " + std::to_string(line_no));
    uint64_t id = 0;
    const auto r = std::from_chars(p, end, id);
    if (r.ec != std::errc() || id >= n)
      fail(F2V_ERANGE, "bad vertex id at line " + std::to_string(line_no));
    if (filled[id]) fail(F2V_ERANGE, "duplicate vertex id at line " + std::to_string(line_no));
    p = r.ptr;
    float* row = z.data() + id * d;
    for (uint64_t j = 0; j < d; ++j) {
      skip_space(p, end);
      float v;
      const auto rv = std::from_chars(p, end, v);
      if (rv.ec != std::errc())
        fail(F2V_ERANGE, "expected " + std::to_string(d + 1) + " tokens at line " +
                             std::to_string(line_no));
      row[j] = v;
      p = rv.ptr;
    }
    skip_space(p, end);
    if (p != end) fail(F2V_ERANGE, "trailing tokens at line " + std::to_string(line_no));
    filled[id] = true;
    ++rows_read;
  }
  if (rows_read != n)
    fail(F2V_ERANGE, "expected " + std::to_string(n) + " body lines, got " +
                         std::to_string(rows_read));
}

void write_layout_tsv(const char* path, const float* z, uint32_t n, uint32_t d,
                      const int32_t* first_label) {
  if (d != 2) fail(F2V_EUSAGE, "layout export requires a 2-D embedding (train with dim 2)");
  File fp(path, "wb");
  if (!fp.f) fail(F2V_EIO, std::string("cannot open ") + path + " for writing");
  std::string buf;
  bool ok = true;
  for (uint32_t u = 0; u < n; ++u) {
    buf.append(std::to_string(u));
    buf.push_back('\t');
    append_float(buf, z[size_t(u) * 2]);
    buf.push_back('\t');
    append_float(buf, z[size_t(u) * 2 + 1]);
    if (first_label && first_label[u] >= 0) {
      buf.push_back('\t');
      buf.append(std::to_string(first_label[u]));
    }
    buf.push_back('\n');
    if (buf.size() > (1u << 20) || u + 1 == n) {
      ok = ok && std::fwrite(buf.data(), 1, buf.size(), fp.f) == buf.size();
      buf.clear();
    }
  }
  if (!ok || std::fflush(fp.f) != 0) fail(F2V_EIO, "failed writing layout tsv");
}

// write_layout_svg (embedding_io.cpp:126-159).  The reference streams its doubles
// with the default ostream format (%g, 6 significant digits); the coordinates
// are float arithmetic widened at the end, as in the reference's expressions.
void write_layout_svg(const char* path, const float* z, uint32_t n, uint32_t d,
                      const int32_t* first_label) {
  if (d != 2) fail(F2V_EUSAGE, "layout export requires a 2-D embedding (train with dim 2)");
  File fp(path, "wb");
  if (!fp.f) fail(F2V_EIO, std::string("cannot open ") + path + " for writing");
  float min_x = INFINITY, max_x = -INFINITY, min_y = INFINITY, max_y = -INFINITY;
  for (uint32_t u = 0; u < n; ++u) {
    min_x = std::min(min_x, z[size_t(u) * 2]);
    max_x = std::max(max_x, z[size_t(u) * 2]);
    min_y = std::min(min_y, z[size_t(u) * 2 + 1]);
    max_y = std::max(max_y, z[size_t(u) * 2 + 1]);
  }
  const float span_x = std::max(max_x - min_x, 1e-9f);
  const float span_y = std::max(max_y - min_y, 1e-9f);
  const int size = 800, margin = 20;
  static const char* kPalette[12] = {"#1f77b4", "#ff7f0e", "#2ca02c", "#d62728", "#9467bd",
                                     "#8c564b", "#e377c2", "#7f7f7f", "#bcbd22", "#17becf",
                                     "#aec7e8", "#ffbb78"};
  std::string buf = "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"800\" height=\"800\" "
                    "viewBox=\"0 0 800 800\">\n";
  bool ok = true;
  char num[64];
  for (uint32_t u = 0; u < n; ++u) {
    const double x = margin + (z[size_t(u) * 2] - min_x) / span_x * (size - 2 * margin);
    const double y = margin + (max_y - z[size_t(u) * 2 + 1]) / span_y * (size - 2 * margin);
    const char* color = kPalette[0];
    if (first_label && first_label[u] >= 0) color = kPalette[first_label[u] % 12];
    buf += "<circle cx=\"";
    std::snprintf(num, sizeof(num), "%g", x);
    buf += num;
    buf += "\" cy=\"";
    std::snprintf(num, sizeof(num), "%g", y);
    buf += num;
    buf += "\" r=\"2.5\" fill=\"";
    buf += color;
    buf += "\" fill-opacity=\"0.8\"/>\n";
    if (buf.size() > (1u << 20)) {
      ok = ok && std::fwrite(buf.data(), 1, buf.size(), fp.f) == buf.size();
      buf.clear();
    }
  }
  buf += "</svg>\n";
  ok = ok && std::fwrite(buf.data(), 1, buf.size(), fp.f) == buf.size();
  if (!ok || std::fflush(fp.f) != 0) fail(F2V_EIO, "failed writing layout svg");
}

// load_labels (evaluation.cpp:175-199)
void load_labels(const char* path, uint32_t n, std::vector<uint64_t>& off, std::vector<int32_t>& ids,
                 int32_t& num_classes, int32_t& multi) {
  const std::vector<char> buf = slurp(path);
  std::vector<std::vector<int32_t>> labels(n);
  const char* cur = buf.data();
  const char* const eof = buf.data() + buf.size();
  uint64_t line_no = 0;
  int max_label = -1;
  while (cur != eof) {
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', size_t(eof - cur)));
    const char* p = cur;
    const char* end = nl ? nl : eof;
    cur = nl ? nl + 1 : eof;
    ++line_no;
    if (end > p && end[-1] == '\r') --end;
    const char* q = p;
    while (q < end && is_space(*q)) ++q;
    if (q == end || *p == '#' || *p == '%') continue;
    uint64_t u = 0, label = 0;
    const auto r1 = std::from_chars(p, end, u);
    p = r1.ptr;
    while (p < end && is_space(*p)) ++p;
    const auto r2 = std::from_chars(p, end, label);
    if (r1.ec != std::errc() || r2.ec != std::errc())
      fail(F2V_ERANGE, "bad label line " + std::to_string(line_no));
    if (u >= n) fail(F2V_ERANGE, "label vertex id out of range at line " + std::to_string(line_no));
    labels[u].push_back(int32_t(label));
    max_label = std::max(max_label, int(label));
  }
  num_classes = max_label + 1;
  multi = 0;
  off.assign(size_t(n) + 1, 0);
  ids.clear();
  for (uint32_t u = 0; u < n; ++u) {
    auto& ls = labels[u];
    std::sort(ls.begin(), ls.end());
    ls.erase(std::unique(ls.begin(), ls.end()), ls.end());
    if (ls.size() > 1) multi = 1;
    ids.insert(ids.end(), ls.begin(), ls.end());
    off[u + 1] = ids.size();
  }
}

// ------------------------------------------------------ link-prediction data
bool has_arc(const uint64_t* rowptr, const uint32_t* col, uint32_t u, uint32_t v) {
  return std::binary_search(col + rowptr[u], col + rowptr[u + 1], v);
}

struct Pair3 {
  uint32_t u, v, e;
};

// build_link_dataset (evaluation.cpp:36-85).  The reference's hash set of seen
// pairs answers two questions; both are answered from the sorted CSR rows
// here: arc (u, v) opens a new undirected pair iff u < v or the reverse arc
// is absent (rows are visited in vertex order), and a drawn non-edge repeats
// iff it is among the negatives drawn so far (the only set kept).
void build_link_dataset(uint32_t n, const uint64_t* rowptr, const uint32_t* col, Stream& rng,
                        std::vector<Pair3>& train, std::vector<Pair3>& test) {
  constexpr size_t kMaxPositives = 1'000'000;
  if (rowptr[n] == 0) fail(F2V_EUSAGE, "link dataset needs at least one edge");
  std::vector<Pair3> pairs;
  for (uint32_t u = 0; u < n; ++u)
    for (uint64_t t = rowptr[u]; t < rowptr[u + 1]; ++t) {
      const uint32_t v = col[t];
      if (u < v || (u > v && !has_arc(rowptr, col, v, u))) pairs.push_back({u, v, 1});
    }
  if (pairs.size() > kMaxPositives) {
    shuffle(pairs, rng);
    pairs.resize(kMaxPositives);
  }
  const size_t positives = pairs.size();
  const uint64_t all_pairs = uint64_t(n) * (n - 1) / 2;
  if (all_pairs <= positives) fail(F2V_EUSAGE, "graph too dense: no non-edges to sample");
  std::unordered_set<uint64_t> drawn;
  drawn.reserve(positives * 2);
  size_t negatives = 0;
  uint64_t attempts = 0;
  const uint64_t max_attempts = 1000 * uint64_t(positives) + 1000;
  while (negatives < positives) {
    if (++attempts > max_attempts)
      fail(F2V_EUSAGE, "could not sample enough distinct non-edges");
    const uint32_t u = uint32_t(rng.below(n));
    const uint32_t v = uint32_t(rng.below(n));
    if (u == v || has_arc(rowptr, col, u, v) || has_arc(rowptr, col, v, u)) continue;
    const uint32_t a = std::min(u, v), b = std::max(u, v);
    if (!drawn.insert((uint64_t(a) << 32) | b).second) continue;
    pairs.push_back({u, v, 0});
    ++negatives;
  }
  shuffle(pairs, rng);
  const size_t half = pairs.size() / 2;
  train.assign(pairs.begin(), pairs.begin() + half);
  test.assign(pairs.begin() + half, pairs.end());
}

// ------------------------------------------------------- node classification
// f1_from_counts (evaluation.cpp:201-215)
struct Counts {
  uint64_t tp = 0, fp = 0, fn = 0;
};
void f1_from_counts(const std::vector<Counts>& counts, double& micro, double& macro_out) {
  uint64_t tp = 0, fp = 0, fn = 0;
  double macro = 0.0;
  for (const Counts& c : counts) {
    tp += c.tp;
    fp += c.fp;
    fn += c.fn;
    const double denom = double(2 * c.tp + c.fp + c.fn);
    macro += denom > 0 ? 2.0 * double(c.tp) / denom : 0.0;
  }
  const double denom = double(2 * tp + fp + fn);
  micro = denom > 0 ? 2.0 * double(tp) / denom : 0.0;
  macro_out = counts.empty() ? 0.0 : macro / double(counts.size());
}

// node_classification (evaluation.cpp:217-321): the split logic and the tallies
// on the host, the num_classes logistic regressions as one device batch
void node_classification(Ctx& c, const uint64_t* loff, const int32_t* lids, int num_classes,
                         double train_fraction, Stream& rng, const f2v_logreg_config& cfg,
                         double& micro, double& macro) {
  if (!(train_fraction > 0.0 && train_fraction < 1.0))
    fail(F2V_EUSAGE, "train_fraction must be in (0, 1)");
  if (num_classes < 2) fail(F2V_EUSAGE, "need at least two classes");
  const uint32_t n = c.n;
  auto nlab = [&](uint32_t u) { return size_t(loff[u + 1] - loff[u]); };
  auto has_label = [&](uint32_t u, int cl) {
    return std::binary_search(lids + loff[u], lids + loff[u + 1], cl);
  };
  std::vector<uint32_t> labeled;
  bool multi = false;
  for (uint32_t u = 0; u < n; ++u) {
    if (nlab(u)) labeled.push_back(u);
    if (nlab(u) > 1) multi = true;
    for (uint64_t t = loff[u]; t < loff[u + 1]; ++t)
      if (lids[t] < 0 || lids[t] >= num_classes) fail(F2V_ERANGE, "label id out of range");
  }
  if (labeled.empty()) fail(F2V_EUSAGE, "no labeled vertices");
  for (int attempt = 0; attempt < 10; ++attempt) {
    std::vector<uint32_t> train_ids, test_ids;
    if (!multi) {  // stratified: each class split separately
      std::vector<std::vector<uint32_t>> by_class(num_classes);
      for (uint32_t u : labeled) by_class[lids[loff[u]]].push_back(u);
      for (auto& members : by_class) {
        shuffle(members, rng);
        const size_t take = std::max<size_t>(
            1, size_t(std::llround(train_fraction * double(members.size()))));
        for (size_t i = 0; i < members.size(); ++i)
          (i < take ? train_ids : test_ids).push_back(members[i]);
      }
    } else {
      std::vector<uint32_t> order = labeled;
      shuffle(order, rng);
      const size_t take =
          std::max<size_t>(1, size_t(std::llround(train_fraction * double(order.size()))));
      train_ids.assign(order.begin(), order.begin() + take);
      test_ids.assign(order.begin() + take, order.end());
    }
    if (test_ids.empty()) fail(F2V_EUSAGE, "train fraction leaves no test set");
    std::vector<bool> present(num_classes, false);
    for (uint32_t u : train_ids)
      for (uint64_t t = loff[u]; t < loff[u + 1]; ++t) present[lids[t]] = true;
    if (!std::all_of(present.begin(), present.end(), [](bool b) { return b; })) continue;

    const size_t ntr = train_ids.size(), nte = test_ids.size();
    std::vector<uint8_t> tgt(size_t(num_classes) * ntr);
    for (int cl = 0; cl < num_classes; ++cl)
      for (size_t i = 0; i < ntr; ++i) tgt[size_t(cl) * ntr + i] = has_label(train_ids[i], cl);
    std::vector<double> prob(nte * size_t(num_classes));
    ev::one_vs_rest(c, c.zcur(), c.d, train_ids.data(), ntr, test_ids.data(), nte,
                    uint32_t(num_classes), tgt.data(), cfg.lr, cfg.iters, cfg.l2, nullptr,
                    prob.data());
    std::vector<Counts> counts(num_classes);
    std::vector<std::pair<double, int>> ranked(num_classes);
    for (size_t i = 0; i < nte; ++i) {
      const uint32_t u = test_ids[i];
      for (int cl = 0; cl < num_classes; ++cl) ranked[cl] = {prob[i * num_classes + cl], cl};
      const size_t l = nlab(u);
      std::vector<int> predicted;
      if (multi) {  // top-l with l = the true label count
        std::partial_sort(ranked.begin(), ranked.begin() + l, ranked.end(), std::greater<>());
        for (size_t t = 0; t < l; ++t) predicted.push_back(ranked[t].second);
      } else {
        predicted.push_back(std::max_element(ranked.begin(), ranked.end())->second);
      }
      std::sort(predicted.begin(), predicted.end());
      for (int cl : predicted) {
        if (has_label(u, cl)) ++counts[cl].tp;
        else ++counts[cl].fp;
      }
      for (uint64_t t = loff[u]; t < loff[u + 1]; ++t)
        if (!std::binary_search(predicted.begin(), predicted.end(), lids[t])) ++counts[lids[t]].fn;
    }
    f1_from_counts(counts, micro, macro);
    return;
  }
  fail(F2V_EERROR, "node_classification: a class was absent from training in 10 splits");
}

void need_eval_state(const Ctx& c, bool graph) {
  if (graph && !c.rowptr.p) fail(F2V_EUSAGE, "no graph uploaded");
  if (!c.z[c.cur].p || c.d == 0) fail(F2V_EUSAGE, "no embedding set");
}

void check_logreg(const f2v_logreg_config& cfg) {
  if (cfg.iters < 0) fail(F2V_EUSAGE, "logreg iters must be >= 0");
}

}  // namespace
}  // namespace f2v

using namespace f2v;

extern "C" {

int32_t f2v_write_embedding(const char* path, const float* z, uint32_t n, uint32_t d) {
  return guard(nullptr, [&] { write_embedding(path, z, n, d); });
}

int32_t f2v_read_embedding(const char* path, float** z_out, uint32_t* n_out, uint32_t* d_out) {
  return guard(nullptr, [&] {
    std::vector<float> z;
    uint64_t n = 0, d = 0;
    read_embedding(path, z, n, d);
    float* out = static_cast<float*>(std::malloc(sizeof(float) * z.size()));
    if (!out) throw std::bad_alloc();
    std::memcpy(out, z.data(), sizeof(float) * z.size());
    *z_out = out;
    *n_out = uint32_t(n);
    *d_out = uint32_t(d);
  });
}

int32_t f2v_write_layout_tsv(const char* path, const float* z, uint32_t n, uint32_t d,
                             const int32_t* first_label) {
  return guard(nullptr, [&] { write_layout_tsv(path, z, n, d, first_label); });
}

int32_t f2v_write_layout_svg(const char* path, const float* z, uint32_t n, uint32_t d,
                             const int32_t* first_label) {
  return guard(nullptr, [&] { write_layout_svg(path, z, n, d, first_label); });
}

int32_t f2v_load_labels(const char* path, uint32_t n, uint64_t** offsets_out, int32_t** ids_out,
                        int32_t* num_classes_out, int32_t* multi_label_out) {
  return guard(nullptr, [&] {
    std::vector<uint64_t> off;
    std::vector<int32_t> ids;
    int32_t nc = 0, multi = 0;
    load_labels(path, n, off, ids, nc, multi);
    uint64_t* o = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * off.size()));
    int32_t* i = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max<size_t>(1, ids.size())));
    if (!o || !i) throw std::bad_alloc();
    std::memcpy(o, off.data(), sizeof(uint64_t) * off.size());
    if (!ids.empty()) std::memcpy(i, ids.data(), sizeof(int32_t) * ids.size());
    *offsets_out = o;
    *ids_out = i;
    *num_classes_out = nc;
    *multi_label_out = multi;
  });
}

uint64_t f2v_rng_state(uint64_t seed, uint64_t stream) { return rng_init(seed, stream); }

int32_t f2v_kmeans(f2v_ctx* h, int32_t k, uint64_t* rng_state, int32_t restarts,
                   int32_t max_iters, int32_t* assignment_out, double* inertia_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_eval_state(c, false);
    F2V_CUDA(cudaSetDevice(c.device));
    const double inertia =
        ev::kmeans(c, c.zcur(), c.n, c.d, k, *rng_state, restarts, max_iters, assignment_out);
    if (inertia_out) *inertia_out = inertia;
  });
}

int32_t f2v_kmeans_inertia(f2v_ctx* h, int32_t k, const int32_t* assignment,
                           double* inertia_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_eval_state(c, false);
    if (k < 1) fail(F2V_EUSAGE, "kmeans_inertia: k must be >= 1");
    F2V_CUDA(cudaSetDevice(c.device));
    *inertia_out = ev::kmeans_inertia(c, c.zcur(), c.n, c.d, k, assignment);
  });
}

int32_t f2v_modularity(f2v_ctx* h, int32_t k, const int32_t* assignment, double* q_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    if (!c.rowptr.p) fail(F2V_EUSAGE, "no graph uploaded");
    if (c.walk_k) fail(F2V_EUSAGE, "modularity needs the graph context (one-hop)");
    F2V_CUDA(cudaSetDevice(c.device));
    *q_out = ev::modularity(c, k, assignment);
  });
}

int32_t f2v_best_modularity_sweep(f2v_ctx* h, uint64_t* rng_state, int32_t kmax, int32_t* k_out,
                                  double* q_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_eval_state(c, true);
    F2V_CUDA(cudaSetDevice(c.device));
    const int upper = int(std::min<int64_t>(kmax, int64_t(c.n)));
    if (upper < 2) fail(F2V_EUSAGE, "best_modularity_sweep needs n >= 2");
    int best_k = 0;
    double best_q = -std::numeric_limits<double>::infinity();
    std::vector<int32_t> assign(c.n);
    for (int k = 2; k <= upper; ++k) {
      ev::kmeans(c, c.zcur(), c.n, c.d, k, *rng_state, 10, 300, assign.data());
      const double q = ev::modularity(c, k, assign.data());
      if (q > best_q) {
        best_q = q;
        best_k = k;
      }
    }
    *k_out = best_k;
    *q_out = best_q;
  });
}

int32_t f2v_fit_logreg(f2v_ctx* h, const float* features, uint64_t rows, uint32_t cols,
                       const int32_t* targets, f2v_logreg_config cfg, double* weights_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    check_logreg(cfg);
    if (rows < 1 || cols < 1) fail(F2V_ERANGE, "fit_logreg: target count mismatch");
    F2V_CUDA(cudaSetDevice(c.device));
    ev::fit_logreg(c, features, rows, cols, targets, cfg.lr, cfg.iters, cfg.l2, weights_out);
  });
}

int32_t f2v_logreg_loss(f2v_ctx* h, const double* weights, const float* features, uint64_t rows,
                        uint32_t cols, const int32_t* targets, double l2, double* loss_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    if (rows < 1 || cols < 1) fail(F2V_ERANGE, "logreg_loss: empty feature matrix");
    F2V_CUDA(cudaSetDevice(c.device));
    *loss_out = ev::logreg_loss(c, weights, features, rows, cols, targets, l2);
  });
}

int32_t f2v_build_link_dataset(uint32_t n, const uint64_t* row_offsets,
                               const uint32_t* col_indices, uint64_t* rng_state,
                               uint32_t** train_out, uint64_t* ntrain_out, uint32_t** test_out,
                               uint64_t* ntest_out) {
  return guard(nullptr, [&] {
    Stream rng{*rng_state};
    std::vector<Pair3> train, test;
    build_link_dataset(n, row_offsets, col_indices, rng, train, test);
    auto dup = [](const std::vector<Pair3>& v) {
      uint32_t* out = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, v.size()) * 12));
      if (!out) throw std::bad_alloc();
      std::memcpy(out, v.data(), v.size() * 12);
      return out;
    };
    static_assert(sizeof(Pair3) == 12, "u32 triples");
    *train_out = dup(train);
    *ntrain_out = train.size();
    *test_out = dup(test);
    *ntest_out = test.size();
  });
}

int32_t f2v_link_prediction_accuracy(f2v_ctx* h, const uint32_t* train, uint64_t ntrain,
                                     const uint32_t* test, uint64_t ntest, f2v_logreg_config cfg,
                                     double* accuracy_out, double* weights_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_eval_state(c, false);
    check_logreg(cfg);
    if (ntrain < 1) fail(F2V_ERANGE, "fit_logreg: target count mismatch");
    F2V_CUDA(cudaSetDevice(c.device));
    *accuracy_out = ev::link_accuracy(c, c.zcur(), c.d, train, ntrain, test, ntest, cfg.lr,
                                      cfg.iters, cfg.l2, weights_out);
  });
}

int32_t f2v_node_classification(f2v_ctx* h, const uint64_t* label_offsets,
                                const int32_t* label_ids, int32_t num_classes,
                                double train_fraction, uint64_t* rng_state,
                                f2v_logreg_config cfg, double* micro_f1_out,
                                double* macro_f1_out) {
  return guard(&h->c, [&] {
    Ctx& c = h->c;
    need_eval_state(c, false);
    check_logreg(cfg);
    F2V_CUDA(cudaSetDevice(c.device));
    Stream rng{*rng_state};
    double micro = 0.0, macro = 0.0;
    node_classification(c, label_offsets, label_ids, num_classes, train_fraction, rng, cfg, micro,
                        macro);
    *micro_f1_out = micro;
    *macro_f1_out = macro;
  });
}

}  // extern "C"
