// Drives the C++ drop-in (include/longctx_b200.hpp) exactly as reference code would,
// with the reference's types and calls, and dumps the results for tests/test_cpp_dropin.py
// to compare against the oracle.
//
//   dropin_parity --errors              error-kind contract (no device needed)
//   dropin_parity <in.bin> <out.bin>    compute on the GPU
//
// in.bin: int64 n, dim, s, c, w, chunk_len, last_q, bv, bs, precision(0 f32 / 1 bf16);
//         double temperature; then q, k, v as n x dim doubles.
// out.bin: a sequence of (int64 count, double values[count]) records in the order
//          written below.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "longctx_b200.hpp"

using namespace longctx;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <typename F>
static std::string kind_of(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.kind();
  }
  return "none";
}

static AttentionInput small_input(std::size_t n, std::size_t dim) {
  AttentionInput in;
  in.q = Matrix(n, dim);
  in.k = Matrix(n, dim);
  in.v = Matrix(n, dim);
  for (std::size_t i = 0; i < n * dim; ++i) {
    in.q.values[i] = 0.01 * double(i % 7);
    in.k.values[i] = 0.02 * double(i % 5);
    in.v.values[i] = 0.03 * double(i % 3);
  }
  in.positions_q.resize(n);
  in.positions_k.resize(n);
  for (std::size_t i = 0; i < n; ++i) in.positions_q[i] = in.positions_k[i] = std::int64_t(i);
  return in;
}

static int errors_mode() {
  // host-side validation: same kinds as the reference (errors.hpp:21-32), thrown before any
  // device work
  AttentionInput in = small_input(8, 4);
  AttentionInput bad = in;
  bad.k = Matrix(7, 4);
  CHECK(kind_of([&] { bad.validate(); }) == "dimension");
  bad = in;
  bad.q = Matrix(8, 3);
  bad.k = Matrix(8, 3);
  bad.v = Matrix(8, 3);
  CHECK(kind_of([&] { bad.validate(); }) == "config");
  bad = in;
  bad.positions_q[2] = -1;
  CHECK(kind_of([&] { bad.validate(); }) == "domain");
  bad = in;
  bad.temperature = 0.0;
  CHECK(kind_of([&] { bad.validate(); }) == "domain");
  bad = in;
  bad.q.values[3] = std::nan("");
  CHECK(kind_of([&] { bad.validate(); }) == "domain");
  CHECK(kind_of([&] { chunked_prefill(in, 0, 4, {1, 1}, PrefillMode::Sparse,
                                      PositionMode::Standard, std::nullopt); }) == "config");
  CHECK(kind_of([&] { chunked_prefill(in, 2, 4, {1, 1}, PrefillMode::Sparse,
                                      PositionMode::Standard, std::nullopt); }) == "config");
  CHECK(kind_of([&] { chunked_prefill(in, 4, 4, {1, 1}, PrefillMode::Sparse,
                                      PositionMode::DcaContinuous, std::nullopt); }) == "config");
  CHECK(kind_of([&] { estimate_block(in.q, in.k, 0, PositionMode::Standard, std::nullopt); }) ==
        "config");
  CHECK(kind_of([&] { estimate_block(Matrix(9, 4), in.k, 4, PositionMode::Standard,
                                     std::nullopt); }) == "dimension");
  CHECK(kind_of([&] { select_critical(Matrix(2, 5), {1, 1}, 6); }) == "dimension");
  CriticalSet crit{{0}, {0}, 7};
  CHECK(kind_of([&] { sparse_attention(in, crit); }) == "dimension");
  CHECK(kind_of([&] { classify_pair(1, 2, ChunkConfig{4, 8, 4}); }) == "causality");
  CHECK(kind_of([&] { ChunkConfig{0, 8, 0}.validate(); }) == "config");
  CHECK(kind_of([&] { ChunkConfig{6, 8, 4}.validate(); }) == "config");
  CHECK(kind_of([&] { yarn_temperature(0.0); }) == "domain");
  CHECK(kind_of([&] { flop_estimate(4, 8, 11); }) == "domain");
  CHECK(kind_of([&] { check_gqa_grouping(28, 3); }) == "config");
  CHECK(kind_of([&] { attention_recall(std::vector<double>{1.0}, std::vector<double>{}); }) ==
        "dimension");
  // host integer helpers (dca.cpp:62-80 hand values, test_dca.cpp)
  const ChunkConfig cfg{4, 10, 4};
  CHECK(dca_relative(7, 5, cfg) == 2);
  CHECK(dca_relative(13, 0, cfg) == 9);
  CHECK(dca_relative(11, 2, cfg) == 7);
  CHECK(selection_position(30, 2, cfg) == 9);
  CHECK(std::abs(yarn_temperature(4.0) - 0.771321) < 1e-6);
  CHECK(flop_estimate(4, 8, 10) == 160.0);
  // density worked example: forced-only selection at n = 4 (sparse.cpp:286-291)
  CriticalSet c4{{0}, {0}, 4};
  CHECK(c4.admitted_row(3) == (std::vector<std::size_t>{0, 3}));
  CHECK(c4.admitted_count() == 7);
  CHECK(std::abs(density(c4) - 0.7) < 1e-15);
  CriticalSet e{{}, {}, 3};
  CHECK(e.admitted_row(2) == std::vector<std::size_t>{2});  // self fallback
  // no device -> loud failure, never a CPU fallback
  if (std::getenv("LCX_EXPECT_NO_GPU")) {
    CHECK(kind_of([&] { full_attention(in); }) == "cuda");
  }
  std::printf("errors: %d failures\n", failures);
  return failures ? 1 : 0;
}

static void put(std::ofstream& o, const std::vector<double>& v) {
  const std::int64_t n = std::int64_t(v.size());
  o.write(reinterpret_cast<const char*>(&n), 8);
  o.write(reinterpret_cast<const char*>(v.data()), std::streamsize(8 * v.size()));
}
static std::vector<double> idx(const std::vector<std::size_t>& v) {
  return std::vector<double>(v.begin(), v.end());
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "--errors") return errors_mode();
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s --errors | <in.bin> <out.bin>\n", argv[0]);
    return 2;
  }
  std::ifstream f(argv[1], std::ios::binary);
  std::int64_t hdr[10];
  double temp;
  f.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
  f.read(reinterpret_cast<char*>(&temp), 8);
  const std::size_t n = std::size_t(hdr[0]), dim = std::size_t(hdr[1]);
  AttentionInput in;
  in.q = Matrix(n, dim);
  in.k = Matrix(n, dim);
  in.v = Matrix(n, dim);
  f.read(reinterpret_cast<char*>(in.q.values.data()), std::streamsize(8 * n * dim));
  f.read(reinterpret_cast<char*>(in.k.values.data()), std::streamsize(8 * n * dim));
  f.read(reinterpret_cast<char*>(in.v.values.data()), std::streamsize(8 * n * dim));
  in.positions_q.resize(n);
  in.positions_k.resize(n);
  for (std::size_t i = 0; i < n; ++i) in.positions_q[i] = in.positions_k[i] = std::int64_t(i);
  in.temperature = temp;
  b200::set_precision(hdr[9] ? b200::Precision::BF16 : b200::Precision::F32);
  const ChunkConfig cfg{std::size_t(hdr[2]), std::size_t(hdr[3]), std::size_t(hdr[4])};
  const HeadBudget budget{std::size_t(hdr[7]), std::size_t(hdr[8])};
  std::ofstream o(argv[2], std::ios::binary);
  // 1. the operator, sparse + DCA-continuous selection
  const PrefillResult pr = chunked_prefill(in, std::size_t(hdr[5]), std::size_t(hdr[6]), budget,
                                           PrefillMode::Sparse, PositionMode::DcaContinuous, cfg);
  put(o, pr.result.output.values);
  put(o, pr.result.lse);
  put(o, {double(pr.state.selections.size())});
  for (const auto& s : pr.state.selections) {
    put(o, idx(s.critical.verticals));
    put(o, idx(s.critical.slashes));
  }
  CHECK(pr.state.cached_k == in.k);
  // 2. one-shot estimate + select + sparse attention (standard positions)
  const Matrix est = estimate_block(in.q, in.k, std::size_t(hdr[6]), PositionMode::Standard,
                                    std::nullopt, in.rope_base);
  put(o, est.values);
  const CriticalSet crit = select_critical(est, budget, n);
  put(o, idx(crit.verticals));
  put(o, idx(crit.slashes));
  const AttentionResult sp = sparse_attention(in, crit);
  put(o, sp.output.values);
  put(o, sp.lse);
  // 3. dense, DCA dense, and the explicit RelPositionMatrix override of the same remap
  const AttentionResult fa = full_attention(in);
  put(o, fa.output.values);
  put(o, fa.lse);
  const AttentionResult da = dca_attention(in, cfg, YarnScale::from_scale(2.0));
  put(o, da.output.values);
  put(o, da.lse);
  AttentionInput t = in;
  t.temperature = YarnScale::from_scale(2.0).temperature;
  const RelPositionMatrix rel = dca_position_matrix(n, cfg);
  const AttentionResult ra = full_attention(t, &rel);
  put(o, ra.output.values);
  // 3b. sparse attention under the explicit override (harness.cpp:399, DCA sparsity check),
  //     once with the selection above and once with lines that leave the first rows empty
  //     (self fallback, sparse.cpp:111)
  const AttentionResult rs = sparse_attention(t, crit, &rel);
  put(o, rs.output.values);
  put(o, rs.lse);
  const CriticalSet late{{5}, {3}, n};
  const AttentionResult rf = sparse_attention(t, late, &rel);
  put(o, rf.output.values);
  put(o, rf.lse);
  // 4. recall
  put(o, {measure_budget_recall(in, budget, RecallMeasurement{})});
  o.close();
  std::printf("dropin: %d failures\n", failures);
  return failures ? 1 : 0;
}
