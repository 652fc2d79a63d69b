// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (/root/reference/proj/core/src/*.cpp, compiled in place by
// oracle/Makefile into oracle/_ref/liblongctx_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (oracle/longctx_oracle.c) and the CUDA path against the reference itself,
// and by bench.py's cpu_baseline / --impl reference legs to time the
// reference CPU path on the box's host cores.  Nothing here is product code.
//
// Error convention: return 0 on success, else the errkind index below
// (errors.hpp:21-32), with the message retrievable by ref_last_error().

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <optional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "longctx/attention.hpp"
#include "longctx/config.hpp"
#include "longctx/dca.hpp"
#include "longctx/errors.hpp"
#include "longctx/planted.hpp"
#include "longctx/refine.hpp"
#include "longctx/sparse.hpp"

using namespace longctx;

namespace {

thread_local std::string g_err;

int kind_code(const std::string& k) {
  static const char* kinds[] = {"",          "dimension", "config",    "domain",
                                "causality", "empty_row", "empty_calibration"};
  for (int i = 1; i < 7; ++i)
    if (k == kinds[i]) return i;
  return 50;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return kind_code(e.kind());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 98;
  }
}

Matrix to_matrix(const double* p, int64_t rows, int64_t cols) {
  Matrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  std::memcpy(m.values.data(), p, sizeof(double) * static_cast<std::size_t>(rows * cols));
  return m;
}

AttentionInput to_input(const double* q, const double* k, const double* v, int64_t n,
                        int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                        double rope_base, double temperature) {
  AttentionInput in;
  in.q = to_matrix(q, n, dim);
  in.k = to_matrix(k, n, dim);
  in.v = to_matrix(v, n, dim);
  in.positions_q.resize(static_cast<std::size_t>(n));
  in.positions_k.resize(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    in.positions_q[i] = pos_q ? pos_q[i] : i;
    in.positions_k[i] = pos_k ? pos_k[i] : i;
  }
  in.rope_base = rope_base;
  in.temperature = temperature;
  return in;
}

CriticalSet to_crit(const int64_t* verts, int64_t nv, const int64_t* slashes, int64_t ns,
                    int64_t n) {
  CriticalSet c;
  c.context_length = static_cast<std::size_t>(n);
  for (int64_t a = 0; a < nv; ++a) c.verticals.push_back(static_cast<std::size_t>(verts[a]));
  for (int64_t a = 0; a < ns; ++a) c.slashes.push_back(static_cast<std::size_t>(slashes[a]));
  return c;
}

void put_result(const AttentionResult& r, double* out, double* lse) {
  std::memcpy(out, r.output.values.data(), sizeof(double) * r.output.values.size());
  std::memcpy(lse, r.lse.data(), sizeof(double) * r.lse.size());
}

std::optional<ChunkConfig> chunk_opt(int use, int64_t s, int64_t c, int64_t w) {
  if (!use) return std::nullopt;
  ChunkConfig cfg;
  cfg.chunk_size = static_cast<std::size_t>(s);
  cfg.train_len = static_cast<std::size_t>(c);
  cfg.local_window = static_cast<std::size_t>(w);
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_estimate_block(const double* q, int64_t nq, const double* k, int64_t nk, int64_t dim,
                       int64_t last_q, int pos_mode, int64_t s, int64_t c, int64_t w,
                       double rope_base, double* est_out) {
  return guarded([&] {
    const Matrix est = estimate_block(
        to_matrix(q, nq, dim), to_matrix(k, nk, dim), static_cast<std::size_t>(last_q),
        pos_mode ? PositionMode::DcaContinuous : PositionMode::Standard,
        chunk_opt(pos_mode, s, c, w), rope_base);
    std::memcpy(est_out, est.values.data(), sizeof(double) * est.values.size());
  });
}

int ref_select_critical(const double* est, int64_t rows, int64_t n, int64_t budget_v,
                        int64_t budget_s, int force_sink, int force_band, int slash_mean,
                        int64_t* out_v, int64_t cap_v, int64_t* nv, int64_t* out_s,
                        int64_t cap_s, int64_t* ns) {
  return guarded([&] {
    SelectionOptions opts{force_sink != 0, force_band != 0, slash_mean != 0};
    const CriticalSet crit = select_critical(
        to_matrix(est, rows, n),
        HeadBudget{static_cast<std::size_t>(budget_v), static_cast<std::size_t>(budget_s)},
        static_cast<std::size_t>(n), opts);
    *nv = static_cast<int64_t>(crit.verticals.size());
    *ns = static_cast<int64_t>(crit.slashes.size());
    for (int64_t a = 0; a < *nv && a < cap_v; ++a) out_v[a] = crit.verticals[a];
    for (int64_t a = 0; a < *ns && a < cap_s; ++a) out_s[a] = crit.slashes[a];
  });
}

int ref_admitted_count(const int64_t* verts, int64_t nv, const int64_t* slashes, int64_t ns,
                       int64_t n, int64_t* count, double* dens) {
  return guarded([&] {
    const CriticalSet crit = to_crit(verts, nv, slashes, ns, n);
    *count = static_cast<int64_t>(crit.admitted_count());
    *dens = density(crit);
  });
}

int ref_sparse_attention(const double* q, const double* k, const double* v, int64_t n,
                         int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                         double rope_base, double temperature, const int64_t* verts, int64_t nv,
                         const int64_t* slashes, int64_t ns, int use_dca, int64_t s, int64_t c,
                         int64_t w, double* out, double* lse) {
  return guarded([&] {
    const AttentionInput in = to_input(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature);
    const CriticalSet crit = to_crit(verts, nv, slashes, ns, n);
    if (use_dca) {
      const RelPositionMatrix rel =
          dca_position_matrix(static_cast<std::size_t>(n), *chunk_opt(1, s, c, w));
      put_result(sparse_attention(in, crit, &rel), out, lse);
    } else {
      put_result(sparse_attention(in, crit), out, lse);
    }
  });
}

int ref_full_attention(const double* q, const double* k, const double* v, int64_t n, int64_t dim,
                       const int64_t* pos_q, const int64_t* pos_k, double rope_base,
                       double temperature, int use_dca, int64_t s, int64_t c, int64_t w,
                       double* out, double* lse) {
  return guarded([&] {
    const AttentionInput in = to_input(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature);
    if (use_dca) {
      const RelPositionMatrix rel =
          dca_position_matrix(static_cast<std::size_t>(n), *chunk_opt(1, s, c, w));
      put_result(full_attention(in, &rel), out, lse);
    } else {
      put_result(full_attention(in), out, lse);
    }
  });
}

int ref_dca_attention(const double* q, const double* k, const double* v, int64_t n, int64_t dim,
                      double rope_base, int64_t s, int64_t c, int64_t w, double scale_factor,
                      double* out, double* lse) {
  return guarded([&] {
    const AttentionInput in = to_input(q, k, v, n, dim, nullptr, nullptr, rope_base, 1.0);
    put_result(dca_attention(in, *chunk_opt(1, s, c, w), YarnScale::from_scale(scale_factor)),
               out, lse);
  });
}

double ref_yarn_temperature(double scale) { return yarn_temperature(scale); }

int64_t ref_dca_relative(int64_t i, int64_t j, int64_t s, int64_t c, int64_t w) {
  return dca_relative(static_cast<std::size_t>(i), static_cast<std::size_t>(j),
                      *chunk_opt(1, s, c, w));
}

int ref_chunked_prefill(const double* q, const double* k, const double* v, int64_t n,
                        int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                        double rope_base, double temperature, int64_t chunk_len, int64_t last_q,
                        int64_t budget_v, int64_t budget_s, int mode, int pos_mode, int64_t s,
                        int64_t c, int64_t w, int force_sink, int force_band, int slash_mean,
                        double* out, double* lse, int64_t* sel_v, int64_t* sel_nv,
                        int64_t cap_v, int64_t* sel_s, int64_t* sel_ns, int64_t cap_s) {
  return guarded([&] {
    const AttentionInput in = to_input(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature);
    SelectionOptions opts{force_sink != 0, force_band != 0, slash_mean != 0};
    const PrefillResult pr = chunked_prefill(
        in, static_cast<std::size_t>(chunk_len), static_cast<std::size_t>(last_q),
        HeadBudget{static_cast<std::size_t>(budget_v), static_cast<std::size_t>(budget_s)},
        mode ? PrefillMode::Sparse : PrefillMode::Full,
        pos_mode ? PositionMode::DcaContinuous : PositionMode::Standard,
        chunk_opt(pos_mode, s, c, w), opts);
    put_result(pr.result, out, lse);
    if (sel_nv) {
      for (std::size_t ci = 0; ci < pr.state.selections.size(); ++ci) {
        const CriticalSet& cr = pr.state.selections[ci].critical;
        sel_nv[ci] = static_cast<int64_t>(cr.verticals.size());
        sel_ns[ci] = static_cast<int64_t>(cr.slashes.size());
        for (std::size_t a = 0; a < cr.verticals.size() && int64_t(a) < cap_v; ++a)
          sel_v[ci * cap_v + a] = cr.verticals[a];
        for (std::size_t a = 0; a < cr.slashes.size() && int64_t(a) < cap_s; ++a)
          sel_s[ci * cap_s + a] = cr.slashes[a];
      }
    }
  });
}

int ref_attention_recall(const double* lse_s, const double* lse_f, int64_t n, double* per_query,
                         double* aggregate) {
  return guarded([&] {
    const RecallReport r = attention_recall(std::span<const double>(lse_s, n),
                                            std::span<const double>(lse_f, n));
    std::memcpy(per_query, r.per_query.data(), sizeof(double) * r.per_query.size());
    *aggregate = r.aggregate;
  });
}

int ref_measure_budget_recall(const double* q, const double* k, const double* v, int64_t n,
                              int64_t dim, double rope_base, int64_t budget_v, int64_t budget_s,
                              int64_t last_q, int force_sink, int force_band, int slash_mean,
                              int fraction_above, double tau, double* value) {
  return guarded([&] {
    const AttentionInput in = to_input(q, k, v, n, dim, nullptr, nullptr, rope_base, 1.0);
    RecallMeasurement m;
    m.last_q = static_cast<std::size_t>(last_q);
    m.selection = SelectionOptions{force_sink != 0, force_band != 0, slash_mean != 0};
    m.aggregate = fraction_above ? RecallAggregate::FractionAbove : RecallAggregate::Mean;
    m.fraction_tau = tau;
    *value = measure_budget_recall(
        in, HeadBudget{static_cast<std::size_t>(budget_v), static_cast<std::size_t>(budget_s)},
        m);
  });
}

int ref_make_planted(int64_t n, int64_t dim, double rope_base, const int64_t* vcols, int64_t nvc,
                     const int64_t* soffs, int64_t nso, double strength, double vstrength,
                     double sstrength, double query_noise, double shared_scale, uint64_t seed,
                     int use_dca, int64_t s, int64_t c, int64_t w, const int64_t* carrier_pairs,
                     int64_t ncp, double* q, double* k, double* v) {
  return guarded([&] {
    PlantedSpec spec;
    spec.n = static_cast<std::size_t>(n);
    spec.head_dim = static_cast<std::size_t>(dim);
    spec.rope_base = rope_base;
    for (int64_t a = 0; a < nvc; ++a) spec.vertical_columns.push_back(vcols[a]);
    for (int64_t a = 0; a < nso; ++a) spec.slash_offsets.push_back(soffs[a]);
    spec.strength = strength;
    spec.vertical_strength = vstrength;
    spec.slash_strength = sstrength;
    spec.query_noise = query_noise;
    spec.shared_scale = shared_scale;
    spec.seed = seed;
    spec.dca = chunk_opt(use_dca, s, c, w);
    for (int64_t a = 0; a < ncp; ++a) spec.carrier_pairs.push_back(carrier_pairs[a]);
    const AttentionInput in = make_planted_input(spec);
    std::memcpy(q, in.q.values.data(), sizeof(double) * in.q.values.size());
    std::memcpy(k, in.k.values.data(), sizeof(double) * in.k.values.size());
    std::memcpy(v, in.v.values.data(), sizeof(double) * in.v.values.size());
  });
}

// testutil.hpp:18-41 recipe (q, k, v uniform(-1, 1) from one mt19937_64), via libstdc++.
void ref_random_input(uint64_t seed, int64_t n, int64_t dim, double* q, double* k, double* v) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uniform(-1.0, 1.0);
  for (int64_t i = 0; i < n * dim; ++i) q[i] = uniform(rng);
  for (int64_t i = 0; i < n * dim; ++i) k[i] = uniform(rng);
  for (int64_t i = 0; i < n * dim; ++i) v[i] = uniform(rng);
}

uint64_t ref_module_seed(uint64_t run_seed, const char* name) { return module_seed(run_seed, name); }

// Reference-side multi-head chunked sparse prefill over [n][H][D] inputs (the
// layout the CUDA path uses), heads distributed over `threads` std::threads
// (concurrent calls on distinct inputs are allowed).  Used by
// bench.py to time the reference CPU path.  GQA: query head h reads kv head
// h / (hq / hkv).  Inputs are float32 (converted to fp64 per head).
int ref_prefill_multihead(const float* q, const float* k, const float* v, int64_t n, int64_t hq,
                          int64_t hkv, int64_t dim, double rope_base, double temperature,
                          int64_t chunk_len, int64_t last_q, int64_t budget_v, int64_t budget_s,
                          int pos_mode, int64_t s, int64_t c, int64_t w, int64_t head_count,
                          int threads, float* out, float* lse) {
  std::atomic<int64_t> next{0};
  std::atomic<int> status{0};
  auto worker = [&] {
    for (;;) {
      const int64_t h = next.fetch_add(1);
      if (h >= head_count) break;
      const int64_t g = h / (hq / hkv);
      std::vector<double> qh(n * dim), kh(n * dim), vh(n * dim);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t d = 0; d < dim; ++d) {
          qh[i * dim + d] = q[(i * hq + h) * dim + d];
          kh[i * dim + d] = k[(i * hkv + g) * dim + d];
          vh[i * dim + d] = v[(i * hkv + g) * dim + d];
        }
      std::vector<double> o(n * dim), l(n);
      const int st = ref_chunked_prefill(qh.data(), kh.data(), vh.data(), n, dim, nullptr,
                                         nullptr, rope_base, temperature, chunk_len, last_q,
                                         budget_v, budget_s, 1, pos_mode, s, c, w, 1, 1, 1,
                                         o.data(), l.data(), nullptr, nullptr, 0, nullptr,
                                         nullptr, 0);
      if (st) status = st;
      if (out)
        for (int64_t i = 0; i < n; ++i)
          for (int64_t d = 0; d < dim; ++d) out[(i * hq + h) * dim + d] = float(o[i * dim + d]);
      if (lse)
        for (int64_t i = 0; i < n; ++i) lse[h * n + i] = float(l[i]);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  return status.load();
}

}  // extern "C"
