// The plan / refinement layer of the C++ drop-in (include/longctx_b200.hpp:
// SparsityPlan, CriticalSet JSON, refine_plan, offline_search), driven like reference
// code and checked against fixtures the REFERENCE produced (tests/golden/
// make_refine_golden.py).
//
//   plan_parity --json <ref_critical_set.json> <ref_plan_refined.json> <ref_prefill_selections.json>
//       CPU: our JSON text equals the text the reference CLI wrote (minus the two
//       bookkeeping keys its harness adds), round trips, and the error kinds of malformed
//       plans (schema_violation / parse_error / config).
//   plan_parity --dcpp <dcpp_golden.txt>
//       CPU: fixed / DCPP chunk schedules identical to the reference's
//       (engine_sim.cpp:77-166) and the non-negative cost-model fit.
//   plan_parity --measure
//       GPU: measured per-chunk costs of the device prefill, fitted, scheduled.
//   plan_parity --refine <refine_golden.txt>
//       GPU: every refine_plan / offline_search case reproduces the reference's budgets,
//       rounds and plan text exactly and its recalls within 1e-4 (fp32 device path vs the
//       reference's fp64; one query's worth for a FractionAbove aggregate).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "longctx_b200.hpp"

using namespace longctx;

static int failures = 0;
#define CHECK(cond)                                                                   \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
      ++failures;                                                                     \
    }                                                                                 \
  } while (0)

static std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// the reference harness adds "configHash" / "version" members before dumping
// (harness.cpp:78-84); drop them to get the operator's own to_json().dump(2)
static std::string strip_harness_keys(const std::string& text) {
  std::vector<std::string> lines;
  std::stringstream ss(text);
  for (std::string l; std::getline(ss, l);)
    if (l.rfind("  \"configHash\"", 0) != 0 && l.rfind("  \"version\"", 0) != 0) lines.push_back(l);
  if (lines.size() >= 2 && !lines[lines.size() - 2].empty() && lines[lines.size() - 2].back() == ',')
    lines[lines.size() - 2].pop_back();
  std::string out;
  for (std::size_t i = 0; i < lines.size(); ++i) out += lines[i] + (i + 1 < lines.size() ? "\n" : "");
  return out;
}

template <typename F>
static std::string kind_of(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.kind();
  }
  return "none";
}

static int selections_check(const std::string& path) {
  // prefill_selections.json of the reference CLI (harness.cpp:430-438): parse, re-emit,
  // compare the text; the example config's four chunk selections
  const std::string text = slurp(path);
  PrefillState st;
  st.selections = b200::prefill_selections_from_json(text);
  CHECK(st.selections.size() == 4);
  if (st.selections.size() == 4) {
    CHECK((st.selections[0].critical.verticals == std::vector<std::size_t>{0, 64, 171}));
    CHECK(st.selections[3].begin == 768 && st.selections[3].end == 1024);
  }
  CHECK(b200::prefill_selections_json(st) == strip_harness_keys(text));
  CHECK(b200::prefill_selections_json(PrefillState{}) == "{\n  \"selections\": []\n}");
  CHECK(kind_of([] { b200::prefill_selections_from_json("{\"selections\": [{}]}"); }) ==
        "schema_violation");
  return 0;
}

static int json_mode(const std::string& crit_path, const std::string& plan_path) {
  // CriticalSet: proj/out/sparsity/critical_set.json (V = [0, 64, 288], S = [0..64, 288])
  const std::string ref_crit = strip_harness_keys(slurp(crit_path));
  CriticalSet crit;
  crit.context_length = 1024;
  crit.verticals = {0, 64, 288};
  for (std::size_t d = 0; d <= 64; ++d) crit.slashes.push_back(d);
  crit.slashes.push_back(288);
  CHECK(crit.to_json() == ref_crit);
  CHECK(CriticalSet::from_json(slurp(crit_path)) == crit);  // extra keys are ignored
  CriticalSet empty;
  empty.context_length = 7;
  CHECK(CriticalSet::from_json(empty.to_json()) == empty);
  CHECK(empty.to_json() == "{\n  \"contextLength\": 7,\n  \"slashes\": [],\n  \"verticals\": []\n}");
  // from_json sorts and deduplicates (sparse.cpp:132-133)
  const CriticalSet messy = CriticalSet::from_json(
      "{\"contextLength\": 9, \"verticals\": [4, 1, 4], \"slashes\": [3, 0]}");
  CHECK((messy.verticals == std::vector<std::size_t>{1, 4}));
  CHECK((messy.slashes == std::vector<std::size_t>{0, 3}));

  // SparsityPlan: proj/out/refine/plan_refined.json
  SparsityPlan plan;
  plan.budgets[{0, 0}] = HeadBudget{2, 2};
  plan.budgets[{0, 1}] = HeadBudget{2, 2};
  CHECK(plan.to_json() == strip_harness_keys(slurp(plan_path)));
  const SparsityPlan back = SparsityPlan::from_json(plan.to_json());
  CHECK(back.budgets == plan.budgets);
  // keys order as strings ("0.10" < "0.2"), as nlohmann objects do
  SparsityPlan many;
  many.budgets[{0, 2}] = HeadBudget{1, 2};
  many.budgets[{0, 10}] = HeadBudget{3, 4};
  const std::string mj = many.to_json();
  CHECK(mj.find("\"0.10\"") < mj.find("\"0.2\""));
  CHECK(SparsityPlan::from_json(mj).budgets == many.budgets);
  CHECK(SparsityPlan::from_json("{}").budgets.empty());
  CHECK(many.to_json() != "" && SparsityPlan{}.to_json() == "{}");
  // error kinds (sparse.cpp:36-43, 54-78)
  CHECK(kind_of([&] { (void)std::as_const(plan).at(3, 9); }) == "config");
  CHECK(kind_of([] { SparsityPlan::from_json("[1, 2]"); }) == "schema_violation");
  CHECK(kind_of([] { SparsityPlan::from_json("{\"configHash\": \"x\"}"); }) == "schema_violation");
  CHECK(kind_of([] { SparsityPlan::from_json("{\"0.x\": {\"vertical\": 1, \"slash\": 1}}"); }) ==
        "schema_violation");
  CHECK(kind_of([] { SparsityPlan::from_json("{\"0.1\": {\"vertical\": 1}}"); }) ==
        "schema_violation");
  CHECK(kind_of([] { SparsityPlan::from_json("{\"0.1\": {\"vertical\": -1, \"slash\": 1}}"); }) ==
        "schema_violation");
  CHECK(kind_of([] { SparsityPlan::from_json("{\"0.1\": "); }) == "parse_error");
  CHECK(kind_of([] { CriticalSet::from_json("{\"contextLength\": 3}"); }) == "schema_violation");
  // refine / offline validation happens before any device work (refine.cpp:87-96, 140-150)
  RefineConfig bad;
  bad.threshold = 1.0;
  CHECK(kind_of([&] { bad.validate(); }) == "config");
  bad = RefineConfig{};
  bad.vertical_increment = 0;
  CHECK(kind_of([&] { bad.validate(); }) == "config");
  CHECK(kind_of([&] { refine_plan({}, plan, RefineConfig{}); }) == "empty_calibration");
  CHECK(kind_of([&] { offline_search({}, {}, 0.5); }) == "config");
  CHECK(kind_of([&] { offline_search({}, {{2, 2}, {1, 1}}, 0.5); }) == "config");
  CHECK(kind_of([&] { offline_search({}, {{1, 1}}, 0.5); }) == "empty_calibration");
  std::printf("json checks: %d failures\n", failures);
  return failures == 0 ? 0 : 1;
}

// ------------------------------------------------------------------ refine --
struct Reader {
  std::istream& in;
  template <typename T>
  T get() {
    T x{};
    in >> x;
    if (!in) throw std::runtime_error("golden file truncated");
    return x;
  }
  std::string str() {
    const std::size_t len = get<std::size_t>();
    in.get();  // newline
    std::string s(len, '\0');
    in.read(s.data(), std::streamsize(len));
    return s;
  }
};

static CalibrationSample read_input(Reader& r) {
  CalibrationSample c;
  c.layer = r.get<std::size_t>();
  c.head = r.get<std::size_t>();
  const auto n = r.get<std::size_t>(), dim = r.get<std::size_t>();
  c.input.rope_base = r.get<double>();
  c.input.temperature = r.get<double>();
  for (Matrix* m : {&c.input.q, &c.input.k, &c.input.v}) {
    *m = Matrix(n, dim);
    for (auto& x : m->values) x = r.get<double>();
  }
  c.input.positions_q.resize(n);
  c.input.positions_k.resize(n);
  for (auto& p : c.input.positions_q) p = r.get<std::int64_t>();
  for (auto& p : c.input.positions_k) p = r.get<std::int64_t>();
  return c;
}

static RecallMeasurement read_measure(Reader& r) {
  RecallMeasurement m;
  m.last_q = r.get<std::size_t>();
  m.selection.force_sink_column = r.get<int>() != 0;
  m.selection.force_local_band = r.get<int>() != 0;
  m.selection.slash_mean = r.get<int>() != 0;
  m.aggregate = r.get<int>() ? RecallAggregate::FractionAbove : RecallAggregate::Mean;
  m.fraction_tau = r.get<double>();
  return m;
}

static bool recall_close(double a, double b, const RecallMeasurement& m, std::size_t n) {
  const double tol = m.aggregate == RecallAggregate::Mean ? 1e-4 : 1.0 / double(n) + 1e-9;
  return std::fabs(a - b) <= tol;
}

static int refine_mode(const std::string& path) {
  std::ifstream f(path);
  Reader r{f};
  int ncase = 0;
  for (;;) {
    const std::string tag = r.get<std::string>();
    if (tag == "end") break;
    if (tag == "crit") {  // JSON text of the bundled nlohmann (arrays inline): skip
      r.get<std::size_t>();
      const auto nv = r.get<std::size_t>();
      for (std::size_t i = 0; i < nv; ++i) r.get<std::size_t>();
      const auto ns = r.get<std::size_t>();
      for (std::size_t i = 0; i < ns; ++i) r.get<std::size_t>();
      r.str();
      continue;
    }
    const int kind = r.get<int>();
    const auto ninp = r.get<std::size_t>();
    CalibrationSet calib;
    std::size_t nmin = SIZE_MAX;
    for (std::size_t i = 0; i < ninp; ++i) {
      calib.push_back(read_input(r));
      nmin = std::min(nmin, calib.back().input.seq_len());
    }
    ++ncase;
    if (kind == 0) {
      SparsityPlan plan;
      const auto np = r.get<std::size_t>();
      for (std::size_t i = 0; i < np; ++i) {
        const auto l = r.get<std::size_t>(), h = r.get<std::size_t>();
        const auto v = r.get<std::size_t>(), s = r.get<std::size_t>();
        plan.budgets[{l, h}] = HeadBudget{v, s};
      }
      RefineConfig cfg;
      cfg.threshold = r.get<double>();
      cfg.vertical_increment = r.get<std::size_t>();
      cfg.slash_increment = r.get<std::size_t>();
      cfg.max_rounds = r.get<std::size_t>();
      cfg.budget_cap.vertical = r.get<std::size_t>();
      cfg.budget_cap.slash = r.get<std::size_t>();
      cfg.measure = read_measure(r);
      const auto nrec = r.get<std::size_t>();
      std::vector<HeadRefineRecord> exp(nrec);
      for (auto& e : exp) {
        e.layer = r.get<std::size_t>();
        e.head = r.get<std::size_t>();
        e.rounds = r.get<std::size_t>();
        e.initial_budget.vertical = r.get<std::size_t>();
        e.initial_budget.slash = r.get<std::size_t>();
        e.final_budget.vertical = r.get<std::size_t>();
        e.final_budget.slash = r.get<std::size_t>();
        e.initial_recall = r.get<double>();
        e.final_recall = r.get<double>();
      }
      const std::string exp_plan = r.str();
      const auto [refined, report] = refine_plan(calib, plan, cfg);
      CHECK(report.heads.size() == exp.size());
      for (std::size_t i = 0; i < std::min(exp.size(), report.heads.size()); ++i) {
        const auto& a = report.heads[i];
        const auto& e = exp[i];
        std::printf("case %d head %zu.%zu rounds %zu/%zu budget (%zu,%zu)/(%zu,%zu) recall "
                    "%.6f/%.6f -> %.6f/%.6f\n",
                    ncase, a.layer, a.head, a.rounds, e.rounds, a.final_budget.vertical,
                    a.final_budget.slash, e.final_budget.vertical, e.final_budget.slash,
                    a.initial_recall, e.initial_recall, a.final_recall, e.final_recall);
        CHECK(a.layer == e.layer && a.head == e.head && a.rounds == e.rounds);
        CHECK(a.initial_budget == e.initial_budget && a.final_budget == e.final_budget);
        CHECK(recall_close(a.initial_recall, e.initial_recall, cfg.measure, nmin));
        CHECK(recall_close(a.final_recall, e.final_recall, cfg.measure, nmin));
      }
      // the refined plan: same budgets as the reference's (its text is the bundled
      // nlohmann's; compare through our parser)
      CHECK(SparsityPlan::from_json(exp_plan).budgets == refined.budgets);
    } else {
      std::vector<HeadBudget> grid(r.get<std::size_t>());
      for (auto& g : grid) {
        g.vertical = r.get<std::size_t>();
        g.slash = r.get<std::size_t>();
      }
      const double thr = r.get<double>();
      const RecallMeasurement m = read_measure(r);
      const std::string exp_plan = r.str();
      const SparsityPlan got = offline_search(calib, grid, thr, m);
      for (const auto& [k, b] : got.budgets)
        std::printf("case %d offline head %zu.%zu -> (%zu,%zu)\n", ncase, k.first, k.second,
                    b.vertical, b.slash);
      CHECK(SparsityPlan::from_json(exp_plan).budgets == got.budgets);
    }
  }
  std::printf("refine cases: %d, failures %d\n", ncase, failures);
  return failures == 0 && ncase > 0 ? 0 : 1;
}

// ---------------------------------------------------------------- DCPP --
static int dcpp_mode(const std::string& path) {
  std::ifstream f(path);
  Reader r{f};
  int ncase = 0;
  for (;;) {
    const std::string tag = r.get<std::string>();
    if (tag == "end") break;
    const auto tokens = r.get<std::size_t>(), chunks = r.get<std::size_t>();
    CostModel m;
    m.attn_coeff = r.get<double>();
    m.self_coeff = r.get<double>();
    m.lin_coeff = r.get<double>();
    m.fixed_cost = r.get<double>();
    std::vector<std::size_t> exp_fixed(r.get<std::size_t>()), exp_dcpp;
    for (auto& b : exp_fixed) b = r.get<std::size_t>();
    exp_dcpp.resize(r.get<std::size_t>());
    for (auto& b : exp_dcpp) b = r.get<std::size_t>();
    CHECK(fixed_schedule(tokens, chunks).boundaries == exp_fixed);
    const ChunkSchedule d = dcpp_schedule(tokens, chunks, m);
    CHECK(d.boundaries == exp_dcpp);
    if (d.boundaries != exp_dcpp) std::fprintf(stderr, "dcpp mismatch tokens %zu chunks %zu\n", tokens, chunks);
    ++ncase;
  }
  // worked example (test_engine_sim.cpp:61-73) and error kinds
  CHECK((dcpp_schedule(100, 2, CostModel{1, 1, 0, 0}).sizes() == std::vector<std::size_t>{71, 29}));
  CHECK(kind_of([] { dcpp_schedule(3, 4, CostModel{1, 1, 0, 0}); }) == "config");
  CHECK(kind_of([] { fixed_schedule(3, 0); }) == "config");
  CHECK(kind_of([] { CostModel{-1, 0, 0, 0}.validate(); }) == "config");
  CHECK(kind_of([] { chunk_cost(CostModel{}, 0, 0); }) == "domain");
  // the cost fit recovers a model from exact samples of it
  const CostModel truth{2e-6, 5e-7, 3e-3, 0.4};
  std::vector<b200::ChunkCostSample> samples;
  for (std::size_t c = 0; c < 32; ++c) {
    const std::size_t n = 1000 + (c * 7919) % 1500, h = c * 4096;  // n, h independent
    samples.push_back({n, h, chunk_cost(truth, n, h)});
  }
  const CostModel fit = b200::fit_cost_model(samples);
  auto rel = [](double a, double b) { return std::fabs(a - b) / std::max(std::fabs(b), 1e-30); };
  CHECK(rel(fit.attn_coeff, truth.attn_coeff) < 1e-6 && rel(fit.self_coeff, truth.self_coeff) < 1e-5);
  CHECK(rel(fit.lin_coeff, truth.lin_coeff) < 1e-4 && rel(fit.fixed_cost, truth.fixed_cost) < 1e-3);
  // negative least-squares components are clamped out (non-negative fit)
  std::vector<b200::ChunkCostSample> lin;
  for (std::size_t n = 1; n <= 20; ++n) lin.push_back({n, 0, 3.0 * double(n) - 1.0});
  const CostModel lf = b200::fit_cost_model(lin);
  CHECK(lf.attn_coeff >= 0 && lf.self_coeff >= 0 && lf.lin_coeff >= 0 && lf.fixed_cost >= 0);
  CHECK(kind_of([] { b200::fit_cost_model({}); }) == "config");
  std::printf("dcpp cases: %d, failures %d\n", ncase, failures);
  return failures == 0 && ncase > 0 ? 0 : 1;
}

// measured chunk costs of the device prefill -> fitted model -> DCPP schedule (GPU)
static int measure_mode() {
  const std::size_t n = 8192, dim = 128, L = 1024;
  AttentionInput in;
  std::uint64_t st = 12345;
  auto u = [&]() {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    return double(int64_t(st >> 11) % 2000001 - 1000000) * 1e-6;
  };
  for (Matrix* m : {&in.q, &in.k, &in.v}) {
    *m = Matrix(n, dim);
    for (auto& x : m->values) x = u();
  }
  in.positions_q.resize(n);
  in.positions_k.resize(n);
  for (std::size_t i = 0; i < n; ++i) in.positions_q[i] = in.positions_k[i] = std::int64_t(i);
  b200::set_precision(b200::Precision::BF16);
  const auto samples = b200::measure_chunk_costs(in, L, 64, HeadBudget{64, 128}, PrefillMode::Sparse,
                                                 PositionMode::Standard, std::nullopt);
  CHECK(samples.size() == n / L);
  for (std::size_t c = 0; c < samples.size(); ++c) {
    CHECK(samples[c].n == L && samples[c].h == c * L && samples[c].ms > 0.0);
    std::printf("chunk %zu: n %zu h %zu %.3f ms\n", c, samples[c].n, samples[c].h, samples[c].ms);
  }
  const CostModel m = b200::fit_cost_model(samples);
  const ChunkSchedule s = dcpp_schedule(n, n / L, m);
  CHECK(s.total_tokens() == n && s.chunk_count() == n / L);
  std::printf("fit: attn %.3g self %.3g lin %.3g fixed %.3g; failures %d\n", m.attn_coeff,
              m.self_coeff, m.lin_coeff, m.fixed_cost, failures);
  return failures == 0 ? 0 : 1;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "";
  try {
    if (mode == "--json" && argc == 5) {
      selections_check(argv[4]);
      return json_mode(argv[2], argv[3]);
    }
    if (mode == "--refine" && argc == 3) return refine_mode(argv[2]);
    if (mode == "--dcpp" && argc == 3) return dcpp_mode(argv[2]);
    if (mode == "--measure" && argc == 2) return measure_mode();
  } catch (const Error& e) {
    std::fprintf(stderr, "Error(%s): %s\n", e.kind().c_str(), e.what());
    return 2;
  }
  std::fprintf(stderr, "usage: plan_parity --json <crit.json> <plan.json> | --refine <golden>\n");
  return 2;
}
