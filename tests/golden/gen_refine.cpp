// Golden fixture generator for the plan / refinement layer,
// driven by the REFERENCE library itself.  Test infrastructure: compiled and run only
// here (where /root/reference exists) by tests/golden/make_refine_golden.py; the GPU box
// only reads the committed tests/golden/refine_golden.txt.
//
// Cases follow the reference's own refinement tests (proj/tests/test_refine.cpp:80-200):
// planted columns that need budget growth, converged heads, a diffuse head capped,
// several heads of one layer, an offline grid search; plus CriticalSet / SparsityPlan
// JSON text exactly as the reference serialises it (nlohmann dump(2)).
//
// Output: a whitespace-separated text stream (read by tests/cpp/plan_parity.cpp):
//   "case" kind(0 refine / 1 offline) ninputs
//     per input: layer head n dim rope_base temperature q[n*dim] k[...] v[...] pq[n] pk[n]
//     refine : nplan (layer head v s)*; threshold vinc sinc rounds capv caps
//     offline: ngrid (v s)*; threshold
//     measure: last_q sink band mean aggregate tau
//     expected refine : nrec (layer head rounds iv is fv fs ir fr)*; plan json (length-prefixed)
//     expected offline: plan json (length-prefixed)
//   "crit" n nv v* ns s* json(length-prefixed)
//   "end"
#include <cstdio>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "longctx/engine_sim.hpp"
#include "longctx/planted.hpp"
#include "longctx/refine.hpp"
#include "longctx/sparse.hpp"

using namespace longctx;

static void put_str(std::ostream& o, const std::string& s) { o << s.size() << "\n" << s << "\n"; }

static void put_input(std::ostream& o, const CalibrationSample& c) {
  const AttentionInput& in = c.input;
  char buf[64];
  o << c.layer << " " << c.head << " " << in.q.rows << " " << in.q.cols << " ";
  std::snprintf(buf, sizeof buf, "%.17g %.17g", in.rope_base, in.temperature);
  o << buf << "\n";
  for (const Matrix* m : {&in.q, &in.k, &in.v}) {
    for (double x : m->values) {
      std::snprintf(buf, sizeof buf, "%.17g", x);
      o << buf << " ";
    }
    o << "\n";
  }
  for (auto p : in.positions_q) o << p << " ";
  o << "\n";
  for (auto p : in.positions_k) o << p << " ";
  o << "\n";
}

static void put_measure(std::ostream& o, const RecallMeasurement& m) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", m.fraction_tau);
  o << m.last_q << " " << int(m.selection.force_sink_column) << " "
    << int(m.selection.force_local_band) << " " << int(m.selection.slash_mean) << " "
    << int(m.aggregate == RecallAggregate::FractionAbove) << " " << buf << "\n";
}

static AttentionInput random_input(std::mt19937_64& rng, std::size_t n, std::size_t dim) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  AttentionInput in;
  for (Matrix* m : {&in.q, &in.k, &in.v}) {
    *m = Matrix(n, dim);
    for (auto& x : m->values) x = u(rng);
  }
  in.positions_q.resize(n);
  in.positions_k.resize(n);
  for (std::size_t i = 0; i < n; ++i) in.positions_q[i] = in.positions_k[i] = std::int64_t(i);
  return in;
}

static AttentionInput planted(std::size_t n, std::size_t dim, double strength, double qnoise,
                              std::uint64_t seed, std::vector<std::size_t> cols,
                              std::vector<std::size_t> slashes) {
  PlantedSpec spec;
  spec.n = n;
  spec.head_dim = dim;
  spec.strength = strength;
  spec.query_noise = qnoise;
  spec.seed = seed;
  spec.vertical_columns = std::move(cols);
  spec.slash_offsets = std::move(slashes);
  return make_planted_input(spec);
}

static RefineConfig basic_config() {  // test_refine.cpp:17-27
  RefineConfig cfg;
  cfg.threshold = 0.9;
  cfg.vertical_increment = 1;
  cfg.slash_increment = 1;
  cfg.max_rounds = 8;
  cfg.budget_cap = HeadBudget{16, 16};
  cfg.measure.last_q = 32;
  return cfg;
}

static void refine_case(std::ostream& o, const CalibrationSet& calib, const SparsityPlan& plan,
                        const RefineConfig& cfg) {
  char buf[64];
  o << "case 0 " << calib.size() << "\n";
  for (const auto& c : calib) put_input(o, c);
  o << plan.budgets.size() << "\n";
  for (const auto& [k, b] : plan.budgets)
    o << k.first << " " << k.second << " " << b.vertical << " " << b.slash << "\n";
  std::snprintf(buf, sizeof buf, "%.17g", cfg.threshold);
  o << buf << " " << cfg.vertical_increment << " " << cfg.slash_increment << " " << cfg.max_rounds
    << " " << cfg.budget_cap.vertical << " " << cfg.budget_cap.slash << "\n";
  put_measure(o, cfg.measure);
  const auto [refined, report] = refine_plan(calib, plan, cfg);
  o << report.heads.size() << "\n";
  for (const auto& r : report.heads) {
    char b2[96];
    std::snprintf(b2, sizeof b2, "%.17g %.17g", r.initial_recall, r.final_recall);
    o << r.layer << " " << r.head << " " << r.rounds << " " << r.initial_budget.vertical << " "
      << r.initial_budget.slash << " " << r.final_budget.vertical << " " << r.final_budget.slash
      << " " << b2 << "\n";
  }
  put_str(o, refined.to_json().dump(2));
}

static void offline_case(std::ostream& o, const CalibrationSet& calib,
                         const std::vector<HeadBudget>& grid, double threshold,
                         const RecallMeasurement& m) {
  char buf[64];
  o << "case 1 " << calib.size() << "\n";
  for (const auto& c : calib) put_input(o, c);
  o << grid.size() << "\n";
  for (const auto& g : grid) o << g.vertical << " " << g.slash << "\n";
  std::snprintf(buf, sizeof buf, "%.17g", threshold);
  o << buf << "\n";
  put_measure(o, m);
  put_str(o, offline_search(calib, grid, threshold, m).to_json().dump(2));
}

// DCPP chunk sizing (engine_sim.cpp:117-166): "dcpp tokens chunks a s l f" then the
// fixed and the DCPP boundaries, one line each ("count b0 b1 ...")
static int dcpp_main() {
  std::ostream& o = std::cout;
  char buf[128];
  auto emit = [&](std::size_t tokens, std::size_t chunks, const CostModel& m) {
    std::snprintf(buf, sizeof buf, "%.17g %.17g %.17g %.17g", m.attn_coeff, m.self_coeff,
                  m.lin_coeff, m.fixed_cost);
    o << "dcpp " << tokens << " " << chunks << " " << buf << "\n";
    for (const ChunkSchedule& s : {fixed_schedule(tokens, chunks), dcpp_schedule(tokens, chunks, m)}) {
      o << s.boundaries.size();
      for (auto b : s.boundaries) o << " " << b;
      o << "\n";
    }
  };
  emit(100, 2, CostModel{1.0, 1.0, 0.0, 0.0});  // test_engine_sim.cpp:61-73
  emit(57, 1, CostModel{1.0, 1.0, 0.5, 2.0});
  emit(57, 57, CostModel{1.0, 1.0, 0.5, 2.0});
  emit(1 << 20, 32, CostModel{1.0, 0.0, 0.0, 0.0});  // pure cross-chunk attention
  emit(1 << 20, 8, CostModel{2e-9, 1e-9, 3e-4, 5.0});
  std::mt19937_64 rng(21);
  std::uniform_real_distribution<double> coeff(0.0, 3.0);
  std::uniform_int_distribution<std::size_t> tokens_pick(10, 4000);
  for (int trial = 0; trial < 24; ++trial) {
    const std::size_t tokens = tokens_pick(rng);
    std::uniform_int_distribution<std::size_t> k_pick(1, std::min<std::size_t>(tokens, 40));
    const std::size_t k = k_pick(rng);
    emit(tokens, k, CostModel{coeff(rng), coeff(rng), coeff(rng), coeff(rng)});
  }
  o << "end\n";
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "dcpp") return dcpp_main();
  std::ostream& o = std::cout;
  const SelectionOptions kNoForced{false, false, true};
  {  // a planted column needs growth (test_refine.cpp:102-124)
    const CalibrationSet calib{{0, 0, planted(128, 16, 64.0, 0.5, 3, {2}, {})}};
    RefineConfig cfg = basic_config();
    cfg.measure.selection = kNoForced;
    SparsityPlan plan;
    plan.budgets[{0, 0}] = HeadBudget{0, 0};
    refine_case(o, calib, plan, cfg);
  }
  {  // converged head untouched (test_refine.cpp:80-100)
    const CalibrationSet calib{{0, 0, planted(96, 16, 64.0, 0.5, 2, {2}, {})}};
    RefineConfig cfg = basic_config();
    cfg.measure.selection = kNoForced;
    SparsityPlan plan;
    plan.budgets[{0, 0}] = HeadBudget{4, 4};
    refine_case(o, calib, plan, cfg);
  }
  {  // a diffuse head stops at the cap (test_refine.cpp:150-165)
    std::mt19937_64 rng(5);
    const CalibrationSet calib{{0, 0, random_input(rng, 128, 8)}};
    RefineConfig cfg = basic_config();
    cfg.threshold = 0.99;
    cfg.budget_cap = HeadBudget{4, 4};
    cfg.vertical_increment = 2;
    cfg.slash_increment = 2;
    cfg.measure.selection = kNoForced;
    SparsityPlan plan;
    plan.budgets[{0, 0}] = HeadBudget{0, 0};
    refine_case(o, calib, plan, cfg);
  }
  {  // planted column + slash, forced lines on, two samples of one head and a second head
    CalibrationSet calib{{1, 2, planted(96, 16, 32.0, 1.0, 7, {5}, {40})},
                         {1, 2, planted(96, 16, 32.0, 1.0, 8, {5}, {40})},
                         {1, 3, planted(80, 16, 48.0, 0.5, 9, {3, 17}, {})}};
    RefineConfig cfg = basic_config();
    SparsityPlan plan;
    plan.budgets[{1, 2}] = HeadBudget{0, 0};
    plan.budgets[{1, 3}] = HeadBudget{1, 0};
    plan.budgets[{0, 7}] = HeadBudget{3, 3};  // absent from the calibration: passes through
    refine_case(o, calib, plan, cfg);
  }
  {  // FractionAbove aggregate
    const CalibrationSet calib{{0, 1, planted(112, 16, 64.0, 0.5, 11, {4}, {})}};
    RefineConfig cfg = basic_config();
    cfg.measure.selection = kNoForced;
    cfg.measure.aggregate = RecallAggregate::FractionAbove;
    cfg.measure.fraction_tau = 0.8;
    SparsityPlan plan;
    plan.budgets[{0, 1}] = HeadBudget{0, 0};
    refine_case(o, calib, plan, cfg);
  }
  {  // offline grid search (refine.cpp:140-164)
    std::mt19937_64 rng(12);
    const CalibrationSet calib{{0, 0, planted(128, 16, 64.0, 0.5, 3, {2}, {})},
                               {0, 1, planted(96, 16, 32.0, 1.0, 7, {5}, {40})},
                               {0, 2, random_input(rng, 64, 8)}};
    const std::vector<HeadBudget> grid{{0, 0}, {1, 1}, {2, 2}, {4, 4}, {8, 8}};
    RecallMeasurement m;
    m.last_q = 32;
    m.selection = kNoForced;
    offline_case(o, calib, grid, 0.9, m);
  }
  {  // CriticalSet JSON text (sparse.cpp:121-125)
    std::vector<CriticalSet> sets(3);
    sets[0].context_length = 1024;
    sets[0].verticals = {0, 64, 288};
    sets[0].slashes = {0, 1, 2, 64, 288};
    sets[1].context_length = 7;
    sets[2].context_length = 300;
    sets[2].verticals = {5};
    for (const auto& c : sets) {
      o << "crit " << c.context_length << " " << c.verticals.size();
      for (auto x : c.verticals) o << " " << x;
      o << " " << c.slashes.size();
      for (auto x : c.slashes) o << " " << x;
      o << "\n";
      put_str(o, c.to_json().dump(2));
    }
  }
  o << "end\n";
  return 0;
}
