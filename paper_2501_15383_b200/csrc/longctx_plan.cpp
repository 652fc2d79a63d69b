// C++ drop-in, part 2: sparsity plans, their JSON text, and budget refinement over a
// calibration set (reference proj/core/src/sparse.cpp:32-78, 121-135 and
// proj/core/src/refine.cpp:85-164).  Host orchestration only: every recall measurement
// runs on the device through the operators of longctx_host.cpp.
//
// JSON: the reference (de)serialises nlohmann::json values; here the same values are
// exchanged as text.  The writer prints what nlohmann's dump(2) prints (object keys in
// std::map order, two-space indent, one array element per line, "[]" / "{}" when
// empty); the reader is a small recursive-descent parser for the JSON grammar.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "longctx_b200.hpp"

namespace longctx {
namespace {

[[noreturn]] void fail(const char* kind, const std::string& message) {
  throw Error(kind, message);
}

// ------------------------------------------------------------------- writer --
std::string indent(int n) { return std::string(std::size_t(n), ' '); }

std::string json_array(const std::vector<std::size_t>& xs, int ind) {
  if (xs.empty()) return "[]";
  std::string out = "[\n";
  for (std::size_t i = 0; i < xs.size(); ++i) {
    out += indent(ind + 2) + std::to_string(xs[i]);
    out += i + 1 < xs.size() ? ",\n" : "\n";
  }
  return out + indent(ind) + "]";
}

// members: already-rendered values, keys in the order given (callers pass map order)
std::string json_object(const std::vector<std::pair<std::string, std::string>>& members,
                        int ind) {
  if (members.empty()) return "{}";
  std::string out = "{\n";
  for (std::size_t i = 0; i < members.size(); ++i) {
    out += indent(ind + 2) + "\"" + members[i].first + "\": " + members[i].second;
    out += i + 1 < members.size() ? ",\n" : "\n";
  }
  return out + indent(ind) + "}";
}

// ------------------------------------------------------------------- reader --
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  bool integral = false;
  unsigned long long u = 0;
  bool negative = false;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;

  const JVal* find(const std::string& key) const {
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& t) : s_(t) {}
  JVal parse() {
    JVal v = value();
    ws();
    if (i_ != s_.size()) err("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  std::size_t i_ = 0;

  [[noreturn]] void err(const std::string& what) {
    fail(errkind::parse, "JSON parse error at offset " + std::to_string(i_) + ": " + what);
  }
  void ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) err(std::string("expected '") + c + "'");
  }
  std::string string_lit() {
    expect('"');
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) err("bad escape");
        const char e = s_[i_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {  // keep the code point if ASCII, else a placeholder
            if (i_ + 4 > s_.size()) err("bad \\u escape");
            const unsigned long cp = std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16);
            i_ += 4;
            out += cp < 128 ? char(cp) : '?';
            break;
          }
          default: err("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) err("unterminated string");
    ++i_;
    return out;
  }
  JVal value() {
    ws();
    if (i_ >= s_.size()) err("unexpected end");
    JVal v;
    const char c = s_[i_];
    if (c == '{') {
      ++i_;
      v.kind = JVal::Obj;
      if (eat('}')) return v;
      do {
        ws();
        std::string key = string_lit();
        expect(':');
        v.obj.emplace_back(std::move(key), value());
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i_;
      v.kind = JVal::Arr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = JVal::Str;
      v.str = string_lit();
    } else if (s_.compare(i_, 4, "true") == 0) {
      i_ += 4;
      v.kind = JVal::Bool;
      v.b = true;
    } else if (s_.compare(i_, 5, "false") == 0) {
      i_ += 5;
      v.kind = JVal::Bool;
    } else if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
      const std::size_t b = i_;
      if (s_[i_] == '-') ++i_;
      while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
      bool integral = true;
      if (i_ < s_.size() && (s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E')) {
        integral = false;
        ++i_;
        while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) ||
                                  s_[i_] == '+' || s_[i_] == '-' || s_[i_] == 'e' ||
                                  s_[i_] == 'E'))
          ++i_;
      }
      const std::string tok = s_.substr(b, i_ - b);
      v.kind = JVal::Num;
      v.integral = integral;
      v.negative = tok[0] == '-';
      v.num = std::strtod(tok.c_str(), nullptr);
      if (integral && !v.negative) v.u = std::strtoull(tok.c_str(), nullptr, 10);
    } else {
      err("unexpected character");
    }
    return v;
  }
};

std::size_t as_size(const JVal& v, const std::string& what) {
  if (v.kind != JVal::Num || !v.integral || v.negative)
    fail(errkind::schema, what + " must be a non-negative integer");
  return std::size_t(v.u);
}

std::vector<std::size_t> as_size_array(const JVal& v, const std::string& what) {
  if (v.kind != JVal::Arr) fail(errkind::schema, what + " must be an array");
  std::vector<std::size_t> out;
  out.reserve(v.arr.size());
  for (const JVal& x : v.arr) out.push_back(as_size(x, what));
  return out;
}

void sort_unique(std::vector<std::size_t>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

// ----------------------------------------------------------- refinement --
using HeadKey = std::pair<std::size_t, std::size_t>;

// Everything of a calibration input that does not depend on the budget: the dense
// LSE and the estimator matrix (refine.cpp:76-79), computed once per call.
struct Prepared {
  const AttentionInput* input = nullptr;
  std::vector<double> full_lse;
  Matrix est;
};

class RecallCache {
 public:
  explicit RecallCache(const RecallMeasurement& m) : m_(m) {}

  // measure_budget_recall (refine.cpp:74-85) on the cached budget-free parts
  double recall(const AttentionInput& input, HeadBudget budget) {
    const Prepared& p = prepare(input);
    const std::size_t n = input.seq_len();
    const CriticalSet crit = select_critical(p.est, budget, n, m_.selection);
    const AttentionResult sparse = sparse_attention(input, crit);
    const RecallReport rep = attention_recall(sparse.lse, p.full_lse);
    if (m_.aggregate == RecallAggregate::Mean) return rep.aggregate;
    std::size_t above = 0;  // refine.cpp:16-27
    for (double r : rep.per_query)
      if (r >= m_.fraction_tau) ++above;
    return double(above) / double(rep.per_query.size());
  }

  // head_recall (refine.cpp:40-47): mean over the head's calibration inputs
  double head_recall(const std::vector<const AttentionInput*>& inputs, HeadBudget budget) {
    double sum = 0.0;
    for (const AttentionInput* in : inputs) sum += recall(*in, budget);
    return sum / double(inputs.size());
  }

 private:
  RecallMeasurement m_;
  std::map<const AttentionInput*, Prepared> cache_;

  const Prepared& prepare(const AttentionInput& input) {
    auto it = cache_.find(&input);
    if (it != cache_.end()) return it->second;
    Prepared p;
    p.input = &input;
    const std::size_t n = input.seq_len();
    p.full_lse = full_attention(input).lse;
    p.est = estimate_block(input.q, input.k, std::min(m_.last_q, n), PositionMode::Standard,
                           std::nullopt, input.rope_base);
    return cache_.emplace(&input, std::move(p)).first->second;
  }
};

std::map<HeadKey, std::vector<const AttentionInput*>> group_by_head(const CalibrationSet& c) {
  std::map<HeadKey, std::vector<const AttentionInput*>> groups;  // refine.cpp:31-38
  for (const auto& s : c) groups[{s.layer, s.head}].push_back(&s.input);
  return groups;
}

}  // namespace

// ------------------------------------------------------------ SparsityPlan --
HeadBudget& SparsityPlan::at(std::size_t layer, std::size_t head) {  // sparse.cpp:32-34
  return budgets[{layer, head}];
}

const HeadBudget& SparsityPlan::at(std::size_t layer, std::size_t head) const {
  auto it = budgets.find({layer, head});  // sparse.cpp:36-43
  if (it == budgets.end())
    fail(errkind::config, "sparsity plan has no entry for layer " + std::to_string(layer) +
                              " head " + std::to_string(head));
  return it->second;
}

std::string SparsityPlan::to_json() const {  // sparse.cpp:45-52
  std::map<std::string, HeadBudget> byname;  // nlohmann objects iterate in key order
  for (const auto& [key, b] : budgets)
    byname[std::to_string(key.first) + "." + std::to_string(key.second)] = b;
  std::vector<std::pair<std::string, std::string>> members;
  for (const auto& [name, b] : byname)
    members.emplace_back(name, json_object({{"slash", std::to_string(b.slash)},
                                            {"vertical", std::to_string(b.vertical)}},
                                           2));
  return json_object(members, 0);
}

SparsityPlan SparsityPlan::from_json(const std::string& text) {  // sparse.cpp:54-78
  const JVal j = Parser(text).parse();
  if (j.kind != JVal::Obj) fail(errkind::schema, "sparsity plan must be a JSON object");
  SparsityPlan plan;
  for (const auto& [name, value] : j.obj) {
    const auto dot = name.find('.');
    const auto bad_key = [&]() {
      fail(errkind::schema, "sparsity plan key \"" + name + "\" is not \"layer.head\"");
    };
    if (dot == std::string::npos) bad_key();
    const std::string a = name.substr(0, dot), b = name.substr(dot + 1);
    const auto digits = [](const std::string& x) {
      return !x.empty() && std::all_of(x.begin(), x.end(), [](char c) {
        return std::isdigit(static_cast<unsigned char>(c)) != 0;
      });
    };
    if (!digits(a) || !digits(b)) bad_key();  // std::stoull accepts a leading number only
    const JVal* v = value.kind == JVal::Obj ? value.find("vertical") : nullptr;
    const JVal* sl = value.kind == JVal::Obj ? value.find("slash") : nullptr;
    if (!v || !sl)
      fail(errkind::schema,
           "sparsity plan entry \"" + name + "\" must carry vertical and slash counts");
    plan.budgets[{std::stoull(a), std::stoull(b)}] =
        HeadBudget{as_size(*v, "vertical"), as_size(*sl, "slash")};
  }
  return plan;
}

// ------------------------------------------------------------ CriticalSet --
namespace {
std::string crit_json(const CriticalSet& c, int ind) {  // sparse.cpp:121-125
  return json_object({{"contextLength", std::to_string(c.context_length)},
                      {"slashes", json_array(c.slashes, ind + 2)},
                      {"verticals", json_array(c.verticals, ind + 2)}},
                     ind);
}
}  // namespace

std::string CriticalSet::to_json() const { return crit_json(*this, 0); }

namespace b200 {
std::string prefill_selections_json(const PrefillState& state) {  // harness.cpp:430-438
  std::string arr;
  if (state.selections.empty()) {
    arr = "[]";
  } else {
    arr = "[\n";
    for (std::size_t x = 0; x < state.selections.size(); ++x) {
      const ChunkSelection& cs = state.selections[x];
      arr += indent(4) + json_object({{"begin", std::to_string(cs.begin)},
                                      {"chunk", std::to_string(cs.chunk_index)},
                                      {"critical", crit_json(cs.critical, 6)},
                                      {"end", std::to_string(cs.end)}},
                                     4);
      arr += x + 1 < state.selections.size() ? ",\n" : "\n";
    }
    arr += indent(2) + "]";
  }
  return json_object({{"selections", arr}}, 0);
}

std::vector<ChunkSelection> prefill_selections_from_json(const std::string& text) {
  const JVal j = Parser(text).parse();
  const JVal* sel = j.kind == JVal::Obj ? j.find("selections") : nullptr;
  if (!sel || sel->kind != JVal::Arr) fail(errkind::schema, "prefill selections need a \"selections\" array");
  std::vector<ChunkSelection> out;
  for (const JVal& e : sel->arr) {
    const JVal* b = e.kind == JVal::Obj ? e.find("begin") : nullptr;
    const JVal* c = e.kind == JVal::Obj ? e.find("chunk") : nullptr;
    const JVal* en = e.kind == JVal::Obj ? e.find("end") : nullptr;
    const JVal* cr = e.kind == JVal::Obj ? e.find("critical") : nullptr;
    if (!b || !c || !en || !cr || cr->kind != JVal::Obj)
      fail(errkind::schema, "a selection needs begin, chunk, end and critical");
    ChunkSelection cs;
    cs.begin = as_size(*b, "begin");
    cs.chunk_index = as_size(*c, "chunk");
    cs.end = as_size(*en, "end");
    const JVal* n = cr->find("contextLength");
    const JVal* v = cr->find("verticals");
    const JVal* sl = cr->find("slashes");
    if (!n || !v || !sl) fail(errkind::schema, "critical set needs contextLength, verticals and slashes");
    cs.critical.context_length = as_size(*n, "contextLength");
    cs.critical.verticals = as_size_array(*v, "verticals");
    cs.critical.slashes = as_size_array(*sl, "slashes");
    sort_unique(cs.critical.verticals);
    sort_unique(cs.critical.slashes);
    out.push_back(std::move(cs));
  }
  return out;
}
}  // namespace b200

CriticalSet CriticalSet::from_json(const std::string& text) {  // sparse.cpp:127-135
  const JVal j = Parser(text).parse();
  if (j.kind != JVal::Obj) fail(errkind::schema, "critical set must be a JSON object");
  const JVal* n = j.find("contextLength");
  const JVal* v = j.find("verticals");
  const JVal* sl = j.find("slashes");
  if (!n || !v || !sl)
    fail(errkind::schema, "critical set needs contextLength, verticals and slashes");
  CriticalSet crit;
  crit.context_length = as_size(*n, "contextLength");
  crit.verticals = as_size_array(*v, "verticals");
  crit.slashes = as_size_array(*sl, "slashes");
  sort_unique(crit.verticals);
  sort_unique(crit.slashes);
  return crit;
}

// ------------------------------------------------------------- refinement --
void RefineConfig::validate() const {  // refine.cpp:87-96
  if (!(threshold > 0.0 && threshold < 1.0)) fail(errkind::config, "threshold must lie in (0, 1)");
  if (vertical_increment == 0 || slash_increment == 0)
    fail(errkind::config, "budget increments must be at least 1");
  if (max_rounds == 0) fail(errkind::config, "maxRounds must be at least 1");
  if (measure.last_q == 0) fail(errkind::config, "lastQ must be positive");
}

std::pair<SparsityPlan, RefineReport> refine_plan(const CalibrationSet& calib,
                                                  const SparsityPlan& plan,
                                                  const RefineConfig& cfg) {  // refine.cpp:98-138
  cfg.validate();
  if (calib.empty())
    fail(errkind::empty_calibration, "refinement requires a non-empty calibration set");
  SparsityPlan refined = plan;
  RefineReport report;
  RecallCache cache(cfg.measure);
  for (const auto& [key, inputs] : group_by_head(calib)) {
    const HeadBudget initial = plan.at(key.first, key.second);
    HeadBudget budget = initial;
    HeadRefineRecord rec;
    rec.layer = key.first;
    rec.head = key.second;
    rec.initial_budget = initial;
    rec.initial_recall = cache.head_recall(inputs, budget);
    double recall = rec.initial_recall;
    std::size_t rounds = 0;
    while (recall < cfg.threshold && rounds < cfg.max_rounds &&
           (budget.vertical < cfg.budget_cap.vertical || budget.slash < cfg.budget_cap.slash)) {
      budget.vertical = std::min(budget.vertical + cfg.vertical_increment, cfg.budget_cap.vertical);
      budget.slash = std::min(budget.slash + cfg.slash_increment, cfg.budget_cap.slash);
      ++rounds;
      recall = cache.head_recall(inputs, budget);
    }
    rec.rounds = rounds;
    rec.final_budget = budget;
    rec.final_recall = recall;
    report.heads.push_back(rec);
    refined.at(key.first, key.second) = budget;
  }
  return {std::move(refined), std::move(report)};
}

SparsityPlan offline_search(const CalibrationSet& calib, const std::vector<HeadBudget>& grid,
                            double threshold, const RecallMeasurement& measure) {
  if (grid.empty()) fail(errkind::config, "search grid must not be empty");  // refine.cpp:140-164
  for (std::size_t g = 1; g < grid.size(); ++g)
    if (grid[g].total() < grid[g - 1].total())
      fail(errkind::config, "search grid must be sorted by total budget ascending");
  if (calib.empty())
    fail(errkind::empty_calibration, "offline search requires a non-empty calibration set");
  SparsityPlan plan;
  RecallCache cache(measure);
  for (const auto& [key, inputs] : group_by_head(calib)) {
    HeadBudget chosen = grid.back();
    for (const HeadBudget& candidate : grid) {
      if (cache.head_recall(inputs, candidate) >= threshold) {
        chosen = candidate;
        break;
      }
    }
    plan.budgets[key] = chosen;
  }
  return plan;
}

}  // namespace longctx

// ------------------------------------------------------- DCPP chunk sizing --
// engine_sim.cpp:33-166 restated: cost model, fixed and cost-balanced schedules.
namespace longctx {

void CostModel::validate() const {
  if (attn_coeff < 0 || self_coeff < 0 || lin_coeff < 0 || fixed_cost < 0)
    fail(errkind::config, "cost coefficients must be non-negative");
}

double chunk_cost(const CostModel& m, std::size_t n, std::size_t h) {
  if (n == 0) fail(errkind::domain, "chunk must contain at least one token");
  const double x = double(n);
  return m.attn_coeff * x * double(h) + m.self_coeff * x * x / 2.0 + m.lin_coeff * x +
         m.fixed_cost;
}

std::vector<std::size_t> ChunkSchedule::sizes() const {
  std::vector<std::size_t> out;
  out.reserve(boundaries.size());
  std::size_t prev = 0;
  for (std::size_t b : boundaries) {
    out.push_back(b - prev);
    prev = b;
  }
  return out;
}

std::pair<std::size_t, std::size_t> ChunkSchedule::chunk(std::size_t idx) const {
  return {idx == 0 ? 0 : boundaries[idx - 1], boundaries[idx]};
}

void ChunkSchedule::validate() const {
  if (boundaries.empty()) fail(errkind::config, "schedule has no chunks");
  std::size_t prev = 0;
  for (std::size_t b : boundaries) {
    if (b <= prev) fail(errkind::config, "chunk boundaries must be strictly increasing");
    prev = b;
  }
}

ChunkSchedule fixed_schedule(std::size_t tokens, std::size_t chunks) {
  if (chunks == 0 || chunks > tokens) fail(errkind::config, "chunk count must lie in [1, tokens]");
  ChunkSchedule s;
  const std::size_t base = tokens / chunks, extra = tokens % chunks;  // remainder to the left
  std::size_t pos = 0;
  for (std::size_t c = 0; c < chunks; ++c) s.boundaries.push_back(pos += base + (c < extra));
  return s;
}

namespace {
// Feasibility of a per-chunk cost bound tau: walk left to right, each chunk taking
// tokens while its cost stays within tau (leaving one token per remaining chunk), the
// last chunk taking the rest.  Empty result = infeasible.
std::vector<std::size_t> walk_under(double tau, std::size_t tokens, std::size_t chunks,
                                    const CostModel& m) {
  std::vector<std::size_t> ends;
  std::size_t pos = 0;
  for (std::size_t c = 0; c < chunks && pos < tokens; ++c) {
    std::size_t take = c + 1 == chunks ? tokens - pos : 1;
    if (chunk_cost(m, take, pos) > tau) return {};
    if (c + 1 < chunks) {
      const std::size_t cap = tokens - pos - (chunks - c - 1);
      while (take < cap && chunk_cost(m, take + 1, pos) <= tau) ++take;
    }
    pos += take;
    ends.push_back(pos);
  }
  if (pos != tokens) return {};
  return ends;
}
}  // namespace

ChunkSchedule dcpp_schedule(std::size_t tokens, std::size_t chunks, const CostModel& m) {
  m.validate();
  if (chunks == 0 || chunks > tokens) fail(errkind::config, "chunk count must lie in [1, tokens]");
  if (chunks == 1) return ChunkSchedule{{tokens}};
  // bisection on the largest admissible chunk cost (the whole prompt as one chunk
  // bounds it from above)
  const double t = double(tokens);
  double lo = 0.0;
  double hi = m.attn_coeff * t * t + m.self_coeff * t * t / 2.0 + m.lin_coeff * t +
              m.fixed_cost + 1.0;
  for (int it = 0; it < 200 && hi > lo; ++it) {
    const double mid = lo + (hi - lo) / 2.0;
    if (!(mid > lo && mid < hi)) break;
    if (walk_under(mid, tokens, chunks, m).empty()) lo = mid;
    else hi = mid;
  }
  ChunkSchedule s{walk_under(hi, tokens, chunks, m)};
  if (s.boundaries.empty()) fail(errkind::domain, "chunk cost search failed to converge");
  // the walk may need fewer chunks: halve the costliest splittable chunk until the count
  // is met (splitting never raises a chunk's cost)
  while (s.chunk_count() < chunks) {
    std::size_t best = s.chunk_count();
    double best_cost = -1.0;
    for (std::size_t c = 0; c < s.chunk_count(); ++c) {
      const auto [b, e] = s.chunk(c);
      if (e - b < 2) continue;
      const double cost = chunk_cost(m, e - b, b);
      if (cost > best_cost) {
        best_cost = cost;
        best = c;
      }
    }
    const auto [b, e] = s.chunk(best);
    s.boundaries.insert(s.boundaries.begin() + std::ptrdiff_t(best), b + (e - b) / 2);
  }
  s.validate();
  return s;
}

namespace b200 {
CostModel fit_cost_model(const std::vector<ChunkCostSample>& samples) {
  if (samples.empty()) fail(errkind::config, "cost fit needs at least one measured chunk");
  // features of a chunk: n*h, n^2/2, n, 1.  Least squares on the active set by
  // Householder QR in long double (the features are nearly collinear over a narrow
  // range of chunk sizes, which squares badly in the normal equations); the most
  // negative coefficient leaves the set until all are >= 0 (4 unknowns: <= 4 passes).
  using LD = long double;
  auto feat = [](const ChunkCostSample& x, int k) -> LD {
    const LD n = LD(x.n), h = LD(x.h);
    return k == 0 ? n * h : k == 1 ? n * n / 2 : k == 2 ? n : LD(1);
  };
  const std::size_t m = samples.size();
  bool active[4] = {true, true, true, true};
  double coef[4] = {0, 0, 0, 0};
  for (int pass = 0; pass < 4; ++pass) {
    int idx[4], na = 0;
    for (int k = 0; k < 4; ++k)
      if (active[k]) idx[na++] = k;
    std::vector<LD> A(m * std::size_t(na)), y(m);
    std::vector<LD> scale(std::size_t(na), 0);
    for (int a = 0; a < na; ++a) {
      for (std::size_t i = 0; i < m; ++i) scale[a] += feat(samples[i], idx[a]) * feat(samples[i], idx[a]);
      scale[a] = scale[a] > 0 ? 1 / std::sqrt(scale[a]) : 0;  // unit-norm columns
      for (std::size_t i = 0; i < m; ++i) A[i * na + a] = feat(samples[i], idx[a]) * scale[a];
    }
    for (std::size_t i = 0; i < m; ++i) y[i] = samples[i].ms;
    // Householder QR: A = Q R, then R c = Q^T y
    const int kc = int(std::min<std::size_t>(std::size_t(na), m));
    for (int j = 0; j < kc; ++j) {
      LD norm = 0;
      for (std::size_t i = std::size_t(j); i < m; ++i) norm += A[i * na + j] * A[i * na + j];
      norm = std::sqrt(norm);
      if (norm == 0) continue;
      const LD alpha = A[std::size_t(j) * na + j] > 0 ? -norm : norm;
      std::vector<LD> v(m, 0);
      for (std::size_t i = std::size_t(j); i < m; ++i) v[i] = A[i * na + j];
      v[std::size_t(j)] -= alpha;
      LD vv = 0;
      for (std::size_t i = std::size_t(j); i < m; ++i) vv += v[i] * v[i];
      if (vv == 0) continue;
      for (int c = j; c < na; ++c) {
        LD d = 0;
        for (std::size_t i = std::size_t(j); i < m; ++i) d += v[i] * A[i * na + c];
        d = 2 * d / vv;
        for (std::size_t i = std::size_t(j); i < m; ++i) A[i * na + c] -= d * v[i];
      }
      LD d = 0;
      for (std::size_t i = std::size_t(j); i < m; ++i) d += v[i] * y[i];
      d = 2 * d / vv;
      for (std::size_t i = std::size_t(j); i < m; ++i) y[i] -= d * v[i];
    }
    LD c[4] = {0, 0, 0, 0};
    for (int j = kc - 1; j >= 0; --j) {  // back substitution; rank-deficient columns -> 0
      const LD r = A[std::size_t(j) * na + j];
      if (std::fabs(double(r)) < 1e-13) continue;
      LD acc = y[std::size_t(j)];
      for (int k = j + 1; k < kc; ++k) acc -= A[std::size_t(j) * na + k] * c[k];
      c[j] = acc / r;
    }
    for (int k = 0; k < 4; ++k) coef[k] = 0.0;
    int worst = -1;
    for (int a = 0; a < na; ++a) {
      coef[idx[a]] = double(c[a] * scale[a]);
      if (coef[idx[a]] < 0 && (worst < 0 || coef[idx[a]] < coef[worst])) worst = idx[a];
    }
    if (worst < 0) break;
    active[worst] = false;
    coef[worst] = 0.0;
  }
  return CostModel{std::max(0.0, coef[0]), std::max(0.0, coef[1]), std::max(0.0, coef[2]),
                   std::max(0.0, coef[3])};
}
}  // namespace b200

}  // namespace longctx
