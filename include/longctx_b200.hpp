// longctx_b200.hpp -- C++ drop-in for the reference `longctx` operator API on the
// prefill attention path, implemented on the B200 (sm_100a) kernels behind the
// C-ABI of longctx_b200.h.
//
// Same namespace, type names, function signatures, argument meaning and error kinds
// as the reference headers (paths relative to /root/reference/proj/core/include/
// longctx/):
//   Matrix, BoolMatrix, RelPositionMatrix ........ matrix.hpp:12-63
//   Error, errkind ............................... errors.hpp:12-39
//   AttentionInput, AttentionResult, kDefaultRopeBase, full_attention,
//   full_attention_f32, flop_estimate, check_gqa_grouping ... attention.hpp:11-89
//   ChunkConfig, PatternKind, YarnScale, yarn_temperature, classify_pair,
//   dca_relative, dca_position_matrix, dca_attention ........ dca.hpp:15-65
//   HeadBudget, CriticalSet, PositionMode, SelectionOptions, estimate_block,
//   select_critical, sparse_attention, selection_position, density, PrefillMode,
//   ChunkSelection, PrefillState, PrefillResult, chunked_prefill .. sparse.hpp:17-129
//   RecallReport, attention_recall, RecallAggregate, RecallMeasurement,
//   measure_budget_recall ....................................... refine.hpp:15-40
//   SparsityPlan, CriticalSet::to_json / from_json ............... sparse.hpp:27-58
//   CalibrationSample, CalibrationSet, RefineConfig, HeadRefineRecord, RefineReport,
//   refine_plan, offline_search ................................. refine.hpp:42-92
//   CostModel, chunk_cost, ChunkSchedule, fixed_schedule, dcpp_schedule
//   ................................................... engine_sim.hpp:10-43
//
// A program written against the reference recompiles against this header and links
// liblongctx_b200.so instead of longctx_core.  Inputs are fp64 host matrices as in
// the reference; they are stored on the device as fp32 (default: the exact parity
// path, 1e-5) or bf16 (b200::set_precision), computed there, and returned as fp64.
// Every compute entry runs on the GPU: there is no CPU fallback (without a usable
// sm_100 device the call throws Error("cuda", ...)).
//
// JSON: the reference exchanges nlohmann::json values; this header exchanges their
// text (to_json returns what nlohmann's dump(2) prints for the same value, from_json
// parses it), so a caller writes / reads the same files without the nlohmann
// dependency.  Not provided: rope_apply / stable_softmax_rows (test helpers of the
// reference).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace longctx {

// ------------------------------------------------------------ matrix.hpp --
struct Matrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<double> values;

  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), values(r * c, 0.0) {}
  double& at(std::size_t i, std::size_t j) { return values[i * cols + j]; }
  double at(std::size_t i, std::size_t j) const { return values[i * cols + j]; }
  std::span<double> row(std::size_t i) { return {values.data() + i * cols, cols}; }
  std::span<const double> row(std::size_t i) const { return {values.data() + i * cols, cols}; }
  bool all_finite() const {
    for (double v : values)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool operator==(const Matrix&) const = default;
};

struct BoolMatrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<std::uint8_t> values;
  BoolMatrix() = default;
  BoolMatrix(std::size_t r, std::size_t c, bool fill = false)
      : rows(r), cols(c), values(r * c, fill ? 1 : 0) {}
  void set(std::size_t i, std::size_t j, bool v) { values[i * cols + j] = v ? 1 : 0; }
  bool at(std::size_t i, std::size_t j) const { return values[i * cols + j] != 0; }
};

struct RelPositionMatrix {
  std::size_t n = 0;
  std::vector<std::int64_t> values;
  RelPositionMatrix() = default;
  explicit RelPositionMatrix(std::size_t n_) : n(n_), values(n_ * n_, 0) {}
  std::int64_t& at(std::size_t i, std::size_t j) { return values[i * n + j]; }
  std::int64_t at(std::size_t i, std::size_t j) const { return values[i * n + j]; }
};

// ------------------------------------------------------------ errors.hpp --
class Error : public std::runtime_error {
 public:
  Error(std::string kind, const std::string& message)
      : std::runtime_error(message), kind_(std::move(kind)) {}
  const std::string& kind() const noexcept { return kind_; }

 private:
  std::string kind_;
};

namespace errkind {
inline constexpr const char* dimension = "dimension";
inline constexpr const char* config = "config";
inline constexpr const char* domain = "domain";
inline constexpr const char* causality = "causality";
inline constexpr const char* empty_row = "empty_row";
inline constexpr const char* empty_calibration = "empty_calibration";
inline constexpr const char* parse = "parse_error";
inline constexpr const char* schema = "schema_violation";
inline constexpr const char* cuda = "cuda";          // B200 build: device / launch failure
inline constexpr const char* internal = "internal";
}  // namespace errkind

// --------------------------------------------------------- attention.hpp --
inline constexpr double kDefaultRopeBase = 10000.0;

struct AttentionInput {
  Matrix q;
  Matrix k;
  Matrix v;
  std::vector<std::int64_t> positions_q;
  std::vector<std::int64_t> positions_k;
  double rope_base = kDefaultRopeBase;
  double temperature = 1.0;
  std::size_t seq_len() const { return q.rows; }
  std::size_t head_dim() const { return q.cols; }
  void validate() const;
};

struct AttentionResult {
  Matrix output;
  std::vector<double> lse;
};

AttentionResult full_attention(const AttentionInput& input,
                               const RelPositionMatrix* rel_override = nullptr);
AttentionResult full_attention_f32(const AttentionInput& input,
                                   const RelPositionMatrix* rel_override = nullptr);
double flop_estimate(std::size_t n, std::size_t head_dim, std::size_t computed_entries);
void check_gqa_grouping(std::size_t query_heads, std::size_t kv_heads);

// --------------------------------------------------------------- dca.hpp --
struct ChunkConfig {
  std::size_t chunk_size = 0;    // s
  std::size_t train_len = 0;     // c
  std::size_t local_window = 0;  // w
  static ChunkConfig with_default_window(std::size_t chunk_size, std::size_t train_len);
  void validate() const;
};

enum class PatternKind { Intra, Successive, Inter };

struct YarnScale {
  double scale_factor = 1.0;
  double temperature = 1.0;
  static YarnScale from_scale(double scale_factor);
  void validate() const;
};

double yarn_temperature(double scale_factor);
PatternKind classify_pair(std::size_t i, std::size_t j, const ChunkConfig& cfg);
std::int64_t dca_relative(std::size_t i, std::size_t j, const ChunkConfig& cfg);
RelPositionMatrix dca_position_matrix(std::size_t n, const ChunkConfig& cfg);
AttentionResult dca_attention(const AttentionInput& input, const ChunkConfig& cfg,
                              const YarnScale& yarn);

// ------------------------------------------------------------ sparse.hpp --
struct HeadBudget {
  std::size_t vertical = 0;
  std::size_t slash = 0;
  std::size_t total() const { return vertical + slash; }
  bool operator==(const HeadBudget&) const = default;
};

// Per (layer, head) budgets; JSON object {"layer.head": {"slash": S, "vertical": V}}.
struct SparsityPlan {
  std::map<std::pair<std::size_t, std::size_t>, HeadBudget> budgets;
  HeadBudget& at(std::size_t layer, std::size_t head);
  const HeadBudget& at(std::size_t layer, std::size_t head) const;  // Error("config") if absent
  std::string to_json() const;
  static SparsityPlan from_json(const std::string& text);
};

struct CriticalSet {
  std::vector<std::size_t> verticals;  // sorted unique column indices
  std::vector<std::size_t> slashes;    // sorted unique diagonal offsets
  std::size_t context_length = 0;
  bool admits(std::size_t i, std::size_t j) const;
  std::vector<std::size_t> admitted_row(std::size_t i) const;
  std::size_t admitted_count() const;
  // {"contextLength": n, "slashes": [...], "verticals": [...]}
  std::string to_json() const;
  static CriticalSet from_json(const std::string& text);
  bool operator==(const CriticalSet&) const = default;
};

enum class PositionMode { Standard, DcaContinuous };

struct SelectionOptions {
  bool force_sink_column = true;
  bool force_local_band = true;
  bool slash_mean = true;
};

Matrix estimate_block(const Matrix& q, const Matrix& k, std::size_t last_q, PositionMode mode,
                      const std::optional<ChunkConfig>& cfg,
                      double rope_base = kDefaultRopeBase);
CriticalSet select_critical(const Matrix& est, HeadBudget budget, std::size_t n,
                            const SelectionOptions& opts = {});
AttentionResult sparse_attention(const AttentionInput& input, const CriticalSet& crit,
                                 const RelPositionMatrix* rel_override = nullptr);
std::int64_t selection_position(std::size_t i, std::size_t j, const ChunkConfig& cfg);
double density(const CriticalSet& crit);

enum class PrefillMode { Full, Sparse };

struct ChunkSelection {
  std::size_t chunk_index = 0;
  std::size_t begin = 0;
  std::size_t end = 0;
  CriticalSet critical;
};

struct PrefillState {
  Matrix cached_k;
  Matrix cached_v;
  std::vector<ChunkSelection> selections;
  std::size_t chunk_len = 0;
  std::size_t last_q = 0;
};

struct PrefillResult {
  AttentionResult result;
  PrefillState state;
};

PrefillResult chunked_prefill(const AttentionInput& input, std::size_t chunk_len,
                              std::size_t last_q, HeadBudget budget, PrefillMode mode,
                              PositionMode pos_mode, const std::optional<ChunkConfig>& cfg,
                              const SelectionOptions& opts = {});

// ------------------------------------------------------------ refine.hpp --
struct RecallReport {
  std::size_t layer = 0;
  std::size_t head = 0;
  std::vector<double> per_query;
  double aggregate = 0.0;
};

RecallReport attention_recall(std::span<const double> lse_sparse,
                              std::span<const double> lse_full);

enum class RecallAggregate { Mean, FractionAbove };

struct RecallMeasurement {
  std::size_t last_q = 64;
  SelectionOptions selection{};
  RecallAggregate aggregate = RecallAggregate::Mean;
  double fraction_tau = 0.9;
};

double measure_budget_recall(const AttentionInput& input, HeadBudget budget,
                             const RecallMeasurement& measure);

struct CalibrationSample {
  std::size_t layer = 0;
  std::size_t head = 0;
  AttentionInput input;
};
using CalibrationSet = std::vector<CalibrationSample>;

struct RefineConfig {
  double threshold = 0.9;
  std::size_t vertical_increment = 4;
  std::size_t slash_increment = 4;
  std::size_t max_rounds = 8;
  HeadBudget budget_cap{64, 64};
  RecallMeasurement measure{};
  void validate() const;
};

struct HeadRefineRecord {
  std::size_t layer = 0;
  std::size_t head = 0;
  std::size_t rounds = 0;
  HeadBudget initial_budget;
  HeadBudget final_budget;
  double initial_recall = 0.0;
  double final_recall = 0.0;
};

struct RefineReport {
  std::vector<HeadRefineRecord> heads;
};

// Grows each sampled head's budget by the increments while its recall over the
// calibration samples stays below the threshold (refine.cpp:98-138).  On the device
// the dense LSE and the estimator matrix of every calibration input are computed once
// per call and reused by every budget tried (they do not depend on the budget).
std::pair<SparsityPlan, RefineReport> refine_plan(const CalibrationSet& calib,
                                                  const SparsityPlan& plan,
                                                  const RefineConfig& cfg);
// Per head, the first grid point (sorted by total budget) whose recall reaches the
// threshold, else the last (refine.cpp:140-164).
SparsityPlan offline_search(const CalibrationSet& calib, const std::vector<HeadBudget>& grid,
                            double threshold, const RecallMeasurement& measure = {});

// -------------------------------------------------------- engine_sim.hpp --
// Prefill chunk cost attn_coeff * n * h + self_coeff * n^2 / 2 + lin_coeff * n +
// fixed_cost for n tokens after h cached ones (engine_sim.hpp:10-21).
struct CostModel {
  double attn_coeff = 0.0;
  double self_coeff = 0.0;
  double lin_coeff = 0.0;
  double fixed_cost = 0.0;
  void validate() const;
};

double chunk_cost(const CostModel& model, std::size_t n, std::size_t h);

// Chunk boundaries as exclusive end indices (engine_sim.hpp:23-35).
struct ChunkSchedule {
  std::vector<std::size_t> boundaries;
  std::size_t total_tokens() const { return boundaries.empty() ? 0 : boundaries.back(); }
  std::size_t chunk_count() const { return boundaries.size(); }
  std::vector<std::size_t> sizes() const;
  std::pair<std::size_t, std::size_t> chunk(std::size_t idx) const;
  void validate() const;
};

ChunkSchedule fixed_schedule(std::size_t tokens, std::size_t chunks);
// DCPP: per-chunk costs as equal as the token grid allows (engine_sim.cpp:117-166).
ChunkSchedule dcpp_schedule(std::size_t tokens, std::size_t chunks, const CostModel& model);

// ------------------------------------------------- B200-specific controls --
namespace b200 {
// One measured prefill chunk: n tokens after h cached ones took `ms` on the device.
struct ChunkCostSample {
  std::size_t n = 0;
  std::size_t h = 0;
  double ms = 0.0;
};
// Runs chunked_prefill (same arguments) on the device with per-chunk CUDA events and
// returns every chunk's (n, h, ms) -- the measured costs a DCPP schedule is fed with.
std::vector<ChunkCostSample> measure_chunk_costs(
    const AttentionInput& input, std::size_t chunk_len, std::size_t last_q, HeadBudget budget,
    PrefillMode mode, PositionMode pos_mode, const std::optional<ChunkConfig>& cfg,
    const SelectionOptions& opts = {});
// Non-negative least-squares fit of the four CostModel coefficients to measured chunk
// costs (Error("config") when fewer than one sample).
CostModel fit_cost_model(const std::vector<ChunkCostSample>& samples);
// The per-chunk selection log of a chunked prefill as the reference CLI writes it
// (prefill_selections.json, harness.cpp:430-438, without its configHash / version keys).
std::string prefill_selections_json(const PrefillState& state);
std::vector<ChunkSelection> prefill_selections_from_json(const std::string& text);

enum class Precision { F32, BF16 };
// Device storage type of q / k / v for the calls made by this thread (default F32:
// the 1e-5 parity path; BF16: the tcgen05 path, 2e-3).
void set_precision(Precision p);
Precision precision();
// CUDA device used by this thread's calls (default 0).
void set_device(int device);
// Recall slack above 1 tolerated by attention_recall before it throws
// Error("domain") (reference: 1e-12 in fp64; scaled to the storage precision).
double recall_slack();
}  // namespace b200

}  // namespace longctx
