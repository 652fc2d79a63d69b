// C++ drop-in (include/longctx_b200.hpp): the reference `longctx` operator API on the
// prefill path, implemented over the C-ABI (include/longctx_b200.h).
//
// Host-side logic that the reference also keeps on the host -- argument validation
// with the same error kinds and messages, the integer DCA / critical-set helpers,
// flop accounting -- is restated here; every floating-point operator (estimate,
// selection scores, attention, recall) runs on the device through the C-ABI.
// References are to /root/reference/proj/core/src.
#include "longctx_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>

#include "longctx_b200.h"

namespace longctx {

namespace {

thread_local b200::Precision g_precision = b200::Precision::F32;
thread_local int g_device = 0;

[[noreturn]] void fail(const char* kind, const std::string& message) {
  throw Error(kind, message);
}

const char* kind_of(int status) {
  switch (status) {
    case LCX_ERR_DIMENSION: return errkind::dimension;
    case LCX_ERR_CONFIG: return errkind::config;
    case LCX_ERR_DOMAIN: return errkind::domain;
    case LCX_ERR_CAUSALITY: return errkind::causality;
    case LCX_ERR_EMPTY_ROW: return errkind::empty_row;
    case LCX_ERR_EMPTY_CALIBRATION: return errkind::empty_calibration;
    case LCX_ERR_CUDA: return errkind::cuda;
    default: return errkind::internal;
  }
}

void check(int status) {
  if (status != LCX_OK) throw Error(kind_of(status), lcx_last_error());
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(errkind::cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

// one C-ABI context per (thread, device)
struct ContextHolder {
  std::map<int, lcx_context*> ctx;
  ~ContextHolder() {
    for (auto& kv : ctx) lcx_context_destroy(kv.second);
  }
};

lcx_context* context() {
  thread_local ContextHolder holder;
  // the device uploads / downloads around each call (DevBuf) go to the selected device too
  check_cuda(cudaSetDevice(g_device), "cudaSetDevice");
  auto it = holder.ctx.find(g_device);
  if (it != holder.ctx.end()) return it->second;
  lcx_context* c = nullptr;
  check(lcx_context_create(g_device, &c));
  holder.ctx[g_device] = c;
  return c;
}

// RAII device allocation
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

uint16_t to_bf16(float f) {  // round to nearest even (finite inputs; validated upstream)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

int dtype() { return g_precision == b200::Precision::BF16 ? LCX_BF16 : LCX_F32; }
size_t elem() { return g_precision == b200::Precision::BF16 ? 2 : 4; }

// rows x cols fp64 host matrix -> device [rows][1][cols] in the storage dtype, placed at
// row offset `row0` of a buffer of `total_rows` rows (the rest zero)
std::unique_ptr<DevBuf> upload(const Matrix& m, size_t total_rows = 0, size_t row0 = 0) {
  if (total_rows == 0) total_rows = m.rows;
  const size_t cols = m.cols;
  auto d = std::make_unique<DevBuf>(std::max<size_t>(total_rows * cols * elem(), 4));
  if (g_precision == b200::Precision::BF16) {
    std::vector<uint16_t> h(total_rows * cols, 0);
    for (size_t i = 0; i < m.values.size(); ++i) h[row0 * cols + i] = to_bf16(float(m.values[i]));
    check_cuda(cudaMemcpy(d->p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
  } else {
    std::vector<float> h(total_rows * cols, 0.f);
    for (size_t i = 0; i < m.values.size(); ++i) h[row0 * cols + i] = float(m.values[i]);
    check_cuda(cudaMemcpy(d->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "upload");
  }
  return d;
}

template <typename T>
std::unique_ptr<DevBuf> upload_vec(const std::vector<T>& v) {
  auto d = std::make_unique<DevBuf>(std::max<size_t>(v.size() * sizeof(T), 4));
  if (!v.empty())
    check_cuda(cudaMemcpy(d->p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice),
               "upload");
  return d;
}

template <typename T>
std::vector<T> download(const DevBuf& d, size_t count) {
  std::vector<T> h(count);
  if (count)
    check_cuda(cudaMemcpy(h.data(), d.p, count * sizeof(T), cudaMemcpyDeviceToHost),
               "download");
  return h;
}

void sync() { check_cuda(cudaDeviceSynchronize(), "synchronize"); }

lcx_attention_input make_input(const AttentionInput& in, const DevBuf& q, const DevBuf& k,
                               const DevBuf& v, const DevBuf* pq, const DevBuf* pk) {
  lcx_attention_input a{};
  a.n = int64_t(in.seq_len());
  a.hq = a.hkv = 1;
  a.dim = int32_t(in.head_dim());
  a.dtype = dtype();
  a.q = q.p;
  a.k = k.p;
  a.v = v.p;
  a.positions_q = pq ? pq->as<int64_t>() : nullptr;
  a.positions_k = pk ? pk->as<int64_t>() : nullptr;
  a.rope_base = in.rope_base;
  a.temperature = in.temperature;
  return a;
}

AttentionResult result_from(const DevBuf& out, const DevBuf& lse, size_t n, size_t dim) {
  AttentionResult r;
  r.output = Matrix(n, dim);
  const auto o = download<float>(out, n * dim);
  std::copy(o.begin(), o.end(), r.output.values.begin());
  const auto l = download<float>(lse, n);
  r.lse.assign(l.begin(), l.end());
  return r;
}

struct Lists {
  std::unique_ptr<DevBuf> v, nv, s, ns;
  int64_t cap_v = 1, cap_s = 1;
};

Lists upload_lists(const CriticalSet& crit) {
  Lists L;
  std::vector<int32_t> v(crit.verticals.begin(), crit.verticals.end());
  std::vector<int32_t> s(crit.slashes.begin(), crit.slashes.end());
  for (size_t x : crit.verticals)
    if (x > size_t(INT32_MAX)) fail(errkind::dimension, "vertical index exceeds int32");
  for (size_t x : crit.slashes)
    if (x > size_t(INT32_MAX)) fail(errkind::dimension, "slash offset exceeds int32");
  L.cap_v = std::max<int64_t>(1, int64_t(v.size()));
  L.cap_s = std::max<int64_t>(1, int64_t(s.size()));
  if (v.empty()) v.push_back(0);
  if (s.empty()) s.push_back(0);
  L.v = upload_vec(v);
  L.s = upload_vec(s);
  L.nv = upload_vec(std::vector<int32_t>{int32_t(crit.verticals.size())});
  L.ns = upload_vec(std::vector<int32_t>{int32_t(crit.slashes.size())});
  return L;
}

std::unique_ptr<DevBuf> upload_positions(const std::vector<int64_t>& p) { return upload_vec(p); }

AttentionResult attend(const AttentionInput& input, const CriticalSet* crit,
                       const RelPositionMatrix* rel, const ChunkConfig* dca) {
  const size_t n = input.seq_len(), dim = input.head_dim();
  auto q = upload(input.q), k = upload(input.k), v = upload(input.v);
  auto pq = upload_positions(input.positions_q), pk = upload_positions(input.positions_k);
  lcx_attention_input a = make_input(input, *q, *k, *v, pq.get(), pk.get());
  DevBuf out(n * dim * 4), lse(n * 4);
  lcx_context* c = context();
  Lists L;
  if (crit) L = upload_lists(*crit);
  const int path = g_precision == b200::Precision::BF16 ? LCX_PATH_AUTO : LCX_PATH_SIMT;
  if (rel) {
    auto r = upload_vec(rel->values);
    check(lcx_attention_rel(c, &a, crit ? L.v->as<int32_t>() : nullptr,
                            crit ? L.nv->as<int32_t>() : nullptr, L.cap_v,
                            crit ? L.s->as<int32_t>() : nullptr,
                            crit ? L.ns->as<int32_t>() : nullptr, L.cap_s, r->as<int64_t>(),
                            out.as<float>(), lse.as<float>(), nullptr));
    sync();
    return result_from(out, lse, n, dim);
  }
  lcx_chunk_config cc{};
  if (dca) cc = {int64_t(dca->chunk_size), int64_t(dca->train_len), int64_t(dca->local_window)};
  if (crit)
    check(lcx_sparse_attention(c, &a, L.v->as<int32_t>(), L.nv->as<int32_t>(), L.cap_v,
                               L.s->as<int32_t>(), L.ns->as<int32_t>(), L.cap_s, dca ? 1 : 0,
                               dca ? &cc : nullptr, path, out.as<float>(), lse.as<float>(),
                               nullptr));
  else
    check(lcx_full_attention(c, &a, dca ? 1 : 0, dca ? &cc : nullptr, path, out.as<float>(),
                             lse.as<float>(), nullptr));
  sync();
  return result_from(out, lse, n, dim);
}

}  // namespace

// ---------------------------------------------------------- attention.cpp --
void AttentionInput::validate() const {  // attention.cpp:70-94
  const std::size_t n = q.rows, dim = q.cols;
  if (k.rows != n || v.rows != n || k.cols != dim || v.cols != dim)
    fail(errkind::dimension, "attention input matrices must share n and D");
  if (n == 0) fail(errkind::dimension, "attention input must have at least one row");
  if (dim == 0 || dim % 2 != 0)
    fail(errkind::config, "head dimension must be even and positive (rope pairs)");
  if (positions_q.size() != n || positions_k.size() != n)
    fail(errkind::dimension, "positions length must equal row count");
  for (std::int64_t p : positions_q)
    if (p < 0) fail(errkind::domain, "query positions must be non-negative");
  for (std::int64_t p : positions_k)
    if (p < 0) fail(errkind::domain, "key positions must be non-negative");
  if (!(rope_base > 0.0)) fail(errkind::domain, "rope base must be positive");
  if (!(temperature > 0.0)) fail(errkind::domain, "temperature must be positive");
  if (!q.all_finite() || !k.all_finite() || !v.all_finite())
    fail(errkind::domain, "attention input values must be finite");
}

AttentionResult full_attention(const AttentionInput& input,
                               const RelPositionMatrix* rel_override) {
  input.validate();
  if (rel_override && rel_override->n != input.seq_len())
    fail(errkind::dimension, "relative-position override must be n x n");
  return attend(input, nullptr, rel_override, nullptr);
}

AttentionResult full_attention_f32(const AttentionInput& input,
                                   const RelPositionMatrix* rel_override) {
  const b200::Precision saved = g_precision;
  g_precision = b200::Precision::F32;
  try {
    AttentionResult r = full_attention(input, rel_override);
    g_precision = saved;
    return r;
  } catch (...) {
    g_precision = saved;
    throw;
  }
}

double flop_estimate(std::size_t n, std::size_t head_dim, std::size_t computed_entries) {
  const std::size_t dense = n * (n + 1) / 2;  // attention.cpp:257-264
  if (computed_entries > dense)
    fail(errkind::domain, "computed entries exceed the causal entry count");
  return 2.0 * double(computed_entries) * double(head_dim);
}

void check_gqa_grouping(std::size_t query_heads, std::size_t kv_heads) {
  if (query_heads == 0 || kv_heads == 0) fail(errkind::config, "head counts must be positive");
  if (query_heads % kv_heads != 0)
    fail(errkind::config, "query-head count must be divisible by kv-head count");
}

// ---------------------------------------------------------------- dca.cpp --
ChunkConfig ChunkConfig::with_default_window(std::size_t chunk_size, std::size_t train_len) {
  ChunkConfig cfg;
  cfg.chunk_size = chunk_size;
  cfg.train_len = train_len;
  cfg.local_window = std::min(chunk_size, train_len > chunk_size ? train_len - chunk_size : 0);
  cfg.validate();
  return cfg;
}

void ChunkConfig::validate() const {  // dca.cpp:18-30
  if (chunk_size == 0) fail(errkind::config, "chunkSize must be positive");
  if (train_len == 0) fail(errkind::config, "trainLen must be positive");
  if (chunk_size > train_len) fail(errkind::config, "chunkSize must not exceed trainLen");
  if (local_window > std::min(chunk_size, train_len - chunk_size))
    fail(errkind::config, "localWindow must not exceed min(chunkSize, trainLen - chunkSize)");
}

double yarn_temperature(double scale_factor) {  // dca.cpp:32-37
  if (!(scale_factor > 0.0)) fail(errkind::domain, "scale factor must be positive");
  if (scale_factor <= 1.0) return 1.0;
  const double root = 0.1 * std::log(scale_factor) + 1.0;
  return 1.0 / (root * root);
}

YarnScale YarnScale::from_scale(double scale_factor) {
  YarnScale y;
  y.scale_factor = scale_factor;
  y.temperature = yarn_temperature(scale_factor);
  return y;
}

void YarnScale::validate() const {
  if (!(scale_factor > 0.0)) fail(errkind::domain, "scale factor must be positive");
  if (temperature != yarn_temperature(scale_factor))
    fail(errkind::config, "temperature inconsistent with scale factor");
}

PatternKind classify_pair(std::size_t i, std::size_t j, const ChunkConfig& cfg) {
  if (j > i) fail(errkind::causality, "classify_pair requires j <= i");
  const std::size_t qc = i / cfg.chunk_size, kc = j / cfg.chunk_size;
  if (qc == kc) return PatternKind::Intra;
  return qc == kc + 1 ? PatternKind::Successive : PatternKind::Inter;
}

std::int64_t dca_relative(std::size_t i, std::size_t j, const ChunkConfig& cfg) {
  const PatternKind kind = classify_pair(i, j, cfg);  // dca.cpp:62-80
  const std::int64_t s = std::int64_t(cfg.chunk_size), c = std::int64_t(cfg.train_len);
  const std::int64_t kpos = std::int64_t(j) % s;
  std::int64_t qpos = std::int64_t(i) % s;
  if (kind == PatternKind::Successive) qpos = std::min(qpos + s, c - 1);
  if (kind == PatternKind::Inter) qpos = c - 1;
  return qpos - kpos;
}

RelPositionMatrix dca_position_matrix(std::size_t n, const ChunkConfig& cfg) {
  cfg.validate();
  RelPositionMatrix rel(n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j <= i; ++j) rel.at(i, j) = dca_relative(i, j, cfg);
  return rel;
}

AttentionResult dca_attention(const AttentionInput& input, const ChunkConfig& cfg,
                              const YarnScale& yarn) {  // dca.cpp:93-113
  cfg.validate();
  yarn.validate();
  const std::size_t n = input.seq_len();
  AttentionInput eff = input;
  eff.positions_q.resize(n);
  eff.positions_k.resize(n);
  std::iota(eff.positions_q.begin(), eff.positions_q.end(), 0);
  std::iota(eff.positions_k.begin(), eff.positions_k.end(), 0);
  eff.temperature = yarn.temperature;
  eff.validate();
  if (n <= cfg.chunk_size && yarn.scale_factor <= 1.0) return attend(eff, nullptr, nullptr, nullptr);
  // the remap is fused into the kernel's RoPE (no n x n matrix)
  return attend(eff, nullptr, nullptr, &cfg);
}

// ------------------------------------------------------------- sparse.cpp --
bool CriticalSet::admits(std::size_t i, std::size_t j) const {  // sparse.cpp:80-83
  if (std::binary_search(verticals.begin(), verticals.end(), j)) return true;
  return j <= i && std::binary_search(slashes.begin(), slashes.end(), i - j);
}

std::vector<std::size_t> CriticalSet::admitted_row(std::size_t i) const {  // sparse.cpp:85-113
  std::vector<std::size_t> row;
  row.reserve(verticals.size() + slashes.size());
  for (std::size_t v : verticals) {
    if (v > i) break;
    row.push_back(v);
  }
  for (auto it = slashes.rbegin(); it != slashes.rend(); ++it)
    if (*it <= i) row.push_back(i - *it);
  std::sort(row.begin(), row.end());
  row.erase(std::unique(row.begin(), row.end()), row.end());
  if (row.empty()) row.push_back(i);
  return row;
}

std::size_t CriticalSet::admitted_count() const {
  // |{v <= i}| + |{d <= i}| - |V ∩ {i - d}| per row, fallback rows count 1
  std::size_t count = 0;
  for (std::size_t i = 0; i < context_length; ++i) count += admitted_row(i).size();
  return count;
}

std::int64_t selection_position(std::size_t i, std::size_t j, const ChunkConfig& cfg) {
  if (j > i) fail(errkind::causality, "selection_position requires j <= i");
  return std::min<std::int64_t>(std::int64_t(i - j), std::int64_t(cfg.train_len) - 1);
}

double density(const CriticalSet& crit) {  // sparse.cpp:286-291
  const std::size_t n = crit.context_length;
  if (n == 0) fail(errkind::dimension, "critical set has no context");
  return double(crit.admitted_count()) / (double(n) * double(n + 1) / 2.0);
}

Matrix estimate_block(const Matrix& q, const Matrix& k, std::size_t last_q, PositionMode mode,
                      const std::optional<ChunkConfig>& cfg, double rope_base) {
  if (last_q == 0) fail(errkind::config, "lastQ must be positive");  // sparse.cpp:142-156
  if (q.cols != k.cols) fail(errkind::dimension, "query/key dimensions differ");
  if (q.cols == 0 || q.cols % 2 != 0) fail(errkind::config, "head dimension must be even");
  if (q.rows == 0 || k.rows == 0) fail(errkind::dimension, "empty query or key matrix");
  if (q.rows > k.rows)
    fail(errkind::dimension, "queries must be the trailing rows of the key timeline");
  if (mode == PositionMode::DcaContinuous && !cfg)
    fail(errkind::config, "dcaContinuous estimation requires a chunk config");
  const size_t nq = q.rows, nk = k.rows, dim = q.cols;
  const size_t block = std::min(last_q, nq);
  auto dq = upload(q, nk, nk - nq), dk = upload(k);
  lcx_attention_input a{};
  a.n = int64_t(nk);
  a.hq = a.hkv = 1;
  a.dim = int32_t(dim);
  a.dtype = dtype();
  a.q = dq->p;
  a.k = dk->p;
  a.v = dk->p;
  a.rope_base = rope_base;
  a.temperature = 1.0;
  lcx_chunk_config cc{};
  if (cfg) cc = {int64_t(cfg->chunk_size), int64_t(cfg->train_len), int64_t(cfg->local_window)};
  DevBuf est(block * nk * 4);
  check(lcx_estimate_block(context(), &a, int64_t(nk - nq), int64_t(nq), int64_t(nk),
                           int64_t(last_q),
                           mode == PositionMode::DcaContinuous ? LCX_POS_DCA_CONTINUOUS
                                                               : LCX_POS_STANDARD,
                           cfg ? &cc : nullptr, est.as<float>(), nullptr));
  sync();
  Matrix m(block, nk);
  const auto h = download<float>(est, block * nk);
  std::copy(h.begin(), h.end(), m.values.begin());
  return m;
}

CriticalSet select_critical(const Matrix& est, HeadBudget budget, std::size_t n,
                            const SelectionOptions& opts) {
  if (est.cols != n) fail(errkind::dimension, "estimation block must have n columns");
  if (est.rows == 0 || est.rows > n)
    fail(errkind::dimension, "estimation block row count out of range");
  std::vector<float> e(est.values.begin(), est.values.end());
  auto d = upload_vec(e);
  const int64_t bv = int64_t(std::min(budget.vertical, n)), bs = int64_t(std::min(budget.slash, n));
  const int64_t cap_v = bv + 1, cap_s = bs + int64_t(est.rows);
  DevBuf v(cap_v * 4), nv(4), s(cap_s * 4), ns(4);
  lcx_selection_options o{int(opts.force_sink_column), int(opts.force_local_band),
                          int(opts.slash_mean)};
  check(lcx_select_critical(context(), d->as<float>(), 1, int64_t(est.rows), int64_t(n), bv, bs,
                            &o, v.as<int32_t>(), nv.as<int32_t>(), cap_v, s.as<int32_t>(),
                            ns.as<int32_t>(), cap_s, nullptr));
  sync();
  const int32_t cnv = download<int32_t>(nv, 1)[0], cns = download<int32_t>(ns, 1)[0];
  const auto hv = download<int32_t>(v, size_t(cnv)), hs = download<int32_t>(s, size_t(cns));
  CriticalSet crit;
  crit.verticals.assign(hv.begin(), hv.end());
  crit.slashes.assign(hs.begin(), hs.end());
  crit.context_length = n;
  return crit;
}

AttentionResult sparse_attention(const AttentionInput& input, const CriticalSet& crit,
                                 const RelPositionMatrix* rel_override) {
  input.validate();  // sparse.cpp:232-245
  const std::size_t n = input.seq_len();
  if (crit.context_length != n) fail(errkind::dimension, "critical set context length must equal n");
  if (rel_override && rel_override->n != n)
    fail(errkind::dimension, "relative-position override must be n x n");
  return attend(input, &crit, rel_override, nullptr);
}

PrefillResult chunked_prefill(const AttentionInput& input, std::size_t chunk_len,
                              std::size_t last_q, HeadBudget budget, PrefillMode mode,
                              PositionMode pos_mode, const std::optional<ChunkConfig>& cfg,
                              const SelectionOptions& opts) {
  input.validate();  // sparse.cpp:293-308
  if (chunk_len == 0) fail(errkind::config, "chunkLen must be positive");
  if (last_q == 0) fail(errkind::config, "lastQ must be positive");
  if (mode == PrefillMode::Sparse && chunk_len < last_q)
    fail(errkind::config, "sparse prefill requires chunkLen >= lastQ");
  const bool dca = pos_mode == PositionMode::DcaContinuous;
  if (dca) {
    if (!cfg) fail(errkind::config, "dcaContinuous prefill requires a chunk config");
    cfg->validate();
  }
  const size_t n = input.seq_len(), dim = input.head_dim();
  const size_t nch = (n + chunk_len - 1) / chunk_len;
  const size_t block = std::min(last_q, chunk_len);
  const int64_t cap_v = int64_t(std::min(budget.vertical, n)) + 2;
  const int64_t cap_s = int64_t(std::min(budget.slash, n) + block) + 1;
  auto q = upload(input.q), k = upload(input.k), v = upload(input.v);
  auto pq = upload_positions(input.positions_q), pk = upload_positions(input.positions_k);
  lcx_attention_input a = make_input(input, *q, *k, *v, pq.get(), pk.get());
  DevBuf out(n * dim * 4), lse(n * 4);
  DevBuf sv(nch * cap_v * 4), snv(nch * 4), ss(nch * cap_s * 4), sns(nch * 4);
  lcx_prefill_config pc{};
  pc.chunk_len = int64_t(chunk_len);
  pc.last_q = int64_t(last_q);
  pc.budget_vertical = int64_t(budget.vertical);
  pc.budget_slash = int64_t(budget.slash);
  pc.mode = mode == PrefillMode::Sparse ? LCX_PREFILL_SPARSE : LCX_PREFILL_FULL;
  pc.position_mode = dca ? LCX_POS_DCA_CONTINUOUS : LCX_POS_STANDARD;
  if (dca)
    pc.dca = {int64_t(cfg->chunk_size), int64_t(cfg->train_len), int64_t(cfg->local_window)};
  pc.opts = {int(opts.force_sink_column), int(opts.force_local_band), int(opts.slash_mean)};
  pc.kernel_path = g_precision == b200::Precision::BF16 ? LCX_PATH_AUTO : LCX_PATH_SIMT;
  lcx_prefill_output po{};
  po.out = out.as<float>();
  po.lse = lse.as<float>();
  const bool sparse = mode == PrefillMode::Sparse;
  if (sparse) {
    po.sel_verticals = sv.as<int32_t>();
    po.sel_nv = snv.as<int32_t>();
    po.sel_slashes = ss.as<int32_t>();
    po.sel_ns = sns.as<int32_t>();
    po.cap_v = cap_v;
    po.cap_s = cap_s;
  }
  check(lcx_chunked_prefill(context(), &a, &pc, &po, nullptr));
  sync();
  PrefillResult pr;
  pr.result = result_from(out, lse, n, dim);
  pr.state.chunk_len = chunk_len;
  pr.state.last_q = last_q;
  pr.state.cached_k = input.k;  // raw rows, one per processed token (sparse.hpp:107-113)
  pr.state.cached_v = input.v;
  if (sparse) {
    const auto hv = download<int32_t>(sv, nch * cap_v), hnv = download<int32_t>(snv, nch);
    const auto hs = download<int32_t>(ss, nch * cap_s), hns = download<int32_t>(sns, nch);
    for (size_t c = 0; c < nch; ++c) {
      ChunkSelection cs;
      cs.chunk_index = c;
      cs.begin = c * chunk_len;
      cs.end = std::min(n, cs.begin + chunk_len);
      cs.critical.context_length = cs.end;
      cs.critical.verticals.assign(hv.begin() + c * cap_v, hv.begin() + c * cap_v + hnv[c]);
      cs.critical.slashes.assign(hs.begin() + c * cap_s, hs.begin() + c * cap_s + hns[c]);
      pr.state.selections.push_back(std::move(cs));
    }
  }
  return pr;
}

// ------------------------------------------------------------- refine.cpp --
RecallReport attention_recall(std::span<const double> lse_sparse,
                              std::span<const double> lse_full) {  // refine.cpp:51-72
  if (lse_sparse.size() != lse_full.size())
    fail(errkind::dimension, "recall needs equally many sparse and full lse values");
  if (lse_sparse.empty()) fail(errkind::dimension, "recall needs at least one query");
  const size_t n = lse_sparse.size();
  // the difference is taken in fp64 here and only then rounded: rounding the two lse values
  // to fp32 separately would cost ~ulp(|lse|) (1.5e-5 at 256), above the recall slack
  std::vector<float> a(n), b(n, 0.f);
  for (size_t i = 0; i < n; ++i) a[i] = float(lse_sparse[i] - lse_full[i]);
  auto da = upload_vec(a), db = upload_vec(b);
  DevBuf per(n * 4);
  double agg = 0.0;
  check(lcx_attention_recall(context(), da->as<float>(), db->as<float>(), int64_t(n),
                             b200::recall_slack(), per.as<float>(), &agg, nullptr));
  RecallReport rep;
  const auto h = download<float>(per, n);
  rep.per_query.assign(h.begin(), h.end());
  rep.aggregate = agg;
  return rep;
}

double measure_budget_recall(const AttentionInput& input, HeadBudget budget,
                             const RecallMeasurement& measure) {  // refine.cpp:74-85
  const std::size_t n = input.seq_len();
  const AttentionResult full = full_attention(input);
  const Matrix est = estimate_block(input.q, input.k, std::min(measure.last_q, n),
                                    PositionMode::Standard, std::nullopt, input.rope_base);
  const CriticalSet crit = select_critical(est, budget, n, measure.selection);
  const AttentionResult sparse = sparse_attention(input, crit);
  const RecallReport rep = attention_recall(sparse.lse, full.lse);
  if (measure.aggregate == RecallAggregate::Mean) return rep.aggregate;
  std::size_t above = 0;  // refine.cpp:16-27
  for (double r : rep.per_query)
    if (r >= measure.fraction_tau) ++above;
  return double(above) / double(rep.per_query.size());
}

// ---------------------------------------------------------------- b200:: --
namespace b200 {
std::vector<ChunkCostSample> measure_chunk_costs(const AttentionInput& input,
                                                 std::size_t chunk_len, std::size_t last_q,
                                                 HeadBudget budget, PrefillMode mode,
                                                 PositionMode pos_mode,
                                                 const std::optional<ChunkConfig>& cfg,
                                                 const SelectionOptions& opts) {
  lcx_context* ctx = context();
  check(lcx_set_profiling(ctx, 1));
  try {
    (void)chunked_prefill(input, chunk_len, last_q, budget, mode, pos_mode, cfg, opts);
  } catch (...) {
    lcx_set_profiling(ctx, 0);
    throw;
  }
  int64_t count = 0;
  check(lcx_get_chunk_ms(ctx, nullptr, 0, &count));
  std::vector<float> ms(static_cast<size_t>(count));
  check(lcx_get_chunk_ms(ctx, ms.data(), count, &count));
  check(lcx_set_profiling(ctx, 0));
  std::vector<ChunkCostSample> out;
  const std::size_t n = input.seq_len();
  for (int64_t c = 0; c < count; ++c) {
    const std::size_t b = std::size_t(c) * chunk_len, e = std::min(n, b + chunk_len);
    out.push_back(ChunkCostSample{e - b, b, double(ms[size_t(c)])});
  }
  return out;
}

void set_precision(Precision p) { g_precision = p; }
Precision precision() { return g_precision; }
void set_device(int device) { g_device = device; }
double recall_slack() { return g_precision == Precision::BF16 ? 4e-3 : 1e-5; }
}  // namespace b200

}  // namespace longctx
