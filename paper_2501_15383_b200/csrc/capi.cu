// C-ABI implementation and per-layer orchestration (include/longctx_b200.h).
//
// lcx_chunked_prefill restates chunked_prefill (reference core/src/sparse.cpp:
// 293-399): for each chunk [t0, t1) the estimator scores the chunk's trailing
// min(last_q, t1 - t0) rows against keys [0, t1), the selection keeps the top
// vertical / slash lines over the t1-key context (one CriticalSet per chunk and
// head), and the attention computes rows [t0, t1) over their admitted entries.
// With Q/K/V given, a chunk depends only on K/V[0:t1]; chunks are issued
// back-to-back on one stream, each launch covering every head.
#include <cstdio>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "attn_gather.cuh"
#include "est_tc.cuh"
#include "attn_tc.cuh"
#include "lcx_internal.cuh"

namespace lcx {

thread_local std::string g_err;
thread_local long long g_launches = 0;
void set_error(const std::string& msg) { g_err = msg; }

int build_rope_table(const double* thetas_dev, int P, int64_t npos, float2* out,
                     cudaStream_t st);

int ensure_workspace(lcx_context* ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return LCX_OK;
  if (ctx->ws) LCX_CHECK_CUDA(cudaFree(ctx->ws));  // implicit device sync
  ctx->ws = nullptr;
  ctx->ws_bytes = 0;
  const size_t want = bytes + bytes / 8 + (1 << 20);
  LCX_CHECK_CUDA(cudaMalloc(&ctx->ws, want));
  ctx->ws_bytes = want;
  return LCX_OK;
}

int ensure_rope(lcx_context* ctx, double base, int dim, int64_t P, cudaStream_t st) {
  if (ctx->rope && ctx->rope_base == base && ctx->rope_dim == dim && ctx->rope_P >= P)
    return LCX_OK;
  if (ctx->rope) LCX_CHECK_CUDA(cudaFree(ctx->rope));
  ctx->rope = nullptr;
  const int pairs = dim / 2;
  const int64_t npos = std::max<int64_t>(P, 128);  // the gather's low table needs 64 rows
  std::vector<double> th(pairs);
  for (int p = 0; p < pairs; ++p) th[p] = std::pow(base, -double(2 * p) / double(dim));
  double* th_dev = nullptr;
  LCX_CHECK_CUDA(cudaMalloc(&th_dev, sizeof(double) * pairs));
  LCX_CHECK_CUDA(cudaMemcpy(th_dev, th.data(), sizeof(double) * pairs, cudaMemcpyHostToDevice));
  LCX_CHECK_CUDA(cudaMalloc(&ctx->rope, sizeof(float2) * size_t(npos) * pairs));
  LCX_TRY(build_rope_table(th_dev, pairs, npos, ctx->rope, st));
  LCX_CHECK_CUDA(cudaStreamSynchronize(st));
  LCX_CHECK_CUDA(cudaFree(th_dev));
  ctx->rope_base = base;
  ctx->rope_dim = dim;
  ctx->rope_P = npos;
  return LCX_OK;
}

namespace {

// slash entries a 64-key relative tile needs to go to tcgen05 rather than the gather:
// profiles/r02/sweep_tcmin_r02.jsonl (1M, 7B): planted flat over 32-160 (482-494 ms),
// structured 5990 -> 5897 ms and iid 8262 -> 7860 ms from 96 to 160, worse again at 192;
// re-swept with the batched gather (sweep_tcmin_r02_gather_batch.jsonl): still the optimum
// for iid / structured (7041 / 5438 ms), planted flat over 160-192 (470 / 469 ms)
constexpr int kDefaultTcMin = 160;
constexpr int64_t kGatherSegment = 32768;  // keys per gather pass (L2-resident K / V)
constexpr int64_t kTcSegment = 32768;      // keys per tcgen05 slash pass (K hi/lo + V^T)
constexpr int64_t kWindowMinSlashes = 512;  // slash capacity from which windows are used

__global__ void dense_count_kernel(int hq, int64_t t0, int64_t t1, int64_t* out) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < hq) out[h] = (t1 * (t1 + 1) - t0 * (t0 + 1)) / 2;  // sum_{i=t0}^{t1-1} (i + 1)
}

// Line sharding: shard r of G keeps the contiguous part [r cnt / G, (r+1) cnt / G) of each
// head's sorted vertical and slash lists (clustered slashes stay together, so dense slash
// runs still become tensor-core tiles on their shard).
__global__ void shard_lists_kernel(const int32_t* __restrict__ v, const int32_t* __restrict__ nv,
                                   int64_t cap_v, const int32_t* __restrict__ sl,
                                   const int32_t* __restrict__ ns, int64_t cap_s, int rank,
                                   int shards, int32_t* __restrict__ ov, int32_t* __restrict__ onv,
                                   int32_t* __restrict__ os, int32_t* __restrict__ ons) {
  const int h = blockIdx.x;
  const int64_t cv = nv[h], cs = ns[h];
  const int64_t v0 = cv * rank / shards, v1 = cv * (rank + 1) / shards;
  const int64_t s0 = cs * rank / shards, s1 = cs * (rank + 1) / shards;
  for (int64_t x = threadIdx.x; x < v1 - v0; x += blockDim.x)
    ov[h * cap_v + x] = v[h * cap_v + v0 + x];
  for (int64_t x = threadIdx.x; x < s1 - s0; x += blockDim.x)
    os[h * cap_s + x] = sl[h * cap_s + s0 + x];
  if (threadIdx.x == 0) {
    onv[h] = int32_t(v1 - v0);
    ons[h] = int32_t(s1 - s0);
  }
}

// far[0] += slashes with d >= far_d, far[1] += all slashes (over heads)
__global__ void store_ints_kernel(const int* __restrict__ src, int* dst, int count) {
  if (int(threadIdx.x) < count) dst[threadIdx.x] = src[threadIdx.x];
  __threadfence_system();
}

__global__ void far_count_kernel(const int32_t* __restrict__ sl, const int32_t* __restrict__ ns,
                                 int64_t cap_s, int64_t far_d, int* far) {
  const int h = blockIdx.x;  // one block per head
  const int cnt = ns[h];
  int f = 0;
  for (int x = threadIdx.x; x < cnt; x += blockDim.x) f += sl[int64_t(h) * cap_s + x] >= far_d;
  f = __reduce_add_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicAdd(far, f);
  if (threadIdx.x == 0) atomicAdd(far + 1, cnt);
}

int dense_counts(int hq, int64_t t0, int64_t t1, int64_t* out, cudaStream_t st) {
  dense_count_kernel<<<(hq + 127) / 128, 128, 0, st>>>(hq, t0, t1, out);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

__global__ void max_pos_kernel(const int64_t* a, const int64_t* b, int64_t n,
                               unsigned long long* out, int* neg) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = a ? a[i] : i, y = b ? b[i] : i;
    if (x < 0 || y < 0) atomicExch(neg, 1);
    const int64_t m = x > y ? x : y;
    atomicMax(out, (unsigned long long)(m < 0 ? 0 : m));
  }
}

__global__ void max_abs_kernel(const int64_t* a, int64_t n, unsigned long long* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = a[i] < 0 ? -a[i] : a[i];
    atomicMax(out, (unsigned long long)x);
  }
}

int validate_input(const lcx_attention_input* in) {
  if (!in) return fail(LCX_ERR_DIMENSION, "null attention input");
  if (in->n <= 0) return fail(LCX_ERR_DIMENSION, "attention input must have at least one row");
  if (in->dim <= 0 || in->dim % 2 != 0)
    return fail(LCX_ERR_CONFIG, "head dimension must be even and positive (rope pairs)");
  if (in->dim > 128) return fail(LCX_ERR_CONFIG, "head dimension > 128 is not supported");
  if (in->hq <= 0 || in->hkv <= 0) return fail(LCX_ERR_CONFIG, "head counts must be positive");
  if (in->hq % in->hkv != 0)
    return fail(LCX_ERR_CONFIG, "query-head count must be divisible by kv-head count");
  if (!(in->rope_base > 0.0)) return fail(LCX_ERR_DOMAIN, "rope base must be positive");
  if (!(in->temperature > 0.0)) return fail(LCX_ERR_DOMAIN, "temperature must be positive");
  if (in->dtype != LCX_F32 && in->dtype != LCX_BF16) return fail(LCX_ERR_CONFIG, "bad dtype");
  if (!in->q || !in->k || !in->v) return fail(LCX_ERR_DIMENSION, "null q/k/v pointer");
  return LCX_OK;
}

int validate_chunk(const lcx_chunk_config* c) {
  if (!c) return fail(LCX_ERR_CONFIG, "dca requires a chunk config");
  if (c->chunk_size <= 0) return fail(LCX_ERR_CONFIG, "chunkSize must be positive");
  if (c->train_len <= 0) return fail(LCX_ERR_CONFIG, "trainLen must be positive");
  if (c->chunk_size > c->train_len)
    return fail(LCX_ERR_CONFIG, "chunkSize must not exceed trainLen");
  const int64_t bound = std::min(c->chunk_size, c->train_len - c->chunk_size);
  if (c->local_window > bound)
    return fail(LCX_ERR_CONFIG,
                "localWindow must not exceed min(chunkSize, trainLen - chunkSize)");
  return LCX_OK;
}

// Largest rotation position any kernel will look up for this input.
int max_position(lcx_context* ctx, const lcx_attention_input* in, int64_t* out,
                 cudaStream_t st) {
  if (!in->positions_q && !in->positions_k) {
    *out = in->n - 1;
    return LCX_OK;
  }
  unsigned long long* dmax = nullptr;
  int* dneg = nullptr;
  LCX_CHECK_CUDA(cudaMallocAsync(&dmax, sizeof(unsigned long long), st));
  LCX_CHECK_CUDA(cudaMallocAsync(&dneg, sizeof(int), st));
  LCX_CHECK_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
  LCX_CHECK_CUDA(cudaMemsetAsync(dneg, 0, sizeof(int), st));
  max_pos_kernel<<<64, 256, 0, st>>>(in->positions_q, in->positions_k, in->n, dmax, dneg);
  LCX_CHECK_LAUNCH();
  unsigned long long hmax = 0;
  int hneg = 0;
  LCX_CHECK_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof(hmax), cudaMemcpyDeviceToHost, st));
  LCX_CHECK_CUDA(cudaMemcpyAsync(&hneg, dneg, sizeof(hneg), cudaMemcpyDeviceToHost, st));
  LCX_CHECK_CUDA(cudaStreamSynchronize(st));
  LCX_CHECK_CUDA(cudaFreeAsync(dmax, st));
  LCX_CHECK_CUDA(cudaFreeAsync(dneg, st));
  if (hneg) return fail(LCX_ERR_DOMAIN, "positions must be non-negative");
  *out = int64_t(hmax);
  (void)ctx;
  return LCX_OK;
}

AttnArgs base_attn(const lcx_attention_input* in, lcx_context* ctx) {
  AttnArgs a{};
  a.q = in->q;
  a.k = in->k;
  a.v = in->v;
  a.dtype = in->dtype;
  a.hq = in->hq;
  a.hkv = in->hkv;
  a.dim = in->dim;
  a.pos_q = in->positions_q;
  a.pos_k = in->positions_k;
  a.scale = float(1.0 / (in->temperature * std::sqrt(double(in->dim))));
  a.rope = ctx->rope;
  a.rope_P = ctx->rope_P;
  return a;
}

EstimateArgs base_est(const lcx_attention_input* in, lcx_context* ctx, int64_t q_row0,
                      int64_t nq, int64_t nk, int64_t last_q, int pos_mode, int64_t c) {
  EstimateArgs e{};
  e.q = in->q;
  e.k = in->k;
  e.dtype = in->dtype;
  e.hq = in->hq;
  e.hkv = in->hkv;
  e.dim = in->dim;
  e.q_row0 = q_row0;
  e.nq = nq;
  e.nk = nk;
  e.block = std::min(last_q, nq);
  e.pos_mode = pos_mode;
  e.c = c;
  e.rope = ctx->rope;
  return e;
}


// ---------------------------------------------------------------------------
// Attention stage shared by sparse_attention / full_attention / chunked_prefill.
// Path: tcgen05 tiles (+ CUDA-core gather for isolated slashes) when the input is
// bf16 with dim 128, the chunk boundaries are 128-aligned and DCA chunks are
// multiples of 128; otherwise the exact CUDA-core path for every entry.
struct FullLists {
  const int32_t* verts; const int32_t* nv; const int32_t* slashes; const int32_t* ns;
  int do_fallback;
};

struct AttnWS {
  bool tc = false;
  int64_t words = 0, U = 0, cap_u = 0, cap_seg = 0;
  uint32_t* vbits = nullptr;
  uint32_t* sbits = nullptr;
  int32_t* hist = nullptr;
  int32_t* tc_u = nullptr;
  int32_t* n_tc_u = nullptr;
  int4* segs = nullptr;
  int32_t* nseg = nullptr;
  bool windows = false;      // key-window passes for this chunk (see prefill_impl)
  int* tc_flags = nullptr;   // per key window: slash tiles present
  int* g_flags = nullptr;    // per key window: gather segments present
  int nwin = 0;
  void* plans = nullptr;
  TcBuffers B;
};

template <class A>
void attn_layout(A& ar, const lcx_attention_input* in, bool tc, bool sparse, int64_t cap_v,
                 int64_t cap_s, int64_t seg_len, AttnWS& w) {
  w.tc = tc;
  w.words = (in->n + 31) / 32 + 4;
  if (sparse) {
    w.vbits = ar.template take<uint32_t>(size_t(in->hq) * w.words);
    if (tc) {
      w.sbits = ar.template take<uint32_t>(size_t(in->hq) * w.words);
      w.U = in->n / 64 + 4;
      w.cap_u = w.U;
      w.cap_seg = cap_s;  // per 64-row half: at most one segment per diagonal
      w.hist = ar.template take<int32_t>(size_t(in->hq) * w.U);
      w.tc_u = ar.template take<int32_t>(size_t(in->hq) * w.cap_u);
      w.n_tc_u = ar.template take<int32_t>(size_t(in->hq));
      w.segs = ar.template take<int4>(size_t(in->hq) * 2 * w.cap_seg);
      w.nseg = ar.template take<int32_t>(size_t(in->hq) * 2);
      w.nwin = int(in->n / kTcSegment + 2);
      w.tc_flags = ar.template take<int>(size_t(w.nwin));
      w.g_flags = ar.template take<int>(size_t(w.nwin));
    }
  }
  if (tc) {
    tc_layout(ar, in->n, in->hq, in->hkv, sparse ? cap_v : 0, seg_len, w.B);
    // one plan per (head, 128-row block) of the largest chunk (<= the whole input)
    w.plans = ar.template take<uint8_t>(size_t(in->hq) * ((in->n + 127) / 128 + 1) *
                                        tc_plan_bytes());
  }
}

bool tc_eligible(const lcx_attention_input* in, int64_t chunk_len, bool dca, int64_t s) {
  if (in->dtype != LCX_BF16 || in->dim != 128) return false;
  if (chunk_len % 128 != 0) return false;
  if (dca && s % 128 != 0) return false;
  if (in->n >= (int64_t(1) << 31)) return false;
  return true;
}

int resolve_path(int32_t kernel_path, const lcx_attention_input* in, int64_t chunk_len, bool dca,
                 int64_t s, bool* tc) {
  const bool ok = tc_eligible(in, chunk_len, dca, s);
  if (kernel_path == LCX_PATH_TC && !ok)
    return fail(LCX_ERR_CONFIG,
                "tcgen05 path needs bf16 q/k/v, head dim 128, 128-aligned chunks and DCA "
                "chunk size");
  *tc = (kernel_path == LCX_PATH_AUTO || kernel_path == LCX_PATH_TC) && ok;
  if (kernel_path == LCX_PATH_AUTO && !ok && in->dtype == LCX_BF16 && in->dim == 128) {
    static bool warned = false;  // the bf16 tensor-core path needs 128-aligned chunks
    if (!warned) {
      warned = true;
      std::fprintf(stderr,
                   "longctx_b200: bf16 prefill on the CUDA-core kernels (chunk length %lld%s"
                   " not a multiple of 128): the tcgen05 path is several times faster\n",
                   (long long)chunk_len, dca ? " or DCA chunk size" : "");
    }
  }
  return LCX_OK;
}

// rows [t0, t1) over keys [0, t1) with the given per-head lists (sparse) or dense.
int attention_chunk(lcx_context* ctx, const lcx_attention_input* in, AttnWS& w, int64_t t0,
                    int64_t t1, bool sparse, const int32_t* verts, const int32_t* nv,
                    int64_t cap_v, const int32_t* slashes, const int32_t* ns, int64_t cap_s,
                    bool dca, int64_t s, int64_t c, int tc_min_entries, float* out, float* lse,
                    int64_t lse_stride, int64_t* admitted, cudaStream_t st,
                    cudaEvent_t ev_tc0 = nullptr, cudaEvent_t ev_tc1 = nullptr,
                    const FullLists* full = nullptr) {
  const int hq = in->hq;
  // line sharding: (verts, slashes) are this rank's lines; the full selection decides
  // V∩S ownership (vertical bitmap) and the self-fallback rows (rank 0 only)
  const int32_t* fv = full ? full->verts : verts;
  const int32_t* fnv = full ? full->nv : nv;
  const int32_t* fs = full ? full->slashes : slashes;
  const int32_t* fns = full ? full->ns : ns;
  const int do_fallback = full ? full->do_fallback : 1;
  if (sparse) LCX_TRY(build_bitmaps(fv, fnv, cap_v, hq, w.words, w.vbits, st));
  if (!w.tc) {
    AttnArgs a = base_attn(in, ctx);
    a.n = t1;
    a.row_begin = t0;
    a.row_end = t1;
    a.rel_mode = dca ? 1 : 0;
    a.s = dca ? s : 1;
    a.c = dca ? c : 1;
    a.dense = sparse ? 0 : 1;
    a.verts = verts;
    a.nv = nv;
    a.cap_v = cap_v;
    a.slashes = slashes;
    a.ns = ns;
    a.cap_s = cap_s;
    a.vbits = w.vbits;
    a.bit_words = w.words;
    a.fverts = fv;
    a.fnv = fnv;
    a.fslashes = fs;
    a.fns = fns;
    a.do_fallback = do_fallback;
    a.out = out;
    a.lse = lse;
    a.lse_stride = lse_stride;
    a.admitted = full && admitted ? nullptr : admitted;
    a.simt_count = ctx->profiling ? ctx->tile_counter + 1 : nullptr;
    LCX_TRY(attention_simt(a, st));
    if (full && admitted) {
      if (do_fallback)
        LCX_TRY(admitted_counts(fv, fnv, cap_v, fs, fns, cap_s, hq, t0, t1, admitted, st));
      else
        LCX_CHECK_CUDA(cudaMemsetAsync(admitted, 0, sizeof(int64_t) * hq, st));
    }
    return LCX_OK;
  }
  if (sparse) {
    LCX_TRY(build_bitmaps(slashes, ns, cap_s, hq, w.words, w.sbits, st));
    LCX_TRY(tc_compact(in->v, hq, in->hkv, verts, nv, cap_v, w.B, st));
    const int64_t U = t1 / 64 + 4;
    LCX_TRY(tc_classify(slashes, ns, cap_s, hq, std::min(U, w.U), tc_min_entries, w.hist,
                        w.tc_u, w.n_tc_u, w.cap_u, w.segs, w.nseg, w.cap_seg, st));
    if (w.windows)
      LCX_TRY(tc_window_flags(w.tc_u, w.n_tc_u, w.cap_u, w.segs, w.nseg, w.cap_seg, hq, t0, t1,
                              kTcSegment, w.nwin, w.tc_flags, w.g_flags, st));
  }
  TcParams p{};
  p.q = reinterpret_cast<const __nv_bfloat16*>(in->q);
  p.hq = hq;
  p.hkv = in->hkv;
  p.group = hq / in->hkv;
  p.n = t1;
  p.t1 = t1;
  p.block0 = t0 / 128;
  p.nblocks = int((t1 - t0 + 127) / 128);
  p.nitems = p.nblocks * hq;
  p.rel_mode = dca ? 1 : 0;
  p.s = dca ? s : 1;
  p.c = dca ? c : 1;
  p.pos_q = in->positions_q;
  p.rope = ctx->rope;
  p.scale_log2 = float(1.4426950408889634 / (in->temperature * std::sqrt(double(in->dim))));
  p.dense = sparse ? 0 : 1;
  p.verts = sparse ? verts : nullptr;
  p.nv = nv;
  p.cap_v = cap_v;
  p.ckeys = w.B.ckeys;
  p.vbase = w.B.vbase;
  p.vfirst = w.B.vfirst;
  p.capp = w.B.capp;
  p.nseg_k = w.B.nseg_k;
  p.seg_len = w.B.seg_len;
  p.ntiles_k = w.B.npad / 64;
  p.tc_u = sparse ? w.tc_u : nullptr;
  p.n_tc_u = w.n_tc_u;
  p.cap_u = w.cap_u;
  p.sbits = w.sbits;
  p.vbits = w.vbits;
  p.words = w.words;
  p.out = out;
  p.lse = lse;
  p.lse_stride = lse_stride;
  p.tile_count = ctx->profiling ? ctx->tile_counter : nullptr;
  p.item_counter = ctx->item_counter;
  p.trace = ctx->trace;
  p.plans = w.plans;
  if (ev_tc0) LCX_CHECK_CUDA(cudaEventRecord(ev_tc0, st));
  if (!sparse) {
    p.key_lo = 0;
    p.key_hi = INT64_MAX;
    p.vert_pass = 1;
    p.init = 0;
    LCX_TRY(tc_attention(p, w.B, ctx->sm_count, st));
  } else {
    // key-window passes: the slash tiles of all (head, block) items sweep one window of
    // keys at a time so that its K hi/lo + V^T tiles stay L2-resident (every block's
    // diagonals hit them); pass 0 also runs the vertical tiles (compacted per head and
    // shared by all blocks of a head), later passes continue from the running state
    // (few slash lines -> one pass: the windows only pay off when slash tiles dominate)
    const int64_t seg = w.windows ? kTcSegment : t1;
    for (int64_t k0 = 0, pass = 0; k0 < t1; k0 += seg, ++pass) {
      p.key_lo = k0;
      p.key_hi = std::min<int64_t>(t1, k0 + seg);
      p.vert_pass = pass == 0;
      p.init = pass > 0;
      p.win_flags = seg == kTcSegment ? w.tc_flags : nullptr;
      p.win = int(pass);
      LCX_TRY(tc_attention(p, w.B, ctx->sm_count, st));
    }
  }
  if (ev_tc1) LCX_CHECK_CUDA(cudaEventRecord(ev_tc1, st));
  if (sparse) {
    // isolated slashes + self-fallback rows on the CUDA-core gather, merged in place
    GatherArgs a{};
    a.q = reinterpret_cast<const __nv_bfloat16*>(in->q);
    a.kf = w.B.kf;
    a.v = reinterpret_cast<const __nv_bfloat16*>(in->v);
    a.hq = hq;
    a.hkv = in->hkv;
    a.group = hq / in->hkv;
    a.row_begin = t0;
    a.row_end = t1;
    a.rel_mode = dca ? 1 : 0;
    a.s = dca ? s : 1;
    a.c = dca ? c : 1;
    a.pos_q = in->positions_q;
    a.pos_k = in->positions_k;
    a.rope = ctx->rope;
    a.scale_log2 = p.scale_log2;
    a.verts = fv;
    a.nv = fnv;
    a.cap_v = cap_v;
    a.slashes = fs;
    a.ns = fns;
    a.cap_s = cap_s;
    a.do_fallback = do_fallback;
    a.vbits = w.vbits;
    a.words = w.words;
    a.segs = w.segs;
    a.nseg = w.nseg;
    a.cap_seg = w.cap_seg;
    a.out = out;
    a.lse = lse;
    a.lse_stride = lse_stride;
    a.simt_count = ctx->profiling ? ctx->tile_counter + 1 : nullptr;
    // key-segment passes: the rows of all heads sweep one key segment at a time, so the
    // K / V rows a pass gathers (kGatherSegment keys x Hkv x 512 B) stay L2-resident
    // while every diagonal of every row reads them; the running (o, lse) state of each row
    // is carried in out / lse between passes
    const int64_t gseg = w.windows ? kGatherSegment : t1;
    a.win_flags = gseg == kGatherSegment ? w.g_flags : nullptr;
    // one pass over all keys: heads fastest (planted 1M: gather 90 -> 82 ms); key-window
    // passes: rows fastest (iid 1M: 5.4 s vs 5.8 s heads fastest)
    a.head_fast = gseg == t1 ? 1 : 0;
    for (int64_t k0 = 0; k0 < t1; k0 += gseg) {
      a.key_lo = k0;
      a.key_hi = std::min<int64_t>(t1, k0 + gseg);
      a.win = int(k0 / gseg);
      LCX_TRY(attention_gather(a, st));
    }
    if (admitted) {
      if (do_fallback)  // exact count of the full selection, reported once (rank 0)
        LCX_TRY(admitted_counts(fv, fnv, cap_v, fs, fns, cap_s, hq, t0, t1, admitted, st));
      else
        LCX_CHECK_CUDA(cudaMemsetAsync(admitted, 0, sizeof(int64_t) * hq, st));
    }
  } else if (admitted) {
    // dense rows: entries = i + 1
    LCX_TRY(dense_counts(hq, t0, t1, admitted, st));
  }
  return LCX_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int64_t words_for(int64_t n) { return (n + 31) / 32 + 1; }

}  // namespace

int prefill_impl(lcx_context* ctx, const lcx_attention_input* in, const lcx_prefill_config* cfg,
                 lcx_prefill_output* out, cudaStream_t st, const cudaEvent_t* ready,
                 const cudaEvent_t* done,
                 const std::function<int(int64_t)>* on_chunk = nullptr);

}  // namespace lcx

using namespace lcx;

extern "C" {

const char* lcx_last_error(void) { return lcx::g_err.c_str(); }
const char* lcx_version(void) { return "longctx-b200 0.1.0 (sm_100a)"; }

int lcx_device_ok(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
  return prop.major == 10 ? 1 : 0;
}

int lcx_context_create(int device, lcx_context** out) {
  if (!out) return fail(LCX_ERR_INTERNAL, "null out");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(LCX_ERR_CUDA, "no CUDA device available (the path has no CPU fallback)");
  cudaDeviceProp prop;
  LCX_CHECK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(LCX_ERR_CUDA, std::string("device ") + prop.name +
                                  " is not sm_100-class; kernels are built for sm_100a only");
  DeviceScope on(device);  // the context's buffers live on `device`
  if (on.err != cudaSuccess) return fail(LCX_ERR_CUDA, "cudaSetDevice failed");
  auto* ctx = new lcx_context();
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  LCX_CHECK_CUDA(cudaMalloc(&ctx->tile_counter, 2 * sizeof(int64_t)));
  LCX_CHECK_CUDA(cudaMalloc(&ctx->item_counter, sizeof(int)));
  LCX_CHECK_CUDA(cudaMalloc(&ctx->far_dev, 2 * sizeof(int)));
  LCX_CHECK_CUDA(cudaHostAlloc(&ctx->far_host, 4 * sizeof(int), cudaHostAllocMapped));
  LCX_CHECK_CUDA(cudaHostGetDevicePointer(&ctx->far_host_dev, ctx->far_host, 0));
  for (auto& e : ctx->far_ev) LCX_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  LCX_CHECK_CUDA(cudaMemset(ctx->tile_counter, 0, 2 * sizeof(int64_t)));
  *out = ctx;
  return LCX_OK;
}

int lcx_context_destroy(lcx_context* ctx) {
  if (!ctx) return LCX_OK;
  DeviceScope on(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->rope) cudaFree(ctx->rope);
  if (ctx->tile_counter) cudaFree(ctx->tile_counter);
  if (ctx->item_counter) cudaFree(ctx->item_counter);
  if (ctx->trace) cudaFree(ctx->trace);
  if (ctx->far_dev) cudaFree(ctx->far_dev);
  if (ctx->far_host) cudaFreeHost(ctx->far_host);
  for (auto& e : ctx->far_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->chunk_done) cudaEventDestroy(e);
  if (ctx->stage) cudaFree(ctx->stage);
  if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
  if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
  if (ctx->est_side) cudaStreamDestroy(ctx->est_side);
  if (ctx->est_fork) cudaEventDestroy(ctx->est_fork);
  if (ctx->est_join) cudaEventDestroy(ctx->est_join);
  if (ctx->prep_side) cudaStreamDestroy(ctx->prep_side);
  if (ctx->prep_fork) cudaEventDestroy(ctx->prep_fork);
  if (ctx->prep_join) cudaEventDestroy(ctx->prep_join);
  delete ctx;
  return LCX_OK;
}

int lcx_set_profiling(lcx_context* ctx, int enabled) {
  LCX_ON_DEVICE(ctx);
  ctx->profiling = enabled;
  return LCX_OK;
}

int lcx_debug_trace(lcx_context* ctx, int enable, long long* host_out) {
  LCX_ON_DEVICE(ctx);
  const size_t bytes = (512 * 8 + 64) * sizeof(long long);  // per-tile marks + wait profile
  if (enable && !ctx->trace) {
    LCX_CHECK_CUDA(cudaMalloc(&ctx->trace, bytes));
    LCX_CHECK_CUDA(cudaMemset(ctx->trace, 0, bytes));
  }
  if (host_out && ctx->trace) {
    LCX_CHECK_CUDA(cudaDeviceSynchronize());
    LCX_CHECK_CUDA(cudaMemcpy(host_out, ctx->trace, bytes, cudaMemcpyDeviceToHost));
  }
  if (!enable && ctx->trace) {
    LCX_CHECK_CUDA(cudaFree(ctx->trace));
    ctx->trace = nullptr;
  }
  return LCX_OK;
}

int lcx_get_stats(lcx_context* ctx, lcx_prefill_stats* out) {
  *out = ctx->stats;
  return LCX_OK;
}

int lcx_get_chunk_ms(lcx_context* ctx, float* out, int64_t cap, int64_t* count) {
  LCX_ON_DEVICE(ctx);
  if (!count) return fail(LCX_ERR_DIMENSION, "null count");
  *count = int64_t(ctx->chunk_ms.size());
  if (out)
    for (int64_t i = 0; i < std::min<int64_t>(cap, *count); ++i) out[i] = ctx->chunk_ms[size_t(i)];
  return LCX_OK;
}

int lcx_estimate_block(lcx_context* ctx, const lcx_attention_input* in, int64_t q_row0,
                       int64_t nq, int64_t nk, int64_t last_q, int32_t pos_mode,
                       const lcx_chunk_config* cfg, float* est_out, void* stream) {
  LCX_ON_DEVICE(ctx);
  LCX_TRY(validate_input(in));
  if (last_q <= 0) return fail(LCX_ERR_CONFIG, "lastQ must be positive");
  if (nq <= 0 || nk <= 0) return fail(LCX_ERR_DIMENSION, "empty query or key matrix");
  if (nq > nk) return fail(LCX_ERR_DIMENSION, "queries must be the trailing rows of the key timeline");
  if (q_row0 + nq != nk || nk > in->n)
    return fail(LCX_ERR_DIMENSION, "query window must end at the key count");
  if (pos_mode == LCX_POS_DCA_CONTINUOUS && !cfg)
    return fail(LCX_ERR_CONFIG, "dcaContinuous estimation requires a chunk config");
  const int64_t c = pos_mode == LCX_POS_DCA_CONTINUOUS ? cfg->train_len : 0;
  if (pos_mode == LCX_POS_DCA_CONTINUOUS && c <= 0)
    return fail(LCX_ERR_CONFIG, "trainLen must be positive");
  cudaStream_t st = S(stream);
  LCX_TRY(ensure_rope(ctx, in->rope_base, in->dim, std::max<int64_t>(nk, c), st));
  EstimateArgs e = base_est(in, ctx, q_row0, nq, nk, last_q, pos_mode, c);
  e.est = est_out;
  Sizer sz;
  estimate_simt_size(e, sz, ctx->sm_count);
  LCX_TRY(ensure_workspace(ctx, sz.off));
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  return estimate_simt(ctx, e, ar, st);
}

int lcx_line_scores(lcx_context* ctx, const lcx_attention_input* in, int64_t q_row0, int64_t nq,
                    int64_t nk, int64_t last_q, int32_t pos_mode, const lcx_chunk_config* cfg,
                    int32_t slash_mean, float* col_score, float* slash_score, void* stream) {
  LCX_ON_DEVICE(ctx);
  LCX_TRY(validate_input(in));
  if (last_q <= 0) return fail(LCX_ERR_CONFIG, "lastQ must be positive");
  if (nq <= 0 || nk <= 0 || nq > nk || q_row0 + nq != nk || nk > in->n)
    return fail(LCX_ERR_DIMENSION, "bad query window");
  if (pos_mode == LCX_POS_DCA_CONTINUOUS && !cfg)
    return fail(LCX_ERR_CONFIG, "dcaContinuous estimation requires a chunk config");
  const int64_t c = pos_mode == LCX_POS_DCA_CONTINUOUS ? cfg->train_len : 0;
  cudaStream_t st = S(stream);
  LCX_TRY(ensure_rope(ctx, in->rope_base, in->dim, std::max<int64_t>(nk, c), st));
  EstimateArgs e = base_est(in, ctx, q_row0, nq, nk, last_q, pos_mode, c);
  e.col = col_score;
  e.slash = slash_score;
  e.slash_mean = slash_mean;
  const bool est_tc = est_tc_eligible(in->dtype, in->dim, e.block);
  const int64_t k3_tiles = (nk + 63) / 64;
  if (est_tc) {
    e.k3 = reinterpret_cast<void*>(1);
    e.k3_tiles = k3_tiles;
  }
  Sizer sz;
  if (est_tc) sz.take<uint8_t>(est_tc_k3_bytes(nk, in->hkv));
  estimate_simt_size(e, sz, ctx->sm_count);
  LCX_TRY(ensure_workspace(ctx, sz.off));
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  if (est_tc) {
    void* k3 = ar.take<uint8_t>(est_tc_k3_bytes(nk, in->hkv));
    LCX_TRY(est_tc_prepare_keys(in->k, 0, nk, in->hkv, k3_tiles, ctx->rope, k3, st));
    e.k3 = k3;
  }
  return estimate_simt(ctx, e, ar, st);
}

int lcx_select_from_scores(lcx_context* ctx, const float* col_score, const float* slash_score,
                           int32_t heads, int64_t n, int64_t block, int64_t budget_vertical,
                           int64_t budget_slash, const lcx_selection_options* opts,
                           int32_t* verticals, int32_t* nv, int64_t cap_v, int32_t* slashes,
                           int32_t* ns, int64_t cap_s, void* stream) {
  LCX_ON_DEVICE(ctx);
  (void)ctx;
  if (n <= 0 || block <= 0 || block > n)
    return fail(LCX_ERR_DIMENSION, "estimation block row count out of range");
  lcx_selection_options o = opts ? *opts : lcx_selection_options{1, 1, 1};
  cudaStream_t st = S(stream);
  LCX_TRY(select_lines(col_score, heads, n, budget_vertical, o.force_sink_column, 1, verticals,
                       nv, cap_v, st));
  LCX_TRY(select_lines(slash_score, heads, n, budget_slash, o.force_local_band, block, slashes,
                       ns, cap_s, st));
  return LCX_OK;
}

int lcx_select_critical(lcx_context* ctx, const float* est, int32_t heads, int64_t block,
                        int64_t n, int64_t budget_vertical, int64_t budget_slash,
                        const lcx_selection_options* opts, int32_t* verticals, int32_t* nv,
                        int64_t cap_v, int32_t* slashes, int32_t* ns, int64_t cap_s,
                        void* stream) {
  LCX_ON_DEVICE(ctx);
  if (n <= 0 || block <= 0 || block > n)
    return fail(LCX_ERR_DIMENSION, "estimation block row count out of range");
  lcx_selection_options o = opts ? *opts : lcx_selection_options{1, 1, 1};
  cudaStream_t st = S(stream);
  Sizer sz;
  sz.take<float>(size_t(heads) * n);
  sz.take<float>(size_t(heads) * n);
  LCX_TRY(ensure_workspace(ctx, sz.off));
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  float* col = ar.take<float>(size_t(heads) * n);
  float* sl = ar.take<float>(size_t(heads) * n);
  LCX_TRY(line_scores_from_est(est, heads, block, n, o.slash_mean, col, sl, st));
  return lcx_select_from_scores(ctx, col, sl, heads, n, block, budget_vertical, budget_slash, &o,
                                verticals, nv, cap_v, slashes, ns, cap_s, stream);
}

int lcx_sparse_attention(lcx_context* ctx, const lcx_attention_input* in,
                         const int32_t* verticals, const int32_t* nv, int64_t cap_v,
                         const int32_t* slashes, const int32_t* ns, int64_t cap_s,
                         int32_t use_dca, const lcx_chunk_config* dca, int32_t kernel_path,
                         float* out, float* lse, void* stream) {
  LCX_ON_DEVICE(ctx);
  LCX_TRY(validate_input(in));
  if (use_dca) LCX_TRY(validate_chunk(dca));
  cudaStream_t st = S(stream);
  bool tc = false;
  const int64_t n = in->n;
  LCX_TRY(resolve_path(kernel_path, in, (n + 127) / 128 * 128, use_dca != 0,
                       use_dca ? dca->chunk_size : 128, &tc));
  int64_t maxpos = 0;
  LCX_TRY(max_position(ctx, in, &maxpos, st));
  const int64_t P = std::max<int64_t>(maxpos + 1, use_dca ? dca->train_len : 0);
  LCX_TRY(ensure_rope(ctx, in->rope_base, in->dim, std::max<int64_t>(P, n), st));
  AttnWS w;
  Sizer sz;
  attn_layout(sz, in, tc, true, cap_v, cap_s, use_dca ? dca->chunk_size : n, w);
  LCX_TRY(ensure_workspace(ctx, sz.off));
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  attn_layout(ar, in, tc, true, cap_v, cap_s, use_dca ? dca->chunk_size : n, w);
  if (tc)
    LCX_TRY(tc_prepare(in->k, in->v, n, in->hq, in->hkv, in->positions_k, use_dca ? 1 : 0,
                       use_dca ? dca->chunk_size : 1, ctx->rope, w.B, st));
  return attention_chunk(ctx, in, w, 0, n, true, verticals, nv, cap_v, slashes, ns, cap_s,
                         use_dca != 0, use_dca ? dca->chunk_size : 1,
                         use_dca ? dca->train_len : 1, kDefaultTcMin, out, lse, n, nullptr, st);
}

int lcx_attention_rel(lcx_context* ctx, const lcx_attention_input* in, const int32_t* verticals,
                      const int32_t* nv, int64_t cap_v, const int32_t* slashes,
                      const int32_t* ns, int64_t cap_s, const int64_t* rel, float* out,
                      float* lse, void* stream) {
  LCX_ON_DEVICE(ctx);
  LCX_TRY(validate_input(in));
  if (!rel) return fail(LCX_ERR_DIMENSION, "relative-position override must be n x n");
  const bool sparse = verticals != nullptr;
  if (sparse && (!nv || !slashes || !ns)) return fail(LCX_ERR_DIMENSION, "null index list");
  cudaStream_t st = S(stream);
  const int64_t n = in->n;
  unsigned long long* dmax = nullptr;
  LCX_CHECK_CUDA(cudaMallocAsync(&dmax, sizeof(unsigned long long), st));
  LCX_CHECK_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
  max_abs_kernel<<<256, 256, 0, st>>>(rel, n * n, dmax);
  LCX_CHECK_LAUNCH();
  unsigned long long hmax = 0;
  LCX_CHECK_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof(hmax), cudaMemcpyDeviceToHost, st));
  LCX_CHECK_CUDA(cudaStreamSynchronize(st));
  LCX_CHECK_CUDA(cudaFreeAsync(dmax, st));
  LCX_TRY(ensure_rope(ctx, in->rope_base, in->dim, std::max<int64_t>(int64_t(hmax) + 1, n), st));
  AttnWS w;
  Sizer sz;
  attn_layout(sz, in, false, sparse, cap_v, cap_s, n, w);
  LCX_TRY(ensure_workspace(ctx, sz.off));
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  attn_layout(ar, in, false, sparse, cap_v, cap_s, n, w);
  if (sparse) LCX_TRY(build_bitmaps(verticals, nv, cap_v, in->hq, w.words, w.vbits, st));
  AttnArgs a = base_attn(in, ctx);
  a.n = n;
  a.row_begin = 0;
  a.row_end = n;
  a.rel_mode = 2;
  a.rel_mat = rel;
  a.rel_n = n;
  a.s = a.c = 1;
  a.dense = sparse ? 0 : 1;
  a.verts = verticals;
  a.nv = nv;
  a.cap_v = cap_v;
  a.slashes = slashes;
  a.ns = ns;
  a.cap_s = cap_s;
  a.vbits = w.vbits;
  a.bit_words = w.words;
  // unsharded: the full selection is this call's selection, and rows with no admitted
  // line attend to themselves (sparse.cpp:111)
  a.fverts = verticals;
  a.fnv = nv;
  a.fslashes = slashes;
  a.fns = ns;
  a.do_fallback = 1;
  a.out = out;
  a.lse = lse;
  a.lse_stride = n;
  return attention_simt(a, st);
}

int lcx_full_attention(lcx_context* ctx, const lcx_attention_input* in, int32_t use_dca,
                       const lcx_chunk_config* dca, int32_t kernel_path, float* out, float* lse,
                       void* stream) {
  LCX_ON_DEVICE(ctx);
  LCX_TRY(validate_input(in));
  if (use_dca) LCX_TRY(validate_chunk(dca));
  cudaStream_t st = S(stream);
  bool tc = false;
  const int64_t n = in->n;
  LCX_TRY(resolve_path(kernel_path, in, (n + 127) / 128 * 128, use_dca != 0,
                       use_dca ? dca->chunk_size : 128, &tc));
  int64_t maxpos = 0;
  LCX_TRY(max_position(ctx, in, &maxpos, st));
  const int64_t P = std::max<int64_t>(maxpos + 1, use_dca ? dca->train_len : 0);
  LCX_TRY(ensure_rope(ctx, in->rope_base, in->dim, std::max<int64_t>(P, n), st));
  AttnWS w;
  Sizer sz;
  attn_layout(sz, in, tc, false, 0, 0, use_dca ? dca->chunk_size : n, w);
  LCX_TRY(ensure_workspace(ctx, sz.off));
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  attn_layout(ar, in, tc, false, 0, 0, use_dca ? dca->chunk_size : n, w);
  if (tc)
    LCX_TRY(tc_prepare(in->k, in->v, n, in->hq, in->hkv, in->positions_k, use_dca ? 1 : 0,
                       use_dca ? dca->chunk_size : 1, ctx->rope, w.B, st));
  return attention_chunk(ctx, in, w, 0, n, false, nullptr, nullptr, 0, nullptr, nullptr, 0,
                         use_dca != 0, use_dca ? dca->chunk_size : 1,
                         use_dca ? dca->train_len : 1, kDefaultTcMin, out, lse, n, nullptr, st);
}

int lcx_chunked_prefill(lcx_context* ctx, const lcx_attention_input* in,
                        const lcx_prefill_config* cfg, lcx_prefill_output* out, void* stream) {
  LCX_ON_DEVICE(ctx);
  return prefill_impl(ctx, in, cfg, out, S(stream), nullptr, nullptr);
}

// Host-buffer entry: chunk-pipelined H2D / compute / D2H over three streams.
int lcx_chunked_prefill_host(lcx_context* ctx, const lcx_attention_input* hin,
                             const lcx_prefill_config* cfg, lcx_prefill_output* hout,
                             void* stream) {
  LCX_ON_DEVICE(ctx);
  LCX_TRY(validate_input(hin));
  if (!cfg || !hout || !hout->out || !hout->lse)
    return fail(LCX_ERR_DIMENSION, "null config/output");
  if (cfg->chunk_len <= 0) return fail(LCX_ERR_CONFIG, "chunkLen must be positive");
  cudaStream_t st = S(stream);
  const int64_t n = hin->n, L = cfg->chunk_len, nch = (n + L - 1) / L;
  const int hq = hin->hq, hkv = hin->hkv, dim = hin->dim;
  const size_t es = hin->dtype == LCX_BF16 ? 2 : 4;
  const bool sel = hout->sel_verticals && hout->sel_nv && hout->sel_slashes && hout->sel_ns;
  const int64_t cap_v = sel ? hout->cap_v : 0, cap_s = sel ? hout->cap_s : 0;
  // device staging (context-owned, grown on demand)
  auto plan = [&](auto& A, void** q, void** k, void** v, int64_t** pq, int64_t** pk, float** o,
                  float** l, int32_t** sv, int32_t** snv, int32_t** ss, int32_t** sns,
                  int64_t** adm) {
    *q = A.template take<char>(size_t(n) * hq * dim * es);
    *k = A.template take<char>(size_t(n) * hkv * dim * es);
    *v = A.template take<char>(size_t(n) * hkv * dim * es);
    *pq = hin->positions_q ? A.template take<int64_t>(size_t(n)) : nullptr;
    *pk = hin->positions_k ? A.template take<int64_t>(size_t(n)) : nullptr;
    *o = A.template take<float>(size_t(n) * hq * dim);
    *l = A.template take<float>(size_t(hq) * n);
    *sv = sel ? A.template take<int32_t>(size_t(nch) * hq * cap_v) : nullptr;
    *snv = sel ? A.template take<int32_t>(size_t(nch) * hq) : nullptr;
    *ss = sel ? A.template take<int32_t>(size_t(nch) * hq * cap_s) : nullptr;
    *sns = sel ? A.template take<int32_t>(size_t(nch) * hq) : nullptr;
    *adm = hout->admitted ? A.template take<int64_t>(size_t(nch) * hq) : nullptr;
  };
  void *dq, *dk, *dv;
  int64_t *dpq, *dpk, *dadm;
  float *dout, *dlse;
  int32_t *dsv, *dsnv, *dss, *dsns;
  Sizer sz;
  plan(sz, &dq, &dk, &dv, &dpq, &dpk, &dout, &dlse, &dsv, &dsnv, &dss, &dsns, &dadm);
  if (sz.off > ctx->stage_bytes) {
    if (ctx->stage) LCX_CHECK_CUDA(cudaFree(ctx->stage));
    ctx->stage = nullptr;
    ctx->stage_bytes = 0;
    LCX_CHECK_CUDA(cudaMalloc(&ctx->stage, sz.off));
    ctx->stage_bytes = sz.off;
  }
  Arena ar{ctx->stage, ctx->stage_bytes, 0};
  plan(ar, &dq, &dk, &dv, &dpq, &dpk, &dout, &dlse, &dsv, &dsnv, &dss, &dsns, &dadm);
  if (sel) {  // list padding past each count reads as 0, as the device entry leaves it
    LCX_CHECK_CUDA(cudaMemsetAsync(dsv, 0, sizeof(int32_t) * size_t(nch) * hq * cap_v, st));
    LCX_CHECK_CUDA(cudaMemsetAsync(dss, 0, sizeof(int32_t) * size_t(nch) * hq * cap_s, st));
  }
  if (!ctx->h2d) LCX_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
  if (!ctx->d2h) LCX_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
  // positions are validated before the chunk loop: upload them first
  if (dpq) LCX_CHECK_CUDA(cudaMemcpy(dpq, hin->positions_q, 8 * n, cudaMemcpyHostToDevice));
  if (dpk) LCX_CHECK_CUDA(cudaMemcpy(dpk, hin->positions_k, 8 * n, cudaMemcpyHostToDevice));
  std::vector<cudaEvent_t> ready(nch), done(nch);
  for (int64_t c = 0; c < nch; ++c) {
    LCX_CHECK_CUDA(cudaEventCreateWithFlags(&ready[c], cudaEventDisableTiming));
    LCX_CHECK_CUDA(cudaEventCreateWithFlags(&done[c], cudaEventDisableTiming));
  }
  cudaEvent_t start;
  LCX_CHECK_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  LCX_CHECK_CUDA(cudaEventRecord(start, st));
  LCX_CHECK_CUDA(cudaStreamWaitEvent(ctx->h2d, start, 0));
  int rc = LCX_OK;
  // H2D: token-major rows [t0, t1) of q, k, v are contiguous slabs
  for (int64_t c = 0; c < nch && rc == LCX_OK; ++c) {
    const int64_t t0 = c * L, t1 = std::min(n, t0 + L);
    auto cp = [&](void* d, const void* h, size_t row_bytes) {
      return cudaMemcpyAsync(static_cast<char*>(d) + t0 * row_bytes,
                             static_cast<const char*>(h) + t0 * row_bytes,
                             (t1 - t0) * row_bytes, cudaMemcpyHostToDevice, ctx->h2d);
    };
    // a chunk range (cfg->chunk_begin / chunk_end) reads the query rows of its chunks only and
    // the keys / values up to its last chunk
    const bool ranged = cfg->chunk_end > cfg->chunk_begin;
    const bool need_q = !ranged || (c >= cfg->chunk_begin && c < cfg->chunk_end);
    const bool need_kv = !ranged || c < cfg->chunk_end;
    if ((need_q && cp(dq, hin->q, size_t(hq) * dim * es) != cudaSuccess) ||
        (need_kv && cp(dk, hin->k, size_t(hkv) * dim * es) != cudaSuccess) ||
        (need_kv && cp(dv, hin->v, size_t(hkv) * dim * es) != cudaSuccess) ||
        cudaEventRecord(ready[c], ctx->h2d) != cudaSuccess)
      rc = fail(LCX_ERR_CUDA, "host-to-device copy failed");
  }
  if (rc == LCX_OK) {
    lcx_attention_input din = *hin;
    din.q = dq;
    din.k = dk;
    din.v = dv;
    din.positions_q = dpq;
    din.positions_k = dpk;
    lcx_prefill_output dout_s{dout, dlse, dsv, dsnv, dss, dsns, cap_v, cap_s, dadm, nullptr};
    // D2H of each chunk's rows, enqueued as soon as the chunk's kernels are (so the copy
    // of chunk c overlaps the compute of chunks c+1, ...)
    const std::function<int(int64_t)> d2h = [&](int64_t c) -> int {
      const int64_t t0 = c * L, t1 = std::min(n, t0 + L);
      cudaError_t e = cudaStreamWaitEvent(ctx->d2h, done[c], 0);
      const size_t orow = size_t(hq) * dim * sizeof(float);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(reinterpret_cast<char*>(hout->out) + t0 * orow,
                            reinterpret_cast<char*>(dout) + t0 * orow, (t1 - t0) * orow,
                            cudaMemcpyDeviceToHost, ctx->d2h);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(hout->lse + t0, sizeof(float) * n, dlse + t0, sizeof(float) * n,
                              sizeof(float) * (t1 - t0), hq, cudaMemcpyDeviceToHost, ctx->d2h);
      if (e == cudaSuccess && sel) {
        e = cudaMemcpyAsync(hout->sel_verticals + c * hq * cap_v, dsv + c * hq * cap_v,
                            sizeof(int32_t) * hq * cap_v, cudaMemcpyDeviceToHost, ctx->d2h);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(hout->sel_slashes + c * hq * cap_s, dss + c * hq * cap_s,
                              sizeof(int32_t) * hq * cap_s, cudaMemcpyDeviceToHost, ctx->d2h);
      }
      return e == cudaSuccess ? LCX_OK : fail(LCX_ERR_CUDA, "device-to-host copy failed");
    };
    rc = prefill_impl(ctx, &din, cfg, &dout_s, st, ready.data(), done.data(), &d2h);
  }
  if (rc == LCX_OK && sel) {
    if (cudaMemcpyAsync(hout->sel_nv, dsnv, sizeof(int32_t) * nch * hq, cudaMemcpyDeviceToHost,
                        ctx->d2h) != cudaSuccess ||
        cudaMemcpyAsync(hout->sel_ns, dsns, sizeof(int32_t) * nch * hq, cudaMemcpyDeviceToHost,
                        ctx->d2h) != cudaSuccess)
      rc = fail(LCX_ERR_CUDA, "device-to-host copy failed");
  }
  if (rc == LCX_OK && hout->admitted) {
    if (cudaMemcpyAsync(hout->admitted, dadm, sizeof(int64_t) * nch * hq, cudaMemcpyDeviceToHost,
                        ctx->d2h) != cudaSuccess)
      rc = fail(LCX_ERR_CUDA, "device-to-host copy failed");
  }
  // the caller's stream observes completion of every copy
  cudaEvent_t fin;
  cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
  cudaEventRecord(fin, ctx->d2h);
  cudaStreamWaitEvent(st, fin, 0);
  const cudaError_t e1 = cudaStreamSynchronize(ctx->h2d);
  const cudaError_t e2 = cudaStreamSynchronize(ctx->d2h);
  const cudaError_t e3 = cudaStreamSynchronize(st);
  for (auto& x : ready) cudaEventDestroy(x);
  for (auto& x : done) cudaEventDestroy(x);
  cudaEventDestroy(start);
  cudaEventDestroy(fin);
  if (rc != LCX_OK) return rc;
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
    return fail(LCX_ERR_CUDA, std::string("host prefill: ") +
                                  cudaGetErrorString(e1 != cudaSuccess ? e1
                                                     : e2 != cudaSuccess ? e2 : e3));
  return LCX_OK;
}

}  // extern "C"

namespace lcx {

// The operator body.  ready[c] (optional) is waited on before chunk c touches its
// rows (host-pipelined entry: Q/K/V rows of chunk c arrive on a copy stream);
// done[c] (optional) is recorded once chunk c's output rows and lse are final.
int prefill_impl(lcx_context* ctx, const lcx_attention_input* in, const lcx_prefill_config* cfg,
                 lcx_prefill_output* out, cudaStream_t st, const cudaEvent_t* ready,
                 const cudaEvent_t* done, const std::function<int(int64_t)>* on_chunk) {
  LCX_TRY(validate_input(in));
  if (!cfg || !out) return fail(LCX_ERR_DIMENSION, "null config/output");
  const int phase = cfg->phase;
  if (phase != LCX_PHASE_ALL && phase != LCX_PHASE_SELECT && phase != LCX_PHASE_ATTEND)
    return fail(LCX_ERR_CONFIG, "unknown prefill phase");
  const bool do_select = phase != LCX_PHASE_ATTEND, do_attend = phase != LCX_PHASE_SELECT;
  if (do_attend && (!out->out || !out->lse)) return fail(LCX_ERR_DIMENSION, "null output");
  if (cfg->chunk_len <= 0) return fail(LCX_ERR_CONFIG, "chunkLen must be positive");
  if (cfg->last_q <= 0) return fail(LCX_ERR_CONFIG, "lastQ must be positive");
  const bool sparse = cfg->mode == LCX_PREFILL_SPARSE;
  if (phase != LCX_PHASE_ALL &&
      (!sparse || !out->sel_verticals || !out->sel_nv || !out->sel_slashes || !out->sel_ns))
    return fail(LCX_ERR_CONFIG, "select / attend phases need sparse mode and a selection log");
  const int eh0 = cfg->est_head_end > 0 ? cfg->est_head_begin : 0;
  const int eh1 = cfg->est_head_end > 0 ? cfg->est_head_end : in->hq;
  if (eh0 < 0 || eh1 > in->hq || eh0 >= eh1)
    return fail(LCX_ERR_CONFIG, "estimator head range out of range");
  if (phase == LCX_PHASE_ALL && (eh0 != 0 || eh1 != in->hq))
    return fail(LCX_ERR_CONFIG, "an estimator head range needs the select phase");
  if (sparse && cfg->chunk_len < cfg->last_q)
    return fail(LCX_ERR_CONFIG, "sparse prefill requires chunkLen >= lastQ");
  const bool dca = cfg->position_mode == LCX_POS_DCA_CONTINUOUS;
  if (dca) LCX_TRY(validate_chunk(&cfg->dca));
  if (cfg->budget_vertical < 0 || cfg->budget_slash < 0)
    return fail(LCX_ERR_CONFIG, "budgets must be non-negative");
  const int shards = cfg->shard_count > 1 ? cfg->shard_count : 1;
  if (shards > 1 && (cfg->shard_rank < 0 || cfg->shard_rank >= shards))
    return fail(LCX_ERR_CONFIG, "shard rank out of range");
  if (shards > 1 && !sparse)
    return fail(LCX_ERR_CONFIG, "line sharding applies to sparse prefill");

  const int64_t n = in->n;
  const int hq = in->hq;
  const int64_t L = cfg->chunk_len;
  const int64_t nchunks = (n + L - 1) / L;
  const int64_t s = dca ? cfg->dca.chunk_size : 1;
  const int64_t c = dca ? cfg->dca.train_len : 0;
  bool tc = false;
  LCX_TRY(resolve_path(cfg->kernel_path, in, L, dca, s, &tc));
  int64_t maxpos = 0;
  LCX_TRY(max_position(ctx, in, &maxpos, st));
  LCX_TRY(ensure_rope(ctx, in->rope_base, in->dim,
                      std::max<int64_t>(std::max<int64_t>(maxpos + 1, n), c), st));

  const int64_t block_max = std::min(cfg->last_q, L);
  const int64_t cap_v = out->sel_verticals ? out->cap_v : cfg->budget_vertical + 2;
  const int64_t cap_s = out->sel_slashes ? out->cap_s : cfg->budget_slash + block_max + 1;
  if (sparse && (cap_v < std::min<int64_t>(cfg->budget_vertical, n) + 1 ||
                 cap_s < std::min<int64_t>(cfg->budget_slash, n) + block_max))
    return fail(LCX_ERR_DIMENSION, "selection capacity below budget + forced lines");
  const int tc_min = cfg->tc_min_entries > 0 ? cfg->tc_min_entries : kDefaultTcMin;
  // recall check scratch rows: the last B rows of a chunk, from a 128-aligned row on the
  // tensor-core path
  const int64_t kRecRows = block_max + (tc ? 127 : 0);

  // workspace plan (largest chunk = the last one: nk = n)
  EstimateArgs e_max = base_est(in, ctx, n - std::min(L, n), std::min(L, n), n, cfg->last_q,
                                dca ? 1 : 0, c);
  e_max.col = reinterpret_cast<float*>(1);
  e_max.slash = reinterpret_cast<float*>(1);
  // tensor-core estimator: keys rotated by their token index and split into 3 bf16 terms,
  // prepared once per chunk for the chunk's new keys (chunks only append keys)
  const bool est_tc = sparse && est_tc_eligible(in->dtype, in->dim, block_max);
  const int64_t k3_tiles = (n + 63) / 64;
  void* k3 = nullptr;
  if (est_tc) {
    e_max.k3 = reinterpret_cast<void*>(1);
    e_max.k3_tiles = k3_tiles;
  }
  int32_t *ov = nullptr, *onv = nullptr, *os = nullptr, *ons = nullptr;
  float *rec_o = nullptr, *rec_l = nullptr;
  if (out->recall && (shards > 1 || phase != LCX_PHASE_ALL))
    return fail(LCX_ERR_CONFIG, "the recall check needs the merged (unsharded) lse");
  auto layout = [&](auto& A, AttnWS& w, float** col, float** sl, int32_t** iv, int32_t** inv,
                    int32_t** is, int32_t** ins, size_t* est_off) {
    *est_off = A.off;
    if (sparse) {
      Sizer es;
      estimate_simt_size(e_max, es, ctx->sm_count);
      A.off += es.off;
      *col = A.template take<float>(size_t(hq) * n);
      *sl = A.template take<float>(size_t(hq) * n);
      if (!out->sel_verticals) {
        *iv = A.template take<int32_t>(size_t(hq) * cap_v);
        *inv = A.template take<int32_t>(size_t(hq));
      }
      if (!out->sel_slashes) {
        *is = A.template take<int32_t>(size_t(hq) * cap_s);
        *ins = A.template take<int32_t>(size_t(hq));
      }
      if (est_tc) k3 = A.template take<uint8_t>(est_tc_k3_bytes(n, in->hkv));
      if (out->recall) {  // dense rows of the recall check: [rows][hq][dim] O + [hq][rows] lse
        rec_o = A.template take<float>(size_t(kRecRows) * hq * in->dim);
        rec_l = A.template take<float>(size_t(hq) * kRecRows);
      }
      if (shards > 1) {  // this shard's lines
        ov = A.template take<int32_t>(size_t(hq) * cap_v);
        onv = A.template take<int32_t>(size_t(hq));
        os = A.template take<int32_t>(size_t(hq) * cap_s);
        ons = A.template take<int32_t>(size_t(hq));
      }
    }
    attn_layout(A, in, tc, sparse, cap_v, cap_s, dca ? s : n, w);
  };
  float *col = nullptr, *sl = nullptr;
  int32_t *iv = nullptr, *inv = nullptr, *is = nullptr, *ins = nullptr;
  size_t est_off = 0;
  AttnWS w;
  {
    Sizer sz;
    layout(sz, w, &col, &sl, &iv, &inv, &is, &ins, &est_off);
    LCX_TRY(ensure_workspace(ctx, sz.off));
  }
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  layout(ar, w, &col, &sl, &iv, &inv, &is, &ins, &est_off);
  Arena est_ar{ctx->ws, ctx->ws_bytes, est_off};
  if (tc) LCX_TRY(tc_prepare_maps(hq, in->hkv, w.B));
  const bool prof = ctx->profiling != 0;
  const long long launches0 = g_launches;
  std::vector<cudaEvent_t> ev;
  if (cfg->record_chunk_events) {
    while (int64_t(ctx->chunk_done.size()) < nchunks) {
      cudaEvent_t e;
      LCX_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ctx->chunk_done.push_back(e);
    }
  }
  ctx->chunk_events = cfg->record_chunk_events ? nchunks : 0;
  if (prof) {
    LCX_CHECK_CUDA(cudaMemsetAsync(ctx->tile_counter, 0, 2 * sizeof(int64_t), st));
    ev.resize(size_t(6 * nchunks + 1));
    for (auto& x : ev) LCX_CHECK_CUDA(cudaEventCreate(&x));
    LCX_CHECK_CUDA(cudaEventRecord(ev[6 * nchunks], st));
  }

  // chunk range of this call (multi-GPU: a head's chunks split over GPUs)
  const int64_t cb = cfg->chunk_end > cfg->chunk_begin ? std::max<int64_t>(0, cfg->chunk_begin) : 0;
  const int64_t ce = cfg->chunk_end > cfg->chunk_begin ? std::min<int64_t>(nchunks, cfg->chunk_end)
                                                        : nchunks;
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int64_t t0 = ci * L, t1 = std::min(n, t0 + L);
    const int64_t block = std::min(cfg->last_q, t1 - t0);
    if (ci < cb || ci >= ce) {
      // outside the range: only the keys this chunk appends are prepared (a later chunk of
      // the range reads them), nothing is computed or written
      cudaEvent_t* e = prof ? &ev[6 * ci] : nullptr;
      if (ready) LCX_CHECK_CUDA(cudaStreamWaitEvent(st, ready[ci], 0));
      if (prof) LCX_CHECK_CUDA(cudaEventRecord(e[0], st));
      if (ci < cb) {
        if (tc && do_attend)
          LCX_TRY(tc_prepare_rows(in->k, in->v, n, t0, t1, in->hkv, in->positions_k, dca ? 1 : 0,
                                  s, ctx->rope, w.B, st));
        if (sparse && do_select && est_tc)
          LCX_TRY(est_tc_prepare_keys(in->k, t0, t1, in->hkv, k3_tiles, ctx->rope, k3, st));
      }
      if (prof)
        for (int x = 1; x < 6; ++x) LCX_CHECK_CUDA(cudaEventRecord(e[x], st));
      if (done) LCX_CHECK_CUDA(cudaEventRecord(done[ci], st));
      if (cfg->record_chunk_events) LCX_CHECK_CUDA(cudaEventRecord(ctx->chunk_done[size_t(ci)], st));
      continue;
    }
    int32_t* vlist = out->sel_verticals ? out->sel_verticals + ci * hq * cap_v : iv;
    int32_t* vcnt = out->sel_nv ? out->sel_nv + ci * hq : inv;
    int32_t* slist = out->sel_slashes ? out->sel_slashes + ci * hq * cap_s : is;
    int32_t* scnt = out->sel_ns ? out->sel_ns + ci * hq : ins;
    cudaEvent_t* e = prof ? &ev[6 * ci] : nullptr;
    if (ready) LCX_CHECK_CUDA(cudaStreamWaitEvent(st, ready[ci], 0));
    if (prof) LCX_CHECK_CUDA(cudaEventRecord(e[0], st));
    // rotated K / V^T of this chunk's new key rows (chunks only ever append keys).  With an
    // estimator to run first, on a side stream beside it (joined before the attention): it
    // writes only rows [t0, t1), which no earlier chunk's attention reads when t0 is
    // 64-aligned (otherwise the shared V^T tile is rewritten: in order, on the main stream)
    const bool prep_beside = tc && do_attend && sparse && do_select && t0 % 64 == 0;
    if (prep_beside) {
      if (!ctx->prep_side) {
        LCX_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx->prep_side, cudaStreamNonBlocking));
        LCX_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->prep_fork, cudaEventDisableTiming));
        LCX_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->prep_join, cudaEventDisableTiming));
      }
      LCX_CHECK_CUDA(cudaEventRecord(ctx->prep_fork, st));
      LCX_CHECK_CUDA(cudaStreamWaitEvent(ctx->prep_side, ctx->prep_fork, 0));
      LCX_TRY(tc_prepare_rows(in->k, in->v, n, t0, t1, in->hkv, in->positions_k, dca ? 1 : 0, s,
                              ctx->rope, w.B, ctx->prep_side));
      LCX_CHECK_CUDA(cudaEventRecord(ctx->prep_join, ctx->prep_side));
    } else if (tc && do_attend) {
      LCX_TRY(tc_prepare_rows(in->k, in->v, n, t0, t1, in->hkv, in->positions_k, dca ? 1 : 0, s,
                              ctx->rope, w.B, st));
    }
    if (sparse && do_select) {
      if (est_tc)
        LCX_TRY(est_tc_prepare_keys(in->k, t0, t1, in->hkv, k3_tiles, ctx->rope, k3, st));
      EstimateArgs es = base_est(in, ctx, t0, t1 - t0, t1, cfg->last_q, dca ? 1 : 0, c);
      es.k3 = k3;
      es.k3_tiles = k3_tiles;
      es.col = col;
      es.slash = sl;
      es.slash_mean = cfg->opts.slash_mean;
      es.h0 = eh0;
      es.h1 = eh1;
      Arena a2 = est_ar;
      LCX_TRY(estimate_simt(ctx, es, a2, st));
      if (prof) LCX_CHECK_CUDA(cudaEventRecord(e[1], st));
      const int neh = eh1 - eh0;
      if (!do_attend) {  // select phase: this call's head slots are written whole, padding 0
        LCX_CHECK_CUDA(cudaMemsetAsync(vlist + eh0 * cap_v, 0, sizeof(int32_t) * neh * cap_v, st));
        LCX_CHECK_CUDA(cudaMemsetAsync(slist + eh0 * cap_s, 0, sizeof(int32_t) * neh * cap_s, st));
      }
      LCX_TRY(select_lines(col + int64_t(eh0) * t1, neh, t1, cfg->budget_vertical,
                           cfg->opts.force_sink_column, 1, vlist + eh0 * cap_v, vcnt + eh0,
                           cap_v, st));
      LCX_TRY(select_lines(sl + int64_t(eh0) * t1, neh, t1, cfg->budget_slash,
                           cfg->opts.force_local_band, block, slist + eh0 * cap_s, scnt + eh0,
                           cap_s, st));
      if (prof) LCX_CHECK_CUDA(cudaEventRecord(e[2], st));
    }
    if (!do_attend) {
      if (prof) {
        LCX_CHECK_CUDA(cudaEventRecord(e[3], st));
        LCX_CHECK_CUDA(cudaEventRecord(e[4], st));
        LCX_CHECK_CUDA(cudaEventRecord(e[5], st));
      }
      continue;
    }
    if (sparse) {
      if (prof && !do_select) {
        LCX_CHECK_CUDA(cudaEventRecord(e[1], st));
        LCX_CHECK_CUDA(cudaEventRecord(e[2], st));
      }
      if (tc) {  // how many selected slashes reach beyond one key window (see below)
        LCX_CHECK_CUDA(cudaMemsetAsync(ctx->far_dev, 0, 2 * sizeof(int), st));
        far_count_kernel<<<hq, 256, 0, st>>>(slist, scnt, cap_s, kTcSegment, ctx->far_dev);
        LCX_CHECK_LAUNCH();
        // stored into mapped host memory by a kernel, not a D2H copy: on the host entry the
        // copy engine is busy with the output rows and a copy on this stream would wait
        store_ints_kernel<<<1, 32, 0, st>>>(ctx->far_dev, ctx->far_host_dev + 2 * (ci & 1), 2);
        LCX_CHECK_LAUNCH();
        LCX_CHECK_CUDA(cudaEventRecord(ctx->far_ev[ci & 1], st));
      }
    }
    // Key-window passes pay off when most slash work lies far from the diagonal (scattered
    // lines: L2-resident windows) and cost a pass per window otherwise.  Decided from the
    // PREVIOUS chunk's selection (the host waits for that selection only, so chunk ci-1's
    // attention still overlaps this enqueue), which keeps the choice -- and the
    // floating-point accumulation order -- deterministic.
    if (sparse && tc) {
      w.windows = false;
      if (ci > cb && cap_s > kWindowMinSlashes) {
        LCX_CHECK_CUDA(cudaEventSynchronize(ctx->far_ev[(ci - 1) & 1]));
        const int* fh = ctx->far_host + 2 * ((ci - 1) & 1);
        w.windows = fh[1] > 0 && 2 * int64_t(fh[0]) > int64_t(fh[1]);
      }
    }
    const int32_t *avl = vlist, *avc = vcnt, *asl = slist, *asc = scnt;
    FullLists full{vlist, vcnt, slist, scnt, cfg->shard_rank == 0 ? 1 : 0};
    if (shards > 1) {
      shard_lists_kernel<<<hq, 256, 0, st>>>(vlist, vcnt, cap_v, slist, scnt, cap_s,
                                             cfg->shard_rank, shards, ov, onv, os, ons);
      LCX_CHECK_LAUNCH();
      avl = ov;
      avc = onv;
      asl = os;
      asc = ons;
    }
    if (prep_beside) LCX_CHECK_CUDA(cudaStreamWaitEvent(st, ctx->prep_join, 0));
    LCX_TRY(attention_chunk(ctx, in, w, t0, t1, sparse, avl, avc, cap_v, asl, asc, cap_s,
                            dca, s, dca ? c : 1, tc_min, out->out, out->lse, n,
                            out->admitted ? out->admitted + ci * hq : nullptr, st,
                            (prof && tc) ? e[4] : nullptr, (prof && tc) ? e[5] : nullptr, shards > 1 ? &full : nullptr));
    if (sparse && out->recall) {
      // dense LSE of the chunk's last rows; the TC path starts them at a 128-aligned row
      // (its chunks are 128-aligned), so at most B + 127 rows
      const int64_t b = std::min(cfg->last_q, t1 - t0);
      const int64_t r0 = tc ? std::max<int64_t>(t0, (t1 - b) / 128 * 128) : t1 - b;
      if (t1 - r0 > kRecRows) return fail(LCX_ERR_INTERNAL, "recall scratch too small");
      float* o_base = rec_o - r0 * hq * in->dim;  // rows [r0, t1) -> scratch rows
      float* l_base = rec_l - r0;                 // lse[h * kRecRows + i - r0]
      LCX_TRY(attention_chunk(ctx, in, w, r0, t1, false, nullptr, nullptr, 0, nullptr, nullptr,
                              0, dca, s, dca ? c : 1, tc_min, o_base, l_base, kRecRows,
                              nullptr, st));
      LCX_TRY(chunk_recall_launch(out->lse, n, rec_l, kRecRows, r0, t1 - b, t1, hq,
                                  out->recall + ci * hq, st));
    }
    if (prof) LCX_CHECK_CUDA(cudaEventRecord(e[3], st));
    if (done) LCX_CHECK_CUDA(cudaEventRecord(done[ci], st));
    if (cfg->record_chunk_events) LCX_CHECK_CUDA(cudaEventRecord(ctx->chunk_done[size_t(ci)], st));
    if (on_chunk) LCX_TRY((*on_chunk)(ci));  // e.g. enqueue this chunk's D2H now
  }
  ctx->stats = lcx_prefill_stats{};
  ctx->stats.chunks = nchunks;
  ctx->stats.tc_path = tc ? 1 : 0;
  ctx->stats.launches = g_launches - launches0;
  if (prof) {
    LCX_CHECK_CUDA(cudaEventSynchronize(ev[6 * (nchunks - 1) + 3]));
    double ms_est = 0, ms_sel = 0, ms_att = 0, ms_tc = 0;
    ctx->chunk_ms.assign(size_t(nchunks), 0.f);
    for (int64_t ci = 0; ci < nchunks; ++ci) {
      cudaEvent_t* e = &ev[6 * ci];
      float t = 0;
      cudaEventElapsedTime(&ctx->chunk_ms[size_t(ci)], e[0], e[3]);
      if (sparse) {
        cudaEventElapsedTime(&t, e[0], e[1]);
        ms_est += t;
        cudaEventElapsedTime(&t, e[1], e[2]);
        ms_sel += t;
        cudaEventElapsedTime(&t, e[2], e[3]);
      } else {
        cudaEventElapsedTime(&t, e[0], e[3]);
      }
      ms_att += t;
      if (tc) {
        cudaEventElapsedTime(&t, e[4], e[5]);
        ms_tc += t;
      }
    }
    float tot = 0;
    cudaEventElapsedTime(&tot, ev[6 * nchunks], ev[6 * (nchunks - 1) + 3]);
    long long cnt[2] = {0, 0};
    LCX_CHECK_CUDA(cudaMemcpy(cnt, ctx->tile_counter, sizeof(cnt), cudaMemcpyDeviceToHost));
    ctx->stats.tc_tiles = cnt[0];
    ctx->stats.simt_entries = cnt[1];
    ctx->stats.ms_estimate = ms_est;
    ctx->stats.ms_select = ms_sel;
    ctx->stats.ms_attention = ms_att;
    ctx->stats.ms_tc_kernel = ms_tc;
    ctx->stats.ms_total = tot;
    for (auto& x : ev) cudaEventDestroy(x);
  }
  return LCX_OK;
}

}  // namespace lcx

extern "C" {

int lcx_attention_recall(lcx_context* ctx, const float* lse_sparse, const float* lse_full,
                         int64_t n, double slack, float* per_query, double* aggregate,
                         void* stream) {
  LCX_ON_DEVICE(ctx);
  if (n <= 0) return fail(LCX_ERR_DIMENSION, "recall needs at least one query");
  cudaStream_t st = S(stream);
  Sizer sz;
  sz.take<double>(1025);
  sz.take<int>(1);
  LCX_TRY(ensure_workspace(ctx, sz.off));
  Arena ar{ctx->ws, ctx->ws_bytes, 0};
  double* dsum = ar.take<double>(1025);  // total + per-block partials (fixed-order sum)
  int* dbad = ar.take<int>(1);
  LCX_TRY(recall_kernel_launch(lse_sparse, lse_full, n, slack, per_query, dsum, dbad, st));
  double hsum = 0;
  int hbad = 0;
  LCX_CHECK_CUDA(cudaMemcpyAsync(&hsum, dsum, sizeof(double), cudaMemcpyDeviceToHost, st));
  LCX_CHECK_CUDA(cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st));
  LCX_CHECK_CUDA(cudaStreamSynchronize(st));
  if (hbad) return fail(LCX_ERR_DOMAIN, "recall above 1: sparse lse exceeds full lse");
  if (aggregate) *aggregate = hsum / double(n);
  return LCX_OK;
}

int lcx_stream_wait_chunk(lcx_context* ctx, int64_t chunk, void* stream) {
  LCX_ON_DEVICE(ctx);
  if (chunk < 0 || chunk >= ctx->chunk_events)
    return fail(LCX_ERR_DIMENSION, "no completion event recorded for this chunk");
  LCX_CHECK_CUDA(cudaStreamWaitEvent(S(stream), ctx->chunk_done[size_t(chunk)], 0));
  return LCX_OK;
}

int lcx_lse_scale_partial(lcx_context* ctx, float* o, const float* lse_own, const float* lse_all,
                          int32_t parts, int64_t n, int32_t hq, int32_t dim, float* lse_out,
                          void* stream) {
  LCX_ON_DEVICE(ctx);
  (void)ctx;
  if (parts <= 0 || n <= 0 || hq <= 0 || dim <= 0)
    return fail(LCX_ERR_DIMENSION, "merge needs at least one part, row, head and dim");
  return lse_scale_launch(o, lse_own, lse_all, parts, n, hq, dim, lse_out, S(stream));
}

int lcx_lse_merge(lcx_context* ctx, const float* o_parts, const float* lse_parts, int32_t parts,
                  int64_t rows, int32_t dim, float* out, float* lse_out, void* stream) {
  LCX_ON_DEVICE(ctx);
  (void)ctx;
  if (parts <= 0) return fail(LCX_ERR_DIMENSION, "merge needs at least one part");
  return lse_merge_launch(o_parts, lse_parts, parts, rows, dim, out, lse_out, S(stream));
}

}  // extern "C"
