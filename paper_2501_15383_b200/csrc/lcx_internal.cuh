// Internal declarations shared by the CUDA translation units of liblongctx_b200.
#pragma once

#include <vector>

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <string>

#include "longctx_b200.h"

namespace lcx {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
struct Status {
  int code = LCX_OK;
};

#define LCX_CHECK_CUDA(expr)                                                        \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::lcx::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));         \
      return LCX_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

extern thread_local long long g_launches;  // kernels launched by this thread (stats)

#define LCX_CHECK_LAUNCH()                                                          \
  do {                                                                              \
    ++::lcx::g_launches;                                                            \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      ::lcx::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e));    \
      return LCX_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

#define LCX_TRY(expr)                                                               \
  do {                                                                              \
    int _s = (expr);                                                                \
    if (_s != LCX_OK) return _s;                                                    \
  } while (0)

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

// Every C-ABI entry runs on its context's device, whatever device the caller has current,
// and restores the caller's device on return.
struct DeviceScope {
  int prev = -1, dev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceScope(int d) : dev(d) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceScope() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};
#define LCX_ON_DEVICE(ctx)                                                          \
  if (!(ctx)) return ::lcx::fail(LCX_ERR_INTERNAL, "null context");                \
  ::lcx::DeviceScope _lcx_dev((ctx)->device);                                       \
  if (_lcx_dev.err != cudaSuccess)                                                  \
  return ::lcx::fail(LCX_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_lcx_dev.err))

// -------------------------------------------------------- device helpers --
__host__ __device__ __forceinline__ int64_t lcx_min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lcx_max64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ float load_elem(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float load_elem(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

__device__ __forceinline__ uint32_t float_to_ordered(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// DCA remap (dca.cpp:62-80)
__device__ __forceinline__ int64_t dca_relative(int64_t i, int64_t j, int64_t s, int64_t c) {
  const int64_t qc = i / s, kc = j / s;
  const int64_t kpos = j - kc * s;
  const int64_t imod = i - qc * s;
  int64_t qpos;
  if (qc == kc) {
    qpos = imod;
  } else if (qc == kc + 1) {
    qpos = (imod + s) < (c - 1) ? (imod + s) : (c - 1);
  } else {
    qpos = c - 1;
  }
  return qpos - kpos;
}

// ------------------------------------------------------------ workspace --
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

// Size accumulator mirroring Arena::take for the dry run.
struct Sizer {
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off += (count * sizeof(T) + 255) & ~size_t(255);
    return nullptr;
  }
};

}  // namespace lcx

struct lcx_context {
  int device = 0;
  int sm_count = 148;
  // RoPE cos/sin table: rope[p * (dim/2) + pair] = (cos, sin)(p * theta_pair), fp64-derived
  double rope_base = 0.0;
  int rope_dim = 0;
  int64_t rope_P = 0;
  float2* rope = nullptr;
  // workspace
  char* ws = nullptr;
  size_t ws_bytes = 0;
  // persistent device scratch (counters)
  int profiling = 0;
  int64_t* tile_counter = nullptr;  // device: [0] executed tcgen05 tiles, [1] CUDA-core entries
  int* item_counter = nullptr;      // device: dynamic item queue of the tcgen05 attention
  long long* trace = nullptr;        // device: optional tcgen05 pipeline trace (debug)
  lcx_prefill_stats stats{};
  std::vector<float> chunk_ms;  // per-chunk device time of the last profiled prefill
  // host-buffer entry: device staging + copy streams (created lazily)
  char* stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  // estimator: the CUDA-core mixed tiles run on a side stream beside the tensor-core passes
  cudaStream_t est_side = nullptr;
  cudaEvent_t est_fork = nullptr, est_join = nullptr;
  // chunked prefill: a chunk's attention-operand prep beside its estimator
  cudaStream_t prep_side = nullptr;
  cudaEvent_t prep_fork = nullptr, prep_join = nullptr;
  // key-window decision of chunked prefill: far-slash counts of the last two chunks
  int* far_dev = nullptr;        // device [2]
  int* far_host = nullptr;       // pinned, mapped [2][2]
  int* far_host_dev = nullptr;   // device alias of far_host (written by a kernel: no copy
                                 // engine, so it never queues behind the host entry's D2H)
  cudaEvent_t far_ev[2] = {nullptr, nullptr};
  // per-chunk completion events of the last prefill run with record_chunk_events
  std::vector<cudaEvent_t> chunk_done;
  int64_t chunk_events = 0;
};

namespace lcx {

int ensure_workspace(lcx_context* ctx, size_t bytes);
int ensure_rope(lcx_context* ctx, double base, int dim, int64_t P, cudaStream_t stream);

// ---------------------------------------------------------- kernel APIs --
// estimate.cu
struct EstimateArgs {
  const void* q;   // [n][hq][dim] full input
  const void* k;   // [n][hkv][dim]
  int dtype;
  int hq, hkv, dim;
  int64_t q_row0;  // first row of the query block window (queries trail keys)
  int64_t nq;      // rows in the window
  int64_t nk;      // keys [0, nk); requires q_row0 + nq == nk
  int64_t block;   // min(last_q, nq)
  int pos_mode;    // 0 standard, 1 dca continuous
  int64_t c;       // train_len (dca)
  const float2* rope;
  float* est;      // optional [hq][block][nk]
  float* col;      // optional [hq][nk]
  float* slash;    // optional [hq][nk]
  int slash_mean;
  // tensor-core estimator (bf16, dim 128): rotated 3-term keys prepared up to nk
  // (est_tc_prepare_keys); nullptr = CUDA-core estimator for every tile
  const void* k3;
  int64_t k3_tiles;
  // query heads [h0, h1) only (sharded estimator); h1 == 0: all heads.  Each head's
  // scores are a function of its own rows and the keys only (bitwise the same whatever
  // range a call covers).
  int h0, h1;
};
int estimate_simt(lcx_context* ctx, const EstimateArgs& a, Arena& ar, cudaStream_t st);
void estimate_simt_size(const EstimateArgs& a, Sizer& sz, int sm_count);

// select.cu
int select_lines(const float* scores, int heads, int64_t n, int64_t k, int force_prefix,
                 int64_t prefix_len, int32_t* out, int32_t* count, int64_t cap,
                 cudaStream_t st);
int line_scores_from_est(const float* est, int heads, int64_t block, int64_t n, int slash_mean,
                         float* col, float* slash, cudaStream_t st);

// attn_simt.cu
struct AttnArgs {
  const void* q;
  const void* k;
  const void* v;
  int dtype;
  int hq, hkv, dim;
  int64_t n;                 // key timeline length visible (keys [0, n))
  int64_t row_begin, row_end;
  const int64_t* pos_q;      // nullptr = iota
  const int64_t* pos_k;
  int rel_mode;              // 0 standard positions, 1 dca remap, 2 explicit matrix
  const int64_t* rel_mat;    // rel_mode 2: [rel_n][rel_n] relative positions
  int64_t rel_n;
  int64_t s, c;
  float scale;               // 1 / (temperature * sqrt(dim))
  const float2* rope;
  int64_t rope_P;
  int dense;                 // 1: every key j <= i
  // sparse lists (per head)
  const int32_t* verts;  const int32_t* nv;  int64_t cap_v;
  const int32_t* slashes; const int32_t* ns; int64_t cap_s;
  const uint32_t* vbits;     // [hq][words] keys that are verticals (skip on the slash path)
  int64_t bit_words;
  // full selection (== the lists above unless line-sharded): self-fallback decision
  const int32_t* fverts; const int32_t* fnv; const int32_t* fslashes; const int32_t* fns;
  int do_fallback;           // this shard computes the self-fallback rows
  float* out;                // [.][hq][dim] rows indexed by absolute row
  float* lse;                // [hq][lse_stride]
  int64_t lse_stride;
  int64_t* admitted;         // optional [hq] counts (atomicAdd)
  int64_t* simt_count;       // optional scalar: entries processed here (atomicAdd)
};
int attention_simt(const AttnArgs& a, cudaStream_t st);

// attn_tc.cu
struct TcBuffers;
struct TcParams;

// index / bitmaps (misc.cu)
int build_bitmaps(const int32_t* lists, const int32_t* counts, int64_t cap, int heads,
                  int64_t words, uint32_t* bits, cudaStream_t st);

// misc.cu
int recall_kernel_launch(const float* ls, const float* lf, int64_t n, double slack,
                         float* per, double* sum_dev, int* bad_dev, cudaStream_t st);
int chunk_recall_launch(const float* lse_s, int64_t s_stride, const float* lse_f,
                        int64_t f_stride, int64_t f0, int64_t i0, int64_t i1, int hq, float* out,
                        cudaStream_t st);
int lse_scale_launch(float* o, const float* lse_own, const float* lse_all, int parts, int64_t n,
                     int hq, int dim, float* lse_out, cudaStream_t st);
int lse_merge_launch(const float* o_parts, const float* lse_parts, int parts, int64_t rows,
                     int dim, float* out, float* lse_out, cudaStream_t st);

}  // namespace lcx
