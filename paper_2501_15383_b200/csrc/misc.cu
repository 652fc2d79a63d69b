// Small kernels: RoPE table, index bitmaps, recall (part d), LSE merge (part e).
#include "lcx_internal.cuh"

namespace lcx {
namespace {

// rope[p][pair] = (cos, sin)(double(p) * theta_pair), theta from the host in fp64
// (attention.cpp:14-33: angle and trig in fp64; only the result is rounded to fp32).
__global__ void rope_table_kernel(const double* __restrict__ thetas, int P, int64_t npos,
                                  float2* __restrict__ out) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= npos * P) return;
  const int64_t pos = idx / P;
  const int pair = int(idx % P);
  double sn, cs;
  sincos(double(pos) * thetas[pair], &sn, &cs);
  out[idx] = make_float2(float(cs), float(sn));
}

__global__ void bitmap_kernel(const int32_t* __restrict__ lists, const int32_t* __restrict__ counts,
                              int64_t cap, int64_t words, uint32_t* __restrict__ bits) {
  const int h = blockIdx.y;
  const int cnt = counts[h];
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < cnt; x += gridDim.x * blockDim.x) {
    const int64_t v = lists[int64_t(h) * cap + x];
    atomicOr(bits + int64_t(h) * words + (v >> 5), 1u << (v & 31));
  }
}

// refine.cpp:51-72: r = exp(lse_s - lse_f); > 1 + slack is an error; clamp to 1.
// The aggregate is deterministic: each block writes its partial sum (fixed grid-stride
// order, fixed shuffle tree, fixed cross-warp order) and recall_final_kernel adds the
// block partials in index order.
constexpr int kRecallBlocks = 1024;
__global__ void recall_kernel(const float* __restrict__ ls, const float* __restrict__ lf,
                              int64_t n, double slack, float* __restrict__ per,
                              double* __restrict__ partial, int* __restrict__ bad) {
  __shared__ double warp_sum[8];
  double local = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double r = exp(double(ls[i]) - double(lf[i]));
    if (r > 1.0 + slack) atomicExch(bad, 1);
    r = r > 1.0 ? 1.0 : r;
    if (per) per[i] = float(r);
    local += r;
  }
  for (int o = 16; o >= 1; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += warp_sum[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void recall_final_kernel(const double* __restrict__ partial, int blocks,
                                    double* __restrict__ sum) {
  double t = 0.0;
  for (int b = 0; b < blocks; ++b) t += partial[b];
  *sum = t;
}

// out = sum_g exp(lse_g - lse) o_g, lse = logsumexp_g lse_g (empty shards: -inf)
__global__ void lse_merge_kernel(const float* __restrict__ o_parts,
                                 const float* __restrict__ lse_parts, int parts, int64_t rows,
                                 int dim, float* __restrict__ out, float* __restrict__ lse_out) {
  const int64_t row = blockIdx.x;
  if (row >= rows) return;
  float m = -INFINITY;
  for (int g = 0; g < parts; ++g) m = fmaxf(m, lse_parts[int64_t(g) * rows + row]);
  float den = 0.f;
  for (int g = 0; g < parts; ++g) {
    const float l = lse_parts[int64_t(g) * rows + row];
    if (l != -INFINITY) den += expf(l - m);
  }
  for (int d = threadIdx.x; d < dim; d += blockDim.x) {
    float acc = 0.f;
    for (int g = 0; g < parts; ++g) {
      const float l = lse_parts[int64_t(g) * rows + row];
      if (l != -INFINITY) acc += expf(l - m) * o_parts[(int64_t(g) * rows + row) * dim + d];
    }
    out[row * dim + d] = acc / den;
  }
  if (threadIdx.x == 0) lse_out[row] = m + logf(den);
}

// lse_out = logsumexp_g lse_all[g]; o *= exp(lse_own - lse_out) (0 where lse_own = -inf)
__global__ void lse_scale_kernel(float* __restrict__ o, const float* __restrict__ lse_own,
                                 const float* __restrict__ lse_all, int parts, int64_t n, int hq,
                                 int dim, float* __restrict__ lse_out) {
  const int64_t idx = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);  // (i, h)
  if (idx >= n * hq) return;
  const int64_t i = idx / hq;
  const int h = int(idx - i * hq);
  const int64_t li = int64_t(h) * n + i;
  float m = -INFINITY;
  for (int g = 0; g < parts; ++g) m = fmaxf(m, lse_all[int64_t(g) * hq * n + li]);
  float den = 0.f;
  for (int g = 0; g < parts; ++g) {
    const float l = lse_all[int64_t(g) * hq * n + li];
    if (l != -INFINITY) den += expf(l - m);
  }
  const float tot = m == -INFINITY ? -INFINITY : m + logf(den);
  const float own = lse_own[li];
  const float w = own == -INFINITY ? 0.f : expf(own - tot);
  float* row = o + idx * dim;
  for (int d = threadIdx.x & 31; d < dim; d += 32) row[d] *= w;
  if ((threadIdx.x & 31) == 0 && lse_out) lse_out[li] = tot;
}

// recall[h] = mean over rows [i0, i1) of min(1, exp(lse_s[h][i] - lse_f[h][i - f0]))
// (refine.cpp:51-72 with the clamp; one block per head)
__global__ void chunk_recall_kernel(const float* __restrict__ lse_s, int64_t s_stride,
                                    const float* __restrict__ lse_f, int64_t f_stride,
                                    int64_t f0, int64_t i0, int64_t i1, float* __restrict__ out) {
  __shared__ float red[32];
  const int h = blockIdx.x;
  float acc = 0.f;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const float d = lse_s[int64_t(h) * s_stride + i] - lse_f[int64_t(h) * f_stride + (i - f0)];
    acc += fminf(1.f, expf(d));
  }
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    out[h] = i1 > i0 ? t / float(i1 - i0) : 1.f;
  }
}

}  // namespace

int chunk_recall_launch(const float* lse_s, int64_t s_stride, const float* lse_f,
                        int64_t f_stride, int64_t f0, int64_t i0, int64_t i1, int hq, float* out,
                        cudaStream_t st) {
  chunk_recall_kernel<<<hq, 256, 0, st>>>(lse_s, s_stride, lse_f, f_stride, f0, i0, i1, out);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int lse_scale_launch(float* o, const float* lse_own, const float* lse_all, int parts, int64_t n,
                     int hq, int dim, float* lse_out, cudaStream_t st) {
  const int64_t rows = n * hq;
  if (rows <= 0) return LCX_OK;
  lse_scale_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(o, lse_own, lse_all, parts, n, hq,
                                                             dim, lse_out);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int build_rope_table(const double* thetas_dev, int P, int64_t npos, float2* out,
                     cudaStream_t st) {
  const int64_t total = npos * P;
  rope_table_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(thetas_dev, P, npos, out);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int build_bitmaps(const int32_t* lists, const int32_t* counts, int64_t cap, int heads,
                  int64_t words, uint32_t* bits, cudaStream_t st) {
  LCX_CHECK_CUDA(cudaMemsetAsync(bits, 0, sizeof(uint32_t) * size_t(words) * heads, st));
  dim3 grid(8, unsigned(heads));
  bitmap_kernel<<<grid, 256, 0, st>>>(lists, counts, cap, words, bits);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

// sum_dev: kRecallBlocks + 1 doubles (block partials, then the total)
int recall_kernel_launch(const float* ls, const float* lf, int64_t n, double slack, float* per,
                         double* sum_dev, int* bad_dev, cudaStream_t st) {
  LCX_CHECK_CUDA(cudaMemsetAsync(bad_dev, 0, sizeof(int), st));
  const int blocks =
      int(std::max<int64_t>(1, std::min<int64_t>(kRecallBlocks, (n + 255) / 256)));
  recall_kernel<<<unsigned(blocks), 256, 0, st>>>(ls, lf, n, slack, per, sum_dev + 1, bad_dev);
  LCX_CHECK_LAUNCH();
  recall_final_kernel<<<1, 1, 0, st>>>(sum_dev + 1, blocks, sum_dev);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int lse_merge_launch(const float* o_parts, const float* lse_parts, int parts, int64_t rows,
                     int dim, float* out, float* lse_out, cudaStream_t st) {
  if (rows <= 0) return LCX_OK;
  lse_merge_kernel<<<unsigned(rows), 128, 0, st>>>(o_parts, lse_parts, parts, rows, dim, out,
                                                   lse_out);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

}  // namespace lcx
