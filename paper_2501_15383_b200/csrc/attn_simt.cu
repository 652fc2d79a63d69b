// K4 (CUDA-core path) -- exact per-entry sparse / dense attention.
//
// One quad (4 lanes) per query row, 32 rows per CTA.  For every admitted entry
// (reference CriticalSet::admitted_row, core/src/sparse.cpp:85-113) the quad
// forms logit = rope(q_i, rel(i, j)) . k_j * scale with
//   rel = pos_q[i] - pos_k[j]           (standard path: rope(q,a).rope(k,b) ==
//                                         rope(q, a-b).k, sparse.cpp:385-398)
//   rel = dca_relative(i, j)            (DCA override path, sparse.cpp:400-412,
//                                         chunked_prefill sparse.cpp:385-393)
// using the fp64-derived cos/sin table, then an fp32 online softmax + value
// accumulation (same result as the reference's two-pass attend_admitted,
// attention.cpp:35-51, within fp32 rounding).
//
// Entry enumeration per row:
//   verticals v <= i (skipped when the tcgen05 path owns them),
//   slashes d <= i -> j = i - d, skipping keys that are verticals (an entry
//   on both a vertical and a selected diagonal is counted once, by the
//   vertical path; sparse.cpp:95-108 dedupe),
//   no admitted entry -> the self entry j = i (sparse.cpp:111).
// This is the complete exact-fp32 path (fp32 storage, any head dim <= 128, any
// positions); in tensor-core mode the isolated slash entries go to attn_gather.cu.
#include "lcx_internal.cuh"

namespace lcx {
namespace {

constexpr int kRowsPerCta = 32;

template <typename T, int PPL>
struct RowState {
  float qx[PPL], qy[PPL];
  float o[2 * PPL];
  float m, l;
};

template <typename T, int PPL>
__device__ __forceinline__ void process_entry(const AttnArgs& a, RowState<T, PPL>& s,
                                              int64_t i, int64_t j, int64_t pq_i, int g,
                                              int lane4, unsigned qmask) {
  const int P = a.dim >> 1;
  int64_t rel;
  if (a.rel_mode == 1) {
    rel = dca_relative(i, j, a.s, a.c);
  } else if (a.rel_mode == 2) {
    rel = a.rel_mat[i * a.rel_n + j];  // explicit RelPositionMatrix (attention.cpp:173-183)
  } else {
    const int64_t pk = a.pos_k ? a.pos_k[j] : j;
    rel = pq_i - pk;
  }
  const float sgn = rel < 0 ? -1.f : 1.f;
  const int64_t arel = rel < 0 ? -rel : rel;
  const float2* cs = a.rope + arel * P;
  const T* kr = reinterpret_cast<const T*>(a.k) + (j * a.hkv + g) * int64_t(a.dim);
  float dot = 0.f;
#pragma unroll
  for (int t = 0; t < PPL; ++t) {
    const int p = lane4 + 4 * t;
    if (p < P) {
      const float2 c = cs[p];
      const float sn = sgn * c.y;
      const float kx = load_elem(kr, 2 * p), ky = load_elem(kr, 2 * p + 1);
      const float rx = s.qx[t] * c.x - s.qy[t] * sn;
      const float ry = s.qx[t] * sn + s.qy[t] * c.x;
      dot = fmaf(rx, kx, dot);
      dot = fmaf(ry, ky, dot);
    }
  }
  dot += __shfl_xor_sync(qmask, dot, 1);
  dot += __shfl_xor_sync(qmask, dot, 2);
  const float logit = dot * a.scale;
  const float mn = fmaxf(s.m, logit);
  const float corr = expf(s.m - mn);  // exp(-inf) = 0 on the first entry
  const float p = expf(logit - mn);
  s.l = s.l * corr + p;
  const T* vr = reinterpret_cast<const T*>(a.v) + (j * a.hkv + g) * int64_t(a.dim);
#pragma unroll
  for (int t = 0; t < PPL; ++t) {
    const int pp = lane4 + 4 * t;
    if (pp < P) {
      const float vx = load_elem(vr, 2 * pp), vy = load_elem(vr, 2 * pp + 1);
      s.o[2 * t] = fmaf(p, vx, s.o[2 * t] * corr);
      s.o[2 * t + 1] = fmaf(p, vy, s.o[2 * t + 1] * corr);
    }
  }
  s.m = mn;
}

__device__ __forceinline__ bool is_vertical(const uint32_t* bits, int64_t j) {
  return (bits[j >> 5] >> (j & 31)) & 1u;
}

template <typename T, int PPL>
__global__ void __launch_bounds__(128) attn_simt_kernel(AttnArgs a) {
  const int lane4 = threadIdx.x & 3;
  const int64_t i = a.row_begin + int64_t(blockIdx.x) * kRowsPerCta + (threadIdx.x >> 2);
  const int h = blockIdx.y;
  const int g = h / (a.hq / a.hkv);
  const unsigned qmask = 0xFu << (threadIdx.x & 28);
  if (i >= a.row_end) return;
  const int P = a.dim >> 1;

  RowState<T, PPL> s;
  const T* qr = reinterpret_cast<const T*>(a.q) + (i * a.hq + h) * int64_t(a.dim);
#pragma unroll
  for (int t = 0; t < PPL; ++t) {
    const int p = lane4 + 4 * t;
    s.qx[t] = p < P ? load_elem(qr, 2 * p) : 0.f;
    s.qy[t] = p < P ? load_elem(qr, 2 * p + 1) : 0.f;
    s.o[2 * t] = 0.f;
    s.o[2 * t + 1] = 0.f;
  }
  s.m = -INFINITY;
  s.l = 0.f;
  const int64_t pq_i = a.pos_q ? a.pos_q[i] : i;
  int64_t entries = 0;

  if (a.dense) {
    for (int64_t j = 0; j <= i; ++j) process_entry<T, PPL>(a, s, i, j, pq_i, g, lane4, qmask);
    entries = i + 1;
  } else {
    const int32_t* verts = a.verts + int64_t(h) * a.cap_v;
    const int32_t* sl = a.slashes + int64_t(h) * a.cap_s;
    const int nv = a.nv[h], ns = a.ns[h];
    const uint32_t* vb = a.vbits + int64_t(h) * a.bit_words;
    const int fnv = a.fnv[h], fns = a.fns[h];
    const bool any = (fnv > 0 && a.fverts[int64_t(h) * a.cap_v] <= i) ||
                     (fns > 0 && a.fslashes[int64_t(h) * a.cap_s] <= i);
    for (int x = 0; x < nv; ++x) {
      const int64_t v = verts[x];
      if (v > i) break;
      process_entry<T, PPL>(a, s, i, v, pq_i, g, lane4, qmask);
      ++entries;
    }
    for (int x = 0; x < ns; ++x) {
      const int64_t d = sl[x];
      if (d > i) break;
      const int64_t j = i - d;
      if (is_vertical(vb, j)) continue;
      process_entry<T, PPL>(a, s, i, j, pq_i, g, lane4, qmask);
      ++entries;
    }
    if (!any && a.do_fallback) {  // self fallback (sparse.cpp:111)
      process_entry<T, PPL>(a, s, i, i, pq_i, g, lane4, qmask);
      entries = 1;
    }
  }

  const float inv_l = s.l > 0.f ? 1.f / s.l : 0.f;  // no entry on this shard: o = 0, lse = -inf
  float* orow = a.out + (i * a.hq + h) * int64_t(a.dim);
#pragma unroll
  for (int t = 0; t < PPL; ++t) {
    const int p = lane4 + 4 * t;
    if (p < P) {
      orow[2 * p] = s.o[2 * t] * inv_l;
      orow[2 * p + 1] = s.o[2 * t + 1] * inv_l;
    }
  }
  if (lane4 == 0) {
    a.lse[int64_t(h) * a.lse_stride + i] = s.m + logf(s.l);
    if (a.admitted) atomicAdd(reinterpret_cast<unsigned long long*>(a.admitted + h),
                                         (unsigned long long)entries);
    if (a.simt_count) atomicAdd(reinterpret_cast<unsigned long long*>(a.simt_count),
                                (unsigned long long)entries);
  }
}

template <typename T>
int launch_t(const AttnArgs& a, cudaStream_t st) {
  const int P = a.dim / 2;
  const int64_t rows = a.row_end - a.row_begin;
  if (rows <= 0) return LCX_OK;
  dim3 grid(unsigned((rows + kRowsPerCta - 1) / kRowsPerCta), unsigned(a.hq));
  if (P <= 4) attn_simt_kernel<T, 1><<<grid, 128, 0, st>>>(a);
  else if (P <= 8) attn_simt_kernel<T, 2><<<grid, 128, 0, st>>>(a);
  else if (P <= 16) attn_simt_kernel<T, 4><<<grid, 128, 0, st>>>(a);
  else if (P <= 32) attn_simt_kernel<T, 8><<<grid, 128, 0, st>>>(a);
  else if (P <= 64) attn_simt_kernel<T, 16><<<grid, 128, 0, st>>>(a);
  else return fail(LCX_ERR_CONFIG, "head dim > 128 not supported");
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

}  // namespace

int attention_simt(const AttnArgs& a, cudaStream_t st) {
  return a.dtype == LCX_BF16 ? launch_t<__nv_bfloat16>(a, st) : launch_t<float>(a, st);
}

}  // namespace lcx
