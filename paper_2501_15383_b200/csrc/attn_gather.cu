// K4b -- CUDA-core gather for the slash entries the tcgen05 tiles do not cover
// (isolated diagonals), bf16 storage / tensor-core mode.
//
// Entry (i, j = i - d) of a selected diagonal d (reference CriticalSet::admitted_row,
// core/src/sparse.cpp:85-113) whose 64-key relative tile was not worth a tensor-core
// tile.  Such an entry shares its K and V rows with no other entry of the row block,
// so this is a gather bounded by HBM traffic; the kernel is laid out for bandwidth:
//   * only the raw bf16 K row and V row are read per entry (2 x 256 B -- the floor for
//     this access pattern); the logit is rope(q_i, rel) . k_j with
//     rel = dca_relative(i, j) (DCA, dca.cpp:62-80) or pos_q[i] - pos_k[j] (standard,
//     sparse.cpp:385-398), and cos / sin(rel * theta_p) is rebuilt by angle addition
//     from the fp64-derived table: rope[rel] = rope[64 * (rel >> 6)] (x) rope[rel & 63],
//     the 64-row low table held in shared memory, the high row an L1 / L2 hit (rel is
//     constant along a diagonal inside one DCA chunk pair and moves by one per row
//     otherwise);
//   * 16 lanes per query row (8 dims each, one 16-byte load per K / V row), and the
//     16 lanes scan 16 diagonals of the row's segment list at once (ballot), so up to
//     four entries' loads are in flight before the first is reduced;
//   * segments (d, first row, last row) come pre-split per 64-row half of the block
//     (classify_kernel), so a row scans only diagonals that can reach it.
// The tensor-core partial (o_tc, lse_tc) of the row is the initial online-softmax state;
// rows with no entry here keep it untouched.  Entries on a vertical column belong to the
// vertical tiles (V∩S counted once, sparse.cpp:95-108).
#include "lcx_internal.cuh"
#include "attn_gather.cuh"

namespace lcx {
namespace {

constexpr int kRows = 16;    // rows per CTA
constexpr int kLanes = 16;   // lanes per row
constexpr int kDims = 8;     // dims per lane (4 RoPE pairs)
constexpr int kThreads = kRows * kLanes;
constexpr int kBatch = 4;    // entries in flight per row

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    f[2 * t] = __uint_as_float(w[t] << 16);
    f[2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u);
  }
}

// relative rotation position of entry (i, j)
__device__ __forceinline__ int64_t rel_of(const GatherArgs& a, int64_t i, int64_t j,
                                          int64_t pq_i, int64_t qc, int64_t imod) {
  if (a.rel_mode == 1) {
    const int64_t c0 = qc * a.s;
    if (j >= c0) return i - j;                                   // intra: (i - c0) - (j - c0)
    if (j >= c0 - a.s) return lcx_min64(imod + a.s, a.c - 1) - (j - (c0 - a.s));  // successive
    return a.c - 1 - int64_t(uint32_t(j) % uint32_t(a.s));       // inter
  }
  return pq_i - (a.pos_k ? a.pos_k[j] : j);
}

__global__ void __launch_bounds__(kThreads, 3) attn_gather_kernel(const GatherArgs a) {
  __shared__ float4 lo_tab[64 * 32];  // rope[0..63][64 pairs] as (cos, sin, cos, sin)
  for (int x = threadIdx.x; x < 64 * 32; x += kThreads)
    lo_tab[x] = reinterpret_cast<const float4*>(a.rope)[x];
  __syncthreads();

  const int lane = threadIdx.x & (kLanes - 1);
  const int rw = threadIdx.x / kLanes;
  const int64_t i = a.row_begin + int64_t(blockIdx.x) * kRows + rw;
  const int h = blockIdx.y;
  const int g = h / a.group;
  const unsigned gmask = 0xffffu << (threadIdx.x & 16);
  if (i >= a.row_end) return;

  float qx[4], qy[4];
  {
    float qf[8];
    bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(a.q + (i * a.hq + h) * 128) + lane), qf);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      qx[t] = qf[2 * t];
      qy[t] = qf[2 * t + 1];
    }
  }
  // initial state = the tensor-core partial of this row (normalised o, lse)
  float o[kDims], m = -INFINITY, l = 0.f;
  const float lp = a.lse[int64_t(h) * a.lse_stride + i];
  float* orow = a.out + (i * a.hq + h) * 128 + lane * kDims;
  if (lp != -INFINITY) {
    m = lp * 1.4426950408889634f;  // log2 domain
    l = 1.f;
    const float4 x0 = reinterpret_cast<const float4*>(orow)[0];
    const float4 x1 = reinterpret_cast<const float4*>(orow)[1];
    o[0] = x0.x; o[1] = x0.y; o[2] = x0.z; o[3] = x0.w;
    o[4] = x1.x; o[5] = x1.y; o[6] = x1.z; o[7] = x1.w;
  } else {
#pragma unroll
    for (int t = 0; t < kDims; ++t) o[t] = 0.f;
  }

  const int r = int((i - a.row_begin) & 127);
  const int half = r >> 6;
  const int4* sg = a.segs + (int64_t(h) * 2 + half) * a.cap_seg;
  const int nseg = a.nseg[h * 2 + half];
  const uint32_t* vb = a.vbits + int64_t(h) * a.words;
  const int64_t qc = a.rel_mode == 1 ? i / a.s : 0;
  const int64_t imod = i - qc * a.s;
  const int64_t pq_i = a.rel_mode == 1 ? 0 : (a.pos_q ? a.pos_q[i] : i);
  const __nv_bfloat16* kbase = a.k + int64_t(g) * 128 + lane * kDims;
  const __nv_bfloat16* vbase = a.v + int64_t(g) * 128 + lane * kDims;
  const int64_t row_stride = int64_t(a.hkv) * 128;

  int64_t entries = 0;
  // one entry: rotate q by rel (angle addition), dot with raw k, online softmax, o += p v
  auto hi_row = [&](int64_t rel) {
    const int64_t ar = rel < 0 ? -rel : rel;
    return reinterpret_cast<const float4*>(a.rope + (ar >> 6) * 64 * 64) + lane * 2;
  };
  auto consume = [&](int64_t rel, const uint4& kr, const uint4& vr) {
    const float sgn = rel < 0 ? -1.f : 1.f;
    const int64_t ar = rel < 0 ? -rel : rel;
    const float4* hp = hi_row(rel);
    const float4 h0 = __ldg(hp), h1 = __ldg(hp + 1);
    const float4 l0 = lo_tab[(ar & 63) * 32 + lane * 2], l1 = lo_tab[(ar & 63) * 32 + lane * 2 + 1];
    const float hc[4] = {h0.x, h0.z, h1.x, h1.z}, hs[4] = {h0.y, h0.w, h1.y, h1.w};
    const float lc[4] = {l0.x, l0.z, l1.x, l1.z}, ls[4] = {l0.y, l0.w, l1.y, l1.w};
    float kf[8];
    bf16x8_to_f32(kr, kf);
    float dot = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float c = hc[t] * lc[t] - hs[t] * ls[t];
      const float s = sgn * (hs[t] * lc[t] + hc[t] * ls[t]);
      const float rx = qx[t] * c - qy[t] * s, ry = qx[t] * s + qy[t] * c;
      dot = fmaf(rx, kf[2 * t], dot);
      dot = fmaf(ry, kf[2 * t + 1], dot);
    }
    dot += __shfl_xor_sync(gmask, dot, 1);
    dot += __shfl_xor_sync(gmask, dot, 2);
    dot += __shfl_xor_sync(gmask, dot, 4);
    dot += __shfl_xor_sync(gmask, dot, 8);
    const float s2 = dot * a.scale_log2;
    const float mn = fmaxf(m, s2);
    const float corr = exp2f(m - mn);
    const float p = exp2f(s2 - mn);
    l = l * corr + p;
    float vf[8];
    bf16x8_to_f32(vr, vf);
#pragma unroll
    for (int t = 0; t < kDims; ++t) o[t] = fmaf(p, vf[t], o[t] * corr);
    m = mn;
    ++entries;
  };

  for (int x0 = 0; x0 < nseg; x0 += kLanes) {
    // lane k examines diagonal x0 + k of the (ascending-d) list
    const int xi = x0 + lane;
    bool ok = false, stop = false;
    int64_t jj = 0;
    if (xi < nseg) {
      const int4 e = sg[xi];
      if (int64_t(e.x) > i) {
        stop = true;
      } else if (r >= e.y && r < e.z) {
        jj = i - e.x;
        ok = !((vb[jj >> 5] >> (jj & 31)) & 1u);
      }
    }
    unsigned okm = __ballot_sync(gmask, ok) >> (threadIdx.x & 16);
    const unsigned stopm = __ballot_sync(gmask, stop) >> (threadIdx.x & 16);
    while (okm) {
      int64_t js[kBatch];
      int nb = 0;
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        if (okm) {
          const int src = __ffs(okm) - 1;
          okm &= okm - 1;
          js[b] = __shfl_sync(gmask, (long long)jj, src, kLanes);
          ++nb;
        } else {
          js[b] = -1;
        }
      }
      uint4 kr[kBatch], vr[kBatch];
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        if (b < nb) {
          kr[b] = __ldg(reinterpret_cast<const uint4*>(kbase + js[b] * row_stride));
          vr[b] = __ldg(reinterpret_cast<const uint4*>(vbase + js[b] * row_stride));
        }
      }
#pragma unroll
      for (int b = 0; b < kBatch; ++b)
        if (b < nb) consume(rel_of(a, i, js[b], pq_i, qc, imod), kr[b], vr[b]);
    }
    if (stopm) break;
  }

  // self fallback (sparse.cpp:111): no vertical <= i and no slash <= i at all
  const int nvh = a.nv[h], nsh = a.ns[h];
  const bool any = (nvh > 0 && int64_t(a.verts[int64_t(h) * a.cap_v]) <= i) ||
                   (nsh > 0 && int64_t(a.slashes[int64_t(h) * a.cap_s]) <= i);
  if (!any && a.do_fallback) {
    m = -INFINITY;
    l = 0.f;
#pragma unroll
    for (int t = 0; t < kDims; ++t) o[t] = 0.f;
    entries = 0;
    consume(rel_of(a, i, i, pq_i, qc, imod),
            __ldg(reinterpret_cast<const uint4*>(kbase + i * row_stride)),
            __ldg(reinterpret_cast<const uint4*>(vbase + i * row_stride)));
  }
  if (entries == 0) return;  // the tensor-core result stands

  const float inv_l = 1.f / l;
  reinterpret_cast<float4*>(orow)[0] = make_float4(o[0] * inv_l, o[1] * inv_l, o[2] * inv_l, o[3] * inv_l);
  reinterpret_cast<float4*>(orow)[1] = make_float4(o[4] * inv_l, o[5] * inv_l, o[6] * inv_l, o[7] * inv_l);
  if (lane == 0) {
    a.lse[int64_t(h) * a.lse_stride + i] = (m + log2f(l)) * 0.6931471805599453f;
    if (a.simt_count)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.simt_count), (unsigned long long)entries);
  }
}

}  // namespace

int attention_gather(const GatherArgs& a, cudaStream_t st) {
  const int64_t rows = a.row_end - a.row_begin;
  if (rows <= 0) return LCX_OK;
  if (a.row_begin % 128 != 0) return fail(LCX_ERR_INTERNAL, "gather rows must start a block");
  dim3 grid(unsigned((rows + kRows - 1) / kRows), unsigned(a.hq));
  attn_gather_kernel<<<grid, kThreads, 0, st>>>(a);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

}  // namespace lcx
