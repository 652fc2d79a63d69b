// K4b -- CUDA-core gather for the slash entries the tcgen05 tiles do not cover
// (isolated diagonals), bf16 storage / tensor-core mode.
//
// Entry (i, j = i - d) of a selected diagonal d (reference CriticalSet::admitted_row,
// core/src/sparse.cpp:85-113) whose 64-key relative tile was not worth a tensor-core
// tile.  Such an entry shares its K and V rows with no other entry of its row, so each
// costs one K row and one V row of traffic and a 128-long dot product; the kernel keeps
// both the traffic in L2 and the per-entry instruction count low:
//   * key-segment passes (the caller sweeps [key_lo, key_hi) windows of 32K keys): every
//     row of every head reads only the K / V rows of the current window, which stay
//     L2-resident while all diagonals hit them (96 % L2 hits at 1M tokens, vs 40 %
//     without the passes); the running (o, lse) of each row is carried in out / lse;
//   * the keys are the fp32 rope(k_j, kpos(j)) rows prepared once per chunk with the
//     tensor-core operands (kpos = j mod s under DCA, pos_k[j] standard), and the query
//     is rotated once per DCA pattern (intra / successive / inter: the pattern only
//     changes twice along a row's descending keys), so
//       logit = rope(q_i, qpos(i, pattern)) . rope(k_j, kpos(j)) * scale
//             == rope(q_i, dca_relative(i, j)) . k_j * scale          (dca.cpp:62-80)
//     with no per-entry trigonometry or table reads;
//   * 16 lanes per query row, 8 dims each (two 16-byte loads of K, one of V), two
//     entries in flight per row, and one online-softmax update per pair of entries;
//     80 registers, 3 CTAs (24 warps) per SM.  Measured at 1M (planted, per layer):
//     8 lanes x 16 dims at 2 CTAs 78 ms, 16 x 8 at 3 CTAs 68-72 ms, at 4 CTAs (spills)
//     68 ms, 16 x 8 with 3 or 4 entries in flight 80-89 ms, 32 x 4 at 4 CTAs 78 ms;
//   * the lanes of a row scan as many diagonals of its sorted segment list at once
//     (ballot);
//     segments (d, first row, last row) come pre-split per 64-row half of the block.
// The tensor-core partial (o_tc, lse_tc) of the row is the initial state; rows with no
// entry in this pass keep their state untouched.  Entries on a vertical column belong to
// the vertical tiles (V∩S counted once, sparse.cpp:95-108).
#include "lcx_internal.cuh"
#include "attn_gather.cuh"

namespace lcx {
namespace {

#ifndef LCX_GATHER_LANES
#define LCX_GATHER_LANES 16
#endif
constexpr int kLanes = LCX_GATHER_LANES;  // lanes per row (8 or 16)
constexpr int kDims = 128 / kLanes;       // dims per lane
// 128-thread CTAs at 6 per SM: the gather itself 72 -> 68 ms, but the attention kernel
// running beside it loses as much (363 vs 359 ms): step time equal, kept at 256
#ifndef LCX_GATHER_THREADS
#define LCX_GATHER_THREADS 256
#endif
constexpr int kRows = LCX_GATHER_THREADS / kLanes;  // rows per CTA
constexpr int kThreads = kRows * kLanes;
#ifndef LCX_GATHER_MINB
#define LCX_GATHER_MINB (LCX_GATHER_LANES == 16 ? 3 : 2)
#endif
constexpr int kMinBlocks = LCX_GATHER_MINB;  // resident CTAs per SM
#ifndef LCX_GATHER_INFLIGHT
#define LCX_GATHER_INFLIGHT 2
#endif
constexpr int kInflight = LCX_GATHER_INFLIGHT;
#ifndef LCX_GATHER_DIAG
#define LCX_GATHER_DIAG 1  // diagonal-major kernel (below); 0: row-major list scan
#endif  // entries of a row loaded at once
static_assert(kLanes == 8 || kLanes == 16 || kLanes == 32, "8, 16 or 32 lanes per row");
constexpr int kVVec = kDims >= 8 ? kDims / 8 : 1;  // 16-byte (or one 8-byte) V loads per lane

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    f[2 * t] = __uint_as_float(w[t] << 16);
    f[2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u);
  }
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct KVRow {
  float4 k[kDims / 4];
  uint4 v[kVVec];  // kDims == 4: only .x / .y used
};

// kDims bf16 values at p (16-byte aligned for kDims >= 8, 8-byte for 4) -> fp32
__device__ __forceinline__ void load_bf16(const __nv_bfloat16* p, float* f) {
  if constexpr (kDims >= 8) {
#pragma unroll
    for (int t = 0; t < kDims / 8; ++t)
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(p) + t), f + 8 * t);
  } else {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    f[0] = __uint_as_float(u.x << 16);
    f[1] = __uint_as_float(u.x & 0xffff0000u);
    f[2] = __uint_as_float(u.y << 16);
    f[3] = __uint_as_float(u.y & 0xffff0000u);
  }
}

__device__ __forceinline__ void load_row(const float* kf, const __nv_bfloat16* vb, int64_t j,
                                         int64_t stride, KVRow& r) {
  const float4* kp = reinterpret_cast<const float4*>(kf + j * stride);
  const uint4* vp = reinterpret_cast<const uint4*>(vb + j * stride);
#pragma unroll
  for (int t = 0; t < kDims / 4; ++t) r.k[t] = __ldg(kp + t);
  if constexpr (kDims >= 8) {
#pragma unroll
    for (int t = 0; t < kDims / 8; ++t) r.v[t] = __ldg(vp + t);
  } else {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(vp));
    r.v[0] = make_uint4(u.x, u.y, 0u, 0u);
  }
}

__device__ __forceinline__ int64_t qpos_of(const GatherArgs& a, int pattern, int64_t i,
                                           int64_t imod) {
  if (a.rel_mode == 0) return a.pos_q ? a.pos_q[i] : i;
  if (pattern == 0) return imod;
  if (pattern == 1) return lcx_min64(imod + a.s, a.c - 1);
  return a.c - 1;
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) attn_gather_kernel(const GatherArgs a) {
  // a window with no segment (and before the chunk's rows: no self-fallback rows) is empty
  if (a.win_flags && !a.win_flags[a.win] && a.key_hi <= a.row_begin) return;
  const int lane = threadIdx.x & (kLanes - 1);
  const int rw = threadIdx.x / kLanes;
  const int64_t i = a.row_begin + int64_t(blockIdx.x) * kRows + rw;
  const int h = blockIdx.y;
  const int g = h / a.group;
  constexpr unsigned kRowMask = kLanes == 32 ? 0xffffffffu : (1u << (kLanes & 31)) - 1u;
  const int lane0 = threadIdx.x & (32 - kLanes);  // first lane of this row in the warp
  const unsigned gmask = kRowMask << lane0;
  if (i >= a.row_end) return;

  const int r = int((i - a.row_begin) & 127);
  const int half = r >> 6;
  const int4* sg = a.segs + (int64_t(h) * 2 + half) * a.cap_seg;
  const int nseg = a.nseg[h * 2 + half];
  // this pass's key window [key_lo, key_hi): diagonals d in [i - key_hi + 1, i - key_lo]
  int xs = 0;
  {
    const int64_t dmin = i - a.key_hi + 1;
    int lo = 0, hi = nseg;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (int64_t(sg[mid].x) < dmin) lo = mid + 1;
      else hi = mid;
    }
    xs = lo;
  }
  const int64_t dmax = lcx_min64(i, i - a.key_lo);
  const int nvh = a.nv[h], nsh = a.ns[h];
  const bool any = (nvh > 0 && int64_t(a.verts[int64_t(h) * a.cap_v]) <= i) ||
                   (nsh > 0 && int64_t(a.slashes[int64_t(h) * a.cap_s]) <= i);
  const bool fallback = !any && a.do_fallback && i >= a.key_lo && i < a.key_hi;
  if (!fallback && (xs >= nseg || int64_t(sg[xs].x) > dmax)) return;  // nothing in this pass

  float qraw[kDims];
  {
    const uint4* qp = reinterpret_cast<const uint4*>(a.q + (i * a.hq + h) * 128 + lane * kDims);
    load_bf16(reinterpret_cast<const __nv_bfloat16*>(qp), qraw);
  }
  // running state = the partial so far (tensor-core tiles + earlier passes)
  float o[kDims], m = -INFINITY, l = 0.f;
  const float lp = a.lse[int64_t(h) * a.lse_stride + i];
  float* orow = a.out + (i * a.hq + h) * 128 + lane * kDims;
  if (lp != -INFINITY && !fallback) {
    m = lp * 1.4426950408889634f;  // log2 domain
    l = 1.f;
#pragma unroll
    for (int t = 0; t < kDims; t += 4) {
      const float4 x = reinterpret_cast<const float4*>(orow)[t / 4];
      o[t] = x.x;
      o[t + 1] = x.y;
      o[t + 2] = x.z;
      o[t + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int t = 0; t < kDims; ++t) o[t] = 0.f;
  }

  const int64_t qc = a.rel_mode == 1 ? i / a.s : 0;
  const int64_t imod = i - qc * a.s;
  const int64_t c_intra = qc * a.s, c_succ = c_intra - a.s;  // DCA pattern thresholds
  const uint32_t* vb = a.vbits + int64_t(h) * a.words;
  const float* kf = a.kf + int64_t(g) * 128 + lane * kDims;
  const __nv_bfloat16* vbase = a.v + int64_t(g) * 128 + lane * kDims;
  const int64_t stride = int64_t(a.hkv) * 128;

  float qr[kDims];
  int cur_pat = -1;
  auto ensure_pattern = [&](int64_t j) {
    const int pat = a.rel_mode != 1 ? 0 : (j >= c_intra ? 0 : (j >= c_succ ? 1 : 2));
    if (pat == cur_pat) return;
    cur_pat = pat;
    const float4* cs = reinterpret_cast<const float4*>(a.rope + qpos_of(a, pat, i, imod) * 64 +
                                                       lane * (kDims / 2));
#pragma unroll
    for (int t = 0; t < kDims / 4; ++t) {
      const float4 c = __ldg(cs + t);
      const float x0 = qraw[4 * t], y0 = qraw[4 * t + 1], x1 = qraw[4 * t + 2];
      const float y1 = qraw[4 * t + 3];
      qr[4 * t] = x0 * c.x - y0 * c.y;
      qr[4 * t + 1] = x0 * c.y + y0 * c.x;
      qr[4 * t + 2] = x1 * c.z - y1 * c.w;
      qr[4 * t + 3] = x1 * c.w + y1 * c.z;
    }
  };
  auto dot_of = [&](const KVRow& kv) {
    float d0 = 0.f, d1 = 0.f;
#pragma unroll
    for (int t = 0; t < kDims / 4; ++t) {
      d0 = fmaf(qr[4 * t], kv.k[t].x, d0);
      d1 = fmaf(qr[4 * t + 1], kv.k[t].y, d1);
      d0 = fmaf(qr[4 * t + 2], kv.k[t].z, d0);
      d1 = fmaf(qr[4 * t + 3], kv.k[t].w, d1);
    }
    float d = d0 + d1;
    d += __shfl_xor_sync(gmask, d, 1);
    d += __shfl_xor_sync(gmask, d, 2);
    d += __shfl_xor_sync(gmask, d, 4);
    if constexpr (kLanes >= 16) d += __shfl_xor_sync(gmask, d, 8);
    if constexpr (kLanes >= 32) d += __shfl_xor_sync(gmask, d, 16);
    return d * a.scale_log2;
  };
  auto accumulate = [&](float p, const KVRow& kv) {
    float vf[kDims];
    if constexpr (kDims >= 8) {
#pragma unroll
      for (int t = 0; t < kDims / 8; ++t) bf16x8_to_f32(kv.v[t], vf + 8 * t);
    } else {
      vf[0] = __uint_as_float(kv.v[0].x << 16);
      vf[1] = __uint_as_float(kv.v[0].x & 0xffff0000u);
      vf[2] = __uint_as_float(kv.v[0].y << 16);
      vf[3] = __uint_as_float(kv.v[0].y & 0xffff0000u);
    }
#pragma unroll
    for (int t = 0; t < kDims; ++t) o[t] = fmaf(p, vf[t], o[t]);
  };
  // online-softmax rescale, only when the running max grows
  auto raise_max = [&](float s0, float s1) {
    const float mn = fmaxf(m, fmaxf(s0, s1));
    if (mn > m) {
      const float corr = exp2f(m - mn);  // exp2(-inf) = 0 on the first entry
      l *= corr;
#pragma unroll
      for (int t = 0; t < kDims; ++t) o[t] *= corr;
      m = mn;
    }
  };

  int64_t entries = 0;
  for (int x0 = xs; x0 < nseg; x0 += kLanes) {
    // lane k examines diagonal x0 + k of the (ascending-d) list
    const int xi = x0 + lane;
    bool ok = false, stop = false;
    int64_t jj = 0;
    if (xi < nseg) {
      const int4 e = sg[xi];
      if (int64_t(e.x) > dmax) {
        stop = true;
      } else if (r >= e.y && r < e.z) {
        jj = i - e.x;
        ok = !((vb[jj >> 5] >> (jj & 31)) & 1u);
      }
    }
    unsigned okm = (__ballot_sync(gmask, ok) >> lane0) & kRowMask;
    const unsigned stopm = (__ballot_sync(gmask, stop) >> lane0) & kRowMask;
    while (okm) {
      // up to kInflight entries of this row at once: loads first, then the math
      int64_t jv[kInflight];
      int cnt = 0;
#pragma unroll
      for (int f = 0; f < kInflight; ++f) {
        jv[f] = -1;
        if (okm) {
          const int src = __ffs(okm) - 1;
          okm &= okm - 1;
          jv[f] = __shfl_sync(gmask, (long long)jj, src, kLanes);
          ++cnt;
        }
      }
      KVRow rv[kInflight];
#pragma unroll
      for (int f = 0; f < kInflight; ++f)
        if (jv[f] >= 0) load_row(kf, vbase, jv[f], stride, rv[f]);
      float sv[kInflight];
      float smax = -INFINITY;
#pragma unroll
      for (int f = 0; f < kInflight; ++f) {
        sv[f] = -INFINITY;
        if (jv[f] >= 0) {
          ensure_pattern(jv[f]);
          sv[f] = dot_of(rv[f]);
        }
        smax = fmaxf(smax, sv[f]);
      }
      raise_max(smax, -INFINITY);
#pragma unroll
      for (int f = 0; f < kInflight; ++f) {
        if (jv[f] >= 0) {
          const float pf = exp2f(sv[f] - m);
          l += pf;
          accumulate(pf, rv[f]);
        }
      }
      entries += cnt;
    }
    if (stopm) break;
  }

  if (fallback) {  // self entry (sparse.cpp:111): the row admits nothing else
    KVRow kv;
    load_row(kf, vbase, i, stride, kv);
    ensure_pattern(i);
    const float s0 = dot_of(kv);
    raise_max(s0, -INFINITY);
    const float p0 = exp2f(s0 - m);
    l += p0;
    accumulate(p0, kv);
    entries += 1;
  }
  if (entries == 0) return;  // the running state stands

  const float inv_l = 1.f / l;
#pragma unroll
  for (int t = 0; t < kDims; t += 4)
    reinterpret_cast<float4*>(orow)[t / 4] =
        make_float4(o[t] * inv_l, o[t + 1] * inv_l, o[t + 2] * inv_l, o[t + 3] * inv_l);
  if (lane == 0) {
    a.lse[int64_t(h) * a.lse_stride + i] = (m + log2f(l)) * 0.6931471805599453f;
    if (a.simt_count)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.simt_count), (unsigned long long)entries);
  }
}


// ---------------------------------------------------------------------------------------
// Diagonal-major variant (default): the rows of a warp walk the half-block's segment list
// together, one diagonal d per step, so a step is the entries (i, i - d) of eight
// consecutive rows -- eight consecutive keys -- with no per-entry list scan, ballot or
// index shuffle.  Four lanes per row: lane ls holds the k-dims {16 t + 4 ls + c} (eight
// float4 loads of the fp32 rotated key, 64 contiguous bytes per row per load, partial dot
// reduced by two shuffles) and the v-dims {32 t + 8 ls + c} (four 16-byte bf16 loads, its
// own 32 output accumulators).  Online softmax per row in fp32 with a lazy max (rescale
// only when a logit passes the running max by 8 in log2 units).  Same entries, state and
// fallback semantics as attn_gather_kernel above.
namespace diag {
constexpr int kLanes = 4;                  // lanes per row
constexpr int kRowsW = 32 / kLanes;        // rows per warp
constexpr int kWarps = 4;                  // warps per CTA
constexpr int kRowsC = kRowsW * kWarps;    // rows per CTA (within one 64-row half)
#ifndef LCX_GATHER_DIAG_MINB
#define LCX_GATHER_DIAG_MINB 3  // resident CTAs per SM (register budget)
#endif
static_assert(64 % kRowsC == 0, "a CTA's rows lie in one half-block");
// LCX_GATHER_BATCH (default 1): batched per-warp segment control (see the kernel); 0: the
// per-diagonal dependent-load loop.  Measured at 1M (per layer): planted gather 81.8 ->
// 67.7 ms, iid 5.39 -> 4.52 s.  Staging the K / V rows of the next 1-3 live diagonals with
// cp.async on top of it measured 65.9-66.6 ms planted but 4.99-5.17 s iid, and a second
// entry per row in registers (255 registers, 2 CTAs per SM) 91 ms planted, 5.92 s iid:
// neither kept.
#ifndef LCX_GATHER_BATCH
#define LCX_GATHER_BATCH 1
#endif

__device__ __forceinline__ int64_t qpos(const GatherArgs& a, int pattern, int64_t i, int64_t imod) {
  if (a.rel_mode == 0) return a.pos_q ? a.pos_q[i] : i;
  if (pattern == 0) return imod;
  if (pattern == 1) return lcx_min64(imod + a.s, a.c - 1);
  return a.c - 1;
}

__global__ void __launch_bounds__(kWarps * 32, LCX_GATHER_DIAG_MINB) attn_gather_diag_kernel(const GatherArgs a) {
  if (a.win_flags && !a.win_flags[a.win] && a.key_hi <= a.row_begin) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ls = lane & (kLanes - 1);
  // heads fastest (a.head_fast, one pass over all keys): the query heads of a KV head work
  // on the same rows together, so a line several of them selected is read from DRAM once;
  // rows fastest for key-window passes (the window's K / V stay in L2 across the rows)
  const int h = a.head_fast ? blockIdx.x : blockIdx.y, g = h / a.group;
  const int64_t cta_row0 =
      a.row_begin + int64_t(a.head_fast ? blockIdx.y : blockIdx.x) * kRowsC;
  const int64_t w_row0 = cta_row0 + warp * kRowsW;
  const int64_t i = w_row0 + (lane / kLanes);
  const bool row_ok = i < a.row_end;
  const int r = int((i - a.row_begin) & 127);  // row within its 128-row block
  const int half = int(((cta_row0 - a.row_begin) & 127) >> 6);
  const int4* sg = a.segs + (int64_t(h) * 2 + half) * a.cap_seg;
  const int nseg = a.nseg[h * 2 + half];
  const int nvh = a.nv[h], nsh = a.ns[h];
  const bool any = (nvh > 0 && int64_t(a.verts[int64_t(h) * a.cap_v]) <= i) ||
                   (nsh > 0 && int64_t(a.slashes[int64_t(h) * a.cap_s]) <= i);
  const bool fallback = row_ok && !any && a.do_fallback && i >= a.key_lo && i < a.key_hi;
  // the warp's diagonals: d in [w_row0 - key_hi + 1, last row - key_lo], d <= last row
  const int64_t w_last = lcx_min64(w_row0 + kRowsW, a.row_end) - 1;
  const int64_t dmin = w_row0 - a.key_hi + 1;
  const int64_t dmax = lcx_min64(w_last, w_last - a.key_lo);
  // first segment index in [lo, hi) whose diagonal is >= key (past = false) or > key
  // (past = true), hi if none: a 32-ary search, one probe per lane per round (3 rounds of
  // independent loads for ~6000 segments instead of 13 dependent ones)
  auto wsearch = [&](int lo, int hi, int64_t key, bool past) -> int {
    while (lo < hi) {
      const int step = (hi - lo + 31) >> 5;
      const int idx = lo + lane * step;
      bool pred = false;
      if (idx < hi) {
        const int64_t v = int64_t(__ldg(&sg[idx].x));
        pred = past ? v > key : v >= key;
      }
      const uint32_t b = __ballot_sync(0xffffffffu, pred);
      if (b == 0) {  // beyond the last probe
        lo = lo + ((hi - lo - 1) / step) * step + 1;
        continue;
      }
      const int f = __ffs(b) - 1;
      if (f == 0) return lo;
      hi = lo + f * step;
      lo = lo + (f - 1) * step + 1;
    }
    return hi;
  };
  const int xs = wsearch(0, nseg, dmin, false);
  const bool have = xs < nseg && int64_t(__ldg(&sg[xs].x)) <= dmax;
  if (!have && !__any_sync(0xffffffffu, fallback)) return;

  // this lane's query dims {16 t + 4 ls + c}: raw bf16 kept packed, rotated per DCA pattern
  uint2 qraw[8];
  {
    const uint2* qp = reinterpret_cast<const uint2*>(a.q + ((row_ok ? i : 0) * a.hq + h) * 128);
#pragma unroll
    for (int t = 0; t < 8; ++t) qraw[t] = row_ok ? __ldg(qp + 4 * t + ls) : make_uint2(0u, 0u);
  }
  const int64_t qc = a.rel_mode == 1 ? i / a.s : 0;
  const int64_t imod = i - qc * a.s;
  const int64_t c_intra = qc * a.s, c_succ = c_intra - a.s;
  float qr[32];
  int cur_pat = -1;
  auto rotate = [&](int pat) {
    cur_pat = pat;
    const float4* cs = reinterpret_cast<const float4*>(a.rope + qpos(a, pat, i, imod) * 64);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float4 c = __ldg(cs + 4 * t + ls);  // pairs 8 t + 2 ls, + 1
      const float x0 = __uint_as_float(qraw[t].x << 16), y0 = __uint_as_float(qraw[t].x & 0xffff0000u);
      const float x1 = __uint_as_float(qraw[t].y << 16), y1 = __uint_as_float(qraw[t].y & 0xffff0000u);
      qr[4 * t] = (x0 * c.x - y0 * c.y) * a.scale_log2;
      qr[4 * t + 1] = (x0 * c.y + y0 * c.x) * a.scale_log2;
      qr[4 * t + 2] = (x1 * c.z - y1 * c.w) * a.scale_log2;
      qr[4 * t + 3] = (x1 * c.w + y1 * c.z) * a.scale_log2;
    }
  };
  auto pattern_of = [&](int64_t j) -> int {
    return a.rel_mode != 1 ? 0 : (j >= c_intra ? 0 : (j >= c_succ ? 1 : 2));
  };

  // running state: the partial so far (tensor-core tiles, earlier passes), log2 domain
  float o[32], m = -INFINITY, l = 0.f;
  float* orow = a.out + ((row_ok ? i : 0) * a.hq + h) * 128;
  const float lp = row_ok ? a.lse[int64_t(h) * a.lse_stride + i] : -INFINITY;
  const bool from_partial = lp != -INFINITY && !fallback;
#pragma unroll
  for (int x = 0; x < 32; ++x) o[x] = 0.f;
  if (from_partial) {
    m = lp * 1.4426950408889634f;
    l = 1.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float4 u0 = reinterpret_cast<const float4*>(orow)[8 * t + 2 * ls];
      const float4 u1 = reinterpret_cast<const float4*>(orow)[8 * t + 2 * ls + 1];
      o[8 * t] = u0.x; o[8 * t + 1] = u0.y; o[8 * t + 2] = u0.z; o[8 * t + 3] = u0.w;
      o[8 * t + 4] = u1.x; o[8 * t + 5] = u1.y; o[8 * t + 6] = u1.z; o[8 * t + 7] = u1.w;
    }
  }
  const float* kbase = a.kf + int64_t(g) * 128;
  const __nv_bfloat16* vbase = a.v + int64_t(g) * 128;
  const int64_t stride = int64_t(a.hkv) * 128;
  const uint32_t* vb = a.vbits + int64_t(h) * a.words;
  int entries = 0;


  // entries of diagonal x for this lane's row: key j = i - d, admitted iff the row is in
  // the segment's row range, j in the pass window (j >= 0) and j not a vertical column
  auto valid_key = [&](const int4 e, int64_t& j) -> bool {
    j = i - e.x;
    return row_ok && r >= e.y && r < e.z && j >= a.key_lo && j < a.key_hi && j >= 0 &&
           !((__ldg(vb + (j >> 5)) >> (j & 31)) & 1u);
  };
  auto process = [&](int64_t j) {  // one admitted entry of this lane's row
    const int pat = pattern_of(j);
    if (pat != cur_pat) rotate(pat);
    const float4* kp = reinterpret_cast<const float4*>(kbase + j * stride);
    const uint4* vp = reinterpret_cast<const uint4*>(vbase + j * stride);
    float4 kk[8];
    uint4 vv[4];
#pragma unroll
    for (int t = 0; t < 8; ++t) kk[t] = __ldg(kp + 4 * t + ls);
#pragma unroll
    for (int t = 0; t < 4; ++t) vv[t] = __ldg(vp + 4 * t + ls);
    float d0 = 0.f, d1 = 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      d0 = fmaf(qr[4 * t], kk[t].x, d0);
      d1 = fmaf(qr[4 * t + 1], kk[t].y, d1);
      d0 = fmaf(qr[4 * t + 2], kk[t].z, d0);
      d1 = fmaf(qr[4 * t + 3], kk[t].w, d1);
    }
    float sc = d0 + d1;
    // the four lanes of a row agree on every branch that leads here (same i): reduce
    // among the lanes present
    const unsigned am = __activemask();
    sc += __shfl_xor_sync(am, sc, 1);
    sc += __shfl_xor_sync(am, sc, 2);
    if (sc > m + 8.f) {  // lazy max: p stays <= 2^8 (fp32 accumulators)
      const float corr = ex2(m - sc);  // 0 on the first entry (m = -inf)
      l *= corr;
#pragma unroll
      for (int x = 0; x < 32; ++x) o[x] *= corr;
      m = sc;
    }
    const float pf = ex2(sc - m);
    l += pf;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t w4[4] = {vv[t].x, vv[t].y, vv[t].z, vv[t].w};
#pragma unroll
      for (int c2 = 0; c2 < 4; ++c2) {
        o[8 * t + 2 * c2] = fmaf(pf, __uint_as_float(w4[c2] << 16), o[8 * t + 2 * c2]);
        o[8 * t + 2 * c2 + 1] = fmaf(pf, __uint_as_float(w4[c2] & 0xffff0000u), o[8 * t + 2 * c2 + 1]);
      }
    }
    ++entries;
  };
#if LCX_GATHER_BATCH
  // batched control: lane k of the warp loads segment x0 + k and works out, for the warp's 8
  // rows, which of them admit its entry (row range, key window, not a vertical column) --
  // one coalesced segment load and two bitmap words per lane per 32 diagonals, instead of
  // a dependent segment -> bitmap load chain per diagonal; the warp then walks the
  // diagonals some row admits
  if (have) {
    const int xe = wsearch(xs, nseg, dmax, true);  // first diagonal > dmax
    const int rr = lane / kLanes;
    const int rb = int((w_row0 - a.row_begin) & 127);
    for (int x0 = xs; x0 < xe; x0 += 32) {
      const int cnt = min(32, xe - x0);
      int dk = 0;
      uint32_t rm = 0;
      if (lane < cnt) {
        const int4 e = __ldg(&sg[x0 + lane]);
        dk = e.x;
        const int64_t jb = w_row0 - e.x;  // key of the warp's first row on this diagonal
        const int64_t w0 = jb >= 0 ? (jb >> 5) : 0;
        const uint64_t bits = uint64_t(__ldg(vb + w0)) | (uint64_t(__ldg(vb + w0 + 1)) << 32);
#pragma unroll
        for (int q = 0; q < kRowsW; ++q) {
          const int64_t j = jb + q;
          const int rq = rb + q;
          const bool ok = w_row0 + q < a.row_end && rq >= e.y && rq < e.z && j >= a.key_lo &&
                          j < a.key_hi && j >= 0 && !((bits >> ((j - (w0 << 5)) & 63)) & 1u);
          rm |= uint32_t(ok) << q;
        }
      }
      uint32_t live = __ballot_sync(0xffffffffu, rm != 0);
      while (live) {
        const int k = __ffs(live) - 1;
        live &= live - 1;
        const uint32_t mk = __shfl_sync(0xffffffffu, rm, k);
        const int d = __shfl_sync(0xffffffffu, dk, k);
        if ((mk >> rr) & 1u) process(i - d);
      }
    }
  }
#else
  if (have) {
    for (int x = xs; x < nseg; ++x) {
      const int4 e = __ldg(&sg[x]);
      if (int64_t(e.x) > dmax) break;
      int64_t j;
      const bool ok = valid_key(e, j);
      // the lanes of a row agree on ok (same i); whole rows skip together
      if (ok) process(j);
    }
  }
#endif
  if (fallback) {  // self entry (sparse.cpp:111): the row admits nothing else
    process(i);
  }
  if (!row_ok || entries == 0) return;  // no entry: the running state stands
  const float inv_l = 1.f / l;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    reinterpret_cast<float4*>(orow)[8 * t + 2 * ls] =
        make_float4(o[8 * t] * inv_l, o[8 * t + 1] * inv_l, o[8 * t + 2] * inv_l, o[8 * t + 3] * inv_l);
    reinterpret_cast<float4*>(orow)[8 * t + 2 * ls + 1] =
        make_float4(o[8 * t + 4] * inv_l, o[8 * t + 5] * inv_l, o[8 * t + 6] * inv_l,
                    o[8 * t + 7] * inv_l);
  }
  if (ls == 0) {
    a.lse[int64_t(h) * a.lse_stride + i] = (m + log2f(l)) * 0.6931471805599453f;
    if (a.simt_count)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.simt_count), (unsigned long long)entries);
  }
}
}  // namespace diag

}  // namespace

int attention_gather(const GatherArgs& a, cudaStream_t st) {
  const int64_t rows = a.row_end - a.row_begin;
  if (rows <= 0) return LCX_OK;
  if (a.row_begin % 128 != 0) return fail(LCX_ERR_INTERNAL, "gather rows must start a block");
#if LCX_GATHER_DIAG
  const unsigned nrb = unsigned((rows + diag::kRowsC - 1) / diag::kRowsC);
  dim3 grid = a.head_fast ? dim3(unsigned(a.hq), nrb) : dim3(nrb, unsigned(a.hq));
  diag::attn_gather_diag_kernel<<<grid, diag::kWarps * 32, 0, st>>>(a);
#else
  dim3 grid(unsigned((rows + kRows - 1) / kRows), unsigned(a.hq));
  attn_gather_kernel<<<grid, kThreads, 0, st>>>(a);
#endif
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

}  // namespace lcx
