// K3 + K4 (tensor-core path) -- index build and block-sparse flash prefill on
// tcgen05 / TMEM / TMA for bf16 inputs with head dim 128.
//
// Semantics (reference core/src/sparse.cpp:85-113, 368-396; attention.cpp:35-51):
// row i of the chunk attends exactly to {verticals v <= i} U {i - d : d in slashes,
// d <= i} (deduplicated), logits scaled by 1/(temperature sqrt(D)); with DCA the
// logit is rope(q_i, dca_relative(i, j)) . k_j, computed here as
// rope(q_i, qpos_pattern(i)) . rope(k_j, j mod s) (identical in exact arithmetic):
// every 128-row query block lies inside one DCA chunk (s % 128 == 0) and every
// 64-key tile inside one key chunk, so a tile has one pattern (intra /
// successive / inter) and the query tile is re-rotated when the pattern changes.
// The standard path rotates q by positions_q and k by positions_k.
//
// Work item = (query head, 128-row block).  Its key tiles (64 keys each):
//   VERT   64 gathered verticals (compacted per (chunk, head) by the index build),
//          mask j <= i;
//   SLASH  a 64-aligned key range holding enough selected diagonals to be worth
//          a tensor-core tile ("relative tile" u = key tile - block/64 is
//          classified once per (chunk, head)); mask (i - j) in slashes and j not a
//          vertical (the vertical path owns entries on both);
//   DENSE  full causal attention (PrefillMode::Full / full_attention).
// Slash entries in the remaining relative tiles go to the CUDA-core gather path
// (attn_simt.cu) as (d, first row, last row) segments and are merged in place.
//
// Precision (bf16 storage, 2e-3 contract): q and k are rotated in fp32 and split
// into bf16 hi + lo; S = q_hi k_hi + q_hi k_lo + q_lo k_hi (3 MMAs, fp32 TMEM
// accumulate); P is fp16 (<= 2^8 under a lazy-rescale threshold of 8 in log2
// units); V is fp16.  Executed MMA work per tile = 4 units vs 2 algorithmic.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (one lane), w2 TMEM
// allocator, w4..w7 softmax / correction / epilogue (thread = query row, TMEM
// lane quadrant = warp % 4).  Pipelines: K (hi+lo) and V^T double-buffered,
// S double-buffered in TMEM (2 x 64 columns), O in TMEM (128 columns), P
// double-buffered in smem.
#include <cuda.h>

#include "lcx_internal.cuh"
#include "tc_ptx.cuh"
#include "attn_tc.cuh"

namespace lcx {



namespace {

constexpr int BM = 128, BN = 64, HD = 128;
constexpr int kThreads = 256;
constexpr uint32_t kQHalf = BM * 64 * 2;             // 16 KB
constexpr uint32_t kKHalf = BN * 64 * 2;             // 8 KB
constexpr uint32_t kKStage = 4 * kKHalf;             // hi0 hi1 lo0 lo1 = 32 KB
constexpr uint32_t kVStage = HD * BN * 2;            // 16 KB
constexpr uint32_t kPBuf = BM * BN * 2;              // 16 KB
constexpr uint32_t OFF_QHI = 0;
constexpr uint32_t OFF_QLO = 2 * kQHalf;
constexpr uint32_t OFF_K = 4 * kQHalf;               // 64 KB
constexpr uint32_t OFF_V = OFF_K + 2 * kKStage;      // 128 KB
constexpr uint32_t OFF_P = OFF_V + 2 * kVStage;      // 160 KB
constexpr uint32_t OFF_BAR = OFF_P + 2 * kPBuf;      // 192 KB
constexpr uint32_t kSmemBytes = OFF_BAR + 256 + 1024;  // + alignment slack
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t COL_O = 128;
constexpr float kRescaleThresh = 8.f;

constexpr uint32_t IDESC_QK = tc::idesc_f16(BM, BN, 1, 1);   // bf16 x bf16
constexpr uint32_t IDESC_PV = tc::idesc_f16(BM, HD, 0, 0);   // f16 x f16

enum { T_VERT = 0, T_SLASH = 1, T_DENSE = 2 };

struct Group {
  int64_t klo, khi;
  int pattern;  // 0 standard / intra, 1 successive, 2 inter
  int vlo, vhi;  // compact positions [vlo, vhi) (64-aligned start)
  int ulo, uhi;
  int nvt, nst;
  int64_t kt0;  // dense: first key tile
};

struct Item {
  int h, g;
  int64_t i0, rend;
  int ng;
  Group grp[3];
  int ntiles;
};

struct Tile {
  int kind, grp, count;
  int64_t key0;  // VERT: compact index; SLASH / DENSE: first key
};

__device__ __forceinline__ int lower_bound32(const int32_t* a, int n, int64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (int64_t(a[mid]) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t ceil_div64(int64_t a) { return (a + 63) >> 6; }

__device__ void setup_item(const TcParams& p, int item, Item& it) {
  it.h = item / p.nblocks;
  const int b = item - it.h * p.nblocks;
  it.g = it.h / p.group;
  it.i0 = (p.block0 + b) * BM;
  it.rend = lcx_min64(it.i0 + BM, p.t1);
  const int64_t kend = it.rend;
  int64_t lo[3], hi[3];
  int pat[3];
  int ng = 0;
  if (p.rel_mode == 0) {
    lo[0] = 0; hi[0] = kend; pat[0] = 0; ng = 1;
  } else {
    const int64_t qc = it.i0 / p.s;
    if (qc >= 2) { lo[ng] = 0; hi[ng] = (qc - 1) * p.s; pat[ng] = 2; ++ng; }
    if (qc >= 1) { lo[ng] = (qc - 1) * p.s; hi[ng] = qc * p.s; pat[ng] = 1; ++ng; }
    lo[ng] = qc * p.s; hi[ng] = kend; pat[ng] = 0; ++ng;
  }
  const int32_t* vh = p.verts ? p.verts + int64_t(it.h) * p.cap_v : nullptr;
  const int nvh = p.verts ? p.nv[it.h] : 0;
  const int32_t* uh = p.tc_u ? p.tc_u + int64_t(it.h) * p.cap_u : nullptr;
  const int nuh = p.tc_u ? p.n_tc_u[it.h] : 0;
  const int64_t ib = it.i0 >> 6;
  it.ng = 0;
  it.ntiles = 0;
  for (int x = 0; x < ng; ++x) {
    Group G{};
    G.klo = lo[x];
    G.khi = hi[x];
    G.pattern = pat[x];
    if (G.khi <= G.klo) continue;
    if (p.dense) {
      G.kt0 = G.klo >> 6;
      G.nvt = 0;
      G.nst = int(ceil_div64(G.khi) - G.kt0);
    } else {
      // compact segment of key chunks [klo / L, ...): 64-aligned start
      const int m_lo = int(G.klo / p.seg_len);
      const int32_t* vb = p.vbase + int64_t(it.h) * (p.nseg_k + 1);
      const int32_t* vf = p.vfirst + int64_t(it.h) * (p.nseg_k + 1);
      G.vlo = vb[m_lo];
      if (G.khi % p.seg_len == 0 && G.khi / p.seg_len <= p.nseg_k) {
        G.vhi = vb[G.khi / p.seg_len];
      } else {
        const int m_hi = int(G.khi / p.seg_len);  // intra group ends inside chunk m_hi
        G.vhi = vb[m_hi] + (lower_bound32(vh, nvh, G.khi) - vf[m_hi]);
      }
      G.nvt = (G.vhi - G.vlo + 63) >> 6;
      G.ulo = lower_bound32(uh, nuh, (G.klo >> 6) - ib);
      G.uhi = lower_bound32(uh, nuh, ceil_div64(G.khi) - ib);
      G.nst = G.uhi - G.ulo;
    }
    if (G.nvt + G.nst == 0) continue;
    it.grp[it.ng++] = G;
    it.ntiles += G.nvt + G.nst;
  }
}

__device__ Tile get_tile(const TcParams& p, const Item& it, int t) {
  Tile T{};
  for (int x = 0; x < it.ng; ++x) {
    const Group& G = it.grp[x];
    if (t < G.nvt) {
      T.kind = T_VERT;
      T.grp = x;
      T.key0 = G.vlo + int64_t(t) * 64;
      T.count = int(lcx_min64(64, G.vhi - T.key0));
      return T;
    }
    t -= G.nvt;
    if (t < G.nst) {
      T.grp = x;
      T.count = 64;
      if (p.dense) {
        T.kind = T_DENSE;
        T.key0 = (G.kt0 + t) * 64;
      } else {
        T.kind = T_SLASH;
        T.key0 = it.i0 + int64_t(p.tc_u[int64_t(it.h) * p.cap_u + G.ulo + t]) * 64;
      }
      return T;
    }
    t -= G.nst;
  }
  return T;
}

// bits [lo, lo + 64) of a bitmap (zeros outside [0, 32 * words))
__device__ __forceinline__ uint64_t bits64(const uint32_t* bits, int64_t words, int64_t lo) {
  if (lo <= -64) return 0;
  const int64_t base = lo < 0 ? 0 : lo;
  const int64_t w = base >> 5;
  const int sh = int(base & 31);
  auto word = [&](int64_t k) -> uint64_t { return k < words ? bits[k] : 0u; };
  const uint64_t a = word(w) | (word(w + 1) << 32);
  const uint64_t b = word(w + 2);
  uint64_t r = sh ? ((a >> sh) | (b << (64 - sh))) : a;
  if (lo < 0) r <<= (-lo);
  return r;
}

__device__ __forceinline__ int64_t qpos_of(const TcParams& p, int pattern, int64_t i) {
  if (p.rel_mode == 0) return p.pos_q ? p.pos_q[i] : i;
  const int64_t im = i % p.s;
  if (pattern == 0) return im;
  if (pattern == 1) return lcx_min64(im + p.s, p.c - 1);
  return p.c - 1;
}

// Rotate this thread's query row by its pattern position and write the bf16
// hi / lo split into the SW128 K-major Q tiles.
__device__ __forceinline__ void rotate_q(const TcParams& p, const Item& it, int pattern, int r,
                                         uint8_t* smem) {
  const int64_t i = it.i0 + r;
  const bool ok = i < it.rend;
  const uint4* src = reinterpret_cast<const uint4*>(p.q + (i * p.hq + it.h) * int64_t(HD));
  const float2* cs = p.rope + (ok ? qpos_of(p, pattern, i) : 0) * (HD / 2);
#pragma unroll 4
  for (int ch = 0; ch < HD / 8; ++ch) {  // 16 chunks of 8 dims (4 pairs)
    uint4 raw = ok ? src[ch] : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 xy = __bfloat1622float2(x2[k]);
      const float2 c = cs[ch * 4 + k];
      const float rx = xy.x * c.x - xy.y * c.y;
      const float ry = xy.x * c.y + xy.y * c.x;
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(rx, ry);
      const float2 hf = __bfloat1622float2(h2);
      const __nv_bfloat162 l2 = __floats2bfloat162_rn(rx - hf.x, ry - hf.y);
      hi[k] = *reinterpret_cast<const uint32_t*>(&h2);
      lo[k] = *reinterpret_cast<const uint32_t*>(&l2);
    }
    const int half = ch >> 3, c16 = ch & 7;
    const uint32_t off = half * kQHalf + tc::sw128_off(r, c16);
    *reinterpret_cast<uint4*>(smem + OFF_QHI + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(smem + OFF_QLO + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
attn_tc_kernel(const TcParams p, const __grid_constant__ CUtensorMap map_k_hi,
               const __grid_constant__ CUtensorMap map_k_lo,
               const __grid_constant__ CUtensorMap map_vt,
               const __grid_constant__ CUtensorMap map_kc_hi,
               const __grid_constant__ CUtensorMap map_kc_lo,
               const __grid_constant__ CUtensorMap map_vct) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* k_full = bars + 0;
  uint64_t* k_empty = bars + 2;
  uint64_t* v_full = bars + 4;
  uint64_t* v_empty = bars + 6;
  uint64_t* s_full = bars + 8;
  uint64_t* s_free = bars + 10;
  uint64_t* p_full = bars + 12;
  uint64_t* p_free = bars + 14;
  uint64_t* q_ready = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(k_full + b, 1);
      tc::mbar_init(k_empty + b, 1);
      tc::mbar_init(v_full + b, 1);
      tc::mbar_init(v_empty + b, 1);
      tc::mbar_init(s_full + b, 1);
      tc::mbar_init(s_free + b, 4);
      tc::mbar_init(p_full + b, 4);
      tc::mbar_init(p_free + b, 1);
    }
    tc::mbar_init(q_ready, 4);
    tc::fence_barrier_init();
    tc::fence_proxy_async();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, kTmemCols);
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&map_k_hi);
    tc::tma_prefetch(&map_k_lo);
    tc::tma_prefetch(&map_vt);
    tc::tma_prefetch(&map_kc_hi);
    tc::tma_prefetch(&map_kc_lo);
    tc::tma_prefetch(&map_vct);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================================================= TMA producer ====
    if (lane == 0) {
      uint32_t T = 0;
      for (int item = blockIdx.x; item < p.nitems; item += gridDim.x) {
        Item it;
        setup_item(p, item, it);
        for (int t = 0; t < it.ntiles; ++t, ++T) {
          const Tile tl = get_tile(p, it, t);
          const int b = T & 1;
          const uint32_t ph = (T >> 1) & 1;
          tc::mbar_wait(k_empty + b, ph ^ 1);
          tc::mbar_expect_tx(k_full + b, kKStage);
          uint8_t* kdst = smem + OFF_K + b * kKStage;
          if (tl.kind == T_VERT) {
            const int r = int(tl.key0);
            tc::tma_load_3d(kdst + 0 * kKHalf, &map_kc_hi, k_full + b, 0, r, it.h);
            tc::tma_load_3d(kdst + 1 * kKHalf, &map_kc_hi, k_full + b, 64, r, it.h);
            tc::tma_load_3d(kdst + 2 * kKHalf, &map_kc_lo, k_full + b, 0, r, it.h);
            tc::tma_load_3d(kdst + 3 * kKHalf, &map_kc_lo, k_full + b, 64, r, it.h);
          } else {
            const int j = int(tl.key0);
            tc::tma_load_3d(kdst + 0 * kKHalf, &map_k_hi, k_full + b, 0, it.g, j);
            tc::tma_load_3d(kdst + 1 * kKHalf, &map_k_hi, k_full + b, 64, it.g, j);
            tc::tma_load_3d(kdst + 2 * kKHalf, &map_k_lo, k_full + b, 0, it.g, j);
            tc::tma_load_3d(kdst + 3 * kKHalf, &map_k_lo, k_full + b, 64, it.g, j);
          }
          tc::mbar_wait(v_empty + b, ph ^ 1);
          tc::mbar_expect_tx(v_full + b, kVStage);
          uint8_t* vdst = smem + OFF_V + b * kVStage;
          if (tl.kind == T_VERT)
            tc::tma_load_3d(vdst, &map_vct, v_full + b, int(tl.key0), 0, it.h);
          else
            tc::tma_load_3d(vdst, &map_vt, v_full + b, int(tl.key0), 0, it.g);
        }
      }
    }
  } else if (warp == 1) {
    // =================================================== MMA issuer ====
    if (lane == 0) {
      uint32_t T = 0, E = 0;
      auto issue_pv = [&](uint32_t Tp, bool first) {
        const int b = Tp & 1;
        const uint32_t ph = (Tp >> 1) & 1;
        tc::mbar_wait(p_full + b, ph);
        tc::mbar_wait(v_full + b, ph);
        tc::tc_fence_after();
        const uint32_t pa = tc::smem_u32(smem + OFF_P + b * kPBuf);
        const uint32_t va = tc::smem_u32(smem + OFF_V + b * kVStage);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          tc::mma_f16_ss(tmem + COL_O, tc::sdesc_sw128(pa + kk * 32), tc::sdesc_sw128(va + kk * 32),
                         IDESC_PV, (first && kk == 0) ? 0u : 1u);
        tc::mma_commit(v_empty + b);
        tc::mma_commit(p_free + b);
      };
      for (int item = blockIdx.x; item < p.nitems; item += gridDim.x) {
        Item it;
        setup_item(p, item, it);
        int prev_grp = -1;
        for (int t = 0; t < it.ntiles; ++t, ++T) {
          const Tile tl = get_tile(p, it, t);
          if (tl.grp != prev_grp) {
            tc::mbar_wait(q_ready, E & 1);
            ++E;
            prev_grp = tl.grp;
          }
          const int b = T & 1;
          const uint32_t ph = (T >> 1) & 1;
          tc::mbar_wait(k_full + b, ph);
          tc::mbar_wait(s_free + b, ph ^ 1);
          tc::tc_fence_after();
          const uint32_t qh = tc::smem_u32(smem + OFF_QHI), ql = tc::smem_u32(smem + OFF_QLO);
          const uint32_t kb = tc::smem_u32(smem + OFF_K + b * kKStage);
          const uint32_t dS = tmem + b * BN;
          uint32_t acc = 0;
#pragma unroll
          for (int combo = 0; combo < 3; ++combo) {
            const uint32_t qa = combo == 2 ? ql : qh;            // hi.hi, hi.lo, lo.hi
            const uint32_t ka = kb + (combo == 1 ? 2 * kKHalf : 0);
#pragma unroll
            for (int half = 0; half < 2; ++half)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                tc::mma_f16_ss(dS, tc::sdesc_sw128(qa + half * kQHalf + kk * 32),
                               tc::sdesc_sw128(ka + half * kKHalf + kk * 32), IDESC_QK, acc);
                acc = 1;
              }
          }
          tc::mma_commit(k_empty + b);
          tc::mma_commit(s_full + b);
          if (t > 0) issue_pv(T - 1, t - 1 == 0);
        }
        if (it.ntiles > 0) issue_pv(T - 1, it.ntiles == 1);
      }
    }
  } else if (warp >= 4) {
    // ============================= softmax / correction / epilogue ====
    const int wq = warp & 3;  // TMEM lane quadrant
    const int r = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    uint32_t T = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x) {
      Item it;
      setup_item(p, item, it);
      const int64_t i = it.i0 + r;
      const bool row_ok = i < it.rend;
      if (it.ntiles == 0) {
        if (row_ok) {
          float4* o = reinterpret_cast<float4*>(p.out + (i * p.hq + it.h) * int64_t(HD));
          for (int x = 0; x < HD / 4; ++x) o[x] = make_float4(0.f, 0.f, 0.f, 0.f);
          p.lse[int64_t(it.h) * p.lse_stride + i] = -INFINITY;
        }
        continue;
      }
      Tile tl = get_tile(p, it, 0);
      rotate_q(p, it, it.grp[tl.grp].pattern, r, smem);
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(q_ready);

      float m = -INFINITY, l = 0.f;
      const int32_t* vh = p.verts ? p.verts + int64_t(it.h) * p.cap_v : nullptr;
      const uint32_t* sb = p.sbits ? p.sbits + int64_t(it.h) * p.words : nullptr;
      const uint32_t* vb = p.vbits ? p.vbits + int64_t(it.h) * p.words : nullptr;
      for (int t = 0; t < it.ntiles; ++t, ++T) {
        const int b = T & 1;
        const uint32_t ph = (T >> 1) & 1;
        float sv[64];
        tc::mbar_wait(s_full + b, ph);
        tc::tc_fence_after();
        tc::tmem_ld32(tmem + lane_base + b * BN, sv);
        tc::tmem_ld32(tmem + lane_base + b * BN + 32, sv + 32);
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(s_free + b);
        Tile nxt{};
        if (t + 1 < it.ntiles) {
          nxt = get_tile(p, it, t + 1);
          if (nxt.grp != tl.grp) {  // all QK of the old pattern are complete
            rotate_q(p, it, it.grp[nxt.grp].pattern, r, smem);
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(q_ready);
          }
        }
        // ---- admission mask (bit c = key c of the tile) ----
        uint64_t mask = 0;
        if (row_ok) {
          if (tl.kind == T_VERT) {
            mask = tl.count >= 64 ? ~0ull : ((1ull << tl.count) - 1);
            // real keys form an ascending prefix of the tile (pads = -1 at the tail)
            const int32_t* ck = p.ckeys + int64_t(it.h) * p.capp + tl.key0;
            int lo = 0, hi = tl.count;  // count of c with 0 <= ck[c] <= i
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              const int32_t kk = ck[mid];
              if (kk >= 0 && int64_t(kk) <= i) lo = mid + 1;
              else hi = mid;
            }
            mask = lo >= 64 ? ~0ull : ((1ull << lo) - 1);
          } else if (tl.kind == T_SLASH) {
            const uint64_t win = bits64(sb, p.words, i - tl.key0 - 63);  // bit k <-> d = lo + k
            const uint64_t vm = bits64(vb, p.words, tl.key0);
            mask = __brevll(win) & ~vm;
          } else {
            const int64_t lim = i - tl.key0;  // keys key0 + c <= i
            mask = lim >= 63 ? ~0ull : (lim < 0 ? 0ull : ((2ull << lim) - 1));
          }
        }
        float tmax = -INFINITY;
#pragma unroll
        for (int cc = 0; cc < 64; ++cc) {
          sv[cc] *= p.scale_log2;
          if ((mask >> cc) & 1ull) tmax = fmaxf(tmax, sv[cc]);
        }
        // lazy rescale (warp-uniform TMEM access)
        const bool need = tmax > m + kRescaleThresh;
        const bool warp_need = __any_sync(0xffffffffu, need && t > 0 && m != -INFINITY);
        float m_new = need ? tmax : m;
        if (warp_need) {
          const uint32_t Tp = T - 1;
          tc::mbar_wait(p_free + (Tp & 1), (Tp >> 1) & 1);
          tc::tc_fence_after();
          const float f = (need && m != -INFINITY) ? exp2f(m - m_new) : 1.f;
          float ov[32];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            tc::tmem_ld32(tmem + lane_base + COL_O + q4 * 32, ov);
            tc::tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 32; ++x) ov[x] *= f;
            tc::tmem_st32(tmem + lane_base + COL_O + q4 * 32, ov);
          }
          tc::tmem_wait_st();
          l *= f;
        } else if (need && m != -INFINITY) {
          // first tile of the item: O is overwritten by this tile's PV
          l *= exp2f(m - m_new);
        }
        m = m_new;
        // ---- P = exp2(x - m) in fp16, row sum from the rounded values ----
        tc::mbar_wait(p_free + b, ph ^ 1);  // PV(T-2) has consumed this P buffer
        uint8_t* pb = smem + OFF_P + b * kPBuf;
        float rs = 0.f;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int c0 = ch * 8 + 2 * k;
            const float p0 = ((mask >> c0) & 1ull) ? exp2f(sv[c0] - m) : 0.f;
            const float p1 = ((mask >> (c0 + 1)) & 1ull) ? exp2f(sv[c0 + 1] - m) : 0.f;
            const __half2 h2 = __floats2half2_rn(p0, p1);
            const float2 hf = __half22float2(h2);
            rs += hf.x + hf.y;
            w[k] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          *reinterpret_cast<uint4*>(pb + tc::sw128_off(r, ch)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        l += rs;
        tc::fence_proxy_async();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full + b);
        tl = nxt;
      }
      // ---- epilogue: wait for the last PV, normalize, store ----
      {
        const uint32_t Tp = T - 1;
        tc::mbar_wait(p_free + (Tp & 1), (Tp >> 1) & 1);
        tc::tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        float4* o = reinterpret_cast<float4*>(p.out + (i * p.hq + it.h) * int64_t(HD));
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float ov[32];
          tc::tmem_ld32(tmem + lane_base + COL_O + q4 * 32, ov);
          tc::tmem_wait_ld();
          if (row_ok) {
#pragma unroll
            for (int x = 0; x < 8; ++x)
              o[q4 * 8 + x] = make_float4(ov[4 * x] * inv, ov[4 * x + 1] * inv,
                                          ov[4 * x + 2] * inv, ov[4 * x + 3] * inv);
          }
        }
        if (row_ok)
          p.lse[int64_t(it.h) * p.lse_stride + i] =
              l > 0.f ? (m + log2f(l)) * 0.69314718055994530942f : -INFINITY;
        tc::tc_fence_before();
      }
      if (p.tile_count && threadIdx.x == 128)
        atomicAdd(reinterpret_cast<unsigned long long*>(p.tile_count),
                  (unsigned long long)it.ntiles);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------- prep --
// K_hi / K_lo [n][hkv][128] bf16 = split(rope(k_j, kpos(j))), kpos = pos_k[j]
// (standard) or j mod s (DCA).
__global__ void k_prep_kernel(const __nv_bfloat16* __restrict__ k, int64_t n, int hkv,
                              const int64_t* __restrict__ pos_k, int rel_mode, int64_t s,
                              const float2* __restrict__ rope, __nv_bfloat16* __restrict__ khi,
                              __nv_bfloat16* __restrict__ klo) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // pair index
  const int64_t total = n * hkv * (HD / 2);
  if (idx >= total) return;
  const int pr = int(idx % (HD / 2));
  const int64_t rowhead = idx / (HD / 2);
  const int64_t j = rowhead / hkv;
  const int64_t kp = rel_mode ? (j % s) : (pos_k ? pos_k[j] : j);
  const float2 xy = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(k)[idx]);
  const float2 c = rope[kp * (HD / 2) + pr];
  const float rx = xy.x * c.x - xy.y * c.y, ry = xy.x * c.y + xy.y * c.x;
  const __nv_bfloat162 h2 = __floats2bfloat162_rn(rx, ry);
  const float2 hf = __bfloat1622float2(h2);
  reinterpret_cast<__nv_bfloat162*>(khi)[idx] = h2;
  reinterpret_cast<__nv_bfloat162*>(klo)[idx] = __floats2bfloat162_rn(rx - hf.x, ry - hf.y);
}

// V^T [hkv][128][npad] fp16 from V [n][hkv][128] bf16 (smem-tiled transpose)
__global__ void vt_prep_kernel(const __nv_bfloat16* __restrict__ v, int64_t n, int hkv,
                               int64_t npad, __half* __restrict__ vt) {
  __shared__ __half tile[64][HD + 8];
  const int g = blockIdx.y;
  const int64_t j0 = int64_t(blockIdx.x) * 64;
  for (int x = threadIdx.x; x < 64 * HD; x += blockDim.x) {
    const int jj = x / HD, d = x % HD;
    const int64_t j = j0 + jj;
    tile[jj][d] = j < n ? __float2half(__bfloat162float(v[(j * hkv + g) * HD + d])) : __half(0.f);
  }
  __syncthreads();
  for (int x = threadIdx.x; x < 64 * HD; x += blockDim.x) {
    const int d = x / 64, jj = x % 64;
    const int64_t j = j0 + jj;
    if (j < npad) vt[(int64_t(g) * HD + d) * npad + j] = tile[jj][d];
  }
}

// Per head: vfirst[m] = first list index of key chunk m (keys [m L, (m+1) L)),
// vbase[m] = 64-aligned compact start of chunk m's segment.
__global__ void vseg_kernel(const int32_t* __restrict__ verts, const int32_t* __restrict__ nv,
                            int64_t cap_v, int64_t seg_len, int nseg_k,
                            int32_t* __restrict__ vbase, int32_t* __restrict__ vfirst) {
  const int h = blockIdx.x;
  const int32_t* vh = verts + int64_t(h) * cap_v;
  const int cnt = nv[h];
  int32_t* vb = vbase + int64_t(h) * (nseg_k + 1);
  int32_t* vf = vfirst + int64_t(h) * (nseg_k + 1);
  int base = 0;
  for (int m = 0; m <= nseg_k; ++m) {
    const int f = lower_bound32(vh, cnt, int64_t(m) * seg_len);
    vf[m] = f;
    vb[m] = base;
    if (m < nseg_k) {
      const int e = lower_bound32(vh, cnt, int64_t(m + 1) * seg_len);
      base += (e - f + 63) & ~63;
    }
  }
}

// Compacted vertical operands per (chunk, head): Kc_hi/lo [hq][capp][128],
// Vc^T [hq][128][capp], ckeys [hq][capp] (key or -1 for padding).
__global__ void compact_kernel(const __nv_bfloat16* __restrict__ khi,
                               const __nv_bfloat16* __restrict__ klo,
                               const __nv_bfloat16* __restrict__ v, int hkv, int group,
                               const int32_t* __restrict__ verts, const int32_t* __restrict__ nv,
                               int64_t cap_v, int64_t capp, int nseg_k,
                               const int32_t* __restrict__ vbase,
                               const int32_t* __restrict__ vfirst,
                               __nv_bfloat16* __restrict__ kchi, __nv_bfloat16* __restrict__ kclo,
                               __half* __restrict__ vct, int32_t* __restrict__ ckeys) {
  __shared__ __half tile[64][HD + 8];
  __shared__ int32_t keys[64];
  const int h = blockIdx.y, g = h / group;
  const int64_t c0 = int64_t(blockIdx.x) * 64;
  const int32_t* vb = vbase + int64_t(h) * (nseg_k + 1);
  const int32_t* vf = vfirst + int64_t(h) * (nseg_k + 1);
  if (threadIdx.x < 64) {
    const int64_t c = c0 + threadIdx.x;
    int32_t key = -1;
    if (c < vb[nseg_k]) {
      int m = 0;  // segment holding compact slot c (vbase ascending)
      while (m + 1 < nseg_k && vb[m + 1] <= c) ++m;
      const int64_t x = vf[m] + (c - vb[m]);
      if (x < vf[m + 1]) key = verts[int64_t(h) * cap_v + x];
    }
    keys[threadIdx.x] = key;
    if (c < capp) ckeys[int64_t(h) * capp + c] = key;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < 64 * (HD / 8); x += blockDim.x) {
    const int cc = x / (HD / 8), ch = x % (HD / 8);
    const int64_t c = c0 + cc;
    uint4 a = make_uint4(0, 0, 0, 0), b = a, vv = a;
    const int32_t j = keys[cc];
    if (j >= 0) {
      a = reinterpret_cast<const uint4*>(khi + (int64_t(j) * hkv + g) * HD)[ch];
      b = reinterpret_cast<const uint4*>(klo + (int64_t(j) * hkv + g) * HD)[ch];
      vv = reinterpret_cast<const uint4*>(v + (int64_t(j) * hkv + g) * HD)[ch];
    }
    if (c < capp) {
      reinterpret_cast<uint4*>(kchi + (int64_t(h) * capp + c) * HD)[ch] = a;
      reinterpret_cast<uint4*>(kclo + (int64_t(h) * capp + c) * HD)[ch] = b;
    }
    const __nv_bfloat16* vbf = reinterpret_cast<const __nv_bfloat16*>(&vv);
#pragma unroll
    for (int k = 0; k < 8; ++k) tile[cc][ch * 8 + k] = __float2half(__bfloat162float(vbf[k]));
  }
  __syncthreads();
  for (int x = threadIdx.x; x < 64 * HD; x += blockDim.x) {
    const int d = x / 64, cc = x % 64;
    const int64_t c = c0 + cc;
    if (c < capp) vct[(int64_t(h) * HD + d) * capp + c] = tile[cc][d];
  }
}

// Relative-tile classification per (chunk, head): one CTA per head.
// hist[1 - u] = slash entries of a 128-row block falling in key tile
// (block/64 + u), u = floor((r - d) / 64); tiles with >= min_entries go to
// tcgen05 (sorted ascending u list); the rest become CUDA-core segments
// (d, r0, r1), sorted by d.
__global__ void __launch_bounds__(1024)
classify_kernel(const int32_t* __restrict__ slashes, const int32_t* __restrict__ ns,
                int64_t cap_s, int64_t U, int min_entries, int32_t* __restrict__ hist_ws,
                int32_t* __restrict__ tc_u, int32_t* __restrict__ n_tc_u, int64_t cap_u,
                int4* __restrict__ segs, int32_t* __restrict__ nseg, int64_t cap_seg) {
  __shared__ int warp_sums[32];
  __shared__ int total;
  const int h = blockIdx.x;
  const int cnt = ns[h];
  const int32_t* sl = slashes + int64_t(h) * cap_s;
  int32_t* hist = hist_ws + int64_t(h) * U;
  for (int64_t x = threadIdx.x; x < U; x += blockDim.x) hist[x] = 0;
  __syncthreads();
  for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
    const int64_t d = sl[x];
    for (int64_t u = -((d + 63) >> 6) - 1; u <= 1; ++u) {  // floor(-d/64) .. 1
      const int64_t r0 = lcx_max64(0, d + 64 * u), r1 = lcx_min64(128, d + 64 * u + 64);
      if (r1 > r0 && 1 - u >= 0 && 1 - u < U) atomicAdd(hist + (1 - u), int(r1 - r0));
    }
  }
  __syncthreads();
  // ascending u <=> descending index
  auto scan = [&](int v) -> int {
    const int ln = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (ln >= o) x += y;
    }
    if (ln == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_sums[ln], ws = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ws, o);
        if (ln >= o) ws += y;
      }
      warp_sums[ln] = ws - w;
      if (ln == 31) total = ws;
    }
    __syncthreads();
    const int res = warp_sums[wid] + x - v;
    __syncthreads();
    return res;
  };
  int base = 0;
  for (int64_t s0 = 0; s0 < U; s0 += blockDim.x) {
    const int64_t x = s0 + threadIdx.x;
    const int64_t idx = U - 1 - x;  // ascending u
    int flag = 0;
    if (x < U) flag = hist[idx] >= min_entries && hist[idx] > 0;
    const int pos = scan(flag);
    const int tot = total;
    if (flag && base + pos < cap_u) tc_u[int64_t(h) * cap_u + base + pos] = int32_t(1 - idx);
    base += tot;
  }
  if (threadIdx.x == 0) n_tc_u[h] = int32_t(base < cap_u ? base : cap_u);
  __syncthreads();
  // segments (the hist array now doubles as the class lookup)
  int sbase = 0;
  for (int s0 = 0; s0 < cnt || s0 == 0; s0 += blockDim.x) {
    const int x = s0 + threadIdx.x;
    int4 sg[2];
    int nsg = 0;
    if (x < cnt) {
      const int64_t d = sl[x];
      int cur0 = -1, cur1 = -1;
      for (int64_t u = -((d + 63) >> 6) - 1; u <= 1; ++u) {
        const int64_t r0 = lcx_max64(0, d + 64 * u), r1 = lcx_min64(128, d + 64 * u + 64);
        if (r1 <= r0) continue;
        const int64_t idx = 1 - u;
        const bool tcu = idx >= 0 && idx < U && hist[idx] >= min_entries && hist[idx] > 0;
        if (!tcu) {
          if (cur1 == int(r0)) {
            cur1 = int(r1);
          } else {
            if (cur0 >= 0 && nsg < 2) sg[nsg++] = make_int4(int(d), cur0, cur1, 0);
            cur0 = int(r0);
            cur1 = int(r1);
          }
        }
      }
      if (cur0 >= 0 && nsg < 2) sg[nsg++] = make_int4(int(d), cur0, cur1, 0);
    }
    const int pos = scan(nsg);
    const int tot = total;
    for (int k = 0; k < nsg; ++k)
      if (sbase + pos + k < cap_seg) segs[int64_t(h) * cap_seg + sbase + pos + k] = sg[k];
    sbase += tot;
    if (s0 + int(blockDim.x) >= cnt) break;
  }
  if (threadIdx.x == 0) nseg[h] = int32_t(sbase < cap_seg ? sbase : cap_seg);
}

// Exact admitted-entry count of rows [t0, t1) per head (CriticalSet::admitted_count
// restricted to the chunk rows, sparse.cpp:115-119), in O(nv log ns + ns):
//   sum_v (t1 - max(t0, v)) + sum_d (t1 - max(t0, d)) - #{(v, d) : t0 <= v + d < t1}
//   + self-fallback rows.
__global__ void __launch_bounds__(256)
admitted_kernel(const int32_t* __restrict__ verts, const int32_t* __restrict__ nv, int64_t cap_v,
                const int32_t* __restrict__ slashes, const int32_t* __restrict__ ns,
                int64_t cap_s, int64_t t0, int64_t t1, int64_t* __restrict__ out) {
  __shared__ long long red[8];
  const int h = blockIdx.x;
  const int nvh = nv[h], nsh = ns[h];
  const int32_t* vh = verts + int64_t(h) * cap_v;
  const int32_t* sh = slashes + int64_t(h) * cap_s;
  long long acc = 0;
  for (int x = threadIdx.x; x < nvh; x += blockDim.x) {
    const int64_t v = vh[x];
    if (v < t1) acc += t1 - lcx_max64(t0, v);
    acc -= lower_bound32(sh, nsh, t1 - v) - lower_bound32(sh, nsh, t0 - v);
  }
  for (int x = threadIdx.x; x < nsh; x += blockDim.x) {
    const int64_t d = sh[x];
    if (d < t1) acc += t1 - lcx_max64(t0, d);
  }
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < 8; ++w) tot += red[w];
    int64_t first = INT64_MAX;
    if (nvh > 0) first = vh[0];
    if (nsh > 0) first = lcx_min64(first, sh[0]);
    tot += lcx_max64(0, lcx_min64(t1, first) - t0);  // rows without any line
    out[h] = tot;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int make_map3(CUtensorMap* m, CUtensorMapDataType dt, void* base, uint64_t d0, uint64_t d1,
              uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0,
              uint32_t b1, uint32_t b2) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(LCX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {b0, b1, b2};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = fn(m, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LCX_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return LCX_OK;
}

}  // namespace

// ------------------------------------------------------------ host API --
int tc_prepare(const void* k, const void* v, int64_t n, int hq, int hkv, const int64_t* pos_k,
               int rel_mode, int64_t s, const float2* rope, TcBuffers& B, cudaStream_t st) {
  const int64_t capp = B.capp;
  if (capp >= (int64_t(1) << 31)) return fail(LCX_ERR_DIMENSION, "vertical capacity too large");
  const int64_t pairs = n * hkv * (HD / 2);
  k_prep_kernel<<<unsigned((pairs + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(k), n, hkv, pos_k, rel_mode, s, rope, B.khi, B.klo);
  LCX_CHECK_LAUNCH();
  vt_prep_kernel<<<dim3(unsigned(B.npad / 64), unsigned(hkv)), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(v), n, hkv, B.npad, B.vt);
  LCX_CHECK_LAUNCH();
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, F16 = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  LCX_TRY(make_map3(&B.m_khi, BF, B.khi, HD, hkv, n, HD * 2, uint64_t(hkv) * HD * 2, 64, 1, 64));
  LCX_TRY(make_map3(&B.m_klo, BF, B.klo, HD, hkv, n, HD * 2, uint64_t(hkv) * HD * 2, 64, 1, 64));
  LCX_TRY(make_map3(&B.m_vt, F16, B.vt, B.npad, HD, hkv, B.npad * 2, uint64_t(HD) * B.npad * 2,
                    64, HD, 1));
  LCX_TRY(make_map3(&B.m_kchi, BF, B.kchi, HD, capp, hq, HD * 2, uint64_t(capp) * HD * 2, 64, 64,
                    1));
  LCX_TRY(make_map3(&B.m_kclo, BF, B.kclo, HD, capp, hq, HD * 2, uint64_t(capp) * HD * 2, 64, 64,
                    1));
  LCX_TRY(make_map3(&B.m_vct, F16, B.vct, capp, HD, hq, capp * 2, uint64_t(HD) * capp * 2, 64, HD,
                    1));
  return LCX_OK;
}

int tc_compact(const void* v, int hq, int hkv, const int32_t* verts, const int32_t* nv,
               int64_t cap_v, TcBuffers& B, cudaStream_t st) {
  vseg_kernel<<<hq, 1, 0, st>>>(verts, nv, cap_v, B.seg_len, B.nseg_k, B.vbase, B.vfirst);
  LCX_CHECK_LAUNCH();
  dim3 grid(unsigned(B.capp / 64), unsigned(hq));
  compact_kernel<<<grid, 256, 0, st>>>(B.khi, B.klo, reinterpret_cast<const __nv_bfloat16*>(v),
                                       hkv, hq / hkv, verts, nv, cap_v, B.capp, B.nseg_k, B.vbase,
                                       B.vfirst, B.kchi, B.kclo, B.vct, B.ckeys);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int tc_classify(const int32_t* slashes, const int32_t* ns, int64_t cap_s, int hq, int64_t U,
                int min_entries, int32_t* hist_ws, int32_t* tc_u, int32_t* n_tc_u, int64_t cap_u,
                int4* segs, int32_t* nseg, int64_t cap_seg, cudaStream_t st) {
  classify_kernel<<<hq, 1024, 0, st>>>(slashes, ns, cap_s, U, min_entries, hist_ws, tc_u, n_tc_u,
                                       cap_u, segs, nseg, cap_seg);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int tc_attention(const TcParams& p, const TcBuffers& B, int sm_count, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    LCX_CHECK_CUDA(cudaFuncSetAttribute(attn_tc_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(kSmemBytes)));
    attr = true;
  }
  if (p.nitems <= 0) return LCX_OK;
  const int grid = std::min(p.nitems, sm_count);
  attn_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(p, B.m_khi, B.m_klo, B.m_vt, B.m_kchi,
                                                     B.m_kclo, B.m_vct);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

}  // namespace lcx

namespace lcx {
int admitted_counts(const int32_t* verts, const int32_t* nv, int64_t cap_v,
                    const int32_t* slashes, const int32_t* ns, int64_t cap_s, int hq,
                    int64_t t0, int64_t t1, int64_t* out, cudaStream_t st) {
  admitted_kernel<<<hq, 256, 0, st>>>(verts, nv, cap_v, slashes, ns, cap_s, t0, t1, out);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}
}  // namespace lcx
