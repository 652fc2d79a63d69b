// K1 on tcgen05 -- the Vertical-Slash estimator for bf16 inputs, head dim 128.
//
// Same semantics as the exact CUDA-core estimator (estimate.cu; reference
// core/src/sparse.cpp:142-217): rows gi = t1 - B + r of the chunk, keys [0, t1),
// logit = rope(q, rel) . k / sqrt(D), rel = gi - j (near) or c - 1 (DcaContinuous far
// region, gi - j > c - 1), token-index positions, causal softmax, then column sums and
// per-diagonal sums of the probabilities.  Near logits are rope(q_gi, gi) .
// rope(k_j, j); far logits rope(q_gi, c - 1) . k_raw_j.
//
// The two matmul passes (pass 1: per-row max / sum-exp; pass 2: probabilities reduced
// into column and diagonal partials) run on the tensor cores with fp32-level accuracy:
// the fp32-rotated operands are scaled by a power of two (one exponent per query row and
// per 64-key tile, so the largest magnitude sits in [2^14, 2^15): exact, and far from the
// fp16 overflow and subnormal ranges) and split into two fp16 terms (x = h + l, 22
// significant bits); the three products of order >= 2^-11 (hh, hl, lh) are accumulated
// in fp32 TMEM and the power-of-two factors come off in the epilogue with the logit
// scale.  The far region's raw keys are exact in fp16 after the scaling (bf16 has 8
// significant bits) and need two products (h., l.).  A CTA owns one pair of query heads
// of one KV head (M = 128 = 2 x 64 estimator rows, its Q terms resident in TMEM) and a
// range of 64-key tiles streamed by TMA (N = 64); tiles whose rows straddle the near /
// far boundary go to the CUDA-core kernel (at most two per chunk).
//
// Warp roles (384 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM owner,
// warps 4-11 epilogue (TMEM lane quadrant = warp % 4, column half = (warp - 4) / 4).
// Pass 2 transposes each tile's probabilities through shared memory so that column
// sums (over a head's 64 rows) and diagonal sums (127 per head and tile) are
// conflict-free strided reads.
#include <cuda.h>

#include "attn_tc.cuh"
#include "est_tc.cuh"
#include "lcx_internal.cuh"
#include "tc_ptx.cuh"

namespace lcx {
namespace {

constexpr int BN = 64;             // keys per tile
#ifndef LCX_EST_PIECES
#define LCX_EST_PIECES 296
#endif
constexpr int kEstPieces = LCX_EST_PIECES;  // tensor-core pieces per head pair (see est_tc_plan)
constexpr int kQBox = 128 * 64 * 2;   // one [128 rows][64 dims] bf16 box = 16 KB
constexpr int kKBox = 64 * 64 * 2;    // one [64 keys][64 dims] box = 8 KB
constexpr int kQTerms = 2;
constexpr int kQBytes = 2 * kQTerms * kQBox;  // 2 terms x 2 halves = 64 KB
// K tile parts in the key buffer: rotated hi, rotated lo, raw (far region), 2 halves each
constexpr int kKParts = 3;
constexpr int kKStage = 4 * kKBox;    // near: 2 terms x 2 halves = 32 KB (far: raw, 16 KB)
constexpr int kTRow = 66;                         // floats per transpose row (bank skew)
constexpr int kTBuf = 128 * kTRow;                // floats per transpose buffer
// Q staging area: Q terms (TMA), then reused: pass-2 transposes [2][128][65] (pass 1:
// two more K stages)
constexpr int kQArea = ((2 * kTBuf * 4 > kQBytes ? 2 * kTBuf * 4 : kQBytes) + 1023) / 1024 * 1024;
constexpr int NKS = 4;          // K stages in the K region
constexpr int NKS_MAX = 6;      // pass 1 adds two stages in the Q staging area once Q is in TMEM
static_assert(2 * kKStage <= kQArea, "pass-1 extra stages must fit the Q staging area");
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + kQArea;
constexpr int OFF_BAR = OFF_K + NKS * kKStage;
constexpr int NSB = 4;                            // S buffers in TMEM
constexpr uint32_t QCOL = NSB * BN;               // TMEM: S [0, 256), Q terms [256, 384)
constexpr int kSmem = OFF_BAR + 256 + 1024;
static_assert(kSmem <= 227 * 1024, "shared memory");
constexpr int kThreads = 384;
constexpr uint32_t IDESC = tc::idesc_f16(128, BN, 0, 0);  // fp16 x fp16

struct Item {
  int pair;      // head pair index
  int far;       // 1: far tiles (raw K, Q at c - 1)
  int t0, t1;    // 64-key tiles [t0, t1)
  int split;     // stats split slot
};

// CTA -> (pair, phase, tile range): far tiles [0, far_end) then near tiles
// [near_begin, ntiles), each cut into `per`-tile pieces; split = piece index of the pair.
// Piece-major order (the call's pairs fastest): the CTAs running together cover every
// pair of a few pieces, so each key tile is fetched from DRAM once and served from L2 to
// the other head pairs of its KV head.
__device__ __forceinline__ Item decode_item(const EstTcParams& p, int idx) {
  const int nf = int((p.far_end + p.per - 1) / p.per);
  const int nn = int((p.ntiles - p.near_begin + p.per - 1) / p.per);
  Item it;
  const int k = idx / p.ncall_pairs;
  it.pair = p.pair0 + (idx - k * p.ncall_pairs);
  it.split = k;
  if (k < nf) {
    it.far = 1;
    it.t0 = k * p.per;
    it.t1 = int(lcx_min64(p.far_end, int64_t(it.t0) + p.per));
  } else {
    it.far = 0;
    it.t0 = int(p.near_begin + int64_t(k - nf) * p.per);
    it.t1 = int(lcx_min64(p.ntiles, int64_t(it.t0) + p.per));
  }
  return it;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Pass 2 epilogue split over specialised warps (LCX_EST_SPLIT_EPI): warps 4-7 turn each
// tile's S into probabilities (all 64 columns of a row per thread) and store them into the
// skewed transpose buffer, warps 8-11 reduce the previous buffer into column and diagonal
// sums, handing the two buffers back and forth on mbarriers -- the two phases of
// consecutive tiles overlap instead of all eight warps alternating between them behind a
// CTA barrier.
#ifndef LCX_EST_SPLIT_EPI
#define LCX_EST_SPLIT_EPI 1
#endif

template <int PASS>
__global__ void __launch_bounds__(kThreads, 1)
est_tc_kernel(const EstTcParams p, const __grid_constant__ CUtensorMap map_q,
              const __grid_constant__ CUtensorMap map_k3) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;          // [NKS_MAX]
  uint64_t* k_empty = k_full + NKS_MAX; // [NKS_MAX]
  uint64_t* s_full = k_empty + NKS_MAX; // [2]
  uint64_t* s_empty = s_full + NSB;     // [NSB]
  uint64_t* q_tmem = s_empty + NSB;     // epilogue warps copied Q into TMEM
  uint64_t* t_full = q_tmem + 1;        // [2] pass 2: transpose buffer written
  uint64_t* t_free = t_full + 2;        // [2] pass 2: transpose buffer reduced
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_free + 2);
  float* T = reinterpret_cast<float*>(smem + OFF_Q);

  const Item it = decode_item(p, blockIdx.x);
  // pass 1 streams through 4 K stages (2 in the K region, 2 in the Q staging area after Q
  // moved to TMEM); pass 2 keeps the Q area for its transposes
  constexpr int kStages = PASS == 1 ? NKS_MAX : NKS;
  auto stage_ptr = [&](int st) -> uint8_t* {
    return st < NKS ? smem + OFF_K + st * kKStage : smem + OFF_Q + (st - NKS) * kKStage;
  };
  const int ntl = it.t1 - it.t0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool kSplitEpi = PASS == 2 && LCX_EST_SPLIT_EPI;
  if (threadIdx.x == 0) {
    tc::mbar_init(q_full, 1);
    for (int b = 0; b < NKS_MAX; ++b) {
      tc::mbar_init(k_full + b, 1);
      tc::mbar_init(k_empty + b, 1);
    }
    for (int b = 0; b < NSB; ++b) {
      tc::mbar_init(s_full + b, 1);
      tc::mbar_init(s_empty + b, kSplitEpi ? 4 : 8);
    }
    tc::mbar_init(q_tmem, 8);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(t_full + b, 4 * 32);  // every lane of the 4 exp warps
      tc::mbar_init(t_free + b, 4 * 32);  // every lane of the 4 reduction warps
    }
    tc::fence_barrier_init();
    tc::fence_proxy_async();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int g = it.pair / p.pairs_per_group;   // kv head

  if (warp == 0) {
    if (lane == 0) {
      // resident Q terms of the pair (near: rope(q, gi); far: rope(q, c - 1))
      tc::mbar_expect_tx(q_full, kQBytes);
      const int qbox0 = ((it.far * p.npairs + it.pair) * 6);
      for (int b = 0; b < 2 * kQTerms; ++b)
        tc::tma_load_3d(smem + OFF_Q + b * kQBox, &map_q, q_full, 0, 0, qbox0 + b);
      for (int t = 0; t < ntl; ++t) {
        const int st = t % kStages;
        tc::mbar_wait(k_empty + st, ((t / kStages) & 1) ^ 1);
        if (st >= NKS && t < kStages) tc::mbar_wait(q_tmem, 0);  // Q staging area now free
        const int kt = it.t0 + t;
        uint8_t* dst = stage_ptr(st);
        // key tile parts: [hi h0, hi h1, lo h0, lo h1, raw h0, raw h1]
        const int b0 = int((int64_t(g) * p.ntiles_k + kt) * (2 * kKParts));
        if (it.far) {
          tc::mbar_expect_tx(k_full + st, 2 * kKBox);
          for (int b = 0; b < 2; ++b)
            tc::tma_load_3d(dst + b * kKBox, &map_k3, k_full + st, 0, 0, b0 + 4 + b);
        } else {
          tc::mbar_expect_tx(k_full + st, 4 * kKBox);
          for (int b = 0; b < 4; ++b)
            tc::tma_load_3d(dst + b * kKBox, &map_k3, k_full + st, 0, 0, b0 + b);
        }
      }
    }
  } else if (warp == 1) {
    // Q is the A operand from TMEM: with N = 64 an A operand in shared memory makes each
    // M128 N64 K16 MMA shared-memory-bound (48 vs 32 cycles, tools/micro/mma_rate.cu)
    tc::mbar_wait(q_tmem, 0);
    // (q term, k term) products of order >= 2^-11: hh hl lh (near), h. l. (far, raw keys
    // in stage part 0)
    const int qt_near[3] = {0, 0, 1}, kt_near[3] = {0, 1, 0};
    for (int t = 0; t < ntl; ++t) {
      const int st = t % kStages, sb = t % NSB;
      tc::mbar_wait(k_full + st, (t / kStages) & 1);
      tc::mbar_wait(s_empty + sb, ((t / NSB) & 1) ^ 1);
      tc::tc_fence_after();
      const uint64_t dk = tc::sdesc_sw128(tc::smem_u32(stage_ptr(st)));
      const uint32_t dS = tmem + sb * BN;
      const int nprod = it.far ? 2 : 3;
      for (int x = 0; x < nprod; ++x) {
        const int qt = it.far ? x : qt_near[x];
        const int kt = it.far ? 0 : kt_near[x];
#pragma unroll
        for (int half = 0; half < 2; ++half)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_f16_ts_warp(dS, tmem + QCOL + qt * 64 + half * 32 + kk * 8,
                                dk + (((kt * 2 + half) * kKBox + kk * 32) >> 4), IDESC,
                                (x | half | kk) ? 1u : 0u);
      }
      tc::mma_commit_warp(k_empty + st);
      tc::mma_commit_warp(s_full + sb);
    }
  } else if (warp >= 4) {
    const int wq = warp & 3, part = (warp - 4) >> 2;
    const int r = wq * 32 + lane;            // TMEM lane = row of the pair tile
    const int hh = r >> 6, rr = r & 63;      // head within the pair, estimator row
    const int h = g * p.group + (it.pair % p.pairs_per_group) * 2 + hh;
    const bool head_ok = (it.pair % p.pairs_per_group) * 2 + hh < p.group;
    const bool row_ok = head_ok && rr < p.block;
    const int64_t gi = p.nk - p.block + rr;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    float m = -INFINITY, s = 0.f, rm = 0.f, rinv = 0.f;
    if (PASS == 2 && row_ok) {
      const float2 ms = p.rowstat[int64_t(h) * p.block + rr];
      rm = ms.x * 1.4426950408889634f;  // natural -> log2 domain
      rinv = ms.y > 0.f ? 1.f / ms.y : 0.f;
    }
    // logit scale with this row's power-of-two Q factor; each tile adds its key factor
    const float sc =
        p.scale_log2 * p.qinv[(int64_t(it.far) * p.npairs + it.pair) * 128 + r];
    const float* kinv = p.kinv + int64_t(g) * p.ntiles_k;
    {  // Q terms: shared memory (TMA, SW128) -> TMEM, this thread's row and dim half
      tc::mbar_wait(q_full, 0);
#pragma unroll
      for (int tm = 0; tm < kQTerms; ++tm) {
        const uint8_t* box = smem + OFF_Q + (tm * 2 + part) * kQBox;
        uint32_t w[32];
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const uint4 x = *reinterpret_cast<const uint4*>(box + tc::sw128_off(r, c8));
          w[c8 * 4] = x.x;
          w[c8 * 4 + 1] = x.y;
          w[c8 * 4 + 2] = x.z;
          w[c8 * 4 + 3] = x.w;
        }
        tc::tmem_st32(tmem + lane_base + QCOL + tm * 64 + part * 32,
                      reinterpret_cast<const float*>(w));
      }
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(q_tmem);
      asm volatile("bar.sync 1, 256;" ::: "memory");  // Q staging area free for reuse
    }
    if constexpr (kSplitEpi) {
      if (part == 0) {
        // ---- exp warps: row r, all 64 columns -> probabilities -> skewed transpose ----
        const int rr64 = r & 63;
        for (int t = 0; t < ntl; ++t) {
          const int sb = t % NSB;
          const int64_t j0 = int64_t(it.t0 + t) * BN;
          tc::mbar_wait(s_full + sb, (t / NSB) & 1);
          tc::tc_fence_after();
          float v[64];
          tc::tmem_ld32(tmem + lane_base + sb * BN, v);
          tc::tmem_ld32_wait(tmem + lane_base + sb * BN + 32, v + 32);
          tc::tmem_wait_ld_dep32(v);
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(s_empty + sb);
          const int64_t lim = (gi < p.nk - 1 ? gi : p.nk - 1) - j0 + 1;
          const int nvalid = !row_ok ? 0 : (lim >= 64 ? 64 : (lim < 0 ? 0 : int(lim)));
          const float sct = sc * __ldg(kinv + it.t0 + t);
          // buffer t & 1 is free once the reduction warps finished tile t - 2
          tc::mbar_wait(t_free + (t & 1), ((t >> 1) & 1) ^ 1);
          float* Trow = T + (t & 1) * kTBuf + r * kTRow;
          if (__all_sync(0xffffffffu, nvalid == 64)) {
#pragma unroll
            for (int c = 0; c < 64; ++c) Trow[(c - rr64) & 63] = ex2(fmaf(v[c], sct, -rm)) * rinv;
          } else {
#pragma unroll
            for (int c = 0; c < 64; ++c)
              Trow[(c - rr64) & 63] = c < nvalid ? ex2(fmaf(v[c], sct, -rm)) * rinv : 0.f;
          }
          __syncwarp();
          tc::mbar_arrive(t_full + (t & 1));  // every lane releases its own stores
        }
      } else {
        // ---- reduction warps: et = (head of the pair) x 64 + key / buffer column ----
        const int et = threadIdx.x - 256;  // 0..127
        const int hh2 = et >> 6, x = et & 63;
        const int hx = g * p.group + (it.pair % p.pairs_per_group) * 2 + hh2;
        const bool hx_ok = (it.pair % p.pairs_per_group) * 2 + hh2 < p.group;
        for (int t = 0; t < ntl; ++t) {
          const int64_t j0 = int64_t(it.t0 + t) * BN;
          tc::mbar_wait(t_full + (t & 1), (t >> 1) & 1);
          const float* hb = T + (t & 1) * kTBuf + hh2 * 64 * kTRow;
          if (hx_ok) {
            // column sum of key x (its row-q element sits at buffer column (x - q) & 63)
            float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int q = 0; q < 64; q += 8)
#pragma unroll
              for (int u = 0; u < 8; ++u) a[u] += hb[(q + u) * kTRow + ((x - q - u) & 63)];
            const int64_t j = j0 + x;
            if (j < p.nk)
              p.col_part[int64_t(hx) * p.nk + j] =
                  ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
            // buffer column x: diagonals e = 63 - x (rows below 64 - x) and 127 - x
            float d1[4] = {0.f, 0.f, 0.f, 0.f}, d2[4] = {0.f, 0.f, 0.f, 0.f};
            const int lim = 64 - x;
#pragma unroll
            for (int q = 0; q < 64; q += 4)
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float y = hb[(q + u) * kTRow + x];
                const bool lo = q + u < lim;
                d1[u] += lo ? y : 0.f;
                d2[u] += lo ? 0.f : y;
              }
            float* dp = p.diag_part + (int64_t(hx) * p.ntiles + it.t0 + t) * 128;
            dp[63 - x] = (d1[0] + d1[1]) + (d1[2] + d1[3]);
            if (x > 0) dp[127 - x] = (d2[0] + d2[1]) + (d2[2] + d2[3]);
          }
          __syncwarp();
          tc::mbar_arrive(t_free + (t & 1));
        }
      }
    } else
    for (int t = 0; t < ntl; ++t) {
      const int sb = t % NSB;
      const int64_t j0 = int64_t(it.t0 + t) * BN;
      tc::mbar_wait(s_full + sb, (t / NSB) & 1);
      tc::tc_fence_after();
      float v[32];
      tc::tmem_ld32_wait(tmem + lane_base + sb * BN + part * 32, v);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(s_empty + sb);
      const int64_t jb = j0 + part * 32;
      // valid columns of this row: c < nvalid (causal j <= gi, j < nk); int32 compares
      const int64_t lim = (gi < p.nk - 1 ? gi : p.nk - 1) - jb + 1;
      const int nvalid = !row_ok ? 0 : (lim >= 32 ? 32 : (lim < 0 ? 0 : int(lim)));
      const float sct = sc * __ldg(kinv + it.t0 + t);
      if (PASS == 1) {
        float tmax = -INFINITY, ts = 0.f;
        if (__all_sync(0xffffffffu, nvalid == 32)) {
          // every column valid (all but the causal edge tiles): the scale is positive, so the
          // scaled max is the max's scaled value and the scaling folds into the exponent's FMA
          float mx[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
          for (int c = 4; c < 32; c += 4)
#pragma unroll
            for (int u = 0; u < 4; ++u) mx[u] = fmaxf(mx[u], v[c + u]);
          tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sct;
          float t4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int c = 0; c < 32; ++c) t4[c & 3] += ex2(fmaf(v[c], sct, -tmax));
          ts = (t4[0] + t4[1]) + (t4[2] + t4[3]);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            v[c] = c < nvalid ? v[c] * sct : -INFINITY;
            tmax = fmaxf(tmax, v[c]);
          }
          if (tmax != -INFINITY) {
#pragma unroll
            for (int c = 0; c < 32; ++c) ts += ex2(v[c] - tmax);
          }
        }
        if (tmax != -INFINITY) {
          const float nm = fmaxf(m, tmax);
          s = s * ex2(m - nm) + ts * ex2(tmax - nm);
          m = nm;
        }
      } else {
        // double-buffered skewed transpose, one barrier per tile (tile t + 2 rewrites this
        // buffer only after every thread passed tile t + 1's barrier, i.e. finished reading
        // it): row rr of a head stores key c at column (c - rr) mod 64, so a column of the
        // buffer holds the two diagonals -s and 64 - s (rows below / from 64 - s) and a key's
        // column walks the rows at a fixed skew -- both conflict-free with a row stride of 66
        // floats, every element read once per reduction.  Rows past the estimator block and
        // masked keys are stored as 0, so every sum has a fixed trip count.
        float* Tb = T + (t & 1) * kTBuf;
        {
          float* Trow = Tb + r * kTRow;
          const int rr64 = r & 63;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            Trow[(part * 32 + c - rr64) & 63] =
                c < nvalid ? ex2(fmaf(v[c], sct, -rm)) * rinv : 0.f;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int et = threadIdx.x - 128;    // 0..255
        const int hh2 = (et >> 6) & 1;       // head of the pair
        const int x = et & 63;               // key (et < 128) / buffer column (et >= 128)
        const int hx = g * p.group + (it.pair % p.pairs_per_group) * 2 + hh2;
        const bool hx_ok = (it.pair % p.pairs_per_group) * 2 + hh2 < p.group;
        const float* hb = Tb + hh2 * 64 * kTRow;
        if (et < 128) {  // column sums: key x of head hh2
          const int64_t j = j0 + x;
          if (hx_ok && j < p.nk) {
            float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 chains, loads up front
#pragma unroll
            for (int q = 0; q < 64; q += 8)
#pragma unroll
              for (int u = 0; u < 8; ++u) a[u] += hb[(q + u) * kTRow + ((x - q - u) & 63)];
            p.col_part[int64_t(hx) * p.nk + j] =
                ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
          }
        } else if (hx_ok) {  // diagonal sums: buffer column x = diagonals e = 63 - x, 127 - x
          float a[4] = {0.f, 0.f, 0.f, 0.f}, b2[4] = {0.f, 0.f, 0.f, 0.f};
          const int lim = 64 - x;  // rows below lim: diagonal 63 - x (e = r - c + 63)
#pragma unroll
          for (int q = 0; q < 64; q += 4)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float y = hb[(q + u) * kTRow + x];
              const bool lo = q + u < lim;
              a[u] += lo ? y : 0.f;
              b2[u] += lo ? 0.f : y;
            }
          float* dp = p.diag_part + (int64_t(hx) * p.ntiles + it.t0 + t) * 128;
          dp[63 - x] = (a[0] + a[1]) + (a[2] + a[3]);
          if (x > 0) dp[127 - x] = (b2[0] + b2[1]) + (b2[2] + b2[3]);
        }
      }
    }
    if (PASS == 1) {
      // combine the two column halves of the row, then write this split's stats
      float* red = T;  // [2][128] (m, s) exchange, pass 1 does not use the transpose
      red[part * 256 + r * 2] = m;
      red[part * 256 + r * 2 + 1] = s;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (part == 0 && row_ok) {
        const float m2 = red[256 + r * 2], s2 = red[256 + r * 2 + 1];
        const float nm = fmaxf(m, m2);
        float tot = 0.f;
        if (nm != -INFINITY) tot = s * ex2(m - nm) + s2 * ex2(m2 - nm);
        // natural-log domain (m, sum), as the CUDA-core estimator writes them
        p.stats[(int64_t(h) * p.nsplit + it.split) * p.block + rr] =
            make_float2(nm == -INFINITY ? -INFINITY : nm * 0.6931471805599453f, tot);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------- prep --
// Power-of-two scale putting the largest magnitude m of a block in [2^14, 2^15): fp16
// terms then stay far from overflow (65504) and from the subnormal range.
__device__ __forceinline__ int pow2_exp(float m) {
  if (!(m > 0.f)) return 0;
  int e = 14 - ilogbf(m);
  return e < -120 ? -120 : (e > 120 ? 120 : e);
}

// 2^e as a float, e in [-120, 120] (pow2_exp's range): x * pow2f(e) == ldexpf(x, e) bitwise
// (scaling by a normal power of two rounds like ldexpf), without ldexpf's special-case code
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

__device__ __forceinline__ float block_max256(float v, float* red) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float m = red[0];
  for (int w = 1; w < int(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
  return m;
}

// Key tiles [tile0, tile1) of KV head blockIdx.y, keys < r1 (the rest of the last tile
// zero; a later call extending the keys rewrites that tile whole):
//   K3 [hkv][ntiles][hi h0, hi h1, lo h0, lo h1, raw h0, raw h1][64 keys][64 dims] fp16
//   hi + lo = rope(k_j, j) * 2^e, raw = k_j * 2^e (exact), kinv [hkv][ntiles] = 2^-e
// with one exponent per tile (pow2_exp of the tile's largest rotated / raw magnitude).
__global__ void __launch_bounds__(256) est_k3_kernel(const __nv_bfloat16* __restrict__ k,
                                                     int64_t tile0, int64_t r1, int hkv,
                                                     int64_t ntiles,
                                                     const float2* __restrict__ rope,
                                                     __half* __restrict__ k3,
                                                     float* __restrict__ kinv) {
  __shared__ float red[8];
  const int64_t tile = tile0 + blockIdx.x;
  const int gg = blockIdx.y;
  constexpr int kPer = 64 * 64 / 256;  // (key, pair) elements per thread
  float2 rot[kPer], raw[kPer];
  float mx = 0.f;
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int e = x * 256 + threadIdx.x;
    const int jj = e >> 6, pr = e & 63;
    const int64_t j = tile * 64 + jj;
    float2 xy = make_float2(0.f, 0.f), rr = xy;
    if (j < r1) {
      xy = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(k)[(j * hkv + gg) * 64 + pr]);
      const float2 cs = rope[j * 64 + pr];
      rr = make_float2(xy.x * cs.x - xy.y * cs.y, xy.x * cs.y + xy.y * cs.x);
    }
    rot[x] = rr;
    raw[x] = xy;
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(rr.x), fabsf(rr.y)), fmaxf(fabsf(xy.x), fabsf(xy.y))));
  }
  const int ex = pow2_exp(block_max256(mx, red));
  if (threadIdx.x == 0) kinv[int64_t(gg) * ntiles + tile] = exp2f(float(-ex));
  const float sc = pow2f(ex);
  __half2* base = reinterpret_cast<__half2*>(k3 + (int64_t(gg) * ntiles + tile) * 6 * 64 * 64);
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int e = x * 256 + threadIdx.x;
    const int jj = e >> 6, pr = e & 63;
    const int d = 2 * pr, half = d >> 6;
    const float2 rs = make_float2(rot[x].x * sc, rot[x].y * sc);
    const __half2 h2 = __floats2half2_rn(rs.x, rs.y);
    const float2 hf = __half22float2(h2);
    const __half2 l2 = __floats2half2_rn(rs.x - hf.x, rs.y - hf.y);
    const __half2 w2 = __floats2half2_rn(raw[x].x * sc, raw[x].y * sc);
    const int64_t o = (int64_t(jj) * 64 + (d & 63)) >> 1;  // within one [64][64] box
    base[(0 + half) * 2048 + o] = h2;
    base[(2 + half) * 2048 + o] = l2;
    base[(4 + half) * 2048 + o] = w2;
  }
}

// Q3 [far 0/1][npairs][2 terms][2 halves][128 rows][64 dims] fp16 (box stride: 6 boxes per
// (far, pair)): row = 64 * (head in pair) + r, hi + lo = rope(q, pos) * 2^e with one
// exponent per row; qinv [far][npairs][128] = 2^-e.
__global__ void __launch_bounds__(64) est_q3_kernel(
    const __nv_bfloat16* __restrict__ q, int hq, int group, int pairs_per_group, int npairs,
    int pair0, int64_t nk, int64_t block, int far_too, int64_t c,
    const float2* __restrict__ rope, __half* __restrict__ q3, float* __restrict__ qinv) {
  __shared__ float red[2];
  const int row = blockIdx.x;        // 0..127
  const int pair = pair0 + int(blockIdx.y);
  const int far = blockIdx.z;
  if (far && !far_too) return;
  const int pr = threadIdx.x;        // 0..63
  const int hh = row >> 6, r = row & 63;
  const int hig = (pair % pairs_per_group) * 2 + hh;
  const int h = (pair / pairs_per_group) * group + hig;
  float rx = 0.f, ry = 0.f;
  if (hig < group && r < block) {
    const int64_t gi = nk - block + r;
    const float2 xy = __bfloat1622float2(
        reinterpret_cast<const __nv_bfloat162*>(q + (gi * hq + h) * 128)[pr]);
    const float2 cs = rope[(far ? c - 1 : gi) * 64 + pr];
    rx = xy.x * cs.x - xy.y * cs.y;
    ry = xy.x * cs.y + xy.y * cs.x;
  }
  float m = fmaxf(fabsf(rx), fabsf(ry));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((pr & 31) == 0) red[pr >> 5] = m;
  __syncthreads();
  const int ex = pow2_exp(fmaxf(red[0], red[1]));
  if (pr == 0) qinv[(int64_t(far) * npairs + pair) * 128 + row] = exp2f(float(-ex));
  rx *= pow2f(ex);
  ry *= pow2f(ex);
  const __half2 h2 = __floats2half2_rn(rx, ry);
  const float2 hf = __half22float2(h2);
  const __half2 l2 = __floats2half2_rn(rx - hf.x, ry - hf.y);
  const __half2 terms[2] = {h2, l2};
  const int d = 2 * pr, half = d >> 6;
#pragma unroll
  for (int tm = 0; tm < 2; ++tm) {
    const int64_t o = (((((int64_t(far) * npairs + pair) * 6 + tm * 2 + half) * 128 + row) * 64 +
                        (d & 63))) >> 1;
    reinterpret_cast<__half2*>(q3)[o] = terms[tm];
  }
}

}  // namespace

// key tile parts (ntiles x hkv x 6 boxes), then the per-tile factors kinv [hkv][ntiles]
static size_t k3_parts_bytes(int64_t ntiles, int hkv) {
  return size_t(ntiles) * hkv * 2 * kKParts * kKBox;
}

size_t est_tc_k3_bytes(int64_t n, int hkv) {
  const int64_t nt = (n + 63) / 64;
  return k3_parts_bytes(nt, hkv) + ((size_t(nt) * hkv * 4 + 255) & ~size_t(255));
}

static float* k3_kinv(const void* k3, int64_t ntiles, int hkv) {
  return reinterpret_cast<float*>(const_cast<uint8_t*>(reinterpret_cast<const uint8_t*>(k3)) +
                                  k3_parts_bytes(ntiles, hkv));
}

int est_tc_prepare_keys(const void* k, int64_t r0, int64_t r1, int hkv, int64_t ntiles,
                        const float2* rope, void* k3, cudaStream_t st) {
  if (r1 <= r0) return LCX_OK;
  // whole tiles: a tile that an earlier call left partial is rebuilt with all its keys
  const int64_t tile0 = r0 / 64, tile1 = (r1 + 63) / 64;
  est_k3_kernel<<<dim3(unsigned(tile1 - tile0), unsigned(hkv)), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(k), tile0, r1, hkv, ntiles, rope,
      reinterpret_cast<__half*>(k3), k3_kinv(k3, ntiles, hkv));
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

bool est_tc_eligible(int dtype, int dim, int64_t block) {
  return dtype == LCX_BF16 && dim == 128 && block <= 64;
}

void est_tc_size(int hq, int hkv, Sizer& sz) {
  const int group = hq / hkv, ppg = (group + 1) / 2, npairs = hkv * ppg;
  sz.take<uint8_t>(size_t(2) * npairs * 6 * kQBox);  // q3
  sz.take<float>(size_t(2) * npairs * 128);          // qinv
}

int est_tc_max_splits() { return 2 * (kEstPieces + 2); }

void est_tc_plan(const EstTcArgs& a, EstTcPlan& pl) {
  const int group = a.hq / a.hkv, ppg = (group + 1) / 2;
  pl.npairs = a.hkv * ppg;
  // head pairs meeting the call's heads [h0, h1): pair of head h = (h / group) * ppg +
  // (h % group) / 2
  auto pair_of = [&](int h) { return (h / group) * ppg + (h % group) / 2; };
  pl.pair0 = a.h1 > a.h0 ? pair_of(a.h0) : 0;
  pl.pair1 = a.h1 > a.h0 ? pair_of(a.h1 - 1) + 1 : 0;
  pl.ntiles = (a.nk + 63) / 64;
  pl.far_end = 0;
  pl.near_begin = 0;
  if (a.pos_mode == 1) {
    // near iff gi - j <= c - 1 (sparse.cpp:169-178), gi in [nk - block, nk):
    // keys < nk - block - c + 1 are far for every row, keys >= nk - c near for every row
    const int64_t lim_far = a.nk - a.block - a.c + 1;
    pl.far_end = lim_far > 0 ? std::min<int64_t>(pl.ntiles, lim_far / 64) : 0;
    const int64_t near_key = a.nk - a.c;
    pl.near_begin = near_key <= 0 ? 0 : std::min<int64_t>(pl.ntiles, (near_key + 63) / 64);
    if (pl.near_begin < pl.far_end) pl.near_begin = pl.far_end;
  }
  // pieces of 1/kEstPieces of the chunk's tensor-core tiles (>= 4 tiles): a function of
  // the key range only, so a head's row statistics (combined over pieces in a fixed
  // order) are bitwise the same whichever heads a call covers -- the estimator shards
  // over GPUs by head pairs with no exchange.  kEstPieces = 37 x 8: 16 head pairs (7B)
  // = 4736 CTAs on one GPU, and still 592 (4 full waves on 148 SMs) for the two pairs of
  // one rank of eight.
  const int64_t tc_tiles = pl.far_end + (pl.ntiles - pl.near_begin);
  pl.per = int(std::max<int64_t>(4, (tc_tiles + kEstPieces - 1) / kEstPieces));
  const int nf = int((pl.far_end + pl.per - 1) / pl.per);
  const int nn = int((pl.ntiles - pl.near_begin + pl.per - 1) / pl.per);
  pl.tc_splits = nf + nn;
  pl.items = (pl.pair1 - pl.pair0) * (nf + nn);
}

// One pass of the estimator for one chunk on the tensor cores over the far and near
// tiles of every head pair; writes the same stats / column / diagonal partials as the
// CUDA-core estimator (which covers the mixed tiles [far_end, near_begin)).
int est_tc_run(const EstTcArgs& a, const EstTcPlan& pl, Arena& ar, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    LCX_CHECK_CUDA(cudaFuncSetAttribute(est_tc_kernel<1>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    LCX_CHECK_CUDA(cudaFuncSetAttribute(est_tc_kernel<2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr = true;
  }
  const int group = a.hq / a.hkv, ppg = (group + 1) / 2, npairs = pl.npairs;
  uint8_t* q3 = ar.take<uint8_t>(size_t(2) * npairs * 6 * kQBox);
  float* qinv = ar.take<float>(size_t(2) * npairs * 128);
  if (pl.items == 0) return LCX_OK;
  const bool dca = a.pos_mode == 1;
  if (a.pass == 1) {  // operands: rotated, 3-term split query rows (near and far)
    dim3 grid(128, unsigned(pl.pair1 - pl.pair0), 2);
    est_q3_kernel<<<grid, 64, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(a.q), a.hq, group,
                                       ppg, npairs, pl.pair0, a.nk, a.block, dca ? 1 : 0, a.c,
                                       a.rope, reinterpret_cast<__half*>(q3), qinv);
    LCX_CHECK_LAUNCH();
  }
  CUtensorMap mq, mk3;
  const auto F16 = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  LCX_TRY(make_tmap3(&mq, F16, q3, 64, 128, uint64_t(2) * npairs * 6, 128, kQBox, 64, 128, 1));
  LCX_TRY(make_tmap3(&mk3, F16, const_cast<void*>(a.k3), 64, 64,
                     uint64_t(a.hkv) * a.k3_tiles * 2 * kKParts, 128, kKBox, 64, 64, 1));
  EstTcParams p{};
  p.group = group;
  p.pairs_per_group = ppg;
  p.npairs = npairs;
  p.pair0 = pl.pair0;
  p.ncall_pairs = pl.pair1 - pl.pair0;
  p.nk = a.nk;
  p.block = int(a.block);
  p.ntiles_k = a.k3_tiles;
  p.ntiles = pl.ntiles;
  p.far_end = pl.far_end;
  p.near_begin = pl.near_begin;
  p.per = pl.per;
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(128.0));
  p.nsplit = a.nsplit;
  p.stats = a.stats;
  p.rowstat = a.rowstat;
  p.col_part = a.col_part;
  p.diag_part = a.diag_part;
  p.qinv = qinv;
  p.kinv = k3_kinv(a.k3, a.k3_tiles, a.hkv);
  if (a.pass == 1)
    est_tc_kernel<1><<<unsigned(pl.items), kThreads, kSmem, st>>>(p, mq, mk3);
  else
    est_tc_kernel<2><<<unsigned(pl.items), kThreads, kSmem, st>>>(p, mq, mk3);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

}  // namespace lcx
