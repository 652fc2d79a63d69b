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
// (attn_gather.cu) as (d, first row, last row) segments and are merged in place.
//
// Precision (bf16 storage, 2e-3 contract): q and k are rotated in fp32 and split
// into bf16 hi + lo; S = q_hi k_hi + q_hi k_lo + q_lo k_hi (3 MMAs, fp32 TMEM
// accumulate); P is fp16 (<= 2^8 under a lazy-rescale threshold of 8 in log2
// units); V is fp16.  Executed MMA work per tile = 4 units vs 2 algorithmic.
//
// Warp roles (384 threads): warps 0-7 softmax / correction / epilogue in two groups
// of four that take alternate tiles (thread = query row, TMEM lane quadrant =
// warp % 4), warp 8 producer (tile metadata ring + K loads), warp 9 QK issuer + TMEM
// owner, warp 10 PV issuer, warp 11 V loads.  Pipelines: K (hi+lo) and V^T in four
// shared-memory stages, S double-buffered in TMEM (2 x 64 columns) with P (fp16)
// written over it, O in TMEM (128 columns), rotated Q hi/lo in TMEM (two buffers, one
// per DCA pattern group parity) as the A operand of every QK MMA.
#include <cuda.h>

#include "lcx_internal.cuh"
#include "tc_ptx.cuh"
#include "attn_tc.cuh"

namespace lcx {



namespace {

constexpr int BM = 128, BN = 64, HD = 128;
// Unit of the pipeline: a DOUBLE TILE (DT) = up to two 64-key tiles of one item and one DCA
// pattern group, sharing one 128-column S buffer, one softmax pass over 128 logits per
// row and one K = 128 PV step.  Every per-tile control cost (metadata ring, mbarrier
// hand-offs, running-max hand-off, TMEM load/store waits) is paid once per 128 keys.
// The two halves are independent 64-key tiles (any kinds, any keys): the QK MMAs of half
// j write S columns [64 j, 64 j + 64) of the buffer, its P (fp16 pairs) lands in columns
// [64 j, 64 j + 32), and the PV MMAs of half j read those with half j's V^T stage.
//
// warps 0-7 softmax (TMEM lane quadrant = warp % 4, group = warp / 4; group g takes the
// DTs T with T % 2 == g), warp 8 producer (DT metadata + K loads), warp 9 QK issuer +
// TMEM allocator, warp 10 PV issuer, warp 11 V loads
constexpr int kGroups = 2;
constexpr int kSoftmaxWarps = 4 * kGroups;
constexpr int kThreads = 32 * (kSoftmaxWarps + 4);
constexpr int kWarpProducer = kSoftmaxWarps, kWarpMma = kSoftmaxWarps + 1,
              kWarpPv = kSoftmaxWarps + 2, kWarpV = kSoftmaxWarps + 3;
constexpr int NK = 4, NV = 4;  // K / V shared-memory stages, one 64-key tile each
constexpr int NS = 2;          // S (+P) TMEM buffers, one DT each
static_assert(NS % kGroups == 0, "each group must see every phase of its S buffers");
constexpr int DTN = 2 * BN;                          // keys per double tile
constexpr uint32_t kKHalf = BN * 64 * 2;             // 8 KB
constexpr uint32_t kKStage = 4 * kKHalf;             // hi0 hi1 lo0 lo1 = 32 KB
constexpr uint32_t kVStage = HD * BN * 2;            // 16 KB
constexpr uint32_t OFF_K = 0;
constexpr uint32_t OFF_V = OFF_K + NK * kKStage;     // 128 KB
constexpr uint32_t OFF_BAR = OFF_V + NV * kVStage;   // 192 KB
constexpr uint32_t OFF_META = OFF_BAR + 1024;
constexpr int kMetaSlots = 8;                        // DT metadata ring
constexpr uint32_t kMetaBytes = 720;
// softmax exchange: running max per group [kGroups][128], partial sums (l, m)
// [2 slot][kGroups][128]
constexpr uint32_t OFF_RED = OFF_META + kMetaSlots * kMetaBytes;
constexpr uint32_t kSmemBytes =
    OFF_RED + kGroups * 128 * 4 + 2 * kGroups * 128 * 8 + 1024;  // + align slack
static_assert(kSmemBytes <= 227 * 1024, "shared memory");
// TMEM (512 columns x 128 lanes): S/P buffers [0, 256) (128 columns per DT), O [256, 384),
// rotated Q [384, 512) (hi, then lo; bf16 pairs per 32-bit column) -- the A operand of
// every QK MMA, so all MMAs read only B from shared memory.  One Q buffer: at a DCA
// pattern change the owner of the old pattern's last DT re-rotates it once that DT's S
// is full (all of the old pattern's QKs are complete).
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t COL_S = 0;
constexpr uint32_t COL_O = NS * DTN;
constexpr uint32_t COL_Q = COL_O + HD;
static_assert(COL_Q + HD <= 512, "TMEM columns");
constexpr float kRescaleThresh = 8.f;
// producer / V-load warps poll with a sleep (ns) instead of a suspended try_wait: their
// waits are off the critical path and would otherwise take issue slots from the softmax
// warps sharing their sub-partitions (round 1: -1 to -1.5 % kernel time at 300 ns)
#ifndef LCX_TC_SLEEPY
#define LCX_TC_SLEEPY 300
#endif

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
  int ndt;  // double tiles: the tiles of each pattern group paired in order
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
  it.ndt = 0;
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
      G.nvt = p.vert_pass ? (G.vhi - G.vlo + 63) >> 6 : 0;
      // slash tiles of this pass's key window [key_lo, key_hi) (64-aligned)
      const int64_t wlo = lcx_max64(G.klo, p.key_lo), whi = lcx_min64(G.khi, p.key_hi);
      if (whi > wlo) {
        G.ulo = lower_bound32(uh, nuh, (wlo >> 6) - ib);
        G.uhi = lower_bound32(uh, nuh, ceil_div64(whi) - ib);
      } else {
        G.ulo = G.uhi = 0;
      }
      G.nst = G.uhi - G.ulo;
    }
    if (G.nvt + G.nst == 0) continue;
    it.grp[it.ng++] = G;
    it.ntiles += G.nvt + G.nst;
    it.ndt += (G.nvt + G.nst + 1) >> 1;
  }
}

__device__ __forceinline__ Tile get_tile(const TcParams& p, const Item& it, int t) {
  Tile T{};
#pragma unroll
  for (int x = 0; x < 3; ++x) {  // compile-time group index: Item stays in registers
    if (x >= it.ng) break;
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

__device__ __forceinline__ int grp_pattern(const Item& it, int g) {
  return g == 0 ? it.grp[0].pattern : (g == 1 ? it.grp[1].pattern : it.grp[2].pattern);
}

__device__ __forceinline__ int64_t qpos_of(const TcParams& p, int pattern, int64_t i) {
  if (p.rel_mode == 0) return p.pos_q ? p.pos_q[i] : i;
  const int64_t im = i % p.s;
  if (pattern == 0) return im;
  if (pattern == 1) return lcx_min64(im + p.s, p.c - 1);
  return p.c - 1;
}

// Rotate this thread's query row (its 64-dim half) by its pattern position and
// store the bf16 hi / lo split into TMEM (row = lane, dim pair = column).
__device__ __forceinline__ void rotate_q(const TcParams& p, const Item& it, int pattern, int r,
                                         int part, uint32_t tmem_row) {
  const int64_t i = it.i0 + r;
  const bool ok = i < it.rend;
  const uint4* src = reinterpret_cast<const uint4*>(p.q + (i * p.hq + it.h) * int64_t(HD));
  const float2* cs = p.rope + (ok ? qpos_of(p, pattern, i) : 0) * (HD / 2);
  uint32_t hi[32], lo[32];
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) {  // 8 chunks of 8 dims in this half
    const int ch = part * 8 + c8;
    uint4 raw = ok ? src[ch] : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 xy = __bfloat1622float2(x2[k]);
      const float2 c = cs[ch * 4 + k];
      // the logit scale log2(e) / (t sqrt(D)) is folded into the rotated query, so S comes
      // out of the MMA in log2 units
      const float rx = (xy.x * c.x - xy.y * c.y) * p.scale_log2;
      const float ry = (xy.x * c.y + xy.y * c.x) * p.scale_log2;
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(rx, ry);
      const float2 hf = __bfloat1622float2(h2);
      const __nv_bfloat162 l2 = __floats2bfloat162_rn(rx - hf.x, ry - hf.y);
      hi[c8 * 4 + k] = *reinterpret_cast<const uint32_t*>(&h2);
      lo[c8 * 4 + k] = *reinterpret_cast<const uint32_t*>(&l2);
    }
  }
  const uint32_t qc = tmem_row + COL_Q;
  tc::tmem_st32(qc + part * 32, reinterpret_cast<const float*>(hi));
  tc::tmem_st32(qc + HD / 2 + part * 32, reinterpret_cast<const float*>(lo));
  tc::tmem_wait_st();
}

// Per-DT control record, written by the producer warp into a shared-memory ring so
// that the MMA and softmax warps never touch global memory for control.
enum { T_TILES = 0, T_EMPTY = 3, T_END = 4 };
enum { F_FIRST = 1, F_LAST = 2, F_EPOCH = 4, F_EPOCH_AFTER = 8 };
struct SubMeta {  // one 64-key half of a DT
  int32_t kind, count, nfar, pad;
  int64_t key0, sbase;
  uint64_t vmask;
  uint32_t sw[8];
  int32_t keys[64];
};
struct DtMeta {
  int32_t kind, flags, pattern, next_pattern;
  int32_t h, nsub, pad0, pad1;
  int64_t i0, rend;
  SubMeta sub[2];
};
static_assert(sizeof(DtMeta) <= kMetaBytes, "DT metadata slot overflow");
static_assert(kMetaBytes % 16 == 0, "DT metadata slot alignment");

// wait profile (LCX_TC_WAITPROF, tools/trace_wait.py): cycles each role spends per wait
// site, summed over all CTAs into trace[4096 + role * 8 + site]
#ifdef LCX_TC_WAITPROF
#define WAITP(site, ...)                      \
  do {                                        \
    const long long _w0 = clock64();          \
    __VA_ARGS__;                              \
    wacc[site] += clock64() - _w0;            \
  } while (0)
#define WAITP_FLUSH(role)                                                                   \
  do {                                                                                      \
    if (lane == 0 && p.trace)                                                               \
      for (int _j = 0; _j < 8; ++_j)                                                        \
        atomicAdd(reinterpret_cast<unsigned long long*>(p.trace + 4096 + (role) * 8 + _j),  \
                  (unsigned long long)wacc[_j]);                                            \
  } while (0)
#else
#define WAITP(site, ...) __VA_ARGS__
#define WAITP_FLUSH(role) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t window64(const uint32_t* sw, int off) {
  // bits [off, off + 64) of the 256-bit array sw (off in [0, 192])
  const int w = off >> 5, sh = off & 31;
  const uint64_t a = uint64_t(sw[w]) | (uint64_t(sw[w + 1]) << 32);
  const uint64_t b = (w + 2 < 8) ? sw[w + 2] : 0u;
  return sh ? ((a >> sh) | (b << (64 - sh))) : a;
}

// admitted-entry mask of row i over the 64 keys of one half (bit c: key c of the tile)
__device__ __forceinline__ uint64_t sub_mask(const SubMeta& sm, int64_t i) {
  if (sm.kind == T_VERT) {
    int cnt = sm.nfar;  // keys below the row block: admitted by every row
    while (cnt < sm.count) {
      const int32_t kk = sm.keys[cnt];
      if (kk < 0 || int64_t(kk) > i) break;
      ++cnt;
    }
    return cnt >= 64 ? ~0ull : ((1ull << cnt) - 1);
  }
  if (sm.kind == T_SLASH) {
    const int off = int(i - sm.key0 - 63 - sm.sbase);
    return __brevll(window64(sm.sw, off)) & ~sm.vmask;
  }
  const int64_t lim = i - sm.key0;  // dense: causal
  return lim >= 63 ? ~0ull : (lim < 0 ? 0ull : ((2ull << lim) - 1));
}

__global__ void __launch_bounds__(kThreads, 1)
attn_tc_kernel(const TcParams p) {
  // key-window pass with no slash tile anywhere in it (and no vertical pass): nothing to do
  if (!p.vert_pass && p.win_flags && !p.win_flags[p.win]) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // stay in the shared address space (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  // barriers as 32-bit shared addresses (no generic -> shared conversion per use)
  const uint32_t smem_base = tc::smem_u32(smem);
  const tc::SBar k_full{smem_base + OFF_BAR};  // [NK] TMA -> MMA
  const tc::SBar k_empty = k_full + NK;        // [NK] QK commit -> producer
  const tc::SBar v_full = k_empty + NK;        // [NV]
  const tc::SBar v_empty = v_full + NV;        // [NV] PV commit -> V loader
  const tc::SBar s_full = v_empty + NV;        // [NS] QK commit -> softmax
  const tc::SBar s_free = s_full + NS;         // [NS] PV commit (S/P buffer, O updated)
  const tc::SBar p_full = s_free + NS;         // [NS] softmax wrote P -> PV issuer
  const tc::SBar q_ready = p_full + NS;        // [1] softmax rotated Q -> QK issuer
  const tc::SBar m_full = q_ready + 1;         // [kMetaSlots]
  const tc::SBar m_empty = m_full + kMetaSlots;  // [kMetaSlots]
  const tc::SBar hand = m_empty + kMetaSlots;    // [kGroups][4] running max of a DT ready
  const tc::SBar lpub = hand + 4 * kGroups;      // [kGroups] partial sums of a DT written
  constexpr int kBars = 2 * NK + 2 * NV + 3 * NS + 1 + 2 * kMetaSlots + 5 * kGroups;
  static_assert((kBars + 1) * 8 <= 1024, "barrier area overflow");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR) + 2 * kBars;
  DtMeta* metas = reinterpret_cast<DtMeta*>(smem + OFF_META);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef LCX_TC_WAITPROF
  long long wacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
#endif
  if (threadIdx.x == 0) {
    for (int b = 0; b < NK; ++b) {
      tc::mbar_init(k_full + b, 1);
      tc::mbar_init(k_empty + b, 1);
    }
    for (int b = 0; b < NV; ++b) {
      tc::mbar_init(v_full + b, 1);
      tc::mbar_init(v_empty + b, 1);
    }
    for (int b = 0; b < NS; ++b) {
      tc::mbar_init(s_full + b, 1);
      tc::mbar_init(s_free + b, 1);
      tc::mbar_init(p_full + b, 4);  // the DT's warp group
    }
    tc::mbar_init(q_ready, 4);
    for (int b = 0; b < 4 * kGroups; ++b) tc::mbar_init(hand + b, 1);
    for (int b = 0; b < kGroups; ++b) tc::mbar_init(lpub + b, 4);
    for (int b = 0; b < kMetaSlots; ++b) {
      tc::mbar_init(m_full + b, 1);
      tc::mbar_init(m_empty + b, kSoftmaxWarps + 3);  // softmax + QK + PV + V warps
    }
    tc::fence_barrier_init();
    tc::fence_proxy_async();
  }
  if (warp == kWarpMma) tc::tmem_alloc(tmem_slot, kTmemCols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpProducer) {
    // ====================================== producer: DT stream + metadata + K loads ====
    // Batches of two DTs (four 64-key halves), one lane per half: lane j resolves half
    // j % 2 of DT db + j / 2 (tile list entry, bitmap window), writes its part of the DT's
    // record into the metadata ring, and issues its K loads.
    uint32_t U = 0, M = 0;  // halves issued, DT records written
    const Item* plans = reinterpret_cast<const Item*>(p.plans);
    auto slot_wait = [&](uint32_t mm) {
      WAITP(0, tc::mbar_wait_sleepy(m_empty + int(mm % kMetaSlots),
                                    ((mm / kMetaSlots) & 1) ^ 1, LCX_TC_SLEEPY));
    };
    // items come from a global queue (ascending, so neighbouring CTAs work on neighbouring
    // row blocks of a head and share their K / V tiles in L2)
    auto next_item = [&]() -> int {
      int v = 0;
      if (lane == 0) v = atomicAdd(p.item_counter, 1);
      return __shfl_sync(0xffffffffu, v, 0);
    };
    for (int item = next_item(); item < p.nitems; item = next_item()) {
      const Item it = plans[item];
      if (it.ndt == 0) {
        slot_wait(M);
        DtMeta& mt = metas[M % kMetaSlots];
        if (lane == 0) {
          mt.kind = T_EMPTY;
          mt.flags = F_FIRST | F_LAST;
          mt.h = it.h;
          mt.i0 = it.i0;
          mt.rend = it.rend;
          mt.nsub = 0;
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(m_full + int(M % kMetaSlots));
        ++M;
        continue;
      }
      for (int db = 0; db < it.ndt; db += 2) {
        const int nd = min(2, it.ndt - db);
        // A: lane j < 4 -> DT d = db + j / 2, half s = j % 2: its pattern group x, the
        // group's first tile and DT indices, the DT's half count
        const int d = db + (lane >> 1), s = lane & 1;
        int x = 0, dl = d, tb = 0, ngt = 0;
#pragma unroll
        for (int y = 0; y < 3; ++y) {
          if (y >= it.ng) break;
          ngt = it.grp[y].nvt + it.grp[y].nst;
          const int ndy = (ngt + 1) >> 1;
          x = y;
          if (dl < ndy) break;
          dl -= ndy;
          tb += ngt;
        }
        const int nsub = min(2, ngt - 2 * dl);
        const bool live = lane < 2 * nd && d < it.ndt;
        const bool valid = live && s < nsub;
        Tile my{};
        my.kind = -1;
        if (valid) my = get_tile(p, it, tb + 2 * dl + s);
        // B: the half's record (SLASH: the 256-bit diagonal window and vertical mask)
        uint32_t swv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint64_t vmask = 0;
        int64_t sbase = 0;
        if (valid && my.kind == T_SLASH) {
          const int64_t lo = it.i0 - my.key0 - 63;
          const int64_t wbase = lo >= 0 ? (lo >> 5) : -((-lo + 31) >> 5);
          sbase = wbase * 32;
          const uint32_t* sb = p.sbits + int64_t(it.h) * p.words;
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const int64_t wi = wbase + w;
            swv[w] = (wi >= 0 && wi < p.words) ? sb[wi] : 0u;
          }
          const uint32_t* vb = p.vbits + int64_t(it.h) * p.words;
          const int64_t kw = my.key0 >> 5;
          const uint32_t v0 = kw < p.words ? vb[kw] : 0u;
          const uint32_t v1 = kw + 1 < p.words ? vb[kw + 1] : 0u;
          vmask = uint64_t(v0) | (uint64_t(v1) << 32);
        }
        // C: the batch's ring slots, then every lane writes its part
        for (int j = 0; j < nd; ++j) slot_wait(M + j);
        if (live) {
          DtMeta& mt = metas[(M + (lane >> 1)) % kMetaSlots];
          if (s == 0) {
            int flags = 0;
            if (d == 0) flags |= F_FIRST;
            if (dl == 0) flags |= F_EPOCH;
            const int ndx = (ngt + 1) >> 1;
            if (d + 1 == it.ndt) flags |= F_LAST;
            else if (dl + 1 == ndx) flags |= F_EPOCH_AFTER;
            mt.kind = T_TILES;
            mt.flags = flags;
            mt.pattern = grp_pattern(it, x);
            mt.next_pattern = (flags & F_EPOCH_AFTER) ? grp_pattern(it, x + 1) : 0;
            mt.h = it.h;
            mt.nsub = nsub;
            mt.i0 = it.i0;
            mt.rend = it.rend;
          }
          if (valid) {
            SubMeta& sm = mt.sub[s];
            sm.kind = my.kind;
            sm.count = my.count;
            sm.key0 = my.key0;
            sm.sbase = sbase;
            sm.vmask = vmask;
            if (my.kind == T_SLASH) {
#pragma unroll
              for (int w = 0; w < 8; ++w) sm.sw[w] = swv[w];
            }
          }
        }
        // vertical halves' key lists, warp-wide
        for (int j = 0; j < 2 * nd; ++j) {
          if (__shfl_sync(0xffffffffu, my.kind, j) != T_VERT) continue;
          const long long key0j = __shfl_sync(0xffffffffu, (long long)my.key0, j);
          const int countj = __shfl_sync(0xffffffffu, my.count, j);
          const int32_t* c = p.ckeys + int64_t(it.h) * p.capp + key0j;
          const int32_t k0 = lane < countj ? c[lane] : -1;
          const int32_t k1 = lane + 32 < countj ? c[lane + 32] : -1;
          SubMeta& sm = metas[(M + (j >> 1)) % kMetaSlots].sub[j & 1];
          sm.keys[lane] = k0;
          sm.keys[lane + 32] = k1;
          const unsigned f0 = __ballot_sync(0xffffffffu, k0 >= 0 && int64_t(k0) < it.i0);
          const unsigned f1 = __ballot_sync(0xffffffffu, k1 >= 0 && int64_t(k1) < it.i0);
          if (lane == 0) sm.nfar = __popc(f0) + __popc(f1);
        }
        // D: publish (lane 2 k: DT db + k), then each valid lane issues its half's K loads
        // (halves in stream order: DT db's, then DT db + 1's)
        __syncwarp();
        if (live && s == 0) tc::mbar_arrive(m_full + int((M + (lane >> 1)) % kMetaSlots));
        const int nsub0 = __shfl_sync(0xffffffffu, nsub, 0);
        const int nsub1 = nd > 1 ? __shfl_sync(0xffffffffu, nsub, 2) : 0;
        if (valid) {
          const uint32_t Uj = U + ((lane >> 1) ? nsub0 : 0) + s;
          const int bk = Uj % NK;
          WAITP(1, tc::mbar_wait_sleepy(k_empty + bk, ((Uj / NK) & 1) ^ 1, LCX_TC_SLEEPY));
          tc::mbar_expect_tx(k_full + bk, kKStage);
          const uint32_t kdst = smem_base + OFF_K + bk * kKStage;
          const int64_t tile = my.kind == T_VERT
                                   ? (int64_t(it.h) * (p.capp / 64) + my.key0 / 64) * 2
                                   : (int64_t(it.g) * p.ntiles_k + my.key0 / 64) * 2;
          // pre-swizzled tiles: hi (2 halves) and lo are one contiguous 16 KB run each
          const __nv_bfloat16* sh = my.kind == T_VERT ? p.kchi : p.khi;
          const __nv_bfloat16* sl = my.kind == T_VERT ? p.kclo : p.klo;
          tc::bulk_load(kdst, sh + tile * (kKHalf / 2), 2 * kKHalf, k_full + bk);
          tc::bulk_load(kdst + 2 * kKHalf, sl + tile * (kKHalf / 2), 2 * kKHalf, k_full + bk);
        }
        __syncwarp();
        M += nd;
        U += nsub0 + nsub1;
      }
    }
    slot_wait(M);
    if (lane == 0) metas[M % kMetaSlots].kind = T_END;
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(m_full + int(M % kMetaSlots));
    ++M;
    if (lane == 0 && p.tile_count)
      atomicAdd(reinterpret_cast<unsigned long long*>(p.tile_count), (unsigned long long)U);
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(0);
  } else if (warp == kWarpMma) {
    // ==================================================== QK issuer ====
    uint32_t T = 0, U = 0, E = 0, M = 0;
    // all 32 lanes run this loop (warp-uniform); one elected lane issues
    const uint64_t dk0 = tc::sdesc_sw128(tc::smem_u32(smem + OFF_K));
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
      const int kind = metas[slot].kind;
      const int flags = metas[slot].flags;
      const int nsub = metas[slot].nsub;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(m_empty + slot);
      ++M;
      if (kind == T_END) break;
      if (kind == T_EMPTY) continue;
      if (flags & F_EPOCH) {  // first DT of a pattern group: its Q is (or will be) rotated
        WAITP(1, tc::mbar_wait(q_ready, E & 1));
        ++E;
      }
      const int bs = T % NS;
      WAITP(3, tc::mbar_wait(s_free + bs, ((T / NS) & 1) ^ 1));  // PV(T - NS) released S/P
      const uint32_t dS = tmem + COL_S + bs * DTN;
      for (int j = 0; j < nsub; ++j) {
        const uint32_t Uj = U + j;
        const int bk = Uj % NK;
        WAITP(2, tc::mbar_wait(k_full + bk, (Uj / NK) & 1));
        tc::tc_fence_after();
        const uint64_t dk = dk0 + ((bk * kKStage) >> 4);
#pragma unroll
        for (int combo = 0; combo < 3; ++combo) {  // hh, hl, lh
          const uint32_t qa = tmem + COL_Q + (combo == 2 ? HD / 2 : 0);
          const uint64_t ka = dk + (combo == 1 ? ((2 * kKHalf) >> 4) : 0);
#pragma unroll
          for (int half = 0; half < 2; ++half)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc::mma_f16_ts_warp(dS + j * BN, qa + half * 32 + kk * 8,
                                  ka + ((half * kKHalf + kk * 32) >> 4), IDESC_QK,
                                  (combo | half | kk) ? 1u : 0u);
        }
        tc::mma_commit_warp(k_empty + bk);
      }
      tc::mma_commit_warp(s_full + bs);
      ++T;
      U += nsub;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(1);
  } else if (warp == kWarpV) {
    // ===================================================== V loads ====
    uint32_t U = 0, M = 0;
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
      const int kind = metas[slot].kind;
      const int h = metas[slot].h;
      const int nsub = metas[slot].nsub;
      const int k0 = metas[slot].sub[0].kind, k1 = metas[slot].sub[1].kind;
      const int64_t key00 = metas[slot].sub[0].key0, key01 = metas[slot].sub[1].key0;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(m_empty + slot);
      ++M;
      if (kind == T_END) break;
      if (kind == T_EMPTY) continue;
      if (lane == 0) {
        for (int j = 0; j < nsub; ++j) {
          const uint32_t Uj = U + j;
          const int bv = Uj % NV;
          const int kd = j ? k1 : k0;
          const int64_t key0 = j ? key01 : key00;
          WAITP(1, tc::mbar_wait_sleepy(v_empty + bv, ((Uj / NV) & 1) ^ 1, LCX_TC_SLEEPY));
          tc::mbar_expect_tx(v_full + bv, kVStage);
          const uint32_t vdst = smem_base + OFF_V + bv * kVStage;
          const int64_t vtile = kd == T_VERT ? int64_t(h) * (p.capp / 64) + key0 / 64
                                             : int64_t(h / p.group) * p.ntiles_k + key0 / 64;
          tc::bulk_load(vdst, (kd == T_VERT ? p.vct : p.vt) + vtile * (kVStage / 2), kVStage,
                        v_full + bv);
        }
      }
      __syncwarp();
      U += nsub;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(2);
  } else if (warp == kWarpPv) {
    // ============================================== PV issuer (O += P V) ====
    uint32_t T = 0, U = 0, M = 0;
    const uint64_t dv0 = tc::sdesc_sw128(tc::smem_u32(smem + OFF_V));
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
      const int kind = metas[slot].kind;
      const int flags = metas[slot].flags;
      const int nsub = metas[slot].nsub;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(m_empty + slot);
      ++M;
      if (kind == T_END) break;
      if (kind == T_EMPTY) continue;
      const int bs = T % NS;
      WAITP(1, tc::mbar_wait(p_full + bs, (T / NS) & 1));
      // the first PV of an item overwrites O (a key-window pass > 0 restored the running O
      // into TMEM before the item's first P was released)
      const bool first = (flags & F_FIRST) && !p.init;
      const uint32_t dO = tmem + COL_O;
      for (int j = 0; j < nsub; ++j) {
        const uint32_t Uj = U + j;
        const int bv = Uj % NV;
        WAITP(2, tc::mbar_wait(v_full + bv, (Uj / NV) & 1));
        tc::tc_fence_after();
        const uint64_t dv = dv0 + ((bv * kVStage) >> 4);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)  // P (fp16, 2 per column) aliases S half j
          tc::mma_f16_ts_warp(dO, tmem + COL_S + bs * DTN + j * BN + kk * 8,
                              dv + ((kk * 32) >> 4), IDESC_PV,
                              (first && j == 0 && kk == 0) ? 0u : 1u);
        tc::mma_commit_warp(v_empty + bv);
      }
      tc::mma_commit_warp(s_free + bs);
      ++T;
      U += nsub;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(3);
  } else {
    // ============================= softmax / correction / epilogue ====
    // The two warp groups take the DTs of the stream in turn (group g: DTs T with
    // T % 2 == g); within a group, warp = TMEM lane quadrant and thread = query row with
    // all 128 columns of the DT.  The groups run out of phase -- one computes a DT's max
    // while the other exponentiates the previous one -- and pass the row's running max on
    // per DT through shared memory, signalled on an mbarrier per (group, quadrant).  Each
    // group keeps its own partial row sum l expressed at the max it last used; the owner
    // of an item's last DT combines both (each published before the group's P release) in
    // the epilogue.
    const int wq = warp & 3;       // TMEM lane quadrant
    const int grp = warp >> 2;     // warp group
    const int r = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    float* mbuf = reinterpret_cast<float*>(smem + OFF_RED);  // [kGroups][128] m after DT
    float2* lbuf = reinterpret_cast<float2*>(smem + OFF_RED + kGroups * 128 * 4);
    const tc::SBar h_in = hand + (((grp + kGroups - 1) % kGroups) * 4 + wq);  // predecessor
    const tc::SBar h_out = hand + (grp * 4 + wq);
    uint32_t T = 0, M = 0, T_first = 0;
    float l = 0.f, m_used = -INFINITY;  // this group's partial sum, at max m_used
    float m_init = -INFINITY;           // running max at the item start (key-window passes)
    Item qi{};  // only i0 / rend / h used by rotate_q
    if (grp == kGroups - 1 && lane == 0) tc::mbar_arrive(h_out);  // DT 0 has no predecessor
    auto rotate_row = [&](int pattern) {
      rotate_q(p, qi, pattern, r, 0, tmem + lane_base);
      rotate_q(p, qi, pattern, r, 1, tmem + lane_base);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(q_ready);
    };
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
      const DtMeta& mt = metas[slot];
      const int kind = mt.kind, flags = mt.flags;
      if (kind == T_END) {
        if (T > 0 && (T - 1) % kGroups != uint32_t(grp))
          tc::mbar_wait(lpub + int((T - 1) % kGroups), ((T - 1) / kGroups) & 1);
        break;
      }
      const int64_t i0 = mt.i0, rend = mt.rend;
      const int h = mt.h;
      const int64_t i = i0 + r;
      const bool row_ok = i < rend;
      const bool mine = kind != T_EMPTY && T % kGroups == uint32_t(grp);
      const int nsub = mt.nsub;
      uint64_t mask0 = 0, mask1 = 0;
      if (mine && row_ok) {
        mask0 = sub_mask(mt.sub[0], i);
        if (nsub > 1) mask1 = sub_mask(mt.sub[1], i);
      }
      const int pattern = mt.pattern, next_pattern = mt.next_pattern;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(m_empty + slot);
      ++M;
      if (kind == T_EMPTY) {
        if (grp == 0 && row_ok && !p.init) {  // init passes keep the running state
          float4* o = reinterpret_cast<float4*>(p.out + (i * p.hq + h) * int64_t(HD));
          for (int x = 0; x < 32; ++x) o[x] = make_float4(0.f, 0.f, 0.f, 0.f);
          p.lse[int64_t(h) * p.lse_stride + i] = -INFINITY;
        }
        continue;
      }
      if (flags & F_FIRST) {  // every group starts the item (partial sums, Q rotation rows)
        l = 0.f;
        m_used = -INFINITY;
        T_first = T;
        qi.i0 = i0;
        qi.rend = rend;
        qi.h = h;
      }
      if (!mine) {
        ++T;
        continue;
      }
      const uint32_t k = T / kGroups;  // this group's DT index (hand-off phase)
      if (flags & F_FIRST) {
        // the previous item's last DT (T - 1, the other group) finished its epilogue: O is
        // read and S(T - 1) consumed, so O / Q of this CTA's TMEM are free
        WAITP(2, tc::mbar_wait(h_in, k & 1));
        tc::tc_fence_after();
        m_init = -INFINITY;
        if (p.init) {
          // key-window pass > 0: continue from the row's running (o, lse) -- O goes back
          // into TMEM (the previous item's last PV completed before its epilogue read O)
          const float lp = row_ok ? p.lse[int64_t(h) * p.lse_stride + i] : -INFINITY;
          const bool alive = lp != -INFINITY;
          m_init = alive ? lp * 1.4426950408889634f : -INFINITY;
          l = alive ? 1.f : 0.f;
          m_used = m_init;
          const float4* o = reinterpret_cast<const float4*>(p.out + (i * p.hq + h) * int64_t(HD));
#pragma unroll 1
          for (int q4 = 0; q4 < 4; ++q4) {
            float ov[32];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              const float4 v = alive ? o[q4 * 8 + x] : make_float4(0.f, 0.f, 0.f, 0.f);
              ov[4 * x] = v.x;
              ov[4 * x + 1] = v.y;
              ov[4 * x + 2] = v.z;
              ov[4 * x + 3] = v.w;
            }
            tc::tmem_st32(tmem + lane_base + COL_O + q4 * 32, ov);
          }
          tc::tmem_wait_st();
        }
        rotate_row(pattern);
      }
      const int b = T % NS;
      const uint32_t ph = (T / NS) & 1;
      const uint32_t sb = tmem + lane_base + COL_S + b * DTN;  // this row's S / P of the DT
      float sv[64];
      WAITP(1, tc::mbar_wait(s_full + b, ph));
      tc::tc_fence_after();
      // the DT's QKs (and every earlier one) are complete: Q takes the next pattern
      if (flags & F_EPOCH_AFTER) rotate_row(next_pattern);
      // masked logits -> -inf (ex2(-inf) = 0), already in log2 units
      auto load_half = [&](int j, uint64_t mk) {
        tc::tmem_ld32(sb + j * BN, sv);
        tc::tmem_ld32_wait(sb + j * BN + 32, sv + 32);
        tc::tmem_wait_ld_dep32(sv);
        if (!__all_sync(0xffffffffu, mk == ~0ull)) {
          const uint32_t lo = uint32_t(mk), hi = uint32_t(mk >> 32);
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) {
            sv[cc] = ((lo >> cc) & 1u) ? sv[cc] : -INFINITY;
            sv[32 + cc] = ((hi >> cc) & 1u) ? sv[32 + cc] : -INFINITY;
          }
        }
      };
      auto half_max = [&]() -> float {
        float t4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int cc = 0; cc < 64; cc += 8)
#pragma unroll
          for (int u = 0; u < 4; ++u) t4[u] = fmaxf(t4[u], fmaxf(sv[cc + u], sv[cc + 4 + u]));
        return fmaxf(fmaxf(t4[0], t4[1]), fmaxf(t4[2], t4[3]));
      };
      // ---- P = exp2(x - m) in fp16, written over half j's S columns in TMEM: key c ->
      // column c / 2 (two fp16 per 32-bit column).  Packed f32x2 subtract / accumulate
      // (FADD2): half the FP32 instructions per key.  Returns the half's row sum.
      auto exps_store = [&](int j, float m) -> float {
        const float mm = m == -INFINITY ? 0.f : m;
        const float2 nm2 = make_float2(-mm, -mm);
        float2 rs2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t pw[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int c = hf * 32 + 2 * q;
            const float2 x = __fadd2_rn(make_float2(sv[c], sv[c + 1]), nm2);
            const float2 pp = make_float2(ex2(x.x), ex2(x.y));
            rs2 = __fadd2_rn(rs2, pp);
            const __half2 h2 = __floats2half2_rn(pp.x, pp.y);
            pw[q] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          tc::tmem_st16(sb + j * BN + hf * 16, pw);
        }
        return rs2.x + rs2.y;
      };
      auto rescale_o = [&](float f) {
#pragma unroll 1
        for (int q8 = 0; q8 < 8; ++q8) {  // 16 columns at a time: S is still live here
          float ov[16];
          const uint32_t ta = tmem + lane_base + COL_O + q8 * 16;
          tc::tmem_ld16_wait(ta, ov);
#pragma unroll
          for (int x = 0; x < 16; ++x) ov[x] *= f;
          tc::tmem_st16f(ta, ov);
        }
        tc::tmem_wait_st();
      };
      // ---- DT max: half 1 (if any) stays in registers for its exponentials
      load_half(0, mask0);
      float tmax = half_max();
      if (nsub > 1) {
        load_half(1, mask1);
        tmax = fmaxf(tmax, half_max());
      }
      // ---- running max: the previous DT's (other group) unless the item starts here
      if (!(flags & F_FIRST)) WAITP(3, tc::mbar_wait(h_in, k & 1));
      const float m_prev =
          (flags & F_FIRST) ? m_init : mbuf[((T + kGroups - 1) % kGroups) * 128 + r];
      // lazy rescale: the max moves only past a threshold (P <= 2^8 in fp16)
      const bool need = tmax > m_prev + kRescaleThresh;
      const float m = need ? tmax : m_prev;
      mbuf[grp * 128 + r] = m;
      // an item's last DT hands over only after its epilogue (next item's O / Q)
      if (!(flags & F_LAST)) {
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(h_out);
      }
      if (__any_sync(0xffffffffu, need && m_prev != -INFINITY)) {
        // O holds PV up to DT T - 1 at max m_prev: complete it, then rescale
        const uint32_t Tp = T - 1;
        WAITP(4, tc::mbar_wait(s_free + (Tp % NS), (Tp / NS) & 1));
        tc::tc_fence_after();
        rescale_o((need && m_prev != -INFINITY) ? ex2(m_prev - m) : 1.f);
      }
      if (m != m_used) {  // this group's partial sum follows the row max
        if (m_used != -INFINITY) l *= ex2(m_used - m);
        m_used = m;
      }
      float rs;
      if (nsub > 1) {
        rs = exps_store(1, m);
        load_half(0, mask0);  // half 0 again (its S columns are untouched so far)
        rs += exps_store(0, m);
      } else {
        rs = exps_store(0, m);
      }
      tc::tmem_wait_st();
      l += rs;
      // partial (l, m) for the item's epilogue (ordered before the P release below)
      lbuf[((k & 1) * kGroups + grp) * 128 + r] = make_float2(l, m_used);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(p_full + b);
        tc::mbar_arrive(lpub + grp);
      }
      // every phase of the other group's partial-sum barrier is waited on: DT T - 1's here,
      // once this DT's P is out (it was published long before); the CTA's last DT at T_END
      if (T > 0) {
        const uint32_t To = T - 1;
        WAITP(5, tc::mbar_wait(lpub + int(To % kGroups), (To / kGroups) & 1));
      }
      if (flags & F_LAST) {
        // ---- epilogue: add the other group's partial sum, wait for the last PV,
        // normalize, store ----
        float lt = l;
        if (T > T_first) {  // the other group's last DT of this item (T - 1)
          const uint32_t To = T - 1, go = To % kGroups, ko = To / kGroups;
          const float2 lo = lbuf[((ko & 1) * kGroups + go) * 128 + r];
          if (lo.x > 0.f) lt += lo.x * ex2(lo.y - m_used);
        }
        WAITP(6, tc::mbar_wait(s_free + b, ph));  // this item's last PV is complete
        tc::tc_fence_after();
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        float4* o = reinterpret_cast<float4*>(p.out + (i * p.hq + h) * int64_t(HD));
#pragma unroll 1
        for (int q4 = 0; q4 < 4; ++q4) {
          float ov[32];
          tc::tmem_ld32_wait(tmem + lane_base + COL_O + q4 * 32, ov);
          if (row_ok) {
#pragma unroll
            for (int x = 0; x < 8; ++x)
              o[q4 * 8 + x] = make_float4(ov[4 * x] * inv, ov[4 * x + 1] * inv,
                                          ov[4 * x + 2] * inv, ov[4 * x + 3] * inv);
          }
        }
        if (row_ok)
          p.lse[int64_t(h) * p.lse_stride + i] =
              lt > 0.f ? (m_used + log2f(lt)) * 0.69314718055994530942f : -INFINITY;
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(h_out);
      }
      ++T;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    if (wq == 0) WAITP_FLUSH(4 + grp);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == kWarpMma) tc::tmem_dealloc(tmem, kTmemCols);
}

__global__ void plan_items_kernel(const TcParams p, Item* __restrict__ plans) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item == 0 && p.item_counter) *p.item_counter = 0;  // the launch that follows draws from 0
  if (item >= p.nitems) return;
  Item it;
  setup_item(p, item, it);
  plans[item] = it;
}

// ---------------------------------------------------------------- prep --
// K_hi / K_lo [n][hkv][128] bf16 = split(rope(k_j, kpos(j))), kpos = pos_k[j]
// (standard) or j mod s (DCA).
__global__ void k_prep_kernel(const __nv_bfloat16* __restrict__ k, int64_t n, int64_t r0,
                              int64_t r1, int hkv, const int64_t* __restrict__ pos_k,
                              int rel_mode, int64_t s, const float2* __restrict__ rope,
                              __nv_bfloat16* __restrict__ khi, __nv_bfloat16* __restrict__ klo,
                              float2* __restrict__ kf) {
  // pair index over rows [r0, r1)
  const int64_t idx = r0 * hkv * (HD / 2) + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = r1 * hkv * (HD / 2);
  if (idx >= total) return;
  const int pr = int(idx % (HD / 2));
  const int64_t rowhead = idx / (HD / 2);
  const int64_t j = rowhead / hkv;
  const int64_t kp = rel_mode ? (j % s) : (pos_k ? pos_k[j] : j);
  const float2 xy = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(k)[idx]);
  const float2 c = rope[kp * (HD / 2) + pr];
  const float rx = xy.x * c.x - xy.y * c.y, ry = xy.x * c.y + xy.y * c.x;
  kf[idx] = make_float2(rx, ry);
  const __nv_bfloat162 h2 = __floats2bfloat162_rn(rx, ry);
  const float2 hf = __bfloat1622float2(h2);
  // tiled [hkv][n/64][half][64 keys][64 dims]: each TMA box is one contiguous 8 KB block
  const int g = int(rowhead % hkv);
  const int64_t nt = (n + 63) / 64;
  const int d = 2 * pr;
  const int jr = int(j % 64), dd = d % 64;
  const int64_t o = ((((int64_t(g) * nt + j / 64) * 2 + d / 64) * 64 + jr) * 64 +
                     sw128_chunk(jr, dd / 8) * 8 + dd % 8) / 2;
  reinterpret_cast<__nv_bfloat162*>(khi)[o] = h2;
  reinterpret_cast<__nv_bfloat162*>(klo)[o] = __floats2bfloat162_rn(rx - hf.x, ry - hf.y);
}

// V^T [hkv][128][npad] fp16 from V [n][hkv][128] bf16 (smem-tiled transpose)
__global__ void vt_prep_kernel(const __nv_bfloat16* __restrict__ v, int64_t n, int64_t tile0,
                               int hkv, int64_t npad, __half* __restrict__ vt) {
  __shared__ __half tile[64][HD + 8];
  const int g = blockIdx.y;
  const int64_t jt = tile0 + blockIdx.x;
  const int64_t j0 = jt * 64;
  for (int x = threadIdx.x; x < 64 * HD; x += blockDim.x) {
    const int jj = x / HD, d = x % HD;
    const int64_t j = j0 + jj;
    tile[jj][d] = j < n ? __float2half(__bfloat162float(v[(j * hkv + g) * HD + d])) : __half(0.f);
  }
  __syncthreads();
  const int64_t nt = npad / 64;
  __half* dst = vt + (int64_t(g) * nt + jt) * (HD * 64);  // [128 dims][64 keys]
  for (int x = threadIdx.x; x < 64 * HD; x += blockDim.x) {
    const int d = x / 64, jj = x % 64;
    dst[d * 64 + sw128_chunk(d, jj / 8) * 8 + jj % 8] = tile[jj][d];
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
                               const int32_t* __restrict__ vfirst, int64_t nt,
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
  const int64_t ct = capp / 64;
  for (int x = threadIdx.x; x < 64 * (HD / 8); x += blockDim.x) {
    const int cc = x / (HD / 8), ch = x % (HD / 8);
    uint4 a = make_uint4(0, 0, 0, 0), b = a, vv = a;
    const int32_t j = keys[cc];
    const int half = ch / 8, c8 = ch % 8;
    if (j >= 0) {
      const int64_t src = (((int64_t(g) * nt + j / 64) * 2 + half) * 64 + j % 64) * 64 +
                          sw128_chunk(j % 64, c8) * 8;
      a = *reinterpret_cast<const uint4*>(khi + src);
      b = *reinterpret_cast<const uint4*>(klo + src);
      vv = reinterpret_cast<const uint4*>(v + (int64_t(j) * hkv + g) * HD)[ch];
    }
    const int64_t dst =
        (((int64_t(h) * ct + blockIdx.x) * 2 + half) * 64 + cc) * 64 + sw128_chunk(cc, c8) * 8;
    *reinterpret_cast<uint4*>(kchi + dst) = a;
    *reinterpret_cast<uint4*>(kclo + dst) = b;
    const __nv_bfloat16* vbf = reinterpret_cast<const __nv_bfloat16*>(&vv);
#pragma unroll
    for (int k = 0; k < 8; ++k) tile[cc][ch * 8 + k] = __float2half(__bfloat162float(vbf[k]));
  }
  __syncthreads();
  __half* vdst = vct + (int64_t(h) * ct + blockIdx.x) * (HD * 64);  // [128 dims][64 slots]
  for (int x = threadIdx.x; x < 64 * HD; x += blockDim.x) {
    const int d = x / 64, cc = x % 64;
    vdst[d * 64 + sw128_chunk(d, cc / 8) * 8 + cc % 8] = tile[cc][d];
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
    const int64_t u_lo = -((d + 63) >> 6) - 1;  // rows [0, 128) meet at most 3 tiles
    for (int64_t u = u_lo; u <= u_lo + 4 && u <= 1; ++u) {
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
  // CUDA-core segments, one list per 64-row half of the block: for every diagonal d the
  // rows of the half whose key lands in a non-tcgen05 relative tile form one contiguous
  // range (a half spans at most two relative tiles).  The hist array doubles as the
  // class lookup.
  for (int hf = 0; hf < 2; ++hf) {
    int sbase = 0;
    for (int s0 = 0; s0 < cnt || s0 == 0; s0 += blockDim.x) {
      const int x = s0 + threadIdx.x;
      int4 sg = make_int4(0, 0, 0, 0);
      int nsg = 0;
      if (x < cnt) {
        const int64_t d = sl[x];
        int cur0 = -1, cur1 = -1;
        const int64_t u_lo = -((d + 63) >> 6) - 1;
        for (int64_t u = u_lo; u <= u_lo + 4 && u <= 1; ++u) {
          const int64_t r0 = lcx_max64(64 * hf, d + 64 * u);
          const int64_t r1 = lcx_min64(64 * hf + 64, d + 64 * u + 64);
          if (r1 <= r0) continue;
          const int64_t idx = 1 - u;
          const bool tcu = idx >= 0 && idx < U && hist[idx] >= min_entries && hist[idx] > 0;
          if (tcu) continue;
          if (cur0 < 0) cur0 = int(r0);
          cur1 = int(r1);  // non-TC pieces of one half are adjacent
        }
        if (cur0 >= 0) {
          sg = make_int4(int(d), cur0, cur1, 0);
          nsg = 1;
        }
      }
      const int pos = scan(nsg);
      const int tot = total;
      if (nsg && sbase + pos < cap_seg)
        segs[(int64_t(h) * 2 + hf) * cap_seg + sbase + pos] = sg;
      sbase += tot;
      if (s0 + int(blockDim.x) >= cnt) break;
    }
    if (threadIdx.x == 0) nseg[h * 2 + hf] = int32_t(sbase < cap_seg ? sbase : cap_seg);
    __syncthreads();
  }
}

// Per key window w = [w W, (w+1) W): 1 if some head has a tcgen05 slash tile or a
// CUDA-core segment whose keys meet it for some row of the chunk [t0, t1) (relative tile
// u covers keys [t0 + 64u, t1 + 64u); segment (d, r0, r1) of half h keys
// [t0 + 64h + r0 - d, t1 - d)), so passes over empty windows exit at once.
__global__ void window_flags_kernel(const int32_t* __restrict__ tc_u,
                                    const int32_t* __restrict__ n_tc_u, int64_t cap_u,
                                    const int4* __restrict__ segs, const int32_t* __restrict__ nseg,
                                    int64_t cap_seg, int64_t t0, int64_t t1, int64_t W, int nwin,
                                    int* __restrict__ tc_flags, int* __restrict__ g_flags) {
  const int h = blockIdx.x;
  auto mark = [&](int* f, int64_t lo, int64_t hi) {  // keys [lo, hi)
    lo = lcx_max64(lo, 0);
    hi = lcx_min64(hi, t1);
    if (hi <= lo) return;
    for (int64_t w = lo / W; w <= (hi - 1) / W && w < nwin; ++w) f[w] = 1;
  };
  const int nu = n_tc_u[h];
  for (int x = threadIdx.x; x < nu; x += blockDim.x) {
    const int64_t u = tc_u[int64_t(h) * cap_u + x];
    mark(tc_flags, t0 + 64 * u, t1 + 64 * u + 64);
  }
  for (int hf = 0; hf < 2; ++hf) {
    const int ns = nseg[h * 2 + hf];
    for (int x = threadIdx.x; x < ns; x += blockDim.x) {
      const int4 e = segs[(int64_t(h) * 2 + hf) * cap_seg + x];
      mark(g_flags, t0 + e.y - e.x, t1 - e.x);
    }
  }
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

int make_map3(CUtensorMap* m, CUtensorMapDataType dt, void* base, uint64_t d0, uint64_t d1,
              uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0,
              uint32_t b1, uint32_t b2) {
  return make_tmap3(m, dt, base, d0, d1, d2, stride1_bytes, stride2_bytes, b0, b1, b2);
}

}  // namespace

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

int make_tmap3(CUtensorMap* m, CUtensorMapDataType dt, void* base, uint64_t d0, uint64_t d1,
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


// ------------------------------------------------------------ host API --
int tc_prepare_rows(const void* k, const void* v, int64_t n, int64_t r0, int64_t r1, int hkv,
                    const int64_t* pos_k, int rel_mode, int64_t s, const float2* rope,
                    const TcBuffers& B, cudaStream_t st) {
  r1 = lcx_min64(r1, n);
  if (r1 <= r0) return LCX_OK;
  const int64_t pairs = (r1 - r0) * hkv * (HD / 2);
  k_prep_kernel<<<unsigned((pairs + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(k), n, r0, r1, hkv, pos_k, rel_mode, s, rope, B.khi,
      B.klo, reinterpret_cast<float2*>(B.kf));
  LCX_CHECK_LAUNCH();
  // V^T tiles covering [r0, r1); a partial trailing tile is rewritten (zero-padded) by the
  // range that completes it, so ranges must be handed in ascending order
  const int64_t tile0 = r0 / 64, tile1 = r1 == n ? B.npad / 64 : (r1 + 63) / 64;
  vt_prep_kernel<<<dim3(unsigned(tile1 - tile0), unsigned(hkv)), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(v), r1, tile0, hkv, B.npad, B.vt);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int tc_prepare_maps(int hq, int hkv, TcBuffers& B) {
  const int64_t capp = B.capp;
  if (capp >= (int64_t(1) << 31)) return fail(LCX_ERR_DIMENSION, "vertical capacity too large");
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, F16 = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const uint64_t nt = uint64_t(B.npad / 64), ct = uint64_t(capp / 64);
  // tiled operands: every box is one contiguous block (8 KB K half-tile, 16 KB V^T tile)
  LCX_TRY(make_map3(&B.m_khi, BF, B.khi, 64, 64, hkv * nt * 2, 128, 8192, 64, 64, 1));
  LCX_TRY(make_map3(&B.m_klo, BF, B.klo, 64, 64, hkv * nt * 2, 128, 8192, 64, 64, 1));
  LCX_TRY(make_map3(&B.m_vt, F16, B.vt, 64, HD, hkv * nt, 128, 16384, 64, HD, 1));
  LCX_TRY(make_map3(&B.m_kchi, BF, B.kchi, 64, 64, hq * ct * 2, 128, 8192, 64, 64, 1));
  LCX_TRY(make_map3(&B.m_kclo, BF, B.kclo, 64, 64, hq * ct * 2, 128, 8192, 64, 64, 1));
  LCX_TRY(make_map3(&B.m_vct, F16, B.vct, 64, HD, hq * ct, 128, 16384, 64, HD, 1));
  return LCX_OK;
}

int tc_prepare(const void* k, const void* v, int64_t n, int hq, int hkv, const int64_t* pos_k,
               int rel_mode, int64_t s, const float2* rope, TcBuffers& B, cudaStream_t st) {
  LCX_TRY(tc_prepare_maps(hq, hkv, B));
  return tc_prepare_rows(k, v, n, 0, n, hkv, pos_k, rel_mode, s, rope, B, st);
}

int tc_compact(const void* v, int hq, int hkv, const int32_t* verts, const int32_t* nv,
               int64_t cap_v, TcBuffers& B, cudaStream_t st) {
  vseg_kernel<<<hq, 1, 0, st>>>(verts, nv, cap_v, B.seg_len, B.nseg_k, B.vbase, B.vfirst);
  LCX_CHECK_LAUNCH();
  dim3 grid(unsigned(B.capp / 64), unsigned(hq));
  compact_kernel<<<grid, 256, 0, st>>>(B.khi, B.klo, reinterpret_cast<const __nv_bfloat16*>(v),
                                       hkv, hq / hkv, verts, nv, cap_v, B.capp, B.nseg_k, B.vbase,
                                       B.vfirst, B.npad / 64, B.kchi, B.kclo, B.vct, B.ckeys);
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

size_t tc_plan_bytes() { return sizeof(Item); }

int tc_window_flags(const int32_t* tc_u, const int32_t* n_tc_u, int64_t cap_u, const int4* segs,
                    const int32_t* nseg, int64_t cap_seg, int hq, int64_t t0, int64_t t1,
                    int64_t W, int nwin, int* tc_flags, int* g_flags, cudaStream_t st) {
  LCX_CHECK_CUDA(cudaMemsetAsync(tc_flags, 0, sizeof(int) * nwin, st));
  LCX_CHECK_CUDA(cudaMemsetAsync(g_flags, 0, sizeof(int) * nwin, st));
  window_flags_kernel<<<hq, 256, 0, st>>>(tc_u, n_tc_u, cap_u, segs, nseg, cap_seg, t0, t1, W,
                                          nwin, tc_flags, g_flags);
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
  if (!p.item_counter) return fail(LCX_ERR_INTERNAL, "tcgen05 attention needs an item counter");
  const int grid = std::min(p.nitems, sm_count);
  plan_items_kernel<<<(p.nitems + 127) / 128, 128, 0, st>>>(p, reinterpret_cast<Item*>(p.plans));
  LCX_CHECK_LAUNCH();
  TcParams q = p;
  q.khi = B.khi;
  q.klo = B.klo;
  q.kchi = B.kchi;
  q.kclo = B.kclo;
  q.vt = B.vt;
  q.vct = B.vct;
  attn_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(q);
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
