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
// Warp roles (352 threads, merged configuration, control warps at the lowest ids):
// warp 0 metadata producer (tile records into a 16-slot shared ring), warp 1 MMA issuer
// (QK(T) on three bf16 products with Q hi/lo resident in TMEM, then PV(T - 2)) + TMEM owner,
// warp 2 K / V^T loader (1-D bulk copies of pre-swizzled tiles), warps 3-10 softmax /
// correction / epilogue in two groups of four that take alternate tiles and read only their
// own ring slots (thread = query row, TMEM lane quadrant = warp % 4).  Pipelines: K (hi+lo)
// and V^T in four shared-memory stages, S in four TMEM buffers of 64 columns with P (fp16)
// written over it, O in TMEM (128 columns), one rotated-Q buffer (hi/lo) re-rotated at DCA
// pattern changes.  Design notes and measurements: DESIGN.md §4.
#include <cuda.h>

#include "lcx_internal.cuh"
#include "tc_ptx.cuh"
#include "attn_tc.cuh"

namespace lcx {



namespace {

constexpr int BM = 128, BN = 64, HD = 128;
// warps 0-7 softmax (TMEM lane quadrant = warp % 4, group = warp / 4),
// warp 8 producer (tile metadata + K TMA), warp 9 QK issuer + TMEM allocator,
// warp 10 PV issuer, warp 11 V TMA
#ifndef LCX_TC_GROUPS
#define LCX_TC_GROUPS 2
#endif
constexpr int kGroups = LCX_TC_GROUPS;          // softmax warp groups (tile T: T % kGroups)
constexpr int kSoftmaxWarps = 4 * kGroups;
// One warp issues both the QK and the PV MMAs (QK(T), then PV(T - 1); PV first at an item
// start) and the producer warp issues the V loads after the K loads of each tile: two fewer
// warps polling barriers (the kernel is issue-bound: ~20 % of its instructions were
// barrier polls), and the sub-partitions they free run only softmax warps.
#ifndef LCX_TC_MERGE
#define LCX_TC_MERGE 1
#endif
constexpr bool kMerge = LCX_TC_MERGE;
// With kMerge the producer warp only builds the tile metadata (running up to the ring's
// depth ahead) and a loader warp issues each tile's K and V^T loads as stages free up: the
// metadata of the next tiles no longer waits behind a stage-empty wait.
#ifndef LCX_TC_MMA_WARP3  // experiment: MMA warp on sub-partition 3 (warp 11), warp 9 idle
#define LCX_TC_MMA_WARP3 0
#endif
// LCX_TC_QK2: the QK MMAs of odd tiles are issued by a second warp on another sub-partition
// (a tcgen05.mma holds its sub-partition's dispatch while it is accepted, so the 24 QK
// MMAs of every tile starved the softmax warp beside the one issuer); PVs stay on the first.
#ifndef LCX_TC_QK2
#define LCX_TC_QK2 0  // measured: 330 vs 322 ms per 1M layer with the own-slot softmax
#endif
constexpr bool kQk2 = LCX_TC_QK2 && kMerge;
// LCX_TC_PRODUCER_LOADS (experiment): the producer issues each batch's K and V loads itself
// (no loader warp), so only the MMA issuer shares a sub-partition with softmax warps
#ifndef LCX_TC_PRODUCER_LOADS
#define LCX_TC_PRODUCER_LOADS 0
#endif
constexpr bool kProdLoads = LCX_TC_PRODUCER_LOADS && kMerge;
// LCX_TC_KV_LOADERS: K and V^T loads from two warps, so a K load never waits behind a V
// stage release (which follows the PV two tiles behind)
#ifndef LCX_TC_KV_LOADERS
#define LCX_TC_KV_LOADERS 0
#endif
constexpr bool kKvLoaders = LCX_TC_KV_LOADERS && kMerge && !kProdLoads && !LCX_TC_QK2;
constexpr int kThreads =
    32 * (kSoftmaxWarps + (kMerge && !LCX_TC_MMA_WARP3 && !kQk2 && !kKvLoaders ? 3 : 4));
constexpr bool kLoaderWarp = kMerge && !kProdLoads;
// Warp ids: each sub-partition's scheduler issues from its highest-id eligible warp first,
// so a softmax warp with a lower id than a control warp of its sub-partition is starved
// whenever that warp is eligible -- and the group that owns it runs at its pace (the
// softmax warp beside the MMA warp lagged its group by ~2000 clk per tile).  With
// LCX_TC_CTRL_FIRST the control warps take the lowest ids and the softmax warps follow.
#ifndef LCX_TC_CTRL_FIRST
#define LCX_TC_CTRL_FIRST 1
#endif
constexpr int kCtrlWarps = kThreads / 32 - kSoftmaxWarps;
constexpr int kSmBase = (LCX_TC_CTRL_FIRST && kMerge) ? kCtrlWarps : 0;  // first softmax warp
constexpr int kCtrlBase = (LCX_TC_CTRL_FIRST && kMerge) ? 0 : kSoftmaxWarps;
constexpr int kWarpProducer = kCtrlBase,
              kWarpMma = LCX_TC_MMA_WARP3 ? kCtrlBase + 3 : kCtrlBase + 1,
              kWarpPv = kMerge ? -1 : kCtrlBase + 2, kWarpV = kMerge ? -1 : kCtrlBase + 3,
              kWarpLoad = kLoaderWarp ? kCtrlBase + 2 : -1,
              kWarpMma2 = kQk2 ? kCtrlBase + 3 : -2,
              kWarpLoadV = kKvLoaders ? kCtrlBase + 3 : -3;
// warps reading each ring slot: one softmax group (slots alternate between the groups) and
// every control warp but the producer
constexpr int kRingConsumers =
    4 + (kMerge ? (kQk2 || kKvLoaders ? 3 : 2) - (kProdLoads ? 1 : 0) : 3);
// The softmax code is written for any number of groups, but a third group needs more
// registers than 65536 / 512 per thread: compiled at 128 it spills ~2.6 KB and ran 3.4x
// slower (setmaxnreg does not help: ptxas still allocates for the launch-time limit).
// With a third group each thread keeps only 32 logits live (kSReread): S is read from
// TMEM twice, once for the tile max and once for the exponentials.
#ifndef LCX_TC_SREREAD
#define LCX_TC_SREREAD (LCX_TC_GROUPS > 2)
#endif
constexpr bool kSReread = LCX_TC_SREREAD;
// Three groups fit in 128 registers this way and are correct (with NS = 3, below), but
// measure slower than two: 397 vs 364 ms per 1M layer on one box (one Q buffer, S read
// twice, spills) -- kept behind LCX_TC_ALLOW_GROUPS3.
#ifndef LCX_TC_ALLOW_GROUPS3
static_assert(kGroups == 2, "two softmax groups");
#endif
// two S buffers suffice (NS = 2, 3, 4 measure the same); the TMEM they free holds a
// second rotated Q, so the Q of the next DCA pattern is in place before its first QK
#ifndef LCX_TC_QBUFS
// one Q buffer and four S buffers: with the merged MMA warp issuing PV(T - 2) after QK(T),
// the QK of the next tiles runs ahead of the softmax (two Q buffers leave room for two S
// buffers only, and QK(T + 2) then waits for PV(T)): 342-344 vs 351-354 ms per 1M layer
#define LCX_TC_QBUFS 1
#endif
// two rotated-Q buffers with two S buffers, or one Q buffer with four S buffers
// Split O (LCX_TC_SPLIT_O): each softmax group accumulates its own tiles into its own O
// in TMEM, at its own running max, and the two are merged in the item's epilogue -- the
// groups no longer hand the running max to each other tile by tile.  TMEM then holds
// two S buffers, two O and one rotated-Q buffer.
#ifndef LCX_TC_SPLIT_O
#define LCX_TC_SPLIT_O 0
#endif
constexpr bool kSplitO = LCX_TC_SPLIT_O;
// split O: exponentiate at the group's running max before the tile max is known (correct,
// measured 2 % slower than max-first: 376 vs 369 ms per layer on one box)
#ifndef LCX_TC_SPEC_EXP
#define LCX_TC_SPEC_EXP 0
#endif
constexpr bool kSpecExp = LCX_TC_SPEC_EXP;
// A softmax group waits for S(T) on buffer T % NS with a phase parity; that is only
// sound if the group itself observed the buffer's previous phase (tile T - NS), i.e. if
// NS is a multiple of the group count -- three groups take three S buffers and one Q.
constexpr int kQBufs = (kSplitO || kGroups == 3) ? 1 : LCX_TC_QBUFS;
constexpr int kOBufs = kSplitO ? kGroups : 1;
constexpr int NK = 4, NV = 4;  // K / V smem stages
constexpr int NS = kGroups == 3 ? 3 : ((kSplitO || kQBufs == 2) ? 2 : 4);  // S (+P) TMEM
static_assert(NS % kGroups == 0, "each group must see every phase of its S buffers");

static_assert(!kSplitO || NS == kGroups, "split O: S(T) full implies PV(T - kGroups) done");
constexpr uint32_t kKHalf = BN * 64 * 2;             // 8 KB
constexpr uint32_t kKStage = 4 * kKHalf;             // hi0 hi1 lo0 lo1 = 32 KB
constexpr uint32_t kVStage = HD * BN * 2;            // 16 KB
constexpr uint32_t OFF_K = 0;
constexpr uint32_t OFF_V = OFF_K + NK * kKStage;     // 128 KB
constexpr uint32_t OFF_BAR = OFF_V + NV * kVStage;   // 192 KB
constexpr uint32_t OFF_META = OFF_BAR + 1024;
constexpr int kMetaSlots = 16;                      // tile metadata ring (448 B slots)
// softmax hand-off area: running max per tile parity [2][128], partial sums
// (l, m) [2 slot][2 warp group][128]
constexpr uint32_t OFF_RED = OFF_META + kMetaSlots * 448;
// softmax exchange: running max per group [kGroups][128], partial sums (l, m)
// [2 slot][kGroups][128]
constexpr uint32_t kSmemBytes =
    OFF_RED + kGroups * 128 * 4 + 2 * kGroups * 128 * 8 + 1024;  // + align slack
// TMEM (512 columns x 128 lanes): S/P buffers [0, 128), O [128, 256), two rotated Q
// buffers [256, 384) and [384, 512) (hi, then lo; bf16 pairs per 32-bit column) as
// the A operand of every QK MMA, so all MMAs read only B from shared memory.  DCA
// pattern group x of an item uses Q buffer x & 1.
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t COL_O = NS * BN;
constexpr uint32_t COL_Q = COL_O + kOBufs * HD;  // Q buffer b: hi at COL_Q + 128 b, lo at + 64
static_assert(COL_Q + kQBufs * HD <= 512, "TMEM columns");
constexpr uint32_t QBUF = HD;
constexpr float kRescaleThresh = 8.f;
// producer / V-load warps: sleepy polling (ns between polls) instead of suspended
// try_wait, 0 = off.  A suspended waiter is woken by other barriers' traffic and
// re-polls: ncu counts ~700 warp instructions per tile in wait loops, taken from the
// softmax warps' sub-partitions.  Same-box A/B (attn_tc ms per 1M layer): off 363 /
// 360, 30 ns 361-363, 100 ns 359-361, 300 ns 357-358, 1000 ns 357-360, 3000 ns 374;
// the PV issuer's wait for P (critical path) at 40 ns: 363.
#ifndef LCX_TC_SLEEPY
#define LCX_TC_SLEEPY 300
#endif
// QK / PV MMAs issued eight / four per asm block (one elect, offsets added in PTX)
#ifndef LCX_TC_MMA_X8
#define LCX_TC_MMA_X8 0
#endif
#ifndef LCX_TC_MMA_DEPTH  // MMA products in flight before the issuer waits (0: no throttle)
#define LCX_TC_MMA_DEPTH 0
#endif
constexpr int kMmaDepth = LCX_TC_MMA_DEPTH;
static_assert(kMmaDepth >= 0 && kMmaDepth <= 4, "throttle ring of 4");
#ifndef LCX_TC_SLEEPY_MMA  // merged MMA warp's wait for P: ns between polls (0 = try_wait)
#define LCX_TC_SLEEPY_MMA 0
#endif
#ifndef LCX_TC_SLEEPY_LOAD  // loader warp's stage-empty waits
#define LCX_TC_SLEEPY_LOAD 0
#endif
#ifndef LCX_TC_SLEEPY_PV  // the PV issuer's wait for P (on the critical path)
#define LCX_TC_SLEEPY_PV 0
#endif

// Barrier arrivals on the metadata ring, the running-max hand-off and the partial-sum
// publication: by every lane that touched the shared data (1), or by lane 0 after a
// __syncwarp (0; the warp barrier orders the other lanes' accesses, but racecheck does
// not credit it and reports those accesses as hazards).
#ifndef LCX_TC_LANE_ARRIVE
#define LCX_TC_LANE_ARRIVE 1
#endif
constexpr uint32_t kArriveLanes = LCX_TC_LANE_ARRIVE ? 32 : 1;
#define LANE_ARRIVE(bar) \
  do {                   \
    if (LCX_TC_LANE_ARRIVE || lane == 0) tc::mbar_arrive(bar); \
  } while (0)

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
  // KV-group-major order: the query heads of one KV head are adjacent for each row block,
  // so CTAs drawing neighbouring items read the same K / V tiles (band, dense) from L2
  // instead of each head re-streaming them from DRAM.
#if defined(LCX_TC_BLOCK_MAJOR)  // experiment: every head of a row block adjacent
  const int b = item / p.hq;
  it.h = item - b * p.hq;
#elif !defined(LCX_TC_HEAD_MAJOR)
  const int per_g = p.nblocks * p.group;
  const int gg = item / per_g;
  const int rem = item - gg * per_g;
  const int b = rem / p.group;
  it.h = gg * p.group + (rem - b * p.group);
#else
  it.h = item / p.nblocks;
  const int b = item - it.h * p.nblocks;
#endif
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
                                         int part, uint32_t tmem_row, int qbuf) {
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
  const uint32_t qc = tmem_row + COL_Q + qbuf * QBUF;
  tc::tmem_st32(qc + part * 32, reinterpret_cast<const float*>(hi));
  tc::tmem_st32(qc + HD / 2 + part * 32, reinterpret_cast<const float*>(lo));
  tc::tmem_wait_st();
}

// Per-tile control record, written by the producer warp into a 4-deep shared
// ring so that the MMA and softmax warps never touch global memory for control.
enum { T_EMPTY = 3, T_END = 4 };
enum { F_FIRST = 1, F_LAST = 2, F_EPOCH = 4, F_EPOCH_AFTER = 8, F_REPEAT = 16 };  // F_REPEAT: a pair's second EMPTY / END slot
struct TileMeta {
  int32_t kind, flags, pattern, next_pattern;
  int32_t h, count, nfar, grp;  // grp: the tile's pattern group within its item
  int32_t gpat[3], ng;          // the item's group patterns and group count
  int32_t item_t0;              // stream index T of the item's first tile
  int32_t item_seq;             // non-empty items this CTA started before this one
  int64_t i0, rend, key0, sbase;
  uint64_t vmask;
  uint32_t sw[8];
  int32_t keys[64];
};
#ifndef LCX_TC_BULK
#define LCX_TC_BULK 1  // 1-D bulk copies of the pre-swizzled tiles (else 3-D tensor TMA)
#endif
[[maybe_unused]] constexpr int kTraceTiles = 512;
// trace columns: 0 meta ready (producer), 1 K TMA issued, 2 V TMA issued,
// 3 QK issued (MMA), 4 PV issued, 5 softmax got S, 6 softmax P written, 7 kind
// pipeline trace (tools/trace_tc.py): compiled in only with -DLCX_TC_TRACE -- the
// per-tile checks cost ~3 % of the kernel's instructions
__device__ __forceinline__ void trace_mark(const TcParams& p, uint32_t T, int col) {
#if defined(LCX_TC_TRACE) && !(defined(LCX_TC_TRACE_Q) && LCX_TC_TRACE_Q == 2)
  if (p.trace && blockIdx.x == 0 && T < kTraceTiles) p.trace[T * 8 + col] = clock64();
#else
  (void)p;
  (void)T;
  (void)col;
#endif
}
static_assert(sizeof(TileMeta) <= 448, "tile metadata slot overflow");
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
#define WAITP2(site, ...)                     \
  do {                                        \
    const long long _w0 = clock64();          \
    __VA_ARGS__;                              \
    wacc2[site] += clock64() - _w0;           \
  } while (0)
#else
#define WAITP(site, ...) __VA_ARGS__
#define WAITP2(site, ...) __VA_ARGS__
#define WAITP_FLUSH(role) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ float ex2(float x) {  // pure: the compiler may schedule it
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t window64(const uint32_t* sw, int off) {
  // bits [off, off + 64) of the 256-bit array sw (off in [0, 192])
  const int w = off >> 5, sh = off & 31;
  const uint64_t a = uint64_t(sw[w]) | (uint64_t(sw[w + 1]) << 32);
  const uint64_t b = (w + 2 < 8) ? sw[w + 2] : 0u;
  return sh ? ((a >> sh) | (b << (64 - sh))) : a;
}

// registers: the register file is split over the four sub-partitions and warps go to them
// round-robin: up to 12 warps put at most 3 on a sub-partition (168 per thread), 13-16 put 4
// (128 per thread)
constexpr int kMaxRegs = (kThreads / 32 + 3) / 4 >= 4 ? 128 : 168;
__global__ void __maxnreg__(kMaxRegs)
attn_tc_kernel(const TcParams p, const __grid_constant__ CUtensorMap map_k_hi,
               const __grid_constant__ CUtensorMap map_k_lo,
               const __grid_constant__ CUtensorMap map_vt,
               const __grid_constant__ CUtensorMap map_kc_hi,
               const __grid_constant__ CUtensorMap map_kc_lo,
               const __grid_constant__ CUtensorMap map_vct) {
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
  const tc::SBar v_empty = v_full + NV;        // [NV] PV commit -> producer
  const tc::SBar s_full = v_empty + NV;        // [NS] QK commit -> softmax
  const tc::SBar s_free = s_full + NS;         // [NS] PV commit (S/P buffer, O updated)
  const tc::SBar p_full = s_free + NS;         // [NS] softmax wrote P -> PV issuer
  const tc::SBar q_ready = p_full + NS;        // [2] softmax rotated Q buffer b -> QK issuer
  const tc::SBar m_full = q_ready + 2;         // [kMetaSlots]
  const tc::SBar m_empty = m_full + kMetaSlots;  // [kMetaSlots]
  const tc::SBar hand = m_empty + kMetaSlots;    // [kGroups][4] running max of a tile ready
  const tc::SBar lpub = hand + 4 * kGroups;      // [kGroups] partial sums of a tile written
  const tc::SBar edone = lpub + kGroups;         // split O: an item's epilogue read both O
  const tc::SBar prog = edone + 1;               // [4] MMA product completions (throttle)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR) +
                        2 * (2 * NK + 2 * NV + 3 * NS + 2 + 2 * kMetaSlots + 5 * kGroups + 5);
  static_assert((2 * NK + 2 * NV + 3 * NS + 2 + 2 * kMetaSlots + 5 * kGroups + 6) * 8 <= 1024,
                "barrier area overflow");
  TileMeta* metas = reinterpret_cast<TileMeta*>(smem + OFF_META);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef LCX_TC_WAITPROF
  long long wacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long wacc2[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // softmax detail (role 5)
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
      tc::mbar_init(p_full + b, 4);  // the tile's warp group
    }
    tc::mbar_init(q_ready, 4);
    tc::mbar_init(q_ready + 1, 4);
    for (int b = 0; b < 4 * kGroups; ++b) tc::mbar_init(hand + b, kArriveLanes);
    for (int b = 0; b < kGroups; ++b) tc::mbar_init(lpub + b, 4 * kArriveLanes);
    tc::mbar_init(edone, 4);
    for (int b = 0; b < 4; ++b) tc::mbar_init(prog + b, 1);
    for (int b = 0; b < kMetaSlots; ++b) {
      tc::mbar_init(m_full + b, 32);  // every producer lane releases its own writes
      tc::mbar_init(m_empty + b, kRingConsumers * kArriveLanes);  // softmax + QK + PV + V warps
    }
    tc::fence_barrier_init();
    tc::fence_proxy_async();
  }
  if (warp == kWarpMma) tc::tmem_alloc(tmem_slot, kTmemCols);
  if (warp == kWarpProducer && lane == 0) {
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

  if (warp == kWarpProducer) {
    // ============================ producer: tile stream + metadata + K loads ====
    // Batches of 4 tiles, one lane per tile: lane j resolves tile j (tile-list entry,
    // bitmap window), waits for nothing but its slot, writes the tile's record into the
    // metadata ring, publishes it and issues its K loads -- the batch's global loads and
    // its four ring slots are all in flight at once.
    uint32_t T = 0, M = 0;
    int32_t item_seq = 0;  // non-empty items started
    const Item* plans = reinterpret_cast<const Item*>(p.plans);
    auto slot_wait = [&](uint32_t mm) {
#if LCX_TC_SLEEPY
      WAITP(0, tc::mbar_wait_sleepy(m_empty + int(mm % kMetaSlots), ((mm / kMetaSlots) & 1) ^ 1,
                                    LCX_TC_SLEEPY));
#else
      WAITP(0, tc::mbar_wait(m_empty + int(mm % kMetaSlots), ((mm / kMetaSlots) & 1) ^ 1));
#endif
    };
    // items come from a global queue (ascending, so neighbouring CTAs still work on
    // neighbouring row blocks of a head and share their K / V tiles in L2) -- CTAs that
    // drew cheap items take more, instead of a fixed round-robin share
    int static_item = int(blockIdx.x);
    auto next_item = [&]() -> int {
      if (!p.item_counter) {
        const int x = static_item;
        static_item += int(gridDim.x);
        return x;
      }
      int v = 0;
      if (lane == 0) v = atomicAdd(p.item_counter, 1);
      return __shfl_sync(0xffffffffu, v, 0);
    };
    for (int item = next_item(); item < p.nitems; item = next_item()) {
      const Item it = plans[item];
      if (it.ntiles == 0) {
        // kGroups slots (one per softmax group: slot ownership is M % kGroups, and tile T
        // keeps T == M mod kGroups); the first slot's group zeroes the rows
        for (int e = 0; e < kGroups; ++e) {
          slot_wait(M);
          TileMeta& mt = metas[M % kMetaSlots];
          if (lane == 0) {
            mt.kind = T_EMPTY;
            mt.flags = (F_FIRST | F_LAST) | (e == 0 ? 0 : F_REPEAT);
            mt.h = it.h;
            mt.i0 = it.i0;
            mt.rend = it.rend;
          }
          __syncwarp();
          tc::mbar_arrive(m_full + int(M % kMetaSlots));
          ++M;
        }
        continue;
      }
      int carry_grp = -1;
      ++item_seq;
      for (int tb = 0; tb < it.ntiles; tb += 4) {
        const int nb = min(4, it.ntiles - tb);
        // A: lane j <= nb resolves tile tb + j (lane nb: the next tile's group)
        Tile my{};
        my.grp = -1;
        my.kind = -1;
        if (lane <= nb && tb + lane < it.ntiles) my = get_tile(p, it, tb + lane);
        const int up_grp = __shfl_up_sync(0xffffffffu, my.grp, 1);
        const int dn_grp = __shfl_down_sync(0xffffffffu, my.grp, 1);
        const int prev_grp = lane == 0 ? carry_grp : up_grp;
        carry_grp = __shfl_sync(0xffffffffu, my.grp, nb - 1);
        // B: lane j < nb builds its tile's record (SLASH: the 256-bit diagonal window)
        const int t = tb + lane;
        int flags = 0, pattern = 0, next_pattern = 0;
        uint32_t swv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint64_t vmask = 0;
        int64_t sbase = 0;
        if (lane < nb) {
          if (t == 0) flags |= F_FIRST;
          if (my.grp != prev_grp) flags |= F_EPOCH;
          if (t + 1 == it.ntiles) flags |= F_LAST;
          else if (dn_grp != my.grp) flags |= F_EPOCH_AFTER;
          pattern = grp_pattern(it, my.grp);
          next_pattern = (flags & F_EPOCH_AFTER) ? grp_pattern(it, dn_grp) : 0;
          if (my.kind == T_SLASH) {
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
        }
        // C: the batch's ring slots, then every lane writes its record; vertical tiles'
        // key lists are written warp-wide
        for (int j = 0; j < nb; ++j) slot_wait(M + j);
        if (lane < nb) {
          TileMeta& mt = metas[(M + lane) % kMetaSlots];
          mt.kind = my.kind;
          mt.flags = flags;
          mt.pattern = pattern;
          mt.next_pattern = next_pattern;
          mt.grp = my.grp;
          mt.gpat[0] = it.grp[0].pattern;
          mt.gpat[1] = it.grp[1].pattern;
          mt.gpat[2] = it.grp[2].pattern;
          mt.ng = it.ng;
          mt.item_t0 = int32_t(T - tb);  // T counts this batch's first tile
          mt.item_seq = item_seq - 1;
          mt.h = it.h;
          mt.count = my.count;
          mt.i0 = it.i0;
          mt.rend = it.rend;
          mt.key0 = my.key0;
          mt.sbase = sbase;
          mt.vmask = vmask;
          if (my.kind == T_SLASH) {
#pragma unroll
            for (int w = 0; w < 8; ++w) mt.sw[w] = swv[w];
          }
        }
        for (int j = 0; j < nb; ++j) {
          if (__shfl_sync(0xffffffffu, my.kind, j) != T_VERT) continue;
          const long long key0j = __shfl_sync(0xffffffffu, (long long)my.key0, j);
          const int countj = __shfl_sync(0xffffffffu, my.count, j);
          const int32_t* c = p.ckeys + int64_t(it.h) * p.capp + key0j;
          const int32_t k0 = lane < countj ? c[lane] : -1;
          const int32_t k1 = lane + 32 < countj ? c[lane + 32] : -1;
          TileMeta& mt = metas[(M + j) % kMetaSlots];
          mt.keys[lane] = k0;
          mt.keys[lane + 32] = k1;
          const unsigned f0 = __ballot_sync(0xffffffffu, k0 >= 0 && int64_t(k0) < it.i0);
          const unsigned f1 = __ballot_sync(0xffffffffu, k1 >= 0 && int64_t(k1) < it.i0);
          if (lane == 0) mt.nfar = __popc(f0) + __popc(f1);
        }
        // D: publish (lane j: slot of tile j), then lane j issues tile j's K loads
        // every lane wrote into the batch's slots (records, vertical key lists): each
        // lane releases its own writes on every slot of the batch (count 32)
        __syncwarp();
        for (int j = 0; j < nb; ++j) tc::mbar_arrive(m_full + int((M + j) % kMetaSlots));
        if (lane < nb) {
          const uint32_t Tj = T + lane;
#if !defined(LCX_TC_TRACE_PV) && !defined(LCX_TC_TRACE_SM)
          trace_mark(p, Tj, 0);
#endif
        }
        if ((!kMerge || kProdLoads) && lane < nb) {
          const uint32_t Tj = T + lane;
          const int bk = Tj % NK;
#if LCX_TC_SLEEPY
          WAITP(1, tc::mbar_wait_sleepy(k_empty + bk, ((Tj / NK) & 1) ^ 1, LCX_TC_SLEEPY));
#else
          WAITP(1, tc::mbar_wait(k_empty + bk, ((Tj / NK) & 1) ^ 1));
#endif
          tc::mbar_expect_tx(k_full + bk, kKStage);
          const uint32_t kdst = smem_base + OFF_K + bk * kKStage;
          int tile = my.kind == T_VERT ? int((int64_t(it.h) * (p.capp / 64) + my.key0 / 64) * 2)
                                       : int((int64_t(it.g) * p.ntiles_k + my.key0 / 64) * 2);
#ifdef LCX_TC_FAKE_LOADS  // timing experiment only: every tile loads from a small L2-resident set
          tile &= 62;
#endif
#if LCX_TC_BULK
          // pre-swizzled tiles: hi (2 halves) and lo are one contiguous 16 KB run each
          const __nv_bfloat16* sh = my.kind == T_VERT ? p.kchi : p.khi;
          const __nv_bfloat16* sl = my.kind == T_VERT ? p.kclo : p.klo;
          tc::bulk_load(kdst, sh + int64_t(tile) * (kKHalf / 2), 2 * kKHalf, k_full + bk);
          tc::bulk_load(kdst + 2 * kKHalf, sl + int64_t(tile) * (kKHalf / 2), 2 * kKHalf,
                        k_full + bk);
#else
          const CUtensorMap* mh = my.kind == T_VERT ? &map_kc_hi : &map_k_hi;
          const CUtensorMap* ml = my.kind == T_VERT ? &map_kc_lo : &map_k_lo;
          tc::tma_load_3d(kdst + 0 * kKHalf, mh, k_full + bk, 0, 0, tile);
          tc::tma_load_3d(kdst + 1 * kKHalf, mh, k_full + bk, 0, 0, tile + 1);
          tc::tma_load_3d(kdst + 2 * kKHalf, ml, k_full + bk, 0, 0, tile);
          tc::tma_load_3d(kdst + 3 * kKHalf, ml, k_full + bk, 0, 0, tile + 1);
#endif
#if !defined(LCX_TC_TRACE_PV) && !defined(LCX_TC_TRACE_SM)
          trace_mark(p, Tj, 1);
#endif
          if constexpr (kProdLoads) {
            const int bv = Tj % NV;
            tc::mbar_wait_sleepy(v_empty + bv, ((Tj / NV) & 1) ^ 1, LCX_TC_SLEEPY);
            tc::mbar_expect_tx(v_full + bv, kVStage);
            const int64_t vtile = my.kind == T_VERT ? int64_t(it.h) * (p.capp / 64) + my.key0 / 64
                                                    : int64_t(it.g) * p.ntiles_k + my.key0 / 64;
            tc::bulk_load(smem_base + OFF_V + bv * kVStage,
                          (my.kind == T_VERT ? p.vct : p.vt) + vtile * (kVStage / 2), kVStage,
                          v_full + bv);
          }
        }
        __syncwarp();
        M += nb;
        T += nb;
      }
    }
    for (int e = 0; e < kGroups; ++e) {  // one end marker per softmax group
      slot_wait(M);
      if (lane == 0) metas[M % kMetaSlots].kind = T_END;
      __syncwarp();
      tc::mbar_arrive(m_full + int(M % kMetaSlots));
      ++M;
    }
    if (lane == 0 && p.tile_count)
      atomicAdd(reinterpret_cast<unsigned long long*>(p.tile_count), (unsigned long long)T);
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(0);
  } else if (warp == kWarpMma || warp == kWarpMma2) {
    // ========================================= QK issuer (+ PV issuer, kMerge) ====
    // kWarpMma: QK of every tile (even tiles with kQk2) and every PV; kWarpMma2: QK of odd
    // tiles.  Both read every ring slot and wait for every Q rotation.
    const bool pv_warp = warp == kWarpMma;
    const uint32_t qk_odd = warp == kWarpMma2 ? 1u : 0u;
    auto qk_mine = [&](uint32_t t) { return !kQk2 || (t & 1u) == qk_odd; };
    uint32_t T = 0, E = 0, M = 0;
    // this warp's barrier waits: suspended try_wait, or test_wait polls with a sleep
    // (LCX_TC_SLEEPY_MMA ns) that keep it out of the barrier unit between polls
    auto mma_wait = [&](tc::SBar bar, uint32_t par) {
      if constexpr (LCX_TC_SLEEPY_MMA > 0) tc::mbar_wait_sleepy(bar, par, LCX_TC_SLEEPY_MMA);
      else tc::mbar_wait(bar, par);
    };
    // all 32 lanes run this loop (warp-uniform); one elected lane issues
    const uint64_t dk0 = tc::sdesc_sw128(tc::smem_u32(smem + OFF_K));
    // merged PV issue: O += P(Tp) V(Tp), P aliasing S buffer Tp % NS (TS-form MMA)
    const uint64_t dv0 = tc::sdesc_sw128(tc::smem_u32(smem + OFF_V));
    uint32_t T_first = 0;
    // PVs not issued yet: tiles T - npend .. T - 1 (flags in pfl, oldest first); the PV of
    // tile T - kPvLag is issued after QK(T), so the QK of the next tiles never waits for a
    // P that the softmax has not produced yet (with NS = 2 S buffers QK(T + 1) needs PV(T - 1)
    // anyway: lag 1; with 4, lag 2)
#ifndef LCX_TC_PV_LAG
#define LCX_TC_PV_LAG 0  // 0: NS / kGroups
#endif
    constexpr int kPvLag = LCX_TC_PV_LAG > 0 ? LCX_TC_PV_LAG : NS / kGroups;
    static_assert(kPvLag >= 1 && kPvLag <= 3 && kPvLag < NS, "PV lag");
    // Issue throttle (LCX_TC_MMA_DEPTH products in flight): a tcgen05.mma that finds the
    // tensor pipe's queue full holds its sub-partition's dispatch, starving the softmax warp
    // that shares it; waiting on a completion barrier instead parks this warp.
    uint32_t nprod = 0;
    auto throttle = [&]() {
      if constexpr (kMmaDepth > 0) {
        if (nprod >= uint32_t(kMmaDepth)) {
          const uint32_t kk = nprod - kMmaDepth;
          mma_wait(prog + int(kk % 4), (kk / 4) & 1);
        }
      }
    };
    auto product_done = [&]() {
      if constexpr (kMmaDepth > 0) tc::mma_commit_warp(prog + int(nprod % 4));
      ++nprod;
    };
    int npend = 0;
    int pfl[3] = {0, 0, 0};
    auto issue_pv = [&](uint32_t Tp, int fl) {
      const int bs = Tp % NS, bv = Tp % NV;
      WAITP(5, mma_wait(p_full + bs, (Tp / NS) & 1));
      WAITP(6, mma_wait(v_full + bv, (Tp / NV) & 1));
      tc::tc_fence_after();
      const uint64_t dv = dv0 + ((bv * kVStage) >> 4);
      if (fl & F_FIRST) T_first = Tp;
      const bool first = kSplitO ? (Tp - T_first < uint32_t(kGroups) && !(p.init && Tp == T_first))
                                 : ((fl & F_FIRST) && !p.init);
      const uint32_t dO = tmem + COL_O + (kSplitO ? (Tp % kGroups) * HD : 0);
      throttle();
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk)
        tc::mma_f16_ts_warp(dO, tmem + bs * BN + kk * 8, dv + ((kk * 32) >> 4), IDESC_PV,
                            (first && kk == 0) ? 0u : 1u);
      product_done();
      tc::mma_commit_warp(v_empty + bv);
      tc::mma_commit_warp(s_free + bs);
#ifndef LCX_TC_TRACE_Q
      if (lane == 0) trace_mark(p, Tp, 4);
#endif
    };
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, mma_wait(m_full + slot, (M / kMetaSlots) & 1));
      const int kind = metas[slot].kind;
      const int flags = metas[slot].flags;
      const int qb = kQBufs == 2 ? (metas[slot].grp & 1) : 0;  // Q buffer of the tile's group
      __syncwarp();
      LANE_ARRIVE(m_empty + slot);
      ++M;
      if constexpr (kMerge) {
        // the previous item's last PV goes first when this tile cannot be issued before it
        // completes (item start: the new item's Q rotation waits for that item's epilogue,
        // which waits for its last PV) or when nothing follows
        if (pv_warp && npend && (kind == T_END || kind == T_EMPTY || (flags & F_FIRST))) {
          for (int x = 0; x < npend; ++x) issue_pv(T - npend + x, pfl[x]);
          npend = 0;
        }
      }
      if (kind == T_END) break;
      if (kind == T_EMPTY) continue;
      if (flags & F_EPOCH) {  // first tile of a group: its Q buffer is (or will be) filled
        WAITP(1, mma_wait(q_ready + qb, (E >> (qb * 16)) & 1));
        E += 1u << (qb * 16);  // per-buffer use counts (low / high half)
      }
      const int bk = T % NK, bs = T % NS;
      if (qk_mine(T)) {
      WAITP(2, mma_wait(k_full + bk, (T / NK) & 1));
      WAITP(3, mma_wait(s_free + bs, ((T / NS) & 1) ^ 1));  // PV(T - NS) released S/P
      tc::tc_fence_after();
#ifndef LCX_TC_TRACE_PV
#ifndef LCX_TC_TRACE_Q
      if (lane == 0) trace_mark(p, T, 7);
#endif
#endif
      const uint64_t dk = dk0 + ((bk * kKStage) >> 4);
      const uint32_t dS = tmem + bs * BN;
#ifdef LCX_TC_WAITPROF
      const long long t_iss = clock64();
#endif
#pragma unroll
#ifdef LCX_TC_ONE_TERM  // timing experiment only: hi.hi product alone
      for (int combo = 0; combo < 1; ++combo) {
#else
      for (int combo = 0; combo < 3; ++combo) {
#endif
        const uint32_t qa = tmem + COL_Q + qb * QBUF + (combo == 2 ? HD / 2 : 0);  // hh, hl, lh
        const uint64_t ka = dk + (combo == 1 ? ((2 * kKHalf) >> 4) : 0);
        if constexpr (kMerge) throttle();
#if LCX_TC_MMA_X8
        tc::mma_f16_ts_x8_warp(dS, qa, ka, kKHalf >> 4, IDESC_QK, combo ? 1u : 0u);
#else
#pragma unroll
        for (int half = 0; half < 2; ++half)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_f16_ts_warp(dS, qa + half * 32 + kk * 8,
                                ka + ((half * kKHalf + kk * 32) >> 4), IDESC_QK,
                                (combo | half | kk) ? 1u : 0u);
#endif
        if constexpr (kMerge) product_done();
      }
      tc::mma_commit_warp(k_empty + bk);
      tc::mma_commit_warp(s_full + bs);
#ifdef LCX_TC_WAITPROF
      wacc[4] += clock64() - t_iss;
#endif
#ifndef LCX_TC_TRACE_PV
#ifndef LCX_TC_TRACE_Q
      if (lane == 0) trace_mark(p, T, 3);
#endif
#endif
      }  // qk_mine
      if (kMerge && pv_warp) {
        if (npend == kPvLag) {  // QK(T) runs while the softmax finishes P(T - kPvLag)
          issue_pv(T - kPvLag, pfl[0]);
          pfl[0] = pfl[1];
          pfl[1] = pfl[2];
          --npend;
        }
        pfl[npend++] = flags;
      }
      ++T;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(1);
  } else if (warp == kWarpLoad || warp == kWarpLoadV) {
    // ===================================== K (hi + lo) and V^T loads (kMerge) ====
    const bool do_k = warp == kWarpLoad, do_v = !kKvLoaders || warp == kWarpLoadV;
    uint32_t T = 0, M = 0;
    for (;;) {
      const int slot = M % kMetaSlots;
      #if LCX_TC_SLEEPY_LOAD
      WAITP(0, tc::mbar_wait_sleepy(m_full + slot, (M / kMetaSlots) & 1, LCX_TC_SLEEPY_LOAD));
#else
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
#endif
      const int kind = metas[slot].kind;
      const int h = metas[slot].h;
      const int64_t key0 = metas[slot].key0;
      __syncwarp();
      LANE_ARRIVE(m_empty + slot);
      ++M;
      if (kind == T_END) break;
      if (kind == T_EMPTY) continue;
      if (lane == 0) {
        const int64_t kt = kind == T_VERT ? int64_t(h) * (p.capp / 64) + key0 / 64
                                          : int64_t(h / p.group) * p.ntiles_k + key0 / 64;
        const int bk = T % NK;
        if (do_k) {
#if LCX_TC_SLEEPY_LOAD
        WAITP(1, tc::mbar_wait_sleepy(k_empty + bk, ((T / NK) & 1) ^ 1, LCX_TC_SLEEPY_LOAD));
#else
        WAITP(1, tc::mbar_wait(k_empty + bk, ((T / NK) & 1) ^ 1));
#endif
        tc::mbar_expect_tx(k_full + bk, kKStage);
        const uint32_t kdst = smem_base + OFF_K + bk * kKStage;
        // pre-swizzled tiles: hi (2 halves) and lo are one contiguous 16 KB run each
        tc::bulk_load(kdst, (kind == T_VERT ? p.kchi : p.khi) + kt * kKHalf, 2 * kKHalf,
                      k_full + bk);
        tc::bulk_load(kdst + 2 * kKHalf, (kind == T_VERT ? p.kclo : p.klo) + kt * kKHalf,
                      2 * kKHalf, k_full + bk);
#ifndef LCX_TC_TRACE_SM
        trace_mark(p, T, 1);
#endif
        }
        const int bv = T % NV;
        if (do_v) {
#if LCX_TC_SLEEPY_LOAD
        WAITP(2, tc::mbar_wait_sleepy(v_empty + bv, ((T / NV) & 1) ^ 1, LCX_TC_SLEEPY_LOAD));
#else
        WAITP(2, tc::mbar_wait(v_empty + bv, ((T / NV) & 1) ^ 1));
#endif
        tc::mbar_expect_tx(v_full + bv, kVStage);
        tc::bulk_load(smem_base + OFF_V + bv * kVStage, (kind == T_VERT ? p.vct : p.vt) + kt * (kVStage / 2),
                      kVStage, v_full + bv);
#ifndef LCX_TC_TRACE_SM
        trace_mark(p, T, 2);
#endif
        }
      }
      __syncwarp();
      ++T;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(2);
  } else if (warp == kWarpV) {
    // ===================================================== V TMA loads ====
    uint32_t T = 0, M = 0;
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
      const int kind = metas[slot].kind;
      const int h = metas[slot].h;
      const int key0 = int(metas[slot].key0);
      __syncwarp();
      LANE_ARRIVE(m_empty + slot);
      ++M;
      if (kind == T_END) break;
      if (kind == T_EMPTY) continue;
      if (lane == 0) {
        const int bv = T % NV;
#if LCX_TC_SLEEPY
        WAITP(1, tc::mbar_wait_sleepy(v_empty + bv, ((T / NV) & 1) ^ 1, LCX_TC_SLEEPY));
#else
        WAITP(1, tc::mbar_wait(v_empty + bv, ((T / NV) & 1) ^ 1));
#endif
        tc::mbar_expect_tx(v_full + bv, kVStage);
        const uint32_t vdst = smem_base + OFF_V + bv * kVStage;
        const int64_t vtile = kind == T_VERT ? int64_t(h) * (p.capp / 64) + key0 / 64
                                             : int64_t(h / p.group) * p.ntiles_k + key0 / 64;
#ifdef LCX_TC_FAKE_LOADS
        const_cast<int64_t&>(vtile) = (vtile & 31);
#endif
#if LCX_TC_BULK
        tc::bulk_load(vdst, (kind == T_VERT ? p.vct : p.vt) + vtile * (kVStage / 2), kVStage,
                      v_full + bv);
#else
        tc::tma_load_3d(vdst, kind == T_VERT ? &map_vct : &map_vt, v_full + bv, 0, 0, int(vtile));
#endif
#ifndef LCX_TC_TRACE_PV
        trace_mark(p, T, 2);
#endif
      }
      __syncwarp();
      ++T;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(2);
  } else if (warp == kWarpPv) {
    // ============================================== PV issuer (O += P V) ====
    uint32_t T = 0, M = 0, T_first = 0;
    const uint64_t dv0 = tc::sdesc_sw128(tc::smem_u32(smem + OFF_V));
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
#ifdef LCX_TC_TRACE_PV
      if (lane == 0) trace_mark(p, T, 0);
#endif
      const int kind = metas[slot].kind;
      const int flags = metas[slot].flags;
      __syncwarp();
      LANE_ARRIVE(m_empty + slot);
      ++M;
      if (kind == T_END) break;
      if (kind == T_EMPTY) continue;
      const int bs = T % NS, bv = T % NV;
#if LCX_TC_SLEEPY_PV
      WAITP(1, tc::mbar_wait_sleepy(p_full + bs, (T / NS) & 1, LCX_TC_SLEEPY_PV));
#else
      WAITP(1, tc::mbar_wait(p_full + bs, (T / NS) & 1));
#endif
#ifdef LCX_TC_TRACE_PV  // columns 0 / 1 / 2: PV issuer passed the meta / P / V waits
      if (lane == 0) trace_mark(p, T, 1);
#endif
      WAITP(2, tc::mbar_wait(v_full + bv, (T / NV) & 1));
#ifdef LCX_TC_TRACE_PV
      if (lane == 0) trace_mark(p, T, 2);
#endif
      tc::tc_fence_after();
      const uint64_t dv = dv0 + ((bv * kVStage) >> 4);
      if (flags & F_FIRST) T_first = T;
      // the first PV into an O of the item overwrites it (a key-window pass > 0 restored
      // the running O into the first tile's O)
      const bool first = kSplitO ? (T - T_first < uint32_t(kGroups) && !(p.init && T == T_first))
                                 : ((flags & F_FIRST) && !p.init);
      const uint32_t dO = tmem + COL_O + (kSplitO ? (T % kGroups) * HD : 0);
#if LCX_TC_MMA_X8
      static_assert(BN / 16 == 4, "four PV MMAs per tile");
      tc::mma_f16_ts_x4_warp(dO, tmem + bs * BN, dv, IDESC_PV, first ? 0u : 1u);
#else
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk)  // P (fp16, 2 per column) aliases S buffer bs
        tc::mma_f16_ts_warp(dO, tmem + bs * BN + kk * 8, dv + ((kk * 32) >> 4),
                            IDESC_PV, (first && kk == 0) ? 0u : 1u);
#endif
      tc::mma_commit_warp(v_empty + bv);
      tc::mma_commit_warp(s_free + bs);
      if (lane == 0) trace_mark(p, T, 4);
      ++T;
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    WAITP_FLUSH(3);
  } else if (warp >= kSmBase && warp < kSmBase + kSoftmaxWarps) {
    // ============================= softmax / correction / epilogue ====
    // kGroups warp groups take the tiles of the stream in turn (group g: tiles T with
    // T % kGroups == g); within a group, warp = TMEM lane quadrant and thread = query
    // row with all 64 columns of the tile.  The groups run out of phase -- one computes
    // a tile's max while the others exponentiate earlier tiles -- and pass the row's
    // running max on per tile through shared memory, signalled on an mbarrier per
    // (group, quadrant).  Each group keeps its own partial row sum l expressed at the max
    // it last used; the owner of an item's last tile combines all of them (each published
    // before the group's P release) in the epilogue.
    const int wq = warp & 3;                 // TMEM lane quadrant (= sub-partition)
    const int grp = (warp - kSmBase) >> 2;   // warp group
    const int r = wq * 32 + lane;
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    const uint32_t col_o = COL_O + (kSplitO ? uint32_t(grp) * HD : 0u);  // this group's O
    uint32_t J_cur = 0;  // split O: the CTA's index of the current item (record item_seq)
    float* mbuf = reinterpret_cast<float*>(smem + OFF_RED);  // [kGroups][128] m after tile
    float2* lbuf = reinterpret_cast<float2*>(smem + OFF_RED + kGroups * 128 * 4);
    const tc::SBar h_in = hand + (((grp + kGroups - 1) % kGroups) * 4 + wq);  // predecessor
    const tc::SBar h_out = hand + (grp * 4 + wq);
    // A group reads only its own ring slots, M == grp mod kGroups (the producer emits EMPTY
    // and END markers once per group), so tile T = M - kGroups * (EMPTY markers seen); it
    // recognises an item's start by the record's first-tile index.
    uint32_t T = 0, M = grp, T_first = 0, empties = 0;
    int32_t cur_t0 = -1;
    float l = 0.f, m_used = -INFINITY;  // this group's partial sum, at max m_used
    float m_init = -INFINITY;           // running max at the item start (key-window passes)
    Item qi{};  // only i0 / rend / h used by rotate_q
    if (!kSplitO && grp == kGroups - 1) LANE_ARRIVE(h_out);  // tile 0
    auto rotate_row = [&](int pattern, int qbuf) {
      rotate_q(p, qi, pattern, r, 0, tmem + lane_base, qbuf);
      rotate_q(p, qi, pattern, r, 1, tmem + lane_base, qbuf);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(q_ready + qbuf);
    };
#ifdef LCX_TC_WAITPROF
    long long t_own = 0;  // start of the last own tile
#endif
    for (;;) {
      const int slot = M % kMetaSlots;
      WAITP(0, tc::mbar_wait(m_full + slot, (M / kMetaSlots) & 1));
#ifdef LCX_TC_WAITPROF
      const long long t_meta = clock64();
#endif
#if defined(LCX_TC_TRACE_Q) && LCX_TC_TRACE_Q == 2
      const long long tq_meta = clock64();
#endif
      const TileMeta& mt = metas[slot];
      const int kind = mt.kind, flags = mt.flags;
      if (kind == T_END) break;
      T = M - uint32_t(kGroups) * empties;
      const int64_t i0 = mt.i0, rend = mt.rend;
      const int h = mt.h;
      const int64_t i = i0 + r;
      const bool row_ok = i < rend;
      const bool mine = kind != T_EMPTY;  // every slot this group reads is its own
      uint64_t mask = 0;
      if (mine && row_ok) {
        if (kind == T_VERT) {
          int cnt = mt.nfar;
          while (cnt < mt.count) {
            const int32_t kk = mt.keys[cnt];
            if (kk < 0 || int64_t(kk) > i) break;
            ++cnt;
          }
          mask = cnt >= 64 ? ~0ull : ((1ull << cnt) - 1);
        } else if (kind == T_SLASH) {
          const int off = int(i - mt.key0 - 63 - mt.sbase);
          mask = __brevll(window64(mt.sw, off)) & ~mt.vmask;
        } else {
          const int64_t lim = i - mt.key0;
          mask = lim >= 63 ? ~0ull : (lim < 0 ? 0ull : ((2ull << lim) - 1));
        }
      }
      const int pattern = mt.pattern, tgrp = mt.grp, ng = mt.ng, next_pattern = mt.next_pattern;
      const int gpat1 = mt.gpat[1], gpat2 = mt.gpat[2];
      const int32_t item_t0 = mt.item_t0;
      const int32_t item_seq = mt.item_seq;
      __syncwarp();
      LANE_ARRIVE(m_empty + slot);
#ifdef LCX_TC_WAITPROF
      wacc[3] += clock64() - t_meta;
#endif
#if defined(LCX_TC_TRACE_Q) && LCX_TC_TRACE_Q == 2  // own tile: meta phase start / end
      if (mine && lane == 0 && p.trace && blockIdx.x == 0 && T < kTraceTiles) {
        p.trace[T * 8 + wq] = tq_meta;
        p.trace[T * 8 + 4 + wq] = clock64();
      }
#endif
      M += kGroups;
      if (kind == T_EMPTY) {
        ++empties;
        if (!(flags & F_REPEAT) && row_ok && !p.init) {  // init passes keep the running state
          float4* o = reinterpret_cast<float4*>(p.out + (i * p.hq + h) * int64_t(HD));
          for (int x = 0; x < 32; ++x) o[x] = make_float4(0.f, 0.f, 0.f, 0.f);
          p.lse[int64_t(h) * p.lse_stride + i] = -INFINITY;
        }
        continue;
      }
      if (item_t0 != cur_t0) {  // this group's first tile of an item: partial sums, Q rows
        cur_t0 = item_t0;
        l = 0.f;
        m_used = -INFINITY;
        T_first = uint32_t(item_t0);
        J_cur = uint32_t(item_seq);
        qi.i0 = i0;
        qi.rend = rend;
        qi.h = h;
      }
#ifdef LCX_TC_WAITPROF
      const long long t_first = clock64();
      t_own = t_first;
#endif
      const uint32_t k = T / kGroups;  // this group's tile index (hand-off phase)
      if (kSplitO && T - T_first < uint32_t(kGroups) && J_cur > 0) {
        // this group's first tile of the item: the previous item's epilogue has read both
        // O (this group's next PV overwrites its O) and its QKs are done (Q is free)
        tc::mbar_wait(edone, (J_cur - 1) & 1);
        tc::tc_fence_after();
      }
      if (flags & F_FIRST) {
        // the previous item's last tile (T - 1, another group) finished its epilogue: O is
        // read and S(T - 1) consumed, so O / Q of this CTA's TMEM are free
        if constexpr (!kSplitO) {
          tc::mbar_wait(h_in, k & 1);
          tc::tc_fence_after();
        }
        m_init = -INFINITY;
        if (p.init) {
          // key-window pass > 0: continue from the row's running (o, lse) -- O goes back
          // into TMEM (the previous item's last PV completed before its epilogue read O)
          const float lp = row_ok ? p.lse[int64_t(h) * p.lse_stride + i] : -INFINITY;
          const bool live = lp != -INFINITY;
          m_init = live ? lp * 1.4426950408889634f : -INFINITY;
          l = live ? 1.f : 0.f;
          m_used = m_init;
          const float4* o = reinterpret_cast<const float4*>(p.out + (i * p.hq + h) * int64_t(HD));
#pragma unroll 1
          for (int q4 = 0; q4 < 4; ++q4) {
            float ov[32];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              const float4 v = live ? o[q4 * 8 + x] : make_float4(0.f, 0.f, 0.f, 0.f);
              ov[4 * x] = v.x;
              ov[4 * x + 1] = v.y;
              ov[4 * x + 2] = v.z;
              ov[4 * x + 3] = v.w;
            }
            tc::tmem_st32(tmem + lane_base + col_o + q4 * 32, ov);
          }
          tc::tmem_wait_st();
        }
        // group 0's Q, and group 1's into the other buffer ahead of its first QK
        if constexpr (kQBufs == 2) {
          rotate_row(pattern, tgrp & 1);
          if (tgrp + 1 < ng) rotate_row(gpat1, (tgrp + 1) & 1);
        } else {
          rotate_row(pattern, 0);
        }
      }
#ifdef LCX_TC_WAITPROF
      wacc[2] += clock64() - t_first;  // item start: hand-over wait, O restore, Q rotations
#endif
      const int b = T % NS;
      const uint32_t ph = (T / NS) & 1;
      float sv[kSReread ? 32 : 64];
      WAITP(1, tc::mbar_wait(s_full + b, ph));
      tc::tc_fence_after();
#ifdef LCX_TC_WAITPROF
      const long long t_ld = clock64();
#endif
      if constexpr (!kSReread) {
        tc::tmem_ld32(tmem + lane_base + b * BN, sv);
        tc::tmem_ld32_wait(tmem + lane_base + b * BN + 32, sv + 32);
        tc::tmem_wait_ld_dep32(sv);
      }
#ifdef LCX_TC_WAITPROF
      wacc2[4] += clock64() - t_ld;
#endif
#ifdef LCX_TC_TRACE_SM  // owner group's quadrant-0 warp: 5 S got, 0 m handed over, 6 P put
#if defined(LCX_TC_TRACE_Q) && LCX_TC_TRACE_Q == 2
#elif defined(LCX_TC_TRACE_Q)  // per quadrant warp: S got in column 4 + wq
      if (lane == 0) trace_mark(p, T, 4 + wq);
#else
      if (wq == 0 && lane == 0) trace_mark(p, T, 5);
#endif
#else
      if (threadIdx.x == 0) trace_mark(p, T, 5);
#endif
#ifdef LCX_TC_WAITPROF
      const long long t_sg = clock64();
#endif
      // the group's QKs are complete: its Q buffer takes the group after next
      if constexpr (kQBufs == 2) {
        if ((flags & F_EPOCH_AFTER) && tgrp + 2 < ng) rotate_row(gpat2, tgrp & 1);
      } else {
        if (flags & F_EPOCH_AFTER) {  // old pattern's QKs done
          if (kQk2 && T >= 1) {  // the other QK issuer's last tile (T - 1) too
            const uint32_t Tp = T - 1;
            tc::mbar_wait(s_full + int(Tp % NS), (Tp / NS) & 1);
          }
          rotate_row(next_pattern, 0);
        }
      }
#ifdef LCX_TC_FAKE_SOFTMAX  // timing experiment only: no softmax math
      for (int cc = 0; cc < int(sizeof(sv) / sizeof(float)); ++cc) sv[cc] = -INFINITY;
      mask = 0ull;
#endif
      // masked logits -> -inf (ex2(-inf) = 0), already in log2 units
      const bool all_in = __all_sync(0xffffffffu, mask == ~0ull);  // no select needed
      if constexpr (!kSReread) {
        if (!all_in) {
          const uint32_t lo = uint32_t(mask), hi = uint32_t(mask >> 32);
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) {
            sv[cc] = ((lo >> cc) & 1u) ? sv[cc] : -INFINITY;
            sv[32 + cc] = ((hi >> cc) & 1u) ? sv[32 + cc] : -INFINITY;
          }
        }
      }
      // ---- P = exp2(x - m) in fp16, written over the tile's S columns in TMEM:
      // key c -> column c / 2 (two fp16 per 32-bit column).  Packed f32x2 subtract /
      // accumulate (FADD2): half the FP32 instructions per key.  Returns the row sum.
      auto exps_store = [&](float m) -> float {
        const float mm = m == -INFINITY ? 0.f : m;
        const float2 nm2 = make_float2(-mm, -mm);
        float2 rs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};  // four independent sum chains
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {  // two 32-key halves: fewer live registers
          if constexpr (kSReread) {  // second read of this half (its P not yet written)
            tc::tmem_ld32_wait(tmem + lane_base + b * BN + hf * 32, sv);
            const uint32_t mb = uint32_t(mask >> (32 * hf));
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) sv[cc] = ((mb >> cc) & 1u) ? sv[cc] : -INFINITY;
          }
          uint32_t pw[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int c = (kSReread ? 0 : hf * 32) + 2 * k;
            const float2 x = __fadd2_rn(make_float2(sv[c], sv[c + 1]), nm2);
            const float2 pp = make_float2(ex2(x.x), ex2(x.y));
            rs2[k & 3] = __fadd2_rn(rs2[k & 3], pp);
            const __half2 h2 = __floats2half2_rn(pp.x, pp.y);
            pw[k] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          tc::tmem_st16(tmem + lane_base + b * BN + hf * 16, pw);
        }
        const float2 ra = __fadd2_rn(rs2[0], rs2[1]), rb = __fadd2_rn(rs2[2], rs2[3]);
        return (ra.x + rb.x) + (ra.y + rb.y);
      };
      auto tile_max = [&]() -> float {
        float t4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if constexpr (!kSReread) {
#pragma unroll
          for (int cc = 0; cc < 64; cc += 8)
#pragma unroll
            for (int u = 0; u < 4; ++u) t4[u] = fmaxf(t4[u], fmaxf(sv[cc + u], sv[cc + 4 + u]));
        } else {
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            tc::tmem_ld32_wait(tmem + lane_base + b * BN + hf * 32, sv);
            const uint32_t mb = uint32_t(mask >> (32 * hf));
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) sv[cc] = ((mb >> cc) & 1u) ? sv[cc] : -INFINITY;
#pragma unroll
            for (int cc = 0; cc < 32; cc += 8)
#pragma unroll
              for (int u = 0; u < 4; ++u)
                t4[u] = fmaxf(t4[u], fmaxf(sv[cc + u], sv[cc + 4 + u]));
          }
        }
        return fmaxf(fmaxf(t4[0], t4[1]), fmaxf(t4[2], t4[3]));
      };
      auto rescale_o = [&](float f) {
#pragma unroll 1
        for (int q8 = 0; q8 < 8; ++q8) {  // 16 columns at a time: S is still live here
          float ov[16];
          const uint32_t ta = tmem + lane_base + col_o + q8 * 16;
          tc::tmem_ld16_wait(ta, ov);
#pragma unroll
          for (int x = 0; x < 16; ++x) ov[x] *= f;
          tc::tmem_st16f(ta, ov);
        }
        tc::tmem_wait_st();
      };
      float rs;
      if (kSplitO && kSpecExp && __all_sync(0xffffffffu, m_used != -INFINITY)) {
        // split O: the group's own running max is known before the tile -- exponentiate
        // at it straight away, independent of the tile max; only when some row's max
        // moved past the threshold (rare after an item's first tiles) rescale and redo.
        // The P written is the same as max-first would write.
        rs = exps_store(m_used);
        const float tmax = tile_max();
        const bool need = tmax > m_used + kRescaleThresh;
        if (__any_sync(0xffffffffu, need)) {
          const float m = need ? tmax : m_used;
          rescale_o(need ? ex2(m_used - m) : 1.f);  // own last PV done (S(T) is full)
          if (need) l *= ex2(m_used - m);
          m_used = m;
          tc::tmem_wait_st();  // the speculative P stores land before their rewrite
          rs = exps_store(m);
        }
#ifdef LCX_TC_WAITPROF
        wacc[5] += clock64() - t_sg;
#endif
      } else {
      const float tmax = tile_max();
#ifdef LCX_TC_WAITPROF
      wacc[5] += clock64() - t_sg;
#endif
#ifdef LCX_TC_TRACE_SM  // column 1: tile max known (before the hand-off wait)
      if (wq == 0 && lane == 0) trace_mark(p, T, 1);
#endif
      // ---- running max: previous tile's (other group) unless the item starts here
      if (!kSplitO && !(flags & F_FIRST)) WAITP2(0, tc::mbar_wait(h_in, k & 1));
      const float m_prev = kSplitO ? m_used
                           : (flags & F_FIRST) ? m_init
                                               : mbuf[((T + kGroups - 1) % kGroups) * 128 + r];
      // lazy rescale: the max moves only past a threshold (P <= 2^8 in fp16)
      const bool need = tmax > m_prev + kRescaleThresh;
      const float m = need ? tmax : m_prev;
      if constexpr (!kSplitO) mbuf[grp * 128 + r] = m;
#ifdef LCX_TC_TRACE_SM
      if (wq == 0 && lane == 0) trace_mark(p, T, 0);
#endif
      // an item's last tile hands over only after its epilogue (next item's O / Q)
      if (!kSplitO && !(flags & F_LAST)) {
        __syncwarp();
        LANE_ARRIVE(h_out);
      }
#ifdef LCX_TC_WAITPROF
      const long long t_rs = clock64();
#endif
      if (__any_sync(0xffffffffu, need && m_prev != -INFINITY)) {
        // O holds PV up to tile T - 1 at max m_prev: complete it, then rescale
        // (split O: this group's last PV, T - kGroups, completed before QK(T) took its S
        // buffer)
        if constexpr (!kSplitO) {
          const uint32_t Tp = T - 1;
          tc::mbar_wait(s_free + (Tp % NS), (Tp / NS) & 1);
          tc::tc_fence_after();
        }
        rescale_o((need && m_prev != -INFINITY) ? ex2(m_prev - m) : 1.f);
      }
      if (m != m_used) {  // this group's partial sum follows the row max
        if (m_used != -INFINITY) l *= ex2(m_used - m);
        m_used = m;
      }
#ifdef LCX_TC_WAITPROF
      wacc2[1] += clock64() - t_rs;
      const long long t_e0 = clock64();
#endif
      rs = exps_store(m);
#ifdef LCX_TC_WAITPROF
      wacc2[2] += clock64() - t_e0;
      ++wacc2[3];  // own tiles
#endif
      }
#ifdef LCX_TC_WAITPROF
      const long long t_ex = clock64();
#endif
#ifdef LCX_TC_TRACE_SM  // column 2: exponentials and P stores issued (before the tail)
      if (wq == 0 && lane == 0) trace_mark(p, T, 2);
#endif
      // P released to the PV first (its stores complete and fenced)
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full + b);
      l += rs;
      // every phase of the predecessor group's partial-sum barrier is consumed (tile T - 1
      // published before this one, so this rarely waits); the epilogue's wait on the same
      // phase then returns at once
#ifndef LCX_TC_NO_LPUB_WAIT  // experiment: skip the per-tile phase consumption
      if (T >= 1) {
        const uint32_t Tp = T - 1;
        tc::mbar_wait(lpub + int(Tp % kGroups), (Tp / kGroups) & 1);
      }
#endif
      // partial (l, m) for the item's epilogue
      lbuf[((k & 1) * kGroups + grp) * 128 + r] = make_float2(l, m_used);
      __syncwarp();
      LANE_ARRIVE(lpub + grp);
#ifdef LCX_TC_WAITPROF
      wacc[6] += clock64() - t_ex;
#endif
#ifdef LCX_TC_TRACE_SM
#if defined(LCX_TC_TRACE_Q) && LCX_TC_TRACE_Q == 2
#elif defined(LCX_TC_TRACE_Q)  // per quadrant warp: P put in column wq
      if (lane == 0) trace_mark(p, T, wq);
#else
      if (wq == 0 && lane == 0) trace_mark(p, T, 6);
#endif
#else
      if (threadIdx.x == 0) trace_mark(p, T, 6);
#endif
#ifdef LCX_TC_WAITPROF
      const long long t_epi = clock64();
#endif
      if (kSplitO && (flags & F_LAST)) {
        // ---- epilogue (split O): merge the other group's O (its last tile T - 1) into
        // this group's, normalize, store; then release both O for the next item ----
        float sx = l > 0.f ? 1.f : 0.f, sy = 0.f, ly = 0.f, mt = m_used;
        const bool other = T > T_first;
        if (other) {
          const uint32_t To = T - 1, go = To % kGroups, ko = To / kGroups;
          tc::mbar_wait(lpub + int(go), ko & 1);
          const float2 lo = lbuf[((ko & 1) * kGroups + go) * 128 + r];
          ly = lo.x;
          if (lo.x > 0.f) {
            if (l > 0.f) {
              mt = fmaxf(m_used, lo.y);
              sx = ex2(m_used - mt);
              sy = ex2(lo.y - mt);
            } else {
              mt = lo.y;
              sy = 1.f;
            }
          }
        }
        const float lt = l * sx + ly * sy;
        tc::mbar_wait(s_free + b, ph);  // PV(T) complete, and every PV before it
        tc::tc_fence_after();
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        const float ax = sx * inv, ay = sy * inv;
        const uint32_t col_y = COL_O + uint32_t((grp + 1) % kGroups) * HD;
        float4* o = reinterpret_cast<float4*>(p.out + (i * p.hq + h) * int64_t(HD));
#pragma unroll 1
        for (int q8 = 0; q8 < 8; ++q8) {
          float ov[16], oy[16];
          tc::tmem_ld16_wait(tmem + lane_base + col_o + q8 * 16, ov);
          if (other) tc::tmem_ld16_wait(tmem + lane_base + col_y + q8 * 16, oy);
          if (!other) {
#pragma unroll
            for (int x = 0; x < 16; ++x) oy[x] = 0.f;
          }
          if (row_ok) {
#pragma unroll
            for (int x = 0; x < 4; ++x)
              o[q8 * 4 + x] = make_float4(ov[4 * x] * ax + oy[4 * x] * ay,
                                          ov[4 * x + 1] * ax + oy[4 * x + 1] * ay,
                                          ov[4 * x + 2] * ax + oy[4 * x + 2] * ay,
                                          ov[4 * x + 3] * ax + oy[4 * x + 3] * ay);
          }
        }
        if (row_ok)
          p.lse[int64_t(h) * p.lse_stride + i] =
              lt > 0.f ? (mt + log2f(lt)) * 0.69314718055994530942f : -INFINITY;
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(edone);
      } else if (flags & F_LAST) {
        // ---- epilogue: add the other group's partial sum, wait for the last PV,
        // normalize, store ----
        float lt = l;
#pragma unroll
        for (uint32_t d = 1; d < uint32_t(kGroups); ++d) {  // the other groups' last tiles
          if (T < T_first + d) break;
          const uint32_t To = T - d, go = To % kGroups, ko = To / kGroups;
          tc::mbar_wait(lpub + int(go), ko & 1);
          const float2 lo = lbuf[((ko & 1) * kGroups + go) * 128 + r];
          if (lo.x > 0.f) lt += lo.x * ex2(lo.y - m_used);
        }
        tc::mbar_wait(s_free + b, ph);  // this item's last PV is complete
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
        LANE_ARRIVE(h_out);

      }
#ifdef LCX_TC_WAITPROF
      wacc2[5] += clock64() - t_epi;
      wacc[4] += clock64() - t_own;  // whole own tile, item start to P release / epilogue
#endif
    }
#ifdef LCX_TC_WAITPROF
    wacc[7] = clock64() - t_start;
#endif
    if (wq == 0) WAITP_FLUSH(4);
#ifdef LCX_TC_WAITPROF
    if (wq == 0) {
      for (int _j = 0; _j < 8; ++_j) wacc[_j] = wacc2[_j];
      wacc[7] = clock64() - t_start;
      WAITP_FLUSH(5);
    }
#endif
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
// One block per key row j (blockIdx.x over [r0, r1)), threadIdx.x = dim pair, threadIdx.y
// striding the KV heads: the row's position is worked out once per block, and no thread
// divides by a runtime 64-bit value.
__global__ void k_prep_kernel(const __nv_bfloat16* __restrict__ k, int64_t n, int64_t r0,
                              int hkv, const int64_t* __restrict__ pos_k, int rel_mode,
                              int64_t s, const float2* __restrict__ rope,
                              __nv_bfloat16* __restrict__ khi, __nv_bfloat16* __restrict__ klo,
                              float2* __restrict__ kf) {
  __shared__ int64_t kp_s;
  const int64_t j = r0 + blockIdx.x;
  const int pr = threadIdx.x;
  if (pr == 0 && threadIdx.y == 0) kp_s = rel_mode ? (j % s) : (pos_k ? pos_k[j] : j);
  __syncthreads();
  const float2 c = rope[kp_s * (HD / 2) + pr];
  // tiled [hkv][n/64][half][64 keys][64 dims]: each TMA box is one contiguous 8 KB block
  const int64_t nt = (n + 63) >> 6;
  const int d = 2 * pr;
  const int jr = int(j & 63), dd = d & 63;
  for (int g = threadIdx.y; g < hkv; g += blockDim.y) {
    const int64_t idx = (j * hkv + g) * (HD / 2) + pr;
    const float2 xy = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(k)[idx]);
    const float rx = xy.x * c.x - xy.y * c.y, ry = xy.x * c.y + xy.y * c.x;
    kf[idx] = make_float2(rx, ry);
    const __nv_bfloat162 h2 = __floats2bfloat162_rn(rx, ry);
    const float2 hf = __bfloat1622float2(h2);
    const int64_t o = ((((int64_t(g) * nt + (j >> 6)) * 2 + (d >> 6)) * 64 + jr) * 64 +
                       sw128_chunk(jr, dd >> 3) * 8 + (dd & 7)) >> 1;
    reinterpret_cast<__nv_bfloat162*>(khi)[o] = h2;
    reinterpret_cast<__nv_bfloat162*>(klo)[o] = __floats2bfloat162_rn(rx - hf.x, ry - hf.y);
  }
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
  k_prep_kernel<<<unsigned(r1 - r0), dim3(HD / 2, unsigned(std::min(hkv, 8))), 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(k), n, r0, hkv, pos_k, rel_mode, s, rope, B.khi,
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
  attn_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(q, B.m_khi, B.m_klo, B.m_vt, B.m_kchi,
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
