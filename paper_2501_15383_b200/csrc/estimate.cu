// K1 -- Vertical-Slash estimator, exact fp32 CUDA-core path.
//
// Restates estimate_block (reference core/src/sparse.cpp:142-188) and the row /
// diagonal reductions of select_critical (sparse.cpp:198-217):
//   row r of the estimate is query gi = nk - block + r (queries trail the keys),
//   logit(r, j) = rope(q_gi, rel) . k_j / sqrt(D), rel = gi - j (Standard) or
//   min(gi - j, c - 1) (DcaContinuous), token-index positions, no temperature;
//   causal softmax over j <= gi; entries j > gi are exactly 0.
// Using rope(q, a) . rope(k, b) = rope(q, a - b) . k, the kernel rotates each
// estimator query once (by gi, and by c - 1 for the DCA far region) and the keys
// once (by j), so the inner loop is a plain fp32 dot product over a 64 x 64
// register-tiled block.  Far-region entries (gi - j > c - 1) use
// rope(q_gi, c-1) . k_raw.
//
// Two passes over the keys: pass 1 produces per-(row, split) (max, sum-exp)
// partials which are combined in ascending split order; pass 2 recomputes the
// logits, forms p = exp(l - m) / S and reduces, per 64-key tile, the column
// sums (over rows, ascending) and the 127 diagonal partial sums; a combine
// kernel adds the two tiles that share each diagonal in ascending tile order.
// All reductions are in a fixed order (bitwise deterministic).
#include "est_tc.cuh"
#include "lcx_internal.cuh"

namespace lcx {
namespace {

constexpr int kRows = 64;      // rows per row-tile
constexpr int kKeys = 64;      // keys per tile
constexpr int kThreads = 256;  // 16 x 16, each 4 rows x 4 keys
constexpr int kMaxDim = 128;

struct EstDev {
  const void* q;
  const void* k;
  int hq, hkv, dim, group;
  int64_t nk, block, gbase;  // gbase = nk - block = global index of estimator row 0
  int pos_mode;
  int64_t c;
  const float2* rope;
  const float* qn;   // [hq][block][dim] rope(q_gi, gi)
  const float* qf;   // [hq][block][dim] rope(q_gi, c - 1)  (dca only)
  const float* kn;   // [nk][hkv][dim]  rope(k_j, j)
  int64_t ntiles;
  int tiles_per_split;
  int nsplit;
  int nrt;           // row tiles
  int64_t tile0, tile_end;  // key tiles this launch covers
  int split0, nsplit_total; // stats slot of split 0, slots per head
  int h0;                    // first query head of this call (grid y = heads of the call)
};

// ---- prep: rotate the estimator query rows and the keys ------------------
template <typename T>
__global__ void est_prep_q(EstDev a) {
  const int64_t r = blockIdx.x;
  const int h = a.h0 + int(blockIdx.y);
  const int64_t gi = a.gbase + r;
  const int P = a.dim / 2;
  const T* qrow = reinterpret_cast<const T*>(a.q) + (gi * a.hq + h) * a.dim;
  float* outn = const_cast<float*>(a.qn) + (int64_t(h) * a.block + r) * a.dim;
  float* outf = a.qf ? const_cast<float*>(a.qf) + (int64_t(h) * a.block + r) * a.dim : nullptr;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const float x = load_elem(qrow, 2 * p), y = load_elem(qrow, 2 * p + 1);
    float2 cs = a.rope[gi * P + p];
    outn[2 * p] = x * cs.x - y * cs.y;
    outn[2 * p + 1] = x * cs.y + y * cs.x;
    if (outf) {
      cs = a.rope[(a.c - 1) * P + p];
      outf[2 * p] = x * cs.x - y * cs.y;
      outf[2 * p + 1] = x * cs.y + y * cs.x;
    }
  }
}

template <typename T>
__global__ void est_prep_k(const T* __restrict__ k, int64_t j0, int64_t nk, int hkv, int dim,
                           const float2* __restrict__ rope, float* __restrict__ kn) {
  const int P = dim / 2;
  const int64_t idx = j0 * hkv * P + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // pair
  const int64_t total = nk * hkv * P;
  if (idx >= total) return;
  const int p = int(idx % P);
  const int64_t rowhead = idx / P;          // j * hkv + g
  const int64_t j = rowhead / hkv;
  const float x = load_elem(k, rowhead * dim + 2 * p), y = load_elem(k, rowhead * dim + 2 * p + 1);
  const float2 cs = rope[j * P + p];
  kn[rowhead * dim + 2 * p] = x * cs.x - y * cs.y;
  kn[rowhead * dim + 2 * p + 1] = x * cs.y + y * cs.x;
}

// ---- main tile kernel -----------------------------------------------------
template <typename T, int PASS>
__global__ void __launch_bounds__(kThreads)
est_tile_kernel(EstDev a, float2* __restrict__ stats, const float2* __restrict__ rowstat,
                float* __restrict__ est, float* __restrict__ col_part,
                float* __restrict__ diag_part) {
  extern __shared__ float smem[];
  const int DP = a.dim + 1;
  float* Qn = smem;                       // [64][DP]
  float* Qf = Qn + kRows * DP;            // [64][DP]
  float* Kn = Qf + kRows * DP;            // [64][DP]
  float* Kf = Kn + kKeys * DP;            // [64][DP]
  float* Ps = Kf + kKeys * DP;            // [64][65]

  const int split = blockIdx.x, h = a.h0 + int(blockIdx.y), rt = blockIdx.z;
  const int g = h / a.group;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t row0 = int64_t(rt) * kRows;
  const int rows = int(lcx_min64(kRows, a.block - row0));
  const bool dca = a.pos_mode == 1;

  for (int idx = tid; idx < kRows * a.dim; idx += kThreads) {
    const int r = idx / a.dim, d = idx % a.dim;
    const int64_t src = (int64_t(h) * a.block + row0 + r) * a.dim + d;
    Qn[r * DP + d] = r < rows ? a.qn[src] : 0.f;
    if (dca) Qf[r * DP + d] = r < rows ? a.qf[src] : 0.f;
  }

  float run_m[4], run_s[4], rm[4], rinv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    run_m[i] = -INFINITY;
    run_s[i] = 0.f;
    rm[i] = 0.f;
    rinv[i] = 0.f;
    if (PASS == 2) {
      const int r = ty * 4 + i;
      if (r < rows) {
        const float2 ms = rowstat[int64_t(h) * a.block + row0 + r];
        rm[i] = ms.x;
        rinv[i] = 1.f / ms.y;
      }
    }
  }
  const float inv_sqrt = rsqrtf(float(a.dim));
  const int64_t t_begin = a.tile0 + int64_t(split) * a.tiles_per_split;
  const int64_t t_end = lcx_min64(a.tile_end, t_begin + a.tiles_per_split);
  const T* kraw = reinterpret_cast<const T*>(a.k);

  for (int64_t t = t_begin; t < t_end; ++t) {
    const int64_t j0 = t * kKeys;
    const int64_t gi_lo = a.gbase + row0, gi_hi = a.gbase + row0 + rows - 1;
    // near iff gi - j <= c - 1 (standard mode: always near)
    const bool all_near = !dca || (gi_hi - j0 <= a.c - 1);
    const bool all_far = dca && (gi_lo - (j0 + kKeys - 1) > a.c - 1);
    __syncthreads();
    for (int idx = tid; idx < kKeys * a.dim; idx += kThreads) {
      const int c = idx / a.dim, d = idx % a.dim;
      const int64_t j = j0 + c;
      const bool ok = j < a.nk;
      if (!all_far) Kn[c * DP + d] = ok ? a.kn[(j * a.hkv + g) * a.dim + d] : 0.f;
      if (!all_near) Kf[c * DP + d] = ok ? load_elem(kraw, (j * a.hkv + g) * a.dim + d) : 0.f;
    }
    __syncthreads();

    float acc_n[4][4], acc_f[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc_n[i][jj] = acc_f[i][jj] = 0.f;
    if (!all_far) {
      for (int d = 0; d < a.dim; ++d) {
        float qa[4], kb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) qa[i] = Qn[(ty * 4 + i) * DP + d];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kb[jj] = Kn[(tx * 4 + jj) * DP + d];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc_n[i][jj] = fmaf(qa[i], kb[jj], acc_n[i][jj]);
      }
    }
    if (!all_near) {
      for (int d = 0; d < a.dim; ++d) {
        float qa[4], kb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) qa[i] = Qf[(ty * 4 + i) * DP + d];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kb[jj] = Kf[(tx * 4 + jj) * DP + d];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc_f[i][jj] = fmaf(qa[i], kb[jj], acc_f[i][jj]);
      }
    }

    float lg[4][4];
    bool valid[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
      const int64_t gi = a.gbase + row0 + r;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int64_t j = j0 + tx * 4 + jj;
        valid[i][jj] = (r < rows) && (j < a.nk) && (j <= gi);
        const bool near = !dca || (gi - j <= a.c - 1);
        lg[i][jj] = (near ? acc_n[i][jj] : acc_f[i][jj]) * inv_sqrt;
      }
    }

    if (PASS == 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float tmax = -INFINITY;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (valid[i][jj]) tmax = fmaxf(tmax, lg[i][jj]);
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1)
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
        float tsum = 0.f;
        if (tmax != -INFINITY) {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            if (valid[i][jj]) tsum += expf(lg[i][jj] - tmax);
        }
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, off);
        if (tmax == -INFINITY) continue;
        const float nm = fmaxf(run_m[i], tmax);
        run_s[i] = run_s[i] * expf(run_m[i] - nm) + tsum * expf(tmax - nm);
        run_m[i] = nm;
      }
    } else {
      // probabilities
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const float p = valid[i][jj] ? expf(lg[i][jj] - rm[i]) * rinv[i] : 0.f;
          Ps[r * 65 + tx * 4 + jj] = p;
          if (est && r < rows) {
            const int64_t j = j0 + tx * 4 + jj;
            if (j < a.nk) est[(int64_t(h) * a.block + row0 + r) * a.nk + j] = p;
          }
        }
      }
      __syncthreads();
      if (col_part && tid < kKeys) {
        const int64_t j = j0 + tid;
        if (j < a.nk) {
          float s = 0.f;
          for (int r = 0; r < rows; ++r) s += Ps[r * 65 + tid];
          col_part[(int64_t(rt) * a.hq + h) * a.nk + j] = s;
        }
      }
      if (diag_part && tid < 2 * kKeys - 1) {
        // e = r - c in [-63, 63]; diagonal d = gbase + row0 - j0 + e
        const int e = tid - (kKeys - 1);
        float s = 0.f;
        for (int r = max(0, e); r < rows && r - e < kKeys; ++r) s += Ps[r * 65 + (r - e)];
        diag_part[((int64_t(rt) * a.hq + h) * a.ntiles + t) * 128 + tid] = s;
      }
    }
  }
  if (PASS == 1 && tx == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
      if (r < rows)
        stats[((int64_t(h) * a.nsplit_total) + a.split0 + split) * a.block + row0 + r] =
            make_float2(run_m[i], run_s[i]);
    }
  }
}

// One warp per (head, row): lane l folds splits l, l + 32, ... in ascending order, then a
// fixed xor tree -- deterministic, and ~600 splits (the tensor-core plan) no longer walked
// by one thread (a latency-bound 65 us per chunk before)
__global__ void est_combine_stats(const float2* __restrict__ stats, int h0, int nh, int nsplit,
                                  int64_t block, float2* __restrict__ rowstat) {
  const int64_t x = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (x >= int64_t(nh) * block) return;  // whole warps
  const int h = h0 + int(x / block);
  const int64_t r = x % block;
  const int64_t idx = int64_t(h) * block + r;
  const float2* sp = stats + int64_t(h) * nsplit * block + r;
  float m = -INFINITY;
  for (int s = lane; s < nsplit; s += 32) m = fmaxf(m, sp[int64_t(s) * block].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float sum = 0.f;
  for (int s = lane; s < nsplit; s += 32) {
    const float2 v = sp[int64_t(s) * block];
    if (v.x != -INFINITY) sum += v.y * expf(v.x - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) rowstat[idx] = make_float2(m, sum);
}

// col_score[h][j] = sum over row tiles ascending; slash_score[h][d] = sum over the
// (row tile, key tile) partials that contain d, ascending, then mean / sum.
__global__ void est_combine_lines(const float* __restrict__ col_part,
                                  const float* __restrict__ diag_part, int hq, int h0, int nh,
                                  int nrt, int64_t nk, int64_t block, int64_t gbase,
                                  int64_t ntiles, int slash_mean, float* __restrict__ col,
                                  float* __restrict__ slash) {
  // grid (key blocks, heads): no 64-bit division per thread
  const int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= nk) return;
  const int h = h0 + int(blockIdx.y);
  const int64_t idx = int64_t(h) * nk + x;
  if (col) {
    float s = 0.f;
    for (int rt = 0; rt < nrt; ++rt) s += col_part[(int64_t(rt) * hq + h) * nk + x];
    col[idx] = s;
  }
  if (slash) {
    const int64_t d = x;
    float s = 0.f;
    for (int rt = 0; rt < nrt; ++rt) {
      // tile t contains d iff e = d - (gbase + 64 rt - 64 t) in [-63, 63]
      const int64_t base = gbase + int64_t(rt) * kRows;
      const int64_t num = base - d - (kKeys - 1);  // t_lo = ceil(num / 64), clipped at 0
      const int64_t t_lo = num <= 0 ? 0 : (num + kKeys - 1) / kKeys;
      for (int64_t t = t_lo; t < ntiles; ++t) {
        const int64_t e = d - (base - t * kKeys);
        if (e > kKeys - 1) break;
        if (e < -(kKeys - 1)) continue;
        s += diag_part[((int64_t(rt) * hq + h) * ntiles + t) * 128 + (e + kKeys - 1)];
      }
    }
    const int64_t cnt = lcx_min64(block, nk - d);
    slash[idx] = slash_mean ? s / float(cnt) : s;
  }
}

// Split plan of the CUDA-core estimator: a function of the key tiles only (not of the head
// count or the device), so a head's scores -- and therefore its selection -- are bitwise
// the same whichever subset of heads a call covers (head-sharded multi-GPU runs).
void plan(const EstimateArgs& a, int sm_count, int64_t tiles, int& nsplit, int& tps, int& nrt) {
  (void)sm_count;
  nrt = int((a.block + kRows - 1) / kRows);
  tps = int(std::max<int64_t>(1, (tiles + 63) / 64));
  nsplit = tiles > 0 ? int((tiles + tps - 1) / tps) : 0;
}

bool use_tc(const EstimateArgs& a) {
  return a.k3 != nullptr && a.est == nullptr && est_tc_eligible(a.dtype, a.dim, a.block);
}

EstTcArgs tc_args(const EstimateArgs& a, int sm_count) {
  EstTcArgs t{};
  t.q = a.q;
  t.k = a.k;
  t.hq = a.hq;
  t.hkv = a.hkv;
  t.nk = a.nk;
  t.block = a.block;
  t.pos_mode = a.pos_mode;
  t.c = a.c;
  t.rope = a.rope;
  t.k3 = a.k3;
  t.k3_tiles = a.k3_tiles;
  t.sm_count = sm_count;
  t.h0 = a.h1 > 0 ? a.h0 : 0;
  t.h1 = a.h1 > 0 ? a.h1 : a.hq;
  return t;
}

// CUDA-core tile range of this launch: all tiles, or the mixed near / far tiles left
// over by the tensor-core estimator
void simt_range(const EstimateArgs& a, int sm_count, int64_t& t0, int64_t& t1, int& tc_splits) {
  const int64_t ntiles = (a.nk + kKeys - 1) / kKeys;
  t0 = 0;
  t1 = ntiles;
  tc_splits = 0;
  if (use_tc(a)) {
    EstTcArgs t = tc_args(a, sm_count);
    EstTcPlan pl;
    est_tc_plan(t, pl);
    t0 = pl.far_end;
    t1 = pl.near_begin;
    tc_splits = pl.tc_splits;
  }
}

}  // namespace

void estimate_simt_size(const EstimateArgs& a, Sizer& sz, int sm_count) {
  int64_t t0, t1;
  int tc_splits, nsplit, tps, nrt;
  simt_range(a, sm_count, t0, t1, tc_splits);
  plan(a, sm_count, t1 - t0, nsplit, tps, nrt);
  const int64_t ntiles = (a.nk + kKeys - 1) / kKeys;
  // stats slots: the worst case over chunk sizes (CUDA-core splits of every tile, or the
  // tensor-core estimator's <= 2 x 66 pieces plus the mixed tiles' splits)
  int nsplit_all, tps_all, nrt_all;
  plan(a, sm_count, ntiles, nsplit_all, tps_all, nrt_all);
  const int nst = std::max(nsplit_all, nsplit + est_tc_max_splits()) + 1;
  sz.take<float>(size_t(a.hq) * a.block * a.dim);                       // qn
  if (a.pos_mode == 1) sz.take<float>(size_t(a.hq) * a.block * a.dim);  // qf
  sz.take<float>(size_t(a.nk) * a.hkv * a.dim);                         // kn
  sz.take<float2>(size_t(a.hq) * nst * a.block);                        // stats
  sz.take<float2>(size_t(a.hq) * a.block);                              // rowstat
  if (a.col || a.slash) {
    sz.take<float>(size_t(nrt) * a.hq * a.nk);                 // col_part
    sz.take<float>(size_t(nrt) * a.hq * ntiles * 128);         // diag_part
  }
  if (use_tc(a)) est_tc_size(a.hq, a.hkv, sz);
}

int estimate_simt(lcx_context* ctx, const EstimateArgs& a, Arena& ar, cudaStream_t st) {
  if (a.dim > kMaxDim) return fail(LCX_ERR_CONFIG, "estimator supports head dim <= 128");
  const bool tc = use_tc(a);
  int64_t s0, s1;
  int tc_splits, nsplit, tps, nrt;
  simt_range(a, ctx->sm_count, s0, s1, tc_splits);
  plan(a, ctx->sm_count, s1 - s0, nsplit, tps, nrt);
  if (tc && nrt != 1) return fail(LCX_ERR_INTERNAL, "tensor-core estimator needs block <= 64");
  const int64_t ntiles = (a.nk + kKeys - 1) / kKeys;
  const int nst = std::max(1, nsplit + tc_splits);
  EstDev d{};
  d.q = a.q;
  d.k = a.k;
  d.hq = a.hq;
  d.hkv = a.hkv;
  d.dim = a.dim;
  d.group = a.hq / a.hkv;
  d.nk = a.nk;
  d.block = a.block;
  d.gbase = a.nk - a.block;
  d.pos_mode = a.pos_mode;
  d.c = a.c;
  d.rope = a.rope;
  d.ntiles = ntiles;
  d.tiles_per_split = tps;
  d.nsplit = nsplit;
  d.nrt = nrt;
  d.tile0 = s0;
  d.tile_end = s1;
  d.split0 = tc_splits;
  d.nsplit_total = nst;
  const int h0 = a.h1 > 0 ? a.h0 : 0, nh = (a.h1 > 0 ? a.h1 : a.hq) - h0;
  d.h0 = h0;
  float* qn = ar.take<float>(size_t(a.hq) * a.block * a.dim);
  float* qf = a.pos_mode == 1 ? ar.take<float>(size_t(a.hq) * a.block * a.dim) : nullptr;
  float* kn = ar.take<float>(size_t(a.nk) * a.hkv * a.dim);
  float2* stats = ar.take<float2>(size_t(a.hq) * nst * a.block);
  float2* rowstat = ar.take<float2>(size_t(a.hq) * a.block);
  float* col_part = nullptr;
  float* diag_part = nullptr;
  if (a.col || a.slash) {
    col_part = ar.take<float>(size_t(nrt) * a.hq * a.nk);
    diag_part = ar.take<float>(size_t(nrt) * a.hq * ntiles * 128);
  }
  d.qn = qn;
  d.qf = qf;
  d.kn = kn;
  Arena tc_ar = ar;  // the tensor-core estimator's operands (same offsets in both passes)
  EstTcArgs ta = tc_args(a, ctx->sm_count);
  EstTcPlan pl{};
  if (tc) {
    est_tc_plan(ta, pl);
    ta.nsplit = nst;
    ta.stats = stats;
    ta.rowstat = rowstat;
    ta.col_part = a.col && nrt == 1 ? a.col : col_part;
    ta.diag_part = diag_part;
  }

  const bool bf = a.dtype == LCX_BF16;
  const bool simt = nsplit > 0;
  if (simt) {
    dim3 grid(unsigned(a.block), unsigned(nh));
    if (bf) est_prep_q<__nv_bfloat16><<<grid, 64, 0, st>>>(d);
    else est_prep_q<float><<<grid, 64, 0, st>>>(d);
    LCX_CHECK_LAUNCH();
    const int64_t j0 = s0 * kKeys, j1 = std::min<int64_t>(a.nk, s1 * kKeys);
    const int64_t pairs = (j1 - j0) * a.hkv * (a.dim / 2);
    const unsigned blocks = unsigned((pairs + 255) / 256);
    if (pairs > 0) {
      if (bf)
        est_prep_k<__nv_bfloat16><<<blocks, 256, 0, st>>>(
            reinterpret_cast<const __nv_bfloat16*>(a.k), j0, j1, a.hkv, a.dim, a.rope, kn);
      else
        est_prep_k<float><<<blocks, 256, 0, st>>>(reinterpret_cast<const float*>(a.k), j0, j1,
                                                   a.hkv, a.dim, a.rope, kn);
      LCX_CHECK_LAUNCH();
    }
  }
  const int DP = a.dim + 1;
  const size_t smem = sizeof(float) * (size_t(2 * kRows + 2 * kKeys) * DP + kRows * 65);
  static bool attr_set[4] = {false, false, false, false};
  auto set_attr = [&](const void* fn, int slot) -> int {
    if (!attr_set[slot]) {
      LCX_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(sizeof(float) * ((2 * kRows + 2 * kKeys) *
                                                                   (kMaxDim + 1) + kRows * 65))));
      attr_set[slot] = true;
    }
    return LCX_OK;
  };
  dim3 grid(unsigned(std::max(nsplit, 1)), unsigned(nh), unsigned(nrt));
  // With both estimators, the CUDA-core mixed tiles (a few dozen CTAs) run on a side stream
  // beside the tensor-core pass instead of after it: disjoint stats slots and partial
  // columns / diagonals, joined before the combines that read them.
  const bool side = tc && simt;
  cudaStream_t ss = st;
  if (side) {
    if (!ctx->est_side) {
      LCX_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx->est_side, cudaStreamNonBlocking));
      LCX_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->est_fork, cudaEventDisableTiming));
      LCX_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->est_join, cudaEventDisableTiming));
    }
    ss = ctx->est_side;
  }
  auto fork = [&]() -> int {
    if (side) {
      LCX_CHECK_CUDA(cudaEventRecord(ctx->est_fork, st));
      LCX_CHECK_CUDA(cudaStreamWaitEvent(ss, ctx->est_fork, 0));
    }
    return LCX_OK;
  };
  auto join = [&]() -> int {
    if (side) {
      LCX_CHECK_CUDA(cudaEventRecord(ctx->est_join, ss));
      LCX_CHECK_CUDA(cudaStreamWaitEvent(st, ctx->est_join, 0));
    }
    return LCX_OK;
  };
  // ---- pass 1: row max / sum-exp ----
  LCX_TRY(fork());
  if (tc) {
    Arena ta_ar = tc_ar;
    ta.pass = 1;
    LCX_TRY(est_tc_run(ta, pl, ta_ar, st));
  }
  if (simt) {
    if (bf) {
      LCX_TRY(set_attr((const void*)est_tile_kernel<__nv_bfloat16, 1>, 0));
      LCX_TRY(set_attr((const void*)est_tile_kernel<__nv_bfloat16, 2>, 1));
      est_tile_kernel<__nv_bfloat16, 1><<<grid, kThreads, smem, ss>>>(d, stats, nullptr, nullptr,
                                                                       nullptr, nullptr);
    } else {
      LCX_TRY(set_attr((const void*)est_tile_kernel<float, 1>, 2));
      LCX_TRY(set_attr((const void*)est_tile_kernel<float, 2>, 3));
      est_tile_kernel<float, 1><<<grid, kThreads, smem, ss>>>(d, stats, nullptr, nullptr,
                                                               nullptr, nullptr);
    }
    LCX_CHECK_LAUNCH();
  }
  LCX_TRY(join());
  {
    const int64_t rows = int64_t(nh) * a.block;
    est_combine_stats<<<unsigned((rows * 32 + 255) / 256), 256, 0, st>>>(stats, h0, nh, nst,
                                                                         a.block, rowstat);
    LCX_CHECK_LAUNCH();
  }
  // ---- pass 2: probabilities -> column / diagonal partials ----
  LCX_TRY(fork());
  if (tc) {
    Arena ta_ar = tc_ar;
    ta.pass = 2;
    LCX_TRY(est_tc_run(ta, pl, ta_ar, st));
  }
  // one row tile: every key's column sum has exactly one writer (its tile), so pass 2
  // writes the column scores in place and the combine only forms the diagonals
  float* colp = a.col && nrt == 1 ? a.col : col_part;
  if (simt) {
    if (bf)
      est_tile_kernel<__nv_bfloat16, 2><<<grid, kThreads, smem, ss>>>(d, nullptr, rowstat,
                                                                       a.est, colp, diag_part);
    else
      est_tile_kernel<float, 2><<<grid, kThreads, smem, ss>>>(d, nullptr, rowstat, a.est,
                                                               colp, diag_part);
    LCX_CHECK_LAUNCH();
  }
  LCX_TRY(join());
  if ((a.col && colp != a.col) || a.slash) {
    est_combine_lines<<<dim3(unsigned((a.nk + 255) / 256), unsigned(nh)), 256, 0, st>>>(
        col_part, diag_part, a.hq, h0, nh, nrt, a.nk, a.block, a.nk - a.block, ntiles,
        a.slash_mean, colp != a.col ? a.col : nullptr, a.slash);
    LCX_CHECK_LAUNCH();
  }
  return LCX_OK;
}

}  // namespace lcx
