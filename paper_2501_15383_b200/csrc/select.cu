// K2 -- deterministic top-k line selection.
//
// Restates top_lines + the forced inclusions of select_critical (reference
// core/src/sparse.cpp:15-24 and 219-229): the k lines with the largest score,
// ties broken toward the smaller index (a total order, so the reference's
// stable_sort and this radix select pick the same set), then the forced prefix
// [0, prefix_len) (column 0 for forceSink, offsets [0, block) for
// forceLocalBand), sorted unique.
//
// One thread-block CLUSTER of 8 CTAs per head (each CTA one contiguous eighth of the
// scores): MSB-first 8-bit radix select on the order-preserving uint32 image of the
// fp32 score finds the k-th largest key T and how many keys equal to T must be taken --
// the per-CTA digit histograms are combined through distributed shared memory between
// cluster barriers, so the 4 passes + the emission are one launch that reads the scores
// at full-chip bandwidth instead of one SM's; the emission then writes, in ascending
// index order, every index with key > T and the first `need` indices with key == T
// (CTA r after CTAs < r: offsets from the other CTAs' counts via DSMEM).  Output is
// sorted by construction.
#include <cooperative_groups.h>

#include "lcx_internal.cuh"

namespace lcx {
namespace {

constexpr int kT = 1024;

__device__ __forceinline__ int block_excl_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < int(blockDim.x >> 5) ? warp_sums[lane] : 0;
    int ws = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ws, o);
      if (lane >= o) ws += y;
    }
    warp_sums[lane] = ws - w;  // exclusive prefix of warp sums
    if (lane == 31) *total = ws;
  }
  __syncthreads();
  const int r = warp_sums[wid] + x - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kT)
select_kernel(const float* __restrict__ scores, int64_t n, int64_t k, int64_t prefix_len,
              int32_t* __restrict__ out, int32_t* __restrict__ count, int64_t cap) {
  __shared__ int hist[256];
  __shared__ int warp_sums[32];
  __shared__ int total;
  __shared__ uint32_t sh_prefix;
  __shared__ int64_t sh_remaining;
  const int h = blockIdx.x;
  const float* sc = scores + int64_t(h) * n;
  int32_t* o = out + int64_t(h) * cap;
  const int tid = threadIdx.x;

  if (k >= n) {  // every line (budget clamps, test_sparse.cpp:123-129)
    for (int64_t i = tid; i < n; i += kT) o[i] = int32_t(i);
    if (tid == 0) count[h] = int32_t(n);
    return;
  }
  for (int64_t i = tid; i < prefix_len; i += kT) o[i] = int32_t(i);
  if (k <= 0) {
    if (tid == 0) count[h] = int32_t(prefix_len);
    return;
  }

  uint32_t prefix = 0, mask = 0;
  int64_t remaining = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += kT) hist[b] = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += kT) {
      const uint32_t u = float_to_ordered(sc[i]);
      if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int64_t cum = 0;
      int chosen = 0;
      for (int dgt = 255; dgt >= 0; --dgt) {
        if (cum + hist[dgt] >= remaining) {
          chosen = dgt;
          break;
        }
        cum += hist[dgt];
      }
      sh_remaining = remaining - cum;
      sh_prefix = prefix | (uint32_t(chosen) << shift);
    }
    __syncthreads();
    prefix = sh_prefix;
    remaining = sh_remaining;
    mask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t T = prefix;
  const int64_t need_eq = remaining;

  int64_t eq_seen = 0, out_seen = 0;
  for (int64_t base = 0; base < n; base += kT) {
    const int64_t i = base + tid;
    uint32_t u = 0;
    if (i < n) u = float_to_ordered(sc[i]);
    const int gt = (i < n) && (u > T);
    const int eq = (i < n) && (u == T);
    const int eq_rank = block_excl_scan(eq, warp_sums, &total);
    const int eq_total = total;
    const int sel = gt || (eq && (eq_seen + eq_rank) < need_eq);
    const int emit = sel && (i >= prefix_len);
    const int pos = block_excl_scan(emit, warp_sums, &total);
    const int emit_total = total;
    if (emit) o[prefix_len + out_seen + pos] = int32_t(i);
    eq_seen += eq_total;
    out_seen += emit_total;
  }
  if (tid == 0) count[h] = int32_t(prefix_len + out_seen);
}

constexpr int kCl = 8;      // CTAs per head (cluster)
constexpr int kCT = 512;    // threads per CTA

// distributed shared memory: address of `p` in cluster CTA `rank`, loads, cluster barrier
__device__ __forceinline__ uint32_t dsmem(const void* p, int rank) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p)), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ int ld_dsmem_i32(uint32_t a) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_dsmem_i64(uint32_t a) {
  long long v;
  asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ int cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return int(r);
}

__global__ void __launch_bounds__(kCT)
select_cluster_kernel(const float* __restrict__ scores, int64_t n, int64_t k,
                      int64_t prefix_len, int32_t* __restrict__ out,
                      int32_t* __restrict__ count, int64_t cap) {
  constexpr int kW = kCT / 32;         // warps per CTA
  __shared__ int whist[kW][256];       // per-warp digit histograms (no atomic contention)
  __shared__ int hist[256];            // this CTA's histogram, read by the cluster via DSMEM
  __shared__ int warp_sums[32];
  __shared__ int total;
  __shared__ uint32_t sh_prefix;
  __shared__ long long sh_remaining;
  __shared__ long long sh_cnt[2];      // [0] emitted by this CTA, [1] its equal count
  __shared__ int w_gt[kW], w_eq[kW], w_eqp[kW];  // per-warp counts of the emission
  __shared__ long long w_base[kW], w_take[kW];
  const int rank = cluster_rank();
  const int h = blockIdx.x / kCl;
  const float* sc = scores + int64_t(h) * n;
  int32_t* o = out + int64_t(h) * cap;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t lo = n * rank / kCl, hi = n * (rank + 1) / kCl;
  // (the k >= n and k <= 0 cases are handled by the single-CTA kernel)
  if (rank == 0)
    for (int64_t i = tid; i < prefix_len; i += kCT) o[i] = int32_t(i);
  uint32_t prefix = 0, mask = 0;
  long long remaining = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = tid; b < kW * 256; b += kCT) (&whist[0][0])[b] = 0;
    __syncthreads();
    for (int64_t i = lo + tid; i < hi; i += kCT) {
      const uint32_t u = float_to_ordered(sc[i]);
      if ((u & mask) == prefix) atomicAdd(&whist[wid][(u >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid < 256) {
      int c = 0;
#pragma unroll
      for (int w = 0; w < kW; ++w) c += whist[w][tid];
      hist[tid] = c;
    }
    cluster_sync();  // all eighths histogrammed
    // digit d = 255 - t for thread t: the cluster-wide count, then the count of all larger
    // digits (exclusive scan in descending digit order); exactly one digit straddles k
    int c = 0;
    if (tid < 256)
      for (int r = 0; r < kCl; ++r) c += ld_dsmem_i32(dsmem(&hist[255 - tid], r));
    const int before = block_excl_scan(c, warp_sums, &total);
    if (tid < 256 && before < remaining && before + c >= remaining) {
      sh_remaining = remaining - before;
      sh_prefix = prefix | (uint32_t(255 - tid) << shift);
    }
    cluster_sync();  // the choice is published; every CTA read every histogram
    prefix = sh_prefix;
    remaining = sh_remaining;
    mask |= 255u << shift;
  }
  const uint32_t T = prefix;
  const long long need_eq = remaining;
  // ---- emission: warp w of the CTA owns a contiguous slice of the CTA's eighth, so the
  // output (ascending indices) needs only per-warp offsets -- no block barrier per element
  const int64_t span = hi - lo;
  const int64_t wlo = lo + span * wid / kW, whi = lo + span * (wid + 1) / kW;
  {  // pass A: per-warp counts
    int gt = 0, eq = 0, eqp = 0;
    for (int64_t i = wlo + lane; i < whi; i += 32) {
      const uint32_t u = float_to_ordered(sc[i]);
      gt += (u > T) && (i >= prefix_len);
      eq += (u == T);
      eqp += (u == T) && (i < prefix_len);
    }
    gt = __reduce_add_sync(0xffffffffu, gt);
    eq = __reduce_add_sync(0xffffffffu, eq);
    eqp = __reduce_add_sync(0xffffffffu, eqp);
    if (lane == 0) {
      w_gt[wid] = gt;
      w_eq[wid] = eq;
      w_eqp[wid] = eqp;
    }
  }
  __syncthreads();
  if (tid == 0) {
    long long e = 0;
    for (int w = 0; w < kW; ++w) e += w_eq[w];
    sh_cnt[1] = e;
  }
  cluster_sync();
  if (tid == 0) {
    // ties go to the lowest indices: this eighth takes the equals ranked
    // [eq_before, eq_before + take) in index order, warp by warp
    long long eq_before = 0;
    for (int r = 0; r < rank; ++r) eq_before += ld_dsmem_i64(dsmem(&sh_cnt[1], r));
    long long take = need_eq - eq_before;
    take = take < 0 ? 0 : (take > sh_cnt[1] ? sh_cnt[1] : take);
    long long emitted = 0;
    for (int w = 0; w < kW; ++w) {
      const long long tw = take < w_eq[w] ? take : w_eq[w];
      take -= tw;
      w_take[w] = tw;
      // the warp's taken equals are its first tw in index order; those inside the forced
      // prefix are written already (prefix indices come first within the slice)
      w_base[w] = emitted;
      emitted += w_gt[w] + tw - (tw < w_eqp[w] ? tw : w_eqp[w]);
    }
    sh_cnt[0] = emitted;
  }
  cluster_sync();
  long long base = prefix_len;
  for (int r = 0; r < rank; ++r) base += ld_dsmem_i64(dsmem(&sh_cnt[0], r));
  {  // pass B: emit the warp's slice in ascending index order
    const long long wb = base + w_base[wid], tw = w_take[wid];
    long long eq_seen = 0, out_seen = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t b0 = wlo; b0 < whi; b0 += 32) {
      const int64_t i = b0 + lane;
      uint32_t u = 0;
      if (i < whi) u = float_to_ordered(sc[i]);
      const bool g = (i < whi) && (u > T);
      const bool e = (i < whi) && (u == T);
      const unsigned em = __ballot_sync(0xffffffffu, e);
      const bool sel = g || (e && eq_seen + __popc(em & lt) < tw);
      const bool emit = sel && (i >= prefix_len);
      const unsigned om = __ballot_sync(0xffffffffu, emit);
      if (emit) o[wb + out_seen + __popc(om & lt)] = int32_t(i);
      eq_seen += __popc(em);
      out_seen += __popc(om);
    }
  }
  if (rank == kCl - 1 && tid == 0) count[h] = int32_t(base + sh_cnt[0]);
  cluster_sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

// col[h][j] = sum_r est[h][r][j]; slash[h][d] = (sum_r est[h][r][gi_r - d]) / cnt
// (sparse.cpp:198-217), ascending r.
__global__ void est_line_scores(const float* __restrict__ est, int heads, int64_t block,
                                int64_t n, int slash_mean, float* __restrict__ col,
                                float* __restrict__ slash) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= int64_t(heads) * n) return;
  const int h = int(idx / n);
  const int64_t x = idx % n;
  const float* e = est + int64_t(h) * block * n;
  float cs = 0.f, ss = 0.f;
  int64_t cnt = 0;
  for (int64_t r = 0; r < block; ++r) {
    const int64_t gi = n - block + r;
    if (x <= gi) cs += e[r * n + x];
    if (x <= gi) {
      ss += e[r * n + (gi - x)];
      ++cnt;
    }
  }
  col[idx] = cs;
  slash[idx] = cnt == 0 ? -INFINITY : (slash_mean ? ss / float(cnt) : ss);
}

}  // namespace

int select_lines(const float* scores, int heads, int64_t n, int64_t k, int force_prefix,
                 int64_t prefix_len, int32_t* out, int32_t* count, int64_t cap,
                 cudaStream_t st) {
  const int64_t pl = force_prefix ? std::min<int64_t>(prefix_len, n) : 0;
  if (pl + std::min<int64_t>(k, n) > cap && std::min<int64_t>(k, n) < n)
    return fail(LCX_ERR_DIMENSION, "selection capacity too small for budget + forced lines");
  if (k >= n && n > cap) return fail(LCX_ERR_DIMENSION, "selection capacity too small");
  if (n >= int64_t(kCl) * kCT && k > 0 && k < n) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(heads * kCl));
    lc.blockDim = dim3(kCT);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    LCX_CHECK_CUDA(cudaLaunchKernelEx(&lc, select_cluster_kernel, scores, n, k, pl, out, count,
                                      cap));
  } else
    select_kernel<<<heads, kT, 0, st>>>(scores, n, k, pl, out, count, cap);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

int line_scores_from_est(const float* est, int heads, int64_t block, int64_t n, int slash_mean,
                         float* col, float* slash, cudaStream_t st) {
  const int64_t total = int64_t(heads) * n;
  est_line_scores<<<unsigned((total + 255) / 256), 256, 0, st>>>(est, heads, block, n,
                                                                  slash_mean, col, slash);
  LCX_CHECK_LAUNCH();
  return LCX_OK;
}

}  // namespace lcx
