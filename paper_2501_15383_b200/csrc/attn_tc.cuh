// Host-visible declarations of the tensor-core attention path (attn_tc.cu).
#pragma once

#include <cuda.h>

#include "lcx_internal.cuh"

namespace lcx {

struct TcParams {
  const __nv_bfloat16* q;
  int hq, hkv, group;
  int64_t n;           // keys visible
  int64_t t1;          // chunk end (row bound)
  int64_t block0;      // first 128-row block index
  int nblocks;
  int nitems;
  int rel_mode;        // 0 standard, 1 dca
  int64_t s, c;
  const int64_t* pos_q;
  const float2* rope;
  float scale_log2;
  int dense;
  const int32_t* verts; const int32_t* nv; int64_t cap_v;
  // compacted verticals: per DCA key chunk m a 64-aligned segment starting at vbase[h][m]
  const int32_t* ckeys; const int32_t* vbase; const int32_t* vfirst; int64_t capp; int nseg_k;
  int64_t seg_len;     // key-chunk length used for the segments (s, or >= n when standard)
  int64_t ntiles_k;    // 64-key tiles of the prepared K / V^T (npad / 64)
  const int32_t* tc_u; const int32_t* n_tc_u; int64_t cap_u;
  const uint32_t* sbits; const uint32_t* vbits; int64_t words;
  float* out; float* lse; int64_t lse_stride;
  int64_t* tile_count;  // optional: executed tiles (atomicAdd)
  long long* trace;     // optional: CTA-0 per-tile timestamps [kTraceTiles][8]
  void* plans;          // workspace: per-item tile plans (filled by plan_items_kernel)
  // key-window pass: slash tiles with keys in [key_lo, key_hi) only; vertical tiles only
  // when vert_pass; init = continue from the running (out, lse) of the rows
  int64_t key_lo, key_hi;
  int vert_pass, init;
  const int* win_flags; int win;  // optional: skip the pass when win_flags[win] == 0
  int* item_counter;  // optional: dynamic item queue (reset by plan_items_kernel)
  // pre-swizzled tiled operands (TcBuffers), loaded with 1-D bulk copies
  const __nv_bfloat16 *khi, *klo, *kchi, *kclo;
  const __half *vt, *vct;
};

struct TcBuffers {
  __nv_bfloat16 *khi = nullptr, *klo = nullptr, *kchi = nullptr, *kclo = nullptr;
  float* kf = nullptr;  // [n][hkv][128] rope(k_j, kpos(j)) in fp32 (CUDA-core gather)
  __half *vt = nullptr, *vct = nullptr;
  int32_t *ckeys = nullptr, *vbase = nullptr, *vfirst = nullptr;
  int64_t npad = 0, capp = 0, seg_len = 0;
  int nseg_k = 0;
  CUtensorMap m_khi, m_klo, m_vt, m_kchi, m_kclo, m_vct;
};

// layout of the tensor-core buffers (Arena or Sizer)
template <class A>
void tc_layout(A& ar, int64_t n, int hq, int hkv, int64_t cap_v, int64_t seg_len, TcBuffers& B) {
  B.npad = (n + 63) / 64 * 64;
  B.seg_len = seg_len;
  B.nseg_k = int((n + seg_len - 1) / seg_len);
  B.capp = (cap_v + 63) / 64 * 64 + 64 * (B.nseg_k + 1);
  const int64_t capp = B.capp;
  B.ckeys = ar.template take<int32_t>(size_t(hq) * capp);
  B.vbase = ar.template take<int32_t>(size_t(hq) * (B.nseg_k + 1));
  B.vfirst = ar.template take<int32_t>(size_t(hq) * (B.nseg_k + 1));
  B.khi = ar.template take<__nv_bfloat16>(size_t(B.npad) * hkv * 128);  // tiled: whole tiles
  B.klo = ar.template take<__nv_bfloat16>(size_t(B.npad) * hkv * 128);
  B.kf = ar.template take<float>(size_t(n) * hkv * 128);  // rotated K, fp32, row-major
  B.vt = ar.template take<__half>(size_t(hkv) * 128 * B.npad);
  B.kchi = ar.template take<__nv_bfloat16>(size_t(hq) * capp * 128);
  B.kclo = ar.template take<__nv_bfloat16>(size_t(hq) * capp * 128);
  B.vct = ar.template take<__half>(size_t(hq) * 128 * capp);
}

// Tiled operand layout: every 64-key tile is a run of 64-row x 128-byte blocks stored
// already in the SWIZZLE_128B shared-memory image (16-byte chunk c of row r at chunk
// c ^ (r & 7)), so one contiguous bulk copy lands a ready UMMA operand.
__host__ __device__ __forceinline__ int sw128_chunk(int row, int chunk) {
  return chunk ^ (row & 7);
}

// 3-D tiled tensor map, SWIZZLE_128B, L2 promotion 256 B
int make_tmap3(CUtensorMap* m, CUtensorMapDataType dt, void* base, uint64_t d0, uint64_t d1,
               uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0,
               uint32_t b1, uint32_t b2);

int tc_prepare(const void* k, const void* v, int64_t n, int hq, int hkv, const int64_t* pos_k,
               int rel_mode, int64_t s, const float2* rope, TcBuffers& B, cudaStream_t st);
int tc_prepare_maps(int hq, int hkv, TcBuffers& B);
// rotated K (hi/lo) and V^T for key rows [r0, r1) only (chunk-incremental preparation)
int tc_prepare_rows(const void* k, const void* v, int64_t n, int64_t r0, int64_t r1, int hkv,
                    const int64_t* pos_k, int rel_mode, int64_t s, const float2* rope,
                    const TcBuffers& B, cudaStream_t st);
int tc_compact(const void* v, int hq, int hkv, const int32_t* verts, const int32_t* nv,
               int64_t cap_v, TcBuffers& B, cudaStream_t st);
int tc_classify(const int32_t* slashes, const int32_t* ns, int64_t cap_s, int hq, int64_t U,
                int min_entries, int32_t* hist_ws, int32_t* tc_u, int32_t* n_tc_u, int64_t cap_u,
                int4* segs, int32_t* nseg, int64_t cap_seg, cudaStream_t st);
int tc_attention(const TcParams& p, const TcBuffers& B, int sm_count, cudaStream_t st);
size_t tc_plan_bytes();  // bytes per work item for the tile plans
// per-key-window work flags of a chunk's slash tiles (tc_flags) and segments (g_flags)
int tc_window_flags(const int32_t* tc_u, const int32_t* n_tc_u, int64_t cap_u, const int4* segs,
                    const int32_t* nseg, int64_t cap_seg, int hq, int64_t t0, int64_t t1,
                    int64_t W, int nwin, int* tc_flags, int* g_flags, cudaStream_t st);
int admitted_counts(const int32_t* verts, const int32_t* nv, int64_t cap_v,
                    const int32_t* slashes, const int32_t* ns, int64_t cap_s, int hq,
                    int64_t t0, int64_t t1, int64_t* out, cudaStream_t st);

}  // namespace lcx
