// K4b: CUDA-core gather of the isolated slash entries in tensor-core mode (attn_gather.cu).
#pragma once

#include "lcx_internal.cuh"

namespace lcx {

struct GatherArgs {
  const __nv_bfloat16* q;                          // [n][hq][128]
  const float* kf;                                 // [n][hkv][128] rope(k_j, kpos(j)) fp32
  const __nv_bfloat16* v;                          // [n][hkv][128]
  int hq, hkv, group;
  int64_t row_begin, row_end;                      // rows (row_begin % 128 == 0)
  int64_t key_lo, key_hi;                          // only entries with key in [key_lo, key_hi)
  const int* win_flags; int win;                   // optional: skip an empty key window
  int rel_mode;                                    // 0 standard, 1 DCA
  int64_t s, c;
  const int64_t* pos_q; const int64_t* pos_k;     // standard mode (nullptr = iota)
  const float2* rope;                              // fp64-derived table, >= 64 rows
  float scale_log2;                                // log2(e) / (temperature sqrt(D))
  // the FULL selection (self-fallback decision) and whether this shard owns fallbacks
  const int32_t* verts; const int32_t* nv; int64_t cap_v;
  const int32_t* slashes; const int32_t* ns; int64_t cap_s;
  int do_fallback;
  const uint32_t* vbits; int64_t words;
  const int4* segs; const int32_t* nseg; int64_t cap_seg;  // [hq][2 halves][cap_seg]
  float* out; float* lse; int64_t lse_stride;      // tensor-core partial in, merged out
  int64_t* simt_count;
  int head_fast;                                   // grid: heads fastest (single pass)
};

int attention_gather(const GatherArgs& a, cudaStream_t st);

}  // namespace lcx
