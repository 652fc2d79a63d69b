// K1 on tcgen05 (est_tc.cu): bf16, head dim 128, estimator rows <= 64.
#pragma once

#include "lcx_internal.cuh"

namespace lcx {

struct EstTcParams {
  int group, pairs_per_group, npairs;
  int pair0;                 // first head pair of this call (items cover pairs [pair0, ...))
  int ncall_pairs;           // head pairs of this call
  int64_t nk;
  int block;
  int64_t ntiles_k;          // 64-key tiles of the K3 buffer (its row stride)
  int64_t ntiles;            // 64-key tiles of this chunk's keys [0, nk)
  int64_t far_end, near_begin;
  int per;                   // tiles per CTA piece
  float scale_log2;          // log2(e) / sqrt(D)  (no temperature, sparse.cpp:159)
  int nsplit;                // stats slots per head
  float2* stats;             // [hq][nsplit][block] (max, sum-exp) natural-log domain
  const float2* rowstat;     // [hq][block]
  float* col_part;           // [hq][nk]
  float* diag_part;          // [hq][ntiles][128]
  const float* qinv;         // [far][npairs][128] power-of-two factor of each Q row
  const float* kinv;         // [hkv][ntiles_k] power-of-two factor of each key tile
};

struct EstTcArgs {
  const void* q; const void* k;  // [n][hq][128], [n][hkv][128] bf16
  int hq, hkv;
  int64_t nk, block;
  int pos_mode;
  int64_t c;
  const float2* rope;
  const void* k3; int64_t k3_tiles;  // scaled fp16 key tiles (est_tc_prepare_keys)
  int sm_count;
  int h0, h1;                    // query heads of the call: pairs meeting [h0, h1)
  int pass;                      // 1 or 2
  int nsplit;                    // total stats slots (TC pieces + CUDA-core mixed splits)
  float2* stats; const float2* rowstat; float* col_part; float* diag_part;
};

struct EstTcPlan {
  int npairs;          // all head pairs (q3 layout)
  int pair0, pair1;    // pairs of this call
  int64_t ntiles, far_end, near_begin;
  int per, tc_splits, items;
};

bool est_tc_eligible(int dtype, int dim, int64_t block);
size_t est_tc_k3_bytes(int64_t n, int hkv);
int est_tc_prepare_keys(const void* k, int64_t r0, int64_t r1, int hkv, int64_t ntiles,
                        const float2* rope, void* k3, cudaStream_t st);
void est_tc_size(int hq, int hkv, Sizer& sz);
void est_tc_plan(const EstTcArgs& a, EstTcPlan& pl);
int est_tc_max_splits();  // upper bound of EstTcPlan::tc_splits (stats slots)
int est_tc_run(const EstTcArgs& a, const EstTcPlan& pl, Arena& ar, cudaStream_t st);

}  // namespace lcx
