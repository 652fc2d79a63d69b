/*
 * longctx_b200.h -- C-ABI of the B200-native Qwen2.5-1M sparse + DCA prefill
 * attention path.  Plain pointers and sizes only; no torch / STL types.
 *
 * Each entry point replaces one reference operator (paths relative to
 * /root/reference/proj); the C++ drop-in (include/longctx_b200.hpp) and the
 * Python mirror (paper_2501_15383_b200/longctx.py) are thin layers over these.
 *
 *   lcx_estimate_block      <- longctx::estimate_block      core/include/longctx/sparse.hpp:74-76
 *                                                         (core/src/sparse.cpp:142-188)
 *   lcx_line_scores         <- the row/diagonal reductions of select_critical
 *                                                         (core/src/sparse.cpp:198-217), fused
 *                                                         with the estimator (no B x t1 matrix)
 *   lcx_select_from_scores  <- top_lines + forced lines of select_critical
 *                                                         (core/src/sparse.cpp:15-24, 219-229)
 *   lcx_select_critical     <- longctx::select_critical     core/include/longctx/sparse.hpp:81-82
 *   lcx_sparse_attention    <- longctx::sparse_attention    core/include/longctx/sparse.hpp:87-88
 *   lcx_full_attention      <- longctx::full_attention      core/include/longctx/attention.hpp:57-58
 *   lcx_attention_rel       <- full_attention / sparse_attention with a RelPositionMatrix
 *                                                         override (attention.cpp:173-183)
 *   lcx_chunked_prefill     <- longctx::chunked_prefill     core/include/longctx/sparse.hpp:125-129
 *   lcx_chunked_prefill_host <- the same operator on HOST buffers (the reference
 *                              API's by-value matrices), chunk-pipelined copies
 *   lcx_attention_recall    <- longctx::attention_recall    core/include/longctx/refine.hpp:25-26
 *   lcx_lse_merge           <- (new) log-sum-exp merge of KV-sequence shards (north star (e))
 *   lcx_lse_scale_partial   <- (new) per-shard scaling step of that merge when the sum
 *                              runs as an NCCL collective
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers; every call takes an explicit
 *     cudaStream_t (passed as void*) and is asynchronous unless stated.
 *   - Token-major layouts: Q [n][hq][dim], K and V [n][hkv][dim]; outputs
 *     O [n][hq][dim] fp32, lse [hq][n] fp32.  Query head h reads kv head
 *     h / (hq / hkv) (GQA, attention.cpp:266-273).
 *   - Index lists are int32, sorted ascending, per (chunk, head) with a
 *     fixed capacity stride (cap_v >= vertical budget + 1, cap_s >= slash
 *     budget + last_q).
 *   - Status: 0 = ok, else an lcx_status whose value equals the reference
 *     error kind (errors.hpp:21-32); lcx_last_error() returns the message
 *     (thread-local).  A C-ABI cannot throw; the C++ wrapper rethrows
 *     longctx::Error(kind, message).
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry returns LCX_ERR_CUDA.
 */
#ifndef LONGCTX_B200_H_
#define LONGCTX_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LCX_OK = 0,
  LCX_ERR_DIMENSION = 1,      /* "dimension"          */
  LCX_ERR_CONFIG = 2,         /* "config"             */
  LCX_ERR_DOMAIN = 3,         /* "domain"             */
  LCX_ERR_CAUSALITY = 4,      /* "causality"          */
  LCX_ERR_EMPTY_ROW = 5,      /* "empty_row"          */
  LCX_ERR_EMPTY_CALIBRATION = 6,
  LCX_ERR_CUDA = 100,         /* device / launch failure (no fallback) */
  LCX_ERR_INTERNAL = 101
} lcx_status;

typedef enum { LCX_F32 = 0, LCX_BF16 = 1 } lcx_dtype;

/* PositionMode (sparse.hpp:63) */
typedef enum { LCX_POS_STANDARD = 0, LCX_POS_DCA_CONTINUOUS = 1 } lcx_position_mode;
/* PrefillMode (sparse.hpp:97) */
typedef enum { LCX_PREFILL_FULL = 0, LCX_PREFILL_SPARSE = 1 } lcx_prefill_mode;
/* Kernel path for the attention stage. AUTO = tcgen05 tiles for verticals,
 * band and dense slash runs + CUDA-core gather for isolated slashes when the
 * input is bf16 and dim == 128; SIMT = exact fp32 CUDA-core path for every
 * entry (the fp32 parity path). */
typedef enum { LCX_PATH_AUTO = 0, LCX_PATH_SIMT = 1, LCX_PATH_TC = 2 } lcx_kernel_path;

/* ChunkConfig (dca.hpp:15-25) */
typedef struct {
  int64_t chunk_size;   /* s */
  int64_t train_len;    /* c */
  int64_t local_window; /* w (validated only, dca.cpp:26-29) */
} lcx_chunk_config;

/* SelectionOptions (sparse.hpp:65-69) */
typedef struct {
  int32_t force_sink_column;
  int32_t force_local_band;
  int32_t slash_mean;
} lcx_selection_options;

/* AttentionInput (attention.hpp:15-30), multi-head, device resident. */
typedef struct {
  int64_t n;
  int32_t hq, hkv, dim;
  int32_t dtype;               /* lcx_dtype of q, k, v */
  const void* q;               /* [n][hq][dim]  */
  const void* k;               /* [n][hkv][dim] */
  const void* v;               /* [n][hkv][dim] */
  const int64_t* positions_q;  /* [n] device, or NULL = 0..n-1 */
  const int64_t* positions_k;  /* [n] device, or NULL = 0..n-1 */
  double rope_base;
  double temperature;
} lcx_attention_input;

typedef struct {
  int64_t chunk_len;
  int64_t last_q;
  int64_t budget_vertical;
  int64_t budget_slash;
  int32_t mode;            /* lcx_prefill_mode */
  int32_t position_mode;   /* lcx_position_mode */
  lcx_chunk_config dca;    /* required when position_mode == DCA_CONTINUOUS */
  lcx_selection_options opts;
  int32_t kernel_path;     /* lcx_kernel_path */
  int32_t tc_min_entries;  /* slash entries per 64-key tile to route it to tcgen05 (0 = default) */
  /* KV-line sharding (north star (e)): with shard_count > 1 this call computes, for every
   * row, the partial attention over shard shard_rank's part of each head's selected
   * lines (contiguous parts of the sorted vertical and slash lists); the estimator and
   * selection run in full on every shard (identical lists, no exchange).  out / lse are
   * then partials (o normalised within the shard, lse = -inf where the shard has no
   * entry) to be combined with lcx_lse_scale_partial + a sum over shards.  Sparse mode
   * only.  0 / 1 = unsharded. */
  int32_t shard_rank;
  int32_t shard_count;
  /* Phases of a sharded layer (multi-GPU, paper_2501_15383_b200/shard.py):
   *   LCX_PHASE_ALL     estimator + selection + attention per chunk (the operator);
   *   LCX_PHASE_SELECT  estimator + selection of every chunk only, into the selection
   *                     log (out->sel_*, required), for query heads
   *                     [est_head_begin, est_head_end) -- those heads' list slots are
   *                     written whole (zero past the count), the other heads' slots are
   *                     left untouched (the shards' slots are combined across GPUs);
   *   LCX_PHASE_ATTEND  attention of every chunk only, over the selection log given in
   *                     out->sel_* (required).
   * A head's selection depends only on its own rows and the keys, so splitting the
   * estimator by heads gives every shard bitwise the unsharded lists. */
  int32_t phase;
  int32_t est_head_begin, est_head_end;  /* 0 / 0 = every head */
  /* != 0: record a context-owned CUDA event once chunk c's out / lse rows are final
   * (see lcx_stream_wait_chunk) */
  int32_t record_chunk_events;
  /* chunks [chunk_begin, chunk_end) only (0 / 0 = every chunk): the keys of the earlier
   * chunks are still prepared, their rows (and those of later chunks) are left untouched --
   * a query head's chunks split over GPUs with no exchange (multi-GPU head sharding when a
   * KV head's query heads do not divide evenly over its GPUs) */
  int32_t chunk_begin, chunk_end;
} lcx_prefill_config;

enum { LCX_PHASE_ALL = 0, LCX_PHASE_SELECT = 1, LCX_PHASE_ATTEND = 2 };

typedef struct {
  float* out;              /* [n][hq][dim] */
  float* lse;              /* [hq][n]      */
  /* optional selection log (ChunkSelection, sparse.hpp:99-104), device, may be NULL */
  int32_t* sel_verticals;  /* [nchunks][hq][cap_v] */
  int32_t* sel_nv;         /* [nchunks][hq]        */
  int32_t* sel_slashes;    /* [nchunks][hq][cap_s] */
  int32_t* sel_ns;         /* [nchunks][hq]        */
  int64_t cap_v, cap_s;
  /* optional exact admitted-entry counts per (chunk, head) (CriticalSet::admitted_count
   * restricted to the chunk's rows), device int64 [nchunks][hq], may be NULL */
  int64_t* admitted;
  /* optional sparsity-refinement recall check (north star (d); refine.cpp:51-85 on the
   * chunk's last queries): recall[chunk][head] = mean over the chunk's last
   * min(lastQ, rows) rows of min(1, exp(lse_sparse - lse_full)), lse_full from a dense
   * pass over those rows against keys [0, t1) with the same positions / DCA remap /
   * temperature.  Device float [nchunks][hq], may be NULL; unsharded calls only. */
  float* recall;
} lcx_prefill_output;

/* Execution statistics of the last lcx_chunked_prefill on a context (host side).
 * Counters and stage times are filled only when profiling is enabled
 * (lcx_set_profiling), which records CUDA events around each stage of each chunk
 * and synchronizes once at the end of the call. */
typedef struct {
  int64_t chunks;
  int64_t launches;        /* kernels launched by the call */
  int64_t tc_tiles;        /* 64-key x 128-row tcgen05 tiles executed */
  int64_t simt_entries;    /* admitted entries computed on the CUDA-core gather path */
  double ms_estimate;      /* K1 estimator (all chunks) */
  double ms_select;        /* K2 selection */
  double ms_attention;     /* K3 index build + K4 attention (tcgen05 + CUDA-core) */
  double ms_tc_kernel;     /* the tcgen05 attention kernel alone */
  double ms_total;
  int64_t tc_path;         /* 1: the call ran the tcgen05 kernels, 0: the CUDA-core kernels
                              (fp32 storage, or bf16 with LCX_PATH_AUTO on a chunk length or
                              DCA chunk size that is not a multiple of 128 -- the AUTO
                              fallback also prints a one-time warning on stderr) */
} lcx_prefill_stats;

typedef struct lcx_context lcx_context;

/* ---- context ------------------------------------------------------------ */
int lcx_context_create(int device, lcx_context** out);
int lcx_context_destroy(lcx_context* ctx);
const char* lcx_last_error(void);
const char* lcx_version(void);
/* 1 if the current device is sm_100 class and kernels can launch. */
int lcx_device_ok(int device);
/* Enables per-stage CUDA-event timing inside lcx_chunked_prefill (synchronizing). */
int lcx_set_profiling(lcx_context* ctx, int enabled);
/* Per-chunk device time (ms, estimator through attention) of the last chunked prefill
 * run with profiling on: *count = number of chunks; up to cap values copied to out (may
 * be NULL).  The measured costs a DCPP chunk schedule is fitted to (engine_sim.cpp:117-166,
 * longctx::b200::measure_chunk_costs). */
int lcx_get_chunk_ms(lcx_context* ctx, float* out, int64_t cap, int64_t* count);
int lcx_get_stats(lcx_context* ctx, lcx_prefill_stats* out);
/* Debug: record CTA-0 per-tile clock64 timestamps of the tcgen05 attention
 * pipeline (512 tiles x 8 columns) and copy them to host_out (may be NULL). */
int lcx_debug_trace(lcx_context* ctx, int enable, long long* host_out);

/* ---- estimator (part a) -------------------------------------------------- */
/* estimate_block: q_rows are the trailing nq rows of the key timeline k[0:nk]
 * (queries trail the keys, sparse.cpp:157-158).  est_out [hq][block][nk] fp32,
 * block = min(last_q, nq).  pos_mode/cfg as in the reference; rope_base from
 * the input (positions are token indices; no temperature, sparse.cpp:159). */
int lcx_estimate_block(lcx_context* ctx, const lcx_attention_input* in, int64_t q_row0,
                       int64_t nq, int64_t nk, int64_t last_q, int32_t pos_mode,
                       const lcx_chunk_config* cfg, float* est_out, void* stream);

/* Fused estimator + line reductions: col_score[hq][nk] and slash_score[hq][nk]
 * exactly as select_critical forms them from the estimate (sum over rows,
 * mean (or sum) over each diagonal's present entries). */
int lcx_line_scores(lcx_context* ctx, const lcx_attention_input* in, int64_t q_row0,
                    int64_t nq, int64_t nk, int64_t last_q, int32_t pos_mode,
                    const lcx_chunk_config* cfg, int32_t slash_mean, float* col_score,
                    float* slash_score, void* stream);

/* ---- selection (part a) -------------------------------------------------- */
/* top-budget columns / diagonals by (score desc, index asc), plus forced lines,
 * sorted unique.  scores [heads][n]; block = estimator rows (forced band width). */
int lcx_select_from_scores(lcx_context* ctx, const float* col_score, const float* slash_score,
                           int32_t heads, int64_t n, int64_t block, int64_t budget_vertical,
                           int64_t budget_slash, const lcx_selection_options* opts,
                           int32_t* verticals, int32_t* nv, int64_t cap_v, int32_t* slashes,
                           int32_t* ns, int64_t cap_s, void* stream);

/* select_critical from an estimate matrix est [heads][block][n] (fp32). */
int lcx_select_critical(lcx_context* ctx, const float* est, int32_t heads, int64_t block,
                        int64_t n, int64_t budget_vertical, int64_t budget_slash,
                        const lcx_selection_options* opts, int32_t* verticals, int32_t* nv,
                        int64_t cap_v, int32_t* slashes, int32_t* ns, int64_t cap_s,
                        void* stream);

/* ---- attention (parts b, c) ---------------------------------------------- */
/* sparse_attention over one critical set per query head (lists [hq][cap]).
 * use_dca != 0: rel_override = dca_position_matrix(n, *dca) (sparse.cpp:400-413). */
int lcx_sparse_attention(lcx_context* ctx, const lcx_attention_input* in,
                         const int32_t* verticals, const int32_t* nv, int64_t cap_v,
                         const int32_t* slashes, const int32_t* ns, int64_t cap_s,
                         int32_t use_dca, const lcx_chunk_config* dca, int32_t kernel_path,
                         float* out, float* lse, void* stream);

/* Dense causal attention (attention.cpp:142-185); use_dca as above. */
int lcx_full_attention(lcx_context* ctx, const lcx_attention_input* in, int32_t use_dca,
                       const lcx_chunk_config* dca, int32_t kernel_path, float* out, float* lse,
                       void* stream);

/* Attention with an explicit relative-position matrix rel [n][n] (device int64):
 * logit(i, j) = rope(q_i, rel[i][j]) . k_j (the reference's RelPositionMatrix
 * override, attention.cpp:173-183 / sparse.cpp:400-413).  verticals == NULL: dense
 * causal (full_attention); else the sparse lists as in lcx_sparse_attention.
 * Exact fp32 CUDA-core path. */
int lcx_attention_rel(lcx_context* ctx, const lcx_attention_input* in, const int32_t* verticals,
                      const int32_t* nv, int64_t cap_v, const int32_t* slashes,
                      const int32_t* ns, int64_t cap_s, const int64_t* rel, float* out,
                      float* lse, void* stream);

/* The operator: chunked prefill over all heads and chunks of one layer. */
int lcx_chunked_prefill(lcx_context* ctx, const lcx_attention_input* in,
                        const lcx_prefill_config* cfg, lcx_prefill_output* out, void* stream);

/* Host-buffer entry of the operator -- what the reference's by-value API
 * (chunked_prefill taking host matrices, sparse.hpp:125-129) maps onto.
 * in->q / k / v / positions_* and every out-> pointer are HOST pointers
 * (page-locked memory gives full copy / compute overlap; a pageable output buffer
 * works but makes each chunk's copy-out block the enqueue of the next chunk).
 * Chunk c's Q/K/V rows are copied host-to-device on a copy stream while
 * earlier chunks compute; chunk c's output rows, lse and selections are copied
 * back on a second stream as soon as chunk c is final.  Device staging is
 * owned by the context.  Synchronous: returns once every host output is
 * written (or on the first error). */
int lcx_chunked_prefill_host(lcx_context* ctx, const lcx_attention_input* in,
                             const lcx_prefill_config* cfg, lcx_prefill_output* out,
                             void* stream);

/* Makes `stream` wait until chunk `chunk` of the last lcx_chunked_prefill on this context
 * (run with record_chunk_events) has its out / lse rows final: per-chunk work on another
 * stream -- e.g. the log-sum-exp merge of KV-line shards over NCCL -- overlaps the
 * attention of the chunks after it. */
int lcx_stream_wait_chunk(lcx_context* ctx, int64_t chunk, void* stream);

/* ---- recall (part d) ----------------------------------------------------- */
/* per_query[i] = min(1, exp(lse_s - lse_f)); LCX_ERR_DOMAIN if any value
 * exceeds 1 + slack (refine.cpp:51-72).  aggregate (host double) = mean.
 * Synchronizes the stream. */
int lcx_attention_recall(lcx_context* ctx, const float* lse_sparse, const float* lse_full,
                         int64_t n, double slack, float* per_query, double* aggregate,
                         void* stream);

/* ---- KV-sequence sharding (part e) --------------------------------------- */
/* In-place log-sum-exp merge of G shard partials: o[g] [rows][dim] fp32
 * (normalized within the shard), lse[g] [rows] (-inf for an empty shard).
 * Writes the merged output/lse into out / lse_out. */
int lcx_lse_merge(lcx_context* ctx, const float* o_parts, const float* lse_parts, int32_t parts,
                  int64_t rows, int32_t dim, float* out, float* lse_out, void* stream);

/* Shard-side half of the log-sum-exp merge of KV-line shards: given this shard's partial
 * o [n][hq][dim] (normalised) and the lse of ALL shards lse_all [parts][hq][n], writes
 * lse_out [hq][n] = logsumexp_g lse_g and scales o in place by exp(lse_own - lse_out)
 * (0 where lse_own = -inf), so that summing the scaled partials over shards (an NCCL
 * reduce-scatter / all-reduce) yields the exact attention output. */
int lcx_lse_scale_partial(lcx_context* ctx, float* o, const float* lse_own, const float* lse_all,
                          int32_t parts, int64_t n, int32_t hq, int32_t dim, float* lse_out,
                          void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LONGCTX_B200_H_ */
