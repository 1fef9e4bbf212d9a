/*
 * dbsa_b200.h -- C ABI of libdbsa_sm100a.so, the B200 (sm_100a) hot path of
 * Dynamic Block-Sparse Attention (arXiv 2503.08640).
 *
 * The reference package (/root/reference/pkg/src/dbsa) has no FFI: its only
 * numeric seam is `kernels.masked_attention` (kernels.py:73-100), called once
 * per (layer, kv-head) from `model._forward` (model.py:338-351), and its
 * data-movement / selection steps are plain numpy (kvstore.py:70-106,
 * kvstore.py:188-221, retrieval.py:352-388).  Each entry point below replaces
 * one of those sites; the Python package `paper_2503_08640_b200` binds them
 * with ctypes behind the reference's own Python API.
 *
 * Conventions
 *   - extern "C", plain pointers and int64_t sizes; no torch types.
 *   - every device buffer is allocated and owned by the caller; the library
 *     never allocates persistent device memory.
 *   - every call takes an explicit cudaStream_t (passed as void*) and is
 *     asynchronous on it; the library keeps no global mutable state, so calls
 *     are reentrant across host threads (reference threading contract:
 *     bench.py:147-150, pipeline.py:322-327).
 *   - return 0 on success; a non-zero DBSA_ERR_* code maps 1:1 onto the
 *     reference exception hierarchy (errors.py:4-29); dbsa_last_error()
 *     returns the thread-local message of the last failure.
 *
 * KV page pool layout (component K2, replaces SegmentedKVCache storage,
 * kvstore.py:36-106).  One pool per cache, bf16:
 *   K   [L][Hkv][rows][HDP]   keys ROTATED at their original positions
 *   V^T [L][Hkv][HDP][rows]   values, transposed (token dim contiguous)
 * rows = n_pages * 64; a group (block) owns a contiguous run of whole pages,
 * pages never span groups; HDP = head_dim padded to {16,32,64,128}, padding
 * columns are zero.  Selecting groups is pointer indirection into this pool
 * (segment tables below), never a copy (replaces assemble, kvstore.py:188-221).
 */
#ifndef DBSA_B200_H
#define DBSA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBSA_ABI_VERSION 12
#define DBSA_PAGE_TOKENS 64

/* Error codes -> reference exceptions (errors.py:4-29). */
#define DBSA_OK 0
#define DBSA_ERR_SHAPE 1       /* ShapeError       errors.py:8  */
#define DBSA_ERR_MASK 2        /* MaskError        errors.py:12 */
#define DBSA_ERR_CONFIG 3      /* ConfigError      errors.py:16 */
#define DBSA_ERR_VALIDATION 4  /* ValidationError  errors.py:20 */
#define DBSA_ERR_COMPAT 5      /* CompatibilityError errors.py:24 */
#define DBSA_ERR_CUDA 6        /* RuntimeError (driver / launch failure) */

/* Segment kinds. */
#define DBSA_SEG_FULL 0 /* context chunk: every key visible to every row */
#define DBSA_SEG_SELF 1 /* the rows' own tokens: causal, optionally a tree */

/* Output modes of a work. */
#define DBSA_OUT_BF16 0    /* normalized bf16 rows into out */
#define DBSA_OUT_PARTIAL 1 /* fp32 partial O + LSE at part_row0 + row */
#define DBSA_OUT_MAPPED 2  /* rows gathered through the row map (chunk-major stage 2): fp32 partial O + LSE
                              at part_row0 + map.part_tok * gs + (row % gs) */

/* Row map entry of a DBSA_OUT_MAPPED work: work-local token i is map entry
 * q_tok0 + i.  Lets one work stack the rows of MANY queries against one
 * selected chunk (each query's delta differs, so the rope row is per entry). */
typedef struct DbsaRowMap {
  int32_t tok;      /* token index into q */
  int32_t rope_row; /* rope_table row of this token for the work's chunk: tok_pos - delta */
  int32_t part_tok; /* partial slot (in tokens) */
  int32_t pad;
} DbsaRowMap;

/* One unit of attention work = one CTA: up to 128*num_m query rows of one kv
 * head (token-major GQA packing: row r = token (r / gs), head (r % gs)),
 * attending to the segment list [seg_begin, seg_end). */
typedef struct DbsaAttnWork {
  int32_t q_tok0;    /* first token of the slab (index into q / tok_* arrays) */
  int32_t n_tok;     /* tokens in the slab; rows = n_tok * gs */
  int32_t self_tok0; /* token index whose local self index is 0 */
  int32_t kv_head;
  int32_t seg_begin;
  int32_t seg_end;
  int32_t prefix;   /* SELF keys with local index < prefix are visible to all rows */
  int32_t out_mode; /* DBSA_OUT_BF16 / DBSA_OUT_PARTIAL / DBSA_OUT_MAPPED (one segment -- FULL, or SELF
                       with self_tok0 / prefix / tok_lo as for plain works -- every shift 0: the
                       rope row comes from the map) */
  int64_t part_row0; /* partial row base (out_mode 1) */
} DbsaAttnWork;

/* A run of consecutive KV rows of one plane. */
typedef struct DbsaAttnSeg {
  int32_t src;   /* 0 = pool planes, 1 = aux planes */
  int32_t layer; /* layer coordinate inside the planes */
  int32_t row0;  /* first row */
  int32_t n_tok; /* > 0 */
  int32_t kind;  /* DBSA_SEG_FULL / DBSA_SEG_SELF */
  int32_t shift; /* stage-2 re-positioning delta = new start - original start of the
                    chunk: the rows' queries use rope row (tok_pos - shift); 0 = none */
  int32_t pad0, pad1;
} DbsaAttnSeg;

/* Components K1 (stage-1 block-sparse prefill) and K3 (stage-2 split-KV
 * query attention) -- one tcgen05/TMEM/TMA kernel.  Replaces
 * kernels.masked_attention (kernels.py:73-100) as called from
 * model._forward (model.py:327-351) including the rotary application of
 * model.py:327-328: queries are read UNROTATED from `q` and rotated in the
 * prologue with rope_table row (tok_pos[t] - seg.shift): the stage-2
 * re-positioning of kvstore.py:201-218 moved to the query side,
 * R(p_q - delta) q . R(p_orig) k == R(p_q) q . R(p_new) k, with the rotation
 * angle formed in float64 for the exact integer position p_q - delta.
 */
typedef struct DbsaAttnArgs {
  const void *q;        /* bf16, element (t, head, d) at q[t*q_tok_stride + head*head_dim + d] */
  int64_t q_tok_stride; /* elements */
  const int32_t *tok_pos; /* [tokens] rotary position of each query token */
  const int32_t *tok_lo;  /* [tokens] tree mask: lowest visible non-prefix SELF key (local); NULL = 0 */
  const float *rope_table; /* float2 [rope_rows][head_dim/2]: cos, sin of pos*theta^(-2i/hd);
                              rows must cover every tok_pos - shift */
  int64_t rope_rows;
  const void *k_pool, *v_pool; /* bf16 planes, see layout above */
  int64_t pool_rows;
  int32_t pool_layers;
  const void *k_aux, *v_aux; /* second plane set (stage-2 new tokens); may alias pool */
  int64_t aux_rows;
  int32_t aux_layers;
  int32_t n_heads, n_kv_heads, head_dim, hd_pad;
  float scale; /* softmax scale, 1/sqrt(head_dim) (model.py:315) */
  int32_t num_m; /* 1 or 2 M-tiles of 128 rows per work */
  const DbsaAttnWork *works; /* device */
  int32_t n_works;
  const DbsaAttnSeg *segs; /* device */
  void *out; /* bf16, element (t, head, d) at out[t*out_tok_stride + head*head_dim + d] */
  int64_t out_tok_stride;
  void *part_o;    /* [rows][head_dim] normalised partial O (out_mode 1 / 2): fp32, or bf16 if part_bf16 */
  float *part_lse; /* fp32 [rows], natural-log LSE (out_mode 1 / 2) */
  const DbsaRowMap *row_map; /* device; required when any work is DBSA_OUT_MAPPED, else may be NULL */
  int32_t part_bf16;         /* partial O element type: 0 fp32, 1 bf16 */
  unsigned long long *pair_count; /* optional (NULL = off): the kernel adds the number of (query row, key)
                                     pairs whose score entered its softmax, i.e. the unmasked entries of every
                                     tile it visited, over all heads.  For stage 1 this equals
                                     n_heads * masks.count_allowed_token_pairs (masks.py:111-123). */
  const int32_t *cta_works; /* optional (NULL = round-robin): device [n_ctas + 1] prefix offsets; CTA b of the
                               num_m == 2 kernel runs works [cta_works[b], cta_works[b+1]) in order, so the
                               host can pack a latency launch (e.g. long chunk works one per CTA, the short
                               SELF works together on the spare CTAs) */
  int32_t n_ctas;           /* grid size when cta_works is set (<= the SM count) */
  int32_t pdl_early_q;      /* 1: q and every table were complete before the stream predecessor kernel STARTED
                               (e.g. the K/V page write that precedes each layer's attention); the launch is then
                               a programmatic dependent launch that stages Q while the predecessor runs and waits
                               for it only before its first K/V tile load.  0: plain stream order. */
  const void *rope_f16;     /* optional (NULL = rotate with rope_table): fp16 (cos, sin) pairs, [rope_rows]
                               [head_dim/2] (dbsa_rope_table_f16), used for the query rotation of the two-tile
                               kernel's Q staging: half the bytes per row of the float32 table.  The rounding
                               (2^-11 relative) is below the bf16 rounding of the rotated query (2^-8). */
  int64_t part_chunk_rows;  /* 0: partial O rows are [rows][head_dim].  > 0 (bf16 partials, head_dim % 16 == 0):
                               16-column chunks, element (row, d) at ((d / 16) * part_chunk_rows + row) * 16 +
                               d % 16 for rows < part_chunk_rows -- the epilogue's 32-byte store of one chunk
                               from 32 consecutive rows (one per TMEM lane) is then 1 KB contiguous instead of
                               32 scattered sectors.  The merge reading them passes the same value. */
  int32_t one_seg_partials; /* 1: every work has exactly one segment and writes a partial (out_mode
                               DBSA_OUT_PARTIAL or DBSA_OUT_MAPPED) -- the chunk-major stage-2 schedule.  With
                               bf16 chunk-layout partials, rope_f16, no pair_count and head_dim == hd_pad (a
                               multiple of 16) the launch then runs a kernel instance specialised for that
                               case; results are identical.  0: the generic kernel. */
} DbsaAttnArgs;
int dbsa_attention(const DbsaAttnArgs *args, void *stream);

/* Component K3m: combine split partials, lse = log sum exp(lse_s),
 * O = sum exp(lse_s - lse) O_s -- reproduces the single softmax over the
 * concatenated key set of kernels.py:52-56. */
typedef struct DbsaMergeGroup {
  int64_t part_row0; /* partial row of split 0, row 0 */
  int32_t rows;      /* rows per split */
  int32_t n_splits;
  int32_t q_tok0; /* output token of row 0 */
  int32_t kv_head;
} DbsaMergeGroup;
typedef struct DbsaMergeArgs {
  const void *part_o; /* fp32, or bf16 if part_bf16 */
  const float *part_lse;
  const DbsaMergeGroup *groups; /* device */
  int32_t n_groups;
  int32_t max_rows;
  int32_t n_heads, n_kv_heads, head_dim;
  void *out; /* bf16 */
  int64_t out_tok_stride;
  int64_t split_stride; /* rows between split s and s+1 of a group; 0 = the group's `rows`
                           (a gathered [world][R] partial buffer uses R: the C5 shard merge) */
  int32_t part_bf16;
  int32_t part_tok_layout; /* 1: partial rows are token-major like `out` -- row r of split s of a group is
                              (q_tok0 + r / gs) * n_heads + kv_head * gs + r % gs + s * split_stride, and
                              part_row0 is unused (the C5 per-layer gather of per-rank merged partials) */
  float *out_lse;          /* optional: write a partial instead of the final output -- the merged O
                              (normalised, bf16) into out and its natural-log LSE into
                              out_lse[t * n_heads + head]; a row with no visible key gets O = 0 and
                              LSE = -inf (the per-rank half of the C5 merge) */
  int64_t part_chunk_rows; /* the partials' layout, as DbsaAttnArgs.part_chunk_rows (part_tok_layout 0 only) */
} DbsaMergeArgs;
int dbsa_lse_merge(const DbsaMergeArgs *args, void *stream);

/* Component K5: the fused label-scoring epilogue of stage 2 -- the reference's
 * logits_from_hidden -> log_softmax_rows -> gather of the label token
 * (model.py:393-397, 414-417, 441-443).  One tcgen05 GEMM pass over
 * x @ lm_head, 256 vocab columns x 256 rows per tile with fp32 accumulators in
 * TMEM, keeps a running (max, sum of exp) per row and tile; no logit reaches
 * HBM.  A second launch folds each scored (row, target) pair's tiles into
 * the row's LSE and subtracts it from the target logit (a dot product of the
 * same bf16 operands with fp32 accumulation). */
typedef struct DbsaLabelScoreArgs {
  const void *x;              /* bf16 [rows, d]: final-normed hidden states of the scored rows */
  int64_t rows;
  int64_t d;                  /* model dim, a multiple of 8 */
  const void *w;              /* bf16 [vocab, d]: lm_head, K-major (transposed from the reference's [d, vocab]) */
  int64_t vocab;
  void *workspace;            /* fp32 [ceil(vocab / 128)][ceil(rows / 128) * 128][2]: per-128-column (max, sum) */
  const int64_t *pair_row;    /* [n_pairs] row of x of each scored pair */
  const int32_t *pair_target; /* [n_pairs] target token */
  int64_t n_pairs;
  float *out;                 /* fp32 [n_pairs]: log p(target | row) */
} DbsaLabelScoreArgs;
int dbsa_label_score(const DbsaLabelScoreArgs *args, void *stream);

/* Component K2w: page write of one layer's K (rotated at tok_pos) and V
 * (transposed) for a set of 64-token pages.  Replaces the per-block copy of
 * SegmentedKVCache.append_block (kvstore.py:103-105) and the rotary
 * transform of model.rope_rotate_heads (model.py:222-239) for keys. */
typedef struct DbsaPage {
  int32_t tok0;  /* first token of the page in the qkv buffer */
  int32_t n_tok; /* 1..64 valid tokens; the rest of the page is zeroed */
  int32_t row0;  /* destination row (multiple of 64) */
  int32_t pad;
} DbsaPage;
typedef struct DbsaKvWriteArgs {
  const void *k_src, *v_src; /* bf16, (t, kvh, d) at src[t*src_tok_stride + kvh*head_dim + d] */
  int64_t src_tok_stride;
  const int32_t *tok_pos;
  const float *rope_table;
  int64_t rope_rows;
  const DbsaPage *pages; /* device */
  int32_t n_pages;
  void *k_dst, *v_dst; /* planes */
  int64_t dst_rows;
  int32_t dst_layers, layer;
  int32_t n_kv_heads, head_dim, hd_pad;
} DbsaKvWriteArgs;
int dbsa_kv_write(const DbsaKvWriteArgs *args, void *stream);

/* Component K2r: page read-back (inverse of K2w) for cache serialisation
 * (kvstore.serialize, kvstore.py:238-258): fp32 pre-rotation K (un-rotated at
 * tok_pos) and V, token-major [t][kvh][head_dim], for a set of pages. */
typedef struct DbsaKvReadArgs {
  const void *k_src, *v_src; /* planes */
  int64_t src_rows;
  int32_t src_layers, layer;
  const int32_t *tok_pos; /* position of each output token */
  const float *rope_table;
  int64_t rope_rows;
  const DbsaPage *pages; /* device; tok0 indexes the output */
  int32_t n_pages;
  int32_t n_kv_heads, head_dim, hd_pad;
  float *k_dst, *v_dst;
} DbsaKvReadArgs;
int dbsa_kv_read(const DbsaKvReadArgs *args, void *stream);

/* Rotary table: table[p][i] = (cos, sin)(p * inv_freq[i]) with the angle
 * formed in float64 exactly as model.rope_angles (model.py:205-209). */
int dbsa_rope_table(float *table, int64_t rows, const double *inv_freq, int32_t half,
                    int64_t pos0, void *stream);
/* The same table rounded once from float64 to fp16 (cos, sin) pairs, for
 * DbsaAttnArgs.rope_f16. */
int dbsa_rope_table_f16(void *table, int64_t rows, const double *inv_freq, int32_t half,
                        int64_t pos0, void *stream);

/* Component K4: per query, [0] + top-(budget-1) of units 1..n-1 under the
 * total order (score desc, id asc), then re-ordered by `ordering`
 * (0 in-order, 1 low-to-high, 2 reverse) -- bit-exact replacement of
 * retrieval.select + retrieval.order (retrieval.py:352-388). */
int dbsa_topk_select(const double *scores, int64_t n_queries, int64_t n_units, int64_t budget,
                     int32_t ordering, int32_t *out_ids, void *stream);

/* GPU BM25: out[q][u] = sum over the query's term ids
 * (row q of term_ids, -1 = skip) of idf[t] * tf[t][u] * k1p1 / (tf[t][u] + norm[u]),
 * float64 in query-term order without FMA contraction -- bit-identical to
 * Bm25Index.score (retrieval.py:129-141) given the host's idf / norm.  tf is a
 * dense uint16 [n_terms][n_units] matrix. */
int dbsa_bm25_scores(const int32_t *term_ids, int64_t n_queries, int32_t max_terms, const uint16_t *tf,
                     const double *idf, const double *norm, int64_t n_units, double k1p1, double *out,
                     void *stream);

/* Dense-path helpers fused for the pre-norm block (model.py:321,355,358;
 * kernels.py:103-123): RMSNorm fp32 -> bf16, and silu(gate) * up. */
int dbsa_rmsnorm(const float *x, const float *weight, void *out, int64_t rows, int64_t dim,
                 float eps, void *stream);
/* Residual add fused with the next norm (model.py:352-359): x += delta (fp32,
 * in place), then out = bf16 RMSNorm(x) * weight. */
int dbsa_add_rmsnorm(float *x, const float *delta, const float *weight, void *out, int64_t rows, int64_t dim,
                     float eps, void *stream);
int dbsa_silu_mul(const void *gate_up, void *out, int64_t rows, int64_t ffn, void *stream);

/* Label scoring gather (model.py:414-417,441-443): for each scored row r,
 * logprob[r] = logits[r, target[r]] - logsumexp(logits[r, :]) in fp32. */
int dbsa_label_logprob(const float *logits, int64_t rows, int64_t vocab, const int32_t *target,
                       float *out, void *stream);
/* Label scores and choice (model.py:441-443, pipeline.py:376-382): output o =
 * q * n_labels + l sums the log-probs of rows label_row0[o] .. label_row0[o+1]
 * in order; best[q] is the first label with the maximum score. */
int dbsa_label_reduce(const float *lp, const int32_t *label_row0, int64_t n_queries, int32_t n_labels,
                      float *scores, int64_t *best, void *stream);

int dbsa_abi_version(void);
const char *dbsa_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DBSA_B200_H */
