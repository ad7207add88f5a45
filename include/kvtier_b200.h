/*
 * kvtier_b200.h -- C ABI of the B200 (sm_100a) KV-selection + sparse-decode library.
 *
 * Drop-in boundary for the reference's hot path (kvtier 0.1.0, pure Python/numpy):
 * every entry point below replaces one reference function, cited as file:line under
 * /root/reference/pkg/src/kvtier/.  The Python host package paper_2506_20187_b200 keeps
 * the reference's module/function names on top of these calls.
 *
 * Conventions
 *   - Pointers are DEVICE pointers unless stated; the caller owns all memory.
 *   - A "lane" is one (batch row, head) KV sequence (reference: one (layer, head),
 *     engine.py:316).  Lane i's rows start at base + i * lane_stride (elements); rows are
 *     contiguous with stride d.
 *   - Token positions are int32 (context < 2^31).
 *   - Every call is stream-ordered on `stream` (a cudaStream_t; NULL = legacy default)
 *     and returns a kvt_status; nothing throws across the ABI; no global mutable state.
 *   - Scores are the canonical float64 logits fl(q.k)/fl(sqrt d);
 *     bounds are widened to be sound for them.  Order for top-k: score desc, index asc.
 */
#ifndef KVTIER_B200_H
#define KVTIER_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define KVT_API __attribute__((visibility("default")))
#else
#define KVT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KVT_OK = 0,
    KVT_ERR_SHAPE = -1,      /* ValueError: shape mismatch (importance.py:31-32) */
    KVT_ERR_K = -2,          /* ValueError: k out of [0, n] (chunk_tree.py:251-252) */
    KVT_ERR_COLD = -3,       /* RuntimeError: cold leaf without a store (chunk_tree.py:275-277) */
    KVT_ERR_OOM = -4,        /* workspace too small */
    KVT_ERR_CUDA = -5,       /* CUDA launch/runtime error */
    KVT_ERR_DTYPE = -6,      /* unsupported dtype combination */
    KVT_ERR_ARG = -7         /* other invalid argument (ValueError) */
} kvt_status;

/* KVT_I4: INT4 KV records produced by kvt_kv_quant -- per token d/2 code bytes (dim 2j in
 * the low nibble, 2j+1 in the high nibble) then d/32 (scale, min) fp16 pairs; dequantised
 * value fmaf(code, scale, min).  For KVT_I4 operands lane strides are in BYTES and d must
 * be a multiple of 128.  Accepted wherever keys/values are read (K1, K4, K7). */
typedef enum { KVT_F32 = 0, KVT_F64 = 1, KVT_BF16 = 2, KVT_F16 = 3, KVT_I4 = 4 } kvt_dtype;

/* Library version (major*10000 + minor*100 + patch) and status text. */
KVT_API int kvt_version(void);
KVT_API const char* kvt_status_string(int status);
/* Last CUDA error text recorded by this thread (for KVT_ERR_CUDA). */
KVT_API const char* kvt_last_error(void);

/* ---- K1: chunk abstracts -------------------------------------------------------------
 * Replaces importance.py:80-87 make_abstract (and the per-leaf loop of chunk_tree.py:
 * 199-208 build_partition).  Uniform grid: chunk c of lane i covers tokens
 * [c*C, min((c+1)*C, n)); chunks [c_begin, c_end) are (re)built.  Outputs are the
 * element-wise max / min key rows at amax + i*abs_lane_stride + c*d, in abs_dtype: F32 for
 * F32/BF16/F16/I4 keys and F64 for F64 keys (exact), or BF16 for any keys (rounded outward:
 * max up, min down -- half the bytes, still a sound summary). */
KVT_API int kvt_abstract_build(const void* keys, int key_dtype, int64_t n_lanes, int64_t lane_stride,
                       int64_t n, int d, int C, int64_t c_begin, int64_t c_end,
                       void* amax, void* amin, int abs_dtype, int64_t abs_lane_stride, void* stream);

/* Arbitrary spans (exact abstracts of keys[start:end) of lane lane_of[j]); used for
 * partition leaves and merged desert runs (importance.py:90-100 merge_abstracts,
 * chunk_tree.py:344-379 merge_desert).  Output row j at amax + j*d. */
KVT_API int kvt_abstract_spans(const void* keys, int key_dtype, int64_t lane_stride, int d,
                       int64_t n_spans, const int32_t* lane_of, const int32_t* starts,
                       const int32_t* ends, void* amax, void* amin, void* stream);
/* K2, merge_abstracts (importance.py:90-100) over segments of consecutive chunk abstracts
 * ([lanes][m][d] rows, lane stride in elements): explicit segments (seg_lane/begin/end,
 * output row s of amax_out/amin_out [n_seg][d]: a merged desert run, chunk_tree.py:344-379)
 * or, with seg_lane == NULL, uniform coarsening by `factor` (segment s = lane s / m_out, chunk
 * j = s % m_out over fine chunks [j factor, (j + 1) factor) < m_in, written at
 * out + lane * out_lane_stride + j * d).  Element-wise max / min: exact in every dtype. */
KVT_API int kvt_abstract_merge(const void* amax, const void* amin, int dtype, int64_t in_lane_stride, int d,
                               int64_t n_seg, const int32_t* seg_lane, const int32_t* seg_begin,
                               const int32_t* seg_end, int factor, int64_t m_in, int64_t m_out, void* amax_out,
                               void* amin_out, int64_t out_lane_stride, void* stream);

/* ---- K8: INT4 KV compression ------------------------------------------------------------
 * North-star item 4 (the reference only models compression, pipeline.py:35-57 delta = 0.25,
 * and has no quantizer): quantise tokens [t_begin, t_end) of every lane from src
 * (F32/BF16/F16, [n_lanes] x src_lane_stride elements) into INT4 records at
 * dst + i*dst_lane_stride (bytes) + t*(d/2 + d/8).  Group 32: scale = fp16((max-min)/15),
 * min = fp16(min), code = clamp(rint((x - min)/scale), 0, 15).  Used at prefill (bulk) and
 * for every appended token. */
KVT_API int kvt_kv_quant(const void* src, int src_dtype, int64_t n_lanes, int64_t src_lane_stride,
                         int64_t t_begin, int64_t t_end, int d, void* dst, int64_t dst_lane_stride,
                         void* stream);
KVT_API int kvt_i4_row_bytes(int d);
/* Test hook: counts (atomically, into *bad_dev) the positive finite fp16 scales s for which
 * the codec's fast reciprocal differs from the correctly rounded fl32(1/s).  Expected: 0. */
KVT_API int kvt_i4_recip_check(int* bad_dev, void* stream);
/* Expand INT4 records (src lane stride in bytes) of tokens [t_begin, t_end) into rows of
 * dst_dtype (F32/BF16/F16): the device half of a compressed host->HBM tier transfer
 * (pipeline.py:79-103 decompress_rate is this kernel's throughput). */
KVT_API int kvt_kv_dequant(const void* src, int64_t src_lane_stride, int64_t n_lanes, int64_t t_begin,
                           int64_t t_end, int d, void* dst, int dst_dtype, int64_t dst_lane_stride,
                           void* stream);

/* ---- K3: query-vs-abstract bounds ----------------------------------------------------
 * Replaces importance.py:108-137 bound_chunk / bound_chunks_batch (logit mode).
 * Leaves of lane i: if leaf_start == NULL the uniform grid of size C over [0, n)
 * (n_leaves = ceil(n/C)); otherwise leaf j = [leaf_start[i*leaf_stride + j],
 * leaf_start[i*leaf_stride + j + 1]) for j < n_leaves[i] (the last end is n).
 * q: [n_lanes][d] of q_dtype (F32 or F64).  U/L: float64 at U + i*bnd_stride + j.
 * scaled != 0: bounds on the logits fl(q.k)/fl(sqrt d) (the importance.py form);
 * scaled == 0: bounds on the raw canonical dots (what the pipeline prunes with).
 * A (optional): sum_j |q_j| max(|max_j|, |min_j|) per chunk, a bound on sum_j |q_j k_j| for
 * every token of the chunk (feeds the f32 scoring error bound). */
KVT_API int kvt_chunk_bounds(const void* q, int q_dtype, int64_t n_lanes, int d, int64_t n, int C,
                     const int32_t* leaf_start, const int32_t* n_leaves, int64_t leaf_stride,
                     const void* amax, const void* amin, int abs_dtype, int64_t abs_lane_stride,
                     double* U, double* L, double* A, int64_t bnd_stride, int scaled, void* stream);

/* ---- K4 (brute force): canonical token logits -----------------------------------------
 * Replaces importance.py:27-33 attention_logits / :46-53 score_tokens (logit mode) for
 * all n tokens of every lane.  out: float64 [n_lanes][n] (row stride out_stride). */
KVT_API int kvt_token_scores(const void* q, int q_dtype, const void* keys, int key_dtype,
                     int64_t n_lanes, int64_t lane_stride, int64_t n, int d,
                     double* out, int64_t out_stride, void* stream);

/* ---- plan: lower-bound threshold tau and candidate work items -------------------------
 * The pruning half of chunk_tree.py:233-338 select_top_k: tau = the k-th largest lower
 * bound counting each leaf's rows; every leaf with U >= tau is a candidate (no top-k
 * token can lie elsewhere).  Candidate leaves are cut into items of <= 64 tokens.
 * Outputs per lane: items (tok_start, count, out_pos) int32 x3 at items + i*item_stride*3,
 * n_items[i], n_cand[i] (candidate tokens), cand_leaf flags (int8, may be NULL) and
 * evals[i] = n_leaves + n_cand (eval_count, chunk_tree.py:256-268,322). */
KVT_API int kvt_select_plan(int64_t n_lanes, int64_t n, int C, const int32_t* leaf_start,
                    const int32_t* n_leaves, int64_t leaf_stride, const double* U, const double* L,
                    int64_t bnd_stride, int64_t k, int32_t* items, int64_t item_stride,
                    int32_t* n_items, int32_t* n_cand, int8_t* cand_leaf, int64_t* evals,
                    void* stream);

/* ---- K4: candidate scoring -------------------------------------------------------------
 * Raw canonical float64 dots q.k of every candidate token (the exact-score half of
 * select_top_k: singleton bounds, chunk_tree.py:291-296,321; logit = dot / sqrt d is a
 * monotone map, so the order is the reference's).  Writes cand_score [i*cand_stride + pos]
 * and cand_tok (token index) for pos < n_cand[i].  Items are streamed through a
 * cp.async.bulk (TMA engine) shared-memory ring by persistent CTAs. */
KVT_API int kvt_cand_score(const void* q, int q_dtype, const void* keys, int key_dtype,
                   int64_t n_lanes, int64_t lane_stride, int d, const int32_t* items,
                   int64_t item_stride, const int32_t* n_items, double* cand_score,
                   int32_t* cand_tok, int64_t cand_stride, int blocks_per_lane, void* stream);

/* ---- fast scoring: f32 estimates + exact band re-scoring ---------------------------------
 * kvt_select_plan2 = kvt_select_plan that also writes a 4-double record per lane:
 * err[4i] = E, a rigorous bound on |f32 estimate - canonical f64 dot| over lane i's
 * candidates (from the chunks' A of kvt_chunk_bounds; d is the head dim), err[4i+1] = tau
 * (<= the k-th canonical dot), err[4i+2] = max U over the candidates.
 * kvt_cand_score_f32 writes the f32 estimates (TMA pipeline, any key dtype but F64).
 * kvt_topk_select_band (one CTA per lane) selects the exact canonical top-k from them:
 * linear-bucket histogram over [tau - 2E, Umax + 2E] + radix select inside the k-th bucket
 * give the exact k-th estimate T; tokens above T + 2E are in, below T - 2E out, and the band
 * in between is re-scored canonically in f64 from the key rows (q: [n_lanes][d]).  A wide
 * band (ties) falls back to canonical re-scoring of every candidate into `scratch` (f64,
 * cand_stride per lane).  Output as kvt_topk_select_runs (sel_score: the estimate for the
 * sure tokens, exact for the band / fallback). */
KVT_API int kvt_select_plan2(int64_t n_lanes, int64_t n, int C, const int32_t* leaf_start,
                    const int32_t* n_leaves, int64_t leaf_stride, const double* U, const double* L,
                    int64_t bnd_stride, int64_t k, int32_t* items, int64_t item_stride,
                    int32_t* n_items, int32_t* n_cand, int8_t* cand_leaf, int64_t* evals,
                    const double* A, double* err, int d, void* stream);
/* kvt_select_plan_group = kvt_select_plan2 for GQA groups of `grp` adjacent query lanes sharing
 * a KV lane (decode path: uniform grid, no leaf_start): tau per query lane, candidates = the
 * union over the group (U_h >= tau_h for any h), items / n_items per KV lane (n_lanes / grp
 * rows), n_cand / evals / err per query lane.  grp = 1 is kvt_select_plan2. */
KVT_API int kvt_select_plan_group(int64_t n_lanes, int64_t n, int C, const int32_t* leaf_start,
                    const int32_t* n_leaves, int64_t leaf_stride, const double* U, const double* L,
                    int64_t bnd_stride, int64_t k, int32_t* items, int64_t item_stride,
                    int32_t* n_items, int32_t* n_cand, int8_t* cand_leaf, int64_t* evals,
                    const double* A, double* err, int d, int grp, void* stream);
KVT_API int kvt_cand_score_f32(const void* q, int q_dtype, const void* keys, int key_dtype,
                    int64_t n_lanes, int64_t lane_stride, int d, const int32_t* items,
                    int64_t item_stride, const int32_t* n_items, float* cand_score32,
                    int32_t* cand_tok, int64_t cand_stride, void* stream);
KVT_API int kvt_topk_select_band(const float* cand_score32, const int32_t* cand_tok,
                    const int32_t* n_cand, int64_t cand_stride, const double* err, int64_t n_lanes,
                    int64_t k, const void* q, int q_dtype, const void* keys, int key_dtype,
                    int64_t lane_stride, int d, double* scratch, int32_t* sel_tok, double* sel_score,
                    int64_t sel_stride, int32_t* n_sel, int32_t* run_start, int32_t* run_len,
                    int64_t run_stride, int32_t* n_runs, void* stream);

/* ---- INT4 keys: fast estimates on the integer tensor cores ------------------------------
 * kvt_i4_qprep writes, per lane, the query as 4 signed 8-bit digits on power-of-two scales
 * laid out as m16n8k32 B fragments in the INT4 nibble order, plus per-group error weights
 * (kvt_i4_qprep_bytes(n_lanes, d) bytes, 16 B aligned; d = 128 or 256).
 * kvt_cand_score_i4mma = kvt_cand_score_f32 for KVT_I4 keys (records of kvt_kv_quant) with
 * the inner products done exactly in int32 by MMA; it also max-es a rigorous per-lane bound
 * on |estimate - canonical f64 dot| into err[4 i + 3] (the kvt_select_plan2 record, which
 * must be written first), which kvt_topk_select_band then uses as E.  Runs kvt_i4_qprep
 * into qprep_ws itself. */
KVT_API size_t kvt_i4_qprep_bytes(int64_t n_lanes, int d);
KVT_API int kvt_i4_qprep(const void* q, int q_dtype, int64_t n_lanes, int d, void* out, void* stream);
KVT_API int kvt_cand_score_i4mma(const void* q, int q_dtype, const void* keys, int64_t n_lanes,
                    int64_t lane_stride, int d, const int32_t* items, int64_t item_stride,
                    const int32_t* n_items, float* cand_score32, int32_t* cand_tok,
                    int64_t cand_stride, double* err, void* qprep_ws, void* stream);

/* ---- K5: exact top-k ---------------------------------------------------------------------
 * Result contract of select_top_k (chunk_tree.py:233-338) / brute force
 * (engine.py:337-339): the k best candidates by (score desc, token asc).  One thread-
 * block cluster per lane runs a 64-bit radix select over the candidates with the
 * histograms reduced through distributed shared memory.  Output ascending token order:
 * sel_tok[i*sel_stride + r], sel_score (float64), n_sel[i] = k. */
KVT_API int kvt_topk_select(const double* cand_score, const int32_t* cand_tok, const int32_t* n_cand,
                    int64_t cand_stride, int64_t n_lanes, int64_t k, int32_t* sel_tok,
                    double* sel_score, int64_t sel_stride, int32_t* n_sel, void* stream);

/* K5 with the K6 run scan fused into the same cluster kernel (what kvt_select_attend uses):
 * additionally writes run_start/run_len [i*run_stride + r] and n_runs[i] for the selected
 * tokens (engine.py:176-183).  run_start == NULL behaves as kvt_topk_select. */
KVT_API int kvt_topk_select_runs(const double* cand_score, const int32_t* cand_tok, const int32_t* n_cand,
                    int64_t cand_stride, int64_t n_lanes, int64_t k, int32_t* sel_tok,
                    double* sel_score, int64_t sel_stride, int32_t* n_sel, int32_t* run_start,
                    int32_t* run_len, int64_t run_stride, int32_t* n_runs, void* stream);

/* ---- K6: runs / canonical partition --------------------------------------------------------
 * engine.py:176-183 _token_runs and the leaf shape of select_top_k + merge_desert
 * (chunk_tree.py:331-379): the selected runs and their complement (desert runs) tile [0,n).
 * run_start/run_len: [i*run_stride + r], n_runs[i].  If part_start != NULL also writes
 * the canonical partition (leaf starts; state 1 = important, 2 = desert) with n_part[i]. */
KVT_API int kvt_runs_scan(const int32_t* sel_tok, const int32_t* n_sel, int64_t sel_stride,
                  int64_t n_lanes, int64_t n, int32_t* run_start, int32_t* run_len,
                  int64_t run_stride, int32_t* n_runs, int32_t* part_start, int8_t* part_state,
                  int64_t part_stride, int32_t* n_part, void* stream);

/* ---- K7: sparse decode attention -----------------------------------------------------------
 * engine.py:145-154 attention_output over the selected set: softmax(sel_score) @ V[sel].
 * sel_score are the scores from K5 (keys are not re-read); the softmax logit of token i is
 * (sel_score_i - max) * logit_scale, i.e. logit_scale = 1/sqrt(d) for raw dots and 1 for
 * logits.  Split over
 * `splits` blocks per lane with an online-softmax (m, l, o) merge; splits <= 0 picks the count
 * (<= 64) that fills whole waves of the kernel at its residency.  out: float32
 * [n_lanes][d] (out64: optional float64 copy).  ws: workspace of
 * kvt_attn_workspace_bytes(n_lanes, d, splits) bytes (splits = 64 when auto), zero-filled
 * once by the caller (the
 * per-lane merge tickets are left at zero by every call).  The last split CTA of each lane
 * performs the log-sum-exp merge, so this is a single kernel launch. */
KVT_API size_t kvt_attn_workspace_bytes(int64_t n_lanes, int d, int splits);
/* Each lane's merged softmax state after kvt_sparse_decode_attn: lse_out[2 i] = m (max selected
 * score), lse_out[2 i + 1] = l = sum exp((s - m) logit_scale).  Device buffer, stream-ordered. */
KVT_API int kvt_attn_lse(const void* ws, int64_t n_lanes, double* lse_out, void* stream);
/* Config 5 (sequence sharding): merge all-gathered shard partials
 * parts[p][lane] = (m, l, o[d]) (o normalised, f64) into out (f32 and/or f64) with the
 * log-sum-exp weights w_p = l_p exp((m_p - max m) logit_scale); n_parts <= 64. */
KVT_API int kvt_lse_merge(const double* parts, int n_parts, int64_t n_lanes, int d, double logit_scale, float* out,
                          double* out64, void* stream);
KVT_API int kvt_sparse_decode_attn(const void* values, int v_dtype, int64_t n_lanes, int64_t lane_stride,
                           int d, const int32_t* sel_tok, const double* sel_score,
                           const int32_t* n_sel, int64_t sel_stride, double logit_scale, int splits,
                           void* ws, float* out, double* out64, void* stream);

/* ---- fused per-layer pipeline -----------------------------------------------------------------
 * K3 -> plan -> K4 -> K5 -> K6 -> K7 for n_lanes lanes on the uniform grid C (or the
 * leaf table), i.e. the body of the engine's per-lane loop (engine.py:316-357) for a whole
 * layer at once.  Workspace size from kvt_layer_workspace_bytes.  Outputs: sel_tok /
 * sel_score / n_sel (K5), runs (K6), out (K7), evals. */
typedef struct {
    int64_t n_lanes, n, k;
    int d, C;
    int key_dtype, v_dtype, q_dtype, abs_dtype;
    const void* q;              /* [n_lanes][d] */
    const void* keys;           /* lane i at keys + i*lane_stride */
    const void* values;
    int64_t lane_stride;
    const void* amax;           /* abstracts [n_lanes][abs_lane_stride] */
    const void* amin;
    int64_t abs_lane_stride;
    const int32_t* leaf_start;  /* NULL = uniform grid C */
    const int32_t* n_leaves;
    int64_t leaf_stride;
    int32_t* sel_tok;           /* [n_lanes][k] */
    double* sel_score;
    int32_t* n_sel;
    int32_t* run_start;         /* [n_lanes][k] (may be NULL: skip K6) */
    int32_t* run_len;
    int32_t* n_runs;
    float* out;                 /* [n_lanes][d] */
    int64_t* evals;             /* [n_lanes] (may be NULL) */
    int attn_splits;            /* 0 = auto */
    int score_blocks;           /* 0 = auto */
    int exact_scores;           /* 1: canonical f64 scoring of every candidate (no f32 band path) */
    const float* abs_mag;       /* [n_lanes][d] per-lane max |key| over all chunks, or NULL.  With bf16
                                   abstracts, f32 q, a uniform grid and d = 128/256 it selects the
                                   directed-rounding f32 bounds (kvt_chunk_bounds_fast) */
    int kv_group;               /* GQA: query lanes per KV lane (0/1 = none).  Query lane i reads keys,
                                   values, abstracts and abs_mag of KV lane i / kv_group; keys/values/
                                   amax/amin/abs_mag then hold n_lanes / kv_group lanes.  Decode path
                                   (abs_mag, bf16 abstracts, f32 q) only */
    float* sel_hint;            /* [n_lanes] f32 state carried across decode steps, or NULL: the bucket
                                   coordinate of the lane's previous k-th estimate in the selector's
                                   estimate histogram (NaN = none), read and rewritten by the selector;
                                   a stale hint costs one extra pass, never exactness */
} kvt_layer_args;

/* K3 for the decode path (bounds_fast.cu): sound f32 bounds of raw dots over bf16 abstracts on a
 * uniform grid C, every fma/add rounded outward (U toward +inf, L toward -inf); A[c] = one
 * per-lane upper bound RU(sum_j |q_j| mag_j) on every chunk's sum |q||k|.  Replaces the
 * canonical kvt_chunk_bounds inside kvt_select_attend when abs_mag is given; the selected set
 * does not depend on it (pruning only needs soundness).  d = 128 or 256; U, L, A f64. */
KVT_API int kvt_chunk_bounds_fast(const float* q, int64_t n_lanes, int d, int64_t n, int C, const void* amax,
                                  const void* amin, int64_t abs_lane_stride, const float* mag, double* U,
                                  double* L, double* A, int64_t bnd_stride, void* stream);

/* Workspace of kvt_select_attend: zero-filled once by the caller and then reusable by every
 * layer with the same n_lanes and d, whatever its chunk size (size it for the largest
 * max_leaves).  Its first region holds the attention merge tickets, which every call leaves
 * at zero. */
KVT_API size_t kvt_layer_workspace_bytes(int64_t n_lanes, int64_t n, int64_t max_leaves, int d);
KVT_API int kvt_select_attend(const kvt_layer_args* a, void* ws, size_t ws_bytes, void* stream);
/* GQA for the standalone decode-path entry points (kvt_chunk_bounds_fast, kvt_cand_score_f32 /
 * _i4mma, kvt_topk_select_band, kvt_sparse_decode_attn) called from this host thread: query
 * lane i reads key/value/abstract lane i / kv_group.  Returns the previous value (1 = none).
 * kvt_select_attend uses its own kv_group field. */
KVT_API int kvt_set_kv_group(int kv_group);
/* GQA union candidates for the standalone entry points (kvt_cand_score_i4mma,
 * kvt_topk_select_band) on this host thread: items from kvt_select_plan_group(grp = g), token
 * ids shared per group (row of the group's first query lane).  kvt_select_attend sets it
 * itself for INT4 keys.  Returns the previous value (1 = one candidate list per lane). */
KVT_API int kvt_set_cand_group(int g);
/* Development aid: when buf (device, >= 8 x n_lanes u64) is non-null, every later
 * kvt_topk_select_band CTA b writes %globaltimer at its phase boundaries p = 0..7 to
 * buf[b * 8 + p] (tools/select_phases.py).  nullptr turns it off (the default). */
KVT_API int kvt_debug_select_phases(unsigned long long* buf);

/* ---- synthetic workload (bench / test input generator; not on the decode path) ----------
 * The planted-desert model of trace.py:270-315 (generate_synthetic) as a counter hash, so
 * any lane can be regenerated bit-identically on the host (oracle ora_synth_lane): fills
 * bf16 keys and/or values [n_lanes] x lane_stride elements, tokens [0, n).  u: [n_lanes, d]
 * f32 unit directions; regions: [n_lanes, n_regions, 2] hot token ranges; planted = 0 gives
 * N(0,1)-like keys.  Recipe in paper_2506_20187_b200/csrc/synth.cu. */
KVT_API int kvt_synth_layer(void* keys, void* values, int64_t n_lanes, int64_t lane_stride, int64_t n, int d,
                            const uint32_t* lane_seed, const float* u, const int32_t* regions, int n_regions,
                            float desert_base, float desert_span, float hot_base, float hot_span,
                            float noise_scale, int planted, void* stream);

/* ---- tiered KV: HBM hot tier over a pinned-host warm tier ----------
 * Replaces the byte movement behind TieredStore.touch / ensure_hot / promote_hot / _evict_hot
 * (tiered_store.py:224-372, driven per lane from engine.py:342-343) for V records of C_rec
 * tokens.  Device state (caller-owned, see paper_2506_20187_b200/host_tier.py):
 *   table [L][kv_lanes][n_rec] i32  slot of each record, -1 = warm only (-2 transient)
 *   owner [n_slots] i64  record id (lk * n_rec + rec, lk = layer * kv_lanes + lane), -1 free
 *   stamp [n_slots] i32  step of the last touch;  free_stack [n_slots] + free_top
 *   pool  [n_slots][C_rec][row] INT4 records;  ctl: kvt_tier_ctl_bytes() zeroed once
 *   host_i4 (+ optional host_raw bf16) = the layer's pinned host rows [kv_lanes][N][row]
 * One kvt_tier_layer call per (step, layer), after the layer's selection: touch the records
 * its runs overlap, evict the least recently touched hot records -- order (stamp, start,
 * layer, lane) = the reference's (last_touch, start, layer, head) -- for the misses, copy the
 * misses host -> pool (a ceil(theta M) share as INT4 records, the rest as raw bf16 rows
 * quantised on the way, when host_raw is given), and add the row's ledger counters
 * (warm_to_hot / hot_to_warm bytes at ledger_rec_bytes per record, promotions) into
 * ledger_row.  The working set of one step must fit (ledger_row[3] = -1 otherwise). */
typedef struct {
    int64_t n_lanes;      /* query lanes of the layer (runs are per query lane) */
    int kv_group, d, crec;
    const int32_t* step;  /* device: the decode step (stamps); read by the kernels, so a
                             captured CUDA graph replays with the current value */
    const int32_t *run_start, *run_len, *n_runs;
    int64_t run_stride;
    int32_t* table;       /* whole table; this layer's rows start at table_base */
    int64_t table_base, table_stride, n_lk;  /* n_rec per lane; n_lk = L * kv_lanes */
    int32_t* stamp;
    int64_t* owner;
    int64_t n_slots;
    int32_t *free_stack, *free_top, *victims, *slot_of_miss;
    int64_t* miss;
    int64_t miss_cap;
    void* ctl;
    void* pool;
    const void* host_i4;  /* this layer's pinned INT4 rows */
    const void* host_raw; /* this layer's pinned bf16 rows, or NULL (all INT4) */
    int64_t host_lane_tokens, n_tok;
    const float* theta;   /* device: compressed share of the misses (pipeline.py solve_theta);
                             NULL = 1 (all INT4) */
    long long ledger_rec_bytes;
    long long* ledger_row; /* device [4]: += warm_to_hot, hot_to_warm bytes, promotions; [3] = -1
                              if the step's working set did not fit (CapacityError) */
} kvt_tier_args;
KVT_API size_t kvt_tier_ctl_bytes(void);
KVT_API int kvt_tier_layer(const kvt_tier_args* a, void* stream);
/* out4 = [misses, evictions, need (< 0: capacity error), victims] of the last call;
 * synchronises the stream (diagnostics). */
KVT_API int kvt_tier_read_ctl(const void* ctl, long long* out4, void* stream);
/* ---- one decode step's appends (the caller side of the path: engine-side KV growth) ---------
 * The new token's K and V rows of every layer and KV lane ([L][kv_lanes][d], element strides,
 * bf16 or f32) become INT4 record t of K / V ([L][kv_lanes][N][row], byte strides) -- the
 * kvt_kv_quant codec, bit-identical -- and each listed bf16 abstract grid has its tail chunk
 * t / C refreshed from the dequantised key (max(old, ru(x)), min(old, rd(x)); a new chunk when
 * t % C == 0), equal to rebuilding that chunk; absmag[layer] ([kv_lanes][d] f32, may be NULL)
 * takes max |.| of the new rounded abstracts.  grids and absmag are DEVICE arrays.  d = 128.
 * One launch for the whole step. */
typedef struct {
    void* amax;           /* bf16 [kv_lanes][lane_stride] */
    void* amin;
    int64_t lane_stride;  /* elements */
    int C;
    int layer;
} kvt_append_grid;
KVT_API int kvt_kv_append(const void* k_new, const void* v_new, int src_dtype, int64_t src_layer_stride,
                          int64_t src_lane_stride, int64_t n_layers, int64_t kv_lanes, int d, int64_t t, void* K,
                          void* V, int64_t layer_stride_b, int64_t lane_stride_b, const kvt_append_grid* grids,
                          int n_grids, float* const* absmag, void* stream);
/* ---- sequence sharding: the all-gather + log-sum-exp merge over NCCL ----------
 * NCCL is bound at run time (dlopen libnccl.so.2; the process's own NCCL when loaded), so the
 * library has no link-time NCCL dependency.  kvt_nccl_available: 1 when it could be bound.
 * kvt_nccl_unique_id writes the 128-byte ncclUniqueId; every rank passes the same id to
 * kvt_nccl_comm_init.  kvt_lse_allgather_merge all-gathers each rank's part_local
 * [n_lanes][d + 2] (m, l, o normalised; kvt_attn_lse + the rank's output) into gather_buf
 * [nranks][n_lanes][d + 2] and merges them (kvt_lse_merge), stream-ordered. */
KVT_API int kvt_nccl_available(void);
KVT_API int kvt_nccl_unique_id(void* id_out);
KVT_API int kvt_nccl_comm_init(void** comm_out, int nranks, int rank, const void* id);
KVT_API int kvt_nccl_comm_destroy(void* comm);
KVT_API int kvt_lse_allgather_merge(void* comm, int nranks, const double* part_local, int64_t n_lanes, int d,
                                    double logit_scale, double* gather_buf, float* out, double* out64,
                                    void* stream);
/* Live chunks of each lane's selection (runs from kvt_topk_select_runs / _band): out[lane][j]
 * = chunks of size 2^(lg0 + j) (j < nlev <= 8) that hold a selected token -- the measured skew
 * behind SparseDecoder.adapt_chunking (the importance density of chunk_tree.py:34-123). */
KVT_API int kvt_live_chunks(const int32_t* run_start, const int32_t* run_len, const int32_t* n_runs,
                            int64_t run_stride, int64_t n_lanes, int lg0, int nlev, long long* out, void* stream);
/* GQA K7 over INT4 values (kv_group g in {2, 4}, d = 128): one pass over the union of each
 * group's selections (query lanes i / g share KV lane i / g), P.V on the tensor cores with the
 * group's heads as MMA rows; tokens < n_ctx.  ws as kvt_sparse_decode_attn (64 splits);
 * scratch >= kvt_attn_gqa_scratch_bytes (the union plan).  KVT_ERR_ARG for shapes it does not
 * cover.  kvt_select_attend runs it for GQA INT4 layers (KVT_GQA_UNION=0 disables). */
KVT_API size_t kvt_attn_gqa_scratch_bytes(int64_t n_lanes, int kvg, int64_t n_ctx);
KVT_API int kvt_sparse_decode_attn_gqa(const void* values, int64_t n_lanes, int64_t lane_stride_b, int d, int kvg,
                                       int64_t n_ctx, const int32_t* sel_tok, const double* sel_score,
                                       const int32_t* n_sel, int64_t sel_stride, double logit_scale, void* ws,
                                       void* scratch, size_t scratch_bytes, float* out, double* out64,
                                       void* stream);
/* K7 over the hot tier: like kvt_sparse_decode_attn with INT4 values, but query lane i's row
 * t is read from pool + (table[(i / kv_group) * table_stride + t / crec] * crec + t % crec)
 * rows (every selected record must be hot: call kvt_tier_layer first). */
KVT_API int kvt_sparse_decode_attn_paged(const void* pool, const int32_t* table, int64_t table_stride, int crec,
                                         int64_t n_lanes, int d, const int32_t* sel_tok, const double* sel_score,
                                         const int32_t* n_sel, int64_t sel_stride, double logit_scale, int splits,
                                         void* ws, float* out, double* out64, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KVTIER_B200_H */
