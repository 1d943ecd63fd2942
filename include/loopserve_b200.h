/*
 * loopserve_b200.h -- C ABI of the B200-native LoopServe hot paths.
 *
 * Drop-in boundary for the two data-parallel hot paths of the reference
 * (arxiv 2507.13681, pkg/src/loopserve): online prefill sparsification +
 * vertical/slash sparse attention, and progressive decode KV compression.
 * Every entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - Stream-ordered: every device entry point enqueues work on `stream` and
 *    returns without synchronising. Buffers are caller-allocated device
 *    memory (the Python layer allocates them with torch); plain pointers and
 *    sizes only, no framework types.
 *  - Status: 0 = OK; negative = one code per reference exception class
 *    (errors.py:4-65) plus CUDA / workspace / unsupported codes.
 *    `ls_last_error()` returns a thread-local message for the last failure.
 *  - Layouts (row-major, bf16 = uint16 storage of bfloat16):
 *      q block      [n_heads][q_rows_stride...]  : q + h*q_head_stride + r*head_dim
 *      K / V archive[n_kv_heads][cap][head_dim]   : k + kv*kv_head_stride + pos*head_dim
 *    q-head h reads kv-head h / (n_heads / n_kv_heads) (GQA; the reference is
 *    MHA, model.py:26-34 -- one reference head == one q-head here).
 *  - Plans on device: per head a sorted int32 id list + count for slashes
 *    (global offsets d = g - c) and verticals (columns c), capacity n_total.
 */
#ifndef LOOPSERVE_B200_H
#define LOOPSERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *ls_stream_t; /* cudaStream_t */

enum ls_status {
  LS_OK = 0,
  LS_ERR_NON_FINITE_INPUT = -1,   /* errors.py:8  NonFiniteInput   */
  LS_ERR_ALL_MASKED_ROW = -2,     /* errors.py:12 AllMaskedRow     */
  LS_ERR_DIMENSION_MISMATCH = -3, /* errors.py:16 DimensionMismatch*/
  LS_ERR_EMPTY_PLAN = -4,         /* errors.py:20 EmptyPlan        */
  LS_ERR_INVALID_CONFIG = -5,     /* errors.py:24 InvalidConfig    */
  LS_ERR_SEQUENCE_TOO_LONG = -6,  /* errors.py:28 SequenceTooLong  */
  LS_ERR_CACHE_CORRUPT = -7,      /* errors.py:32 CacheCorrupt     */
  LS_ERR_EMPTY_BLOCK = -8,        /* errors.py:36 EmptyBlock       */
  LS_ERR_INVALID_ALPHA = -9,      /* errors.py:40 InvalidAlpha     */
  LS_ERR_EMPTY_WINDOW = -11,      /* errors.py:48 EmptyWindow      */
  LS_ERR_SIZE_MISMATCH = -12,     /* errors.py:52 SizeMismatch     */
  LS_ERR_INVALID_IDS = -13,       /* errors.py:56 InvalidIds       */
  LS_ERR_CUDA = -100,
  LS_ERR_WORKSPACE = -101,
  LS_ERR_UNSUPPORTED = -102
};

/* Shape of one attention layer call (all q-heads of a layer, or a shard). */
typedef struct ls_layer_desc {
  int32_t n_heads;        /* q-heads in this call                          */
  int32_t n_kv_heads;     /* kv-heads; n_heads % n_kv_heads == 0           */
  int32_t head_dim;       /* 64 or 128                                      */
  int32_t n_new;          /* block rows (session.py:122 block)              */
  int32_t n_total;        /* keys = row_offset + n_new                      */
  int32_t row_offset;     /* global position of block row 0                 */
  int64_t q_head_stride;  /* elements between q-heads in q                  */
  int64_t kv_head_stride; /* elements between kv-heads in k / v             */
  int64_t out_row_stride; /* elements between attention-output rows; 0 =
                             n_heads * head_dim (a head group writes its
                             columns of the full [n_new][H][d] output)     */
} ls_layer_desc;

const char *ls_last_error(void);
/* Device-side validation: kernels record the first reference error they find
 * on the device (NonFiniteInput / AllMaskedRow in the sampled-row softmax of
 * ls_score_lines, tensor_ops.py:34-38; EmptyPlan for a head with no selected
 * line in ls_vs_attention, tensor_ops.py:165-166) in a device status word.
 * ls_device_status synchronises `stream`, writes the code (0 = none) to
 * *host_status and clears the word. */
int ls_device_status(int32_t *host_status, ls_stream_t stream);
int ls_version(void);
/* Debugging: host-mapped int buffer where the pipelined kernels record the
 * progress of each role per CTA (NULL disables). */
int ls_debug_set_buffer(void *host_mapped);
/* number of SMs / device name of the current device (diagnostics) */
int ls_device_info(int *sm_count, char *name, int name_len);

/* ---------------------------------------------------------------- K0 ---
 * Row sampling, bit-exact with numpy: replaces Session.head_seed
 * (session.py:84-86) + sample_rows (prefill.py:125-135), i.e. for each layer
 * l in [layer_begin, +n_layers) and head h in [head_begin, +n_heads): rows of
 *   sample_rows(n_new, rate, floor, SeedSequence(session_seed,
 *               spawn_key=(turn, l, h)).generate_state(1, uint64)[0])
 * written sorted to out_rows[l - layer_begin][h - head_begin][0..n_s). n_s is returned by
 * ls_sample_size (prefill.py:132). turn < 0 selects raw-seed mode: session_seed
 * is used directly as the PCG64 seed (sample_rows(..., seed)). alpha >= 1 (session.py:136-137) is the
 * caller's choice: pass rate=1, floor=n_new to get every row.
 * Workspace: ls_sample_rows_workspace(n_layers * n_heads, n_new) bytes.  */
int ls_sample_size(int32_t n_new, double rate, int32_t floor_, int32_t *n_s);
size_t ls_sample_rows_workspace(int32_t n_units, int32_t n_new);
int ls_sample_rows(uint64_t session_seed, int32_t turn, int32_t layer_begin, int32_t n_layers,
                   int32_t head_begin, int32_t n_heads, int32_t n_new, double rate, int32_t floor_,
                   int32_t *out_rows, void *ws, size_t ws_bytes, ls_stream_t stream);
/* Host build of the same generator (used by the CPU tests to pin the bits
 * against numpy; not used by any device path). */
int ls_sample_rows_host(uint64_t session_seed, int32_t turn, int32_t layer, int32_t head,
                        int32_t n_new, double rate, int32_t floor_, int32_t *out_rows);
uint64_t ls_head_seed_host(uint64_t session_seed, int32_t turn, int32_t layer, int32_t head);

/* ---------------------------------------------------------------- K1 ---
 * Sampled-row scoring + line sums: replaces the scoring part of
 * sparsify_head (prefill.py:377-390), softmax_rows (tensor_ops.py:24-40) and
 * _line_sums (prefill.py:138-169) for every head of a layer.
 * rows[h][n_s]: sorted local block rows (K0 output).
 * Outputs (per head, capacity n_total):
 *   v_w[h][c] fp64, v_max[h][c] fp32  (vertical weight / max cell)
 *   s_w[h][d] fp64, s_max[h][d] fp32  (slash weight / max cell)
 *   row_stats[h][n_s][2] fp32 (row max in log2 units, 1/row-sum)
 *   total[h] fp64 (sum of all sampled weights, prefill.py:392)
 *   score_count[h] int64 (OpCounter increments, prefill.py:388-389)     */
size_t ls_score_lines_workspace(const ls_layer_desc *L, int32_t n_s);
int ls_score_lines(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k,
                   const int32_t *rows, double *v_w, float *v_max, double *s_w, float *s_max,
                   float *row_stats, double *total, int64_t *score_count, void *ws,
                   size_t ws_bytes, ls_stream_t stream);
/* Same contract on CUDA cores (tests cross-check the tcgen05 kernel).    */
int ls_score_lines_simt(const ls_layer_desc *L, int32_t n_s, const uint16_t *q, const uint16_t *k,
                        const int32_t *rows, double *v_w, float *v_max, double *s_w, float *s_max,
                        float *row_stats, double *total, int64_t *score_count, void *ws,
                        size_t ws_bytes, ls_stream_t stream);

/* ------------------------------------------------------------- K2+K3+K4 -
 * Line sort + greedy coverage-alpha selection: replaces the sort of
 * _line_sums (prefill.py:168-169) and _greedy (prefill.py:178-229).
 * Consumes ls_score_lines outputs; crossing cells (prefill.py:116-122) are
 * recomputed from q/k and row_stats. Outputs per head:
 *   slash_ids[h][n_total] / vert_ids[h][n_total] sorted ascending,
 *   counts[h][2] = (|S|, |V|), coverage[h], approx[h] (SparsePlan fields),
 *   picks[h][...] pick sequence (kind<<31 | index) in selection order
 *   (capacity 2*n_total) and n_picks[h].                               */
size_t ls_select_lines_workspace(const ls_layer_desc *L, int32_t n_s);
int ls_select_lines(const ls_layer_desc *L, int32_t n_s, double alpha, const uint16_t *q,
                    const uint16_t *k, const int32_t *rows, const double *v_w,
                    const float *v_max, const double *s_w, const float *s_max,
                    const float *row_stats, const double *total, int32_t *slash_ids,
                    int32_t *vert_ids, int32_t *counts, double *coverage, double *approx,
                    int32_t *picks, int32_t *n_picks, void *ws, size_t ws_bytes,
                    ls_stream_t stream);

/* ls_select_lines with the plan build (K4) fused into each head's K3 CTA: head h's
 * slash_ids / vert_ids / counts / picks are written by its CTA, which then sets
 * plan_ready[h] = epoch (device memory, monotonically increasing epochs), so the
 * caller can start the head's sparse attention on another stream with
 * ls_stream_wait_value while slower heads are still selecting. */
int ls_select_lines_ready(const ls_layer_desc *L, int32_t n_s, double alpha, const uint16_t *q,
                          const uint16_t *k, const int32_t *rows, const double *v_w, const float *v_max,
                          const double *s_w, const float *s_max, const float *row_stats, const double *total,
                          int32_t *slash_ids, int32_t *vert_ids, int32_t *counts, double *coverage, double *approx,
                          int32_t *picks, int32_t *n_picks, int32_t *plan_ready, int32_t epoch, void *ws,
                          size_t ws_bytes, ls_stream_t stream);

/* Stream-ordered wait until *addr >= value (device memory; cuStreamWaitValue32 GEQ). */
int ls_stream_wait_value(ls_stream_t stream, const int32_t *addr, int32_t value);

/* Greedy on caller-provided sorted line lists with a dense weight matrix as
 * the cell source: replaces greedy_select_lines (prefill.py:232-251). One
 * head. lines are (index, weight, length, max_cell) sorted by (-w, index);
 * weights[n_rows][n_total] fp64 with positions[n_rows]. Diagnostics/parity. */
int ls_greedy_dense(int32_t n_slash, const int32_t *s_idx, const double *s_w,
                    const int32_t *s_len, const double *s_max, int32_t n_vert,
                    const int32_t *v_idx, const double *v_w, const int32_t *v_len,
                    const double *v_max, double alpha, double total_weight,
                    const double *weights, const int32_t *positions, int32_t n_rows,
                    int32_t n_total, int32_t *slash_ids, int32_t *vert_ids,
                    int32_t *counts, double *coverage, double *approx, void *ws,
                    size_t ws_bytes, ls_stream_t stream);

/* ---------------------------------------------------------------- K5 ---
 * Vertical/slash sparse attention: replaces masked_sparse_attention
 * (tensor_ops.py:141-183) for every head of a layer, with the exact
 * `_row_columns` cell set (tensor_ops.py:130-138) incl. the diagonal
 * fallback. out[r][h][d] (token-major, the head concat of model.py:259),
 * fp32 if out_bf16 == 0 else bf16. cells[h] int64 = OpCounter increments
 * (tensor_ops.py:172-174). Heads with an empty plan -> LS_ERR_EMPTY_PLAN
 * is checked by the host layer (tensor_ops.py:165-166).                 */
size_t ls_vs_attention_workspace(const ls_layer_desc *L);
int ls_vs_attention(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k,
                    const uint16_t *v, const int32_t *slash_ids, const int32_t *vert_ids,
                    const int32_t *counts, void *out, int32_t out_bf16, int64_t *cells,
                    void *ws, size_t ws_bytes, ls_stream_t stream);
/* Same, also counting the 128x128 tensor-core tiles each head executed
 * (tiles[h] int64, the executed-FLOP denominator of the K5 roofline).    */
int ls_vs_attention_ex(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k,
                       const uint16_t *v, const int32_t *slash_ids, const int32_t *vert_ids,
                       const int32_t *counts, void *out, int32_t out_bf16, int64_t *cells,
                       int64_t *tiles, void *ws, size_t ws_bytes, ls_stream_t stream);
/* Same contract on CUDA cores (FFMA, no tensor cores): the cross-check the
 * GPU tests compare the tcgen05 kernel against at full sizes.           */
int ls_vs_attention_simt(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k,
                         const uint16_t *v, const int32_t *slash_ids, const int32_t *vert_ids,
                         const int32_t *counts, void *out, int32_t out_bf16, int64_t *cells,
                         void *ws, size_t ws_bytes, ls_stream_t stream);

/* Dense probability rows of block rows [n_new - n_rows, n_new) under the
 * plan (the decode observation seeds, session.py:89-95):
 * out[h*out_head_stride + i*out_row_stride + c] fp32, zeros off-plan.    */
int ls_plan_rows(const ls_layer_desc *L, int32_t n_rows, const uint16_t *q, const uint16_t *k,
                 const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts,
                 float *out, int64_t out_row_stride, int64_t out_head_stride,
                 ls_stream_t stream);

/* Dense causal attention (scaled_dot_attention, tensor_ops.py:104-127):
 * the lossless baseline / speed-up denominator. out[r][h][d].           */
int ls_dense_attention(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k,
                       const uint16_t *v, void *out, int32_t out_bf16, ls_stream_t stream);

/* ----------------------------------------------------- plan diagnostics ---
 * coverage_ratio (prefill.py:254-281) for every head of
 * a layer: the fraction of the block's FULL causal attention mass (all n_new
 * rows, dense softmax) covered by the plan's lines -- inclusion-exclusion over
 * the single crossing cells == the mass of the union of plan cells. Runs K1's
 * statistics pass over every row (dense normaliser) and K5 with per-row
 * plan-cell normalisers; coverage[h] = mean_r 2^(lse_plan - lse_full).
 * Workspace: ls_plan_coverage_workspace(L) bytes. */
size_t ls_plan_coverage_workspace(const ls_layer_desc *L);
int ls_plan_coverage(const ls_layer_desc *L, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                     const int32_t *slash_ids, const int32_t *vert_ids, const int32_t *counts,
                     double *coverage, void *ws, size_t ws_bytes, ls_stream_t stream);

/* ------------------------------------------------------------- decode ---
 * Decode state of ALL layers of one session, caller-allocated device arrays
 * (see paper_2507_13681_b200/kvcompress.py DecodeStack). The step counters
 * live in device memory so a decode step / an event is a fixed launch
 * sequence (CUDA-graph capturable):
 *   step[0] = cache length before this step's append (= the new token's position)
 *   step[1] = rows appended to the observation deque so far (seeds included);
 *             this step's row goes to slot step[1] % window.
 * Per (layer, q-head) row hr = layer*n_heads + h:
 *   ring_s   [hr][window][row_cap]  fp32 raw log2-domain logits of a row
 *   ring_ml  [hr][window][2]        fp32 (max, sum) of the row; sum == 0 means
 *                                   ring_s holds probabilities (prefill seeds)
 *   ring_ids [hr][window][sparse_cap] int32 ids of compressed rows
 *   ring_n, ring_dense [hr][window] int32; ring_dense: 1 = dense row (ids 0..n-1),
 *            0 = ids in ring_ids, LS_RING_WORKING_SET = the working set of the
 *            current selection (ids: sel_ids[0, n_a) then lo, lo+1, ...; n_a and
 *            lo in ring_ids[0..1]) -- valid until the next compression event
 *   sel_ids  [hr][budget_cap], n_sel [hr]      picked ids (kvcompress.py:212)
 *   ck, cv   [hr][budget_cap][head_dim] bf16   compacted K/V of sel_ids
 *   partials [ls_decode_partials_size() bytes] fp32 split-K partials of a decode step
 *   counters [2 * n_heads] int32, zeroed once: per-unit split arrival / departure counts
 *                      Both may be NULL: splits then combine inside one thread-block
 *                      cluster (at most 16 splits per unit).
 *   n_a      [hr] int32  picked ids below the recent window at the current step
 *                        (written by ls_decode_event, advanced by ls_decode_advance)
 * Archive K/V of layer l, kv-head j at k_all + l*kv_layer_stride + j*kv_head_stride. */
typedef struct ls_decode_stack {
  int32_t n_layers, n_heads, n_kv_heads, head_dim;
  int32_t window;      /* obs_window (kvcompress.py:29-30)   */
  int32_t row_cap;     /* >= max cache length + 1            */
  int32_t sparse_cap;  /* >= budget_cap + window + 1         */
  int32_t budget_cap;  /* >= budget                          */
  int64_t kv_layer_stride, kv_head_stride;
  float *ring_s;
  float *ring_ml;
  int32_t *ring_ids;
  int32_t *ring_n;
  int32_t *ring_dense;
  int32_t *sel_ids;
  int32_t *n_sel;
  uint16_t *ck;
  uint16_t *cv;
  float *partials;
  int32_t *counters;
  int32_t *step;
  int32_t *n_a;
} ls_decode_stack;

/* Working-set decode attention of one layer for the current step
 * (model.py:232-241 inside decode_step, model.py:289-311): out[h][d] and the
 * observation row into the ring. compressed = an event has happened
 * (kvcompress.py:234-237); max_cols bounds the columns of any head. */
size_t ls_decode_partials_size(const ls_decode_stack *S, int32_t max_len);
int ls_decode_step(const ls_decode_stack *S, int32_t layer, const uint16_t *q, const uint16_t *k_layer,
                   const uint16_t *v_layer, int32_t compressed, int32_t max_cols, void *out,
                   int32_t out_bf16, ls_stream_t stream);
/* Same step with q read from the layer's Q archive at position step[0]
 * (q_layer + h*q_head_stride + step[0]*head_dim): no per-step q gather, so a
 * decode step of every layer is one launch per layer. flags: LS_DECODE_PDL
 * launches it as a programmatic dependent of the previous kernel on the stream
 * (its K/V tile prefetch overlaps that kernel's tail; q and all writes wait
 * for it, as the next layer of a full model would). */
#define LS_DECODE_PDL 1
/* compressed rows record (n_a, lo) and K7 derives their ids from the current
 * selection (no per-column id writes): only when every buffered row is consumed
 * before the selection changes again, i.e. interval >= obs_window */
#define LS_DECODE_DERIVED_IDS 2
#define LS_RING_WORKING_SET 2
int ls_decode_step_archive(const ls_decode_stack *S, int32_t layer, const uint16_t *q_layer,
                           int64_t q_head_stride, const uint16_t *k_layer, const uint16_t *v_layer,
                           int32_t compressed, int32_t max_cols, void *out, int32_t out_bf16, int32_t flags,
                           ls_stream_t stream);
/* step[0] += 1 (the new token is in the cache), step[1] += 1 (its row was appended);
 * n_a follows the window start. */
int ls_decode_advance(const ls_decode_stack *S, ls_stream_t stream);
/* Compression event for every layer and head (kvcompress.py:210-224):
 * accumulate the buffered rows oldest first, top-B by (score desc, id asc),
 * sel_ids / n_sel, then the coalesced gather-compaction of K/V (compact_cache,
 * kvcompress.py:133-147). retained_n / score_coverage [n_layers*n_heads]
 * (optional) are the event-log fields. */
size_t ls_decode_select_workspace(const ls_decode_stack *S);
int ls_decode_event(const ls_decode_stack *S, int32_t budget, int32_t max_len, const uint16_t *k_all,
                    const uint16_t *v_all, int32_t *retained_n, double *score_coverage, void *ws,
                    size_t ws_bytes, ls_stream_t stream);

/* ------------------------------------------ reference-API decode pieces ---
 * One call per reference function, for callers that keep the decode state in
 * the reference's own types (numpy ids / rows) -- the drop-in patched onto
 * loopserve.kvcompress / loopserve.model (paper_2507_13681_b200/dropin.py).
 *
 * accumulate_scores (kvcompress.py:67-83): rows r = 0..n_rows-1 oldest first,
 * row r = ids/w[row_ptr[r] .. row_ptr[r+1]), ids distinct within a row and in
 * [0, id_cap). acc[id] = 0.0 + w_0 + w_1 + ... in row order (fp64, the
 * reference's order); touched[id] = 1 for every id some row holds (only those
 * are candidates, kvcompress.py:73-83). LS_ERR_EMPTY_WINDOW for n_rows < 1. */
int ls_accumulate_scores(int32_t n_rows, const int64_t *row_ptr, const int32_t *ids, const double *w,
                         int32_t id_cap, double *acc, uint8_t *touched, ls_stream_t stream);
/* _top_by_score (kvcompress.py:86-90): the budget highest of n (id, score)
 * pairs by (score desc, id asc), written to out[0..budget) in ascending id
 * order; ids distinct, inside [id_lo, id_lo + id_range). *n_out = ids written.
 * Workspace: ls_top_by_score_workspace(id_range) bytes. */
size_t ls_top_by_score_workspace(int32_t id_range);
int ls_top_by_score(int32_t n, const int32_t *ids, const double *scores, int32_t budget, int32_t id_lo,
                    int32_t id_range, int32_t *out, int32_t *n_out, void *ws, size_t ws_bytes, ls_stream_t stream);
/* retained_union (kvcompress.py:126-130): sorted unique union of sel[0..n_sel)
 * and [full_len - recent_window, full_len); ids in [0, cap). out capacity
 * n_sel + recent_window; *n_out = its length. Workspace (cap + 31) / 32 * 4 bytes. */
int ls_retained_union(int32_t n_sel, const int32_t *sel, int32_t recent_window, int32_t full_len, int32_t cap,
                      int32_t *out, int32_t *n_out, void *ws, size_t ws_bytes, ls_stream_t stream);
/* compact_cache's gather (kvcompress.py:133-147, K8): dst row r = the source
 * row whose id (src_ids strictly increasing) equals keep_ids[r], for K rows of
 * k_row_bytes and V rows of v_row_bytes (multiples of 16; 16-byte coalesced
 * copies). *status = 0, or 1 + a keep index whose id is not in the source
 * (-> InvalidIds). */
int ls_kv_compact(int32_t n_src, const int32_t *src_ids, const void *src_k, const void *src_v, int32_t n_keep,
                  const int32_t *keep_ids, int32_t k_row_bytes, int32_t v_row_bytes, void *dst_k, void *dst_v,
                  int32_t *status, ls_stream_t stream);
/* Working-set attention of one decode token for every head of a layer
 * (forward_extend's working-set branch, model.py:232-241): head h attends to
 * cols[col_ptr[h] .. col_ptr[h+1]) of kv-head h / (n_heads / n_kv_heads);
 * bf16 q / K / V (q + h*q_head_stride, k / v + kv*kv_head_stride + pos*head_dim),
 * fp64 arithmetic as the reference's branch. out[h][head_dim] = w . V[cols];
 * w_out[col_ptr[h] + j] = softmax weight of column j (the observation row). */
int ls_gather_attention(int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, const uint16_t *q,
                        int64_t q_head_stride, const uint16_t *k, const uint16_t *v, int64_t kv_head_stride,
                        const int64_t *col_ptr, const int32_t *cols, double *out, double *w_out, ls_stream_t stream);

/* ------------------------------------------------ obswindow baseline ---
 * The observation-window (SnapKV-style) baseline's one-shot selection
 * (session.py:204-230): scores[c] = sum over units u = 0..n_units-1 (every
 * (layer, head), in order) of accumulate_scores of that unit's n_rows dense
 * observation rows (rows + u*unit_stride + r*row_stride, fp32 probabilities,
 * oldest first) -- the summed_over_heads input of select_topB_obs; fp64, the
 * reference's addition order. */
int ls_obs_window_scores(int32_t n_units, int32_t n_rows, const float *rows, int64_t unit_stride,
                         int64_t row_stride, int32_t n_cols, double *scores, ls_stream_t stream);
/* dst + s*dst_slice_bytes + r*row_bytes = src + s*src_slice_bytes + ids[r]*row_bytes
 * for s < n_slices, r < n_ids (row_bytes a multiple of 16): the baseline's
 * compaction of the shared working set for every (layer, kv-head) slice. */
int ls_gather_rows(int32_t n_slices, int32_t n_ids, const int32_t *ids, const void *src, int64_t src_slice_bytes,
                   void *dst, int64_t dst_slice_bytes, int32_t row_bytes, ls_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LOOPSERVE_B200_H */
