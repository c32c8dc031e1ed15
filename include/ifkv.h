/*
 * ifkv.h -- C ABI of the B200 (sm_100a) kernels behind InfoFlow-KV's
 * query-time context-assembly path (assemble -> select -> recompute, reorder).
 *
 * The reference (chunkkv 0.1.0, /root/reference/pkg/src/chunkkv) is pure
 * Python/NumPy and has no FFI layer; its boundary is the Python module API
 * (__init__.py:3-81).  Each entry point below replaces the NumPy arithmetic of
 * one reference function, cited per declaration.  The Python package
 * paper_2603_05353_b200 binds these through ctypes and
 * keeps the reference's names, argument meaning and exceptions.
 *
 * Conventions (all entry points):
 *   - plain device pointers and sizes; no torch types, no allocation inside;
 *   - all work is enqueued on the caller's stream (cudaStream_t passed as
 *     void*), no host synchronisation;
 *   - return 0 on success, IFKV_ERR_ARG for an invalid argument (the Python
 *     layer raises ConfigurationError, errors.py:5), IFKV_ERR_CUDA for a CUDA
 *     launch failure; ifkv_last_error() gives a thread-local message;
 *   - dtype codes: IFKV_F32 (float) or IFKV_BF16 (__nv_bfloat16) for K/V slabs,
 *     weights and activations as stated per argument;
 *   - KV slabs are layer-major [L][rows][Hkv][Dh], rows contiguous, one layer
 *     view = base + l * layer_stride elements.
 */
#ifndef IFKV_H_
#define IFKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IFKV_OK 0
#define IFKV_ERR_ARG 2
#define IFKV_ERR_CUDA 4

#define IFKV_F32 0
#define IFKV_BF16 1

/* output modes of the fused elementwise kernels */
#define IFKV_OUT_F32 0     /* float [rows][d]                                  */
#define IFKV_OUT_BF16 1    /* bf16  [rows][d]                                  */
#define IFKV_OUT_SPLIT3 2  /* bf16  [3][rows][d]: x = hi + mid + lo (fp32-exact
                              operands for the fp32-accurate scoring GEMMs)   */

/* aggregation modes of ifkv_topk_segments (reorder.py:45-54) */
#define IFKV_AGG_NONE (-1)
#define IFKV_AGG_SUM 0
#define IFKV_AGG_MEAN 1
#define IFKV_AGG_MAX 2

const char* ifkv_last_error(void);
int ifkv_abi_version(void);

/* ---- RoPE (model.py:226-270) ------------------------------------------
 * cs[i][j] = (cos, sin)(pos[i] * theta_j), theta_j = base^(-2j/d_head); the
 * angle and the trig are evaluated in fp64 and rounded to fp32 (the reference
 * computes angles in f64, model.py:263).  cs is float[n][d_head/2][2]. */
int ifkv_rope_table(const int64_t* pos, int n, int d_head, double rope_base, float* cs, void* stream);

/* Kernel 1 -- re-rotation of cached keys (rotate_heads model.py:254-270 as
 * used by decode_view cache.py:382-403, score_attention_norm
 * selection.py:152-158 and recompute.py:106-109).
 * dst[l][r] = R(cs[row_table[r]]) src[l][r] over interleaved pairs, for
 * l < n_layers, r < n_rows; row_table[r] < 0 means "delta 0": the row is
 * copied bit-exactly (dst != src) or left untouched (dst == src, in place).
 * src/dst element type = dtype; row_table is a device int32 array. */
int ifkv_rotate_rows(int dtype, const void* src, void* dst, int64_t layer_stride, int n_layers, int n_rows,
                     int heads, int d_head, const int32_t* row_table, const float* cs, void* stream);

/* ---- assemble (cache.py:259-322) ----------------------------------------
 * Gather n_chunks chunk KV caches (each [L][len_c][Hkv][Dh], layer stride
 * src_layer_stride[c] elements) into the slab rows dst_row0[c] ..
 * dst_row0[c]+len_c-1 of dst_k/dst_v (layer stride dst_layer_stride).
 * Pointer / length arrays are HOST arrays (copied into the launch). */
int ifkv_assemble_gather(int dtype, int n_chunks, const void* const* src_k, const void* const* src_v,
                         const int64_t* src_layer_stride, const int32_t* chunk_len, const int32_t* dst_row0,
                         void* dst_k, void* dst_v, int64_t dst_layer_stride, int n_layers, int row_elems,
                         void* stream);

/* ---- fused elementwise (model.py:278-294, recompute.py:95) --------------- */
/* h[rows][d] (fp32) += sum_p delta_p (delta_dtype IFKV_F32/IFKV_BF16, n_parts
 * blocks of rows*d elements, n_parts = 0: no add); then
 * out = rms_norm(h) * gain in out_mode (IFKV_OUT_*).  out may be NULL. */
int ifkv_add_rmsnorm(float* h, const void* delta, int delta_dtype, int n_parts, const float* gain, int rows,
                     int d, int out_mode, void* out, void* stream);
/* a = silu(g) * u with gu = [rows][2*d_ff], gate and up columns interleaved
 * in blocks of gu_block (gate j..j+gu_block-1, then up j.., ...; gu_block =
 * d_ff is the plain [gate | up] layout), summed over n_parts part blocks;
 * out in out_mode. */
int ifkv_silu_mul(const void* gu, int gu_dtype, int n_parts, int rows, int d_ff, int gu_block, int out_mode,
                  void* out, void* stream);
/* h[r] = (float) table[ids[r]] (embedding gather, recompute.py:95). */
int ifkv_embed_rows(const void* table, int dtype, const int64_t* ids, int rows, int d, float* h, void* stream);
/* out = sum over n_parts of x (fp32 blocks of n elements) -> fp32 or split3. */
int ifkv_split3(const float* x, int64_t n, void* out, void* stream);
/* acc[r] += || a[r] - b[r] ||_2 for fp32 [rows][d] (fp64 accumulator): the
 * CacheBlend baseline's per-token hidden-state deviation
 * (replaces np.linalg.norm in selection.py:219-222). */
int ifkv_row_dist_accum(const float* a, const float* b, int rows, int d, double* acc, void* stream);
/* Prompt-row GEMM of the scoring pass (x @ W of model.py:435-455 for the M
 * prompt rows, selection.py:127-169): out[s][r][n] = sum_{p<P} sum_{k in
 * split s} x[p][r][k] w[n][k]; x bf16 [P][R][K] (the split3 terms), w bf16
 * [N][K] ("out x in", W^T of x @ W), out fp32 [splits][R][N] (per-split partials, summed by the
 * consumer's n_parts).  R % 32 == 0, P*R <= 256, K % 64 == 0, N % 128 == 0,
 * 1 <= splits <= K/64.  HBM-bound weight stream on tcgen05 (replaces the
 * cuBLAS calls of the scoring layers). */
int ifkv_prompt_mm(const void* x, int P, int R, int K, const void* w, int N, int splits, float* out, void* stream);

/* ---- projection GEMMs of the layer stack (tcgen05 CTA pairs) -------------
 * C[M][N] = A[M][K] . W[N][K]^T: A bf16 activations (row stride lda), W a bf16
 * weight stored "out x in" (K-major, row stride K).  Replaces the x @ W of
 * recompute.py:98-116 / model.py:433-455 (cuBLAS in round 1).  tile_n: the
 * CTA-pair tile as 1000 + BN (256 rows x BN = 256/224/192/160/128 columns),
 * 0 = chosen by shape.
 *
 * ifkv_gemm: out fp32 or bf16 [M][ldo]; accumulate != 0 (fp32 only) adds into
 * out (h += ctx Wo, h += a Wdown: the residual adds of model.py:448-452). */
int ifkv_gemm(const void* a, int64_t lda, int M, int K, const void* w, int N, int out_dtype, void* out, int64_t ldo,
              int accumulate, int tile_n, void* stream);
/* QKV projection with RoPE and the in-place K/V scatter in the epilogue
 * (recompute.py:99-112 + replace_entries cache.py:354-363): W rows are
 * [wq^T; wk^T; wv^T] (Dh = 128), or only [wk^T; wv^T] when kv_only.  q, k
 * rotated by cs[m] (fp32 (cos, sin) [M][64]); q -> q_out [M][H][128]; k, v ->
 * k_dst / v_dst rows dst_rows[m] (NULL = m) of [*][Hkv][128] bf16 views. */
int ifkv_gemm_qkv_rope_scatter(const void* a, int64_t lda, int M, int K, const void* w, int H, int Hkv,
                               int kv_only, const float* cs, void* q_out, void* k_dst, void* v_dst,
                               const int64_t* dst_rows, int tile_n, void* stream);
/* gate|up projection with SwiGLU in the epilogue (model.py:283-294): W rows
 * interleaved in 64-row blocks (gate j..j+63 | up j..j+63 | ...), 2 d_ff
 * rows; out[m][j] = silu(g_j) u_j, bf16 [M][d_ff]. */
int ifkv_gemm_swiglu(const void* a, int64_t lda, int M, int K, const void* w, int d_ff, void* out, int tile_n,
                     void* stream);

/* ---- fresh q/k/v (model.py:433-437, recompute.py:99-112) ----------------
 * qkv = [rows][(H + 2 Hkv) Dh] (GEMM output, qkv_dtype, n_parts part blocks
 * summed).  q and k are rotated by cs[r] (table rows aligned with qkv rows).
 * q_out [rows][H][Dh] (out_dtype) may be NULL; k/v go to k_dst/v_dst rows
 * dst_rows[r] (device int64; NULL = compact rows r) of a [*][Hkv][Dh] view in
 * out_dtype -- the in-place scatter of replace_entries (cache.py:354-363). */
int ifkv_qkv_rope_scatter(const void* qkv, int qkv_dtype, int n_parts, int rows, int H, int Hkv, int Dh,
                          const float* cs, int out_dtype, void* q_out, void* k_dst, void* v_dst,
                          const int64_t* dst_rows, void* stream);

/* ---- prompt attention over an injected prefix (selection.py:127-169,
 * model.py:297-315 with the causal-with-prefix mask model.py:352-360) -----
 * Work is a list of items; each item attends the query rows of one query
 * group (M prompt rows x H heads) to <= 128 keys: either context slab rows
 * [key_row0, key_row0 + n_keys) read with a rotation delta folded into the
 * query set qset (q . R(d) k == (R(-d) q) . k), or the group's own prompt
 * rows (causal).  Queries are fp32 and pre-rotated per qset:
 * qd [n_qsets][H][M][Dh]. */
typedef struct {
  int32_t group;    /* query group                                          */
  int32_t qset;     /* rotated query set (qd index)                         */
  int32_t key_row0; /* first key row (slab row, or prompt row 0)            */
  int32_t n_keys;   /* number of keys (<= 128 for the SIMT kernels)         */
  int32_t prompt;   /* 1: keys are the group's prompt rows, causal          */
  int32_t score;    /* 1: context item whose columns are scored             */
} ifkv_attn_item;

/* Partial softmax state per (item, head, row): ml = (max, sum exp), o = sum p v.
 * max_keys (<= 128) bounds every item's n_keys and sizes the staging smem
 * (prompt items: M keys -> several CTAs per SM). */
int ifkv_prompt_attn_partial(int kv_dtype, const float* qd, const void* k_slab, const void* v_slab,
                             const float* k_prompt, const float* v_prompt, const ifkv_attn_item* items,
                             int n_items, int max_keys, int H, int Hkv, int M, int Dh, float scale,
                             float* part_ml, float* part_o, void* stream);
/* Merge the partials of each group's items in a fixed order -- its context
 * items [item_begin[g], item_begin[g+1]) then, if prompt_item0 >= 0, its
 * prompt items prompt_item0 + g * n_prompt_items + [0, n_prompt_items) (the
 * prompt's own keys in blocks of <= 128, so any prompt length M works):
 * ctx [G][M][H][Dh] fp32, final ml [G][H][M][2]; ctx_split3 (optional, bf16
 * [3][G*M][H*Dh]) also receives its hi/mid/lo terms (the O-projection GEMM
 * operand). */
int ifkv_prompt_attn_merge(const float* part_ml, const float* part_o, const int32_t* item_begin, int prompt_item0,
                           int n_prompt_items, int G, int H, int M, int Dh, float* ctx, float* ml, void* ctx_split3,
                           void* stream);
/* ifkv_prompt_attn_merge with one warp per (g, h, m) row instead of a CTA:
 * the same contract and item order, for groups of few items (the reorder
 * first pass); its fp32 sums run in item order, so the two entry points may
 * differ in the last bits. */
int ifkv_prompt_attn_merge_rows(const float* part_ml, const float* part_o, const int32_t* item_begin,
                                int prompt_item0, int n_prompt_items, int G, int H, int M, int Dh, float* ctx,
                                float* ml, void* ctx_split3, void* stream);
/* Capture-layer column scores (score_from_attention selection.py:108-124):
 * for each scored item column j, scores[key_row0 + j] =
 * (1/H) sum_h sum_m exp(s_hmj - m_hm) / l_hm, deterministic order. */
int ifkv_score_columns(int kv_dtype, const float* qd, const void* k_slab, const ifkv_attn_item* items, int n_items,
                       const float* ml, int H, int Hkv, int M, int Dh, float scale, float* scores, void* stream);
/* Prompt-row q/k/v of the scoring pass in one pass (model.py:435-437 for the
 * prompt rows + the query-side form of the key re-rotation,
 * selection.py:152-158): qkv = sum of n_parts fp32 blocks [G*M][(H+2Hkv)Dh];
 * q, k rotated by cs[row]; kp, vp fp32 [G*M][Hkv][Dh]; for every query set s
 * of the row's group g (qs_list[qs_begin[g] .. qs_begin[g+1])) qd[s][h][m] =
 * R(-cs_delta[qset_cs[s]]) q (qset_cs < 0: no rotation), qd3 (optional) its
 * bf16 hi/mid/lo terms [n_qsets][3][H][M][Dh]; with qd3 given, qd is written
 * only for the unrotated sets (the SIMT prompt items' input).  max_group_qsets:
 * an upper bound of any group's query-set count (the launch's extent over
 * query sets; the total count is always a valid bound). */
int ifkv_prompt_qkv(const float* qkv, int n_parts, int G, int M, int H, int Hkv, int Dh, const float* cs,
                    const int32_t* qs_begin, const int32_t* qs_list, const int32_t* qset_cs, int max_group_qsets,
                    const float* cs_delta, float* kp, float* vp, float* qd, void* qd3, void* stream);
/* Rotated query sets: qd[s] = R(-cs[qset_cs[s]]) q[qset_group[s]], transposed
 * from q [G][M][H][Dh] to [H][M][Dh]; qset_cs[s] < 0 means no rotation.
 * qd3 (optional, bf16 [n_qsets][3][H][M][Dh]) receives the hi/mid/lo split
 * terms the tensor-core scorer consumes. */
int ifkv_rotate_queries(const float* q, int G, int M, int H, int Dh, const int32_t* qset_group,
                        const int32_t* qset_cs, int n_qsets, const float* cs, float* qd, void* qd3, void* stream);

/* Tensor-core (tcgen05/TMEM/TMA) versions for bf16 slabs with Dh = 128:
 * S = sum_t Q_t K^T and O = sum_t P_t V over hi/mid/lo bf16 terms of the fp32
 * queries / probabilities (exact products, fp32 sums), one CTA per (context
 * item, kv head, <=128-row head chunk); an item may span several 128-key
 * blocks (n_keys <= item_keys, a multiple of 128), streamed through a TMA
 * ring with an online softmax.  Context items only (prompt items go to the
 * SIMT kernel).  n_rows = rows of the slab layer view. */
int ifkv_prompt_attn_tc_supported(int kv_dtype, int H, int Hkv, int M, int Dh);
int ifkv_prompt_attn_partial_tc(const void* qd3, int n_qsets, const void* k_slab, const void* v_slab, int n_rows,
                                const ifkv_attn_item* items, int n_items, int item_keys, int H, int Hkv, int M,
                                float scale, float* part_ml, float* part_o, void* stream);
/* colsum_ws: fp32 [n_items][Hkv * head_chunks][item_keys] workspace. */
int ifkv_score_columns_tc(const void* qd3, int n_qsets, const void* k_slab, int n_rows, const ifkv_attn_item* items,
                          int n_items, int item_keys, const float* ml, int H, int Hkv, int M, float scale,
                          float* colsum_ws, float* scores, void* stream);

/* ---- top-k (selection.py:172-183) and per-chunk importance
 * (reorder.py:84-112) -----------------------------------------------------
 * For each segment s (scores[seg_begin[s] .. seg_begin[s+1])), write the
 * seg_k[s] best indices by (score desc, index asc), ascending, as GLOBAL
 * indices into out_idx[out_begin[s] ...]; optionally aggregate the selected
 * scores (IFKV_AGG_*) into agg[s] (fp64 accumulation).  All arrays device. */
int ifkv_topk_segments(const float* scores, const int32_t* seg_begin, const int32_t* seg_k,
                       const int32_t* out_begin, int n_seg, int64_t* out_idx, int agg_mode, double* agg,
                       void* stream);

/* ---- selective recompute attention (recompute.py:92-114) ----------------
 * Query row i (head h) attends keys 0..horizon[i] of the layer's K/V view
 * [n_rows][Hkv][Dh] (kv head h / (H/Hkv)); horizons ascending, < n_rows.
 * q [S][H][Dh], out [S][H][Dh], element type dtype, fp32 softmax. */
int ifkv_recompute_attn(int dtype, const void* q, const void* k_layer, const void* v_layer,
                        const int64_t* horizon, int S, int H, int Hkv, int Dh, int n_rows, float scale, void* out,
                        void* stream);
/* Key ranges instead of prefixes: query row i attends keys key_start[i] ..
 * horizon[i] (device int64; the block-diagonal causal mask of the batched
 * chunk prefill, cache.py:74-99 for all chunks in one launch: every chunk's
 * tokens see only their own chunk).  Tiles are consecutive rows, so
 * key_start should be non-decreasing for efficiency (not for correctness). */
int ifkv_recompute_attn_range(int dtype, const void* q, const void* k_layer, const void* v_layer,
                              const int64_t* key_start, const int64_t* horizon, int S, int H, int Hkv, int Dh,
                              int n_rows, float scale, void* out, void* stream);
/* The two implementations behind it (selected automatically): the tcgen05 /
 * TMEM / TMA kernel for bf16, Dh = 128, H/Hkv <= 16; and the generic
 * SIMT fp32-softmax kernel (fp32 mode, other head sizes). */
int ifkv_recompute_attn_tc_supported(int dtype, int H, int Hkv, int Dh);
int ifkv_recompute_attn_simt(int dtype, const void* q, const void* k_layer, const void* v_layer,
                             const int64_t* horizon, int S, int H, int Hkv, int Dh, int n_rows, float scale,
                             void* out, void* stream);
/* Chunk-sharded recompute: the same attention over this rank's
 * local keys only, returning the partial softmax state -- out = normalised
 * local context (0 when no key is visible), ml_out [S][H][2] = (max, sum exp)
 * -- for the cross-rank merge.  horizon[i] may be -1 (no local key <= the
 * query's global index). */
/* Merge P partial attentions of the same queries over disjoint key sets (the
 * chunk-sharded recompute, recompute.py:114 over every rank's keys): part_o
 * bf16 [P][rows][Dh] each normalised by its own sum, part_ml fp32
 * [P][rows][2] = (max in natural-log units, sum); out bf16 [rows][Dh],
 * optional ml_out [rows][2].  Fixed p order (deterministic). */
int ifkv_merge_partials(const void* part_o, const float* part_ml, int P, int64_t rows, int Dh, void* out,
                        float* ml_out, void* stream);
/* The same merge for the scoring pass's per-layer prompt states (chunk
 * sharding, selection.py:127-169 over every rank's keys): part_ctx fp32
 * [P][G][M][H][Dh], part_ml fp32 [P][G][H][M][2] -> out_ctx [G][M][H][Dh],
 * out_ml [G][H][M][2]. */
int ifkv_merge_prompt_states(const float* part_ctx, const float* part_ml, int P, int G, int M, int H, int Dh,
                             float* out_ctx, float* out_ml, void* stream);
int ifkv_recompute_attn_partial(int dtype, const void* q, const void* k_layer, const void* v_layer,
                                const int64_t* horizon, int S, int H, int Hkv, int Dh, int n_rows, float scale,
                                void* out, float* ml_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IFKV_H_ */
