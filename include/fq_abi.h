/*
 * fq_abi.h — C-ABI of the B200 (sm_100a) LightSeq inference hot path.
 *
 * This is the drop-in boundary under the reference's Python operator API
 * (`fuseq`, /root/reference/pkg/src/fuseq). Every entry point below replaces
 * one call site of the reference's kernel layer (`kernels.py`, numba) or GEMM
 * layer (`tensor.py`, numpy->OpenBLAS); the comment on each names it. The
 * Python package `paper_2010_13887_b200` binds these with ctypes exactly where
 * the reference calls `kernels.*` / `np.matmul`.
 *
 * Conventions:
 *  - plain device pointers, element counts and leading dimensions (in
 *    elements), plus the CUDA stream (`fq_stream_t` = cudaStream_t);
 *  - no allocation inside, no hidden global state, stream-ordered, reentrant;
 *    every workspace comes from the caller's (torch-held) arena;
 *  - return int: 0 = OK; < 0 = error (enum fq_status, message via
 *    fq_last_error()); the softmax/bad-row count is reported through a device
 *    int written by the kernel (kernels never raise, kernels.py:139).
 *  - graph-capturable: entry points that depend on the decode position read it
 *    from a device int (`d_cur`) so a captured step can be replayed.
 */
#ifndef FQ_ABI_H
#define FQ_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* fq_stream_t;

enum fq_status {
  FQ_OK = 0,
  FQ_ERR_DIMENSION = -1,   /* errors.py:8  DimensionError  */
  FQ_ERR_PARAMETER = -2,   /* errors.py:36 ParameterError  */
  FQ_ERR_ALIASING = -3,    /* errors.py:12 AliasingError   */
  FQ_ERR_CAPACITY = -4,    /* errors.py:20 CapacityError   */
  FQ_ERR_CUDA = -5,        /* launch / runtime failure      */
  FQ_ERR_UNSUPPORTED = -6  /* dtype/shape combination not built */
};

enum fq_dtype { FQ_F32 = 0, FQ_F16 = 1 };
enum fq_act { FQ_ACT_NONE = 0, FQ_ACT_RELU = 1, FQ_ACT_GELU = 2 }; /* ops.py:61 */

/* ---- library ---------------------------------------------------------- */
int fq_abi_version(void);
const char* fq_last_error(void);
int fq_num_sms(void);
/* Programmatic dependent launch for later launches / captures: 1 on, 0 off,
 * -1 back to the FQ_PDL environment default (on). Not a reference interface:
 * the benchmark's clean kernel timeline (PDL overlaps kernel durations). */
int fq_set_pdl(int mode);
/* Opt every kernel into the shared-memory sizes it may request, once, before
 * any stream capture (cudaFuncSetAttribute is not a stream operation). */
int fq_prepare(void);

/* ---- fused elementwise passes (kernels.py) ---------------------------- */

/* kernels.py:22 layer_norm_kernel. x fp32 [rows, d] (ldx); outputs optional:
 * out (fp32, ldo) and/or out16 (fp16, ldo16; the next GEMM's operand). */
int fq_layer_norm(const float* x, int64_t ldx, const float* gamma, const float* beta,
                  double eps, int64_t rows, int64_t d, float* out, int64_t ldo,
                  void* out16, int64_t ldo16, fq_stream_t stream);

/* kernels.py:57 bias_residual_layer_norm_kernel: LN((x + bias) + residual). */
int fq_bias_residual_layer_norm(const float* x, int64_t ldx, const float* bias,
                                const float* residual, int64_t ldr, const float* gamma,
                                const float* beta, double eps, int64_t rows, int64_t d,
                                float* out, int64_t ldo, void* out16, int64_t ldo16,
                                fq_stream_t stream);

/* The split-K consumer of fq_gemm_ln's slab path: LN((sum_s slabs[s] +
 * bias) + residual), slabs [nslab][rows][ld] fp32 (slab s = the GEMM's K
 * slice s), summed in slab order — bit-identical to the split-K GEMM's
 * in-kernel reduction followed by fq_layer_norm. nslab in {2, 4}, d in
 * {512, 1024, 2048}, 16-byte aligned rows. */
int fq_splitk_bias_residual_layer_norm(const float* slabs, int nslab, int64_t ld,
                                       const float* bias, const float* residual, int64_t ldr,
                                       const float* gamma, const float* beta, double eps,
                                       int64_t rows, int64_t d, float* out, int64_t ldo,
                                       void* out16, int64_t ldo16, fq_stream_t stream);

/* kernels.py:39 bias_residual_act_kernel: act(x + bias) (+ residual). In place
 * allowed (out == x). act: enum fq_act. residual may be NULL. */
int fq_bias_residual_act(const float* x, int64_t ldx, const float* bias,
                         const float* residual, int64_t ldr, int act, int64_t rows,
                         int64_t d, float* out, int64_t ldo, fq_stream_t stream);

/* kernels.py:77 qkv_bias_reshape_kernel: [batch*seq, 3d] + bias -> q,k,v each
 * contiguous [batch, heads, seq, head_dim]. */
int fq_qkv_bias_reshape(const float* qkv, int64_t ldq, const float* bias, int64_t batch,
                        int64_t seq, int64_t heads, int64_t head_dim, float* q, float* k,
                        float* v, fq_stream_t stream);

/* kernels.py:93 bias_reshape_heads_kernel: [batch*seq, d] + bias -> [batch, heads, seq, hd]. */
int fq_bias_reshape_heads(const float* x, int64_t ldx, const float* bias, int64_t batch,
                          int64_t seq, int64_t heads, int64_t head_dim, float* out,
                          fq_stream_t stream);

/* kernels.py:106 scale_mask_softmax_kernel over a [b, h, q, l] view whose
 * rows (length l) are `ld` apart (the decoder's sscores[..., :cur] slice,
 * model.py:574). mask: NULL or [b, l] of {0,-inf}. The number of fully masked
 * rows is written to *d_bad (device int, may be NULL). In place allowed. */
int fq_scale_mask_softmax(const float* scores, int64_t ld, float* out, int64_t ldo,
                          int64_t b, int64_t h, int64_t q, int64_t l, float scale,
                          const float* mask, int* d_bad, fq_stream_t stream);

/* kernels.py:143 embed_scale_pos_kernel: out[i] = emb[tok[i]]*scale + pos[i%seq + off].
 * If d_off != NULL the offset is read from device memory (graph replay).
 * out (fp32) and/or out16 (fp16) may be NULL. */
int fq_embed_scale_pos(const int64_t* tokens, int64_t n, const float* emb, int64_t d,
                       float scale, const float* pos, int64_t pos_offset,
                       const int32_t* d_off, int64_t seq, float* out, void* out16,
                       fq_stream_t stream);

/* Diversity penalty of diverse beam search, decode.py:291-295 ->
 * kernels.py:215-219: out[r, j] = logits[r, j] - lam * counts[j] (f64
 * arithmetic, rounded to fp32, as numba types it). */
int fq_penalize_counts(const float* logits, int64_t ld, int64_t rows, int64_t vocab,
                       const int32_t* counts, float lam, float* out, int64_t ldo,
                       fq_stream_t stream);

/* kernels.py:205 kv_append_kernel: dst[r,:,cur,:] = new[r,:,0,:], dst [R,h,S,hd]. */
int fq_kv_append(const float* new_k, const float* new_v, int64_t cur, int64_t rows,
                 int64_t heads, int64_t max_seq, int64_t head_dim, float* dst_k,
                 float* dst_v, fq_stream_t stream);

/* kernels.py:189 kv_gather_append_kernel (ping-pong beam reorder):
 * dst[r,:,:cur] = src[parents[r],:,:cur]; dst[r,:,cur] = new[r,:,0]. */
int fq_kv_gather_append(const float* src_k, const float* src_v, const float* new_k,
                        const float* new_v, const int64_t* parents, int64_t cur,
                        int64_t rows, int64_t heads, int64_t max_seq, int64_t head_dim,
                        float* dst_k, float* dst_v, fq_stream_t stream);

/* ---- GEMM (tensor.py:179 gemm, :207 gemm_batched) --------------------- */

/* out = LN(a . w^T + bias + residual) (fp16 operands, fp32 out, optional fp16
 * copy): model.py:596-627's GEMM + fused_bias_residual_layer_norm pairs
 * (kernels.py:57-73). When the GEMM runs split-K over 128-column tiles:
 * - ws >= split * M * N * 4 bytes (slab path, the engine default): the split-K
 *   GEMM writes one fp32 partial slab per K slice into ws with no in-kernel
 *   reduction, then fq_splitk_bias_residual_layer_norm sums them (same order,
 *   same bits as the reduced GEMM + LN);
 * - else ws >= M * (N/128) * 16 + ceil(M/128) * 8 bytes, zeroed once, and all
 *   clusters fit on the GPU at once: one launch, the LN statistics of a row
 *   block exchanged between its CTAs through ws (the counters reset
 *   themselves).
 * Otherwise the GEMM then fq_layer_norm. One launch per stream at a time. */
int fq_gemm_ln(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
               const float* res, int64_t ldr, const float* gamma, const float* beta, double eps,
               float* out, int64_t ldo, void* out16, int64_t ldo16, void* ws, int64_t ws_bytes,
               int64_t M, int64_t N, int64_t K, fq_stream_t stream);

/* The split-K fp16 GEMM's per-K-slice fp32 partials without the reduction:
 * ws [nslab][M][N], slab s = a[:, slice s] . w[:, slice s]^T (a [M,K], w
 * [N,K]). Sets *nslab = 0 and launches nothing when this shape's plan is not
 * split-K or ws < split * M * N * 4 bytes. The consumer sums the slabs in slab
 * order (fq_splitk_bias_residual_layer_norm, fq_cross_attention_slabs), which
 * reproduces the split-K kernel's own reduction bit for bit. */
int fq_gemm_splitk_slabs(const void* a, int64_t lda, const void* w, int64_t ldw, void* ws,
                         int64_t ws_bytes, int64_t M, int64_t N, int64_t K, int* nslab,
                         fq_stream_t stream);

/* C[M,N] = epilogue(A[M,K] @ op(B)); op(B) = B [K,N] (ldb) or B^T with B
 * [N,K] when transpose_b. Epilogue (fused, fp32 math): t = acc (+ C if
 * accumulate) (+ bias[N]); t = act(t); t = t + residual[M,N] (ldr).
 * dtypes: a_dtype == b_dtype. FQ_F32 operands with transpose_b (K-major B),
 * 16-byte aligned rows and an fp32 C: the exact-mode 3xTF32 tcgen05 kernel
 * (fq_gemm_f32x3 with b_lo = NULL); other FQ_F32 layouts: the SIMT FFMA
 * kernel (sequential K order, M-independent; API use only). FQ_F16 operands
 * require transpose_b (weights pre-laid-out [N,K]) and run on tcgen05 tensor
 * cores (TMEM accumulators, TMA-fed, fp32 accumulate). c_dtype: FQ_F32 or
 * FQ_F16. */
int fq_gemm(const void* a, int a_dtype, int64_t lda, const void* b, int b_dtype, int64_t ldb,
            int transpose_b, void* c, int c_dtype, int64_t ldc, int64_t M, int64_t N,
            int64_t K, int accumulate, const float* bias, const float* residual, int64_t ldr,
            int act, fq_stream_t stream);

/* Exact fp32 mode on the tensor cores (replaces tensor.py:179-204's OpenBLAS
 * SGEMM on the engine path): C = epilogue(A . B^T) as in fq_gemm, A [M,K]
 * fp32, B [N,K] fp32 K-major. Each operand is split into tf32 hi + lo (x =
 * hi + lo to 2^-22) and the product is accumulated as a_hi.b_lo + a_lo.b_hi +
 * a_hi.b_hi on kind::tf32 tcgen05 MMAs into an fp32 TMEM accumulator (3xTF32).
 * b_lo = NULL: B is raw fp32 and is split in shared memory next to A; else b /
 * b_lo are B's pre-split hi / lo (fq_split_tf32, once at weight load). The K
 * order depends on (N, K) only: results are bitwise independent of M. */
int fq_gemm_f32x3(const float* a, int64_t lda, const float* b, const float* b_lo, int64_t ldb,
                  float* c, int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate,
                  const float* bias, const float* residual, int64_t ldr, int act,
                  fq_stream_t stream);

/* out = LN(a . b^T + bias + residual) in exact mode (fq_gemm_f32x3 operands):
 * when the plan splits K in 4 and ws >= 4 * M * N * 4 bytes, the K-slice
 * partials go to ws as slabs summed by fq_splitk_bias_residual_layer_norm in
 * slice order; else the GEMM (bias + residual fused) then fq_layer_norm. */
int fq_gemm_f32x3_ln(const float* a, int64_t lda, const float* b, const float* b_lo,
                     int64_t ldb, const float* bias, const float* res, int64_t ldr,
                     const float* gamma, const float* beta, double eps, float* out, int64_t ldo,
                     void* ws, int64_t ws_bytes, int64_t M, int64_t N, int64_t K,
                     fq_stream_t stream);

/* Exact fp32 mode, 3xFP16 (replaces tensor.py:179-204's OpenBLAS SGEMM on the
 * engine path): C = epilogue(A . B^T) as in fq_gemm with A [M,K] and B [N,K]
 * given as fp16 pairs x = hi + lo * 2^-11 (fq_split_f16; the producing
 * kernels write them directly). tcgen05 kind::f16 MMAs accumulate
 * a_hi.b_hi and a_hi.b_lo + a_lo.b_hi into two fp32 TMEM accumulators, summed
 * with RN adds every 128 K elements; the K order depends on (N, K) only
 * (bitwise independent of M). 22-bit operand precision, like 3xTF32, at the
 * kind::f16 rate and half the operand bytes. Operands |x| < 65504. */
int fq_gemm_x3h(const void* a, const void* a_lo, int64_t lda, const void* b, const void* b_lo,
                int64_t ldb, float* c, int64_t ldc, int64_t M, int64_t N, int64_t K,
                int accumulate, const float* bias, const float* residual, int64_t ldr, int act,
                fq_stream_t stream);

/* fq_gemm_x3h whose output act(a . b^T + bias) is written only as the next
 * exact-mode GEMM's fp16 pair: c = hi, c_lo = lo, both [M, ldc] fp16 (the
 * FFN1 and cross-K/V projections, whose only consumers read the pair). */
int fq_gemm_x3h_pair(const void* a, const void* a_lo, int64_t lda, const void* b,
                     const void* b_lo, int64_t ldb, void* c, void* c_lo, int64_t ldc, int64_t M,
                     int64_t N, int64_t K, const float* bias, int act, fq_stream_t stream);

/* out = LN(a . b^T + bias + residual) with fq_gemm_x3h operands (the closing
 * GEMM + LN pairs, model.py:339-358 / :582-626); out16 / out16_lo (optional)
 * receive the output's fp16 pair for the next exact-mode GEMM. The 4-slice
 * plan writes K-slice slabs to ws, summed in slice order by the LN kernel. */
/* Exact-mode GEMM as split-K partial slabs only ([S][M][N] fp32 in ws, slab s
 * = K slice s) for the K/4-slice shapes (N <= 1024, K >= 1024); *nslab (host
 * int) receives S. FQ_ERR_UNSUPPORTED for other shapes. */
int fq_gemm_x3h_slabs(const void* a, const void* a_lo, int64_t lda, const void* b,
                      const void* b_lo, int64_t ldb, void* ws, int64_t ws_bytes, int64_t M,
                      int64_t N, int64_t K, int32_t* nslab, fq_stream_t stream);
int fq_gemm_x3h_ln(const void* a, const void* a_lo, int64_t lda, const void* b,
                   const void* b_lo, int64_t ldb, const float* bias, const float* res,
                   int64_t ldr, const float* gamma, const float* beta, double eps, float* out,
                   int64_t ldo, void* out16, void* out16_lo, int64_t ldo16, void* ws,
                   int64_t ws_bytes, int64_t M, int64_t N, int64_t K, fq_stream_t stream);

/* fp16 pairs (hi, lo) of a row-major fp32 [rows, cols] matrix (leading dim
 * lds): x = hi + lo * 2^-11. transpose: hi/lo are [cols, rows] (the K-major
 * layout of a [K, N] weight; ldo >= rows), else [rows, cols] (ldo >= cols). */
int fq_split_f16(const float* src, int64_t lds, int64_t rows, int64_t cols, int transpose,
                 void* hi, void* lo, int64_t ldo, fq_stream_t stream);

/* fq_layer_norm / fq_splitk_bias_residual_layer_norm whose fp16 output is the
 * exact mode's pair: out16 = hi, out16_lo = lo (fq_split_f16 semantics). */
int fq_layer_norm_xh(const float* x, int64_t ldx, const float* gamma, const float* beta,
                     double eps, int64_t rows, int64_t d, float* out, int64_t ldo, void* out16,
                     void* out16_lo, int64_t ldo16, fq_stream_t stream);
int fq_splitk_bias_residual_layer_norm_xh(const float* slabs, int nslab, int64_t ld,
                                          const float* bias, const float* residual, int64_t ldr,
                                          const float* gamma, const float* beta, double eps,
                                          int64_t rows, int64_t d, float* out, int64_t ldo,
                                          void* out16, void* out16_lo, int64_t ldo16,
                                          fq_stream_t stream);

/* Weight preparation for fq_gemm_f32x3 (once, at load): hi = tf32(src) (round
 * to nearest, ties away), lo = tf32(src - hi); src [rows, cols] row-major;
 * transpose: hi/lo are [cols, rows] (the K-major layout of a [K, N] weight). */
int fq_split_tf32(const float* src, int64_t rows, int64_t cols, int transpose, float* hi,
                  float* lo, fq_stream_t stream);

/* Tile width and thread-block-cluster shape (cm x cn CTAs sharing A/B tiles
 * through TMA multicast) the fp16 dispatcher picks for an M x N x K GEMM. */
int fq_gemm_plan(int64_t M, int64_t N, int64_t K, int* bn, int* cm, int* cn, int* split);

/* Strided batched fp32 GEMM over a two-level batch (i0 < n0, i1 < n1):
 * operand X of batch (i0,i1) starts at X + i0*sX0 + i1*sX1 (elements).
 * Covers every gemm_batched call site of model.py (QK^T, P.V into the
 * merged-head strided view, the sscores[..., :cur] slice). */
int fq_gemm_batched(const float* a, int64_t lda, int64_t sa0, int64_t sa1, const float* b,
                    int64_t ldb, int64_t sb0, int64_t sb1, int transpose_b, float* c,
                    int64_t ldc, int64_t sc0, int64_t sc1, int64_t n0, int64_t n1,
                    int64_t M, int64_t N, int64_t K, fq_stream_t stream);

/* ---- HARS output layer (decode.py) ------------------------------------ */

/* Stage 1, decode.py:58 retrieve -> kernels.py:155 retrieve_kernel, one HBM
 * sweep per row: strided group maxima (token j -> group j % k), threshold
 * R = min_g m_g, lse = f64(row_max) + log(sum f64(expf(x - row_max))), and the
 * candidates x >= R in ascending token order (cand_idx [rows, cand_ld]; rows
 * whose count exceeds cand_ld are flagged by count > cand_ld and truncated).
 * k per row: d_k[row] if d_k != NULL (0 = skip row) else k; with d_k, k is an
 * upper bound on the d_k entries. */
int fq_retrieve(const float* logits, int64_t ld, int64_t rows, int64_t vocab, int64_t k,
                const int32_t* d_k, float* group_max, int64_t gm_ld, float* threshold,
                double* lse, int32_t* cand_idx, int64_t cand_ld, int64_t* cand_count,
                fq_stream_t stream);

/* Device-resident beam state for `batch` items of beam K (decode.py:140). */
typedef struct fq_beam_state {
  int32_t* live;        /* [B] number of live beams (prefixes)            */
  int32_t* step;        /* [B] BeamState.step                             */
  int32_t* done;        /* [B] engine.py:154 done flags                    */
  int32_t* prefix;      /* [B, K, max_len] live prefixes                  */
  double* cum;          /* [B, K] cum_log_prob                            */
  int32_t* fin_count;   /* [B]                                            */
  int32_t* fin_tok;     /* [B, K, max_len] finished sequences             */
  int32_t* fin_len;     /* [B, K]                                         */
  double* fin_score;    /* [B, K]                                         */
  int32_t* last_tok;    /* [B, K] last_tokens                             */
  int32_t* parent;      /* [B, K] parents (item-local)                    */
  int32_t* n_done;      /* [1] count of done items                        */
} fq_beam_state;

/* Stage 2, decode.py:217-240 beam_search_step + :192 _apply_selection +
 * :186 _finished_insert + :160 should_stop, and the engine's per-item loop
 * engine.py:148-169, for every item at once (one CTA per item):
 * rerank score = cum + (f64(logit) - lse), order (-score, token, beam), walk.
 * len_pow: NULL when the length penalty alpha is 0, else a device table
 * len_pow[l] = l ** alpha (l = 0..max_len) computed by the host's libm, so the
 * penalised scores are bit-identical to decode.py:203 / :170.
 * Writes next-step row tokens/parents (int64 [B*K]) and, when hist != NULL,
 * the copy-free KV history table hist [B*K, max_len] (positions 0..cur).
 * The step t (= *d_cur, else the item's step) is the engine's last when
 * t == max_steps-1 (engine.py:150). Workspace: unused, may be NULL. */
int fq_hars_select(const float* logits, int64_t ld, const double* lse,
                   const int32_t* cand_idx, int64_t cand_ld, const int64_t* cand_count,
                   fq_beam_state st, int64_t batch, int64_t beam, int64_t vocab,
                   int64_t max_len, int64_t eos, const double* len_pow, const int32_t* d_cur,
                   int64_t max_steps, int64_t* row_tokens, int64_t* row_parents, int32_t* hist,
                   void* workspace, int64_t ws_bytes, fq_stream_t stream);

/* groups per row for stage 1: d_k[b*K+i] = i < live[b] && !done[b] ?
 * min(K + live[b], V) : 0 (decode.py:230). exhaustive -> V. */
int fq_hars_groups(fq_beam_state st, int64_t batch, int64_t beam, int64_t vocab,
                   int exhaustive, int32_t* d_k, fq_stream_t stream);

/* The whole HARS step of a decode step in one launch (engine.py:148-169 +
 * decode.py:217-240 + model.py:508-512): per row the group count
 * min(K + live, V) (decode.py:230), stage 1 (single-sweep retrieve), and for
 * each item, run by the last of its rows to finish, stage 2 (fq_hars_select
 * semantics); the last item advances *d_cur. counters: int32
 * [batch + 1 + batch*beam] (item, all-items and per-row counters: the split
 * layout's row arrivals, the row layout's top-list marks; zero between launches),
 * zero-initialised once (they reset themselves). For long rows (V >= 64k) or
 * <= 8 rows stage 1 runs on the balanced split (every CTA of one wave streams
 * an equal share of the [rows, V] block; the CTA completing a row merges it). Needs 2*beam <= 32 and
 * 16-byte aligned rows; exhaustive search uses the separate entry points.
 * With x_next != NULL the item's rows of the next step's decoder input are
 * also written (embed_scale_pos at position *d_cur + 1, kernels.py:143-151:
 * fp32 emb[token] * emb_scale + pos[position], row-major [rows, d_model],
 * x16_next an optional fp16 copy; with x16_next_lo the exact mode's fp16 pair hi / lo),
 * replacing the next step's embedding launch. */
int fq_hars_step(const float* logits, int64_t ld, fq_beam_state st, int64_t batch, int64_t beam,
                 int64_t vocab, int64_t max_len, int64_t eos, const double* len_pow,
                 int32_t* d_cur, int64_t max_steps, double* lse, int32_t* cand_idx,
                 int64_t cand_ld, int64_t* cand_count, int32_t* counters, int64_t* row_tokens,
                 int64_t* row_parents, int32_t* hist, const float* emb, int64_t d_model,
                 float emb_scale, const float* pos, float* x_next, void* x16_next,
                 void* x16_next_lo, fq_stream_t stream);

/* The decode step's output layer without materialising the [rows, V]
 * logits: the tied-embedding logits GEMM (x16 [rows, d] fp16 .
 * emb16 [vocab, d]^T, tcgen05) whose epilogue computes HARS stage 1's
 * statistics per row and column tile: strided group maxima folded into the
 * row's running maxima gmax [rows][32] (ordered ints, -inf between steps) with
 * global atomics, the tile-row maximum tmax and sum of exp(x - tmax) tsum
 * ([rows][ldt], column tiles of 224: ldt >= ceil(vocab/224)), and every element >= the
 * tile-local bound min_g(tile group max) <= R stored in the tile-row's own slots
 * sv [rows][ldt][sv_cap] (int2 column, value bits) with its count in
 * sv_cnt [rows][ldt] (> sv_cap: overflow). dk [rows]: group count per row (0 =
 * skip). Replaces model.py:627-629 + decode.py:58-92 stage 1. */
int fq_logits_hars(const void* x16, int64_t ldx, const void* emb16, int64_t lde, int64_t rows,
                   int64_t vocab, int64_t d, const int32_t* dk, int32_t* gmax, float* tmax,
                   double* tsum, int64_t ldt, int32_t* sv_cnt, void* sv, int64_t sv_cap,
                   fq_stream_t stream);

/* Completes fq_logits_hars: per row R, M, lse (fixed-order f64 merge of the
 * tile sums) and the ordered candidates x >= R from the survivors; then per
 * item stage 2 + next-step embedding + position advance exactly as
 * fq_hars_step, and the item's group counts for the next step in dk. Resets
 * gmax. ntiles <= 256. counters: int32 [batch + 1] zeroed once; d_ovf counts
 * survivor-slot overflows and rows with more than 2048 candidates (tie-heavy
 * logits; not supported on this path). */
int fq_hars_merge_step(fq_beam_state st, int64_t batch, int64_t beam, int64_t vocab,
                       int64_t max_len, int64_t eos, const double* len_pow, int32_t* d_cur,
                       int64_t max_steps, int32_t* dk, int32_t* gmax, const float* tmax,
                       const double* tsum, int64_t ldt, int64_t ntiles, int32_t* sv_cnt,
                       const void* sv, int64_t sv_cap, double* lse, int32_t* cand_idx,
                       int64_t cand_ld, int64_t* cand_count, int32_t* counters, int32_t* d_ovf,
                       int64_t* row_tokens, int64_t* row_parents, int32_t* hist,
                       const float* emb, int64_t d_model, float emb_scale, const float* pos,
                       float* x_next, void* x16_next, void* x16_next_lo,
                       fq_stream_t stream);

/* Reset beam state to BeamState() (decode.py:145-151) for every item. */
int fq_beam_state_init(fq_beam_state st, int64_t batch, int64_t beam, int64_t max_len,
                       fq_stream_t stream);

/* HOST helper (no device work): BeamState.finalize (decode.py:173-183) for a
 * whole batch from the host copy of an fq_beam_state (all pointers HOST
 * arrays): finished list + non-empty live prefixes not already finished
 * (score cum / len**alpha), stably sorted by (-score, sequence), the first
 * `keep` per item into out_tok [batch][keep][max_len], out_len, out_score,
 * out_n [batch]. */
int fq_finalize_beams(const int32_t* live, const int32_t* step, const int32_t* prefix,
                      const double* cum, const int32_t* fin_count, const int32_t* fin_tok,
                      const int32_t* fin_len, const double* fin_score, int64_t batch, int64_t K,
                      int64_t max_len, double alpha, int64_t keep, int32_t* out_tok,
                      int32_t* out_len, double* out_score, int32_t* out_n);

/* *d_cur += 1 (KVCache.end_step, model.py:508-512). */
int fq_step_advance(int32_t* d_cur, fq_stream_t stream);

/* Device-resident sampling step (Session._sampling_step, engine.py:175-195;
 * sample_top_k / sample_top_p + _draw, decode.py:378-430) for every row of one
 * decode step, after fq_retrieve with per-row group counts dk (live rows: k
 * for top-k, `groups` for top-p; 0 done): survivors sorted by (-logit, token),
 * probs exp(f64 logit - lse); top-k (k >= 1) keeps the first k, top-p (k = 0)
 * cuts the sorted prefix at the first cumulative sum >= top_p
 * (np.searchsorted "left"); r = u * probs.sum() (numpy pairwise order), the
 * first token with r <= the running sum. uniforms: the reference's PCG64
 * stream in its draw order (one per live row per step, rows in batch order),
 * consumed through *draw. done int32 [2][batch] (step parity t = *d_cur: read
 * [t & 1], write [(t + 1) & 1]); writes out_tok[b][t] (int32
 * [batch][max_len]), out_len, fin (EOS), the next step's dk_next / tokens (0
 * for done rows); the last CTA advances *draw and *d_cur and stores the
 * live-row count in counters[1] (counters int32 [2], zero once). err != 0: a
 * row had > 1024 survivors (1), the uniform stream ran out (2), or a top-p
 * row's survivors miss the nucleus (3, the reference escalates its group
 * count) -- re-run the request on the host-driven path. */
int fq_sample_step(const float* logits, int64_t ld, const double* lse, const int32_t* cand_idx,
                   int64_t cand_ld, const int64_t* cand_count, int64_t batch, int64_t k,
                   double top_p, int64_t groups, int64_t vocab, int64_t eos,
                   const double* uniforms, int64_t n_uniforms, int64_t* draw, int32_t* done,
                   int32_t* d_cur, int64_t max_steps, int64_t max_len, int32_t* dk_next,
                   int64_t* tokens, int32_t* out_tok, int32_t* out_len, int32_t* fin,
                   int32_t* counters, int32_t* err, fq_stream_t stream);

/* ---- fused attention for the device engine (model.py:329-336, :572-604) --- */

/* Encoder self-attention, one pass per (item, head): q,k,v read from the packed
 * [n, 3d] projection (bias already added), softmax(qk^T*scale + mask) with the
 * kernels.py:106 numerics (exact mode: f64 exp/sum), ctx written merged-head
 * [n, d] (ldo) as fp32 (out) and/or fp16 (out16). mask [batch, seq] or NULL.
 * d_bad counts fully masked rows. exact: 1 = f64 softmax internals. */
int fq_encoder_attention(const float* qkv, int64_t ldq, int64_t batch, int64_t seq,
                         int64_t heads, int64_t head_dim, float scale, const float* mask,
                         float* out, void* out16, int64_t ldo, int exact, int* d_bad,
                         fq_stream_t stream);

/* Decoder incremental self-attention with copy-free beam reorder: row r at
 * step cur attends positions t < cur through cache slot (t, hist[r, t]) and
 * position cur through its own new K/V (taken from the packed sqkv [R, 3d]
 * projection, bias added), which this call also stores into slot (cur, r).
 * Cache layout [max_len, R, d] (kv_dtype fp32 or fp16). */
int fq_decoder_self_attention(const float* sqkv, int64_t ldq, void* kcache, void* vcache,
                              int kv_dtype, const int32_t* hist, const int32_t* d_cur,
                              int64_t rows, int64_t heads, int64_t head_dim, int64_t max_len,
                              float scale, float* out, void* out16, int64_t ldo, int exact,
                              fq_stream_t stream);

/* Cross-attention: the K beam rows of item b attend to that item's encoder
 * memory K/V (not replicated per beam, model.py:594-604). ck/cv rows are
 * [batch*seq] with leading dim ldkv (bias added). mask [batch, seq] or NULL. */
int fq_cross_attention(const float* cq, int64_t ldcq, const void* ck, const void* cv,
                       int kv_dtype, int64_t ldkv, int64_t batch, int64_t beam, int64_t seq,
                       int64_t heads, int64_t head_dim, float scale, const float* mask,
                       float* out, void* out16, int64_t ldo, int exact, int* d_bad,
                       fq_stream_t stream);

/* fq_cross_attention (fp16 K/V, head_dim 64, seq <= 64, beam <= 8) whose
 * query is given as the nslab K-slice slabs of the split-K query GEMM
 * (fq_gemm_splitk_slabs; slab s at q_slabs + s * batch*beam*ldq) plus q_bias:
 * q = ((slab0 + slab1) + ...) + bias, the GEMM's own epilogue order. */
int fq_cross_attention_slabs(const float* q_slabs, int nslab, int64_t ldq, const float* q_bias,
                             const void* ck, const void* cv, int64_t ldkv, int64_t batch,
                             int64_t beam, int64_t seq, int64_t heads, int64_t head_dim,
                             float scale, const float* mask, float* out, void* out16, int64_t ldo,
                             int* d_bad, fq_stream_t stream);

/* ---- weight preparation (cast once at load) -------------- */

/* Exact mode's output layer (SURVEY §8(f)1 for fp32): the 3xFP16 logits GEMM
 * whose epilogue emits the HARS stage-1 statistics per (row, 128-column tile)
 * for fq_hars_merge_step (ldt = ntiles = vocab / 128) — group maxima, tile max,
 * f64 sum of exp, survivors x >= a bound <= R; the [rows, V] logits are never
 * written. x / emb: fp16 pairs (fq_gemm_x3h operands); vocab % 128 == 0. */
int fq_logits_hars_x3h(const void* x, const void* x_lo, int64_t ldx, const void* emb,
                       const void* emb_lo, int64_t lde, int64_t rows, int64_t vocab, int64_t d,
                       const int32_t* dk, int32_t* gmax, float* tmax, double* tsum, int64_t ldt,
                       int32_t* sv_cnt, void* sv, int64_t sv_cap, fq_stream_t stream);

/* Exact fp32 mode attention on warp MMAs (3xFP16: every fp32 operand as its
 * fp16 pair, three MMAs per product; the reference's exact f64 softmax in
 * between), replacing model.py:565-578 (decoder self-attention over the
 * KVCache) and :594-604 (cross-attention). Self-attention cache: fp16 pair
 * planes, hi at kcache / vcache and lo at + plane elements, each [max_len,
 * rows, d]; this step's K/V are split and written to slot (cur, r). Cross K/V:
 * pair planes of the [batch*seq, ldkv] cross-K/V buffer. ctx goes to out
 * (fp32) and/or its pair (out_hi, out_lo) for the next exact-mode GEMM. */
int fq_decoder_self_attention_xh(const float* sqkv, int64_t ldq, void* kcache, void* vcache,
                                 int64_t plane, const int32_t* hist, const int32_t* d_cur,
                                 int64_t rows, int64_t heads, int64_t head_dim, int64_t max_len,
                                 float scale, float* out, void* out_hi, void* out_lo,
                                 int64_t ldo, fq_stream_t stream);
/* The same decoder self-attention, one warp per (item, head) with the beams
 * (rows item*beam .. item*beam + beam-1, beam <= 8, head_dim 64) as the MMA's
 * query columns: each distinct history slot the item's beams share (via hist)
 * is read once. Scores and probabilities equal fq_decoder_self_attention_xh's
 * bit for bit; the context may differ in the last fp32 bit (the P.V terms are
 * grouped by shared slot, not by position). Opt-in in the engine
 * (FQ_SELF_ITEMS=1): fewer bytes, but slower at C2 than the per-row kernel. */
int fq_decoder_self_attention_xh_items(const float* sqkv, int64_t ldq, void* kcache,
                                       void* vcache, int64_t plane, const int32_t* hist,
                                       const int32_t* d_cur, int64_t items, int64_t beam,
                                       int64_t heads, int64_t head_dim, int64_t max_len,
                                       float scale, float* out, void* out_hi, void* out_lo,
                                       int64_t ldo, fq_stream_t stream);
/* Exact-mode encoder self-attention on 3xFP16 warp MMAs (head_dim 64, seq <=
 * 64; model.py:329-336, kernels.py:106-139 softmax): ctx written as the
 * out-projection GEMM's fp16 pair (out_hi, out_lo) and optionally fp32 `out`. */
int fq_encoder_attention_xh(const float* qkv, int64_t ldq, int64_t batch, int64_t seq,
                            int64_t heads, int64_t head_dim, float scale, const float* mask,
                            float* out, void* out_hi, void* out_lo, int64_t ldo, int* d_bad,
                            fq_stream_t stream);
/* fq_cross_attention_xh with the query as the nslab split-K slabs of its GEMM
 * (fq_gemm_x3h_slabs: q_slabs + s * slab_stride, row stride ldq) summed in
 * slab order, + q_bias -- the DSMEM epilogue's additions, so the same bits. */
int fq_cross_attention_xh_slabs(const float* q_slabs, int64_t nslab, int64_t ldq,
                                int64_t slab_stride, const float* q_bias, const void* ck,
                                const void* cv, int64_t plane, int64_t ldkv, int64_t batch,
                                int64_t beam, int64_t seq, int64_t heads, int64_t head_dim,
                                float scale, const float* mask, float* out, void* out_hi,
                                void* out_lo, int64_t ldo, int* d_bad, fq_stream_t stream);
int fq_cross_attention_xh(const float* cq, int64_t ldcq, const void* ck, const void* cv,
                          int64_t plane, int64_t ldkv, int64_t batch, int64_t beam, int64_t seq,
                          int64_t heads, int64_t head_dim, float scale, const float* mask,
                          float* out, void* out_hi, void* out_lo, int64_t ldo, int* d_bad,
                          fq_stream_t stream);

/* dst16[N, K] (fp16, row-major) = src[K, N]^T (fp32) when transpose, else cast. */
int fq_cast_f16(const float* src, int64_t rows, int64_t cols, int transpose, void* dst16,
                 fq_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FQ_ABI_H */
