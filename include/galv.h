/*
 * galv.h -- C ABI of the B200 (sm_100a) kernel library behind the hybrid-parallel
 * runtime (paper_2504_21411_b200/csrc, built into libgalv_b200.so).
 *
 * The reference planner (/root/reference/pkg/src/hybridplan) stops at the Plan
 * boundary: its "runtime" is the simulator pipesim.py and the paper's
 * get_hybrid_parallel_configs / construct_hybrid_parallel_model (PAPER.md:82,
 * SPEC.md:10) have no reference code.  Each entry point below realizes one term
 * of the reference cost model (costmodel.py:90-213); the comment on each names it.
 *
 * Conventions
 *   - status: 0 ok; < 0 invalid argument; > 0 CUDA error code.  galv_last_error()
 *     returns a thread-local message for the last failure on the calling thread.
 *   - all pointers are device pointers owned by the caller (PyTorch caching
 *     allocator); kernels never allocate.  Row-major, strides in elements.
 *   - dtype: GALV_F32 = 0, GALV_BF16 = 1.
 *   - every call is asynchronous on `stream` (a cudaStream_t passed as void*);
 *     no host synchronization, callable from any host thread.
 */
#ifndef GALV_H_
#define GALV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GALV_ABI_VERSION 1
#define GALV_F32 0
#define GALV_BF16 1

int32_t galv_abi_version(void);
const char* galv_last_error(void);
/* number of SMs / sm major.minor of the current device (for host-side heuristics) */
int32_t galv_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/*
 * C[M,N] = alpha * op(A) @ op(B) (+ bias[N]) (+ C if accumulate)
 * op(A) is [M,K]: A stored [M,K] (trans_a = 0, lda >= K) or [K,M] (trans_a = 1, lda >= M).
 * op(B) is [K,N]: B stored [N,K] (trans_b = 1, the nn.Linear weight layout) or [K,N]
 * (trans_b = 0).  bf16 inputs run on tcgen05 (TMA -> smem -> UMMA -> TMEM), fp32
 * inputs on the exact SIMT FP32 path.  c_dtype may differ from ab_dtype (fp32
 * accumulation buffers for bf16 GEMMs).  Realizes fwd_compute / bwd_compute
 * (costmodel.py:104-106): column/row-parallel forward, dgrad and wgrad.
 */
int32_t galv_gemm(const void* A, const void* B, void* C, const void* bias,
                  int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                  int32_t trans_a, int32_t trans_b, float alpha, int32_t accumulate,
                  int32_t ab_dtype, int32_t c_dtype, int32_t bias_dtype, void* stream);

/*
 * Split-K variant of galv_gemm for bf16 operands (same op semantics): the K loop is cut into
 * `splits` ranges computed as separate 2-CTA work units, fp32 partial tiles land in `ws`
 * (>= splits*M*N*4 bytes, caller-owned), and one reduction pass applies alpha/bias/accumulate.
 * galv_gemm_splits(M, N, K) returns the split count the cost heuristic picks (1 = none);
 * it is > 1 only for GEMMs whose tiles cannot fill the chip (narrow-layer wgrad).
 */
int32_t galv_gemm_splits(int64_t M, int64_t N, int64_t K);
/* Workspace queries (the caller owns all memory): bytes the matching call needs in `ws`. */
int64_t galv_gemm_splitk_workspace(int64_t M, int64_t N, int64_t K);
int64_t galv_colsum_workspace(int64_t rows, int64_t cols, int32_t dtype);
int32_t galv_gemm_splitk(const void* A, const void* B, void* C, const void* bias, int64_t M,
                         int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                         int32_t trans_a, int32_t trans_b, float alpha, int32_t accumulate,
                         int32_t c_dtype, int32_t bias_dtype, int32_t splits, void* ws,
                         int64_t ws_bytes, void* stream);

/*
 * Batched strided GEMM (same op semantics), `batch` problems at element offsets
 * stride_a/b/c.  Used by the small-head attention path and tests.
 */
int32_t galv_gemm_batched(const void* A, const void* B, void* C, int64_t batch,
                          int64_t stride_a, int64_t stride_b, int64_t stride_c,
                          int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
                          int64_t ldc, int32_t trans_a, int32_t trans_b, float alpha,
                          int32_t accumulate, int32_t ab_dtype, int32_t c_dtype, void* stream);

/*
 * Causal/non-causal attention over q,k,v laid out [B, S, H, D] (token-major, the
 * layout the QKV GEMM produces; strides given in elements for token and head).
 * o: [B, S, H, D]; lse: fp32 [B, H, S] (natural-log logsumexp of scaled scores).
 * Realizes the flops_per_token_sq term (costmodel.py:104; flash assumption,
 * profiles.py:207-208: no S^2 memory).
 */
int32_t galv_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                      int64_t B, int64_t S, int64_t H, int64_t D,
                      int64_t stride_tok, int64_t stride_head, int64_t o_stride_tok,
                      float scale, int32_t causal, int32_t dtype, void* stream);
/* dq/dk/dv same layout as q/k/v; ws: fp32 workspace of galv_attn_bwd_workspace bytes. */
int64_t galv_attn_bwd_workspace(int64_t B, int64_t S, int64_t H, int64_t D, int32_t dtype);
int32_t galv_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                      const void* dout, const float* lse, void* dq, void* dk, void* dv,
                      int64_t B, int64_t S, int64_t H, int64_t D, int64_t stride_tok,
                      int64_t stride_head, int64_t o_stride_tok, float scale, int32_t causal,
                      int32_t dtype, void* ws, void* stream);
/* galv_attn_bwd with dq/dk returned through the inverse rotate-half RoPE of q/k (bf16,
 * head_dim 128); rope_table = fp32 [2][S][D/2] cos|sin planes (the galv_rope_table layout).
 * epilogue 1: rotate in the dq/dk store epilogues; 0: backward + streaming inverse-RoPE
 * pass; <0: library default (0, measured faster).  Replaces galv_attn_bwd +
 * galv_rope_table(inverse=1) on dq|dk in the decoder backward (costmodel.py:104). */
int32_t galv_attn_bwd_rope(const void* q, const void* k, const void* v, const void* o,
                           const void* dout, const float* lse, void* dq, void* dk, void* dv,
                           int64_t B, int64_t S, int64_t H, int64_t D, int64_t stride_tok,
                           int64_t stride_head, int64_t o_stride_tok, float scale,
                           int32_t causal, const float* rope_table, int32_t epilogue,
                           int32_t dtype, void* ws, void* stream);
/* Softmax-dropout variants (SURVEY.md §8(b) attn_fwd / attn_bwd with p, seed, offset;
 * north_star (1) softmax-dropout).  Attention probabilities are dropped with probability
 * dropout_p and the kept ones scaled by 1/(1-p); the keep mask is Philox4x32-10 of
 * (counter = (key/4, query, (b0+b)*H_total + h0+h, offset), key = seed) -- csrc/dropout.cuh,
 * regenerated identically by the forward and both backward kernels (nothing stored).
 * b0 / h0 / H_total place this call's local (b, h) in the global batch / head grid, so the
 * mask does not depend on how dp / tp / Ulysses shard the call.  dropout_p = 0: exactly
 * galv_attn_fwd / galv_attn_bwd(_rope).  rope_table NULL: no inverse RoPE. */
int32_t galv_attn_fwd_dropout(const void* q, const void* k, const void* v, void* o, float* lse,
                              int64_t B, int64_t S, int64_t H, int64_t D, int64_t stride_tok,
                              int64_t stride_head, int64_t o_stride_tok, float scale,
                              int32_t causal, float dropout_p, uint64_t seed, uint64_t offset,
                              int64_t b0, int64_t h0, int64_t H_total, int32_t dtype,
                              void* stream);
int32_t galv_attn_bwd_dropout(const void* q, const void* k, const void* v, const void* o,
                              const void* dout, const float* lse, void* dq, void* dk, void* dv,
                              int64_t B, int64_t S, int64_t H, int64_t D, int64_t stride_tok,
                              int64_t stride_head, int64_t o_stride_tok, float scale,
                              int32_t causal, float dropout_p, uint64_t seed, uint64_t offset,
                              int64_t b0, int64_t h0, int64_t H_total, const float* rope_table,
                              int32_t epilogue, int32_t dtype, void* ws, void* stream);
/* The keep mask itself, uint8 [B][H][S][S] (tests: cross-checked against the CPU Philox). */
int32_t galv_dropout_mask(uint8_t* mask, int64_t B, int64_t S, int64_t H, float dropout_p,
                          uint64_t seed, uint64_t offset, int64_t b0, int64_t h0,
                          int64_t H_total, void* stream);

/* y = norm(x (+ residual)) * gamma (+ beta).  rows x cols; residual/res_out optional:
 * when residual != NULL, res_out = x + residual is written and normalized.
 * rstd/mean: fp32 [rows] saved for backward (mean unused for RMSNorm). */
int32_t galv_rmsnorm_fwd(const void* x, const void* residual, void* res_out,
                         const void* gamma, void* y, float* rstd, int64_t rows, int64_t cols,
                         float eps, int32_t dtype, void* stream);
/* dx = d(norm)/dx^T dy (+ dres_in if not NULL); dgamma accumulated into fp32 dgamma_acc. */
int32_t galv_rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy,
                         const void* dres_in, void* dx, float* dgamma_acc, int64_t rows,
                         int64_t cols, int32_t dtype, void* ws, void* stream);
int32_t galv_layernorm_fwd(const void* x, const void* residual, void* res_out,
                           const void* gamma, const void* beta, void* y, float* mean,
                           float* rstd, int64_t rows, int64_t cols, float eps, int32_t dtype,
                           void* stream);
int32_t galv_layernorm_bwd(const void* x, const void* gamma, const float* mean,
                           const float* rstd, const void* dy, const void* dres_in, void* dx,
                           float* dgamma_acc, float* dbeta_acc, int64_t rows, int64_t cols,
                           int32_t dtype, void* ws, void* stream);
int64_t galv_norm_bwd_workspace(int64_t rows, int64_t cols);

/* Rotary embedding in place on x [T, H, D] (rows of stride_tok), positions pos0 + t % S.
 * inverse = 1 applies the transpose rotation (backward). theta base e.g. 10000. */
int32_t galv_rope(void* x, int64_t T, int64_t S, int64_t H, int64_t D, int64_t stride_tok,
                  int64_t stride_head, int64_t pos0, float theta, int32_t inverse,
                  int32_t dtype, void* stream);

/* Same rotation from a precomputed fp32 table [2][S][D/2] (cos plane, then sin plane). */
int32_t galv_rope_table(void* x, const float* table, int64_t T, int64_t S, int64_t H, int64_t D,
                        int64_t stride_tok, int64_t stride_head, int64_t pos0, int32_t inverse,
                        int32_t dtype, void* stream);

/* SwiGLU on a fused [T, 2F] gate|up tensor -> h [T, F]; backward -> d(gate|up). */
int32_t galv_swiglu_fwd(const void* gu, void* h, int64_t T, int64_t F, int32_t dtype,
                        void* stream);
int32_t galv_swiglu_bwd(const void* gu, const void* dh, void* dgu, int64_t T, int64_t F,
                        int32_t dtype, void* stream);
/* bf16 SwiGLU backward with dh rows ld_dh elements apart (dh may alias dgu's up half). */
int32_t galv_swiglu_bwd_strided(const void* gu, const void* dh, int64_t ld_dh, void* dgu,
                                int64_t T, int64_t F, void* stream);
/*
 * Llama MLP GEMMs with the SwiGLU fused into the tcgen05 epilogue (bf16):
 *   fwd: gu[M,2F] = X[M,K] W_gu[2F,K]^T (rows gate then up), h[M,F] = silu(gate) * up;
 *        each CTA pair accumulates 128 gate + the matching 128 up columns, so the
 *        activation is computed from TMEM and h is written by the same epilogue.
 *   bwd: dgu[M,2F] = swiglu_bwd(gu, dh) with dh = dY[M,K] W_down[K,F] (nn.Linear layout
 *        of the down projection) kept in TMEM -- dh never reaches HBM.
 * Same values as galv_gemm + galv_swiglu_fwd/bwd (gate/up/dh rounded to bf16 first);
 * shapes the 2-CTA path cannot take run exactly that unfused sequence.
 * Realizes fwd_compute/bwd_compute of the MLP (costmodel.py:104-106).
 */
int32_t galv_gemm_swiglu_fwd(const void* X, const void* Wgu, void* gu, void* h, int64_t M,
                             int64_t F, int64_t K, int64_t ldx, int64_t ldw, int64_t ld_gu,
                             int64_t ld_h, void* stream);
int32_t galv_gemm_swiglu_bwd(const void* dY, const void* Wdown, const void* gu, void* dgu,
                             int64_t M, int64_t F, int64_t K, int64_t ldy, int64_t ldw,
                             int64_t ld_gu, int64_t ld_dgu, void* stream);
/* GeLU(tanh) with bias: y = gelu(x + b); backward dx = dy * gelu'(x + b). */
int32_t galv_bias_gelu_fwd(const void* x, const void* bias, void* y, int64_t T, int64_t F,
                           int32_t dtype, void* stream);
int32_t galv_bias_gelu_bwd(const void* x, const void* bias, const void* dy, void* dx,
                           int64_t T, int64_t F, int32_t dtype, void* stream);
/* Llama QKV projection with RoPE in the tcgen05 epilogue (bf16):
 *   qkv[M,N] = X[M,K] Wqkv[N,K]^T, then rotate-half RoPE on columns [0, n_rot) as heads
 *   of 128 (q | k), position = row % S, cos/sin from table [2][S][64] fp32 -- the same
 *   arithmetic as galv_gemm followed by galv_rope_table on the stored bf16 values.
 * n_rot, N multiples of 128.  Falls back to exactly that pair when the fused path does not
 * apply (M <= 128, unaligned operands, S % 8 != 0, GALV_ROPE_UNFUSED=1).
 * Realizes K1 + K6 inside fwd_compute (costmodel.py:104-105). */
int32_t galv_gemm_rope_qkv(const void* X, const void* Wqkv, void* qkv, const float* table,
                           int64_t M, int64_t N, int64_t K, int64_t ldx, int64_t ldw,
                           int64_t ldc, int64_t n_rot, int64_t S, void* stream);
/* bias-GeLU backward with the bias gradient fused: dx as galv_bias_gelu_bwd and
 * dbias_acc[f] += sum_t dx[t, f] (fp32; equals galv_colsum(dx, accumulate=1)).
 * x, dy, dx 16-byte aligned, F * element size a multiple of 16 B (bias: any alignment).
 * Realizes K8 inside the bwd_compute term (costmodel.py:106). */
int32_t galv_bias_gelu_bwd_colsum(const void* x, const void* bias, const void* dy, void* dx,
                                  float* dbias_acc, int64_t T, int64_t F, int32_t dtype,
                                  void* stream);
/*
 * GPT MLP GEMMs with the bias-GeLU(tanh) fused into the tcgen05 epilogue (bf16):
 *   fwd: pre[M,F] = X[M,K] W1[F,K]^T, act[M,F] = gelu(pre + bias)   (fc1)
 *   bwd: dpre[M,F] = (dY[M,K] W2[K,F]) * gelu'(pre + bias)          (fc2 dgrad)
 * GeLU/tanh on MUFU (tanh.approx); same roundings as galv_gemm + galv_bias_gelu_*
 * otherwise.  bias may be null; bias_dtype GALV_BF16 or GALV_F32.
 */
int32_t galv_gemm_bias_gelu_fwd(const void* X, const void* W1, const void* bias, void* pre,
                                void* act, int64_t M, int64_t F, int64_t K, int64_t ldx,
                                int64_t ldw, int64_t ld_pre, int64_t ld_act, int32_t bias_dtype,
                                void* stream);
int32_t galv_gemm_bias_gelu_bwd(const void* dY, const void* W2, const void* pre,
                                const void* bias, void* dpre, int64_t M, int64_t F, int64_t K,
                                int64_t ldy, int64_t ldw, int64_t ld_pre, int64_t ld_dpre,
                                int32_t bias_dtype, void* stream);
/* x[T, F] += bias[F] (row broadcast) */
int32_t galv_bias_add(void* x, const void* bias, int64_t T, int64_t F, int32_t dtype, void* stream);
/* column sums: out[c] (+)= sum_r x[r, c] (fp32 out, for bias gradients) */
int32_t galv_colsum(const void* x, float* out, int64_t rows, int64_t cols, int32_t accumulate,
                    int32_t dtype, void* ws, void* stream);

/* Embedding gather/scatter-add over a vocab shard [vocab_lo, vocab_lo + V_local). */
int32_t galv_embed_fwd(const int64_t* ids, const void* table, void* out, int64_t T,
                       int64_t V_local, int64_t vocab_lo, int64_t Hd, int32_t dtype,
                       void* stream);
int32_t galv_embed_bwd(const int64_t* ids, const void* dout, float* dtable_acc, int64_t T,
                       int64_t V_local, int64_t vocab_lo, int64_t Hd, int32_t dtype,
                       void* stream);
/* Deterministic embedding backward: ids sorted (stable) with their token order; grad rows
 * of this vocab shard += the fp32 sum of their dout rows, stored in grad_dtype (bf16/f32).
 * Replaces the fp32 scatter table + atomics of galv_embed_bwd on the training path. */
int32_t galv_embed_bwd_sorted(const int64_t* sorted_ids, const int64_t* order,
                              const void* dout, void* grad, int64_t T, int64_t V_local,
                              int64_t vocab_lo, int64_t Hd, int32_t dtype, int32_t grad_dtype,
                              void* stream);

/* Vocab-parallel cross entropy over a logits shard [T, V_local].
 *  stage 0: row max -> stats[T*3+0] ; (caller all-reduces MAX over tp)
 *  stage 1: sum exp(x - max) -> stats[1], target logit -> stats[2] ; (caller all-reduces SUM)
 *  stage 2: loss[T] = log(sum) + max - target; dlogits = (softmax - onehot) * grad_scale
 *  (in place over logits when dlogits == logits). ignore_index rows give 0. */
int32_t galv_xent(void* logits, const int64_t* labels, float* stats, float* loss,
                  void* dlogits, int64_t T, int64_t V_local, int64_t vocab_lo,
                  float grad_scale, int64_t ignore_index, int32_t stage, int32_t dtype,
                  void* stream);

/* Fused AdamW over flat fp32 master/m/v shards; grad in `grad_dtype` scaled by
 * grad_scale; writes the updated param copy (bf16 or fp32) to param_out (may be NULL). */
int32_t galv_adamw(float* master, float* m, float* v, const void* grad, void* param_out,
                   int64_t n, float lr, float beta1, float beta2, float eps,
                   float weight_decay, float grad_scale, int64_t step, int32_t grad_dtype,
                   int32_t param_dtype, void* stream);

/* Reshard pack/unpack: dst[i] = src[idx[i]] row gather (rows of `row_bytes`). */
int32_t galv_gather_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows,
                         int64_t row_bytes, void* stream);
/* dst[idx[i]] = src[i] row scatter. */
int32_t galv_scatter_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows,
                          int64_t row_bytes, void* stream);

/* Elementwise helpers: y = a*x + b*y (axpby, any of f32/bf16 in/out), cast, fill. */
int32_t galv_axpby(const void* x, void* y, int64_t n, float a, float b, int32_t x_dtype,
                   int32_t y_dtype, void* stream);
int32_t galv_sumsq(const void* x, int64_t n, float* out, int32_t dtype, void* stream);

/* ---- NVLink / NVSwitch collectives over symmetric (peer-mapped) buffers ----------------
 * Replace the NCCL collectives the cost model charges (collectives.py:49-69 ring passes;
 * costmodel.py:110-118 TP all-reduce, :199-213 dp_sync).  Flag arrays hold one uint32 per
 * source rank; epochs increase monotonically per (buffer, stream).  `*_ptrs` arguments are
 * DEVICE arrays of per-rank base addresses (rank order of the group). */

/* Row-parallel GEMM C = op(A) op(B) whose epilogue stores output rows r into
 * peer_c[r / rows_per_rank] at row slot my_slot (Megatron-SP reduce-scatter fused into the
 * GEMM; bf16 only). */
int32_t galv_gemm_rs(const void* A, const void* B, void* const* peer_c, int64_t rows_per_rank,
                     int32_t my_slot, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
                     int64_t ldc, int32_t trans_a, int32_t trans_b, void* stream);
/* Signal + wait (one CTA), then out[n] = sum_s recv[s*n + i] over the t slots. */
int32_t galv_tp_signal_reduce(void* const* flag_ptrs, int32_t me, int32_t t, uint32_t epoch,
                              const void* recv, void* out, int64_t n, int32_t dtype,
                              void* stream);
/* Store `bytes` of src into slot `me` of every rank's dst buffer, then signal + wait. */
int32_t galv_tp_allgather(const void* src, void* const* dst_ptrs, void* const* flag_ptrs,
                          int32_t me, int32_t t, uint32_t epoch, int64_t bytes, void* stream);
/* Raise flag[me] = epoch in every rank's flag array (release, system scope). */
int32_t galv_nvl_signal(void* const* flag_ptrs, int32_t me, int32_t t, uint32_t epoch,
                        void* stream);
/* One CTA spins until my_flags[0..t) >= epoch (acquire, system scope). */
int32_t galv_nvl_wait(const uint32_t* my_flags, int32_t t, uint32_t epoch, void* stream);
/* dp reduce over bf16 chunks [offset, offset+n): sum over ranks read from the multicast
 * address mc_src (NVSwitch multimem.ld_reduce, fp32 accumulate) or, if mc_src is NULL, from
 * peer_src[r] + offset; out = sum (+ out if accumulate); the result is also stored to every
 * rank at mc_dst (multimem.st) or peer_dst[r] + offset when given (all-reduce).
 * max_ctas > 0 caps the grid (leave SMs to the concurrent GEMMs). */
int32_t galv_dp_reduce(const void* mc_src, void* const* peer_src, int32_t t, int64_t offset,
                       void* out, int32_t accumulate, void* mc_dst, void* const* peer_dst,
                       int64_t n, int32_t max_ctas, void* stream);
/* AdamW (as galv_adamw) on this rank's fp32 shard of n params whose bf16 result is stored to
 * every dp rank's full parameter buffer: multicast address mc_dst, or peer_dst[r] + offset
 * (ZeRO-1/2 parameter all-gather fused into the optimizer; n, offset multiples of 8). */
int32_t galv_adamw_bcast(float* master, float* m, float* v, const void* grad, void* mc_dst,
                         void* const* peer_dst, int32_t t, int64_t offset, int64_t n, float lr,
                         float beta1, float beta2, float eps, float weight_decay,
                         float grad_scale, int64_t step, int32_t grad_dtype, void* stream);

/* ---- NCCL communicators (opaque ncclComm_t as void*), collectives.py:49-89 ring passes --
 * libnccl.so.2 is dlopen'ed on first use (no link-time dependency).  dtype 0 = f32, 1 = bf16;
 * counts in elements; the ncclResult_t is returned on failure. */
int32_t galv_comm_unique_id(void* out /* 128 bytes */);
int32_t galv_comm_init(const void* unique_id, int32_t nranks, int32_t rank, void** comm);
int32_t galv_comm_split(void* comm, int32_t color, int32_t key, void** out);
int32_t galv_comm_destroy(void* comm);
int32_t galv_all_reduce(void* comm, const void* send, void* recv, int64_t count, int32_t dtype,
                        void* stream);
int32_t galv_reduce_scatter(void* comm, const void* send, void* recv, int64_t recv_count,
                            int32_t dtype, void* stream);
int32_t galv_all_gather(void* comm, const void* send, void* recv, int64_t send_count,
                        int32_t dtype, void* stream);
/* one grouped send + recv of raw bytes (pipeline-stage boundary exchange) */
int32_t galv_sendrecv(void* comm, const void* send, int64_t send_bytes, int32_t peer_send,
                      void* recv, int64_t recv_bytes, int32_t peer_recv, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GALV_H_ */
