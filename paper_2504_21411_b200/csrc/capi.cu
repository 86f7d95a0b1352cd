// C ABI entry points (include/galv.h): argument validation, dtype dispatch, error state.
#include <mutex>
#include <string>

#include "common.cuh"

namespace galv {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

int sm_count() {
  static int count = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    if (count <= 0) count = 148;
  });
  return count;
}

int32_t gemm_bf16_sm100(const void* A, const void* B, void* C, const void* bias, int64_t M,
                        int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                        int32_t trans_a, int32_t trans_b, float alpha, int32_t accumulate,
                        int32_t c_dtype, int32_t bias_dtype, cudaStream_t stream,
                        void* const* peer_c = nullptr, int64_t rows_per_rank = 0,
                        int32_t my_slot = 0, int32_t epi = 0, const void* aux = nullptr,
                        int64_t aux_ld = 0, int64_t ff = 0, int32_t splits = 1,
                        float* ws = nullptr);
int32_t gemm_pick_splits(int64_t M, int64_t N, int64_t K);
bool epilogue_fusable(const void* A, const void* B, const void* C, const void* aux, int64_t M,
                    int64_t ldc, int64_t aux_ld, int64_t ff, int32_t trans_b, int32_t epi);
int32_t gemm_f32_simt(const float* A, const float* B, void* C, const float* bias, int64_t batch,
                      int64_t sa, int64_t sb, int64_t sc, int64_t M, int64_t N, int64_t K,
                      int64_t lda, int64_t ldb, int64_t ldc, int32_t ta, int32_t tb, float alpha,
                      int32_t accumulate, int32_t c_dtype, cudaStream_t stream);

}  // namespace galv

extern "C" {

int32_t galv_abi_version(void) { return GALV_ABI_VERSION; }

const char* galv_last_error(void) { return galv::g_last_error.c_str(); }

int32_t galv_device_info(int32_t* sm, int32_t* major, int32_t* minor) {
  int dev = 0;
  GALV_CUDA_RET(cudaGetDevice(&dev));
  int a = 0, b = 0, c = 0;
  GALV_CUDA_RET(cudaDeviceGetAttribute(&a, cudaDevAttrMultiProcessorCount, dev));
  GALV_CUDA_RET(cudaDeviceGetAttribute(&b, cudaDevAttrComputeCapabilityMajor, dev));
  GALV_CUDA_RET(cudaDeviceGetAttribute(&c, cudaDevAttrComputeCapabilityMinor, dev));
  if (sm) *sm = a;
  if (major) *major = b;
  if (minor) *minor = c;
  return 0;
}

int32_t galv_gemm(const void* A, const void* B, void* C, const void* bias, int64_t M, int64_t N,
                  int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int32_t trans_a,
                  int32_t trans_b, float alpha, int32_t accumulate, int32_t ab_dtype,
                  int32_t c_dtype, int32_t bias_dtype, void* stream) {
  GALV_CHECK_ARG(A && B && C, "null operand");
  GALV_CHECK_ARG(c_dtype == GALV_F32 || c_dtype == GALV_BF16, "bad c_dtype");
  if (ab_dtype == GALV_BF16)
    return galv::gemm_bf16_sm100(A, B, C, bias, M, N, K, lda, ldb, ldc, trans_a, trans_b, alpha,
                                 accumulate, c_dtype, bias_dtype, galv::as_stream(stream));
  GALV_CHECK_ARG(ab_dtype == GALV_F32, "bad ab_dtype");
  GALV_CHECK_ARG(bias == nullptr || bias_dtype == GALV_F32, "fp32 gemm needs fp32 bias");
  return galv::gemm_f32_simt((const float*)A, (const float*)B, C, (const float*)bias, 1, 0, 0, 0,
                             M, N, K, lda, ldb, ldc, trans_a, trans_b, alpha, accumulate, c_dtype,
                             galv::as_stream(stream));
}

int32_t galv_gemm_splits(int64_t M, int64_t N, int64_t K) {
  return M > 0 && N > 0 && K > 0 ? galv::gemm_pick_splits(M, N, K) : 1;
}

// Workspace queries (the caller owns all memory; kernels never allocate).
// split-K: splits * M * N fp32 partial tiles when galv_gemm_splits picks > 1, else 0.
int64_t galv_gemm_splitk_workspace(int64_t M, int64_t N, int64_t K) {
  const int64_t s = galv_gemm_splits(M, N, K);
  return s > 1 ? s * M * N * (int64_t)sizeof(float) : 0;
}
// The column-sum kernels need no scratch (their `ws` argument is reserved): 0 bytes.
// (galv_norm_bwd_workspace lives with the norm kernels, norm.cu.)
int64_t galv_colsum_workspace(int64_t rows, int64_t cols, int32_t dtype) {
  (void)rows;
  (void)cols;
  (void)dtype;
  return 0;
}

int32_t galv_gemm_splitk(const void* A, const void* B, void* C, const void* bias, int64_t M,
                         int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                         int32_t trans_a, int32_t trans_b, float alpha, int32_t accumulate,
                         int32_t c_dtype, int32_t bias_dtype, int32_t splits, void* ws,
                         int64_t ws_bytes, void* stream) {
  GALV_CHECK_ARG(A && B && C && splits >= 1, "bad arguments");
  GALV_CHECK_ARG(c_dtype == GALV_F32 || c_dtype == GALV_BF16, "bad c_dtype");
  GALV_CHECK_ARG(splits == 1 || (ws != nullptr && ws_bytes >= (int64_t)splits * M * N * 4 &&
                                 (reinterpret_cast<uintptr_t>(ws) & 15) == 0),
                 "split-K workspace must hold splits*M*N fp32 (16-byte aligned)");
  return galv::gemm_bf16_sm100(A, B, C, bias, M, N, K, lda, ldb, ldc, trans_a, trans_b, alpha,
                               accumulate, c_dtype, bias_dtype, galv::as_stream(stream), nullptr,
                               0, 0, 0, nullptr, 0, 0, splits, static_cast<float*>(ws));
}

int32_t galv_gemm_batched(const void* A, const void* B, void* C, int64_t batch, int64_t sa,
                          int64_t sb, int64_t sc, int64_t M, int64_t N, int64_t K, int64_t lda,
                          int64_t ldb, int64_t ldc, int32_t trans_a, int32_t trans_b,
                          float alpha, int32_t accumulate, int32_t ab_dtype, int32_t c_dtype,
                          void* stream) {
  GALV_CHECK_ARG(A && B && C && batch > 0, "bad arguments");
  if (ab_dtype == GALV_F32)
    return galv::gemm_f32_simt((const float*)A, (const float*)B, C, nullptr, batch, sa, sb, sc,
                               M, N, K, lda, ldb, ldc, trans_a, trans_b, alpha, accumulate,
                               c_dtype, galv::as_stream(stream));
  GALV_CHECK_ARG(ab_dtype == GALV_BF16, "bad ab_dtype");
  const size_t esz_c = c_dtype == GALV_F32 ? 4 : 2;
  for (int64_t b = 0; b < batch; ++b) {
    int32_t rc = galv::gemm_bf16_sm100((const char*)A + 2 * sa * b, (const char*)B + 2 * sb * b,
                                       (char*)C + esz_c * sc * b, nullptr, M, N, K, lda, ldb,
                                       ldc, trans_a, trans_b, alpha, accumulate, c_dtype,
                                       GALV_F32, galv::as_stream(stream));
    if (rc) return rc;
  }
  return 0;
}

// GALV_ROPE_UNFUSED=1 runs the QKV GEMM and the standalone RoPE kernel (A/B).
static bool rope_unfused() {
  static const bool off = [] {
    const char* e = getenv("GALV_ROPE_UNFUSED");
    return e && e[0] == '1';
  }();
  return off;
}

// qkv = X Wqkv^T (Wqkv [N, K], nn.Linear layout; rows q heads | k heads | v heads of 128)
// with RoPE (rotate-half, table [2][S][64] fp32 as kernels.rope_table builds it) applied to
// the first n_rot columns in the GEMM epilogue; otherwise the GEMM then galv_rope_table.
int32_t galv_gemm_rope_qkv(const void* X, const void* Wqkv, void* qkv, const float* table,
                           int64_t M, int64_t N, int64_t K, int64_t ldx, int64_t ldw,
                           int64_t ldc, int64_t n_rot, int64_t S, void* stream) {
  GALV_CHECK_ARG(X && Wqkv && qkv && table && M > 0 && N > 0 && K > 0 && S > 0,
                 "bad arguments");
  GALV_CHECK_ARG(n_rot % 128 == 0 && n_rot <= N && N % 128 == 0,
                 "q|k|v must be whole heads of 128 columns");
  if (!rope_unfused() && S % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(table) & 15) == 0 &&
      galv::epilogue_fusable(X, Wqkv, qkv, table, M, ldc, S, n_rot > 0 ? n_rot : 8, 1, 5))
    return galv::gemm_bf16_sm100(X, Wqkv, qkv, nullptr, M, N, K, ldx, ldw, ldc, 0, 1, 1.0f, 0,
                                 GALV_BF16, GALV_F32, galv::as_stream(stream), nullptr, 0, 0, 5,
                                 table, S, n_rot);
  int32_t rc = galv::gemm_bf16_sm100(X, Wqkv, qkv, nullptr, M, N, K, ldx, ldw, ldc, 0, 1, 1.0f,
                                     0, GALV_BF16, GALV_F32, galv::as_stream(stream));
  if (rc || n_rot == 0) return rc;
  return galv_rope_table(qkv, table, M, S, n_rot / 128, 128, ldc, 128, 0, 0, GALV_BF16, stream);
}

// gate|up = X W_gu^T (W_gu [2F, K], rows gate then up) and h = silu(gate) * up, with the
// SwiGLU in the GEMM epilogue (each CTA pair computes 128 gate and the matching 128 up
// columns); other shapes run the GEMM and then the standalone SwiGLU kernel.
int32_t galv_gemm_swiglu_fwd(const void* X, const void* Wgu, void* gu, void* h, int64_t M,
                             int64_t F, int64_t K, int64_t ldx, int64_t ldw, int64_t ld_gu,
                             int64_t ld_h, void* stream) {
  GALV_CHECK_ARG(X && Wgu && gu && h && M > 0 && F > 0 && K > 0 && F % 8 == 0, "bad arguments");
  GALV_CHECK_ARG(ld_gu == 2 * F && ld_h == F, "gate|up and h must be dense [M,2F] / [M,F]");
  if (galv::epilogue_fusable(X, Wgu, gu, h, M, ld_gu, ld_h, F, 1, 2))
    return galv::gemm_bf16_sm100(X, Wgu, gu, nullptr, M, 2 * F, K, ldx, ldw, ld_gu, 0, 1, 1.0f, 0,
                                 GALV_BF16, GALV_F32, galv::as_stream(stream), nullptr, 0, 0, 2, h,
                                 ld_h, F);
  int32_t rc = galv::gemm_bf16_sm100(X, Wgu, gu, nullptr, M, 2 * F, K, ldx, ldw, ld_gu, 0, 1, 1.0f,
                                     0, GALV_BF16, GALV_F32, galv::as_stream(stream));
  return rc ? rc : galv_swiglu_fwd(gu, h, M, F, GALV_BF16, stream);
}

// d(gate|up) [M, 2F] from dh = dY W_down (W_down [K=hidden, F], the nn.Linear layout of the
// down projection) and the saved gate|up, with the SwiGLU backward in the dgrad epilogue
// (dh never reaches HBM); the unfused fallback stages dh in the up half of dgu.
int32_t galv_gemm_swiglu_bwd(const void* dY, const void* Wdown, const void* gu, void* dgu,
                             int64_t M, int64_t F, int64_t K, int64_t ldy, int64_t ldw,
                             int64_t ld_gu, int64_t ld_dgu, void* stream) {
  GALV_CHECK_ARG(dY && Wdown && gu && dgu && M > 0 && F > 0 && K > 0 && F % 8 == 0,
                 "bad arguments");
  GALV_CHECK_ARG(ld_gu == 2 * F && ld_dgu == 2 * F, "gate|up tensors must be dense [M,2F]");
  if (galv::epilogue_fusable(dY, Wdown, dgu, gu, M, ld_dgu, ld_gu, F, 0, 1))
    return galv::gemm_bf16_sm100(dY, Wdown, dgu, nullptr, M, F, K, ldy, ldw, ld_dgu, 0, 0, 1.0f, 0,
                                 GALV_BF16, GALV_F32, galv::as_stream(stream), nullptr, 0, 0, 1, gu,
                                 ld_gu, F);
  char* up_half = static_cast<char*>(dgu) + 2 * F;  // dh staged where du will land
  int32_t rc = galv::gemm_bf16_sm100(dY, Wdown, up_half, nullptr, M, F, K, ldy, ldw, ld_dgu, 0, 0,
                                     1.0f, 0, GALV_BF16, GALV_F32, galv::as_stream(stream));
  return rc ? rc : galv_swiglu_bwd_strided(gu, up_half, ld_dgu, dgu, M, F, stream);
}

// GPT fc1: pre = X W1^T (W1 [F, K]) and act = gelu_tanh(pre + bias), the activation in the
// GEMM epilogue; unfused fallback = GEMM + galv_bias_gelu_fwd.
int32_t galv_gemm_bias_gelu_fwd(const void* X, const void* W1, const void* bias, void* pre,
                                void* act, int64_t M, int64_t F, int64_t K, int64_t ldx,
                                int64_t ldw, int64_t ld_pre, int64_t ld_act, int32_t bias_dtype,
                                void* stream) {
  GALV_CHECK_ARG(X && W1 && pre && act && M > 0 && F > 0 && K > 0 && F % 8 == 0,
                 "bad arguments");
  GALV_CHECK_ARG(bias_dtype == GALV_BF16 || bias_dtype == GALV_F32, "bad bias dtype");
  if (galv::epilogue_fusable(X, W1, pre, act, M, ld_pre, ld_act, F, 1, 3))
    return galv::gemm_bf16_sm100(X, W1, pre, bias, M, F, K, ldx, ldw, ld_pre, 0, 1, 1.0f, 0,
                                 GALV_BF16, bias_dtype, galv::as_stream(stream), nullptr, 0, 0, 3,
                                 act, ld_act, F);
  GALV_CHECK_ARG(ld_pre == F && ld_act == F && (bias == nullptr || bias_dtype == GALV_BF16),
                 "unfused fallback needs dense pre/act and a bf16 bias");
  int32_t rc = galv::gemm_bf16_sm100(X, W1, pre, nullptr, M, F, K, ldx, ldw, ld_pre, 0, 1, 1.0f,
                                     0, GALV_BF16, GALV_F32, galv::as_stream(stream));
  return rc ? rc : galv_bias_gelu_fwd(pre, bias, act, M, F, GALV_BF16, stream);
}

// GPT fc2 dgrad: dpre = (dY W2) * gelu_tanh'(pre + bias) with W2 [K=hidden, F] (nn.Linear
// layout of fc2); d(act) stays in TMEM.  The fallback stages d(act) in dpre and transforms
// it in place (each element is read before it is overwritten).
int32_t galv_gemm_bias_gelu_bwd(const void* dY, const void* W2, const void* pre,
                                const void* bias, void* dpre, int64_t M, int64_t F, int64_t K,
                                int64_t ldy, int64_t ldw, int64_t ld_pre, int64_t ld_dpre,
                                int32_t bias_dtype, void* stream) {
  GALV_CHECK_ARG(dY && W2 && pre && dpre && M > 0 && F > 0 && K > 0 && F % 8 == 0,
                 "bad arguments");
  GALV_CHECK_ARG(bias_dtype == GALV_BF16 || bias_dtype == GALV_F32, "bad bias dtype");
  if (galv::epilogue_fusable(dY, W2, dpre, pre, M, ld_dpre, ld_pre, F, 0, 4))
    return galv::gemm_bf16_sm100(dY, W2, dpre, bias, M, F, K, ldy, ldw, ld_dpre, 0, 0, 1.0f, 0,
                                 GALV_BF16, bias_dtype, galv::as_stream(stream), nullptr, 0, 0, 4,
                                 pre, ld_pre, F);
  GALV_CHECK_ARG(ld_pre == F && ld_dpre == F && (bias == nullptr || bias_dtype == GALV_BF16),
                 "unfused fallback needs dense pre/dpre and a bf16 bias");
  int32_t rc = galv::gemm_bf16_sm100(dY, W2, dpre, nullptr, M, F, K, ldy, ldw, ld_dpre, 0, 0,
                                     1.0f, 0, GALV_BF16, GALV_F32, galv::as_stream(stream));
  return rc ? rc : galv_bias_gelu_bwd(pre, bias, dpre, dpre, M, F, GALV_BF16, stream);
}

}  // extern "C"
