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
                        int32_t my_slot = 0);
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

}  // extern "C"
