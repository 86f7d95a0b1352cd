// Exact FP32 SIMT GEMM (tcgen05 has no fp32 kind): the fp32 parity configuration's
// contraction path (BASELINE config 1, <= 1e-5 relative vs the CPU restatement).
// 64x64 tile, 256 threads, 4x4 micro-tile per thread, K step 16; any transpose combo.
#include "common.cuh"

namespace galv {
namespace f32 {

constexpr int TM = 64, TN = 64, TK = 16;

template <typename TC>
__global__ void __launch_bounds__(256) gemm_f32_kernel(
    const float* __restrict__ A, const float* __restrict__ B, TC* __restrict__ C,
    const float* __restrict__ bias, int M, int N, int K, long long lda, long long ldb,
    long long ldc, int ta, int tb, float alpha, int accumulate, long long sa, long long sb,
    long long sc) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  A += blockIdx.z * sa;
  B += blockIdx.z * sb;
  C += blockIdx.z * sc;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TK * TM; i += 256) {
      int kk, mm;
      if (ta) { mm = i % TM; kk = i / TM; } else { kk = i % TK; mm = i / TK; }
      const int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < K) v = ta ? A[(long long)gk * lda + gm] : A[(long long)gm * lda + gk];
      As[kk][mm] = v;
    }
    for (int i = threadIdx.x; i < TK * TN; i += 256) {
      int kk, nn;
      if (tb) { kk = i % TK; nn = i / TK; } else { nn = i % TN; kk = i / TN; }
      const int gn = n0 + nn, gk = k0 + kk;
      float v = 0.f;
      if (gn < N && gk < K) v = tb ? B[(long long)gn * ldb + gk] : B[(long long)gk * ldb + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j] * alpha;
      if (bias) v += bias[gn];
      TC* c = C + (long long)gm * ldc + gn;
      if (accumulate) v += to_f(*c);
      *c = from_f<TC>(v);
    }
  }
}

}  // namespace f32

int32_t gemm_f32_simt(const float* A, const float* B, void* C, const float* bias, int64_t batch,
                      int64_t sa, int64_t sb, int64_t sc, int64_t M, int64_t N, int64_t K,
                      int64_t lda, int64_t ldb, int64_t ldc, int32_t ta, int32_t tb, float alpha,
                      int32_t accumulate, int32_t c_dtype, cudaStream_t stream) {
  GALV_CHECK_ARG(M > 0 && N > 0 && K > 0 && batch > 0, "empty problem");
  dim3 grid((unsigned)((N + f32::TN - 1) / f32::TN), (unsigned)((M + f32::TM - 1) / f32::TM),
            (unsigned)batch);
  if (c_dtype == GALV_F32)
    f32::gemm_f32_kernel<float><<<grid, 256, 0, stream>>>(
        A, B, (float*)C, bias, (int)M, (int)N, (int)K, lda, ldb, ldc, ta, tb, alpha, accumulate,
        sa, sb, sc);
  else
    f32::gemm_f32_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(
        A, B, (__nv_bfloat16*)C, bias, (int)M, (int)N, (int)K, lda, ldb, ldc, ta, tb, alpha,
        accumulate, sa, sb, sc);
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // namespace galv
