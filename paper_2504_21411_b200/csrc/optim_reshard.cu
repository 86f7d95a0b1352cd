// Fused AdamW over flat fp32 shards (one HBM pass over master/m/v/grad + bf16 param
// write: 28 B/param for bf16 grads) and the reshard row gather/scatter used around the
// single collective of an inter-layer strategy transition.
#include "common.cuh"

namespace galv {
namespace opt {

template <typename TG, typename TP>
__global__ void adamw_kernel(float* __restrict__ master, float* __restrict__ m,
                             float* __restrict__ v, const TG* __restrict__ g,
                             TP* __restrict__ pout, int64_t n, float lr, float b1, float b2,
                             float eps, float wd, float gscale, float bc1, float bc2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gr = to_f(g[i]) * gscale;
    float p = master[i];
    const float mi = b1 * m[i] + (1.f - b1) * gr;
    const float vi = b2 * v[i] + (1.f - b2) * gr * gr;
    m[i] = mi;
    v[i] = vi;
    const float mhat = mi / bc1, vhat = vi / bc2;
    p = p - lr * (mhat / (sqrtf(vhat) + eps) + wd * p);
    master[i] = p;
    if (pout) pout[i] = from_f<TP>(p);
  }
}

// 4 parameters per thread-iteration with 16B master/m/v accesses (n % 4 == 0)
template <typename TG, typename TP>
__global__ void adamw_vec4(float* __restrict__ master, float* __restrict__ m,
                           float* __restrict__ v, const TG* __restrict__ g,
                           TP* __restrict__ pout, int64_t n4, float lr, float b1, float b2,
                           float eps, float wd, float gscale, float bc1, float bc2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 p4 = reinterpret_cast<float4*>(master)[i];
    float4 m4 = reinterpret_cast<float4*>(m)[i];
    float4 v4 = reinterpret_cast<float4*>(v)[i];
    float gr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) gr[k] = to_f(g[i * 4 + k]) * gscale;
    float* pp = &p4.x;
    float* mm = &m4.x;
    float* vv = &v4.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mm[k] = b1 * mm[k] + (1.f - b1) * gr[k];
      vv[k] = b2 * vv[k] + (1.f - b2) * gr[k] * gr[k];
      pp[k] = pp[k] - lr * ((mm[k] / bc1) / (sqrtf(vv[k] / bc2) + eps) + wd * pp[k]);
    }
    reinterpret_cast<float4*>(master)[i] = p4;
    reinterpret_cast<float4*>(m)[i] = m4;
    reinterpret_cast<float4*>(v)[i] = v4;
    if (pout) {
#pragma unroll
      for (int k = 0; k < 4; ++k) pout[i * 4 + k] = from_f<TP>(pp[k]);
    }
  }
}

}  // namespace opt

namespace rs {

__global__ void gather_rows16(const uint4* __restrict__ src, uint4* __restrict__ dst,
                              const int64_t* __restrict__ idx, int64_t n_rows, int64_t vpr) {
  const int64_t total = n_rows * vpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / vpr, c = i - r * vpr;
    dst[i] = src[idx[r] * vpr + c];
  }
}
__global__ void scatter_rows16(const uint4* __restrict__ src, uint4* __restrict__ dst,
                               const int64_t* __restrict__ idx, int64_t n_rows, int64_t vpr) {
  const int64_t total = n_rows * vpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / vpr, c = i - r * vpr;
    dst[idx[r] * vpr + c] = src[i];
  }
}

}  // namespace rs
}  // namespace galv

using namespace galv;

extern "C" {

int32_t galv_adamw(float* master, float* m, float* v, const void* grad, void* param_out,
                   int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay,
                   float grad_scale, int64_t step, int32_t grad_dtype, int32_t param_dtype,
                   void* stream) {
  GALV_CHECK_ARG(master && m && v && grad && n >= 0 && step >= 1, "bad arguments");
  if (n == 0) return 0;
  const float bc1 = 1.f - powf(beta1, (float)step), bc2 = 1.f - powf(beta2, (float)step);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, sm_count() * 8);
  GALV_DISPATCH(grad_dtype, TG, {
    GALV_DISPATCH(param_dtype, TP, {
      if (n % 4 == 0)
        opt::adamw_vec4<TG, TP><<<grid, 256, 0, as_stream(stream)>>>(
            master, m, v, (const TG*)grad, (TP*)param_out, n / 4, lr, beta1, beta2, eps,
            weight_decay, grad_scale, bc1, bc2);
      else
        opt::adamw_kernel<TG, TP><<<grid, 256, 0, as_stream(stream)>>>(
            master, m, v, (const TG*)grad, (TP*)param_out, n, lr, beta1, beta2, eps,
            weight_decay, grad_scale, bc1, bc2);
    });
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_gather_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows,
                         int64_t row_bytes, void* stream) {
  GALV_CHECK_ARG(src && dst && idx && n_rows >= 0 && row_bytes % 16 == 0, "bad arguments");
  if (n_rows == 0) return 0;
  const int64_t vpr = row_bytes / 16, total = n_rows * vpr;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, sm_count() * 8);
  rs::gather_rows16<<<grid, 256, 0, as_stream(stream)>>>((const uint4*)src, (uint4*)dst, idx,
                                                         n_rows, vpr);
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_scatter_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows,
                          int64_t row_bytes, void* stream) {
  GALV_CHECK_ARG(src && dst && idx && n_rows >= 0 && row_bytes % 16 == 0, "bad arguments");
  if (n_rows == 0) return 0;
  const int64_t vpr = row_bytes / 16, total = n_rows * vpr;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, sm_count() * 8);
  rs::scatter_rows16<<<grid, 256, 0, as_stream(stream)>>>((const uint4*)src, (uint4*)dst, idx,
                                                          n_rows, vpr);
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
