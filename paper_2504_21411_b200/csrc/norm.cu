// RMSNorm (Llama) / LayerNorm (GPT) forward+backward with an optional fused residual add.
// HBM-bound: one warp per row, 16-byte vector loads, warp-shuffle reductions; the
// second pass over the row hits L1.  dgamma/dbeta are reduced per CTA in shared memory
// (grid-stride over rows, one CTA set per SM) and flushed with one atomic per column
// per CTA into fp32 accumulators.
#include "common.cuh"

namespace galv {
namespace norm {

constexpr int WARPS = 8;

template <typename T, bool LAYER, bool RESID>
__global__ void __launch_bounds__(WARPS * 32) fwd_kernel(
    const T* __restrict__ x, const T* __restrict__ res, T* __restrict__ res_out,
    const T* __restrict__ gamma, const T* __restrict__ beta, T* __restrict__ y,
    float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows, int cols,
    float eps) {
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* xr = x + row * cols;
  const T* rr = RESID ? res + row * cols : nullptr;
  T* ro = RESID ? res_out + row * cols : nullptr;
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V];
    load16(xr + c, v);
    if (RESID) {
      float r[V];
      load16(rr + c, r);
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] += r[i];
      store16(ro + c, v);
      // re-round to T so the normalized value matches the stored residual stream
      load16(ro + c, v);
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      s1 += v[i];
      s2 += v[i] * v[i];
    }
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  float mu = 0.f, rstd;
  if (LAYER) {
    mu = s1 / cols;
    float var = fmaxf(s2 / cols - mu * mu, 0.f);
    rstd = rsqrtf(var + eps);
  } else {
    rstd = rsqrtf(s2 / cols + eps);
  }
  if (lane == 0) {
    rstd_out[row] = rstd;
    if (LAYER) mean_out[row] = mu;
  }
  const T* src = RESID ? ro : xr;
  T* yr = y + row * cols;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V], g[V], b[V];
    load16(src + c, v);
    load16(gamma + c, g);
    if (LAYER) load16(beta + c, b);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = (v[i] - mu) * rstd * g[i] + (LAYER ? b[i] : 0.f);
    store16(yr + c, v);
  }
}

// dx = rstd * (g*dy - xhat * mean(g*dy*xhat) [- mean(g*dy) for LayerNorm]) (+ dres)
// dgamma/dbeta partials are accumulated in warp-private shared-memory rows (no atomics),
// summed per CTA at the end and flushed with one global atomic per column per CTA.
constexpr int BWD_WARPS = 4;
template <typename T, bool LAYER>
__global__ void __launch_bounds__(BWD_WARPS * 32) bwd_kernel(
    const T* __restrict__ x, const T* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, const T* __restrict__ dy, const T* __restrict__ dres,
    T* __restrict__ dx, float* __restrict__ dgamma, float* __restrict__ dbeta, int64_t rows,
    int cols) {
  constexpr int V = 16 / sizeof(T);
  extern __shared__ float sacc[];  // [BWD_WARPS][(LAYER ? 2 : 1) * cols]
  const int per = cols * (LAYER ? 2 : 1);
  for (int c = threadIdx.x; c < per * BWD_WARPS; c += blockDim.x) sacc[c] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* mine = sacc + w * per;
  for (int64_t row = (int64_t)blockIdx.x * BWD_WARPS + w; row < rows;
       row += (int64_t)gridDim.x * BWD_WARPS) {
    const T* xr = x + row * cols;
    const T* dyr = dy + row * cols;
    const float mu = LAYER ? mean[row] : 0.f, rs = rstd[row];
    float a1 = 0.f, a2 = 0.f;  // sum(g*dy*xhat), sum(g*dy)
    for (int c = lane * V; c < cols; c += 32 * V) {
      float v[V], d[V], g[V];
      load16(xr + c, v);
      load16(dyr + c, d);
      load16(gamma + c, g);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = (v[i] - mu) * rs;
        const float gd = g[i] * d[i];
        a1 += gd * xh;
        a2 += gd;
        mine[c + i] += d[i] * xh;
        if (LAYER) mine[cols + c + i] += d[i];
      }
    }
    a1 = warp_sum(a1) / cols;
    a2 = warp_sum(a2) / cols;
    T* dxr = dx + row * cols;
    const T* drr = dres ? dres + row * cols : nullptr;
    for (int c = lane * V; c < cols; c += 32 * V) {
      float v[V], d[V], g[V], r[V];
      load16(xr + c, v);
      load16(dyr + c, d);
      load16(gamma + c, g);
      if (drr) load16(drr + c, r);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = (v[i] - mu) * rs;
        float o = rs * (g[i] * d[i] - xh * a1 - (LAYER ? a2 : 0.f));
        if (drr) o += r[i];
        v[i] = o;
      }
      store16(dxr + c, v);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < per; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < BWD_WARPS; ++k) t += sacc[k * per + c];
    if (c < cols)
      atomicAdd(&dgamma[c], t);
    else
      atomicAdd(&dbeta[c - cols], t);
  }
}

}  // namespace norm
}  // namespace galv

using namespace galv;

template <bool LAYER>
static int32_t norm_fwd(const void* x, const void* residual, void* res_out, const void* gamma,
                        const void* beta, void* y, float* mean, float* rstd, int64_t rows,
                        int64_t cols, float eps, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && gamma && y && rstd && rows > 0 && cols > 0, "bad arguments");
  GALV_CHECK_ARG(!LAYER || (beta && mean), "layernorm needs beta and mean");
  GALV_CHECK_ARG(!residual || res_out, "residual needs res_out");
  GALV_CHECK_ARG(cols % 8 == 0, "cols must be a multiple of 8");
  const unsigned grid = (unsigned)((rows + norm::WARPS - 1) / norm::WARPS);
  GALV_DISPATCH(dtype, T, {
    if (residual)
      norm::fwd_kernel<T, LAYER, true><<<grid, norm::WARPS * 32, 0, as_stream(stream)>>>(
          (const T*)x, (const T*)residual, (T*)res_out, (const T*)gamma, (const T*)beta, (T*)y,
          mean, rstd, rows, (int)cols, eps);
    else
      norm::fwd_kernel<T, LAYER, false><<<grid, norm::WARPS * 32, 0, as_stream(stream)>>>(
          (const T*)x, nullptr, nullptr, (const T*)gamma, (const T*)beta, (T*)y, mean, rstd,
          rows, (int)cols, eps);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

template <bool LAYER>
static int32_t norm_bwd(const void* x, const void* gamma, const float* mean, const float* rstd,
                        const void* dy, const void* dres, void* dx, float* dgamma, float* dbeta,
                        int64_t rows, int64_t cols, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && gamma && rstd && dy && dx && dgamma && rows > 0, "bad arguments");
  GALV_CHECK_ARG(!LAYER || (mean && dbeta), "layernorm needs mean and dbeta");
  GALV_CHECK_ARG(cols % 8 == 0, "cols must be a multiple of 8");
  const size_t smem = sizeof(float) * cols * (LAYER ? 2 : 1) * norm::BWD_WARPS;
  GALV_CHECK_ARG(smem <= 220 * 1024, "cols too large for the dgamma reduction");
  int64_t want = (rows + norm::BWD_WARPS - 1) / norm::BWD_WARPS;
  const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)sm_count());
  GALV_DISPATCH(dtype, T, {
    auto k = norm::bwd_kernel<T, LAYER>;
    if (smem > 48 * 1024)
      GALV_CUDA_RET(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    k<<<grid, norm::BWD_WARPS * 32, smem, as_stream(stream)>>>(
        (const T*)x, (const T*)gamma, mean, rstd, (const T*)dy, (const T*)dres, (T*)dx, dgamma,
        dbeta, rows, (int)cols);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

extern "C" {

int32_t galv_rmsnorm_fwd(const void* x, const void* residual, void* res_out, const void* gamma,
                         void* y, float* rstd, int64_t rows, int64_t cols, float eps,
                         int32_t dtype, void* stream) {
  return norm_fwd<false>(x, residual, res_out, gamma, nullptr, y, nullptr, rstd, rows, cols, eps,
                         dtype, stream);
}

int32_t galv_rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy,
                         const void* dres_in, void* dx, float* dgamma_acc, int64_t rows,
                         int64_t cols, int32_t dtype, void* ws, void* stream) {
  (void)ws;
  return norm_bwd<false>(x, gamma, nullptr, rstd, dy, dres_in, dx, dgamma_acc, nullptr, rows,
                         cols, dtype, stream);
}

int32_t galv_layernorm_fwd(const void* x, const void* residual, void* res_out, const void* gamma,
                           const void* beta, void* y, float* mean, float* rstd, int64_t rows,
                           int64_t cols, float eps, int32_t dtype, void* stream) {
  return norm_fwd<true>(x, residual, res_out, gamma, beta, y, mean, rstd, rows, cols, eps, dtype,
                        stream);
}

int32_t galv_layernorm_bwd(const void* x, const void* gamma, const float* mean, const float* rstd,
                           const void* dy, const void* dres_in, void* dx, float* dgamma_acc,
                           float* dbeta_acc, int64_t rows, int64_t cols, int32_t dtype, void* ws,
                           void* stream) {
  (void)ws;
  return norm_bwd<true>(x, gamma, mean, rstd, dy, dres_in, dx, dgamma_acc, dbeta_acc, rows, cols,
                        dtype, stream);
}

int64_t galv_norm_bwd_workspace(int64_t rows, int64_t cols) {
  (void)rows;
  (void)cols;
  return 0;
}

}  // extern "C"
