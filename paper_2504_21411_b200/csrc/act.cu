// Elementwise activation kernels (HBM-bound, 16-byte vectors, grid-stride):
//   SwiGLU (Llama MLP) on the fused gate|up GEMM output, bias+GeLU(tanh) (GPT MLP),
//   column sums for bias gradients, axpby / cast, sum of squares (grad-norm).
#include "common.cuh"

namespace galv {
namespace act {

__device__ __forceinline__ float silu(float x) { return x / (1.f + expf(-x)); }

// gu: [T, 2F] (gate | up), h: [T, F]
template <typename T>
__global__ void swiglu_fwd(const T* __restrict__ gu, T* __restrict__ h, int64_t T_, int64_t F) {
  constexpr int V = 16 / sizeof(T);
  const int64_t nvec = T_ * F / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * V, t = e / F, f = e - t * F;
    float g[V], u[V], o[V];
    load16(gu + t * 2 * F + f, g);
    load16(gu + t * 2 * F + F + f, u);
#pragma unroll
    for (int k = 0; k < V; ++k) o[k] = silu(g[k]) * u[k];
    store16(h + e, o);
  }
}

template <typename T>
__global__ void swiglu_bwd(const T* gu, const T* dh, T* dgu, int64_t T_, int64_t F,
                           int64_t ld_dh) {  // dh may alias dgu's up half (read before write)
  constexpr int V = 16 / sizeof(T);
  const int64_t nvec = T_ * F / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * V, t = e / F, f = e - t * F;
    float g[V], u[V], d[V], dg[V], du[V];
    load16(gu + t * 2 * F + f, g);
    load16(gu + t * 2 * F + F + f, u);
    load16(dh + t * ld_dh + f, d);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const float s = 1.f / (1.f + expf(-g[k]));
      du[k] = d[k] * g[k] * s;
      dg[k] = d[k] * u[k] * s * (1.f + g[k] * (1.f - s));
    }
    store16(dgu + t * 2 * F + f, dg);
    store16(dgu + t * 2 * F + F + f, du);
  }
}

// tanh: bf16 activations use the MUFU tanh.approx.f32 (max rel err ~2^-11, below the bf16
// rounding of the result); fp32 (the exact-parity config) keeps tanhf
template <bool FAST>
__device__ __forceinline__ float tanh_sel(float u) {
  if constexpr (FAST) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
    return t;
  } else {
    return tanhf(u);
  }
}
template <bool FAST = false>
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanh_sel<FAST>(k0 * (x + k1 * x * x * x)));
}
template <bool FAST = false>
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float u = k0 * (x + k1 * x * x * x);
  const float th = tanh_sel<FAST>(u);
  return 0.5f * (1.f + th) + 0.5f * x * (1.f - th * th) * k0 * (1.f + 3.f * k1 * x * x);
}

template <typename T>
__global__ void bias_gelu_fwd(const T* __restrict__ x, const T* __restrict__ b, T* __restrict__ y,
                              int64_t T_, int64_t F) {
  constexpr int V = 16 / sizeof(T);
  constexpr bool FAST = sizeof(T) == 2;
  const int64_t nvec = T_ * F / V;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // column of the vector: one 64-bit modulo per thread, then stepped (stride*V mod F < F)
  const int64_t fstep = (stride * V) % F;
  int64_t f = (i0 * V) % F;
  for (int64_t i = i0; i < nvec; i += stride) {
    const int64_t e = i * V;
    float v[V], bb[V];
    load16(x + e, v);
    if (b) load16(b + f, bb);
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = gelu_tanh<FAST>(v[k] + (b ? bb[k] : 0.f));
    store16(y + e, v);
    f += fstep;
    if (f >= F) f -= F;
  }
}

template <typename T>
__global__ void bias_gelu_bwd(const T* __restrict__ x, const T* __restrict__ b,
                              const T* __restrict__ dy, T* __restrict__ dx, int64_t T_,
                              int64_t F) {
  constexpr int V = 16 / sizeof(T);
  constexpr bool FAST = sizeof(T) == 2;
  const int64_t nvec = T_ * F / V;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t fstep = (stride * V) % F;
  int64_t f = (i0 * V) % F;
  for (int64_t i = i0; i < nvec; i += stride) {
    const int64_t e = i * V;
    float v[V], bb[V], d[V];
    load16(x + e, v);
    load16(dy + e, d);
    if (b) load16(b + f, bb);
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = d[k] * gelu_tanh_grad<FAST>(v[k] + (b ? bb[k] : 0.f));
    store16(dx + e, v);
    f += fstep;
    if (f >= F) f -= F;
  }
}

// out[c] (+)= sum_r x[r, c]: CTA = 128 threads x 2 columns (coalesced 512 B row segments
// for bf16), a chunk of rows per blockIdx.y, register accumulation, one atomic per column.
template <typename T>
__global__ void __launch_bounds__(128) colsum_kernel(const T* __restrict__ x,
                                                     float* __restrict__ out, int64_t rows,
                                                     int64_t cols, int64_t rows_per_cta) {
  const int64_t c = (blockIdx.x * 128 + threadIdx.x) * 2;
  if (c >= cols) return;
  const int64_t r0 = blockIdx.y * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  float s0 = 0.f, s1 = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    s0 += to_f(x[r * cols + c]);
    s1 += to_f(x[r * cols + c + 1]);
  }
  atomicAdd(&out[c], s0);
  atomicAdd(&out[c + 1], s1);
}

// vectorized column sums: CTA = 8 column-threads (16-byte vectors) x 32 row lanes over a
// 16-byte-aligned matrix; row lanes are reduced through smem, so each column gets one
// atomic per CTA (few CTAs per column strip -> no L2 atomic contention)
template <typename T>
__global__ void __launch_bounds__(256) colsum_vec(const T* __restrict__ x, float* __restrict__ out,
                                                  int64_t rows, int64_t cols,
                                                  int64_t rows_per_cta) {
  constexpr int V = 16 / sizeof(T);
  __shared__ float red[32][8 * V + 1];
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int64_t c = ((int64_t)blockIdx.x * 8 + tx) * V;
  const int64_t r0 = blockIdx.y * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  float s[V];
#pragma unroll
  for (int e = 0; e < V; ++e) s[e] = 0.f;
  if (c < cols) {
#pragma unroll 4
    for (int64_t r = r0 + ty; r < r1; r += 32) {
      float v[V];
      load16(x + r * cols + c, v);
#pragma unroll
      for (int e = 0; e < V; ++e) s[e] += v[e];
    }
  }
#pragma unroll
  for (int e = 0; e < V; ++e) red[ty][tx * V + e] = s[e];
  __syncthreads();
  if (threadIdx.x < 8 * V) {
    const int64_t col = (int64_t)blockIdx.x * 8 * V + threadIdx.x;
    float t = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) t += red[k][threadIdx.x];
    if (col < cols) atomicAdd(&out[col], t);
  }
}

// bias-GeLU backward with the bias gradient fused: dx = dy * gelu'(x + b) and
// dbias[f] += sum_t dx[t, f] (of the stored, T-rounded dx, as galv_colsum would see it).
#ifndef GELU_BWD_UNROLL
#define GELU_BWD_UNROLL 1  // 16384x4096 bf16: unroll 1 82.3 us, 2 96.0, 4 142.2 (kernels_ab/gelu)
#endif
constexpr int kGeluBwdUnroll = GELU_BWD_UNROLL;  // (#pragma unroll does not expand macros)
// colsum_vec's geometry: CTA = 8 column-threads (16-byte vectors) x 32 row lanes, row lanes
// reduced through smem, one atomic per column per CTA.  Saves the colsum re-read of dx.
template <typename T>
__global__ void __launch_bounds__(256) bias_gelu_bwd_colsum(
    const T* __restrict__ x, const T* __restrict__ b, const T* __restrict__ dy,
    T* __restrict__ dx, float* __restrict__ dbias, int64_t rows, int64_t cols,
    int64_t rows_per_cta) {
  constexpr int V = 16 / sizeof(T);
  __shared__ float red[32][8 * V + 1];
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int64_t c = ((int64_t)blockIdx.x * 8 + tx) * V;
  const int64_t r0 = blockIdx.y * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  float s[V], bb[V];
#pragma unroll
  for (int e = 0; e < V; ++e) s[e] = bb[e] = 0.f;
  if (c < cols) {
    if (b) {  // bias may be an unaligned view into a flat parameter buffer: scalar loads
#pragma unroll
      for (int e = 0; e < V; ++e) bb[e] = to_f(b[c + e]);
    }
#pragma unroll kGeluBwdUnroll
    for (int64_t r = r0 + ty; r < r1; r += 32) {
      float v[V], d[V];
      load16(x + r * cols + c, v);
      load16(dy + r * cols + c, d);
#pragma unroll
      for (int e = 0; e < V; ++e) v[e] = d[e] * gelu_tanh_grad<sizeof(T) == 2>(v[e] + bb[e]);
      // round once: store the packed values and sum exactly what was stored
      uint4 raw;
      T* pe = reinterpret_cast<T*>(&raw);
#pragma unroll
      for (int e = 0; e < V; ++e) pe[e] = from_f<T>(v[e]);
      *reinterpret_cast<uint4*>(dx + r * cols + c) = raw;
#pragma unroll
      for (int e = 0; e < V; ++e) s[e] += to_f(pe[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < V; ++e) red[ty][tx * V + e] = s[e];
  __syncthreads();
  if (threadIdx.x < 8 * V) {
    const int64_t col = (int64_t)blockIdx.x * 8 * V + threadIdx.x;
    float t = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) t += red[k][threadIdx.x];
    if (col < cols) atomicAdd(&dbias[col], t);
  }
}

template <typename TX, typename TY>
__global__ void axpby_kernel(const TX* __restrict__ x, TY* __restrict__ y, int64_t n, float a,
                             float b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float yv = b != 0.f ? to_f(y[i]) : 0.f;
    y[i] = from_f<TY>(a * to_f(x[i]) + b * yv);
  }
}

// vectorized variant: 8 elements per thread-iteration (n % 8 == 0, 16B-aligned pointers)
template <typename TX, typename TY>
__global__ void axpby_vec8(const TX* __restrict__ x, TY* __restrict__ y, int64_t n8, float a,
                           float b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    float xv[8], yv[8];
#pragma unroll
    for (int h = 0; h < 8; h += 16 / (int)sizeof(TX)) load16(x + i * 8 + h, xv + h);
    if (b != 0.f) {
#pragma unroll
      for (int h = 0; h < 8; h += 16 / (int)sizeof(TY)) load16(y + i * 8 + h, yv + h);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) yv[k] = a * xv[k] + (b != 0.f ? b * yv[k] : 0.f);
#pragma unroll
    for (int h = 0; h < 8; h += 16 / (int)sizeof(TY)) store16(y + i * 8 + h, yv + h);
  }
}

template <typename T>
__global__ void sumsq_kernel(const T* __restrict__ x, int64_t n, float* out) {
  __shared__ float red[33];
  float s = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = to_f(x[i]);
    s += v * v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) atomicAdd(out, s);
}

inline unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * 8;
  return (unsigned)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace act
}  // namespace galv

using namespace galv;

extern "C" {

int32_t galv_swiglu_fwd(const void* gu, void* h, int64_t T_, int64_t F, int32_t dtype,
                        void* stream) {
  GALV_CHECK_ARG(gu && h && T_ > 0 && F > 0 && F % 8 == 0, "bad arguments");
  GALV_DISPATCH(dtype, T, {
    const int64_t nvec = T_ * F / (16 / sizeof(T));
    act::swiglu_fwd<T><<<act::grid_for(nvec, 256), 256, 0, as_stream(stream)>>>(
        (const T*)gu, (T*)h, T_, F);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_swiglu_bwd(const void* gu, const void* dh, void* dgu, int64_t T_, int64_t F,
                        int32_t dtype, void* stream) {
  GALV_CHECK_ARG(gu && dh && dgu && T_ > 0 && F % 8 == 0, "bad arguments");
  GALV_DISPATCH(dtype, T, {
    const int64_t nvec = T_ * F / (16 / sizeof(T));
    act::swiglu_bwd<T><<<act::grid_for(nvec, 256), 256, 0, as_stream(stream)>>>(
        (const T*)gu, (const T*)dh, (T*)dgu, T_, F, F);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

// bf16 SwiGLU backward with dh rows `ld_dh` apart (the fused-GEMM fallback stages dh in the
// up half of dgu)
int32_t galv_swiglu_bwd_strided(const void* gu, const void* dh, int64_t ld_dh, void* dgu,
                                int64_t T_, int64_t F, void* stream) {
  GALV_CHECK_ARG(gu && dh && dgu && T_ > 0 && F % 8 == 0 && ld_dh % 8 == 0, "bad arguments");
  using T = __nv_bfloat16;
  const int64_t nvec = T_ * F / 8;
  act::swiglu_bwd<T><<<act::grid_for(nvec, 256), 256, 0, as_stream(stream)>>>(
      (const T*)gu, (const T*)dh, (T*)dgu, T_, F, ld_dh);
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_bias_gelu_fwd(const void* x, const void* bias, void* y, int64_t T_, int64_t F,
                           int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && y && T_ > 0 && F % 8 == 0, "bad arguments");
  GALV_CHECK_ARG(((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(bias)) & 15) == 0,
                 "x and bias must be 16-byte aligned (16-byte vector loads)");
  GALV_DISPATCH(dtype, T, {
    const int64_t nvec = T_ * F / (16 / sizeof(T));
    act::bias_gelu_fwd<T><<<act::grid_for(nvec, 256), 256, 0, as_stream(stream)>>>(
        (const T*)x, (const T*)bias, (T*)y, T_, F);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_bias_gelu_bwd(const void* x, const void* bias, const void* dy, void* dx, int64_t T_,
                           int64_t F, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && dy && dx && T_ > 0 && F % 8 == 0, "bad arguments");
  GALV_CHECK_ARG(((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(bias)) & 15) == 0,
                 "x and bias must be 16-byte aligned (16-byte vector loads)");
  GALV_DISPATCH(dtype, T, {
    const int64_t nvec = T_ * F / (16 / sizeof(T));
    act::bias_gelu_bwd<T><<<act::grid_for(nvec, 256), 256, 0, as_stream(stream)>>>(
        (const T*)x, (const T*)bias, (const T*)dy, (T*)dx, T_, F);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_bias_gelu_bwd_colsum(const void* x, const void* bias, const void* dy, void* dx,
                                  float* dbias_acc, int64_t T_, int64_t F, int32_t dtype,
                                  void* stream) {
  GALV_CHECK_ARG(x && dy && dx && dbias_acc && T_ > 0 && F > 0, "bad arguments");
  const int esz = dtype == GALV_BF16 ? 2 : 4;
  GALV_CHECK_ARG((F * esz) % 16 == 0, "F * element size must be a multiple of 16 bytes");
  GALV_CHECK_ARG(((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) |
                   reinterpret_cast<uintptr_t>(dx)) & 15) == 0,
                 "x, dy, dx must be 16-byte aligned");
  const int64_t per = 8 * (16 / esz);  // columns per CTA
  const int64_t strips = (F + per - 1) / per;
  const int64_t ych = std::max<int64_t>(
      1, std::min<int64_t>((T_ + 31) / 32, (int64_t)sm_count() * 8 / strips));
  const int64_t rpc = (T_ + ych - 1) / ych;
  GALV_DISPATCH(dtype, T, {
    act::bias_gelu_bwd_colsum<T><<<dim3((unsigned)strips, (unsigned)ych), 256, 0,
                                   as_stream(stream)>>>((const T*)x, (const T*)bias,
                                                        (const T*)dy, (T*)dx, dbias_acc, T_, F,
                                                        rpc);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

#ifndef COLSUM_CTAS_PER_SM
#define COLSUM_CTAS_PER_SM 4  // 8 or 16 measured the same (11-16 us at 16384x1024, noise)
#endif
int32_t galv_colsum(const void* x, float* out, int64_t rows, int64_t cols, int32_t accumulate,
                    int32_t dtype, void* ws, void* stream) {
  (void)ws;
  GALV_CHECK_ARG(x && out && rows > 0 && cols > 0, "bad arguments");
  if (!accumulate) GALV_CUDA_RET(cudaMemsetAsync(out, 0, sizeof(float) * cols, as_stream(stream)));
  GALV_CHECK_ARG(cols % 2 == 0, "cols must be even");
  const int esz = dtype == GALV_BF16 ? 2 : 4;
  if ((cols * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const int64_t per = 8 * (16 / esz);  // columns per CTA
    const int64_t strips_v = (cols + per - 1) / per;
    const int64_t ych = std::max<int64_t>(
        1, std::min<int64_t>((rows + 31) / 32, (int64_t)sm_count() * COLSUM_CTAS_PER_SM / strips_v));
    const int64_t rpc_v = (rows + ych - 1) / ych;
    dim3 g((unsigned)strips_v, (unsigned)ych);
    GALV_DISPATCH(dtype, T, {
      act::colsum_vec<T><<<g, 256, 0, as_stream(stream)>>>((const T*)x, out, rows, cols, rpc_v);
    });
    GALV_LAUNCH_CHECK();
    return 0;
  }
  const int64_t strips = (cols / 2 + 127) / 128;
  const int64_t ychunks = std::max<int64_t>(
      1, std::min<int64_t>(rows / 16 + 1, sm_count() * 16 / std::max<int64_t>(1, strips) + 1));
  const int64_t rpc = (rows + ychunks - 1) / ychunks;
  dim3 grid((unsigned)strips, (unsigned)ychunks);
  GALV_DISPATCH(dtype, T, {
    act::colsum_kernel<T><<<grid, 128, 0, as_stream(stream)>>>((const T*)x, out, rows, cols, rpc);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_axpby(const void* x, void* y, int64_t n, float a, float b, int32_t x_dtype,
                   int32_t y_dtype, void* stream) {
  GALV_CHECK_ARG(x && y && n >= 0, "bad arguments");
  if (n == 0) return 0;
  const bool vec = (n % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  GALV_DISPATCH(x_dtype, TX, {
    GALV_DISPATCH(y_dtype, TY, {
      if (vec)
        act::axpby_vec8<TX, TY><<<act::grid_for(n / 8, 256), 256, 0, as_stream(stream)>>>(
            (const TX*)x, (TY*)y, n / 8, a, b);
      else
        act::axpby_kernel<TX, TY><<<act::grid_for(n, 256), 256, 0, as_stream(stream)>>>(
            (const TX*)x, (TY*)y, n, a, b);
    });
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_sumsq(const void* x, int64_t n, float* out, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && out && n >= 0, "bad arguments");
  if (n == 0) return 0;
  GALV_DISPATCH(dtype, T, {
    act::sumsq_kernel<T><<<act::grid_for(n, 256), 256, 0, as_stream(stream)>>>((const T*)x, n,
                                                                                out);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"

namespace galv {
namespace act {
template <typename T>
__global__ void bias_add_kernel(T* __restrict__ x, const T* __restrict__ b, int64_t T_,
                                int64_t F) {
  constexpr int V = 16 / sizeof(T);
  const int64_t nvec = T_ * F / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * V, f = e % F;
    float v[V], bb[V];
    load16(x + e, v);
    load16(b + f, bb);
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] += bb[k];
    store16(x + e, v);
  }
}
}  // namespace act
}  // namespace galv

extern "C" int32_t galv_bias_add(void* x, const void* bias, int64_t T_, int64_t F, int32_t dtype,
                                 void* stream) {
  GALV_CHECK_ARG(x && bias && T_ > 0 && F % 8 == 0, "bad arguments");
  GALV_CHECK_ARG(((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(bias)) & 15) == 0,
                 "x and bias must be 16-byte aligned (16-byte vector loads)");
  GALV_DISPATCH(dtype, T, {
    const int64_t nvec = T_ * F / (16 / sizeof(T));
    act::bias_add_kernel<T><<<act::grid_for(nvec, 256), 256, 0, as_stream(stream)>>>(
        (T*)x, (const T*)bias, T_, F);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}
