// Rotary position embedding (rotate-half convention) applied in place to the q and k
// slices of the fused QKV GEMM output.  Angles are computed in fp32 from the position
// (token index mod S, plus an offset for sequence-sharded layouts) -- no tables in HBM.
#include "common.cuh"

namespace galv {
namespace rope {

template <typename T>
__global__ void rope_kernel(T* __restrict__ x, int64_t T_, int64_t S, int H, int D,
                            int64_t stride_tok, int64_t stride_head, int64_t pos0, float theta,
                            int inverse) {
  const int half = D / 2;
  const int64_t total = T_ * H * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % half);
    const int64_t th = i / half;
    const int h = (int)(th % H);
    const int64_t t = th / H;
    const float pos = (float)(pos0 + t % S);
    // inv_freq = theta^(-2j/D), evaluated like the CPU restatement (fp32 pow)
    const float inv_freq = 1.0f / powf(theta, (float)(2 * j) / (float)D);
    float s, c;
    sincosf(pos * inv_freq, &s, &c);
    if (inverse) s = -s;
    T* p = x + t * stride_tok + h * stride_head;
    const float a = to_f(p[j]), b = to_f(p[j + half]);
    p[j] = from_f<T>(a * c - b * s);
    p[j + half] = from_f<T>(b * c + a * s);
  }
}

// table-driven, vectorized: each thread rotates 8 (or 4 for fp32) pairs; cs = [S, D/2] x
// {cos, sin} fp32 interleaved as two planes: cos at cs[p*D/2 + j], sin at cs[S*D/2 + ...]
template <typename T>
__global__ void rope_table_kernel(T* __restrict__ x, const float* __restrict__ cs, int64_t T_,
                                  int64_t S, int H, int D, int64_t stride_tok,
                                  int64_t stride_head, int64_t pos0, int inverse) {
  constexpr int V = 16 / sizeof(T);
  const int half = D / 2, vec_per_head = half / V;
  const int64_t total = T_ * H * vec_per_head;
  const float* sn = cs + S * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int jv = (int)(i % vec_per_head);
    const int64_t th = i / vec_per_head;
    const int h = (int)(th % H);
    const int64_t t = th / H;
    const int64_t pos = (pos0 + t) % S;
    T* p = x + t * stride_tok + h * stride_head + jv * V;
    float a[V], b[V], c[V], s[V];
    load16(p, a);
    load16(p + half, b);
#pragma unroll
    for (int k = 0; k < V; k += 4) {
      *reinterpret_cast<float4*>(c + k) =
          *reinterpret_cast<const float4*>(cs + pos * half + jv * V + k);
      *reinterpret_cast<float4*>(s + k) =
          *reinterpret_cast<const float4*>(sn + pos * half + jv * V + k);
    }
    float o1[V], o2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const float sk = inverse ? -s[k] : s[k];
      o1[k] = a[k] * c[k] - b[k] * sk;
      o2[k] = b[k] * c[k] + a[k] * sk;
    }
    store16(p, o1);
    store16(p + half, o2);
  }
}

}  // namespace rope
}  // namespace galv

using namespace galv;

extern "C" int32_t galv_rope_table(void* x, const float* table, int64_t T_, int64_t S,
                                   int64_t H, int64_t D, int64_t stride_tok, int64_t stride_head,
                                   int64_t pos0, int32_t inverse, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && table && T_ > 0 && S > 0 && H > 0 && D % 16 == 0, "bad arguments");
  GALV_CHECK_ARG(stride_tok % 8 == 0 && stride_head % 8 == 0, "strides must be multiples of 8");
  GALV_DISPATCH(dtype, T, {
    const int64_t total = T_ * H * (D / 2) / (16 / sizeof(T));
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, sm_count() * 16);
    rope::rope_table_kernel<T><<<grid, 256, 0, as_stream(stream)>>>(
        (T*)x, table, T_, S, (int)H, (int)D, stride_tok, stride_head, pos0, inverse);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

extern "C" int32_t galv_rope(void* x, int64_t T_, int64_t S, int64_t H, int64_t D,
                             int64_t stride_tok, int64_t stride_head, int64_t pos0, float theta,
                             int32_t inverse, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && T_ > 0 && S > 0 && H > 0 && D > 0 && D % 2 == 0, "bad arguments");
  const int64_t total = T_ * H * (D / 2);
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, sm_count() * 16);
  GALV_DISPATCH(dtype, T, {
    rope::rope_kernel<T><<<grid, 256, 0, as_stream(stream)>>>(
        (T*)x, T_, S, (int)H, (int)D, stride_tok, stride_head, pos0, theta, inverse);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}
