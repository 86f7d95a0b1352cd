// Attention C ABI entry points over [B, S, H, D] token-major q/k/v (the layout the fused QKV
// GEMM writes; no transposes), lse [B, H, S] fp32 natural-log logsumexp.
//   bf16 -> tcgen05/TMEM flash attention (attn_sm100.cu)
//   fp32 -> exact SIMT kernels below (thread per row), for the fp32 parity configuration.
#include "common.cuh"
#include "dropout.cuh"

namespace galv {
namespace attn {

// ------------------------------------------------------------------ fp32 SIMT path
// Dvec[b,h,i] = sum_d dO[i,d] * O[i,d]
__global__ void bwd_dot_f32(const float* __restrict__ o, const float* __restrict__ dout,
                            float* __restrict__ dvec, int S, int H, int D, int64_t ost,
                            int64_t sh) {
  const int64_t row = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);  // over S*H of batch y
  const int lane = threadIdx.x & 31;
  if (row >= (int64_t)S * H) return;
  const int b = blockIdx.y, i = (int)(row / H), h = (int)(row % H);
  const float* orow = o + (int64_t)b * S * ost + (int64_t)i * ost + (int64_t)h * sh;
  const float* drow = dout + (int64_t)b * S * ost + (int64_t)i * ost + (int64_t)h * sh;
  float s = 0.f;
  for (int d = lane; d < D; d += 32) s += orow[d] * drow[d];
  s = warp_sum(s);
  if (lane == 0) dvec[((int64_t)b * H + h) * S + i] = s;
}

// forward: thread per query row, K/V tiles staged in smem (padded rows)
template <int D>
__global__ void __launch_bounds__(64) fwd_f32(const float* __restrict__ q,
                                              const float* __restrict__ k,
                                              const float* __restrict__ v, float* __restrict__ o,
                                              float* __restrict__ lse, int S, int H, int64_t st,
                                              int64_t sh, int64_t ost, float scale, int causal,
                                              const DropoutParams drop) {
  __shared__ float ks[64][D + 1], vs[64][D + 1];
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int i = blockIdx.x * 64 + threadIdx.x;
  const int64_t off = (int64_t)b * S * st + (int64_t)h * sh;
  float qr[D], acc[D];
  const bool live = i < S;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    qr[d] = live ? q[off + (int64_t)i * st + d] : 0.f;
    acc[d] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const int kmax = causal ? min(S, blockIdx.x * 64 + 64) : S;
  for (int j0 = 0; j0 < kmax; j0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * D; e += 64) {
      const int r = e / D, d = e % D;
      const bool ok = j0 + r < S;
      ks[r][d] = ok ? k[off + (int64_t)(j0 + r) * st + d] : 0.f;
      vs[r][d] = ok ? v[off + (int64_t)(j0 + r) * st + d] : 0.f;
    }
    __syncthreads();
    if (!live) continue;
    for (int r = 0; r < 64; ++r) {
      const int j = j0 + r;
      if (j >= S || (causal && j > i)) break;
      float s = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) s = fmaf(qr[d], ks[r][d], s);
      s *= scale;
      const float mn = fmaxf(m, s);
      const float c = expf(m - mn), p = expf(s - mn);
      l = l * c + p;  // normalizer: undropped probabilities
      const float pd = (drop.thresh == 0 || dropout_keep(drop, b, h, i, j)) ? p : 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] = acc[d] * c + pd * vs[r][d];
      m = mn;
    }
  }
  if (!live) return;
  const float inv = (drop.thresh ? drop.inv_keep : 1.f) / l;
  const int64_t oo = (int64_t)b * S * ost + (int64_t)h * sh + (int64_t)i * ost;
#pragma unroll
  for (int d = 0; d < D; ++d) o[oo + d] = acc[d] * inv;
  lse[((int64_t)b * H + h) * S + i] = m + logf(l);
}

// dK/dV: thread per key row
template <int D>
__global__ void __launch_bounds__(64) bwd_dkdv_f32(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ dout, const float* __restrict__ lse, const float* __restrict__ dvec,
    float* __restrict__ dk, float* __restrict__ dv, int S, int H, int64_t st, int64_t sh,
    int64_t ost, float scale, int causal, const DropoutParams drop) {
  __shared__ float qs[64][D + 1], ds_[64][D + 1], ls[64], dd[64];
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int j = blockIdx.x * 64 + threadIdx.x;
  const int64_t off = (int64_t)b * S * st + (int64_t)h * sh;
  const int64_t ooff = (int64_t)b * S * ost + (int64_t)h * sh;
  const bool live = j < S;
  float kr[D], vr[D], gk[D], gv[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    kr[d] = live ? k[off + (int64_t)j * st + d] : 0.f;
    vr[d] = live ? v[off + (int64_t)j * st + d] : 0.f;
    gk[d] = gv[d] = 0.f;
  }
  const float* lg = lse + ((int64_t)b * H + h) * S;
  const float* dg = dvec + ((int64_t)b * H + h) * S;
  const int i_start = causal ? blockIdx.x * 64 : 0;
  for (int i0 = i_start; i0 < S; i0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * D; e += 64) {
      const int r = e / D, d = e % D;
      const bool ok = i0 + r < S;
      qs[r][d] = ok ? q[off + (int64_t)(i0 + r) * st + d] : 0.f;
      ds_[r][d] = ok ? dout[ooff + (int64_t)(i0 + r) * ost + d] : 0.f;
    }
    if (threadIdx.x < 64) {
      const int r = i0 + threadIdx.x;
      ls[threadIdx.x] = r < S ? lg[r] : 0.f;
      dd[threadIdx.x] = r < S ? dg[r] : 0.f;
    }
    __syncthreads();
    if (!live) continue;
    for (int r = 0; r < 64; ++r) {
      const int i = i0 + r;
      if (i >= S) break;
      if (causal && j > i) continue;
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        s = fmaf(qs[r][d], kr[d], s);
        dp = fmaf(ds_[r][d], vr[d], dp);
      }
      const float p = expf(s * scale - ls[r]);
      // dropout: dV from the kept, scaled P; dS = P * (dP * mask / (1-p) - D)
      const float kp = drop.thresh == 0 ? 1.f
                       : (dropout_keep(drop, b, h, i, j) ? drop.inv_keep : 0.f);
      const float dsv = p * (dp * kp - dd[r]);
      const float pk = p * kp;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        gv[d] = fmaf(pk, ds_[r][d], gv[d]);
        gk[d] = fmaf(dsv, qs[r][d], gk[d]);
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    dk[off + (int64_t)j * st + d] = gk[d] * scale;
    dv[off + (int64_t)j * st + d] = gv[d];
  }
}

// dQ: thread per query row
template <int D>
__global__ void __launch_bounds__(64) bwd_dq_f32(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ dout, const float* __restrict__ lse, const float* __restrict__ dvec,
    float* __restrict__ dq, int S, int H, int64_t st, int64_t sh, int64_t ost, float scale,
    int causal, const DropoutParams drop) {
  __shared__ float ks[64][D + 1], vs[64][D + 1];
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int i = blockIdx.x * 64 + threadIdx.x;
  const int64_t off = (int64_t)b * S * st + (int64_t)h * sh;
  const int64_t ooff = (int64_t)b * S * ost + (int64_t)h * sh;
  const bool live = i < S;
  float qr[D], dor[D], g[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    qr[d] = live ? q[off + (int64_t)i * st + d] : 0.f;
    dor[d] = live ? dout[ooff + (int64_t)i * ost + d] : 0.f;
    g[d] = 0.f;
  }
  const float l = live ? lse[((int64_t)b * H + h) * S + i] : 0.f;
  const float dd = live ? dvec[((int64_t)b * H + h) * S + i] : 0.f;
  const int kmax = causal ? min(S, blockIdx.x * 64 + 64) : S;
  for (int j0 = 0; j0 < kmax; j0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * D; e += 64) {
      const int r = e / D, d = e % D;
      const bool ok = j0 + r < S;
      ks[r][d] = ok ? k[off + (int64_t)(j0 + r) * st + d] : 0.f;
      vs[r][d] = ok ? v[off + (int64_t)(j0 + r) * st + d] : 0.f;
    }
    __syncthreads();
    if (!live) continue;
    for (int r = 0; r < 64; ++r) {
      const int j = j0 + r;
      if (j >= S || (causal && j > i)) break;
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        s = fmaf(qr[d], ks[r][d], s);
        dp = fmaf(dor[d], vs[r][d], dp);
      }
      const float p = expf(s * scale - l);
      const float kp = drop.thresh == 0 ? 1.f
                       : (dropout_keep(drop, b, h, i, j) ? drop.inv_keep : 0.f);
      const float dsv = p * (dp * kp - dd);
#pragma unroll
      for (int d = 0; d < D; ++d) g[d] = fmaf(dsv, ks[r][d], g[d]);
    }
  }
  if (!live) return;
#pragma unroll
  for (int d = 0; d < D; ++d) dq[off + (int64_t)i * st + d] = g[d] * scale;
}

}  // namespace attn
}  // namespace galv

using namespace galv;

template <typename K>
static int32_t set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    GALV_CUDA_RET(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes));
  return 0;
}

namespace galv {
int32_t attn_fwd_sm100(const void* q, const void* k, const void* v, void* o, float* lse,
                       int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                       int64_t ost, float scale, int32_t causal, cudaStream_t stream,
                       const DropoutParams& drop);
int64_t attn_bwd_ws_sm100(int64_t B, int64_t S, int64_t H);
int32_t attn_bwd_sm100(const void* q, const void* k, const void* v, const void* o,
                       const void* dout, const float* lse, void* dq, void* dk, void* dv,
                       int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                       int64_t ost, float scale, int32_t causal, void* ws, cudaStream_t stream,
                       const float* rope_table, const DropoutParams& drop);
}

extern "C" {

int32_t galv_attn_fwd_dropout(const void* q, const void* k, const void* v, void* o, float* lse,
                              int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                              int64_t ost, float scale, int32_t causal, float dropout_p,
                              uint64_t seed, uint64_t offset, int64_t b0, int64_t h0,
                              int64_t H_total, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(q && k && v && o && lse && B > 0 && S > 0 && H > 0, "bad arguments");
  GALV_CHECK_ARG(D == 64 || D == 128, "head_dim must be 64 or 128");
  GALV_CHECK_ARG(dropout_p >= 0.f && dropout_p < 1.f, "dropout_p must be in [0, 1)");
  GALV_CHECK_ARG(H_total >= h0 + H && b0 >= 0 && h0 >= 0, "bad dropout coordinates");
  const DropoutParams drop = make_dropout(dropout_p, seed, offset, b0, h0, H_total);
  const dim3 grid((unsigned)((S + 63) / 64), (unsigned)(B * H));
  cudaStream_t s = as_stream(stream);
  if (dtype == GALV_BF16) {
    GALV_CHECK_ARG(st % 8 == 0 && sh % 8 == 0 && ost % 8 == 0, "strides must be multiples of 8");
    return attn_fwd_sm100(q, k, v, o, lse, B, S, H, D, st, sh, ost, scale, causal, s, drop);
  } else {
    GALV_CHECK_ARG(dtype == GALV_F32, "bad dtype");
    if (D == 64)
      attn::fwd_f32<64><<<grid, 64, 0, s>>>((const float*)q, (const float*)k, (const float*)v,
                                            (float*)o, lse, (int)S, (int)H, st, sh, ost, scale,
                                            causal, drop);
    else
      GALV_CHECK_ARG(false, "fp32 attention supports head_dim 64");
  }
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t B,
                      int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh, int64_t ost,
                      float scale, int32_t causal, int32_t dtype, void* stream) {
  return galv_attn_fwd_dropout(q, k, v, o, lse, B, S, H, D, st, sh, ost, scale, causal, 0.f, 0, 0,
                               0, 0, H, dtype, stream);
}

// Device keep-mask of the attention dropout (test / oracle cross-check): mask[b][h][i][j] =
// 1 if element (query i, key j) of the call-local (b, h) is kept (dropout.cuh).
__global__ void dropout_mask_kernel(uint8_t* mask, int S, int H, DropoutParams d) {
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)S * S) return;
  const int i = (int)(e / S), j = (int)(e % S);
  mask[(int64_t)bh * S * S + e] = dropout_keep(d, b, h, i, j) ? 1 : 0;
}

int32_t galv_dropout_mask(uint8_t* mask, int64_t B, int64_t S, int64_t H, float dropout_p,
                          uint64_t seed, uint64_t offset, int64_t b0, int64_t h0, int64_t H_total,
                          void* stream) {
  GALV_CHECK_ARG(mask && B > 0 && S > 0 && H > 0 && dropout_p > 0.f && dropout_p < 1.f,
                 "bad arguments");
  const DropoutParams d = make_dropout(dropout_p, seed, offset, b0, h0, H_total);
  const dim3 grid((unsigned)((S * S + 255) / 256), (unsigned)(B * H));
  dropout_mask_kernel<<<grid, 256, 0, as_stream(stream)>>>(mask, (int)S, (int)H, d);
  GALV_LAUNCH_CHECK();
  return 0;
}

int64_t galv_attn_bwd_workspace(int64_t B, int64_t S, int64_t H, int64_t D, int32_t dtype) {
  (void)D;
  if (dtype == GALV_BF16) return galv::attn_bwd_ws_sm100(B, S, H);
  return B * H * S * (int64_t)sizeof(float);
}

// galv_attn_bwd with dq / dk returned through the inverse RoPE of q / k (bf16, head_dim
// 128); rope_table: fp32 [2][S][D/2] cos|sin planes, positions = token index mod S.
//   epilogue 1: rotated in the kernels' dq / dk store epilogues (attn_sm100.cu
//               store_row_out_rope) -- no extra pass over dq|dk, but the lane-per-row table
//               reads sit on the CTA's critical path (1 CTA/SM);
//   epilogue 0: the plain backward, then the streaming inverse-RoPE pass (rope.cu) -- one
//               launch over q|k heads when dk directly follows dq in the row;
//   epilogue < 0: library default = 0, the faster of the two as measured on B200
//               (Llama-2-7B shapes: 1015 + 48 us vs 1095-1210 us).
int32_t galv_attn_bwd_dropout(const void* q, const void* k, const void* v, const void* o,
                              const void* dout, const float* lse, void* dq, void* dk, void* dv,
                              int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                              int64_t ost, float scale, int32_t causal, float dropout_p,
                              uint64_t seed, uint64_t offset, int64_t b0, int64_t h0,
                              int64_t H_total, const float* rope_table, int32_t epilogue,
                              int32_t dtype, void* ws, void* stream) {
  GALV_CHECK_ARG(q && k && v && o && dout && lse && dq && dk && dv && ws, "bad arguments");
  GALV_CHECK_ARG(D == 64 || D == 128, "head_dim must be 64 or 128");
  GALV_CHECK_ARG(dropout_p >= 0.f && dropout_p < 1.f, "dropout_p must be in [0, 1)");
  GALV_CHECK_ARG(H_total >= h0 + H && b0 >= 0 && h0 >= 0, "bad dropout coordinates");
  const DropoutParams drop = make_dropout(dropout_p, seed, offset, b0, h0, H_total);
  cudaStream_t s = as_stream(stream);
  if (rope_table != nullptr) {
    GALV_CHECK_ARG(dtype == GALV_BF16 && D == 128, "RoPE backward: bf16, head_dim 128");
    GALV_CHECK_ARG(st % 8 == 0 && sh % 8 == 0 && ost % 8 == 0, "strides must be multiples of 8");
    if (epilogue > 0) {
      GALV_CHECK_ARG((reinterpret_cast<uintptr_t>(rope_table) & 15) == 0,
                     "rope_table must be 16-byte aligned");
      return attn_bwd_sm100(q, k, v, o, dout, lse, dq, dk, dv, B, S, H, D, st, sh, ost, scale,
                            causal, ws, s, rope_table, drop);
    }
    int32_t rc = attn_bwd_sm100(q, k, v, o, dout, lse, dq, dk, dv, B, S, H, D, st, sh, ost, scale,
                                causal, ws, s, nullptr, drop);
    if (rc) return rc;
    const __nv_bfloat16* q_end = static_cast<const __nv_bfloat16*>(dq) + H * sh;
    if (q_end == static_cast<const __nv_bfloat16*>(dk))  // [q heads | k heads]: one launch
      return galv_rope_table(dq, rope_table, B * S, S, 2 * H, D, st, sh, 0, 1, dtype, stream);
    rc = galv_rope_table(dq, rope_table, B * S, S, H, D, st, sh, 0, 1, dtype, stream);
    if (rc) return rc;
    return galv_rope_table(dk, rope_table, B * S, S, H, D, st, sh, 0, 1, dtype, stream);
  }
  float* dvec = (float*)ws;
  const dim3 grid((unsigned)((S + 63) / 64), (unsigned)(B * H));
  const dim3 gdot((unsigned)((S * H + 3) / 4), (unsigned)B);
  if (dtype == GALV_BF16) {
    GALV_CHECK_ARG(st % 8 == 0 && sh % 8 == 0 && ost % 8 == 0, "strides must be multiples of 8");
    return attn_bwd_sm100(q, k, v, o, dout, lse, dq, dk, dv, B, S, H, D, st, sh, ost, scale,
                          causal, ws, s, nullptr, drop);
  }
  GALV_CHECK_ARG(dtype == GALV_F32 && D == 64, "fp32 attention supports head_dim 64");
  attn::bwd_dot_f32<<<gdot, 128, 0, s>>>((const float*)o, (const float*)dout, dvec, (int)S,
                                         (int)H, (int)D, ost, sh);
  attn::bwd_dkdv_f32<64><<<grid, 64, 0, s>>>(
      (const float*)q, (const float*)k, (const float*)v, (const float*)dout, lse, dvec,
      (float*)dk, (float*)dv, (int)S, (int)H, st, sh, ost, scale, causal, drop);
  attn::bwd_dq_f32<64><<<grid, 64, 0, s>>>((const float*)q, (const float*)k, (const float*)v,
                                           (const float*)dout, lse, dvec, (float*)dq, (int)S,
                                           (int)H, st, sh, ost, scale, causal, drop);
  GALV_LAUNCH_CHECK();
  return 0;
}

// galv_attn_bwd with dq / dk returned through the inverse RoPE of q / k (bf16, head_dim
// 128); rope_table: fp32 [2][S][D/2] cos|sin planes, positions = token index mod S.
//   epilogue 1: rotated in the kernels' dq / dk store epilogues (attn_sm100.cu
//               store_row_out_rope) -- no extra pass over dq|dk, but the lane-per-row table
//               reads sit on the CTA's critical path (1 CTA/SM);
//   epilogue 0: the plain backward, then the streaming inverse-RoPE pass (rope.cu) -- one
//               launch over q|k heads when dk directly follows dq in the row;
//   epilogue < 0: library default = 0, the faster of the two as measured on B200
//               (Llama-2-7B shapes: 1015 + 48 us vs 1095-1210 us).
int32_t galv_attn_bwd_rope(const void* q, const void* k, const void* v, const void* o,
                           const void* dout, const float* lse, void* dq, void* dk, void* dv,
                           int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                           int64_t ost, float scale, int32_t causal, const float* rope_table,
                           int32_t epilogue, int32_t dtype, void* ws, void* stream) {
  GALV_CHECK_ARG(rope_table, "bad arguments");
  return galv_attn_bwd_dropout(q, k, v, o, dout, lse, dq, dk, dv, B, S, H, D, st, sh, ost, scale,
                               causal, 0.f, 0, 0, 0, 0, H, rope_table, epilogue, dtype, ws,
                               stream);
}

int32_t galv_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                      const void* dout, const float* lse, void* dq, void* dk, void* dv, int64_t B,
                      int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh, int64_t ost,
                      float scale, int32_t causal, int32_t dtype, void* ws, void* stream) {
  return galv_attn_bwd_dropout(q, k, v, o, dout, lse, dq, dk, dv, B, S, H, D, st, sh, ost, scale,
                               causal, 0.f, 0, 0, 0, 0, H, nullptr, 0, dtype, ws, stream);
}

}  // extern "C"
