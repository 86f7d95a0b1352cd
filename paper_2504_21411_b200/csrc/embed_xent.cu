// Token embedding (vocab-sharded gather / fp32 scatter-add) and vocab-parallel
// cross-entropy.  The cross-entropy never materializes fp32 [T, V] probabilities: the
// gradient is written in place over the logits in the GEMM's dtype.
#include "common.cuh"

namespace galv {
namespace emb {

template <typename T>
__global__ void embed_fwd(const int64_t* __restrict__ ids, const T* __restrict__ table,
                          T* __restrict__ out, int64_t T_, int64_t V_local, int64_t lo,
                          int64_t Hd) {
  constexpr int V = 16 / sizeof(T);
  const int64_t t = blockIdx.x;
  const int64_t id = ids[t] - lo;
  const bool mine = id >= 0 && id < V_local;
  for (int64_t c = threadIdx.x * V; c < Hd; c += blockDim.x * V) {
    float v[V];
    if (mine)
      load16(table + id * Hd + c, v);
    else
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = 0.f;
    store16(out + t * Hd + c, v);
  }
}

template <typename T>
__global__ void embed_bwd(const int64_t* __restrict__ ids, const T* __restrict__ dout,
                          float* __restrict__ dtable, int64_t T_, int64_t V_local, int64_t lo,
                          int64_t Hd) {
  const int64_t t = blockIdx.x;
  const int64_t id = ids[t] - lo;
  if (id < 0 || id >= V_local) return;
  for (int64_t c = threadIdx.x; c < Hd; c += blockDim.x)
    atomicAdd(&dtable[id * Hd + c], to_f(dout[t * Hd + c]));
}

// Deterministic embedding backward over token ids sorted by id (stable): the CTA at the
// first position of each id's run sums that id's dout rows in fp32 registers (each thread
// owns 8 columns per 2048-column chunk) and adds the sum once into the gradient row, in the
// gradient's own dtype (bf16 or fp32).  No fp32 [V, h] scratch table, no atomics: dout is
// read once and each touched gradient row is read and written once.
template <typename T, typename G>
__global__ void __launch_bounds__(256) embed_bwd_sorted(const int64_t* __restrict__ sorted,
                                                        const int64_t* __restrict__ order,
                                                        const T* __restrict__ dout,
                                                        G* __restrict__ grad, int64_t T_,
                                                        int64_t V_local, int64_t lo,
                                                        int64_t Hd) {
  const int64_t t = blockIdx.x;
  const int64_t key = sorted[t];
  if (t > 0 && sorted[t - 1] == key) return;  // not the first of its run
  const int64_t id = key - lo;
  if (id < 0 || id >= V_local) return;        // another rank's vocab shard
  int64_t end = t + 1;
  while (end < T_ && sorted[end] == key) ++end;
  for (int64_t c0 = threadIdx.x * 8; c0 < Hd; c0 += 256 * 8) {
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int64_t r = t; r < end; ++r) {
      const T* row = dout + order[r] * Hd + c0;
      float v[8];
      if constexpr (sizeof(T) == 2) {
        load16(row, v);
      } else {
        load16(row, v);
        load16(row + 4, v + 4);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
    G* g = grad + id * Hd + c0;
    float cur[8];
    if constexpr (sizeof(G) == 2) {
      load16(g, cur);
    } else {
      load16(g, cur);
      load16(g + 4, cur + 4);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) cur[i] += acc[i];
    if constexpr (sizeof(G) == 2) {
      store16(g, cur);
    } else {
      store16(g, cur);
      store16(g + 4, cur + 4);
    }
  }
}

}  // namespace emb

namespace xent {

// one CTA per row. stats layout per row: [max, sumexp, target_logit]
template <typename T>
__global__ void __launch_bounds__(256) xent_kernel(T* __restrict__ logits,
                                                   const int64_t* __restrict__ labels,
                                                   float* __restrict__ stats,
                                                   float* __restrict__ loss, T* __restrict__ dl,
                                                   int64_t V_local, int64_t lo, float gscale,
                                                   int64_t ignore, int stage) {
  __shared__ float red[33];
  const int64_t row = blockIdx.x;
  T* x = logits + row * V_local;
  const int64_t lab = labels[row];
  const int64_t tgt = lab - lo;
  float* st = stats + row * 3;
  if (stage == 0 || stage == 3) {
    float m = -INFINITY;
    for (int64_t c = threadIdx.x; c < V_local; c += blockDim.x) m = fmaxf(m, to_f(x[c]));
    // block max via shuffles
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
      t = warp_max(t);
      if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) st[0] = red[32];
    __syncthreads();
    if (stage == 0) return;
  }
  if (stage == 1 || stage == 3) {
    const float m = st[0];
    float s = 0.f;
    for (int64_t c = threadIdx.x; c < V_local; c += blockDim.x) s += expf(to_f(x[c]) - m);
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      st[1] = s;
      st[2] = (tgt >= 0 && tgt < V_local) ? to_f(x[tgt]) : 0.f;
    }
    __syncthreads();
    if (stage == 1) return;
  }
  // stage 2 (or 3): loss + gradient
  const float m = st[0], s = st[1];
  const bool ign = lab == ignore;
  if (threadIdx.x == 0) loss[row] = ign ? 0.f : (logf(s) + m - st[2]);
  T* d = dl + row * V_local;
  const float inv = 1.f / s;
  for (int64_t c = threadIdx.x; c < V_local; c += blockDim.x) {
    float g = ign ? 0.f : expf(to_f(x[c]) - m) * inv;
    if (!ign && c == tgt) g -= 1.f;
    d[c] = from_f<T>(g * gscale);
  }
}

// Vectorized variant (rows 16-byte aligned, V_local a multiple of the 16-byte vector):
// stage 3 makes ONE pass over the logits for the row statistics -- an online (max, sum of
// exp) per thread, merged across the CTA -- and a second pass (an L2 hit: the row was just
// read) writing the gradient in place, so HBM sees the logits read once and written once;
// the scalar kernel above read them three times with 2-byte loads.
constexpr float XLOG2E = 1.4426950408889634f;

__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  if (mm == -INFINITY) return;
  s = s * exp2f((m - mm) * XLOG2E) + s2 * exp2f((m2 - mm) * XLOG2E);
  m = mm;
}

template <typename T>
__global__ void __launch_bounds__(256) xent_vec(T* __restrict__ logits,
                                                const int64_t* __restrict__ labels,
                                                float* __restrict__ stats,
                                                float* __restrict__ loss, T* __restrict__ dl,
                                                int64_t V_local, int64_t lo, float gscale,
                                                int64_t ignore, int stage) {
  constexpr int VEC = 16 / sizeof(T);
  __shared__ float red_m[8], red_s[8], bc[2];
  const int64_t row = blockIdx.x;
  const T* x = logits + row * V_local;
  const int64_t lab = labels[row];
  const int64_t tgt = lab - lo;
  float* st = stats + row * 3;
  const int nvec = (int)(V_local / VEC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float m = -INFINITY, sum = 0.f;
  if (stage == 0 || stage == 3) {
    for (int v = threadIdx.x; v < nvec; v += 256) {
      float e[VEC];
      load16(x + (int64_t)v * VEC, e);
      float mv = e[0];
#pragma unroll
      for (int i = 1; i < VEC; ++i) mv = fmaxf(mv, e[i]);
      if (stage == 3) {
        const float mn = fmaxf(m, mv);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc += exp2f((e[i] - mn) * XLOG2E);
        sum = (m == -INFINITY ? 0.f : sum * exp2f((m - mn) * XLOG2E)) + acc;
      }
      m = fmaxf(m, mv);
    }
    // merge (max, sum) across the warp, then across warps
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      online_merge(m, sum, m2, s2);
    }
    if (lane == 0) {
      red_m[warp] = m;
      red_s[warp] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float mm = red_m[0], ss = red_s[0];
      for (int w = 1; w < 8; ++w) online_merge(mm, ss, red_m[w], red_s[w]);
      bc[0] = mm;
      bc[1] = ss;
      st[0] = mm;
      if (stage == 3) {
        st[1] = ss;
        st[2] = (tgt >= 0 && tgt < V_local) ? to_f(x[tgt]) : 0.f;
      }
    }
    __syncthreads();
    if (stage == 0) return;
    m = bc[0];
    sum = bc[1];
  }
  if (stage == 1) {
    const float mg = st[0];
    float acc = 0.f;
    for (int v = threadIdx.x; v < nvec; v += 256) {
      float e[VEC];
      load16(x + (int64_t)v * VEC, e);
#pragma unroll
      for (int i = 0; i < VEC; ++i) acc += exp2f((e[i] - mg) * XLOG2E);
    }
    acc = warp_sum(acc);
    if (lane == 0) red_s[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < 8; ++w) t += red_s[w];
      st[1] = t;
      st[2] = (tgt >= 0 && tgt < V_local) ? to_f(x[tgt]) : 0.f;
    }
    return;
  }
  // stage 2 (or 3): loss + gradient, in place over the logits
  if (stage == 2) {
    m = st[0];
    sum = st[1];
  }
  const bool ign = lab == ignore;
  if (threadIdx.x == 0) loss[row] = ign ? 0.f : (logf(sum) + m - st[2]);
  T* d = dl + row * V_local;
  const float scale = ign ? 0.f : gscale / sum;
  for (int v = threadIdx.x; v < nvec; v += 256) {
    float e[VEC];
    load16(x + (int64_t)v * VEC, e);
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      e[i] = exp2f((e[i] - m) * XLOG2E) * scale;
      if (!ign && (int64_t)v * VEC + i == tgt) e[i] -= gscale;
    }
    store16(d + (int64_t)v * VEC, e);
  }
}

}  // namespace xent
}  // namespace galv

using namespace galv;

extern "C" {

int32_t galv_embed_fwd(const int64_t* ids, const void* table, void* out, int64_t T_,
                       int64_t V_local, int64_t vocab_lo, int64_t Hd, int32_t dtype,
                       void* stream) {
  GALV_CHECK_ARG(ids && table && out && T_ > 0 && Hd % 8 == 0, "bad arguments");
  GALV_DISPATCH(dtype, T, {
    emb::embed_fwd<T><<<(unsigned)T_, 128, 0, as_stream(stream)>>>(ids, (const T*)table, (T*)out,
                                                                  T_, V_local, vocab_lo, Hd);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_embed_bwd(const int64_t* ids, const void* dout, float* dtable, int64_t T_,
                       int64_t V_local, int64_t vocab_lo, int64_t Hd, int32_t dtype,
                       void* stream) {
  GALV_CHECK_ARG(ids && dout && dtable && T_ > 0, "bad arguments");
  GALV_DISPATCH(dtype, T, {
    emb::embed_bwd<T><<<(unsigned)T_, 256, 0, as_stream(stream)>>>(ids, (const T*)dout, dtable,
                                                                  T_, V_local, vocab_lo, Hd);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_embed_bwd_sorted(const int64_t* sorted_ids, const int64_t* order, const void* dout,
                              void* grad, int64_t T_, int64_t V_local, int64_t vocab_lo,
                              int64_t Hd, int32_t dtype, int32_t grad_dtype, void* stream) {
  GALV_CHECK_ARG(sorted_ids && order && dout && grad && T_ > 0 && Hd % 8 == 0, "bad arguments");
  GALV_CHECK_ARG((reinterpret_cast<uintptr_t>(dout) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(grad) & 15) == 0,
                 "dout and grad must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  GALV_DISPATCH(dtype, T, {
    if (grad_dtype == GALV_BF16)
      emb::embed_bwd_sorted<T, __nv_bfloat16><<<(unsigned)T_, 256, 0, s>>>(
          sorted_ids, order, (const T*)dout, (__nv_bfloat16*)grad, T_, V_local, vocab_lo, Hd);
    else if (grad_dtype == GALV_F32)
      emb::embed_bwd_sorted<T, float><<<(unsigned)T_, 256, 0, s>>>(
          sorted_ids, order, (const T*)dout, (float*)grad, T_, V_local, vocab_lo, Hd);
    else
      GALV_CHECK_ARG(false, "grad dtype must be bf16 or f32");
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_xent(void* logits, const int64_t* labels, float* stats, float* loss, void* dlogits,
                  int64_t T_, int64_t V_local, int64_t vocab_lo, float grad_scale,
                  int64_t ignore_index, int32_t stage, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(logits && labels && stats && T_ > 0 && V_local > 0, "bad arguments");
  GALV_CHECK_ARG(stage >= 0 && stage <= 3, "stage must be 0..3");
  GALV_CHECK_ARG(stage < 2 || (loss && dlogits), "stage 2/3 need loss and dlogits");
  GALV_DISPATCH(dtype, T, {
    const bool vec = (V_local * (int64_t)sizeof(T)) % 16 == 0 &&
                     (reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
                     (dlogits == nullptr || (reinterpret_cast<uintptr_t>(dlogits) & 15) == 0);
    if (vec)
      xent::xent_vec<T><<<(unsigned)T_, 256, 0, as_stream(stream)>>>(
          (T*)logits, labels, stats, loss, (T*)dlogits, V_local, vocab_lo, grad_scale,
          ignore_index, stage);
    else
      xent::xent_kernel<T><<<(unsigned)T_, 256, 0, as_stream(stream)>>>(
          (T*)logits, labels, stats, loss, (T*)dlogits, V_local, vocab_lo, grad_scale,
          ignore_index, stage);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
