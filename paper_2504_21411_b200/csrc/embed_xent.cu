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
    xent::xent_kernel<T><<<(unsigned)T_, 256, 0, as_stream(stream)>>>(
        (T*)logits, labels, stats, loss, (T*)dlogits, V_local, vocab_lo, grad_scale, ignore_index,
        stage);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
