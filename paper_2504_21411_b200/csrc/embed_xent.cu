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
