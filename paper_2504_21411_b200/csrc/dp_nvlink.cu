// Data-parallel collectives over NVLink / NVSwitch for the ZeRO gradient and parameter
// buffers (costmodel.py:199-213 dp_sync: z0 all-reduce, z>=1 reduce-scatter + all-gather).
//
// Every dp rank's flat grad / param buffers live in one symmetric allocation, mapped into
// all peers and (when the fabric supports it) bound to an NVSwitch multicast object:
//   * reduce-scatter = each rank pulls ITS chunk summed over all ranks with
//     multimem.ld_reduce (the switch adds the dp copies; every byte crosses NVLink once)
//     and accumulates it into its shard in the same pass (ZeRO-2 microbatch accumulation);
//   * all-reduce (z0) = the same pull, then multimem.st of the reduced chunk to all ranks;
//   * parameter all-gather (z1/z2) is fused into AdamW: the updated bf16 parameters are
//     stored once to the multicast address and the switch replicates them into every
//     rank's full parameter buffer -- no separate gather pass, no staging copy.
// Without multicast the same kernels use unicast NVLink loads/stores to each peer pointer.
// Synchronisation: monotonic per-source epochs in a flag area of the symmetric buffer
// (st.release.sys / ld.acquire.sys, tp_nvlink.cu); the waits are single-CTA kernels.
#include "common.cuh"

namespace galv {
namespace dpl {

__device__ __forceinline__ void mc_st16(void* addr, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// 8 bf16 summed over every rank of the multicast group (fp32 accumulation in the switch)
__device__ __forceinline__ uint4 mc_ld_reduce_bf16x8(const void* addr) {
  uint4 v;
  asm volatile(
      "multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(addr)
      : "memory");
  return v;
}

__device__ __forceinline__ void bf16x8_to_f(const uint4 raw, float* f) {
  const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(e[i]);
}
__device__ __forceinline__ uint4 f_to_bf16x8(const float* f) {
  uint4 raw;
  __nv_bfloat16* e = reinterpret_cast<__nv_bfloat16*>(&raw);
#pragma unroll
  for (int i = 0; i < 8; ++i) e[i] = __float2bfloat16_rn(f[i]);
  return raw;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// flag_ptrs[r] = rank r's flag array (uint32 per source rank)
__global__ void signal_kernel(void* const* flag_ptrs, int me, int t, uint32_t epoch) {
  if (threadIdx.x < (unsigned)t) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint32_t*>(flag_ptrs[threadIdx.x]) + me, epoch);
  }
}
__global__ void wait_kernel(const uint32_t* my_flags, int t, uint32_t epoch) {
  if (threadIdx.x < (unsigned)t) {
    while ((int)(ld_acquire_sys(my_flags + threadIdx.x) - epoch) < 0) {
    }
  }
  __syncthreads();
}

// out[i] (+)= sum over ranks of src[i], i over this rank's chunk (8 bf16 per vector).
// mc_src: multicast address of the chunk, or null -> unicast loads from peer_src[r] + off.
// bcast: also store the reduced chunk to every rank (multicast or peer_dst[r] + off).
// U vectors per thread are loaded before any is consumed, so a small grid keeps enough
// NVLink round trips in flight (the kernel runs next to the backward GEMMs and should
// occupy as few SMs as possible).
constexpr int RU = 4;

__device__ __forceinline__ void reduce_store(uint4 raw_sum, float* extra, int64_t i, uint4* out,
                                             int accumulate, uint4* mc_dst,
                                             void* const* peer_dst, int t, int64_t off16) {
  float acc[8];
  bf16x8_to_f(raw_sum, acc);
  if (extra) {
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = extra[e];
  }
  if (accumulate) {
    float v[8];
    bf16x8_to_f(out[i], v);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += v[e];
  }
  const uint4 res = f_to_bf16x8(acc);
  if (out) out[i] = res;
  if (mc_dst) {
    mc_st16(mc_dst + i, res);
  } else if (peer_dst) {
    for (int r = 0; r < t; ++r) reinterpret_cast<uint4*>(peer_dst[r])[off16 + i] = res;
  }
}

__global__ void __launch_bounds__(512) reduce_chunk(const uint4* mc_src, void* const* peer_src,
                                                    int t, int64_t off16, uint4* out,
                                                    int accumulate, uint4* mc_dst,
                                                    void* const* peer_dst, int64_t n8) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (mc_src) {
    // RU independent multimem loads in flight per thread
    for (; base + (RU - 1) * stride < n8; base += stride * RU) {
      uint4 raw[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) raw[u] = mc_ld_reduce_bf16x8(mc_src + base + u * stride);
#pragma unroll
      for (int u = 0; u < RU; ++u)
        reduce_store(raw[u], nullptr, base + u * stride, out, accumulate, mc_dst, peer_dst, t,
                     off16);
    }
    for (; base < n8; base += stride)
      reduce_store(mc_ld_reduce_bf16x8(mc_src + base), nullptr, base, out, accumulate, mc_dst,
                   peer_dst, t, off16);
    return;
  }
  for (; base < n8; base += stride) {  // unicast: sum the peers' copies over NVLink
    float acc[8], v[8];
    bf16x8_to_f(reinterpret_cast<const uint4*>(peer_src[0])[off16 + base], acc);
    for (int r = 1; r < t; ++r) {
      bf16x8_to_f(reinterpret_cast<const uint4*>(peer_src[r])[off16 + base], v);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
    }
    reduce_store(make_uint4(0, 0, 0, 0), acc, base, out, accumulate, mc_dst, peer_dst, t, off16);
  }
}

// AdamW over this rank's fp32 master shard, 8 params per step; the bf16 parameters go to
// every rank's full parameter buffer at the same offset (multicast or unicast peer stores).
template <typename TG>
__global__ void __launch_bounds__(256) adamw_bcast(float* __restrict__ master,
                                                   float* __restrict__ m, float* __restrict__ v,
                                                   const TG* __restrict__ g, uint4* mc_dst,
                                                   void* const* peer_dst, int t, int64_t off16,
                                                   int64_t n8, float lr, float b1, float b2,
                                                   float eps, float wd, float gscale, float bc1,
                                                   float bc2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    float p[8], mm[8], vv[8], gr[8];
    *reinterpret_cast<float4*>(p) = reinterpret_cast<float4*>(master)[2 * i];
    *reinterpret_cast<float4*>(p + 4) = reinterpret_cast<float4*>(master)[2 * i + 1];
    *reinterpret_cast<float4*>(mm) = reinterpret_cast<float4*>(m)[2 * i];
    *reinterpret_cast<float4*>(mm + 4) = reinterpret_cast<float4*>(m)[2 * i + 1];
    *reinterpret_cast<float4*>(vv) = reinterpret_cast<float4*>(v)[2 * i];
    *reinterpret_cast<float4*>(vv + 4) = reinterpret_cast<float4*>(v)[2 * i + 1];
    load16(g + i * 8, gr);
    if (sizeof(TG) == 4) load16(g + i * 8 + 4, gr + 4);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float gk = gr[k] * gscale;
      mm[k] = b1 * mm[k] + (1.f - b1) * gk;
      vv[k] = b2 * vv[k] + (1.f - b2) * gk * gk;
      p[k] = p[k] - lr * ((mm[k] / bc1) / (sqrtf(vv[k] / bc2) + eps) + wd * p[k]);
    }
    reinterpret_cast<float4*>(master)[2 * i] = *reinterpret_cast<float4*>(p);
    reinterpret_cast<float4*>(master)[2 * i + 1] = *reinterpret_cast<float4*>(p + 4);
    reinterpret_cast<float4*>(m)[2 * i] = *reinterpret_cast<float4*>(mm);
    reinterpret_cast<float4*>(m)[2 * i + 1] = *reinterpret_cast<float4*>(mm + 4);
    reinterpret_cast<float4*>(v)[2 * i] = *reinterpret_cast<float4*>(vv);
    reinterpret_cast<float4*>(v)[2 * i + 1] = *reinterpret_cast<float4*>(vv + 4);
    const uint4 res = f_to_bf16x8(p);
    if (mc_dst) {
      mc_st16(mc_dst + i, res);
    } else {
      for (int r = 0; r < t; ++r) reinterpret_cast<uint4*>(peer_dst[r])[off16 + i] = res;
    }
  }
}

inline unsigned grid_for(int64_t n, int threads, int per_sm) {
  return (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)sm_count() * per_sm));
}

}  // namespace dpl
}  // namespace galv

using namespace galv;

extern "C" {

int32_t galv_nvl_signal(void* const* flag_ptrs, int32_t me, int32_t t, uint32_t epoch,
                        void* stream) {
  GALV_CHECK_ARG(flag_ptrs && t >= 1 && t <= 32 && me >= 0 && me < t, "bad arguments");
  dpl::signal_kernel<<<1, 32, 0, as_stream(stream)>>>(flag_ptrs, me, t, epoch);
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_nvl_wait(const uint32_t* my_flags, int32_t t, uint32_t epoch, void* stream) {
  GALV_CHECK_ARG(my_flags && t >= 1 && t <= 32, "bad arguments");
  dpl::wait_kernel<<<1, 32, 0, as_stream(stream)>>>(my_flags, t, epoch);
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_dp_reduce(const void* mc_src, void* const* peer_src, int32_t t, int64_t offset,
                       void* out, int32_t accumulate, void* mc_dst, void* const* peer_dst,
                       int64_t n, int32_t max_ctas, void* stream) {
  GALV_CHECK_ARG((mc_src || peer_src) && t >= 1 && t <= 32 && n % 8 == 0 && offset % 8 == 0 &&
                     (out || mc_dst || peer_dst) && !(accumulate && !out),
                 "bad arguments");
  if (n == 0) return 0;
  const int64_t n8 = n / 8;
  unsigned grid = dpl::grid_for(n8, 512, 2);
  if (max_ctas > 0) grid = std::min<unsigned>(grid, (unsigned)max_ctas);
  dpl::reduce_chunk<<<grid, 512, 0, as_stream(stream)>>>(
      (const uint4*)mc_src, peer_src, t, offset / 8, (uint4*)out, accumulate, (uint4*)mc_dst,
      peer_dst, n8);
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_adamw_bcast(float* master, float* m, float* v, const void* grad, void* mc_dst,
                         void* const* peer_dst, int32_t t, int64_t offset, int64_t n, float lr,
                         float beta1, float beta2, float eps, float weight_decay,
                         float grad_scale, int64_t step, int32_t grad_dtype, void* stream) {
  GALV_CHECK_ARG(master && m && v && grad && (mc_dst || peer_dst) && n % 8 == 0 &&
                     offset % 8 == 0 && step >= 1 && t >= 1 && t <= 32,
                 "bad arguments");
  if (n == 0) return 0;
  const float bc1 = 1.f - powf(beta1, (float)step), bc2 = 1.f - powf(beta2, (float)step);
  const int64_t n8 = n / 8;
  const unsigned grid = dpl::grid_for(n8, 256, 8);
  GALV_DISPATCH(grad_dtype, TG, {
    dpl::adamw_bcast<TG><<<grid, 256, 0, as_stream(stream)>>>(
        master, m, v, (const TG*)grad, (uint4*)mc_dst, peer_dst, t, offset / 8, n8, lr, beta1,
        beta2, eps, weight_decay, grad_scale, bc1, bc2);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
