// Tensor-parallel collectives over NVLink peer memory (symmetric buffers mapped into every
// rank of the tp group):
//   * reduce-scatter fused into the row-parallel GEMM: the GEMM epilogue (gemm_sm100.cu,
//     galv_gemm_rs) stores each output row straight into the owning rank's receive slot,
//     so the NVLink transfer overlaps the tensor-core work tile by tile; this file then
//     signals arrival and sums the tp slots (fp32 accumulate) into the local chunk;
//   * all-gather by direct peer stores (every rank writes its chunk into all peers).
// Flags: one uint32 per source rank in each rank's flag area; epochs increase monotonically
// (release.sys stores after a system fence, acquire.sys polling).
#include "common.cuh"

namespace galv {
namespace tpl {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// signal every peer that this rank's stores for `epoch` are complete, then wait for all
__device__ __forceinline__ void signal_and_wait(void* const* flag_ptrs, int me, int t,
                                                uint32_t epoch) {
  if (blockIdx.x == 0 && threadIdx.x < (unsigned)t) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint32_t*>(flag_ptrs[threadIdx.x]) + me, epoch);
  }
  if (threadIdx.x < (unsigned)t) {
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(flag_ptrs[me]) + threadIdx.x;
    while ((int)(ld_acquire_sys(mine) - epoch) < 0) {
    }
  }
  __syncthreads();
}

// out[n] = sum_s recv[s][n]; launched after signal_wait_kernel on the same stream.  The
// wait is a single spinning CTA so NCCL kernels on other streams (dp collectives launched by
// the optimizer / ZeRO overlap) can always get SMs -- a full-grid spin could starve them.
template <typename T>
__global__ void __launch_bounds__(256) slot_reduce(int t, const T* __restrict__ recv,
                                                   T* __restrict__ out, int64_t n) {
  constexpr int V = 16 / sizeof(T);
  const int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc[V], v[V];
    load16(recv + i * V, acc);
    for (int s = 1; s < t; ++s) {
      load16(recv + s * n + i * V, v);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] += v[e];
    }
    store16(out + i * V, acc);
  }
}

// every rank copies its chunk (n_bytes) into slot `me` of every peer's gather buffer
__global__ void __launch_bounds__(256) peer_copy(const uint4* __restrict__ src,
                                                 void* const* dst_ptrs, int me, int t,
                                                 int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    for (int r = 0; r < t; ++r) reinterpret_cast<uint4*>(dst_ptrs[r])[me * n16 + i] = v;
  }
}

__global__ void signal_wait_kernel(void* const* flag_ptrs, int me, int t, uint32_t epoch) {
  signal_and_wait(flag_ptrs, me, t, epoch);
}

}  // namespace tpl
}  // namespace galv

using namespace galv;

extern "C" {

int32_t galv_tp_signal_reduce(void* const* flag_ptrs, int32_t me, int32_t t, uint32_t epoch,
                              const void* recv, void* out, int64_t n, int32_t dtype,
                              void* stream) {
  GALV_CHECK_ARG(flag_ptrs && recv && out && t >= 1 && t <= 32 && n % 8 == 0, "bad arguments");
  tpl::signal_wait_kernel<<<1, 32, 0, as_stream(stream)>>>(flag_ptrs, me, t, epoch);
  GALV_LAUNCH_CHECK();
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((n / 8 + 255) / 256, sm_count()));
  GALV_DISPATCH(dtype, T, {
    tpl::slot_reduce<T><<<grid, 256, 0, as_stream(stream)>>>(t, (const T*)recv, (T*)out, n);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

int32_t galv_tp_allgather(const void* src, void* const* dst_ptrs, void* const* flag_ptrs,
                          int32_t me, int32_t t, uint32_t epoch, int64_t bytes, void* stream) {
  GALV_CHECK_ARG(src && dst_ptrs && flag_ptrs && bytes % 16 == 0, "bad arguments");
  const int64_t n16 = bytes / 16;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256,
                                                                         sm_count()));
  tpl::peer_copy<<<grid, 256, 0, as_stream(stream)>>>((const uint4*)src, dst_ptrs, me, t, n16);
  GALV_LAUNCH_CHECK();
  tpl::signal_wait_kernel<<<1, 32, 0, as_stream(stream)>>>(flag_ptrs, me, t, epoch);
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
