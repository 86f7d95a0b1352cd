// tcgen05 bf16 GEMM for sm_100a: TMA -> 128B-swizzled smem ring -> UMMA (M=128, N=256,
// K=16 per instruction) -> double-buffered TMEM accumulators -> epilogue warps.
//
// Persistent kernel, one CTA per SM, warp-specialized:
//   warp 0 : TMA producer (one elected lane)
//   warp 1 : MMA issuer  (one elected lane)
//   warp 2 : TMEM allocator (512 columns = 2 x 256 fp32 accumulators)
//   warps 4-7 : epilogue (TMEM lane quarter w%4 -> rows), fused alpha/bias/accumulate
// Operands may be K-major or MN-major independently (idesc bits 15/16), which covers
// forward (X W^T), dgrad (dY W) and wgrad (dY^T X) without transposes.
#include <cuda.h>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace galv {
namespace tc {
using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;          // 16 KB
constexpr int B_STAGE = BN * BK * 2;          // 32 KB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int GROUP_M = 8;  // raster group (256-row pair tiles); sustained sweep: 8 >= 16 > 4 > 32

struct Params {
  int M, N, K;
  int a_mn, b_mn;
  void* C;
  long long ldc;
  int c_bf16;
  const void* bias;
  int bias_bf16;
  float alpha;
  int accumulate;
  int tiles_m, tiles_n, num_tiles, k_blocks;
  // fused reduce-scatter epilogue over NVLink peer memory (tensor-parallel row GEMMs):
  // row r goes to rank j = r / rows_per_rank, slot `my_slot`, of that rank's receive buffer
  void* const* peer_c;
  int rows_per_rank, my_slot;
  // tile raster: groups of `group` tiles along M (gdim 0) or N (gdim 1); L2 cache hints
  int group, gdim, hint;
  // fused SwiGLU epilogues (Llama MLP): 1 = backward (C = d(gate|up) from dh = acc, aux =
  // saved gate|up), 2 = forward (pair tile = 128 gate + 128 up columns; C = gate|up,
  // aux = h = silu(gate) * up); ff = F (gate/up split), aux_ld its leading dim
  int epi, ff;
  const void* aux;
  long long aux_ld;
  // split-K (2-CTA path): work unit u = tile (u % num_tiles) x K-split (u / num_tiles), each
  // split covering kb_per k-blocks; partial fp32 tiles go to ws[split][M][N]
  int splits, kb_per, num_units;
  float* ws;
};

__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mt, int& nt) {
  if (p.gdim == 0) {
    const int per_group = p.group * p.tiles_n;
    const int group = t / per_group;
    const int first_m = group * p.group;
    const int gm = min(p.tiles_m - first_m, p.group);
    const int r = t - group * per_group;
    mt = first_m + r % gm;
    nt = r / gm;
  } else {
    const int per_group = p.group * p.tiles_m;
    const int group = t / per_group;
    const int first_n = group * p.group;
    const int gn = min(p.tiles_n - first_n, p.group);
    const int r = t - group * per_group;
    nt = first_n + r % gn;
    mt = r / gn;
  }
}

// Epilogue of one 128-lane accumulator slice: this thread owns output row `row` and
// the BN columns starting at `col_base`; alpha, bias and accumulate-into-C fused.
__device__ __forceinline__ void epilogue_tile(const Params& p, uint32_t taddr, int row,
                                              int col_base, bool vec_ok) {
  const bool row_ok = row < p.M;
  char* cbase = reinterpret_cast<char*>(p.C);
  long long row_off = (long long)row * p.ldc;
  if (p.peer_c != nullptr && row_ok) {  // store straight into the owning rank's buffer
    const int j = row / p.rows_per_rank;
    cbase = reinterpret_cast<char*>(p.peer_c[j]);
    row_off = (long long)(p.my_slot * p.rows_per_rank + (row - j * p.rows_per_rank)) * p.ldc;
  }
#pragma unroll 1
  for (int cc = 0; cc < BN; cc += 32) {
    uint32_t r[32];
    tmem_ld32(taddr + cc, r);
    const int col0 = col_base + cc;
    if (!row_ok || col0 >= p.N) continue;
        float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
    const int ncol = min(32, p.N - col0);
    if (p.bias) {
      for (int i = 0; i < ncol; ++i)
        v[i] += p.bias_bf16 ? __bfloat162float(
                                  reinterpret_cast<const __nv_bfloat16*>(p.bias)[col0 + i])
                            : reinterpret_cast<const float*>(p.bias)[col0 + i];
    }
    const long long off = row_off + col0;
    if (p.c_bf16) {
      __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(cbase) + off;
      if (ncol == 32 && vec_ok) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float tmp[8];
          if (p.accumulate) load16(c + j * 8, tmp);
#pragma unroll
          for (int e = 0; e < 8; ++e) tmp[e] = p.accumulate ? tmp[e] + v[j * 8 + e] : v[j * 8 + e];
          store16(c + j * 8, tmp);
        }
      } else {
        for (int i = 0; i < ncol; ++i) {
          float o = v[i];
          if (p.accumulate) o += __bfloat162float(c[i]);
          c[i] = __float2bfloat16_rn(o);
        }
      }
    } else {
      float* c = reinterpret_cast<float*>(cbase) + off;
      if (ncol == 32 && (p.ldc % 4) == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o = make_float4(v[j * 4], v[j * 4 + 1], v[j * 4 + 2], v[j * 4 + 3]);
          if (p.accumulate) {
            float4 old = *reinterpret_cast<const float4*>(c + j * 4);
            o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
          }
          *reinterpret_cast<float4*>(c + j * 4) = o;
        }
      } else {
        for (int i = 0; i < ncol; ++i) c[i] = p.accumulate ? c[i] + v[i] : v[i];
      }
    }
  }
}

__global__ void __launch_bounds__(256, 1)
    gemm_bf16_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared window
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    prefetch_map(&tmA);
    prefetch_map(&tmB);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mt, nt;
        tile_coords(p, t, mt, nt);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          uint8_t* a_dst = sA + stage * A_STAGE;
          uint8_t* b_dst = sB + stage * B_STAGE;
          if (!p.a_mn) {
            tma_load_2d(&tmA, &full[stage], a_dst, kb * BK, mt * BM);
          } else {
#pragma unroll
            for (int g = 0; g < BM / 64; ++g)
              tma_load_2d(&tmA, &full[stage], a_dst + g * 8192, mt * BM + g * 64, kb * BK);
          }
          if (!p.b_mn) {
            tma_load_2d(&tmB, &full[stage], b_dst, kb * BK, nt * BN);
          } else {
#pragma unroll
            for (int g = 0; g < BN / 64; ++g)
              tma_load_2d(&tmB, &full[stage], b_dst + g * 8192, nt * BN + g * 64, kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(BM, BN, p.a_mn, p.b_mn);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_STAGE);
          const uint32_t b_base = smem_u32(sB + stage * B_STAGE);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = p.a_mn ? sdesc(a_base + k * 2048, 8192, 1024)
                                       : sdesc(a_base + k * 32, 16, 1024);
            const uint64_t bd = p.b_mn ? sdesc(b_base + k * 2048, 8192, 1024)
                                       : sdesc(b_base + k * 32, 16, 1024);
            umma_bf16(d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool vec_ok = (p.ldc % 8) == 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int mt, nt;
      tile_coords(p, t, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      epilogue_tile(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16), mt * BM + q * 32 + lane,
                    nt * BN, vec_ok);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}


// ---------------------------------------------------------------- 2-CTA variant
// CTA pair (cluster of 2 on one TPC) computes a 256x256 tile with tcgen05.mma.cta_group::2:
// each CTA stages its 128 rows of A and 128 rows (N) of B, so per-SM shared-memory
// operand traffic is halved relative to the 1-CTA 128x256 kernel.  Only the leader CTA
// issues MMAs; TMA bytes of both CTAs complete on the leader's `full` barriers; MMA
// completion is multicast to both CTAs' `empty` / `tfull` barriers; both CTAs' epilogues
// release the accumulator by arriving remotely on the leader's `tempty` barrier.
constexpr int HALF_STAGE = 128 * BK * 2;  // 16 KB: 128 rows of A (or of B)
template <bool PEER> struct Cfg2 {
  // 5 pipeline stages + an epilogue staging area so every output store leaves the SM as a
  // full row segment: plain = 32 rows x 64 fp32 columns per warp (128/256-byte segments,
  // read-modify-write capable); PEER = 32 rows x 128 bf16 columns (256-byte NVLink stores)
  static constexpr int STAGES = 5;
  static constexpr int STAGE_PITCH = PEER ? 128 * 2 + 16 : 64 * 4 + 16;
  static constexpr int STAGING = 4 * 32 * STAGE_PITCH;
  static constexpr int SMEM = STAGES * 2 * HALF_STAGE + STAGING + 1024 + 256;
};

// fused reduce-scatter epilogue: rows -> bf16 -> smem -> 256-byte stores into the owning
// rank's receive buffer (two 128-column halves per 256-column tile)
__device__ __forceinline__ void epilogue_peer(const Params& p, uint32_t taddr, int row0,
                                              int col_base, uint8_t* stage) {
  constexpr int PITCH = Cfg2<true>::STAGE_PITCH;
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
#pragma unroll 1
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t r[32];
      tmem_ld32(taddr + half * 128 + cc * 32, r);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(r[2 * i]) * p.alpha,
                                                 __uint_as_float(r[2 * i + 1]) * p.alpha);
        pk[i] = *reinterpret_cast<uint32_t*>(&v);
      }
      uint4* dst = reinterpret_cast<uint4*>(stage + lane * PITCH + cc * 64);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        dst[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
    }
    __syncwarp();
    const int col0 = col_base + half * 128;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {  // 32 rows x 16 chunks of 16 B
      const int c = i * 32 + lane, rr = c >> 4, part = c & 15;
      const int row = row0 + rr, col = col0 + part * 8;
      if (row < p.M && col < p.N) {
        const int j = row / p.rows_per_rank;
        __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(p.peer_c[j]);
        const long long off =
            (long long)(p.my_slot * p.rows_per_rank + (row - j * p.rows_per_rank)) * p.ldc + col;
        *reinterpret_cast<uint4*>(base + off) =
            *reinterpret_cast<const uint4*>(stage + rr * PITCH + part * 16);
      }
    }
    __syncwarp();
  }
}

// Staged epilogue: a warp's 32 rows x 256 columns go TMEM -> (alpha, bias) fp32 -> smem ->
// coalesced row-segment stores (+ read-modify-write when accumulating).  With PEER the
// destination row lives in rank row / rows_per_rank's receive buffer (fused NVLink RS).
template <bool PEER>
__device__ __forceinline__ void epilogue_staged(const Params& p, uint32_t taddr, int row0,
                                                int col_base, uint8_t* stage) {
  constexpr int PITCH = Cfg2<PEER>::STAGE_PITCH;
  const int lane = threadIdx.x & 31;
  const uint64_t st_pol = l2_evict_first();
#pragma unroll 1
  for (int q4 = 0; q4 < 4; ++q4) {
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      uint32_t r[32];
      tmem_ld32(taddr + q4 * 64 + cc * 32, r);
      const int c0 = col_base + q4 * 64 + cc * 32;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
      if (p.bias != nullptr) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int c = min(c0 + i, p.N - 1);
          v[i] += p.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.bias)[c])
                              : reinterpret_cast<const float*>(p.bias)[c];
        }
      }
      float4* dst = reinterpret_cast<float4*>(stage + lane * PITCH + cc * 128);
#pragma unroll
      for (int u = 0; u < 8; ++u) dst[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    }
    __syncwarp();
    const int colq = col_base + q4 * 64;
    if (p.c_bf16) {
#pragma unroll 2
      for (int it = 0; it < 8; ++it) {  // 32 rows x 8 units of 8 bf16
        const int u = it * 32 + lane, rr = u >> 3, part = u & 7;
        const int row = row0 + rr, col = colq + part * 8;
        if (row < p.M && col < p.N) {
          __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(p.C);
          long long off = (long long)row * p.ldc + col;
          if (PEER) {
            const int j = row / p.rows_per_rank;
            base = reinterpret_cast<__nv_bfloat16*>(p.peer_c[j]);
            off = (long long)(p.my_slot * p.rows_per_rank + (row - j * p.rows_per_rank)) * p.ldc +
                  col;
          }
          const float4* src = reinterpret_cast<const float4*>(stage + rr * PITCH + part * 32);
          float4 a = src[0], b = src[1];
          float o[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
          if (p.accumulate) {
            float old[8];
            load16(base + off, old);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] += old[e];
          }
          if (p.hint & 2) {
            uint4 raw;
            __nv_bfloat16* e8 = reinterpret_cast<__nv_bfloat16*>(&raw);
#pragma unroll
            for (int e = 0; e < 8; ++e) e8[e] = __float2bfloat16_rn(o[e]);
            st_global_hint(base + off, raw, st_pol);
          } else {
            store16(base + off, o);
          }
        }
      }
    } else {
#pragma unroll 2
      for (int it = 0; it < 16; ++it) {  // 32 rows x 16 units of 4 fp32
        const int u = it * 32 + lane, rr = u >> 4, part = u & 15;
        const int row = row0 + rr, col = colq + part * 4;
        if (row < p.M && col < p.N) {
          float* base = reinterpret_cast<float*>(p.C);
          long long off = (long long)row * p.ldc + col;
          if (PEER) {
            const int j = row / p.rows_per_rank;
            base = reinterpret_cast<float*>(p.peer_c[j]);
            off = (long long)(p.my_slot * p.rows_per_rank + (row - j * p.rows_per_rank)) * p.ldc +
                  col;
          }
          float4 o = *reinterpret_cast<const float4*>(stage + rr * PITCH + part * 16);
          if (p.accumulate) {
            const float4 old = *reinterpret_cast<const float4*>(base + off);
            o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
          }
          *reinterpret_cast<float4*>(base + off) = o;
        }
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {  // bf16x2, round to nearest
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 bf2_to_f2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
// sigmoid on MUFU (ex2 + rcp): the fused epilogues must keep pace with the MMA mainloop;
// saturates cleanly (x -> -inf gives 0) without the IEEE-division slow path
__device__ __forceinline__ float fast_sigmoid(float x) {
  return __fdividef(1.f, 1.f + __expf(-x));
}

// Fused SwiGLU epilogues.  A warp owns 32 rows; global traffic goes through the warp's
// smem staging rows (PITCH bytes each) so every load/store is a coalesced row segment.
constexpr int SW_PITCH = Cfg2<false>::STAGE_PITCH;  // 272 >= 2 x 128-byte halves + pad

// epi 1 (backward): 64-column chunks of dh (fp32 in TMEM, rounded to bf16 as the unfused
// dgrad would store it); gate/up row segments are loaded coalesced into smem, each lane
// turns its row into d(gate)/d(up) in place, then the chunk is stored coalesced.
__device__ __forceinline__ void epilogue_swiglu_bwd(const Params& p, uint32_t taddr, int row0,
                                                    int col_base, uint8_t* stage) {
  const int lane = threadIdx.x & 31;
  const __nv_bfloat16* gu = reinterpret_cast<const __nv_bfloat16*>(p.aux);
  __nv_bfloat16* dgu = reinterpret_cast<__nv_bfloat16*>(p.C);
#pragma unroll 1
  for (int q4 = 0; q4 < 4; ++q4) {
    const int colq = col_base + q4 * 64;
    // coalesced loads: 32 rows x (gate 8 units | up 8 units) of 16 bytes
    uint4 ld[16];
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int u = it * 32 + lane, rr = u >> 4, part = u & 15;
      const int row = row0 + rr, col = colq + (part & 7) * 8;
      ld[it] = make_uint4(0, 0, 0, 0);
      if (row < p.M && col < p.N)
        ld[it] = *reinterpret_cast<const uint4*>(gu + (long long)row * p.aux_ld +
                                                 (part >> 3) * p.ff + col);
    }
    uint32_t r[64];
    tmem_ld32(taddr + q4 * 64, r);
    tmem_ld32(taddr + q4 * 64 + 32, r + 32);
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int u = it * 32 + lane, rr = u >> 4, part = u & 15;
      *reinterpret_cast<uint4*>(stage + rr * SW_PITCH + part * 16) = ld[it];
    }
    __syncwarp();
    // this lane's row: gate at bytes [0,128), up at [128,256)
    __nv_bfloat16* srow = reinterpret_cast<__nv_bfloat16*>(stage + lane * SW_PITCH);
#pragma unroll
    for (int c = 0; c < 64; c += 8) {
      uint4 graw = *reinterpret_cast<const uint4*>(srow + c);
      uint4 uraw = *reinterpret_cast<const uint4*>(srow + 64 + c);
      const uint32_t* gw = reinterpret_cast<const uint32_t*>(&graw);
      const uint32_t* uw = reinterpret_cast<const uint32_t*>(&uraw);
      uint32_t dgw[4], duw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 g = bf2_to_f2(gw[e]), u = bf2_to_f2(uw[e]);
        const float2 d = bf2_to_f2(pack2(__uint_as_float(r[c + 2 * e]), __uint_as_float(r[c + 2 * e + 1])));
        const float s0 = fast_sigmoid(g.x), s1 = fast_sigmoid(g.y);
        duw[e] = pack2(d.x * g.x * s0, d.y * g.y * s1);
        dgw[e] = pack2(d.x * u.x * s0 * (1.f + g.x * (1.f - s0)),
                       d.y * u.y * s1 * (1.f + g.y * (1.f - s1)));
      }
      *reinterpret_cast<uint4*>(srow + c) = make_uint4(dgw[0], dgw[1], dgw[2], dgw[3]);
      *reinterpret_cast<uint4*>(srow + 64 + c) = make_uint4(duw[0], duw[1], duw[2], duw[3]);
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int u = it * 32 + lane, rr = u >> 4, part = u & 15;
      const int row = row0 + rr, col = colq + (part & 7) * 8;
      if (row < p.M && col < p.N)
        *reinterpret_cast<uint4*>(dgu + (long long)row * p.ldc + (part >> 3) * p.ff + col) =
            *reinterpret_cast<const uint4*>(stage + rr * SW_PITCH + part * 16);
    }
    __syncwarp();
  }
}

// epi 2 (forward): accumulator columns [0,128) are gate columns [col_base, +128), [128,256)
// the matching up columns.  gate/up are rounded to bf16 (what the unfused GEMM stores) and
// h = silu(g) * u from the rounded values, as act::swiglu_fwd; per 32-column chunk the lane
// writes its row's gate | up | h (3 x 64 bytes) to smem, then the warp stores coalesced.
__device__ __forceinline__ void epilogue_swiglu_fwd(const Params& p, uint32_t taddr, int row0,
                                                    int col_base, uint8_t* stage) {
  const int lane = threadIdx.x & 31;
  __nv_bfloat16* gu = reinterpret_cast<__nv_bfloat16*>(p.C);
  __nv_bfloat16* hout = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(p.aux));
  __nv_bfloat16* srow = reinterpret_cast<__nv_bfloat16*>(stage + lane * SW_PITCH);
#pragma unroll 1
  for (int cc = 0; cc < 128; cc += 32) {
    uint32_t rg[32], ru[32];
    tmem_ld32(taddr + cc, rg);
    tmem_ld32(taddr + 128 + cc, ru);
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      uint32_t gw[4], uw[4], hw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        gw[e] = pack2(__uint_as_float(rg[c + 2 * e]), __uint_as_float(rg[c + 2 * e + 1]));
        uw[e] = pack2(__uint_as_float(ru[c + 2 * e]), __uint_as_float(ru[c + 2 * e + 1]));
        const float2 g = bf2_to_f2(gw[e]), u = bf2_to_f2(uw[e]);
        hw[e] = pack2(g.x * fast_sigmoid(g.x) * u.x, g.y * fast_sigmoid(g.y) * u.y);
      }
      *reinterpret_cast<uint4*>(srow + c) = make_uint4(gw[0], gw[1], gw[2], gw[3]);
      *reinterpret_cast<uint4*>(srow + 32 + c) = make_uint4(uw[0], uw[1], uw[2], uw[3]);
      *reinterpret_cast<uint4*>(srow + 64 + c) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    }
    __syncwarp();
    const int colq = col_base + cc;
#pragma unroll
    for (int it = 0; it < 12; ++it) {  // 32 rows x (gate 4 | up 4 | h 4) units of 16 bytes
      const int u = it * 32 + lane, rr = u / 12, part = u % 12, arr = part >> 2;
      const int row = row0 + rr, col = colq + (part & 3) * 8;
      if (row < p.M && col < p.ff) {
        __nv_bfloat16* dst = arr == 2 ? hout + (long long)row * p.aux_ld + col
                                      : gu + (long long)row * p.ldc + arr * p.ff + col;
        *reinterpret_cast<uint4*>(dst) =
            *reinterpret_cast<const uint4*>(stage + rr * SW_PITCH + part * 16);
      }
    }
    __syncwarp();
  }
}

// tanh-GeLU on MUFU (tanh.approx), as used by the GPT MLP epilogues
__device__ __forceinline__ float fast_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_fast(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + fast_tanh(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float th = fast_tanh(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + th) + 0.5f * x * (1.f - th * th) * k0 * (1.f + 3.f * k1 * x * x);
}
__device__ __forceinline__ float2 bias_pair(const Params& p, int col) {  // bias[col], [col+1]
  if (p.bias_bf16) return bf2_to_f2(*reinterpret_cast<const uint32_t*>(
                       reinterpret_cast<const __nv_bfloat16*>(p.bias) + col));
  return *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(p.bias) + col);
}

// epi 3 (GPT fc1 forward): C = pre = acc (bf16, what the unfused GEMM stores), aux = act =
// gelu(pre + bias); per 32-column chunk the lane stages its row's pre | act (2 x 64 B)
__device__ __forceinline__ void epilogue_bias_gelu_fwd(const Params& p, uint32_t taddr, int row0,
                                                       int col_base, uint8_t* stage) {
  const int lane = threadIdx.x & 31;
  __nv_bfloat16* pre = reinterpret_cast<__nv_bfloat16*>(p.C);
  __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(p.aux));
  __nv_bfloat16* srow = reinterpret_cast<__nv_bfloat16*>(stage + lane * SW_PITCH);
#pragma unroll 1
  for (int cc = 0; cc < BN; cc += 32) {
    const int colq = col_base + cc;
    if (colq >= p.N) break;
    uint32_t r[32];
    tmem_ld32(taddr + cc, r);
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      uint32_t pw[4], aw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        pw[e] = pack2(__uint_as_float(r[c + 2 * e]), __uint_as_float(r[c + 2 * e + 1]));
        const float2 x = bf2_to_f2(pw[e]);
        const int col = min(colq + c + 2 * e, p.N - 2);
        const float2 b = p.bias ? bias_pair(p, col) : make_float2(0.f, 0.f);
        aw[e] = pack2(gelu_fast(x.x + b.x), gelu_fast(x.y + b.y));
      }
      *reinterpret_cast<uint4*>(srow + c) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
      *reinterpret_cast<uint4*>(srow + 32 + c) = make_uint4(aw[0], aw[1], aw[2], aw[3]);
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 8; ++it) {  // 32 rows x (pre 4 | act 4) units of 16 bytes
      const int u = it * 32 + lane, rr = u >> 3, part = u & 7;
      const int row = row0 + rr, col = colq + (part & 3) * 8;
      if (row < p.M && col < p.N) {
        __nv_bfloat16* dst = (part >> 2) ? act + (long long)row * p.aux_ld + col
                                         : pre + (long long)row * p.ldc + col;
        *reinterpret_cast<uint4*>(dst) =
            *reinterpret_cast<const uint4*>(stage + rr * SW_PITCH + part * 16);
      }
    }
    __syncwarp();
  }
}

// epi 5 (Llama QKV forward): C = qkv = acc rounded to bf16 (what the plain GEMM stores),
// then RoPE rotate-half on columns < ff (the q | k heads, head_dim 128) in fp32 with the
// cos/sin table aux = [2][S][64] (S = aux_ld, position = row % S), exactly the arithmetic of
// galv_rope_table on the stored values; v columns pass through.  Per head (128 columns of
// the 256-column tile) and 32-column quarter: the lane's row pairs columns j and j + 64.
__device__ __forceinline__ void epilogue_rope_qkv(const Params& p, uint32_t taddr, int row0,
                                                  int col_base, uint8_t* stage) {
  const int lane = threadIdx.x & 31;
  __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(p.C);
  const float* cs = reinterpret_cast<const float*>(p.aux);
  const float* sn = cs + p.aux_ld * 64;
  const int my_row = row0 + lane;
  const long long pos = (my_row < p.M ? my_row : 0) % p.aux_ld;
  __nv_bfloat16* srow = reinterpret_cast<__nv_bfloat16*>(stage + lane * SW_PITCH);
#pragma unroll 1
  for (int hb = 0; hb < BN; hb += 128) {
    const int colh = col_base + hb;
    if (colh >= p.N) break;
    const bool rot = colh < p.ff;
#pragma unroll 1
    for (int cc = 0; cc < 64; cc += 32) {
      uint32_t ra[32], rb[32];
      tmem_ld32(taddr + hb + cc, ra);
      tmem_ld32(taddr + hb + 64 + cc, rb);
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          lo[e] = pack2(__uint_as_float(ra[c + 2 * e]), __uint_as_float(ra[c + 2 * e + 1]));
          hi[e] = pack2(__uint_as_float(rb[c + 2 * e]), __uint_as_float(rb[c + 2 * e + 1]));
        }
        if (rot) {
          const int j = cc + c;
          float cv[8], sv[8];
          *reinterpret_cast<float4*>(cv) = *reinterpret_cast<const float4*>(cs + pos * 64 + j);
          *reinterpret_cast<float4*>(cv + 4) =
              *reinterpret_cast<const float4*>(cs + pos * 64 + j + 4);
          *reinterpret_cast<float4*>(sv) = *reinterpret_cast<const float4*>(sn + pos * 64 + j);
          *reinterpret_cast<float4*>(sv + 4) =
              *reinterpret_cast<const float4*>(sn + pos * 64 + j + 4);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a = bf2_to_f2(lo[e]), b = bf2_to_f2(hi[e]);
            const float c0 = cv[2 * e], c1 = cv[2 * e + 1], s0 = sv[2 * e], s1 = sv[2 * e + 1];
            lo[e] = pack2(a.x * c0 - b.x * s0, a.y * c1 - b.y * s1);
            hi[e] = pack2(b.x * c0 + a.x * s0, b.y * c1 + a.y * s1);
          }
        }
        *reinterpret_cast<uint4*>(srow + c) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        *reinterpret_cast<uint4*>(srow + 32 + c) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 8; ++it) {  // 32 rows x (first 4 | second 4) units of 16 bytes
        const int u = it * 32 + lane, rr = u >> 3, part = u & 7;
        const int row = row0 + rr, col = colh + (part >> 2) * 64 + cc + (part & 3) * 8;
        if (row < p.M && col < p.N)
          *reinterpret_cast<uint4*>(C + (long long)row * p.ldc + col) =
              *reinterpret_cast<const uint4*>(stage + rr * SW_PITCH + part * 16);
      }
      __syncwarp();
    }
  }
}

// epi 4 (GPT fc2 dgrad): acc = d(act) (rounded to bf16 as the unfused dgrad stores it),
// aux = saved pre; C = d(pre) = d(act) * gelu'(pre + bias).  64-column chunks: pre loaded
// coalesced into smem, transformed in place per row, stored coalesced.
__device__ __forceinline__ void epilogue_bias_gelu_bwd(const Params& p, uint32_t taddr, int row0,
                                                       int col_base, uint8_t* stage) {
  const int lane = threadIdx.x & 31;
  const __nv_bfloat16* pre = reinterpret_cast<const __nv_bfloat16*>(p.aux);
  __nv_bfloat16* dpre = reinterpret_cast<__nv_bfloat16*>(p.C);
  __nv_bfloat16* srow = reinterpret_cast<__nv_bfloat16*>(stage + lane * SW_PITCH);
#pragma unroll 1
  for (int q4 = 0; q4 < 4; ++q4) {
    const int colq = col_base + q4 * 64;
    if (colq >= p.N) break;
    uint4 ld[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {  // 32 rows x 8 units of 16 bytes
      const int u = it * 32 + lane, rr = u >> 3, part = u & 7;
      const int row = row0 + rr, col = colq + part * 8;
      ld[it] = make_uint4(0, 0, 0, 0);
      if (row < p.M && col < p.N)
        ld[it] = *reinterpret_cast<const uint4*>(pre + (long long)row * p.aux_ld + col);
    }
    uint32_t r[64];
    tmem_ld32(taddr + q4 * 64, r);
    tmem_ld32(taddr + q4 * 64 + 32, r + 32);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int u = it * 32 + lane, rr = u >> 3, part = u & 7;
      *reinterpret_cast<uint4*>(stage + rr * SW_PITCH + part * 16) = ld[it];
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 64; c += 8) {
      uint4 xr = *reinterpret_cast<const uint4*>(srow + c);
      const uint32_t* xw = reinterpret_cast<const uint32_t*>(&xr);
      uint32_t ow[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = bf2_to_f2(xw[e]);
        const float2 d = bf2_to_f2(pack2(__uint_as_float(r[c + 2 * e]), __uint_as_float(r[c + 2 * e + 1])));
        const int col = min(colq + c + 2 * e, p.N - 2);
        const float2 b = p.bias ? bias_pair(p, col) : make_float2(0.f, 0.f);
        ow[e] = pack2(d.x * gelu_grad_fast(x.x + b.x), d.y * gelu_grad_fast(x.y + b.y));
      }
      *reinterpret_cast<uint4*>(srow + c) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int u = it * 32 + lane, rr = u >> 3, part = u & 7;
      const int row = row0 + rr, col = colq + part * 8;
      if (row < p.M && col < p.N)
        *reinterpret_cast<uint4*>(dpre + (long long)row * p.ldc + col) =
            *reinterpret_cast<const uint4*>(stage + rr * SW_PITCH + part * 16);
    }
    __syncwarp();
  }
}

// plain bf16 epilogue (alpha only: no bias, no accumulate): TMEM -> bf16 pairs -> smem
// (128 columns = 256 bytes per row) -> 16-byte coalesced row-segment stores.  Half the
// staging bytes and no conversions in the store loop compared with the fp32 staging.
__device__ __forceinline__ void epilogue_bf16(const Params& p, uint32_t taddr, int row0,
                                              int col_base, uint8_t* stage) {
  const int lane = threadIdx.x & 31;
  __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(p.C);
  uint8_t* srow = stage + lane * SW_PITCH;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t r[32];
      tmem_ld32(taddr + h * 128 + cc * 32, r);
      uint32_t w[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        w[i] = pack2(__uint_as_float(r[2 * i]) * p.alpha, __uint_as_float(r[2 * i + 1]) * p.alpha);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        *reinterpret_cast<uint4*>(srow + cc * 64 + u * 16) =
            make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
    }
    __syncwarp();
    const int colq = col_base + h * 128;
#pragma unroll 4
    for (int it = 0; it < 16; ++it) {  // 32 rows x 16 units of 16 bytes
      const int u = it * 32 + lane, rr = u >> 4, part = u & 15;
      const int row = row0 + rr, col = colq + part * 8;
      if (row < p.M && col < p.N)
        *reinterpret_cast<uint4*>(C + (long long)row * p.ldc + col) =
            *reinterpret_cast<const uint4*>(stage + rr * SW_PITCH + part * 16);
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void tile_coords2(const Params& p, int t, int& mt, int& nt) {
  tile_coords(p, t, mt, nt);  // pair tiles are 256 x 256; p.tiles_m counts 256-row tiles
}

template <bool PEER>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_bf16_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const Params p) {
  constexpr int STAGES2 = Cfg2<PEER>::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared window
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * HALF_STAGE;
  uint8_t* staging = smem + STAGES2 * 2 * HALF_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + Cfg2<PEER>::STAGING);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
    prefetch_map(&tmA);
    prefetch_map(&tmB);
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // TMA producer: the whole warp runs the loop (warp-uniform state), one elected lane
    // issues each stage's loads
    int stage = 0;
    uint32_t phase = 0;
    const uint64_t pol = l2_evict_last();
    for (int u = pair; u < p.num_units; u += npairs) {
      int mt, nt;
      tile_coords2(p, u % p.num_tiles, mt, nt);
      const int kb0 = (u / p.num_tiles) * p.kb_per, kb1 = min(p.k_blocks, kb0 + p.kb_per);
      const int m0 = mt * 256 + (int)cr * 128;
      const int n0 = p.epi == 2 ? (cr == 0 ? nt * 128 : p.ff + nt * 128) : nt * 256 + (int)cr * 128;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          if (cr == 0) mbar_expect_tx(&full[stage], 4 * HALF_STAGE);
          uint8_t* a_dst = sA + stage * HALF_STAGE;
          uint8_t* b_dst = sB + stage * HALF_STAGE;
          if (p.hint & 1) {
            if (!p.a_mn) {
              tma_load_2d_2sm_hint(&tmA, &full[stage], a_dst, kb * BK, m0, pol);
            } else {
              tma_load_2d_2sm_hint(&tmA, &full[stage], a_dst, m0, kb * BK, pol);
              tma_load_2d_2sm_hint(&tmA, &full[stage], a_dst + 8192, m0 + 64, kb * BK, pol);
            }
            if (!p.b_mn) {
              tma_load_2d_2sm_hint(&tmB, &full[stage], b_dst, kb * BK, n0, pol);
            } else {
              tma_load_2d_2sm_hint(&tmB, &full[stage], b_dst, n0, kb * BK, pol);
              tma_load_2d_2sm_hint(&tmB, &full[stage], b_dst + 8192, n0 + 64, kb * BK, pol);
            }
          } else {
            if (!p.a_mn) {
              tma_load_2d_2sm(&tmA, &full[stage], a_dst, kb * BK, m0);
            } else {
              tma_load_2d_2sm(&tmA, &full[stage], a_dst, m0, kb * BK);
              tma_load_2d_2sm(&tmA, &full[stage], a_dst + 8192, m0 + 64, kb * BK);
            }
            if (!p.b_mn) {
              tma_load_2d_2sm(&tmB, &full[stage], b_dst, kb * BK, n0);
            } else {
              tma_load_2d_2sm(&tmB, &full[stage], b_dst, n0, kb * BK);
              tma_load_2d_2sm(&tmB, &full[stage], b_dst + 8192, n0 + 64, kb * BK);
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES2) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer (leader CTA): descriptors precomputed once and advanced by constant
    // offsets; one elected lane issues a stage's four UMMAs back to back
    if (cr == 0) {
      const uint32_t idesc = make_idesc(256, 256, p.a_mn, p.b_mn);
      const uint64_t a0 = p.a_mn ? sdesc(smem_u32(sA), 8192, 1024) : sdesc(smem_u32(sA), 16, 1024);
      const uint64_t b0 = p.b_mn ? sdesc(smem_u32(sB), 8192, 1024) : sdesc(smem_u32(sB), 16, 1024);
      const uint64_t a_k = p.a_mn ? (2048 >> 4) : (32 >> 4);
      const uint64_t b_k = p.b_mn ? (2048 >> 4) : (32 >> 4);
      constexpr uint64_t STG = HALF_STAGE >> 4;
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = pair; u < p.num_units; u += npairs) {
        const int kb0 = (u / p.num_tiles) * p.kb_per, kb1 = min(p.k_blocks, kb0 + p.kb_per);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = a0 + (uint64_t)stage * STG, bd = b0 + (uint64_t)stage * STG;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_2sm(d, ad + k * a_k, bd + k * b_k, idesc, (kb > kb0) || (k > 0));
            umma_commit_2sm(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_2sm(&tfull[acc], 0x3);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < p.num_units; u += npairs) {
      int mt, nt;
      tile_coords2(p, u % p.num_tiles, mt, nt);
      if (p.hint & 8) mbar_wait(&tfull[acc], acc_phase);
      else mbar_wait_sleep(&tfull[acc], acc_phase, 512);
      tc_fence_after();
      if constexpr (PEER)
        epilogue_peer(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                      mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                      staging + q * 32 * Cfg2<true>::STAGE_PITCH);
      else if (p.epi == 1)
        epilogue_swiglu_bwd(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                            mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                            staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      else if (p.epi == 2)
        epilogue_swiglu_fwd(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                            mt * 256 + (int)cr * 128 + q * 32, nt * 128,
                            staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      else if (p.epi == 3)
        epilogue_bias_gelu_fwd(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                               mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                               staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      else if (p.epi == 4)
        epilogue_bias_gelu_bwd(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                               mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                               staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      else if (p.epi == 5)
        epilogue_rope_qkv(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                          mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                          staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      else if (p.splits > 1) {  // fp32 partial tile of this K-split -> workspace
        Params w = p;
        w.C = p.ws + (long long)(u / p.num_tiles) * p.M * p.N;
        w.ldc = p.N;
        w.c_bf16 = 0;
        w.accumulate = 0;
        w.bias = nullptr;
        w.alpha = 1.f;
        epilogue_staged<false>(w, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                               mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                               staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      } else if (p.c_bf16 && p.bias == nullptr && !p.accumulate && !(p.hint & 32))
        epilogue_bf16(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                      mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                      staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      else
        epilogue_staged<false>(p, tmem + acc * BN + ((uint32_t)(q * 32) << 16),
                               mt * 256 + (int)cr * 128 + q * 32, nt * BN,
                               staging + q * 32 * Cfg2<false>::STAGE_PITCH);
      tc_fence_before();
      mbar_arrive_remote(&tempty[acc], 0);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, TMEM_COLS);
  }
}

// split-K reduction: C[m, n] (+)= alpha * sum_s ws[s][m][n] (+ bias[n]), 4 columns/thread
__global__ void splitk_reduce(const float* __restrict__ ws, int splits, int M, int N, void* C,
                              long long ldc, int c_bf16, float alpha, const void* bias,
                              int bias_bf16, int accumulate) {
  const long long n4 = N / 4, total = (long long)M * n4;
  const long long MN = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / n4), col = (int)(i - (long long)row * n4) * 4;
    const long long src = (long long)row * N + col;
    float4 a = *reinterpret_cast<const float4*>(ws + src);
    for (int s = 1; s < splits; ++s) {
      const float4 b = *reinterpret_cast<const float4*>(ws + s * MN + src);
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    float v[4] = {a.x * alpha, a.y * alpha, a.z * alpha, a.w * alpha};
    if (bias) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        v[e] += bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(bias)[col + e])
                          : reinterpret_cast<const float*>(bias)[col + e];
    }
    const long long dst = (long long)row * ldc + col;
    if (c_bf16) {
      __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(C) + dst;
#pragma unroll
      for (int e = 0; e < 4; ++e) c[e] = __float2bfloat16_rn(v[e] + (accumulate ? __bfloat162float(c[e]) : 0.f));
    } else {
      float* c = reinterpret_cast<float*>(C) + dst;
#pragma unroll
      for (int e = 0; e < 4; ++e) c[e] = v[e] + (accumulate ? c[e] : 0.f);
    }
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// 2-D bf16 map over a row-major matrix [outer, inner] with leading dim `ld` elements
static bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace tc

// K-split count for the 2-CTA path: minimise waves x k-blocks per unit (one k-block of a
// 256x256 pair tile ~ 0.35 us) plus the fp32 partial round trip through HBM and one extra
// launch; small-output / long-K GEMMs (wgrad of narrow layers) fill 74 pairs this way
int32_t gemm_pick_splits(int64_t M, int64_t N, int64_t K) {
  if (M <= 128 || N % 4 != 0) return 1;
  const int64_t pairs = sm_count() / 2;
  const int64_t tiles = ((M + 255) / 256) * ((N + 255) / 256), kb = (K + tc::BK - 1) / tc::BK;
  auto cost = [&](int64_t s) {
    const int64_t kbs = (kb + s - 1) / s, units = tiles * ((kb + kbs - 1) / kbs);
    double t = (double)((units + pairs - 1) / pairs) * kbs * 0.35e-6;
    if (s > 1) t += (double)M * N * 4.0 * (s + 1) / 6.0e12 + 4e-6;
    return t;
  };
  int32_t best = 1;
  double best_t = cost(1);
  for (int64_t s = 2; s <= 16; ++s) {
    if (kb / s < 8) break;
    const double t = cost(s);
    if (t < 0.9 * best_t) {
      best = (int32_t)s;
      best_t = t;
    }
  }
  return best;
}

// the fused activation epilogues (SwiGLU / bias-GeLU) need the 2-CTA path (M > 128, 16-byte aligned rows) and
// 8-element aligned gate/up/h rows; epi 2 also needs the nn.Linear (K-major) weight
bool epilogue_fusable(const void* A, const void* B, const void* C, const void* aux, int64_t M,
                    int64_t ldc, int64_t aux_ld, int64_t ff, int32_t trans_b, int32_t epi) {
  auto al = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; };
  return M > 128 && al(A) && al(B) && al(C) && al(aux) && ldc % 8 == 0 && aux_ld % 8 == 0 &&
         ff % 8 == 0 && ff > 0 && (epi != 2 || trans_b);
}

int32_t gemm_bf16_sm100(const void* A, const void* B, void* C, const void* bias, int64_t M,
                        int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                        int32_t trans_a, int32_t trans_b, float alpha, int32_t accumulate,
                        int32_t c_dtype, int32_t bias_dtype, cudaStream_t stream,
                        void* const* peer_c, int64_t rows_per_rank, int32_t my_slot,
                        int32_t epi, const void* aux, int64_t aux_ld, int64_t ff,
                        int32_t splits, float* ws) {
  using namespace tc;
  GALV_CHECK_ARG(M > 0 && N > 0 && K > 0, "empty problem");
  GALV_CHECK_ARG(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31), "problem too large");
  GALV_CHECK_ARG((lda % 8) == 0 && (ldb % 8) == 0, "lda/ldb must be multiples of 8 (TMA)");
  GALV_CHECK_ARG((reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(B) & 15) == 0,
                 "A/B must be 16-byte aligned");
  const int a_mn = trans_a ? 1 : 0;  // A stored [K, M] -> M contiguous
  const int b_mn = trans_b ? 0 : 1;  // B stored [K, N] -> N contiguous
  CUtensorMap ma, mb;
  bool ok = a_mn ? make_map(&ma, A, M, K, lda, 64, 64) : make_map(&ma, A, K, M, lda, 64, BM);
  ok = ok && (b_mn ? make_map(&mb, B, N, K, ldb, 64, 64) : make_map(&mb, B, K, N, ldb, 64, BN));
  GALV_CHECK_ARG(ok, "cuTensorMapEncodeTiled failed");
  Params p;
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.a_mn = a_mn;
  p.b_mn = b_mn;
  p.C = C;
  p.ldc = ldc;
  p.c_bf16 = c_dtype == GALV_BF16;
  p.bias = bias;
  p.bias_bf16 = bias_dtype == GALV_BF16;
  p.alpha = alpha;
  p.accumulate = accumulate;
  p.tiles_m = (int)((M + BM - 1) / BM);
  p.tiles_n = (int)((N + BN - 1) / BN);
  p.num_tiles = p.tiles_m * p.tiles_n;
  p.num_units = p.num_tiles;
  p.k_blocks = (int)((K + BK - 1) / BK);
  p.peer_c = peer_c;
  p.rows_per_rank = (int)rows_per_rank;
  p.my_slot = my_slot;
  p.splits = 1;
  p.kb_per = (int)((K + BK - 1) / BK);
  p.ws = nullptr;
  p.epi = epi;
  p.aux = aux;
  p.aux_ld = aux_ld;
  p.ff = (int)ff;
  {
    static int v_group = -1, v_gdim = 0, v_hint = 0;
    if (v_group < 0) {  // GALV_GEMM_RASTER="group,gdim,hint" (tuning sweeps only)
      v_group = GROUP_M;
      if (const char* e = getenv("GALV_GEMM_RASTER")) sscanf(e, "%d,%d,%d", &v_group, &v_gdim, &v_hint);
      if (v_group < 1) v_group = 1;
    }
    p.group = v_group;
    p.gdim = v_gdim;
    p.hint = v_hint;
  }
  static bool attr_set = false;
  if (!attr_set) {
    GALV_CUDA_RET(cudaFuncSetAttribute(gemm_bf16_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SMEM_BYTES));
    attr_set = true;
  }
  const bool c_aligned = (ldc % 8) == 0 &&
                         ((reinterpret_cast<uintptr_t>(C) & 15) == 0 || peer_c != nullptr);
  if (epi != 0) {  // fused SwiGLU epilogues exist on the 2-CTA path only (callers check)
    GALV_CHECK_ARG(epilogue_fusable(A, B, C, aux, M, ldc, aux_ld, ff, trans_b, epi) &&
                       peer_c == nullptr && (bias == nullptr || epi == 3 || epi == 4) &&
                       !accumulate &&
                       c_dtype == GALV_BF16 && alpha == 1.0f,
                   "fused activation epilogue: unsupported operands");
  }
  if (M > 128 && c_aligned) {
    // 2-CTA path: 256x256 pair tiles, per-CTA boxes of 128 rows
    CUtensorMap ma2, mb2;
    bool ok2 = a_mn ? make_map(&ma2, A, M, K, lda, 64, 64) : make_map(&ma2, A, K, M, lda, 64, 128);
    ok2 = ok2 && (b_mn ? make_map(&mb2, B, N, K, ldb, 64, 64) : make_map(&mb2, B, K, N, ldb, 64, 128));
    GALV_CHECK_ARG(ok2, "cuTensorMapEncodeTiled failed");
    Params p2 = p;
    p2.tiles_m = (int)((M + 255) / 256);
    if (epi == 2) p2.tiles_n = (int)((ff + 127) / 128);  // pair tile = 128 gate + 128 up cols
    p2.num_tiles = p2.tiles_m * p2.tiles_n;
    const bool split = splits > 1 && ws != nullptr && epi == 0 && peer_c == nullptr && N % 4 == 0;
    p2.kb_per = split ? (p.k_blocks + splits - 1) / splits : p.k_blocks;
    p2.splits = split ? (p.k_blocks + p2.kb_per - 1) / p2.kb_per : 1;
    p2.num_units = p2.num_tiles * p2.splits;
    p2.ws = split ? ws : nullptr;
    static bool attr2 = false;
    if (!attr2) {
      GALV_CUDA_RET(cudaFuncSetAttribute(gemm_bf16_tc2<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg2<false>::SMEM));
      GALV_CUDA_RET(cudaFuncSetAttribute(gemm_bf16_tc2<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg2<true>::SMEM));
      attr2 = true;
    }
    const int pairs = min(p2.num_units, sm_count() / 2);
    if (peer_c != nullptr)
      gemm_bf16_tc2<true><<<2 * pairs, 256, Cfg2<true>::SMEM, stream>>>(ma2, mb2, p2);
    else
      gemm_bf16_tc2<false><<<2 * pairs, 256, Cfg2<false>::SMEM, stream>>>(ma2, mb2, p2);
    GALV_LAUNCH_CHECK();
    if (p2.splits > 1) {
      const long long work = M * (N / 4);
      const int blocks = (int)std::min<long long>((work + 255) / 256, (long long)sm_count() * 8);
      splitk_reduce<<<blocks, 256, 0, stream>>>(ws, p2.splits, (int)M, (int)N, C, ldc,
                                                c_dtype == GALV_BF16, alpha, bias,
                                                bias_dtype == GALV_BF16, accumulate);
      GALV_LAUNCH_CHECK();
    }
    return 0;
  }
  const int grid = min(p.num_tiles, sm_count());
  gemm_bf16_tc<<<grid, 256, SMEM_BYTES, stream>>>(ma, mb, p);
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // namespace galv

extern "C" int32_t galv_gemm_rs(const void* A, const void* B, void* const* peer_c,
                                int64_t rows_per_rank, int32_t my_slot, int64_t M, int64_t N,
                                int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int32_t trans_a,
                                int32_t trans_b, void* stream) {
  GALV_CHECK_ARG(A && B && peer_c && rows_per_rank > 0 && M % rows_per_rank == 0,
                 "bad arguments");
  return galv::gemm_bf16_sm100(A, B, nullptr, nullptr, M, N, K, lda, ldb, ldc, trans_a, trans_b,
                               1.0f, 0, GALV_BF16, GALV_F32, galv::as_stream(stream), peer_c,
                               rows_per_rank, my_slot, 0, nullptr, 0, 0, 1, nullptr);
}
