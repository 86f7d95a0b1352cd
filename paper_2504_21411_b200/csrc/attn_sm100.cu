// tcgen05 flash-attention forward for sm_100a (bf16 in, fp32 softmax/accumulate).
//
// CTA = 128 queries of one (batch, head); K/V streamed in 128-key blocks by TMA into a
// 2-stage ring; S = Q K^T and O += P V on the 5th-gen tensor cores with accumulators in
// TMEM (S double-buffered: cols [0,128) and [128,256); O at cols [256, 256+D)).
//   warp 0   : TMA producer (Q once, K/V ring; 3-D maps over [tokens, heads, head_dim])
//   warp 1   : MMA issuer; issues S_{j+1} before PV_j so QK^T overlaps the softmax
//   warp 2   : TMEM allocator
//   warps 4-7: softmax -- thread = query row = TMEM lane; online softmax with a lazy
//              rescale (O in TMEM is rescaled only when a row max grows by > 2^8),
//              P written to smem as a 128B-swizzled K-major bf16 operand, epilogue.
#include "common.cuh"
#include "dropout.cuh"
#include "sm100.cuh"

namespace galv {
namespace fa {
using namespace sm100;

constexpr int BQ = 128, BKV = 128;
#ifdef GALV_ATTN_TRACE  // scratch builds only: clock64 timeline of CTA (0, 0)
__device__ unsigned long long g_trace[8192];
#define TRACE(slot)                                                        \
  do {                                                                     \
    if (blockIdx.x == 0 && blockIdx.y == 0) g_trace[(slot)] = clock64();   \
  } while (0)
// per-CTA [start, end, smid] in globaltimer ns (forward kernel only)
__device__ unsigned long long g_cta[3 * 65536];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CTA_TRACE(k)                                                                   \
  do {                                                                                 \
    const unsigned id = blockIdx.y * gridDim.x + blockIdx.x;                           \
    if (id < 65536) {                                                                  \
      g_cta[3 * id + (k)] = gtimer();                                                  \
      if ((k) == 0) {                                                                  \
        unsigned smid;                                                                 \
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));                               \
        g_cta[3 * id + 2] = smid;                                                      \
      }                                                                                \
    }                                                                                  \
  } while (0)
#else
#define CTA_TRACE(k) \
  do {               \
  } while (0)
#define TRACE(slot) \
  do {              \
  } while (0)
#endif
// K/V multicast across CTA pairs (fwd_tc<D, true>) is correct but measured slower on B200
// (663 vs 701 TF at S=4K, 933 vs 942 TF at S=32K, 203 vs 237 TF at D=64): the forward is not
// L2-bandwidth bound, and pairing couples the two CTAs' pipelines.  Off by default.
#ifndef ATTN_FWD_MC
#define ATTN_FWD_MC 0
#endif
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units
// exponentials stay on MUFU: measured on B200, offloading 1/2..1/4 of them to the FMA pipe
// (exp2_fma) made the forward 2-8 % slower -- the softmax is latency-, not XU-bound
#ifndef EXP_POLY_EVERY
#define EXP_POLY_EVERY 0
#endif

template <int D>
struct Smem {
  static constexpr int TILE = D * BQ * 2;        // one [128 rows][D] bf16 tile
  static constexpr int Q = 0;
  static constexpr int K0 = Q + TILE;
  static constexpr int V0 = K0 + 2 * TILE;
  static constexpr int BAR = V0 + 2 * TILE;      // P lives in TMEM (over its S buffer)
  static constexpr int BYTES = BAR + 160 + 3 * 1024 + 1024;  // barriers, xch, slack
};

struct FwdParams {
  int S, H, n_qblocks;
  int bh_total;  // batch * heads (fwd_tc2 work-item decode)
  int causal;
  float scale_log2;
  __nv_bfloat16* o;
  float* lse;
  long long o_st;  // o token stride (elements)
  long long sh;    // head stride (elements)
  DropoutParams drop;  // attention-probability dropout (fwd_tc2 only; thresh 0 = off)
};

// 2^x on the FMA/ALU pipes (Cody-Waite split + degree-4 minimax, rel err 5e-6): used for
// half of the softmax exponentials so the MUFU (XU) pipe is not the bottleneck.
__device__ __forceinline__ float exp2_fma(float x) {
  const float xc = fmaxf(x, -125.f);
  const float magic = 12582912.f;  // 1.5 * 2^23: rounds to an integer in the low bits
  const float r = xc + magic;
  const float n = r - magic;
  const float f = xc - n;  // [-0.5, 0.5]
  float p = fmaf(0.009554105163799703f, f, 0.05587040851370001f);
  p = fmaf(p, f, 0.24024696601651352f);
  p = fmaf(p, f, 0.6931280281735204f);
  p = fmaf(p, f, 0.9999994397927999f);
  const int bits = __float_as_int(p) + (__float_as_int(r) << 23);
  return x < -125.f ? 0.f : __int_as_float(bits);
}
// 2^x (x <= 0) on the FMA/ALU pipes: x = n + f, n = floor(x), 2^f by a degree-3 minimax
// (max rel err 8.6e-5, below the bf16 rounding of P), exponent by an integer add
__device__ __forceinline__ float exp2_poly3(float x) {
  const float xc = fmaxf(x, -126.f);
  const float n = floorf(xc);
  const float f = xc - n;
  float q = fmaf(0.07706213f, f, 0.22764884f);
  q = fmaf(q, f, 0.69511681f);
  q = fmaf(q, f, 1.0f);
  return __int_as_float(__float_as_int(q) + (static_cast<int>(n) << 23));
}
// head_dim 64 forward: the exp work is 2x the MMA work per block (MUFU-bound); every
// ATTN_POLY64-th exponential pair goes to the FMA pipe (0 = all on MUFU); ATTN_POLY128 the
// same at head_dim 128 -- measured slower at every fraction for both (fwd_poly/)
#ifndef ATTN_POLY128
#define ATTN_POLY128 0
#endif
#ifndef ATTN_POLY_FN
#define ATTN_POLY_FN exp2_poly3
#endif
#ifndef ATTN_POLY64
#define ATTN_POLY64 0
#endif
__device__ __forceinline__ float exp2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// MC: CTA pairs (cluster of 2 on adjacent query blocks of the same (b, h)) share every K/V
// tile: the leader loads it once with a multicast TMA into both CTAs' rings (halving L2->SM
// traffic per FLOP); both CTAs' MMA completions release the leader's k/v_empty barriers.
template <int D, bool MC>
__global__ void __launch_bounds__(384, 1)
    fwd_tc(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
           const __grid_constant__ CUtensorMap mv, const FwdParams p) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared window
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* v_full = bar + 3;    // [2]
  uint64_t* k_empty = bar + 5;   // [2]  K stage free once S_j is computed
  uint64_t* s_full = bar + 7;    // [3]
  uint64_t* s_empty = bar + 10;  // [3]  S buffer free once PV of its block is done
  uint64_t* p_full = bar + 13;   // [3]  P (bf16) packed over its S buffer
  uint64_t* o_done = bar + 16;
  uint64_t* v_empty = bar + 17;  // [2]  V stage free once PV_j is computed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 19);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = p.n_qblocks - 1 - blockIdx.x;  // heavy causal blocks first
  const int bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int q0 = qb * BQ;
  const uint32_t cr = MC ? cluster_ctarank() : 0;
  // a cluster pair iterates the leader's (larger) KV range; the extra causal block is fully
  // masked for the peer and contributes nothing
  const int qb_lead = MC ? p.n_qblocks - 1 - (int)(blockIdx.x & ~1u) : qb;
  const int n_kv = p.causal ? min(qb_lead + 1, (p.S + BKV - 1) / BKV) : (p.S + BKV - 1) / BKV;
  const int tok0 = b * p.S;
  constexpr uint32_t TILE_BYTES = L::TILE;

  if (threadIdx.x == 0) CTA_TRACE(0);
  if (threadIdx.x == 0) TRACE(8000);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&k_empty[i], MC ? 2 : 1);
      mbar_init(&v_empty[i], MC ? 2 : 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 1);
      mbar_init(&p_full[i], 256);
    }
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
    if (MC) {  // every CTA arms its own K/V barriers for the first use of each stage
      for (int i = 0; i < 2 && i < n_kv; ++i) {
        mbar_expect_tx(&k_full[i], TILE_BYTES);
        mbar_expect_tx(&v_full[i], TILE_BYTES);
      }
    }
    prefetch_map(&mq);
    prefetch_map(&mk);
    prefetch_map(&mv);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  if (MC)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S triple-buffered (cols 0-383; P(j) bf16 is packed over the first half of each
  // softmax half's S columns and read by PV as the A operand), O at cols 384-511
  const uint32_t t_s = tmem, t_o = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, TILE_BYTES);
#pragma unroll
      for (int c = 0; c < D / 64; ++c)
        tma_load_3d(&mq, q_full, sm + L::Q + c * 16384, c * 64, h, tok0 + q0);
      if (!MC || cr == 0) {
        for (int j = 0; j < n_kv; ++j) {
          const int st = j & 1;
          mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
          if (!MC) mbar_expect_tx(&k_full[st], TILE_BYTES);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            uint8_t* dst = sm + L::K0 + st * L::TILE + c * 16384;
            if (MC)
              tma_load_3d_mc(&mk, &k_full[st], dst, c * 64, h, tok0 + j * BKV, 0x3);
            else
              tma_load_3d(&mk, &k_full[st], dst, c * 64, h, tok0 + j * BKV);
          }
          mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
          if (!MC) mbar_expect_tx(&v_full[st], TILE_BYTES);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            uint8_t* dst = sm + L::V0 + st * L::TILE + c * 16384;
            if (MC)
              tma_load_3d_mc(&mv, &v_full[st], dst, c * 64, h, tok0 + j * BKV, 0x3);
            else
              tma_load_3d(&mv, &v_full[st], dst, c * 64, h, tok0 + j * BKV);
          }
        }
        if (MC) {  // drain: the peer's final releases must land before this CTA exits
          for (int j = n_kv; j < n_kv + 2; ++j) {
            mbar_wait(&k_empty[j & 1], ((j >> 1) & 1) ^ 1);
            mbar_wait(&v_empty[j & 1], ((j >> 1) & 1) ^ 1);
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA warp: all lanes run the loop (warp-uniform state, descriptors precomputed once and
    // advanced by constant offsets); one elected lane issues each group of tcgen05.mma
    const uint32_t id_s = make_idesc(BQ, BKV, 0, 0);  // Q (K-major) x K (K-major)
    const uint32_t id_o = make_idesc(BQ, D, 0, 1);    // P (K-major) x V (MN-major)
    const uint64_t d_q = sdesc(smem_u32(sm + L::Q), 16, 1024);
    const uint64_t d_k = sdesc(smem_u32(sm + L::K0), 16, 1024);
    const uint64_t d_v = sdesc(smem_u32(sm + L::V0), 16384, 1024);
    mbar_wait_fast(q_full, 0);
    // O += P V: A = P from TMEM (keys 16k.. packed at col 64*(k/4) + 8*(k%4) of the block's S
    // buffer), B = the V tile as an MN-major operand
    auto issue_pv = [&](int j) {
      const int st = j & 1, sb = j % 3;
      mbar_wait_fast(&p_full[sb], (j / 3) & 1);
      mbar_wait_fast(&v_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (lane == 0) TRACE(6144 + j * 8 + 1);
      const uint64_t bv = d_v + (uint64_t)((st * L::TILE) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          umma_bf16_ts(t_o, t_s + sb * BKV + (k >> 2) * 64 + (k & 3) * 8,
                       bv + (uint64_t)((k * 2048) >> 4), id_o, (j | k) != 0);
        umma_commit(o_done);
        umma_commit(&s_empty[sb]);
        if (MC) {
          umma_commit_mc(&v_empty[st], 0x1);  // release to the leader's producer
          if (j + 2 < n_kv) mbar_expect_tx(&v_full[st], TILE_BYTES);  // re-arm own stage
        } else {
          umma_commit(&v_empty[st]);
        }
      }
      __syncwarp();
    };
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1, sb = j % 3;
      if (lane == 0) TRACE(6144 + j * 8 + 6);
      mbar_wait_fast(&k_full[st], (j >> 1) & 1);
      if (lane == 0) TRACE(6144 + j * 8 + 7);
      mbar_wait_fast(&s_empty[sb], ((j / 3) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) TRACE(6144 + j * 8 + 0);
      const uint64_t bk = d_k + (uint64_t)((st * L::TILE) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t off = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
          umma_bf16(t_s + sb * BKV, d_q + off, bk + off, id_s, k != 0);
        }
        umma_commit(&s_full[sb]);
        if (MC) {
          umma_commit_mc(&k_empty[st], 0x1);
          if (j + 2 < n_kv) mbar_expect_tx(&k_full[st], TILE_BYTES);
        } else {
          umma_commit(&k_empty[st]);
        }
      }
      __syncwarp();
      if (j > 0) issue_pv(j - 1);
    }
    issue_pv(n_kv - 1);
  } else if (warp >= 4) {
    // softmax: warps 4..11; quarter q = warp % 4 owns TMEM lanes (rows) [32q, 32q+32),
    // half = (warp - 4) / 4 owns key columns [64*half, 64*half + 64) of every S block and
    // O columns [half*D/2, half*D/2 + D/2).  Row maxima are exchanged through smem.
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    const int qi = q0 + r;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // [2][256] partial maxima + [256] partial sums, after the 20 barrier words (160 bytes)
    float* xch = reinterpret_cast<float*>(bar + 20);
    float m_used = -INFINITY, l = 0.f;
    constexpr int HC = BKV / 2;  // columns per half
    for (int j = 0; j < n_kv; ++j) {
      const int sb = j % 3;
      mbar_wait(&s_full[sb], (j / 3) & 1);
      tc_fence_after();
      if (warp == 4 && lane == 0) TRACE(6144 + j * 8 + 2);
      float s[HC];
#pragma unroll
      for (int c = 0; c < HC / 32; ++c)
        tmem_ld32_nowait(t_s + sb * BKV + half * HC + c * 32 + lane_off,
                         reinterpret_cast<uint32_t*>(s) + c * 32);
      tmem_wait_ld();
      if (warp == 4 && lane == 0) TRACE(6144 + j * 8 + 3);
      const int k0 = j * BKV + half * HC;
      const bool mask = (k0 + HC > p.S) || (p.causal && k0 + HC - 1 > q0);
      if (mask) {  // diagonal / tail block: keys >= lim are invisible to this row
        const int lim = (p.causal ? min(p.S, qi + 1) : p.S) - k0;
#pragma unroll
        for (int i = 0; i < HC; ++i) s[i] = i < lim ? s[i] : -INFINITY;
      }
      // row max as a tree (8 independent chains): a serial fmax chain over 64 columns is
      // ~256 cycles of dependent latency per block on the softmax critical path
      float m8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = s[u];
#pragma unroll
      for (int i = 8; i < HC; ++i) m8[i & 7] = fmaxf(m8[i & 7], s[i]);
      float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                       fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      // combine the two halves' row maxima (pair barrier: 64 threads of this quarter)
      xch[(j & 1) * 256 + half * 128 + r] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      mx = fmaxf(mx, xch[(j & 1) * 256 + (half ^ 1) * 128 + r]);
      mx *= p.scale_log2;
      float alpha = 1.f;
      if ((mx > m_used + RESCALE_THRESHOLD || m_used == -INFINITY) && mx != -INFINITY) {
        alpha = (m_used == -INFINITY) ? 0.f : exp2f(m_used - mx);
        m_used = mx;
      }
      const float mu = (m_used == -INFINITY) ? 0.f : m_used;
      float r4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent partial row sums
      uint32_t pk[HC / 2];
#pragma unroll
      for (int i = 0; i < HC; i += 2) {
        // FA4-style split: EXP_POLY_EVERY-th pairs on the FMA pipe, the rest on MUFU
        const float x0 = fmaf(s[i], p.scale_log2, -mu), x1 = fmaf(s[i + 1], p.scale_log2, -mu);
        float p0, p1;
        if (EXP_POLY_EVERY > 0 && ((i >> 1) % (EXP_POLY_EVERY > 0 ? EXP_POLY_EVERY : 1)) ==
                                      (EXP_POLY_EVERY > 0 ? EXP_POLY_EVERY : 1) - 1) {
          p0 = exp2_fma(x0);
          p1 = exp2_fma(x1);
        } else {
          p0 = exp2_mufu(x0);
          p1 = exp2_mufu(x1);
        }
        r4[(i >> 1) & 3] += p0 + p1;
        pk[i / 2] = pack2(p0, p1);
      }
      const float rs = (r4[0] + r4[1]) + (r4[2] + r4[3]);
      l = l * alpha + rs;
      if (warp == 4 && lane == 0) TRACE(6144 + j * 8 + 4);
      // lazy rescale: O must hold PV(j-1) first.  When S(j) completed, PV(j-2) had too and
      // PV(j) needs this P, so o_done has completed j-1 or j phases: the parity wait is exact
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 64; ++c) {
          uint32_t ov[32];
          const uint32_t ta = t_o + half * (D / 2) + c * 32 + lane_off;
          tmem_ld32(ta, ov);
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
          tmem_st32(ta, ov);
        }
      }
      // P half-row (bf16 pairs) -> TMEM over this half's first 32 S columns
      tmem_st32(t_s + sb * BKV + half * HC + lane_off, pk);  // includes wait::st
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
      if (warp == 4 && lane == 0) TRACE(6144 + j * 8 + 5);
    }
    // full row sum = both halves
    xch[512 + half * 128 + r] = l;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
    l += xch[512 + (half ^ 1) * 128 + r];
    mbar_wait(o_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = p.o + (long long)(tok0 + qi) * p.o_st + (long long)h * p.sh + half * (D / 2);
#pragma unroll 1
    for (int c = 0; c < D / 64; ++c) {
      uint32_t ov[32];
      tmem_ld32(t_o + half * (D / 2) + c * 32 + lane_off, ov);
      if (qi < p.S) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 w;
          w.x = pack2(__uint_as_float(ov[u * 8 + 0]) * inv_l, __uint_as_float(ov[u * 8 + 1]) * inv_l);
          w.y = pack2(__uint_as_float(ov[u * 8 + 2]) * inv_l, __uint_as_float(ov[u * 8 + 3]) * inv_l);
          w.z = pack2(__uint_as_float(ov[u * 8 + 4]) * inv_l, __uint_as_float(ov[u * 8 + 5]) * inv_l);
          w.w = pack2(__uint_as_float(ov[u * 8 + 6]) * inv_l, __uint_as_float(ov[u * 8 + 7]) * inv_l);
          *reinterpret_cast<uint4*>(orow + c * 32 + u * 8) = w;
        }
      }
    }
    if (qi < p.S && half == 0)
      p.lse[((long long)b * p.H + h) * p.S + qi] =
          (m_used + log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  if (MC)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- forward, two Q tiles
// CTA = 256 queries (two 128-row tiles t = 0, 1) of one (batch, head), so every K/V tile
// loaded by TMA feeds two QK^T and two PV MMAs, and the tensor pipe alternates between the
// tiles: while softmax warpgroup-pair t works on S_t(j), the MMA warp runs the other tile's
// PV(j) and S(j+1).  TMEM (512 columns): S_0 [0,128), S_1 [128,256), O_0 [256, 256+D),
// O_1 [384, 384+D); P_t (bf16) is packed over the first half of each 64-column half of S_t
// and read by PV as the A operand.  tcgen05.mma instructions from one thread execute in
// issue order, so S_t(j+1) -- issued after PV_t(j) -- never overwrites P_t(j) before PV
// has read it.
// Work items (query pair, batch*head) go heaviest causal pair first; with fwd_ctas(S) > 0
// each CTA loops over items c, c + gridDim.x, ... (persistent: TMEM and barriers set up once,
// the next item's Q load and first S MMAs overlap this item's epilogue; q_empty and o_free
// hand Q and O_t over between items).
//   warp 0    : TMA producer (Q_0, Q_1 per item; K/V 2-stage ring)
//   warp 1    : MMA issuer: S_0(0), S_1(0), then per block j: PV_0(j), S_0(j+1), PV_1(j),
//               S_1(j+1)
//   warp 2    : TMEM allocator;  warp 3: idle
//   warps 4-7 : softmax of tile 0;  warps 8-11: softmax of tile 1 (one thread per query
//               row = TMEM lane, quarter = warp % 4, all 128 key columns in registers)
template <int D>
struct Smem2 {
  static constexpr int TILE = D * 128 * 2;
  static constexpr int Q = 0;                    // [2 tiles]
  static constexpr int K0 = 2 * TILE;            // [2 stages]
  static constexpr int V0 = K0 + 2 * TILE;       // [2 stages]
  static constexpr int BAR = V0 + 2 * TILE;
  static constexpr int XCH = BAR + 256;          // per tile: [2][256] maxima + [256] sums
  static constexpr int BYTES = XCH + 2 * 768 * 4 + 1024;
};
constexpr int FWD2_THREADS = 384;
#ifndef FWD_PSPLIT
#define FWD_PSPLIT 2  // parts of P per tile and block handed to PV separately (1, 2, 4, 8)
#endif
#ifndef ATTN_FWD_PERSIST_MAX_S
#define ATTN_FWD_PERSIST_MAX_S 2048
#endif

template <int D, bool DROP>
__global__ void __launch_bounds__(FWD2_THREADS, 1)
    fwd_tc2(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
            const __grid_constant__ CUtensorMap mv, const FwdParams p) {
  using L = Smem2<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* v_full = bar + 3;    // [2]
  uint64_t* k_empty = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;   // [2]
  uint64_t* s_full = bar + 9;    // [tile]
  constexpr int NP = FWD_PSPLIT;  // P parts per tile (PV over part q starts once it is stored)
  static_assert(NP >= 2 && NP <= 8 && (NP & (NP - 1)) == 0, "FWD_PSPLIT: 2, 4 or 8");
  uint64_t* p_full = bar + 11;        // [tile][part] P_t of keys [128 q / NP, ...) stored
  uint64_t* o_done = p_full + 2 * NP; // [tile]
  uint64_t* q_empty = o_done + 2;     // the item's last S MMA done: Q tiles reusable
  uint64_t* o_free = q_empty + 1;     // [tile] the item's epilogue has read O_t out of TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_pairs = (p.n_qblocks + 1) / 2;
  const int nkb = (p.S + BKV - 1) / BKV;
  const int n_items = n_pairs * p.bh_total;
  constexpr uint32_t TILE_BYTES = L::TILE;
  // Work item w = (query pair, batch*head), ordered heaviest causal pair first with
  // (batch, head) fastest; CTA c runs items c, c + gridDim.x, ... (one item per CTA when the
  // grid covers them all; persistent CTAs otherwise -- the next item's Q load and S MMAs then
  // overlap this item's epilogue, and the CTA set-up is paid once).
  struct Item {
    int b, h, q0, nkv0, nkv1, tok0;
  };
  auto decode = [&](int w) {
    Item it;
    const int qp = n_pairs - 1 - w / p.bh_total, bh = w % p.bh_total;
    it.b = bh / p.H;
    it.h = bh % p.H;
    it.q0 = qp * 2 * BQ;
    auto blocks_of = [&](int qt) {
      return qt >= p.S ? 0 : (p.causal ? min(qt / BKV + 1, nkb) : nkb);
    };
    it.nkv0 = blocks_of(it.q0);
    it.nkv1 = blocks_of(it.q0 + BQ);  // 0 = tile beyond the sequence
    it.tok0 = it.b * p.S;
    return it;
  };

  if (threadIdx.x == 0) CTA_TRACE(0);
  if (threadIdx.x == 0) TRACE(8000);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      for (int q = 0; q < NP; ++q) mbar_init(&p_full[NP * i + q], 128);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_free[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
    prefetch_map(&mq);
    prefetch_map(&mk);
    prefetch_map(&mv);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE(8001);
  if (warp == 0) {
    if (lane == 0) {
      uint32_t kv = 0;  // K/V blocks loaded so far (ring stage and parity)
      int n_it = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n_it) {
        const Item I = decode(w);
        mbar_wait(q_empty, (n_it & 1) ^ 1);
        const int nq = I.nkv1 > 0 ? 2 : 1;
        mbar_expect_tx(q_full, nq * TILE_BYTES);
        for (int t = 0; t < nq; ++t)
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(&mq, q_full, sm + L::Q + t * L::TILE + c * 16384, c * 64, I.h,
                        I.tok0 + I.q0 + t * BQ);
        const int n_kv = max(I.nkv0, I.nkv1);
        for (int j = 0; j < n_kv; ++j, ++kv) {
          const int st = kv & 1;
          mbar_wait(&k_empty[st], ((kv >> 1) & 1) ^ 1);
          mbar_expect_tx(&k_full[st], TILE_BYTES);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(&mk, &k_full[st], sm + L::K0 + st * L::TILE + c * 16384, c * 64, I.h,
                        I.tok0 + j * BKV);
          mbar_wait(&v_empty[st], ((kv >> 1) & 1) ^ 1);
          mbar_expect_tx(&v_full[st], TILE_BYTES);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(&mv, &v_full[st], sm + L::V0 + st * L::TILE + c * 16384, c * 64, I.h,
                        I.tok0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t id_s = make_idesc(BQ, BKV, 0, 0);
    const uint32_t id_o = make_idesc(BQ, D, 0, 1);
    const uint64_t d_q = sdesc(smem_u32(sm + L::Q), 16, 1024);
    const uint64_t d_k = sdesc(smem_u32(sm + L::K0), 16, 1024);
    const uint64_t d_v = sdesc(smem_u32(sm + L::V0), 16384, 1024);
    uint32_t kv0 = 0;                        // first K/V block of the item (ring position)
    uint32_t base0 = 0, base1 = 0;           // blocks of tile 0 / 1 in earlier items
    uint32_t done0 = 0, done1 = 0;           // earlier items with a tile-0 / tile-1 epilogue
    int n_it = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n_it) {
      const Item I = decode(w);
      const int nkv0 = I.nkv0, nkv1 = I.nkv1, n_kv = max(nkv0, nkv1);
      mbar_wait_fast(q_full, n_it & 1);
      if (lane == 0) TRACE(8002);
      // the last S MMA of the item reads Q for the last time (S_1 when tile 1 exists)
      const int last_t = nkv1 > 0 ? 1 : 0, last_j = (last_t ? nkv1 : nkv0) - 1;
      auto issue_s = [&](int t, int j) {
        const uint32_t g = kv0 + j;
        const int st = g & 1;
        if (lane == 0) TRACE(4096 + t * 1024 + j * 8 + 0);
        mbar_wait_fast(&k_full[st], (g >> 1) & 1);
        tc_fence_after();
        if (lane == 0) TRACE(4096 + t * 1024 + j * 8 + 1);
        const uint64_t bk = d_k + (uint64_t)((st * L::TILE) >> 4);
        const uint64_t bq = d_q + (uint64_t)((t * L::TILE) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t off = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
            umma_bf16(tmem + t * 128, bq + off, bk + off, id_s, k != 0);
          }
          umma_commit(&s_full[t]);
          if (t == 1 || j >= nkv1) umma_commit(&k_empty[st]);  // last reader of K_j
          if (t == last_t && j == last_j) umma_commit(q_empty);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j) {
        const uint32_t g = kv0 + j;
        const int st = g & 1;
        const uint32_t bt = (t ? base1 : base0) + j;
        if (lane == 0) TRACE(4096 + t * 1024 + j * 8 + 2);
        if (j == 0) {  // O_t is overwritten: the previous item's epilogue must have read it
          const uint32_t dn = t ? done1 : done0;
          if (dn > 0) mbar_wait_fast(&o_free[t], (dn - 1) & 1);
        }
        mbar_wait_fast(&p_full[NP * t], bt & 1);
        if (lane == 0) TRACE(4096 + t * 1024 + j * 8 + 3);
        mbar_wait_fast(&v_full[st], (g >> 1) & 1);
        tc_fence_after();
        if (lane == 0) TRACE(4096 + t * 1024 + j * 8 + 4);
        const uint64_t bv = d_v + (uint64_t)((st * L::TILE) >> 4);
        const uint32_t t_o = tmem + 256 + t * 128, t_p = tmem + t * 128;
        // PV over each part of the keys as soon as that part of P is stored; the softmax
        // computes the next part meanwhile (P of keys 16k.. at column 64*(k/4) + 8*(k%4))
        constexpr int KP = BKV / 16 / NP;  // K-steps per part
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (q > 0) {
            mbar_wait_fast(&p_full[NP * t + q], bt & 1);
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int k = q * KP; k < (q + 1) * KP; ++k)
              umma_bf16_ts(t_o, t_p + (k >> 2) * 64 + (k & 3) * 8,
                           bv + (uint64_t)((k * 2048) >> 4), id_o, (j | k) != 0);
          }
          __syncwarp();
        }
        if (elect_one()) {
          umma_commit(&o_done[t]);
          if (t == 1 || j >= nkv1) umma_commit(&v_empty[st]);  // last reader of V_j
        }
        __syncwarp();
      };
      if (nkv0 > 0) issue_s(0, 0);
      if (nkv1 > 0) issue_s(1, 0);
      for (int j = 0; j < n_kv; ++j) {
        if (j < nkv0) {
          issue_pv(0, j);
          if (j + 1 < nkv0) issue_s(0, j + 1);
        }
        if (j < nkv1) {
          issue_pv(1, j);
          if (j + 1 < nkv1) issue_s(1, j + 1);
        }
      }
      kv0 += n_kv;
      base0 += nkv0;
      base1 += nkv1;
      done0 += nkv0 > 0;
      done1 += nkv1 > 0;
    }
  } else if (warp >= 4) {
    // softmax: one thread per query row (warp % 4 = TMEM lane quarter), all 128 key columns
    // of a block in registers -- no cross-warp row-max exchange (the two-threads-per-row
    // split spent ~300 of ~1800 cycles per block in that smem exchange + named barrier)
    const int t = (warp - 4) >> 2;              // tile
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t t_s = tmem + t * 128, t_o = tmem + 256 + t * 128;
    const bool tr = (warp == 4 || warp == 8) && lane == 0;
    uint32_t base = 0;  // blocks of this tile in earlier items (barrier parities)
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const Item I = decode(w);
      const int b = I.b, h = I.h, tok0 = I.tok0;
      const int qt = I.q0 + t * BQ, qi = qt + r;
      const int n_t = t == 0 ? I.nkv0 : I.nkv1;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_t; ++j) {
        const uint32_t bt = base + j;
        if (tr) TRACE(t * 1024 + j * 8 + 0);
        mbar_wait(&s_full[t], bt & 1);
        tc_fence_after();
        if (tr) TRACE(t * 1024 + j * 8 + 1);
        float s[BKV];
#pragma unroll
        for (int c = 0; c < BKV / 32; ++c)
          tmem_ld32_nowait(t_s + c * 32 + lane_off, reinterpret_cast<uint32_t*>(s) + c * 32);
        tmem_wait_ld();
        const int k0 = j * BKV;
        const bool mask = (k0 + BKV > p.S) || (p.causal && k0 + BKV - 1 > qt);
        if (mask) {  // diagonal / tail block: keys >= lim are invisible to this row
          const int lim = (p.causal ? min(p.S, qi + 1) : p.S) - k0;
#pragma unroll
          for (int i = 0; i < BKV; ++i) s[i] = i < lim ? s[i] : -INFINITY;
        }
        float m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = s[u];
#pragma unroll
        for (int i = 8; i < BKV; ++i) m8[i & 7] = fmaxf(m8[i & 7], s[i]);
        float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        if (tr) TRACE(t * 1024 + j * 8 + 2);
        mx *= p.scale_log2;
        float alpha = 1.f;
        if ((mx > m_used + RESCALE_THRESHOLD || m_used == -INFINITY) && mx != -INFINITY) {
          alpha = (m_used == -INFINITY) ? 0.f : exp2f(m_used - mx);
          m_used = mx;
        }
        const float mu = (m_used == -INFINITY) ? 0.f : m_used;
        float r4[4] = {0.f, 0.f, 0.f, 0.f};
        // P in chunks of 16 keys -> 8 packed bf16x2 columns, placed where the PV MMA reads
        // its A operand: keys 16c.. at column 64*(c/4) + 8*(c%4) of the tile's S columns
#pragma unroll
        for (int c = 0; c < BKV / 16; ++c) {
          uint32_t pk[8];
          uint32_t keep = 0xFFFFu;  // dropout: keep bits of the chunk's 16 keys
          if constexpr (DROP) {
            keep = 0;
#pragma unroll
            for (int g = 0; g < 4; ++g)
              keep |= dropout_keep4(p.drop, b, h, qi, k0 + c * 16 + g * 4) << (4 * g);
          }
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const int e = c * 16 + i;
            // all exponentials on MUFU: moving 1/4 or 1/2 of them to an FMA-pipe polynomial
            // measured 4-14 % slower (D 64 and 128, two-threads-per-row variant)
            constexpr int PE = D == 64 ? ATTN_POLY64 : ATTN_POLY128;
            const bool poly = PE > 0 && ((i >> 1) % (PE > 0 ? PE : 1)) == (PE > 0 ? PE : 1) - 1;
            const float x0 = fmaf(s[e], p.scale_log2, -mu), x1 = fmaf(s[e + 1], p.scale_log2, -mu);
            const float p0 = poly ? ATTN_POLY_FN(x0) : exp2_mufu(x0);
            const float p1 = poly ? ATTN_POLY_FN(x1) : exp2_mufu(x1);
            r4[(i >> 1) & 3] += p0 + p1;  // the normalizer uses the undropped probabilities
            if constexpr (DROP)
              pk[i / 2] = pack2((keep >> i) & 1u ? p0 : 0.f, (keep >> (i + 1)) & 1u ? p1 : 0.f);
            else
              pk[i / 2] = pack2(p0, p1);
          }
          tmem_st8(t_s + (c >> 2) * 64 + (c & 3) * 8 + lane_off, pk);
          constexpr int CP = BKV / 16 / NP;  // 16-key chunks per part
          if (c % CP == CP - 1 && c != BKV / 16 - 1) {  // a part stored: PV over it may start
            tmem_wait_st();
            if (tr) TRACE(t * 1024 + j * 8 + 4);
            // lazy rescale of O (after half of P is out of registers): O must hold PV(j-1)
            // first; o_done has completed j-1 phases here (PV(j) needs this P), so the
            // parity wait is exact
            if (c == CP - 1 && j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
              mbar_wait(&o_done[t], (bt - 1) & 1);
              tc_fence_after();
#pragma unroll 1
              for (int cc = 0; cc < D / 32; ++cc) {
                uint32_t ov[32];
                const uint32_t ta = t_o + cc * 32 + lane_off;
                tmem_ld32(ta, ov);
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                tmem_st32(ta, ov);
              }
            }
            tc_fence_before();
            mbar_arrive(&p_full[NP * t + c / CP]);
          }
        }
        l = l * alpha + ((r4[0] + r4[1]) + (r4[2] + r4[3]));
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[NP * t + NP - 1]);
        if (tr) TRACE(t * 1024 + j * 8 + 5);
      }
      if (tr) TRACE(8003 + 2 * t);
      if (n_t > 0) {
        mbar_wait(&o_done[t], (base + n_t - 1) & 1);
        tc_fence_after();
        // dropout: kept probabilities carry 1 / (1 - p)
        const float inv_l = l > 0.f ? (DROP ? p.drop.inv_keep : 1.f) / l : 0.f;
        __nv_bfloat16* orow = p.o + (long long)(tok0 + qi) * p.o_st + (long long)h * p.sh;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t ov[32];
          tmem_ld32(t_o + c * 32 + lane_off, ov);
          if (qi < p.S) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              uint4 v;
              v.x = pack2(__uint_as_float(ov[u * 8 + 0]) * inv_l, __uint_as_float(ov[u * 8 + 1]) * inv_l);
              v.y = pack2(__uint_as_float(ov[u * 8 + 2]) * inv_l, __uint_as_float(ov[u * 8 + 3]) * inv_l);
              v.z = pack2(__uint_as_float(ov[u * 8 + 4]) * inv_l, __uint_as_float(ov[u * 8 + 5]) * inv_l);
              v.w = pack2(__uint_as_float(ov[u * 8 + 6]) * inv_l, __uint_as_float(ov[u * 8 + 7]) * inv_l);
              *reinterpret_cast<uint4*>(orow + c * 32 + u * 8) = v;
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&o_free[t]);  // O_t may now be overwritten by the next item's PV
        if (qi < p.S)
          p.lse[((long long)b * p.H + h) * p.S + qi] = (m_used + log2f(l)) * 0.6931471805599453f;
      }
      if (tr) TRACE(8004 + 2 * t);
      base += n_t;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) CTA_TRACE(1);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- backward
// Two deterministic kernels (no atomics), both on tcgen05 with 8 math warps:
//   dkdv: CTA = 128 keys; per 64-query step  S^T = K Q^T, dP^T = V dO^T (TMEM, double
//         buffered), P^T / dS^T -> smem (bf16, K-major), dV += P^T dO, dK += dS^T Q (TMEM)
//   dq:   CTA = 128 queries; per 64-key step S = Q K^T, dP = dO V^T, dS -> smem,
//         dQ += dS K (TMEM)
// Q/dO (resp. K/V) tiles are loaded once by TMA and read as K-major operands for the
// score GEMMs and as MN-major operands for the gradient GEMMs (same bytes).
// lse*log2(e) and D = rowsum(dO*O) come from a padded workspace written by bwd_prep
// (padded rows: lse2 = +inf so their P is exactly 0).

// D = rowsum(dO * O) and lse * log2(e) per (batch*head, query) row into the padded workspace.
// D/8 lanes per row (one 16-byte load of O and of dO each), 32/(D/8) rows per warp, and
// PREP_ROWS row groups per warp with every load issued before the first use (HBM-bound:
// 2*D*2 bytes read per row; the one-group-per-warp version ran at ~2 TB/s at D=64).
constexpr int PREP_ROWS = 4;
template <int D>
__global__ void __launch_bounds__(256) bwd_prep(const __nv_bfloat16* __restrict__ o,
                                                const __nv_bfloat16* __restrict__ dout,
                                                const float* __restrict__ lse,
                                                float* __restrict__ lse2, float* __restrict__ dvec,
                                                int S, int S_pad, int H, long long n_rows,
                                                long long ost, long long sh) {
  constexpr int LPR = D / 8, RPW = 32 / LPR;  // lanes per row, rows per warp
  const int lane = threadIdx.x & 31, sub = lane % LPR;
  const long long warp_id = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long row0 = warp_id * (RPW * PREP_ROWS) + lane / LPR;
  float a[PREP_ROWS][8], c[PREP_ROWS][8];
  bool ok[PREP_ROWS];
#pragma unroll
  for (int u = 0; u < PREP_ROWS; ++u) {
    const long long row = row0 + u * RPW;
    const int bh = (int)(row / S_pad), i = (int)(row - (long long)bh * S_pad);
    ok[u] = row < n_rows && i < S;
    if (ok[u]) {
      const long long off = ((long long)(bh / H) * S + i) * ost + (long long)(bh % H) * sh + sub * 8;
      load16(o + off, a[u]);
      load16(dout + off, c[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < PREP_ROWS; ++u) {
    const long long row = row0 + u * RPW;
    float s = 0.f;
    if (ok[u]) {
#pragma unroll
      for (int e = 0; e < 8; ++e) s += a[u][e] * c[u][e];
    }
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (sub == 0 && row < n_rows) {
      const int bh = (int)(row / S_pad), i = (int)(row - (long long)bh * S_pad);
      dvec[row] = i < S ? s : 0.f;
      lse2[row] = i < S ? lse[(long long)bh * S + i] * LOG2E : INFINITY;
    }
  }
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

struct BwdParams {
  int S, S_pad, H;
  int causal;
  float scale, scale_log2;
  const float* lse2;
  const float* dvec;
  __nv_bfloat16* g0;   // dkdv: dk ; dq: dq
  __nv_bfloat16* g1;   // dkdv: dv
  long long st, sh;    // output (q layout) strides
  const float* rope;   // optional fp32 [2][S][D/2] cos|sin planes: inverse RoPE on dq / dk
  DropoutParams drop;  // attention-probability dropout (thresh 0 = off)
  int bh_total;        // batch * heads (work-item decode)
  int persist;         // 1: persistent CTAs (heaviest item first, (batch, head) fastest)
};

template <int D>
struct SmemKV {
  static constexpr int NST = 3;  // Q/dO pipeline depth
  static constexpr int KT = D * 128 * 2, QT = D * 64 * 2;
  static constexpr int K = 0, V = KT, Q0 = 2 * KT, O0 = Q0 + NST * QT;
  static constexpr int PT = O0 + NST * QT, DST = PT + 128 * 64 * 2;
  static constexpr int LSE = DST + 128 * 64 * 2, DV = LSE + NST * 64 * 4;
  static constexpr int BAR = DV + NST * 64 * 4;
  static constexpr int BYTES = BAR + 256 + 1024;
};

constexpr int BWD_SPLIT = 4;                    // math warps per TMEM lane quarter
constexpr int BWD_CP = 64 / BWD_SPLIT;          // columns per math warp (16)
constexpr int BWD_THREADS = 128 + 128 * BWD_SPLIT;

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 16 values of row r, column part `part` -> bf16 into a K-major SW128 [rows][64] tile
__device__ __forceinline__ void store_part_row(uint8_t* tile, int r, int part, const float* v) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    uint4 w = make_uint4(pack2(v[u * 8 + 0], v[u * 8 + 1]), pack2(v[u * 8 + 2], v[u * 8 + 3]),
                         pack2(v[u * 8 + 4], v[u * 8 + 5]), pack2(v[u * 8 + 6], v[u * 8 + 7]));
    *reinterpret_cast<uint4*>(tile + r * 128 + (((part * 2 + u) ^ (r & 7)) * 16)) = w;
  }
}

// rows of a half-row (32 values) -> bf16 into a K-major SW128 [rows][64] tile
__device__ __forceinline__ void store_half_row(uint8_t* tile, int r, int half, const float* v) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint4 w = make_uint4(pack2(v[u * 8 + 0], v[u * 8 + 1]), pack2(v[u * 8 + 2], v[u * 8 + 3]),
                         pack2(v[u * 8 + 4], v[u * 8 + 5]), pack2(v[u * 8 + 6], v[u * 8 + 7]));
    *reinterpret_cast<uint4*>(tile + r * 128 + (((half * 4 + u) ^ (r & 7)) * 16)) = w;
  }
}

__device__ __forceinline__ void store_row_out(__nv_bfloat16* dst, uint32_t taddr, float mul,
                                              bool write) {
  uint32_t ov[32];
  tmem_ld32(taddr, ov);  // warp-collective: every lane loads, only valid rows store
  if (!write) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint4 w;
    w.x = pack2(__uint_as_float(ov[u * 8 + 0]) * mul, __uint_as_float(ov[u * 8 + 1]) * mul);
    w.y = pack2(__uint_as_float(ov[u * 8 + 2]) * mul, __uint_as_float(ov[u * 8 + 3]) * mul);
    w.z = pack2(__uint_as_float(ov[u * 8 + 4]) * mul, __uint_as_float(ov[u * 8 + 5]) * mul);
    w.w = pack2(__uint_as_float(ov[u * 8 + 6]) * mul, __uint_as_float(ov[u * 8 + 7]) * mul);
    *reinterpret_cast<uint4*>(dst + u * 8) = w;
  }
}

// Inverse rotate-half RoPE fused into the dq / dk store (replaces the standalone
// rope_table_kernel pass over dq|dk, rope.cu): the warp's 32 columns [c0, c0+32) pair with
// the partner chunk c0 +- D/2, loaded from TMEM by the same warp (same lanes = same rows).
// Angles come from the fp32 table cs (cos plane, sin plane at +S*D/2) at the row's position.
//   j <  D/2:  out_j = x_j cos + x_{j+D/2} sin;   j >= D/2:  out_j = x_j cos - x_{j-D/2} sin
template <int D>
__device__ __forceinline__ void store_row_out_rope(__nv_bfloat16* dst, uint32_t t_self,
                                                   uint32_t t_pair, float mul, bool write,
                                                   const float* cs, int S, int pos, int c0) {
  uint32_t xv[32], yv[32];
  tmem_ld32_nowait(t_self, xv);
  tmem_ld32_nowait(t_pair, yv);
  tmem_wait_ld();
  if (!write) return;
  constexpr int HALF = D / 2;
  const float sgn = c0 < HALF ? 1.f : -1.f;
  const float* cr = cs + (long long)pos * HALF + (c0 & (HALF - 1));
  const float* sr = cr + (long long)S * HALF;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    float o[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 c = __ldg(reinterpret_cast<const float4*>(cr + u * 8 + h * 4));
      const float4 sn = __ldg(reinterpret_cast<const float4*>(sr + u * 8 + h * 4));
      const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = u * 8 + h * 4 + e;
        const float x = __uint_as_float(xv[i]) * mul, y = __uint_as_float(yv[i]) * mul;
        o[h * 4 + e] = x * cc[e] + sgn * y * ss[e];
      }
    }
    uint4 w;
    w.x = pack2(o[0], o[1]);
    w.y = pack2(o[2], o[3]);
    w.z = pack2(o[4], o[5]);
    w.w = pack2(o[6], o[7]);
    *reinterpret_cast<uint4*>(dst + u * 8) = w;
  }
}

// 16 output columns of one row: TMEM -> bf16 -> global (warp-collective load)
__device__ __forceinline__ void store_row_out16(__nv_bfloat16* dst, uint32_t taddr, float mul,
                                                bool write) {
  uint32_t ov[16];
  tmem_ld16_nowait(taddr, ov);
  tmem_wait_ld();
  if (!write) return;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    uint4 w;
    w.x = pack2(__uint_as_float(ov[u * 8 + 0]) * mul, __uint_as_float(ov[u * 8 + 1]) * mul);
    w.y = pack2(__uint_as_float(ov[u * 8 + 2]) * mul, __uint_as_float(ov[u * 8 + 3]) * mul);
    w.z = pack2(__uint_as_float(ov[u * 8 + 4]) * mul, __uint_as_float(ov[u * 8 + 5]) * mul);
    w.w = pack2(__uint_as_float(ov[u * 8 + 6]) * mul, __uint_as_float(ov[u * 8 + 7]) * mul);
    *reinterpret_cast<uint4*>(dst + u * 8) = w;
  }
}

template <int D, bool DROP>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    bwd_dkdv_tc(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                const BwdParams p) {
  using L = SmemKV<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared window
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  constexpr int NST = L::NST;
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;          // [NST]
  uint64_t* q_empty = q_full + NST;    // [NST]
  uint64_t* st_full = q_empty + NST;   // [2]
  uint64_t* st_empty = st_full + 2;    // [2]  buffer free once dV/dK of its step are done
  uint64_t* p_full = st_empty + 2;     // [2]  P^T / dS^T packed into the buffer (TMEM)
  uint64_t* mm_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mm_done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x;
  const int bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int k0 = kb * 128, tok0 = b * p.S;
  const int n_qb = (p.S + 63) / 64;
  const int i0 = p.causal ? (k0 / 64) : 0;
  const int n_it = n_qb - i0;
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
      mbar_init(&p_full[i], 128 * BWD_SPLIT);
    }
    mbar_init(mm_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dv = tmem + 256, t_dk = tmem + 384;
  const float* lse2_g = p.lse2 + (long long)bh * p.S_pad;
  const float* dv_g = p.dvec + (long long)bh * p.S_pad;

  if (warp == 0) {
    if (lane == 0 && n_it > 0) {
      mbar_expect_tx(kv_full, 2 * L::KT);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tma_load_3d(&mk, kv_full, sm + L::K + c * 16384, c * 64, h, tok0 + k0);
        tma_load_3d(&mv, kv_full, sm + L::V + c * 16384, c * 64, h, tok0 + k0);
      }
      for (int it = 0; it < n_it; ++it) {
        const int st = it % NST, q0 = (i0 + it) * 64;
        mbar_wait(&q_empty[st], ((it / NST) & 1) ^ 1);
        mbar_expect_tx(&q_full[st], 2 * L::QT + 512);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tma_load_3d(&mq, &q_full[st], sm + L::Q0 + st * L::QT + c * 8192, c * 64, h, tok0 + q0);
          tma_load_3d(&mdo, &q_full[st], sm + L::O0 + st * L::QT + c * 8192, c * 64, h, tok0 + q0);
        }
        bulk_load(sm + L::LSE + st * 256, lse2_g + q0, 256, &q_full[st]);
        bulk_load(sm + L::DV + st * 256, dv_g + q0, 256, &q_full[st]);
      }
    }
  } else if (warp == 1) {
    if (n_it > 0) {  // whole warp; elected lane issues (see fwd_tc)
      const uint32_t id_st = make_idesc(128, 64, 0, 0);
      const uint32_t id_g = make_idesc(128, D, 0, 1);
      const uint64_t d_k = sdesc(smem_u32(sm + L::K), 16, 1024);
      const uint64_t d_v = sdesc(smem_u32(sm + L::V), 16, 1024);
      const uint64_t d_q = sdesc(smem_u32(sm + L::Q0), 16, 1024);
      const uint64_t d_o = sdesc(smem_u32(sm + L::O0), 16, 1024);
      const uint64_t m_q = sdesc(smem_u32(sm + L::Q0), 8192, 1024);   // MN-major views
      const uint64_t m_o = sdesc(smem_u32(sm + L::O0), 8192, 1024);
      mbar_wait_fast(kv_full, 0);
      // dV += P^T dO, dK += dS^T Q with A read from TMEM (P^T / dS^T packed by the math
      // warps into the first 8 of every 16 columns of the S^T / dP^T buffer)
      auto grads = [&](int it) {
        const int st = it % NST, sb = it & 1;
        mbar_wait_fast(&p_full[sb], (it >> 1) & 1);
        tc_fence_after();
        if (lane == 0) TRACE(4096 + it * 8 + 3);
        const uint64_t so = (uint64_t)((st * L::QT) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_ts(t_dv, tmem + sb * 128 + k * 16, m_o + so + (uint64_t)((k * 2048) >> 4),
                         id_g, (it | k) != 0);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_ts(t_dk, tmem + sb * 128 + 64 + k * 16,
                         m_q + so + (uint64_t)((k * 2048) >> 4), id_g, (it | k) != 0);
          if (it == n_it - 1) umma_commit(mm_done);  // single phase: final dK/dV complete
          umma_commit(&st_empty[sb]);
          umma_commit(&q_empty[st]);
        }
        __syncwarp();
      };
      for (int it = 0; it < n_it; ++it) {
        const int st = it % NST, sb = it & 1;
        if (lane == 0) TRACE(4096 + it * 8 + 0);
        mbar_wait_fast(&q_full[st], (it / NST) & 1);
        if (lane == 0) TRACE(4096 + it * 8 + 2);
        mbar_wait_fast(&st_empty[sb], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) TRACE(4096 + it * 8 + 1);
        const uint64_t so = (uint64_t)((st * L::QT) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t oa = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
            const uint64_t ob = (uint64_t)(((k >> 2) * 8192 + (k & 3) * 32) >> 4);
            umma_bf16(tmem + sb * 128, d_k + oa, d_q + so + ob, id_st, k != 0);
          }
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t oa = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
            const uint64_t ob = (uint64_t)(((k >> 2) * 8192 + (k & 3) * 32) >> 4);
            umma_bf16(tmem + sb * 128 + 64, d_v + oa, d_o + so + ob, id_st, k != 0);
          }
          umma_commit(&st_full[sb]);
        }
        __syncwarp();
        if (it > 0) grads(it - 1);
      }
      grads(n_it - 1);
    }
  } else if (warp >= 4) {
    const int q = warp & 3, part = (warp - 4) >> 2;
    const int r = q * 32 + lane, key = k0 + r;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    for (int it = 0; it < n_it; ++it) {
      const int st = it % NST, sb = it & 1, q0 = (i0 + it) * 64;
      mbar_wait(&st_full[sb], (it >> 1) & 1);
      tc_fence_after();
      if (warp == 4 && lane == 0) TRACE(4096 + it * 8 + 4);
      float s[BWD_CP], dp[BWD_CP];
      tmem_ld16_nowait(tmem + sb * 128 + part * BWD_CP + lane_off, reinterpret_cast<uint32_t*>(s));
      tmem_ld16_nowait(tmem + sb * 128 + 64 + part * BWD_CP + lane_off,
                       reinterpret_cast<uint32_t*>(dp));
      tmem_wait_ld();
      if (warp == 4 && lane == 0) TRACE(4096 + it * 8 + 5);
      const float* l2 = reinterpret_cast<const float*>(sm + L::LSE + st * 256) + part * BWD_CP;
      const float* dd = reinterpret_cast<const float*>(sm + L::DV + st * 256) + part * BWD_CP;
      const int qbase = q0 + part * BWD_CP;
      const float sl2 = p.scale_log2;
      if constexpr (DROP) {
        // dropout: dV uses the kept, 1/(1-p)-scaled P; dS = P * (dP * mask / (1-p) - D)
        const int first = p.causal ? key - qbase : -1;
#pragma unroll
        for (int i = 0; i < BWD_CP; ++i) {
          const float pv = i >= first ? exp2_mufu(fmaf(s[i], sl2, -l2[i])) : 0.f;
          const float kp = dropout_keep(p.drop, b, h, qbase + i, key) ? p.drop.inv_keep : 0.f;
          s[i] = pv * kp;
          dp[i] = pv * (dp[i] * kp - dd[i]);
        }
      } else if (p.causal && key > qbase) {  // diagonal: queries < key are masked
        const int first = key - qbase;
#pragma unroll
        for (int i = 0; i < BWD_CP; ++i) {
          const float pv = i >= first ? exp2_mufu(fmaf(s[i], sl2, -l2[i])) : 0.f;
          s[i] = pv;
          dp[i] = pv * (dp[i] - dd[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < BWD_CP; ++i) {
          const float pv = exp2_mufu(fmaf(s[i], sl2, -l2[i]));
          s[i] = pv;
          dp[i] = pv * (dp[i] - dd[i]);
        }
      }
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) pk[i] = pack2(s[2 * i], s[2 * i + 1]);
      if (warp == 4 && lane == 0) TRACE(4096 + it * 8 + 6);
      tmem_st8(tmem + sb * 128 + part * BWD_CP + lane_off, pk);
#pragma unroll
      for (int i = 0; i < 8; ++i) pk[i] = pack2(dp[2 * i], dp[2 * i + 1]);
      tmem_st8(tmem + sb * 128 + 64 + part * BWD_CP + lane_off, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
      if (warp == 4 && lane == 0) TRACE(4096 + it * 8 + 7);
    }
    if (n_it > 0) {
      mbar_wait(mm_done, 0);
      tc_fence_after();
      const bool ok = key < p.S;
      constexpr int OC = D / BWD_SPLIT;  // output columns per warp
      const long long off =
          (long long)(tok0 + (ok ? key : 0)) * p.st + (long long)h * p.sh + part * OC;
      if constexpr (OC >= 32) {
#pragma unroll 1
        for (int c = 0; c < OC / 32; ++c) {
          const int c0 = part * OC + c * 32;
          store_row_out(p.g1 + off + c * 32, t_dv + c0 + lane_off, 1.f, ok);
          if (p.rope != nullptr)
            store_row_out_rope<D>(p.g0 + off + c * 32, t_dk + c0 + lane_off,
                                  t_dk + ((c0 + D / 2) & (D - 1)) + lane_off, p.scale, ok,
                                  p.rope, p.S, ok ? key : 0, c0);
          else
            store_row_out(p.g0 + off + c * 32, t_dk + c0 + lane_off, p.scale, ok);
        }
      } else {
        store_row_out16(p.g1 + off, t_dv + part * OC + lane_off, 1.f, ok);
        store_row_out16(p.g0 + off, t_dk + part * OC + lane_off, p.scale, ok);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// dkdv, 128-query steps (default): CTA = 128 keys.  The N=128 score MMAs read 8 KB of smem
// per 64 tensor cycles (the N=64 ones of bwd_dkdv_tc read 6 KB per 32 and are smem-bound).
// TMEM (512 columns at D=128): S^T [0,128), dP^T [128,256), dV [256,256+D), dK [256+D,..).
// The scores are single-buffered; instead the MMA warp interleaves two steps so that each
// softmax phase overlaps other MMAs:
//     ... dV(it-1) S(it) dK(it-1) dP(it) | dV(it) S(it+1) dK(it) dP(it+1) | ...
//   phase 1 (P^T = exp2(S^T - lse), packed bf16 over S^T) runs under dK(it-1), dP(it)
//   phase 2 (dS^T = P^T (dP^T - D), packed over dP^T) runs under dV(it), S(it+1)
// Both phases go in two query halves with their own barriers, so dV / dK over the first
// 64 queries start while the second half is computed (phase 1 is MUFU-bound: 16K exp2 per
// step = 1024 cycles at 16/clk/SM; measured period 2730 cycles per 128-query step vs 3400
// for two 64-query steps of bwd_dkdv_tc).  tcgen05.mma from one thread execute in issue
// order, so S(it+1) (issued after dV(it)) never overwrites P^T(it) before dV has read it;
// likewise dP(it+1) after dK(it).  Q (+ lse, D vectors) and dO come through separate
// 2-stage rings: dO(it) is released by dV(it), Q(it) by dK(it), the last reader of the
// step's vectors being phase 2 (before dK(it) issues).  Splitting S(it+1) into two N=64
// halves (so S half 0 can follow dV half 0) measured slower (period 3010): N=64 score MMAs
// are smem-bound.
// every DKDV_POLY-th phase-1 exponential on the FMA pipe: measured neutral to slower (poly 4:
// 925-929 vs 907-934 us at B2 S4096 H32; poly 2: 993): the phase is issue-bound once the
// polynomial's ~11 instructions are added.  0 = all on MUFU.
#ifndef DKDV_POLY
#define DKDV_POLY 0
#endif
// Grid order of the backward kernels.  1 = (batch, head) fastest, i.e. the whole grid issued
// heaviest-first (what the forward does); measured slower for both backward kernels on B200
// (B2 S4096 H32: 941-958 vs 921 us, B4 S8192 H16: 3785-4110 vs 3627 us): a key (query)
// block sweeps every query (key) block of its head, and with the blocks of one head running
// side by side those sweeps share L2.  0 = block index fastest (heaviest-first per head).
// (Two MMA-issuing warps for the dK/dV kernel, chain A = dV, S and chain B = dK, dP on
// disjoint TMEM, measured slower: 936 vs 884 us at B2 S4096 H32 -- the tensor pipe then runs
// dP(it+1) ahead of S(it+1).  profiles/r02/attention/bwd2/.)
#ifndef ATTN_BWD_PERSIST_MAX_S
#define ATTN_BWD_PERSIST_MAX_S 2048
#endif
#ifndef DKDV_GRID_BH_FAST
#define DKDV_GRID_BH_FAST 0
#endif
#ifndef DQ_GRID_BH_FAST
#define DQ_GRID_BH_FAST 0
#endif
template <int D>
struct SmemKV2 {
  static constexpr int NST = 2;
  static constexpr int KVB = D == 64 ? 2 : 1;  // K/V buffers (persistent CTAs prefetch the next item's)
  static constexpr int KT = D * 128 * 2;       // every tile is 128 rows x D
  static constexpr int KV = 0, Q0 = KVB * 2 * KT, O0 = Q0 + NST * KT;
  static constexpr int LSE = O0 + NST * KT, DV = LSE + NST * 512;
  static constexpr int BAR = DV + NST * 512;
  static constexpr int BYTES = BAR + 256 + 1024;
};

// Work items (key block, batch*head): one per CTA, or persistent CTAs looping over items c,
// c + gridDim.x, ... (short sequences; see bwd_ctas).  Persistent order is heaviest key block
// first with (batch, head) fastest (balanced round-robin); one-per-CTA order is key block
// fastest (the head's sweeps share L2, DKDV_GRID_BH_FAST).  Between items, the K/V buffers
// are handed over by kv_empty / kv_full and the dK/dV accumulators by acc_free (the
// epilogue has read them); every per-step barrier's parity runs on the CTA's global step count.
template <int D, bool DROP>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    bwd_dkdv2_tc(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                 const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                 const BwdParams p) {
  using L = SmemKV2<D>;
  constexpr int NST = L::NST, KVB = L::KVB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* kv_full = bar + 0;          // [KVB]
  uint64_t* kv_empty = kv_full + KVB;   // [KVB]
  uint64_t* q_full = kv_empty + KVB;    // [NST] Q tile + lse2 / D vectors
  uint64_t* q_empty = q_full + NST;     // [NST]
  uint64_t* o_full = q_empty + NST;     // [NST] dO tile
  uint64_t* o_empty = o_full + NST;     // [NST]
  uint64_t* s_full = o_empty + NST;     // S^T(it) complete
  uint64_t* dp_full = s_full + 1;       // dP^T(it) complete
  uint64_t* p_full = dp_full + 1;       // [2] P^T(it) query half packed (all math threads)
  uint64_t* ds_full = p_full + 2;       // [2] dS^T(it) query half packed (all math threads)
  uint64_t* mm_done = ds_full + 2;      // the item's last dK / dV MMA complete
  uint64_t* acc_free = mm_done + 1;     // the item's epilogue has read dK / dV
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qb = (p.S + 127) / 128;
  const int n_items = n_qb * p.bh_total;
  struct Item {
    int b, h, bh, k0, i0, n_it, tok0;
  };
  auto decode = [&](int w) {
    Item I;
    int kb;
    if (p.persist || DKDV_GRID_BH_FAST) {
      kb = w / p.bh_total;
      I.bh = w % p.bh_total;
    } else {
      kb = w % n_qb;
      I.bh = w / n_qb;
    }
    I.b = I.bh / p.H;
    I.h = I.bh % p.H;
    I.k0 = kb * 128;
    I.i0 = p.causal ? kb : 0;  // causal: low key blocks carry the most query blocks
    I.n_it = n_qb - I.i0;
    I.tok0 = I.b * p.S;
    return I;
  };
  if (threadIdx.x == 0) TRACE(4096 + 16 * 64 + 3);
  if (threadIdx.x == 0) {
    for (int i = 0; i < KVB; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < NST; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], 128 * BWD_SPLIT);
      mbar_init(&ds_full[i], 128 * BWD_SPLIT);
    }
    mbar_init(mm_done, 1);
    mbar_init(acc_free, 128 * BWD_SPLIT);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 256 + D;

  if (warp == 0) {  // Q ring (+ vectors)
    if (lane == 0) {
      uint32_t g = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const Item I = decode(w);
        const float* lse2_g = p.lse2 + (long long)I.bh * p.S_pad;
        const float* dv_g = p.dvec + (long long)I.bh * p.S_pad;
        for (int it = 0; it < I.n_it; ++it, ++g) {
          const int st = g % NST, q0 = (I.i0 + it) * 128;
          mbar_wait(&q_empty[st], ((g / NST) & 1) ^ 1);
          mbar_expect_tx(&q_full[st], L::KT + 1024);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(&mq, &q_full[st], sm + L::Q0 + st * L::KT + c * 16384, c * 64, I.h,
                        I.tok0 + q0);
          bulk_load(sm + L::LSE + st * 512, lse2_g + q0, 512, &q_full[st]);
          bulk_load(sm + L::DV + st * 512, dv_g + q0, 512, &q_full[st]);
        }
      }
    }
  } else if (warp == 2) {  // K / V per item (after the TMEM allocation)
    if (lane == 0) {
      int n = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n) {
        const Item I = decode(w);
        const int kb = n % KVB;
        mbar_wait(&kv_empty[kb], ((n / KVB) & 1) ^ 1);
        mbar_expect_tx(&kv_full[kb], 2 * L::KT);
        uint8_t* kvs = sm + L::KV + kb * 2 * L::KT;
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tma_load_3d(&mk, &kv_full[kb], kvs + c * 16384, c * 64, I.h, I.tok0 + I.k0);
          tma_load_3d(&mv, &kv_full[kb], kvs + L::KT + c * 16384, c * 64, I.h, I.tok0 + I.k0);
        }
      }
    }
  } else if (warp == 3) {  // dO ring
    if (lane == 0) {
      uint32_t g = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const Item I = decode(w);
        for (int it = 0; it < I.n_it; ++it, ++g) {
          const int st = g % NST, q0 = (I.i0 + it) * 128;
          mbar_wait(&o_empty[st], ((g / NST) & 1) ^ 1);
          mbar_expect_tx(&o_full[st], L::KT);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(&mdo, &o_full[st], sm + L::O0 + st * L::KT + c * 16384, c * 64, I.h,
                        I.tok0 + q0);
        }
      }
    }
  } else if (warp == 1) {
    // issue order dV(it) S(it+1) dK(it) dP(it+1): S(it+1) overwrites the S^T columns dV(it)
    // has read, dP(it+1) the dP^T columns dK(it) has read (one thread's MMAs run in order)
    const uint32_t id_s = make_idesc(128, 128, 0, 0);
    const uint32_t id_g = make_idesc(128, D, 0, 1);
    const uint64_t d_q = sdesc(smem_u32(sm + L::Q0), 16, 1024);
    const uint64_t d_o = sdesc(smem_u32(sm + L::O0), 16, 1024);
    const uint64_t m_q = sdesc(smem_u32(sm + L::Q0), 16384, 1024);  // MN-major views
    const uint64_t m_o = sdesc(smem_u32(sm + L::O0), 16384, 1024);
    auto so = [&](uint32_t g) { return (uint64_t)(((g % NST) * L::KT) >> 4); };
    auto scores = [&](uint32_t dst, uint64_t da, uint64_t db) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t o = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
          umma_bf16(dst, da + o, db + o, id_s, k != 0);
        }
      }
    };
    // dst += A^T B over query half hf, A^T packed in TMEM (queries 16k.. at col 16k of src)
    auto grad = [&](uint32_t dst, uint32_t src, uint64_t mb, int hf, bool acc) {
      if (elect_one()) {
#pragma unroll
        for (int k = 4 * hf; k < 4 * hf + 4; ++k)
          umma_bf16_ts(dst, src + k * 16, mb + (uint64_t)((k * 2048) >> 4), id_g, acc || k != 0);
      }
    };
    uint32_t g0 = 0;
    int n = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n) {
      const Item I = decode(w);
      const int n_it = I.n_it, kb = n % KVB;
      const uint64_t d_k = sdesc(smem_u32(sm + L::KV + kb * 2 * L::KT), 16, 1024);
      const uint64_t d_v = sdesc(smem_u32(sm + L::KV + kb * 2 * L::KT + L::KT), 16, 1024);
      auto s_mma = [&](uint32_t g) {
        mbar_wait_fast(&q_full[g % NST], (g / NST) & 1);
        tc_fence_after();
        scores(tmem, d_k, d_q + so(g));
        if (elect_one()) umma_commit(s_full);
        __syncwarp();
      };
      auto dp_mma = [&](uint32_t g) {
        mbar_wait_fast(&o_full[g % NST], (g / NST) & 1);
        tc_fence_after();
        scores(t_dp, d_v, d_o + so(g));
        if (elect_one()) umma_commit(dp_full);
        __syncwarp();
      };
      mbar_wait_fast(&kv_full[kb], (n / KVB) & 1);
      if (n == 0 && lane == 0) TRACE(4096 + 16 * 64 + 2);
      s_mma(g0);
      dp_mma(g0);
      if (n > 0) mbar_wait_fast(acc_free, (n - 1) & 1);  // dK / dV of the last item read out
      for (int it = 0; it < n_it; ++it) {
        const uint32_t g = g0 + it;
        const int st = g % NST;
        const bool more = it + 1 < n_it;
        if (n == 0 && lane == 0) TRACE(4096 + it * 16 + 0);
        mbar_wait_fast(&p_full[0], g & 1);
        tc_fence_after();
        if (n == 0 && lane == 0) TRACE(4096 + it * 16 + 1);
        grad(t_dv, tmem, m_o + so(g), 0, it != 0);
        __syncwarp();
        mbar_wait_fast(&p_full[1], g & 1);
        tc_fence_after();
        grad(t_dv, tmem, m_o + so(g), 1, true);
        if (elect_one()) umma_commit(&o_empty[st]);
        __syncwarp();
        if (n == 0 && lane == 0) TRACE(4096 + it * 16 + 2);
        if (more) s_mma(g + 1);
        mbar_wait_fast(&ds_full[0], g & 1);
        tc_fence_after();
        if (n == 0 && lane == 0) TRACE(4096 + it * 16 + 3);
        grad(t_dk, t_dp, m_q + so(g), 0, it != 0);
        __syncwarp();
        mbar_wait_fast(&ds_full[1], g & 1);
        tc_fence_after();
        grad(t_dk, t_dp, m_q + so(g), 1, true);
        if (elect_one()) {
          umma_commit(&q_empty[st]);
          if (!more) {
            umma_commit(mm_done);
            umma_commit(&kv_empty[kb]);
          }
        }
        __syncwarp();
        if (n == 0 && lane == 0) TRACE(4096 + it * 16 + 4);
        if (more) dp_mma(g + 1);
      }
      g0 += n_it;
    }
  } else if (warp >= 4) {
    // part p owns query columns [16p, 16p+16) (half 0) and [64+16p, 64+16p+16) (half 1), so
    // the packed bf16 of query slice k lands on the thread's own columns 16k.. and the dV / dK
    // MMAs of half 0 start while half 1 is still being computed
    const int q = warp & 3, part = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float sl2 = p.scale_log2;
    uint32_t g0 = 0;
    int n = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n) {
    const Item I = decode(w);
    const int b = I.b, h = I.h, tok0 = I.tok0, key = I.k0 + r, n_it = I.n_it;
    const bool tr = n == 0 && warp == 4 && lane == 0;
    for (int it = 0; it < n_it; ++it) {
      const uint32_t g = g0 + it;
      const int st = g % NST, q0 = (I.i0 + it) * 128;
      const float* l2 = reinterpret_cast<const float*>(sm + L::LSE + st * 512) + part * 16;
      const float* dd = reinterpret_cast<const float*>(sm + L::DV + st * 512) + part * 16;
      // ---- phase 1: P^T
      mbar_wait(s_full, g & 1);
      tc_fence_after();
      if (tr) TRACE(4096 + it * 16 + 8);
      float pv[32];
      tmem_ld16_nowait(tmem + part * 16 + lane_off, reinterpret_cast<uint32_t*>(pv));
      tmem_ld16_nowait(tmem + 64 + part * 16 + lane_off, reinterpret_cast<uint32_t*>(pv + 16));
      tmem_wait_ld();
      if (tr) TRACE(4096 + it * 16 + 13);
      uint32_t keep = 0xffffffffu;
      if constexpr (DROP) {
        keep = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          keep |= (uint32_t)dropout_keep(p.drop, b, h, q0 + (i >> 4) * 64 + part * 16 + (i & 15),
                                         key) << i;
      }
      // every DKDV_POLY-th exponential on the FMA pipe (exp2_fma, rel err 5e-6); 0 = MUFU only
      auto ex = [](int i, float x) {
        if constexpr (DKDV_POLY > 0) {
          if (i % (DKDV_POLY > 0 ? DKDV_POLY : 1) == DKDV_POLY - 1) return exp2_fma(x);
        }
        return exp2_mufu(x);
      };
      uint32_t pk[8];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float* v = pv + hf * 16;
        const float* lh = l2 + hf * 64;
        const int qb = q0 + hf * 64 + part * 16;
        if (p.causal && key > qb) {  // diagonal block: queries < key are masked
          const int first = key - qb;
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = i >= first ? ex(i, fmaf(v[i], sl2, -lh[i])) : 0.f;
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = ex(i, fmaf(v[i], sl2, -lh[i]));
        }
        if constexpr (DROP) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c = hf * 16 + 2 * i;
            pk[i] = pack2((keep >> c) & 1u ? v[2 * i] * p.drop.inv_keep : 0.f,
                          (keep >> (c + 1)) & 1u ? v[2 * i + 1] * p.drop.inv_keep : 0.f);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) pk[i] = pack2(v[2 * i], v[2 * i + 1]);
        }
        tmem_st8(tmem + hf * 64 + part * 16 + lane_off, pk);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[hf]);
        if (tr) TRACE(4096 + it * 16 + 9 + hf);
      }
      // ---- phase 2: dS^T = P^T (dP^T * mask / (1-p) - D)
      mbar_wait(dp_full, g & 1);
      tc_fence_after();
      if (tr) TRACE(4096 + it * 16 + 11);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float dp[16];
        tmem_ld16_nowait(t_dp + hf * 64 + part * 16 + lane_off, reinterpret_cast<uint32_t*>(dp));
        tmem_wait_ld();
        if (tr && hf == 0) TRACE(4096 + it * 16 + 14);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = hf * 16 + i;
          float g = dp[i];
          if constexpr (DROP) g = (keep >> c) & 1u ? g * p.drop.inv_keep : 0.f;
          dp[i] = pv[c] * (g - dd[hf * 64 + i]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) pk[i] = pack2(dp[2 * i], dp[2 * i + 1]);
        tmem_st8(t_dp + hf * 64 + part * 16 + lane_off, pk);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&ds_full[hf]);
      }
      if (tr) TRACE(4096 + it * 16 + 12);
    }
    {
      mbar_wait(mm_done, n & 1);
      tc_fence_after();
      if (tr) TRACE(4096 + 16 * 64 + 0);
      const bool ok = key < p.S;
      constexpr int OC = D / BWD_SPLIT;  // output columns per warp
      const long long off =
          (long long)(tok0 + (ok ? key : 0)) * p.st + (long long)h * p.sh + part * OC;
      if constexpr (OC >= 32) {
#pragma unroll 1
        for (int c = 0; c < OC / 32; ++c) {
          const int c0 = part * OC + c * 32;
          store_row_out(p.g1 + off + c * 32, t_dv + c0 + lane_off, 1.f, ok);
          if (p.rope != nullptr)
            store_row_out_rope<D>(p.g0 + off + c * 32, t_dk + c0 + lane_off,
                                  t_dk + ((c0 + D / 2) & (D - 1)) + lane_off, p.scale, ok,
                                  p.rope, p.S, ok ? key : 0, c0);
          else
            store_row_out(p.g0 + off + c * 32, t_dk + c0 + lane_off, p.scale, ok);
        }
      } else {
        store_row_out16(p.g1 + off, t_dv + part * OC + lane_off, 1.f, ok);
        store_row_out16(p.g0 + off, t_dk + part * OC + lane_off, p.scale, ok);
      }
      if (tr) TRACE(4096 + 16 * 64 + 1);
      tc_fence_before();
      mbar_arrive(acc_free);  // dK / dV are out of TMEM: the next item may overwrite them
    }
    g0 += n_it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// dq kernel: CTA = 128 queries, 128-key steps.  TMEM: S double-buffered (cols 0-255), dP
// single (256-383; released as soon as the math warps have loaded it), dQ (384-).  dS is
// packed (bf16) over the first half of its own S columns and read from TMEM as the A
// operand of dQ += dS K, so S(it+1)/dP(it+1) overlap the softmax of step it and only the
// dQ MMA of step it-1 separates them.
template <int D>
struct SmemQ {
  // K is used by S(it) and dQ(it) (released late), V only by dP(it): separate rings, K one
  // stage deeper so its TMA load for step it+2 starts a full step before S(it+2) needs it.
  // Q / dO: QOB buffers (persistent CTAs load the next item's while this one runs; D=64 only,
  // D=128 has no shared memory left for a second pair)
  static constexpr int NK = 3, NV = 2, QOB = D == 64 ? 2 : 1;
  static constexpr int QT = D * 128 * 2, KT = D * 128 * 2;
  static constexpr int QO = 0, K0 = QOB * 2 * QT, V0 = K0 + NK * KT;
  static constexpr int BAR = V0 + NV * KT;
  static constexpr int BYTES = BAR + 256 + 1024;
};

// Work items (query block, batch*head): one per CTA (query block fastest, heaviest first per
// head, DQ_GRID_BH_FAST) or persistent CTAs for short sequences (heaviest block first over the
// whole grid, (batch, head) fastest).  Q/dO buffers are handed over by qo_empty (the item's
// last S and dP done: one commit from each issuing warp) and the dQ accumulator by acc_free.
// MMA issuers: warp 1 issues S(it) and dQ(it-1); warp 2 issues dP(it) as soon as the math
// warps have loaded dP(it-1), so it never queues behind warp 1's waits for dS (measured B2
// S4096 H32 whole backward 912 -> 895 us, period 2080 -> 1860 cycles per 128-key step, where
// the step's smem traffic -- 224 KB: S and dP read A and B, dQ reads B, TMA writes K and V --
// is 1750 cycles at 128 B/clk; issuing dQ(it-2), dP(it), S(it) from one warp was neutral).
template <int D, bool DROP>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    bwd_dq_tc(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
              const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
              const BwdParams p) {
  using L = SmemQ<D>;
  constexpr int QOB = L::QOB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared window
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* qo_full = bar + 0;          // [QOB]
  uint64_t* qo_empty = qo_full + QOB;   // [QOB]
  uint64_t* k_full = qo_empty + QOB;    // [NK]
  uint64_t* k_empty = k_full + L::NK;   // [NK]
  uint64_t* v_full = k_empty + L::NK;   // [NV]
  uint64_t* v_empty = v_full + L::NV;   // [NV]
  uint64_t* st_full = v_empty + L::NV;  // [2]  S (buffer sb) computed
  uint64_t* ds_full = st_full + 2;      // [2]  dS packed into the S buffer
  uint64_t* dp_free = ds_full + 2;      // dP loaded by every math thread
  uint64_t* dq_done = dp_free + 1;      // the item's last dQ MMA complete
  uint64_t* dp_full = dq_done + 1;      // dP(it) complete
  uint64_t* acc_free = dp_full + 1;     // the item's epilogue has read dQ
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_q = (p.S + 127) / 128;
  const int n_kb = n_q;
  const int n_items = n_q * p.bh_total;
  struct Item {
    int b, h, bh, q0, n_it, tok0;
  };
  auto decode = [&](int w) {
    Item I;
    int qb;
    if (p.persist || DQ_GRID_BH_FAST) {
      qb = n_q - 1 - w / p.bh_total;
      I.bh = w % p.bh_total;
    } else {
      qb = n_q - 1 - w % n_q;
      I.bh = w / n_q;
    }
    I.b = I.bh / p.H;
    I.h = I.bh % p.H;
    I.q0 = qb * 128;
    I.n_it = p.causal ? min(n_kb, qb + 1) : n_kb;
    I.tok0 = I.b * p.S;
    return I;
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < QOB; ++i) {
      mbar_init(&qo_full[i], 1);
      mbar_init(&qo_empty[i], 2);  // last S (warp 1) + last dP (warp 2)
    }
    for (int i = 0; i < L::NK; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < L::NV; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&ds_full[i], 128 * BWD_SPLIT);
    }
    mbar_init(dp_free, 128 * BWD_SPLIT);
    mbar_init(dq_done, 1);
    mbar_init(dp_full, 1);
    mbar_init(acc_free, 128 * BWD_SPLIT);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dp = tmem + 256, t_dq = tmem + 384;

  if (warp == 0) {  // Q / dO per item, K ring
    if (lane == 0) {
      uint32_t g = 0;
      int n = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n) {
        const Item I = decode(w);
        const int qb = n % QOB;
        mbar_wait(&qo_empty[qb], ((n / QOB) & 1) ^ 1);
        mbar_expect_tx(&qo_full[qb], 2 * L::QT);
        uint8_t* qo = sm + L::QO + qb * 2 * L::QT;
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tma_load_3d(&mq, &qo_full[qb], qo + c * 16384, c * 64, I.h, I.tok0 + I.q0);
          tma_load_3d(&mdo, &qo_full[qb], qo + L::QT + c * 16384, c * 64, I.h, I.tok0 + I.q0);
        }
        for (int it = 0; it < I.n_it; ++it, ++g) {
          const int st = g % L::NK;
          mbar_wait(&k_empty[st], ((g / L::NK) & 1) ^ 1);
          mbar_expect_tx(&k_full[st], L::KT);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(&mk, &k_full[st], sm + L::K0 + st * L::KT + c * 16384, c * 64, I.h,
                        I.tok0 + it * 128);
        }
      }
    }
  } else if (warp == 3) {  // V ring
    if (lane == 0) {
      uint32_t g = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const Item I = decode(w);
        for (int it = 0; it < I.n_it; ++it, ++g) {
          const int st = g % L::NV;
          mbar_wait(&v_empty[st], ((g / L::NV) & 1) ^ 1);
          mbar_expect_tx(&v_full[st], L::KT);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(&mv, &v_full[st], sm + L::V0 + st * L::KT + c * 16384, c * 64, I.h,
                        I.tok0 + it * 128);
        }
      }
    }
  } else if (warp == 2) {  // dP issuer (after the TMEM allocation)
    const uint32_t id_s = make_idesc(128, 128, 0, 0);
    const uint64_t d_v = sdesc(smem_u32(sm + L::V0), 16, 1024);
    uint32_t g = 0;
    int n = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n) {
      const Item I = decode(w);
      const int qb = n % QOB;
      const uint64_t d_o = sdesc(smem_u32(sm + L::QO + qb * 2 * L::QT + L::QT), 16, 1024);
      mbar_wait_fast(&qo_full[qb], (n / QOB) & 1);
      for (int it = 0; it < I.n_it; ++it, ++g) {
        const int sv = g % L::NV;
        mbar_wait_fast(&v_full[sv], (g / L::NV) & 1);
        if (g > 0) mbar_wait_fast(dp_free, (g - 1) & 1);
        tc_fence_after();
        if (n == 0 && lane == 0) TRACE(it * 8 + 2);
        const uint64_t ov = (uint64_t)((sv * L::KT) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t o = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
            umma_bf16(t_dp, d_o + o, d_v + ov + o, id_s, k != 0);
          }
          umma_commit(dp_full);
          umma_commit(&v_empty[sv]);
          if (it == I.n_it - 1) umma_commit(&qo_empty[qb]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // S and dQ issuer
    const uint32_t id_s = make_idesc(128, 128, 0, 0);
    const uint32_t id_g = make_idesc(128, D, 0, 1);
    const uint64_t d_k = sdesc(smem_u32(sm + L::K0), 16, 1024);
    const uint64_t m_k = sdesc(smem_u32(sm + L::K0), 16384, 1024);  // K as MN-major B
    uint32_t g0 = 0;
    int n = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n) {
      const Item I = decode(w);
      const int n_it = I.n_it, qb = n % QOB;
      const uint64_t d_q = sdesc(smem_u32(sm + L::QO + qb * 2 * L::QT), 16, 1024);
      mbar_wait_fast(&qo_full[qb], (n / QOB) & 1);
      // dQ += dS K: A = dS from TMEM (keys 16k.. packed at col 32*(k/2) + 8*(k%2) of the S
      // buffer), B = the K tile as an MN-major operand (same smem bytes as the S GEMM's B)
      auto grads = [&](int it) {
        const uint32_t g = g0 + it;
        const int st = g % L::NK, sb = g & 1;
        if (it == 0 && n > 0) mbar_wait_fast(acc_free, (n - 1) & 1);  // last item's dQ read
        mbar_wait_fast(&ds_full[sb], (g >> 1) & 1);
        tc_fence_after();
        if (n == 0 && lane == 0) TRACE(it * 8 + 3);
        const uint64_t so = (uint64_t)((st * L::KT) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            umma_bf16_ts(t_dq, tmem + sb * 128 + (k >> 1) * 32 + (k & 1) * 8,
                         m_k + so + (uint64_t)((k * 2048) >> 4), id_g, (it | k) != 0);
          if (it == n_it - 1) umma_commit(dq_done);
          umma_commit(&k_empty[st]);
        }
        __syncwarp();
      };
      // S(it) into buffer g&1: this warp issued dQ(g-2), the buffer's last reader, before it
      // (one thread's MMAs execute in issue order), so no completion wait is needed
      auto s_mma = [&](int it) {
        const uint32_t g = g0 + it;
        const int sk = g % L::NK, sb = g & 1;
        mbar_wait_fast(&k_full[sk], (g / L::NK) & 1);
        tc_fence_after();
        if (n == 0 && lane == 0) TRACE(it * 8 + 1);
        const uint64_t ok = (uint64_t)((sk * L::KT) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t o = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
            umma_bf16(tmem + sb * 128, d_q + o, d_k + ok + o, id_s, k != 0);
          }
          umma_commit(&st_full[sb]);
          if (it == n_it - 1) umma_commit(&qo_empty[qb]);
        }
        __syncwarp();
      };
      for (int it = 0; it < n_it; ++it) {
        if (n == 0 && lane == 0) TRACE(it * 8 + 0);
        s_mma(it);
        if (it > 0) grads(it - 1);
      }
      grads(n_it - 1);
      g0 += n_it;
    }
  } else if (warp >= 4) {
    const int q = warp & 3, part = (warp - 4) >> 2;  // part: keys [32 part, 32 part + 32)
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float sl2 = p.scale_log2;
    uint32_t g0 = 0;
    int n = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++n) {
    const Item I = decode(w);
    const int b = I.b, h = I.h, tok0 = I.tok0, qi = I.q0 + r, n_it = I.n_it;
    const float l2 = p.lse2[(long long)I.bh * p.S_pad + qi];
    const float dd = p.dvec[(long long)I.bh * p.S_pad + qi];
    const bool tr = n == 0 && warp == 4 && lane == 0;
    for (int it = 0; it < n_it; ++it) {
      const uint32_t g = g0 + it;
      const int sb = g & 1;
      mbar_wait(&st_full[sb], (g >> 1) & 1);
      mbar_wait(dp_full, g & 1);
      tc_fence_after();
      if (tr) TRACE(it * 8 + 4);
      float s[32], dp[32];
      tmem_ld32_nowait(tmem + sb * 128 + part * 32 + lane_off, reinterpret_cast<uint32_t*>(s));
      tmem_ld32_nowait(t_dp + part * 32 + lane_off, reinterpret_cast<uint32_t*>(dp));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(dp_free);
      if (tr) TRACE(it * 8 + 5);
      const int kbase = it * 128 + part * 32;
      if constexpr (DROP) {
        const int lim = (p.causal ? min(p.S, qi + 1) : p.S) - kbase;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const uint32_t keep = dropout_keep4(p.drop, b, h, qi, kbase + g * 4);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = g * 4 + e;
            const float pv = i < lim ? exp2_mufu(fmaf(s[i], sl2, -l2)) : 0.f;
            const float kp = (keep >> e) & 1u ? p.drop.inv_keep : 0.f;
            dp[i] = pv * (dp[i] * kp - dd);
          }
        }
      } else if ((kbase + 32 > p.S) || (p.causal && kbase + 31 > qi)) {
        const int lim = (p.causal ? min(p.S, qi + 1) : p.S) - kbase;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float pv = i < lim ? exp2_mufu(fmaf(s[i], sl2, -l2)) : 0.f;
          dp[i] = pv * (dp[i] - dd);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float pv = exp2_mufu(fmaf(s[i], sl2, -l2));
          dp[i] = pv * (dp[i] - dd);
        }
      }
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = pack2(dp[2 * i], dp[2 * i + 1]);
      if (tr) TRACE(it * 8 + 6);
      tmem_st8(tmem + sb * 128 + part * 32 + lane_off, pk);
      tmem_st8(tmem + sb * 128 + part * 32 + 8 + lane_off, pk + 8);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ds_full[sb]);
      if (tr) TRACE(it * 8 + 7);
    }
    mbar_wait(dq_done, n & 1);
    tc_fence_after();
    const bool ok = qi < p.S;
    constexpr int OC = D / BWD_SPLIT;
    const long long off =
        (long long)(tok0 + (ok ? qi : 0)) * p.st + (long long)h * p.sh + part * OC;
    if constexpr (OC >= 32) {
#pragma unroll 1
      for (int c = 0; c < OC / 32; ++c) {
        const int c0 = part * OC + c * 32;
        if (p.rope != nullptr)
          store_row_out_rope<D>(p.g0 + off + c * 32, t_dq + c0 + lane_off,
                                t_dq + ((c0 + D / 2) & (D - 1)) + lane_off, p.scale, ok, p.rope,
                                p.S, ok ? qi : 0, c0);
        else
          store_row_out(p.g0 + off + c * 32, t_dq + c0 + lane_off, p.scale, ok);
      }
    } else {
      store_row_out16(p.g0 + off, t_dq + part * OC + lane_off, p.scale, ok);
    }
    tc_fence_before();
    mbar_arrive(acc_free);  // dQ is out of TMEM: the next item may overwrite it
    g0 += n_it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 3-D map over [tokens, heads, head_dim] with box [128 tokens, 1 head, 64 dims]
static bool qkv_map(CUtensorMap* m, const void* base, int64_t tokens, int64_t H, int64_t D,
                    int64_t st, int64_t sh, uint32_t rows = 128) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)tokens};
  cuuint64_t strides[2] = {(cuuint64_t)sh * 2, (cuuint64_t)st * 2};
  cuuint32_t box[3] = {64, 1, rows};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// GALV_ATTN_FWD=1 selects the one-Q-tile forward (fwd_tc) for A/B runs
static bool fwd_two_tiles() {
  static const bool two = [] {
    const char* e = getenv("GALV_ATTN_FWD");
    return !(e && e[0] == '1');
  }();
  return two;
}

// Forward CTA count: persistent CTAs (one per SM) for short sequences, one CTA per work item
// otherwise.  Measured (same box, `profiles/r02/attention/persistent/`): B16 S1024 H16 D64
// 141 -> 120 us, B8 S2048 H16 D64 190-196 -> 184 us, but B2 S4096 H32 D128 280 -> 292 and
// B1 S32768 H8 1884 -> 2000+ (the static round-robin of long items balances worse than the
// hardware block scheduler).  GALV_ATTN_FWD_CTAS overrides (0 = one CTA per item).
static int fwd_ctas(int64_t S) {
  static const int env = [] {
    const char* e = getenv("GALV_ATTN_FWD_CTAS");
    return e ? atoi(e) : -1;
  }();
  if (env >= 0) return env;
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return S <= ATTN_FWD_PERSIST_MAX_S ? sms : 0;
}

// Backward CTA count (dK/dV kernel): persistent CTAs for short sequences as in the forward.
// GALV_ATTN_BWD_CTAS overrides (0 = one CTA per item).
static int bwd_ctas(int64_t S) {
  static const int env = [] {
    const char* e = getenv("GALV_ATTN_BWD_CTAS");
    return e ? atoi(e) : -1;
  }();
  if (env >= 0) return env;
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return S <= ATTN_BWD_PERSIST_MAX_S ? sms : 0;
}

// GALV_ATTN_DKDV=1 selects the 64-query-step dK/dV kernel (bwd_dkdv_tc) for A/B runs
static bool dkdv_64q_steps() {
  static const bool old = [] {
    const char* e = getenv("GALV_ATTN_DKDV");
    return e && e[0] == '1';
  }();
  return old;
}

}  // namespace fa

int32_t attn_fwd_sm100(const void* q, const void* k, const void* v, void* o, float* lse,
                       int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                       int64_t ost, float scale, int32_t causal, cudaStream_t stream,
                       const DropoutParams& drop) {
  using namespace fa;
  CUtensorMap mq, mk, mv;
  const int64_t tokens = B * S;
  bool ok = qkv_map(&mq, q, tokens, H, D, st, sh) && qkv_map(&mk, k, tokens, H, D, st, sh) &&
            qkv_map(&mv, v, tokens, H, D, st, sh);
  GALV_CHECK_ARG(ok, "tensor map encode failed (alignment?)");
  FwdParams p;
  p.S = (int)S;
  p.H = (int)H;
  p.n_qblocks = (int)((S + BQ - 1) / BQ);
  p.causal = causal;
  p.scale_log2 = scale * LOG2E;
  p.o = (__nv_bfloat16*)o;
  p.lse = lse;
  p.o_st = ost;
  p.sh = sh;
  p.drop = drop;
  const dim3 grid((unsigned)p.n_qblocks, (unsigned)(B * H));
  const bool mc = ATTN_FWD_MC && (p.n_qblocks % 2) == 0;  // cluster pairs share K/V loads
  auto launch = [&](auto kernel, int smem) -> int32_t {
    GALV_CUDA_RET(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = mc ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GALV_CUDA_RET(cudaLaunchKernelEx(&cfg, kernel, mq, mk, mv, p));
    return 0;
  };
  int32_t rc;
  // default: the two-Q-tile kernel (fwd_tc2); dropout is implemented there only
  if (fwd_two_tiles() || p.drop.thresh != 0) {
    p.bh_total = (int)(B * H);
    const long long n_items = (long long)p.bh_total * ((p.n_qblocks + 1) / 2);
    const int ctas = fwd_ctas(S);
    const dim3 grid2((unsigned)(ctas > 0 ? std::min<long long>(n_items, ctas) : n_items));
    const bool drop = p.drop.thresh != 0;
    auto kern = D == 128 ? (drop ? fwd_tc2<128, true> : fwd_tc2<128, false>)
                         : (drop ? fwd_tc2<64, true> : fwd_tc2<64, false>);
    const int smem = D == 128 ? Smem2<128>::BYTES : Smem2<64>::BYTES;
    GALV_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid2, FWD2_THREADS, smem, stream>>>(mq, mk, mv, p);
    GALV_LAUNCH_CHECK();
    return 0;
  }
  if (D == 128)
    rc = mc ? launch(fwd_tc<128, true>, Smem<128>::BYTES)
            : launch(fwd_tc<128, false>, Smem<128>::BYTES);
  else
    rc = mc ? launch(fwd_tc<64, true>, Smem<64>::BYTES)
            : launch(fwd_tc<64, false>, Smem<64>::BYTES);
  if (rc) return rc;
  GALV_LAUNCH_CHECK();
  return 0;
}


#ifdef GALV_ATTN_TRACE
extern "C" int32_t galv_attn_trace_read(void* host) {
  return (int32_t)cudaMemcpyFromSymbol(host, fa::g_trace, sizeof(fa::g_trace));
}
extern "C" int32_t galv_attn_cta_trace_read(void* host) {
  return (int32_t)cudaMemcpyFromSymbol(host, fa::g_cta, sizeof(fa::g_cta));
}
#endif

int64_t attn_bwd_ws_sm100(int64_t B, int64_t S, int64_t H) {
  const int64_t S_pad = (S + 127) / 128 * 128;
  return 2 * B * H * S_pad * (int64_t)sizeof(float);
}

int32_t attn_bwd_sm100(const void* q, const void* k, const void* v, const void* o,
                       const void* dout, const float* lse, void* dq, void* dk, void* dv,
                       int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                       int64_t ost, float scale, int32_t causal, void* ws, cudaStream_t stream,
                       const float* rope_table, const DropoutParams& drop) {
  using namespace fa;
  const int64_t S_pad = (S + 127) / 128 * 128;
  float* lse2 = reinterpret_cast<float*>(ws);
  float* dvec = lse2 + B * H * S_pad;
  {
    const long long n_rows = B * H * S_pad;
    const int rows_per_block = 8 * (32 / (int)(D / 8)) * PREP_ROWS;  // 8 warps
    const unsigned blocks = (unsigned)((n_rows + rows_per_block - 1) / rows_per_block);
    auto prep = D == 128 ? bwd_prep<128> : bwd_prep<64>;
    prep<<<blocks, 256, 0, stream>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, lse,
                                     lse2, dvec, (int)S, (int)S_pad, (int)H, n_rows, ost, sh);
  }
  GALV_LAUNCH_CHECK();
  const int64_t tokens = B * S;
  CUtensorMap mq64, mdo64, mk128, mv128, mq128, mdo128;
  bool ok = qkv_map(&mq64, q, tokens, H, D, st, sh, 64) &&
            qkv_map(&mdo64, dout, tokens, H, D, ost, sh, 64) &&
            qkv_map(&mk128, k, tokens, H, D, st, sh, 128) &&
            qkv_map(&mv128, v, tokens, H, D, st, sh, 128) &&
            qkv_map(&mq128, q, tokens, H, D, st, sh, 128) &&
            qkv_map(&mdo128, dout, tokens, H, D, ost, sh, 128);
  GALV_CHECK_ARG(ok, "tensor map encode failed (alignment?)");
  BwdParams p;
  p.S = (int)S;
  p.S_pad = (int)S_pad;
  p.H = (int)H;
  p.causal = causal;
  p.scale = scale;
  p.scale_log2 = scale * LOG2E;
  p.lse2 = lse2;
  p.dvec = dvec;
  p.st = st;
  p.sh = sh;
  p.rope = rope_table;
  p.drop = drop;
  GALV_CHECK_ARG(rope_table == nullptr || D == 128, "fused inverse RoPE needs head_dim 128");
  const dim3 g_kv((unsigned)((S + 127) / 128), (unsigned)(B * H));
  p.bh_total = (int)(B * H);
  const long long bwd_items = (long long)p.bh_total * ((S + 127) / 128);
  const int bctas = bwd_ctas(S);
  p.persist = bctas > 0;
  const dim3 g_kv2((unsigned)(bctas > 0 ? std::min<long long>(bwd_items, bctas) : bwd_items));
  const dim3 g_q = g_kv2;  // same item count and CTA policy for the dq kernel
#define GALV_FA_BWD(DD, DR)                                                                      \
  do {                                                                                           \
    static bool set = false;                                                                     \
    if (!set) {                                                                                  \
      GALV_CUDA_RET(cudaFuncSetAttribute(bwd_dkdv_tc<DD, DR>,                                    \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                                         SmemKV<DD>::BYTES));                                    \
      GALV_CUDA_RET(cudaFuncSetAttribute(bwd_dkdv2_tc<DD, DR>,                                   \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                                         SmemKV2<DD>::BYTES));                                   \
      GALV_CUDA_RET(cudaFuncSetAttribute(bwd_dq_tc<DD, DR>,                                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                                         SmemQ<DD>::BYTES));                                     \
      set = true;                                                                                \
    }                                                                                            \
    p.g0 = (__nv_bfloat16*)dk;                                                                   \
    p.g1 = (__nv_bfloat16*)dv;                                                                   \
    if (dkdv_64q_steps())                                                                        \
      bwd_dkdv_tc<DD, DR><<<g_kv, BWD_THREADS, SmemKV<DD>::BYTES, stream>>>(mq64, mk128, mv128,  \
                                                                           mdo64, p);            \
    else                                                                                         \
      bwd_dkdv2_tc<DD, DR><<<g_kv2, BWD_THREADS, SmemKV2<DD>::BYTES, stream>>>(mq128, mk128,      \
                                                                             mv128, mdo128, p);  \
    GALV_LAUNCH_CHECK();                                                                         \
    p.g0 = (__nv_bfloat16*)dq;                                                                   \
    p.g1 = nullptr;                                                                              \
    bwd_dq_tc<DD, DR><<<g_q, BWD_THREADS, SmemQ<DD>::BYTES, stream>>>(mq128, mk128, mv128,       \
                                                                     mdo128, p);                 \
    GALV_LAUNCH_CHECK();                                                                         \
  } while (0)
  const bool drp = drop.thresh != 0;
  if (D == 128) {
    if (drp)
      GALV_FA_BWD(128, true);
    else
      GALV_FA_BWD(128, false);
  } else {
    if (drp)
      GALV_FA_BWD(64, true);
    else
      GALV_FA_BWD(64, false);
  }
#undef GALV_FA_BWD
  return 0;
}

}  // namespace galv
