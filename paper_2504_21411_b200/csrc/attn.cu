// Flash attention forward/backward (causal or full) over [B, S, H, D] token-major q/k/v
// (the layout the fused QKV GEMM writes; no transposes), lse [B, H, S] fp32.
//
// bf16 path (v1): mma.sync m16n8k16 tensor-core tiles, 64x64 blocks, 4 warps, swizzled
// smem + cp.async double buffering, online softmax in registers (S/P never touch HBM).
// Backward is two deterministic kernels (no fp32 atomics): dK/dV per key block and dQ
// per query block, each recomputing P from the saved logsumexp.
// fp32 path: exact SIMT kernels (thread per row) for the fp32 parity configuration.
#include <cstdlib>

#include "common.cuh"

namespace galv {
namespace attn {

constexpr int BLK = 64;     // rows per tile (queries or keys)
constexpr int WARPS = 4;    // 16 rows per warp
constexpr float LOG2E = 1.4426950408889634f;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s_u32(smem)), "l"(gmem),
               "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// A [BLK][D] bf16 tile in smem, 16-byte chunks XOR-swizzled by (row & 7)
template <int D>
struct Tile {
  static constexpr int CH = D / 8;  // 16B chunks per row
  __nv_bfloat16* base;
  __device__ __forceinline__ uint32_t addr(int row, int chunk) const {
    return s_u32(base) + (uint32_t)((row * CH + (chunk ^ (row & 7))) * 16);
  }
  // rows [row0, row0+BLK) of a [.., stride_tok] global tensor; rows >= limit zero-filled
  __device__ __forceinline__ void load(const __nv_bfloat16* g, int64_t stride_tok, int row0,
                                       int limit) const {
    for (int i = threadIdx.x; i < BLK * CH; i += WARPS * 32) {
      const int r = i / CH, c = i % CH;
      const bool ok = row0 + r < limit;
      const __nv_bfloat16* src = g + (int64_t)(ok ? row0 + r : 0) * stride_tok + c * 8;
      cp_async16(base + (r * CH + (c ^ (r & 7))) * 8, src, ok);
    }
  }
  // A fragment (16 rows x 16 k) from [row][k] storage
  __device__ __forceinline__ void frag_a(int r0, int k0, uint32_t* a) const {
    const int lane = threadIdx.x & 31;
    ldsm4(addr(r0 + (lane & 15), (k0 >> 3) + (lane >> 4)), a);
  }
  // B fragments for two n8 tiles from [n][k] storage: b[0],b[1] tile n0; b[2],b[3] tile n0+8
  __device__ __forceinline__ void frag_b_nk(int n0, int k0, uint32_t* b) const {
    const int lane = threadIdx.x & 31;
    ldsm4(addr(n0 + (lane & 7) + ((lane >> 4) << 3), (k0 >> 3) + ((lane >> 3) & 1)), b);
  }
  // B fragments for two n8 tiles from [k][n] storage (transposing load)
  __device__ __forceinline__ void frag_b_kn(int k0, int n0, uint32_t* b) const {
    const int lane = threadIdx.x & 31;
    ldsm4t(addr(k0 + (lane & 7) + (((lane >> 3) & 1) << 3), (n0 >> 3) + (lane >> 4)), b);
  }
};

// ------------------------------------------------------------------ forward (bf16)
template <int D>
__global__ void __launch_bounds__(WARPS * 32) fwd_bf16(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
    const __nv_bfloat16* __restrict__ v, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
    int S, int H, int64_t st, int64_t sh, int64_t ost, float scale_log2, int causal) {
  extern __shared__ __align__(128) uint8_t smem[];
  Tile<D> tq{reinterpret_cast<__nv_bfloat16*>(smem)};
  Tile<D> tk[2] = {{tq.base + BLK * D}, {tq.base + 2 * BLK * D}};
  Tile<D> tv[2] = {{tq.base + 3 * BLK * D}, {tq.base + 4 * BLK * D}};
  const int mb = gridDim.x - 1 - blockIdx.x;  // heavy (late) query blocks first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t off = (int64_t)b * S * st + (int64_t)h * sh;
  const __nv_bfloat16 *qg = q + off, *kg = k + off, *vg = v + off;
  const int q0 = mb * BLK;
  const int n_blocks = causal ? min((S + BLK - 1) / BLK, mb + 1) : (S + BLK - 1) / BLK;

  tq.load(qg, st, q0, S);
  tk[0].load(kg, st, 0, S);
  tv[0].load(vg, st, 0, S);
  cp_commit();

  float oacc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  uint32_t qf[D / 16][4];
  const int g = lane >> 2, t4 = lane & 3;
  const int row_a = q0 + warp * 16 + g, row_b = row_a + 8;

  for (int nb = 0; nb < n_blocks; ++nb) {
    const int cur = nb & 1;
    if (nb + 1 < n_blocks) {
      tk[cur ^ 1].load(kg, st, (nb + 1) * BLK, S);
      tv[cur ^ 1].load(vg, st, (nb + 1) * BLK, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (nb == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) tq.frag_a(warp * 16, kk * 16, qf[kk]);
    }
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t bf[4];
        tk[cur].frag_b_nk(j * 16, kk * 16, bf);
        mma16816(s[2 * j], qf[kk], bf[0], bf[1]);
        mma16816(s[2 * j + 1], qf[kk], bf[2], bf[3]);
      }
    }
    // mask (causal diagonal block / sequence tail) and online softmax
    const int k0 = nb * BLK;
    const bool need_mask = (k0 + BLK > S) || (causal && k0 + BLK - 1 > q0);
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + j * 8 + 2 * t4 + (e & 1);
        const int row = (e < 2) ? row_a : row_b;
        if (need_mask && (key >= S || (causal && key > row))) s[j][e] = -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], s[j][e]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], msc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      msc[r] = (mx[r] == -INFINITY) ? 0.f : mx[r] * scale_log2;
      corr[r] = (mrow[r] == -INFINITY) ? 0.f : exp2f(mrow[r] * scale_log2 - msc[r]);
      mrow[r] = mx[r];
      lrow[r] *= corr[r];
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      oacc[i][0] *= corr[0];
      oacc[i][1] *= corr[0];
      oacc[i][2] *= corr[1];
      oacc[i][3] *= corr[1];
    }
    uint32_t pf[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        p[e] = exp2f(s[j][e] * scale_log2 - msc[e >> 1]);
        lrow[e >> 1] += p[e];
      }
      pf[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
      pf[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t bf[4];
        tv[cur].frag_b_kn(kk * 16, dn * 16, bf);
        mma16816(oacc[2 * dn], pf[kk], bf[0], bf[1]);
        mma16816(oacc[2 * dn + 1], pf[kk], bf[2], bf[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const float inv[2] = {lrow[0] > 0.f ? 1.f / lrow[0] : 0.f, lrow[1] > 0.f ? 1.f / lrow[1] : 0.f};
  __nv_bfloat16* og = o + (int64_t)b * S * ost + (int64_t)h * sh;
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    const int col = i * 8 + 2 * t4;
    if (row_a < S)
      *reinterpret_cast<__nv_bfloat162*>(og + (int64_t)row_a * ost + col) =
          __floats2bfloat162_rn(oacc[i][0] * inv[0], oacc[i][1] * inv[0]);
    if (row_b < S)
      *reinterpret_cast<__nv_bfloat162*>(og + (int64_t)row_b * ost + col) =
          __floats2bfloat162_rn(oacc[i][2] * inv[1], oacc[i][3] * inv[1]);
  }
  if (t4 == 0) {
    float* lg = lse + ((int64_t)b * H + h) * S;
    const float ln2 = 0.6931471805599453f;
    if (row_a < S) lg[row_a] = (mrow[0] * scale_log2 + log2f(lrow[0])) * ln2;
    if (row_b < S) lg[row_b] = (mrow[1] * scale_log2 + log2f(lrow[1])) * ln2;
  }
}

// Dvec[b,h,i] = sum_d dO[i,d] * O[i,d]
template <typename T>
__global__ void bwd_dot(const T* __restrict__ o, const T* __restrict__ dout,
                        float* __restrict__ dvec, int S, int H, int D, int64_t ost, int64_t sh) {
  const int64_t row = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);  // over S*H of batch y
  const int lane = threadIdx.x & 31;
  if (row >= (int64_t)S * H) return;
  const int b = blockIdx.y, i = (int)(row / H), h = (int)(row % H);
  const T* orow = o + (int64_t)b * S * ost + (int64_t)i * ost + (int64_t)h * sh;
  const T* drow = dout + (int64_t)b * S * ost + (int64_t)i * ost + (int64_t)h * sh;
  float s = 0.f;
  for (int d = lane; d < D; d += 32) s += to_f(orow[d]) * to_f(drow[d]);
  s = warp_sum(s);
  if (lane == 0) dvec[((int64_t)b * H + h) * S + i] = s;
}

// dK, dV for one key block; loops over query blocks (causal: m >= n)
template <int D>
__global__ void __launch_bounds__(WARPS * 32) bwd_dkdv_bf16(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
    const __nv_bfloat16* __restrict__ v, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ dvec, __nv_bfloat16* __restrict__ dk,
    __nv_bfloat16* __restrict__ dv, int S, int H, int64_t st, int64_t sh, int64_t ost,
    float scale, int causal) {
  extern __shared__ __align__(128) uint8_t smem[];
  Tile<D> tk{reinterpret_cast<__nv_bfloat16*>(smem)};
  Tile<D> tv{tk.base + BLK * D};
  Tile<D> tq[2] = {{tk.base + 2 * BLK * D}, {tk.base + 3 * BLK * D}};
  Tile<D> tdo[2] = {{tk.base + 4 * BLK * D}, {tk.base + 5 * BLK * D}};
  float* s_lse = reinterpret_cast<float*>(tk.base + 6 * BLK * D);  // [2][BLK]
  float* s_dv = s_lse + 2 * BLK;                                   // [2][BLK]
  const int nb = blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t off = (int64_t)b * S * st + (int64_t)h * sh;
  const int64_t ooff = (int64_t)b * S * ost + (int64_t)h * sh;
  const float* lse_g = lse + ((int64_t)b * H + h) * S;
  const float* dv_g = dvec + ((int64_t)b * H + h) * S;
  const int k0 = nb * BLK;
  const int n_qb = (S + BLK - 1) / BLK;
  const int m_start = causal ? nb : 0;
  const float scale_log2 = scale * LOG2E;

  tk.load(k + off, st, k0, S);
  tv.load(v + off, st, k0, S);
  auto load_q = [&](int mb, int buf) {
    tq[buf].load(q + off, st, mb * BLK, S);
    tdo[buf].load(dout + ooff, ost, mb * BLK, S);
    for (int i = threadIdx.x; i < BLK; i += WARPS * 32) {
      const int r = mb * BLK + i;
      s_lse[buf * BLK + i] = r < S ? lse_g[r] * LOG2E : 0.f;
      s_dv[buf * BLK + i] = r < S ? dv_g[r] : 0.f;
    }
  };
  if (m_start < n_qb) load_q(m_start, 0);
  cp_commit();

  float dk_acc[D / 8][4], dv_acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk_acc[i][e] = dv_acc[i][e] = 0.f;
  const int key_a = k0 + warp * 16 + g, key_b = key_a + 8;

  for (int mb = m_start; mb < n_qb; ++mb) {
    const int cur = (mb - m_start) & 1;
    if (mb + 1 < n_qb) load_q(mb + 1, cur ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const int q0 = mb * BLK;
    // S^T (keys x queries) and dP^T
    float st_[8][4], dpt[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) st_[j][e] = dpt[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ka[4], va[4];
      tk.frag_a(warp * 16, kk * 16, ka);
      tv.frag_a(warp * 16, kk * 16, va);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t bq[4], bd[4];
        tq[cur].frag_b_nk(j * 16, kk * 16, bq);
        tdo[cur].frag_b_nk(j * 16, kk * 16, bd);
        mma16816(st_[2 * j], ka, bq[0], bq[1]);
        mma16816(st_[2 * j + 1], ka, bq[2], bq[3]);
        mma16816(dpt[2 * j], va, bd[0], bd[1]);
        mma16816(dpt[2 * j + 1], va, bd[2], bd[3]);
      }
    }
    const bool need_mask = (q0 + BLK > S) || (k0 + BLK > S) || (causal && k0 + BLK - 1 > q0);
    uint32_t pa[4][4], dsa[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p[4], ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = j * 8 + 2 * t4 + (e & 1);  // query within block
        const int key = (e < 2) ? key_a : key_b;
        const int qrow = q0 + qi;
        const bool masked = need_mask && (qrow >= S || key >= S || (causal && key > qrow));
        p[e] = masked ? 0.f : exp2f(st_[j][e] * scale_log2 - s_lse[cur * BLK + qi]);
        ds[e] = p[e] * (dpt[j][e] - s_dv[cur * BLK + qi]);
      }
      pa[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
      pa[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
      dsa[j >> 1][(j & 1) * 2 + 0] = pack_bf16(ds[0], ds[1]);
      dsa[j >> 1][(j & 1) * 2 + 1] = pack_bf16(ds[2], ds[3]);
    }
    // dV += P^T dO ; dK += dS^T Q   (reduction over the 64 queries)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t bd[4], bq[4];
        tdo[cur].frag_b_kn(kk * 16, dn * 16, bd);
        tq[cur].frag_b_kn(kk * 16, dn * 16, bq);
        mma16816(dv_acc[2 * dn], pa[kk], bd[0], bd[1]);
        mma16816(dv_acc[2 * dn + 1], pa[kk], bd[2], bd[3]);
        mma16816(dk_acc[2 * dn], dsa[kk], bq[0], bq[1]);
        mma16816(dk_acc[2 * dn + 1], dsa[kk], bq[2], bq[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    const int col = i * 8 + 2 * t4;
    if (key_a < S) {
      *reinterpret_cast<__nv_bfloat162*>(dk + off + (int64_t)key_a * st + col) =
          __floats2bfloat162_rn(dk_acc[i][0] * scale, dk_acc[i][1] * scale);
      *reinterpret_cast<__nv_bfloat162*>(dv + off + (int64_t)key_a * st + col) =
          __floats2bfloat162_rn(dv_acc[i][0], dv_acc[i][1]);
    }
    if (key_b < S) {
      *reinterpret_cast<__nv_bfloat162*>(dk + off + (int64_t)key_b * st + col) =
          __floats2bfloat162_rn(dk_acc[i][2] * scale, dk_acc[i][3] * scale);
      *reinterpret_cast<__nv_bfloat162*>(dv + off + (int64_t)key_b * st + col) =
          __floats2bfloat162_rn(dv_acc[i][2], dv_acc[i][3]);
    }
  }
}

// dQ for one query block; loops over key blocks (causal: n <= m)
template <int D>
__global__ void __launch_bounds__(WARPS * 32) bwd_dq_bf16(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
    const __nv_bfloat16* __restrict__ v, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ dvec, __nv_bfloat16* __restrict__ dq,
    int S, int H, int64_t st, int64_t sh, int64_t ost, float scale, int causal) {
  extern __shared__ __align__(128) uint8_t smem[];
  Tile<D> tq{reinterpret_cast<__nv_bfloat16*>(smem)};
  Tile<D> tdo{tq.base + BLK * D};
  Tile<D> tk[2] = {{tq.base + 2 * BLK * D}, {tq.base + 3 * BLK * D}};
  Tile<D> tv[2] = {{tq.base + 4 * BLK * D}, {tq.base + 5 * BLK * D}};
  const int mb = gridDim.x - 1 - blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t off = (int64_t)b * S * st + (int64_t)h * sh;
  const int64_t ooff = (int64_t)b * S * ost + (int64_t)h * sh;
  const int q0 = mb * BLK;
  const int n_blocks = causal ? min((S + BLK - 1) / BLK, mb + 1) : (S + BLK - 1) / BLK;
  const float scale_log2 = scale * LOG2E;
  const int row_a = q0 + warp * 16 + g, row_b = row_a + 8;
  const float* lse_g = lse + ((int64_t)b * H + h) * S;
  const float* dv_g = dvec + ((int64_t)b * H + h) * S;
  const float l2a = row_a < S ? lse_g[row_a] * LOG2E : 0.f;
  const float l2b = row_b < S ? lse_g[row_b] * LOG2E : 0.f;
  const float dva = row_a < S ? dv_g[row_a] : 0.f;
  const float dvb = row_b < S ? dv_g[row_b] : 0.f;

  tq.load(q + off, st, q0, S);
  tdo.load(dout + ooff, ost, q0, S);
  tk[0].load(k + off, st, 0, S);
  tv[0].load(v + off, st, 0, S);
  cp_commit();
  float dq_acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dq_acc[i][0] = dq_acc[i][1] = dq_acc[i][2] = dq_acc[i][3] = 0.f;

  for (int nb = 0; nb < n_blocks; ++nb) {
    const int cur = nb & 1;
    if (nb + 1 < n_blocks) {
      tk[cur ^ 1].load(k + off, st, (nb + 1) * BLK, S);
      tv[cur ^ 1].load(v + off, st, (nb + 1) * BLK, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    float s[8][4], dp[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = dp[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t qa[4], da[4];
      tq.frag_a(warp * 16, kk * 16, qa);
      tdo.frag_a(warp * 16, kk * 16, da);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t bk[4], bv[4];
        tk[cur].frag_b_nk(j * 16, kk * 16, bk);
        tv[cur].frag_b_nk(j * 16, kk * 16, bv);
        mma16816(s[2 * j], qa, bk[0], bk[1]);
        mma16816(s[2 * j + 1], qa, bk[2], bk[3]);
        mma16816(dp[2 * j], da, bv[0], bv[1]);
        mma16816(dp[2 * j + 1], da, bv[2], bv[3]);
      }
    }
    const int k0 = nb * BLK;
    const bool need_mask = (k0 + BLK > S) || (causal && k0 + BLK - 1 > q0);
    uint32_t dsa[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + j * 8 + 2 * t4 + (e & 1);
        const int row = (e < 2) ? row_a : row_b;
        const bool masked = need_mask && (key >= S || (causal && key > row));
        const float p = masked ? 0.f : exp2f(s[j][e] * scale_log2 - ((e < 2) ? l2a : l2b));
        ds[e] = p * (dp[j][e] - ((e < 2) ? dva : dvb));
      }
      dsa[j >> 1][(j & 1) * 2 + 0] = pack_bf16(ds[0], ds[1]);
      dsa[j >> 1][(j & 1) * 2 + 1] = pack_bf16(ds[2], ds[3]);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t bk[4];
        tk[cur].frag_b_kn(kk * 16, dn * 16, bk);
        mma16816(dq_acc[2 * dn], dsa[kk], bk[0], bk[1]);
        mma16816(dq_acc[2 * dn + 1], dsa[kk], bk[2], bk[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    const int col = i * 8 + 2 * t4;
    if (row_a < S)
      *reinterpret_cast<__nv_bfloat162*>(dq + off + (int64_t)row_a * st + col) =
          __floats2bfloat162_rn(dq_acc[i][0] * scale, dq_acc[i][1] * scale);
    if (row_b < S)
      *reinterpret_cast<__nv_bfloat162*>(dq + off + (int64_t)row_b * st + col) =
          __floats2bfloat162_rn(dq_acc[i][2] * scale, dq_acc[i][3] * scale);
  }
}

// ------------------------------------------------------------------ fp32 SIMT path
// forward: thread per query row, K/V tiles staged in smem (padded rows)
template <int D>
__global__ void __launch_bounds__(64) fwd_f32(const float* __restrict__ q,
                                              const float* __restrict__ k,
                                              const float* __restrict__ v, float* __restrict__ o,
                                              float* __restrict__ lse, int S, int H, int64_t st,
                                              int64_t sh, int64_t ost, float scale, int causal) {
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
      l = l * c + p;
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] = acc[d] * c + p * vs[r][d];
      m = mn;
    }
  }
  if (!live) return;
  const float inv = 1.f / l;
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
    int64_t ost, float scale, int causal) {
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
      const float dsv = p * (dp - dd[r]);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        gv[d] = fmaf(p, ds_[r][d], gv[d]);
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
    int causal) {
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
      const float dsv = p * (dp - dd);
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
                       int64_t ost, float scale, int32_t causal, cudaStream_t stream);
int64_t attn_bwd_ws_sm100(int64_t B, int64_t S, int64_t H);
int32_t attn_bwd_sm100(const void* q, const void* k, const void* v, const void* o,
                       const void* dout, const float* lse, void* dq, void* dk, void* dv,
                       int64_t B, int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh,
                       int64_t ost, float scale, int32_t causal, void* ws, cudaStream_t stream);
}

extern "C" {

int32_t galv_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t B,
                      int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh, int64_t ost,
                      float scale, int32_t causal, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(q && k && v && o && lse && B > 0 && S > 0 && H > 0, "bad arguments");
  GALV_CHECK_ARG(D == 64 || D == 128, "head_dim must be 64 or 128");
  const dim3 grid((unsigned)((S + 63) / 64), (unsigned)(B * H));
  cudaStream_t s = as_stream(stream);
  if (dtype == GALV_BF16) {
    GALV_CHECK_ARG(st % 8 == 0 && sh % 8 == 0 && ost % 8 == 0, "strides must be multiples of 8");
    if (getenv("GALV_ATTN_MMA_SYNC") == nullptr)  // tcgen05 path (default)
      return attn_fwd_sm100(q, k, v, o, lse, B, S, H, D, st, sh, ost, scale, causal, s);
    const size_t smem = 5 * attn::BLK * D * 2;
    if (D == 64) {
      if (int32_t rc = set_smem(attn::fwd_bf16<64>, smem)) return rc;
      attn::fwd_bf16<64><<<grid, 128, smem, s>>>(
          (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
          (__nv_bfloat16*)o, lse, (int)S, (int)H, st, sh, ost, scale * attn::LOG2E, causal);
    } else {
      if (int32_t rc = set_smem(attn::fwd_bf16<128>, smem)) return rc;
      attn::fwd_bf16<128><<<grid, 128, smem, s>>>(
          (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
          (__nv_bfloat16*)o, lse, (int)S, (int)H, st, sh, ost, scale * attn::LOG2E, causal);
    }
  } else {
    GALV_CHECK_ARG(dtype == GALV_F32, "bad dtype");
    if (D == 64)
      attn::fwd_f32<64><<<grid, 64, 0, s>>>((const float*)q, (const float*)k, (const float*)v,
                                            (float*)o, lse, (int)S, (int)H, st, sh, ost, scale,
                                            causal);
    else
      GALV_CHECK_ARG(false, "fp32 attention supports head_dim 64");
  }
  GALV_LAUNCH_CHECK();
  return 0;
}

int64_t galv_attn_bwd_workspace(int64_t B, int64_t S, int64_t H, int64_t D, int32_t dtype) {
  (void)D;
  if (dtype == GALV_BF16) return galv::attn_bwd_ws_sm100(B, S, H);
  return B * H * S * (int64_t)sizeof(float);
}

int32_t galv_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                      const void* dout, const float* lse, void* dq, void* dk, void* dv, int64_t B,
                      int64_t S, int64_t H, int64_t D, int64_t st, int64_t sh, int64_t ost,
                      float scale, int32_t causal, int32_t dtype, void* ws, void* stream) {
  GALV_CHECK_ARG(q && k && v && o && dout && lse && dq && dk && dv && ws, "bad arguments");
  GALV_CHECK_ARG(D == 64 || D == 128, "head_dim must be 64 or 128");
  cudaStream_t s = as_stream(stream);
  float* dvec = (float*)ws;
  const dim3 grid((unsigned)((S + 63) / 64), (unsigned)(B * H));
  const dim3 gdot((unsigned)((S * H + 3) / 4), (unsigned)B);
  if (dtype == GALV_BF16) {
    GALV_CHECK_ARG(st % 8 == 0 && sh % 8 == 0 && ost % 8 == 0, "strides must be multiples of 8");
    if (getenv("GALV_ATTN_MMA_SYNC") == nullptr)  // tcgen05 path (default)
      return attn_bwd_sm100(q, k, v, o, dout, lse, dq, dk, dv, B, S, H, D, st, sh, ost, scale,
                            causal, ws, s);
    attn::bwd_dot<__nv_bfloat16><<<gdot, 128, 0, s>>>(
        (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, dvec, (int)S, (int)H, (int)D, ost, sh);
    const size_t smem_kv = 6 * attn::BLK * D * 2 + 4 * attn::BLK * sizeof(float);
    const size_t smem_q = 6 * attn::BLK * D * 2;
#define GALV_ATTN_BWD(DD)                                                                      \
  do {                                                                                         \
    if (int32_t rc = set_smem(attn::bwd_dkdv_bf16<DD>, smem_kv)) return rc;                    \
    if (int32_t rc = set_smem(attn::bwd_dq_bf16<DD>, smem_q)) return rc;                       \
    attn::bwd_dkdv_bf16<DD><<<grid, 128, smem_kv, s>>>(                                        \
        (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,            \
        (const __nv_bfloat16*)dout, lse, dvec, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, (int)S, \
        (int)H, st, sh, ost, scale, causal);                                                   \
    attn::bwd_dq_bf16<DD><<<grid, 128, smem_q, s>>>(                                           \
        (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,            \
        (const __nv_bfloat16*)dout, lse, dvec, (__nv_bfloat16*)dq, (int)S, (int)H, st, sh, ost, \
        scale, causal);                                                                        \
  } while (0)
    if (D == 64)
      GALV_ATTN_BWD(64);
    else
      GALV_ATTN_BWD(128);
#undef GALV_ATTN_BWD
  } else {
    GALV_CHECK_ARG(dtype == GALV_F32 && D == 64, "fp32 attention supports head_dim 64");
    attn::bwd_dot<float><<<gdot, 128, 0, s>>>((const float*)o, (const float*)dout, dvec, (int)S,
                                              (int)H, (int)D, ost, sh);
    attn::bwd_dkdv_f32<64><<<grid, 64, 0, s>>>(
        (const float*)q, (const float*)k, (const float*)v, (const float*)dout, lse, dvec,
        (float*)dk, (float*)dv, (int)S, (int)H, st, sh, ost, scale, causal);
    attn::bwd_dq_f32<64><<<grid, 64, 0, s>>>((const float*)q, (const float*)k, (const float*)v,
                                             (const float*)dout, lse, dvec, (float*)dq, (int)S,
                                             (int)H, st, sh, ost, scale, causal);
  }
  GALV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
