// RMSNorm (Llama) / LayerNorm (GPT) forward+backward with an optional fused residual add.
// HBM-bound: one warp per row, 16-byte vector loads, warp-shuffle reductions; the
// second pass over the row hits L1.  dgamma/dbeta are reduced per CTA in shared memory
// (grid-stride over rows, one CTA set per SM) and flushed with one atomic per column
// per CTA into fp32 accumulators.
#include "common.cuh"

namespace galv {
namespace norm {

constexpr int WARPS = 8;

// GALV_NORM_UNFUSED=1 selects the two-kernel backward (dx pass, then dgamma pass) for A/B.
// GALV_NORM_WARP=1 opts narrow rows into the warp-per-row kernel.  Off by default: B200,
// 16384 x 1024 LayerNorm backward 77.1 us vs 48.3 us for the dx + dgamma pair
// (tools/pointwise_bench.py, profiles/r02/kernels_ab/pointwise.jsonl) -- the per-element
// smem read-modify-write of the partials costs more than the pair's second read.
static bool warp_rows_enabled() {
  static const bool on = [] {
    const char* e = getenv("GALV_NORM_WARP");
    return e && e[0] == '1';
  }();
  return on;
}
static bool fused_disabled() {
  static const bool off = [] {
    const char* e = getenv("GALV_NORM_UNFUSED");
    return e && e[0] == '1';
  }();
  return off;
}

template <typename T, bool LAYER, bool RESID>
__global__ void __launch_bounds__(WARPS * 32) fwd_kernel(
    const T* __restrict__ x, const T* __restrict__ res, T* __restrict__ res_out,
    const T* __restrict__ gamma, const T* __restrict__ beta, T* __restrict__ y,
    float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows, int cols,
    float eps) {
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* xr = x + row * cols;
  const T* rr = RESID ? res + row * cols : nullptr;
  T* ro = RESID ? res_out + row * cols : nullptr;
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V];
    load16(xr + c, v);
    if (RESID) {
      float r[V];
      load16(rr + c, r);
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] += r[i];
      store16(ro + c, v);
      // re-round to T so the normalized value matches the stored residual stream
      load16(ro + c, v);
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      s1 += v[i];
      s2 += v[i] * v[i];
    }
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  float mu = 0.f, rstd;
  if (LAYER) {
    mu = s1 / cols;
    float var = fmaxf(s2 / cols - mu * mu, 0.f);
    rstd = rsqrtf(var + eps);
  } else {
    rstd = rsqrtf(s2 / cols + eps);
  }
  if (lane == 0) {
    rstd_out[row] = rstd;
    if (LAYER) mean_out[row] = mu;
  }
  const T* src = RESID ? ro : xr;
  T* yr = y + row * cols;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V], g[V], b[V];
    load16(src + c, v);
    load16(gamma + c, g);
    if (LAYER) load16(beta + c, b);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = (v[i] - mu) * rstd * g[i] + (LAYER ? b[i] : 0.f);
    store16(yr + c, v);
  }
}

// dx = rstd * (g*dy - xhat * mean(g*dy*xhat) [- mean(g*dy) for LayerNorm]) (+ dres):
// warp per row, 8 warps per CTA, full occupancy (HBM-bound, 16-byte vectors).
template <typename T, bool LAYER>
__global__ void __launch_bounds__(WARPS * 32) bwd_dx_kernel(
    const T* __restrict__ x, const T* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, const T* __restrict__ dy, const T* __restrict__ dres,
    T* __restrict__ dx, int64_t rows, int cols) {
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* xr = x + row * cols;
  const T* dyr = dy + row * cols;
  const float mu = LAYER ? mean[row] : 0.f, rs = rstd[row];
  float a1 = 0.f, a2 = 0.f;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V], d[V], g[V];
    load16(xr + c, v);
    load16(dyr + c, d);
    load16(gamma + c, g);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float gd = g[i] * d[i];
      a1 += gd * (v[i] - mu) * rs;
      a2 += gd;
    }
  }
  a1 = warp_sum(a1) / cols;
  a2 = warp_sum(a2) / cols;
  T* dxr = dx + row * cols;
  const T* drr = dres ? dres + row * cols : nullptr;
  for (int c = lane * V; c < cols; c += 32 * V) {
    float v[V], d[V], g[V], r[V];
    load16(xr + c, v);
    load16(dyr + c, d);
    load16(gamma + c, g);
    if (drr) load16(drr + c, r);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float xh = (v[i] - mu) * rs;
      float o = rs * (g[i] * d[i] - xh * a1 - (LAYER ? a2 : 0.f));
      if (drr) o += r[i];
      v[i] = o;
    }
    store16(dxr + c, v);
  }
}

// Single-pass variant for rows of up to 128 * NV vectors: one 128-thread CTA per row keeps
// its x / dy vectors in registers between the reduction and the output pass, so x and dy
// are read from HBM once (the warp-per-row kernel above re-reads them).
template <typename T, bool LAYER, int NV>
__global__ void __launch_bounds__(128) bwd_dx_row(
    const T* __restrict__ x, const T* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, const T* __restrict__ dy, const T* __restrict__ dres,
    T* __restrict__ dx, int cols) {
  constexpr int V = 16 / sizeof(T);
  __shared__ float red[2][4];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * cols;
  const T* dyr = dy + row * cols;
  const float mu = LAYER ? mean[row] : 0.f, rs = rstd[row];
  uint4 xv[NV], dv[NV];
  float a1 = 0.f, a2 = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = (j * 128 + threadIdx.x) * V;
    if (c < cols) {
      xv[j] = *reinterpret_cast<const uint4*>(xr + c);
      dv[j] = *reinterpret_cast<const uint4*>(dyr + c);
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = (j * 128 + threadIdx.x) * V;
    if (c < cols) {
      float v[V], d[V], g[V];
      load16(reinterpret_cast<const T*>(&xv[j]), v);
      load16(reinterpret_cast<const T*>(&dv[j]), d);
      load16(gamma + c, g);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float gd = g[i] * d[i];
        a1 += gd * (v[i] - mu) * rs;
        a2 += gd;
      }
    }
  }
  a1 = warp_sum(a1);
  a2 = warp_sum(a2);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a1;
    red[1][threadIdx.x >> 5] = a2;
  }
  __syncthreads();
  a1 = (red[0][0] + red[0][1] + red[0][2] + red[0][3]) / cols;
  a2 = (red[1][0] + red[1][1] + red[1][2] + red[1][3]) / cols;
  T* dxr = dx + row * cols;
  const T* drr = dres ? dres + row * cols : nullptr;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = (j * 128 + threadIdx.x) * V;
    if (c < cols) {
      float v[V], d[V], g[V], r[V];
      load16(reinterpret_cast<const T*>(&xv[j]), v);
      load16(reinterpret_cast<const T*>(&dv[j]), d);
      load16(gamma + c, g);
      if (drr) load16(drr + c, r);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = (v[i] - mu) * rs;
        float o = rs * (g[i] * d[i] - xh * a1 - (LAYER ? a2 : 0.f));
        if (drr) o += r[i];
        v[i] = o;
      }
      store16(dxr + c, v);
    }
  }
}

// Fused dx + dgamma(/dbeta): persistent NT-thread CTAs stride over rows; every thread owns
// the same NV column vectors in every row, so its dgamma partials stay in registers across
// rows and x / dy are read from HBM exactly once per backward (the dx-then-dgamma pair
// above reads them twice).  The partials live in shared memory (each column is owned by
// exactly one thread of the CTA, so plain read-modify-write, no atomics) to leave the
// registers to the in-flight x / dy vectors, and are flushed once per CTA with 16-byte
// atomics.
// Per row: 2 reads (x, dy) [+ dres] + 1 write of rows*cols*sizeof(T).
#ifndef NORM_FUSED_PREFETCH
#define NORM_FUSED_PREFETCH 1
#endif
template <typename T, bool LAYER, int NV, int NT>
__global__ void __launch_bounds__(NT) bwd_fused_rows(
    const T* __restrict__ x, const T* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, const T* __restrict__ dy, const T* __restrict__ dres,
    T* __restrict__ dx, float* __restrict__ dgamma, float* __restrict__ dbeta, int64_t rows,
    int cols) {
  constexpr int V = 16 / sizeof(T);
  constexpr int NW = NT / 32;
  __shared__ float red[2][2][NW];
  extern __shared__ float4 sacc4[];  // [cols] dgamma partials (+ [cols] dbeta)
  float* gacc = reinterpret_cast<float*>(sacc4);
  float* bacc = gacc + cols;
  uint4 gv[NV];  // gamma kept packed (T) in registers for the whole kernel
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = (j * NT + threadIdx.x) * V;
    if (c < cols) {
      gv[j] = *reinterpret_cast<const uint4*>(gamma + c);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        gacc[c + i] = 0.f;
        if (LAYER) bacc[c + i] = 0.f;
      }
    }
  }
  int parity = 0;
  // the next row's x / dy (and mean / rstd) are loaded before this row's barrier and
  // arithmetic (NORM_FUSED_PREFETCH): two rows in flight per CTA
  uint4 xv[NV], dv[NV], xn[NV], dn[NV];
  float mun = 0.f, rsn = 0.f;
  auto fetch = [&](int64_t r, uint4* xo, uint4* doo, float& m, float& q) {
    if (r >= rows) return;
    const T* xr = x + r * cols;
    const T* dyr = dy + r * cols;
    m = LAYER ? mean[r] : 0.f;
    q = rstd[r];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * NT + threadIdx.x) * V;
      if (c < cols) {
        xo[j] = __ldcs(reinterpret_cast<const uint4*>(xr + c));
        doo[j] = __ldcs(reinterpret_cast<const uint4*>(dyr + c));
      }
    }
  };
  if (NORM_FUSED_PREFETCH) fetch(blockIdx.x, xn, dn, mun, rsn);
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x, parity ^= 1) {
    float mu, rs;
    if (NORM_FUSED_PREFETCH) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        xv[j] = xn[j];
        dv[j] = dn[j];
      }
      mu = mun;
      rs = rsn;
      fetch(row + gridDim.x, xn, dn, mun, rsn);
    } else {
      fetch(row, xv, dv, mu, rs);
    }
    float a1 = 0.f, a2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * NT + threadIdx.x) * V;
      if (c < cols) {
        float v[V], d[V], g[V];
        load16(reinterpret_cast<const T*>(&xv[j]), v);
        load16(reinterpret_cast<const T*>(&dv[j]), d);
        load16(reinterpret_cast<const T*>(&gv[j]), g);
        float ga[V], ba[V];
#pragma unroll
        for (int i = 0; i < V; i += 4) {
          *reinterpret_cast<float4*>(ga + i) = *reinterpret_cast<const float4*>(gacc + c + i);
          if (LAYER)
            *reinterpret_cast<float4*>(ba + i) = *reinterpret_cast<const float4*>(bacc + c + i);
        }
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float xh = (v[i] - mu) * rs;
          const float gd = g[i] * d[i];
          a1 += gd * xh;
          a2 += gd;
          ga[i] += d[i] * xh;
          if (LAYER) ba[i] += d[i];
        }
#pragma unroll
        for (int i = 0; i < V; i += 4) {
          *reinterpret_cast<float4*>(gacc + c + i) = *reinterpret_cast<const float4*>(ga + i);
          if (LAYER)
            *reinterpret_cast<float4*>(bacc + c + i) = *reinterpret_cast<const float4*>(ba + i);
        }
      }
    }
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    // double-buffered by row parity: one barrier per row suffices
    if ((threadIdx.x & 31) == 0) {
      red[parity][0][threadIdx.x >> 5] = a1;
      red[parity][1][threadIdx.x >> 5] = a2;
    }
    __syncthreads();
    a1 = 0.f;
    a2 = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      a1 += red[parity][0][w];
      a2 += red[parity][1][w];
    }
    a1 /= cols;
    a2 /= cols;
    T* dxr = dx + row * cols;
    const T* drr = dres ? dres + row * cols : nullptr;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * NT + threadIdx.x) * V;
      if (c < cols) {
        float v[V], d[V], g[V], r[V];
        load16(reinterpret_cast<const T*>(&xv[j]), v);
        load16(reinterpret_cast<const T*>(&dv[j]), d);
        load16(reinterpret_cast<const T*>(&gv[j]), g);
        if (drr) load16(drr + c, r);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float xh = (v[i] - mu) * rs;
          float o = rs * (g[i] * d[i] - xh * a1 - (LAYER ? a2 : 0.f));
          if (drr) o += r[i];
          v[i] = o;
        }
        store16(dxr + c, v);
      }
    }
  }
  const bool vec = ((reinterpret_cast<uintptr_t>(dgamma) |
                     (LAYER ? reinterpret_cast<uintptr_t>(dbeta) : 0)) & 15) == 0;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = (j * NT + threadIdx.x) * V;
    if (c >= cols) continue;
#pragma unroll
    for (int i = 0; i < V; i += 4) {
      if (vec) {
        atomicAdd(reinterpret_cast<float4*>(dgamma + c + i),
                  *reinterpret_cast<const float4*>(gacc + c + i));
        if (LAYER)
          atomicAdd(reinterpret_cast<float4*>(dbeta + c + i),
                    *reinterpret_cast<const float4*>(bacc + c + i));
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          atomicAdd(dgamma + c + i + k, gacc[c + i + k]);
          if (LAYER) atomicAdd(dbeta + c + i + k, bacc[c + i + k]);
        }
      }
    }
  }
}

// Narrow rows (<= 1024 bf16 / 512 fp32 columns): a WARP per row instead of a CTA per row.
// Each lane owns VPL fixed 16-byte column vectors (columns lane*V + j*32*V), so its dgamma
// (/dbeta) partials stay in registers across all the rows the warp visits; the row
// reductions are warp shuffles (no CTA barrier per row, which is what starved the
// CTA-per-row kernel at width 1024: one short row per barrier interval).  x and dy are read
// once; the partials are summed over the CTA's warps through smem and flushed with one
// atomic per column per CTA.
template <typename T, bool LAYER, int VPL>
__global__ void __launch_bounds__(256, 2) bwd_fused_warp_rows(
    const T* __restrict__ x, const T* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, const T* __restrict__ dy, const T* __restrict__ dres,
    T* __restrict__ dx, float* __restrict__ dgamma, float* __restrict__ dbeta, int64_t rows,
    int cols) {
  constexpr int V = 16 / sizeof(T);
  constexpr int NW = 8;
  // per-warp dgamma (/dbeta) partials in smem ([NW][cols] each): every lane owns its
  // columns, so read-modify-write needs no atomics; x / dy / gamma stay packed in registers
  // (a register-resident version used 223 registers: one CTA per SM, latency-bound)
  extern __shared__ float sred[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* ga = sred + warp * cols;
  float* ba = sred + (NW + warp) * cols;
  uint4 gv[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int c = (j * 32 + lane) * V;
    if (c < cols) {
      gv[j] = *reinterpret_cast<const uint4*>(gamma + c);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        ga[c + i] = 0.f;
        if (LAYER) ba[c + i] = 0.f;
      }
    }
  }
  const float inv_cols = 1.f / cols;
  for (int64_t row = (int64_t)blockIdx.x * NW + warp; row < rows; row += (int64_t)gridDim.x * NW) {
    const T* xr = x + row * cols;
    const T* dyr = dy + row * cols;
    const float mu = LAYER ? mean[row] : 0.f, rs = rstd[row];
    uint4 xv[VPL], dv[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = (j * 32 + lane) * V;
      if (c < cols) {
        xv[j] = __ldcs(reinterpret_cast<const uint4*>(xr + c));
        dv[j] = __ldcs(reinterpret_cast<const uint4*>(dyr + c));
      }
    }
    float a1 = 0.f, a2 = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = (j * 32 + lane) * V;
      if (c >= cols) continue;
      float v[V], d[V], g[V];
      load16(reinterpret_cast<const T*>(&xv[j]), v);
      load16(reinterpret_cast<const T*>(&dv[j]), d);
      load16(reinterpret_cast<const T*>(&gv[j]), g);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = (v[i] - mu) * rs;
        const float gd = g[i] * d[i];
        a1 += gd * xh;
        a2 += gd;
        ga[c + i] += d[i] * xh;
        if (LAYER) ba[c + i] += d[i];
      }
    }
    a1 = warp_sum(a1) * inv_cols;
    a2 = warp_sum(a2) * inv_cols;
    T* dxr = dx + row * cols;
    const T* drr = dres ? dres + row * cols : nullptr;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = (j * 32 + lane) * V;
      if (c >= cols) continue;
      float v[V], d[V], g[V], r[V];
      load16(reinterpret_cast<const T*>(&xv[j]), v);
      load16(reinterpret_cast<const T*>(&dv[j]), d);
      load16(reinterpret_cast<const T*>(&gv[j]), g);
      if (drr) load16(drr + c, r);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = (v[i] - mu) * rs;
        float o = rs * (g[i] * d[i] - xh * a1 - (LAYER ? a2 : 0.f));
        if (drr) o += r[i];
        v[i] = o;
      }
      store16(dxr + c, v);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float sg = 0.f, sb = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      sg += sred[w * cols + c];
      if (LAYER) sb += sred[(NW + w) * cols + c];
    }
    atomicAdd(dgamma + c, sg);
    if (LAYER) atomicAdd(dbeta + c, sb);
  }
}

// Narrow rows (<= 1024 bf16 columns), register partials: a warp per row, each lane owning
// VPL fixed 16-byte column vectors (columns (j*32 + lane)*V), so its dgamma (/dbeta)
// partials are VPL*V (*2) floats in registers across every row the warp visits; gamma is
// re-read through L1 (2 KB) instead of pinned in registers; the row reductions are warp
// shuffles.  x / dy are read once and dx written once (the dx + dgamma pair reads x and dy
// twice); per CTA the partials meet in smem and are flushed with one 16-byte atomic per 4
// columns.  (The smem-partials warp kernel above pays an 8-way bank-conflicted
// read-modify-write per element.)
#ifndef NORM_NARROW_WARPS
#define NORM_NARROW_WARPS 12  // 8: 39.1 us, 12: 33.1, 16 (128 regs, spills): 37.3 at LN 16384x1024
#endif
template <typename T, bool LAYER, int VPL>
__global__ void __launch_bounds__(NORM_NARROW_WARPS * 32, 1) bwd_narrow_reg(
    const T* __restrict__ x, const T* __restrict__ gamma, const float* __restrict__ mean,
    const float* __restrict__ rstd, const T* __restrict__ dy, const T* __restrict__ dres,
    T* __restrict__ dx, float* __restrict__ dgamma, float* __restrict__ dbeta, int64_t rows,
    int cols) {
  constexpr int V = 16 / sizeof(T);
  constexpr int NW = NORM_NARROW_WARPS;
  extern __shared__ float4 sred4[];  // [NW][cols] dgamma partials (+ [NW][cols] dbeta)
  float* sred = reinterpret_cast<float*>(sred4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float pg[VPL][V], pb[LAYER ? VPL : 1][V];
#pragma unroll
  for (int j = 0; j < VPL; ++j)
#pragma unroll
    for (int i = 0; i < V; ++i) {
      pg[j][i] = 0.f;
      if (LAYER) pb[j][i] = 0.f;
    }
  const float inv_cols = 1.f / cols;
  for (int64_t row = (int64_t)blockIdx.x * NW + warp; row < rows;
       row += (int64_t)gridDim.x * NW) {
    const T* xr = x + row * cols;
    const T* dyr = dy + row * cols;
    const float mu = LAYER ? mean[row] : 0.f, rs = rstd[row];
    uint4 xv[VPL], dv[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = (j * 32 + lane) * V;
      if (c < cols) {
        xv[j] = __ldcs(reinterpret_cast<const uint4*>(xr + c));
        dv[j] = __ldcs(reinterpret_cast<const uint4*>(dyr + c));
      }
    }
    float a1 = 0.f, a2 = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = (j * 32 + lane) * V;
      if (c >= cols) continue;
      float v[V], d[V], g[V];
      load16(reinterpret_cast<const T*>(&xv[j]), v);
      load16(reinterpret_cast<const T*>(&dv[j]), d);
      load16(gamma + c, g);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = (v[i] - mu) * rs;
        const float gd = g[i] * d[i];
        a1 += gd * xh;
        a2 += gd;
        pg[j][i] += d[i] * xh;
        if (LAYER) pb[j][i] += d[i];
      }
    }
    a1 = warp_sum(a1) * inv_cols;
    a2 = warp_sum(a2) * inv_cols;
    T* dxr = dx + row * cols;
    const T* drr = dres ? dres + row * cols : nullptr;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = (j * 32 + lane) * V;
      if (c >= cols) continue;
      float v[V], d[V], g[V], r[V];
      load16(reinterpret_cast<const T*>(&xv[j]), v);
      load16(reinterpret_cast<const T*>(&dv[j]), d);
      load16(gamma + c, g);
      if (drr) load16(drr + c, r);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = (v[i] - mu) * rs;
        float o = rs * (g[i] * d[i] - xh * a1 - (LAYER ? a2 : 0.f));
        if (drr) o += r[i];
        v[i] = o;
      }
      store16(dxr + c, v);
    }
  }
  // CTA reduction of the partials, then 16-byte atomics
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int c = (j * 32 + lane) * V;
    if (c >= cols) continue;
#pragma unroll
    for (int i = 0; i < V; i += 4) {
      *reinterpret_cast<float4*>(sred + warp * cols + c + i) =
          make_float4(pg[j][i], pg[j][i + 1], pg[j][i + 2], pg[j][i + 3]);
      if (LAYER)
        *reinterpret_cast<float4*>(sred + (NW + warp) * cols + c + i) =
            make_float4(pb[j][i], pb[j][i + 1], pb[j][i + 2], pb[j][i + 3]);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x * 4; c < cols; c += blockDim.x * 4) {
    float4 sg = make_float4(0.f, 0.f, 0.f, 0.f), sb = sg;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float4 a = *reinterpret_cast<const float4*>(sred + w * cols + c);
      sg.x += a.x; sg.y += a.y; sg.z += a.z; sg.w += a.w;
      if (LAYER) {
        const float4 bb = *reinterpret_cast<const float4*>(sred + (NW + w) * cols + c);
        sb.x += bb.x; sb.y += bb.y; sb.z += bb.z; sb.w += bb.w;
      }
    }
    atomicAdd(reinterpret_cast<float4*>(dgamma + c), sg);
    if (LAYER) atomicAdd(reinterpret_cast<float4*>(dbeta + c), sb);
  }
}

// GALV_NORM_NARROW=0 turns the register-partials narrow kernel off (A/B)
static bool narrow_enabled() {
  static const bool on = [] {
    const char* e = getenv("GALV_NORM_NARROW");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename T, bool LAYER>
bool launch_narrow_reg(const void* x, const void* gamma, const float* mean, const float* rstd,
                       const void* dy, const void* dres, void* dx, float* dgamma, float* dbeta,
                       int64_t rows, int64_t cols, void* stream) {
  constexpr int V = 16 / (int)sizeof(T);
  if (!narrow_enabled() || cols % (4 * V) != 0 || cols > 32 * V * 4 || cols < 32 * V * 2)
    return false;
  if ((reinterpret_cast<uintptr_t>(dgamma) & 15) || (LAYER && (reinterpret_cast<uintptr_t>(dbeta) & 15)))
    return false;
  const int64_t vpl = (cols / V + 31) / 32;
  auto go = [&](auto kernel) {
    constexpr int NW = NORM_NARROW_WARPS;
    const size_t smem = (size_t)(LAYER ? 2 : 1) * NW * cols * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t grid = std::min<int64_t>((rows + NW - 1) / NW, (int64_t)sm_count());
    kernel<<<(unsigned)grid, NW * 32, smem, as_stream(stream)>>>(
        (const T*)x, (const T*)gamma, mean, rstd, (const T*)dy, (const T*)dres, (T*)dx, dgamma,
        dbeta, rows, (int)cols);
  };
  if (vpl <= 2) go(bwd_narrow_reg<T, LAYER, 2>);
  else if (vpl <= 3) go(bwd_narrow_reg<T, LAYER, 3>);
  else go(bwd_narrow_reg<T, LAYER, 4>);
  return true;
}

template <typename T, bool LAYER>
bool launch_fused_warp(const void* x, const void* gamma, const float* mean, const float* rstd,
                       const void* dy, const void* dres, void* dx, float* dgamma, float* dbeta,
                       int64_t rows, int64_t cols, void* stream) {
  constexpr int V = 16 / (int)sizeof(T);
  if (cols % V != 0 || cols > 32 * V * 4) return false;
  const int64_t vpl = (cols / V + 31) / 32;
  auto go = [&](auto kernel) {
    const size_t smem = (size_t)(LAYER ? 2 : 1) * 8 * cols * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem);
    const int64_t grid =
        std::min<int64_t>((rows + 7) / 8, (int64_t)sm_count() * std::max(per_sm, 1));
    kernel<<<(unsigned)grid, 256, smem, as_stream(stream)>>>(
        (const T*)x, (const T*)gamma, mean, rstd, (const T*)dy, (const T*)dres, (T*)dx, dgamma,
        dbeta, rows, (int)cols);
  };
  if (vpl <= 1) go(bwd_fused_warp_rows<T, LAYER, 1>);
  else if (vpl <= 2) go(bwd_fused_warp_rows<T, LAYER, 2>);
  else if (vpl <= 3) go(bwd_fused_warp_rows<T, LAYER, 3>);
  else go(bwd_fused_warp_rows<T, LAYER, 4>);
  return true;
}

// GALV_NORM_NT=128|256 forces the CTA width (A/B).  Default (B200 A/B, scratch/norm_ab.py,
// profiles/r01/kernels_ab/norm_bwd_ab.jsonl): 256 threads, and the fused kernel only for rows of
// >= 256 vectors (bf16 width >= 2048): 8192x4096 RMS 89.9 -> 65.3 us, 8192x5120 145.9 ->
// 84.8 us, 16384x2048 LN 89.7 -> 84.6 us; at width 1024 the two-kernel pair is faster
// (48.2 vs 53.3 us: one short row per CTA iteration leaves too little in flight).
static int forced_nt() {
  static const int nt = [] {
    const char* e = getenv("GALV_NORM_NT");
    const int v = e ? atoi(e) : 0;
    return (v == 128 || v == 256) ? v : 0;  // the only instantiated widths; else default
  }();
  return nt;
}

template <typename T, bool LAYER>
bool launch_fused(const void* x, const void* gamma, const float* mean, const float* rstd,
                  const void* dy, const void* dres, void* dx, float* dgamma, float* dbeta,
                  int64_t rows, int64_t cols, void* stream) {
  if (fused_disabled()) return false;
  const int64_t vecs = cols / (16 / (int64_t)sizeof(T));
  if (!forced_nt() && vecs < 256) return false;
  const int nt = forced_nt() ? forced_nt() : 256;
  const int64_t nv = (vecs + nt - 1) / nt;
  auto go = [&](auto kernel, int threads) {
    const size_t smem = (size_t)cols * sizeof(float) * (LAYER ? 2 : 1);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    const int64_t grid = std::min<int64_t>(rows, (int64_t)sm_count() * std::max(per_sm, 1));
    kernel<<<(unsigned)grid, threads, smem, as_stream(stream)>>>(
        (const T*)x, (const T*)gamma, mean, rstd, (const T*)dy, (const T*)dres, (T*)dx, dgamma,
        dbeta, rows, (int)cols);
  };
  if (nt == 256) {
    if (nv <= 1) go(bwd_fused_rows<T, LAYER, 1, 256>, 256);
    else if (nv <= 2) go(bwd_fused_rows<T, LAYER, 2, 256>, 256);
    else if constexpr (!LAYER) {
      if (nv <= 3) go(bwd_fused_rows<T, LAYER, 3, 256>, 256);
      else if (nv <= 4) go(bwd_fused_rows<T, LAYER, 4, 256>, 256);
      else return false;
    } else {
      return false;
    }
    return true;
  }
  if (nv <= 1) go(bwd_fused_rows<T, LAYER, 1, 128>, 128);
  else if (nv <= 2) go(bwd_fused_rows<T, LAYER, 2, 128>, 128);
  else if (nv <= 4) go(bwd_fused_rows<T, LAYER, 4, 128>, 128);
  else if constexpr (!LAYER) {  // LayerNorm keeps 2 accumulators per column: NV <= 4
    if (nv <= 5) go(bwd_fused_rows<T, LAYER, 5, 128>, 128);
    else if (nv <= 8) go(bwd_fused_rows<T, LAYER, 8, 128>, 128);
    else return false;
  } else {
    return false;
  }
  return true;
}

template <typename T, bool LAYER>
bool launch_dx_row(const void* x, const void* gamma, const float* mean, const float* rstd,
                   const void* dy, const void* dres, void* dx, int64_t rows, int64_t cols,
                   void* stream) {
  const int64_t nv = (cols / (16 / (int64_t)sizeof(T)) + 127) / 128;
  auto go = [&](auto kernel) {
    kernel<<<(unsigned)rows, 128, 0, as_stream(stream)>>>(
        (const T*)x, (const T*)gamma, mean, rstd, (const T*)dy, (const T*)dres, (T*)dx,
        (int)cols);
  };
  if (rows > 2147483647LL) return false;
  if (nv <= 1) go(bwd_dx_row<T, LAYER, 1>);
  else if (nv <= 2) go(bwd_dx_row<T, LAYER, 2>);
  else if (nv <= 4) go(bwd_dx_row<T, LAYER, 4>);
  else if (nv <= 8) go(bwd_dx_row<T, LAYER, 8>);
  else return false;
  return true;
}

// dgamma[c] += sum_r dy[r,c] * xhat[r,c] (and dbeta[c] += sum_r dy[r,c]): column strips of
// 2*blockDim columns (bf16x2 / float2 loads, coalesced), row chunks across blockIdx.y.
template <typename T, bool LAYER>
__global__ void __launch_bounds__(128) bwd_dgamma_kernel(
    const T* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ rstd,
    const T* __restrict__ dy, float* __restrict__ dgamma, float* __restrict__ dbeta,
    int64_t rows, int cols, int64_t rows_per_cta) {
  const int c = (blockIdx.x * 128 + threadIdx.x) * 2;
  if (c >= cols) return;
  const int64_t r0 = blockIdx.y * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  float g0 = 0.f, g1 = 0.f, b0 = 0.f, b1 = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    const float mu = LAYER ? mean[r] : 0.f, rs = rstd[r];
    float xv0, xv1, d0, d1;
    if constexpr (sizeof(T) == 2) {
      const __nv_bfloat162 xx = *reinterpret_cast<const __nv_bfloat162*>(x + r * cols + c);
      const __nv_bfloat162 dd = *reinterpret_cast<const __nv_bfloat162*>(dy + r * cols + c);
      xv0 = __bfloat162float(xx.x); xv1 = __bfloat162float(xx.y);
      d0 = __bfloat162float(dd.x); d1 = __bfloat162float(dd.y);
    } else {
      const float2 xx = *reinterpret_cast<const float2*>(x + r * cols + c);
      const float2 dd = *reinterpret_cast<const float2*>(dy + r * cols + c);
      xv0 = xx.x; xv1 = xx.y; d0 = dd.x; d1 = dd.y;
    }
    g0 += d0 * (xv0 - mu) * rs;
    g1 += d1 * (xv1 - mu) * rs;
    b0 += d0;
    b1 += d1;
  }
  atomicAdd(&dgamma[c], g0);
  atomicAdd(&dgamma[c + 1], g1);
  if (LAYER) {
    atomicAdd(&dbeta[c], b0);
    atomicAdd(&dbeta[c + 1], b1);
  }
}

}  // namespace norm
}  // namespace galv

using namespace galv;

template <bool LAYER>
static int32_t norm_fwd(const void* x, const void* residual, void* res_out, const void* gamma,
                        const void* beta, void* y, float* mean, float* rstd, int64_t rows,
                        int64_t cols, float eps, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && gamma && y && rstd && rows > 0 && cols > 0, "bad arguments");
  GALV_CHECK_ARG(!LAYER || (beta && mean), "layernorm needs beta and mean");
  GALV_CHECK_ARG(!residual || res_out, "residual needs res_out");
  GALV_CHECK_ARG(cols % 8 == 0, "cols must be a multiple of 8");
  const unsigned grid = (unsigned)((rows + norm::WARPS - 1) / norm::WARPS);
  GALV_DISPATCH(dtype, T, {
    if (residual)
      norm::fwd_kernel<T, LAYER, true><<<grid, norm::WARPS * 32, 0, as_stream(stream)>>>(
          (const T*)x, (const T*)residual, (T*)res_out, (const T*)gamma, (const T*)beta, (T*)y,
          mean, rstd, rows, (int)cols, eps);
    else
      norm::fwd_kernel<T, LAYER, false><<<grid, norm::WARPS * 32, 0, as_stream(stream)>>>(
          (const T*)x, nullptr, nullptr, (const T*)gamma, (const T*)beta, (T*)y, mean, rstd,
          rows, (int)cols, eps);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

template <bool LAYER>
static int32_t norm_bwd(const void* x, const void* gamma, const float* mean, const float* rstd,
                        const void* dy, const void* dres, void* dx, float* dgamma, float* dbeta,
                        int64_t rows, int64_t cols, int32_t dtype, void* stream) {
  GALV_CHECK_ARG(x && gamma && rstd && dy && dx && dgamma && rows > 0, "bad arguments");
  GALV_CHECK_ARG(!LAYER || (mean && dbeta), "layernorm needs mean and dbeta");
  GALV_CHECK_ARG(cols % 8 == 0, "cols must be a multiple of 8");
  const unsigned grid = (unsigned)((rows + norm::WARPS - 1) / norm::WARPS);
  const int64_t strips = (cols / 2 + 127) / 128;
  const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(rows / 32 + 1,
                                                                (int64_t)sm_count() * 8 / strips + 1));
  const int64_t rpc = (rows + chunks - 1) / chunks;
  GALV_DISPATCH(dtype, T, {
    if (norm::launch_fused<T, LAYER>(x, gamma, mean, rstd, dy, dres, dx, dgamma, dbeta, rows,
                                     cols, stream))
      break;
    if (!norm::fused_disabled() &&
        norm::launch_narrow_reg<T, LAYER>(x, gamma, mean, rstd, dy, dres, dx, dgamma, dbeta,
                                          rows, cols, stream))
      break;
    if (!norm::fused_disabled() && norm::warp_rows_enabled() &&
        (reinterpret_cast<uintptr_t>(gamma) & 15) == 0 &&
        norm::launch_fused_warp<T, LAYER>(x, gamma, mean, rstd, dy, dres, dx, dgamma, dbeta,
                                          rows, cols, stream))
      break;
    if (!norm::launch_dx_row<T, LAYER>(x, gamma, mean, rstd, dy, dres, dx, rows, cols, stream))
      norm::bwd_dx_kernel<T, LAYER><<<grid, norm::WARPS * 32, 0, as_stream(stream)>>>(
          (const T*)x, (const T*)gamma, mean, rstd, (const T*)dy, (const T*)dres, (T*)dx, rows,
          (int)cols);
    norm::bwd_dgamma_kernel<T, LAYER><<<dim3((unsigned)strips, (unsigned)chunks), 128, 0,
                                        as_stream(stream)>>>(
        (const T*)x, mean, rstd, (const T*)dy, dgamma, dbeta, rows, (int)cols, rpc);
  });
  GALV_LAUNCH_CHECK();
  return 0;
}

extern "C" {

int32_t galv_rmsnorm_fwd(const void* x, const void* residual, void* res_out, const void* gamma,
                         void* y, float* rstd, int64_t rows, int64_t cols, float eps,
                         int32_t dtype, void* stream) {
  return norm_fwd<false>(x, residual, res_out, gamma, nullptr, y, nullptr, rstd, rows, cols, eps,
                         dtype, stream);
}

int32_t galv_rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy,
                         const void* dres_in, void* dx, float* dgamma_acc, int64_t rows,
                         int64_t cols, int32_t dtype, void* ws, void* stream) {
  (void)ws;
  return norm_bwd<false>(x, gamma, nullptr, rstd, dy, dres_in, dx, dgamma_acc, nullptr, rows,
                         cols, dtype, stream);
}

int32_t galv_layernorm_fwd(const void* x, const void* residual, void* res_out, const void* gamma,
                           const void* beta, void* y, float* mean, float* rstd, int64_t rows,
                           int64_t cols, float eps, int32_t dtype, void* stream) {
  return norm_fwd<true>(x, residual, res_out, gamma, beta, y, mean, rstd, rows, cols, eps, dtype,
                        stream);
}

int32_t galv_layernorm_bwd(const void* x, const void* gamma, const float* mean, const float* rstd,
                           const void* dy, const void* dres_in, void* dx, float* dgamma_acc,
                           float* dbeta_acc, int64_t rows, int64_t cols, int32_t dtype, void* ws,
                           void* stream) {
  (void)ws;
  return norm_bwd<true>(x, gamma, mean, rstd, dy, dres_in, dx, dgamma_acc, dbeta_acc, rows, cols,
                        dtype, stream);
}

int64_t galv_norm_bwd_workspace(int64_t rows, int64_t cols) {
  (void)rows;
  (void)cols;
  return 0;
}

}  // extern "C"
