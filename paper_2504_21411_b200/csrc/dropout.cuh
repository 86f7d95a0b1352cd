// Attention-probability dropout: a counter-based keep mask from Philox4x32-10 (Salmon et
// al., SC'11; the Random123 round / key schedule), so every kernel that touches P -- the
// forward and both backward kernels, bf16 tcgen05 and fp32 SIMT -- regenerates the same
// mask from coordinates alone, with nothing stored.  The CPU restatement used by the tests
// is oracle/dropout_ref.py.
//
// Element (query i, key j) of global sample bg = b0 + b and global head hg = h0 + h:
//   counter = (j / 4, i, bg * H_total + hg, offset), key = (seed_lo, seed_hi)
//   u = philox4x32_10(counter, key)[j % 4];  kept iff u >= thresh, thresh = p * 2^32.
// Kept probabilities are scaled by 1 / (1 - p); the softmax normalization (and the lse the
// backward recomputes P from) uses the undropped probabilities.
#pragma once
#include <stdint.h>

namespace galv {

struct DropoutParams {
  uint32_t thresh = 0;  // 0: no dropout
  uint32_t seed_lo = 0, seed_hi = 0;
  uint32_t offset = 0;
  int32_t b0 = 0, h0 = 0, H_total = 1;
  float inv_keep = 1.f;
};

__host__ inline DropoutParams make_dropout(float p, uint64_t seed, uint64_t offset, int64_t b0,
                                           int64_t h0, int64_t H_total) {
  DropoutParams d;
  if (p > 0.f) {
    const double t = (double)p * 4294967296.0;
    d.thresh = t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
    if (d.thresh == 0) d.thresh = 1;
    d.inv_keep = (float)(1.0 / (1.0 - (double)p));
  }
  d.seed_lo = (uint32_t)seed;
  d.seed_hi = (uint32_t)(seed >> 32);
  d.offset = (uint32_t)offset;
  d.b0 = (int32_t)b0;
  d.h0 = (int32_t)h0;
  d.H_total = (int32_t)H_total;
  return d;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// keep bits (bit e = key j4 + e) of the 4 keys j4..j4+3 (j4 % 4 == 0) for query row i of the
// call-local (b, h)
__device__ __forceinline__ uint32_t dropout_keep4(const DropoutParams& d, int b, int h, int i,
                                                  int j4) {
  const uint32_t bh = (uint32_t)((d.b0 + b) * d.H_total + d.h0 + h);
  const uint4 r = philox4x32_10(make_uint4((uint32_t)j4 >> 2, (uint32_t)i, bh, d.offset),
                                d.seed_lo, d.seed_hi);
  return (uint32_t)(r.x >= d.thresh) | ((uint32_t)(r.y >= d.thresh) << 1) |
         ((uint32_t)(r.z >= d.thresh) << 2) | ((uint32_t)(r.w >= d.thresh) << 3);
}

__device__ __forceinline__ bool dropout_keep(const DropoutParams& d, int b, int h, int i, int j) {
  return (dropout_keep4(d, b, h, i, j & ~3) >> (j & 3)) & 1u;
}

}  // namespace galv
