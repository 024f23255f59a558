// kvf_rc_model.cuh — the adaptive order-0 model of the reference range coder
// (fk/rangecoder.py:44-103) as the GPU decoder and encoder hold it, plus the
// exact `rng / total` both need.  One thread owns one stream's model.
#pragma once

#include "kvf_common.cuh"

namespace kvf {
namespace rc {

constexpr uint32_t kTop = 1u << 24;
constexpr uint32_t kBot = 1u << 16;
constexpr uint32_t kInc = 32;
constexpr uint32_t kLimit = 1u << 16;

// The reference model (fk/rangecoder.py:53-103: 256 counts starting at 1,
// +INC per coded symbol, halving at TOTAL_LIMIT) held as cumulative counts in
// 16 blocks of 16 symbols:
//   CB[k]        = count of symbols in blocks < k           (registers, CB[0] = 0)
//   incl[16b+j]  = sum of counts of block b symbols 0..j    (u16 in shared memory)
// so cum(16b + j) = CB[b] + incl[16b + j - 1].  Counts fit 16 bits: total <
// 2^16 while decoding (fk/rangecoder.py:186-188).  A thread's 256 entries are
// 32 x 16 B: chunk (b, half) of thread t at ((2b + half) * 32 + t) * 16 B, so a
// block is two conflict-free 128-bit loads and two 128-bit stores.
constexpr int kDecThreads = 32;  // one warp per CTA: 16 KB of models, 14 CTAs per SM

__device__ __forceinline__ uint32_t lo16(uint32_t w) { return w & 0xFFFFu; }

// 1/t to ~1 ulp (MUFU.RCP): the exact division below tolerates 4 ulp.
__device__ __forceinline__ float rcp_approx(uint32_t t) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint2float_rn(t)));
  return y;
}
__device__ __forceinline__ uint32_t hi16(uint32_t w) { return w >> 16; }

// Halve every count ((f + 1) >> 1, fk/rangecoder.py:93-103) and rebuild the
// cumulative arrays; returns the new total.
__device__ __forceinline__ uint32_t rebuild(uint4* m, uint32_t (&P)[8]) {
  uint32_t total = 0;
#pragma unroll 1
  for (int b = 0; b < 16; ++b) {
    uint4 c0 = m[(2 * b) * kDecThreads], c1 = m[(2 * b + 1) * kDecThreads];
    const uint32_t wv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    uint32_t out[8], prev = 0, acc = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t inc = (j & 1) ? hi16(wv[j >> 1]) : lo16(wv[j >> 1]);
      const uint32_t f = ((inc - prev) + 1) >> 1;
      prev = inc;
      acc += f;
      if (j & 1) out[j >> 1] |= acc << 16; else out[j >> 1] = acc;
    }
    m[(2 * b) * kDecThreads] = make_uint4(out[0], out[1], out[2], out[3]);
    m[(2 * b + 1) * kDecThreads] = make_uint4(out[4], out[5], out[6], out[7]);
    total += acc;
  }
  uint32_t run = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    if (b & 1) P[b >> 1] |= run << 16; else P[b >> 1] = run;
    const uint4 c1 = m[(2 * b + 1) * kDecThreads];
    run += hi16(c1.w);
  }
  return total;
}

// r = rng / total exactly (fk/rangecoder.py:118,163) in fp32: with rcp within
// 4 ulp of 1/total, q0 = RZ(RN(rng) * rcp) is within 8 of the quotient
// (rng < 2^32, total in [256, 2^16)); one floor((rng - q0 total) * rcp) step
// and a +-1 fix-up make it exact (checked against integer division on 3.5e7
// cases incl. every k*total +- 1 edge, with rcp perturbed 1-4 ulp).
__device__ __forceinline__ uint32_t exact_div(uint32_t rng, uint32_t total, float rcp) {
  const uint32_t q0 = __float2uint_rz(__fmul_rn(__uint2float_rn(rng), rcp));
  const int32_t rem0 = (int32_t)(rng - q0 * total);
  const int32_t d = __float2int_rd(__fmul_rn((float)rem0, rcp));
  const int32_t rem1 = rem0 - d * (int32_t)total;
  return q0 + (uint32_t)d + (rem1 >= (int32_t)total ? 1u : 0u) - (rem1 < 0 ? 1u : 0u);
}

// counts start at 1: incl[16b + j] = j + 1, CB[k] = 16k (packed: P[w] = CB[2w] | CB[2w+1] << 16)
__device__ __forceinline__ void model_init(uint4* m, uint32_t (&P)[8]) {
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const uint32_t j0 = (c & 1) * 8 + 1;
    m[c * kDecThreads] = make_uint4(j0 | (j0 + 1) << 16, (j0 + 2) | (j0 + 3) << 16,
                                    (j0 + 4) | (j0 + 5) << 16, (j0 + 6) | (j0 + 7) << 16);
  }
#pragma unroll
  for (int w = 0; w < 8; ++w) P[w] = (32u * w) | ((32u * w + 16u) << 16);
}

// Increment rows: row t (t = 0..16) is 8 packed words, word w holding INC in
// its low half if 2w >= t and in its high half if 2w + 1 >= t.  Row sl is
// what a symbol at block slot sl adds to its block's inclusive sums; row
// blk + 1 is what it adds to the packed block prefixes (CB[q] for q > blk).
// One table per CTA in shared memory (544 B); the kernels load row blk + 1 as
// soon as blk is known, so the load is off the next symbol's search chain.
constexpr int kAddRows = 17;
__device__ __forceinline__ void add_table_init(uint4* T) {
  for (uint32_t i = threadIdx.x; i < 2 * kAddRows; i += 32) {
    const uint32_t t = i >> 1, w0 = (i & 1) * 4;
    uint32_t a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t w = w0 + k;
      a[k] = (2u * w >= t ? kInc : 0u) | (2u * w + 1 >= t ? kInc << 16 : 0u);
    }
    T[i] = make_uint4(a[0], a[1], a[2], a[3]);
  }
  __syncwarp();
}

__device__ __forceinline__ uint32_t cb_lo(uint32_t w) { return w & 0xFFFFu; }
__device__ __forceinline__ uint32_t cb_hi(uint32_t w) { return w >> 16; }

// freq[s] += INC (fk/rangecoder.py:60-66): incl[16 blk + j] += INC for j >= sl
// (the block's 8 packed words `wv` plus table row sl, two 128-bit stores) and
// CB[q] += INC for q > blk (the packed prefixes plus row blk + 1, `cbi`,
// loaded by the caller as soon as blk was known).
__device__ __forceinline__ void model_update(uint4* m, uint32_t (&P)[8], uint32_t blk,
                                             uint32_t sl, const uint32_t (&wv)[8],
                                             const uint4* T, const uint4 (&cbi)[2]) {
  const uint4 a0 = T[2 * sl], a1 = T[2 * sl + 1];
  const uint32_t add[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
  uint32_t nv[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) nv[w] = wv[w] + add[w];
  m[(2 * blk) * kDecThreads] = make_uint4(nv[0], nv[1], nv[2], nv[3]);
  m[(2 * blk + 1) * kDecThreads] = make_uint4(nv[4], nv[5], nv[6], nv[7]);
  P[0] += cbi[0].x; P[1] += cbi[0].y; P[2] += cbi[0].z; P[3] += cbi[0].w;
  P[4] += cbi[1].x; P[5] += cbi[1].y; P[6] += cbi[1].z; P[7] += cbi[1].w;
}

}  // namespace rc
}  // namespace kvf
