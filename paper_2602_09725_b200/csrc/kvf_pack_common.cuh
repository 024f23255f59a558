// kvf_pack_common.cuh — pieces shared by the phase-split and the single-read
// (persistent) pack kernels: unit descriptor, source vector loads, |x| maxima,
// the exact quantiser and the per-warp frame-item loop.
//
// Quantisation is the reference's (fk/kvmodel.py:127-144): per (layer, group)
// scale = fp32(fp64(max|x|)/127) or 1.0, q = clip(rint_half_even(fp64 x / fp64 s),
// -127, 127); the frame sample is q + 128 (fk/layout.py:246-250).
#pragma once

#include "kvf_common.cuh"

namespace kvf {

constexpr int kPackThreads = 256;
constexpr int kPackWarps = kPackThreads / 32;
constexpr int kMaxPackUnits = 96;  // descriptors per launch (kernel params <= 32 KB)

// Scratch words of a unit (kvf_pack_scratch_words): [3, G] |x| maxima (f32
// bit patterns) | [3, G] counter words.
inline int64_t pack_scratch_words(const kvf_plan& p) {
  const int64_t G = (int64_t)p.H * p.D / p.group_size;
  return 6 * G;
}

struct PackUnitDev {
  kvf_paged src;
  Geom g;
  uint32_t* absmax;       // [3, G] maxima (f32 bit patterns)
  uint32_t* counters;     // absmax + 3G: [3, G] counter words
  float* scales;
  kvf_surface fr;
  FastDiv div_bs;
  int32_t n_items;  // frame_count * tiles_per_frame (per plane)
  int32_t G;
  int32_t n_scratch;
};

inline PackUnitDev make_pack_unit_dev(const kvf_pack_unit& u) {
  PackUnitDev d;
  d.src = u.src;
  d.g = make_geom(u.plan);
  d.G = (u.plan.H * u.plan.D) / u.plan.group_size;
  d.absmax = u.absmax;
  d.counters = u.absmax ? u.absmax + 3 * d.G : nullptr;
  d.n_scratch = 6 * d.G;  // the phase-split kernels use maxima + counters only
  d.scales = u.scales;
  d.fr = u.frames;
  d.div_bs = make_fastdiv(u.src.block_size);
  d.n_items = u.plan.frame_count * u.plan.tiles_per_frame;
  return d;
}

// Source vector loads (optionally tagged with an L2 eviction policy).
struct NoPolicy {
  __device__ __forceinline__ uint4 load(const char* p) const { return ld_nc_v4(p); }
};
struct KeepLoad {  // coherent path: the line stays in L2 for a re-read
  __device__ __forceinline__ uint4 load(const char* p) const { return ld_keep_v4(p); }
};
struct WithPolicy {
  uint64_t pol;
  __device__ __forceinline__ uint4 load(const char* p) const { return ld_nc_v4_pol(p, pol); }
};

// max |x| bit pattern over 8 values (16-bit patterns for bf16/fp16, which order
// like the magnitudes they encode; f32 bits for fp32).
template <int SRC, typename LD = NoPolicy>
__device__ __forceinline__ uint32_t vec_absmax_bits(const char* p, LD ld = LD()) {
  if constexpr (SRC == KVF_F32) {
    uint4 a = ld.load(p), b = ld.load(p + 16);
    uint32_t m = max(max(a.x & 0x7FFFFFFFu, a.y & 0x7FFFFFFFu),
                     max(a.z & 0x7FFFFFFFu, a.w & 0x7FFFFFFFu));
    m = max(m, max(max(b.x & 0x7FFFFFFFu, b.y & 0x7FFFFFFFu),
                   max(b.z & 0x7FFFFFFFu, b.w & 0x7FFFFFFFu)));
    return m;
  } else {
    uint4 a = ld.load(p);
    uint32_t w0 = a.x & 0x7FFF7FFFu, w1 = a.y & 0x7FFF7FFFu;
    uint32_t w2 = a.z & 0x7FFF7FFFu, w3 = a.w & 0x7FFF7FFFu;
    uint32_t hi = max(max(w0, w1), max(w2, w3)) & 0xFFFF0000u;  // high halves
    uint32_t lo = max(max(w0 & 0xFFFFu, w1 & 0xFFFFu), max(w2 & 0xFFFFu, w3 & 0xFFFFu));
    return max(hi >> 16, lo);
  }
}

// 16-bit |x| pattern (or f32 bits) -> f32 bits of |x|.
template <int SRC>
__device__ __forceinline__ uint32_t absmax_to_f32_bits(uint32_t m) {
  if constexpr (SRC == KVF_BF16) return m << 16;
  if constexpr (SRC == KVF_F16)
    return __float_as_uint(__half2float(__ushort_as_half((unsigned short)m)));
  return m;
}

// Raw source words of one 8-value vector (bf16/fp16: 16 B; fp32: 32 B).
template <int SRC>
struct Raw8 {
  uint4 a;
  uint4 b;  // fp32 only
};

template <int SRC, typename LD = NoPolicy>
__device__ __forceinline__ Raw8<SRC> load_raw8(const char* p, LD ld = LD()) {
  Raw8<SRC> r;
  r.a = ld.load(p);
  if constexpr (SRC == KVF_F32) r.b = ld.load(p + 16);
  return r;
}

template <int SRC>
__device__ __forceinline__ void raw8_to_float(const Raw8<SRC>& r, float (&x)[8]) {
  if constexpr (SRC == KVF_F32) {
    x[0] = __uint_as_float(r.a.x); x[1] = __uint_as_float(r.a.y);
    x[2] = __uint_as_float(r.a.z); x[3] = __uint_as_float(r.a.w);
    x[4] = __uint_as_float(r.b.x); x[5] = __uint_as_float(r.b.y);
    x[6] = __uint_as_float(r.b.z); x[7] = __uint_as_float(r.b.w);
  } else {
    const uint32_t w[4] = {r.a.x, r.a.y, r.a.z, r.a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (SRC == KVF_BF16) {
        x[2 * k] = __uint_as_float(w[k] << 16);
        x[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
      } else {
        __half2 h = *reinterpret_cast<const __half2*>(&w[k]);
        float2 f = __half22float2(h);
        x[2 * k] = f.x;
        x[2 * k + 1] = f.y;
      }
    }
  }
}

template <int SRC, typename LD = NoPolicy>
__device__ __forceinline__ void load_vec8(const char* p, float (&x)[8], LD ld = LD()) {
  raw8_to_float<SRC>(load_raw8<SRC>(p, ld), x);
}

__device__ __forceinline__ uint32_t pack_codes4(int a, int b, int c, int d) {
  return (uint32_t)((a + 128) & 0xFF) | ((uint32_t)((b + 128) & 0xFF) << 8) |
         ((uint32_t)((c + 128) & 0xFF) << 16) | ((uint32_t)((d + 128) & 0xFF) << 24);
}

// Exact path for a whole vector (rare): out of line to keep the hot loop small.
static __device__ __noinline__ uint2 quantize8_exact(float x0, float x1, float x2, float x3,
                                                     float x4, float x5, float x6, float x7,
                                                     float s, float inv) {
  return make_uint2(pack_codes4(quantize_exact(x0, s, inv), quantize_exact(x1, s, inv),
                                quantize_exact(x2, s, inv), quantize_exact(x3, s, inv)),
                    pack_codes4(quantize_exact(x4, s, inv), quantize_exact(x5, s, inv),
                                quantize_exact(x6, s, inv), quantize_exact(x7, s, inv)));
}

// Packed FP32 pair arithmetic (sm_100a FFMA2/FADD2/FMUL2 via PTX .f32x2).
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t v;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(lo), "f"(hi));
  return v;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// 8 values -> 8 frame bytes (q + 128), bit-identical to quantize_exact.
// Fast path (packed FP32 pairs): y = x * (1/s), RNE to an integer by adding
// 1.5*2^23 (the sum's ulp is 1, so the add itself rounds half-to-even) whose
// low mantissa byte is q mod 256; XOR 0x80 turns it into q + 128.  y is within
// 2^-16 of x/s, so only a vector with some |y - r| within 2^-14 of 1/2 can
// round differently from the reference's fp64 division: such vectors (and,
// when kRange, any |y| beyond the clip range) are redone exactly.  Without
// kRange the caller guarantees |x| <= the group max the scale came from, which
// bounds |y| <= 127 * (1 + 2^-22).
// Fast path only; `bad` is set when the vector must be redone exactly.  The
// rounding residual d is within 2^-16 of the exact one (reciprocal error
// <= 2^-17 at |x/s| <= 128, plus at most one fp32 rounding of the product), so
// only |d| > 1/2 - 2^-15 can round differently from the reference.
template <bool kRange = true>
__device__ __forceinline__ uint2 quantize8_fast(const float (&x)[8], float inv, bool& bad) {
  const uint64_t kMagic2 = 0x4B4000004B400000ull;  // {1.5*2^23, 1.5*2^23}
  const uint64_t inv2 = f2_pack(inv, inv);
  uint32_t w[8];
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    const uint64_t y = f2_mul(f2_pack(x[e], x[e + 1]), inv2);
    const uint64_t rp = f2_add(y, kMagic2);
    const uint64_t d = f2_sub(y, f2_sub(rp, kMagic2));
    float d0, d1, y0, y1, r0, r1;
    f2_unpack(d, d0, d1);
    bad |= (fabsf(d0) > 0.499969482421875f) | (fabsf(d1) > 0.499969482421875f);
    if constexpr (kRange) {
      f2_unpack(y, y0, y1);
      bad |= (fabsf(y0) > 127.25f) | (fabsf(y1) > 127.25f);
    }
    f2_unpack(rp, r0, r1);
    w[e] = __float_as_uint(r0);
    w[e + 1] = __float_as_uint(r1);
  }
  uint2 out;
  out.x = __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410) ^
          0x80808080u;
  out.y = __byte_perm(__byte_perm(w[4], w[5], 0x0040), __byte_perm(w[6], w[7], 0x0040), 0x5410) ^
          0x80808080u;
  return out;
}

template <bool kRange = true>
__device__ __forceinline__ uint2 quantize8(const float (&x)[8], float s, float inv) {
  const uint64_t kMagic2 = 0x4B4000004B400000ull;  // {1.5*2^23, 1.5*2^23}
  const uint64_t inv2 = f2_pack(inv, inv);
  uint32_t w[8];
  bool bad = false;
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    const uint64_t y = f2_mul(f2_pack(x[e], x[e + 1]), inv2);
    const uint64_t rp = f2_add(y, kMagic2);
    const uint64_t d = f2_sub(y, f2_sub(rp, kMagic2));
    float d0, d1, y0, y1, r0, r1;
    f2_unpack(d, d0, d1);
    bad |= (fabsf(d0) > 0.49993896484375f) | (fabsf(d1) > 0.49993896484375f);
    if constexpr (kRange) {
      f2_unpack(y, y0, y1);
      bad |= (fabsf(y0) > 127.25f) | (fabsf(y1) > 127.25f);
    }
    f2_unpack(rp, r0, r1);
    w[e] = __float_as_uint(r0);
    w[e + 1] = __float_as_uint(r1);
  }
  uint2 out;
  out.x = __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410) ^
          0x80808080u;
  out.y = __byte_perm(__byte_perm(w[4], w[5], 0x0040), __byte_perm(w[6], w[7], 0x0040), 0x5410) ^
          0x80808080u;
  if (__builtin_expect(bad, 0))
    out = quantize8_exact(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], s, inv);
  return out;
}

// ------------------------------------------------------------ frame items
constexpr int kIPW = 8;  // frame items per warp run

// absmax tokens per warp (phase-split absmax kernel): 8 for C >= 1024 channels,
// more for narrow slots so a CTA still reads ~128 KB
__host__ __device__ constexpr int tok_per_warp(int vpl) { return vpl >= 4 ? 8 : 32 / vpl; }

// Narrow slots (VPL 1 / 2) run SUB items side by side in a warp, 32/SUB lanes
// each, so a lane still handles 4 vectors per item round (as in restore).
template <int SRC, int VPL>
__host__ __device__ constexpr int pack_sub() {
  return (SRC != KVF_I8 && VPL < 4) ? 4 / VPL : 1;
}

// Warp-group reduction of per-lane maxima into s_max[group] (lanes lane+32k of
// one group are gs/8 consecutive lanes when gs <= 256, else the whole warp).
template <int SRC, int VPL>
__device__ __forceinline__ void reduce_groups(const uint32_t (&m)[VPL], int group_size,
                                              uint32_t* s_max) {
  const int lane = threadIdx.x & 31;
  const int lpg = group_size >> 3;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    uint32_t v = absmax_to_f32_bits<SRC>(m[k]);
    for (int o = 1; o < 32 && o < lpg; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((lane & (min(lpg, 32) - 1)) == 0 && v) atomicMax(&s_max[(lane + 32 * k) / lpg], v);
  }
}

// Per-lane constants of one (unit, plane) for the frame-item loop: source and
// tile offsets of the lane's 8-channel vectors and their group scales.
template <int SRC, int VPL>
struct PackLane {
  static constexpr int SUB = pack_sub<SRC, VPL>();
  static constexpr int LPI = 32 / SUB;
  static constexpr int VL = VPL * SUB;
  int32_t in_off[VL], tile_off[VL];
  float s[VL], inv[VL];

  // `scales`: the plane's [G] scales (ignored for int8 sources).
  __device__ __forceinline__ void init(const PackUnitDev& U, int p, const float* scales) {
    constexpr int ES = SRC == KVF_F32 ? 4 : (SRC == KVF_I8 ? 1 : 2);
    const int sl = (threadIdx.x & 31) % LPI;
#pragma unroll
    for (int k = 0; k < VL; ++k) {
      const int c = (sl + LPI * k) * 8;
      in_off[k] = (int32_t)slot_channel_offset(U.g, c, U.src.head_stride) * ES;
      tile_off[k] = (int32_t)tile_offset(U.g, c, U.fr.row_pitch);
      if constexpr (SRC != KVF_I8) {
        s[k] = scales[c >> U.g.lg_gs];
        inv[k] = __frcp_rn(s[k]);
      }
    }
  }
};

// One warp packs frame items of plane p in `rounds` rounds: round r takes items
// item0 + r*stride + sub (sub < SUB, lanes split SUB ways), those below `end`.
// Item q = (frame, tile slot) -> its token's quantised slot at the tile origin,
// or a pad tile of 128s.  Rounds are software-pipelined (the loads of round
// r+1 are in flight while round r is quantised and stored).
template <int SRC, int VPL, bool kRange, typename LD = NoPolicy>
__device__ __forceinline__ void pack_items(const PackUnitDev& U, int p,
                                           const PackLane<SRC, VPL>& L, int item0, int stride,
                                           int rounds, int end, LD ld = LD()) {
  constexpr int SUB = PackLane<SRC, VPL>::SUB;
  constexpr int LPI = PackLane<SRC, VPL>::LPI;
  constexpr int VL = PackLane<SRC, VPL>::VL;
  constexpr int ES = SRC == KVF_F32 ? 4 : (SRC == KVF_I8 ? 1 : 2);
  const int sub = (threadIdx.x & 31) / LPI;
  const char* layer = reinterpret_cast<const char*>(U.src.layer[p]);
  uint8_t* plane_base = U.fr.base + (int64_t)p * U.fr.plane_stride;
  // Item q -> (tile origin in the plane, source slot or null for a pad tile).
  auto locate = [&](int q, uint8_t*& dst, const char*& srcp) {
    const int f = fdiv(U.g.div_tpf, q);
    const int slot = q - f * U.g.tpf;
    const int i = token_of(U.g, f, slot);
    const int tr = fdiv(U.g.div_cols, slot);
    const int tc = slot - tr * U.g.grid_cols;
    dst = plane_base + (int64_t)f * U.fr.frame_stride +
          (int64_t)tr * U.g.tile_h * U.fr.row_pitch + (int64_t)tc * U.g.tile_w;
    srcp = (i < U.g.T && layer != nullptr)
               ? layer + paged_slot_offset_fd(U.src, U.div_bs, i) * ES
               : nullptr;
  };
  if constexpr (SRC == KVF_I8 || VPL > 4) {
    for (int it = 0; it < rounds; ++it) {
      const int q = item0 + it * stride + sub;
      if (q >= end) break;
      uint8_t* dst;
      const char* slotp;
      locate(q, dst, slotp);
      if (slotp == nullptr) {
#pragma unroll
        for (int k = 0; k < VL; ++k)
          st_v2(dst + L.tile_off[k], make_uint2(0x80808080u, 0x80808080u));
        continue;
      }
      if constexpr (SRC == KVF_I8) {
        uint2 v[VL];
#pragma unroll
        for (int k = 0; k < VL; ++k) v[k] = ld_nc_v2(slotp + L.in_off[k]);
#pragma unroll
        for (int k = 0; k < VL; ++k)
          st_v2(dst + L.tile_off[k], make_uint2(v[k].x ^ 0x80808080u, v[k].y ^ 0x80808080u));
      } else {
#pragma unroll
        for (int k0 = 0; k0 < VL; k0 += 4) {  // at most 32 live values per lane
          float x[4][8];
#pragma unroll
          for (int k = 0; k < 4; ++k) load_vec8<SRC>(slotp + L.in_off[k0 + k], x[k], ld);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            st_v2(dst + L.tile_off[k0 + k],
                  quantize8<kRange>(x[k], L.s[k0 + k], L.inv[k0 + k]));
        }
      }
    }
  } else if constexpr (SUB == 1) {
    // Software pipeline: the loads of item it+1 are in flight while item it is
    // quantised and stored.  The item addresses are located lane-parallel:
    // lane l locates round r0 + l once for the warp (instead of every lane
    // locating every round) and round it takes them with two shuffles.
    const int lane = threadIdx.x & 31;
    uint8_t* my_dst = nullptr;
    const char* my_src = nullptr;
    auto fill = [&](int r0) {
      const int q = item0 + (r0 + lane) * stride;
      my_dst = nullptr;
      my_src = nullptr;
      if (r0 + lane < rounds && q < end) locate(q, my_dst, my_src);
    };
    auto get = [&](int it, uint8_t*& d, const char*& sp) {
      d = reinterpret_cast<uint8_t*>(__shfl_sync(
          0xffffffffu, (unsigned long long)reinterpret_cast<uintptr_t>(my_dst), it & 31));
      sp = reinterpret_cast<const char*>(__shfl_sync(
          0xffffffffu, (unsigned long long)reinterpret_cast<uintptr_t>(my_src), it & 31));
    };
    Raw8<SRC> cur[VL], nxt[VL];
    uint8_t* dst_cur = nullptr;
    const char* src_cur = nullptr;
    const int n_it = rounds;  // warp-uniform
    fill(0);
    get(0, dst_cur, src_cur);
    if (src_cur)
#pragma unroll
      for (int k = 0; k < VL; ++k) cur[k] = load_raw8<SRC>(src_cur + L.in_off[k], ld);
    for (int it = 0; it < n_it; ++it) {
      uint8_t* dst_nxt = nullptr;
      const char* src_nxt = nullptr;
      if (it + 1 < n_it) {
        if (((it + 1) & 31) == 0) fill(it + 1);
        get(it + 1, dst_nxt, src_nxt);
        if (src_nxt)
#pragma unroll
          for (int k = 0; k < VL; ++k) nxt[k] = load_raw8<SRC>(src_nxt + L.in_off[k], ld);
      }
      if (dst_cur != nullptr) {
#pragma unroll
        for (int k = 0; k < VL; ++k) {
          uint2 out = make_uint2(0x80808080u, 0x80808080u);
          if (src_cur) {
            float x[8];
            raw8_to_float<SRC>(cur[k], x);
            out = quantize8<kRange>(x, L.s[k], L.inv[k]);
          }
          st_v2(dst_cur + L.tile_off[k], out);
        }
      }
#pragma unroll
      for (int k = 0; k < VL; ++k) cur[k] = nxt[k];
      dst_cur = dst_nxt;
      src_cur = src_nxt;
    }
  } else {
    // Software pipeline: the loads of item it+1 are in flight while item it is
    // quantised and stored.
    Raw8<SRC> cur[VL], nxt[VL];
    uint8_t* dst_cur = nullptr;
    const char* src_cur = nullptr;
    const int n_it = rounds;  // warp-uniform
    if (item0 + sub < end) locate(item0 + sub, dst_cur, src_cur);
    if (src_cur)
#pragma unroll
      for (int k = 0; k < VL; ++k) cur[k] = load_raw8<SRC>(src_cur + L.in_off[k], ld);
    for (int it = 0; it < n_it; ++it) {
      uint8_t* dst_nxt = nullptr;
      const char* src_nxt = nullptr;
      const int qn = item0 + (it + 1) * stride + sub;
      if (it + 1 < n_it && qn < end) {
        locate(qn, dst_nxt, src_nxt);
        if (src_nxt)
#pragma unroll
          for (int k = 0; k < VL; ++k) nxt[k] = load_raw8<SRC>(src_nxt + L.in_off[k], ld);
      }
      if (dst_cur != nullptr) {
#pragma unroll
        for (int k = 0; k < VL; ++k) {
          uint2 out = make_uint2(0x80808080u, 0x80808080u);
          if (src_cur) {
            float x[8];
            raw8_to_float<SRC>(cur[k], x);
            out = quantize8<kRange>(x, L.s[k], L.inv[k]);
          }
          st_v2(dst_cur + L.tile_off[k], out);
        }
      }
#pragma unroll
      for (int k = 0; k < VL; ++k) cur[k] = nxt[k];
      dst_cur = dst_nxt;
      src_cur = src_nxt;
    }
  }
}

}  // namespace kvf
