// kvf_common.cuh — shared device/host helpers for the sm_100a KV-frame kernels.
//
// Index conventions follow the reference framekv package (see include/kvf.h):
//   channel c = h*D + d; tile (row, col) = (i_h*a_d + i_d, j_h*b_d + j_d)
//   (fk/layout.py:31-36, 244-250); token placement fk/layout.py:195-201.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/kvf.h"

namespace kvf {

// ---------------------------------------------------------------- host errors
void set_error(const char* fmt, ...);
kvf_status cuda_status(cudaError_t e, const char* what);

#define KVF_CHECK_CUDA(expr)                                   \
  do {                                                         \
    cudaError_t e_ = (expr);                                   \
    if (e_ != cudaSuccess) return ::kvf::cuda_status(e_, #expr); \
  } while (0)

#define KVF_FAIL(code, ...)            \
  do {                                 \
    ::kvf::set_error(__VA_ARGS__);     \
    return (code);                     \
  } while (0)

inline int ilog2(int64_t v) {
  int r = 0;
  while ((int64_t(1) << r) < v) ++r;
  return r;
}
inline bool is_pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }

// Host-side validation of a plan filled by kvf_plan_init (fields consistent).
kvf_status check_plan(const kvf_plan& p);
size_t dtype_size(int32_t dt);

// Division by a runtime-constant divisor d >= 1 for dividends n < 2^31:
// q = umulhi(n, m) >> s with m = ceil(2^(31+ceil(log2 d)) / d), s = ceil(log2 d)-1
// (the multiply-high scheme of Granlund & Montgomery); d == 1 passes through.
struct FastDiv {
  uint32_t m;
  int32_t s;
  int32_t d;
};

inline FastDiv make_fastdiv(int32_t d) {
  FastDiv f;
  f.d = d;
  if (d <= 1) {
    f.m = 0;
    f.s = 0;
    return f;
  }
  int l = ilog2(d);
  uint64_t p = 31 + l;
  f.m = (uint32_t)(((uint64_t(1) << p) + d - 1) / d);
  f.s = l - 1;
  return f;
}

__host__ __device__ __forceinline__ int32_t fdiv(const FastDiv& f, int32_t n) {
#ifdef __CUDA_ARCH__
  return f.d == 1 ? n : (int32_t)(__umulhi((uint32_t)n, f.m) >> f.s);
#else
  return n / f.d;
#endif
}

// Plan fields the kernels need, with log2 of the power-of-two extents.
struct Geom {
  int32_t T, F, tpf, grid_cols, tile_h, tile_w, frame_count;
  int32_t lg_D, lg_bh, lg_bd, a_d, C, lg_C, group_size;
  int32_t lg_gs;  // group_size divides the power-of-two channel count: a power of two
  FastDiv div_tpf, div_F, div_cols;
};

inline Geom make_geom(const kvf_plan& p) {
  Geom g;
  g.T = p.T;
  g.F = p.F;
  g.tpf = p.tiles_per_frame;
  g.grid_cols = p.grid_cols;
  g.tile_h = p.a_h * p.a_d;
  g.tile_w = p.b_h * p.b_d;
  g.frame_count = p.frame_count;
  g.lg_D = ilog2(p.D);
  g.lg_bh = ilog2(p.b_h);
  g.lg_bd = ilog2(p.b_d);
  g.a_d = p.a_d;
  g.C = p.H * p.D;
  g.lg_C = ilog2(g.C);
  g.group_size = p.group_size;
  g.lg_gs = ilog2(p.group_size);
  g.div_tpf = make_fastdiv(p.tiles_per_frame);
  g.div_F = make_fastdiv(p.F);
  g.div_cols = make_fastdiv(p.grid_cols);
  return g;
}

// ------------------------------------------------------------- device helpers

// Channel c -> byte offset of its sample inside a tile whose rows are
// `row_pitch` bytes apart (fk/layout.py:244-250; inverse fk/layout.py:142-146).
__device__ __forceinline__ int64_t tile_offset(const Geom& g, int c,
                                               int64_t row_pitch) {
  int h = c >> g.lg_D;
  int d = c & ((1 << g.lg_D) - 1);
  int i_h = h >> g.lg_bh, j_h = h & ((1 << g.lg_bh) - 1);
  int i_d = d >> g.lg_bd, j_d = d & ((1 << g.lg_bd) - 1);
  int row = i_h * g.a_d + i_d;
  int col = (j_h << g.lg_bd) + j_d;
  return (int64_t)row * row_pitch + col;
}

// Element offset of channel c inside a token slot of a paged cache.
__device__ __forceinline__ int64_t slot_channel_offset(const Geom& g, int c,
                                                       int64_t head_stride) {
  int h = c >> g.lg_D;
  int d = c & ((1 << g.lg_D) - 1);
  return (int64_t)h * head_stride + d;
}

// Token placement (fk/layout.py:195-201) in the frame-major direction used by
// frame_slots (fk/layout.py:203-212): frame f, slot -> chunk token index.
__device__ __forceinline__ int token_of(const Geom& g, int f, int slot) {
  int seg = fdiv(g.div_F, f);
  int o = f - seg * g.F;
  return (seg * g.tpf + slot) * g.F + o;
}

// Element offset of chunk token i's slot in layer p of a paged cache.
__device__ __forceinline__ int64_t paged_slot_offset(const kvf_paged& pg, int i) {
  int64_t t = (int64_t)pg.token_base + i;
  int64_t blk_logical = t / pg.block_size;
  int64_t in_blk = t - blk_logical * pg.block_size;
  int64_t blk = pg.block_table ? (int64_t)__ldg(pg.block_table + blk_logical)
                               : blk_logical;
  return blk * pg.block_stride + in_blk * pg.slot_stride;
}

// Same with a fast divisor for the block size (t < 2^31).
__device__ __forceinline__ int64_t paged_slot_offset_fd(const kvf_paged& pg,
                                                        const FastDiv& bs, int i) {
  int32_t t = pg.token_base + i;
  int32_t blk_logical = fdiv(bs, t);
  int32_t in_blk = t - blk_logical * pg.block_size;
  int64_t blk = pg.block_table ? (int64_t)__ldg(pg.block_table + blk_logical)
                               : (int64_t)blk_logical;
  return blk * pg.block_stride + (int64_t)in_blk * pg.slot_stride;
}

// Quantization scale of one group from its |x| maximum (fk/kvmodel.py:139-140):
// fp32(fp64(max)/127.0), or 1.0 for an all-zero group.
__device__ __forceinline__ float scale_from_absmax_bits(uint32_t bits) {
  float m = __uint_as_float(bits);
  if (!(m > 0.0f)) return 1.0f;
  return __double2float_rn(__ddiv_rn((double)m, 127.0));
}

// rint(fp64(x) / fp64(s)) with round-half-to-even, clipped to [-127, 127]
// (fk/kvmodel.py:141-142).  The quotient via the fp32 reciprocal is within
// 2^-16 of x/s for |x/s| <= 128, so only samples whose fractional part lies
// within 2^-14 of one half can round differently; those take an exact fp64
// residual test (x - r*s is exact in fp64: r has 8 and s 24 significant bits).
// An fp64 quotient of two fp32 values can never land on a half-integer it is
// not exactly equal to, so this is bit-identical to the reference.
__device__ __forceinline__ int quantize_exact(float x, float s, float inv) {
  float y = x * inv;
  float r = rintf(y);
  float fr = fabsf(y - r);
  if (fr > 0.49993896484375f) {
    double sd = (double)s;
    double two_d = 2.0 * ((double)x - (double)r * sd);
    if (two_d > sd) {
      r += 1.0f;
    } else if (two_d == sd) {
      // tie between r and r+1: keep the even one
      if (fmodf(r, 2.0f) != 0.0f) r += 1.0f;
    } else if (two_d < -sd) {
      r -= 1.0f;
    } else if (two_d == -sd) {
      if (fmodf(r, 2.0f) != 0.0f) r -= 1.0f;
    }
  }
  r = fminf(fmaxf(r, -127.0f), 127.0f);
  return (int)r;
}

// 8 u8 samples -> exact floats of (sample - 128) without an I2F:
// float bits 0x4B0000bb = 2^23 + b, minus (2^23 + 128).
__device__ __forceinline__ void bytes8_to_float(uint32_t lo, uint32_t hi,
                                                float (&q)[8]) {
  // __byte_perm(x, y, s): result byte i is byte s[i] of {y:x}; bytes 4..7 are
  // y = 0x4B000000 -> 0x00,0x00,0x00,0x4B, so selector 0x744k gives 0x4B0000bk.
  const uint32_t magic = 0x4B000000u;
  uint32_t w[8];
  w[0] = __byte_perm(lo, magic, 0x7440);
  w[1] = __byte_perm(lo, magic, 0x7441);
  w[2] = __byte_perm(lo, magic, 0x7442);
  w[3] = __byte_perm(lo, magic, 0x7443);
  w[4] = __byte_perm(hi, magic, 0x7440);
  w[5] = __byte_perm(hi, magic, 0x7441);
  w[6] = __byte_perm(hi, magic, 0x7442);
  w[7] = __byte_perm(hi, magic, 0x7443);
#pragma unroll
  for (int k = 0; k < 8; ++k) q[k] = __uint_as_float(w[k]) - 8388736.0f;  // 2^23+128
}

// Streaming loads / stores.
__device__ __forceinline__ uint2 ld_nc_v2(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// Plain load that leaves the line in L2 with the normal eviction priority.
// (Measured on B200, tools/l2_probe2.cu: a re-read after an
// ld.global.nc.L1::no_allocate misses L2 as if the line had been evicted at
// once; after a plain ld.global, or a .nc load with an evict_last policy, a
// 48 MB re-read runs at ~9 TB/s.)
__device__ __forceinline__ uint4 ld_keep_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- mbarrier helpers ------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

// L2 eviction-priority policies (createpolicy) and loads/stores that carry them.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_nc_v4_pol(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_v2_pol(void* p, uint2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(v.x),
               "r"(v.y), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_v2(void* p, uint2 v) {
  asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack_f16x2(float a, float b) {
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Scalar element load/convert of any source dtype to float.
__device__ __forceinline__ float load_as_float(const void* base, int64_t idx,
                                               int32_t dtype) {
  switch (dtype) {
    case KVF_BF16:
      return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
    case KVF_F16:
      return __half2float(reinterpret_cast<const __half*>(base)[idx]);
    case KVF_F32:
      return reinterpret_cast<const float*>(base)[idx];
    default:
      return (float)reinterpret_cast<const int8_t*>(base)[idx];
  }
}

__device__ __forceinline__ void store_from_float(void* base, int64_t idx,
                                                 int32_t dtype, float v, int q) {
  switch (dtype) {
    case KVF_BF16:
      reinterpret_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(v);
      break;
    case KVF_F16:
      reinterpret_cast<__half*>(base)[idx] = __float2half_rn(v);
      break;
    case KVF_F32:
      reinterpret_cast<float*>(base)[idx] = v;
      break;
    default:
      reinterpret_cast<int8_t*>(base)[idx] = (int8_t)q;
      break;
  }
}

// |x| as an order-preserving u32 (non-negative float bits).
__device__ __forceinline__ uint32_t absbits(float x) {
  return __float_as_uint(x) & 0x7FFFFFFFu;
}

}  // namespace kvf
