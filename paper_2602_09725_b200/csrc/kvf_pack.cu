// kvf_pack.cu — (paged) KV -> quantised 3-plane frames, sm_100a.
//
// Replaces quantize (fk/kvmodel.py:127-144) + slice_tokens (fk/layout.py:109-114)
// + assemble_frames (fk/layout.py:234-258) for one (layer triplet, token chunk)
// unit, in three launches per batch:
//   1. absmax  — per (plane, group) max |x| over the chunk's tokens
//                (fk/kvmodel.py:138-139): warp-per-token, lanes keep running
//                maxima of the 16-bit |x| patterns (order-preserving for
//                non-negative bf16/fp16), xor-shuffle reduce inside the group,
//                shared atomicMax across warps, one global atomicMax per CTA.
//   2. scales  — fp32(fp64(max)/127) or 1.0 (fk/kvmodel.py:140).
//   3. frames  — warp per (frame, tile slot) of one plane (grid.z = plane):
//                16-byte source loads, exact half-even rounding + clip
//                (fk/kvmodel.py:141-142), +128, 8-byte stores at the tile
//                position; slots past T and pad layers get PAD_BYTE 128
//                (fk/layout.py:231, 251-253).
// An int8 source skips 1-2 and places the codes (assemble_frames).
#include <algorithm>
#include <vector>

#include "kvf_common.cuh"

namespace kvf {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kIPW = 2;          // frame items per warp
constexpr int kTokPerWarp = 8;   // absmax tokens per warp

struct PackUnitDev {
  kvf_paged src;
  Geom g;
  uint32_t* absmax;
  float* scales;
  kvf_surface fr;
  int32_t n_items;  // frame_count * tiles_per_frame (per plane)
  int32_t G;
};

struct PackParams {
  int32_t n_units;
  PackUnitDev u[KVF_MAX_UNITS];
};

// ------------------------------------------------------------------ phase 0/2
__global__ void zero_absmax_kernel(const __grid_constant__ PackParams P) {
  const PackUnitDev& U = P.u[blockIdx.y];
  for (int k = threadIdx.x; k < 3 * U.G; k += blockDim.x) U.absmax[k] = 0u;
}

__global__ void finalize_scales_kernel(const __grid_constant__ PackParams P) {
  const PackUnitDev& U = P.u[blockIdx.y];
  for (int k = threadIdx.x; k < 3 * U.G; k += blockDim.x)
    U.scales[k] = scale_from_absmax_bits(U.absmax[k]);
}

// -------------------------------------------------------------------- phase 1
template <int SRC>
__device__ __forceinline__ uint32_t vec_absmax_bits(const char* p) {
  if constexpr (SRC == KVF_F32) {
    uint4 a = ld_nc_v4(p), b = ld_nc_v4(p + 16);
    uint32_t m = max(max(a.x & 0x7FFFFFFFu, a.y & 0x7FFFFFFFu),
                     max(a.z & 0x7FFFFFFFu, a.w & 0x7FFFFFFFu));
    m = max(m, max(max(b.x & 0x7FFFFFFFu, b.y & 0x7FFFFFFFu),
                   max(b.z & 0x7FFFFFFFu, b.w & 0x7FFFFFFFu)));
    return m;
  } else {
    uint4 a = ld_nc_v4(p);
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

template <int SRC, int VPL>
__global__ void __launch_bounds__(kThreads)
    absmax_fast_kernel(const __grid_constant__ PackParams P) {
  extern __shared__ uint32_t s_max[];  // [G]
  const PackUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tok0 = (blockIdx.x * kWarps + warp) * kTokPerWarp;
  const char* layer = reinterpret_cast<const char*>(U.src.layer[p]);
  if (blockIdx.x * kWarps * kTokPerWarp >= U.g.T || layer == nullptr) return;
  for (int k = threadIdx.x; k < U.G; k += kThreads) s_max[k] = 0u;
  __syncthreads();

  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  int32_t off[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k)
    off[k] = (int32_t)slot_channel_offset(U.g, (lane + 32 * k) * 8, U.src.head_stride) * ES;
  uint32_t m[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) m[k] = 0u;

#pragma unroll 2
  for (int t = 0; t < kTokPerWarp; ++t) {
    int i = tok0 + t;
    if (i >= U.g.T) break;
    const char* slot = layer + paged_slot_offset(U.src, i) * ES;
#pragma unroll
    for (int k = 0; k < VPL; ++k) m[k] = max(m[k], vec_absmax_bits<SRC>(slot + off[k]));
  }

  // Lanes (lane + 32k) of one group are gs/8 consecutive lanes (gs <= 256) or
  // the whole warp over several k (gs > 256).
  const int lpg = U.g.group_size >> 3;  // lanes per group (vectors per group)
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    uint32_t v = absmax_to_f32_bits<SRC>(m[k]);
    for (int o = 1; o < 32 && o < lpg; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    int vec = lane + 32 * k;
    if ((lane & (min(lpg, 32) - 1)) == 0 && v) atomicMax(&s_max[vec / lpg], v);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < U.G; k += kThreads)
    if (s_max[k]) atomicMax(&U.absmax[p * U.G + k], s_max[k]);
}

__global__ void __launch_bounds__(kThreads)
    absmax_generic_kernel(const __grid_constant__ PackParams P) {
  extern __shared__ uint32_t s_max[];
  const PackUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const void* layer = U.src.layer[p];
  int64_t base = (int64_t)blockIdx.x * kThreads;
  if (base >= (int64_t)U.g.T * U.g.C || layer == nullptr) return;
  for (int k = threadIdx.x; k < U.G; k += kThreads) s_max[k] = 0u;
  __syncthreads();
  int64_t x = base + threadIdx.x;
  if (x < (int64_t)U.g.T * U.g.C) {
    int i = (int)(x >> U.g.lg_C);
    int c = (int)(x & (U.g.C - 1));
    int64_t o = paged_slot_offset(U.src, i) + slot_channel_offset(U.g, c, U.src.head_stride);
    uint32_t v = absbits(load_as_float(layer, o, U.src.dtype));
    if (v) atomicMax(&s_max[c / U.g.group_size], v);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < U.G; k += kThreads)
    if (s_max[k]) atomicMax(&U.absmax[p * U.G + k], s_max[k]);
}

// -------------------------------------------------------------------- phase 3
template <int SRC>
__device__ __forceinline__ void load_vec8(const char* p, float (&x)[8]) {
  if constexpr (SRC == KVF_F32) {
    uint4 a = ld_nc_v4(p), b = ld_nc_v4(p + 16);
    x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y);
    x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
    x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y);
    x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
  } else {
    uint4 a = ld_nc_v4(p);
    uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (SRC == KVF_BF16) {
        x[2 * k] = __uint_as_float(w[k] << 16);
        x[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
      } else {
        __half2 h = *reinterpret_cast<__half2*>(&w[k]);
        float2 f = __half22float2(h);
        x[2 * k] = f.x;
        x[2 * k + 1] = f.y;
      }
    }
  }
}

__device__ __forceinline__ uint32_t pack_codes4(int a, int b, int c, int d) {
  return (uint32_t)((a + 128) & 0xFF) | ((uint32_t)((b + 128) & 0xFF) << 8) |
         ((uint32_t)((c + 128) & 0xFF) << 16) | ((uint32_t)((d + 128) & 0xFF) << 24);
}

template <int SRC, int VPL>
__global__ void __launch_bounds__(kThreads)
    pack_fast_kernel(const __grid_constant__ PackParams P) {
  const PackUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item0 = ((int64_t)blockIdx.x * kWarps + warp) * kIPW;
  if (item0 >= U.n_items) return;
  constexpr int ES = SRC == KVF_F32 ? 4 : (SRC == KVF_I8 ? 1 : 2);
  const char* layer = reinterpret_cast<const char*>(U.src.layer[p]);

  int32_t in_off[VPL], tile_off[VPL];
  float s[VPL], inv[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    int c = (lane + 32 * k) * 8;
    in_off[k] = (int32_t)slot_channel_offset(U.g, c, U.src.head_stride) * ES;
    tile_off[k] = (int32_t)tile_offset(U.g, c, U.fr.row_pitch);
    if constexpr (SRC != KVF_I8) {
      s[k] = U.scales[p * U.G + c / U.g.group_size];
      inv[k] = __frcp_rn(s[k]);
    }
  }

#pragma unroll
  for (int it = 0; it < kIPW; ++it) {
    int j = (int)(item0 + it);
    if (j >= U.n_items) break;
    int f = j / U.g.tpf;
    int slot = j - f * U.g.tpf;
    int i = token_of(U.g, f, slot);
    int tr = slot / U.g.grid_cols;
    int tc = slot - tr * U.g.grid_cols;
    uint8_t* dst = U.fr.base + (int64_t)f * U.fr.frame_stride +
                   (int64_t)p * U.fr.plane_stride +
                   (int64_t)tr * U.g.tile_h * U.fr.row_pitch + (int64_t)tc * U.g.tile_w;
    if (i >= U.g.T || layer == nullptr) {
#pragma unroll
      for (int k = 0; k < VPL; ++k) st_v2(dst + tile_off[k], make_uint2(0x80808080u, 0x80808080u));
      continue;
    }
    const char* slotp = layer + paged_slot_offset(U.src, i) * ES;
    if constexpr (SRC == KVF_I8) {
      uint2 v[VPL];
#pragma unroll
      for (int k = 0; k < VPL; ++k) v[k] = ld_nc_v2(slotp + in_off[k]);
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        st_v2(dst + tile_off[k], make_uint2(v[k].x ^ 0x80808080u, v[k].y ^ 0x80808080u));
    } else {
      // At most 4 vectors (32 values) live at once to bound register use.
      constexpr int KB = VPL < 4 ? VPL : 4;
#pragma unroll
      for (int k0 = 0; k0 < VPL; k0 += KB) {
        float x[KB][8];
#pragma unroll
        for (int k = 0; k < KB; ++k) load_vec8<SRC>(slotp + in_off[k0 + k], x[k]);
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          int q[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) q[e] = quantize_exact(x[k][e], s[k0 + k], inv[k0 + k]);
          st_v2(dst + tile_off[k0 + k], make_uint2(pack_codes4(q[0], q[1], q[2], q[3]),
                                                   pack_codes4(q[4], q[5], q[6], q[7])));
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads)
    pack_generic_kernel(const __grid_constant__ PackParams P) {
  const PackUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  int64_t x = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  int64_t j = x >> U.g.lg_C;
  if (j >= U.n_items) return;
  int c = (int)(x & (U.g.C - 1));
  int f = (int)(j / U.g.tpf);
  int slot = (int)(j - (int64_t)f * U.g.tpf);
  int i = token_of(U.g, f, slot);
  int tr = slot / U.g.grid_cols;
  int tc = slot - tr * U.g.grid_cols;
  uint8_t* dst = U.fr.base + (int64_t)f * U.fr.frame_stride +
                 (int64_t)p * U.fr.plane_stride +
                 (int64_t)tr * U.g.tile_h * U.fr.row_pitch + (int64_t)tc * U.g.tile_w +
                 tile_offset(U.g, c, U.fr.row_pitch);
  const void* layer = U.src.layer[p];
  if (i >= U.g.T || layer == nullptr) {
    *dst = 128;
    return;
  }
  int64_t o = paged_slot_offset(U.src, i) + slot_channel_offset(U.g, c, U.src.head_stride);
  int q;
  if (U.src.dtype == KVF_I8) {
    q = reinterpret_cast<const int8_t*>(layer)[o];
  } else {
    float s = U.scales[p * U.G + c / U.g.group_size];
    q = quantize_exact(load_as_float(layer, o, U.src.dtype), s, __frcp_rn(s));
  }
  *dst = (uint8_t)(q + 128);
}

bool aligned(const void* p, int64_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

int pack_variant(const kvf_pack_unit& u) {
  const kvf_plan& p = u.plan;
  int64_t C = (int64_t)p.H * p.D;
  if (C % 256 != 0) return 0;
  int vpl = (int)(C / 256);
  if (vpl != 1 && vpl != 2 && vpl != 4 && vpl != 8 && vpl != 16) return 0;
  if (p.b_d % 8 != 0) return 0;
  if (u.src.dtype != KVF_I8 && p.group_size % 8 != 0) return 0;
  if (!aligned(u.frames.base, 8) || u.frames.frame_stride % 8 ||
      u.frames.plane_stride % 8 || u.frames.row_pitch % 8)
    return 0;
  int64_t es = (int64_t)dtype_size(u.src.dtype);
  int64_t va = u.src.dtype == KVF_I8 ? 8 : 16;
  for (int l = 0; l < 3; ++l)
    if (u.src.layer[l] && !aligned(u.src.layer[l], va)) return 0;
  if ((u.src.head_stride * es) % va || (u.src.slot_stride * es) % va ||
      (u.src.block_stride * es) % va)
    return 0;
  return vpl;
}

kvf_status check_unit(const kvf_pack_unit& u) {
  kvf_status st = check_plan(u.plan);
  if (st != KVF_OK) return st;
  if (u.frames.base == nullptr) KVF_FAIL(KVF_EINVAL, "null frame surface");
  if (u.frames.row_pitch < u.plan.frame_w)
    KVF_FAIL(KVF_EINVAL, "row pitch below frame width");
  if (u.src.dtype < KVF_BF16 || u.src.dtype > KVF_I8)
    KVF_FAIL(KVF_EINVAL, "bad source dtype %d", u.src.dtype);
  if (u.src.dtype != KVF_I8 && (u.absmax == nullptr || u.scales == nullptr))
    KVF_FAIL(KVF_EINVAL, "quantising pack needs absmax scratch and scales");
  if (u.src.block_size < 1) KVF_FAIL(KVF_EINVAL, "block_size must be >= 1");
  if (u.src.token_base < 0) KVF_FAIL(KVF_EINVAL, "negative token_base");
  return KVF_OK;
}

PackUnitDev to_dev(const kvf_pack_unit& u) {
  PackUnitDev d;
  d.src = u.src;
  d.g = make_geom(u.plan);
  d.absmax = u.absmax;
  d.scales = u.scales;
  d.fr = u.frames;
  d.n_items = u.plan.frame_count * u.plan.tiles_per_frame;
  d.G = (u.plan.H * u.plan.D) / u.plan.group_size;
  return d;
}

template <int SRC>
void launch_absmax_fast(int vpl, const PackParams& P, dim3 grid, size_t smem,
                        cudaStream_t s) {
  switch (vpl) {
    case 1: absmax_fast_kernel<SRC, 1><<<grid, kThreads, smem, s>>>(P); break;
    case 2: absmax_fast_kernel<SRC, 2><<<grid, kThreads, smem, s>>>(P); break;
    case 4: absmax_fast_kernel<SRC, 4><<<grid, kThreads, smem, s>>>(P); break;
    case 8: absmax_fast_kernel<SRC, 8><<<grid, kThreads, smem, s>>>(P); break;
    case 16: absmax_fast_kernel<SRC, 16><<<grid, kThreads, smem, s>>>(P); break;
  }
}

template <int SRC>
void launch_pack_fast(int vpl, const PackParams& P, dim3 grid, cudaStream_t s) {
  switch (vpl) {
    case 1: pack_fast_kernel<SRC, 1><<<grid, kThreads, 0, s>>>(P); break;
    case 2: pack_fast_kernel<SRC, 2><<<grid, kThreads, 0, s>>>(P); break;
    case 4: pack_fast_kernel<SRC, 4><<<grid, kThreads, 0, s>>>(P); break;
    case 8: pack_fast_kernel<SRC, 8><<<grid, kThreads, 0, s>>>(P); break;
    case 16: pack_fast_kernel<SRC, 16><<<grid, kThreads, 0, s>>>(P); break;
  }
}

// phases: bit 0 = zero absmax, bit 1 = absmax, bit 2 = scales, bit 3 = frames.
kvf_status launch_group(const std::vector<kvf_pack_unit>& units, int vpl,
                        int32_t dtype, int phases, cudaStream_t s) {
  for (size_t at = 0; at < units.size(); at += KVF_MAX_UNITS) {
    size_t n = std::min<size_t>(KVF_MAX_UNITS, units.size() - at);
    PackParams P;
    P.n_units = (int32_t)n;
    int64_t max_items = 0, max_T = 0, max_G = 1, max_C = 1;
    for (size_t k = 0; k < n; ++k) {
      P.u[k] = to_dev(units[at + k]);
      max_items = std::max<int64_t>(max_items, P.u[k].n_items);
      max_T = std::max<int64_t>(max_T, P.u[k].g.T);
      max_G = std::max<int64_t>(max_G, P.u[k].G);
      max_C = std::max<int64_t>(max_C, P.u[k].g.C);
    }
    const bool quant = dtype != KVF_I8;
    size_t smem = (size_t)max_G * sizeof(uint32_t);
    if (smem > 48 * 1024) KVF_FAIL(KVF_EUNSUPPORTED, "too many quantisation groups");
    if (quant && (phases & 1)) {
      zero_absmax_kernel<<<dim3(1, (unsigned)n), 256, 0, s>>>(P);
      KVF_CHECK_CUDA(cudaGetLastError());
    }
    if (quant && (phases & 2) && max_T > 0) {
      if (vpl) {
        int64_t per = (int64_t)kWarps * kTokPerWarp;
        dim3 grid((unsigned)((max_T + per - 1) / per), (unsigned)n, 3);
        switch (dtype) {
          case KVF_BF16: launch_absmax_fast<KVF_BF16>(vpl, P, grid, smem, s); break;
          case KVF_F16: launch_absmax_fast<KVF_F16>(vpl, P, grid, smem, s); break;
          case KVF_F32: launch_absmax_fast<KVF_F32>(vpl, P, grid, smem, s); break;
        }
      } else {
        int64_t work = max_T * max_C;
        dim3 grid((unsigned)((work + kThreads - 1) / kThreads), (unsigned)n, 3);
        absmax_generic_kernel<<<grid, kThreads, smem, s>>>(P);
      }
      KVF_CHECK_CUDA(cudaGetLastError());
    }
    if (quant && (phases & 4)) {
      finalize_scales_kernel<<<dim3(1, (unsigned)n), 256, 0, s>>>(P);
      KVF_CHECK_CUDA(cudaGetLastError());
    }
    if ((phases & 8) && max_items > 0) {
      if (vpl) {
        int64_t per = (int64_t)kWarps * kIPW;
        dim3 grid((unsigned)((max_items + per - 1) / per), (unsigned)n, 3);
        switch (dtype) {
          case KVF_BF16: launch_pack_fast<KVF_BF16>(vpl, P, grid, s); break;
          case KVF_F16: launch_pack_fast<KVF_F16>(vpl, P, grid, s); break;
          case KVF_F32: launch_pack_fast<KVF_F32>(vpl, P, grid, s); break;
          case KVF_I8: launch_pack_fast<KVF_I8>(vpl, P, grid, s); break;
        }
      } else {
        int64_t work = max_items * max_C;
        if ((work + kThreads - 1) / kThreads > 0x7FFFFFFF)
          KVF_FAIL(KVF_EUNSUPPORTED, "pack grid too large");
        dim3 grid((unsigned)((work + kThreads - 1) / kThreads), (unsigned)n, 3);
        pack_generic_kernel<<<grid, kThreads, 0, s>>>(P);
      }
      KVF_CHECK_CUDA(cudaGetLastError());
    }
  }
  return KVF_OK;
}

kvf_status run(const kvf_pack_unit* units, int32_t n_units, int phases,
               cudaStream_t s) {
  if (n_units < 0 || (n_units > 0 && units == nullptr))
    KVF_FAIL(KVF_EINVAL, "bad unit array");
  std::vector<kvf_pack_unit> groups[17][4];
  for (int32_t k = 0; k < n_units; ++k) {
    kvf_status st = check_unit(units[k]);
    if (st != KVF_OK) return st;
    groups[pack_variant(units[k])][units[k].src.dtype].push_back(units[k]);
  }
  for (int v = 0; v <= 16; ++v)
    for (int dt = 0; dt < 4; ++dt)
      if (!groups[v][dt].empty()) {
        kvf_status st = launch_group(groups[v][dt], v, dt, phases, s);
        if (st != KVF_OK) return st;
      }
  return KVF_OK;
}

kvf_pack_unit single(const kvf_paged* src, const kvf_plan* plan,
                     const uint32_t* absmax, float* scales,
                     const kvf_surface* frames) {
  kvf_pack_unit u;
  u.src = *src;
  u.plan = *plan;
  u.absmax = const_cast<uint32_t*>(absmax);
  u.scales = scales;
  if (frames) {
    u.frames = *frames;
  } else {
    // absmax-only call: any non-null surface passes validation, never touched.
    u.frames.base = reinterpret_cast<uint8_t*>(1);
    u.frames.row_pitch = plan->frame_w;
    u.frames.plane_stride = (int64_t)plan->frame_w * plan->frame_h;
    u.frames.frame_stride = 3 * u.frames.plane_stride;
  }
  return u;
}

}  // namespace
}  // namespace kvf

using namespace kvf;

extern "C" kvf_status kvf_pack_batch(const kvf_pack_unit* units, int32_t n_units,
                                     void* stream) {
  return run(units, n_units, 1 | 2 | 4 | 8, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" kvf_status kvf_pack_absmax(const kvf_paged* src, const kvf_plan* plan,
                                      uint32_t* absmax, void* stream) {
  if (!src || !plan || !absmax) KVF_FAIL(KVF_EINVAL, "null argument");
  if (src->dtype == KVF_I8) KVF_FAIL(KVF_EINVAL, "int8 codes have no absmax phase");
  float dummy_scales_never_written;
  kvf_pack_unit u = single(src, plan, absmax, &dummy_scales_never_written, nullptr);
  return run(&u, 1, 2, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" kvf_status kvf_pack_frames(const kvf_paged* src, const kvf_plan* plan,
                                      const uint32_t* absmax, float* scales,
                                      const kvf_surface* frames, void* stream) {
  if (!src || !plan || !frames) KVF_FAIL(KVF_EINVAL, "null argument");
  kvf_pack_unit u = single(src, plan, absmax, scales, frames);
  return run(&u, 1, 4 | 8, reinterpret_cast<cudaStream_t>(stream));
}
