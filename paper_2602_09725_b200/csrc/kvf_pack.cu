// kvf_pack.cu — (paged) KV -> quantised 3-plane frames, sm_100a: entry points
// and the phase-split kernels.
//
// Replaces quantize (fk/kvmodel.py:127-144) + slice_tokens (fk/layout.py:109-114)
// + assemble_frames (fk/layout.py:234-258) for (layer triplet, token chunk) units.
//
// kvf_pack_batch runs, per group of units sharing (variant, dtype):
//   zero scratch -> absmax (max |x| per (plane, group) over all chunk tokens) ->
//   scales -> frames (exact quantise + tile + place, pad tiles 128).
// The reference scale spans all chunk tokens, so these kernels read the source
// twice; the single-HBM-read schedule is kvf_pack_stream.cu.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {

kvf_status launch_pack_stream(const std::vector<kvf_pack_unit>& units, int32_t dtype,
                              int cluster, int probe, cudaStream_t s,
                              std::vector<kvf_pack_unit>* rest);
bool pack_band_ok(const kvf_pack_unit& u);
kvf_status launch_pack_band(const std::vector<kvf_pack_unit>& units, int32_t dtype,
                            cudaStream_t s);
// pack group variants: 0 generic, 1..16 fast kernels (VPL), kBandBase + v =
// shared-memory band frames kernel with the absmax of variant v
constexpr int kBandBase = 20;

namespace {

constexpr int kThreads = kPackThreads;
constexpr int kWarps = kPackWarps;
struct PackParams {
  int32_t n_units;
  PackUnitDev u[kMaxPackUnits];
};

// ------------------------------------------------------------------ phase 0/2
__global__ void zero_absmax_kernel(const __grid_constant__ PackParams P) {
  const PackUnitDev& U = P.u[blockIdx.y];
  for (int k = threadIdx.x; k < U.n_scratch; k += blockDim.x) U.absmax[k] = 0u;
}

__global__ void finalize_scales_kernel(const __grid_constant__ PackParams P) {
  const PackUnitDev& U = P.u[blockIdx.y];
  for (int k = threadIdx.x; k < 3 * U.G; k += blockDim.x)
    U.scales[k] = scale_from_absmax_bits(U.absmax[k]);
}

// -------------------------------------------------------------------- phase 1
template <int SRC, int VPL>
__global__ void __launch_bounds__(kThreads)
    absmax_fast_kernel(const __grid_constant__ PackParams P) {
  extern __shared__ uint32_t s_max[];  // [G]
  const PackUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kTokPerWarp = tok_per_warp(VPL);
  const int tok0 = (blockIdx.x * kWarps + warp) * kTokPerWarp;
  const char* layer = reinterpret_cast<const char*>(U.src.layer[p]);
  if (blockIdx.x * kWarps * kTokPerWarp >= U.g.T || layer == nullptr) return;
  for (int k = threadIdx.x; k < U.G; k += kThreads) s_max[k] = 0u;
  __syncthreads();
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  int32_t off[VPL];
  uint32_t m[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    off[k] = (int32_t)slot_channel_offset(U.g, (lane + 32 * k) * 8, U.src.head_stride) * ES;
    m[k] = 0u;
  }
#pragma unroll(VPL >= 4 ? 2 : 8 / VPL)  // ~8 vectors per lane in flight
  for (int t = 0; t < kTokPerWarp; ++t) {
    int i = tok0 + t;
    if (i >= U.g.T) break;
    const char* slot = layer + paged_slot_offset_fd(U.src, U.div_bs, i) * ES;
#pragma unroll
    for (int k = 0; k < VPL; ++k) m[k] = max(m[k], vec_absmax_bits<SRC>(slot + off[k]));
  }
  reduce_groups<SRC, VPL>(m, U.g.group_size, s_max);
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
// kRange: scales may come from a caller's absmax (kvf_pack_frames), so |x/s|
// is not bounded by 127 and the clip must be checked.
// 4 CTAs per SM (64 registers): more loads in flight beat the few spilled
// registers (1.86 -> 1.80 ms on C2).
template <int SRC, int VPL, bool kRange>
__global__ void __launch_bounds__(kThreads, 4)
    pack_fast_kernel(const __grid_constant__ PackParams P) {
  const PackUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const int warp = threadIdx.x >> 5;
  constexpr int SUB = pack_sub<SRC, VPL>();
  const int item0 = (blockIdx.x * kWarps + warp) * kIPW * SUB;
  if (item0 >= U.n_items) return;
  PackLane<SRC, VPL> L;
  L.init(U, p, U.scales + p * U.G);
  const int rounds = min(kIPW, (U.n_items - item0 + SUB - 1) / SUB);
  pack_items<SRC, VPL, kRange>(U, p, L, item0, SUB, rounds, U.n_items);
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
  uint8_t* dst = U.fr.base + (int64_t)f * U.fr.frame_stride + (int64_t)p * U.fr.plane_stride +
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

// ------------------------------------------------------------------- host
bool aligned(const void* p, int64_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// VPL of the vectorised source kernels (absmax, frames) or 0: source-side
// conditions only (the absmax ignores the tiling).
int source_vpl(const kvf_pack_unit& u) {
  const kvf_plan& p = u.plan;
  int64_t C = (int64_t)p.H * p.D;
  if (C % 256 != 0) return 0;
  int vpl = (int)(C / 256);
  if (vpl != 1 && vpl != 2 && vpl != 4 && vpl != 8 && vpl != 16) return 0;
  if (u.src.dtype != KVF_I8 && p.group_size % 8 != 0) return 0;
  int64_t es = (int64_t)dtype_size(u.src.dtype);
  int64_t va = u.src.dtype == KVF_I8 ? 8 : 16;
  for (int l = 0; l < 3; ++l)
    if (u.src.layer[l] && !aligned(u.src.layer[l], va)) return 0;
  if ((u.src.head_stride * es) % va || (u.src.slot_stride * es) % va ||
      (u.src.block_stride * es) % va)
    return 0;
  return vpl;
}

int pack_variant(const kvf_pack_unit& u) {
  const kvf_plan& p = u.plan;
  if (p.b_d % 8 != 0) return 0;
  if (!aligned(u.frames.base, 8) || u.frames.frame_stride % 8 || u.frames.plane_stride % 8 ||
      u.frames.row_pitch % 8)
    return 0;
  return source_vpl(u);
}

kvf_status check_unit(const kvf_pack_unit& u) {
  kvf_status st = check_plan(u.plan);
  if (st != KVF_OK) return st;
  if (u.frames.base == nullptr) KVF_FAIL(KVF_EINVAL, "null frame surface");
  if (u.frames.row_pitch < u.plan.frame_w) KVF_FAIL(KVF_EINVAL, "row pitch below frame width");
  if (u.src.dtype < KVF_BF16 || u.src.dtype > KVF_I8)
    KVF_FAIL(KVF_EINVAL, "bad source dtype %d", u.src.dtype);
  if (u.src.dtype != KVF_I8 && (u.absmax == nullptr || u.scales == nullptr))
    KVF_FAIL(KVF_EINVAL, "quantising pack needs absmax scratch and scales");
  if (u.src.block_size < 1) KVF_FAIL(KVF_EINVAL, "block_size must be >= 1");
  if (u.src.token_base < 0) KVF_FAIL(KVF_EINVAL, "negative token_base");
  if ((int64_t)u.src.token_base + u.plan.T >= (int64_t(1) << 31))
    KVF_FAIL(KVF_EUNSUPPORTED, "token index beyond 2^31");
  return KVF_OK;
}

template <int SRC>
void launch_absmax_fast(int vpl, const PackParams& P, dim3 grid, size_t smem, cudaStream_t s) {
  switch (vpl) {
    case 1: absmax_fast_kernel<SRC, 1><<<grid, kThreads, smem, s>>>(P); break;
    case 2: absmax_fast_kernel<SRC, 2><<<grid, kThreads, smem, s>>>(P); break;
    case 4: absmax_fast_kernel<SRC, 4><<<grid, kThreads, smem, s>>>(P); break;
    case 8: absmax_fast_kernel<SRC, 8><<<grid, kThreads, smem, s>>>(P); break;
    case 16: absmax_fast_kernel<SRC, 16><<<grid, kThreads, smem, s>>>(P); break;
  }
}

template <int SRC, bool kRange>
void launch_pack_fast_r(int vpl, const PackParams& P, dim3 grid, cudaStream_t s) {
  switch (vpl) {
    case 1: pack_fast_kernel<SRC, 1, kRange><<<grid, kThreads, 0, s>>>(P); break;
    case 2: pack_fast_kernel<SRC, 2, kRange><<<grid, kThreads, 0, s>>>(P); break;
    case 4: pack_fast_kernel<SRC, 4, kRange><<<grid, kThreads, 0, s>>>(P); break;
    case 8: pack_fast_kernel<SRC, 8, kRange><<<grid, kThreads, 0, s>>>(P); break;
    case 16: pack_fast_kernel<SRC, 16, kRange><<<grid, kThreads, 0, s>>>(P); break;
  }
}

// trusted: the scales were derived in this call from the same source's maxima.
template <int SRC>
void launch_pack_fast(int vpl, const PackParams& P, dim3 grid, cudaStream_t s, bool trusted) {
  if (trusted || SRC == KVF_I8)
    launch_pack_fast_r<SRC, false>(vpl, P, grid, s);
  else
    launch_pack_fast_r<SRC, true>(vpl, P, grid, s);
}

PackParams* make_params(const std::vector<kvf_pack_unit>& units, size_t at, size_t n) {
  PackParams* P = new PackParams();
  P->n_units = (int32_t)n;
  for (size_t k = 0; k < n; ++k) P->u[k] = make_pack_unit_dev(units[at + k]);
  return P;
}

// phases: bit 0 = zero scratch, bit 1 = absmax, bit 2 = scales, bit 3 = frames.
kvf_status launch_phases(const std::vector<kvf_pack_unit>& units, int variant, int32_t dtype,
                         int phases, cudaStream_t s) {
  const bool band = variant >= kBandBase;
  const int vpl = band ? variant - kBandBase : variant;
  if (band && (phases & 8)) {
    if (phases & 7) {
      kvf_status st = launch_phases(units, vpl, dtype, phases & 7, s);
      if (st != KVF_OK) return st;
    }
    return launch_pack_band(units, dtype, s);
  }
  for (size_t at = 0; at < units.size(); at += kMaxPackUnits) {
    size_t n = std::min<size_t>(kMaxPackUnits, units.size() - at);
    PackParams* P = make_params(units, at, n);
    int64_t max_items = 0, max_T = 0, max_G = 1, max_C = 1;
    for (size_t k = 0; k < n; ++k) {
      max_items = std::max<int64_t>(max_items, P->u[k].n_items);
      max_T = std::max<int64_t>(max_T, P->u[k].g.T);
      max_G = std::max<int64_t>(max_G, P->u[k].G);
      max_C = std::max<int64_t>(max_C, P->u[k].g.C);
    }
    const bool quant = dtype != KVF_I8;
    size_t smem = (size_t)max_G * sizeof(uint32_t);
    cudaError_t e = cudaSuccess;
    if (smem > 48 * 1024) {
      delete P;
      KVF_FAIL(KVF_EUNSUPPORTED, "too many quantisation groups");
    }
    if (quant && (phases & 1)) zero_absmax_kernel<<<dim3(1, (unsigned)n), 256, 0, s>>>(*P);
    if (quant && (phases & 2) && max_T > 0) {
      if (vpl) {
        int64_t per = (int64_t)kWarps * tok_per_warp(vpl);
        dim3 grid((unsigned)((max_T + per - 1) / per), (unsigned)n, 3);
        switch (dtype) {
          case KVF_BF16: launch_absmax_fast<KVF_BF16>(vpl, *P, grid, smem, s); break;
          case KVF_F16: launch_absmax_fast<KVF_F16>(vpl, *P, grid, smem, s); break;
          case KVF_F32: launch_absmax_fast<KVF_F32>(vpl, *P, grid, smem, s); break;
        }
      } else {
        int64_t work = max_T * max_C;
        dim3 grid((unsigned)((work + kThreads - 1) / kThreads), (unsigned)n, 3);
        absmax_generic_kernel<<<grid, kThreads, smem, s>>>(*P);
      }
    }
    if (quant && (phases & 4)) finalize_scales_kernel<<<dim3(1, (unsigned)n), 256, 0, s>>>(*P);
    if ((phases & 8) && max_items > 0) {
      if (vpl) {
        const int sub = (dtype != KVF_I8 && vpl < 4) ? 4 / vpl : 1;  // pack_sub<SRC, VPL>
        int64_t per = (int64_t)kWarps * kIPW * sub;
        dim3 grid((unsigned)((max_items + per - 1) / per), (unsigned)n, 3);
        const bool trusted = (phases & 2) != 0;
        switch (dtype) {
          case KVF_BF16: launch_pack_fast<KVF_BF16>(vpl, *P, grid, s, trusted); break;
          case KVF_F16: launch_pack_fast<KVF_F16>(vpl, *P, grid, s, trusted); break;
          case KVF_F32: launch_pack_fast<KVF_F32>(vpl, *P, grid, s, trusted); break;
          case KVF_I8: launch_pack_fast<KVF_I8>(vpl, *P, grid, s, trusted); break;
        }
      } else {
        int64_t work = max_items * max_C;
        if ((work + kThreads - 1) / kThreads > 0x7FFFFFFF) {
          delete P;
          KVF_FAIL(KVF_EUNSUPPORTED, "pack grid too large");
        }
        dim3 grid((unsigned)((work + kThreads - 1) / kThreads), (unsigned)n, 3);
        pack_generic_kernel<<<grid, kThreads, 0, s>>>(*P);
      }
    }
    e = cudaGetLastError();
    delete P;
    if (e != cudaSuccess) return cuda_status(e, "pack phase kernels");
  }
  return KVF_OK;
}

kvf_status run(const kvf_pack_unit* units, int32_t n_units, int phases, int32_t schedule,
               int64_t param, cudaStream_t s) {
  if (n_units < 0 || (n_units > 0 && units == nullptr)) KVF_FAIL(KVF_EINVAL, "bad unit array");
  if (schedule < KVF_PACK_AUTO || schedule > KVF_PACK_SINGLE_READ)
    KVF_FAIL(KVF_EINVAL, "bad pack schedule %d", schedule);
  if (param < 0) KVF_FAIL(KVF_EINVAL, "negative schedule parameter");
  const bool single = schedule == KVF_PACK_SINGLE_READ && phases == (1 | 2 | 4 | 8);
  std::vector<kvf_pack_unit> by_dtype[4];
  for (int32_t k = 0; k < n_units; ++k) {
    kvf_status st = check_unit(units[k]);
    if (st != KVF_OK) return st;
    by_dtype[units[k].src.dtype].push_back(units[k]);
  }
  std::vector<kvf_pack_unit> groups[kBandBase + 17][4];
  for (int dt = 0; dt < 4; ++dt) {
    std::vector<kvf_pack_unit> rest;
    if (single && dt != KVF_I8) {
      kvf_status st = launch_pack_stream(by_dtype[dt], dt, (int)(param & 0xFF),
                                         (int)((param >> 8) & 0xFF), s, &rest);
      if (st != KVF_OK) return st;
    } else {
      rest.swap(by_dtype[dt]);
    }
    for (const auto& u : rest) {
      int v = pack_variant(u);
      if (v == 0 && pack_band_ok(u)) v = kBandBase + source_vpl(u);  // narrow tile rows
      groups[v][dt].push_back(u);
    }
  }
  for (int v = 0; v < kBandBase + 17; ++v)
    for (int dt = 0; dt < 4; ++dt)
      if (!groups[v][dt].empty()) {
        kvf_status st = launch_phases(groups[v][dt], v, dt, phases, s);
        if (st != KVF_OK) return st;
      }
  return KVF_OK;
}

kvf_pack_unit single(const kvf_paged* src, const kvf_plan* plan, const uint32_t* absmax,
                     float* scales, const kvf_surface* frames) {
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

extern "C" kvf_status kvf_pack_batch(const kvf_pack_unit* units, int32_t n_units, void* stream) {
  return run(units, n_units, 1 | 2 | 4 | 8, KVF_PACK_AUTO, 0,
             reinterpret_cast<cudaStream_t>(stream));
}

extern "C" kvf_status kvf_pack_batch_ex(const kvf_pack_unit* units, int32_t n_units,
                                        int32_t schedule, int64_t param, void* stream) {
  return run(units, n_units, 1 | 2 | 4 | 8, schedule, param,
             reinterpret_cast<cudaStream_t>(stream));
}

extern "C" kvf_status kvf_pack_frames_batch(const kvf_pack_unit* units, int32_t n_units,
                                            void* stream) {
  return run(units, n_units, 4 | 8, KVF_PACK_AUTO, 0, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" kvf_status kvf_pack_absmax(const kvf_paged* src, const kvf_plan* plan,
                                      uint32_t* absmax, void* stream) {
  if (!src || !plan || !absmax) KVF_FAIL(KVF_EINVAL, "null argument");
  if (src->dtype == KVF_I8) KVF_FAIL(KVF_EINVAL, "int8 codes have no absmax phase");
  float unused_scales;
  kvf_pack_unit u = single(src, plan, absmax, &unused_scales, nullptr);
  return run(&u, 1, 2, KVF_PACK_AUTO, 0, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" kvf_status kvf_pack_frames(const kvf_paged* src, const kvf_plan* plan,
                                      const uint32_t* absmax, float* scales,
                                      const kvf_surface* frames, void* stream) {
  if (!src || !plan || !frames) KVF_FAIL(KVF_EINVAL, "null argument");
  kvf_pack_unit u = single(src, plan, absmax, scales, frames);
  return run(&u, 1, 4 | 8, KVF_PACK_AUTO, 0, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int64_t kvf_pack_scratch_words(const kvf_plan* plan) {
  if (!plan || check_plan(*plan) != KVF_OK) return -1;
  return pack_scratch_words(*plan);
}
