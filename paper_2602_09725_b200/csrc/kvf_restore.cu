// kvf_restore.cu — frames -> (dequantised) paged KV cache, sm_100a.
//
// Replaces, for a batch of decoded frames, the reference's frame-wise restore
// callback fk/fetchsim.py:347-355 (frame_slots -> tile -> int16-128 -> int8 ->
// inverse_layout -> PagedMemory.page_write, fk/layout.py:137-147,203-212 and
// fk/kvmodel.py:216-229) fused with dequantize (fk/kvmodel.py:147-152).
//
// Work decomposition: one warp per (frame, tile slot, plane) "item" = one token
// slot of one layer.  Each lane owns VPL 8-channel vectors of the slot; its tile
// offsets are computed once per CTA (the layout is per unit), so the per-item
// cost is the item decode (frame/slot/token/page) amortised over the warp.  A
// vector is one 8-byte read of 8 u8 samples (contiguous because b_d % 8 == 0)
// and one 16-byte bf16 store into the 2*C-byte contiguous slot.  Each warp keeps
// IPW*VPL loads in flight before it converts and stores.
//
// Bound: HBM.  Algorithmic bytes per channel element: 1 (u8 read) + sizeof(out).
#include <algorithm>
#include <type_traits>
#include <vector>

#include "kvf_common.cuh"

namespace kvf {

bool restore_band_ok(const kvf_restore_unit& u);
kvf_status launch_restore_band(const std::vector<kvf_restore_unit>& units, int32_t dtype,
                               cudaStream_t s);

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kIPW = 4;  // item rounds per warp (loads in flight per lane: kIPW * 4 or VPL)
// Narrow slots (C = 256 / 512 channels: VPL 1 / 2 vectors per lane) put
// SUB = 4 / VPL items side by side in a warp, 32 / SUB lanes each, so every
// lane still moves 4 vectors per item round and the per-item index math is
// amortised over as many bytes as for C = 1024.
// VPL 0 stands for C = 128 channels (half a vector per lane of a 32-lane
// item): 8 items side by side, 4 lanes of 4 vectors each.
__host__ __device__ constexpr int sub_for(int vpl) {
  return vpl == 0 ? 8 : (vpl >= 4 ? 1 : 4 / vpl);
}
__host__ __device__ constexpr int vl_for(int vpl) { return vpl == 0 ? 4 : vpl * sub_for(vpl); }
constexpr int kVariantC128 = 3;  // restore_variant code of C = 128 (VPL 0)
__host__ __device__ constexpr int ipw_for(int vpl) { return kIPW * sub_for(vpl); }

struct RestoreUnitDev {
  kvf_surface fr;
  Geom g;
  const float* scales;
  kvf_paged dst;
  FastDiv div_bs;
  int32_t first_frame;
  int32_t n_plane_items;  // n_frames * tiles_per_frame (per plane)
  int32_t G;              // groups per layer
};

// Head windows of kvf_restore_batch_heads (the same for every unit of a launch;
// else the whole slot: head_lo 0, head_hi = win_heads = H).
struct HeadWin {
  int32_t head_lo, head_hi;  // heads restored
  int32_t win_heads;         // heads per window; window w lands at + w * win_stride
  int32_t raw;               // int8 destination gets the samples (q + 128), not q
  int64_t win_stride;        // bytes
};

struct RestoreParams {
  int32_t n_units;
  HeadWin hw;
  RestoreUnitDev u[KVF_MAX_UNITS];
};

// grid = (item tiles, unit, plane): the plane (layer of the triplet) is uniform
// per CTA, so each lane loads its VPL group scales once and the per-item index
// math is a handful of multiply-high divisions by host-precomputed constants.
// HW: head window (kvf_restore_batch_heads): only heads [head_lo, head_hi)
// move, to local head h - head_lo of the destination.
template <int OUT, int VPL, bool HW = false>
__global__ void __launch_bounds__(kThreads)
    restore_fast_kernel(const __grid_constant__ RestoreParams P) {
  const RestoreUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int SUB = sub_for(VPL);         // items side by side in the warp
  constexpr int LPI = 32 / SUB;             // lanes per item
  constexpr int VL = vl_for(VPL);           // vectors per lane per item
  const int sub = lane / LPI, sl = lane % LPI;
  const int item0 = (blockIdx.x * kWarps + warp) * ipw_for(VPL);
  char* layer = reinterpret_cast<char*>(U.dst.layer[p]);
  if (item0 >= U.n_plane_items || layer == nullptr) return;

  constexpr int ES = OUT == KVF_F32 ? 4 : (OUT == KVF_I8 ? 1 : 2);
  int32_t in_off[VL];
  using OffT = std::conditional_t<HW, int64_t, int32_t>;
  OffT out_off[VL];
  float s[VL];
  uint32_t live = ~0u;  // HW: the lane's vectors inside the head windows
#pragma unroll
  for (int k = 0; k < VL; ++k) {
    int c = (sl + LPI * k) * 8;
    in_off[k] = (int32_t)tile_offset(U.g, c, U.fr.row_pitch);
    if constexpr (HW) {
      const int h = c >> U.g.lg_D;
      if (h < P.hw.head_lo || h >= P.hw.head_hi) live &= ~(1u << k);
      const int r = h - P.hw.head_lo, w = r / P.hw.win_heads;
      const int local = (r - w * P.hw.win_heads) << U.g.lg_D | (c & ((1 << U.g.lg_D) - 1));
      out_off[k] = (int64_t)w * P.hw.win_stride +
                   slot_channel_offset(U.g, local, U.dst.head_stride) * ES;
    } else {
      out_off[k] = (int32_t)slot_channel_offset(U.g, c, U.dst.head_stride) * ES;
    }
    if constexpr (OUT != KVF_I8) s[k] = __ldg(U.scales + p * U.G + (c >> U.g.lg_gs));
  }
  const uint32_t flip = (HW && P.hw.raw) ? 0u : 0x80808080u;
  const uint8_t* plane_base = U.fr.base + (int64_t)p * U.fr.plane_stride;

  uint2 v[kIPW][VL];
  char* outp[kIPW];
#pragma unroll
  for (int it = 0; it < kIPW; ++it) {
    outp[it] = nullptr;
    const int q = item0 + it * SUB + sub;  // (frame, slot) item of this plane
    if (q < U.n_plane_items) {
      const int fl = fdiv(U.g.div_tpf, q);
      const int slot = q - fl * U.g.tpf;
      const int f = U.first_frame + fl;
      const int i = token_of(U.g, f, slot);
      if (i < U.g.T) {
        const int tr = fdiv(U.g.div_cols, slot);
        const int tc = slot - tr * U.g.grid_cols;
        const uint8_t* src = plane_base + (int64_t)f * U.fr.frame_stride +
                             (int64_t)tr * U.g.tile_h * U.fr.row_pitch + tc * U.g.tile_w;
#pragma unroll
        for (int k = 0; k < VL; ++k)
          if (!HW || ((live >> k) & 1)) v[it][k] = ld_nc_v2(src + in_off[k]);
        outp[it] = layer + paged_slot_offset_fd(U.dst, U.div_bs, i) * ES;
      }
    }
  }

#pragma unroll
  for (int it = 0; it < kIPW; ++it) {
    if (outp[it] == nullptr) continue;
#pragma unroll
    for (int k = 0; k < VL; ++k) {
      if (HW && !((live >> k) & 1)) continue;
      char* dst = outp[it] + out_off[k];
      if constexpr (OUT == KVF_I8) {
        // int8 code = u8 sample - 128 = sample ^ 0x80 (fk/fetchsim.py:351).
        st_v2(dst, make_uint2(v[it][k].x ^ flip, v[it][k].y ^ flip));
      } else {
        float q[8];
        bytes8_to_float(v[it][k].x, v[it][k].y, q);
#pragma unroll
        for (int e = 0; e < 8; ++e) q[e] *= s[k];
        if constexpr (OUT == KVF_F32) {
          st_v4(dst, make_uint4(__float_as_uint(q[0]), __float_as_uint(q[1]),
                                __float_as_uint(q[2]), __float_as_uint(q[3])));
          st_v4(dst + 16, make_uint4(__float_as_uint(q[4]), __float_as_uint(q[5]),
                                     __float_as_uint(q[6]), __float_as_uint(q[7])));
        } else if constexpr (OUT == KVF_BF16) {
          st_v4(dst, make_uint4(pack_bf16x2(q[0], q[1]), pack_bf16x2(q[2], q[3]),
                                pack_bf16x2(q[4], q[5]), pack_bf16x2(q[6], q[7])));
        } else {
          st_v4(dst, make_uint4(pack_f16x2(q[0], q[1]), pack_f16x2(q[2], q[3]),
                                pack_f16x2(q[4], q[5]), pack_f16x2(q[6], q[7])));
        }
      }
    }
  }
}

// One thread per (item, channel): any layout, group size, alignment.
__global__ void __launch_bounds__(kThreads)
    restore_generic_kernel(const __grid_constant__ RestoreParams P) {
  const RestoreUnitDev& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  int64_t x = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  int64_t q_item = x >> U.g.lg_C;
  void* layer = U.dst.layer[p];
  if (q_item >= U.n_plane_items || layer == nullptr) return;
  int c = (int)(x & (U.g.C - 1));
  const int h = c >> U.g.lg_D;
  const bool win = P.hw.win_heads > 0;  // kvf_restore_batch_heads
  if (win && (h < P.hw.head_lo || h >= P.hw.head_hi)) return;
  const int hr = win ? h - P.hw.head_lo : 0, hw = win ? hr / P.hw.win_heads : 0;
  const int local = win ? ((hr - hw * P.hw.win_heads) << U.g.lg_D | (c & ((1 << U.g.lg_D) - 1)))
                        : c;
  int fl = (int)q_item / U.g.tpf;
  int slot = (int)q_item - fl * U.g.tpf;
  int f = U.first_frame + fl;
  int i = token_of(U.g, f, slot);
  if (i >= U.g.T) return;
  int tr = slot / U.g.grid_cols;
  int tc = slot - tr * U.g.grid_cols;
  const uint8_t* src = U.fr.base + (int64_t)f * U.fr.frame_stride +
                       (int64_t)p * U.fr.plane_stride +
                       (int64_t)tr * U.g.tile_h * U.fr.row_pitch + (int64_t)tc * U.g.tile_w +
                       tile_offset(U.g, c, U.fr.row_pitch);
  int q = (int)*src - 128;
  float val = 0.0f;
  if (U.dst.dtype != KVF_I8)
    val = (float)q * __ldg(U.scales + p * U.G + c / U.g.group_size);
  int64_t o = paged_slot_offset(U.dst, i) + slot_channel_offset(U.g, local, U.dst.head_stride);
  void* base = static_cast<char*>(layer) + (int64_t)hw * P.hw.win_stride;
  store_from_float(base, o, U.dst.dtype, val, P.hw.raw ? q + 128 : q);
}

bool aligned(const void* p, int64_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

// 0 = generic, else VPL of the fast kernel.
int restore_variant(const kvf_restore_unit& u) {
  const kvf_plan& p = u.plan;
  int64_t C = (int64_t)p.H * p.D;
  if (C != 128 && C % 256 != 0) return 0;
  int vpl = C == 128 ? kVariantC128 : (int)(C / 256);
  if (vpl != 1 && vpl != 2 && vpl != kVariantC128 && vpl != 4 && vpl != 8 && vpl != 16)
    return 0;
  if (p.b_d % 8 != 0) return 0;
  if (u.dst.dtype != KVF_I8 && p.group_size % 8 != 0) return 0;
  if (!aligned(u.frames.base, 8) || u.frames.frame_stride % 8 ||
      u.frames.plane_stride % 8 || u.frames.row_pitch % 8)
    return 0;
  int64_t es = (int64_t)dtype_size(u.dst.dtype);
  int64_t va = u.dst.dtype == KVF_I8 ? 8 : 16;  // bytes per vector store
  for (int l = 0; l < 3; ++l)
    if (u.dst.layer[l] && !aligned(u.dst.layer[l], va)) return 0;
  if ((u.dst.head_stride * es) % va || (u.dst.slot_stride * es) % va ||
      (u.dst.block_stride * es) % va)
    return 0;
  return vpl;
}

kvf_status check_unit(const kvf_restore_unit& u) {
  kvf_status st = check_plan(u.plan);
  if (st != KVF_OK) return st;
  if (u.first_frame < 0 || u.n_frames < 0 ||
      (int64_t)u.first_frame + u.n_frames > u.plan.frame_count)
    KVF_FAIL(KVF_EINVAL, "frame range [%d, %d) outside the plan's %d frames",
             u.first_frame, u.first_frame + u.n_frames, u.plan.frame_count);
  if (u.n_frames > 0 && u.frames.base == nullptr)
    KVF_FAIL(KVF_EINVAL, "null frame surface");
  if (u.frames.row_pitch < u.plan.frame_w)
    KVF_FAIL(KVF_EINVAL, "row pitch %lld below frame width %d",
             (long long)u.frames.row_pitch, u.plan.frame_w);
  if (u.dst.dtype < KVF_BF16 || u.dst.dtype > KVF_I8)
    KVF_FAIL(KVF_EINVAL, "bad destination dtype %d", u.dst.dtype);
  if (u.dst.dtype != KVF_I8 && u.scales == nullptr)
    KVF_FAIL(KVF_EINVAL, "dequantising restore needs scales");
  if (u.dst.block_size < 1) KVF_FAIL(KVF_EINVAL, "block_size must be >= 1");
  if (u.dst.token_base < 0) KVF_FAIL(KVF_EINVAL, "negative token_base");
  if ((int64_t)u.dst.token_base + u.plan.T >= (int64_t(1) << 31))
    KVF_FAIL(KVF_EUNSUPPORTED, "token index beyond 2^31");
  return KVF_OK;
}

RestoreUnitDev to_dev(const kvf_restore_unit& u) {
  RestoreUnitDev d;
  d.fr = u.frames;
  d.g = make_geom(u.plan);
  d.scales = u.scales;
  d.dst = u.dst;
  d.div_bs = make_fastdiv(u.dst.block_size);
  d.first_frame = u.first_frame;
  d.n_plane_items = u.n_frames * u.plan.tiles_per_frame;
  d.G = (u.plan.H * u.plan.D) / u.plan.group_size;
  return d;
}

template <int OUT, bool HW>
void launch_fast(int vpl, const RestoreParams& P, dim3 grid, cudaStream_t s) {
  switch (vpl) {
    case 1: restore_fast_kernel<OUT, 1, HW><<<grid, kThreads, 0, s>>>(P); break;
    case 2: restore_fast_kernel<OUT, 2, HW><<<grid, kThreads, 0, s>>>(P); break;
    case kVariantC128: restore_fast_kernel<OUT, 0, HW><<<grid, kThreads, 0, s>>>(P); break;
    case 4: restore_fast_kernel<OUT, 4, HW><<<grid, kThreads, 0, s>>>(P); break;
    case 8: restore_fast_kernel<OUT, 8, HW><<<grid, kThreads, 0, s>>>(P); break;
    case 16: restore_fast_kernel<OUT, 16, HW><<<grid, kThreads, 0, s>>>(P); break;
  }
}

// Launch one group of units that share (variant, dtype).
struct HeadWindow {
  int32_t lo, hi, win_heads, raw;
  int64_t win_stride;
  bool on;
};

kvf_status launch_group(const std::vector<kvf_restore_unit>& units, int vpl,
                        int32_t dtype, cudaStream_t s,
                        HeadWindow hw = {0, 0, 1, 0, 0, false}) {
  // equal launches (e.g. 280 units: 94 + 93 + 93, not 128 + 128 + 24, whose
  // last small launch would leave most SMs idle)
  const size_t n_launch = (units.size() + KVF_MAX_UNITS - 1) / KVF_MAX_UNITS;
  const size_t per = n_launch ? (units.size() + n_launch - 1) / n_launch : 0;
  for (size_t at = 0; at < units.size(); at += per) {
    size_t n = std::min<size_t>(per, units.size() - at);
    RestoreParams P;
    P.n_units = (int32_t)n;
    P.hw = hw.on ? HeadWin{hw.lo, hw.hi, hw.win_heads, hw.raw, hw.win_stride}
                 : HeadWin{0, 0, 0, 0, 0};
    int64_t max_work = 0;
    for (size_t k = 0; k < n; ++k) {
      P.u[k] = to_dev(units[at + k]);
      int64_t w = vpl ? P.u[k].n_plane_items : (int64_t)P.u[k].n_plane_items * P.u[k].g.C;
      max_work = std::max(max_work, w);
    }
    if (max_work == 0) continue;
    int64_t per_cta =
        vpl ? (int64_t)kWarps * ipw_for(vpl == kVariantC128 ? 0 : vpl) : kThreads;
    int64_t gx = (max_work + per_cta - 1) / per_cta;
    if (gx > 0x7FFFFFFF) KVF_FAIL(KVF_EUNSUPPORTED, "restore grid too large");
    dim3 grid((unsigned)gx, (unsigned)n, 3);
    if (vpl == 0) {
      restore_generic_kernel<<<grid, kThreads, 0, s>>>(P);
    } else {
      if (hw.on) {
        switch (dtype) {
          case KVF_BF16: launch_fast<KVF_BF16, true>(vpl, P, grid, s); break;
          case KVF_F16: launch_fast<KVF_F16, true>(vpl, P, grid, s); break;
          case KVF_F32: launch_fast<KVF_F32, true>(vpl, P, grid, s); break;
          case KVF_I8: launch_fast<KVF_I8, true>(vpl, P, grid, s); break;
        }
      } else {
        switch (dtype) {
          case KVF_BF16: launch_fast<KVF_BF16, false>(vpl, P, grid, s); break;
          case KVF_F16: launch_fast<KVF_F16, false>(vpl, P, grid, s); break;
          case KVF_F32: launch_fast<KVF_F32, false>(vpl, P, grid, s); break;
          case KVF_I8: launch_fast<KVF_I8, false>(vpl, P, grid, s); break;
        }
      }
    }
    KVF_CHECK_CUDA(cudaGetLastError());
  }
  return KVF_OK;
}

}  // namespace
}  // namespace kvf

using namespace kvf;

extern "C" kvf_status kvf_restore_batch(const kvf_restore_unit* units,
                                        int32_t n_units, void* stream) {
  if (n_units < 0 || (n_units > 0 && units == nullptr))
    KVF_FAIL(KVF_EINVAL, "bad unit array");
  // Group by (variant, dtype) so each launch instantiates one kernel; variant
  // 17 = shared-memory band transpose (tile rows narrower than 8 channels).
  constexpr int kBand = 17;
  std::vector<kvf_restore_unit> groups[kBand + 1][4];
  for (int32_t k = 0; k < n_units; ++k) {
    kvf_status st = check_unit(units[k]);
    if (st != KVF_OK) return st;
    if (units[k].n_frames == 0) continue;
    int v = restore_variant(units[k]);
    if (v == 0 && restore_band_ok(units[k])) v = kBand;
    groups[v][units[k].dst.dtype].push_back(units[k]);
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int v = 0; v <= kBand; ++v)
    for (int dt = 0; dt < 4; ++dt)
      if (!groups[v][dt].empty()) {
        kvf_status st = v == kBand ? launch_restore_band(groups[v][dt], dt, s)
                                   : launch_group(groups[v][dt], v, dt, s);
        if (st != KVF_OK) return st;
      }
  return KVF_OK;
}

extern "C" kvf_status kvf_restore_batch_heads(const kvf_restore_unit* units, int32_t n_units,
                                              int32_t head_lo, int32_t n_heads,
                                              int32_t n_windows, int64_t window_stride,
                                              int32_t raw_samples, void* stream) {
  if (n_units < 0 || (n_units > 0 && units == nullptr))
    KVF_FAIL(KVF_EINVAL, "bad unit array");
  std::vector<kvf_restore_unit> groups[17][4];
  for (int32_t k = 0; k < n_units; ++k) {
    kvf_status st = check_unit(units[k]);
    if (st != KVF_OK) return st;
    if (head_lo < 0 || n_heads < 1 || n_windows < 1 ||
        head_lo + (int64_t)n_windows * n_heads > units[k].plan.H)
      KVF_FAIL(KVF_EINVAL, "head windows [%d, %lld) outside %d heads", head_lo,
               (long long)head_lo + (long long)n_windows * n_heads, units[k].plan.H);
    if (raw_samples && units[k].dst.dtype != KVF_I8)
      KVF_FAIL(KVF_EINVAL, "raw samples need an int8 destination");
    if (units[k].n_frames == 0) continue;
    // the fast kernel when its conditions hold for the local cache, else the
    // one-thread-per-sample kernel (tile rows narrower than 8 channels too)
    groups[restore_variant(units[k])][units[k].dst.dtype].push_back(units[k]);
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const HeadWindow hw{head_lo, head_lo + n_windows * n_heads, n_heads, raw_samples ? 1 : 0,
                      window_stride, true};
  for (int v = 0; v < 17; ++v)
    for (int dt = 0; dt < 4; ++dt)
      if (!groups[v][dt].empty()) {
        kvf_status st = launch_group(groups[v][dt], v, dt, s, hw);
        if (st != KVF_OK) return st;
      }
  return KVF_OK;
}

extern "C" kvf_status kvf_restore(const kvf_surface* frames, int32_t first_frame,
                                  int32_t n_frames, const kvf_plan* plan,
                                  const float* scales, const kvf_paged* dst,
                                  void* stream) {
  if (!frames || !plan || !dst) KVF_FAIL(KVF_EINVAL, "null argument");
  kvf_restore_unit u;
  u.frames = *frames;
  u.plan = *plan;
  u.scales = scales;
  u.dst = *dst;
  u.first_frame = first_frame;
  u.n_frames = n_frames;
  return kvf_restore_batch(&u, 1, stream);
}
