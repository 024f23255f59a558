// kvf_pack_persist.cu — single-HBM-read pack, sm_100a: one persistent
// cooperative grid walks the (unit, plane) slabs of a pack batch with a
// one-step lag between the two halves of the reference quantiser.
//
// The reference scale of a (unit, plane, group) is the max |x| over ALL chunk
// tokens (fk/kvmodel.py:138-140), so no sample can be quantised (:141-143) and
// placed (fk/layout.py:234-258) before the whole group has been read.  The
// phase-split kernels (kvf_pack.cu) read the source twice from HBM (5 B/elem
// against 3 algorithmic).  Here every CTA owns a fixed 1/N share of every
// slab (a slab = whole (unit, plane)s, ~16 MB of source) and runs, at step j:
//
//   A(j):   max |x| of its share of slab j's token rows -> shared-memory
//           reduction -> atomicMax into the unit's [3, G] maxima; then one
//           release-add on slab j's counter.
//   B(j-1): wait until slab j-1's counter reached N (every CTA finished its
//           A(j-1) one step earlier, so the wait is normally already over),
//           derive the scales, then quantise + tile + place its share of slab
//           j-1's frame items.  Slab j-1 was read from HBM one step ago and is
//           still in L2 (two slabs + the frames in flight, ~40 MB of 126 MB):
//           the re-read costs L2 bandwidth, not HBM.
//
// HBM traffic is the algorithmic 2 B read + 1 B written per element.  The grid
// must be co-resident (CTAs wait on each other's counters): it is launched
// cooperatively with the occupancy-limited CTA count.
#include <algorithm>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kThreads = kPackThreads;
constexpr int kWarps = kPackWarps;
constexpr int kMaxUps = 3 * kMaxPackUnits;  // (unit, plane) pairs per launch
constexpr int kMaxG = 512;                  // groups per plane: C <= 4096, gs >= 8

struct PersistParams {
  int32_t n_units;
  int32_t n_slabs;
  int32_t ra, rb;   // A : B CTA ratio
  int32_t lag;      // A-CTAs run at most `lag` slabs ahead of the B-CTAs
  PackUnitDev u[kMaxPackUnits];
  uint16_t up[kMaxUps];             // (unit << 2) | plane, in slab order
  int16_t slab_first[kMaxUps + 1];  // first up of each slab; [n_slabs] = end
};
static_assert(sizeof(PersistParams) <= 32000, "kernel parameters above 32 KB");

__device__ __forceinline__ const PackUnitDev& up_unit(const PersistParams& P, int k) {
  return P.u[P.up[k] >> 2];
}
__device__ __forceinline__ int up_plane(const PersistParams& P, int k) { return P.up[k] & 3; }

// Slab j's step counter: the first counter word of its first (unit, plane).
__device__ __forceinline__ uint32_t* slab_counter(const PersistParams& P, int j) {
  const int k = P.slab_first[j];
  const PackUnitDev& U = up_unit(P, k);
  return U.counters + up_plane(P, k) * U.G;
}

__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// A(j): this CTA's share of slab j's token rows -> per-group maxima.
template <int SRC, int VPL, typename LD>
__device__ __forceinline__ void phase_absmax(const PersistParams& P, int j, uint32_t* s_max,
                                             LD ld, int me, int n) {
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = P.slab_first[j], k1 = P.slab_first[j + 1];
  int64_t R = 0;
  for (int k = k0; k < k1; ++k) R += up_unit(P, k).g.T;
  const int64_t r0 = R * me / n, r1 = R * (me + 1) / n;
  int64_t base = 0;
  for (int k = k0; k < k1; ++k) {
    const PackUnitDev& U = up_unit(P, k);
    const int p = up_plane(P, k);
    const int lo = (int)(max(r0, base) - base), hi = (int)(min(r1, base + U.g.T) - base);
    base += U.g.T;
    const char* layer = reinterpret_cast<const char*>(U.src.layer[p]);
    if (lo >= hi || layer == nullptr) continue;  // uniform over the CTA
    for (int g = threadIdx.x; g < U.G; g += kThreads) s_max[g] = 0u;
    __syncthreads();
    int32_t off[VPL];
    uint32_t m[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      off[v] = (int32_t)slot_channel_offset(U.g, (lane + 32 * v) * 8, U.src.head_stride) * ES;
      m[v] = 0u;
    }
#pragma unroll(VPL >= 4 ? 2 : 8 / VPL)  // ~8 vectors per lane in flight
    for (int i = lo + warp; i < hi; i += kWarps) {
      const char* slot = layer + paged_slot_offset_fd(U.src, U.div_bs, i) * ES;
#pragma unroll
      for (int v = 0; v < VPL; ++v) m[v] = max(m[v], vec_absmax_bits<SRC>(slot + off[v], ld));
    }
    reduce_groups<SRC, VPL>(m, U.g.group_size, s_max);
    __syncthreads();
    for (int g = threadIdx.x; g < U.G; g += kThreads)
      if (s_max[g]) atomicMax(&U.absmax[p * U.G + g], s_max[g]);
    __syncthreads();
  }
}

// B(j): once every CTA has contributed its maxima of slab j, this CTA's share
// of slab j's frame items.
template <int SRC, int VPL, typename LD>
__device__ __forceinline__ void phase_frames(const PersistParams& P, int j, float* s_sc, LD ld,
                                             int me, int n) {
  constexpr int SUB = pack_sub<SRC, VPL>();
  const int warp = threadIdx.x >> 5;
  const int k0 = P.slab_first[j], k1 = P.slab_first[j + 1];
  int64_t I = 0;
  for (int k = k0; k < k1; ++k) I += up_unit(P, k).n_items;
  const int64_t q0 = I * me / n, q1 = I * (me + 1) / n;
  int64_t base = 0;
  for (int k = k0; k < k1; ++k) {
    const PackUnitDev& U = up_unit(P, k);
    const int p = up_plane(P, k);
    const int lo = (int)(max(q0, base) - base), hi = (int)(min(q1, base + U.n_items) - base);
    base += U.n_items;
    if (lo >= hi) continue;  // uniform over the CTA
    // Scales from the complete maxima (written by atomics in this kernel: read
    // through L2, not the non-coherent path).  The CTA holding item 0 of the
    // plane publishes them (fk/kvmodel.py:140).
    for (int g = threadIdx.x; g < U.G; g += kThreads) {
      const float sc = scale_from_absmax_bits(__ldcg(&U.absmax[p * U.G + g]));
      s_sc[g] = sc;
      if (lo == 0) U.scales[p * U.G + g] = sc;
    }
    __syncthreads();
    PackLane<SRC, VPL> L;
    L.init(U, p, s_sc);
    // items spread round-robin over the warps (a CTA's share of a step is a
    // few items per warp: one pipelined pass, not a latency chain per warp)
    const int item0 = lo + warp * SUB;
    if (item0 < hi) {
      const int rounds = (hi - item0 + kWarps * SUB - 1) / (kWarps * SUB);
      pack_items<SRC, VPL, false>(U, p, L, item0, kWarps * SUB, rounds, hi, ld);
    }
    __syncthreads();  // s_sc is reused by the next plane
  }
}

// Thread 0 waits until *c >= target (acquire), then the CTA proceeds.
__device__ __forceinline__ void cta_wait(const uint32_t* c, uint32_t target) {
  if (threadIdx.x == 0)
    while (ld_acquire_u32(c) < target) __nanosleep(20);
  __syncthreads();
}
// Release (cumulative over the CTA barrier): everything the CTA did before is
// ordered before the add.
__device__ __forceinline__ void cta_arrive(uint32_t* c) {
  __syncthreads();
  if (threadIdx.x == 0) red_release_add(c, 1u);
}

// Role-split schedule: CTAs b with b % (ra + rb) < ra are A-CTAs (maxima),
// the others B-CTAs (frames).  Slab j's counter counts the A arrivals (n_a:
// its maxima are complete) and then the B arrivals (n_a + n_b: its frames are
// done).  A-CTAs run at most `lag` slabs ahead of the B-CTAs, which bounds the
// L2 footprint to ~lag slabs.
template <int SRC, int VPL>
__global__ void __launch_bounds__(kThreads, 4)
    pack_persist_kernel(const __grid_constant__ PersistParams P) {
  __shared__ uint32_t s_max[kMaxG];
  __shared__ float s_sc[kMaxG];
  const int ra = P.ra, rb = P.rb, per = ra + rb;
  const int b = blockIdx.x, cyc = b / per, pos = b % per;
  const int full = gridDim.x / per, rem = gridDim.x % per;
  const uint32_t n_a = full * ra + min(rem, ra);
  const uint32_t n_b = gridDim.x - n_a;
  if (pos < ra) {
    const int me = cyc * ra + pos;
    for (int j = 0; j < P.n_slabs; ++j) {
      if (j >= P.lag) cta_wait(slab_counter(P, j - P.lag), n_a + n_b);
      phase_absmax<SRC, VPL>(P, j, s_max, KeepLoad(), me, n_a);
      cta_arrive(slab_counter(P, j));
    }
  } else {
    const int me = cyc * rb + pos - ra;
    const auto lb = WithPolicy{l2_policy_evict_first()};
    for (int j = 0; j < P.n_slabs; ++j) {
      cta_wait(slab_counter(P, j), n_a);
      phase_frames<SRC, VPL>(P, j, s_sc, lb, me, n_b);
      cta_arrive(slab_counter(P, j));
    }
  }
}

template <int SRC>
const void* kernel_for(int vpl) {
  switch (vpl) {
    case 1: return (const void*)pack_persist_kernel<SRC, 1>;
    case 2: return (const void*)pack_persist_kernel<SRC, 2>;
    case 4: return (const void*)pack_persist_kernel<SRC, 4>;
    case 8: return (const void*)pack_persist_kernel<SRC, 8>;
    case 16: return (const void*)pack_persist_kernel<SRC, 16>;
    default: return nullptr;
  }
}

struct DeviceInfo {
  int sms = 0;
  bool coop = false;
};

DeviceInfo device_info() {
  int dev = 0, sms = 0, coop = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess) {
    cudaGetLastError();
    return DeviceInfo();
  }
  DeviceInfo d;
  d.sms = sms;
  d.coop = coop != 0;
  return d;
}

}  // namespace

// Source bytes a slab aims at (slab_bytes == 0): two slabs and the frames of
// one stay well inside L2 (126 MB on B200) while a step stays long against the
// counter hand-off latency.
constexpr int64_t kDefaultSlabBytes = 16ll << 20;

// Single-read pack of quantising fast-variant units (zeroed scratch required:
// maxima and counters).  *launched = false when the device or the shapes do
// not allow it (the caller then runs the phase-split kernels).
kvf_status launch_pack_persist(const std::vector<kvf_pack_unit>& units, int vpl, int32_t dtype,
                               int64_t slab_bytes, cudaStream_t s, bool* launched) {
  const int tune = (int)(slab_bytes & 0xFF);  // tuning hook (low bits): lag | ratio
  slab_bytes &= ~int64_t(0xFF);
  if (slab_bytes <= 0) slab_bytes = kDefaultSlabBytes;
  *launched = false;
  if (units.empty() || units.size() > (size_t)kMaxPackUnits || dtype == KVF_I8) return KVF_OK;
  const void* fn = dtype == KVF_BF16  ? kernel_for<KVF_BF16>(vpl)
                   : dtype == KVF_F16 ? kernel_for<KVF_F16>(vpl)
                                      : kernel_for<KVF_F32>(vpl);
  if (fn == nullptr) return KVF_OK;
  for (const auto& u : units)
    if ((int64_t)u.plan.H * u.plan.D / u.plan.group_size > kMaxG) return KVF_OK;
  const DeviceInfo di = device_info();
  int occ = 0;
  if (!di.coop || di.sms < 1 ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, 0) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    return KVF_OK;
  }
  PersistParams* P = new PersistParams();
  P->n_units = (int32_t)units.size();
  P->lag = tune & 0xF ? (tune & 0xF) : 2;
  P->ra = (tune >> 4) & 3 ? (tune >> 4) & 3 : 1;
  P->rb = (tune >> 6) & 3 ? (tune >> 6) & 3 : 1;
  const size_t es = dtype_size(dtype);
  int n_up = 0, n_slab = 0;
  int64_t acc = 0;
  for (size_t k = 0; k < units.size(); ++k) {
    P->u[k] = make_pack_unit_dev(units[k]);
    const int64_t plane_bytes = (int64_t)units[k].plan.T * units[k].plan.H * units[k].plan.D * es;
    for (int p = 0; p < 3; ++p) {
      if (acc == 0) P->slab_first[n_slab++] = (int16_t)n_up;
      P->up[n_up++] = (uint16_t)((k << 2) | p);
      acc += plane_bytes;
      if (acc >= slab_bytes) acc = 0;
    }
  }
  P->n_slabs = n_slab;
  P->slab_first[n_slab] = (int16_t)n_up;
  void* args[] = {P};
  cudaError_t e =
      cudaLaunchCooperativeKernel(fn, dim3(di.sms * occ), dim3(kThreads), args, 0, s);
  delete P;
  if (e != cudaSuccess) return cuda_status(e, "pack_persist_kernel launch");
  *launched = true;
  return KVF_OK;
}

}  // namespace kvf
