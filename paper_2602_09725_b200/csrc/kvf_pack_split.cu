// kvf_pack_split.cu — single-HBM-read pack, sm_100a: CTA roles over one
// persistent (cooperative) grid, plane by plane.
//
// The reference scale of a (unit, plane, group) is the max |x| over ALL chunk
// tokens (fk/kvmodel.py:138-140), so a plane's samples can be quantised
// (:141-143) and placed (fk/layout.py:234-258) only after the whole plane was
// read.  The phase-split kernels (kvf_pack.cu) read the source twice from HBM.
// Here the CTAs of one grid take two roles over the launch's PLANE-UNITS
// ((unit, plane): 20 MB of bf16 for a 10,000-token chunk), in order:
//
//   * A CTAs (blockIdx < n_a): each folds |x| maxima over its token share of
//     plane-unit i (16-byte loads that leave the lines in L2), red.max of the
//     group maxima, fence, one count on the plane-unit's A counter.
//   * Q CTAs: wait until every A CTA counted plane-unit i, derive the scales,
//     quantise and place their frame-item share of it (the frames-pass loop of
//     kvf_pack.cu), re-reading the tokens from L2 (evict-first), then count it
//     done on the Q counter.
//   * A CTAs run at most kLagPU plane-units ahead of the Q CTAs, so the lines
//     they read are still in L2 when the Q CTAs re-read them (~3 x 20 MB).
//
// One sync per plane-unit per CTA (not per tile): its latency is hidden behind
// the next plane-unit's fold.  HBM traffic is the algorithmic 2 B read + 1 B
// written per element when the re-reads hit L2 (ncu on C2: 4.31 GB read +
// 2.24 GB written, 1.02x algorithmic), but 2.45-2.9 ms against 1.85 ms for the
// two-pass kernels: each role has only its share of the CTAs, whose loads in
// flight cannot keep HBM busy (warps mostly wait at the role barriers).
#include <algorithm>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kSThreads = 256;
constexpr int kSWarps = kSThreads / 32;
constexpr int kLagPU = 2;
constexpr int kMaxSplitUnits = 88;

struct SplitParams {
  int32_t n_units, n_pu, n_a, n_q, lag;
  PackUnitDev u[kMaxSplitUnits];
};
static_assert(sizeof(SplitParams) <= 32000, "kernel parameters above 32 KB");

// plane-unit counters after the unit's [3, G] maxima and [3, G] counter words
__device__ __forceinline__ uint32_t* a_cnt(const PackUnitDev& U, int p) {
  return U.absmax + 6 * U.G + 2 * p;
}
__device__ __forceinline__ uint32_t* q_cnt(const PackUnitDev& U, int p) {
  return U.absmax + 6 * U.G + 2 * p + 1;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_count(const uint32_t* p, uint32_t target) {
  while (ld_acquire_u32(p) < target) __nanosleep(128);
}

template <int SRC, int VPL>
__global__ void __launch_bounds__(kSThreads, 4) pack_split_kernel(const __grid_constant__ SplitParams P) {
  __shared__ uint32_t s_max[64];
  __shared__ float s_sc[64];
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool role_a = (int)blockIdx.x < P.n_a;
  const int rank = role_a ? (int)blockIdx.x : (int)blockIdx.x - P.n_a;
  const int nr = role_a ? P.n_a : P.n_q;
  for (int pu = 0; pu < P.n_pu; ++pu) {
    const PackUnitDev& U = P.u[pu / 3];
    const int p = pu % 3;
    const char* layer = reinterpret_cast<const char*>(U.src.layer[p]);
    if (role_a) {
      // ---------------------------------------------------------- fold (A)
      if (layer == nullptr) continue;  // pad layer: zeros, maxima stay 0
      if (pu >= P.lag) {
        // the plane-unit `lag` back is quantised everywhere (its lines may go)
        const PackUnitDev& V = P.u[(pu - P.lag) / 3];
        const int vp = (pu - P.lag) % 3;
        if (threadIdx.x == 0 && V.src.layer[vp] != nullptr) wait_count(q_cnt(V, vp), P.n_q);
      }
      for (int k = threadIdx.x; k < U.G; k += kSThreads) s_max[k] = 0u;
      __syncthreads();
      const int T = U.g.T;
      const int t0 = (int)((int64_t)T * rank / nr), t1 = (int)((int64_t)T * (rank + 1) / nr);
      int32_t off[VPL];
      uint32_t m[VPL];
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        off[k] = (int32_t)slot_channel_offset(U.g, (lane + 32 * k) * 8, U.src.head_stride) * ES;
        m[k] = 0u;
      }
#pragma unroll 2
      for (int i = t0 + warp; i < t1; i += kSWarps) {
        const char* slot = layer + paged_slot_offset_fd(U.src, U.div_bs, i) * ES;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          m[k] = max(m[k], vec_absmax_bits<SRC, KeepLoad>(slot + off[k]));
      }
      reduce_groups<SRC, VPL>(m, U.g.group_size, s_max);
      __syncthreads();
      for (int k = threadIdx.x; k < U.G; k += kSThreads) {
        if (s_max[k]) atomicMax(&U.absmax[p * U.G + k], s_max[k]);
        __threadfence();
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(a_cnt(U, p), 1u);
      }
    } else {
      // ------------------------------------------------------ quantise (Q)
      if (layer != nullptr && threadIdx.x == 0) wait_count(a_cnt(U, p), P.n_a);
      __syncthreads();
      for (int k = threadIdx.x; k < U.G; k += kSThreads) {
        const uint32_t bits = layer ? ld_relaxed(&U.absmax[p * U.G + k]) : 0u;
        const float sc = scale_from_absmax_bits(bits);  // fk/kvmodel.py:139-140
        s_sc[k] = sc;
        if (rank == 0) U.scales[p * U.G + k] = sc;
      }
      __syncthreads();
      constexpr int SUB = pack_sub<SRC, VPL>();
      const int n = U.n_items;
      const int q0 = (int)((int64_t)n * rank / nr), q1 = (int)((int64_t)n * (rank + 1) / nr);
      const int item0 = q0 + warp * SUB;
      if (item0 < q1) {
        PackLane<SRC, VPL> L;
        L.init(U, p, s_sc);
        const int rounds = (q1 - item0 + kSWarps * SUB - 1) / (kSWarps * SUB);
        pack_items<SRC, VPL, false>(U, p, L, item0, kSWarps * SUB, rounds, q1,
                                    WithPolicy{l2_policy_evict_first()});
      }
      __syncthreads();
      if (threadIdx.x == 0 && layer != nullptr) {
        __threadfence();
        atomicAdd(q_cnt(U, p), 1u);
      }
    }
  }
}

__global__ void zero_split_scratch(const __grid_constant__ SplitParams P) {
  const PackUnitDev& U = P.u[blockIdx.x];
  for (int k = threadIdx.x; k < 6 * U.G + 8; k += blockDim.x) U.absmax[k] = 0u;
}

template <int SRC>
const void* split_kernel_for(int vpl) {
  switch (vpl) {
    case 1: return (const void*)pack_split_kernel<SRC, 1>;
    case 2: return (const void*)pack_split_kernel<SRC, 2>;
    case 4: return (const void*)pack_split_kernel<SRC, 4>;
    case 8: return (const void*)pack_split_kernel<SRC, 8>;
    case 16: return (const void*)pack_split_kernel<SRC, 16>;
    default: return nullptr;
  }
}

}  // namespace

// Single-read pack of the quantising units of one (variant = VPL, dtype)
// group on CTA roles.  `frac_a`: per-mille of the CTAs folding (0 = 400);
// `lag`: plane-units the folds may run ahead (0 = kLagPU).
// Returns false in *launched when the grid can not be made co-resident.
kvf_status launch_pack_split(const std::vector<kvf_pack_unit>& units, int vpl, int32_t dtype,
                             int frac_a, int lag, cudaStream_t s, bool* launched) {
  lag = lag > 0 ? lag : kLagPU;
  *launched = false;
  if (units.empty() || dtype == KVF_I8) return KVF_OK;
  for (const auto& u : units)
    if (u.plan.H * u.plan.D / u.plan.group_size > 64) return KVF_OK;  // s_max / s_sc
  const void* fn = dtype == KVF_BF16  ? split_kernel_for<KVF_BF16>(vpl)
                   : dtype == KVF_F16 ? split_kernel_for<KVF_F16>(vpl)
                                      : split_kernel_for<KVF_F32>(vpl);
  if (fn == nullptr) return KVF_OK;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSThreads, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return KVF_OK;
  }
  const int grid = sms * std::min(per_sm, 4);
  const int n_a = std::max(1, std::min(grid - 1, grid * (frac_a ? frac_a : 400) / 1000));
  for (size_t at = 0; at < units.size(); at += kMaxSplitUnits) {
    const size_t n = std::min<size_t>(kMaxSplitUnits, units.size() - at);
    SplitParams* P = new SplitParams();
    P->n_units = (int32_t)n;
    P->n_pu = (int32_t)(3 * n);
    P->n_a = n_a;
    P->n_q = grid - n_a;
    P->lag = lag;
    for (size_t k = 0; k < n; ++k) P->u[k] = make_pack_unit_dev(units[at + k]);
    zero_split_scratch<<<(unsigned)n, 256, 0, s>>>(*P);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kSThreads);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {P};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    delete P;
    if (e != cudaSuccess) return cuda_status(e, "pack_split_kernel launch");
  }
  *launched = true;
  return KVF_OK;
}

}  // namespace kvf
