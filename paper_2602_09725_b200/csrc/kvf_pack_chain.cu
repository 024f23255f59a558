// kvf_pack_chain.cu — single-HBM-read pack, sm_100a: a chain of small kernels,
// one per (unit, plane) PLANE-UNIT, linked by programmatic dependent launch.
//
// The reference scale of a (unit, plane, group) is the max |x| over ALL chunk
// tokens (fk/kvmodel.py:138-140): a plane's samples can be quantised
// (:141-143) and placed (fk/layout.py:234-258) only once the whole plane was
// read.  The two-pass kernels (kvf_pack.cu) read the source twice from HBM.
// Here launch i of the chain, on every SM:
//
//   1. folds the |x| maxima of plane-unit i+1 (16-byte loads that leave the
//      lines in L2; red.max into the unit's scratch) -- it depends on nothing,
//      so it starts while launch i-1 is still finishing (PDL: the previous
//      launch triggers its dependents at once);
//   2. griddepcontrol.wait: launch i-1 is complete, so the maxima of
//      plane-unit i (folded by launch i-1) are final;
//   3. quantises and places plane-unit i (the frames-pass loop of kvf_pack.cu),
//      re-reading its tokens from L2 (evict-first).
//
// The kernel boundary is the only synchronisation (no spin waits); PDL hides
// the launch gaps and tails behind the next fold.  L2 holds about three
// plane-units (20 MB each for a 10,000-token bf16 chunk).  HBM traffic is the
// algorithmic 2 B read + 1 B written per element when the re-reads hit L2.
#include <algorithm>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kCThreads = 256;
constexpr int kCWarps = kCThreads / 32;

struct ChainParams {
  PackUnitDev uf, uq;  // fold plane-unit (uf, pf); quantise plane-unit (uq, pq)
  int32_t pf, pq;      // plane index, -1: none
};

template <int SRC, int VPL>
__global__ void __launch_bounds__(kCThreads, 4) pack_chain_kernel(const __grid_constant__ ChainParams P) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ uint32_t s_max[64];
  __shared__ float s_sc[64];
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = gridDim.x, b = blockIdx.x;
  // 1. fold plane-unit (uf, pf)
  if (P.pf >= 0) {
    const PackUnitDev& U = P.uf;
    const char* layer = reinterpret_cast<const char*>(U.src.layer[P.pf]);
    if (layer != nullptr) {
      for (int k = threadIdx.x; k < U.G; k += kCThreads) s_max[k] = 0u;
      __syncthreads();
      const int T = U.g.T;
      const int t0 = (int)((int64_t)T * b / nb), t1 = (int)((int64_t)T * (b + 1) / nb);
      int32_t off[VPL];
      uint32_t m[VPL];
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        off[k] = (int32_t)slot_channel_offset(U.g, (lane + 32 * k) * 8, U.src.head_stride) * ES;
        m[k] = 0u;
      }
#pragma unroll 2
      for (int i = t0 + warp; i < t1; i += kCWarps) {
        const char* slot = layer + paged_slot_offset_fd(U.src, U.div_bs, i) * ES;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          m[k] = max(m[k], vec_absmax_bits<SRC, KeepLoad>(slot + off[k]));
      }
      reduce_groups<SRC, VPL>(m, U.g.group_size, s_max);
      __syncthreads();
      for (int k = threadIdx.x; k < U.G; k += kCThreads)
        if (s_max[k]) atomicMax(&U.absmax[P.pf * U.G + k], s_max[k]);
    }
  }
  // 2. the previous launch (the fold of this launch's quantise plane-unit) is complete
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // 3. quantise and place plane-unit (uq, pq)
  if (P.pq >= 0) {
    const PackUnitDev& U = P.uq;
    const int p = P.pq;
    const bool real = U.src.layer[p] != nullptr;
    for (int k = threadIdx.x; k < U.G; k += kCThreads) {
      uint32_t bits = 0u;
      if (real) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(bits) : "l"(U.absmax + p * U.G + k));
      const float sc = scale_from_absmax_bits(bits);  // fk/kvmodel.py:139-140
      s_sc[k] = sc;
      if (b == 0) U.scales[p * U.G + k] = sc;
    }
    __syncthreads();
    constexpr int SUB = pack_sub<SRC, VPL>();
    const int n = U.n_items;
    const int q0 = (int)((int64_t)n * b / nb), q1 = (int)((int64_t)n * (b + 1) / nb);
    const int item0 = q0 + warp * SUB;
    if (item0 < q1) {
      PackLane<SRC, VPL> L;
      L.init(U, p, s_sc);
      const int rounds = (q1 - item0 + kCWarps * SUB - 1) / (kCWarps * SUB);
      pack_items<SRC, VPL, false>(U, p, L, item0, kCWarps * SUB, rounds, q1,
                                  WithPolicy{l2_policy_evict_first()});
    }
  }
}

constexpr int kZeroUnits = 256;
struct ZeroParams {
  uint32_t* absmax[kZeroUnits];
  int32_t words[kZeroUnits];
  int32_t n;
};
__global__ void zero_chain_scratch(const __grid_constant__ ZeroParams Z) {
  for (int u = blockIdx.x; u < Z.n; u += gridDim.x)
    for (int k = threadIdx.x; k < Z.words[u]; k += blockDim.x) Z.absmax[u][k] = 0u;
}

template <int SRC>
const void* chain_kernel_for(int vpl) {
  switch (vpl) {
    case 1: return (const void*)pack_chain_kernel<SRC, 1>;
    case 2: return (const void*)pack_chain_kernel<SRC, 2>;
    case 4: return (const void*)pack_chain_kernel<SRC, 4>;
    case 8: return (const void*)pack_chain_kernel<SRC, 8>;
    case 16: return (const void*)pack_chain_kernel<SRC, 16>;
    default: return nullptr;
  }
}

}  // namespace

// Single-read pack of the quantising units of one (variant = VPL, dtype) group
// as a PDL chain of plane-unit kernels.  *launched = false when the device or
// the shapes do not allow it (the caller then runs the phase-split kernels).
kvf_status launch_pack_chain(const std::vector<kvf_pack_unit>& units, int vpl, int32_t dtype,
                             int ctas_per_sm, cudaStream_t s, bool* launched) {
  *launched = false;
  if (units.empty() || dtype == KVF_I8) return KVF_OK;
  for (const auto& u : units)
    if (u.plan.H * u.plan.D / u.plan.group_size > 64) return KVF_OK;  // s_max / s_sc
  const void* fn = dtype == KVF_BF16  ? chain_kernel_for<KVF_BF16>(vpl)
                   : dtype == KVF_F16 ? chain_kernel_for<KVF_F16>(vpl)
                                      : chain_kernel_for<KVF_F32>(vpl);
  if (fn == nullptr) return KVF_OK;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kCThreads, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return KVF_OK;
  }
  // every unit's maxima to zero first (one small launch per 256 units; the
  // chain's first kernel starts when it completed)
  for (size_t at = 0; at < units.size(); at += kZeroUnits) {
    ZeroParams Z;
    Z.n = (int32_t)std::min<size_t>(kZeroUnits, units.size() - at);
    for (int k = 0; k < Z.n; ++k) {
      const kvf_pack_unit& u = units[at + k];
      Z.absmax[k] = u.absmax;
      Z.words[k] = 3 * u.plan.H * u.plan.D / u.plan.group_size;
    }
    zero_chain_scratch<<<std::min(Z.n, 64), 128, 0, s>>>(Z);
    KVF_CHECK_CUDA(cudaGetLastError());
  }
  const int grid = sms * std::min(per_sm, ctas_per_sm > 0 ? ctas_per_sm : 4);
  // plane-units in order: (unit k, plane p)
  const int n_pu = (int)(3 * units.size());
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kCThreads);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ChainParams P;
  for (int i = 0; i <= n_pu; ++i) {
    // launch i folds plane-unit i and quantises plane-unit i - 1
    P.pf = i < n_pu ? i % 3 : -1;
    P.pq = i > 0 ? (i - 1) % 3 : -1;
    if (P.pf >= 0) P.uf = make_pack_unit_dev(units[i / 3]);
    if (P.pq >= 0) P.uq = make_pack_unit_dev(units[(i - 1) / 3]);
    if (P.pf < 0) P.uf = P.uq;
    if (P.pq < 0) P.uq = P.uf;
    void* args[] = {&P};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return cuda_status(e, "pack_chain_kernel launch");
  }
  *launched = true;
  return KVF_OK;
}

}  // namespace kvf
