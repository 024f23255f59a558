// kvf_pack_multi.cu — single-HBM-read pack, sm_100a: per-plane fold and
// quantise kernels spread over several CUDA streams.
//
// The reference scale of a (unit, plane, group) is the max |x| over ALL chunk
// tokens (fk/kvmodel.py:138-140): a plane's samples can be quantised
// (:141-143) and placed (fk/layout.py:234-258) only once the whole plane was
// read.  The two-pass kernels (kvf_pack.cu) fold every unit, then quantise
// every unit, reading the source twice from HBM.  Here each (unit, plane)
// PLANE-UNIT gets its own pair of kernels on one of S streams:
//
//   fold(i)      |x| maxima of plane-unit i (16-byte loads that leave the
//                lines in L2; red.max into the unit's scratch)
//   quantise(i)  scales from the maxima, then the frames-pass loop of
//                kvf_pack.cu over plane-unit i, re-reading its tokens from L2
//                (evict-first)
//
// Stream k runs plane-units k, k+S, k+2S, ...  The kernel boundary is the only
// synchronisation, as in the two-pass schedule; the other streams' kernels
// fill the gaps a stream leaves between its launches (grid drain, launch
// latency).  At most S plane-units (~20 MB each for a 10,000-token bf16
// chunk) are between their fold and their quantise, so the re-reads hit L2.
#include <algorithm>
#include <mutex>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kMThreads = 256;
constexpr int kMWarps = kMThreads / 32;
constexpr int kMaxStreams = 8;

struct PlaneParams {
  PackUnitDev u;
  int32_t p;  // plane (layer of the triplet)
};

template <int SRC, int VPL>
__global__ void __launch_bounds__(kMThreads) fold_plane_kernel(const __grid_constant__ PlaneParams P) {
  __shared__ uint32_t s_max[64];
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  const PackUnitDev& U = P.u;
  const char* layer = reinterpret_cast<const char*>(U.src.layer[P.p]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < U.G; k += kMThreads) s_max[k] = 0u;
  __syncthreads();
  const int T = U.g.T, nb = gridDim.x, b = blockIdx.x;
  const int t0 = (int)((int64_t)T * b / nb), t1 = (int)((int64_t)T * (b + 1) / nb);
  int32_t off[VPL];
  uint32_t m[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    off[k] = (int32_t)slot_channel_offset(U.g, (lane + 32 * k) * 8, U.src.head_stride) * ES;
    m[k] = 0u;
  }
#pragma unroll 2
  for (int i = t0 + warp; i < t1; i += kMWarps) {
    const char* slot = layer + paged_slot_offset_fd(U.src, U.div_bs, i) * ES;
#pragma unroll
    for (int k = 0; k < VPL; ++k) m[k] = max(m[k], vec_absmax_bits<SRC, KeepLoad>(slot + off[k]));
  }
  reduce_groups<SRC, VPL>(m, U.g.group_size, s_max);
  __syncthreads();
  for (int k = threadIdx.x; k < U.G; k += kMThreads)
    if (s_max[k]) atomicMax(&U.absmax[P.p * U.G + k], s_max[k]);
}

// Quantise and place plane P.p of P.u; a pad plane (null layer) writes 128s.
template <int SRC, int VPL>
__global__ void __launch_bounds__(kMThreads) quant_plane_kernel(const __grid_constant__ PlaneParams P) {
  __shared__ float s_sc[64];
  const PackUnitDev& U = P.u;
  const int p = P.p;
  const int warp = threadIdx.x >> 5, nb = gridDim.x, b = blockIdx.x;
  const bool real = U.src.layer[p] != nullptr;
  for (int k = threadIdx.x; k < U.G; k += kMThreads) {
    const uint32_t bits = real ? U.absmax[p * U.G + k] : 0u;
    const float sc = scale_from_absmax_bits(bits);  // fk/kvmodel.py:139-140
    s_sc[k] = sc;
    if (b == 0) U.scales[p * U.G + k] = sc;
  }
  __syncthreads();
  constexpr int SUB = pack_sub<SRC, VPL>();
  const int n = U.n_items;
  const int q0 = (int)((int64_t)n * b / nb), q1 = (int)((int64_t)n * (b + 1) / nb);
  const int item0 = q0 + warp * SUB;
  if (item0 >= q1) return;
  PackLane<SRC, VPL> L;
  L.init(U, p, s_sc);
  const int rounds = (q1 - item0 + kMWarps * SUB - 1) / (kMWarps * SUB);
  pack_items<SRC, VPL, false>(U, p, L, item0, kMWarps * SUB, rounds, q1,
                              WithPolicy{l2_policy_evict_first()});
}

constexpr int kZeroUnits = 256;
struct ZeroParams {
  uint32_t* absmax[kZeroUnits];
  int32_t words[kZeroUnits];
  int32_t n;
};
__global__ void zero_plane_scratch(const __grid_constant__ ZeroParams Z) {
  for (int u = blockIdx.x; u < Z.n; u += gridDim.x)
    for (int k = threadIdx.x; k < Z.words[u]; k += blockDim.x) Z.absmax[u][k] = 0u;
}

template <int SRC, int VPL>
void launch_plane(bool fold, const PlaneParams& P, int grid, cudaStream_t s) {
  if (fold)
    fold_plane_kernel<SRC, VPL><<<grid, kMThreads, 0, s>>>(P);
  else
    quant_plane_kernel<SRC, VPL><<<grid, kMThreads, 0, s>>>(P);
}

template <int SRC>
void launch_plane_v(int vpl, bool fold, const PlaneParams& P, int grid, cudaStream_t s) {
  switch (vpl) {
    case 1: launch_plane<SRC, 1>(fold, P, grid, s); break;
    case 2: launch_plane<SRC, 2>(fold, P, grid, s); break;
    case 4: launch_plane<SRC, 4>(fold, P, grid, s); break;
    case 8: launch_plane<SRC, 8>(fold, P, grid, s); break;
    case 16: launch_plane<SRC, 16>(fold, P, grid, s); break;
  }
}

// Side streams and fork/join events of one device, created on first use and
// kept for the life of the process.
struct SideStreams {
  int device = -1;
  cudaStream_t st[kMaxStreams] = {};
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[kMaxStreams] = {};
};
std::mutex g_side_mu;
SideStreams g_side[64];

kvf_status side_streams(int dev, SideStreams** out) {
  if (dev < 0 || dev >= 64) KVF_FAIL(KVF_EUNSUPPORTED, "device index %d", dev);
  std::lock_guard<std::mutex> lock(g_side_mu);
  SideStreams& S = g_side[dev];
  if (S.device != dev) {
    for (int k = 0; k < kMaxStreams; ++k) {
      KVF_CHECK_CUDA(cudaStreamCreateWithFlags(&S.st[k], cudaStreamNonBlocking));
      KVF_CHECK_CUDA(cudaEventCreateWithFlags(&S.join[k], cudaEventDisableTiming));
    }
    KVF_CHECK_CUDA(cudaEventCreateWithFlags(&S.fork, cudaEventDisableTiming));
    S.device = dev;
  }
  *out = &S;
  return KVF_OK;
}

}  // namespace

// Single-read pack of the quantising units of one (variant = VPL, dtype)
// group.  param: bits 0-3 streams (0: 4), bits 4-7 fold CTAs per SM (0: 2),
// bits 8-11 quantise CTAs per SM (0: 2).  *launched = false when the shapes
// do not allow it (the caller then runs the phase-split kernels).
kvf_status launch_pack_multi(const std::vector<kvf_pack_unit>& units, int vpl, int32_t dtype,
                             int64_t param, cudaStream_t s, bool* launched) {
  *launched = false;
  if (units.empty() || dtype == KVF_I8) return KVF_OK;
  if (vpl != 1 && vpl != 2 && vpl != 4 && vpl != 8 && vpl != 16) return KVF_OK;
  for (const auto& u : units)
    if (u.plan.H * u.plan.D / u.plan.group_size > 64) return KVF_OK;  // s_max / s_sc
  int dev = 0, sms = 0;
  KVF_CHECK_CUDA(cudaGetDevice(&dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SideStreams* S = nullptr;
  kvf_status st = side_streams(dev, &S);
  if (st != KVF_OK) return st;
  const int n_st = std::min(kMaxStreams, (int)(param & 0xF) ? (int)(param & 0xF) : 4);
  const int fold_grid = sms * ((param >> 4) & 0xF ? (int)((param >> 4) & 0xF) : 2);
  const int quant_grid = sms * ((param >> 8) & 0xF ? (int)((param >> 8) & 0xF) : 2);
  for (size_t at = 0; at < units.size(); at += kZeroUnits) {
    ZeroParams Z;
    Z.n = (int32_t)std::min<size_t>(kZeroUnits, units.size() - at);
    for (int k = 0; k < Z.n; ++k) {
      const kvf_pack_unit& u = units[at + k];
      Z.absmax[k] = u.absmax;
      Z.words[k] = 3 * u.plan.H * u.plan.D / u.plan.group_size;
    }
    zero_plane_scratch<<<std::min(Z.n, 64), 128, 0, s>>>(Z);
  }
  KVF_CHECK_CUDA(cudaGetLastError());
  KVF_CHECK_CUDA(cudaEventRecord(S->fork, s));
  for (int k = 0; k < n_st; ++k) KVF_CHECK_CUDA(cudaStreamWaitEvent(S->st[k], S->fork, 0));
  const int n_pu = (int)(3 * units.size());
  PlaneParams P;
  for (int i = 0; i < n_pu; ++i) {
    P.u = make_pack_unit_dev(units[i / 3]);
    P.p = i % 3;
    cudaStream_t ss = S->st[i % n_st];
    const bool real = P.u.src.layer[P.p] != nullptr;
    for (int fold = real ? 1 : 0; fold >= 0; --fold) {
      if ((param >> 12) & (fold ? 2 : 1)) continue;  // timing probes: bit 12 no quantise, bit 13 no fold
      const int grid = fold ? fold_grid : quant_grid;
      switch (dtype) {
        case KVF_BF16: launch_plane_v<KVF_BF16>(vpl, fold, P, grid, ss); break;
        case KVF_F16: launch_plane_v<KVF_F16>(vpl, fold, P, grid, ss); break;
        case KVF_F32: launch_plane_v<KVF_F32>(vpl, fold, P, grid, ss); break;
      }
    }
  }
  KVF_CHECK_CUDA(cudaGetLastError());
  for (int k = 0; k < n_st; ++k) {
    KVF_CHECK_CUDA(cudaEventRecord(S->join[k], S->st[k]));
    KVF_CHECK_CUDA(cudaStreamWaitEvent(s, S->join[k], 0));
  }
  *launched = true;
  return KVF_OK;
}

}  // namespace kvf
