// kvf_pack_stream.cu — single-HBM-read pack on sm_100a: thread-block clusters
// own whole sub-units, TMA tensor-map loads stream the source through shared
// memory, the all-token maxima are exchanged through distributed shared memory,
// and the quantising pass re-reads the tokens from L2.
//
// The reference scale of a (unit, plane, group) SUB-UNIT is the max |x| over
// ALL chunk tokens (fk/kvmodel.py:138-140), so no sample of it can be quantised
// (:141-143) and placed (fk/layout.py:234-258) before the whole group has been
// read.  The phase-split kernels (kvf_pack.cu) read the source twice from HBM
// (5 B/elem against 3 algorithmic).  Here HBM sees each source byte once:
//
//   * An ITEM is IT tokens x group_size channels (8 KB) of one sub-unit.  A
//     cluster of NC CTAs (8 or 16, one per SM) owns a sub-unit at a time (cluster c
//     takes sub-units c, c + clusters, ...); CTA r of the cluster takes items
//     [n*r/NC, n*(r+1)/NC) of it.
//   * fold producer (one thread): TMA box copy of each item from the layer's
//     4-D tensor map {D, H, block_size, blocks} (a paged block through the
//     block table, or IT rows of a contiguous cache) into ring A.
//   * fold warps: max |x| of the item's chunk tokens (packed u16 maxima).
//   * publisher: when the CTA's items of a sub-unit are folded, its maximum
//     goes to every CTA of the cluster (st.shared::cluster + a remote mbarrier
//     arrive with release semantics): no global memory, no grid-wide sync.
//   * quantise producer: waits for the NC maxima of the sub-unit, derives the
//     scale, and re-reads each item with TMA into ring Q (an L2 hit: the fold
//     pass read it microseconds before; the fold pass runs at most one
//     sub-unit ahead, ~2 sub-units x 2.56 MB per cluster in L2).
//   * quantise warps: FFMA2 quantiser with the exact near-tie redo, tile
//     placement, 16-byte frame stores.
//
// HBM traffic is the algorithmic 2 B read + 1 B written per element.  No
// cross-cluster dependency exists, so the launch needs no co-residency.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kSlotBytes = 16384;
constexpr int kRingA = 8;   // fold ring: TMA loads in flight + folds
constexpr int kLagSU = 1;   // fold pass at most this many sub-units ahead of the re-reads
constexpr int kXSlots = 8;  // maxima exchange slots (sub-units in flight per cluster)
constexpr int kMaxNC = 16;  // CTAs per cluster (16: non-portable, opt-in)
constexpr int kMaxMaps = 72;
constexpr int kMaxSU = 80;  // units per launch (kernel parameters <= 32 KB)
constexpr int kNA = 4;      // fold warps
constexpr int kNQ = 10;     // quantise warps
constexpr int kWarpsS = 2 + kNA + kNQ;  // + fold producer, publisher
// A ring slot is always consumed by the same fold warp, so every mbarrier
// phase is waited for in order (a parity wait can not alias a phase two
// completions ahead).
static_assert(kRingA % kNA == 0, "ring slots per fold warp");

struct StreamUnit {
  uint8_t* fr_base;
  int64_t frame_stride, plane_stride, row_pitch;
  float* scales;
  uint32_t* absmax;  // [3, G] maxima (output copy)
  const int32_t* table;
  int32_t bs, base, T;
  int32_t it0;       // first item's absolute token / IT
  int32_t n_it;      // items per sub-unit
  int32_t G, lg_G, lg_gs;
  int32_t planes;    // real planes, 2 bits each (rank order)
  int32_t n_real;
  int16_t map[3];    // tensor map of each plane, -1: pad layer
  int16_t lg_D, lg_bh, lg_bd, a_d;
  int32_t F, tpf, cols, tile_h, tile_w, n_slots, frame_count;
  FastDiv div_F, div_tpf, div_cols, div_bs;
  const char* layer[3];       // source layers (quantise-pass re-reads)
  int64_t slot_b, block_b;    // source byte strides
  int32_t head_b;             // source head stride in bytes
  int32_t pad_;
};

struct __align__(64) StreamParams {
  CUtensorMap maps[kMaxMaps];
  int32_t n_units, n_sub;
  int32_t probe;                  // measurement probes: bit 0 = no quantise pass
  int32_t sub_first[kMaxSU + 1];  // first sub-unit of each unit
  StreamUnit u[kMaxSU];
};
static_assert(sizeof(StreamParams) <= 32700, "kernel parameters above 32 KB");
static_assert(sizeof(StreamUnit) % 4 == 0, "unit table copy");
constexpr int kStreamSmem = kRingA * kSlotBytes + kMaxSU * sizeof(StreamUnit) + (kMaxSU + 1) * 4;

// Stage trace (tools/trace_stream.py builds a -DKVF_TRACE library): globaltimer
// per (CTA, local item < 4096, event).
#ifdef KVF_TRACE
__device__ unsigned long long* g_trace;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(k, e)                                                                   \
  do {                                                                                \
    if (g_trace && (k) < 4096) g_trace[((size_t)blockIdx.x * 4096 + (k)) * 8 + (e)] = gtime(); \
  } while (0)
#else
#define TRACE(k, e) \
  do {              \
  } while (0)
#endif

// ---- PTX helpers -----------------------------------------------------------
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// Wait (acquire, cluster scope): the phase's arrivals came from other CTAs.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
// st.shared::cluster of v into CTA `rank`'s copy of *p, then a release arrive
// on its copy of *bar (orders the store before the arrive).
__device__ __forceinline__ void publish_remote(const uint32_t* p, uint64_t* bar, uint32_t rank,
                                               uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa(p, rank)), "r"(v) : "memory");
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(bar, rank))
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_idx() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint32_t vmax2_u16(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// The unit table, copied to shared memory at kernel start (dynamically indexed
// kernel-parameter loads go through the small constant cache and miss).
struct Tab {
  const StreamUnit* u;
  const int32_t* first;  // sub_first
};
// Sub-unit S of the launch -> unit, plane, group; `hint`: unit of an earlier
// sub-unit of the same (monotone) walk.
struct Loc {
  int u, plane, group, m, sub;  // sub = plane * G + group (scratch word)
};
__device__ __forceinline__ Loc locate_sub(const Tab& P, int S, int& hint) {
  while (P.first[hint + 1] <= S) ++hint;
  const StreamUnit& U = P.u[hint];
  const int s = S - P.first[hint];
  Loc L;
  L.u = hint;
  L.m = 0;
  const int rp = s >> U.lg_G;
  L.group = s & ((1 << U.lg_G) - 1);
  L.plane = (U.planes >> (2 * rp)) & 3;
  L.sub = L.plane * U.G + L.group;
  return L;
}

// Frame bytes of chunk token i's tile in one plane (fk/layout.py:195-201).
__device__ __forceinline__ uint8_t* tile_of(const StreamUnit& U, int plane, int i) {
  const int gi = fdiv(U.div_F, i);
  const int o = i - gi * U.F;
  const int seg = fdiv(U.div_tpf, gi);
  const int slot = gi - seg * U.tpf;
  const int tr = fdiv(U.div_cols, slot);
  const int tc = slot - tr * U.cols;
  return U.fr_base + (int64_t)plane * U.plane_stride + (int64_t)(seg * U.F + o) * U.frame_stride +
         (int64_t)tr * U.tile_h * U.row_pitch + tc * U.tile_w;
}
// Byte offset of channel c inside a tile (fk/layout.py:244-250).
__device__ __forceinline__ int32_t chan_off(const StreamUnit& U, int c) {
  const int h = c >> U.lg_D, d = c & ((1 << U.lg_D) - 1);
  const int i_h = h >> U.lg_bh, j_h = h & ((1 << U.lg_bh) - 1);
  const int i_d = d >> U.lg_bd, j_d = d & ((1 << U.lg_bd) - 1);
  return (int32_t)((i_h * U.a_d + i_d) * U.row_pitch + (j_h << U.lg_bd) + j_d);
}

// Pad tiles (tokens >= T of a real plane; every tile of a pad plane) and pad
// planes' scales: bytes 128 (fk/layout.py:231, 251-253), scale 1.0
// (fk/kvmodel.py:56-69, 140).  Spread over every warp of the grid.
__device__ __noinline__ void write_pads(const StreamParams& P) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarpsS + warp, nw = gridDim.x * kWarpsS;
  const uint2 pad = make_uint2(0x80808080u, 0x80808080u);
  for (int k = 0; k < P.n_units; ++k) {
    const StreamUnit& U = P.u[k];
    const int per_seg = U.F * U.tpf;
    for (int p = 0; p < 3; ++p) {
      const bool pad_plane = U.map[p] < 0;
      if (pad_plane && blockIdx.x == 0)
        for (int e = threadIdx.x; e < U.G; e += blockDim.x) {
          U.scales[p * U.G + e] = 1.0f;
          U.absmax[p * U.G + e] = 0u;
        }
      const int q0 = pad_plane ? 0 : (U.T / per_seg) * per_seg;
      uint8_t* plane = U.fr_base + (int64_t)p * U.plane_stride;
      // one warp per pad tile: tile_h rows of tile_w bytes (8-byte pieces)
      const int pieces = U.tile_w >> 3;
      for (int q = q0 + gw; q < U.n_slots; q += nw) {
        const int f = fdiv(U.div_tpf, q);
        const int slot = q - f * U.tpf;
        const int seg = fdiv(U.div_F, f);
        const int o = f - seg * U.F;
        if (!pad_plane && (seg * U.tpf + slot) * U.F + o < U.T) continue;
        const int tr = fdiv(U.div_cols, slot);
        const int tc = slot - tr * U.cols;
        uint8_t* t = plane + (int64_t)f * U.frame_stride + (int64_t)tr * U.tile_h * U.row_pitch +
                     tc * U.tile_w;
        for (int e = lane; e < U.tile_h * pieces; e += 32) {
          const int r = e / pieces, c = e - r * pieces;
          st_v2(t + (int64_t)r * U.row_pitch + c * 8, pad);
        }
      }
    }
  }
}

// Issue the TMA copy(ies) of item m of sub-unit L (IT tokens x gs channels)
// into `dst`, completing on `bar`.
template <int IT, int ROW>
__device__ __forceinline__ void issue_item(const StreamParams& P, const StreamUnit& U,
                                           const Loc& L, int m, char* dst, uint64_t* bar,
                                           uint64_t pol) {
  const CUtensorMap* map = &P.maps[U.map[L.plane]];
  const int c = L.group << U.lg_gs;
  const int c0 = c & ((1 << U.lg_D) - 1), c1 = c >> U.lg_D;
  const int t0 = (U.it0 + m) * IT;
  if (U.table == nullptr && U.bs == 1) {
    mbar_expect_tx(bar, kSlotBytes);
    tma_load_4d(dst, map, c0, c1, 0, t0, bar, pol);
  } else if (U.bs >= IT) {
    const int lb = t0 / U.bs;
    const int blk = U.table ? __ldg(U.table + lb) : lb;
    mbar_expect_tx(bar, kSlotBytes);
    tma_load_4d(dst, map, c0, c1, t0 - lb * U.bs, blk, bar, pol);
  } else {
    // IT / bs whole blocks; only those holding chunk tokens are read
    const int lo = max(t0, U.base), hi = min(t0 + IT, U.base + U.T);
    const int b0 = lo / U.bs, b1 = (hi - 1) / U.bs;
    mbar_expect_tx(bar, (uint32_t)((b1 - b0 + 1) * U.bs * ROW));
    for (int b = b0; b <= b1; ++b) {
      const int blk = U.table ? __ldg(U.table + b) : b;
      tma_load_4d(dst + (b * U.bs - t0) * ROW, map, c0, c1, 0, blk, bar, pol);
    }
  }
}

// Exact quantisation of one 8-value vector (near-ties), out of line.
template <int SRC>
__device__ __noinline__ uint2 redo_raw(Raw8<SRC> r, float sc, float inv) {
  float x[8];
  raw8_to_float<SRC>(r, x);
  return quantize8_exact(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], sc, inv);
}

// The walk every role makes: the cluster's sub-units j = 0, 1, ... (global
// sub-unit cid + j * clusters) and, inside each, this CTA's items
// [m0, m1); k counts the CTA's items (ring slots).
#define FOR_SUBUNITS(...)                                                       \
  for (int j = 0, S = cid; S < P.n_sub; ++j, S += ncl) {                        \
    const Loc L = locate_sub(Tb, S, hint);                                      \
    const StreamUnit& U = Tb.u[L.u];                                            \
    const int m0 = (int)(((int64_t)U.n_it * rank) / nc);                        \
    const int m1 = (int)(((int64_t)U.n_it * (rank + 1)) / nc);                  \
    __VA_ARGS__                                                                 \
  }

// SRC: source dtype; GS: group size; CPL: channels per lane per row in the
// quantise warps (16: one 16-byte tile store, needs b_d >= 16; 8: b_d == 8).
// Roles (warps): 0 fold producer, 1 publisher, 2 .. 2+kNA-1 fold, the rest
// quantise (they re-read their items from L2 with 16-byte loads: the TMA unit
// of an SM streams ~40 GB/s of these boxes, enough for one pass, not two).
template <int SRC, int GS, int CPL>
__global__ void __launch_bounds__(kWarpsS * 32, 1)
    pack_stream_kernel(const __grid_constant__ StreamParams P) {
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  constexpr int ROW = GS * ES;            // bytes of one token row of an item
  constexpr int IT = kSlotBytes / ROW;    // tokens per item
  extern __shared__ __align__(128) char s_ring[];  // [ring A | unit table]
  __shared__ __align__(8) uint64_t s_fullA[kRingA], s_emptyA[kRingA], s_fold[kRingA];
  __shared__ __align__(8) uint64_t s_xfull[kXSlots];
  __shared__ uint32_t s_xpart[kXSlots][kMaxNC];  // CTA maxima of a sub-unit
  __shared__ uint32_t s_pmax[kRingA];
  __shared__ volatile int s_qj[kNQ];  // sub-unit each quantise warp is on
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank(), nc = (int)cluster_nctarank();
  const int cid = (int)cluster_idx(), ncl = (int)cluster_count();
  if (threadIdx.x < kRingA) {
    mbar_init(&s_fullA[threadIdx.x], 1);
    mbar_init(&s_emptyA[threadIdx.x], 2);  // fold warp + publisher
    mbar_init(&s_fold[threadIdx.x], 1);
  }
  if (threadIdx.x < kXSlots) mbar_init(&s_xfull[threadIdx.x], nc);
  if (threadIdx.x < kNQ) s_qj[threadIdx.x] = 0;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  char* const ringA = s_ring;
  char* const tab = s_ring + kRingA * kSlotBytes;
  {
    uint32_t* dst = reinterpret_cast<uint32_t*>(tab);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(P.u);
    const int nw = P.n_units * (int)(sizeof(StreamUnit) / 4);
    for (int e = threadIdx.x; e < nw; e += blockDim.x) dst[e] = src[e];
    for (int e = threadIdx.x; e <= P.n_units; e += blockDim.x)
      dst[kMaxSU * (sizeof(StreamUnit) / 4) + e] = P.sub_first[e];
  }
  __syncthreads();
  cluster_sync_all();  // every CTA's exchange barriers exist before any remote arrive
  const Tab Tb{reinterpret_cast<const StreamUnit*>(tab),
               reinterpret_cast<const int32_t*>(tab + kMaxSU * sizeof(StreamUnit))};
  int hint = 0;

  if (warp == 0) {
    // --------------------------------------------------- fold producer (A)
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();  // re-read by the quantise pass
      int k = 0;
      FOR_SUBUNITS({
        // at most kLagSU sub-units ahead of the slowest quantise warp
        for (;;) {
          int mq = s_qj[0];
#pragma unroll
          for (int q = 1; q < kNQ; ++q) mq = min(mq, s_qj[q]);
          if (j <= mq + kLagSU) break;
          __nanosleep(64);
        }
        for (int m = m0; m < m1; ++m, ++k) {
          const int slot = k % kRingA, round = k / kRingA;
          TRACE(k, 0);
          if (round > 0) mbar_wait(&s_emptyA[slot], (round - 1) & 1);
          TRACE(k, 1);
          issue_item<IT, ROW>(P, U, L, m, ringA + slot * kSlotBytes, &s_fullA[slot], pol);
        }
      })
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- publisher
    int k = 0;
    FOR_SUBUNITS({
      uint32_t mx = 0;
      for (int m = m0; m < m1; ++m, ++k) {
        const int slot = k % kRingA;
        mbar_wait(&s_fold[slot], (k / kRingA) & 1);
        mx = max(mx, s_pmax[slot]);
        __syncwarp();
        if (lane == 0) {
          TRACE(k, 3);
          mbar_arrive(&s_emptyA[slot]);
        }
      }
      // The publication of sub-unit j obeys the fold lead too (a CTA without
      // items of a sub-unit would otherwise publish far ahead and overwrite
      // exchange slots other CTAs have not read): every quantise warp of this
      // CTA is on sub-unit >= j - kLagSU, so every CTA has published j - 2 and
      // read its slot j - 8.
      for (;;) {
        int mq = s_qj[0];
#pragma unroll
        for (int q = 1; q < kNQ; ++q) mq = min(mq, s_qj[q]);
        if (j <= mq + kLagSU) break;
        __nanosleep(64);
      }
      // this CTA's maximum of sub-unit j -> every CTA of the cluster
      if (lane < nc) publish_remote(&s_xpart[j % kXSlots][rank], &s_xfull[j % kXSlots], lane, mx);
    })
  } else if (warp < 2 + kNA) {
    // ------------------------------------------------- fold |x| maxima (A)
    constexpr int VPR = GS / 8;  // 8-value vectors per row
    constexpr int RPS = 32 / VPR;
    static_assert(32 % VPR == 0, "group size");
    const int fw = warp - 2;
    int k = 0;
    FOR_SUBUNITS({
      for (int m = m0; m < m1; ++m, ++k) {
        if (k % kNA != fw) continue;
        const int slot = k % kRingA;
        const int t0 = (U.it0 + m) * IT;
        const int r0 = max(0, U.base - t0), r1 = min(IT, U.base + U.T - t0);
        mbar_wait(&s_fullA[slot], (k / kRingA) & 1);
        const char* base = ringA + slot * kSlotBytes + (lane % VPR) * (8 * ES);
        uint32_t mx = 0;
#pragma unroll 4
        for (int st = 0; st < IT / RPS; ++st) {
          const int row = st * RPS + lane / VPR;
          if (row < r0 || row >= r1) continue;
          const char* a = base + row * ROW;
          if constexpr (SRC == KVF_F32) {
            const uint4 x = *reinterpret_cast<const uint4*>(a);
            const uint4 y = *reinterpret_cast<const uint4*>(a + 16);
            mx = max(mx, max(max(x.x & 0x7FFFFFFFu, x.y & 0x7FFFFFFFu),
                             max(x.z & 0x7FFFFFFFu, x.w & 0x7FFFFFFFu)));
            mx = max(mx, max(max(y.x & 0x7FFFFFFFu, y.y & 0x7FFFFFFFu),
                             max(y.z & 0x7FFFFFFFu, y.w & 0x7FFFFFFFu)));
          } else {
            const uint4 x = *reinterpret_cast<const uint4*>(a);
            mx = vmax2_u16(mx, vmax2_u16(vmax2_u16(x.x & 0x7FFF7FFFu, x.y & 0x7FFF7FFFu),
                                         vmax2_u16(x.z & 0x7FFF7FFFu, x.w & 0x7FFF7FFFu)));
          }
        }
        if constexpr (SRC != KVF_F32) mx = absmax_to_f32_bits<SRC>(max(mx >> 16, mx & 0xFFFFu));
        mx = __reduce_max_sync(0xffffffffu, mx);
        __syncwarp();
        if (lane == 0) {
          s_pmax[slot] = mx;
          TRACE(k, 2);
          mbar_arrive(&s_fold[slot]);
          mbar_arrive(&s_emptyA[slot]);
        }
      }
    })
  } else if (!(P.probe & 1)) {
    // ------------------------------------------------------- quantise (Q)
    // Per sub-unit: wait for the cluster's NC maxima, scale (fk/kvmodel.py:
    // 139-140); per item: 16-byte re-reads of the item's rows from L2 (QB rows
    // per lane in flight), FFMA2 quantiser with the exact near-tie redo
    // (fk/kvmodel.py:141-143), tile placement (fk/layout.py:244-258).
    constexpr int LPR = GS / CPL;  // lanes per row
    constexpr int RPS = 32 / LPR;  // rows per step
    constexpr int NV = CPL / 8;    // 8-value vectors per lane per row
    constexpr int STEPS = IT / RPS;
    constexpr int QB = STEPS >= 4 ? 4 : STEPS;  // rows of a lane in flight
    static_assert(32 % LPR == 0 && STEPS % QB == 0, "group size");
    constexpr int VB = SRC == KVF_F32 ? 32 : 16;  // source bytes of an 8-value vector
    const int qw = warp - 2 - kNA;
    const int lr = lane / LPR, lc = lane % LPR;
    const uint64_t pol = l2_policy_evict_first();
    int k = 0;
    FOR_SUBUNITS({
      if (lane == 0) s_qj[qw] = j;
      mbar_wait_cluster(&s_xfull[j % kXSlots], (j / kXSlots) & 1);
      const uint32_t mb = __reduce_max_sync(0xffffffffu, lane < nc ? s_xpart[j % kXSlots][lane] : 0u);
      const float sc = scale_from_absmax_bits(mb);
      const float inv = __frcp_rn(sc);
      if (rank == 0 && qw == 0 && lane == 0) {
        U.scales[L.sub] = sc;
        U.absmax[L.sub] = mb;
      }
      const int c = (L.group << U.lg_gs) + lc * CPL;
      const int32_t toff = chan_off(U, c);  // the lane's CPL channels are contiguous
      const char* layer = U.layer[L.plane] + (c >> U.lg_D) * U.head_b + (c & ((1 << U.lg_D) - 1)) * ES;
      for (int m = m0; m < m1; ++m, ++k) {
        if (k % kNQ != qw) continue;
        const int t0 = (U.it0 + m) * IT;
        const int r0 = max(0, U.base - t0), r1 = min(IT, U.base + U.T - t0);
#pragma unroll 1
        for (int s0 = 0; s0 < STEPS; s0 += QB) {
          Raw8<SRC> raw[QB][NV];
#pragma unroll
          for (int u = 0; u < QB; ++u) {
            const int row = (s0 + u) * RPS + lr;
            const int t = min(max(t0 + row, U.base), U.base + U.T - 1);  // clamp: stay in bounds
            const int blk = fdiv(U.div_bs, t);
            const int in = t - blk * U.bs;
            const int64_t pb = U.table ? (int64_t)__ldg(U.table + blk) : (int64_t)blk;
            const char* a = layer + pb * U.block_b + (int64_t)in * U.slot_b;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              raw[u][v].a = ld_nc_v4_pol(a + v * VB, pol);
              if constexpr (SRC == KVF_F32) raw[u][v].b = ld_nc_v4_pol(a + v * VB + 16, pol);
            }
          }
#pragma unroll
          for (int u = 0; u < QB; ++u) {
            const int row = (s0 + u) * RPS + lr;
            uint2 out[NV];
            uint32_t badm = 0;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              float x[8];
              bool bad = false;
              raw8_to_float<SRC>(raw[u][v], x);
              out[v] = quantize8_fast<false>(x, inv, bad);
              badm |= (uint32_t)bad << v;
            }
            if (__builtin_expect(badm != 0, 0)) {
#pragma unroll
              for (int v = 0; v < NV; ++v)
                if ((badm >> v) & 1) out[v] = redo_raw<SRC>(raw[u][v], sc, inv);
            }
            if (row < r0 || row >= r1) continue;
            uint8_t* d = tile_of(U, L.plane, t0 + row - U.base) + toff;
            if constexpr (CPL == 16) {
              st_v4(d, make_uint4(out[0].x, out[0].y, out[1].x, out[1].y));
            } else {
              st_v2(d, out[0]);
            }
          }
        }
        if (lane == 0) TRACE(k, 6);
      }
    })
    if (lane == 0) s_qj[qw] = 1 << 30;
  }
  if (warp >= 2 + kNA && (P.probe & 1) && lane == 0) s_qj[warp - 2 - kNA] = 1 << 30;
  write_pads(P);
  cluster_sync_all();  // no CTA exits while a remote arrive may still target it
}

template <int SRC, int GS>
const void* kernel_for(bool bd16) {
  return bd16 ? (const void*)pack_stream_kernel<SRC, GS, 16>
              : (const void*)pack_stream_kernel<SRC, GS, 8>;
}
template <int SRC>
const void* kernel_for(int gs, bool bd16) {
  switch (gs) {
    case 64: return kernel_for<SRC, 64>(bd16);
    case 128: return kernel_for<SRC, 128>(bd16);
    case 256: return kernel_for<SRC, 256>(bd16);
    default: return nullptr;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;  // a driver symbol, resolved once
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Units sharing a tensor map: same layer pointer and source geometry.
bool same_src(const kvf_pack_unit& a, const kvf_pack_unit& b) {
  return a.src.block_table == b.src.block_table && a.src.block_size == b.src.block_size &&
         a.src.block_stride == b.src.block_stride && a.src.slot_stride == b.src.slot_stride &&
         a.src.head_stride == b.src.head_stride && a.src.dtype == b.src.dtype &&
         a.plan.H == b.plan.H && a.plan.D == b.plan.D;
}

int64_t layer_extent(const std::vector<kvf_pack_unit>& units, const kvf_pack_unit& ref,
                     const void* layer) {
  int64_t e = 0;
  for (const auto& u : units)
    for (int p = 0; p < 3; ++p)
      if (u.src.layer[p] == layer && same_src(u, ref))
        e = std::max<int64_t>(e, (int64_t)u.src.token_base + u.plan.T);
  return e;
}

// The layer's tensor map {D, H, block_size, blocks}; box = one item (IT tokens
// x gs channels) or, for block_size < IT, one block.
CUresult encode_map(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* map,
                    const kvf_pack_unit& u, void* layer, int gs, int es, int it,
                    int64_t extent) {
  const kvf_plan& pl = u.plan;
  const kvf_paged& src = u.src;
  const bool contig = src.block_table == nullptr && src.block_size == 1;
  cuuint64_t gdim[4] = {(cuuint64_t)pl.D, (cuuint64_t)pl.H, (cuuint64_t)src.block_size,
                        contig ? (cuuint64_t)extent : (cuuint64_t)0x7FFFFFFF};
  cuuint64_t gstr[3] = {(cuuint64_t)(src.head_stride * es), (cuuint64_t)(src.slot_stride * es),
                        (cuuint64_t)(src.block_stride * es)};
  cuuint32_t box[4] = {(cuuint32_t)std::min(gs, pl.D), (cuuint32_t)std::max(1, gs / pl.D),
                       contig ? 1u : (cuuint32_t)std::min(src.block_size, it),
                       contig ? (cuuint32_t)it : 1u};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
             layer, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// Can this unit take the stream schedule (given the item size IT)?
bool unit_ok(PFN_cuTensorMapEncodeTiled_v12000 enc, const kvf_pack_unit& u, int gs, int es,
             int it) {
  const kvf_plan& p = u.plan;
  if (p.group_size != gs || p.b_d < 8 || gs % 8) return false;
  if (gs < p.D ? p.D % gs : gs % p.D) return false;
  const kvf_paged& s = u.src;
  for (int l = 0; l < 3; ++l)
    if (s.layer[l] && reinterpret_cast<uintptr_t>(s.layer[l]) % 16) return false;
  if ((s.head_stride * es) % 16 || (s.slot_stride * es) % 16 || (s.block_stride * es) % 16)
    return false;
  if (s.head_stride * es >= (int64_t(1) << 40) || s.slot_stride * es >= (int64_t(1) << 40) ||
      s.block_stride * es >= (int64_t(1) << 40))
    return false;
  const bool contig = s.block_table == nullptr && s.block_size == 1;
  if (!contig && !(s.block_size >= it ? s.block_size % it == 0 : it % s.block_size == 0))
    return false;
  if (!contig && s.block_size > 256) return false;
  if (reinterpret_cast<uintptr_t>(u.frames.base) % 8 || u.frames.frame_stride % 8 ||
      u.frames.plane_stride % 8 || u.frames.row_pitch % 8)
    return false;
  if (p.b_d >= 16 && (reinterpret_cast<uintptr_t>(u.frames.base) % 16 ||
                      u.frames.frame_stride % 16 || u.frames.plane_stride % 16 ||
                      u.frames.row_pitch % 16))
    return false;
  // the driver accepts the layer's tensor map (strides, box)
  for (int l = 0; l < 3; ++l) {
    if (!s.layer[l]) continue;
    CUtensorMap m;
    if (encode_map(enc, &m, u, s.layer[l], gs, es, it, (int64_t)s.token_base + p.T) !=
        CUDA_SUCCESS)
      return false;
  }
  return true;
}

}  // namespace

#ifdef KVF_TRACE
extern "C" int kvf_trace_set(void* p) { return (int)cudaMemcpyToSymbol(g_trace, &p, sizeof(p)); }
#endif

// Single-read pack of quantising units on thread-block clusters.  Units this
// schedule cannot take (int8 sources, group sizes other than 64/128/256,
// b_d < 8, strides the tensor maps reject) are appended to *rest for the
// phase-split kernels.  `cluster`: CTAs per cluster (8 or 16; 0 = 8, the
// faster on C2: 15 clusters cover 120 SMs against 7 x 16 = 112).
kvf_status launch_pack_stream(const std::vector<kvf_pack_unit>& units, int32_t dtype,
                              int cluster, int probe, cudaStream_t s,
                              std::vector<kvf_pack_unit>* rest) {
  if (units.empty()) return KVF_OK;
  if (dtype == KVF_I8) {
    rest->insert(rest->end(), units.begin(), units.end());
    return KVF_OK;
  }
  const int es = (int)dtype_size(dtype);
  auto enc = encode_fn();
  if (enc == nullptr) {
    rest->insert(rest->end(), units.begin(), units.end());
    return KVF_OK;
  }
  // group units by (group size, b_d >= 16); others go to the caller
  struct Key {
    int gs;
    bool bd16;
  };
  std::vector<std::pair<Key, std::vector<kvf_pack_unit>>> groups;
  for (const auto& u : units) {
    const int gs = u.plan.group_size;
    const int it = (gs == 64 || gs == 128 || gs == 256) ? kSlotBytes / (gs * es) : 0;
    if (it == 0 || !unit_ok(enc, u, gs, es, it)) {
      rest->push_back(u);
      continue;
    }
    const Key key{gs, u.plan.b_d >= 16};
    auto g = std::find_if(groups.begin(), groups.end(), [&](const auto& e) {
      return e.first.gs == key.gs && e.first.bd16 == key.bd16;
    });
    if (g == groups.end()) {
      groups.push_back({key, {}});
      g = groups.end() - 1;
    }
    g->second.push_back(u);
  }
  for (auto& [key, list] : groups) {
    const void* fn = dtype == KVF_BF16  ? kernel_for<KVF_BF16>(key.gs, key.bd16)
                     : dtype == KVF_F16 ? kernel_for<KVF_F16>(key.gs, key.bd16)
                                        : kernel_for<KVF_F32>(key.gs, key.bd16);
    const int smem = kStreamSmem;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess) {
      cudaGetLastError();
      rest->insert(rest->end(), list.begin(), list.end());
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kWarpsS * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0, ncl = 0;
    for (int c : {8, 16}) {
      if (cluster && c != cluster) continue;
      int n = 0;
      attr[0].val.clusterDim.x = c;
      cfg.gridDim = dim3(c * 64);
      if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (n > 0) {
        nc = c;
        ncl = n;
        break;
      }
    }
    if (nc == 0) {
      rest->insert(rest->end(), list.begin(), list.end());
      continue;
    }
    const int it = kSlotBytes / (key.gs * es);
    size_t at = 0;
    while (at < list.size()) {
      StreamParams* P = new StreamParams();
      std::vector<std::pair<const void*, const kvf_pack_unit*>> maps;  // (layer, geometry)
      int n = 0, n_sub = 0;
      while (at + n < list.size() && n < kMaxSU) {
        const kvf_pack_unit& u = list[at + n];
        auto find_map = [&](const void* layer) {
          for (size_t i = 0; i < maps.size(); ++i)
            if (maps[i].first == layer && same_src(*maps[i].second, u)) return (int)i;
          return -1;
        };
        int need = 0;
        for (int p = 0; p < 3; ++p)
          if (u.src.layer[p] && find_map(u.src.layer[p]) < 0) ++need;
        if ((int)maps.size() + need > kMaxMaps) break;
        StreamUnit& D = P->u[n];
        const kvf_plan& pl = u.plan;
        const kvf_paged& src = u.src;
        D.fr_base = u.frames.base;
        D.frame_stride = u.frames.frame_stride;
        D.plane_stride = u.frames.plane_stride;
        D.row_pitch = u.frames.row_pitch;
        D.scales = u.scales;
        D.absmax = u.absmax;
        D.table = src.block_table;
        D.bs = src.block_size;
        D.base = src.token_base;
        D.T = pl.T;
        D.it0 = src.token_base / it;
        D.n_it = (src.token_base + pl.T - 1) / it - D.it0 + 1;
        D.G = pl.H * pl.D / key.gs;
        D.lg_G = ilog2(D.G);
        D.lg_gs = ilog2(key.gs);
        D.planes = 0;
        D.n_real = 0;
        for (int p = 0; p < 3; ++p) {
          if (!src.layer[p]) {
            D.map[p] = -1;
            continue;
          }
          int mi = find_map(src.layer[p]);
          if (mi < 0) {
            mi = (int)maps.size();
            maps.push_back({src.layer[p], &u});
            CUresult r = encode_map(enc, &P->maps[mi], u, src.layer[p], key.gs, es, it,
                                    layer_extent(list, u, src.layer[p]));
            if (r != CUDA_SUCCESS) {  // accepted by unit_ok: not expected
              delete P;
              KVF_FAIL(KVF_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
            }
          }
          D.map[p] = (int16_t)mi;
          D.planes |= p << (2 * D.n_real);
          ++D.n_real;
        }
        D.lg_D = (int16_t)ilog2(pl.D);
        D.lg_bh = (int16_t)ilog2(pl.b_h);
        D.lg_bd = (int16_t)ilog2(pl.b_d);
        D.a_d = (int16_t)pl.a_d;
        D.F = pl.F;
        D.tpf = pl.tiles_per_frame;
        D.cols = pl.grid_cols;
        D.tile_h = pl.a_h * pl.a_d;
        D.tile_w = pl.b_h * pl.b_d;
        D.frame_count = pl.frame_count;
        D.n_slots = pl.frame_count * pl.tiles_per_frame;
        D.div_F = make_fastdiv(pl.F);
        D.div_tpf = make_fastdiv(pl.tiles_per_frame);
        D.div_cols = make_fastdiv(pl.grid_cols);
        D.div_bs = make_fastdiv(src.block_size);
        for (int p = 0; p < 3; ++p) D.layer[p] = reinterpret_cast<const char*>(src.layer[p]);
        D.slot_b = src.slot_stride * es;
        D.block_b = src.block_stride * es;
        D.head_b = (int32_t)(src.head_stride * es);
        P->sub_first[n] = n_sub;
        n_sub += D.n_real * D.G;
        ++n;
      }
      P->sub_first[n] = n_sub;
      P->n_units = n;
      P->n_sub = n_sub;
      P->probe = (int32_t)(probe & 0xFF);
      attr[0].val.clusterDim.x = nc;
      cfg.gridDim = dim3(nc * std::max(1, std::min(ncl, n_sub)));
      void* args[] = {P};
      cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
      delete P;
      if (e != cudaSuccess) return cuda_status(e, "pack_stream_kernel launch");
      at += n;
    }
  }
  return KVF_OK;
}

}  // namespace kvf
