// kvf_pack_cluster.cu — single-HBM-read pack, sm_100a: thread-block clusters
// exchange the quantisation maxima through distributed shared memory.
//
// The reference scale of a (unit, plane, group) is the max |x| over ALL chunk
// tokens (fk/kvmodel.py:138-140), so no sample can be quantised (:141-143) and
// placed (fk/layout.py:234-258) before the whole group has been read.  The
// phase-split kernels (kvf_pack.cu) read the source twice from HBM (5 B/elem
// against 3 algorithmic).
//
// Here a SUB-UNIT is one (unit, plane, group): T tokens x group_size channels
// (10,000 x 128 bf16 = 2.56 MB for a full reference chunk).  One cluster of NC
// CTAs (one per SM) owns a sub-unit at a time, CTA r of the cluster holding
// tokens [T*r/NC, T*(r+1)/NC).  Clusters walk the sub-unit list round-robin
// (persistent grid), and every CTA runs, per step k of its cluster's list:
//
//   A(k+2): read its token share of sub-unit k+2 from HBM, |x| maxima in
//           registers (lines left in L2);
//   B(k):   re-read its share of sub-unit k (read two steps ago: an L2 hit),
//           quantise with the complete maxima, tile, store the frame bytes;
//
// interleaved in one loop so the HBM stream of A never stops while B works.
// At the end of the step the CTA's partial max of sub-unit k+2 goes to every
// CTA of the cluster (st.shared::cluster into slot (k+2)%3) followed by
// barrier.cluster.arrive.release; the matching barrier.cluster.wait.acquire
// runs one step later, so the cluster barrier's latency is hidden behind a
// whole step.  Three slots make the reuse safe: slot (k+2)%3 last held
// sub-unit k-1, read at the start of step k-1 by every CTA before its arrive
// that the wait of step k observes.
//
// HBM traffic is the algorithmic 2 B read + 1 B written per element: the
// re-read is served by L2 (~3 sub-units per cluster in flight, ~55 MB of the
// 126 MB L2 with 7 clusters of 16).
#include <algorithm>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kMaxCWarps = 16;
constexpr int kMaxNC = 16;  // CTAs per cluster (16 = non-portable, opt-in)

struct ClusterParams {
  int32_t n_units;
  int32_t n_sub;                         // sub-units in the launch
  int32_t sub_first[kMaxPackUnits + 1];  // first sub-unit of unit k (3*G per unit)
  PackUnitDev u[kMaxPackUnits];
};
static_assert(sizeof(ClusterParams) <= 32000, "kernel parameters above 32 KB");

// ---- cluster PTX ---------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive (release, cluster scope) on CTA `rank`'s copy of the mbarrier at `bar`.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(remote)
               : "r"(smem_addr(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
// Wait (acquire, cluster scope) for the phase of parity `parity` of a local mbarrier.
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
// Store a word into CTA `rank`'s copy of the shared variable at `p`.
__device__ __forceinline__ void st_cluster_u32(const void* p, uint32_t rank, uint32_t v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(remote)
               : "r"(smem_addr(p)), "r"(rank));
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(v) : "memory");
}

// max of three packed u16 pairs, per half
__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  asm("max.u16x2 %0, %0, %1;" : "+r"(r) : "r"(c));
  return r;
}

// Which (unit, plane, group) sub-unit s is.  `u` is a hint: the unit of an
// earlier sub-unit of the same walk (the walk only moves forward).
struct Sub {
  int unit, plane, group;
};
__device__ __forceinline__ Sub sub_of(const ClusterParams& P, int s, int& u) {
  while (u + 1 < P.n_units && P.sub_first[u + 1] <= s) ++u;
  const int local = s - P.sub_first[u];
  const int lg_G = P.u[u].g.lg_C - P.u[u].g.lg_gs;  // G = C / gs, both powers of two
  return Sub{u, local >> lg_G, local & ((1 << lg_G) - 1)};
}

// Where a sub-unit's source tokens are: the paged-slot offset of chunk token i
// (fk/kvmodel.py:223-225 page/slot, as a block table), held in registers.
struct SrcView {
  const char* layer;  // plane p's layer, null: pad layer (zeros)
  const int32_t* table;
  int64_t slot_b, block_b;  // byte strides
  FastDiv bs;
  int32_t base;             // token_base
  __device__ __forceinline__ void init(const PackUnitDev& U, int p, int es) {
    layer = reinterpret_cast<const char*>(U.src.layer[p]);
    table = U.src.block_table;
    slot_b = U.src.slot_stride * es;
    block_b = U.src.block_stride * es;
    bs = U.div_bs;
    base = U.src.token_base;
  }
  __device__ __forceinline__ const char* at(int i) const {
    const int t = base + i;
    if (table == nullptr && bs.d == 1) return layer + (int64_t)t * slot_b;
    const int blk = fdiv(bs, t);
    const int in = t - blk * bs.d;
    const int64_t b = table ? (int64_t)__ldg(table + blk) : (int64_t)blk;
    return layer + b * block_b + (int64_t)in * slot_b;
  }
};

// Where chunk token i's tile lies in one plane (fk/layout.py:195-201).
struct DstView {
  uint8_t* plane;
  int64_t frame_b, row_b;  // frame stride, tile-row stride (tile_h * pitch) in bytes
  FastDiv F, tpf, cols;
  int32_t tile_w;
  __device__ __forceinline__ void init(const PackUnitDev& U, int p) {
    plane = U.fr.base + (int64_t)p * U.fr.plane_stride;
    frame_b = U.fr.frame_stride;
    row_b = (int64_t)U.g.tile_h * U.fr.row_pitch;
    F = U.g.div_F;
    tpf = U.g.div_tpf;
    cols = U.g.div_cols;
    tile_w = U.g.tile_w;
  }
  __device__ __forceinline__ uint8_t* item(int f, int slot) const {
    const int tr = fdiv(cols, slot);
    const int tc = slot - tr * cols.d;
    return plane + (int64_t)f * frame_b + (int64_t)tr * row_b + tc * tile_w;
  }
  __device__ __forceinline__ uint8_t* at(int i) const {
    const int gi = fdiv(F, i);
    const int o = i - gi * F.d;
    const int seg = fdiv(tpf, gi);
    const int slot = gi - seg * tpf.d;
    return item(seg * F.d + o, slot);
  }
};

// This CTA's token share of a sub-unit and the lane's channel offsets.
template <int SRC, int LPT, int VPT, int NW>
struct Share {
  static constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  static constexpr int TPW = 32 / LPT;        // tokens per warp step
  static constexpr int TPS = TPW * NW;        // tokens per CTA step
  int unit, plane, group;
  int tok0, tok1;
  int32_t in_off[VPT];
  bool valid;
  __device__ __forceinline__ void init(const ClusterParams& P, int s, int rank, int lg_nc,
                                       int& hint) {
    valid = s < P.n_sub;
    tok0 = tok1 = 0;
    unit = plane = group = 0;
    if (!valid) return;
    const Sub q = sub_of(P, s, hint);
    unit = q.unit;
    plane = q.plane;
    group = q.group;
    const PackUnitDev& U = P.u[q.unit];
    const int T = U.g.T;
    tok0 = (T * rank) >> lg_nc;  // T < 2^26 (checked on the host)
    tok1 = (T * (rank + 1)) >> lg_nc;
    const int sl = (threadIdx.x & 31) % LPT;
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c = q.group * U.g.group_size + (v * LPT + sl) * 8;
      in_off[v] = (int32_t)(slot_channel_offset(U.g, c, U.src.head_stride) * ES);
    }
  }
  // the lane's token at CTA step `st` (>= tok1: none)
  __device__ __forceinline__ int token(int st) const {
    return tok0 + st * TPS + (threadIdx.x >> 5) * TPW + (threadIdx.x & 31) / LPT;
  }
  __device__ __forceinline__ int steps() const { return (tok1 - tok0 + TPS - 1) / TPS; }
};

// 8 frame bytes of one vector -> the tile: one 8-byte store when b_d >= 8,
// else 8/b_d pieces of b_d bytes in consecutive tile rows (fk/layout.py:244-250).
__device__ __forceinline__ void store_vec(uint8_t* p, uint2 v, int lg_bd, int64_t pitch) {
  if (lg_bd >= 3) {
    st_v2(p, v);
    return;
  }
  const uint64_t w = ((uint64_t)v.y << 32) | v.x;
  const int bd = 1 << lg_bd;
  for (int j = 0; j < 8 / bd; ++j) {
    const uint64_t piece = w >> (8 * bd * j);
    uint8_t* q = p + j * pitch;
    if (bd == 4) *reinterpret_cast<uint32_t*>(q) = (uint32_t)piece;
    else if (bd == 2) *reinterpret_cast<uint16_t*>(q) = (uint16_t)piece;
    else *q = (uint8_t)piece;
  }
}

// Pad tiles of the sub-unit's last segment (tokens >= T) and, for a pad layer,
// every tile: the group's bytes are 128 (fk/layout.py:231, 251-253).
template <int LPT, int VPT, int NW>
__device__ __noinline__ void write_pads(const ClusterParams& P, int unit, int plane, int group,
                                        bool pad_layer, int rank, int nc) {
  const PackUnitDev& U = P.u[unit];
  const Geom& g = U.g;
  DstView D;
  D.init(U, plane);
  const int per_seg = g.F * g.tpf;
  const int q0 = pad_layer ? 0 : (g.T / per_seg) * per_seg;  // first item that can be a pad
  constexpr int TPW = 32 / LPT;
  const int sl = (threadIdx.x & 31) % LPT;
  int32_t tile_off[VPT];
#pragma unroll
  for (int v = 0; v < VPT; ++v)
    tile_off[v] = (int32_t)tile_offset(g, group * g.group_size + (v * LPT + sl) * 8,
                                       U.fr.row_pitch);
  const uint2 pad = make_uint2(0x80808080u, 0x80808080u);
  for (int q = q0 + (rank * NW + (threadIdx.x >> 5)) * TPW + (threadIdx.x & 31) / LPT;
       q < U.n_items; q += nc * NW * TPW) {
    const int f = fdiv(g.div_tpf, q);
    const int slot = q - f * g.tpf;
    if (!pad_layer && token_of(g, f, slot) < g.T) continue;
    uint8_t* d = D.item(f, slot);
#pragma unroll
    for (int v = 0; v < VPT; ++v) store_vec(d + tile_off[v], pad, g.lg_bd, U.fr.row_pitch);
  }
}

// ---- per-thread async copies (cp.async, 16 B) into the warp's stage ring ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_addr(p)));
  return v;
}


// Bytes of one lane's vectors of one phase in a stage: VPT x 8 values.
template <int SRC, int VPT>
__host__ __device__ constexpr int lane_bytes() { return VPT * 8 * (SRC == KVF_F32 ? 4 : 2); }
template <int SRC, int VPT>
__host__ __device__ constexpr int stage_bytes() { return 2 * 32 * lane_bytes<SRC, VPT>(); }
// NW warps per CTA, NS stages per warp ring (NS - 1 steps in flight)
template <int SRC, int VPT, int NW, int NS>
__host__ __device__ constexpr int cluster_smem_bytes() {
  return NW * NS * stage_bytes<SRC, VPT>();
}

// One phase's walk state: the sub-unit share, where its tokens are, the step count.
template <int SRC, int LPT, int VPT, int NW>
struct Walk {
  Share<SRC, LPT, VPT, NW> sh;
  SrcView src;
  int n;  // CTA steps (0: nothing to read: invalid or pad layer)
  __device__ __forceinline__ void init(const ClusterParams& P, int s, int rank, int lg_nc,
                                       int& hint) {
    sh.init(P, s, rank, lg_nc, hint);
    src.init(P.u[sh.unit], sh.plane, Share<SRC, LPT, VPT, NW>::ES);
    n = (sh.valid && src.layer != nullptr) ? sh.steps() : 0;
  }
  // Copy the lane's vectors of step j (token clamped into the share) to `dst`
  // (layout [VPT][32 lanes] of 16-B pieces, bank-conflict free).
  __device__ __forceinline__ void issue(int j, char* dst) const {
    const char* p = src.at(min(sh.token(j), sh.tok1 - 1));
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      cp_async16(dst + (v * (SRC == KVF_F32 ? 2 : 1) * 32 + lane) * 16, p + sh.in_off[v]);
      if constexpr (SRC == KVF_F32)
        cp_async16(dst + ((2 * v + 1) * 32 + lane) * 16, p + sh.in_off[v] + 16);
    }
  }
};

template <int SRC, int VPT>
__device__ __forceinline__ Raw8<SRC> stage_vec(const char* base, int v) {
  const int lane = threadIdx.x & 31;
  Raw8<SRC> r;
  if constexpr (SRC == KVF_F32) {
    r.a = lds128(base + ((2 * v) * 32 + lane) * 16);
    r.b = lds128(base + ((2 * v + 1) * 32 + lane) * 16);
  } else {
    r.a = lds128(base + (v * 32 + lane) * 16);
  }
  return r;
}

template <int SRC, int LPT, int VPT, bool BD8, int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 1)
    pack_cluster_kernel(const __grid_constant__ ClusterParams P) {
  extern __shared__ __align__(16) char s_ring[];  // [warps][stages][A | B] lane vectors
  // Partial maxima (f32 bits) of every (CTA, warp) of the cluster, 4 slots by
  // sub-unit; s_full[slot] completes a phase when all nc * NW warps published.
  __shared__ uint32_t s_part[4][kMaxNC * NW];
  __shared__ __align__(8) uint64_t s_full[4];
  using W = Walk<SRC, LPT, VPT, NW>;
  constexpr int LB = 32 * lane_bytes<SRC, VPT>();  // one phase of a stage
  const int rank = (int)cluster_rank(), nc = (int)cluster_size();
  const int lg_nc = 31 - __clz(nc);  // cluster sizes are powers of two
  const int cid = (int)cluster_id(), ncl = (int)cluster_count();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_mine = P.n_sub > cid ? (P.n_sub - cid + ncl - 1) / ncl : 0;
  char* ring = s_ring + warp * NS * 2 * LB;
  // k-th sub-unit of this cluster's walk (k < 0 or k >= n_mine: none)
  auto sub_at = [&](int k) { return (k >= 0 && k < n_mine) ? cid + k * ncl : P.n_sub; };

  if (threadIdx.x < 4) mbar_init(&s_full[threadIdx.x], nc * NW);
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cluster_arrive();  // every CTA's barriers exist before any remote arrive
  cluster_wait();

  auto vmax = [&](uint32_t m, const Raw8<SRC>& r) {
    if constexpr (SRC == KVF_F32) {
      m = max(m, max(max(r.a.x & 0x7FFFFFFFu, r.a.y & 0x7FFFFFFFu),
                     max(r.a.z & 0x7FFFFFFFu, r.a.w & 0x7FFFFFFFu)));
      return max(m, max(max(r.b.x & 0x7FFFFFFFu, r.b.y & 0x7FFFFFFFu),
                        max(r.b.z & 0x7FFFFFFFu, r.b.w & 0x7FFFFFFFu)));
    } else {
      // packed |x| maxima of the 16-bit patterns (magnitude order = value order)
      return vmax_u16x2(vmax_u16x2(m, r.a.x & 0x7FFF7FFFu, r.a.y & 0x7FFF7FFFu),
                        r.a.z & 0x7FFF7FFFu, r.a.w & 0x7FFF7FFFu);
    }
  };

  // Iteration k in [-2, n_mine): A = max of sub-unit k+2, B = frames of
  // sub-unit k (iterations -2, -1 are the prologue: A only).  Steps of all
  // iterations form one stream; the producer side runs NS-1 steps ahead
  // of the consumer side, across iteration boundaries (loads never need the
  // maxima, only the quantisation does).
  // producer
  int kp = -2, jp = 0, hint_pa = 0, hint_pb = 0;
  W pa, pb;
  pa.init(P, sub_at(0), rank, lg_nc, hint_pa);
  pb.init(P, sub_at(-2), rank, lg_nc, hint_pb);
  int sp = 0;  // stage slot of the next issue
  auto issue_next = [&]() {
    // skip empty iterations
    while (kp < n_mine && jp >= max(pa.n, pb.n)) {
      ++kp;
      jp = 0;
      if (kp < n_mine) {
        pa.init(P, sub_at(kp + 2), rank, lg_nc, hint_pa);
        pb.init(P, sub_at(kp), rank, lg_nc, hint_pb);
      }
    }
    if (kp < n_mine) {
      char* st = ring + sp * 2 * LB;
      if (jp < pa.n) pa.issue(jp, st);
      if (jp < pb.n) pb.issue(jp, st + LB);
      ++jp;
    }
    cp_async_commit();  // (an empty group past the end keeps the count uniform)
    sp = sp + 1 == NS ? 0 : sp + 1;
  };
#pragma unroll 1
  for (int q = 0; q < NS - 1; ++q) issue_next();

  int sc_slot = 0;  // consumer stage slot
  int hint_ca = 0, hint_cb = 0;
  for (int k = -2; k < n_mine; ++k) {
    W ca, cb;
    ca.init(P, sub_at(k + 2), rank, lg_nc, hint_ca);
    cb.init(P, sub_at(k), rank, lg_nc, hint_cb);
    const int steps = max(ca.n, cb.n);
    // B side: complete max of sub-unit k -> scale (fk/kvmodel.py:139-140)
    float sc = 1.0f, inv = 1.0f;
    int32_t tile_off[VPT];
    DstView db;
    int lg_bd = 3;
    int64_t pitch = 0;
    if (k >= 0) {
      mbar_wait_cluster(&s_full[k & 3], (k >> 2) & 1);
      uint32_t mb = 0;
      for (int e = lane; e < nc * NW; e += 32) mb = max(mb, s_part[k & 3][e]);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      sc = scale_from_absmax_bits(mb);
      inv = __frcp_rn(sc);
      const PackUnitDev& UB = P.u[cb.sh.unit];
      if (rank == 0 && threadIdx.x == 0) {
        UB.scales[cb.sh.plane * UB.G + cb.sh.group] = sc;
        UB.absmax[cb.sh.plane * UB.G + cb.sh.group] = mb;
      }
      db.init(UB, cb.sh.plane);
      lg_bd = UB.g.lg_bd;
      pitch = UB.fr.row_pitch;
      const int sl = lane % LPT;
#pragma unroll
      for (int v = 0; v < VPT; ++v)
        tile_off[v] = (int32_t)tile_offset(
            UB.g, cb.sh.group * UB.g.group_size + (v * LPT + sl) * 8, pitch);
    }
    uint32_t ma = 0;
    for (int j = 0; j < steps; ++j) {
      issue_next();              // step (consumed + NS - 1)
      cp_async_wait<NS - 1>();   // this step's copies (the lane's own) have landed
      const char* st = ring + sc_slot * 2 * LB;
      sc_slot = sc_slot + 1 == NS ? 0 : sc_slot + 1;
      if (j < ca.n) {
#pragma unroll
        for (int v = 0; v < VPT; ++v) ma = vmax(ma, stage_vec<SRC, VPT>(st, v));
      }
      if (j < cb.n) {
        uint8_t* d = db.at(min(cb.sh.token(j), cb.sh.tok1 - 1));
        // all vectors' fast quantisation first (independent chains), the rare
        // exact redo of near-ties after (fk/kvmodel.py:141)
        uint2 out[VPT];
        uint32_t badm = 0;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
          float x[8];
          bool bad = false;
          raw8_to_float<SRC>(stage_vec<SRC, VPT>(st + LB, v), x);
          out[v] = quantize8_fast<false>(x, inv, bad);
          badm |= (uint32_t)bad << v;
        }
        if (__builtin_expect(badm != 0, 0)) {
#pragma unroll 1
          for (int v = 0; v < VPT; ++v) {
            if (!((badm >> v) & 1)) continue;
            float x[8];
            raw8_to_float<SRC>(stage_vec<SRC, VPT>(st + LB, v), x);
            out[v] = quantize8_exact(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], sc, inv);
          }
        }
        if (BD8) {
#pragma unroll
          for (int v = 0; v < VPT; ++v) st_v2(d + tile_off[v], out[v]);
        } else {
#pragma unroll
          for (int v = 0; v < VPT; ++v) store_vec(d + tile_off[v], out[v], lg_bd, pitch);
        }
      }
    }
    // a pad layer's tiles, or the chunk's last-segment pad tiles
    if (cb.sh.valid) {
      const PackUnitDev& UB = P.u[cb.sh.unit];
      if (cb.src.layer == nullptr || UB.n_items > UB.g.T)
        write_pads<LPT, VPT, NW>(P, cb.sh.unit, cb.sh.plane, cb.sh.group, cb.src.layer == nullptr,
                             rank, nc);
    }
    // this CTA's partial max of sub-unit k+2 -> every CTA of the cluster
    uint32_t m = ma;
    if constexpr (SRC != KVF_F32) m = max(m >> 16, m & 0xFFFFu);
    m = absmax_to_f32_bits<SRC>(m);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    // Slot (k+2)%4 last held sub-unit k-2: every warp of the cluster read it at
    // the start of its iteration k-2, before publishing its part of sub-unit k
    // (iteration k-2's end), which this warp's B(k) waited for.  No barrier.
    if (lane < nc) {
      st_cluster_u32(&s_part[(k + 2) & 3][rank * NW + warp], lane, m);
      mbar_arrive_remote(&s_full[(k + 2) & 3], lane);
    }
  }
  cp_async_wait<0>();
  cluster_arrive();  // no CTA exits while another may still store into its smem
  cluster_wait();
}

#define VPT_OF(SRC) ((SRC) == KVF_F32 ? 2 : 4)
// CTA shapes: (warps, ring stages) with ~192 KB of stage ring; the first is
// the default (measured fastest on C2: 16 warps)
constexpr int kShapes[3][2] = {{16, 3}, {12, 4}, {8, 6}};

// bf16/fp16: 4 vectors (32 channels) per lane per token; fp32: 2
template <int SRC, bool BD8, int NW, int NS>
const void* kernel_for(int group_size) {
  constexpr int V = VPT_OF(SRC);
  switch (group_size) {
    case 64: return (const void*)pack_cluster_kernel<SRC, 64 / (8 * V), V, BD8, NW, NS>;
    case 128: return (const void*)pack_cluster_kernel<SRC, 128 / (8 * V), V, BD8, NW, NS>;
    case 256: return (const void*)pack_cluster_kernel<SRC, 256 / (8 * V), V, BD8, NW, NS>;
    case 512: return (const void*)pack_cluster_kernel<SRC, 512 / (8 * V), V, BD8, NW, NS>;
    default: return nullptr;
  }
}

template <int SRC, bool BD8>
const void* kernel_for(int group_size, int shape) {
  switch (shape) {
    case 0: return kernel_for<SRC, BD8, kShapes[0][0], kShapes[0][1]>(group_size);
    case 1: return kernel_for<SRC, BD8, kShapes[1][0], kShapes[1][1]>(group_size);
    default: return kernel_for<SRC, BD8, kShapes[2][0], kShapes[2][1]>(group_size);
  }
}

template <int SRC>
const void* kernel_for(int group_size, bool bd8, int shape) {
  return bd8 ? kernel_for<SRC, true>(group_size, shape) : kernel_for<SRC, false>(group_size, shape);
}

}  // namespace

// Single-read pack of quantising units (bf16/fp16/fp32 sources, group sizes
// 64-512).  `param` = CTAs per cluster (0 = the largest the device takes).
// *launched = false when the device or the shapes do not allow it (the caller
// then runs the phase-split kernels).
kvf_status launch_pack_cluster(const std::vector<kvf_pack_unit>& units, int32_t dtype,
                               int64_t param, cudaStream_t s, bool* launched) {
  *launched = false;
  if (units.empty() || units.size() > (size_t)kMaxPackUnits || dtype == KVF_I8) return KVF_OK;
  const int gs = units[0].plan.group_size;
  for (const auto& u : units)
    if (u.plan.group_size != gs || u.plan.D % 8 || gs > u.plan.H * u.plan.D ||
        u.plan.T >= (1 << 26))  // T * rank fits 32 bits
      return KVF_OK;
  bool bd8 = true;  // every tile row piece of a vector is 8 bytes (b_d >= 8)
  for (const auto& u : units) bd8 = bd8 && u.plan.b_d >= 8;
  const int shape = std::min<int>(2, (int)((param >> 9) & 3));  // bits 9-10: CTA shape
  const void* fn = dtype == KVF_BF16  ? kernel_for<KVF_BF16>(gs, bd8, shape)
                   : dtype == KVF_F16 ? kernel_for<KVF_F16>(gs, bd8, shape)
                                      : kernel_for<KVF_F32>(gs, bd8, shape);
  if (fn == nullptr) return KVF_OK;
  // 16-B source vectors and 8-B tile stores (b_d >= 8) must be aligned
  const int64_t es = (int64_t)dtype_size(dtype);
  for (const auto& u : units) {
    for (int l = 0; l < 3; ++l)
      if (u.src.layer[l] && reinterpret_cast<uintptr_t>(u.src.layer[l]) % 16) return KVF_OK;
    if ((u.src.head_stride * es) % 16 || (u.src.slot_stride * es) % 16 ||
        (u.src.block_stride * es) % 16)
      return KVF_OK;
    const int64_t a = std::min<int64_t>(8, u.plan.b_d);
    if (reinterpret_cast<uintptr_t>(u.frames.base) % a || u.frames.frame_stride % a ||
        u.frames.plane_stride % a || u.frames.row_pitch % a)
      return KVF_OK;
  }
  const int nw = kShapes[shape][0];
  const int smem = nw * kShapes[shape][1] * (dtype == KVF_F32 ? stage_bytes<KVF_F32, 2>()
                                                               : stage_bytes<KVF_BF16, 4>());
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaGetLastError();

  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(32 * nw);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // L2 budget: every cluster keeps ~3 sub-units in flight between their HBM
  // read and the quantising re-read; keep that under ~45% of L2.
  int dev = 0, l2 = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess) {
    cudaGetLastError();
    return KVF_OK;
  }
  int64_t src_bytes = 0, n_sub_all = 0;
  for (const auto& u : units) {
    src_bytes += (int64_t)u.plan.T * u.plan.H * u.plan.D * es * 3;
    n_sub_all += 3 * (int64_t)u.plan.H * u.plan.D / gs;
  }
  const int64_t sub_bytes = std::max<int64_t>(1, src_bytes / std::max<int64_t>(1, n_sub_all));
  const bool capped = (param & 0x100) == 0;  // bit 8: no L2 cap (exploration)
  const int64_t max_cl = std::max<int64_t>(1, (int64_t)l2 * 45 / 100 / (3 * sub_bytes));
  int nc = 0, ncl = 0;
  const int want = (int)(param & 0xFF);
  for (int c : {16, 8, 4, 2}) {
    if (want && c != want) continue;
    int n = 0;
    attr[0].val.clusterDim.x = c;
    cfg.gridDim = dim3(c * 64);
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (capped) n = (int)std::min<int64_t>(n, max_cl);
    if (n * c > ncl * nc) {  // the most SMs covered within the budget
      nc = c;
      ncl = n;
    }
  }
  if (nc == 0 || ncl == 0) return KVF_OK;

  ClusterParams* P = new ClusterParams();
  P->n_units = (int32_t)units.size();
  int n_sub = 0;
  for (size_t k = 0; k < units.size(); ++k) {
    P->u[k] = make_pack_unit_dev(units[k]);
    P->sub_first[k] = n_sub;
    n_sub += 3 * P->u[k].G;
  }
  P->sub_first[units.size()] = n_sub;
  P->n_sub = n_sub;
  ncl = std::min(ncl, n_sub);
  attr[0].val.clusterDim.x = nc;
  cfg.gridDim = dim3(nc * ncl);
  void* args[] = {P};
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  delete P;
  if (e != cudaSuccess) return cuda_status(e, "pack_cluster_kernel launch");
  *launched = true;
  return KVF_OK;
}

}  // namespace kvf
