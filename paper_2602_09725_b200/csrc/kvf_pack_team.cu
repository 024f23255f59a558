// kvf_pack_team.cu — single-HBM-read pack: co-resident CTA teams, sm_100a.
//
// Replaces quantize (fk/kvmodel.py:127-144) + slice_tokens/assemble_frames
// (fk/layout.py:109-114, 234-258) for bf16/fp16/fp32 sources.  The reference
// scale of a (layer, 128-channel group) is the max |x| over ALL tokens of the
// chunk (fk/kvmodel.py:138-140), so every sample is needed twice: once for the
// maximum, once to quantise.  The second read must not go to HBM.
//
// Sub-unit s = (unit, plane p, group g): tokens x group_size channels, at most
// 10,000 x 128 x 2 B = 2.56 MB.  The persistent cooperative grid (one CTA per
// SM, all co-resident) is cut into teams of ~16 CTAs; team t owns sub-units
// t, t + n_teams, ...  Each CTA of a team takes a 1/16 token slice of the
// sub-unit.  Round r of a CTA streams, warp by warp and fully pipelined:
//   A(s_r)     : HBM read of its token slice of s_r (L2 evict_last), running
//                max |x| -> warp max -> CTA max (smem) -> the last warp of the
//                CTA publishes atomicMax + a release increment of s_r's counter;
//   Q(s_{r-2}) : re-read of its frame-item slice of s_{r-2} — an L2 hit, the
//                team read it two rounds earlier — quantise with the team
//                scale (acquire-spin on the counter, normally already full)
//                and store the tiled frame bytes (evict_first).
// Loads of a batch are issued before the counter wait, so the wait never
// drains the pipeline.  L2 working set ~ n_teams x 3 sub-units (~69 MB).
// HBM traffic: 2 B read + 1 B written per element (bf16).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kTeamThreads = 512;
constexpr int kTeamWarps = kTeamThreads / 32;
constexpr int kMaxTeamUnits = 88;
constexpr int kUnroll = 2;  // tokens in flight per lane (each: A and Q vectors)
constexpr int kMaxLag = 2;  // Q(s) runs P.lag <= kMaxLag rounds after A(s)
constexpr int kSlots = kMaxLag + 1;  // CTA-count slots in flight (see the reuse argument)

struct TeamParams {
  int32_t n_units;
  int32_t n_sub;       // 3 * G * n_units
  int32_t G;           // groups per plane (uniform in a launch)
  int32_t n_teams;
  int32_t lag;
  PackUnitDev u[kMaxTeamUnits];
};
static_assert(sizeof(TeamParams) <= 32000, "kernel parameters exceed 32 KB");

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sub-unit s -> (unit, plane, group); consecutive s share (unit, plane), so
// concurrently running teams read neighbouring 256-B pieces of the same slots.
struct Sub {
  int unit, p, g;
};
__device__ __forceinline__ Sub sub_of(const TeamParams& P, int s) {
  const int pg = s % (3 * P.G);
  return Sub{s / (3 * P.G), pg / P.G, pg % P.G};
}

// Scale of sub-unit (U, pg) once all `ts` CTAs of the team have published
// their maxima (acquire-spin of lane 0, broadcast to the warp).
__device__ __forceinline__ float team_scale(const PackUnitDev* U, int pg, int ts, int lane) {
  uint32_t bits = 0u;
  if (lane == 0) {
    uint32_t spins = 0;
    while (ld_relaxed_u32(&U->team_done[pg]) < (uint32_t)ts) {
      __nanosleep(128);
      if (++spins == (1u << 23)) __trap();  // broken schedule: fail fast, never hang
    }
    __threadfence();  // acquire: the counter is read before the maxima it covers
    bits = __ldcg(&U->absmax[pg]);
  }
  bits = __shfl_sync(0xffffffffu, bits, 0);
  return scale_from_absmax_bits(bits);
}

// |x| maximum bits of one source vector (16-bit patterns for bf16/fp16).
template <int SRC>
__device__ __forceinline__ uint32_t raw_absmax(const Raw8<SRC>& v) {
  if constexpr (SRC == KVF_F32) {
    const uint4 a = v.a, c = v.b;
    return max(max(max(a.x & 0x7FFFFFFFu, a.y & 0x7FFFFFFFu),
                   max(a.z & 0x7FFFFFFFu, a.w & 0x7FFFFFFFu)),
               max(max(c.x & 0x7FFFFFFFu, c.y & 0x7FFFFFFFu),
                   max(c.z & 0x7FFFFFFFu, c.w & 0x7FFFFFFFu)));
  } else {
    const uint4 a = v.a;
    const uint32_t w0 = a.x & 0x7FFF7FFFu, w1 = a.y & 0x7FFF7FFFu;
    const uint32_t w2 = a.z & 0x7FFF7FFFu, w3 = a.w & 0x7FFF7FFFu;
    const uint32_t hi = max(max(w0, w1), max(w2, w3)) >> 16;
    const uint32_t lo = max(max(w0 & 0xFFFFu, w1 & 0xFFFFu), max(w2 & 0xFFFFu, w3 & 0xFFFFu));
    return max(hi, lo);
  }
}

// LPG lanes share one (token, group) row; each lane owns VPL 8-channel vectors
// of it (vector v of sub-lane sl = channels (v*LPG + sl)*8 of the group), so
// the per-token address math is amortised over VPL loads.
template <int SRC, int LPG, int VPL, int UNR>
__global__ void __launch_bounds__(kTeamThreads, 1)
    pack_team_kernel(const __grid_constant__ TeamParams P) {
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  constexpr int TPI = 32 / LPG;  // tokens (or frame items) per warp instruction
  __shared__ uint32_t s_max[kSlots], s_cnt[kSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sl = lane % LPG, tl = lane / LPG;
  // team membership: team t = CTAs [ceil(t*nb/n_teams), ceil((t+1)*nb/n_teams))
  const int nb = gridDim.x, b = blockIdx.x;
  const int team = (int)(((int64_t)b * P.n_teams) / nb);
  const int c_lo = (int)(((int64_t)team * nb + P.n_teams - 1) / P.n_teams);
  const int c_hi = (int)(((int64_t)(team + 1) * nb + P.n_teams - 1) / P.n_teams);
  const int ts = c_hi - c_lo, m = b - c_lo;
  const int n_mine = team < P.n_sub ? (P.n_sub - team + P.n_teams - 1) / P.n_teams : 0;
  if (threadIdx.x < kSlots) {
    s_max[threadIdx.x] = 0u;
    s_cnt[threadIdx.x] = 0u;
  }
  __syncthreads();
  // First reads keep the default (evict_normal) priority: evict_last would pin
  // 4 GB of once-used lines; re-reads and frame stores are evict_first.
  const uint64_t drop = l2_policy_evict_first();
  const WithPolicy ld_drop{drop};

  const int kLag = P.lag;
  for (int r = 0; r < n_mine + kLag; ++r) {
    // ---- A side: sub-unit s_r, token slice [a_lo, a_lo + a_n) of this CTA
    const bool hasA = r < n_mine;
    const PackUnitDev* UA = nullptr;
    const char* a_layer = nullptr;
    int a_lo = 0, a_n = 0, a_pg = 0;
    int32_t a_off[VPL];
    if (hasA) {
      const Sub sa = sub_of(P, team + r * P.n_teams);
      UA = &P.u[sa.unit];
      a_layer = reinterpret_cast<const char*>(UA->src.layer[sa.p]);
      a_lo = (int)(((int64_t)UA->g.T * m) / ts);
      a_n = (int)(((int64_t)UA->g.T * (m + 1)) / ts) - a_lo;
      a_pg = sa.p * P.G + sa.g;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        a_off[v] = (int32_t)slot_channel_offset(
                       UA->g, sa.g * UA->g.group_size + (v * LPG + sl) * 8, UA->src.head_stride) *
                   ES;
      if (a_layer == nullptr) a_n = 0;
    }
    // ---- Q side: sub-unit s_{r-kLag}, the SAME token slice this CTA read in
    // its A pass (so the re-read hits the L2 next to this SM)
    const bool hasQ = r >= kLag;
    const PackUnitDev* UQ = nullptr;
    const char* q_layer = nullptr;
    uint8_t* q_plane = nullptr;
    int q_lo = 0, q_n = 0, q_pg = 0;
    int32_t q_off[VPL], q_toff[VPL];
    if (hasQ) {
      const Sub sq = sub_of(P, team + (r - kLag) * P.n_teams);
      UQ = &P.u[sq.unit];
      q_layer = reinterpret_cast<const char*>(UQ->src.layer[sq.p]);
      q_plane = UQ->fr.base + (int64_t)sq.p * UQ->fr.plane_stride;
      q_lo = (int)(((int64_t)UQ->g.T * m) / ts);
      q_n = (int)(((int64_t)UQ->g.T * (m + 1)) / ts) - q_lo;
      q_pg = sq.p * P.G + sq.g;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = sq.g * UQ->g.group_size + (v * LPG + sl) * 8;
        q_off[v] = (int32_t)slot_channel_offset(UQ->g, c, UQ->src.head_stride) * ES;
        q_toff[v] = (int32_t)tile_offset(UQ->g, c, UQ->fr.row_pitch);
      }
    }
    const int nA = (a_n + TPI - 1) / TPI, nQ = (q_n + TPI - 1) / TPI;
    const int n_it = max(nA, nQ);
    uint32_t amax = 0u;
    float s = 1.0f, inv = 1.0f;
    bool have_scale = !hasQ;
    for (int j0 = warp; j0 < n_it; j0 += kTeamWarps * UNR) {
      Raw8<SRC> va[UNR][VPL], vq[UNR][VPL];
      uint8_t* dq[UNR];
      bool vq_ok[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int j = j0 + u * kTeamWarps;
        const int ia = j * TPI + tl;
        if (j < nA && ia < a_n) {
          const char* sp = a_layer + paged_slot_offset_fd(UA->src, UA->div_bs, a_lo + ia) * ES;
#pragma unroll
          for (int v = 0; v < VPL; ++v) va[u][v] = load_raw8<SRC>(sp + a_off[v]);
        } else {
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            va[u][v].a = make_uint4(0u, 0u, 0u, 0u);
            if constexpr (SRC == KVF_F32) va[u][v].b = make_uint4(0u, 0u, 0u, 0u);
          }
        }
        const int iq = j * TPI + tl;
        dq[u] = nullptr;
        vq_ok[u] = false;
        if (j < nQ && iq < q_n) {
          // placement of token i (fk/layout.py:195-201)
          const int i = q_lo + iq;
          const int gq = fdiv(UQ->g.div_F, i);
          const int o = i - gq * UQ->g.F;
          const int seg = fdiv(UQ->g.div_tpf, gq);
          const int slot = gq - seg * UQ->g.tpf;
          const int f = seg * UQ->g.F + o;
          const int tr = fdiv(UQ->g.div_cols, slot);
          const int tc = slot - tr * UQ->g.grid_cols;
          dq[u] = q_plane + (int64_t)f * UQ->fr.frame_stride +
                  (int64_t)tr * UQ->g.tile_h * UQ->fr.row_pitch + tc * UQ->g.tile_w;
          if (q_layer != nullptr) {
            const char* sp = q_layer + paged_slot_offset_fd(UQ->src, UQ->div_bs, i) * ES;
#pragma unroll
            for (int v = 0; v < VPL; ++v) vq[u][v] = load_raw8<SRC>(sp + q_off[v], ld_drop);
            vq_ok[u] = true;
          }
        }
      }
      if (!have_scale) {  // counter of s_{r-kLag}: all team CTAs published their A
        s = team_scale(UQ, q_pg, ts, lane);
        inv = __frcp_rn(s);
        have_scale = true;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) amax = max(amax, raw_absmax<SRC>(va[u][v]));
        if (dq[u] != nullptr) {
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            uint2 out = make_uint2(0x80808080u, 0x80808080u);
            if (vq_ok[u]) {
              float x[8];
              raw8_to_float<SRC>(vq[u][v], x);
              out = quantize8<false>(x, s, inv);
            }
            st_v2_pol(dq[u] + q_toff[v], out, drop);
          }
        }
      }
    }
    // Pad slots of the trailing segment (token >= T, fk/layout.py:251-253):
    // PAD_BYTE 128 in this group's channels, split over the team.
    if (hasQ) {
      const int seg_items = UQ->g.F * UQ->g.tpf;
      const int q_tail = (UQ->g.T / seg_items) * seg_items;
      for (int q = q_tail + (m * kTeamWarps + warp) * TPI + tl; q < UQ->n_items;
           q += ts * kTeamWarps * TPI) {
        const int f = fdiv(UQ->g.div_tpf, q);
        const int slot = q - f * UQ->g.tpf;
        if (token_of(UQ->g, f, slot) < UQ->g.T) continue;
        const int tr = fdiv(UQ->g.div_cols, slot);
        const int tc = slot - tr * UQ->g.grid_cols;
        uint8_t* d = q_plane + (int64_t)f * UQ->fr.frame_stride +
                     (int64_t)tr * UQ->g.tile_h * UQ->fr.row_pitch + tc * UQ->g.tile_w;
#pragma unroll
        for (int v = 0; v < VPL; ++v) st_v2_pol(d + q_toff[v], make_uint2(0x80808080u, 0x80808080u), drop);
      }
    }
    // Every warp passes the wait of s_{r-kLag} each round, items or not: a
    // warp may only arrive at slot r % kSlots after the CTA published
    // s_{r-kLag}, i.e. after every warp left round r-kSlots' count (reuse).
    if (hasQ && !have_scale) s = team_scale(UQ, q_pg, ts, lane);
    if (hasQ && m == 0 && warp == 0 && lane == 0) UQ->scales[q_pg] = s;
    // ---- publish A(s_r): warp max -> CTA max -> team max
    if (hasA) {
      amax = __reduce_max_sync(0xffffffffu, amax);
      if (lane == 0) {
        const uint32_t bits = absmax_to_f32_bits<SRC>(amax);
        const int k = r % kSlots;
        if (bits) atomicMax(&s_max[k], bits);
        __threadfence_block();
        if (atomicAdd(&s_cnt[k], 1u) == kTeamWarps - 1) {
          __threadfence_block();
          const uint32_t cta_max = atomicExch(&s_max[k], 0u);
          s_cnt[k] = 0u;
          if (cta_max) atomicMax(&UA->absmax[a_pg], cta_max);
          red_release_add(&UA->team_done[a_pg], 1u);
        }
      }
    }
  }
}

template <int SRC>
const void* kernel_for(int gs) {
  constexpr int V = SRC == KVF_F32 ? 2 : 4;  // vectors per lane (16 data registers)
  switch (gs / (8 * V)) {
    case 1: return (const void*)pack_team_kernel<SRC, 1, V, kUnroll>;
    case 2: return (const void*)pack_team_kernel<SRC, 2, V, kUnroll>;
    case 4: return (const void*)pack_team_kernel<SRC, 4, V, kUnroll>;
    case 8: return (const void*)pack_team_kernel<SRC, 8, V, kUnroll>;
    case 16: return (const void*)pack_team_kernel<SRC, 16, V, kUnroll>;
    default: return nullptr;
  }
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

}  // namespace

// Launch the team kernel for quantising fast-variant units sharing one source
// dtype.  Sets *launched = false (and launches nothing) when the shapes or the
// device do not allow it; the caller then uses the phase-split kernels.  The
// units' scratch must already be zeroed (counters and maxima).
kvf_status launch_pack_team(const std::vector<kvf_pack_unit>& units, int32_t dtype,
                            cudaStream_t s, bool* launched) {
  *launched = false;
  if (units.empty() || units.size() > (size_t)kMaxTeamUnits || dtype == KVF_I8) return KVF_OK;
  const int gs = units[0].plan.group_size;
  const int C = units[0].plan.H * units[0].plan.D;
  for (const auto& u : units)
    if (u.plan.group_size != gs || u.plan.H * u.plan.D != C) return KVF_OK;
  const void* fn = dtype == KVF_BF16  ? kernel_for<KVF_BF16>(gs)
                   : dtype == KVF_F16 ? kernel_for<KVF_F16>(gs)
                                      : kernel_for<KVF_F32>(gs);
  if (fn == nullptr || gs % 8) return KVF_OK;
  TeamParams* P = new TeamParams();
  P->n_units = (int32_t)units.size();
  P->G = C / gs;
  P->n_sub = 3 * P->G * P->n_units;
  for (size_t k = 0; k < units.size(); ++k) P->u[k] = make_pack_unit_dev(units[k]);
  int dev = 0, sms = 0, occ = 0, coop = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTeamThreads, 0);
  if (e != cudaSuccess) {
    delete P;
    return cuda_status(e, "team pack setup");
  }
  const int grid = sms * std::min(occ, 1);
  const int team_size = std::max(1, env_int("KVF_TEAM_SIZE", 16));
  P->n_teams = std::max(1, grid / team_size);
  P->lag = std::min(kMaxLag, std::max(1, env_int("KVF_TEAM_LAG", 1)));
  if (!coop || grid < 1) {
    delete P;
    return KVF_OK;
  }
  void* args[] = {P};
  e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kTeamThreads), args, 0, s);
  delete P;
  if (e != cudaSuccess) return cuda_status(e, "pack_team_kernel launch");
  *launched = true;
  return KVF_OK;
}

}  // namespace kvf
