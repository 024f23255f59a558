// kvf_pack_coop.cu — single-read fused pack: TMA-staged stripes + grid-wide
// per-stripe counters, sm_100a.
//
// The reference quantises per (layer, 128-channel group) with the maximum
// taken over ALL tokens of the chunk (fk/kvmodel.py:138-140), so a streaming
// kernel would have to read the source twice.  Here the whole chip holds the
// data instead: one CTA per SM (cooperative launch, all co-resident), and a
// "stripe" = (unit, plane, SC contiguous channels) is split across the CTAs by
// token range.  Each CTA bulk-copies (cp.async.bulk, TMA engine, mbarrier
// completion) its tokens' stripe slice into shared memory once; then
//   A(k): local |x| max from SMEM -> atomicMax to the stripe's group maxima ->
//         one arrival on the plane's counter;
//   Q(k-2): wait until all CTAs arrived for stripe k-2, scale = fp32(max/127),
//         quantise its slice from SMEM and write the tiled frame bytes
//         (fk/kvmodel.py:141-143, fk/layout.py:234-258).
// Four SMEM buffers rotate: stripe k+2 is in flight while A(k) and Q(k-2)
// run, so neither the copy nor the grid barrier is on the critical path.
// HBM traffic: exactly 2 B read + 1 B written per element (bf16 source).
#include <algorithm>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {
namespace {

constexpr int kCoopThreads = 512;
constexpr int kCoopWarps = kCoopThreads / 32;
constexpr int kNBuf = 4;
constexpr int kQLag = 2;         // Q(k - kQLag) runs in iteration k
constexpr int kNTab = 4;         // per-unit token tables alive at once
constexpr int kMaxCoopUnits = 64;
constexpr int kMaxStripes = 3 * kMaxCoopUnits * 8;
constexpr int kSmemBudget = 220 * 1024;

struct Stripe {
  uint16_t unit;
  uint8_t plane;
  uint8_t first_of_unit;
  int16_t c0;       // first channel
  int16_t j;        // stripe index within its plane
};

struct CoopParams {
  int32_t n_units;
  int32_t n_stripes;
  int32_t SC;          // channels per stripe
  int32_t tok_cap;     // max tokens per CTA (buffer rows)
  int32_t stripes_per_plane;
  PackUnitDev u[kMaxCoopUnits];
  Stripe st[kMaxStripes];
};

struct TokTab {
  int64_t src;  // element offset of the token slot in the source layer
  int64_t dst;  // byte offset of the token's tile origin inside a plane
};

__device__ __forceinline__ void cta_tokens(const PackUnitDev& U, int b, int nb, int& lo,
                                           int& n) {
  lo = (int)(((int64_t)U.g.T * b) / nb);
  n = (int)(((int64_t)U.g.T * (b + 1)) / nb) - lo;
}

template <int SRC>
__device__ void fill_table_and_load(const CoopParams& P, int m, uint8_t* buf, uint64_t* bar,
                                    TokTab* tabs, uint64_t pol) {
  // warp 0 only
  const int lane = threadIdx.x & 31;
  const Stripe st = P.st[m];
  const PackUnitDev& U = P.u[st.unit];
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  int lo, n;
  cta_tokens(U, blockIdx.x, gridDim.x, lo, n);
  TokTab* tab = tabs + (st.unit % kNTab) * P.tok_cap;
  if (st.first_of_unit) {
    for (int j = lane; j < n; j += 32) {
      const int i = lo + j;
      tab[j].src = paged_slot_offset_fd(U.src, U.div_bs, i);
      // placement (fk/layout.py:195-201)
      const int g = fdiv(U.g.div_F, i);
      const int o = i - g * U.g.F;
      const int seg = fdiv(U.g.div_tpf, g);
      const int slot = g - seg * U.g.tpf;
      const int f = seg * U.g.F + o;
      const int tr = fdiv(U.g.div_cols, slot);
      const int tc = slot - tr * U.g.grid_cols;
      tab[j].dst = (int64_t)f * U.fr.frame_stride + (int64_t)tr * U.g.tile_h * U.fr.row_pitch +
                   (int64_t)tc * U.g.tile_w;
    }
    __syncwarp();
  }
  const char* layer = reinterpret_cast<const char*>(U.src.layer[st.plane]);
  const int SC = P.SC;
  const bool contiguous = U.src.head_stride == (1 << U.g.lg_D);
  const int D = 1 << U.g.lg_D;
  const int hs = SC >> U.g.lg_D;  // heads per stripe
  const int h0 = st.c0 >> U.g.lg_D;
  uint32_t bytes = layer ? (uint32_t)(n * SC * ES) : 0u;
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (!layer || n == 0) return;
  if (contiguous) {
    for (int j = lane; j < n; j += 32)
      tma_bulk_g2s(buf + (size_t)j * SC * ES, layer + (tab[j].src + st.c0) * ES, SC * ES, bar,
                   pol);
  } else {
    for (int q = lane; q < n * hs; q += 32) {
      const int j = q / hs, h = q - j * hs;
      tma_bulk_g2s(buf + ((size_t)j * SC + h * D) * ES,
                   layer + (tab[j].src + (int64_t)(h0 + h) * U.src.head_stride) * ES, D * ES, bar,
                   pol);
    }
  }
}

template <int SRC, int VPS>
__global__ void __launch_bounds__(kCoopThreads, 1)
    pack_coop_kernel(const __grid_constant__ CoopParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[kNBuf];
  constexpr int ES = SRC == KVF_F32 ? 4 : 2;
  const int SC = P.SC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x, nb = gridDim.x;
  const size_t buf_bytes = (size_t)P.tok_cap * SC * ES;
  uint8_t* bufs = smem;
  TokTab* tabs = reinterpret_cast<TokTab*>(smem + kNBuf * buf_bytes);
  uint32_t* s_max = reinterpret_cast<uint32_t*>(tabs + kNTab * P.tok_cap);  // [SC/8]

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNBuf; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  for (int k = threadIdx.x; k < SC / 8; k += kCoopThreads) s_max[k] = 0u;
  __syncthreads();
  const uint64_t keep = l2_policy_evict_first();  // source is read exactly once
  if (warp == 0)
    for (int m = 0; m < kNBuf && m < P.n_stripes; ++m)
      fill_table_and_load<SRC>(P, m, bufs + m * buf_bytes, &bars[m], tabs, keep);
  __syncthreads();

  const int S = P.n_stripes;
  for (int k = 0; k < S + kQLag; ++k) {
    // ------------------------------------------------------------ A(k)
    if (k < S) {
      const Stripe st = P.st[k];
      const PackUnitDev& U = P.u[st.unit];
      const char* layer = reinterpret_cast<const char*>(U.src.layer[st.plane]);
      mbar_wait_parity(&bars[k % kNBuf], (uint32_t)((k / kNBuf) & 1));
      if (layer) {
        int lo, n;
        cta_tokens(U, b, nb, lo, n);
        const uint8_t* buf = bufs + (k % kNBuf) * buf_bytes;
        uint32_t m[VPS];
#pragma unroll
        for (int v = 0; v < VPS; ++v) m[v] = 0u;
        for (int j = warp; j < n; j += kCoopWarps) {
#pragma unroll
          for (int v = 0; v < VPS; ++v)
            m[v] = max(m[v], vec_absmax_bits<SRC>(
                                 reinterpret_cast<const char*>(buf) +
                                     ((size_t)j * SC + (lane + 32 * v) * 8) * ES,
                                 SmemLoad()));
        }
        const int lpg = U.g.group_size >> 3;
#pragma unroll
        for (int v = 0; v < VPS; ++v) {
          uint32_t x = absmax_to_f32_bits<SRC>(m[v]);
          for (int o = 1; o < 32 && o < lpg; o <<= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
          if ((lane & (min(lpg, 32) - 1)) == 0 && x) atomicMax(&s_max[(lane + 32 * v) / lpg], x);
        }
        __syncthreads();
        const int ng = SC / U.g.group_size;
        const int g0 = st.c0 / U.g.group_size;
        for (int i = threadIdx.x; i < ng; i += kCoopThreads) {
          if (s_max[i]) atomicMax(&U.absmax[st.plane * U.G + g0 + i], s_max[i]);
          s_max[i] = 0u;
          __threadfence();  // each writer makes its reduction visible before the barrier
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // then this CTA's arrival for stripe k
          atomicAdd(&U.stripe_done[st.plane * P.stripes_per_plane + st.j], 1u);
        }
      }
    }
    // ---------------------------------------------------------- Q(k-lag)
    const int kq = k - kQLag;
    if (kq >= 0) {
      const Stripe st = P.st[kq];
      const PackUnitDev& U = P.u[st.unit];
      const char* layer = reinterpret_cast<const char*>(U.src.layer[st.plane]);
      if (layer && threadIdx.x == 0) {
        // Every CTA arrives exactly once per stripe on the stripe's own counter
        // (a shared per-plane counter would let early arrivals for stripe j+1
        // stand in for late ones of stripe j).
        const uint32_t need = (uint32_t)nb;
        const uint32_t* ctr = &U.stripe_done[st.plane * P.stripes_per_plane + st.j];
        long long spins = 0;
        while (ld_acquire_u32(ctr) < need) {
          __nanosleep(64);
          if (++spins == (1ll << 28)) __trap();  // broken schedule: fail hard
        }
      }
      __syncthreads();
      const int gs = U.g.group_size;
      float s[VPS], inv[VPS];
      int32_t toff[VPS];
#pragma unroll
      for (int v = 0; v < VPS; ++v) {
        const int c = st.c0 + (lane + 32 * v) * 8;
        s[v] = scale_from_absmax_bits(__ldcg(&U.absmax[st.plane * U.G + (c >> U.g.lg_gs)]));
        inv[v] = __frcp_rn(s[v]);
        toff[v] = (int32_t)tile_offset(U.g, c, U.fr.row_pitch);
      }
      if (b == 0)  // publish the stripe's scales (fk/kvmodel.py:140)
        for (int i = threadIdx.x; i < SC / gs; i += kCoopThreads) {
          const int g = st.c0 / gs + i;
          U.scales[st.plane * U.G + g] =
              scale_from_absmax_bits(__ldcg(&U.absmax[st.plane * U.G + g]));
        }
      uint8_t* plane_base = U.fr.base + (int64_t)st.plane * U.fr.plane_stride;
      const uint64_t drop = l2_policy_evict_first();
      int lo, n;
      cta_tokens(U, b, nb, lo, n);
      const TokTab* tab = tabs + (st.unit % kNTab) * P.tok_cap;
      const uint8_t* buf = bufs + (kq % kNBuf) * buf_bytes;
      for (int j = warp; j < n; j += kCoopWarps) {
        uint8_t* dst = plane_base + tab[j].dst;
#pragma unroll
        for (int v = 0; v < VPS; ++v) {
          uint2 out;
          if (layer) {
            float x[8];
            load_vec8<SRC>(reinterpret_cast<const char*>(buf) +
                               ((size_t)j * SC + (lane + 32 * v) * 8) * ES,
                           x, SmemLoad());
            out = quantize8<false>(x, s[v], inv[v]);
          } else {
            out = make_uint2(0x80808080u, 0x80808080u);  // pad layer: quantised zero
          }
          st_v2_pol(dst + toff[v], out, drop);
        }
      }
      // Pad slots of the trailing segment (token index >= T): PAD_BYTE 128.
      {
        const int seg_items = U.g.F * U.g.tpf;
        const int q_tail = (U.g.T / seg_items) * seg_items;
        for (int q = q_tail + b * kCoopWarps + warp; q < U.n_items; q += nb * kCoopWarps) {
          const int f = fdiv(U.g.div_tpf, q);
          const int slot = q - f * U.g.tpf;
          if (token_of(U.g, f, slot) < U.g.T) continue;
          const int tr = fdiv(U.g.div_cols, slot);
          const int tc = slot - tr * U.g.grid_cols;
          uint8_t* dst = plane_base + (int64_t)f * U.fr.frame_stride +
                         (int64_t)tr * U.g.tile_h * U.fr.row_pitch + (int64_t)tc * U.g.tile_w;
#pragma unroll
          for (int v = 0; v < VPS; ++v)
            st_v2_pol(dst + toff[v], make_uint2(0x80808080u, 0x80808080u), drop);
        }
      }
      __syncthreads();  // buffer kq % kNBuf is free
      const int m = kq + kNBuf;
      if (warp == 0 && m < S)
        fill_table_and_load<SRC>(P, m, bufs + (m % kNBuf) * buf_bytes, &bars[m % kNBuf], tabs,
                                 keep);
    }
  }
}

// ------------------------------------------------------------------- host
template <int SRC, int VPS>
kvf_status launch_t(const CoopParams& P, size_t smem, cudaStream_t s, bool* launched) {
  auto fn = pack_coop_kernel<SRC, VPS>;
  KVF_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0, occ = 0;
  KVF_CHECK_CUDA(cudaGetDevice(&dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  KVF_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kCoopThreads, smem));
  if (occ < 1) return KVF_OK;  // not launchable: caller falls back
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(kCoopThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KVF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, fn, P));
  *launched = true;
  return KVF_OK;
}

template <int SRC>
kvf_status launch_vps(int vps, const CoopParams& P, size_t smem, cudaStream_t s, bool* ok) {
  switch (vps) {
    case 1: return launch_t<SRC, 1>(P, smem, s, ok);
    case 2: return launch_t<SRC, 2>(P, smem, s, ok);
    case 4: return launch_t<SRC, 4>(P, smem, s, ok);
    default: return KVF_OK;
  }
}

}  // namespace

// Plan the stripes for a group of fast-variant quantising units; returns
// false (and launches nothing) when the stripes do not fit the SMEM budget.
kvf_status launch_pack_coop(const std::vector<kvf_pack_unit>& units, int32_t dtype,
                            cudaStream_t s, bool* launched) {
  *launched = false;
  if (units.empty() || units.size() > (size_t)kMaxCoopUnits) return KVF_OK;
  int dev = 0, sms = 0;
  KVF_CHECK_CUDA(cudaGetDevice(&dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int ES = (int)dtype_size(dtype);
  const kvf_plan& p0 = units[0].plan;
  const int C = p0.H * p0.D;
  int max_T = 0;
  for (const auto& u : units) {
    const kvf_plan& p = u.plan;
    if (p.H * p.D != C || p.D != p0.D || p.group_size != p0.group_size) return KVF_OK;
    max_T = std::max(max_T, p.T);
  }
  const int tok_cap = (max_T + sms - 1) / sms;
  int SC = 0;
  for (int sc = C; sc >= 256; sc /= 2) {
    if (C % sc || sc % p0.group_size || sc % p0.D || sc / 256 > 4 || sc % 256) continue;
    size_t smem = (size_t)kNBuf * tok_cap * sc * ES + (size_t)kNTab * tok_cap * sizeof(TokTab) +
                  (size_t)(sc / 8) * 4;
    if (smem <= (size_t)kSmemBudget) {
      SC = sc;
      break;
    }
  }
  if (SC == 0) return KVF_OK;
  const int per_plane = C / SC;
  if ((size_t)units.size() * 3 * per_plane > (size_t)kMaxStripes) return KVF_OK;

  CoopParams* P = new CoopParams();
  P->n_units = (int32_t)units.size();
  P->SC = SC;
  P->tok_cap = tok_cap;
  P->stripes_per_plane = per_plane;
  int S = 0;
  for (size_t k = 0; k < units.size(); ++k) {
    P->u[k] = make_pack_unit_dev(units[k]);
    for (int pl = 0; pl < 3; ++pl)
      for (int j = 0; j < per_plane; ++j) {
        Stripe& st = P->st[S++];
        st.unit = (uint16_t)k;
        st.plane = (uint8_t)pl;
        st.first_of_unit = (uint8_t)(pl == 0 && j == 0);
        st.c0 = (int16_t)(j * SC);
        st.j = (int16_t)j;
      }
  }
  P->n_stripes = S;
  size_t smem = (size_t)kNBuf * tok_cap * SC * ES + (size_t)kNTab * tok_cap * sizeof(TokTab) +
                (size_t)(SC / 8) * 4;
  kvf_status st = KVF_OK;
  switch (dtype) {
    case KVF_BF16: st = launch_vps<KVF_BF16>(SC / 256, *P, smem, s, launched); break;
    case KVF_F16: st = launch_vps<KVF_F16>(SC / 256, *P, smem, s, launched); break;
    default: st = launch_vps<KVF_F32>(SC / 256, *P, smem, s, launched); break;
  }
  delete P;
  return st;
}

}  // namespace kvf
