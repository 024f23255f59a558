// kvf_kvfc.cu — KVFC frame-stream decode on the GPU, sm_100a.
//
// 1. rc_decode_kernel: the reference's adaptive range decoder
//    (fk/rangecoder.py:146-189), one thread per (frame, plane) stream — every
//    stream resets its model and is length-prefixed, so they are independent.
//    The model lives in shared memory as 256 packed words per thread,
//      W[i] = fen[i+1] << 16 | freq[i]      (fen = Fenwick tree of freq),
//    stored [i][thread] so each thread always hits its own bank.  Counts fit
//    16 bits: freq <= total - 255 and every Fenwick node below the root covers
//    at most 128 symbols, while total < 2^16 + 32 (fk/rangecoder.py:48-50).
//    The root node (total) is never read by the search and is not stored.
// 2. recon_kernel: per-sample prediction (fk/codec.py:131-144) as segmented
//    prefix sums mod 256.  One CTA per chain of same-plane frames starting at
//    an intra frame.  A 16-pixel run of a row never crosses a 16x16 block, so a
//    run is wholly inter (absolute: prev + d) or intra (relative: + d); a warp
//    scans 32 runs at a time with the operator
//      (a, b) -> b.abs ? b : (a.abs, a.v + b.v),
//    after the first column (predicted from above) was scanned down the rows.
#include <algorithm>

#include "kvf_common.cuh"

namespace kvf {
namespace {

constexpr uint32_t kTop = 1u << 24;
constexpr uint32_t kBot = 1u << 16;
constexpr uint32_t kInc = 32;
constexpr uint32_t kLimit = 1u << 16;

// Sequential byte reader over a device payload; bytes past the end are 0.
struct ByteReader {
  const uint8_t* p;
  int64_t len;
  int64_t pos;
  uint32_t word;    // the aligned 4-byte word holding byte `pos`, when cached
  uintptr_t waddr;  // address of that word (0 = nothing cached)
  __device__ __forceinline__ uint32_t next() {
    const int64_t i = pos++;
    if (i >= len) return 0u;
    const uintptr_t a = reinterpret_cast<uintptr_t>(p + i);
    const uintptr_t wa = a & ~uintptr_t(3);
    if (wa != waddr) {
      word = __ldg(reinterpret_cast<const uint32_t*>(wa));
      waddr = wa;
    }
    return (word >> (8 * (a & 3))) & 0xFFu;
  }
};

__global__ void __launch_bounds__(224)
    rc_decode_kernel(const kvf_rc_stream* __restrict__ streams, int n) {
  extern __shared__ uint32_t W[];  // [256][blockDim.x]
  const int nt = blockDim.x, tid = threadIdx.x;
  const int sidx = blockIdx.x * nt + tid;
  if (sidx >= n) return;
  const kvf_rc_stream st = streams[sidx];
#define MW(i) W[(i) * nt + tid]
  for (int i = 0; i < 256; ++i) {
    const int j = i + 1;
    MW(i) = ((uint32_t)(j & -j) << 16) | 1u;  // freq 1, fen[j] = lowbit(j)
  }
  uint32_t total = 256, low = 0, rng = 0xFFFFFFFFu, code = 0;
  ByteReader br{st.payload, st.len, 0, 0u, 0};
  for (int k = 0; k < 4; ++k) code = (code << 8) | br.next();

  uint8_t* out = st.symbols;
  uint32_t pack = 0;
  const bool aligned4 = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  for (int64_t k = 0; k < st.n_symbols; ++k) {
    const uint32_t r = rng / total;
    uint32_t v = (code - low) / r;
    if (v >= total) v = total - 1;
    // Fenwick descent: largest s with cum(s) <= v (fk/rangecoder.py:79-90)
    uint32_t idx = 0, rem = v;
#pragma unroll
    for (uint32_t bit = 128; bit; bit >>= 1) {
      const uint32_t f = MW(idx + bit - 1) >> 16;
      if (f <= rem) {
        rem -= f;
        idx += bit;
      }
    }
    const uint32_t s = idx;
    const uint32_t cum = v - rem;
    const uint32_t fr = MW(s) & 0xFFFFu;
    low += r * cum;
    rng = r * fr;
    for (;;) {
      if ((low ^ (low + rng)) >= kTop) {
        if (rng >= kBot) break;
        rng = (0u - low) & (kBot - 1);
      }
      code = (code << 8) | br.next();
      low <<= 8;
      rng <<= 8;
    }
    // emit (4 symbols per store when aligned)
    if (aligned4) {
      pack |= s << (8 * (k & 3));
      if ((k & 3) == 3) {
        *reinterpret_cast<uint32_t*>(out + (k - 3)) = pack;
        pack = 0;
      }
    } else {
      out[k] = (uint8_t)s;
    }
    // model update: freq[s] += INC and Fenwick path (fk/rangecoder.py:60-66)
    MW(s) += (kInc << 16) | kInc;
    for (uint32_t j = (s + 1) + ((s + 1) & (0u - (s + 1))); j <= 255; j += j & (0u - j))
      MW(j - 1) += kInc << 16;
    total += kInc;
    if (total >= kLimit) {  // halve counts, rebuild the tree (fk/rangecoder.py:93-103)
      total = 0;
      for (int i = 0; i < 256; ++i) {
        const uint32_t f = ((MW(i) & 0xFFFFu) + 1) >> 1;
        total += f;
        MW(i) = (f << 16) | f;
      }
      for (int j = 1; j <= 255; ++j) {
        const int par = j + (j & -j);
        if (par <= 255) MW(par - 1) += MW(j - 1) & 0xFFFF0000u;
      }
    }
  }
  if (aligned4 && (st.n_symbols & 3)) {
    const int64_t base = st.n_symbols & ~int64_t(3);
    for (int64_t k = base; k < st.n_symbols; ++k) out[k] = (uint8_t)(pack >> (8 * (k - base)));
  }
#undef MW
}

// ----------------------------------------------------------- reconstruction
struct Seg {
  uint32_t abs;  // 1 = value is absolute
  uint32_t v;    // value (abs) or increment (relative), mod 256 in the low byte
};

__device__ __forceinline__ Seg seg_combine(Seg a, Seg b) {
  return b.abs ? b : Seg{a.abs, a.v + b.v};
}

// Inclusive warp scan of Seg; returns the inclusive value for this lane.
__device__ __forceinline__ Seg warp_seg_scan(Seg x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg y;
    y.abs = __shfl_up_sync(0xffffffffu, x.abs, o);
    y.v = __shfl_up_sync(0xffffffffu, x.v, o);
    if (lane >= o) x = seg_combine(y, x);
  }
  return x;
}

__device__ __forceinline__ int unzig(uint32_t z) {
  return (z & 1) ? -(int)((z + 1) >> 1) : (int)(z >> 1);
}

__device__ __forceinline__ bool mode_bit(const uint8_t* modes, int bw, int by, int bx) {
  if (!modes) return false;
  const int b = by * bw + bx;
  return (modes[b >> 3] >> (7 - (b & 7))) & 1;  // np.packbits: MSB first
}

constexpr int kReconThreads = 512;

__global__ void __launch_bounds__(kReconThreads)
    recon_kernel(const kvf_recon_plane* __restrict__ planes,
                 const kvf_recon_chain* __restrict__ chains) {
  const kvf_recon_chain ch = chains[blockIdx.x];
  const int h = ch.height, w = ch.width;
  const int bw = (w + 15) / 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int e = 0; e < ch.count; ++e) {
    const kvf_recon_plane P = planes[ch.first + e];
    const uint8_t* prev = e > 0 ? planes[ch.first + e - 1].out : nullptr;
    const int64_t prev_pitch = e > 0 ? planes[ch.first + e - 1].out_pitch : 0;
    const uint8_t* modes = e > 0 ? P.modes : nullptr;
    // Phase A: first column, scanned down the rows by warp 0 (carry starts at
    // the corner prediction 128).
    if (warp == 0) {
      uint32_t carry = 128;
      for (int y0 = 0; y0 < h; y0 += 32) {
        const int y = y0 + lane;
        Seg x{0u, 0u};
        if (y < h) {
          const int d = unzig(P.symbols[(int64_t)y * w]);
          if (mode_bit(modes, bw, y >> 4, 0))
            x = Seg{1u, (uint32_t)(prev[(int64_t)y * prev_pitch] + d)};
          else
            x = Seg{0u, (uint32_t)d};
        }
        Seg inc = warp_seg_scan(x);
        const uint32_t val = inc.abs ? inc.v : carry + inc.v;
        if (y < h) P.out[(int64_t)y * P.out_pitch] = (uint8_t)val;
        carry = __shfl_sync(0xffffffffu, val, 31);
      }
    }
    __syncthreads();
    // Phase B: each warp scans whole rows in spans of 32 runs x 16 pixels.
    for (int y = warp; y < h; y += nwarps) {
      const uint8_t* sym = P.symbols + (int64_t)y * w;
      uint8_t* orow = P.out + (int64_t)y * P.out_pitch;
      const uint8_t* prow = prev ? prev + (int64_t)y * prev_pitch : nullptr;
      uint32_t carry = orow[0];  // column 0 from phase A
      for (int x0 = 0; x0 < w; x0 += 32 * 16) {
        const int xs = x0 + lane * 16;
        const int nrun = max(0, min(16, w - xs));
        const bool inter = nrun > 0 && mode_bit(modes, bw, y >> 4, xs >> 4);
        uint8_t vals[16];
        Seg run{0u, 0u};
        for (int k = 0; k < nrun; ++k) {
          const int x = xs + k;
          const int d = unzig(sym[x]);
          if (x == 0) {
            vals[k] = (uint8_t)carry;  // already final
            run = Seg{1u, carry};
          } else if (inter) {
            vals[k] = (uint8_t)(prow[x] + d);
            run = Seg{1u, vals[k]};
          } else {
            vals[k] = (uint8_t)d;  // relative increment for now
            run = seg_combine(run, Seg{0u, (uint32_t)d});
          }
        }
        const Seg inc = warp_seg_scan(run);
        // exclusive prefix = value just before this run
        Seg exc;
        exc.abs = __shfl_up_sync(0xffffffffu, inc.abs, 1);
        exc.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
        uint32_t before = carry;
        if (lane > 0) before = exc.abs ? exc.v : carry + exc.v;
        if (!inter) {
          uint32_t acc = before;
          for (int k = 0; k < nrun; ++k) {
            if (xs + k == 0) {
              acc = carry;
              continue;
            }
            acc += vals[k];
            vals[k] = (uint8_t)acc;
          }
        }
        for (int k = 0; k < nrun; ++k) orow[xs + k] = vals[k];
        const uint32_t last = inc.abs ? inc.v : carry + inc.v;
        carry = __shfl_sync(0xffffffffu, last, 31);
      }
    }
    __syncthreads();  // frame e complete before e+1 predicts from it
  }
}

}  // namespace
}  // namespace kvf

using namespace kvf;

extern "C" kvf_status kvf_rc_decode(const kvf_rc_stream* d_streams, int32_t n_streams,
                                    void* stream) {
  if (n_streams < 0 || (n_streams > 0 && !d_streams)) KVF_FAIL(KVF_EINVAL, "bad stream array");
  if (n_streams == 0) return KVF_OK;
  int dev = 0, sms = 0;
  KVF_CHECK_CUDA(cudaGetDevice(&dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // Spread the streams over every SM: threads per CTA = ceil(n / SMs), in
  // warps, capped by the 224 x 1 KB model footprint per CTA.
  int per = (n_streams + sms - 1) / sms;
  per = std::min(224, std::max(32, (per + 31) / 32 * 32));
  const size_t smem = (size_t)per * 256 * sizeof(uint32_t);
  KVF_CHECK_CUDA(cudaFuncSetAttribute(rc_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(224 * 256 * sizeof(uint32_t))));
  const int grid = (n_streams + per - 1) / per;
  rc_decode_kernel<<<grid, per, smem, reinterpret_cast<cudaStream_t>(stream)>>>(d_streams,
                                                                                n_streams);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}

extern "C" kvf_status kvf_kvfc_reconstruct(const kvf_recon_plane* d_planes,
                                           const kvf_recon_chain* d_chains, int32_t n_chains,
                                           void* stream) {
  if (n_chains < 0 || (n_chains > 0 && (!d_planes || !d_chains)))
    KVF_FAIL(KVF_EINVAL, "bad chain arrays");
  if (n_chains == 0) return KVF_OK;
  recon_kernel<<<n_chains, kReconThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_planes,
                                                                                     d_chains);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}
