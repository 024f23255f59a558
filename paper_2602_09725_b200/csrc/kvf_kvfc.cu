// kvf_kvfc.cu — KVFC frame-stream decode on the GPU, sm_100a.
//
// 1. rc_decode_kernel: the reference's adaptive range decoder
//    (fk/rangecoder.py:146-189), one thread per (frame, plane) stream — every
//    stream resets its model and is length-prefixed, so they are independent.
//    The per-symbol work is a serial dependency chain, so the kernel is built
//    for latency: the top four Fenwick levels are registers, the second
//    division is replaced by multiplies inside the descent, tree updates are
//    fire-and-forget shared atomics, the halving rebuild is block-parallel,
//    and payload words are prefetched one word ahead.  The root node (total)
//    is never read by the search and is not stored.
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
// Two aligned words are held: the one being consumed and the next one, whose
// load is issued four bytes ahead so the dependent decode chain rarely waits.
struct ByteStream {
  uintptr_t wa;    // address of the aligned word `cur`
  uintptr_t end;   // payload end address
  uintptr_t a;     // address of the next byte
  uint32_t cur, nxt;
  __device__ __forceinline__ void init(const uint8_t* p, uint32_t n) {
    a = reinterpret_cast<uintptr_t>(p);
    end = a + n;
    wa = a & ~uintptr_t(3);
    cur = n ? __ldg(reinterpret_cast<const uint32_t*>(wa)) : 0u;
    nxt = wa + 4 < end ? __ldg(reinterpret_cast<const uint32_t*>(wa + 4)) : 0u;
  }
  // Straight-line (predicated) so the per-symbol renormalisation does not
  // branch: the byte, then the word rotation when `a` crosses into `nxt`.
  __device__ __forceinline__ uint32_t next() {
    const uint32_t b = a < end ? (cur >> (8 * (a & 3))) & 0xFFu : 0u;
    ++a;
    if ((a & 3) == 0) {
      wa += 4;
      cur = nxt;
      nxt = wa + 4 < end ? __ldg(reinterpret_cast<const uint32_t*>(wa + 4)) : 0u;
    }
    return b;
  }
};

// The reference model (fk/rangecoder.py:53-103): 256 counts, a Fenwick tree of
// cumulative counts, +INC per coded symbol, halving at TOTAL_LIMIT.  Here the
// 15 tree nodes that are multiples of 16 (the top four levels of the descent)
// live in registers R[1..15]; the other nodes and every count live in shared
// memory as W[i] = fen[i+1] << 16 | freq[i], [i][thread]-major so each thread
// always hits its own bank.  Counts fit 16 bits: total < 2^16 + 32 and a node
// below the multiples of 16 covers at most 8 symbols (fk/rangecoder.py:48-50).
constexpr int kDecThreads = 32;  // one warp per CTA: 32 KB of models, 7 CTAs per SM

__device__ __forceinline__ uint32_t lowbit(uint32_t j) { return j & (0u - j); }


// Halve every count ((f + 1) >> 1, fk/rangecoder.py:93-103) and rebuild the
// tree block by block (16 symbols per block); returns the new total.
__device__ __forceinline__ uint32_t rebuild(uint32_t* w, uint32_t (&R)[16]) {
  uint32_t B[16];
  uint32_t total = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    uint32_t pre[17];
    pre[0] = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) pre[q + 1] = pre[q] + (((w[(16 * b + q) * kDecThreads] & 0xFFFFu) + 1) >> 1);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int jl = q + 1;
      const uint32_t node = pre[jl] - pre[jl - (jl & -jl)];
      w[(16 * b + q) * kDecThreads] = (node << 16) | (pre[q + 1] - pre[q]);
    }
    B[b] = pre[16];
    total += pre[16];
  }
#pragma unroll
  for (int k = 1; k < 16; ++k) {  // node 16k covers blocks (k - lowbit(k), k]
    uint32_t v = 0;
#pragma unroll
    for (int b = k - (k & -k); b < k; ++b) v += B[b];
    R[k] = v;
  }
  return total;
}

__global__ void __launch_bounds__(kDecThreads)
    rc_decode_kernel(const kvf_rc_stream* __restrict__ streams, int n) {
  extern __shared__ uint32_t W[];  // [256][kDecThreads]
  const int tid = threadIdx.x;
  const int sidx = blockIdx.x * kDecThreads + tid;
  if (sidx >= n) return;
  const kvf_rc_stream st = streams[sidx];
  uint32_t* w = W + tid;  // word i of this thread's model at w[i * kDecThreads]
#pragma unroll 8
  for (int i = 0; i < 256; ++i) w[i * kDecThreads] = (lowbit(i + 1) << 16) | 1u;
  uint32_t R[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) R[k] = 16u * (uint32_t)(k & -k);
  uint32_t total = 256, low = 0, rng = 0xFFFFFFFFu, code = 0;
  ByteStream bs;
  bs.init(st.payload, (uint32_t)st.len);
  for (int k = 0; k < 4; ++k) code = (code << 8) | bs.next();

  uint8_t* out = st.symbols;
  const uint32_t nsym = (uint32_t)st.n_symbols;
  uint32_t pack = 0;
  const bool aligned4 = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  double inv = 1.0 / (double)total;  // 1/total of the symbol being decoded
  for (uint32_t k = 0; k < nsym; ++k) {
    // r = rng / total (fk/rangecoder.py:163), exact: inv = RN(1/total) has a
    // relative error <= 2^-53, so rng*inv is within 2^-28 of rng/total, whose
    // fraction is 0 or in [1/total, 1 - 1/total] with total < 2^16 + 32;
    // adding 2^-19 before the floor therefore never changes it wrongly.
    const uint32_t r = __double2uint_rd(__fma_rn((double)rng, inv, 0x1p-19));
    const double inv_next = 1.0 / (double)(total + kInc);  // off the critical path
    // Largest s with cum(s) <= min((code - low) / r, total - 1) (fk/rangecoder.py:163-166,
    // 79-90), found without the second division: cum <= x / r  <=>  cum * r <= x.
    const uint32_t x = code - low;
    uint32_t rem = x, f;
    // top four levels: register nodes 128 | 64,192 | 32..224 | 16..240
    f = R[8] * r;
    const bool b7 = f <= rem;
    if (b7) rem -= f;
    f = (b7 ? R[12] : R[4]) * r;
    const bool b6 = f <= rem;
    if (b6) rem -= f;
    {
      const uint32_t a = b7 ? R[10] : R[2], b = b7 ? R[14] : R[6];
      f = (b6 ? b : a) * r;
    }
    const bool b5 = f <= rem;
    if (b5) rem -= f;
    {
      const uint32_t a0 = b7 ? R[9] : R[1], a1 = b7 ? R[11] : R[3];
      const uint32_t a2 = b7 ? R[13] : R[5], a3 = b7 ? R[15] : R[7];
      const uint32_t c0 = b6 ? a2 : a0, c1 = b6 ? a3 : a1;
      f = (b5 ? c1 : c0) * r;
    }
    const bool b4 = f <= rem;
    if (b4) rem -= f;
    const uint32_t blk = (b7 ? 128u : 0u) + (b6 ? 64u : 0u) + (b5 ? 32u : 0u) + (b4 ? 16u : 0u);
    // bottom four levels inside the 16-symbol block: all 16 words in one go
    uint32_t Wb[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) Wb[q] = w[(blk + q) * kDecThreads];
    uint32_t F8[8], F4[4], F2[2];  // freq candidates narrowed bit by bit
    f = (Wb[7] >> 16) * r;
    const bool b3 = f <= rem;
    if (b3) rem -= f;
#pragma unroll
    for (int i = 0; i < 8; ++i) F8[i] = b3 ? Wb[8 + i] : Wb[i];
    f = (F8[3] >> 16) * r;
    const bool b2 = f <= rem;
    if (b2) rem -= f;
#pragma unroll
    for (int i = 0; i < 4; ++i) F4[i] = b2 ? F8[4 + i] : F8[i];
    f = (F4[1] >> 16) * r;
    const bool b1 = f <= rem;
    if (b1) rem -= f;
#pragma unroll
    for (int i = 0; i < 2; ++i) F2[i] = b1 ? F4[2 + i] : F4[i];
    f = (F2[0] >> 16) * r;
    const bool b0 = f <= rem;
    if (b0) rem -= f;
    const uint32_t sl = (b3 ? 8u : 0u) + (b2 ? 4u : 0u) + (b1 ? 2u : 0u) + (b0 ? 1u : 0u);
    const uint32_t s = blk + sl;
    low = code - rem;                                      // low + r * cum(s)
    rng = r * ((b0 ? F2[1] : F2[0]) & 0xFFFFu);            // r * freq(s)
    for (;;) {                                             // fk/rangecoder.py:172-183
      if ((low ^ (low + rng)) >= kTop) {
        if (rng >= kBot) break;
        rng = (0u - low) & (kBot - 1);
      }
      code = (code << 8) | bs.next();
      low <<= 8;
      rng <<= 8;
    }
    pack = (pack >> 8) | (s << 24);  // 4 symbols per 32-bit store
    if ((k & 3) == 3) {
      if (aligned4) {
        *reinterpret_cast<uint32_t*>(out + (k - 3)) = pack;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) out[k - 3 + e] = (uint8_t)(pack >> (8 * e));
      }
    }
    // freq[s] += INC and the Fenwick path of s (fk/rangecoder.py:60-66, 185-186),
    // branch-free: the shared nodes below the block end (at most four: lowbits
    // 1, 2, 4, 8) as unconditional atomics (+0 when off the path), then every
    // register node covering s.
    {
      const uint32_t j0 = s + 1, j1 = j0 + lowbit(j0), j2 = j1 + lowbit(j1), j3 = j2 + lowbit(j2);
      const bool p0 = (j0 & 15) != 0, p1 = p0 && (j1 & 15), p2 = p1 && (j2 & 15),
                 p3 = p2 && (j3 & 15);
      atomicAdd(&w[s * kDecThreads], p0 ? ((kInc << 16) | kInc) : kInc);
      atomicAdd(&w[(p1 ? j1 - 1 : s) * kDecThreads], p1 ? kInc << 16 : 0u);
      atomicAdd(&w[(p2 ? j2 - 1 : s) * kDecThreads], p2 ? kInc << 16 : 0u);
      atomicAdd(&w[(p3 ? j3 - 1 : s) * kDecThreads], p3 ? kInc << 16 : 0u);
    }
#pragma unroll
    for (int q = 1; q < 16; ++q) {  // node 16q covers s in [16(q - lowbit(q)), 16q)
      const uint32_t lo = 16u * (uint32_t)(q - (q & -q)), len = 16u * (uint32_t)(q & -q);
      R[q] += (s - lo < len) ? kInc : 0u;
    }
    total += kInc;
    inv = inv_next;
    if (total >= kLimit) {
      total = rebuild(w, R);
      inv = 1.0 / (double)total;
    }
  }
  if (nsym & 3) {  // tail: the last nsym % 4 symbols sit in the top bytes of `pack`
    const uint32_t base = nsym & ~3u, n_tail = nsym & 3;
    for (uint32_t k = base; k < nsym; ++k) out[k] = (uint8_t)(pack >> (8 * (4 - n_tail + k - base)));
  }
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
  // One warp per CTA; its 32 models take 32 KB of shared memory, so seven CTAs
  // (224 streams) are resident per SM and the grid spreads over every SM.
  const size_t smem = (size_t)kDecThreads * 256 * sizeof(uint32_t);
  const int grid = (n_streams + kDecThreads - 1) / kDecThreads;
  rc_decode_kernel<<<grid, kDecThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(d_streams,
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
