// kvf_kvfc_enc.cu — KVFC frame-stream encode on the GPU, sm_100a.
//
// 1. resid_kernel: one thread per 16x16 block of one frame plane: intra and
//    inter residual SADs, mode = inter iff SAD_inter <= SAD_intra, then the
//    zigzag symbols of the chosen residual (fk/codec.py:77-123).
// 2. rc_encode_kernel: the reference's adaptive range encoder
//    (fk/rangecoder.py:106-143), one thread per (frame, plane) stream, on the
//    decoder's cumulative-count model (kvf_rc_model.cuh).
// 3. gather_kernel: scatters payloads and packed mode bitmaps into the final
//    stream buffer at host-computed offsets (fk/codec.py:16-20 layout).
#include <algorithm>

#include "kvf_rc_model.cuh"

namespace kvf {
namespace {

using rc::kBot;
using rc::kInc;
using rc::kLimit;
using rc::kTop;

__device__ __forceinline__ uint32_t zig(int r) {
  const int s = (int)(int8_t)(uint8_t)(r & 0xFF);  // residual mod 256 as signed byte
  return s >= 0 ? (uint32_t)(2 * s) : (uint32_t)(-2 * s - 1);
}

__global__ void resid_kernel(const kvf_resid_plane* __restrict__ planes) {
  const kvf_resid_plane P = planes[blockIdx.x];  // planes on x: up to 2^31 - 1 of them
  const int bw = (P.width + 15) / 16, bh = (P.height + 15) / 16;
  const int b = blockIdx.y * blockDim.x + threadIdx.x;
  if (b >= bw * bh) return;
  const int by = b / bw, bx = b - by * bw;
  const int y0 = by * 16, x0 = bx * 16;
  const int y1 = min(y0 + 16, P.height), x1 = min(x0 + 16, P.width);
  const uint8_t* cur = P.cur;
  const uint8_t* prev = P.prev;
  auto intra = [&](int y, int x) -> int {
    const int v = cur[(int64_t)y * P.pitch + x];
    if (x > 0) return v - cur[(int64_t)y * P.pitch + x - 1];
    if (y > 0) return v - cur[(int64_t)(y - 1) * P.pitch];
    return v - 128;
  };
  bool inter = false;
  if (prev) {
    int64_t sad_a = 0, sad_e = 0;  // intra, inter
    for (int y = y0; y < y1; ++y)
      for (int x = x0; x < x1; ++x) {
        sad_a += abs(intra(y, x));
        sad_e += abs((int)cur[(int64_t)y * P.pitch + x] - (int)prev[(int64_t)y * P.pitch + x]);
      }
    inter = sad_e <= sad_a;  // ties go to inter (fk/codec.py:113-118)
    P.modes[b] = inter ? 1 : 0;
  }
  for (int y = y0; y < y1; ++y)
    for (int x = x0; x < x1; ++x) {
      const int r = inter ? (int)cur[(int64_t)y * P.pitch + x] - (int)prev[(int64_t)y * P.pitch + x]
                          : intra(y, x);
      P.symbols[(int64_t)y * P.width + x] = (uint8_t)zig(r);
    }
}

// The encoder runs the decoder's model (kvf_rc_model.cuh): a symbol's cum and
// count come straight from its block (two u16 reads), the division is the exact
// fp32 one, the "top byte settled" output phase is clz(low ^ (low + rng)) / 8
// bytes at once, and output bytes collect in a 64-bit accumulator so a 4-byte
// aligned stream is written a word at a time.
__global__ void __launch_bounds__(rc::kDecThreads)
    rc_encode_kernel(const kvf_rc_stream* __restrict__ streams, int n, int64_t* out_len) {
  using namespace rc;
  extern __shared__ uint4 M[];  // [32 chunks][kDecThreads] x 16 B, as the decoder's
  __shared__ uint4 T_add[2 * kAddRows];  // increment rows (rc::add_table_init)
  add_table_init(T_add);       // the whole warp, before any thread leaves
  const int tid = threadIdx.x;
  const int sidx = blockIdx.x * kDecThreads + tid;
  if (sidx >= n) return;
  const kvf_rc_stream st = streams[sidx];
  uint4* m = M + tid;
  uint32_t P[8];  // block prefixes CB[2w] | CB[2w+1] << 16
  model_init(m, P);
  uint32_t total = 256, low = 0, rng = 0xFFFFFFFFu;
  uint8_t* out = const_cast<uint8_t*>(st.payload);
  const bool aligned4 = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  uint64_t acc = 0;    // pending output bytes, first byte lowest
  uint32_t pend = 0;   // number of pending bytes (< 4 between symbols)
  int64_t n_out = 0;   // bytes written to `out`
  auto emit = [&](uint32_t v, uint32_t nb) {  // v: nb bytes, first in the low byte
    acc |= (uint64_t)v << (8 * pend);
    pend += nb;
    if (pend >= 4) {
      if (aligned4) {
        *reinterpret_cast<uint32_t*>(out + n_out) = (uint32_t)acc;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) out[n_out + e] = (uint8_t)(acc >> (8 * e));
      }
      n_out += 4;
      acc >>= 32;
      pend -= 4;
    }
  };
  const uint8_t* sym = st.symbols;
  const uint32_t nsym = (uint32_t)st.n_symbols;
  float rcp = rcp_approx(total);
  for (uint32_t k = 0; k < nsym; ++k) {
    const uint32_t s = __ldg(sym + k);
    const float rcp_next = rcp_approx(total + kInc);
    const uint32_t blk = s >> 4, sl = s & 15;
    const uint4 ca = m[(2 * blk) * kDecThreads], cb = m[(2 * blk + 1) * kDecThreads];
    const uint32_t wv[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    // incl[sl] and incl[sl - 1] (0 at sl = 0): two direct u16 loads
    const uint16_t* m16 = reinterpret_cast<const uint16_t*>(m);
    const uint32_t hi_v = m16[((2 * blk + (sl >> 3)) * kDecThreads) * 8 + (sl & 7)];
    const uint32_t j1 = sl - 1;  // wraps for sl == 0 (value unused then)
    const uint32_t lo_raw = m16[((2 * blk + ((j1 >> 3) & 1)) * kDecThreads) * 8 + (j1 & 7)];
    const uint32_t lo_v = sl == 0 ? 0u : lo_raw;
    // CB[blk]: a 3-level select tree picks the packed word P[blk >> 1], the
    // low bit of blk its half
    uint32_t base;
    {
      const bool k3 = blk & 8, k2 = blk & 4, k1 = blk & 2;
      uint32_t e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = k3 ? P[4 + i] : P[i];
      const uint32_t f0 = k2 ? e[2] : e[0], f1 = k2 ? e[3] : e[1];
      const uint32_t w = k1 ? f1 : f0;
      base = (blk & 1) ? cb_hi(w) : cb_lo(w);
    }
    const uint4 cbi[2] = {T_add[2 * (blk + 1)], T_add[2 * (blk + 1) + 1]};
    const uint32_t cum = base + lo_v, fr = hi_v - lo_v;     // fk/rangecoder.py:114-115
    const uint32_t r = exact_div(rng, total, rcp);          // fk/rangecoder.py:117
    low += r * cum;
    rng = r * fr;
    {  // fk/rangecoder.py:120-131: settled top bytes, then (rarely) squeezes
      const uint32_t nb = __clz(low ^ (low + rng)) >> 3;
      if (nb) {
        emit(__byte_perm(low, 0u, 0x0123) & ((1u << (8 * nb)) - 1u), nb);
        low <<= 8 * nb;
        rng <<= 8 * nb;
      }
      while (rng < kBot || (low ^ (low + rng)) < kTop) {
        if ((low ^ (low + rng)) >= kTop) rng = (0u - low) & (kBot - 1);
        emit(low >> 24, 1);
        low <<= 8;
        rng <<= 8;
      }
    }
    model_update(m, P, blk, sl, wv, T_add, cbi);            // fk/rangecoder.py:133-135
    total += kInc;
    rcp = rcp_next;
    if (total >= kLimit) {                                  // fk/rangecoder.py:136-137
      total = rebuild(m, P);
      rcp = rcp_approx(total);
    }
  }
  for (int k = 0; k < 4; ++k) {  // flush: four bytes pin down the final interval
    emit(low >> 24, 1);
    low <<= 8;
  }
  for (uint32_t e = 0; e < pend; ++e) out[n_out + e] = (uint8_t)(acc >> (8 * e));
  out_len[sidx] = n_out + pend;
}

__global__ void gather_kernel(const kvf_piece* __restrict__ pieces, uint8_t* dst) {
  const kvf_piece P = pieces[blockIdx.x];
  if (!P.pack_bits) {
    for (int64_t i = threadIdx.x; i < P.len; i += blockDim.x) dst[P.dst_off + i] = P.src[i];
  } else {
    const int64_t nbytes = (P.len + 7) / 8;
    for (int64_t i = threadIdx.x; i < nbytes; i += blockDim.x) {
      uint32_t v = 0;
      for (int k = 0; k < 8; ++k) {
        const int64_t b = i * 8 + k;
        if (b < P.len && P.src[b]) v |= 0x80u >> k;
      }
      dst[P.dst_off + i] = (uint8_t)v;
    }
  }
}

}  // namespace
}  // namespace kvf

using namespace kvf;

extern "C" kvf_status kvf_kvfc_residuals(const kvf_resid_plane* d_planes, int32_t n_planes,
                                         int32_t max_blocks, void* stream) {
  if (n_planes < 0 || max_blocks < 0 || (n_planes > 0 && !d_planes))
    KVF_FAIL(KVF_EINVAL, "bad residual plane array");
  if (n_planes == 0 || max_blocks == 0) return KVF_OK;
  if ((max_blocks + 127) / 128 > 65535) KVF_FAIL(KVF_EUNSUPPORTED, "plane too large");
  dim3 grid((unsigned)n_planes, (unsigned)((max_blocks + 127) / 128));
  resid_kernel<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_planes);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}

extern "C" kvf_status kvf_rc_encode(const kvf_rc_stream* d_streams, int32_t n_streams,
                                    int64_t* d_out_len, void* stream) {
  if (n_streams < 0 || (n_streams > 0 && (!d_streams || !d_out_len)))
    KVF_FAIL(KVF_EINVAL, "bad stream array");
  if (n_streams == 0) return KVF_OK;
  // one warp per CTA, 16 KB of models (the decoder's layout)
  const size_t smem = (size_t)rc::kDecThreads * 256 * sizeof(uint16_t);
  const int grid = (n_streams + rc::kDecThreads - 1) / rc::kDecThreads;
  rc_encode_kernel<<<grid, rc::kDecThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      d_streams, n_streams, d_out_len);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}

extern "C" kvf_status kvf_gather(const kvf_piece* d_pieces, int32_t n_pieces, uint8_t* dst,
                                 void* stream) {
  if (n_pieces < 0 || (n_pieces > 0 && (!d_pieces || !dst))) KVF_FAIL(KVF_EINVAL, "bad pieces");
  if (n_pieces == 0) return KVF_OK;
  gather_kernel<<<n_pieces, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_pieces, dst);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}
