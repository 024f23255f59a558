// kvf_kvfc_enc.cu — KVFC frame-stream encode on the GPU, sm_100a.
//
// 1. resid_kernel: one thread per 16x16 block of one frame plane: intra and
//    inter residual SADs, mode = inter iff SAD_inter <= SAD_intra, then the
//    zigzag symbols of the chosen residual (fk/codec.py:77-123).
// 2. rc_encode_kernel: the reference's adaptive range encoder
//    (fk/rangecoder.py:106-143), one thread per (frame, plane) stream, with the
//    same packed Fenwick model in shared memory as the decoder (kvf_kvfc.cu).
// 3. gather_kernel: scatters payloads and packed mode bitmaps into the final
//    stream buffer at host-computed offsets (fk/codec.py:16-20 layout).
#include <algorithm>

#include "kvf_common.cuh"

namespace kvf {
namespace {

constexpr uint32_t kTop = 1u << 24;
constexpr uint32_t kBot = 1u << 16;
constexpr uint32_t kInc = 32;
constexpr uint32_t kLimit = 1u << 16;

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

__global__ void __launch_bounds__(224)
    rc_encode_kernel(const kvf_rc_stream* __restrict__ streams, int n, int64_t* out_len) {
  extern __shared__ uint32_t W[];  // [256][blockDim.x], W[i] = fen[i+1] << 16 | freq[i]
  const int nt = blockDim.x, tid = threadIdx.x;
  const int sidx = blockIdx.x * nt + tid;
  if (sidx >= n) return;
  const kvf_rc_stream st = streams[sidx];
#define MW(i) W[(i) * nt + tid]
  for (int i = 0; i < 256; ++i) {
    const int j = i + 1;
    MW(i) = ((uint32_t)(j & -j) << 16) | 1u;
  }
  uint32_t total = 256, low = 0, rng = 0xFFFFFFFFu;
  uint8_t* out = const_cast<uint8_t*>(st.payload);
  int64_t n_out = 0;
  const uint8_t* sym = st.symbols;
  for (int64_t k = 0; k < st.n_symbols; ++k) {
    const uint32_t s = __ldg(sym + k);
    uint32_t cum = 0;  // Fenwick prefix sum of freq[0..s-1]
    for (uint32_t j = s; j > 0; j -= j & (0u - j)) cum += MW(j - 1) >> 16;
    const uint32_t fr = MW(s) & 0xFFFFu;
    const uint32_t r = rng / total;
    low += r * cum;
    rng = r * fr;
    for (;;) {
      if ((low ^ (low + rng)) >= kTop) {
        if (rng >= kBot) break;
        rng = (0u - low) & (kBot - 1);
      }
      out[n_out++] = (uint8_t)(low >> 24);
      low <<= 8;
      rng <<= 8;
    }
    MW(s) += (kInc << 16) | kInc;
    for (uint32_t j = (s + 1) + ((s + 1) & (0u - (s + 1))); j <= 255; j += j & (0u - j))
      MW(j - 1) += kInc << 16;
    total += kInc;
    if (total >= kLimit) {
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
  for (int k = 0; k < 4; ++k) {  // flush: four bytes pin down the final interval
    out[n_out++] = (uint8_t)(low >> 24);
    low <<= 8;
  }
  out_len[sidx] = n_out;
#undef MW
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
  int dev = 0, sms = 0;
  KVF_CHECK_CUDA(cudaGetDevice(&dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int per = (n_streams + sms - 1) / sms;
  per = std::min(224, std::max(32, (per + 31) / 32 * 32));
  const size_t smem = (size_t)per * 256 * sizeof(uint32_t);
  KVF_CHECK_CUDA(cudaFuncSetAttribute(rc_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(224 * 256 * sizeof(uint32_t))));
  const int grid = (n_streams + per - 1) / per;
  rc_encode_kernel<<<grid, per, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
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
