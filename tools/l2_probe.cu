// l2_probe.cu — does a re-read of recently read data hit the B200 L2?
//
// touch: SM s reads chunk s of a buffer (persistent grid, one CTA per SM,
// chunk chosen by %smid); reread: SM s reads chunk (s + shift) % 148.
// Run under ncu and compare dram__bytes_read.sum of the reread launch with the
// buffer size, for several sizes, shifts (same SM / same die / other die) and
// load flavours.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_probe tools/l2_probe.cu
//   ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct /tmp/l2_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ uint32_t g_sink;

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

template <int FLAVOR>
__device__ __forceinline__ uint4 load(const void* p, uint64_t pol) {
  uint4 v;
  if (FLAVOR == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (FLAVOR == 1)
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}

// Reads chunk ((smid + shift) % n_chunks) of `buf` (chunk = bytes / n_chunks).
template <int FLAVOR>
__global__ void __launch_bounds__(1024) read_chunk(const uint8_t* buf, int64_t chunk, int shift,
                                                   int n_chunks, int evict_last) {
  uint64_t pol;
  if (evict_last)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int c = (int)((smid() + shift) % n_chunks);
  const uint8_t* p = buf + c * chunk;
  uint32_t acc = 0;
  for (int64_t o = (int64_t)threadIdx.x * 16; o < chunk; o += 1024 * 16) {
    uint4 v = load<FLAVOR>(p + o, pol);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) g_sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t max_bytes = 256ll << 20;
  uint8_t* buf;
  uint8_t* flush;
  cudaMalloc(&buf, max_bytes);
  cudaMalloc(&flush, 512ll << 20);
  cudaMemset(buf, 1, max_bytes);
  cudaFuncSetAttribute(read_chunk<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 << 10);
  cudaFuncSetAttribute(read_chunk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 << 10);
  cudaFuncSetAttribute(read_chunk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 << 10);
  const int sizes_mb[] = {8, 16, 32, 48, 64, 96};
  const int shifts[] = {0, 1, 74};
  for (int flavor = 0; flavor < 3; ++flavor)
    for (int sz : sizes_mb)
      for (int sh : shifts) {
        const int64_t bytes = (int64_t)sz << 20;
        const int64_t chunk = (bytes / sms) & ~int64_t(16383);
        cudaMemset(flush, 0, 512ll << 20);  // evict everything
        // touch (shift 0) then re-read (shift sh): ncu reports both launches
        // 150 KB of dynamic shared memory: one CTA per SM, so %smid picks
        // every chunk exactly once
        const size_t smem = 150 << 10;
        auto launch = [&](int shift) {
          if (flavor == 0) read_chunk<0><<<sms, 1024, smem>>>(buf, chunk, shift, sms, 1);
          if (flavor == 1) read_chunk<1><<<sms, 1024, smem>>>(buf, chunk, shift, sms, 1);
          if (flavor == 2) read_chunk<2><<<sms, 1024, smem>>>(buf, chunk, shift, sms, 1);
        };
        launch(0);
        launch(sh);
        cudaDeviceSynchronize();
        printf("flavor %d size_mb %d shift %d chunk %lld\n", flavor, sz, sh, (long long)chunk);
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(e));
  return 0;
}
