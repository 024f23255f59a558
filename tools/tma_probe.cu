// tools/tma_probe.cu — TMA streaming-read probe on one B200 (measurement tool).
// One CTA per SM streams boxes of a [T, 3, 8, 128] bf16 tensor (the bench's
// contiguous C2 source: 6 KB token stride) through a ring of shared-memory
// slots: a producer thread issues cp.async.bulk.tensor, a consumer warp waits
// and releases (optionally reading every byte).  Prints GB/s per box shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
}
struct Args { CUtensorMap map; int n_items; int box_tok; int box_ch; int ch_groups; int slot_bytes; int nslots; int touch; int four_d; int hint; };

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ Args A, unsigned long long* sink) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) uint64_t full[64], empty[64];
  if (threadIdx.x < A.nslots) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[threadIdx.x])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[threadIdx.x])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int per = (A.n_items + gridDim.x - 1) / gridDim.x;
  const int k0 = blockIdx.x * per, k1 = min(A.n_items, k0 + per);
  if (threadIdx.x == 0) {
    for (int k = k0; k < k1; ++k) {
      int i = k - k0, s = i % A.nslots, r = i / A.nslots;
      if (r > 0) wait(&empty[s], (r - 1) & 1);
      int g = k % A.ch_groups, t = (k / A.ch_groups) * A.box_tok;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(A.slot_bytes) : "memory");
      if (A.four_d) {
        uint64_t pol;
        if (A.hint) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
                     ::"r"(sa(ring + s * A.slot_bytes)), "l"((unsigned long long)&A.map), "r"(0), "r"(g), "r"(0), "r"(t), "r"(sa(&full[s])), "l"(pol) : "memory");
      } else {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sa(ring + s * A.slot_bytes)), "l"((unsigned long long)&A.map), "r"(g * A.box_ch), "r"(0), "r"(t), "r"(sa(&full[s])) : "memory");
      }
    }
  } else if (threadIdx.x >= 32) {
    unsigned long long acc = 0;
    for (int k = k0; k < k1; ++k) {
      int i = k - k0, s = i % A.nslots, r = i / A.nslots;
      wait(&full[s], r & 1);
      if (A.touch) {
        const uint4* p = reinterpret_cast<const uint4*>(ring + s * A.slot_bytes);
        for (int e = threadIdx.x - 32; e < A.slot_bytes / 16; e += 32) acc += p[e].x;
      }
      __syncwarp();
      if (threadIdx.x == 32) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
    if (acc == 12345) sink[0] = acc;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const long T = 32768 * 11;  // tokens (rows of 3 planes x 1024 ch)
  void* src; cudaMalloc(&src, T * 3 * 1024 * 2); cudaMemset(src, 1, T * 3 * 1024 * 2);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int box_ch, box_tok, nslots, touch, four_d, hint; };
  std::vector<Cfg> cfgs = {{128, 32, 12, 0, 0, 0}, {128, 32, 12, 0, 1, 0}, {128, 32, 12, 0, 1, 1}, {128, 32, 12, 1, 1, 1}};
  for (int grid : {16, 128, 148})
  for (auto c : cfgs) {
    Args A;
    cuuint64_t gdim[3] = {1024, 3, (cuuint64_t)T};       // channels, planes, tokens (plane 0 only used)
    cuuint64_t gstr[2] = {2048, 6144};
    cuuint32_t box[3] = {(cuuint32_t)c.box_ch, 1, (cuuint32_t)c.box_tok};
    cuuint32_t es[3] = {1, 1, 1};
    cuuint64_t gdim4[4] = {128, 8, 1, (cuuint64_t)T};
    cuuint64_t gstr4[3] = {256, 6144, 6144};
    cuuint32_t box4[4] = {128, 1, 1, (cuuint32_t)c.box_tok};
    cuuint32_t es4[4] = {1, 1, 1, 1};
    A.four_d = c.four_d; A.hint = c.hint;
    CUresult r = c.four_d ? enc(&A.map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, src, gdim4, gstr4, box4, es4,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                          : enc(&A.map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, src, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode %d\n", r); continue; }
    A.box_ch = c.box_ch; A.box_tok = c.box_tok; A.ch_groups = 1024 / c.box_ch;
    A.slot_bytes = c.box_ch * c.box_tok * 2; A.nslots = c.nslots; A.touch = c.touch;
    A.n_items = (int)(T / c.box_tok) * A.ch_groups;
    if (grid < sms) A.n_items = A.n_items * grid / sms / 4;  // small grids: L2-resident re-reads
    int smem = A.slot_bytes * c.nslots;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      probe<<<grid, 64, smem>>>(A, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)A.n_items * A.slot_bytes;
    printf("4d %d hint %d | grid %3d per-SM %.1f GB/s | box %4d ch x %3d tok  slot %6d B  slots %2d touch %d : %.3f ms  %.0f GB/s  (%s)\n", c.four_d, c.hint, grid, bytes / ms / 1e6 / grid, c.box_ch, c.box_tok,
           A.slot_bytes, c.nslots, c.touch, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
