/*
 * abi_roundtrip.c — the C ABI of include/kvf.h used from plain C (no torch, no
 * Python): what a non-Python binding of the reference API would do.
 *
 * One Llama-shaped unit (T tokens x 3 layers x 8 heads x 128, bf16, contiguous
 * [T, 3, H, D]) is packed into frames (kvf_pack_batch: quantize + tile + place),
 * restored into int8 and bf16 paged caches through a shuffled block table
 * (kvf_restore_batch), and checked on the host: the int8 cache must hold the
 * codes the quantiser produced (kvf_quantize on the same input), the bf16 cache
 * RNE(code * scale).  Exit code 0 = pass.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "kvf.h"

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) {                                              \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 2;                                                           \
    }                                                                     \
  } while (0)
#define KV(x)                                                             \
  do {                                                                    \
    kvf_status s_ = (x);                                                  \
    if (s_ != KVF_OK) {                                                   \
      fprintf(stderr, "%s:%d kvf status %d: %s\n", __FILE__, __LINE__, s_, kvf_last_error()); \
      return 3;                                                           \
    }                                                                     \
  } while (0)

static uint16_t f32_to_bf16(float f) {  /* round to nearest even */
  uint32_t b;
  memcpy(&b, &f, 4);
  return (uint16_t)((b + 0x7FFF + ((b >> 16) & 1)) >> 16);
}
static float bf16_to_f32(uint16_t h) {
  uint32_t b = (uint32_t)h << 16;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

int main(void) {
  const int T = 333, H = 8, D = 128, C = H * D, GS = 128, G = C / GS, BS = 16;
  const int nblk = (T + BS - 1) / BS;
  if (kvf_abi_version() != KVF_ABI_VERSION) return 4;

  /* synthetic bf16 input: a smooth ramp plus a hash, so every group differs */
  size_t n = (size_t)T * 3 * C;
  uint16_t* hx = (uint16_t*)malloc(n * 2);
  for (size_t i = 0; i < n; ++i) {
    uint32_t h = (uint32_t)i * 2654435761u;
    hx[i] = f32_to_bf16(((float)((h >> 8) % 2001) - 1000.0f) / 333.0f);
  }
  void *x, *frames, *cache8, *cache16;
  uint32_t *absmax, *qabs;
  float *scales, *qscales;
  int8_t* codes;
  int32_t* table;
  kvf_plan plan;
  memset(&plan, 0, sizeof plan);
  plan.T = T; plan.H = H; plan.D = D; plan.a_h = 1; plan.b_h = H; plan.a_d = 1; plan.b_d = D;
  plan.F = 4; plan.tiles_per_frame = 16; plan.grid_rows = 4; plan.grid_cols = 4;
  plan.group_size = GS;
  KV(kvf_plan_init(&plan));
  const int64_t fbytes = kvf_plan_frame_bytes(&plan);
  const int64_t scratch = kvf_pack_scratch_words(&plan);
  CK(cudaMalloc(&x, n * 2));
  CK(cudaMalloc(&frames, fbytes));
  CK(cudaMalloc((void**)&absmax, scratch * 4));
  CK(cudaMalloc((void**)&scales, 3 * G * 4));
  CK(cudaMalloc((void**)&qabs, 3 * G * 4));
  CK(cudaMalloc((void**)&qscales, 3 * G * 4));
  CK(cudaMalloc((void**)&codes, n));
  CK(cudaMalloc(&cache8, (size_t)3 * (nblk + 3) * BS * C));
  CK(cudaMalloc(&cache16, (size_t)3 * (nblk + 3) * BS * C * 2));
  CK(cudaMalloc((void**)&table, nblk * 4));
  CK(cudaMemcpy(x, hx, n * 2, cudaMemcpyHostToDevice));
  int32_t* htab = (int32_t*)malloc(nblk * 4);
  for (int b = 0; b < nblk; ++b) htab[b] = (b * 7 + 3) % (nblk + 3); /* a permutation's prefix */
  for (int b = 0; b < nblk; ++b)
    for (int c = 0; c < b; ++c)
      if (htab[b] == htab[c]) return 5; /* not injective: bad test setup */
  CK(cudaMemcpy(table, htab, nblk * 4, cudaMemcpyHostToDevice));

  /* pack: the unit reads layers 0..2 of the contiguous [T, 3, H, D] tensor */
  kvf_pack_unit pu;
  memset(&pu, 0, sizeof pu);
  for (int p = 0; p < 3; ++p) pu.src.layer[p] = (char*)x + (size_t)p * C * 2;
  pu.src.block_size = 1;
  pu.src.dtype = KVF_BF16;
  pu.src.block_stride = pu.src.slot_stride = 3 * C;
  pu.src.head_stride = D;
  pu.plan = plan;
  pu.absmax = absmax;
  pu.scales = scales;
  pu.frames.base = (uint8_t*)frames;
  pu.frames.row_pitch = plan.frame_w;
  pu.frames.plane_stride = (int64_t)plan.frame_w * plan.frame_h;
  pu.frames.frame_stride = 3 * pu.frames.plane_stride;
  KV(kvf_pack_batch(&pu, 1, NULL));
  /* reference codes: whole-tensor quantize of the same input ([T, 3, C]) */
  KV(kvf_quantize(x, KVF_BF16, T, 3, C, GS, qabs, qscales, codes, NULL));

  /* restore into int8 and bf16 paged caches [3 layers][blocks][BS][H][D] */
  int ok = 1;
  for (int mode = 0; mode < 2; ++mode) {
    kvf_restore_unit ru;
    memset(&ru, 0, sizeof ru);
    ru.frames = pu.frames;
    ru.plan = plan;
    ru.scales = scales;
    const int es = mode ? 2 : 1;
    char* cache = (char*)(mode ? cache16 : cache8);
    for (int p = 0; p < 3; ++p) ru.dst.layer[p] = cache + (size_t)p * (nblk + 3) * BS * C * es;
    ru.dst.block_table = table;
    ru.dst.block_size = BS;
    ru.dst.dtype = mode ? KVF_BF16 : KVF_I8;
    ru.dst.block_stride = (int64_t)BS * C;
    ru.dst.slot_stride = C;
    ru.dst.head_stride = D;
    ru.first_frame = 0;
    ru.n_frames = plan.frame_count;
    KV(kvf_restore_batch(&ru, 1, NULL));
  }
  CK(cudaDeviceSynchronize());

  int8_t* hcodes = (int8_t*)malloc(n);
  float* hsc = (float*)malloc(3 * G * 4);
  float* hqsc = (float*)malloc(3 * G * 4);
  size_t csz = (size_t)3 * (nblk + 3) * BS * C;
  int8_t* h8 = (int8_t*)malloc(csz);
  uint16_t* h16 = (uint16_t*)malloc(csz * 2);
  CK(cudaMemcpy(hcodes, codes, n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hsc, scales, 3 * G * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hqsc, qscales, 3 * G * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h8, cache8, csz, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h16, cache16, csz * 2, cudaMemcpyDeviceToHost));
  if (memcmp(hsc, hqsc, 3 * G * 4) != 0) ok = 0, fprintf(stderr, "scales differ\n");
  long bad8 = 0, bad16 = 0;
  for (int t = 0; t < T; ++t)
    for (int p = 0; p < 3; ++p)
      for (int c = 0; c < C; ++c) {
        const size_t slot = ((size_t)p * (nblk + 3) + htab[t / BS]) * BS * C + (size_t)(t % BS) * C + c;
        const int8_t q = hcodes[((size_t)t * 3 + p) * C + c];
        if (h8[slot] != q) ++bad8;
        if (h16[slot] != f32_to_bf16((float)q * hsc[p * G + c / GS])) ++bad16;
      }
  if (bad8 || bad16) ok = 0;
  printf("abi_roundtrip: T=%d frames=%d int8 mismatches=%ld bf16 mismatches=%ld -> %s\n", T,
         plan.frame_count, bad8, bad16, ok ? "PASS" : "FAIL");
  (void)bf16_to_f32;
  return ok ? 0 : 1;
}
