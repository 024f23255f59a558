// kvf_api.cu — housekeeping entry points, plan validation, and whole-tensor
// quantize / dequantize (fk/kvmodel.py:127-152) for the C ABI in include/kvf.h.
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>

#include "kvf_common.cuh"

namespace kvf {

namespace {
thread_local char g_err[512] = "";
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

kvf_status cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return KVF_ECUDA;
}

size_t dtype_size(int32_t dt) {
  switch (dt) {
    case KVF_BF16:
    case KVF_F16:
      return 2;
    case KVF_F32:
      return 4;
    default:
      return 1;
  }
}

// Checks of LayoutConfig.__init__ (fk/layout.py:38-50), FramePlan.__init__
// (fk/layout.py:166-193) and plan_inter_frame (fk/layout.py:224-228).
static kvf_status validate_layout(const kvf_plan& p) {
  if (p.T < 1) KVF_FAIL(KVF_EINVAL, "T must be >= 1");
  if (p.F < 1) KVF_FAIL(KVF_EINVAL, "F must be >= 1");
  if (!is_pow2(p.H) || !is_pow2(p.D))
    KVF_FAIL(KVF_EINVAL, "H and D must be powers of two");
  if ((int64_t)p.a_h * p.b_h != p.H || (int64_t)p.a_d * p.b_d != p.D)
    KVF_FAIL(KVF_EINVAL, "factor pairs must multiply back to H and D");
  if (!is_pow2(p.a_h) || !is_pow2(p.b_h) || !is_pow2(p.a_d) || !is_pow2(p.b_d))
    KVF_FAIL(KVF_EINVAL, "factors must be powers of two");
  if (p.tiles_per_frame < 1) KVF_FAIL(KVF_EINVAL, "tiles_per_frame must be >= 1");
  if (p.grid_rows < 1 || p.grid_cols < 1 ||
      (int64_t)p.grid_rows * p.grid_cols != p.tiles_per_frame)
    KVF_FAIL(KVF_EINVAL, "tile grid %dx%d does not hold %d tiles", p.grid_rows,
             p.grid_cols, p.tiles_per_frame);
  int64_t C = (int64_t)p.H * p.D;
  if (p.group_size <= 0 || C % p.group_size != 0)
    KVF_FAIL(KVF_EINVAL, "group_size must be positive and divide channel");
  return KVF_OK;
}

static int32_t frame_count_of(const kvf_plan& p) {
  // frame_count = full*F + min(rem, F) if rem (fk/layout.py:189-193)
  int64_t seg_cap = (int64_t)p.F * p.tiles_per_frame;
  int64_t full = p.T / seg_cap, rem = p.T % seg_cap;
  return (int32_t)(full * p.F + (rem ? std::min<int64_t>(rem, p.F) : 0));
}

kvf_status check_plan(const kvf_plan& p) {
  kvf_status st = validate_layout(p);
  if (st != KVF_OK) return st;
  if (p.frame_h != p.grid_rows * p.a_h * p.a_d || p.frame_w != p.grid_cols * p.b_h * p.b_d ||
      p.frame_count != frame_count_of(p))
    KVF_FAIL(KVF_EINVAL, "plan derived fields inconsistent (call kvf_plan_init)");
  return KVF_OK;
}

namespace {

constexpr int kThreads = 256;

// Per-(layer, group) max |x| of a contiguous [T, L, C] tensor.
__global__ void tensor_absmax_kernel(const void* x, int32_t dtype, int64_t T,
                                     int32_t L, int32_t C, int32_t gs,
                                     uint32_t* absmax) {
  extern __shared__ uint32_t s_max[];
  const int l = blockIdx.y;
  const int G = C / gs;
  for (int k = threadIdx.x; k < G; k += blockDim.x) s_max[k] = 0u;
  __syncthreads();
  int64_t n = T * C;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e / C;
    int c = (int)(e - t * C);
    uint32_t v = absbits(load_as_float(x, (t * L + l) * C + c, dtype));
    if (v) atomicMax(&s_max[c / gs], v);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < G; k += blockDim.x)
    if (s_max[k]) atomicMax(&absmax[l * G + k], s_max[k]);
}

__global__ void tensor_scales_kernel(const uint32_t* absmax, float* scales, int n) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) scales[k] = scale_from_absmax_bits(absmax[k]);
}

__global__ void tensor_quantize_kernel(const void* x, int32_t dtype, int64_t n,
                                       int32_t L, int32_t C, int32_t gs,
                                       const float* scales, int8_t* values) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int64_t row = e / C;  // t*L + l
  int c = (int)(e - row * C);
  int l = (int)(row % L);
  float s = scales[l * (C / gs) + c / gs];
  values[e] = (int8_t)quantize_exact(load_as_float(x, e, dtype), s, __frcp_rn(s));
}

__global__ void tensor_dequantize_kernel(const int8_t* values, const float* scales,
                                         int64_t n, int32_t L, int32_t C, int32_t gs,
                                         void* out, int32_t out_dtype) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int64_t row = e / C;
  int c = (int)(e - row * C);
  int l = (int)(row % L);
  int q = values[e];
  // fp32 product == fp32(fp64(q) * fp64(s)): q has 8, s 24 significant bits.
  store_from_float(out, e, out_dtype, (float)q * scales[l * (C / gs) + c / gs], q);
}

kvf_status check_tensor(int64_t T, int32_t L, int32_t C, int32_t gs) {
  if (T < 1 || L < 1 || C < 1) KVF_FAIL(KVF_EINVAL, "all extents must be >= 1");
  if (gs <= 0 || C % gs != 0)
    KVF_FAIL(KVF_EINVAL, "group_size must be positive and divide channel");
  if ((int64_t)(C / gs) * sizeof(uint32_t) > 48 * 1024)
    KVF_FAIL(KVF_EUNSUPPORTED, "too many quantisation groups per layer");
  return KVF_OK;
}

}  // namespace
}  // namespace kvf

using namespace kvf;

extern "C" int32_t kvf_abi_version(void) { return KVF_ABI_VERSION; }

extern "C" const char* kvf_last_error(void) { return g_err; }

extern "C" kvf_status kvf_plan_init(kvf_plan* plan) {
  if (!plan) KVF_FAIL(KVF_EINVAL, "null plan");
  kvf_status st = validate_layout(*plan);
  if (st != KVF_OK) return st;
  plan->frame_h = plan->grid_rows * plan->a_h * plan->a_d;
  plan->frame_w = plan->grid_cols * plan->b_h * plan->b_d;
  plan->frame_count = frame_count_of(*plan);
  return KVF_OK;
}

extern "C" int64_t kvf_plan_frame_bytes(const kvf_plan* plan) {
  if (!plan || check_plan(*plan) != KVF_OK) return -1;
  return (int64_t)plan->frame_count * 3 * plan->frame_h * plan->frame_w;
}

extern "C" kvf_status kvf_quantize(const void* x, int32_t src_dtype, int64_t T,
                                   int32_t L, int32_t C, int32_t group_size,
                                   uint32_t* absmax, float* scales, int8_t* values,
                                   void* stream) {
  kvf_status st = check_tensor(T, L, C, group_size);
  if (st != KVF_OK) return st;
  if (src_dtype == KVF_I8 || src_dtype < 0 || src_dtype > KVF_I8)
    KVF_FAIL(KVF_EINVAL, "quantize needs a floating-point source");
  if (!x || !absmax || !scales || !values) KVF_FAIL(KVF_EINVAL, "null argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int G = C / group_size;
  KVF_CHECK_CUDA(cudaMemsetAsync(absmax, 0, sizeof(uint32_t) * L * G, s));
  int64_t per_layer = T * C;
  unsigned gx = (unsigned)std::min<int64_t>((per_layer + kThreads - 1) / kThreads, 4096);
  tensor_absmax_kernel<<<dim3(gx, L), kThreads, G * sizeof(uint32_t), s>>>(
      x, src_dtype, T, L, C, group_size, absmax);
  KVF_CHECK_CUDA(cudaGetLastError());
  tensor_scales_kernel<<<(L * G + kThreads - 1) / kThreads, kThreads, 0, s>>>(
      absmax, scales, L * G);
  KVF_CHECK_CUDA(cudaGetLastError());
  int64_t n = T * L * C;
  tensor_quantize_kernel<<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      x, src_dtype, n, L, C, group_size, scales, values);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}

extern "C" kvf_status kvf_dequantize(const int8_t* values, const float* scales,
                                     int64_t T, int32_t L, int32_t C,
                                     int32_t group_size, void* out, int32_t out_dtype,
                                     void* stream) {
  kvf_status st = check_tensor(T, L, C, group_size);
  if (st != KVF_OK) return st;
  if (out_dtype < 0 || out_dtype > KVF_I8) KVF_FAIL(KVF_EINVAL, "bad output dtype");
  if (!values || !scales || !out) KVF_FAIL(KVF_EINVAL, "null argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t n = T * L * C;
  tensor_dequantize_kernel<<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      values, scales, n, L, C, group_size, out, out_dtype);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}

namespace kvf {
namespace {
// x viewed as [outer, len, inner] fp32; in place x[o, t, i] = s*x[o, t-1, i] +
// (1-s)*x[o, t, i] for t >= 1 (the AR(1) law of gen_synthetic_kv,
// fk/kvmodel.py:176-188).  One thread per (outer, inner) series.
__global__ void ar1_scan_kernel(float* x, int64_t outer, int64_t len, int64_t inner,
                                float s) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= outer * inner) return;
  int64_t o = k / inner, i = k - o * inner;
  float* p = x + o * len * inner + i;
  float prev = p[0];
  for (int64_t t = 1; t < len; ++t) {
    float cur = s * prev + (1.0f - s) * p[t * inner];
    p[t * inner] = cur;
    prev = cur;
  }
}
}  // namespace
}  // namespace kvf

extern "C" kvf_status kvf_ar1_scan(float* x, int64_t outer, int64_t len, int64_t inner,
                                   float s, void* stream) {
  if (!x || outer < 1 || len < 1 || inner < 1) KVF_FAIL(KVF_EINVAL, "bad AR(1) extents");
  int64_t n = outer * inner;
  ar1_scan_kernel<<<(unsigned)((n + 255) / 256), 256, 0,
                    reinterpret_cast<cudaStream_t>(stream)>>>(x, outer, len, inner, s);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}
