// Memory-bound elementwise kernels (K8/K9/K13 + helpers), f32 and bf16.
//
// Replaces (reference pkg/src/nsk/):
//   elementwise()  tensor.py:247-283   -> nsk_eltwise        (add/sub/hadamard/scalar-*/relu/sigmoid/tanh/neg)
//   gradient_rule  autodiff.py:259-281 -> nsk_eltwise_bwd    (relu, sigmoid, tanh, scalar-mul, neg, hadamard)
//   bias_add       tensor.py:286-296   -> nsk_bias_add;  its rule (g, sum_rows g) autodiff.py:282-283 -> nsk_colsum
//   onehot         tensor.py:299-317   -> nsk_onehot (range errors reported through a device flag)
//   np.add(out=)   autodiff.py:359/384, GradCache.accumulate tensor.py:350 -> nsk_axpy
//   Pool poison / GradCache.zero_after_step tensor.py:98-99/360-364 -> nsk_fill_*
// Vectorised 16-byte accesses, grid sized to a multiple of the SM count.
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* p, float* f) {
    float4 v = *(const float4*)p;
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
  __device__ static void store(float* p, const float* f) { *(float4*)p = make_float4(f[0], f[1], f[2], f[3]); }
  __device__ static float ld1(const float* p) { return *p; }
  __device__ static void st1(float* p, float v) { *p = v; }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const __nv_bfloat16* p, float* f) {
    uint4 u = *(const uint4*)p;
    const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float* f) {
    uint4 u;
    u.x = pack_bf16x2(f[0], f[1]);
    u.y = pack_bf16x2(f[2], f[3]);
    u.z = pack_bf16x2(f[4], f[5]);
    u.w = pack_bf16x2(f[6], f[7]);
    *(uint4*)p = u;
  }
  __device__ static float ld1(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  __device__ static void st1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

__device__ __forceinline__ float stable_sigmoid(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  float e = expf(z);
  return e / (1.f + e);
}

__device__ __forceinline__ float ew_fwd(int kind, float a, float b, float s) {
  switch (kind) {
    case NSK_EW_ADD: return a + b;
    case NSK_EW_SUB: return a - b;
    case NSK_EW_HADAMARD: return a * b;
    case NSK_EW_SCALAR_ADD: return a + s;
    case NSK_EW_SCALAR_MUL: return a * s;
    case NSK_EW_RELU: return a > 0.f ? a : 0.f;
    case NSK_EW_SIGMOID: return stable_sigmoid(a);
    case NSK_EW_TANH: return tanhf(a);
    case NSK_EW_NEG: return -a;
    default: return a;  // COPY
  }
}

// g = incoming gradient, v = saved tensor
__device__ __forceinline__ float ew_bwd(int kind, float g, float v, float s) {
  switch (kind) {
    case NSK_EW_RELU: return v > 0.f ? g : 0.f;
    case NSK_EW_SIGMOID: return g * v * (1.f - v);
    case NSK_EW_TANH: return g * (1.f - v * v);
    case NSK_EW_SCALAR_MUL: return g * s;
    case NSK_EW_NEG: return -g;
    case NSK_EW_HADAMARD: return g * v;
    default: return g;
  }
}

constexpr bool binary(int k) { return k == NSK_EW_ADD || k == NSK_EW_SUB || k == NSK_EW_HADAMARD; }

template <typename T, bool BWD>
__global__ void ew_kernel(int kind, const T* __restrict__ a, const T* __restrict__ b, float s, T* __restrict__ out,
                          uint64_t n, bool vec) {
  pdl_wait();
  using V = Vec<T>;
  const bool needb = BWD ? (kind == NSK_EW_RELU || kind == NSK_EW_SIGMOID || kind == NSK_EW_TANH ||
                            kind == NSK_EW_HADAMARD)
                         : binary(kind);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    const uint64_t nv = n / V::N;
    for (uint64_t i = tid; i < nv; i += stride) {
      float fa[V::N], fb[V::N], fo[V::N];
      V::load(a + i * V::N, fa);
      if (needb) V::load(b + i * V::N, fb);
#pragma unroll
      for (int j = 0; j < V::N; ++j) fo[j] = BWD ? ew_bwd(kind, fa[j], needb ? fb[j] : 0.f, s)
                                                 : ew_fwd(kind, fa[j], needb ? fb[j] : 0.f, s);
      V::store(out + i * V::N, fo);
    }
    for (uint64_t i = nv * V::N + tid; i < n; i += stride) {
      float x = V::ld1(a + i), y = needb ? V::ld1(b + i) : 0.f;
      V::st1(out + i, BWD ? ew_bwd(kind, x, y, s) : ew_fwd(kind, x, y, s));
    }
  } else {
    for (uint64_t i = tid; i < n; i += stride) {
      float x = V::ld1(a + i), y = needb ? V::ld1(b + i) : 0.f;
      V::st1(out + i, BWD ? ew_bwd(kind, x, y, s) : ew_fwd(kind, x, y, s));
    }
  }
}

template <typename T>
__global__ void axpy_kernel(T* y, const T* __restrict__ x, float alpha, uint64_t n, bool vec) {
  pdl_wait();
  using V = Vec<T>;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t start = 0;
  if (vec) {
    const uint64_t nv = n / V::N;
    for (uint64_t i = tid; i < nv; i += stride) {
      float fy[V::N], fx[V::N];
      V::load(y + i * V::N, fy);
      V::load(x + i * V::N, fx);
#pragma unroll
      for (int j = 0; j < V::N; ++j) fy[j] += alpha * fx[j];
      V::store(y + i * V::N, fy);
    }
    start = nv * V::N;
  }
  for (uint64_t i = start + tid; i < n; i += stride) V::st1(y + i, V::ld1(y + i) + alpha * V::ld1(x + i));
}

template <typename T>
__global__ void fill_kernel(T* p, uint64_t n, float v) {
  pdl_wait();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) Vec<T>::st1(p + i, v);
}

template <typename S, typename D>
__global__ void cast_kernel(const S* __restrict__ s, D* __restrict__ d, uint64_t n) {
  pdl_wait();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    Vec<D>::st1(d + i, Vec<S>::ld1(s + i));
}

template <typename T>
__global__ void bias_add_kernel(const T* __restrict__ x, const float* __restrict__ b, T* __restrict__ out,
                                uint64_t rows, uint64_t cols) {
  pdl_wait();
  const uint64_t n = rows * cols;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    Vec<T>::st1(out + i, Vec<T>::ld1(x + i) + b[i % cols]);
}

// column sums (bias gradient): one block of 32x8 threads per 32 columns, rows strided over threadIdx.y,
// fixed-order shared-memory fold -> deterministic. out = sum (+ beta*out).
template <typename T>
__global__ void colsum_kernel(const T* __restrict__ g, float* __restrict__ out, uint64_t rows, uint64_t cols,
                              float beta) {
  pdl_wait();
  __shared__ float red[8][33];
  const uint64_t c = (uint64_t)blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (c < cols)
    for (uint64_t r = threadIdx.y; r < rows; r += 8) s += Vec<T>::ld1(g + r * cols + c);
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    out[c] = beta != 0.f ? t + beta * out[c] : t;
  }
}

__global__ void check_idx_kernel(const float* idx, uint64_t m, int classes, int* err) {
  pdl_wait();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    float v = idx[i];
    if (!(v >= 0.f && v < (float)classes && v == floorf(v))) atomicMin(err, (int)i);
  }
}

__global__ void onehot_kernel(const float* idx, uint64_t m, int classes, float* out) {
  pdl_wait();
  const uint64_t n = m * (uint64_t)classes;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = i / classes;
    int c = (int)(i - r * classes);
    out[i] = ((float)c == idx[r]) ? 1.f : 0.f;
  }
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ s, T* __restrict__ d, uint64_t rows, uint64_t cols) {
  pdl_wait();
  __shared__ T tile[32][33];
  uint64_t c = (uint64_t)blockIdx.x * 32 + threadIdx.x;
  uint64_t r = (uint64_t)blockIdx.y * 32 + threadIdx.y;
  for (int k = 0; k < 32; k += 8)
    if (r + k < rows && c < cols) tile[threadIdx.y + k][threadIdx.x] = s[(r + k) * cols + c];
  __syncthreads();
  c = (uint64_t)blockIdx.y * 32 + threadIdx.x;
  r = (uint64_t)blockIdx.x * 32 + threadIdx.y;
  for (int k = 0; k < 32; k += 8)
    if (r + k < cols && c < rows) d[(r + k) * rows + c] = tile[threadIdx.x][threadIdx.y + k];
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace

extern "C" {

int nsk_fill_f32(float* p, uint64_t n, float value, void* stream) {
  if (n == 0) return NSK_OK;
  nsk::launch_pdl(fill_kernel<float>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, p, n, value);
  NSK_LAUNCH_CHECK("fill_f32");
  return NSK_OK;
}

int nsk_fill_bf16(void* p, uint64_t n, float value, void* stream) {
  if (n == 0) return NSK_OK;
  nsk::launch_pdl(fill_kernel<__nv_bfloat16>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, (__nv_bfloat16*)p, n, value);
  NSK_LAUNCH_CHECK("fill_bf16");
  return NSK_OK;
}

int nsk_cast(int sdt, const void* src, int ddt, void* dst, uint64_t n, void* stream) {
  if (n == 0) return NSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned g = nsk::grid_for(n, 256);
  if (sdt == NSK_DTYPE_F32 && ddt == NSK_DTYPE_BF16)
    nsk::launch_pdl(cast_kernel<float, __nv_bfloat16>, g, 256, 0, st, (const float*)src, (__nv_bfloat16*)dst, n);
  else if (sdt == NSK_DTYPE_BF16 && ddt == NSK_DTYPE_F32)
    nsk::launch_pdl(cast_kernel<__nv_bfloat16, float>, g, 256, 0, st, (const __nv_bfloat16*)src, (float*)dst, n);
  else if (sdt == ddt)
    NSK_CUDA(cudaMemcpyAsync(dst, src, n * (sdt == NSK_DTYPE_F32 ? 4 : 2), cudaMemcpyDeviceToDevice, st));
  else
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "cast: bad dtypes");
  NSK_LAUNCH_CHECK("cast");
  return NSK_OK;
}

int nsk_eltwise(int kind, int dtype, const void* a, const void* b, float scalar, void* out, uint64_t n, void* stream) {
  if (n == 0) return NSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  bool vec = aligned16(a) && aligned16(out) && (!b || aligned16(b));
  if (dtype == NSK_DTYPE_F32)
    nsk::launch_pdl(ew_kernel<float, false>, nsk::grid_for(n, 256, 4), 256, 0, st, kind, (const float*)a, (const float*)b, scalar,
                                                                       (float*)out, n, vec);
  else
    nsk::launch_pdl(ew_kernel<__nv_bfloat16, false>, nsk::grid_for(n, 256, 8), 256, 0, st, 
        kind, (const __nv_bfloat16*)a, (const __nv_bfloat16*)b, scalar, (__nv_bfloat16*)out, n, vec);
  NSK_LAUNCH_CHECK("eltwise");
  return NSK_OK;
}

int nsk_eltwise_bwd(int kind, int dtype, const void* g, const void* saved, float scalar, void* out, uint64_t n,
                    void* stream) {
  if (n == 0) return NSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  bool vec = aligned16(g) && aligned16(out) && (!saved || aligned16(saved));
  if (dtype == NSK_DTYPE_F32)
    nsk::launch_pdl(ew_kernel<float, true>, nsk::grid_for(n, 256, 4), 256, 0, st, kind, (const float*)g, (const float*)saved,
                                                                      scalar, (float*)out, n, vec);
  else
    nsk::launch_pdl(ew_kernel<__nv_bfloat16, true>, nsk::grid_for(n, 256, 8), 256, 0, st, 
        kind, (const __nv_bfloat16*)g, (const __nv_bfloat16*)saved, scalar, (__nv_bfloat16*)out, n, vec);
  NSK_LAUNCH_CHECK("eltwise_bwd");
  return NSK_OK;
}

int nsk_axpy(int dtype, void* y, const void* x, float alpha, uint64_t n, void* stream) {
  if (n == 0) return NSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  bool vec = aligned16(y) && aligned16(x);
  if (dtype == NSK_DTYPE_F32)
    nsk::launch_pdl(axpy_kernel<float>, nsk::grid_for(n, 256, 4), 256, 0, st, (float*)y, (const float*)x, alpha, n, vec);
  else
    nsk::launch_pdl(axpy_kernel<__nv_bfloat16>, nsk::grid_for(n, 256, 8), 256, 0, st, (__nv_bfloat16*)y,
                                                                           (const __nv_bfloat16*)x, alpha, n, vec);
  NSK_LAUNCH_CHECK("axpy");
  return NSK_OK;
}

int nsk_bias_add(int dtype, const void* x, const float* b, void* out, uint64_t rows, uint64_t cols, void* stream) {
  uint64_t n = rows * cols;
  if (n == 0) return NSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == NSK_DTYPE_F32)
    nsk::launch_pdl(bias_add_kernel<float>, nsk::grid_for(n, 256), 256, 0, st, (const float*)x, b, (float*)out, rows, cols);
  else
    nsk::launch_pdl(bias_add_kernel<__nv_bfloat16>, nsk::grid_for(n, 256), 256, 0, st, (const __nv_bfloat16*)x, b,
                                                                            (__nv_bfloat16*)out, rows, cols);
  NSK_LAUNCH_CHECK("bias_add");
  return NSK_OK;
}

int nsk_colsum(int dtype, const void* g, float* out, uint64_t rows, uint64_t cols, float beta, void* stream) {
  if (cols == 0) return NSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)((cols + 31) / 32)), block(32, 8);
  if (dtype == NSK_DTYPE_F32)
    nsk::launch_pdl(colsum_kernel<float>, grid, block, 0, st, (const float*)g, out, rows, cols, beta);
  else
    nsk::launch_pdl(colsum_kernel<__nv_bfloat16>, grid, block, 0, st, (const __nv_bfloat16*)g, out, rows, cols, beta);
  NSK_LAUNCH_CHECK("colsum");
  return NSK_OK;
}

int nsk_check_indices(const float* idx, uint64_t m, int classes, int* err_flag, void* stream) {
  if (m == 0) return NSK_OK;
  nsk::launch_pdl(check_idx_kernel, nsk::grid_for(m, 256), 256, 0, (cudaStream_t)stream, idx, m, classes, err_flag);
  NSK_LAUNCH_CHECK("check_indices");
  return NSK_OK;
}

int nsk_onehot(const float* idx, uint64_t m, int classes, float* out, int* err_flag, void* stream) {
  if (err_flag) {
    int rc = nsk_check_indices(idx, m, classes, err_flag, stream);
    if (rc) return rc;
  }
  uint64_t n = m * (uint64_t)classes;
  if (n == 0) return NSK_OK;
  nsk::launch_pdl(onehot_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, idx, m, classes, out);
  NSK_LAUNCH_CHECK("onehot");
  return NSK_OK;
}

int nsk_transpose_2d(int dtype, const void* src, void* dst, uint64_t rows, uint64_t cols, void* stream) {
  if (rows == 0 || cols == 0) return NSK_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32)), block(32, 8);
  if (dtype == NSK_DTYPE_F32)
    nsk::launch_pdl(transpose_kernel<float>, grid, block, 0, (cudaStream_t)stream, (const float*)src, (float*)dst, rows, cols);
  else
    nsk::launch_pdl(transpose_kernel<__nv_bfloat16>, grid, block, 0, (cudaStream_t)stream, 
        (const __nv_bfloat16*)src, (__nv_bfloat16*)dst, rows, cols);
  NSK_LAUNCH_CHECK("transpose_2d");
  return NSK_OK;
}

}  // extern "C"
