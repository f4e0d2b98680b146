// Embedding gather / scatter-add (K15).
//
// Reference: the GRU input path is onehot(tokens) @ E (tensor.py:299-317 then matmul_t
// tensor.py:213-229, the substitution PAPER.md:173). The forward of onehot@E in float64 is an exact
// copy of row E[tok] (a one-term sum), so the gather is bit-identical to it; the backward
// dE = onehot^T @ dx is a scatter-add of dx rows into dE (fp32 atomics).
// Token ids arrive as float32 (the reference's data tensors are float32 with integer values, checked
// as in onehot). With seq_T > 0 the ids are [B][T] (batch-major, as loaded) and output rows are
// time-major: row t*B + b holds token [b][t].
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

__device__ __forceinline__ uint64_t src_index(uint64_t r, int seq_T, uint64_t n) {
  if (seq_T <= 0) return r;
  const uint64_t B = n / (uint64_t)seq_T;
  const uint64_t t = r / B, b = r - t * B;
  return b * (uint64_t)seq_T + t;
}

template <typename T>
__device__ __forceinline__ void stv(T* p, float v);
template <>
__device__ __forceinline__ void stv<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void stv<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
template <typename T>
__device__ __forceinline__ float ldv(const T* p);
template <>
__device__ __forceinline__ float ldv<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ldv<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T>
__global__ void embed_fwd_kernel(const float* __restrict__ table, const float* __restrict__ tok, uint64_t n, int E,
                                 int V, int seq_T, T* __restrict__ out, int* err) {
  pdl_wait();
  const uint64_t total = n * (uint64_t)E;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / E;
    const int e = (int)(i - r * E);
    const float tv = tok[src_index(r, seq_T, n)];
    const int t = (int)tv;
    if (!(tv >= 0.f && tv < (float)V && tv == floorf(tv))) {
      if (e == 0 && err) atomicMin(err, (int)r);
      stv<T>(out + i, 0.f);
    } else {
      stv<T>(out + i, table[(uint64_t)t * E + e]);
    }
  }
}

template <typename T>
__global__ void embed_bwd_kernel(const T* __restrict__ dout, const float* __restrict__ tok, uint64_t n, int E,
                                 int seq_T, float* dtable) {
  pdl_wait();
  const uint64_t total = n * (uint64_t)E;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / E;
    const int e = (int)(i - r * E);
    const int t = (int)tok[src_index(r, seq_T, n)];
    atomicAdd(dtable + (uint64_t)t * E + e, ldv<T>(dout + i));
  }
}

}  // namespace

extern "C" {

int nsk_embedding_fwd(const float* table, const float* tokens, uint64_t n, int E, int V, int seq_T, int dtype_out,
                      void* out, int* err_flag, void* stream) {
  uint64_t total = n * (uint64_t)E;
  if (!total) return NSK_OK;
  if (seq_T > 0 && n % (uint64_t)seq_T) return nsk::set_error(NSK_ERR_SHAPE, "embedding: n is not a multiple of T");
  if (dtype_out == NSK_DTYPE_F32)
    nsk::launch_pdl(embed_fwd_kernel<float>, nsk::grid_for(total, 256), 256, 0, (cudaStream_t)stream, table, tokens, n, E, V, seq_T,
                                                                                          (float*)out, err_flag);
  else
    nsk::launch_pdl(embed_fwd_kernel<__nv_bfloat16>, nsk::grid_for(total, 256), 256, 0, (cudaStream_t)stream, 
        table, tokens, n, E, V, seq_T, (__nv_bfloat16*)out, err_flag);
  NSK_LAUNCH_CHECK("embedding_fwd");
  return NSK_OK;
}

int nsk_embedding_bwd(const void* dout, int dtype_in, const float* tokens, uint64_t n, int E, int seq_T, float* dtable,
                      void* stream) {
  uint64_t total = n * (uint64_t)E;
  if (!total) return NSK_OK;
  if (dtype_in == NSK_DTYPE_F32)
    nsk::launch_pdl(embed_bwd_kernel<float>, nsk::grid_for(total, 256), 256, 0, (cudaStream_t)stream, (const float*)dout, tokens, n,
                                                                                          E, seq_T, dtable);
  else
    nsk::launch_pdl(embed_bwd_kernel<__nv_bfloat16>, nsk::grid_for(total, 256), 256, 0, (cudaStream_t)stream, 
        (const __nv_bfloat16*)dout, tokens, n, E, seq_T, dtable);
  NSK_LAUNCH_CHECK("embedding_bwd");
  return NSK_OK;
}

}  // extern "C"
