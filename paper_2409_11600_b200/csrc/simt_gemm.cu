// SIMT GEMM with fp64 accumulation for small or unaligned f32 problems.
//
// The reference accumulates matmul_t / plain_matmul in float64 and casts to
// float32 on store (pkg/src/nsk/tensor.py:213-234). Shapes too small or too
// ragged for TMA (row pitch not a multiple of 16 bytes, e.g. the 1x2 @ 1x2
// known-answer test tensor.py / test_tensor.py:124-130) run here instead of on
// the tensor cores; the result then matches the reference to f32 rounding.
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

constexpr int TS = 16;

__global__ void simt_gemm_kernel(int a_mn, int b_mn, int M, int N, int K, const float* __restrict__ A, long long lda,
                                 const float* __restrict__ B, long long ldb, float* C, long long ldc,
                                 const float* __restrict__ bias, float beta) {
  pdl_wait();
  __shared__ float As[TS][TS + 1];
  __shared__ float Bs[TS][TS + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int m = blockIdx.y * TS + ty;
  const int n = blockIdx.x * TS + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += TS) {
    {
      int mm = blockIdx.y * TS + ty, kk = k0 + tx;
      As[ty][tx] = (mm < M && kk < K) ? (a_mn ? A[(long long)kk * lda + mm] : A[(long long)mm * lda + kk]) : 0.f;
      int nn = blockIdx.x * TS + ty;
      Bs[ty][tx] = (nn < N && kk < K) ? (b_mn ? B[(long long)kk * ldb + nn] : B[(long long)nn * ldb + kk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TS; ++k) acc += (double)As[ty][k] * (double)Bs[tx][k];
    __syncthreads();
  }
  if (m < M && n < N) {
    if (bias) acc += (double)bias[n];
    float* c = C + (long long)m * ldc + n;
    float r = (float)acc;
    *c = beta != 0.f ? r + beta * *c : r;
  }
}

// Skinny products (few outputs, long K: the classifier layer and its weight gradient): one warp per output,
// lanes stride K (coalesced along K-major rows), float64 warp reduction.
__global__ void simt_dot_kernel(int a_mn, int b_mn, int M, int N, int K, const float* __restrict__ A, long long lda,
                                const float* __restrict__ B, long long ldb, float* C, long long ldc,
                                const float* __restrict__ bias, float beta) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long o = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); o < (long long)M * N;
       o += warps) {
    const int m = (int)(o / N), n = (int)(o - (long long)m * N);
    double acc = 0.0;
    for (int k = lane; k < K; k += 32) {
      const float a = a_mn ? A[(long long)k * lda + m] : A[(long long)m * lda + k];
      const float b = b_mn ? B[(long long)k * ldb + n] : B[(long long)n * ldb + k];
      acc += (double)a * (double)b;
    }
    acc = warp_sum_d(acc);
    if (lane == 0) {
      if (bias) acc += (double)bias[n];
      float* c = C + (long long)m * ldc + n;
      const float r = (float)acc;
      *c = beta != 0.f ? r + beta * *c : r;
    }
  }
}

// Short K (e.g. the classifier's input gradient, K = classes): one thread per output.
__global__ void simt_short_k_kernel(int a_mn, int b_mn, int M, int N, int K, const float* __restrict__ A,
                                    long long lda, const float* __restrict__ B, long long ldb, float* C,
                                    long long ldc, const float* __restrict__ bias, float beta) {
  pdl_wait();
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < (long long)M * N;
       o += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(o / N), n = (int)(o - (long long)m * N);
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
      const float a = a_mn ? A[(long long)k * lda + m] : A[(long long)m * lda + k];
      const float b = b_mn ? B[(long long)k * ldb + n] : B[(long long)n * ldb + k];
      acc += (double)a * (double)b;
    }
    if (bias) acc += (double)bias[n];
    float* c = C + (long long)m * ldc + n;
    const float r = (float)acc;
    *c = beta != 0.f ? r + beta * *c : r;
  }
}

}  // namespace

extern "C" int nsk_gemm_simt(int a_mn, int b_mn, int M, int N, int K, const float* A, long long lda, const float* B,
                             long long ldb, float* C, long long ldc, const float* bias, float beta, void* stream) {
  if (M < 1 || N < 1 || K < 1) return nsk::set_error(NSK_ERR_SHAPE, "gemm: empty problem");
  const long long outs = (long long)M * N;
  if (K <= 32) {
    nsk::launch_pdl(simt_short_k_kernel, nsk::grid_for(outs, 256), 256, 0, (cudaStream_t)stream, a_mn, b_mn, M, N, K, A, lda, B,
                                                                                   ldb, C, ldc, bias, beta);
    NSK_LAUNCH_CHECK("simt_short_k");
    return NSK_OK;
  }
  if (outs <= 65536) {
    nsk::launch_pdl(simt_dot_kernel, nsk::grid_for(outs * 32, 256), 256, 0, (cudaStream_t)stream, a_mn, b_mn, M, N, K, A, lda, B,
                                                                                    ldb, C, ldc, bias, beta);
    NSK_LAUNCH_CHECK("simt_dot");
    return NSK_OK;
  }
  dim3 grid((N + TS - 1) / TS, (M + TS - 1) / TS), block(TS, TS);
  nsk::launch_pdl(simt_gemm_kernel, grid, block, 0, (cudaStream_t)stream, a_mn, b_mn, M, N, K, A, lda, B, ldb, C, ldc, bias, beta);
  NSK_LAUNCH_CHECK("simt_gemm");
  return NSK_OK;
}
