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

}  // namespace

extern "C" int nsk_gemm_simt(int a_mn, int b_mn, int M, int N, int K, const float* A, long long lda, const float* B,
                             long long ldb, float* C, long long ldc, const float* bias, float beta, void* stream) {
  if (M < 1 || N < 1 || K < 1) return nsk::set_error(NSK_ERR_SHAPE, "gemm: empty problem");
  dim3 grid((N + TS - 1) / TS, (M + TS - 1) / TS), block(TS, TS);
  simt_gemm_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(a_mn, b_mn, M, N, K, A, lda, B, ldb, C, ldc, bias, beta);
  NSK_LAUNCH_CHECK("simt_gemm");
  return NSK_OK;
}
