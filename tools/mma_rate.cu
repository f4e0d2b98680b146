// Microbenchmark: back-to-back tcgen05.mma (bf16, M=128, SS operands) throughput per N, no memory traffic.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include tools/mma_rate.cu -o gpurun_out/mma_rate
#include <cstdio>
#include "../paper_2409_11600_b200/csrc/common.cuh"

template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + N) * 64; i += blockDim.x) ((uint16_t*)sm)[i] = 0x3c00;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tslot, N * NACC < 32 ? 32 : (N * NACC <= 64 ? 64 : (N * NACC <= 128 ? 128 : (N * NACC <= 256 ? 256 : 512))));
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(sm), sb = sa + 128 * 128;
    const uint32_t idesc = make_idesc(1, 0, 0, 128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int q = 0; q < 4; ++q)  // NACC independent accumulator chains, round-robin
        umma_bf16(t + (q % NACC) * N, sdesc_sw128(sa + q * 32, 16, 1024), sdesc_sw128(sb + q * 32, 16, 1024), idesc, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, N * NACC < 32 ? 32 : (N * NACC <= 64 ? 64 : (N * NACC <= 128 ? 128 : (N * NACC <= 256 ? 256 : 512))));
}

template <int N, int NACC = 1>
void run(int blocks) {
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  int smem = (128 + N) * 128 + 2048;
  cudaFuncSetAttribute(mma_loop<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  mma_loop<N, NACC><<<blocks, 128, smem>>>(16, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<N, NACC><<<blocks, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, d, sizeof c, cudaMemcpyDeviceToHost);
  double flops = 2.0 * 128 * N * 16 * 4 * (double)iters * blocks;
  printf("N=%3d acc=%d blocks=%4d: %.1f cycles/MMA(128x%dx16), %.0f TFLOP/s (err=%s)\n", N, NACC, blocks,
         (double)c / (iters * 4), N, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64>(148);
  run<64, 2>(148);
  run<64, 4>(148);
  run<128>(148);
  run<128, 2>(148);
  run<256>(148);
  run<256, 2>(148);
  run<64>(296);
  run<64, 2>(296);
  run<128>(296);
  return 0;
}
