// Microbenchmark: back-to-back tcgen05.mma, 1-CTA M=128 vs 2-CTA (cta_group::2) M=256, bf16, SS operands,
// N = 64 / 128: per-SM cycles per 128xNx16 MMA-equivalent (does halving each SM's B reads lift the 64-wide MMAs
// off the shared-memory bound?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include tools/mma_rate2.cu -o gpurun_out/mma_rate2
#include <cstdio>
#include "../paper_2409_11600_b200/csrc/common.cuh"

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_loop(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = ctarank();
  // A: 128 rows per CTA; B: N/2 rows per CTA (each CTA holds its half of N)
  for (int i = threadIdx.x; i < (128 + N / 2) * 64; i += blockDim.x) ((uint16_t*)sm)[i] = 0x3c00;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  constexpr int COLS = N < 32 ? 32 : N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const uint32_t t = tslot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t sa = smem_u32(sm), sb = sa + 128 * 128;
    const uint32_t idesc = make_idesc(1, 0, 0, 256, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t ad = sdesc_sw128(sa + q * 32, 16, 1024), bd = sdesc_sw128(sb + q * 32, 16, 1024);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1));
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3));
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(COLS));
  }
}

template <int N>
void run(int blocks) {
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  int smem = (128 + N / 2) * 128 + 2048;
  cudaFuncSetAttribute(mma2_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  mma2_loop<N><<<blocks, 128, smem>>>(16, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma2_loop<N><<<blocks, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, d, sizeof c, cudaMemcpyDeviceToHost);
  double flops = 2.0 * 256 * N * 16 * 4 * (double)iters * (blocks / 2);
  printf("2-CTA N=%3d pairs=%4d: %.1f cycles per 256x%dx16 MMA (= per 128x%dx16 per SM), %.0f TFLOP/s (err=%s)\n", N,
         blocks / 2, (double)c / (iters * 4), N, N, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64>(148);
  run<128>(148);
  run<256>(148);
  return 0;
}
