// Microbenchmark: what each per-stage step of the MMA issue loop costs when the MMAs are small (128x64x16 bf16,
// ~48 cycles each). The tensor pipe buffers almost nothing, so every cycle the issuing warp spends between
// stages is a pipe bubble. Variants are template-specialised so each loop compiles to exactly its own steps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_gap tools/mma_gap.cu -lcuda
#include <cstdio>
#include "../paper_2409_11600_b200/csrc/common.cuh"

constexpr int kA = 24576, kStages = 4, kW = 9 * 8192;

enum { F_FENCE = 1, F_WAIT = 2, F_TEST = 4, F_NOCOMMIT = 8, F_SPLITWAIT = 16, F_LANE0 = 32, F_FLAG = 64, F_NAMED = 128 };

template <int FLAGS, int PER_STAGE>
__global__ void __launch_bounds__(128, 1) gap(int stages_total, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bars[kStages + 1];
  __shared__ uint32_t tslot;
  __shared__ volatile int flag;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  for (int i = threadIdx.x; i < (kStages * kA + kW) / 2; i += blockDim.x) ((uint16_t*)sm)[i] = 0x3f80;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages + 1; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    flag = 1;
    mbar_arrive(&bars[kStages]);  // phase 0 of the "ready" barrier completes: waits on parity 0 succeed at once
  }
  if (warp == 0) {
    tmem_alloc(&tslot, 128);
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (warp == 1 && ((FLAGS & F_LANE0) == 0 || (threadIdx.x & 31) == 0)) {
    const uint32_t s0 = smem_u32(sm);
    const uint32_t idesc = make_idesc(1, 0, 0, 128, 64);
    int s = 0;
    for (int st = 0; st < stages_total; ++st) {
      if (FLAGS & F_WAIT) mbar_wait(&bars[kStages], 0);
      if (FLAGS & F_TEST) mbar_wait_test(&bars[kStages], 0);
      if (FLAGS & F_FLAG) {
        while (flag != 1) {
        }
      }
      if (FLAGS & F_NAMED) asm volatile("bar.sync %0, 64;" ::"r"(8 + s) : "memory");
      if (FLAGS & F_FENCE) tc_fence_after();
      const uint64_t ad0 = sdesc_sw128(s0 + s * kA, 16, 1024), bd0 = sdesc_sw128(s0 + kStages * kA, 16, 1024);
      const bool leader = (FLAGS & F_LANE0) ? true : elect_one();
      if (leader) {
#pragma unroll
        for (int t = 0; t < PER_STAGE / 4; ++t)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            umma_bf16(tm, ad0 + (((t % 3) * 4096 + q * 32) >> 4), bd0 + (((t % 3) * 8192 + q * 32) >> 4), idesc,
                      (st | t | q) ? 1u : 0u);
        if (!(FLAGS & F_NOCOMMIT)) umma_commit(&bars[s]);
      }
      if (!(FLAGS & F_LANE0)) __syncwarp();
      if (++s == kStages) s = 0;
    }
  }
  if ((FLAGS & F_NAMED) && warp == 2) {
    // a waiter warp stands in for the MMA warp's full-barrier wait: it waits on the mbarrier (here: the commit of
    // the stage's previous use, i.e. a producer's empty wait) and releases the MMA warp through a named barrier
    // per ring slot, so the MMA warp itself never reads shared memory
    for (int st = 0; st < stages_total; ++st) {
      const int s = st % kStages;
      if (st >= kStages) mbar_wait(&bars[s], ((st / kStages) - 1) & 1);
      asm volatile("bar.arrive %0, 64;" ::"r"(8 + s) : "memory");
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 128);
}

template <int FLAGS, int PER_STAGE>
void run(const char* name) {
  long long* d = nullptr;
  const int blocks = 148, smem = kStages * kA + kW + 2048;
  cudaFuncSetAttribute(gap<FLAGS, PER_STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 72000 / PER_STAGE;
  gap<FLAGS, PER_STAGE><<<blocks, 128, smem>>>(8, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  gap<FLAGS, PER_STAGE><<<blocks, 128, smem>>>(stages, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s %2d MMAs/stage: %.1f cycles/MMA at 1.9 GHz (err=%s)\n", name, PER_STAGE,
         ms * 1e-3 * 1.9e9 / (stages * PER_STAGE), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0, 12>("elect + commit");
  run<F_WAIT, 12>("+ try_wait (complete)");
  run<F_NAMED, 12>("+ named-barrier release by a waiter warp");
  run<F_NAMED, 4>("+ named-barrier release by a waiter warp");
  run<F_WAIT, 4>("+ try_wait (complete)");
  run<0, 4>("elect + commit");
  return 0;
}
