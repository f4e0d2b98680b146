// Microbenchmark: tcgen05.mma issue rate for the row-reuse conv sequence (128 x 64 x 16 bf16 MMAs over a
// 4-stage ring of row-extended A boxes and 9 resident 8 KB filter taps), against simpler address patterns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_rr tools/mma_rr.cu -lcuda
#include <cstdio>
#include "../paper_2409_11600_b200/csrc/common.cuh"

constexpr int kA = 24576, kStages = 4, kW = 9 * 8192;

// mode 0: real pattern (tap row offsets, resident B per group, commit per stage, accumulator flip per tile)
// mode 1: fixed A/B addresses (like tools/mma_rate.cu), same commits
// mode 2: real pattern, no per-stage commits
// mode 3: real pattern, B from the A ring instead of the resident region
__global__ void __launch_bounds__(128, 1) mma_rr(int tiles, int mode, long long* cycles, int spin) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bars[kStages + 2];
  __shared__ uint32_t tslot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  for (int i = threadIdx.x; i < (kStages * kA + kW) / 2; i += blockDim.x) ((uint16_t*)sm)[i] = 0x3c00;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages + 2; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
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
  if (warp == 1) {
    const uint32_t s0 = smem_u32(sm);
    const uint32_t idesc = make_idesc(1, 0, 0, 128, 64);
    long long t0 = clock64();
    int s = 0;
    for (int tile = 0; tile < tiles; ++tile) {
      const uint32_t d = tm + (tile & 1) * 64;
      for (int g = 0; g < 3; ++g) {
        const uint32_t sa = mode == 1 ? s0 : s0 + s * kA;
        const uint32_t sb = mode == 1 ? s0 + kStages * kA : (mode == 3 ? s0 + ((s + 1) % kStages) * kA
                                                                          : s0 + kStages * kA + g * 3 * 8192);
        const uint64_t ad0 = sdesc_sw128(sa, 16, 1024), bd0 = sdesc_sw128(sb, 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              umma_bf16(d, ad0 + (((mode == 1 ? 0 : t * 4096) + q * 32) >> 4),
                        bd0 + (((mode == 1 ? 0 : t * 8192) + q * 32) >> 4), idesc, (g | t | q) ? 1u : 0u);
          if (mode != 2) umma_commit(&bars[s]);
        }
        __syncwarp();
        if (spin) {  // a fixed gap between stages: how much issue-side work does the MMA queue absorb?
          const long long c0 = clock64();
          while (clock64() - c0 < spin) {
          }
        }
        s = (s + 1) % kStages;
      }
      if (elect_one()) umma_commit(&bars[kStages + (tile & 1)]);
      __syncwarp();
    }
    if (elect_one()) {
      umma_commit(&bars[kStages]);
    }
    __syncwarp();
    // wait for everything: the last commit's phase on bars[kStages] is unknown, so poll completion via a fresh
    // commit + an arrival count: simply spin on clock until the tensor pipe drains (commit ordering)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    long long t1 = clock64();
    if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 128);
}

// mode 4: the kernel's pipeline: producer warp 0 waits empty[s] and arrives on full[s] (no data), MMA warp 1 waits
// full[s], issues, commits empty[s]; mode 5: + epilogue warps 4..7 handshake (tfull/tempty) per tile;
// mode 6: as 5 but the MMA warp does not wait for full[s]; 7: one elected lane waits; 8: suspend-hint wait.
// 9: test_wait probe loop; 10: wait only on 2 of 3 stages per tile.
// backoff 1: nanosleep polling, 3: test_wait probe loop, 2: try_wait with a suspend-time hint (producer and epilogue waits). `ring` = barrier ring depth (data buffers stay 4).
__global__ void __launch_bounds__(256, 1) mma_pipe(int tiles, int mode, int backoff, int ring) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16], empty[16], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (kStages * kA + kW) / 2; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;  // pattern: 1.0, or pseudo-random bf16 in [-2, 2]
    ((uint16_t*)sm)[i] = mode >= 100 ? (uint16_t)(0x3c00 ^ ((h >> 16) & 0x80ff)) : (uint16_t)0x3f80;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mode %= 100;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(&tslot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  const int steps = tiles * 3;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % ring;
      if (i >= ring) {
        if (backoff == 1) mbar_wait_backoff(&empty[s], ((i / ring) - 1) & 1);
        else if (backoff == 2) mbar_wait_suspend(&empty[s], ((i / ring) - 1) & 1);
        else if (backoff == 3) mbar_wait_test(&empty[s], ((i / ring) - 1) & 1);
        else mbar_wait(&empty[s], ((i / ring) - 1) & 1);
      }
      mbar_arrive(&full[s]);
    }
  } else if (warp == 1) {
    const uint32_t s0 = smem_u32(sm);
    const uint32_t idesc = make_idesc(1, 0, 0, 128, 64);
    int s = 0;
    uint32_t ph = 0;
    for (int tile = 0; tile < tiles; ++tile) {
      const int acc = tile & 1;
      if (mode >= 5 && tile >= 2) mbar_wait(&tempty[acc], ((tile >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tm + acc * 64;
      for (int g = 0; g < 3; ++g) {
        if (mode == 7) {
          if (elect_one()) mbar_wait(&full[s], ph);
          __syncwarp();
        } else if (mode == 8) {
          mbar_wait_suspend(&full[s], ph);
        } else if (mode == 9) {
          mbar_wait_test(&full[s], ph);
        } else if (mode == 10) {
          if (g != 1) mbar_wait(&full[s], ph);
        } else if (mode != 6) {
          mbar_wait(&full[s], ph);
        }
        tc_fence_after();
        const uint64_t ad0 = sdesc_sw128(s0 + (s % kStages) * kA, 16, 1024), bd0 = sdesc_sw128(s0 + kStages * kA + g * 3 * 8192, 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              umma_bf16(d, ad0 + ((t * 4096 + q * 32) >> 4), bd0 + ((t * 8192 + q * 32) >> 4), idesc, (g | t | q) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == ring) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= 4 && mode >= 5) {
    for (int tile = 0; tile < tiles; ++tile) {
      const int acc = tile & 1;
      if (backoff == 1) mbar_wait_backoff(&tfull[acc], (tile >> 1) & 1);
      else if (backoff == 2) mbar_wait_suspend(&tfull[acc], (tile >> 1) & 1);
      else if (backoff == 3) mbar_wait_test(&tfull[acc], (tile >> 1) & 1);
      else mbar_wait(&tfull[acc], (tile >> 1) & 1);
      tc_fence_after();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) tmem_dealloc(tm, 128);
}

int main() {
  long long* d;
  const int blocks = 148;
  cudaMalloc(&d, blocks * sizeof(long long));
  const int smem = kStages * kA + kW + 2048;
  cudaFuncSetAttribute(mma_rr, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 2000;
  for (int run = 0; run < 9; ++run) {
    const int mode = run < 4 ? run : 0, spin = run < 4 ? 0 : (50 << (run - 4));
    mma_rr<<<blocks, 128, smem>>>(4, mode, d, spin);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_rr<<<blocks, 128, smem>>>(tiles, mode, d, spin);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = 36.0 * tiles;
    printf("mode %d spin %4d: %.1f SM-cycles/MMA by event time at 1.9 GHz, %.0f TFLOP/s (err=%s)\n", mode, spin,
           ms * 1e-3 * 1.9e9 / mmas, 2.0 * 128 * 64 * 16 * mmas * blocks / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  const int cfg[][3] = {{5, 0, 4}, {6, 0, 4}};
  for (auto& c : cfg) {
    cudaFuncSetAttribute(mma_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_pipe<<<blocks, 256, smem>>>(4, c[0], c[1], c[2]);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_pipe<<<blocks, 256, smem>>>(tiles, c[0], c[1], c[2]);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = 36.0 * tiles;
    printf("pipe mode %d backoff %d ring %2d: %.1f SM-cycles/MMA at 1.9 GHz (err=%s)\n", c[0], c[1], c[2],
           ms * 1e-3 * 1.9e9 / mmas, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
