// Microbenchmark: TMA load throughput (L2 -> SMEM) per box shape / tensor-map mode, 148 persistent CTAs,
// one issuing thread each, STAGES-deep ring of 16 KB boxes, no consumer work.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tma_rate.cu -o gpurun_out/tma_rate -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2409_11600_b200/csrc/common.cuh"

namespace nsk {
int set_error(int, const std::string&) { return 1; }
int sm_count() { return 148; }
}  // namespace nsk

int BOX_ROWS_HOST = 128;

struct Job {
  int box;    // bytes per box
  int rows;   // 2D box rows
  int mode;   // 0: 2D, 1: 4D tiled, 2: 4D im2col
  int n_tiles;
  int d1, d2, d3;  // tile grid extents (mode-specific)
  int halo;        // 4D: coordinate offset (-1 = OOB halo rows/cols)
  int boxes_per_stage;
  int lane_issuers;
};

template <int STAGES>
__global__ void __launch_bounds__(256, 1) tma_loop(const __grid_constant__ CUtensorMap map, Job j, int iters,
                                                  long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int issuers = j.lane_issuers ? j.lane_issuers : blockDim.x / 32;
  int me;
  if (j.lane_issuers) {
    if (threadIdx.x >= j.lane_issuers) return;
    me = threadIdx.x;
  } else {
    if (threadIdx.x % 32 != 0) return;
    me = threadIdx.x / 32;
  }
  long long t0 = clock64();
  const int bps = j.boxes_per_stage;
  for (int i = 0; i < iters; ++i) {
    const int s = i % STAGES;
    if (s % issuers != me) continue;
    if (i >= STAGES) mbar_wait(&full[s], ((i / STAGES) - 1) & 1);
    mbar_expect_tx(&full[s], j.box * bps);
    for (int b = 0; b < bps; ++b) {
      const int t = (blockIdx.x + (long long)(i * bps + b) * gridDim.x) % j.n_tiles;
      uint8_t* dst = sm + (s * bps + b) * j.box;
      if (j.mode == 0) {
        tma_load_2d(&map, &full[s], dst, 0, t * j.rows);
      } else if (j.mode == 1) {
        const int a = t % j.d1, r = t / j.d1;
        const int bb = r % j.d2, n = r / j.d2;
        tma_load_4d(&map, &full[s], dst, 0, a * j.d3 + j.halo, bb * (j.rows / j.d3) + j.halo, n);
      } else {
        // im2col: 128 consecutive output pixels from linear pixel t*128 of a d1 x d1 grid (pad 1)
        const int p0 = t * 128;
        const int hw = j.d1 * j.d1;
        const int n = p0 / hw, rem = p0 % hw;
        tma_load_4d_im2col(&map, &full[s], dst, 0, rem % j.d1 - 1, rem / j.d1 - 1, n, (uint16_t)(i % 3),
                           (uint16_t)((i / 3) % 3));
      }
    }
  }
  for (int s = 0; s < STAGES; ++s) {
    int last = iters - 1 - ((iters - 1 - s) % STAGES);
    if (last >= 0 && last % STAGES == s) mbar_wait(&full[s], (last / STAGES) & 1);
  }
  cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* buf;
  const size_t bytes = 256ull * 32 * 32 * 256 * 2;  // 134 MB
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  long long* cyc;
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  cuTensorMapEncodeTiled(nullptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, nullptr, nullptr, nullptr, nullptr, nullptr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  struct Case {
    const char* name;
    int mode, C, H, W, N, rows_k, bw, bh, bn, halo, bps;
    int rows = 128, ctas = 1, stages = 8, issuers = 1, lanes = 0;
  };
  // NHWC bf16 tensors; 2D cases view [N*H*W, C] with 64-element (128 B) boxes of 128 rows
  std::vector<Case> cases = {
      {"2D  box 64x128 x8 stages, 4 issuer lanes/1 warp", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 8, 1, 4},
      {"2D  box 64x128 x8 stages, 8 issuer lanes/1 warp", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 8, 1, 8},
      {"2D  box 64x256 x4 stages, 4 issuer warps", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 256, 1, 4, 4},
      {"2D  box 64x128 x8 stages, 8 issuer warps", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 8, 8},
      {"4D  box 64x32x4x1 x8, 8 issuer warps", 1, 64, 32, 32, 256, 0, 32, 4, 1, 0, 1, 128, 1, 8, 8},
      {"I2C 32x32x64 x8, 8 issuer warps", 2, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 8, 8},
      {"2D  box 64x128 x8 stages, 2 issuer warps", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 8, 2},
      {"2D  box 64x128 x8 stages, 4 issuer warps", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 8, 4},
      {"4D  box 64x32x8x1 (32KB) x4", 1, 64, 32, 32, 256, 0, 32, 8, 1, 0, 1, 256, 1, 4},
      {"4D  box 64x32x4x1 x8, 4 issuer warps", 1, 64, 32, 32, 256, 0, 32, 4, 1, 0, 1, 128, 1, 8, 4},
      {"4D  box 64x32x4x1 x4, 2 CTA/SM 2 issuers", 1, 64, 32, 32, 256, 0, 32, 4, 1, 0, 1, 128, 2, 4, 2},
      {"2D  [262144 x 64] box 64x128 (contig rows)", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1},
      {"2D  [262144 x 256] box 64x128 (1 KB pitch)", 0, 256, 32, 32, 256, 0, 0, 0, 0, 0, 1},
      {"2D  [262144 x 64] 2 boxes/stage", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 2},
      {"2D  box 64x256 (32 KB) x4 stages", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 256, 1, 4},
      {"2D  box 64x64 (8 KB) x16 stages", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 64, 1, 16},
      {"2D  box 64x128 x4 stages, 2 CTA/SM", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 2, 4},
      {"2D  box 64x128 x4 stages, 4 CTA/SM", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 4, 2},
      {"2D  box 64x128 x2 stages", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 2},
      {"2D  box 64x128 x4 stages", 0, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1, 128, 1, 4},
      {"4D  box 64x32x4x1, 2 CTA/SM", 1, 64, 32, 32, 256, 0, 32, 4, 1, 0, 1, 128, 2, 4},
      {"4D  NHWC 32x32x64 box 64x32x4x1", 1, 64, 32, 32, 256, 0, 32, 4, 1, 0, 1},
      {"4D  NHWC 32x32x64 box 64x32x4x1 halo", 1, 64, 32, 32, 256, 0, 32, 4, 1, -1, 1},
      {"4D  NHWC 8x8x256 box 64x8x8x2", 1, 256, 8, 8, 256, 0, 8, 8, 2, 0, 1},
      {"4D  NHWC 8x8x256 box 64x8x8x2 halo", 1, 256, 8, 8, 256, 0, 8, 8, 2, -1, 1},
      {"4D  NHWC 4x4x512 box 64x4x4x8 halo", 1, 512, 4, 4, 256, 0, 4, 4, 8, -1, 1},
      {"I2C NHWC 32x32x64 128px", 2, 64, 32, 32, 256, 0, 0, 0, 0, 0, 1},
      {"I2C NHWC 56x56x64 128px", 2, 64, 56, 56, 64, 0, 0, 0, 0, 0, 1},
  };
  auto enc = cuTensorMapEncodeTiled;
  for (auto& c : cases) {
    CUtensorMap m;
    Job j{};
    j.mode = c.mode;
    j.halo = c.halo;
    j.boxes_per_stage = c.bps;
    j.lane_issuers = c.lanes;
    CUresult r;
    const long long npix = (long long)c.N * c.H * c.W;
    if (c.mode == 0) {
      cuuint64_t dims[2] = {(cuuint64_t)c.C, (cuuint64_t)npix};
      cuuint64_t str[1] = {(cuuint64_t)c.C * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)c.rows}, es[2] = {1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      j.n_tiles = (int)(npix / c.rows);
    } else if (c.mode == 1) {
      cuuint64_t dims[4] = {(cuuint64_t)c.C, (cuuint64_t)c.W, (cuuint64_t)c.H, (cuuint64_t)c.N};
      cuuint64_t str[3] = {(cuuint64_t)c.C * 2, (cuuint64_t)c.W * c.C * 2, (cuuint64_t)c.H * c.W * c.C * 2};
      cuuint32_t box[4] = {64, (cuuint32_t)c.bw, (cuuint32_t)c.bh, (cuuint32_t)c.bn}, es[4] = {1, 1, 1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      j.d1 = c.W / c.bw;
      j.d2 = c.H / c.bh;
      j.d3 = c.bw;
      j.n_tiles = (int)(npix / c.rows);
      if (c.bn > 1) j.d2 = 1;
    } else {
      cuuint64_t dims[4] = {(cuuint64_t)c.C, (cuuint64_t)c.W, (cuuint64_t)c.H, (cuuint64_t)c.N};
      cuuint64_t str[3] = {(cuuint64_t)c.C * 2, (cuuint64_t)c.W * c.C * 2, (cuuint64_t)c.H * c.W * c.C * 2};
      int lo[2] = {-1, -1}, hi[2] = {-1, -1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      r = cuTensorMapEncodeIm2col(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, lo, hi, 64, 128, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      j.d1 = c.W;
      j.n_tiles = (int)(npix / 128);
    }
    if (r != CUDA_SUCCESS) {
      printf("%-45s encode failed %d\n", c.name, (int)r);
      continue;
    }
    j.rows = c.mode == 2 ? 128 : c.rows;
    j.box = j.rows * 128;
    const int stages = c.bps == 2 ? 4 : c.stages;
    const int smem = stages * c.bps * j.box + 1024;
    cudaFuncSetAttribute(tma_loop<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tma_loop<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tma_loop<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tma_loop<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = 148 * c.ctas;
    const int iters = 4000 * 128 / j.rows / c.bps / c.ctas;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (stages == 16) tma_loop<16><<<grid, 32 * c.issuers, smem>>>(m, j, iters, cyc);
      if (stages == 8) tma_loop<8><<<grid, 32 * c.issuers, smem>>>(m, j, iters, cyc);
      if (stages == 4) tma_loop<4><<<grid, 32 * c.issuers, smem>>>(m, j, iters, cyc);
      if (stages == 2) tma_loop<2><<<grid, 32 * c.issuers, smem>>>(m, j, iters, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double gb = (double)grid * iters * c.bps * j.box / 1e9;
    std::vector<long long> hc(grid);
    cudaMemcpy(hc.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double mc = 0;
    for (long long v : hc) mc = v > mc ? v : mc;
    printf("%-45s %8.1f us  %6.2f TB/s  %5.1f B/clk/SM (SM clock %.0f MHz) %s\n", c.name, ms * 1e3, gb / (ms * 1e-3) / 1e3,
           (double)iters * c.bps * j.box * c.ctas / mc, mc / (ms * 1e-3) / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
