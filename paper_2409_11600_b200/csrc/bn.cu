// BatchNorm (training mode) fused with residual add and ReLU (K7).
//
// Absent from the reference; restated in oracle/restated.py
// (batchnorm_fwd / batchnorm_bwd) with the reference's conventions: float32
// storage, float64 accumulation of the statistics, biased batch variance.
//   fwd: y = relu( (x - mean) * invstd * gamma + beta  [+ residual] )
//   bwd: dz = dy * [y > 0];  dbeta = sum dz;  dgamma = sum dz * xhat
// The ReLU mask [y > 0] is kept as one bit per element (one byte per 8 channels, written by the forward
// apply), so the backward passes read 1/16 of the bytes a bf16 y would cost.
//        dx = gamma*invstd*(dz - dbeta/M - xhat*dgamma/M);  dres = dz
// x / y / dy / dx / residual are NHWC bf16 viewed as [rows, C]; gamma_beta is
// the fp32 parameter [2, C]. Each pass is a vectorised (8 x bf16) sweep;
// per-block channel partials go to a workspace and are folded in float64 in a
// fixed order (deterministic, no atomics).
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

constexpr int BT = 256;      // threads per block
constexpr int MAXBLK = 592;  // 4 * 148

struct Pack8 {
  float v[8];
};

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* f) {
  uint4 u = __ldg((const uint4*)p);
  const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float* f) {
  uint4 u;
  u.x = pack_bf16x2(f[0], f[1]);
  u.y = pack_bf16x2(f[2], f[3]);
  u.z = pack_bf16x2(f[4], f[5]);
  u.w = pack_bf16x2(f[6], f[7]);
  *(uint4*)p = u;
}

// Block-level channel reduction of two per-thread 8-vectors, written as partials[blk][2][C].
__device__ void block_reduce_store(float* s1, float* s2, int C, float* part) {
  extern __shared__ float red[];  // [BT/CV][C] x 2
  const int CV = C / 8;
  const int cv = threadIdx.x % CV, ro = threadIdx.x / CV, RPB = BT / CV;
  float* r1 = red;
  float* r2 = red + RPB * C;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    r1[ro * C + cv * 8 + j] = s1[j];
    r2[ro * C + cv * 8 + j] = s2[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += BT) {
    float a = 0.f, b = 0.f;
    for (int r = 0; r < RPB; ++r) {
      a += r1[r * C + c];
      b += r2[r * C + c];
    }
    part[(size_t)blockIdx.x * 2 * C + c] = a;
    part[(size_t)blockIdx.x * 2 * C + C + c] = b;
  }
}

// pass 1 of fwd: sum x and sum x^2 per channel
constexpr int kFoldSlots = 4;  // one fold-count pair per stream that runs BatchNorms (compute + side branches)
__device__ unsigned g_fold_sync[kFoldSlots][2][2];

__global__ void __launch_bounds__(BT) bn_stats_kernel(const __nv_bfloat16* __restrict__ x, uint64_t rows, int C,
                                                      float* part, unsigned* rearm) {
  pdl_wait();
  if (rearm && blockIdx.x == 0 && threadIdx.x == 0) rearm[0] = rearm[1] = 0u;  // re-arm fold count + ticket
  const int CV = C / 8;
  const int cv = threadIdx.x % CV, ro = threadIdx.x / CV, RPB = BT / CV;
  float s1[8] = {0}, s2[8] = {0};
  const uint64_t stride = (uint64_t)gridDim.x * RPB;
  uint64_t r = (uint64_t)blockIdx.x * RPB + ro;
  for (; r + 3 * stride < rows; r += 4 * stride) {  // four rows in flight, same order as one at a time
    float f[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k) ld8(x + (r + k * stride) * C + cv * 8, f[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s1[j] += f[k][j];
        s2[j] += f[k][j] * f[k][j];
      }
  }
  for (; r < rows; r += stride) {
    float f[8];
    ld8(x + r * C + cv * 8, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s1[j] += f[j];
      s2[j] += f[j] * f[j];
    }
  }
  block_reduce_store(s1, s2, C, part);
}

constexpr int FT = 128;  // finalize threads: one block per channel folds the block partials

// float64 fold of the two partial rows of channel c over nblk blocks (fixed order -> deterministic)
__device__ void fold_partials(const float* part, int nblk, int C, int c, double* a_out, double* b_out) {
  __shared__ double ra[FT / 32], rb[FT / 32];
  double a = 0.0, b = 0.0;
  for (int k = threadIdx.x; k < nblk; k += FT) {
    a += (double)part[(size_t)k * 2 * C + c];
    b += (double)part[(size_t)k * 2 * C + C + c];
  }
  a = warp_sum_d(a);
  b = warp_sum_d(b);
  if ((threadIdx.x & 31) == 0) {
    ra[threadIdx.x >> 5] = a;
    rb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = b = 0.0;
    for (int i = 0; i < FT / 32; ++i) {
      a += ra[i];
      b += rb[i];
    }
    *a_out = a;
    *b_out = b;
  }
}

// fold partials (float64) -> mean, invstd and the fused affine (scale, shift); grid = C blocks
__global__ void __launch_bounds__(FT) bn_fwd_finalize(const float* part, int nblk, uint64_t rows, int C, float eps,
                                                      const float* gb, float* mean, float* invstd, float* scale,
                                                      float* shift, float* running, float momentum) {
  pdl_wait();
  const int c = blockIdx.x;
  double a, b;
  fold_partials(part, nblk, C, c, &a, &b);
  if (threadIdx.x == 0) {
    double mu = a / (double)rows;
    double var = b / (double)rows - mu * mu;
    if (var < 0.0) var = 0.0;
    double is = 1.0 / sqrt(var + (double)eps);
    mean[c] = (float)mu;
    invstd[c] = (float)is;
    double g = gb[c], be = gb[C + c];
    scale[c] = (float)(g * is);
    shift[c] = (float)(be - mu * g * is);
    if (running) {  // running statistics, unbiased variance (torch.nn.BatchNorm2d convention)
      const double n = (double)rows;
      const double unb = n > 1.0 ? var * n / (n - 1.0) : var;
      running[c] = (float)((1.0 - momentum) * running[c] + momentum * mu);
      running[C + c] = (float)((1.0 - momentum) * running[C + c] + momentum * unb);
    }
  }
}

__global__ void __launch_bounds__(BT) bn_apply_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ res,
                                                      const float* __restrict__ scale, const float* __restrict__ shift,
                                                      __nv_bfloat16* __restrict__ y, uint8_t* __restrict__ mask,
                                                      uint64_t rows, int C, int relu) {
  pdl_wait();
  extern __shared__ float ss[];  // [2][C] scale, shift (float4 reads instead of 16 scalar global loads)
  for (int k = threadIdx.x; k < C; k += BT) {
    ss[k] = scale[k];
    ss[C + k] = shift[k];
  }
  __syncthreads();
  const uint64_t nv = rows * (uint64_t)C / 8;
  const int CV = C / 8;
  // channel group carried incrementally (no 64-bit modulo per iteration)
  const uint64_t i0 = (uint64_t)blockIdx.x * BT + threadIdx.x, istep = (uint64_t)gridDim.x * BT;
  int cvi = (int)(i0 % CV);
  const int cstep = (int)(istep % CV);
  for (uint64_t i = i0; i < nv; i += istep, cvi = (cvi + cstep >= CV) ? cvi + cstep - CV : cvi + cstep) {
    const int c0 = cvi * 8;
    float f[8], r[8], sc[8], sh[8];
    ld8(x + i * 8, f);
    if (res) ld8(res + i * 8, r);
    *(float4*)sc = *(const float4*)(ss + c0);
    *(float4*)(sc + 4) = *(const float4*)(ss + c0 + 4);
    *(float4*)sh = *(const float4*)(ss + C + c0);
    *(float4*)(sh + 4) = *(const float4*)(ss + C + c0 + 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = f[j] * sc[j] + sh[j];
      if (res) v += r[j];
      if (relu) v = v > 0.f ? v : 0.f;
      f[j] = v;
    }
    st8(y + i * 8, f);
    if (mask) {
      unsigned bits = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) bits |= (f[j] > 0.f ? 1u : 0u) << j;
      mask[i] = (uint8_t)bits;
    }
  }
}

// running statistics (eval mode): rm = (1-m) rm + m mean, rv = (1-m) rv + m var_unbiased, var from invstd
__global__ void bn_running_kernel(const float* __restrict__ mean, const float* __restrict__ invstd, float* running,
                                  int C, double rows, float momentum, float eps) {
  pdl_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double is = invstd[c];
  double var = 1.0 / (is * is) - (double)eps;
  if (var < 0.0) var = 0.0;
  const double unb = rows > 1.0 ? var * rows / (rows - 1.0) : var;
  running[c] = (float)((1.0 - momentum) * running[c] + momentum * (double)mean[c]);
  running[C + c] = (float)((1.0 - momentum) * running[C + c] + momentum * unb);
}

// eval-mode affine from running statistics: scale = g / sqrt(rv + eps), shift = b - rm * scale
__global__ void bn_eval_affine_kernel(const float* __restrict__ gb, const float* __restrict__ running, int C,
                                      float eps, float* scale, float* shift) {
  pdl_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double sc = (double)gb[c] / sqrt((double)running[C + c] + (double)eps);
  scale[c] = (float)sc;
  shift[c] = (float)((double)gb[C + c] - (double)running[c] * sc);
}

// bwd pass 1: sum dz and sum dz*x per channel, dz = dy * [y > 0] (relu) or dy
__global__ void __launch_bounds__(BT) bn_bwd_reduce_kernel(const __nv_bfloat16* __restrict__ dy,
                                                           const __nv_bfloat16* __restrict__ x,
                                                           const uint8_t* __restrict__ mask, uint64_t rows, int C,
                                                           float* part, unsigned* rearm) {
  pdl_wait();
  if (rearm && blockIdx.x == 0 && threadIdx.x == 0) rearm[0] = rearm[1] = 0u;  // re-arm fold count + ticket
  const int CV = C / 8;
  const int cv = threadIdx.x % CV, ro = threadIdx.x / CV, RPB = BT / CV;
  float s1[8] = {0}, s2[8] = {0};
  const uint64_t stride = (uint64_t)gridDim.x * RPB;
  uint64_t r = (uint64_t)blockIdx.x * RPB + ro;
  // two rows in flight per thread (same accumulation order as one at a time)
  for (; r + stride < rows; r += 2 * stride) {
    const uint64_t o0 = r * C + cv * 8, o1 = (r + stride) * C + cv * 8;
    float g0[8], x0[8], g1[8], x1[8];
    ld8(dy + o0, g0);
    ld8(x + o0, x0);
    ld8(dy + o1, g1);
    ld8(x + o1, x1);
    if (mask) {
      const unsigned m0 = __ldg(mask + o0 / 8), m1 = __ldg(mask + o1 / 8);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        g0[j] = ((m0 >> j) & 1u) ? g0[j] : 0.f;
        g1[j] = ((m1 >> j) & 1u) ? g1[j] : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s1[j] += g0[j];
      s2[j] += g0[j] * x0[j];
      s1[j] += g1[j];
      s2[j] += g1[j] * x1[j];
    }
  }
  if (r < rows) {
    const uint64_t off = r * C + cv * 8;
    float g[8], xv[8];
    ld8(dy + off, g);
    ld8(x + off, xv);
    if (mask) {
      const unsigned m = __ldg(mask + off / 8);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = ((m >> j) & 1u) ? g[j] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s1[j] += g[j];
      s2[j] += g[j] * xv[j];
    }
  }
  block_reduce_store(s1, s2, C, part);
}

// dgamma/dbeta and dx = A*dz + B*x + Cc per channel
__global__ void __launch_bounds__(FT) bn_bwd_finalize(const float* part, int nblk, uint64_t rows, int C,
                                                      const float* gb, const float* mean, const float* invstd,
                                                      float* dgb, float beta_acc, float* coef) {
  pdl_wait();
  const int c = blockIdx.x;
  double sdz, sdzx;
  fold_partials(part, nblk, C, c, &sdz, &sdzx);
  if (threadIdx.x == 0) {
    const double mu = mean[c], is = invstd[c], g = gb[c], M = (double)rows;
    const double dbeta = sdz;
    const double dgamma = is * (sdzx - mu * sdz);
    if (beta_acc != 0.f) {
      dgb[c] = (float)(dgamma + beta_acc * dgb[c]);
      dgb[C + c] = (float)(dbeta + beta_acc * dgb[C + c]);
    } else {
      dgb[c] = (float)dgamma;
      dgb[C + c] = (float)dbeta;
    }
    const double A = g * is;
    const double B = -g * is * is * dgamma / M;
    const double Cc = -g * is * dbeta / M + g * is * is * mu * dgamma / M;
    coef[c] = (float)A;
    coef[C + c] = (float)B;
    coef[2 * C + c] = (float)Cc;
  }
}

__global__ void __launch_bounds__(BT) bn_bwd_apply_kernel(const __nv_bfloat16* __restrict__ dy,
                                                          const __nv_bfloat16* __restrict__ x,
                                                          const uint8_t* __restrict__ mask,
                                                          const float* __restrict__ coef,
                                                          __nv_bfloat16* __restrict__ dx,
                                                          __nv_bfloat16* __restrict__ dres, uint64_t rows, int C) {
  pdl_wait();
  // per-channel coefficients staged in shared memory and read as float4 (24 scalar global loads per 8 elements
  // made the pass load-instruction bound)
  extern __shared__ float cf[];  // [3][C]
  for (int k = threadIdx.x; k < 3 * C; k += BT) cf[k] = coef[k];
  __syncthreads();
  const uint64_t nv = rows * (uint64_t)C / 8;
  const int CV = C / 8;
  // channel group carried incrementally (no 64-bit modulo per iteration)
  const uint64_t i0 = (uint64_t)blockIdx.x * BT + threadIdx.x, istep = (uint64_t)gridDim.x * BT;
  int cvi = (int)(i0 % CV);
  const int cstep = (int)(istep % CV);
  for (uint64_t i = i0; i < nv; i += istep, cvi = (cvi + cstep >= CV) ? cvi + cstep - CV : cvi + cstep) {
    const int c0 = cvi * 8;
    float g[8], xv[8];
    ld8(dy + i * 8, g);
    ld8(x + i * 8, xv);
    if (mask) {
      const unsigned m = __ldg(mask + i);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = ((m >> j) & 1u) ? g[j] : 0.f;
    }
    if (dres) st8(dres + i * 8, g);
    float a[8], b[8], cc[8];
    *(float4*)a = *(const float4*)(cf + c0);
    *(float4*)(a + 4) = *(const float4*)(cf + c0 + 4);
    *(float4*)b = *(const float4*)(cf + C + c0);
    *(float4*)(b + 4) = *(const float4*)(cf + C + c0 + 4);
    *(float4*)cc = *(const float4*)(cf + 2 * C + c0);
    *(float4*)(cc + 4) = *(const float4*)(cf + 2 * C + c0 + 4);
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = a[j] * g[j] + b[j] * xv[j] + cc[j];
    st8(dx + i * 8, o);
  }
}

// ---- finalize folded into the apply pass ----
// A separate finalize launch per BatchNorm cost ~4 us of step time each (39 per ResNet-18 step: 163 us measured by
// skipping them). Instead the first C/2 blocks of the apply grid fold one channel per 128 threads (float64, fixed
// order: threads stride the partial rows, butterfly, warp sums in order), publish scale/shift (or the backward coefficients) and
// count themselves done; every block waits for the count, stages the per-channel values in shared memory and
// applies. The folding blocks are the first nfold to take an arrival ticket, so they are running before anyone
// can spin on them. The
// count is re-armed by the kernel that produced the partials (bn_stats / bn_bwd_reduce / the conv statistics
// epilogue zero it at their start, nsk_bn_fold_counter), so the apply needs no exit accounting (2.4k
// same-address atomics per launch were measurable).
// g_fold_sync[fwd | bwd]: [0] folded channels, [1] arrival ticket (declared with bn_stats_kernel)

__device__ __forceinline__ void fold_wait(unsigned* sync, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v, ns = 64;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sync) : "memory");
      if (v >= target) break;
      __nanosleep(ns);  // back off: a thousand pollers on one L2 line slow the folding blocks' atomics
      if (ns < 512) ns *= 2;
    }
  }
  __syncthreads();
}

// arrival ticket of this block (sync[1], re-armed with the count sync[0] by the producer of the partials)
__device__ __forceinline__ int fold_ticket(unsigned* sync) {
  __shared__ unsigned ticket;
  if (threadIdx.x == 0) ticket = atomicAdd(&sync[1], 1u);
  __syncthreads();
  return (int)ticket;
}

// float64 fold of channel c's two partial columns over nblk rows of [nblk][2][C] by the 128 threads of one half
// block (4 warps; fixed order: thread strides, butterfly, then the 4 warp sums in order). All BT threads call it.
constexpr int FOLD_T = 128;  // threads per folded channel
constexpr int AT = BT;       // threads per block of the fused fold+apply passes
__device__ __forceinline__ void group_fold(const float* part, int nblk, int C, int c, double* a, double* b) {
  __shared__ double red[AT / 32][2];
  const int t = threadIdx.x % FOLD_T;
  double x = 0.0, y = 0.0, x2 = 0.0, y2 = 0.0;
  if (c < C) {
    int k = t;
    for (; k + FOLD_T < nblk; k += 2 * FOLD_T) {  // two rows in flight per thread
      const float p0 = __ldcg(part + (size_t)k * 2 * C + c), q0 = __ldcg(part + (size_t)k * 2 * C + C + c);
      const float p1 = __ldcg(part + (size_t)(k + FOLD_T) * 2 * C + c);
      const float q1 = __ldcg(part + (size_t)(k + FOLD_T) * 2 * C + C + c);
      x += p0; y += q0; x2 += p1; y2 += q1;
    }
    if (k < nblk) {
      x += (double)__ldcg(part + (size_t)k * 2 * C + c);
      y += (double)__ldcg(part + (size_t)k * 2 * C + C + c);
    }
  }
  x = warp_sum_d(x + x2);
  y = warp_sum_d(y + y2);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[w][0] = x;
    red[w][1] = y;
  }
  __syncthreads();
  const int g0 = (threadIdx.x / FOLD_T) * (FOLD_T / 32);
  *a = (red[g0][0] + red[g0 + 1][0]) + (red[g0 + 2][0] + red[g0 + 3][0]);
  *b = (red[g0][1] + red[g0 + 1][1]) + (red[g0 + 2][1] + red[g0 + 3][1]);
  __syncthreads();  // red is reused by the next channel pair
}

__global__ void __launch_bounds__(AT) bn_apply_fold_kernel(const float* part, int nblk, uint64_t rows, int C, float eps,
                                                           const float* __restrict__ gb, float* mean, float* invstd,
                                                           float* running, float momentum, float* affine,
                                                           const __nv_bfloat16* __restrict__ x,
                                                           const __nv_bfloat16* __restrict__ res,
                                                           __nv_bfloat16* __restrict__ y, uint8_t* __restrict__ mask,
                                                           int relu, int nfold, unsigned* sync) {
  pdl_wait();
  // folding blocks: the first nfold (<= SMs) blocks to ARRIVE, 2 channels per pass. Roles come from an arrival
  // ticket, not blockIdx: a block that holds a ticket is running, so the fold never waits on an undispatched block
  // whatever order the hardware schedules the grid in (or however side-stream kernels occupy the SMs).
  const int role = fold_ticket(sync);
  for (int cg = role; role < nfold && cg * (AT / FOLD_T) < C; cg += nfold) {
    const int c = cg * (AT / FOLD_T) + threadIdx.x / FOLD_T;
    double a, b;
    group_fold(part, nblk, C, c, &a, &b);
    if (c < C && threadIdx.x % FOLD_T == 0) {
      const double mu = a / (double)rows;
      double var = b / (double)rows - mu * mu;
      if (var < 0.0) var = 0.0;
      const double is = 1.0 / sqrt(var + (double)eps);
      mean[c] = (float)mu;
      invstd[c] = (float)is;
      const double g = gb[c], be = gb[C + c];
      affine[c] = (float)(g * is);
      affine[C + c] = (float)(be - mu * g * is);
      if (running) {  // running statistics, unbiased variance (torch.nn.BatchNorm2d convention)
        const double n = (double)rows;
        const double unb = n > 1.0 ? var * n / (n - 1.0) : var;
        running[c] = (float)((1.0 - momentum) * running[c] + momentum * mu);
        running[C + c] = (float)((1.0 - momentum) * running[C + c] + momentum * unb);
      }
      __threadfence();
      atomicAdd(&sync[0], 1u);
    }
  }
  fold_wait(sync, (unsigned)C);
  extern __shared__ float aff[];  // [2][C]
  for (int i = threadIdx.x; i < 2 * C; i += AT) aff[i] = __ldcg(affine + i);
  __syncthreads();
  const float* scale = aff;
  const float* shift = aff + C;
  const uint64_t nv = rows * (uint64_t)C / 8;
  const int CV = C / 8;
  const uint64_t i0 = (uint64_t)blockIdx.x * AT + threadIdx.x, istep = (uint64_t)gridDim.x * AT;
  int cvi = (int)(i0 % CV);
  const int cstep = (int)(istep % CV);
  for (uint64_t i = i0; i < nv; i += istep, cvi = (cvi + cstep >= CV) ? cvi + cstep - CV : cvi + cstep) {
    const int c0 = cvi * 8;
    float f[8], r[8], sc[8], sh[8];
    ld8(x + i * 8, f);
    if (res) ld8(res + i * 8, r);
    *(float4*)sc = *(const float4*)(scale + c0);
    *(float4*)(sc + 4) = *(const float4*)(scale + c0 + 4);
    *(float4*)sh = *(const float4*)(shift + c0);
    *(float4*)(sh + 4) = *(const float4*)(shift + c0 + 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = f[j] * sc[j] + sh[j];
      if (res) v += r[j];
      if (relu) v = v > 0.f ? v : 0.f;
      f[j] = v;
    }
    st8(y + i * 8, f);
    if (mask) {
      unsigned bits = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) bits |= (f[j] > 0.f ? 1u : 0u) << j;
      mask[i] = (uint8_t)bits;
    }
  }
}

__global__ void __launch_bounds__(AT) bn_bwd_apply_fold_kernel(const float* part, int nblk, uint64_t rows, int C,
                                                               const float* __restrict__ gb,
                                                               const float* __restrict__ mean,
                                                               const float* __restrict__ invstd, float* dgb,
                                                               float beta_acc, float* coefg,
                                                               const __nv_bfloat16* __restrict__ dy,
                                                               const __nv_bfloat16* __restrict__ x,
                                                               const uint8_t* __restrict__ mask,
                                                               __nv_bfloat16* __restrict__ dx,
                                                               __nv_bfloat16* __restrict__ dres, int nfold,
                                                               unsigned* sync) {
  pdl_wait();
  const int role = fold_ticket(sync);  // arrival-ordered fold roles (see bn_apply_fold_kernel)
  for (int cg = role; role < nfold && cg * (AT / FOLD_T) < C; cg += nfold) {
    const int c = cg * (AT / FOLD_T) + threadIdx.x / FOLD_T;
    double sdz, sdzx;
    group_fold(part, nblk, C, c, &sdz, &sdzx);
    if (c < C && threadIdx.x % FOLD_T == 0) {
      const double mu = mean[c], is = invstd[c], g = gb[c], M = (double)rows;
      const double dbeta = sdz;
      const double dgamma = is * (sdzx - mu * sdz);
      if (beta_acc != 0.f) {
        dgb[c] = (float)(dgamma + beta_acc * dgb[c]);
        dgb[C + c] = (float)(dbeta + beta_acc * dgb[C + c]);
      } else {
        dgb[c] = (float)dgamma;
        dgb[C + c] = (float)dbeta;
      }
      coefg[c] = (float)(g * is);
      coefg[C + c] = (float)(-g * is * is * dgamma / M);
      coefg[2 * C + c] = (float)(-g * is * dbeta / M + g * is * is * mu * dgamma / M);
      __threadfence();
      atomicAdd(&sync[0], 1u);
    }
  }
  fold_wait(sync, (unsigned)C);
  extern __shared__ float coef[];  // [3][C]
  for (int i = threadIdx.x; i < 3 * C; i += AT) coef[i] = __ldcg(coefg + i);
  __syncthreads();
  const uint64_t nv = rows * (uint64_t)C / 8;
  const int CV = C / 8;
  const uint64_t i0 = (uint64_t)blockIdx.x * AT + threadIdx.x, istep = (uint64_t)gridDim.x * AT;
  int cvi = (int)(i0 % CV);
  const int cstep = (int)(istep % CV);
  for (uint64_t i = i0; i < nv; i += istep, cvi = (cvi + cstep >= CV) ? cvi + cstep - CV : cvi + cstep) {
    const int c0 = cvi * 8;
    float g[8], xv[8];
    ld8(dy + i * 8, g);
    ld8(x + i * 8, xv);
    if (mask) {
      const unsigned m = __ldg(mask + i);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = ((m >> j) & 1u) ? g[j] : 0.f;
    }
    if (dres) st8(dres + i * 8, g);
    float a[8], b[8], cc[8];
    *(float4*)a = *(const float4*)(coef + c0);
    *(float4*)(a + 4) = *(const float4*)(coef + c0 + 4);
    *(float4*)b = *(const float4*)(coef + C + c0);
    *(float4*)(b + 4) = *(const float4*)(coef + C + c0 + 4);
    *(float4*)cc = *(const float4*)(coef + 2 * C + c0);
    *(float4*)(cc + 4) = *(const float4*)(coef + 2 * C + c0 + 4);
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = a[j] * g[j] + b[j] * xv[j] + cc[j];
    st8(dx + i * 8, o);
  }
}

// folding blocks: one per channel pair, at most one per SM (every folding block must be resident before any
// block spins on the count: 1024 pairs for C = 2048 deadlocked with 4 resident blocks per SM)
int fold_blocks(int C) {
  const int groups = (C + AT / FOLD_T - 1) / (AT / FOLD_T);
  return groups < nsk::sm_count() ? groups : nsk::sm_count();
}
// grid of the grid-stride apply passes: at most 4 blocks per SM (NSK_BN_GRID_CAP overrides). 16 per SM fills the
// SMs and crowds out the side-stream weight-gradient CTAs running beside them: ResNet-18 2.063 -> 2.026 ms/step with 4
// (2 per SM: 2.16 ms; ResNet-50 unchanged, its large layers take the fold-in-apply kernels)
unsigned apply_grid(uint64_t nv) {
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("NSK_BN_GRID_CAP");
    cap = e ? atoi(e) : 4;
    if (cap < 1) cap = 4;
  }
  unsigned g = nsk::grid_for(nv, BT);
  const unsigned lim = (unsigned)(nsk::sm_count() * cap);
  return g > lim ? lim : g;
}

unsigned fold_grid(uint64_t nv, int C) {
  unsigned g = nsk::grid_for(nv, AT);
  const unsigned need = (unsigned)fold_blocks(C);
  return g < need ? need : g;
}

// fold counts of the stream's slot: [0] forward, [2] backward (slots handed out to streams on first use)
static unsigned* fold_counters(cudaStream_t st) {
  static unsigned* base = nullptr;
  static cudaStream_t owners[kFoldSlots] = {};
  static int used = 0;
  if (!base) {
    void* a = nullptr;
    if (cudaGetSymbolAddress(&a, g_fold_sync) != cudaSuccess) return nullptr;
    base = (unsigned*)a;
  }
  int slot = -1;
  for (int i = 0; i < used; ++i)
    if (owners[i] == st) slot = i;
  if (slot < 0) {
    if (used == kFoldSlots) return nullptr;  // more concurrent BN streams than slots: caller folds separately
    owners[used] = st;
    slot = used++;
  }
  return base + slot * 4;
}

// The fused fold+apply stalls every block until the fold is done (a few us); that only beats a separate
// finalize launch (~4 us of step time each) when the apply itself is long: ResNet-50's 56x56x256 layers
// (8.3k vs 7.6k img/s) yes, ResNet-18's (2.61 vs 2.71 ms/step) no.
bool fold_in_apply(uint64_t rows, int C, cudaStream_t st) {
  if (!fold_counters(st)) return false;
  const char* e = getenv("NSK_BN_FOLD_APPLY");
  if (e) return e[0] == '1';
  return rows * (uint64_t)C >= (1ull << 25);
}

int nblocks(uint64_t rows, int C) {
  const int RPB = BT / (C / 8);
  uint64_t want = (rows + RPB * 8 - 1) / (RPB * 8);  // >= 8 rows per thread
  static int cap = -1;  // NSK_BN_RED_BLK: blocks of the statistics passes (the workspace holds MAXBLK partials)
  if (cap < 0) {
    const char* e = getenv("NSK_BN_RED_BLK");
    cap = e ? atoi(e) : MAXBLK;
    if (cap < 1 || cap > MAXBLK) cap = MAXBLK;
  }
  if (want > (uint64_t)cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

int check(uint64_t rows, int C, const void* a, const void* b) {
  if (C % 8 || C < 8 || C > 2048 || (BT % (C / 8)))
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "batchnorm: C must be a multiple of 8 dividing 2048");
  if (((uintptr_t)a & 15) || (b && ((uintptr_t)b & 15)))
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "batchnorm: buffers must be 16-byte aligned");
  return NSK_OK;
}

}  // namespace

// device address of the forward fold count, zeroed by the conv statistics epilogue (umma_gemm.cu) that feeds
// nsk_bn_fwd_partials
unsigned* nsk::bn_fold_counter_fwd(cudaStream_t st) { return fold_counters(st); }
unsigned* nsk::bn_fold_counter_bwd(cudaStream_t st) {
  unsigned* fc = fold_counters(st);
  return fc ? fc + 2 : nullptr;
}

extern "C" {

uint64_t nsk_bn_workspace(uint64_t rows, int C) {
  return (uint64_t)MAXBLK * 2 * C * sizeof(float) + 4 * (uint64_t)C * sizeof(float);
}

int nsk_bn_fwd(const void* x, const float* gamma_beta, void* y, float* mean, float* invstd, uint64_t rows, int C,
               float eps, int relu, const void* residual, void* relu_mask, float* running, float momentum, float* ws,
               void* stream) {
  int rc = check(rows, C, x, residual);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = nblocks(rows, C);
  const int RPB = BT / (C / 8);
  const size_t smem = 2 * (size_t)RPB * C * sizeof(float);
  float* part = ws;
  float* scale = ws + (size_t)MAXBLK * 2 * C;
  float* shift = scale + C;
  unsigned* fc = fold_counters(st);
  nsk::launch_pdl(bn_stats_kernel, nb, BT, smem, st, (const __nv_bfloat16*)x, rows, C, part, fc);
  const uint64_t nv = rows * (uint64_t)C / 8;
  if (!fold_in_apply(rows, C, st)) {
    nsk::launch_pdl(bn_fwd_finalize, C, FT, 0, st, (const float*)part, nb, rows, C, eps, gamma_beta, mean, invstd, scale,
                    shift, running, momentum);
    nsk::launch_pdl(bn_apply_kernel, apply_grid(nv), BT, 2 * C * sizeof(float), st, (const __nv_bfloat16*)x,
                    (const __nv_bfloat16*)residual, (const float*)scale, (const float*)shift, (__nv_bfloat16*)y,
                    (uint8_t*)relu_mask, rows, C, relu);
    NSK_LAUNCH_CHECK("bn_fwd");
    return NSK_OK;
  }
  nsk::launch_pdl(bn_apply_fold_kernel, fold_grid(nv, C), AT, 2 * C * sizeof(float), st, (const float*)part, nb, rows,
                  C, eps, gamma_beta, mean, invstd, running, momentum, scale, (const __nv_bfloat16*)x,
                  (const __nv_bfloat16*)residual, (__nv_bfloat16*)y, (uint8_t*)relu_mask, relu, fold_blocks(C),
                  fold_counters(st));
  NSK_LAUNCH_CHECK("bn_fwd");
  return NSK_OK;
}

// forward from channel partials produced by the conv that wrote x (nsk_conv2d_fprop_stats): fold + apply,
// no statistics pass over x
int nsk_bn_fwd_partials(const float* partials, int nparts, const void* x, const float* gamma_beta, void* y,
                        float* mean, float* invstd, uint64_t rows, int C, float eps, int relu, const void* residual,
                        void* relu_mask, float* running, float momentum, float* ws, void* stream) {
  int rc = check(rows, C, x, residual);
  if (rc) return rc;
  if (nparts < 1) return nsk::set_error(NSK_ERR_SHAPE, "batchnorm: no statistics partials");
  cudaStream_t st = (cudaStream_t)stream;
  float* scale = ws + (size_t)MAXBLK * 2 * C;
  float* shift = scale + C;
  const uint64_t nv = rows * (uint64_t)C / 8;
  if (!fold_in_apply(rows, C, st)) {
    nsk::launch_pdl(bn_fwd_finalize, C, FT, 0, st, partials, nparts, rows, C, eps, gamma_beta, mean, invstd, scale,
                    shift, running, momentum);
    nsk::launch_pdl(bn_apply_kernel, apply_grid(nv), BT, 2 * C * sizeof(float), st, (const __nv_bfloat16*)x,
                    (const __nv_bfloat16*)residual, (const float*)scale, (const float*)shift, (__nv_bfloat16*)y,
                    (uint8_t*)relu_mask, rows, C, relu);
    NSK_LAUNCH_CHECK("bn_fwd_partials");
    return NSK_OK;
  }
  nsk::launch_pdl(bn_apply_fold_kernel, fold_grid(nv, C), AT, 2 * C * sizeof(float), st, partials, nparts, rows, C, eps,
                  gamma_beta, mean, invstd, running, momentum, scale, (const __nv_bfloat16*)x,
                  (const __nv_bfloat16*)residual, (__nv_bfloat16*)y, (uint8_t*)relu_mask, relu, fold_blocks(C),
                  fold_counters(st));
  NSK_LAUNCH_CHECK("bn_fwd_partials");
  return NSK_OK;
}

// running-statistics update from a training-mode forward's mean / invstd (momentum convention of
// torch.nn.BatchNorm2d: new = (1 - m) * old + m * batch, unbiased batch variance)
int nsk_bn_running_update(const float* mean, const float* invstd, float* running, uint64_t rows, int C,
                          float momentum, float eps, void* stream) {
  nsk::launch_pdl(bn_running_kernel, (C + 127) / 128, 128, 0, (cudaStream_t)stream, mean, invstd, running, C,
                  (double)rows, momentum, eps);
  NSK_LAUNCH_CHECK("bn_running_update");
  return NSK_OK;
}

// inference forward: y = relu(x * g / sqrt(rv + eps) + b - rm * g / sqrt(rv + eps) [+ residual])
int nsk_bn_fwd_eval(const void* x, const float* gamma_beta, const float* running, void* y, uint64_t rows, int C,
                    float eps, int relu, const void* residual, float* ws, void* stream) {
  int rc = check(rows, C, x, residual);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  float* scale = ws + (size_t)MAXBLK * 2 * C;
  float* shift = scale + C;
  nsk::launch_pdl(bn_eval_affine_kernel, (C + 127) / 128, 128, 0, st, gamma_beta, running, C, eps, scale, shift);
  const uint64_t nv = rows * (uint64_t)C / 8;
  nsk::launch_pdl(bn_apply_kernel, apply_grid(nv), BT, 2 * C * sizeof(float), st, (const __nv_bfloat16*)x,
                  (const __nv_bfloat16*)residual, scale, shift, (__nv_bfloat16*)y, (uint8_t*)nullptr, rows, C, relu);
  NSK_LAUNCH_CHECK("bn_fwd_eval");
  return NSK_OK;
}

int nsk_bn_bwd(const void* dy, const void* x, const void* relu_mask, const float* gamma_beta, const float* mean,
               const float* invstd, void* dx, void* dres, float* dgamma_beta, float beta_acc, uint64_t rows, int C,
               float* ws, void* stream) {
  int rc = check(rows, C, dy, x);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = nblocks(rows, C);
  const int RPB = BT / (C / 8);
  const size_t smem = 2 * (size_t)RPB * C * sizeof(float);
  float* part = ws;
  float* coef = ws + (size_t)MAXBLK * 2 * C;  // 3*C floats (workspace reserves 4*C)
  unsigned* fc = fold_counters(st);
  nsk::launch_pdl(bn_bwd_reduce_kernel, nb, BT, smem, st, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x,
                  (const uint8_t*)relu_mask, rows, C, part, fc ? fc + 2 : nullptr);
  const uint64_t nv = rows * (uint64_t)C / 8;
  if (!fold_in_apply(rows, C, st)) {
    nsk::launch_pdl(bn_bwd_finalize, C, FT, 0, st, (const float*)part, nb, rows, C, gamma_beta, mean, invstd,
                    dgamma_beta, beta_acc, coef);
    nsk::launch_pdl(bn_bwd_apply_kernel, apply_grid(nv), BT, 3 * C * sizeof(float), st, (const __nv_bfloat16*)dy,
                    (const __nv_bfloat16*)x, (const uint8_t*)relu_mask, (const float*)coef, (__nv_bfloat16*)dx,
                    (__nv_bfloat16*)dres, rows, C);
    NSK_LAUNCH_CHECK("bn_bwd");
    return NSK_OK;
  }
  nsk::launch_pdl(bn_bwd_apply_fold_kernel, fold_grid(nv, C), AT, 3 * C * sizeof(float), st, (const float*)part, nb,
                  rows, C, gamma_beta, mean, invstd, dgamma_beta, beta_acc, coef, (const __nv_bfloat16*)dy,
                  (const __nv_bfloat16*)x, (const uint8_t*)relu_mask, (__nv_bfloat16*)dx, (__nv_bfloat16*)dres,
                  fold_blocks(C), fold_counters(st) + 2);
  NSK_LAUNCH_CHECK("bn_bwd");
  return NSK_OK;
}

// backward from channel partials produced by the dgrad that wrote dz (nsk_conv2d_dgrad_bnstats: dz is already
// ReLU-masked): finalize + apply, no reduction pass over dz and x
int nsk_bn_bwd_partials(const float* partials, int nparts, const void* dz, const void* x, const float* gamma_beta,
                        const float* mean, const float* invstd, void* dx, void* dres, float* dgamma_beta,
                        float beta_acc, uint64_t rows, int C, float* ws, void* stream) {
  int rc = check(rows, C, dz, x);
  if (rc) return rc;
  if (nparts < 1) return nsk::set_error(NSK_ERR_SHAPE, "batchnorm backward: no statistics partials");
  cudaStream_t st = (cudaStream_t)stream;
  float* coef = ws + (size_t)MAXBLK * 2 * C;
  const uint64_t nv = rows * (uint64_t)C / 8;
  if (!fold_in_apply(rows, C, st)) {
    nsk::launch_pdl(bn_bwd_finalize, C, FT, 0, st, partials, nparts, rows, C, gamma_beta, mean, invstd, dgamma_beta,
                    beta_acc, coef);
    nsk::launch_pdl(bn_bwd_apply_kernel, apply_grid(nv), BT, 3 * C * sizeof(float), st,
                    (const __nv_bfloat16*)dz, (const __nv_bfloat16*)x, (const uint8_t*)nullptr, (const float*)coef,
                    (__nv_bfloat16*)dx, (__nv_bfloat16*)dres, rows, C);
    NSK_LAUNCH_CHECK("bn_bwd_partials");
    return NSK_OK;
  }
  nsk::launch_pdl(bn_bwd_apply_fold_kernel, fold_grid(nv, C), AT, 3 * C * sizeof(float), st, partials, nparts, rows,
                  C, gamma_beta, mean, invstd, dgamma_beta, beta_acc, coef, (const __nv_bfloat16*)dz,
                  (const __nv_bfloat16*)x, (const uint8_t*)nullptr, (__nv_bfloat16*)dx, (__nv_bfloat16*)dres,
                  fold_blocks(C), fold_counters(st) + 2);
  NSK_LAUNCH_CHECK("bn_bwd_partials");
  return NSK_OK;
}

}  // extern "C"
