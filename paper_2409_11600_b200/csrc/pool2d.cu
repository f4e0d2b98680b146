// Pooling (K17), layout conversion, stem im2col and GPU augmentation (K18).
//
// All absent from the reference; restated in
// oracle/restated.py. Augmentation applies crop offsets and flip bits drawn
// on the host in a fixed order (bit-exact indexing, north star), as the
// paper ran its crop/flip preprocessing on the GPU.
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

template <typename T>
__device__ __forceinline__ float ldv(const T* p);
template <>
__device__ __forceinline__ float ldv<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ldv<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T>
__device__ __forceinline__ void stv(T* p, float v);
template <>
__device__ __forceinline__ void stv<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void stv<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// global average pool: x [N, HW, C] -> y [N, C] (fp32), float64 accumulate
template <typename T>
__global__ void avgpool_fwd_kernel(const T* __restrict__ x, float* __restrict__ y, int N, int HW, int C) {
  pdl_wait();
  const long long n_out = (long long)N * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_out; i += (long long)gridDim.x * blockDim.x) {
    long long n = i / C;
    int c = (int)(i - n * C);
    const T* p = x + n * (long long)HW * C + c;
    double s = 0.0;
    for (int k = 0; k < HW; ++k) s += (double)ldv<T>(p + (long long)k * C);
    y[i] = (float)(s / (double)HW);
  }
}

template <typename T>
__global__ void avgpool_bwd_kernel(const float* __restrict__ dy, T* __restrict__ dx, int N, int HW, int C) {
  pdl_wait();
  const long long n = (long long)N * HW * C;
  const float inv = 1.f / (float)HW;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    long long img = i / ((long long)HW * C);
    int c = (int)(i % C);
    stv<T>(dx + i, dy[img * C + c] * inv);
  }
}

// max pool (NHWC bf16): window k x k, stride, pad (padding = -inf); first maximum wins (numpy argmax convention)
// 8 channels per thread (16-byte loads); the window position of the first maximum (row-major window order,
// strictly greater wins: restated.maxpool_bwd) is saved per output element as one byte for the backward.
// KC > 0: the window size as a compile-time constant, the K*K loads issued together; KC = 0: runtime k.
template <int KC>
__global__ void maxpool_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                   uint8_t* __restrict__ arg, int N, int H, int W, int C, int k_rt, int st, int pad,
                                   int P, int Q) {
  const int k = KC > 0 ? KC : k_rt;
  pdl_wait();
  const int CV = C / 8;
  const long long n_out = (long long)N * P * Q * CV;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_out; i += (long long)gridDim.x * blockDim.x) {
    // 32-bit index arithmetic (the host checks N*P*Q*C/8 < 2^31): 64-bit divisions cost ~4x more
    const unsigned iu = (unsigned)i;
    const int cv = (int)(iu % (unsigned)CV);
    unsigned t = iu / (unsigned)CV;
    const int q = (int)(t % (unsigned)Q);
    t /= (unsigned)Q;
    const int p = (int)(t % (unsigned)P);
    const long long n = t / (unsigned)P;
    float best[8];
    uint32_t at[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      best[j] = -INFINITY;
      at[j] = 0;
    }
    bool first = true;
    if constexpr (KC > 0) {
      uint4 u[KC * KC];
      bool ok[KC * KC];
#pragma unroll
      for (int r = 0; r < KC; ++r)
#pragma unroll
        for (int s = 0; s < KC; ++s) {
          const int h = p * st - pad + r, w = q * st - pad + s;
          ok[r * KC + s] = h >= 0 && h < H && w >= 0 && w < W;
          u[r * KC + s] = ok[r * KC + s] ? __ldg((const uint4*)(x + ((n * H + h) * W + w) * C + cv * 8))
                                        : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
      for (int t = 0; t < KC * KC; ++t) {
        if (!ok[t]) continue;
        const __nv_bfloat162* h2 = (const __nv_bfloat162*)&u[t];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(h2[j]);
          if (first || f.x > best[2 * j]) {
            best[2 * j] = f.x;
            at[2 * j] = t;
          }
          if (first || f.y > best[2 * j + 1]) {
            best[2 * j + 1] = f.y;
            at[2 * j + 1] = t;
          }
        }
        first = false;
      }
    }
    for (int r = 0; KC == 0 && r < k; ++r) {
      const int h = p * st - pad + r;
      if (h < 0 || h >= H) continue;
      for (int s = 0; s < k; ++s) {
        const int w = q * st - pad + s;
        if (w < 0 || w >= W) continue;
        const uint4 u = __ldg((const uint4*)(x + ((n * H + h) * W + w) * C + cv * 8));
        const __nv_bfloat162* h2 = (const __nv_bfloat162*)&u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(h2[j]);
          if (first || f.x > best[2 * j]) {
            best[2 * j] = f.x;
            at[2 * j] = r * k + s;
          }
          if (first || f.y > best[2 * j + 1]) {
            best[2 * j + 1] = f.y;
            at[2 * j + 1] = r * k + s;
          }
        }
        first = false;
      }
    }
    uint4 o;
    o.x = pack_bf16x2(best[0], best[1]);
    o.y = pack_bf16x2(best[2], best[3]);
    o.z = pack_bf16x2(best[4], best[5]);
    o.w = pack_bf16x2(best[6], best[7]);
    *(uint4*)(y + i * 8) = o;
    uint2 a8;
    a8.x = at[0] | (at[1] << 8) | (at[2] << 16) | (at[3] << 24);
    a8.y = at[4] | (at[5] << 8) | (at[6] << 16) | (at[7] << 24);
    *(uint2*)(arg + i * 8) = a8;
  }
}

// gather formulation: each input element sums dy over the windows whose saved first-argmax it is. No atomics,
// fixed summation order (window row-major), 8 channels per thread.
// KC > 0: compile-time window and stride (SC): the at most ceil(K/S)^2 (argmax, dy) pairs an input element gathers
// are loaded together; KC = 0: runtime k, stride.
template <int KC, int SC>
__global__ void maxpool_bwd_kernel(const uint8_t* __restrict__ arg, const __nv_bfloat16* __restrict__ dy,
                                   __nv_bfloat16* __restrict__ dx, int N, int H, int W, int C, int k_rt, int st_rt,
                                   int pad, int P, int Q) {
  const int k = KC > 0 ? KC : k_rt, st = KC > 0 ? SC : st_rt;
  pdl_wait();
  const int CV = C / 8;
  const long long n_in = (long long)N * H * W * CV;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_in; i += (long long)gridDim.x * blockDim.x) {
    const unsigned iu = (unsigned)i;  // 32-bit index arithmetic (host-checked)
    const int cv = (int)(iu % (unsigned)CV);
    unsigned t = iu / (unsigned)CV;
    const int w = (int)(t % (unsigned)W);
    t /= (unsigned)W;
    const int h = (int)(t % (unsigned)H);
    const long long n = t / (unsigned)H;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // outputs p with p*st - pad <= h <= p*st - pad + k - 1
    int p_lo = h + pad - k + 1 <= 0 ? 0 : (h + pad - k + 1 + st - 1) / st;
    const int p_hi = (h + pad) / st;
    int q_lo = w + pad - k + 1 <= 0 ? 0 : (w + pad - k + 1 + st - 1) / st;
    const int q_hi = (w + pad) / st;
    if constexpr (KC > 0) {
      constexpr int NP = (KC + SC - 1) / SC;  // output rows (cols) whose window covers one input row (col)
      uint2 a8[NP * NP];
      uint4 g[NP * NP];
      bool ok[NP * NP];
#pragma unroll
      for (int a = 0; a < NP; ++a)
#pragma unroll
        for (int b = 0; b < NP; ++b) {
          const int p = p_lo + a, q = q_lo + b;
          const int t = a * NP + b;
          ok[t] = p <= p_hi && p < P && q <= q_hi && q < Q;
          const long long o = ((n * P + p) * Q + q) * C + cv * 8;
          a8[t] = ok[t] ? __ldg((const uint2*)(arg + o)) : make_uint2(0xffffffffu, 0xffffffffu);
          g[t] = ok[t] ? __ldg((const uint4*)(dy + o)) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
      for (int a = 0; a < NP; ++a)
#pragma unroll
        for (int b = 0; b < NP; ++b) {  // window row-major order: the same summation order as the loop below
          const int t = a * NP + b;
          if (!ok[t]) continue;
          const uint32_t tap = (h - ((p_lo + a) * st - pad)) * k + (w - ((q_lo + b) * st - pad));
          const __nv_bfloat162* g2 = (const __nv_bfloat162*)&g[t];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(g2[j]);
            const uint32_t word = j < 2 ? a8[t].x : a8[t].y;
            const int sh = (j & 1) * 16;
            if (((word >> sh) & 0xff) == tap) acc[2 * j] += f.x;
            if (((word >> (sh + 8)) & 0xff) == tap) acc[2 * j + 1] += f.y;
          }
        }
    }
    for (int p = p_lo; KC == 0 && p <= p_hi && p < P; ++p) {
      const uint32_t r = h - (p * st - pad);
      for (int q = q_lo; q <= q_hi && q < Q; ++q) {
        const uint32_t tap = r * k + (w - (q * st - pad));
        const long long o = ((n * P + p) * Q + q) * C + cv * 8;
        const uint2 a8 = __ldg((const uint2*)(arg + o));
        const uint4 g = __ldg((const uint4*)(dy + o));
        const __nv_bfloat162* g2 = (const __nv_bfloat162*)&g;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(g2[j]);
          const uint32_t word = j < 2 ? a8.x : a8.y;
          const int sh = (j & 1) * 16;
          if (((word >> sh) & 0xff) == tap) acc[2 * j] += f.x;
          if (((word >> (sh + 8)) & 0xff) == tap) acc[2 * j + 1] += f.y;
        }
      }
    }
    uint4 u;
    u.x = pack_bf16x2(acc[0], acc[1]);
    u.y = pack_bf16x2(acc[2], acc[3]);
    u.z = pack_bf16x2(acc[4], acc[5]);
    u.w = pack_bf16x2(acc[6], acc[7]);
    *(uint4*)(dx + i * 8) = u;
  }
}

__global__ void nchw_to_nhwc_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int N, int C, int H,
                                    int W, int Cp) {
  pdl_wait();
  const long long n = (long long)N * H * W * Cp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % Cp);
    long long t = i / Cp;
    int w = (int)(t % W);
    t /= W;
    int h = (int)(t % H);
    long long b = t / H;
    float v = c < C ? x[((b * C + c) * H + h) * W + w] : 0.f;
    y[i] = __float2bfloat16_rn(v);
  }
}

template <typename T>
__global__ void nhwc_to_nchw_kernel(const T* __restrict__ x, float* __restrict__ y, int N, int C, int H, int W, int Cp) {
  pdl_wait();
  const long long n = (long long)N * C * H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int w = (int)(i % W);
    long long t = i / W;
    int h = (int)(t % H);
    t /= H;
    int c = (int)(t % C);
    long long b = t / C;
    y[i] = ldv<T>(x + ((b * H + h) * W + w) * Cp + c);
  }
}

// im2col for small-channel stems: out[(n,p,q), k], k = (r*S + s)*C + c, zero for k >= R*S*C or padding
__global__ void im2col_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ out, int N, int H,
                              int W, int C, int R, int S, int st, int pad, int P, int Q, int Kp) {
  pdl_wait();
  const long long n = (long long)N * P * Q * Kp;
  const int RSC = R * S * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int kk = (int)(i % Kp);
    long long pix = i / Kp;
    float v = 0.f;
    if (kk < RSC) {
      int c = kk % C;
      int rs = kk / C;
      int s = rs % S, r = rs / S;
      int q = (int)(pix % Q);
      long long t = pix / Q;
      int p = (int)(t % P);
      long long b = t / P;
      int h = p * st - pad + r, w = q * st - pad + s;
      if (h >= 0 && h < H && w >= 0 && w < W) v = __bfloat162float(x[((b * H + h) * W + w) * C + c]);
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

// Fused layout change + im2col for image stems (x is the host-layout NCHW float32 batch).
// One thread per (output pixel, 8-column group) of the [N*P*Q, Kp] bf16 cols matrix; column kk = (r*S + s)*C + c
// (KRSC filter order) gathers x[n, c, p*st - pad + r, q*st - pad + s] from the NCHW float32 batch. The kk ->
// (c, r, s) decode comes from a shared-memory table so the loop body is loads and converts only.
// Row-tiled variant: one CTA per output row (n, p). The input window it needs -- C planes x R rows x the
// (Q-1)*st + S columns the row's taps span -- is loaded once, coalesced along W, into shared memory (zero outside
// the image); the Q x Kp im2col rows are then written as consecutive 16-byte pieces. The per-element gather from
// L2 it replaces was 4.6x off HBM bandwidth on the 224x224 ResNet-50 stem.
__global__ void __launch_bounds__(256) im2col_nchw_rows_kernel(const float* __restrict__ x,
                                                               __nv_bfloat16* __restrict__ out, int N, int C, int H,
                                                               int W, int R, int S, int st, int pad, int P, int Q,
                                                               int Kp, int Wp) {
  pdl_wait();
  extern __shared__ float patch[];  // [C][R][Wp] then int off[Kp]: column k's patch offset (-1: padding column)
  int* off = (int*)(patch + (size_t)C * R * Wp);
  const int RSC = R * S * C;
  for (int kk = threadIdx.x; kk < Kp; kk += blockDim.x) {
    if (kk < RSC) {
      const int c = kk % C, rs = kk / C;
      off[kk] = (c * R + rs / S) * Wp + rs % S;
    } else {
      off[kk] = -1;
    }
  }
  const int n = blockIdx.x / P, p = blockIdx.x - n * P;
  const int h0 = p * st - pad, w0 = -pad;
  const long long HW = (long long)H * W;
  const float* xb = x + (long long)n * C * HW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int row = warp; row < C * R; row += blockDim.x >> 5) {  // one patch row per warp, coalesced along W
    const int c = row / R, h = h0 + row - c * R;
    const bool hok = h >= 0 && h < H;
    const float* src = xb + c * HW + (long long)h * W;
    for (int col = lane; col < Wp; col += 32) {
      const int w = w0 + col;
      patch[row * Wp + col] = (hok && w >= 0 && w < W) ? __ldg(src + w) : 0.f;
    }
  }
  __syncthreads();
  // thread -> (column group g, first pixel q0); pixels step by qstep: no divisions in the loop
  const int groups = Kp / 8;
  const int qstep = blockDim.x / groups;
  const int g = threadIdx.x % groups, q0 = threadIdx.x / groups;
  if (q0 >= qstep) return;
  int o[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) o[e] = off[g * 8 + e];
  __nv_bfloat16* ob = out + (long long)blockIdx.x * Q * Kp + g * 8;
  for (int q = q0; q < Q; q += qstep) {
    const float* pq = patch + q * st;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = o[e] >= 0 ? pq[o[e]] : 0.f;
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]);
    u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]);
    u.w = pack_bf16x2(v[6], v[7]);
    *(uint4*)(ob + (long long)q * Kp) = u;
  }
}

__global__ void im2col_nchw_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int N, int C, int H,
                                   int W, int R, int S, int st, int pad, int P, int Q, int Kp) {
  pdl_wait();
  extern __shared__ int tab[];  // [Kp]: (c << 16) | (r << 8) | s, or -1 for padding columns
  const int RSC = R * S * C;
  for (int kk = threadIdx.x; kk < Kp; kk += blockDim.x) {
    if (kk < RSC) {
      const int c = kk % C, rs = kk / C;
      tab[kk] = (c << 16) | ((rs / S) << 8) | (rs % S);
    } else {
      tab[kk] = -1;
    }
  }
  __syncthreads();
  const int groups = Kp / 8;
  const long long total = (long long)N * P * Q * groups;
  const long long HW = (long long)H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(i % groups);
    const long long pix = i / groups;
    const int q = (int)(pix % Q);
    const long long np = pix / Q;
    const int p = (int)(np % P);
    const long long n = np / P;
    const int h0 = p * st - pad, w0 = q * st - pad;
    const float* xb = x + n * C * HW;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int t = tab[g * 8 + e];
      float val = 0.f;
      if (t >= 0) {
        const int h = h0 + ((t >> 8) & 0xff), w = w0 + (t & 0xff);
        if (h >= 0 && h < H && w >= 0 && w < W) val = __ldg(xb + (t >> 16) * HW + (long long)h * W + w);
      }
      v[e] = val;
    }
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]);
    u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]);
    u.w = pack_bf16x2(v[6], v[7]);
    *(uint4*)(out + pix * Kp + g * 8) = u;
  }
}

// col2im (gather form, deterministic): dx[n,h,w,c] = sum_{r,s: h = p*st-pad+r, w = q*st-pad+s} dcols[(n,p,q), k]
__global__ void col2im_kernel(const float* __restrict__ dcols, __nv_bfloat16* __restrict__ dx, int N, int H,
                              int W, int C, int R, int S, int st, int pad, int P, int Q, int Kp) {
  pdl_wait();
  const long long n = (long long)N * H * W * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    long long t = i / C;
    int w = (int)(t % W);
    t /= W;
    int h = (int)(t % H);
    long long b = t / H;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
      int hp = h + pad - r;
      if (hp < 0 || hp % st) continue;
      int p = hp / st;
      if (p >= P) continue;
      for (int s = 0; s < S; ++s) {
        int wq = w + pad - s;
        if (wq < 0 || wq % st) continue;
        int q = wq / st;
        if (q >= Q) continue;
        acc += dcols[((b * P + p) * Q + q) * (long long)Kp + (r * S + s) * C + c];
      }
    }
    dx[i] = __float2bfloat16_rn(acc);
  }
}

// out[n,h,w,c] = ((img[n, h+dy-pad, w'+dx-pad, c] or 0) / 255 - mean[c]) / std[c],  w' = flip ? W-1-w : w
__global__ void augment_kernel(const uint8_t* __restrict__ img, const int32_t* __restrict__ offs,
                               __nv_bfloat16* __restrict__ out, int N, int H, int W, int C, int pad,
                               const float* __restrict__ mean, const float* __restrict__ stdv, int Cp) {
  pdl_wait();
  const long long n = (long long)N * H * W * Cp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % Cp);
    long long t = i / Cp;
    int w = (int)(t % W);
    t /= W;
    int h = (int)(t % H);
    long long b = t / H;
    float v = 0.f;
    if (c < C) {
      const int oy = offs[b * 3 + 0], ox = offs[b * 3 + 1], flip = offs[b * 3 + 2];
      int ww = flip ? (W - 1 - w) : w;
      int sh = h + oy - pad, sw = ww + ox - pad;
      float raw = 0.f;
      if (sh >= 0 && sh < H && sw >= 0 && sw < W) raw = (float)img[((b * H + sh) * W + sw) * C + c];
      v = (raw / 255.f - mean[c]) / stdv[c];
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

}  // namespace

extern "C" {

int nsk_avgpool_fwd(int dtype_in, const void* x, float* y, int N, int HW, int C, void* stream) {
  long long n = (long long)N * C;
  if (dtype_in == NSK_DTYPE_F32)
    nsk::launch_pdl(avgpool_fwd_kernel<float>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, (const float*)x, y, N, HW, C);
  else
    nsk::launch_pdl(avgpool_fwd_kernel<__nv_bfloat16>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, 
        (const __nv_bfloat16*)x, y, N, HW, C);
  NSK_LAUNCH_CHECK("avgpool_fwd");
  return NSK_OK;
}

int nsk_avgpool_bwd(const float* dy, int dtype_out, void* dx, int N, int HW, int C, void* stream) {
  long long n = (long long)N * HW * C;
  if (dtype_out == NSK_DTYPE_F32)
    nsk::launch_pdl(avgpool_bwd_kernel<float>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, dy, (float*)dx, N, HW, C);
  else
    nsk::launch_pdl(avgpool_bwd_kernel<__nv_bfloat16>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, 
        dy, (__nv_bfloat16*)dx, N, HW, C);
  NSK_LAUNCH_CHECK("avgpool_bwd");
  return NSK_OK;
}

int nsk_maxpool_fwd(const void* x, void* y, void* argmax, int N, int H, int W, int C, int k, int stride, int pad,
                    int P, int Q, void* stream) {
  if (C % 8 || ((uintptr_t)x & 15) || ((uintptr_t)y & 15) || ((uintptr_t)argmax & 7) || k * k > 255)
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "maxpool: C must be a multiple of 8, buffers aligned, k*k < 256");
  long long n = (long long)N * P * Q * C;
  if ((long long)N * P * Q * (C / 8) >= (1ll << 31) || (long long)N * H * W * (C / 8) >= (1ll << 31))
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "maxpool: more than 2^31 channel groups");
  // (a compile-time 3x3 window that issues the nine loads together measured slower: 83 registers, 25% occupancy)
  nsk::launch_pdl(maxpool_fwd_kernel<0>, nsk::grid_for(n / 8, 256), 256, 0, (cudaStream_t)stream,
                  (const __nv_bfloat16*)x, (__nv_bfloat16*)y, (uint8_t*)argmax, N, H, W, C, k, stride, pad, P, Q);
  NSK_LAUNCH_CHECK("maxpool_fwd");
  return NSK_OK;
}

int nsk_maxpool_bwd(const void* argmax, const void* dy, void* dx, int N, int H, int W, int C, int k, int stride,
                    int pad, int P, int Q, void* stream) {
  if (C % 8 || ((uintptr_t)dy & 15) || ((uintptr_t)dx & 15) || ((uintptr_t)argmax & 7))
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "maxpool: C must be a multiple of 8, buffers aligned");
  long long n = (long long)N * H * W * C;
  if (n / 8 >= (1ll << 31)) return nsk::set_error(NSK_ERR_UNSUPPORTED, "maxpool: more than 2^31 channel groups");
  if (k == 3 && stride == 2)
    nsk::launch_pdl(maxpool_bwd_kernel<3, 2>, nsk::grid_for(n / 8, 256), 256, 0, (cudaStream_t)stream,
                    (const uint8_t*)argmax, (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, N, H, W, C, k, stride, pad,
                    P, Q);
  else
    nsk::launch_pdl(maxpool_bwd_kernel<0, 1>, nsk::grid_for(n / 8, 256), 256, 0, (cudaStream_t)stream,
                    (const uint8_t*)argmax, (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, N, H, W, C, k, stride, pad,
                    P, Q);
  NSK_LAUNCH_CHECK("maxpool_bwd");
  return NSK_OK;
}

int nsk_nchw_to_nhwc(const float* x, void* y, int N, int C, int H, int W, int Cp, void* stream) {
  long long n = (long long)N * H * W * Cp;
  nsk::launch_pdl(nchw_to_nhwc_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, x, (__nv_bfloat16*)y, N, C, H, W, Cp);
  NSK_LAUNCH_CHECK("nchw_to_nhwc");
  return NSK_OK;
}

int nsk_nhwc_to_nchw(int dtype_in, const void* x, float* y, int N, int C, int H, int W, int Cp, void* stream) {
  long long n = (long long)N * C * H * W;
  if (dtype_in == NSK_DTYPE_F32)
    nsk::launch_pdl(nhwc_to_nchw_kernel<float>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, (const float*)x, y, N, C, H, W,
                                                                                         Cp);
  else
    nsk::launch_pdl(nhwc_to_nchw_kernel<__nv_bfloat16>, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, 
        (const __nv_bfloat16*)x, y, N, C, H, W, Cp);
  NSK_LAUNCH_CHECK("nhwc_to_nchw");
  return NSK_OK;
}

int nsk_im2col(const void* x, void* out, int N, int H, int W, int C, int R, int S, int stride, int pad, int P, int Q,
               int Kp, void* stream) {
  long long n = (long long)N * P * Q * Kp;
  nsk::launch_pdl(im2col_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)x, (__nv_bfloat16*)out, N, H, W, C, R, S, stride, pad, P, Q, Kp);
  NSK_LAUNCH_CHECK("im2col");
  return NSK_OK;
}

int nsk_im2col_nchw(const float* x, void* out, int N, int C, int H, int W, int R, int S, int stride, int pad, int P,
                    int Q, int Kp, void* stream) {
  if (Kp % 8) return nsk::set_error(NSK_ERR_UNSUPPORTED, "im2col_nchw: Kp must be a multiple of 8");
  if (R > 255 || S > 255 || C > 32767 || Kp > 8192)
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "im2col_nchw: filter too large");
  const int Wp = (Q - 1) * stride + S;  // input columns one output row's taps span
  const size_t tiled = ((size_t)C * R * Wp + Kp) * sizeof(float);
  if (tiled <= 48 * 1024 && Kp / 8 <= 256) {
    nsk::launch_pdl(im2col_nchw_rows_kernel, (unsigned)(N * P), 256, tiled, (cudaStream_t)stream, x,
                    (__nv_bfloat16*)out, N, C, H, W, R, S, stride, pad, P, Q, Kp, Wp);
    NSK_LAUNCH_CHECK("im2col_nchw_rows");
    return NSK_OK;
  }
  const size_t smem = (size_t)Kp * sizeof(int);
  const long long n = (long long)N * P * Q * (Kp / 8);
  nsk::launch_pdl(im2col_nchw_kernel, nsk::grid_for(n, 256), 256, smem, (cudaStream_t)stream, x, (__nv_bfloat16*)out, N, C, H, W, R, S, stride, pad,
                                                                P, Q, Kp);
  NSK_LAUNCH_CHECK("im2col_nchw");
  return NSK_OK;
}

int nsk_col2im(const void* dcols, void* dx, int N, int H, int W, int C, int R, int S, int stride, int pad, int P, int Q,
               int Kp, void* stream) {
  long long n = (long long)N * H * W * C;
  nsk::launch_pdl(col2im_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, 
      (const float*)dcols, (__nv_bfloat16*)dx, N, H, W, C, R, S, stride, pad, P, Q, Kp);
  NSK_LAUNCH_CHECK("col2im");
  return NSK_OK;
}

int nsk_augment_crop_flip(const uint8_t* img, const int32_t* offs, void* out, int N, int H, int W, int C, int pad,
                          const float* mean, const float* stdv, int Cp, void* stream) {
  long long n = (long long)N * H * W * Cp;
  nsk::launch_pdl(augment_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, img, offs, (__nv_bfloat16*)out, N, H, W, C,
                                                                          pad, mean, stdv, Cp);
  NSK_LAUNCH_CHECK("augment_crop_flip");
  return NSK_OK;
}

}  // extern "C"
