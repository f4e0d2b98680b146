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
__global__ void maxpool_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, int N, int H,
                                   int W, int C, int k, int st, int pad, int P, int Q) {
  pdl_wait();
  const long long n_out = (long long)N * P * Q * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_out; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    long long t = i / C;
    int q = (int)(t % Q);
    t /= Q;
    int p = (int)(t % P);
    long long n = t / P;
    float best = -INFINITY;
    for (int r = 0; r < k; ++r) {
      int h = p * st - pad + r;
      if (h < 0 || h >= H) continue;
      for (int s = 0; s < k; ++s) {
        int w = q * st - pad + s;
        if (w < 0 || w >= W) continue;
        float v = __bfloat162float(x[((n * H + h) * W + w) * C + c]);
        if (v > best) best = v;
      }
    }
    y[i] = __float2bfloat16_rn(best);
  }
}

// gather formulation: each input element sums dy over the windows whose (first) argmax it is. No atomics.
__global__ void maxpool_bwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy,
                                   __nv_bfloat16* __restrict__ dx, int N, int H, int W, int C, int k, int st, int pad,
                                   int P, int Q) {
  pdl_wait();
  const long long n_in = (long long)N * H * W * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_in; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    long long t = i / C;
    int w = (int)(t % W);
    t /= W;
    int h = (int)(t % H);
    long long n = t / H;
    float acc = 0.f;
    // outputs p with p*st - pad <= h <= p*st - pad + k - 1
    int p_lo = (h + pad - k + 1 + st - 1) / st;
    if (h + pad - k + 1 < 0) p_lo = 0;
    int p_hi = (h + pad) / st;
    int q_lo = (w + pad - k + 1 + st - 1) / st;
    if (w + pad - k + 1 < 0) q_lo = 0;
    int q_hi = (w + pad) / st;
    for (int p = p_lo; p <= p_hi && p < P; ++p)
      for (int q = q_lo; q <= q_hi && q < Q; ++q) {
        float best = -INFINITY;
        int bh = -1, bw = -1;
        for (int r = 0; r < k; ++r) {
          int hh = p * st - pad + r;
          if (hh < 0 || hh >= H) continue;
          for (int s = 0; s < k; ++s) {
            int ww = q * st - pad + s;
            if (ww < 0 || ww >= W) continue;
            float v = __bfloat162float(x[((n * H + hh) * W + ww) * C + c]);
            if (bh < 0 || v > best) {
              best = v;
              bh = hh;
              bw = ww;
            }
          }
        }
        if (bh == h && bw == w) acc += __bfloat162float(dy[((n * P + p) * Q + q) * C + c]);
      }
    dx[i] = __float2bfloat16_rn(acc);
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

int nsk_maxpool_fwd(const void* x, void* y, int N, int H, int W, int C, int k, int stride, int pad, int P, int Q,
                    void* stream) {
  long long n = (long long)N * P * Q * C;
  nsk::launch_pdl(maxpool_fwd_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)x, (__nv_bfloat16*)y, N, H, W, C, k, stride, pad, P, Q);
  NSK_LAUNCH_CHECK("maxpool_fwd");
  return NSK_OK;
}

int nsk_maxpool_bwd(const void* x, const void* dy, void* dx, int N, int H, int W, int C, int k, int stride, int pad,
                    int P, int Q, void* stream) {
  long long n = (long long)N * H * W * C;
  nsk::launch_pdl(maxpool_bwd_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, N, H, W, C, k, stride, pad, P, Q);
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
