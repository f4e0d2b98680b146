// Multi-tensor optimizers (K11 SGD-momentum, K12 AdamW + global-norm clip).
//
// Reference (pkg/src/nsk/nn.py):
//   sgd_step      nn.py:91-99   v <- mu*v + g ; w <- w - lr*v          (float64 math, float32 store)
//   adamw_step    nn.py:102-119 w *= 1 - lr*wd ; bias-corrected Adam  (float64 math, float32 store)
//   clip_grad_norm nn.py:122-139 global float64 L2, grads scaled by float32(max/norm)
// One launch covers every parameter: blockIdx.y selects the tensor, blocks
// stride over its elements. Tensor tables (pointers, sizes) are device arrays
// built once by the Python ParamGroup. The optimizer also refreshes the bf16
// shadow copy of each weight that conv/GEMM kernels read (w_bf16 may be NULL).
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

__global__ void sgd_kernel(float* const* w, const float* const* g, float* const* v, void* const* wb,
                           const uint64_t* numel, double lr, double mu, float gscale) {
  pdl_wait();
  const int t = blockIdx.y;
  const uint64_t n = numel[t];
  float* W = w[t];
  const float* G = g[t];
  float* V = v[t];
  __nv_bfloat16* B = (__nv_bfloat16*)wb[t];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // explicit _rn ops: no FMA contraction, so results match numpy's float64 arithmetic bit for bit
  auto step = [&](float w0, float g0, float v0, float* wo, float* vo) {
    const double gi = (double)__fmul_rn(g0, gscale);
    const double vi = __dadd_rn(__dmul_rn(mu, (double)v0), gi);
    *vo = (float)vi;
    *wo = (float)__dsub_rn((double)w0, __dmul_rn(lr, vi));
  };
  uint64_t head = 0;
  // 16-byte vectors when the tensors allow it (the flat parameter arena does): the update streams 22 B per
  // parameter, so load/store width decides how close it gets to HBM bandwidth
  if ((((uintptr_t)W | (uintptr_t)G | (uintptr_t)V) & 15) == 0 && (((uintptr_t)B) & 7) == 0) {
    const uint64_t n4 = n / 4;
    for (uint64_t i = tid; i < n4; i += stride) {
      const float4 w4 = ((const float4*)W)[i], g4 = __ldg((const float4*)G + i), v4 = ((const float4*)V)[i];
      float4 wo, vo;
      step(w4.x, g4.x, v4.x, &wo.x, &vo.x);
      step(w4.y, g4.y, v4.y, &wo.y, &vo.y);
      step(w4.z, g4.z, v4.z, &wo.z, &vo.z);
      step(w4.w, g4.w, v4.w, &wo.w, &vo.w);
      ((float4*)W)[i] = wo;
      ((float4*)V)[i] = vo;
      if (B) {
        uint2 b;
        b.x = pack_bf16x2(wo.x, wo.y);
        b.y = pack_bf16x2(wo.z, wo.w);
        ((uint2*)B)[i] = b;
      }
    }
    head = n4 * 4;
  }
  for (uint64_t i = head + tid; i < n; i += stride) {
    float wo, vo;
    step(W[i], G[i], V[i], &wo, &vo);
    V[i] = vo;
    W[i] = wo;
    if (B) B[i] = __float2bfloat16_rn(wo);
  }
}

// the optimizer step counter lives on the device so a captured step graph replays with t = 1, 2, 3, ...
__global__ void step_inc_kernel(int* step) {
  pdl_wait(); step[0] += 1; }

__global__ void adamw_kernel(float* const* w, const float* const* g, float* const* m, float* const* v, void* const* wb,
                             const uint64_t* numel, double lr, double wd, double b1, double b2, double eps,
                             const int* step_dev, const float* gscale_dev) {
  pdl_wait();
  __shared__ double bc[2];
  if (threadIdx.x == 0) {
    const double st = (double)step_dev[0];
    bc[0] = 1.0 - pow(b1, st);  // same libm pow as the reference's b1 ** t (nn.py:116-117)
    bc[1] = 1.0 - pow(b2, st);
  }
  __syncthreads();
  const double bc1 = bc[0], bc2 = bc[1];
  const int t = blockIdx.y;
  const uint64_t n = numel[t];
  float* W = w[t];
  const float* G = g[t];
  float* Mm = m[t];
  float* Vv = v[t];
  __nv_bfloat16* B = (__nv_bfloat16*)wb[t];
  const float gs = gscale_dev ? gscale_dev[0] : 1.f;
  const double decay = __dsub_rn(1.0, __dmul_rn(lr, wd)), ob1 = __dsub_rn(1.0, b1), ob2 = __dsub_rn(1.0, b2);
  // the bias corrections as reciprocal multiplies (within one float64 ulp of the reference's m / (1 - b1^t): far
  // below the float32 rounding of the stored results) -- the float64 divisions made the sweep compute-bound
  const double rb1 = 1.0 / bc1, rb2 = 1.0 / bc2;
  // nn.py:108-119 in float64 with explicit _rn ops (no FMA contraction)
  auto step = [&](float w0, float g0, float m0, float v0, float* wo, float* mo, float* vo) {
    const double gi = (double)(gscale_dev ? __fmul_rn(g0, gs) : g0);
    const double wi = __dmul_rn((double)w0, decay);
    const double mi = __dadd_rn(__dmul_rn(b1, (double)m0), __dmul_rn(ob1, gi));
    const double vi = __dadd_rn(__dmul_rn(b2, (double)v0), __dmul_rn(__dmul_rn(ob2, gi), gi));
    *mo = (float)mi;
    *vo = (float)vi;
    const double mh = __dmul_rn(mi, rb1), vh = __dmul_rn(vi, rb2);
    *wo = (float)__dsub_rn(wi, __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps)));
  };
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t head = 0;
  // 16-byte vectors (the flat parameter arena allows them): four independent updates per thread keep the loads of
  // the next elements in flight behind the float64 divisions
  if ((((uintptr_t)W | (uintptr_t)G | (uintptr_t)Mm | (uintptr_t)Vv) & 15) == 0 && (((uintptr_t)B) & 7) == 0) {
    const uint64_t n4 = n / 4;
    for (uint64_t i = tid; i < n4; i += stride) {
      const float4 w4 = ((const float4*)W)[i], g4 = __ldg((const float4*)G + i);
      const float4 m4 = ((const float4*)Mm)[i], v4 = ((const float4*)Vv)[i];
      float4 wo, mo, vo;
      step(w4.x, g4.x, m4.x, v4.x, &wo.x, &mo.x, &vo.x);
      step(w4.y, g4.y, m4.y, v4.y, &wo.y, &mo.y, &vo.y);
      step(w4.z, g4.z, m4.z, v4.z, &wo.z, &mo.z, &vo.z);
      step(w4.w, g4.w, m4.w, v4.w, &wo.w, &mo.w, &vo.w);
      ((float4*)W)[i] = wo;
      ((float4*)Mm)[i] = mo;
      ((float4*)Vv)[i] = vo;
      if (B) {
        uint2 b;
        b.x = pack_bf16x2(wo.x, wo.y);
        b.y = pack_bf16x2(wo.z, wo.w);
        ((uint2*)B)[i] = b;
      }
    }
    head = n4 * 4;
  }
  for (uint64_t i = head + tid; i < n; i += stride) {
    float wo, mo, vo;
    step(W[i], G[i], Mm[i], Vv[i], &wo, &mo, &vo);
    Mm[i] = mo;
    Vv[i] = vo;
    W[i] = wo;
    if (B) B[i] = __float2bfloat16_rn(wo);
  }
}

constexpr int NB = 1024;  // partial slots for the norm reduction

__global__ void sqnorm_partial_kernel(const float* const* g, const uint64_t* numel, int nt, double* part) {
  pdl_wait();
  __shared__ double red[256 / 32];
  double s0 = 0.0, s1 = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int t = 0; t < nt; ++t) {
    const float* G = g[t];
    const uint64_t n = numel[t];
    uint64_t head = 0;
    if (((uintptr_t)G & 15) == 0) {  // 16-byte loads, two in flight per thread
      const uint64_t n4 = n / 4;
      uint64_t i = tid;
      for (; i + stride < n4; i += 2 * stride) {
        const float4 a = __ldg((const float4*)G + i), b = __ldg((const float4*)G + i + stride);
        s0 += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
        s1 += (double)b.x * b.x + (double)b.y * b.y + (double)b.z * b.z + (double)b.w * b.w;
      }
      if (i < n4) {
        const float4 a = __ldg((const float4*)G + i);
        s0 += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
      }
      head = n4 * 4;
    }
    for (uint64_t i = head + tid; i < n; i += stride) {
      const double x = (double)G[i];
      s0 += x * x;
    }
  }
  double s = warp_sum_d(s0 + s1);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 256 / 32; ++i) t += red[i];
    part[1 + blockIdx.x] = t;
  }
}

__global__ void sqnorm_final_kernel(double* part, int nb) {
  pdl_wait();
  double t = 0.0;  // one warp, fixed order: lane strides, then the butterfly
  for (int i = threadIdx.x; i < nb; i += 32) t += part[1 + i];
  t = warp_sum_d(t);
  if (threadIdx.x == 0) part[0] = t;
}

__global__ void clip_scale_kernel(const double* sq, float max_norm, float* scale) {
  pdl_wait();
  double norm = sqrt(sq[0]);
  scale[0] = norm <= (double)max_norm ? 1.f : (float)((double)max_norm / norm);
}

__global__ void scale_kernel(float* const* g, const uint64_t* numel, const float* scale) {
  pdl_wait();
  const float s = scale[0];
  if (s == 1.f) return;
  const int t = blockIdx.y;
  float* G = g[t];
  const uint64_t n = numel[t];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t head = 0;
  if (((uintptr_t)G & 15) == 0) {
    const uint64_t n4 = n / 4;
    for (uint64_t i = tid; i < n4; i += stride) {
      float4 a = ((float4*)G)[i];
      a.x *= s;
      a.y *= s;
      a.z *= s;
      a.w *= s;
      ((float4*)G)[i] = a;
    }
    head = n4 * 4;
  }
  for (uint64_t i = head + tid; i < n; i += stride) G[i] *= s;
}

// blocks per tensor: ~16 resident blocks per SM across the whole launch
unsigned blocks_x(int nt) {
  int b = (16 * nsk::sm_count() + nt - 1) / (nt > 0 ? nt : 1);
  if (b < 16) b = 16;
  if (b > 4096) b = 4096;
  return (unsigned)b;
}

}  // namespace

extern "C" {

int nsk_sgd_multi(int nt, float* const* w, const float* const* g, float* const* v, void* const* wb,
                  const uint64_t* numel, double lr, double momentum, float grad_scale, void* stream) {
  if (nt < 1) return NSK_OK;
  dim3 grid(blocks_x(nt), nt);
  nsk::launch_pdl(sgd_kernel, grid, 256, 0, (cudaStream_t)stream, w, g, v, wb, numel, lr, momentum, grad_scale);
  NSK_LAUNCH_CHECK("sgd_multi");
  return NSK_OK;
}

int nsk_adamw_multi(int nt, float* const* w, const float* const* g, float* const* m, float* const* v,
                    void* const* wb, const uint64_t* numel, int* step_dev, double lr, double wd, double beta1,
                    double beta2, double eps, const float* grad_scale_dev, void* stream) {
  if (nt < 1) return NSK_OK;
  nsk::launch_pdl(step_inc_kernel, 1, 1, 0, (cudaStream_t)stream, step_dev);
  dim3 grid(blocks_x(nt), nt);
  nsk::launch_pdl(adamw_kernel, grid, 256, 0, (cudaStream_t)stream, w, g, m, v, wb, numel, lr, wd, beta1, beta2, eps, step_dev,
                                                       grad_scale_dev);
  NSK_LAUNCH_CHECK("adamw_multi");
  return NSK_OK;
}

// out must hold 1 + 1024 doubles; out[0] receives the sum of squares.
int nsk_sqnorm_multi(int nt, const float* const* g, const uint64_t* numel, double* out, void* stream) {
  int nb = 6 * nsk::sm_count();  // enough 16-byte loads in flight to stream the gradients at HBM rate
  if (nb > NB) nb = NB;
  nsk::launch_pdl(sqnorm_partial_kernel, nb, 256, 0, (cudaStream_t)stream, g, numel, nt, out);
  nsk::launch_pdl(sqnorm_final_kernel, 1, 32, 0, (cudaStream_t)stream, out, nb);
  NSK_LAUNCH_CHECK("sqnorm_multi");
  return NSK_OK;
}

int nsk_clip_scale(const double* sqnorm, float max_norm, float* scale_dev, void* stream) {
  nsk::launch_pdl(clip_scale_kernel, 1, 1, 0, (cudaStream_t)stream, sqnorm, max_norm, scale_dev);
  NSK_LAUNCH_CHECK("clip_scale");
  return NSK_OK;
}

int nsk_scale_multi(int nt, float* const* g, const uint64_t* numel, const float* scale_dev, void* stream) {
  if (nt < 1) return NSK_OK;
  dim3 grid(blocks_x(nt), nt);
  nsk::launch_pdl(scale_kernel, grid, 256, 0, (cudaStream_t)stream, g, numel, scale_dev);
  NSK_LAUNCH_CHECK("scale_multi");
  return NSK_OK;
}

}  // extern "C"
