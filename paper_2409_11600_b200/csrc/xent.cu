// Softmax cross-entropy (K10), sum-loss, argmax accuracy (K14).
//
// Reference (pkg/src/nsk/):
//   rec_cross_entropy autodiff.py:220-248  loss = mean(lse - z_t) in float64 after max-subtraction,
//                                          probs = exp(z - lse) saved as float32
//   gradient_rule("cross-entropy-loss") autodiff.py:286-292  d = (probs - onehot) * g / m  (float64 math)
//   rec_sum_loss autodiff.py:213-217 (float64 sum); rule autodiff.py:284-285 (broadcast g)
//   _accuracy builtins.py:70-80 (numpy argmax: first maximum wins, NaN counts as the maximum)
// The loss is written to a device scalar: no host synchronisation inside a step.
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

constexpr int XT = 1024;

// One warp per row, XW rows per block; block partial sums of (lse - z_t) go to a library scratch and the last
// block to finish (ticket) folds them in block order: deterministic, one launch, any batch size.
constexpr int XW = 8;

struct XentScratch {
  double* part = nullptr;
  unsigned* ticket = nullptr;
  int cap = 0;
};

__global__ void __launch_bounds__(XW * 32) xent_fwd_kernel(const float* __restrict__ z, const float* __restrict__ tgt,
                                                           int m, int c, float* __restrict__ probs, float* loss,
                                                           int* err, double* part, unsigned* ticket) {
  pdl_wait();
  __shared__ double wpart[XW];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * XW + warp;
  double term = 0.0;
  if (row < m) {
    const float* zr = z + (long long)row * c;
    double mx = -INFINITY;
    for (int j = lane; j < c; j += 32) mx = fmax(mx, (double)zr[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double se = 0.0;
    for (int j = lane; j < c; j += 32) se += exp((double)zr[j] - mx);
    se = warp_sum_d(se);
    const double lse = log(se);
    float* pr = probs + (long long)row * c;
    for (int j = lane; j < c; j += 32) pr[j] = (float)exp((double)zr[j] - mx - lse);
    float tv = tgt[row];
    int t = (int)tv;
    bool ok = tv >= 0.f && tv < (float)c && tv == floorf(tv);
    if (!ok) {
      if (lane == 0 && err) atomicMin(err, row);
      t = 0;
    }
    term = lse - ((double)zr[t] - mx);
  }
  if (lane == 0) wpart[warp] = term;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < XW; ++i) s += wpart[i];
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += ((volatile double*)part)[b];
    loss[0] = (float)(s / (double)m);
    *ticket = 0;  // ready for the next launch (graph replays)
  }
}

__global__ void xent_bwd_kernel(const float* __restrict__ probs, const float* __restrict__ tgt, const float* g, int m,
                                int c, float* __restrict__ d) {
  pdl_wait();
  const double scale = (double)g[0] / (double)m;
  const long long n = (long long)m * c;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int row = (int)(i / c);
    int j = (int)(i - (long long)row * c);
    double v = (double)probs[i];
    if ((float)j == tgt[row]) v -= 1.0;
    d[i] = (float)(v * scale);
  }
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T>
__global__ void __launch_bounds__(XT) sum_kernel(const T* __restrict__ x, uint64_t n, float* out) {
  pdl_wait();
  __shared__ double part[XT / 32];
  double s = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += XT) s += (double)ldf<T>(x + i);
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < XT / 32; ++i) t += part[i];
    out[0] = (float)t;
  }
}

__global__ void fill_scalar_kernel(const float* g, float* out, uint64_t n) {
  pdl_wait();
  const float v = g[0];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

__global__ void argmax_kernel(const float* __restrict__ z, const float* __restrict__ labels, int m, int c, int* count) {
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int local = 0;
  for (int row = warp; row < m; row += nwarps) {
    const float* zr = z + (long long)row * c;
    float best = -INFINITY;
    int bi = -1;
    for (int j = lane; j < c; j += 32) {
      float v = zr[j];
      bool better = (bi < 0) || (isnan(v) && !isnan(best)) || (!isnan(best) && v > best);
      if (better) {
        best = v;
        bi = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      bool take;
      if (oi < 0) take = false;
      else if (bi < 0) take = true;
      else if (isnan(ov) != isnan(best)) take = isnan(ov);
      else if (isnan(ov) || ov == best) take = oi < bi;
      else take = ov > best;
      if (take) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0 && (double)bi == (double)(long long)labels[row]) ++local;
  }
  if (lane == 0 && local) atomicAdd(count, local);
}

}  // namespace

extern "C" {

int nsk_xent_fwd(const float* logits, const float* targets, int m, int c, float* probs, float* loss_out, int* err_flag,
                 void* stream) {
  if (m < 1 || c < 1) return nsk::set_error(NSK_ERR_SHAPE, "cross_entropy: empty logits");
  static XentScratch sc;
  const int blocks = (m + XW - 1) / XW;
  if (blocks > sc.cap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing((cudaStream_t)stream, &cs);
    if (cs != cudaStreamCaptureStatusNone)
      return nsk::set_error(NSK_ERR_UNSUPPORTED, "cross_entropy: scratch must be sized before graph capture");
    if (sc.part) {
      cudaStreamSynchronize((cudaStream_t)stream);
      cudaFree(sc.part);
    }
    const int cap = blocks < 1024 ? 1024 : blocks;
    NSK_CUDA(cudaMalloc(&sc.part, cap * sizeof(double) + 64));
    sc.ticket = (unsigned*)(sc.part + cap);
    NSK_CUDA(cudaMemset(sc.ticket, 0, sizeof(unsigned)));
    sc.cap = cap;
  }
  nsk::launch_pdl(xent_fwd_kernel, blocks, XW * 32, 0, (cudaStream_t)stream, logits, targets, m, c, probs, loss_out, err_flag,
                                                                sc.part, sc.ticket);
  NSK_LAUNCH_CHECK("xent_fwd");
  return NSK_OK;
}

int nsk_xent_bwd(const float* probs, const float* targets, const float* g, int m, int c, float* dlogits,
                 void* stream) {
  long long n = (long long)m * c;
  nsk::launch_pdl(xent_bwd_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, probs, targets, g, m, c, dlogits);
  NSK_LAUNCH_CHECK("xent_bwd");
  return NSK_OK;
}

int nsk_sum_f32(int dtype, const void* x, uint64_t n, float* out, void* stream) {
  if (dtype == NSK_DTYPE_F32)
    nsk::launch_pdl(sum_kernel<float>, 1, XT, 0, (cudaStream_t)stream, (const float*)x, n, out);
  else
    nsk::launch_pdl(sum_kernel<__nv_bfloat16>, 1, XT, 0, (cudaStream_t)stream, (const __nv_bfloat16*)x, n, out);
  NSK_LAUNCH_CHECK("sum");
  return NSK_OK;
}

int nsk_fill_like_scalar(const float* g, float* out, uint64_t n, void* stream) {
  nsk::launch_pdl(fill_scalar_kernel, nsk::grid_for(n, 256), 256, 0, (cudaStream_t)stream, g, out, n);
  NSK_LAUNCH_CHECK("fill_like_scalar");
  return NSK_OK;
}

int nsk_argmax_correct(const float* logits, const float* labels, int m, int c, int* count_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  NSK_CUDA(cudaMemsetAsync(count_out, 0, sizeof(int), st));
  int blocks = (m + 7) / 8;
  if (blocks > 4 * nsk::sm_count()) blocks = 4 * nsk::sm_count();
  if (blocks < 1) blocks = 1;
  nsk::launch_pdl(argmax_kernel, blocks, 256, 0, st, logits, labels, m, c, count_out);
  NSK_LAUNCH_CHECK("argmax_correct");
  return NSK_OK;
}

}  // extern "C"
