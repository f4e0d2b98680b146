// Fused GRU sequence kernels (K16): one persistent cooperative launch per direction.
//
// The reference builds a GRU from primitives (linear, sigmoid, tanh, hadamard, add,
// neg, scalar-add -- tensor.py:247-296, autodiff.py:253-293), one op and one tape node per gate per
// step. Here the input projection for all T steps is one tcgen05 GEMM (host side), and the whole
// recurrence runs in ONE kernel: CTA j owns HU hidden units (all three gates), keeps its slice of U
// resident in shared memory for all T steps, and the CTAs meet at a grid barrier once per step.
//
//   r = s(gx_r + h U_r^T + c_r)      z = s(gx_z + h U_z^T + c_z)
//   a = h U_n^T + c_n                 n = tanh(gx_n + r * a)
//   h' = (1 - z) * n + z * h          (== n - z*n + z*h, the reference composition)
//
// Backward (BPTT, reverse sweep): per step the gate derivatives are elementwise on saved
// (r, z, n, a); the recurrent part dh_prev = dh*z + dgh U is formed split-K over the CTAs
// (partials through global memory, one grid barrier per step). dW, dU, db, dc, dX are batched GEMMs/column
// sums over all steps afterwards (host side), using the dgx / dgh these kernels emit.
// fp32 throughout (the recurrence compounds rounding over T steps).
#include <cooperative_groups.h>

#include "common.cuh"
#include "../../include/nskb.h"

namespace cg = cooperative_groups;

namespace {

constexpr int GT = 256;  // threads per CTA
constexpr int PAD = 4;   // row padding (floats) for conflict-free float4 reads

__device__ __forceinline__ float sigm(float x) {
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

// gx [T][B][3H] (includes b), U [3H][H], c [3H]; hs [T+1][B][H] with hs[0] = h0; gates [T][B][4][H]
__global__ void __launch_bounds__(GT, 1) gru_fwd_kernel(const float* __restrict__ gx, const float* __restrict__ U,
                                                        const float* __restrict__ c, int T, int B, int H, int HU,
                                                        float* hs, float* gates) {
  pdl_wait();
  extern __shared__ float sm[];
  const int HP = H + PAD;
  float* hsm = sm;                    // [B][HP]
  float* usm = sm + (size_t)B * HP;   // [3*HU][HP]: r rows, z rows, n rows of this CTA's units
  cg::grid_group grid = cg::this_grid();
  const int j0 = blockIdx.x * HU;
  for (int i = threadIdx.x; i < 3 * HU * H; i += GT) {
    const int row = i / H, k = i - row * H;
    const int g = row / HU, u = row - g * HU;
    usm[row * HP + k] = U[(size_t)(g * H + j0 + u) * H + k];
  }
  for (int t = 0; t < T; ++t) {
    const float* hprev = hs + (size_t)t * B * H;
    __syncthreads();
    for (int i = threadIdx.x * 4; i < B * H; i += GT * 4) {
      const int b = i / H, k = i - b * H;
      *(float4*)(hsm + b * HP + k) = *(const float4*)(hprev + i);
    }
    __syncthreads();
    for (int o = threadIdx.x; o < B * HU; o += GT) {
      const int b = o / HU, u = o - b * HU, j = j0 + u;
      const float* hr = hsm + b * HP;
      const float* ur = usm + (0 * HU + u) * HP;
      const float* uz = usm + (1 * HU + u) * HP;
      const float* un = usm + (2 * HU + u) * HP;
      float ar = 0.f, az = 0.f, an = 0.f;
#pragma unroll 4
      for (int k = 0; k < H; k += 4) {
        const float4 h4 = *(const float4*)(hr + k);
        const float4 r4 = *(const float4*)(ur + k);
        const float4 z4 = *(const float4*)(uz + k);
        const float4 n4 = *(const float4*)(un + k);
        ar = fmaf(h4.x, r4.x, ar); ar = fmaf(h4.y, r4.y, ar); ar = fmaf(h4.z, r4.z, ar); ar = fmaf(h4.w, r4.w, ar);
        az = fmaf(h4.x, z4.x, az); az = fmaf(h4.y, z4.y, az); az = fmaf(h4.z, z4.z, az); az = fmaf(h4.w, z4.w, az);
        an = fmaf(h4.x, n4.x, an); an = fmaf(h4.y, n4.y, an); an = fmaf(h4.z, n4.z, an); an = fmaf(h4.w, n4.w, an);
      }
      const float* g3 = gx + ((size_t)t * B + b) * 3 * H;
      const float r = sigm(g3[j] + ar + c[j]);
      const float z = sigm(g3[H + j] + az + c[H + j]);
      const float a = an + c[2 * H + j];
      const float n = tanhf(g3[2 * H + j] + r * a);
      const float hp = hr[j];
      const float hn = n - z * n + z * hp;
      hs[((size_t)(t + 1) * B + b) * H + j] = hn;
      float* gs = gates + ((size_t)t * B + b) * 4 * H;
      gs[j] = r;
      gs[H + j] = z;
      gs[2 * H + j] = n;
      gs[3 * H + j] = a;
    }
    grid.sync();  // h_t complete before any CTA reads it
  }
}

// dhs [T][B][H]: external gradient of each h_{t+1} (t = 0..T-1); U [3H][H]; hs, gates from forward.
// Writes dgx [T][B][3H] (= d pre-activation of gx: r, z, n) and dgh [T][B][3H] (r, z, and d a), dh0 [B][H].
// Recurrent term dh_prev = dh*z + dgh U is formed split-K over the CTAs: CTA g multiplies only the dgh of
// its own 3*HU gate rows with its own U rows (the same smem-resident slice the forward uses) into a
// partial [B][H]; after one grid barrier each CTA sums the G partials for its own units.
// scratch: dhcur [2][B][H] running dh, part [2][G][B][H] partials (double-buffered by step parity).
__global__ void __launch_bounds__(GT, 1) gru_bwd_kernel(const float* __restrict__ dhs, const float* __restrict__ U,
                                                        const float* __restrict__ hs, const float* __restrict__ gates,
                                                        int T, int B, int H, int HU, float* dgx, float* dgh,
                                                        float* dh0, float* dhcur, float* part) {
  pdl_wait();
  extern __shared__ float sm[];
  const int H3 = 3 * H;
  const int HP = H + PAD;
  const int R3 = 3 * HU;
  float* usm = sm;                        // [3*HU][HP] own U rows (r rows, z rows, n rows)
  float* gsm = sm + (size_t)R3 * HP;      // [B][3*HU] own dgh for this step
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  const int j0 = blockIdx.x * HU;
  for (int i = threadIdx.x; i < R3 * H; i += GT) {
    const int row = i / H, k = i - row * H;
    const int g = row / HU, u = row - g * HU;
    usm[row * HP + k] = U[(size_t)(g * H + j0 + u) * H + k];
  }
  // dh for step T-1 starts as the external gradient of h_T (each CTA only touches its own units' dh)
  for (int o = threadIdx.x; o < B * HU; o += GT) {
    const int b = o / HU, j = j0 + o - (o / HU) * HU;
    dhcur[(size_t)((T - 1) & 1) * B * H + (size_t)b * H + j] = dhs[((size_t)(T - 1) * B + b) * H + j];
  }
  __syncthreads();
  for (int t = T - 1; t >= 0; --t) {
    float* dcur = dhcur + (size_t)(t & 1) * B * H;
    float* dnext = dhcur + (size_t)((t + 1) & 1) * B * H;
    float* pbuf = part + (size_t)(t & 1) * G * B * H;
    // 1) gate derivatives for this CTA's units (also kept in smem for the partial product)
    for (int o = threadIdx.x; o < B * HU; o += GT) {
      const int b = o / HU, u = o - b * HU, j = j0 + u;
      const float dh = dcur[(size_t)b * H + j];
      const float* gs = gates + ((size_t)t * B + b) * 4 * H;
      const float r = gs[j], z = gs[H + j], n = gs[2 * H + j], a = gs[3 * H + j];
      const float hp = hs[((size_t)t * B + b) * H + j];
      const float dn = dh * (1.f - z);
      const float dz = dh * (hp - n);
      const float dnp = dn * (1.f - n * n);
      const float drp = dnp * a * r * (1.f - r);
      const float dzp = dz * z * (1.f - z);
      float* gxo = dgx + ((size_t)t * B + b) * H3;
      float* gho = dgh + ((size_t)t * B + b) * H3;
      gxo[j] = drp;
      gxo[H + j] = dzp;
      gxo[2 * H + j] = dnp;
      gho[j] = drp;
      gho[H + j] = dzp;
      gho[2 * H + j] = dnp * r;
      gsm[b * R3 + u] = drp;
      gsm[b * R3 + HU + u] = dzp;
      gsm[b * R3 + 2 * HU + u] = dnp * r;
    }
    __syncthreads();
    // 2) partial[g][b][k] = sum over own rows of dgh[b,row] * U[row,k]
    for (int o = threadIdx.x * 4; o < B * H; o += GT * 4) {
      const int b = o / H, k = o - b * H;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int row = 0; row < R3; ++row) {
        const float gv = gsm[b * R3 + row];
        const float4 u4 = *(const float4*)(usm + row * HP + k);
        acc.x = fmaf(gv, u4.x, acc.x);
        acc.y = fmaf(gv, u4.y, acc.y);
        acc.z = fmaf(gv, u4.z, acc.z);
        acc.w = fmaf(gv, u4.w, acc.w);
      }
      *(float4*)(pbuf + ((size_t)blockIdx.x * B + b) * H + k) = acc;
    }
    grid.sync();  // all partials of step t written
    // 3) dh_prev for own units = dh*z + sum_g partial[g] (+ external dhs[t-1]); fixed order over g
    for (int o = threadIdx.x; o < B * HU; o += GT) {
      const int b = o / HU, u = o - b * HU, j = j0 + u;
      float acc = 0.f;
      for (int g = 0; g < G; ++g) acc += __ldcg(pbuf + ((size_t)g * B + b) * H + j);
      const float z = gates[((size_t)t * B + b) * 4 * H + H + j];
      const float dh = dcur[(size_t)b * H + j];
      float dprev = dh * z + acc;
      if (t > 0) {
        dprev += dhs[((size_t)(t - 1) * B + b) * H + j];
        dnext[(size_t)b * H + j] = dprev;
      } else {
        dh0[(size_t)b * H + j] = dprev;
      }
    }
    // no barrier: step t-1 reads only this CTA's dh entries and writes the other partial buffer
    __syncthreads();
  }
}

int pick_hu(int H, int* hu) {
  const int sms = nsk::sm_count();
  for (int u = 1; u <= H; ++u)
    if (H % u == 0 && H / u <= sms) {
      *hu = u;
      return NSK_OK;
    }
  return nsk::set_error(NSK_ERR_UNSUPPORTED, "gru: hidden size does not partition over the SMs");
}

int coop_launch(const void* fn, int grid, size_t smem, void** args, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return nsk::cuda_status(e, "gru: cudaFuncSetAttribute");
  e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(GT), args, smem, st);
  if (e != cudaSuccess) return nsk::cuda_status(e, "gru: cudaLaunchCooperativeKernel");
  return NSK_OK;
}

}  // namespace

extern "C" {

int nsk_gru_fwd(const float* gx, const float* U, const float* c, int T, int B, int H, float* hs, float* gates,
                void* stream) {
  if (T < 1 || B < 1 || H < 4 || H % 4) return nsk::set_error(NSK_ERR_SHAPE, "gru: need T, B >= 1 and H % 4 == 0");
  int HU;
  int rc = pick_hu(H, &HU);
  if (rc) return rc;
  const size_t smem = ((size_t)B * (H + PAD) + (size_t)3 * HU * (H + PAD)) * sizeof(float);
  if (smem > 220 * 1024) return nsk::set_error(NSK_ERR_UNSUPPORTED, "gru: batch x hidden too large for one CTA");
  void* args[] = {(void*)&gx, (void*)&U, (void*)&c, (void*)&T, (void*)&B, (void*)&H, (void*)&HU, (void*)&hs,
                  (void*)&gates};
  return coop_launch((const void*)gru_fwd_kernel, H / HU, smem, args, (cudaStream_t)stream);
}

uint64_t nsk_gru_bwd_workspace(int T, int B, int H) {
  int HU = 1;
  pick_hu(H, &HU);
  const uint64_t G = (uint64_t)(H / HU);
  return (uint64_t)2 * B * H * sizeof(float) + 2 * G * B * H * sizeof(float);
}

int nsk_gru_bwd(const float* dhs, const float* U, const float* hs, const float* gates, int T, int B, int H, float* dgx,
                float* dgh, float* dh0, void* ws, uint64_t ws_bytes, void* stream) {
  if (ws_bytes < nsk_gru_bwd_workspace(T, B, H)) return nsk::set_error(NSK_ERR_SHAPE, "gru: workspace too small");
  int HU;
  int rc = pick_hu(H, &HU);
  if (rc) return rc;
  const size_t smem = ((size_t)3 * HU * (H + PAD) + (size_t)B * 3 * HU) * sizeof(float);
  if (smem > 220 * 1024) return nsk::set_error(NSK_ERR_UNSUPPORTED, "gru bwd: hidden slice too large for one CTA");
  float* dhcur = (float*)ws;
  float* part = dhcur + (size_t)2 * B * H;
  void* args[] = {(void*)&dhs, (void*)&U, (void*)&hs, (void*)&gates, (void*)&T, (void*)&B, (void*)&H, (void*)&HU,
                  (void*)&dgx, (void*)&dgh, (void*)&dh0, (void*)&dhcur, (void*)&part};
  return coop_launch((const void*)gru_bwd_kernel, H / HU, smem, args, (cudaStream_t)stream);
}

}  // extern "C"
