// Fused GRU recurrence on the tensor cores (K16, tcgen05): thread-block clusters walk all T steps.
//
// Reference: the reference has no GRU op; SURVEY.md A26 defines it as the composition of its primitives
// (linear = matmul_t + bias-add, sigmoid, tanh, hadamard, add, neg, scalar-add: tensor.py:213-296,
// autodiff.py:253-293):
//   r = s(gx_r + h U_r^T + c_r)      z = s(gx_z + h U_z^T + c_z)
//   a = h U_n^T + c_n                 n = tanh(gx_n + r * a)
//   h' = n - z * n + z * h
// gx = x W^T + b for all T steps is one tcgen05 GEMM on the host side; this file is the recurrence.
//
// Batch groups: rows of the batch never interact inside the recurrence, so B / Bc independent clusters of
// CL = H / 32 CTAs each take Bc rows (4 groups of 16 at C3); CTA q of a cluster owns hidden units [32q, 32q + 32).
//
// Forward (gru_fwd_tc_kernel): the CTA's 96 rows of U live in tensor memory as the MMA's A operand; per step
// 32 tcgen05.mma compute D^T = U_q h_t^T (N = the batch rows), all eight warps share the gate math through a
// shared-memory tile, and each CTA's bf16 slice of h_{t+1} is TMA-multicast from a global ring into every CTA.
//
// Backward (BPTT, reverse sweep; the cluster arranged RG x CG):
//   dh_{t-1} = dh_t * z_t + dgh_t U       (dgh = [dr', dz', dn' * r], the gradient w.r.t. h U^T + c)
// CTA (i, j) owns units [j*H/CG + 32 i, +32) and keeps U[rows of row group i, cols of column group j] (in tensor
// memory, transposed: the A operand). Per step: A) form dh_t from the partial products of step t+1 and the gate
// derivatives (fp32), write dgx / dgh for the batched weight-gradient GEMMs, and send this CTA's dgh piece to the
// CTAs of its row group; B) P^T = U^T dgh^T over the row group's gate rows, each 32-column slice to its owner in the
// column group. gru_bwd_push_kernel moves both exchanges by DSMEM bulk copies into double-buffered receive buffers
// (no global rings, no barriers inside the sweep); gru_bwd_tc_kernel (rings in global memory, two split cluster
// barriers per step) covers the shapes the push kernel's buffers do not fit.
//
// Precision: the MMA operands are bf16 (h, dgh, U), accumulation and all gate math / state fp32 (SURVEY.md
// §7 hard part 5; oracle/restated.gru_*_bf16 emulates exactly these roundings).
#include "common.cuh"
#include "../../include/nskb.h"

namespace {

constexpr int kUC = 32;         // hidden units per CTA
constexpr int kThreads = 256;   // 8 warps: 0,1,4,5 epilogue | 2 TMA | 3 MMA + TMEM | 6,7 idle
constexpr int kMaxB = 64;       // batch rows (A operand rows that are read back)
constexpr int kDP = 100;        // row pitch (floats) of the forward's accumulator tile: conflict-free float4 rows
long long* g_trace = nullptr;   // NSK_GRU_TRACE: per-step timestamps of the forward (diagnostics)

// split cluster barrier: the arrive publishes (release) what the peers need, work that only this CTA needs runs
// between arrive and wait, off the critical path
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// 32 lanes x 16 consecutive fp32 columns (thread t of the warp: lane base + t)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* f) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(r[i]);
}

// Gate nonlinearities, branch-free (MUFU ex2 + rcp, no IEEE slow paths, so the 8 units of a thread interleave):
// the reference's stable sigmoid (tensor.py:237-244: exp of -|x| only, nothing overflows) and tanh from the same
// e = exp(-2|x|). Relative error ~1e-6 (absolute ~1e-7 near 0), far below the bf16 rounding of the recurrent
// product's operands.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigm(float x) {
  const float e = ex2_approx(-1.4426950408889634f * fabsf(x));
  const float r = rcp_approx(1.f + e);
  return x >= 0.f ? r : e * r;
}
__device__ __forceinline__ float tanh_fast(float x) {
  const float e = ex2_approx(-2.8853900817779268f * fabsf(x));
  const float t = (1.f - e) * rcp_approx(1.f + e);
  return copysignf(t, x);
}

// 32 lanes x 8 consecutive fp32 columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* f) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 consecutive 32-bit columns from registers (thread t of the warp: lane base + t)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] . B[smem]: A (M = 128 lanes, K = 16 as 8 columns of packed bf16 pairs) read from tensor
// memory, so only B comes from shared memory; BOFF is added to B's descriptor
template <int BOFF>
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\tadd.s64 bd, %2, %5;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], bd, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum), "n"(BOFF)
      : "memory");
}

__device__ __forceinline__ void ld16(const float* p, float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) *(float4*)(v + 4 * i) = __ldcg((const float4*)(p + 4 * i));
}
__device__ __forceinline__ void st16(float* p, const float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) *(float4*)(p + 4 * i) = *(const float4*)(v + 4 * i);
}
__device__ __forceinline__ void ld8(const float* p, float* v) {
  *(float4*)v = __ldcg((const float4*)p);
  *(float4*)(v + 4) = __ldcg((const float4*)(p + 4));
}
__device__ __forceinline__ void st8(float* p, const float* v) {
  *(float4*)p = *(const float4*)v;
  *(float4*)(p + 4) = *(const float4*)(v + 4);
}
__device__ __forceinline__ void st8_bf16(__nv_bfloat16* p, const float* v) {
  uint4 a;
  a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]); a.z = pack_bf16x2(v[4], v[5]);
  a.w = pack_bf16x2(v[6], v[7]);
  *(uint4*)p = a;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// N consecutive fp32 / bf16 values per thread (N = units per thread: 8, 4, 2 or 1)
template <int N>
__device__ __forceinline__ void ldv(const float* p, float* v) {
  if constexpr (N == 8) {
    ld8(p, v);
  } else if constexpr (N == 4) {
    *(float4*)v = __ldcg((const float4*)p);
  } else if constexpr (N == 2) {
    *(float2*)v = __ldcg((const float2*)p);
  } else {
    v[0] = __ldcg(p);
  }
}
template <int N>
__device__ __forceinline__ void ldvs(const float* p, float* v) {  // shared memory
  if constexpr (N >= 4) {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) *(float4*)(v + 4 * i) = *(const float4*)(p + 4 * i);
  } else if constexpr (N == 2) {
    *(float2*)v = *(const float2*)p;
  } else {
    v[0] = p[0];
  }
}
template <int N>
__device__ __forceinline__ void stv(float* p, const float* v) {
  if constexpr (N >= 4) {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) *(float4*)(p + 4 * i) = *(const float4*)(v + 4 * i);
  } else if constexpr (N == 2) {
    *(float2*)p = *(const float2*)v;
  } else {
    p[0] = v[0];
  }
}
template <int N>
__device__ __forceinline__ void stvb(__nv_bfloat16* p, const float* v) {
  if constexpr (N == 8) {
    st8_bf16(p, v);
  } else if constexpr (N == 4) {
    uint2 a;
    a.x = pack_bf16x2(v[0], v[1]);
    a.y = pack_bf16x2(v[2], v[3]);
    *(uint2*)p = a;
  } else if constexpr (N == 2) {
    *(uint32_t*)p = pack_bf16x2(v[0], v[1]);
  } else {
    p[0] = __float2bfloat16_rn(v[0]);
  }
}

__device__ __forceinline__ void st16_bf16(__nv_bfloat16* p, const float* v) {
  uint4 a, b;
  a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]); a.z = pack_bf16x2(v[4], v[5]);
  a.w = pack_bf16x2(v[6], v[7]);
  b.x = pack_bf16x2(v[8], v[9]); b.y = pack_bf16x2(v[10], v[11]); b.z = pack_bf16x2(v[12], v[13]);
  b.w = pack_bf16x2(v[14], v[15]);
  ((uint4*)p)[0] = a;
  ((uint4*)p)[1] = b;
}

// ---------------------------------------------------------------------------------------------------------
// forward
// smem: [U rows: H/64 chunks x 96 rows x 128 B] [h: H/32 slices x 4 KB] [4 KB slack] [accumulator tile] [mbarriers]
struct FwdArgs {
  const float* gx;   // [T][B][3H] (includes b)
  const float* c;    // [3H]
  float* hs;         // [T+1][B][H], hs[0] = h0 on entry
  float* gates;      // [T][B][4][H]  (r, z, n, a)
  __nv_bfloat16* hsb;  // [T+1][B][H] bf16 copy of hs (operand of the recurrent weight gradient dU = dgh^T h)
  __nv_bfloat16* hx; // [2][B][H] exchange ring
  int T, B, H;
  int Bc;            // batch rows per cluster (cluster k owns rows [k Bc, (k + 1) Bc))
  long long* trace;  // optional per-step timestamps of the first cluster's CTAs (NSK_GRU_TRACE), 8 per step
};

__device__ __forceinline__ long long gclock() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// SW64 K-major shared-memory descriptor (sm_100 layout type 4): rows of 64 B (32 bf16), 8-row groups 512 B apart
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;    // SBO
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// one box of the h ring, multicast to every CTA of the cluster (same smem offset / mbarrier in each)
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// Batch groups: the rows of the batch are independent through the recurrence, so the grid is B / Bc clusters, each
// the full H / 32 CTAs (U resident in every cluster) over its own Bc rows.
// Per CTA (units [32q, 32q + 32)) and step:
//   * D^T = U_q h^T: the CTA's 96 gate rows of U (copied once into tensor memory, packed bf16 pairs: the MMA's A
//     operand, M = 128 lanes of which 96 are used) times h_t (bf16, the Bc batch rows as N, K-major in shared memory)
//     -- 32 tcgen05.mma (K = 16) issued 16 per elected thread (the issue loop, not the tensor pipe, bounded it);
//   * the accumulator (lane = gate row, column = batch row) goes through a shared-memory tile so all eight warps
//     share the gate math (fp32, state h kept in registers);
//   * each CTA writes its bf16 slice of h_{t+1} to a global ring and multicasts it (one TMA box) into every CTA's
//     h buffer, all slices completing one mbarrier per step. A split cluster barrier protects the buffer: the
//     arrive follows the MMAs' reads of h_t, the wait precedes the multicast (its latency hides behind the math).
template <int UPT>  // hidden units per thread in the gate math: Bc <= 8 UPT rows x 32 / UPT threads per row
__global__ void __launch_bounds__(kThreads, 1) gru_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmU,
                                                                 const __grid_constant__ CUtensorMap tmH,
                                                                 const FwdArgs p) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  const int H = p.H, B = p.B, T = p.T, H3 = 3 * H, Bc = p.Bc;
  const int NCH = H / 64;                  // 64-wide K chunks of U
  const int NS = H / kUC;                  // 32-wide h slices = CTAs of the cluster
  const int b0 = (int)(blockIdx.x / NS) * Bc;  // first batch row of this cluster
  uint8_t* us = smem;                      // NCH x 12 KB (SW128): staging of U on its way into tensor memory
  uint8_t* hsm = us + NCH * 12288;         // NS x 4 KB (SW64, B operand) + 4 KB slack
  float* dsm = (float*)(hsm + NS * 4096 + 4096);   // [64][kDP] accumulator tile for the gate math
  uint64_t* bars = (uint64_t*)(dsm + 64 * kDP);
  uint64_t* ufull = bars;
  uint64_t* hfull = bars + 1;              // every CTA's slice of h_t
  uint64_t* mdone = bars + 2;
  uint32_t* tmem_slot = (uint32_t*)(bars + 3);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int q = (int)cluster_rank();
  const int j0 = q * kUC;
  const uint16_t all = (uint16_t)((1u << NS) - 1u);
  const uint32_t hbytes = (uint32_t)(NS * Bc * 64);
  if (threadIdx.x == 0) {
    mbar_init(ufull, 1);
    mbar_init(hfull, 1);
    mbar_init(mdone, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmH);
    mbar_expect_tx(hfull, hbytes);  // phase 0
  }
  constexpr uint32_t kUCol = 256;  // U at columns [256, 256 + H/2), the accumulator at [0, NP)
  if (warp == 3) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // gate math: thread -> batch row gb = tid / TPR, units [UPT gq, UPT gq + UPT) of this CTA
  constexpr int TPR = kUC / UPT;  // threads per batch row
  const int hf = warp >> 2;
  const int gb = threadIdx.x / TPR, gq = threadIdx.x % TPR;
  const bool row_ok = gb < Bc;
  const size_t grow = (size_t)(b0 + gb);  // global batch row
  const int ju = j0 + gq * UPT;  // first global unit of this thread
  float h[UPT], cr[UPT], cz[UPT], cn[UPT], gr[UPT], gz[UPT], gn[UPT];
  if (row_ok) {
    ldv<UPT>(p.hs + grow * H + ju, h);
    ldv<UPT>(p.c + ju, cr);
    ldv<UPT>(p.c + H + ju, cz);
    ldv<UPT>(p.c + 2 * H + ju, cn);
    stvb<UPT>(p.hx + grow * H + ju, h);  // ring slot 0 = bf16(h0)
    stvb<UPT>(p.hsb + grow * H + ju, h);
    const float* g3 = p.gx + grow * H3 + ju;  // step 0's input projections
    ldv<UPT>(g3, gr);
    ldv<UPT>(g3 + H, gz);
    ldv<UPT>(g3 + 2 * H, gn);
  }
  if (warp == 2 && elect_one()) {  // U rows of this CTA: 3 gates x NCH chunks of {64 k, 32 rows}
    mbar_expect_tx(ufull, (uint32_t)(NCH * 12288));
    for (int c = 0; c < NCH; ++c)
      for (int g = 0; g < 3; ++g) tma_load_2d(&tmU, ufull, us + c * 12288 + g * 4096, c * 64, g * H + j0);
  }
  fence_proxy_async_global();
  tc_fence_before();
  cluster_sync_all();  // every CTA's mbarriers are initialised and its h0 slice is in the ring
  if (threadIdx.x == 0) tma_load_2d_mc(&tmH, hfull, hsm + q * 4096, j0, b0, all);
  if (warp < 4) {  // U rows (gate row m = lane, rows 96..127 zero) from the 128B-swizzled chunks into TMEM, once
    mbar_wait(ufull, 0);
    const int m = warp * 32 + lane;
    for (int c = 0; c < NCH; ++c) {  // 64 k = 32 packed columns per chunk
      uint32_t w[32];
#pragma unroll
      for (int g8 = 0; g8 < 8; ++g8) {
        const uint4 v = m < 3 * kUC ? *(const uint4*)(us + c * 12288 + m * 128 + ((g8 ^ (m & 7)) << 4))
                                    : make_uint4(0u, 0u, 0u, 0u);
        w[g8 * 4 + 0] = v.x;
        w[g8 * 4 + 1] = v.y;
        w[g8 * 4 + 2] = v.z;
        w[g8 * 4 + 3] = v.w;
      }
      tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + kUCol + c * 32, w);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const int NP = Bc <= 16 ? 16 : (Bc + 15) / 16 * 16;  // MMA N (batch rows, rows past Bc unused)
  const uint32_t idesc = make_idesc(1u, 0u, 0u, 128u, (uint32_t)NP);
  const uint64_t hd0 = sdesc_sw64(smem_u32(hsm));
  for (int t = 0; t < T; ++t) {
    long long* tr = p.trace && b0 == 0 ? p.trace + ((size_t)q * T + t) * 16 : nullptr;
    if (warp == 3) {
      // slice pair k: h slices 2k, 2k + 1 (4 KB apart), U k-steps 4k .. 4k+3 (8 packed columns each)
      mbar_wait(hfull, t & 1);
      if (tr && lane == 0) tr[1] = tr[2] = gclock();
      tc_fence_after();
      for (int k = 0; k < NS / 2; k += 4) {
        const uint64_t hd = hd0 + (uint64_t)(k * 512);
        const uint32_t ua = tmem + kUCol + (uint32_t)(k * 32);
        const int np = NS / 2 - k < 4 ? NS / 2 - k : 4;  // slice pairs in this issue
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i >= np) break;
            const uint64_t h2 = hd + (uint64_t)(i * 512);
            const uint32_t u2 = ua + (uint32_t)(i * 32);
            umma_ts<0>(tmem, u2, h2, idesc, k + i > 0 ? 1u : 0u);
            umma_ts<2>(tmem, u2 + 8, h2, idesc, 1u);
            umma_ts<256>(tmem, u2 + 16, h2, idesc, 1u);
            umma_ts<258>(tmem, u2 + 24, h2, idesc, 1u);
          }
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(mdone);
      __syncwarp();
    }
    // ---- epilogue: all warps ----
    mbar_wait_backoff(mdone, t & 1);
    if (tr && threadIdx.x == 0) tr[3] = gclock();
    tc_fence_after();
    if (threadIdx.x == 0 && t + 1 < T) mbar_expect_tx(hfull, hbytes);  // next phase (this one is complete)
    {  // D^T lane = gate row m (sub-partitions 0..2), column = batch row b -> dsm[b][m]
      const int sub = warp & 3;
      if (sub < 3) {
        const int nh = NP / 2;
        for (int cb = hf * nh; cb < hf * nh + nh; cb += 8) {
          float d[8];
          tmem_ld8(tmem + ((uint32_t)(sub * 32) << 16) + cb, d);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (cb + i < Bc) dsm[(cb + i) * kDP + sub * 32 + lane] = d[i];
        }
      }
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // done reading this step's h buffer
    named_sync(1, kThreads);
    if (tr && threadIdx.x == 0) tr[5] = gclock();
    float dr[UPT], dz[UPT], dn[UPT];
    if (row_ok) {
      const float* drow = dsm + gb * kDP + gq * UPT;
      ldvs<UPT>(drow, dr);
      ldvs<UPT>(drow + 32, dz);
      ldvs<UPT>(drow + 64, dn);
#pragma unroll
      for (int u = 0; u < UPT; ++u) {
        dr[u] = sigm(gr[u] + dr[u] + cr[u]);            // r
        dz[u] = sigm(gz[u] + dz[u] + cz[u]);            // z
        dn[u] = dn[u] + cn[u];                          // a
        gn[u] = tanh_fast(gn[u] + dr[u] * dn[u]);       // n
        h[u] = gn[u] - dz[u] * gn[u] + dz[u] * h[u];
      }
      if (tr && threadIdx.x == 0) tr[6] = gclock();
      if (t + 1 < T) stvb<UPT>(p.hx + ((size_t)((t + 1) & 1) * B + grow) * H + ju, h);
    }
    fence_proxy_async_global();  // this slice of h_{t+1} is read by this CTA's multicast (async proxy)
    named_sync(1, kThreads);
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every CTA is done with h_t: buffers are free
    if (tr && threadIdx.x == 0) tr[7] = gclock();
    if (threadIdx.x == 0 && t + 1 < T)
      tma_load_2d_mc(&tmH, hfull, hsm + q * 4096, j0, ((t + 1) & 1) * B + b0, all);
    if (row_ok) {  // needed only by backward: off the critical path
      stv<UPT>(p.hs + ((size_t)(t + 1) * B + grow) * H + ju, h);
      stvb<UPT>(p.hsb + ((size_t)(t + 1) * B + grow) * H + ju, h);
      float* gs = p.gates + ((size_t)t * B + grow) * 4 * H + ju;
      stv<UPT>(gs, dr);
      stv<UPT>(gs + H, dz);
      stv<UPT>(gs + 2 * H, gn);
      stv<UPT>(gs + 3 * H, dn);
      if (t + 1 < T) {  // next step's input projections
        const float* g3 = p.gx + ((size_t)(t + 1) * B + grow) * H3 + ju;
        ldv<UPT>(g3, gr);
        ldv<UPT>(g3 + H, gz);
        ldv<UPT>(g3 + 2 * H, gn);
      }
    }
    if (tr && threadIdx.x == 0) tr[4] = gclock();
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while a peer's multicast may still target it
  if (warp == 3) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------------------------------
// backward
struct BwdArgs {
  const float* dhs;    // [T][B][H] external gradient of each h_{t+1}
  const float* hs;     // [T+1][B][H]
  const float* gates;  // [T][B][4][H]
  __nv_bfloat16* dgx;  // [T][B][3H] bf16: operand of dW = dgx^T x and dx = dgx W
  __nv_bfloat16* dgh;  // [T][B][3H] bf16: operand of dU = dgh^T h
  float* dh0;          // [B][H]
  float* db;           // [3H]  sum over (t, b) of dgx (fp32, fixed order), accumulated with beta_b
  float* dc;           // [3H]  sum over (t, b) of dgh, accumulated with beta_c
  float beta_b, beta_c;
  __nv_bfloat16* gex;  // [2][RG][B][KR] dgh exchange ring (bf16)
  float* pex;          // [2][CL][RG][B][32] partial-product ring
  float* bpart;        // [clusters][4][H] per-cluster bias-gradient sums (nullptr: one cluster writes db / dc)
  int T, B, H, RG, CG;
  int Bc;              // batch rows per cluster (see the forward)
  long long* trace;    // optional per-step timestamps of the first cluster's CTAs (NSK_GRU_TRACE=2)
};

template <int UPT>
__global__ void __launch_bounds__(kThreads, 1) gru_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmU,
                                                                 const __grid_constant__ CUtensorMap tmG,
                                                                 const BwdArgs p) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  const int H = p.H, B = p.B, T = p.T, H3 = 3 * H, RG = p.RG, CG = p.CG, Bc = p.Bc;
  const int CL = RG * CG;
  const int cid = (int)(blockIdx.x / CL), b0 = cid * Bc;  // batch group of this cluster
  const int NC = H / CG;            // column-group width (MMA N)
  const int KR = 3 * kUC * CG;      // gate rows of a row group (MMA K)
  const int NB = NC / 64;           // 64-column MN blocks of the U block
  const int NKC = KR / 64;          // 64-row K chunks of the dgh block
  uint8_t* ub = smem;                              // NB x (KR x 128 B)
  uint8_t* gsm = ub + NB * KR * 128;               // NKC x 8 KB (+8 KB slack)
  uint64_t* bars = (uint64_t*)(gsm + NKC * 8192 + 8192);
  uint64_t* ufull = bars;
  uint64_t* gfull = bars + 1;                      // 1: the step's dgh block (four issuers arrive)
  uint64_t* mdone = gfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(mdone + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int q = (int)cluster_rank();
  const int gi = q / CG, gj = q % CG;              // row group, column group
  const int j0 = gj * NC + gi * kUC;               // first owned unit
  if (threadIdx.x == 0) {
    mbar_init(ufull, 1);
    mbar_init(gfull, 4);
    mbar_init(mdone, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmG);
  }
  if (warp == 3) {
    tmem_alloc(tmem_slot, NC <= 32 ? 32 : (NC <= 64 ? 64 : (NC <= 128 ? 128 : 256)));
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 2 && elect_one()) {
    // U block: for each owner column j' of row group gi and gate g, the 32 rows g*H + (j' NC + 32 gi) .. +32,
    // as MN-major K rows (128 B = 64 columns per block)
    mbar_expect_tx(ufull, (uint32_t)(NB * KR * 128));
    for (int nb = 0; nb < NB; ++nb)
      for (int jj = 0; jj < CG; ++jj)
        for (int g = 0; g < 3; ++g)
          tma_load_2d(&tmU, ufull, ub + nb * KR * 128 + (jj * 3 + g) * kUC * 128, gj * NC + nb * 64,
                      g * H + jj * NC + gi * kUC);
  }
  // phase A runs on all eight warps: thread -> batch row gb = tid / TPR, units [UPT gq, UPT gq + UPT) of this
  // CTA; phase B's TMEM readers are warps 0,1,4,5 (accumulator rows = batch rows live in sub-partitions 0 and 1)
  constexpr int TPR = kUC / UPT;
  const bool epi = (warp & 2) == 0;
  const int sp = warp & 1, hf = warp >> 2;
  const int b = sp * 32 + lane;
  const int gb = threadIdx.x / TPR, gq = threadIdx.x % TPR;
  const bool arow = gb < Bc;
  const size_t grow = (size_t)(b0 + gb);  // global batch row (phase A)
  const int ju = j0 + gq * UPT;  // first global unit of this thread (phase A)
  const int uo = gq * UPT;       // its offset inside the CTA's 32 units
  float dhz[UPT];                // dh_{t+1} * z_{t+1} carried to the next (earlier) step
  float cs[4][UPT];              // running column sums of dr', dz', dn', dn'*r (bias gradients db, dc)
#pragma unroll
  for (int u = 0; u < UPT; ++u) {
    dhz[u] = 0.f;
    cs[0][u] = cs[1][u] = cs[2][u] = cs[3][u] = 0.f;
  }
  const uint32_t idesc = make_idesc(1u, 0u, 1u, 128u, (uint32_t)NC);
  const int NP = Bc <= 16 ? 16 : (Bc + 15) / 16 * 16;  // swapped: MMA N (batch rows, rows past Bc unused)
  const bool swap = NC == 128;  // P^T = U^T dgh^T: M = the column group's 128 columns, N = the batch rows
  const uint32_t idesc_s = make_idesc(1u, 1u, 0u, 128u, (uint32_t)NP);
  // step t's external gradient, saved gates and h_t do not depend on the recurrence: they are loaded during step
  // t + 1's exchange and MMA phase, so only the partial products stay on the per-step critical path
  float pdh[UPT], pr[UPT], pz[UPT], pn[UPT], pa[UPT], php[UPT];
  auto prefetch = [&](int tt) {
    if (!arow || tt < 0) return;
    ldv<UPT>(p.dhs + ((size_t)tt * B + grow) * H + ju, pdh);
    const float* gs = p.gates + ((size_t)tt * B + grow) * 4 * H + ju;
    ldv<UPT>(gs, pr);
    ldv<UPT>(gs + H, pz);
    ldv<UPT>(gs + 2 * H, pn);
    ldv<UPT>(gs + 3 * H, pa);
    ldv<UPT>(p.hs + ((size_t)tt * B + grow) * H + ju, php);
  };
  prefetch(T - 1);
  for (int t = T - 1; t >= 0; --t) {
    long long* tr = p.trace && b0 == 0 ? p.trace + ((size_t)q * T + (T - 1 - t)) * 16 : nullptr;
    // ---- A: dh_t for own units, gate derivatives, dgh block ----
    if (t < T - 1) {
      cluster_wait();  // partial products of step t+1 visible
      tc_fence_after();
    }
    if (tr && threadIdx.x == 0) tr[0] = gclock();
    float drp[UPT], dzp[UPT], dnp[UPT], dnr[UPT];
    if (arow) {
      float dh[UPT], v[UPT];
#pragma unroll
      for (int u = 0; u < UPT; ++u) dh[u] = pdh[u] + dhz[u];
      if (t < T - 1) {
        const float* pp = p.pex + ((size_t)(((t + 1) & 1) * CL + q) * RG) * B * kUC + grow * kUC + uo;
        for (int s = 0; s < RG; ++s) {  // fixed order over the row groups
          ldv<UPT>(pp + (size_t)s * B * kUC, v);
#pragma unroll
          for (int u = 0; u < UPT; ++u) dh[u] += v[u];
        }
      }
      float r[UPT], z[UPT], n[UPT], a[UPT], hp[UPT];
#pragma unroll
      for (int u = 0; u < UPT; ++u) {
        r[u] = pr[u];
        z[u] = pz[u];
        n[u] = pn[u];
        a[u] = pa[u];
        hp[u] = php[u];
      }
#pragma unroll
      for (int u = 0; u < UPT; ++u) {
        const float dn = dh[u] * (1.f - z[u]);
        const float dz = dh[u] * (hp[u] - n[u]);
        dnp[u] = dn * (1.f - n[u] * n[u]);
        drp[u] = dnp[u] * a[u] * r[u] * (1.f - r[u]);
        dzp[u] = dz * z[u] * (1.f - z[u]);
        dnr[u] = dnp[u] * r[u];
        dhz[u] = dh[u] * z[u];
        cs[0][u] += drp[u];
        cs[1][u] += dzp[u];
        cs[2][u] += dnp[u];
        cs[3][u] += dnr[u];
      }
      __nv_bfloat16* ge = p.gex + ((size_t)((t & 1) * RG + gi) * B + grow) * KR + gj * 3 * kUC + uo;
      stvb<UPT>(ge, drp);
      stvb<UPT>(ge + kUC, dzp);
      stvb<UPT>(ge + 2 * kUC, dnr);
    }
    fence_proxy_async_global();
    tc_fence_before();
    if (tr && threadIdx.x == 0) tr[1] = gclock();
    cluster_arrive();  // publish this step's dgh block; the fp32 copies below are only read after the kernel
    prefetch(t - 1);
    if (arow) {
      __nv_bfloat16* gxo = p.dgx + ((size_t)t * B + grow) * H3 + ju;
      __nv_bfloat16* gho = p.dgh + ((size_t)t * B + grow) * H3 + ju;
      stvb<UPT>(gxo, drp);
      stvb<UPT>(gxo + H, dzp);
      stvb<UPT>(gxo + 2 * H, dnp);
      stvb<UPT>(gho, drp);
      stvb<UPT>(gho + H, dzp);
      stvb<UPT>(gho + 2 * H, dnr);
      if (t == 0) {
        // dh0 = dh_0 * z_0 + (dgh_0 U)[own units], the partials of step 0 are added after the last barrier
        stv<UPT>(p.dh0 + grow * H + ju, dhz);
      }
    }
    cluster_wait();  // every dgh block of step t is in the ring
    tc_fence_after();
    if (tr && threadIdx.x == 0) tr[2] = gclock();
    // ---- B: P = dgh(row group) . U(row group rows, column group cols), slices to the column group ----
    fence_proxy_async_global();
    if ((warp & 2) && lane == 0) {  // four issuing threads (warps 2, 3, 6, 7), one barrier for the whole block
      const int w4 = (warp & 1) | ((warp >> 1) & 2);
      mbar_expect_tx(gfull, (uint32_t)(((NKC - w4 + 3) / 4) * Bc * 128));
      for (int c = w4; c < NKC; c += 4)
        tma_load_2d(&tmG, gfull, gsm + c * 8192, c * 64, ((t & 1) * RG + gi) * B + b0);
    }
    __syncwarp();
    if (warp == 3) {
      if (t == T - 1) mbar_wait(ufull, 0);
      const uint64_t gd0 = sdesc_sw128(smem_u32(gsm), 16, 1024);
      const uint64_t ud0 = sdesc_sw128(smem_u32(ub), (uint32_t)(KR * 128), 1024);
      mbar_wait(gfull, (T - 1 - t) & 1);
      if (tr && lane == 0) tr[3] = gclock();
      tc_fence_after();
      for (int c = 0; c < NKC; ++c) {  // chunk c: dgh + 8 KB, U + 64 K rows
        const uint64_t gd = gd0 + (uint64_t)(c * 512), ud = ud0 + (uint64_t)(c * 512);
        if (elect_one()) {
          if (swap) {  // U block (MN-major) as A: the MMA reads Bc rows of dgh, not 128
            umma_off<0, 0, false>(tmem, ud, gd, idesc_s, c > 0 ? 1u : 0u);
            umma_off<128, 2, false>(tmem, ud, gd, idesc_s, 1u);
            umma_off<256, 4, false>(tmem, ud, gd, idesc_s, 1u);
            umma_off<384, 6, false>(tmem, ud, gd, idesc_s, 1u);
          } else {
            umma_off<0, 0, false>(tmem, gd, ud, idesc, c > 0 ? 1u : 0u);
            umma_off<2, 128, false>(tmem, gd, ud, idesc, 1u);
            umma_off<4, 256, false>(tmem, gd, ud, idesc, 1u);
            umma_off<6, 384, false>(tmem, gd, ud, idesc, 1u);
          }
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(mdone);
      __syncwarp();
    }
    if (swap) {  // P^T lane = column n = 32 s + u (sub-partition s = the slice of row group s), column = batch row
      mbar_wait_backoff(mdone, (T - 1 - t) & 1);
      tc_fence_after();
      if (tr && threadIdx.x == 0) tr[4] = gclock();
      const int s = warp & 3, nh = NP / 2;
      float* po = p.pex + ((size_t)((t & 1) * CL + s * CG + gj) * RG + gi) * B * kUC + (size_t)b0 * kUC + lane;
      for (int cb = hf * nh; cb < hf * nh + nh; cb += 8) {
        float d[8];
        tmem_ld8(tmem + ((uint32_t)(s * 32) << 16) + cb, d);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (cb + i < Bc) po[(size_t)(cb + i) * kUC] = d[i];
      }
    } else if (epi) {
      mbar_wait_backoff(mdone, (T - 1 - t) & 1);
      tc_fence_after();
      // thread (b, hf) holds columns [hf NC/2, (hf+1) NC/2) = the slices of row groups s in [hf RG/2, (hf+1) RG/2)
      const uint32_t ta = tmem + ((uint32_t)(sp * 32) << 16);
      for (int s = hf * (RG / 2); s < (hf + 1) * (RG / 2); ++s) {
        float v0[16], v1[16];
        tmem_ld16(ta + s * kUC, v0);
        tmem_ld16(ta + s * kUC + 16, v1);
        tmem_ld_wait();
        if (b < Bc) {
          const int dest = s * CG + gj;
          float* po = p.pex + ((size_t)((t & 1) * CL + dest) * RG + gi) * B * kUC + (size_t)(b0 + b) * kUC;
          st16(po, v0);
          st16(po + 16, v1);
        }
      }
    }
    tc_fence_before();
    if (tr && threadIdx.x == 0) tr[5] = gclock();
    cluster_arrive();  // partials of step t published (read in A of step t-1)
  }
  cluster_wait();
  tc_fence_after();
  // dh0 += the step-0 partial products of this CTA's units
  if (arow) {
    float dh[UPT], v[UPT];
    ldv<UPT>(p.dh0 + grow * H + ju, dh);
    const float* pp = p.pex + ((size_t)q * RG) * B * kUC + grow * kUC + uo;  // slot (0 & 1) = 0
    for (int s = 0; s < RG; ++s) {
      ldv<UPT>(pp + (size_t)s * B * kUC, v);
#pragma unroll
      for (int u = 0; u < UPT; ++u) dh[u] += v[u];
    }
    stv<UPT>(p.dh0 + grow * H + ju, dh);
  }
  // bias gradients: the running column sums of the cluster's batch rows, added in row order (deterministic);
  // the dgh block ring in shared memory is free now. Several clusters: per-cluster sums, folded in cluster
  // order by gru_bias_fold_kernel
  float* red = (float*)gsm;  // [Bc rows][4 sums][32 units]
  if (arow) {
#pragma unroll
    for (int k = 0; k < 4; ++k) stv<UPT>(red + ((size_t)gb * 4 + k) * kUC + uo, cs[k]);
  }
  __syncthreads();
  if (threadIdx.x < 4 * kUC) {
    const int k = threadIdx.x / kUC, u = threadIdx.x % kUC;
    float acc = 0.f;
    for (int r = 0; r < Bc; ++r) acc += red[((size_t)r * 4 + k) * kUC + u];
    const int j = j0 + u;
    if (p.bpart) {
      p.bpart[((size_t)cid * 4 + k) * H + j] = acc;
    } else if (k < 2) {  // r and z parts: dgx and dgh agree
      float* o1 = p.db + k * H + j;
      float* o2 = p.dc + k * H + j;
      *o1 = acc + p.beta_b * *o1;
      *o2 = acc + p.beta_c * *o2;
    } else if (k == 2) {
      float* o = p.db + 2 * H + j;
      *o = acc + p.beta_b * *o;
    } else {
      float* o = p.dc + 2 * H + j;
      *o = acc + p.beta_c * *o;
    }
  }
  if (warp == 3) {
    tc_fence_after();
    tmem_dealloc(tmem, NC <= 32 ? 32 : (NC <= 64 ? 64 : (NC <= 128 ? 128 : 256)));
  }
}

// Backward with DSMEM pushes (batch groups of Bc <= 32 rows, 128-column column groups): no global rings and no
// cluster barriers inside the sweep. Per step
//   A) wait for the RG partial-product blocks of step t+1 (pushed into this CTA's shared memory), form dh_t and the
//      gate derivatives, stage this CTA's dgh piece (its 3 x 32 gate rows) directly in the MMA operand layout
//      (K-major, 64-byte swizzle, one 32-wide K chunk per gate) and push it with one bulk copy into the dgh
//      buffer of every CTA of its row group;
//   B) once the row group's CG pieces have landed, 6 CG tcgen05.mma (U block as the MN-major A operand, M = the 128
//      columns of the column group, N = the batch rows) and push each 32-column slice of P^T to its owner.
// Every buffer is double-buffered by step parity. A buffer of step t is rewritten at step t-2 only after its
// reader has consumed it: the producer of step t-2's data transitively needs, through the alternating
// row-group / column-group dependencies, data that every reader produced after consuming step t -- so no barrier
// guards the rewrite, and every re-arm of a receive barrier precedes the pushes it counts.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void bulk_s2c(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct PushLayout {  // byte sizes of the push kernel's shared-memory regions
  int NB, KR, NK32, NP, CP, GSZ, PSZ;
  __host__ __device__ PushLayout(int H, int CG, int Bc) {
    NB = H / CG / 64;
    KR = 3 * kUC * CG;
    NK32 = KR / 32;
    NP = Bc <= 16 ? 16 : 32;
    CP = NP * 64;
    GSZ = NK32 * CP;
    PSZ = (H / CG / kUC) * Bc * 128;
  }
  __host__ __device__ size_t bytes() const {
    return (size_t)NB * KR * 128 + 2 * (size_t)GSZ + 6 * (size_t)CP + 4 * (size_t)PSZ + 64;
  }
};

template <int UPT>
__global__ void __launch_bounds__(kThreads, 1) gru_bwd_push_kernel(const __grid_constant__ CUtensorMap tmU,
                                                                   const BwdArgs p) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  const int H = p.H, B = p.B, T = p.T, H3 = 3 * H, RG = p.RG, CG = p.CG, Bc = p.Bc;
  const int CL = RG * CG;
  const int cid = (int)(blockIdx.x / CL), b0 = cid * Bc;
  const int NC = H / CG;  // 128 = RG slices of 32
  const PushLayout L(H, CG, Bc);
  uint8_t* ub = smem;                         // NB x (KR x 128 B): U block, MN-major
  uint8_t* gsm = ub + L.NB * L.KR * 128;      // [2][GSZ]: the row group's dgh, NK32 chunks of NP rows x 64 B
  uint8_t* gst = gsm + 2 * L.GSZ;             // [2][3 CP]: this CTA's dgh piece, staged in operand layout
  uint8_t* prx = gst + 6 * L.CP;              // [2][PSZ]: received partial products, RG blocks of [Bc][32] fp32
  uint8_t* pst = prx + 2 * L.PSZ;             // [2][PSZ]: outgoing P^T slices, [RG][Bc][32] fp32
  uint64_t* bars = (uint64_t*)(pst + 2 * L.PSZ);
  uint64_t* ufull = bars;
  uint64_t* gfull = bars + 1;  // [2]
  uint64_t* pfull = bars + 3;  // [2]
  uint64_t* mdone = bars + 5;
  uint32_t* tmem_slot = (uint32_t*)(bars + 6);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int q = (int)cluster_rank();
  const int gi = q / CG, gj = q % CG;
  const int j0 = gj * NC + gi * kUC;
  const uint32_t gbytes = (uint32_t)(CG * 3 * L.CP), pbytes = (uint32_t)L.PSZ;
  if (threadIdx.x == 0) {
    mbar_init(ufull, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&gfull[i], 1);
      mbar_init(&pfull[i], 1);
    }
    mbar_init(mdone, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmU);
    for (int i = 0; i < 2; ++i) {  // the first use of each buffer
      mbar_expect_tx(&gfull[i], gbytes);
      mbar_expect_tx(&pfull[i], pbytes);
    }
  }
  constexpr uint32_t kUCol = 64;  // U^T at columns [64, 64 + KR/2), the accumulator at [0, NP)
  if (warp == 3) {
    tmem_alloc(tmem_slot, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 2 && elect_one()) {
    mbar_expect_tx(ufull, (uint32_t)(L.NB * L.KR * 128));
    for (int nb = 0; nb < L.NB; ++nb)
      for (int jj = 0; jj < CG; ++jj)
        for (int g = 0; g < 3; ++g)
          tma_load_2d(&tmU, ufull, ub + nb * L.KR * 128 + (jj * 3 + g) * kUC * 128, gj * NC + nb * 64,
                      g * H + jj * NC + gi * kUC);
  }
  cluster_sync_all();  // every CTA's receive barriers are initialised and armed before the first push
  {  // A[n][k] = U block[k][n] into tensor memory: lane n gathers its column (2 bytes per 128B-swizzled row), packs
     // k pairs; the per-step MMAs then read only the dgh block from shared memory
    if (warp < 4) {
      mbar_wait(ufull, 0);
      const int n = warp * 32 + lane;
      const uint8_t* col = ub + (n >> 6) * L.KR * 128 + ((n & 7) << 1);
      const int g0 = (n & 63) >> 3;
      for (int c = 0; c < L.KR / 64; ++c) {  // 64 k = 32 packed columns
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int k = c * 64 + 2 * i;  // k and k+1 share k / 8 (k even)
          const uint32_t lo = *(const uint16_t*)(col + k * 128 + ((g0 ^ (k & 7)) << 4));
          const uint32_t hi = *(const uint16_t*)(col + (k + 1) * 128 + ((g0 ^ ((k + 1) & 7)) << 4));
          w[i] = lo | (hi << 16);
        }
        tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + kUCol + c * 32, w);
      }
      tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  constexpr int TPR = kUC / UPT;
  const int hf = warp >> 2;
  const int gb = threadIdx.x / TPR, gq = threadIdx.x % TPR;
  const bool arow = gb < Bc;
  const size_t grow = (size_t)(b0 + gb);
  const int ju = j0 + gq * UPT;
  const int uo = gq * UPT;
  // this thread's dgh values in the SW64 K-major chunk: row gb (64 B), 16-byte granule uo / 8 XOR (gb / 2) % 4
  const uint32_t soff = (uint32_t)(gb * 64 + ((((uo >> 3) ^ ((gb >> 1) & 3))) << 4) + (uo & 7) * 2);
  float dhz[UPT], cs[4][UPT];
#pragma unroll
  for (int u = 0; u < UPT; ++u) {
    dhz[u] = 0.f;
    cs[0][u] = cs[1][u] = cs[2][u] = cs[3][u] = 0.f;
  }
  const uint32_t idesc_t = make_idesc(1u, 0u, 0u, 128u, (uint32_t)L.NP);  // A from tensor memory (K-major)
  float pdh[UPT], pr[UPT], pz[UPT], pn[UPT], pa[UPT], php[UPT];
  auto prefetch = [&](int tt) {
    if (!arow || tt < 0) return;
    ldv<UPT>(p.dhs + ((size_t)tt * B + grow) * H + ju, pdh);
    const float* gs = p.gates + ((size_t)tt * B + grow) * 4 * H + ju;
    ldv<UPT>(gs, pr);
    ldv<UPT>(gs + H, pz);
    ldv<UPT>(gs + 2 * H, pn);
    ldv<UPT>(gs + 3 * H, pa);
    ldv<UPT>(p.hs + ((size_t)tt * B + grow) * H + ju, php);
  };
  prefetch(T - 1);
  for (int t = T - 1; t >= 0; --t) {
    const int par = t & 1;
    long long* tr = p.trace && b0 == 0 ? p.trace + ((size_t)q * T + (T - 1 - t)) * 16 : nullptr;
    // ---- A ----
    float dh[UPT];
#pragma unroll
    for (int u = 0; u < UPT; ++u) dh[u] = pdh[u] + dhz[u];
    if (t < T - 1) {
      const int pp = (t + 1) & 1;
      mbar_wait(&pfull[pp], (uint32_t)(((T - 2 - t) >> 1) & 1));
      if (threadIdx.x == 0 && t >= 1) mbar_expect_tx(&pfull[pp], pbytes);  // next: the partials of step t-1
      if (arow) {
        const float* src = (const float*)(prx + pp * L.PSZ) + (size_t)gb * kUC + uo;
        for (int s = 0; s < RG; ++s) {  // fixed order over the row groups
          float v[UPT];
          ldvs<UPT>(src + (size_t)s * Bc * kUC, v);
#pragma unroll
          for (int u = 0; u < UPT; ++u) dh[u] += v[u];
        }
      }
    }
    if (tr && threadIdx.x == 0) tr[0] = gclock();
    float drp[UPT], dzp[UPT], dnp[UPT], dnr[UPT];
    uint8_t* stg = gst + par * 3 * L.CP;
    if (arow) {
#pragma unroll
      for (int u = 0; u < UPT; ++u) {
        const float dn = dh[u] * (1.f - pz[u]);
        const float dz = dh[u] * (php[u] - pn[u]);
        dnp[u] = dn * (1.f - pn[u] * pn[u]);
        drp[u] = dnp[u] * pa[u] * pr[u] * (1.f - pr[u]);
        dzp[u] = dz * pz[u] * (1.f - pz[u]);
        dnr[u] = dnp[u] * pr[u];
        dhz[u] = dh[u] * pz[u];
        cs[0][u] += drp[u];
        cs[1][u] += dzp[u];
        cs[2][u] += dnp[u];
        cs[3][u] += dnr[u];
      }
      stvb<UPT>((__nv_bfloat16*)(stg + soff), drp);
      stvb<UPT>((__nv_bfloat16*)(stg + L.CP + soff), dzp);
      stvb<UPT>((__nv_bfloat16*)(stg + 2 * L.CP + soff), dnr);
    }
    fence_proxy_async_smem();
    named_sync(1, kThreads);
    if (threadIdx.x == 0) {  // the piece (3 chunks, rows past Bc unused) into every CTA of the row group
      if (tr) tr[1] = gclock();
      const uint32_t dst = smem_u32(gsm + par * L.GSZ + gj * 3 * L.CP), bar = smem_u32(&gfull[par]);
      for (int j = 0; j < CG; ++j) {
        const uint32_t r = (uint32_t)(gi * CG + j);
        bulk_s2c(mapa_u32(dst, r), smem_u32(stg), (uint32_t)(3 * L.CP), mapa_u32(bar, r));
      }
    }
    prefetch(t - 1);
    if (arow) {  // bf16 operands of the weight-gradient GEMMs and dh0: off the critical path
      __nv_bfloat16* gxo = p.dgx + ((size_t)t * B + grow) * H3 + ju;
      __nv_bfloat16* gho = p.dgh + ((size_t)t * B + grow) * H3 + ju;
      stvb<UPT>(gxo, drp);
      stvb<UPT>(gxo + H, dzp);
      stvb<UPT>(gxo + 2 * H, dnp);
      stvb<UPT>(gho, drp);
      stvb<UPT>(gho + H, dzp);
      stvb<UPT>(gho + 2 * H, dnr);
      if (t == 0) stv<UPT>(p.dh0 + grow * H + ju, dhz);
    }
    // ---- B ----
    if (warp == 3) {
      if (t == T - 1) mbar_wait(ufull, 0);
      if (tr && lane == 0) tr[2] = gclock();
      mbar_wait(&gfull[par], (uint32_t)(((T - 1 - t) >> 1) & 1));
      if (t >= 2 && elect_one()) mbar_expect_tx(&gfull[par], gbytes);  // next: the dgh of step t-2
      __syncwarp();
      if (tr && lane == 0) tr[3] = gclock();
      tc_fence_after();
      const uint64_t gd0 = sdesc_sw64(smem_u32(gsm + par * L.GSZ));
      const int cpd = L.CP >> 4;
      for (int c = 0; c < L.NK32; c += 8) {  // eight chunks (16 MMAs) per elected issue
        const uint32_t ua = tmem + kUCol + (uint32_t)(c * 16);  // chunk c = 16 packed columns of U^T
        const int nc = L.NK32 - c < 8 ? L.NK32 - c : 8;         // NK32 = 3 CG
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i >= nc) break;
            const uint64_t gd = gd0 + (uint64_t)((c + i) * cpd);
            umma_ts<0>(tmem, ua + 16 * i, gd, idesc_t, c + i > 0 ? 1u : 0u);
            umma_ts<2>(tmem, ua + 16 * i + 8, gd, idesc_t, 1u);
          }
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(mdone);
      __syncwarp();
    }
    mbar_wait_backoff(mdone, (uint32_t)((T - 1 - t) & 1));
    tc_fence_after();
    if (tr && threadIdx.x == 0) tr[4] = gclock();
    {  // P^T lane 32 s + u = unit u of slice s (owner: row group s of this column group), column = batch row
      const int s = warp & 3, nh = L.NP / 2;
      float* ps = (float*)(pst + par * L.PSZ) + (size_t)s * Bc * kUC;
      const int r0 = hf * nh, r1 = r0 + nh < Bc ? r0 + nh : Bc;
      for (int cb = r0; cb < r0 + nh; cb += 8) {
        float d[8];
        tmem_ld8(tmem + ((uint32_t)(s * 32) << 16) + cb, d);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (cb + i < Bc) ps[(size_t)(cb + i) * kUC + lane] = d[i];
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && r1 > r0) {
        const uint32_t r = (uint32_t)(s * CG + gj);
        const uint32_t dst = smem_u32(prx + par * L.PSZ) + (uint32_t)((gi * Bc + r0) * 128);
        bulk_s2c(mapa_u32(dst, r), smem_u32(ps + (size_t)r0 * kUC), (uint32_t)((r1 - r0) * 128),
                 mapa_u32(smem_u32(&pfull[par]), r));
      }
    }
    if (tr && threadIdx.x == 0) tr[5] = gclock();
  }
  // dh0 += the step-0 partial products of this CTA's units
  mbar_wait(&pfull[0], (uint32_t)(((T - 1) >> 1) & 1));
  if (arow) {
    float dh[UPT], v[UPT];
    ldv<UPT>(p.dh0 + grow * H + ju, dh);
    const float* src = (const float*)prx + (size_t)gb * kUC + uo;
    for (int s = 0; s < RG; ++s) {
      ldvs<UPT>(src + (size_t)s * Bc * kUC, v);
#pragma unroll
      for (int u = 0; u < UPT; ++u) dh[u] += v[u];
    }
    stv<UPT>(p.dh0 + grow * H + ju, dh);
  }
  // bias gradients as in gru_bwd_tc_kernel (the dgh buffers are free: every push into them was consumed)
  float* red = (float*)gsm;  // [Bc rows][4 sums][32 units]
  if (arow) {
#pragma unroll
    for (int k = 0; k < 4; ++k) stv<UPT>(red + ((size_t)gb * 4 + k) * kUC + uo, cs[k]);
  }
  __syncthreads();
  if (threadIdx.x < 4 * kUC) {
    const int k = threadIdx.x / kUC, u = threadIdx.x % kUC;
    float acc = 0.f;
    for (int r = 0; r < Bc; ++r) acc += red[((size_t)r * 4 + k) * kUC + u];
    const int j = j0 + u;
    if (p.bpart) {
      p.bpart[((size_t)cid * 4 + k) * H + j] = acc;
    } else if (k < 2) {
      p.db[k * H + j] = acc + p.beta_b * p.db[k * H + j];
      p.dc[k * H + j] = acc + p.beta_c * p.dc[k * H + j];
    } else if (k == 2) {
      p.db[2 * H + j] = acc + p.beta_b * p.db[2 * H + j];
    } else {
      p.dc[2 * H + j] = acc + p.beta_c * p.dc[2 * H + j];
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while a push may still read its shared memory
  if (warp == 3) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// backward arrangement: CG column groups x RG row groups of CL = H / 32 CTAs with NC = H / CG and KR = 96 CG
// multiples of 64 (NSK_GRU_CG overrides the choice)
int bwd_groups(int H, int* rg, int* cg) {
  const int CL = H / kUC;
  const char* e = getenv("NSK_GRU_CG");
  const int want = e ? atoi(e) : 0;
  int best = 0;
  for (int c = 1; c <= CL; ++c) {
    if (CL % c || (H / c) % 64 || (3 * kUC * c) % 64 || H / c > 256 || (CL / c) % 2) continue;
    if (want ? c == want : (best == 0 || (c <= 4 && c > best))) best = c;
  }
  if (!best) return 0;
  *cg = best;
  *rg = CL / best;
  return 1;
}

// bias gradients of several batch groups: the per-cluster sums added in cluster order (deterministic)
__global__ void gru_bias_fold_kernel(const float* __restrict__ part, int groups, int H, float* db, float beta_b,
                                     float* dc, float beta_c) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * H) return;
  const int k = i / H, j = i - k * H;
  float acc = 0.f;
  for (int c = 0; c < groups; ++c) acc += part[((size_t)c * 4 + k) * H + j];
  if (k < 2) {  // r and z parts: dgx and dgh agree
    db[k * H + j] = acc + beta_b * db[k * H + j];
    dc[k * H + j] = acc + beta_c * dc[k * H + j];
  } else if (k == 2) {
    db[2 * H + j] = acc + beta_b * db[2 * H + j];
  } else {
    dc[2 * H + j] = acc + beta_c * dc[2 * H + j];
  }
}

constexpr int kMaxGroups = 8;

size_t fwd_smem(int H) { return 1024 + (size_t)(H / 64) * 12288 + (size_t)(H / kUC) * 4096 + 4096 + 64 * kDP * 4 + 256; }
size_t bwd_smem(int H, int rg, int cg) {
  const int NB = H / cg / 64, KR = 3 * kUC * cg;
  return 1024 + (size_t)NB * KR * 128 + (size_t)(KR / 64) * 8192 + 8192 + 256;
}

int set_cluster_attrs(const void* fn, int cl, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && cl > 8) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return nsk::cuda_status(e, "gru_tc: cudaFuncSetAttribute");
  return NSK_OK;
}

// Batch groups (independent clusters over B / groups rows each): the largest power of two <= NSK_GRU_GROUPS
// (default 4) dividing B whose clusters can all be resident at once
int batch_groups(const void* fn, int cl, size_t smem, int B) {
  const char* e = getenv("NSK_GRU_GROUPS");
  int want = e ? atoi(e) : 4;
  if (want > kMaxGroups) want = kMaxGroups;
  if (want < 2 || set_cluster_attrs(fn, cl, smem)) return 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl * want);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  for (int g = want; g > 1; g >>= 1)
    if (B % g == 0 && g <= n) return g;
  return 1;
}

int launch_cluster(const void* fn, int cl, int groups, size_t smem, void** args, cudaStream_t st) {
  int rc = set_cluster_attrs(fn, cl, smem);
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl * groups);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return nsk::cuda_status(e, "gru_tc: cluster launch");
  return NSK_OK;
}

int tmap_2d_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  const uint64_t dims[2] = {cols, rows};
  const uint64_t str[1] = {cols * 2};
  const uint32_t box[2] = {64, box_rows};
  return nsk::encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, nullptr,
                          CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace

extern "C" {

// diagnostics: copy the forward trace (16 globaltimer stamps per CTA and step) of the last traced launch
int nsk_gru_trace(long long* out, int steps) {
  if (!g_trace) return nsk::set_error(NSK_ERR_UNSUPPORTED, "gru_tc: run with NSK_GRU_TRACE=1");
  NSK_CUDA(cudaDeviceSynchronize());
  NSK_CUDA(cudaMemcpy(out, g_trace, (size_t)16 * steps * sizeof(long long), cudaMemcpyDeviceToHost));  // steps: T x CTAs
  return NSK_OK;
}

int nsk_gru_tc_supported(int B, int H) {
  int rg, cg;
  return B >= 1 && B <= kMaxB && H % 64 == 0 && H >= 128 && H <= 16 * kUC && bwd_groups(H, &rg, &cg);
}

uint64_t nsk_gru_tc_workspace(int B, int H) {
  int rg = 1, cg = 1;
  bwd_groups(H, &rg, &cg);
  const uint64_t CL = (uint64_t)H / kUC, KR = 3ull * kUC * cg;
  const uint64_t hx = 2ull * B * H * 2;                // forward ring
  const uint64_t gex = 2ull * rg * B * KR * 2;         // backward dgh ring
  const uint64_t pex = 2ull * CL * rg * B * kUC * 4;   // backward partial ring
  const uint64_t bpart = (uint64_t)kMaxGroups * 4 * H * 4;  // per-cluster bias-gradient sums
  return ((hx + 255) / 256 + (gex + 255) / 256 + (pex + 255) / 256) * 256 + bpart;
}

int nsk_gru_fwd_tc(const float* gx, const void* Ubf, const float* c, int T, int B, int H, float* hs, void* hsb,
                   float* gates, void* ws, uint64_t ws_bytes, void* stream) {
  if (!nsk_gru_tc_supported(B, H) || T < 1)
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "gru_tc: needs 1 <= B <= 64 and H in 128..512, H % 64 == 0");
  if (ws_bytes < nsk_gru_tc_workspace(B, H)) return nsk::set_error(NSK_ERR_SHAPE, "gru_tc: workspace too small");
  const int CL = H / kUC;
  const size_t smem = fwd_smem(H);
  const int groups = batch_groups((const void*)gru_fwd_tc_kernel<8>, CL, smem, B);
  const int Bc = B / groups;
  const void* fn = Bc > 32 ? (const void*)gru_fwd_tc_kernel<8>
                 : Bc > 16 ? (const void*)gru_fwd_tc_kernel<4>
                 : Bc > 8  ? (const void*)gru_fwd_tc_kernel<2>
                           : (const void*)gru_fwd_tc_kernel<1>;
  CUtensorMap tmU, tmH;
  int rc = tmap_2d_bf16(&tmU, Ubf, (uint64_t)3 * H, (uint64_t)H, kUC);
  if (rc) return rc;
  __nv_bfloat16* hx = (__nv_bfloat16*)ws;
  {  // h ring as 32-column (64-byte) boxes of one batch group's rows, 64B-swizzled: one box = one CTA's slice
    const uint64_t dims[2] = {(uint64_t)H, (uint64_t)2 * B};
    const uint64_t str[1] = {(uint64_t)H * 2};
    const uint32_t box[2] = {(uint32_t)kUC, (uint32_t)Bc};
    if ((rc = nsk::encode_tmap(&tmH, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, hx, dims, str, box, nullptr,
                               CU_TENSOR_MAP_SWIZZLE_64B)))
      return rc;
  }
  if (getenv("NSK_GRU_TRACE") && !g_trace) cudaMalloc(&g_trace, (size_t)16 * 16 * 4096 * sizeof(long long));
  const bool trace_fwd = getenv("NSK_GRU_TRACE") && getenv("NSK_GRU_TRACE")[0] != '2';
  FwdArgs a{gx, c, hs, gates, (__nv_bfloat16*)hsb, hx, T, B, H, Bc, trace_fwd && T <= 4096 ? g_trace : nullptr};
  void* args[] = {(void*)&tmU, (void*)&tmH, (void*)&a};
  return launch_cluster(fn, CL, groups, smem, args, (cudaStream_t)stream);
}

int nsk_gru_bwd_tc(const float* dhs, const void* Ubf, const float* hs, const float* gates, int T, int B, int H,
                   void* dgx, void* dgh, float* dh0, float* db, float beta_b, float* dc, float beta_c, void* ws,
                   uint64_t ws_bytes, void* stream) {
  if (!nsk_gru_tc_supported(B, H) || T < 1)
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "gru_tc: needs 1 <= B <= 64 and H in 128..512, H % 64 == 0");
  if (ws_bytes < nsk_gru_tc_workspace(B, H)) return nsk::set_error(NSK_ERR_SHAPE, "gru_tc: workspace too small");
  int rg, cg;
  bwd_groups(H, &rg, &cg);
  const int CL = H / kUC, KR = 3 * kUC * cg;
  const size_t smem = bwd_smem(H, rg, cg);
  const int groups = batch_groups((const void*)gru_bwd_tc_kernel<8>, CL, smem, B);
  const int Bc = B / groups;
  const void* fn = Bc > 32 ? (const void*)gru_bwd_tc_kernel<8>
                 : Bc > 16 ? (const void*)gru_bwd_tc_kernel<4>
                 : Bc > 8  ? (const void*)gru_bwd_tc_kernel<2>
                           : (const void*)gru_bwd_tc_kernel<1>;
  // DSMEM-push variant (no global rings, no per-step cluster barriers) where its buffers fit
  const PushLayout PL(H, cg, Bc);
  const size_t push_smem = 1024 + PL.bytes();
  const bool push = Bc <= 32 && H / cg == 128 && push_smem <= 227 * 1024 &&
                    !(getenv("NSK_GRU_PUSH") && getenv("NSK_GRU_PUSH")[0] == '0');
  uint8_t* w = (uint8_t*)ws;
  const uint64_t hx_bytes = ((2ull * B * H * 2 + 255) / 256) * 256;
  const uint64_t gex_bytes = ((2ull * rg * B * KR * 2 + 255) / 256) * 256;
  const uint64_t pex_bytes = ((2ull * CL * rg * B * kUC * 4 + 255) / 256) * 256;
  __nv_bfloat16* gex = (__nv_bfloat16*)(w + hx_bytes);
  float* pex = (float*)(w + hx_bytes + gex_bytes);
  float* bpart = groups > 1 ? (float*)(w + hx_bytes + gex_bytes + pex_bytes) : nullptr;
  CUtensorMap tmU, tmG;
  int rc = tmap_2d_bf16(&tmU, Ubf, (uint64_t)3 * H, (uint64_t)H, kUC);
  if (rc) return rc;
  if ((rc = tmap_2d_bf16(&tmG, gex, (uint64_t)2 * rg * B, (uint64_t)KR, (uint32_t)Bc))) return rc;
  const char* tre = getenv("NSK_GRU_TRACE");
  if (tre && tre[0] == '2' && !g_trace) cudaMalloc(&g_trace, (size_t)16 * 16 * 4096 * sizeof(long long));
  BwdArgs a{dhs, hs, gates, (__nv_bfloat16*)dgx, (__nv_bfloat16*)dgh, dh0, db, dc, beta_b, beta_c, gex, pex,
            bpart, T, B, H, rg, cg, Bc, tre && tre[0] == '2' && T <= 4096 ? g_trace : nullptr};
  if (push) {
    const void* pf = Bc > 16 ? (const void*)gru_bwd_push_kernel<4>
                   : Bc > 8  ? (const void*)gru_bwd_push_kernel<2>
                             : (const void*)gru_bwd_push_kernel<1>;
    void* pargs[] = {(void*)&tmU, (void*)&a};
    rc = launch_cluster(pf, CL, groups, push_smem, pargs, (cudaStream_t)stream);
  } else {
    void* args[] = {(void*)&tmU, (void*)&tmG, (void*)&a};
    rc = launch_cluster(fn, CL, groups, smem, args, (cudaStream_t)stream);
  }
  if (rc) return rc;
  if (bpart) {
    nsk::launch_pdl(gru_bias_fold_kernel, (4 * H + 255) / 256, 256, 0, (cudaStream_t)stream, (const float*)bpart,
                    groups, H, db, beta_b, dc, beta_c);
    NSK_LAUNCH_CHECK("gru_bias_fold_kernel");
  }
  return NSK_OK;
}

}  // extern "C"
