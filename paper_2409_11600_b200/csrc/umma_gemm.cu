// tcgen05/TMEM implicit-GEMM engine: dense GEMM (linear layers) and conv2d
// fprop / dgrad / wgrad on NHWC bf16 activations, fed by TMA.
//
// Replaces (reference): matmul_t   pkg/src/nsk/tensor.py:213-229
//                       plain_matmul pkg/src/nsk/tensor.py:232-234 (via gradient_rule autodiff.py:265-267)
//                       conv2d (absent in the reference; restated in oracle/restated.py)
//
// Persistent: one CTA per SM walks 128 x BN output tiles (or K-splits); double-buffered TMEM accumulators.
//   warp 0 lane 0 : TMA producer   (STAGES-deep smem ring, mbarrier full/empty)
//   warp 1 lane 0 : MMA issuer     (tcgen05.mma kind::f16 | kind::tf32, fp32 accum in TMEM)
//   warp 2        : TMEM allocator
//   warps 4..7    : epilogue       (tcgen05.ld -> bias/beta/convert -> global)
// Every smem stage holds 128 bytes of K per operand row: 4 UMMA k-substeps.
// Operands can be K-major (TMA box {128B of K, rows}) or MN-major
// (boxes of 64 bf16 / 32 fp32 MN-elements x KS K-rows), all 128B-swizzled.
#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "common.cuh"
#include "../../include/nskb.h"

namespace {

enum { MODE_GEMM = 0, MODE_CONV = 1, MODE_WGRAD = 2 };
// BMODE_RR3: row-reuse fprop, the three taps of a column group (filter taps tw, tw+3, tw+6) fetched as ONE
// 3-D box {64 channels, BN filters, 3 taps (element stride 3)} -- one TMA op instead of three
// (BMODE_RR3T: the same box for dgrad, where the 64-channel box dimension is the output (N) side)
enum { BMODE_2D = 0, BMODE_DGRAD3D = 1, BMODE_RR3 = 2, BMODE_RR3T = 3 };

constexpr int kMaxTaps = 9;

struct UmmaProb {
  int mode, bmode;
  int a_mn, b_mn;
  int M, N;
  int k_steps;      // K-steps for this launch (per class for conv; total for wgrad)
  int k_per_split;  // wgrad: K-steps per split
  // conv / wgrad pixel tiling (A operand is a 4D NHWC tensor map)
  int Wt, Ht, Nt;   // pixel tile extents (output-grid units)
  int Wo, Ho;       // output grid (fprop/dgrad) or dy grid (wgrad)
  int cs;           // coordinate stride (conv stride)
  int cchunks;      // reduction channel chunks of 64 per tap
  int ntaps[4];
  signed char tdh[4][kMaxTaps], tdw[4][kMaxTaps], tw[4][kMaxTaps];
  int os, Hd, Wd;   // output pixel mapping: (n, i*os+ph, j*os+pw) in an [Hd x Wd] grid
  signed char cph[4], cpw[4];  // (ph, pw) of class z (dgrad parity classes; classes without taps may be dropped)
  int atoms_total;  // wgrad: M / 64
  int cin_atoms;    // wgrad: Cin / 64
  // epilogue
  void* out;
  long long ldc;
  int out_f32;
  const float* bias;
  float beta;
  int Mpad;         // wgrad workspace row pitch (M padded to the tile)
  // persistent schedule: units = mt * nt * (classes | splits), n-tile fastest
  int mt, nt, units;
  // row-reuse conv schedule (stride-1 gathers, tiles of whole image rows, W % 8 == 0): taps are grouped
  // by column offset dw; one TMA box of Ht + (dh_max - dh_min) rows feeds every tap of the group, each
  // tap's A operand being a view shifted by whole rows (W*128 B, a multiple of the 1 KB swizzle atom).
  int rr;
  int ngroups[4];
  signed char gdw[4][kMaxTaps], gdhmin[4][kMaxTaps], gnt[4][kMaxTaps];
  signed char gdh[4][kMaxTaps][3], gw[4][kMaxTaps][3];
  int ext_rows;  // rows of the A box in rr mode (Ht + dh range)
  int probe;     // diagnostics (env NSK_PROBE): bit0 skip MMAs, bit1 skip stores, bit2 skip B loads,
                 // bit4 no A loads in weight-resident mode, bit5 accumulator never read
  // im2col-mode A operand (any output width): the tile's first pixel sits at bounding-box position
  // (lw + j*cs, lh + i*cs, n) and every tap is an unsigned im2col offset (tdw - lw, tdh - lh)
  int i2c, lw, lh;
  int tma_store;  // bf16 output rows contiguous in m (fprop, stride-1 dgrad, GEMM): epilogue writes via TMA
                  // (2: TMA reduce-add into the existing output, i.e. beta == 1 accumulation)
  int bslab;      // MN-major B (wgrad dy): all BN/64 slabs of a k-step as ONE 3-D box {64, K rows, slabs}
  // conv fprop feeding a BatchNorm: per-CTA channel partials [gridDim.x][2][N] (sum, sum of squares of
  // the bf16-rounded outputs) so the BN statistics need no extra pass over the activation
  float* stats;
  unsigned* fold_reset;  // statistics feeding a fused BatchNorm apply: zero its fold count (bn.cu) at start
  int wres;    // weight-resident row-reuse (see Smem WRES)
  int rr_fast;  // row-reuse 3x3 on 32-wide rows, taps t = 0..2 at row offsets t (1: fprop, 2: dgrad) or 2 - t
                // (4: fprop, 3: dgrad): the MMA issuer uses immediate descriptor offsets
  int asplit;  // WRES: each stage's A box is asplit row bands, one per producer warp (more boxes in flight)
  // dgrad feeding a BatchNorm's backward (nsk_conv2d_dgrad_bnstats): the output is the gradient dz of that
  // BatchNorm's output, stored ReLU-masked (bmask bits; dz = g * [y > 0]); `stats` then receives per-CTA partials
  // [gridDim.x][2][N] of sum dz and sum dz * x (bx = the BatchNorm's input) so the backward needs no reduction
  // pass. bacc: dz = mask * bf16(old + dgrad), the pending gradient accumulated before masking and statistics.
  const __nv_bfloat16* bx;
  const uint8_t* bmask;
  int bacc;
  int stats_shared;  // STATS 1 with wide N: one [2][N] CTA accumulator combined per chunk (per-warp ones do not fit)
  // CTA-pair multicast of the B operand (conv passes with 256-wide tiles, whose few-tile grids are L2-bound: every
  // CTA streams the same filter): launched as 2-CTA clusters, the pair takes adjacent M tiles of one (N tile,
  // class / split) unit, each CTA loads half of every B stage and multicasts it into both; a stage is free again
  // once BOTH CTAs' MMAs are done with it (the MMA commit arrives on both CTAs' empty barriers). mt counts pairs.
  int mc;
};

constexpr int kRRMaxA = 6 * 32 * 128;  // largest rr A box: (4 + 2) rows x 32 pixels x 128 B
constexpr int kStgPitch = 64;          // epilogue staging: 32 x 32 bf16 blocks, 64B-swizzled (TMA-store source)
constexpr int kStgBytes = 32 * kStgPitch;
// byte offset of 16-byte chunk c (of 4) in row r of a staging block: the SWIZZLE_64B pattern (chunk ^= row / 2 % 4)
__device__ __forceinline__ int stg_off(int r, int c) { return r * kStgPitch + ((c ^ ((r >> 1) & 3)) << 4); }

template <int ESZ>
struct KT {
  static constexpr int KE = 128 / ESZ;  // elements per 128B row
  static constexpr int KS = 128 / ESZ;  // K rows per stage for MN-major operands (64 bf16 / 32 fp32)
  static constexpr int UK = 32 / ESZ;   // UMMA K per instruction (16 bf16 / 8 tf32)
};

// WRES: weight-resident row-reuse conv (one 64-channel chunk, 3x3, N = BN): all 9 filter taps are loaded once
// per CTA into a resident region and the ring stages carry only the row-extended A boxes.
template <int BN, int ESZ, int STAGES, bool RR = false, int EPI = 4, bool WRES = false>
struct Smem {
  static constexpr int A_BYTES = RR ? kRRMaxA : 128 * 128;
  static constexpr int B1_BYTES = BN * 128;                                // one tap's B tile
  static constexpr int B_BYTES = WRES ? 0 : B1_BYTES * (RR ? 3 : 1);      // rr: up to 3 taps per column group
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int W_OFF = STAGES * STAGE_BYTES;                      // resident filter taps (WRES)
  static constexpr int BAR_OFF = W_OFF + (WRES ? 9 * B1_BYTES : 0);
  // TMA-store source; 512-byte aligned: the SWIZZLE_64B pattern is taken from address bits 7-8
  static constexpr int STG_OFF = (BAR_OFF + 8 * (2 * STAGES + 9) + 16 + 511) / 512 * 512;
  // staging buffers per epilogue warp: double-buffered with 8 warps (one CTA per SM anyway); single with 4 so
  // the 64/128-wide tiles keep two CTAs per SM
  static constexpr int NSTG = EPI == 8 ? 2 : 1;
  static constexpr int TOTAL = STG_OFF + EPI * NSTG * kStgBytes + 1024;  // + epilogue staging
  // TMEM accumulator buffers: four when they fit the 512 columns beside the co-resident CTA (the epilogue of a tile
  // may then lag the MMAs by up to three tiles), else two
  static constexpr bool kTwoPerSM = 2 * TOTAL + 8192 <= 227 * 1024;
  static constexpr int NACC = (kTwoPerSM ? 256 : 512) / BN >= 4 ? 4 : 2;
  static constexpr int TMEM_COLS = NACC * BN < 32 ? 32 : NACC * BN;
};

// bf16x8 beta*old + v (fp32 math, one rounding): the same value the axpy kernel would produce
__device__ __forceinline__ uint4 bf16x8_axpby(uint4 old, float beta, uint4 v) {
  const __nv_bfloat162* o2 = (const __nv_bfloat162*)&old;
  const __nv_bfloat162* v2 = (const __nv_bfloat162*)&v;
  uint4 r;
  uint32_t* r32 = (uint32_t*)&r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 a = __bfloat1622float2(o2[i]), b = __bfloat1622float2(v2[i]);
    r32[i] = pack_bf16x2(beta * a.x + b.x, beta * a.y + b.y);
  }
  return r;
}

// named barriers: one per epilogue warpgroup (ids 1, 2; 128 threads), one over all epilogue warps (id 3)
__device__ __forceinline__ void epi_bar_group(int group) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + group) : "memory");
}
__device__ __forceinline__ void epi_bar_all(int threads) { asm volatile("bar.sync 3, %0;" ::"r"(threads) : "memory"); }
// MMA gate: the gate warp waits on the mbarriers and releases the MMA warp through named barriers 4..4+STAGES-1
// (stage s full) and 8, 9 (accumulator a drained), 64 threads each (gate warp arrives, MMA warp syncs)
constexpr int kBarFull = 4, kBarAcc = 8;
#ifdef NSK_NO_GATE
constexpr bool kNoGate = true;
#else
constexpr bool kNoGate = false;
#endif
// Two co-resident CTAs per SM hide each other's MMA-issue gaps; the gate warp only pays off for one CTA per SM
// (measured: -3 us on the weight-resident 64-channel conv, +1-2% on the two-per-SM configurations).
template <class S>
struct Launch {
  static constexpr bool kTwoPerSM = 2 * S::TOTAL + 8192 <= 227 * 1024;
#ifdef NSK_GATE_ALL
  static constexpr bool kGate = !kNoGate;
#else
  static constexpr bool kGate = !kTwoPerSM && !kNoGate;
#endif
  template <int EPI>
  static constexpr int threads() { return 128 + 32 * EPI + (kGate ? 32 : 0); }
};
__device__ __forceinline__ void gate_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void gate_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                               int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

// One 64-element K slab (4 UMMA k-steps) with compile-time descriptor steps: the offsets fold into immediates
// of the uniform-register descriptor adds, so the issuing warp runs ~2 instructions per MMA.
template <int AOFF0, int BOFF0, int AST, int BST, bool TF32>
__device__ __forceinline__ void mma_slab_at(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, bool acc) {
  umma_off<((AOFF0 + 0 * AST) >> 4), ((BOFF0 + 0 * BST) >> 4), TF32>(d, ad, bd, idesc, acc ? 1u : 0u);
  umma_off<((AOFF0 + 1 * AST) >> 4), ((BOFF0 + 1 * BST) >> 4), TF32>(d, ad, bd, idesc, 1u);
  umma_off<((AOFF0 + 2 * AST) >> 4), ((BOFF0 + 2 * BST) >> 4), TF32>(d, ad, bd, idesc, 1u);
  umma_off<((AOFF0 + 3 * AST) >> 4), ((BOFF0 + 3 * BST) >> 4), TF32>(d, ad, bd, idesc, 1u);
}

// One 64-element K slab (4 UMMA k-steps) with compile-time descriptor steps (offsets are PTX immediates).
template <int AST, int BST, bool TF32>
__device__ __forceinline__ void mma_slab(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, bool acc) {
  mma_slab_at<0, 0, AST, BST, TF32>(d, ad, bd, idesc, acc);
}

// Row-reuse column group of a 32-wide image: taps t = 0..2 read A shifted by whole rows (4 KB) in ascending
// (DESC = false) or descending order, B at tap t of the strided box; BST = B k-step (32: K-major, 2048: MN-major).
template <int B1, int BST, bool DESC>
__device__ __forceinline__ void mma_rr32(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, bool acc) {
  mma_slab_at<(DESC ? 2 : 0) * 4096, 0 * B1, 32, BST, false>(d, ad, bd, idesc, acc);
  mma_slab_at<1 * 4096, 1 * B1, 32, BST, false>(d, ad, bd, idesc, true);
  mma_slab_at<(DESC ? 0 : 2) * 4096, 2 * B1, 32, BST, false>(d, ad, bd, idesc, true);
}

struct Unit {
  int m0, n0, z;  // tile origin and class (conv) / split (wgrad)
  int kb, nk;     // first k-step and number of k-steps
};

__device__ __forceinline__ Unit decode_unit(const UmmaProb& p, int u, int BN, int crank) {
  Unit w;
  const int mn = p.mt * p.nt;
  w.z = u / mn;
  const int r = u - w.z * mn;
  const int mi = r / p.nt;
  w.m0 = (p.mc ? 2 * mi + crank : mi) * 128;  // pair multicast: adjacent M tiles (past M: all rows masked)
  w.n0 = (r - mi * p.nt) * BN;
  if (p.mode == MODE_WGRAD || p.k_per_split > 0) {  // wgrad, or a split-K GEMM
    w.kb = w.z * p.k_per_split;
    int ke = min(p.k_steps, w.kb + p.k_per_split);
    w.nk = ke > w.kb ? ke - w.kb : 0;
  } else if (p.mode == MODE_CONV) {
    w.kb = 0;
    w.nk = (p.rr ? p.ngroups[w.z] : p.ntaps[w.z]) * p.cchunks;
  } else {
    w.kb = 0;
    w.nk = p.k_steps;
  }
  return w;
}

// Persistent warp-specialised tcgen05 kernel: each CTA walks work units u = blockIdx.x, +gridDim.x, ...
// The smem ring runs continuously across units; two TMEM accumulators let the epilogue of unit j
// overlap the MMAs of unit j+1.
// EPI epilogue warps (4 or 8): with 8, two warpgroups take alternate 32-column chunks of each tile, doubling the
// TMEM-drain / store parallelism for the wide (BN = 256) tiles whose epilogue is the bottleneck.
// STATS (separate instantiations, so the passes without statistics keep their register budget):
//   1: conv fprop feeding a BatchNorm -- per-CTA column sums of y and y^2 of the stored bf16 outputs into p.stats
//   2: dgrad producing the gradient of a BatchNorm's output (feeding nsk_bn_bwd_partials) -- the epilogue masks it
//      with the BatchNorm's ReLU bits, adds the pending gradient (bacc) and sums dz and dz * x (p.bx = BN input)
// Column sums are warp butterflies over the thread-per-row registers into per-warp accumulators: no shared-memory
// traffic beside the MMAs' operand reads (the 64-channel convs are shared-memory bound) and no per-chunk barrier.
template <int BN, int ESZ, int STAGES, bool RR, int EPI, bool WRES, int STATS>
__global__ void __launch_bounds__(Launch<Smem<BN, ESZ, STAGES, RR, EPI, WRES>>::template threads<EPI>(),
                                  Launch<Smem<BN, ESZ, STAGES, RR, EPI, WRES>>::kTwoPerSM ? 2 : 1)
    umma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const UmmaProb p) {
  pdl_wait();
  if (p.fold_reset && blockIdx.x == 0 && threadIdx.x == 0) p.fold_reset[0] = p.fold_reset[1] = 0u;
  using S = Smem<BN, ESZ, STAGES, RR, EPI, WRES>;
  using T = KT<ESZ>;
  constexpr bool kGate = Launch<S>::kGate;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint64_t* full = (uint64_t*)(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  constexpr int NACC = S::NACC;
  uint64_t* tfull = empty + STAGES;  // [NACC] accumulator ready for the epilogue
  uint64_t* tempty = tfull + NACC;   // [NACC] accumulator drained by the epilogue
  uint64_t* wfull = tempty + NACC;   // resident filter taps landed (WRES)
  uint32_t* tmem_slot = (uint32_t*)(wfull + 1);
  // STATS 3 stages fp32 32 x 32 tiles for 128B-swizzled TMA stores: 1 KB aligned (the host adds 512 bytes)
  uint8_t* stage_base = smem + (STATS == 3 ? (S::STG_OFF + 1023) / 1024 * 1024 : S::STG_OFF);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform role index
  const int lane = threadIdx.x & 31;
  const int units = p.units;
  // pair multicast (p.mc): the 2-CTA cluster walks the pair units together; rank = the M tile within the pair
  const int crank = p.mc ? (int)(blockIdx.x & 1) : 0;
  const int u0 = p.mc ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ustep = p.mc ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], WRES ? p.asplit : 1);
      mbar_init(&empty[s], p.mc ? 2 : 1);  // pair multicast: both CTAs' MMAs release the stage
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI);  // one arrival per epilogue warp
    }
    if (WRES) mbar_init(wfull, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, S::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  if (p.mc) cluster_sync_all();  // the peer's barriers are initialised before any multicast targets them
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Up to three TMA issuing threads (warps 0, 2, 3) take k-steps round-robin: one thread only sustains about
  // one TMA box per L2 round trip (tools/tma_rate.cu), so independent issuers multiply the per-SM feed
  // rate. At most STAGES issuers: a producer is then never more than one empty-barrier phase ahead of the
  // MMA consumer, which keeps the parity waits unambiguous.
  constexpr int kProducers = STAGES < 3 ? STAGES : 3;
  const int prod = warp == 0 ? 0 : warp - 1;
  if (lane == 0 && (warp == 0 || warp == 2 || warp == 3) && prod < kProducers) {
    // ---------------- TMA producers ----------------
    int i = 0;  // global k-step counter (smem ring position)
    if (WRES && prod == 0) {
      mbar_expect_tx(wfull, (uint32_t)(p.ngroups[0] * 3 * S::B1_BYTES));
      for (int g = 0; g < p.ngroups[0]; ++g) {
        tma_load_3d(&tmB, wfull, smem + S::W_OFF + g * 3 * S::B1_BYTES, 0, 0, p.gw[0][g][0]);  // N = C = 64
      }
    }
    for (int u = u0; u < units; u += ustep) {
      const Unit w = decode_unit(p, u, BN, crank);
      int n_img = 0, h_img = 0, w_img = 0;
      if (p.mode == MODE_CONV) {
        const int hw = p.Ho * p.Wo;
        n_img = w.m0 / hw;
        const int rem = w.m0 - n_img * hw;
        h_img = rem / p.Wo;
        w_img = rem - h_img * p.Wo;
      }
      const bool half_a = (p.mode == MODE_WGRAD) && (w.m0 / 64 + 1 >= p.atoms_total);
      for (int kk = w.kb; kk < w.kb + w.nk; ++kk, ++i) {
        if (!(WRES && p.asplit > 1) && i % kProducers != prod) continue;  // banded A: every warp, every stage
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait_backoff(&empty[s], ((i / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * S::STAGE_BYTES;
        uint8_t* sb = sa + S::A_BYTES;
        if constexpr (RR) {
          // one row-extended A box for the column group, then the B tile of each tap in the group
          const int ng = p.ngroups[w.z];
          const int chunk = kk / ng;
          const int g = kk - chunk * ng;
          const int c0 = chunk * 64;
          const int nt = p.gnt[w.z][g];
          if (WRES) {
            const int rows = p.ext_rows / p.asplit, band = p.asplit > 1 ? prod : 0;
            if (p.probe & 16) {  // diagnostics: no A traffic (MMAs on stale stages)
              mbar_arrive(&full[s]);
              continue;
            }
            mbar_expect_tx(&full[s], (uint32_t)(rows * p.Wt * 128));
            tma_load_4d(&tmA, &full[s], sa + band * rows * p.Wt * 128, c0, w_img + p.gdw[w.z][g],
                        h_img + p.gdhmin[w.z][g] + band * rows, n_img);
            continue;
          }
          mbar_expect_tx(&full[s], (uint32_t)(p.ext_rows * p.Wt * 128 + nt * S::B1_BYTES));
          tma_load_4d(&tmA, &full[s], sa, c0, w_img + p.gdw[w.z][g], h_img + p.gdhmin[w.z][g], n_img);
          if (p.bmode == BMODE_RR3 || p.bmode == BMODE_RR3T) {
            if (p.bmode == BMODE_RR3)
              tma_load_3d(&tmB, &full[s], sb, c0, w.n0, p.gw[w.z][g][0]);
            else
              tma_load_3d(&tmB, &full[s], sb, w.n0, c0, p.gw[w.z][g][0]);
            continue;
          }
          for (int t = 0; t < nt; ++t) {
            if (p.bmode == BMODE_2D) {
              tma_load_2d(&tmB, &full[s], sb + t * S::B1_BYTES, p.gw[w.z][g][t] * (p.cchunks * 64) + c0, w.n0);
            } else {
#pragma unroll
              for (int b = 0; b < BN / 64; ++b)
                tma_load_3d(&tmB, &full[s], sb + t * S::B1_BYTES + b * 8192, w.n0 + b * 64, p.gw[w.z][g][t], c0);
            }
          }
          continue;
        }
        mbar_expect_tx(&full[s], S::A_BYTES + ((p.probe & 4) ? 0 : S::B_BYTES) - (half_a ? 8192 : 0));
        // ---- A ----
        if (p.mode == MODE_GEMM) {
          if (!p.a_mn) {
            tma_load_2d(&tmA, &full[s], sa, kk * T::KE, w.m0);
          } else {
#pragma unroll
            for (int a = 0; a < 128 / T::KE; ++a)
              tma_load_2d(&tmA, &full[s], sa + a * (T::KS * 128), w.m0 + a * T::KE, kk * T::KS);
          }
        } else if (p.mode == MODE_CONV) {
          const int tap = kk / p.cchunks;
          const int c0 = (kk - tap * p.cchunks) * 64;
          const int cls = p.k_per_split > 0 ? 0 : w.z;  // split-K convs: z is the split, the class is 0
          if (p.i2c)
            tma_load_4d_im2col(&tmA, &full[s], sa, c0, p.lw + w_img * p.cs, p.lh + h_img * p.cs, n_img,
                               (uint16_t)(p.tdw[cls][tap] - p.lw), (uint16_t)(p.tdh[cls][tap] - p.lh));
          else
            tma_load_4d(&tmA, &full[s], sa, c0, w_img * p.cs + p.tdw[cls][tap], h_img * p.cs + p.tdh[cls][tap],
                        n_img);
        } else {  // WGRAD: A = x, MN-major atoms of 64 channels at tap offsets; K = 64 dy pixels
          const int pix0 = kk * 64;
          const int hw = p.Ho * p.Wo;
          const int nn = pix0 / hw;
          const int rem = pix0 - nn * hw;
          const int hh = rem / p.Wo;
          const int ww = rem - hh * p.Wo;
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const int ga = w.m0 / 64 + a;
            if (ga < p.atoms_total) {
              const int tap = ga / p.cin_atoms;
              const int c0 = (ga - tap * p.cin_atoms) * 64;
              if (p.i2c)
                tma_load_4d_im2col(&tmA, &full[s], sa + a * 8192, c0, p.lw + ww * p.cs, p.lh + hh * p.cs, nn,
                                   (uint16_t)(p.tdw[0][tap] - p.lw), (uint16_t)(p.tdh[0][tap] - p.lh));
              else
                tma_load_4d(&tmA, &full[s], sa + a * 8192, c0, ww * p.cs + p.tdw[0][tap], hh * p.cs + p.tdh[0][tap],
                            nn);
            }
          }
        }
        // ---- B ----
        if (p.probe & 4) continue;
        if (p.mode == MODE_GEMM || p.mode == MODE_WGRAD) {
          if (!p.b_mn) {
            tma_load_2d(&tmB, &full[s], sb, kk * T::KE, w.n0);
          } else if (p.bslab) {
            tma_load_3d(&tmB, &full[s], sb, 0, kk * T::KS, w.n0 / T::KE);
          } else {
#pragma unroll
            for (int b = 0; b < BN / T::KE; ++b)
              tma_load_2d(&tmB, &full[s], sb + b * (T::KS * 128), w.n0 + b * T::KE, kk * T::KS);
          }
        } else {
          const int tap = kk / p.cchunks;
          const int c0 = (kk - tap * p.cchunks) * 64;
          const int cls = p.k_per_split > 0 ? 0 : w.z;
          if (p.mc) {  // this CTA's half of the B stage, into both CTAs of the pair (host map: BN/2-row boxes)
            if (p.bmode == BMODE_2D) {
              tma_load_2d_mc(&tmB, &full[s], sb + crank * (BN / 2) * 128, p.tw[cls][tap] * (p.cchunks * 64) + c0,
                             w.n0 + crank * (BN / 2), (uint16_t)3);
            } else {
              for (int b = crank * (BN / 128); b < (crank + 1) * (BN / 128); ++b)
                tma_load_3d_mc(&tmB, &full[s], sb + b * 8192, w.n0 + b * 64, p.tw[cls][tap], c0, (uint16_t)3);
            }
          } else if (p.bmode == BMODE_2D) {
            tma_load_2d(&tmB, &full[s], sb, p.tw[cls][tap] * (p.cchunks * 64) + c0, w.n0);
          } else {
#pragma unroll
            for (int b = 0; b < BN / 64; ++b)
              tma_load_3d(&tmB, &full[s], sb + b * 8192, w.n0 + b * 64, p.tw[cls][tap], c0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp walks the pipeline (converged, so descriptors and ring state stay in uniform registers)
    // and one elected lane issues: issuing from a divergent `lane == 0` branch made ptxas wrap every
    // tcgen05.mma in a waterfall loop with vector->uniform moves, ~130 cycles per MMA instead of ~48.
    const int a_mn = (p.mode == MODE_WGRAD) ? 1 : (p.mode == MODE_CONV ? 0 : p.a_mn);
    const int b_mn = (p.mode == MODE_WGRAD) ? 1 : (p.mode == MODE_CONV ? (p.bmode == BMODE_DGRAD3D || p.bmode == BMODE_RR3T) : p.b_mn);
    const uint32_t idesc = make_idesc(ESZ == 2 ? 1u : 2u, (uint32_t)a_mn, (uint32_t)b_mn, 128u, (uint32_t)BN);
    const uint32_t a_lbo = a_mn ? (T::KS * 128) : 16;
    const uint32_t b_lbo = b_mn ? (T::KS * 128) : 16;
    constexpr int MNS = T::UK * 128;  // MN-major k-step (bytes)
    const int rr_groups = RR ? p.ngroups[0] : 1;  // row reuse runs single-class launches only
    const uint32_t smem0 = smem_u32(smem);
    if (WRES) mbar_wait(wfull, 0);
    // The loop is instantiated per MMA kind (KIND: 1..4 fixed-order 32-wide row reuse, 0 general row reuse,
    // 10..13 one K slab with operand majors a_mn*2+b_mn, -1 no MMAs) so nothing between two MMA bursts reads
    // parameter space or branches through a jump table. Ring position and phase are carried incrementally;
    // the shared-memory descriptors are built once per stage and advanced by immediates.
    auto mma_loop = [&](auto kind_c) {
      constexpr int KIND = decltype(kind_c)::value;
      int s = 0;
      uint32_t ph = 0;
      int j = 0;
      // fixed-order row reuse: every unit has the same k-steps (single class, no split) -- no per-tile decode
      const int nk_fixed = (KIND >= 1 && KIND <= 4) ? rr_groups * p.cchunks : 0;
      for (int u = u0; u < units; u += ustep, ++j) {
        Unit w;
        if constexpr (KIND >= 1 && KIND <= 4) {
          w.z = 0;
          w.nk = nk_fixed;
        } else {
          w = decode_unit(p, u, BN, crank);
        }
        const int acc = j % NACC;
        if (j >= NACC) {
          if constexpr (kGate)
            gate_sync(kBarAcc + acc);
          else
            mbar_wait(&tempty[acc], (j / NACC - 1) & 1);
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int g = 0;  // RR column group of k-step k
        for (int k = 0; k < w.nk; ++k) {
          if constexpr (kGate)
            gate_sync(kBarFull + s);
          else
            mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem0 + s * S::STAGE_BYTES;
          const uint64_t ad0 = sdesc_sw128(sa, a_lbo, 1024);
          const uint64_t bd0 =
              sdesc_sw128(WRES ? smem0 + S::W_OFF + g * 3 * S::B1_BYTES : sa + S::A_BYTES, b_lbo, 1024);
          if (elect_one()) {
            constexpr int B1 = S::B1_BYTES;
            constexpr bool TF = ESZ == 4;
            if constexpr (KIND == 1) {
              mma_rr32<B1, 32, false>(d_tmem, ad0, bd0, idesc, k > 0);
            } else if constexpr (KIND == 2) {
              mma_rr32<B1, 2048, false>(d_tmem, ad0, bd0, idesc, k > 0);
            } else if constexpr (KIND == 3) {
              mma_rr32<B1, 2048, true>(d_tmem, ad0, bd0, idesc, k > 0);
            } else if constexpr (KIND == 4) {
              mma_rr32<B1, 32, true>(d_tmem, ad0, bd0, idesc, k > 0);
            } else if constexpr (KIND == 0) {
              const uint32_t b_step = b_mn ? MNS : 32;
              const int nt = p.gnt[w.z][g];
              for (int t = 0; t < nt; ++t) {
                // tap view: rows shifted by (dh - dh_min) whole image rows of Wt pixels
                const uint32_t aoff = (uint32_t)((p.gdh[w.z][g][t] - p.gdhmin[w.z][g]) * p.Wt * 128);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  umma_bf16(d_tmem, ad0 + ((aoff + q * 32) >> 4), bd0 + ((uint32_t)(t * B1 + q * b_step) >> 4),
                            idesc, (k > 0 || t > 0 || q > 0) ? 1u : 0u);
              }
            } else if constexpr (KIND == 10) {
              mma_slab<32, 32, TF>(d_tmem, ad0, bd0, idesc, k > 0);
            } else if constexpr (KIND == 11) {
              mma_slab<32, MNS, TF>(d_tmem, ad0, bd0, idesc, k > 0);
            } else if constexpr (KIND == 12) {
              mma_slab<MNS, 32, TF>(d_tmem, ad0, bd0, idesc, k > 0);
            } else if constexpr (KIND == 13) {
              mma_slab<MNS, MNS, TF>(d_tmem, ad0, bd0, idesc, k > 0);
            }
            if (p.mc)
              umma_commit_mc(&empty[s], (uint16_t)3);
            else
              umma_commit(&empty[s]);
          }
          __syncwarp();
          if (RR && ++g == rr_groups) g = 0;
          if (++s == STAGES) {
            s = 0;
            ph ^= 1u;
          }
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
      }
    };
    using std::integral_constant;
    if constexpr (RR) {
      switch (p.rr_fast) {
        case 1: mma_loop(integral_constant<int, 1>{}); break;
        case 2: mma_loop(integral_constant<int, 2>{}); break;
        case 3: mma_loop(integral_constant<int, 3>{}); break;
        case 4: mma_loop(integral_constant<int, 4>{}); break;
        default: mma_loop(integral_constant<int, 0>{}); break;
      }
    } else if (p.probe & 1) {
      mma_loop(integral_constant<int, -1>{});
    } else {
      switch (a_mn * 2 + b_mn) {
        case 0: mma_loop(integral_constant<int, 10>{}); break;
        case 1: mma_loop(integral_constant<int, 11>{}); break;
        case 2: mma_loop(integral_constant<int, 12>{}); break;
        default: mma_loop(integral_constant<int, 13>{}); break;
      }
    }
  } else if (kGate && warp == 4 + EPI) {
    // ---------------- MMA gate ----------------
    // Any shared-memory read by the MMA warp (an mbarrier try_wait, even on a completed phase) waits for the
    // tensor pipe's queued operand reads and leaves it idle for ~130 cycles per stage -- a third of the time
    // with 64-wide MMAs (tools/mma_gap.cu). This warp does the mbarrier waits in the MMA warp's order and
    // releases it through named barriers, which cost the MMA warp nothing.
    int s = 0;
    uint32_t phase = 0;
    int j = 0;
    for (int u = u0; u < units; u += ustep, ++j) {
      const Unit w = decode_unit(p, u, BN, crank);
      const int acc = j % NACC;
      if (j >= NACC) {
        mbar_wait(&tempty[acc], (j / NACC - 1) & 1);
        gate_arrive(kBarAcc + acc);
      }
      for (int k = 0; k < w.nk; ++k) {
        mbar_wait(&full[s], phase);
        gate_arrive(kBarFull + s);
        if (++s == STAGES) {
          s = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp >= 4 && warp < 4 + EPI) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;         // TMEM lane quarter (a warp may only access lanes 32*(warp%4) .. +31)
    const int eg = (warp - 4) >> 2;  // epilogue warpgroup: chunks eg, eg + EPI/4, ...
    const int r = q * 32 + lane;  // tile row == TMEM lane
    const bool vec_ok = ((p.ldc * (p.out_f32 ? 4 : 2)) % 16 == 0);
    int sbuf = 0;  // staging double buffer (TMA stores of the previous chunk may still be reading the other)
    // output element offset of this thread's row of unit w
    auto row_of = [&](const Unit& w) -> long long {
      const int m = w.m0 + r;
      if (p.mode == MODE_WGRAD) return (long long)w.z * p.N * p.Mpad + m;  // transposed partials: ws[split][n][m]
      if (p.mode == MODE_CONV && p.k_per_split > 0) return ((long long)w.z * p.M + m) * p.ldc;  // split-K conv
      if (p.mode == MODE_CONV) {
        const int hw = p.Ho * p.Wo;
        const int nn = m / hw;
        const int rem = m - nn * hw;
        const int ii = rem / p.Wo;
        const int jj = rem - ii * p.Wo;
        const int ph = p.cph[w.z], pw = p.cpw[w.z];
        const long long pix = ((long long)nn * p.Hd + ii * p.os + ph) * p.Wd + (jj * p.os + pw);
        return pix * p.ldc;
      }
      // split-K GEMM: fp32 partials of split z into ws[z][M][N] (p.out / p.ldc set up by the host)
      return ((long long)(p.k_per_split > 0 ? w.z : 0) * p.M + m) * p.ldc;
    };
    auto chunks_of = [&](const Unit& w) {
      const int n = (p.N - w.n0 + 31) / 32;
      return n > BN / 32 ? BN / 32 : n;
    };
    // statistics (STATS): per-warp column sums, [EPI warps][2][N / G] floats (G = EPI / 4 warpgroups; warp (q, eg)
    // owns the 32-column chunks gc = eg mod G of the output)
    constexpr int G = EPI / 4;
    float* st_col = (float*)(stage_base + EPI * S::NSTG * kStgBytes);
    const int ncol_w = (p.N / 32 + G - 1) / G * 32;  // columns per warp
    if constexpr (STATS == 1 || STATS == 2) {
      if (p.stats_shared) {
        for (int i = threadIdx.x - 128; i < 2 * p.N; i += 32 * EPI) st_col[i] = 0.f;
        epi_bar_all(32 * EPI);
      } else {
        for (int i = lane; i < 2 * ncol_w; i += 32) st_col[(warp - 4) * 2 * ncol_w + i] = 0.f;
        __syncwarp();
      }
    }
    int j = 0;
    for (int u = u0; u < units; u += ustep, ++j) {
      const Unit w = decode_unit(p, u, BN, crank);
      const int acc = j % NACC;
      mbar_wait_backoff(&tfull[acc], (j / NACC) & 1);
      tc_fence_after();
      const int m = w.m0 + r;
      const bool row_ok = m < p.M;
      const long long row_off = row_of(w);
      const int nchunks = chunks_of(w);
#pragma unroll 1
      for (int c = eg; c < nchunks; c += EPI / 4) {
        uint32_t v[32];
        if (p.probe & 32) continue;  // diagnostics: accumulator never read
        // STATS 2: this row's ReLU-mask word, requested before the TMEM load
        uint32_t bmw = 0xffffffffu;
        if constexpr (STATS == 2) {
          if (row_ok && p.bmask) bmw = __ldg((const uint32_t*)(p.bmask + ((row_off + w.n0 + c * 32) >> 3)));
        }
        if (w.nk > 0) {
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) v[t] = 0;
        }
        const int col0 = w.n0 + c * 32;
        if (p.probe & 2) continue;
        float f[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) f[t] = __uint_as_float(v[t]);
        if (p.mode == MODE_WGRAD) {
          if (row_ok) {
            float* o = (float*)p.out + row_off + (long long)col0 * p.Mpad;
            for (int t = 0; t < 32; ++t)
              if (col0 + t < p.N) o[(long long)t * p.Mpad] = f[t];
          }
          continue;
        }
        if constexpr (S::NSTG == 2 && STATS == 3) {
          if (p.out_f32 && p.tma_store && (col0 + 32 <= p.N) && !((uintptr_t)p.bias & 15)) {
            // beta = 0: the swizzled staging tile is the TMA store's source (SWIZZLE_128B map over [splits][M][N]
            // fp32, so a ragged M tile clips inside its split). The hardware swizzle follows address bits 7-9: the
            // tile starts on a 1 KB boundary (stage_base above)
            if (p.bias) {
#pragma unroll
              for (int g = 0; g < 8; ++g) {
                const float4 b4 = __ldg((const float4*)(p.bias + col0) + g);
                f[4 * g] += b4.x;
                f[4 * g + 1] += b4.y;
                f[4 * g + 2] += b4.z;
                f[4 * g + 3] += b4.w;
              }
            }
            float* sf = (float*)(stage_base + (warp - 4) * S::NSTG * kStgBytes);
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous store read it
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 8; ++g)
              *(float4*)(sf + lane * 32 + ((g ^ (lane & 7)) << 2)) = make_float4(f[4 * g], f[4 * g + 1], f[4 * g + 2],
                                                                                 f[4 * g + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(&tmC),
                  "r"(smem_u32(sf)), "r"(col0), "r"(w.m0 + q * 32), "r"(p.k_per_split > 0 ? w.z : 0)
                  : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            continue;
          }
          if (p.out_f32 && (col0 + 32 <= p.N) && vec_ok && !((uintptr_t)p.bias & 15)) {
            // fp32 through the warp's two staging buffers (32 x 32 floats, 16-byte granule g of row r at g ^ (r % 8):
            // conflict-free both ways), then 8 lanes per row: each store instruction covers 4 rows x 128 contiguous
            // bytes instead of 32 rows x 16 bytes; lane owns columns 4 (lane % 8) .. +3, so the bias is one float4 per
            // lane. A separate instantiation (STATS 3, fp32-output GEMMs and split-K partials): compiled into the
            // conv kernels it raised them from 96 to 119 registers (ResNet-18 2.10 -> 2.14 ms/step)
            const int part = lane & 7;
            const float4 bv = p.bias ? __ldg((const float4*)(p.bias + col0) + part) : make_float4(0.f, 0.f, 0.f, 0.f);
            // GEMM and split-K rows are linear in m: row pr of this warp's 32 sits pr * ldc after row 0
            const long long ro0 = __shfl_sync(0xffffffffu, row_off, 0);
            const int mrow0 = w.m0 + q * 32;
            float* sf = (float*)(stage_base + (warp - 4) * S::NSTG * kStgBytes);
            __syncwarp();  // the previous chunk's reads of the staging tile are done
#pragma unroll
            for (int g = 0; g < 8; ++g)
              *(float4*)(sf + lane * 32 + ((g ^ (lane & 7)) << 2)) = make_float4(f[4 * g], f[4 * g + 1], f[4 * g + 2],
                                                                                 f[4 * g + 3]);
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int pr = it * 4 + (lane >> 3);
              const long long ro = ro0 + (long long)pr * p.ldc;
              if (mrow0 + pr < p.M) {
                float4 v = *(const float4*)(sf + pr * 32 + ((part ^ (pr & 7)) << 2));
                v.x += bv.x;
                v.y += bv.y;
                v.z += bv.z;
                v.w += bv.w;
                float4* dst = (float4*)((float*)p.out + ro + col0 + part * 4);
                if (p.beta != 0.f) {
                  const float4 o = *dst;
                  v.x += p.beta * o.x;
                  v.y += p.beta * o.y;
                  v.z += p.beta * o.z;
                  v.w += p.beta * o.w;
                }
                *dst = v;
              }
            }
            continue;
          }
        }
        if (p.bias) {
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (col0 + t < p.N) f[t] += p.bias[col0 + t];
        }
        const bool full_chunk = (col0 + 32 <= p.N) && vec_ok;
        if (p.out_f32) {
          if (row_ok) {
            float* o = (float*)p.out + row_off + col0;
            if (p.beta != 0.f) {
              for (int t = 0; t < 32; ++t)
                if (col0 + t < p.N) f[t] += p.beta * o[t];
            }
            if (full_chunk) {
#pragma unroll
              for (int t = 0; t < 32; t += 4) *(float4*)(o + t) = make_float4(f[t], f[t + 1], f[t + 2], f[t + 3]);
            } else {
              for (int t = 0; t < 32; ++t)
                if (col0 + t < p.N) o[t] = f[t];
            }
          }
        } else if (full_chunk) {
          // bf16: stage this warp's 32 rows x 32 columns in shared memory, then write 16-byte pieces so
          // one store instruction covers 8 rows x 64 contiguous bytes instead of 32 scattered rows.
          uint8_t* stg = stage_base + ((warp - 4) * S::NSTG + sbuf) * kStgBytes;
          if (p.tma_store) {
            if (lane == 0) {  // the TMA store that last read this buffer is done with it
              if constexpr (S::NSTG == 2)
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              else
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
          }
          uint4 u4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            u4[t].x = pack_bf16x2(f[8 * t], f[8 * t + 1]);
            u4[t].y = pack_bf16x2(f[8 * t + 2], f[8 * t + 3]);
            u4[t].z = pack_bf16x2(f[8 * t + 4], f[8 * t + 5]);
            u4[t].w = pack_bf16x2(f[8 * t + 6], f[8 * t + 7]);
          }
          if constexpr (STATS == 2) {
            // dz = [y > 0] * bf16(pending + bf16(dgrad)) -- the pending gradient added as the TMA reduce-add / axpby
            // accumulation paths add it; masking commutes with the rounding
            const uint4* o4 = (const uint4*)((const __nv_bfloat16*)p.out + row_off + col0);
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              uint4 v4 = u4[c4];
              if (p.bacc && row_ok) v4 = bf16x8_axpby(o4[c4], 1.f, v4);
              const uint32_t m8 = bmw >> (8 * c4);
              uint32_t* v32 = (uint32_t*)&v4;
#pragma unroll
              for (int i = 0; i < 4; ++i)
                v32[i] &= (((m8 >> (2 * i)) & 1u) ? 0x0000ffffu : 0u) | (((m8 >> (2 * i + 1)) & 1u) ? 0xffff0000u : 0u);
              u4[c4] = v4;
            }
          }
          // 64-byte-swizzled staging (the TMA store map uses SWIZZLE_64B): 16-byte chunk c of row r sits at chunk
          // c ^ ((r >> 1) & 3). Each quarter-warp store then covers all 32 banks exactly once, and the chunk index
          // of the register operand stays static (a lane-dependent register index spilled u4 to local memory)
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) *(uint4*)(stg + stg_off(lane, c4)) = u4[c4];
          if (p.tma_store) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if constexpr (STATS == 1) {
            // column sums of the staged (bf16-rounded) tile: lane = column, this warp's 32 rows, into the warp's own
            // accumulators (no cross-warp barrier per chunk)
            const unsigned okm = __ballot_sync(0xffffffffu, row_ok);
            float s1 = 0.f, s2 = 0.f;
#pragma unroll 8
            for (int rr = 0; rr < 32; ++rr) {
              const float v =
                  __bfloat162float(*(const __nv_bfloat16*)(stg + stg_off(rr, lane >> 3) + (lane & 7) * 2));
              if ((okm >> rr) & 1u) {
                s1 += v;
                s2 += v * v;
              }
            }
            if (p.stats_shared) {
              // [2][N] CTA accumulator: the four lane-quarter warps of this warpgroup combine in fixed order
              float* st_red = st_col + 2 * p.N + eg * 256;  // per warpgroup: [4 warps][2][32]
              st_red[q * 64 + lane] = s1;
              st_red[q * 64 + 32 + lane] = s2;
              epi_bar_group(eg);
              if (q == 0) {
                st_col[col0 + lane] += (st_red[lane] + st_red[64 + lane]) + (st_red[128 + lane] + st_red[192 + lane]);
                st_col[p.N + col0 + lane] +=
                    (st_red[32 + lane] + st_red[96 + lane]) + (st_red[160 + lane] + st_red[224 + lane]);
              }
              epi_bar_group(eg);
            } else {
              float* col = st_col + (warp - 4) * 2 * ncol_w + (col0 / 32 / G) * 32 + lane;
              col[0] += s1;
              col[ncol_w] += s2;
            }
          } else if constexpr (STATS == 2) {
            // column sums over this warp's 32 rows (thread = row) by a butterfly reduce-scatter: lane ends with column
            // col0 + lane (the BatchNorm input is read per row straight from global memory)
            float red[32];
            const uint4* x4 = (const uint4*)(p.bx + row_off + col0);
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const __nv_bfloat162* hz = (const __nv_bfloat162*)&u4[c4];
              const uint4 xv = row_ok ? __ldg(x4 + c4) : make_uint4(0u, 0u, 0u, 0u);
              const __nv_bfloat162* hx = (const __nv_bfloat162*)&xv;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 z = __bfloat1622float2(hz[i]), xx = __bfloat1622float2(hx[i]);
                red[8 * c4 + 2 * i] = z.x * xx.x;
                red[8 * c4 + 2 * i + 1] = z.y * xx.y;
              }
            }
            const float s2 = warp_colsum32(red, lane);
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const __nv_bfloat162* hz = (const __nv_bfloat162*)&u4[c4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 z = __bfloat1622float2(hz[i]);
                red[8 * c4 + 2 * i] = row_ok ? z.x : 0.f;
                red[8 * c4 + 2 * i + 1] = row_ok ? z.y : 0.f;
              }
            }
            const float s1 = warp_colsum32(red, lane);
            float* col = st_col + (warp - 4) * 2 * ncol_w + (col0 / 32 / G) * 32 + lane;
            col[0] += s1;
            col[ncol_w] += s2;
          }
          if (p.tma_store) {
            if (lane == 0) {
              if (p.tma_store == 2)
                asm volatile(
                    "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                        &tmC),
                    "r"(smem_u32(stg)), "r"(col0), "r"(w.m0 + q * 32)
                    : "memory");
              else
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmC),
                    "r"(smem_u32(stg)), "r"(col0), "r"(w.m0 + q * 32)
                    : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            sbuf = (sbuf + 1) % S::NSTG;
            continue;
          }
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int piece = it * 32 + lane;
            const int pr = piece >> 2, part = piece & 3;
            const long long ro = __shfl_sync(0xffffffffu, row_off, pr);
            const int ok = __shfl_sync(0xffffffffu, (int)row_ok, pr);
            if (ok) {
              uint4* dst = (uint4*)((__nv_bfloat16*)p.out + ro + col0 + part * 8);
              uint4 val = *(const uint4*)(stg + stg_off(pr, part));
              if (p.beta != 0.f) val = bf16x8_axpby(*dst, p.beta, val);  // accumulate into an existing gradient
              *dst = val;
            }
          }
          __syncwarp();
        } else if (row_ok) {
          __nv_bfloat16* o = (__nv_bfloat16*)p.out + row_off + col0;
          for (int t = 0; t < 32; ++t)
            if (col0 + t < p.N) o[t] = __float2bfloat16_rn(f[t]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if (p.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if constexpr (STATS == 1 || STATS == 2) {
      // CTA partials [2][N]: the four lane-quarter warps of the owning warpgroup, in fixed order
      epi_bar_all(32 * EPI);
      float* out = p.stats + (size_t)blockIdx.x * 2 * p.N;
      for (int i = threadIdx.x - 128; i < 2 * p.N; i += 32 * EPI) {
        if (p.stats_shared) {
          out[i] = st_col[i];
          continue;
        }
        const int k = i / p.N, n = i - k * p.N;
        const int gc = n / 32, e = gc % G, li = (gc / G) * 32 + (n & 31);
        float t = 0.f;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) t += st_col[(e * 4 + qq) * 2 * ncol_w + k * ncol_w + li];
        out[i] = t;
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, S::TMEM_COLS);
  }
  if (p.mc) cluster_sync_all();  // no CTA leaves while its peer may still multicast into it
}

// wgrad split-K reduction: ws[split][N][Mpad] (rows = cout, cols = (tap, cin)) -> dw[cout][tap][cin] (+= if beta).
// Both sides are contiguous in the (tap, cin) index. Block (32, SL): 32 float4 columns x SL split slices (slice s
// takes splits s, s+SL, ...), slices combined in slice order: deterministic. Small outputs with many splits (576 x 64
// is only 9216 float4 columns) use 8 slices for 8x the loads in flight; large outputs one.
template <int kWgSlices>
__global__ void __launch_bounds__(256) wgrad_reduce_kernel(const float* __restrict__ ws, int splits, int Mpad, int M,
                                                           int N, float* dw, float beta) {
  pdl_wait();
  constexpr int XT = 256 / kWgSlices;
  __shared__ float4 red[kWgSlices][XT];
  const long long total4 = (long long)M * N / 4;
  const long long i4 = (long long)blockIdx.x * XT + threadIdx.x;
  const int sl = threadIdx.y;
  const long long plane = (long long)N * Mpad;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  long long idx = 0;
  if (i4 < total4) {
    idx = i4 * 4;
    const int n = (int)(idx / M);
    const int m = (int)(idx - (long long)n * M);
    const float* src = ws + (long long)n * Mpad + m;
    int s = sl;
    for (; s + 3 * kWgSlices < splits; s += 4 * kWgSlices) {
      const float4 v0 = __ldg((const float4*)(src + (s + 0 * kWgSlices) * plane));
      const float4 v1 = __ldg((const float4*)(src + (s + 1 * kWgSlices) * plane));
      const float4 v2 = __ldg((const float4*)(src + (s + 2 * kWgSlices) * plane));
      const float4 v3 = __ldg((const float4*)(src + (s + 3 * kWgSlices) * plane));
      acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
      acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w;
      acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w;
      acc.x += v3.x; acc.y += v3.y; acc.z += v3.z; acc.w += v3.w;
    }
    for (; s < splits; s += kWgSlices) {
      const float4 v = __ldg((const float4*)(src + s * plane));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (kWgSlices > 1) {
    red[sl][threadIdx.x] = acc;
    __syncthreads();
  }
  if (sl != 0 || i4 >= total4) return;
  float4 t = acc;
#pragma unroll
  for (int k = 1; k < kWgSlices; ++k) {
    const float4 v = red[k][threadIdx.x];
    t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
  }
  float4* d = (float4*)(dw + idx);
  if (beta != 0.f) {
    const float4 o = *d;
    t.x += beta * o.x; t.y += beta * o.y; t.z += beta * o.z; t.w += beta * o.w;
  }
  *d = t;
}


// ---- row-reuse weight gradient for 3x3 / stride 1 / 64 -> 64 channels on 32-wide images ----
// dW[co][tap][ci] = sum_pix dy[pix][co] x[pix + tap][ci]. One work unit = a range of 64-pixel k-steps (two image
// rows) for ALL nine taps: per k-step three 4-row x boxes (one per column offset dw, rows h-1..h+2, 16 KB each)
// serve the three row offsets dh as K-views shifted by whole rows (32 pixels = 4 KB, a multiple of the 1 KB
// swizzle atom), and the dy box (8 KB) is loaded once for all taps -- 56 KB per k-step instead of 5 x 24 KB.
// M = 9 taps x 64 channels is issued as five 128-row MMA tiles whose two 64-channel atoms sit at a per-tile
// leading-byte offset: (dh -1, dh +1) of one box (8 KB apart) x3, (dh 0 of dw -1, dh 0 of dw 0) across two
// boxes (16 KB), and (dh 0 of dw +1, unused). Five TMEM accumulators (320 columns), fp32 partials per unit
// into ws[split][co][Mpad] (rows m = tap * 64 + ci), folded by wgrad_reduce_kernel.
struct WgrrProb {
  int k_steps, per, units;
  int HW, Wimg;  // pixels per image, image width (32)
  float* ws;
  int Mpad;
};
constexpr int kWgrrStages = 3;
constexpr int kWgrrStage = 3 * 16384 + 8192;
__constant__ signed char c_wgrr_tap[5][2] = {{0, 6}, {1, 7}, {2, 8}, {3, 4}, {5, -1}};

__global__ void __launch_bounds__(256, 1) wgrad_rr64_kernel(const __grid_constant__ CUtensorMap tmX,
                                                            const __grid_constant__ CUtensorMap tmDY,
                                                            const WgrrProb p) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint64_t* full = (uint64_t*)(smem + kWgrrStages * kWgrrStage);
  uint64_t* empty = full + kWgrrStages;
  uint64_t* tfull = empty + kWgrrStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWgrrStages; ++s) {
      mbar_init(&full[s], 2);  // two producer threads arrive per stage
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmDY);
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if ((warp == 0 || warp == 2) && lane == 0) {
    // producers: warp 0 the dw = -1 box and dy, warp 2 the dw = 0 and +1 boxes
    int i = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int kb = u * p.per, ke = min(p.k_steps, kb + p.per);
      for (int kk = kb; kk < ke; ++kk, ++i) {
        const int s = i % kWgrrStages;
        if (i >= kWgrrStages) mbar_wait_backoff(&empty[s], ((i / kWgrrStages) - 1) & 1);
        uint8_t* st = smem + s * kWgrrStage;
        const int pix0 = kk * 64;
        const int n = pix0 / p.HW;
        const int hh = (pix0 - n * p.HW) / p.Wimg;
        if (warp == 0) {
          mbar_expect_tx(&full[s], 16384 + 8192);
          tma_load_4d(&tmX, &full[s], st, 0, -1, hh - 1, n);
          tma_load_2d(&tmDY, &full[s], st + 3 * 16384, 0, pix0);
        } else {
          mbar_expect_tx(&full[s], 2 * 16384);
          tma_load_4d(&tmX, &full[s], st + 16384, 0, 0, hh - 1, n);
          tma_load_4d(&tmX, &full[s], st + 2 * 16384, 0, 1, hh - 1, n);
        }
      }
    }
  } else if (warp == 3) {
    // gate: mbarrier waits on behalf of the MMA warp (released through named barriers)
    int i = 0, j = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++j) {
      if (j >= 1) {
        mbar_wait(tempty, (j - 1) & 1);
        gate_arrive(kBarAcc);
      }
      const int kb = u * p.per, ke = min(p.k_steps, kb + p.per);
      for (int kk = kb; kk < ke; ++kk, ++i) {
        const int s = i % kWgrrStages;
        mbar_wait(&full[s], (i / kWgrrStages) & 1);
        gate_arrive(kBarFull + s);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(1u, 1u, 1u, 128u, 64u);
    const uint32_t smem0 = smem_u32(smem);
    int s = 0, j = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++j) {
      if (j >= 1) gate_sync(kBarAcc);
      tc_fence_after();
      const int kb = u * p.per, ke = min(p.k_steps, kb + p.per);
      for (int kk = kb; kk < ke; ++kk) {
        gate_sync(kBarFull + s);
        tc_fence_after();
        const uint32_t st = smem0 + s * kWgrrStage;
        const uint64_t b0 = sdesc_sw128(st + 3 * 16384, 8192, 1024);
        const uint64_t t0 = sdesc_sw128(st, 8192, 1024), t1 = sdesc_sw128(st + 16384, 8192, 1024);
        const uint64_t t2 = sdesc_sw128(st + 2 * 16384, 8192, 1024), t3 = sdesc_sw128(st + 4096, 16384, 1024);
        const uint64_t t4 = sdesc_sw128(st + 2 * 16384 + 4096, 8192, 1024);
        if (elect_one()) {
          const bool acc = kk > kb;
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 0 * 64, t0, b0, idesc, acc);
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 1 * 64, t1, b0, idesc, acc);
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 2 * 64, t2, b0, idesc, acc);
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 3 * 64, t3, b0, idesc, acc);
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 4 * 64, t4, b0, idesc, acc);
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == kWgrrStages) s = 0;
      }
      if (elect_one()) umma_commit(tfull);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int r = q * 32 + lane;  // accumulator row: atom r / 64, input channel r % 64
    const int atom = r >> 6, ci = r & 63;
    int j = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++j) {
      mbar_wait_backoff(tfull, j & 1);
      tc_fence_after();
      float* out = p.ws + (size_t)u * 64 * p.Mpad;
#pragma unroll 1
      for (int T = 0; T < 5; ++T) {
        const int tap = c_wgrr_tap[T][atom];
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + T * 64 + c * 32, v);
          tmem_ld_wait();
          if (tap >= 0) {
            float* o = out + (size_t)(c * 32) * p.Mpad + tap * 64 + ci;
#pragma unroll
            for (int t = 0; t < 32; ++t) o[(size_t)t * p.Mpad] = __uint_as_float(v[t]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}


// Row-reuse weight gradient for 3x3 / stride 1 / 128 -> 128 channels on 16-wide images. Nine 128-row tiles do not
// fit TMEM at N = 128, so a work unit is (column offset dw, range of k-steps): per 64-pixel k-step (4 rows) two
// 6-row x boxes (the two 64-channel halves, 12 KB each) serve the three row offsets dh as K views shifted by
// 16 pixels (2 KB), dy (both 64-wide halves of the 128 outputs) is one 16 KB load; three 128x128 tiles (one per
// dh; atoms = the two channel halves, 12 KB apart) accumulate in TMEM. 40 KB per k-step for 12 MMAs of N = 128,
// against 32 KB per 4 MMAs in the generic tiling.
constexpr int kWg128Stages = 4;
constexpr int kWg128Stage = 2 * 12288 + 16384;

__global__ void __launch_bounds__(256, 1) wgrad_rr128_kernel(const __grid_constant__ CUtensorMap tmX,
                                                             const __grid_constant__ CUtensorMap tmDY,
                                                             const WgrrProb p) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint64_t* full = (uint64_t*)(smem + kWg128Stages * kWg128Stage);
  uint64_t* empty = full + kWg128Stages;
  uint64_t* tfull = empty + kWg128Stages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWg128Stages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmDY);
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if ((warp == 0 || warp == 2) && lane == 0) {
    // warp 0: channel half 0 and dy; warp 2: channel half 1
    int i = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int dw = u % 3 - 1, z = u / 3;
      const int kb = z * p.per, ke = min(p.k_steps, kb + p.per);
      for (int kk = kb; kk < ke; ++kk, ++i) {
        const int s = i % kWg128Stages;
        if (i >= kWg128Stages) mbar_wait_backoff(&empty[s], ((i / kWg128Stages) - 1) & 1);
        uint8_t* st = smem + s * kWg128Stage;
        const int pix0 = kk * 64;
        const int n = pix0 / p.HW;
        const int hh = (pix0 - n * p.HW) / p.Wimg;
        if (warp == 0) {
          mbar_expect_tx(&full[s], 12288 + 16384);
          tma_load_4d(&tmX, &full[s], st, 0, dw, hh - 1, n);
          tma_load_3d(&tmDY, &full[s], st + 2 * 12288, 0, pix0, 0);
        } else {
          mbar_expect_tx(&full[s], 12288);
          tma_load_4d(&tmX, &full[s], st + 12288, 64, dw, hh - 1, n);
        }
      }
    }
  } else if (warp == 3) {
    int i = 0, j = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++j) {
      if (j >= 1) {
        mbar_wait(tempty, (j - 1) & 1);
        gate_arrive(kBarAcc);
      }
      const int z = u / 3;
      const int kb = z * p.per, ke = min(p.k_steps, kb + p.per);
      for (int kk = kb; kk < ke; ++kk, ++i) {
        const int s = i % kWg128Stages;
        mbar_wait(&full[s], (i / kWg128Stages) & 1);
        gate_arrive(kBarFull + s);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(1u, 1u, 1u, 128u, 128u);
    const uint32_t smem0 = smem_u32(smem);
    int s = 0, j = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++j) {
      if (j >= 1) gate_sync(kBarAcc);
      tc_fence_after();
      const int z = u / 3;
      const int kb = z * p.per, ke = min(p.k_steps, kb + p.per);
      for (int kk = kb; kk < ke; ++kk) {
        gate_sync(kBarFull + s);
        tc_fence_after();
        const uint32_t st = smem0 + s * kWg128Stage;
        const uint64_t b0 = sdesc_sw128(st + 2 * 12288, 8192, 1024);  // two 64-wide output halves, 8 KB apart
        const uint64_t a0 = sdesc_sw128(st, 12288, 1024);             // dh = -1: rows 0..63 of both halves
        const uint64_t a1 = sdesc_sw128(st + 2048, 12288, 1024);      // dh =  0: rows 16..79
        const uint64_t a2 = sdesc_sw128(st + 4096, 12288, 1024);      // dh = +1: rows 32..95
        if (elect_one()) {
          const bool acc = kk > kb;
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 0 * 128, a0, b0, idesc, acc);
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 1 * 128, a1, b0, idesc, acc);
          mma_slab_at<0, 0, 2048, 2048, false>(tmem_base + 2 * 128, a2, b0, idesc, acc);
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == kWg128Stages) s = 0;
      }
      if (elect_one()) umma_commit(tfull);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int ci = (r >> 6) * 64 + (r & 63);  // atom = channel half
    int j = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++j) {
      const int dw = u % 3, z = u / 3;
      mbar_wait_backoff(tfull, j & 1);
      tc_fence_after();
      float* out = p.ws + (size_t)z * 128 * p.Mpad;
#pragma unroll 1
      for (int T = 0; T < 3; ++T) {
        const int tap = T * 3 + dw;  // (dh + 1) * 3 + (dw + 1)
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + T * 128 + c * 32, v);
          tmem_ld_wait();
          float* o = out + (size_t)(c * 32) * p.Mpad + tap * 128 + ci;
#pragma unroll
          for (int t = 0; t < 32; ++t) o[(size_t)t * p.Mpad] = __uint_as_float(v[t]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// split-K conv fold: y[m, :] = bf16(sum_z ws[z][m][:] (+ beta * y[m, :])) in split order, 8 channels per thread;
// with `stats`, also per-block channel partials [gridDim.x][2][N] (sum, sum of squares of the stored bf16 values)
// for the BatchNorm consuming y (nsk_bn_fwd_partials), as the conv epilogue would have written them.
constexpr int kFoldThreads = 256;
__global__ void __launch_bounds__(kFoldThreads) conv_split_fold_kernel(const float* __restrict__ ws, int splits, int M,
                                                                       int N, __nv_bfloat16* y, float beta, float* stats,
                                                                       const __nv_bfloat16* __restrict__ bx,
                                                                       const uint8_t* __restrict__ bmask) {
  pdl_wait();
  extern __shared__ float fold_red[];  // [RPB][N] (stats)
  const int CV = N / 8;
  const int cv = threadIdx.x % CV, ro = threadIdx.x / CV, RPB = kFoldThreads / CV;
  const long long plane = (long long)M * N;
  float s1[8] = {0}, s2[8] = {0};
  if (ro < RPB) {
    for (long long r = (long long)blockIdx.x * RPB + ro; r < M; r += (long long)gridDim.x * RPB) {
      const float* src = ws + r * N + cv * 8;
      float a[8];
      {
        const float4 u0 = __ldg((const float4*)src), u1 = __ldg((const float4*)(src + 4));
        a[0] = u0.x; a[1] = u0.y; a[2] = u0.z; a[3] = u0.w; a[4] = u1.x; a[5] = u1.y; a[6] = u1.z; a[7] = u1.w;
      }
      for (int z = 1; z < splits; ++z) {
        const float4 u0 = __ldg((const float4*)(src + z * plane)), u1 = __ldg((const float4*)(src + z * plane + 4));
        a[0] += u0.x; a[1] += u0.y; a[2] += u0.z; a[3] += u0.w; a[4] += u1.x; a[5] += u1.y; a[6] += u1.z; a[7] += u1.w;
      }
      uint4* dst = (uint4*)(y + r * N + cv * 8);
      uint4 v;
      v.x = pack_bf16x2(a[0], a[1]); v.y = pack_bf16x2(a[2], a[3]);
      v.z = pack_bf16x2(a[4], a[5]); v.w = pack_bf16x2(a[6], a[7]);
      if (beta != 0.f) v = bf16x8_axpby(*dst, beta, v);
      if (bmask) {  // BatchNorm-backward mode: dz = [y > 0] * g
        const unsigned m = bmask[(r * N + cv * 8) >> 3];
        uint32_t* v32 = (uint32_t*)&v;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          v32[i] &= (((m >> (2 * i)) & 1u) ? 0x0000ffffu : 0u) | (((m >> (2 * i + 1)) & 1u) ? 0xffff0000u : 0u);
      }
      *dst = v;
      if (stats && bx) {  // sum dz, sum dz * x (x = the BatchNorm input)
        float xv[8];
        {
          const uint4 xu = __ldg((const uint4*)(bx + r * N + cv * 8));
          const __nv_bfloat162* xh = (const __nv_bfloat162*)&xu;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 t = __bfloat1622float2(xh[i]);
            xv[2 * i] = t.x;
            xv[2 * i + 1] = t.y;
          }
        }
        const __nv_bfloat162* h = (const __nv_bfloat162*)&v;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          s1[2 * i] += f.x; s2[2 * i] += f.x * xv[2 * i];
          s1[2 * i + 1] += f.y; s2[2 * i + 1] += f.y * xv[2 * i + 1];
        }
      } else if (stats) {
        const __nv_bfloat162* h = (const __nv_bfloat162*)&v;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          s1[2 * i] += f.x; s2[2 * i] += f.x * f.x;
          s1[2 * i + 1] += f.y; s2[2 * i + 1] += f.y * f.y;
        }
      }
    }
  }
  if (!stats) return;
  for (int pass = 0; pass < 2; ++pass) {
    const float* sv = pass ? s2 : s1;
    if (ro < RPB)
#pragma unroll
      for (int j = 0; j < 8; ++j) fold_red[ro * N + cv * 8 + j] = sv[j];
    __syncthreads();
    for (int c = threadIdx.x; c < N; c += kFoldThreads) {
      float t = 0.f;
      for (int r = 0; r < RPB; ++r) t += fold_red[r * N + c];
      stats[(size_t)blockIdx.x * 2 * N + pass * N + c] = t;
    }
    __syncthreads();
  }
}

// split-K GEMM fold: C[m, n] = sum_z ws[z][m][n] (+ bias[n]) (+ beta * C[m, n]), fp32 or bf16 out
// 16-byte variant (N, ldc multiples of 4, aligned buffers): four columns per thread, the splits' loads all in
// flight, the same per-element summation order (split 0, 1, ...) -- bit-identical to the scalar fold
__global__ void splitk_fold4_kernel(const float* __restrict__ ws, int splits, int M, int N, void* C, long long ldc,
                                    int c_f32, const float* __restrict__ bias, float beta) {
  pdl_wait();
  const long long total = (long long)M * N, total4 = total / 4;
  const int N4 = N / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total4;
       i += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(i / N4), n = (int)(i - (long long)m * N4) * 4;
    float4 acc = __ldg((const float4*)ws + i);
    for (int z = 1; z < splits; ++z) {
      const float4 v = __ldg((const float4*)(ws + (long long)z * total) + i);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (bias) {
      const float4 b4 = __ldg((const float4*)(bias + n));
      acc.x += b4.x;
      acc.y += b4.y;
      acc.z += b4.z;
      acc.w += b4.w;
    }
    if (c_f32) {
      float4* o = (float4*)((float*)C + (long long)m * ldc + n);
      if (beta != 0.f) {
        const float4 old = *o;
        acc.x += beta * old.x;
        acc.y += beta * old.y;
        acc.z += beta * old.z;
        acc.w += beta * old.w;
      }
      *o = acc;
    } else {
      uint2 u;
      u.x = pack_bf16x2(acc.x, acc.y);
      u.y = pack_bf16x2(acc.z, acc.w);
      *(uint2*)((__nv_bfloat16*)C + (long long)m * ldc + n) = u;
    }
  }
}

__global__ void splitk_fold_kernel(const float* __restrict__ ws, int splits, int M, int N, void* C, long long ldc,
                                   int c_f32, const float* __restrict__ bias, float beta) {
  pdl_wait();
  const long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(i / N), n = (int)(i - (long long)m * N);
    float acc = 0.f;
    for (int z = 0; z < splits; ++z) acc += ws[(long long)z * total + i];
    if (bias) acc += bias[n];
    if (c_f32) {
      float* o = (float*)C + (long long)m * ldc + n;
      *o = beta != 0.f ? acc + beta * *o : acc;
    } else {
      ((__nv_bfloat16*)C)[(long long)m * ldc + n] = __float2bfloat16_rn(acc);
    }
  }
}

// Library-owned grow-only scratch for split-K partials, one buffer per launching stream: split-K problems
// issued concurrently on the compute stream and a side stream never share partials. Grows only outside
// stream capture (the first, eager execution of a captured step sizes it); an outgrown buffer is freed
// after a device-wide synchronize, since kernels on any stream may still read it.
int gemm_scratch(size_t floats, cudaStream_t st, float** out) {
  struct Slot { float* buf = nullptr; size_t cap = 0; };
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, Slot> slots;
  std::lock_guard<std::mutex> lk(mu);
  Slot& s = slots[st];
  if (floats > s.cap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone)
      return nsk::set_error(NSK_ERR_UNSUPPORTED, "gemm: split-K scratch must be sized before graph capture");
    if (s.buf) {
      cudaDeviceSynchronize();
      cudaFree(s.buf);
    }
    size_t want = floats < (1u << 20) ? (1u << 20) : floats;
    if (cudaMalloc(&s.buf, want * sizeof(float)) != cudaSuccess) {
      cudaGetLastError();
      s.buf = nullptr;
      s.cap = 0;
      return nsk::set_error(NSK_ERR_OOM, "out of memory: gemm split-K scratch");
    }
    s.cap = want;
  }
  *out = s.buf;
  return NSK_OK;
}

int g_wgrad_grid_cap = 0;  // CTAs per wgrad launch (0: two per SM as usual)

// dynamic shared memory past Smem::TOTAL: statistics accumulators [2][N] + per-warpgroup reduction slots, and
// for the BatchNorm-backward statistics a staging block of the BatchNorm input per epilogue warp
// dynamic shared memory past Smem::TOTAL: the statistics' per-warp column sums [epi warps][2][columns per warp], or
// with stats_shared one [2][N] CTA accumulator + per-warpgroup combine slots [4][2][32]
int epi_extra_smem(const UmmaProb& p, int epi) {
  if (!p.stats) return 0;
  if (p.stats_shared) return (2 * p.N + epi * 64) * (int)sizeof(float);
  const int g = epi / 4;
  return epi * 2 * ((p.N / 32 + g - 1) / g * 32) * (int)sizeof(float);
}

template <int BN, int ESZ, int STAGES, bool RR = false, int EPI = 4, bool WRES = false, int STATS = 0>
int launch_umma(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, UmmaProb p, cudaStream_t st,
                int* grid_out) {
  using S = Smem<BN, ESZ, STAGES, RR, EPI, WRES>;
  auto kern = umma_kernel<BN, ESZ, STAGES, RR, EPI, WRES, STATS>;
  const int smem = S::TOTAL + epi_extra_smem(p, EPI) + (STATS == 3 ? 512 : 0);
  if (smem > 227 * 1024) return nsk::set_error(NSK_ERR_UNSUPPORTED, "umma: shared memory budget exceeded");
  static int configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return nsk::cuda_status(e, "cudaFuncSetAttribute(umma)");
    configured = smem;
  }
  const int per_sm = (2 * smem <= 227 * 1024) ? 2 : 1;  // small-N tiles: two co-resident CTAs per SM
  int grid = per_sm * nsk::sm_count();
  if (p.mode == MODE_WGRAD) {  // weight gradients beside the compute stream: leave it SMs (nsk_wgrad_grid_cap)
    int cap = g_wgrad_grid_cap;
    if (const char* e = getenv("NSK_WGRAD_GRID")) cap = atoi(e);
    if (cap > 0 && cap < grid) grid = cap;
  }
  if (p.mc) {  // CTA pairs (2-CTA clusters) walking pair units
    if (grid > 2 * p.units) grid = 2 * p.units;
    grid &= ~1;
    if (grid < 2) grid = 2;
    if (grid_out) *grid_out = grid;
    nsk::launch_pdl_cluster(kern, grid, Launch<S>::template threads<EPI>(), smem, st, 2, a, b, c, p);
    NSK_LAUNCH_CHECK("umma_kernel (pair multicast)");
    return NSK_OK;
  }
  if (grid > p.units) grid = p.units;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = grid;
  nsk::launch_pdl(kern, grid, Launch<S>::template threads<EPI>(), smem, st, a, b, c, p);
  NSK_LAUNCH_CHECK("umma_kernel");
  return NSK_OK;
}

// STATS: 0 none, 1 forward BatchNorm statistics, 2 BatchNorm-backward statistics, 3 fp32-output GEMM (staged
// coalesced stores; 256-wide tiles only, everything else falls back to 0)
template <int ESZ, int STATS>
int dispatch_bn_main(int BN, const CUtensorMap& a, const CUtensorMap& b, UmmaProb p, int mt, int nt, int nz,
                     cudaStream_t st, int* grid_out, const CUtensorMap* cmap) {
  static CUtensorMap dummy{};
  const CUtensorMap& c = cmap ? *cmap : dummy;
  if (!cmap) p.tma_store = 0;
  p.mt = p.mc ? (mt + 1) / 2 : mt;  // pair multicast: units are pairs of M tiles
  p.nt = nt;
  p.units = p.mt * nt * nz;
  if (p.rr) {
    if constexpr (ESZ == 2) {
      switch (BN) {  // rr stages carry 3 taps of B: one CTA per SM, ~190-220 KB of ring
        case 64: {
          // one 64-channel chunk, N = 64, 3x3 in strided tap boxes: keep all 9 taps resident (the ring then
          // moves only A; re-fetching the 72 KB filter per tile was half the L2->smem traffic)
          if (p.wres && nt == 1 && nz == 1) return launch_umma<64, 2, 4, true, 8, true, STATS>(a, b, c, p, st, grid_out);
          if (p.wres) return nsk::set_error(NSK_ERR_UNSUPPORTED, "weight-resident conv needs a single 64-wide tile");
          return launch_umma<64, 2, 2, true, 4, false, STATS>(a, b, c, p, st, grid_out);
        }
        case 128:
          return launch_umma<128, 2, 2, true, 4, false, STATS>(a, b, c, p, st, grid_out);
      }
    }
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "row-reuse conv needs bf16 and N <= 128");
  }
  switch (BN) {  // ~192 KB of smem ring per CTA, one persistent CTA per SM
    case 64:
      return launch_umma<64, ESZ, 4, false, 4, false, STATS>(a, b, c, p, st, grid_out);
    case 128:
      return launch_umma<128, ESZ, 3, false, 4, false, STATS>(a, b, c, p, st, grid_out);
    case 256: {
      // 8 epilogue warps unless the statistics buffers would not fit beside them
      using S8 = Smem<256, ESZ, 4, false, 8>;
      const int need = S8::TOTAL + epi_extra_smem(p, 8);
      // 8 epilogue warps pay on store-bound passes (large M, or short-K expands to >= 1024 channels: ResNet-50's
      // 1x1 layers); the long-K ResNet-18 layers (M <= 16k) measured 0.9 % faster per step with 4. NSK_EPI8=0/1 forces
      const char* e8 = getenv("NSK_EPI8");
      const bool store_bound = p.M >= (1 << 15) || (p.k_steps <= 16 && p.N >= 1024);
      const bool epi8 = e8 ? e8[0] != '0' : store_bound;
      if (need <= 227 * 1024 && epi8)
        return launch_umma<256, ESZ, 4, false, 8, false, STATS>(a, b, c, p, st, grid_out);
      if constexpr (STATS == 1) {
        // the statistics do not fit beside four stages: the store-bound layers (large M, or ResNet-50's short-K
        // 1x1 expands to >= 1024 channels) keep the 8-warp epilogue with three stages (R50 9.85k -> 10.24k
        // img/s); ResNet-18's small 8x8 layers measure 0.15 % faster on the deeper 4-warp ring
        if (epi8 && store_bound && !(getenv("NSK_STATS_S3") && getenv("NSK_STATS_S3")[0] == '0'))
          return launch_umma<256, ESZ, 3, false, 8, false, STATS>(a, b, c, p, st, grid_out);
      }
      return launch_umma<256, ESZ, 4, false, 4, false, STATS>(a, b, c, p, st, grid_out);
    }
  }
  return nsk::set_error(NSK_ERR_UNSUPPORTED, "unsupported BN");
}

template <int ESZ, int STATS = 0>
int dispatch_bn(int BN, const CUtensorMap& a, const CUtensorMap& b, UmmaProb p, int mt, int nt, int nz,
                cudaStream_t st, int* grid_out = nullptr, const CUtensorMap* cmap = nullptr) {
  if constexpr (STATS == 3) {
    if (p.rr || p.mc || BN != 256 || !p.out_f32) {
      if (p.out_f32) p.tma_store = 0;  // an fp32 store map is only read by this instantiation
      return dispatch_bn_main<ESZ, 0>(BN, a, b, p, mt, nt, nz, st, grid_out, p.out_f32 ? nullptr : cmap);
    }
    static CUtensorMap dummy{};
    const CUtensorMap& c = cmap ? *cmap : dummy;
    if (!cmap) p.tma_store = 0;
    p.mt = mt;
    p.nt = nt;
    p.units = mt * nt * nz;
    return launch_umma<256, ESZ, 4, false, 8, false, 3>(a, b, c, p, st, grid_out);
  } else {
    return dispatch_bn_main<ESZ, STATS>(BN, a, b, p, mt, nt, nz, st, grid_out, cmap);
  }
}

// CTA-pair multicast of B for the 256-wide conv tiles: opt-in (NSK_MC=1). Measured on B200 it halves each CTA's
// filter traffic but is 5 % slower on the 8x8 and 4x4 layers (19.5 -> 20.6 us, 26.7 -> 28.0 us): those passes are
// not L2-bandwidth bound, and the pair's shared stage release couples the two CTAs' pipelines.
bool mc_ok(int BN, int mt) {
  const char* e = getenv("NSK_MC");
  return e && e[0] == '1' && BN == 256 && mt >= 2;
}

int pick_bn(int N) {
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  return 256;
}

// conv tiles: the widest N tile that still gives every SM a work unit (small late-stage grids
// otherwise leave most of the 148 SMs idle: 4x4x512 at B=256 is only 32 M tiles)
int pick_bn_units(int N, int m_tiles, int classes) {
  if (const char* e = getenv("NSK_CONV_BN")) {  // experiment: force the conv N tile
    const int f = atoi(e);
    if ((f == 64 || f == 128 || f == 256) && f <= pick_bn(N)) return f;
  }
  int bn = pick_bn(N);
  while (bn > 64 && 2 * m_tiles * classes * ((N + bn - 1) / bn) < nsk::sm_count()) bn /= 2;
  return bn;
}

// pixel tile (Wt, Ht, Nt) covering `rows` consecutive output pixels in (n,h,w) raster order
bool pixel_tile(int Wo, int Ho, int rows, int* Wt, int* Ht, int* Nt) {
  if (Wo > rows || rows % Wo != 0) return false;
  int per = rows / Wo;
  if (per <= Ho) {
    if (Ho % per != 0) return false;
    *Wt = Wo;
    *Ht = per;
    *Nt = 1;
  } else {
    if (per % Ho != 0) return false;
    *Wt = Wo;
    *Ht = Ho;
    *Nt = per / Ho;
  }
  return true;
}

int nhwc_map(CUtensorMap* m, const void* ptr, int N, int H, int W, int C, int c_box, int Wt, int Ht, int Nt, int cs) {
  uint64_t dims[4] = {(uint64_t)C, (uint64_t)W, (uint64_t)H, (uint64_t)N};
  uint64_t strides[3] = {(uint64_t)C * 2, (uint64_t)W * C * 2, (uint64_t)H * W * C * 2};
  uint32_t box[4] = {(uint32_t)c_box, (uint32_t)(Wt * cs), (uint32_t)(Ht * cs), (uint32_t)Nt};
  uint32_t es[4] = {1, (uint32_t)cs, (uint32_t)cs, 1};
  return nsk::encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, ptr, dims, strides, box, es,
                          CU_TENSOR_MAP_SWIZZLE_128B);
}

// Switch a single-class stride-1 conv gather to the row-reuse schedule when the tile shape allows it:
// group class-0 taps by column offset, one A box of Ht + (dh range) rows per group. `act` is the
// gathered NHWC tensor [N, Hin, Win, Cin].
bool try_rowreuse(UmmaProb& p, CUtensorMap* ma, const void* act, int N, int Hin, int Win, int Cin, int BN) {
  const char* env = getenv("NSK_CONV_RR");
  if (env && env[0] == '0') return false;
  // default: N=64 tiles (2 CTAs/SM). NSK_CONV_RR=1 adds the 128-wide ones: 0.3 % faster per step on the round-2
  // kernels, but it reorders their fp32 accumulation over taps, and the lr-0.1 C2 trajectory test (chaotic after its
  // blow-up) then leaves its 1 % bar in one window -- not worth it
  if (BN != 64 && !(env && env[0] == '1')) return false;
  if (p.cs != 1 || p.Nt != 1 || p.Wt != p.Wo || (p.Wo % 8) || BN > 128 || p.ntaps[0] < 1) return false;
  int dhmin = 127, dhmax = -128;
  for (int t = 0; t < p.ntaps[0]; ++t) {
    dhmin = p.tdh[0][t] < dhmin ? p.tdh[0][t] : dhmin;
    dhmax = p.tdh[0][t] > dhmax ? p.tdh[0][t] : dhmax;
  }
  const int ext = p.Ht + dhmax - dhmin;
  if (ext * p.Wt * 128 > kRRMaxA || ext > 256) return false;
  int ng = 0;
  for (int t = 0; t < p.ntaps[0]; ++t) {
    int g = 0;
    while (g < ng && p.gdw[0][g] != p.tdw[0][t]) ++g;
    if (g == ng) {
      p.gdw[0][g] = p.tdw[0][t];
      p.gdhmin[0][g] = (signed char)dhmin;
      p.gnt[0][g] = 0;
      ++ng;
    }
    if (p.gnt[0][g] >= 3) return false;
    p.gdh[0][g][p.gnt[0][g]] = p.tdh[0][t];
    p.gw[0][g][p.gnt[0][g]] = p.tw[0][t];
    ++p.gnt[0][g];
  }
  if (nhwc_map(ma, act, N, Hin, Win, Cin, 64, p.Wt, ext, 1, 1)) return false;
  p.ngroups[0] = ng;
  p.ext_rows = ext;
  p.rr = 1;
  return true;
}

// im2col-mode A map for a gather over `act` [N, Hin, Win, Cin]: an output grid Gh x Gw walked with
// coordinate stride p.cs, taps of every class in p.tdh/p.tdw. The bounding box starts at the smallest tap
// offset (TMA im2col offsets are unsigned) and is sized so it holds exactly Gh x Gw positions per image.
int i2c_map(UmmaProb& p, CUtensorMap* m, const void* act, int N, int Hin, int Win, int Cin, int Gh, int Gw, int ncls,
            int pixels) {
  int mh = 127, mw = 127;
  for (int c = 0; c < ncls; ++c)
    for (int t = 0; t < p.ntaps[c]; ++t) {
      mh = p.tdh[c][t] < mh ? p.tdh[c][t] : mh;
      mw = p.tdw[c][t] < mw ? p.tdw[c][t] : mw;
    }
  if (mh == 127) mh = mw = 0;
  const int lower[2] = {mw, mh};
  const int upper[2] = {mw + (Gw - 1) * p.cs - (Win - 1), mh + (Gh - 1) * p.cs - (Hin - 1)};
  int rc = nsk::encode_tmap_im2col(m, act, N, Hin, Win, Cin, lower, upper, pixels, p.cs);
  if (rc) return rc;
  p.i2c = 1;
  p.lw = mw;
  p.lh = mh;
  return NSK_OK;
}

// TMA-store map of a bf16 [M, N] output with row pitch ldc: 32 x 32 boxes (one epilogue warp's chunk)
bool out_map(CUtensorMap* m, void* out, long long M, int N, long long ldc) {
  if (N % 32 || (ldc * 2) % 16 || ((uintptr_t)out & 15)) return false;
  const char* env = getenv("NSK_TMA_STORE");
  if (env && env[0] == '0') return false;
  uint64_t dims[2] = {(uint64_t)N, (uint64_t)M};
  uint64_t str[1] = {(uint64_t)ldc * 2};
  uint32_t box[2] = {32, 32};
  return nsk::encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, str, box, nullptr,
                          CU_TENSOR_MAP_SWIZZLE_64B) == NSK_OK;  // matches the staging layout (stg_off)
}

// fp32 output (or split-K partials [splits][M][N]) for the staged STATS 3 epilogue: 32 x 32 boxes, 128-byte swizzle
bool out_map_f32(CUtensorMap* m, void* out, long long M, int N, long long ldc, int splits) {
  if ((ldc * 4) % 16 || ((uintptr_t)out & 15)) return false;
  const char* env = getenv("NSK_TMA_STORE_F32");
  if (env && env[0] == '0') return false;
  uint64_t dims[3] = {(uint64_t)N, (uint64_t)M, (uint64_t)splits};
  uint64_t str[2] = {(uint64_t)ldc * 4, (uint64_t)M * ldc * 4};
  uint32_t box[3] = {32, 32, 1};
  return nsk::encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, str, box, nullptr,
                          CU_TENSOR_MAP_SWIZZLE_128B) == NSK_OK;
}

bool force_i2c() {
  const char* env = getenv("NSK_CONV_I2C");
  return env && env[0] == '1';
}

// Row-reuse 3x3: every column group holds taps (dh -1, 0, +1) = filter taps tw, tw+3, tw+6, so the group's B
// tiles are ONE strided 3-D box {64 channels, 64|BN rows, 3 taps (element stride 3)} over the KRSC filter
// viewed as {C, K, R*S} -- one TMA op instead of three.
void try_rr3(UmmaProb& p, CUtensorMap* mb, const NskConvDesc* d, const void* w, int BN, int mode) {
  bool three = d->R == 3 && d->S == 3 && p.ngroups[0] == 3;
  for (int g = 0; three && g < 3; ++g)
    three = p.gnt[0][g] == 3 && p.gw[0][g][1] == p.gw[0][g][0] + 3 && p.gw[0][g][2] == p.gw[0][g][0] + 6;
  const char* env = getenv("NSK_RR3");
  if (!three || (env && env[0] == '0')) return;
  const int RS = d->R * d->S;
  uint64_t dims[3] = {(uint64_t)d->C, (uint64_t)d->K, (uint64_t)RS};
  uint64_t str[2] = {(uint64_t)RS * d->C * 2, (uint64_t)d->C * 2};
  uint32_t box[3] = {64, (uint32_t)(mode == BMODE_RR3 ? BN : 64), 9};  // span 9, stride 3 -> 3 taps loaded
  uint32_t es[3] = {1, 1, 3};
  CUtensorMap m;
  if (nsk::encode_tmap(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w, dims, str, box, es, CU_TENSOR_MAP_SWIZZLE_128B) ==
      NSK_OK) {
    *mb = m;
    p.bmode = mode;
    if (p.Wt == 32) {
      bool asc = true, desc = true;
      for (int g = 0; g < 3; ++g)
        for (int t = 0; t < 3; ++t) {
          asc = asc && p.gdh[0][g][t] - p.gdhmin[0][g] == t;
          desc = desc && p.gdh[0][g][t] - p.gdhmin[0][g] == 2 - t;
        }
      const char* ef = getenv("NSK_RR_FAST");
      if (!(ef && ef[0] == '0'))
        p.rr_fast = asc ? (mode == BMODE_RR3 ? 1 : 2) : (desc ? (mode == BMODE_RR3 ? 4 : 3) : 0);
    }
  }
}

// Weight-resident row-reuse (Smem WRES): a 3x3 over one 64-channel chunk with 64 outputs whose taps come in
// strided boxes. The A map is re-encoded as row bands so the three producer warps each keep a box in flight
// per stage (one 4-D box per issuing thread is latency-bound at ~15 B/clk/SM, tools/tma_rate.cu).
void try_wres(UmmaProb& p, CUtensorMap* ma, const void* act, int N, int Hin, int Win, int Cin, int Nout) {
  const char* env = getenv("NSK_WRES");
  if (env && env[0] == '0') return;
  if (!(p.bmode == BMODE_RR3 || p.bmode == BMODE_RR3T) || p.cchunks != 1 || Nout != 64 || p.ngroups[0] != 3) return;
  // A box per stage: one band (default) or split into 3 row bands, one per producer warp (NSK_ASPLIT=3; round 1's
  // choice, now measured 0.6 % slower per step than one box)
  const char* es = getenv("NSK_ASPLIT");
  int split = es ? atoi(es) : 1;
  if (split != 3 || p.ext_rows % 3) split = 1;
  if (split > 1 && nhwc_map(ma, act, N, Hin, Win, Cin, 64, p.Wt, p.ext_rows / split, 1, 1)) split = 1;
  p.asplit = split;
  p.wres = 1;
}

// Few output tiles over a long reduction (the 4x4 and 7x7 layers: 32 m-tiles x 512 channels): 256-wide tiles,
// whose 128x256 MMAs read 25 % less shared memory per flop than 64-wide ones, with the K range split across work
// units so every SM still has one -- fp32 partials in the library scratch, folded in split order
// (conv_split_fold_kernel). Returns the split count (1: no split). NSK_CONV_SPLIT=0 disables.
int conv_splits(int m_tiles, int N, int k_steps) {
  const char* e = getenv("NSK_CONV_SPLIT");
  if (e && e[0] == '0') return 1;
  if (N < 256 || N % 256 || N > 2048) return 1;
  const int units = m_tiles * (N / 256);
  if (units >= nsk::sm_count() || k_steps < 64) return 1;  // 8x8 256->512 s2 (36 k-steps): 17.3 -> 19.7 us split
  int splits = nsk::sm_count() / units;
  if (e && atoi(e) > 1) splits = atoi(e);  // experiment: forced split count
  if (splits > k_steps / 16) splits = k_steps / 16;
  return splits < 2 ? 1 : splits;
}

// launch the split-K conv and its fold into the bf16 output (beta: accumulate; stats: BN partials, nparts out)
int conv_split_run(UmmaProb p, const CUtensorMap& ma, const CUtensorMap& mb, int splits, int k_steps, void* out,
                   float beta, float* stats, int* nparts, cudaStream_t st) {
  const int M = p.M, N = p.N;
  const int per = (k_steps + splits - 1) / splits;
  splits = (k_steps + per - 1) / per;
  float* ws = nullptr;
  int rc = gemm_scratch((size_t)splits * M * N, st, &ws);
  if (rc) return rc;
  p.k_steps = k_steps;
  p.k_per_split = per;
  p.out = ws;
  p.ldc = N;
  p.out_f32 = 1;
  p.beta = 0.f;
  p.tma_store = 0;
  p.stats = nullptr;
  p.rr = 0;
  const __nv_bfloat16* bx = p.bx;
  const uint8_t* bmask = p.bmask;
  p.bx = nullptr;
  p.bmask = nullptr;
  p.bacc = 0;
  const bool staged = !(getenv("NSK_SPLIT_STAGED") && getenv("NSK_SPLIT_STAGED")[0] == '0');
  CUtensorMap mw;
  const bool tw = staged && out_map_f32(&mw, ws, M, N, N, splits);
  p.tma_store = tw;
  if ((rc = staged ? dispatch_bn<2, 3>(256, ma, mb, p, (M + 127) / 128, N / 256, splits, st, nullptr, tw ? &mw : nullptr)
                   : dispatch_bn<2>(256, ma, mb, p, (M + 127) / 128, N / 256, splits, st)))
    return rc;
  const int CV = N / 8, RPB = kFoldThreads / CV;
  unsigned grid = (unsigned)((M + RPB - 1) / RPB);
  if (stats && grid > (unsigned)(2 * nsk::sm_count())) grid = 2 * nsk::sm_count();
  if (!stats && grid > (unsigned)(16 * nsk::sm_count())) grid = 16 * nsk::sm_count();
  const size_t smem = stats ? (size_t)RPB * N * sizeof(float) : 0;
  nsk::launch_pdl(conv_split_fold_kernel, grid, kFoldThreads, smem, st, (const float*)ws, splits, M, N,
                  (__nv_bfloat16*)out, beta, stats, bx, bmask);
  NSK_LAUNCH_CHECK("conv_split_fold_kernel");
  if (nparts) *nparts = (int)grid;
  return NSK_OK;
}

bool wgrad_rr128_ok(const NskConvDesc* d) {
  const char* e = getenv("NSK_WGRAD_RR");
  if (e && (e[0] == '0' || e[0] == '1')) return e[0] != '0' && e[1] != '6';  // "64": the 64-channel path only
  return d->C == 128 && d->K == 128 && d->R == 3 && d->S == 3 && d->stride == 1 && d->pad == 1 && d->W == 16 &&
         d->Q == 16 && d->H == d->P && d->H % 4 == 0 && ((long long)d->N * d->P * d->Q) % 64 == 0;
}

bool wgrad_rr64_ok(const NskConvDesc* d) {
  const char* e = getenv("NSK_WGRAD_RR");
  if (e && e[0] == '0') return false;
  return d->C == 64 && d->K == 64 && d->R == 3 && d->S == 3 && d->stride == 1 && d->pad == 1 && d->W == 32 &&
         d->Q == 32 && d->H == d->P && d->H % 2 == 0 && ((long long)d->N * d->P * d->Q) % 64 == 0;
}

int check_desc(const NskConvDesc* d) {
  if (d->N < 1 || d->H < 1 || d->W < 1 || d->C < 1 || d->K < 1 || d->R < 1 || d->S < 1 || d->stride < 1)
    return nsk::set_error(NSK_ERR_SHAPE, "conv2d: invalid descriptor");
  if (d->R * d->S > kMaxTaps) return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d: filter larger than 3x3");
  if (d->C % 64 != 0 || d->K % 64 != 0)
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d: channel counts must be multiples of 64 (pad the stem)");
  return NSK_OK;
}

}  // namespace

extern "C" {

int nsk_gemm(int dtype, int a_mn, int b_mn, int M, int N, int K, const void* A, long long lda, const void* B,
             long long ldb, void* C, long long ldc, int c_f32, const float* bias, float beta, void* stream) {
  if (M < 1 || N < 1 || K < 1) return nsk::set_error(NSK_ERR_SHAPE, "gemm: empty problem");
  const int esz = dtype == NSK_DTYPE_BF16 ? 2 : 4;
  if ((lda * esz) % 16 || (ldb * esz) % 16 || ((uintptr_t)A % 16) || ((uintptr_t)B % 16))
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "gemm: operands must be 16-byte aligned with 16-byte row pitch");
  if (beta != 0.f && !c_f32) return nsk::set_error(NSK_ERR_UNSUPPORTED, "gemm: beta needs an fp32 output");
  const int KE = 128 / esz;
  const int BN = pick_bn(N);
  CUtensorMapDataType dt = esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap ma, mb;
  int rc;
  {
    uint64_t dims[2], str[1];
    uint32_t box[2];
    if (!a_mn) {
      dims[0] = K; dims[1] = M; box[0] = KE; box[1] = 128;
    } else {
      dims[0] = M; dims[1] = K; box[0] = KE; box[1] = KE;
    }
    str[0] = (uint64_t)lda * esz;
    if ((rc = nsk::encode_tmap(&ma, dt, 2, A, dims, str, box, nullptr, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if (!b_mn) {
      dims[0] = K; dims[1] = N; box[0] = KE; box[1] = BN;
    } else {
      dims[0] = N; dims[1] = K; box[0] = KE; box[1] = KE;
    }
    str[0] = (uint64_t)ldb * esz;
    if ((rc = nsk::encode_tmap(&mb, dt, 2, B, dims, str, box, nullptr, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  }
  UmmaProb p{};
  p.mode = MODE_GEMM;
  p.a_mn = a_mn;
  p.b_mn = b_mn;
  p.M = M;
  p.N = N;
  p.k_steps = (K + KE - 1) / KE;
  p.out = C;
  p.ldc = ldc;
  p.out_f32 = c_f32;
  p.bias = bias;
  p.beta = beta;
  const int mt = (M + 127) / 128, nt = (N + BN - 1) / BN;
  if (const char* pr = getenv("NSK_PROBE")) p.probe = atoi(pr);
  // Few output tiles but a long K (e.g. the stem's weight gradient, K = all pixels): split K across
  // work units, fp32 partials in a library scratch, fixed-order fold (deterministic).
  int splits = 1;
  if (mt * nt * 2 <= nsk::sm_count() && p.k_steps >= 16) {
    splits = nsk::sm_count() / (mt * nt);
    if (splits > p.k_steps / 8) splits = p.k_steps / 8;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (splits > 1) {
    const int per = (p.k_steps + splits - 1) / splits;
    splits = (p.k_steps + per - 1) / per;
    float* ws = nullptr;
    if ((rc = gemm_scratch((size_t)splits * M * N, st, &ws))) return rc;
    p.k_per_split = per;
    p.out = ws;
    p.ldc = N;
    p.out_f32 = 1;
    p.bias = nullptr;
    p.beta = 0.f;
    CUtensorMap mw;
    const bool tw = out_map_f32(&mw, ws, M, N, N, splits);
    p.tma_store = tw;
    rc = esz == 2 ? dispatch_bn<2, 3>(BN, ma, mb, p, mt, nt, splits, st, nullptr, tw ? &mw : nullptr)
                  : dispatch_bn<4, 3>(BN, ma, mb, p, mt, nt, splits, st, nullptr, tw ? &mw : nullptr);
    if (rc) return rc;
    const long long total = (long long)M * N;
    const bool vec = N % 4 == 0 && ldc % 4 == 0 && ((uintptr_t)C & 15) == 0 && (!bias || ((uintptr_t)bias & 15) == 0);
    if (vec)
      nsk::launch_pdl(splitk_fold4_kernel, nsk::grid_for(total / 4, 256), 256, 0, st, ws, splits, M, N, C, ldc, c_f32,
                      bias, beta);
    else
      nsk::launch_pdl(splitk_fold_kernel, nsk::grid_for(total, 256), 256, 0, st, ws, splits, M, N, C, ldc, c_f32,
                      bias, beta);
    NSK_LAUNCH_CHECK("splitk_fold_kernel");
    return NSK_OK;
  }
  CUtensorMap mc;
  const bool ts = beta == 0.f && (c_f32 ? out_map_f32(&mc, C, M, N, ldc, 1) : out_map(&mc, C, M, N, ldc));
  p.tma_store = ts;
  if (esz == 2) return dispatch_bn<2, 3>(BN, ma, mb, p, mt, nt, 1, st, nullptr, ts ? &mc : nullptr);
  return dispatch_bn<4, 3>(BN, ma, mb, p, mt, nt, 1, st, nullptr, ts ? &mc : nullptr);
}

}  // extern "C"

namespace {

int conv_fprop(const NskConvDesc* d, const void* x, const void* w, void* y, int y_f32, float* stats,
               uint64_t stats_floats, int* nparts, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  const int P = d->P, Q = d->Q;
  int Wt = 0, Ht = 0, Nt = 0;
  const bool i2c = !pixel_tile(Q, P, 128, &Wt, &Ht, &Nt) || force_i2c();
  const int fsteps = d->R * d->S * (d->C / 64);
  const int splits = y_f32 ? 1 : conv_splits((d->N * P * Q + 127) / 128, d->K, fsteps);
  const int BN = splits > 1 ? 256 : pick_bn_units(d->K, (d->N * P * Q + 127) / 128, 1);
  CUtensorMap ma, mb;
  if (!i2c && (rc = nhwc_map(&ma, x, d->N, d->H, d->W, d->C, 64, Wt, Ht, Nt, d->stride))) return rc;
  const bool pair_mc = !y_f32 && mc_ok(BN, (d->N * P * Q + 127) / 128);
  {
    const int RS = d->R * d->S;
    uint64_t dims[2] = {(uint64_t)RS * d->C, (uint64_t)d->K};
    uint64_t str[1] = {(uint64_t)RS * d->C * 2};
    uint32_t box[2] = {64, (uint32_t)(pair_mc ? BN / 2 : BN)};  // pair multicast: each CTA loads half the rows
    if ((rc = nsk::encode_tmap(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, nullptr,
                               CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
  }
  UmmaProb p{};
  p.mode = MODE_CONV;
  p.bmode = BMODE_2D;
  p.M = d->N * P * Q;
  p.N = d->K;
  p.Wt = Wt; p.Ht = Ht; p.Nt = Nt;
  p.Wo = Q; p.Ho = P;
  p.cs = d->stride;
  p.cchunks = d->C / 64;
  int t = 0;
  for (int r = 0; r < d->R; ++r)
    for (int s = 0; s < d->S; ++s, ++t) {
      p.tdh[0][t] = (signed char)(r - d->pad);
      p.tdw[0][t] = (signed char)(s - d->pad);
      p.tw[0][t] = (signed char)t;
    }
  p.ntaps[0] = t;
  p.os = 1; p.Hd = P; p.Wd = Q;
  p.out = y;
  p.ldc = d->K;
  p.out_f32 = y_f32;
  p.mc = pair_mc;
  if (i2c) {
    if ((rc = i2c_map(p, &ma, x, d->N, d->H, d->W, d->C, P, Q, 1, 128))) return rc;
  } else if (splits == 1 && try_rowreuse(p, &ma, x, d->N, d->H, d->W, d->C, BN)) {
    try_rr3(p, &mb, d, w, BN, BMODE_RR3);
    try_wres(p, &ma, x, d->N, d->H, d->W, d->C, d->K);
  }
  if (const char* pr = getenv("NSK_PROBE")) p.probe = atoi(pr);
  if (stats) {
    if (y_f32) return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d fprop: channel statistics need a bf16 output");
    if (stats_floats < (uint64_t)2 * nsk::sm_count() * 2 * d->K)
      return nsk::set_error(NSK_ERR_SHAPE, "conv2d fprop: statistics buffer smaller than 2*SMs x 2 x K floats");
    p.stats = stats;
    p.fold_reset = nsk::bn_fold_counter_fwd((cudaStream_t)stream);
    p.stats_shared = 32 * d->K > 8192;  // per-warp accumulators cost 32 B per channel: wide layers share one
  }
  if (splits > 1) return conv_split_run(p, ma, mb, splits, fsteps, y, 0.f, stats, nparts, (cudaStream_t)stream);
  CUtensorMap mc;
  const bool ts = !y_f32 && out_map(&mc, y, p.M, d->K, d->K);
  p.tma_store = ts;
  if (stats)
    return dispatch_bn<2, 1>(BN, ma, mb, p, (p.M + 127) / 128, (d->K + BN - 1) / BN, 1, (cudaStream_t)stream, nparts,
                             ts ? &mc : nullptr);
  return dispatch_bn<2>(BN, ma, mb, p, (p.M + 127) / 128, (d->K + BN - 1) / BN, 1, (cudaStream_t)stream, nparts,
                        ts ? &mc : nullptr);
}

int conv_dgrad(const NskConvDesc* d, const void* dy, const void* w, void* dx, float beta, const __nv_bfloat16* bx,
               const uint8_t* bmask, float* stats, uint64_t stats_floats, int* nparts, void* stream);

}  // namespace

extern "C" {

// y[n,p,q,k] = sum_{c,r,s} x[n, p*st-pad+r, q*st-pad+s, c] * w[k,r,s,c]   (NHWC / KRSC, bf16)
int nsk_conv2d_fprop(const NskConvDesc* d, const void* x, const void* w, void* y, int y_f32, void* stream) {
  return conv_fprop(d, x, w, y, y_f32, nullptr, 0, nullptr, stream);
}

// fprop that also emits per-CTA channel partials for the BatchNorm consuming y (nsk_bn_fwd_partials)
int nsk_conv2d_fprop_stats(const NskConvDesc* d, const void* x, const void* w, void* y, float* partials,
                           uint64_t partial_floats, int* nparts, void* stream) {
  return conv_fprop(d, x, w, y, 0, partials, partial_floats, nparts, stream);
}

// dx[n,h,w,c] = sum_{k,r,s : h = p*st-pad+r} dy[n,p,q,k] * w[k,r,s,c]
// stride 1: one launch over all taps; stride 2: four output-parity classes
// (blockIdx.z), each a stride-1 gather over dy with its subset of taps.
int nsk_conv2d_dgrad(const NskConvDesc* d, const void* dy, const void* w, void* dx, void* stream) {
  return nsk_conv2d_dgrad_acc(d, dy, w, dx, 0.f, stream);
}

// dx = dgrad + beta * dx (bf16 in place): a second gradient contribution accumulated in the epilogue
int nsk_conv2d_dgrad_acc(const NskConvDesc* d, const void* dy, const void* w, void* dx, float beta, void* stream) {
  return conv_dgrad(d, dy, w, dx, beta, nullptr, nullptr, nullptr, 0, nullptr, stream);
}

// dgrad whose result is the gradient of a BatchNorm's output (the last contribution to it): stores
// dz = relu_mask * (dgrad + beta * dx) and per-CTA partials [nparts][2][C] of sum dz and sum dz * bn_x for
// nsk_bn_bwd_partials (no reduction pass over dz and x)
int nsk_conv2d_dgrad_bnstats(const NskConvDesc* d, const void* dy, const void* w, void* dx, float beta,
                             const void* bn_x, const void* relu_mask, float* partials, uint64_t partial_floats,
                             int* nparts, void* stream) {
  if (!bn_x || !partials || !nparts) return nsk::set_error(NSK_ERR_SHAPE, "conv2d dgrad_bnstats: null argument");
  if (beta != 0.f && beta != 1.f) return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d dgrad_bnstats: beta 0 or 1");
  if (partial_floats < (uint64_t)2 * nsk::sm_count() * 2 * d->C)
    return nsk::set_error(NSK_ERR_SHAPE, "conv2d dgrad_bnstats: partials buffer smaller than 2*SMs x 2 x C floats");
  if (((uintptr_t)bn_x & 15) || ((uintptr_t)relu_mask & 3))
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d dgrad_bnstats: misaligned BatchNorm input or mask");
  return conv_dgrad(d, dy, w, dx, beta, (const __nv_bfloat16*)bn_x, (const uint8_t*)relu_mask, partials,
                    partial_floats, nparts, stream);
}

}  // extern "C"

namespace {

int conv_dgrad(const NskConvDesc* d, const void* dy, const void* w, void* dx, float beta, const __nv_bfloat16* bx,
               const uint8_t* bmask, float* stats, uint64_t stats_floats, int* nparts, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  const int P = d->P, Q = d->Q, st = d->stride;
  if (st > 2) return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d dgrad: stride > 2");
  if (d->H % st || d->W % st) return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d dgrad: H, W must divide stride");
  // output grid of each class
  const int Hg = d->H / st, Wg = d->W / st;
  int Wt = 0, Ht = 0, Nt = 0;
  const bool i2c = !pixel_tile(Wg, Hg, 128, &Wt, &Ht, &Nt) || force_i2c();
  int active = 0;  // parity classes with at least one tap
  for (int c = 0; c < st * st; ++c) {
    bool any = false;
    for (int r = 0; r < d->R; ++r)
      for (int q = 0; q < d->S; ++q)
        any = any || (((st == 2 ? (c >> 1) : 0) + d->pad - r) % st == 0 && ((st == 2 ? (c & 1) : 0) + d->pad - q) % st == 0);
    active += any;
  }
  const int dsteps = d->R * d->S * (d->K / 64);
  const int splits = st == 1 ? conv_splits((d->N * Hg * Wg + 127) / 128, d->C, dsteps) : 1;
  const int BN = splits > 1 ? 256 : pick_bn_units(d->C, (d->N * Hg * Wg + 127) / 128, beta == 1.f ? active : st * st);
  CUtensorMap ma, mb;
  if (!i2c && (rc = nhwc_map(&ma, dy, d->N, P, Q, d->K, 64, Wt, Ht, Nt, 1))) return rc;
  {
    const int RS = d->R * d->S;
    uint64_t dims[3] = {(uint64_t)d->C, (uint64_t)RS, (uint64_t)d->K};
    uint64_t str[2] = {(uint64_t)d->C * 2, (uint64_t)RS * d->C * 2};
    uint32_t box[3] = {64, 1, 64};
    if ((rc = nsk::encode_tmap(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w, dims, str, box, nullptr,
                               CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
  }
  UmmaProb p{};
  p.mode = MODE_CONV;
  p.bmode = BMODE_DGRAD3D;
  p.M = d->N * Hg * Wg;
  p.N = d->C;
  p.Wt = Wt; p.Ht = Ht; p.Nt = Nt;
  p.Wo = Wg; p.Ho = Hg;
  p.cs = 1;
  p.cchunks = d->K / 64;
  const int ncls = st * st;
  for (int c = 0; c < ncls; ++c) {
    const int ph = st == 2 ? (c >> 1) : 0, pw = st == 2 ? (c & 1) : 0;
    int t = 0;
    for (int r = 0; r < d->R; ++r)
      for (int s = 0; s < d->S; ++s) {
        // h = i*st + ph = p*st - pad + r  =>  p = i + (ph + pad - r)/st when divisible
        int nh = ph + d->pad - r, nw = pw + d->pad - s;
        if (((nh % st) + st) % st || ((nw % st) + st) % st) continue;
        int dh = nh >= 0 ? nh / st : -((-nh + st - 1) / st);
        int dw = nw >= 0 ? nw / st : -((-nw + st - 1) / st);
        p.tdh[c][t] = (signed char)dh;
        p.tdw[c][t] = (signed char)dw;
        p.tw[c][t] = (signed char)(r * d->S + s);
        ++t;
      }
    p.ntaps[c] = t;
    p.cph[c] = (signed char)ph;
    p.cpw[c] = (signed char)pw;
  }
  // accumulating into an existing gradient: a parity class without taps (1x1 stride 2: three of four) adds
  // nothing, so its work units are dropped instead of re-writing dx unchanged
  int ncls_run = ncls;
  if (beta == 1.f && ncls > 1 && !bx) {  // (statistics need every pixel through the epilogue)
    ncls_run = 0;
    for (int c = 0; c < ncls; ++c) {
      if (p.ntaps[c] == 0) continue;
      if (ncls_run != c) {
        p.ntaps[ncls_run] = p.ntaps[c];
        for (int t = 0; t < p.ntaps[c]; ++t) {
          p.tdh[ncls_run][t] = p.tdh[c][t];
          p.tdw[ncls_run][t] = p.tdw[c][t];
          p.tw[ncls_run][t] = p.tw[c][t];
        }
        p.cph[ncls_run] = p.cph[c];
        p.cpw[ncls_run] = p.cpw[c];
      }
      ++ncls_run;
    }
    if (ncls_run == 0) return NSK_OK;  // nothing to add
  }
  p.os = st; p.Hd = d->H; p.Wd = d->W;
  p.out = dx;
  p.ldc = d->C;
  p.out_f32 = 0;
  p.beta = beta;
  if (i2c) {
    if ((rc = i2c_map(p, &ma, dy, d->N, P, Q, d->K, Hg, Wg, ncls_run, 128))) return rc;
  } else if (ncls == 1 && splits == 1 && try_rowreuse(p, &ma, dy, d->N, P, Q, d->K, BN)) {
    if (BN == 64) {
      try_rr3(p, &mb, d, w, BN, BMODE_RR3T);
      try_wres(p, &ma, dy, d->N, P, Q, d->K, d->C);
    }
  }
  p.mc = !p.rr && mc_ok(BN, (p.M + 127) / 128);  // (the dgrad B boxes are per 64-channel slab: no map change)
  if (const char* pr = getenv("NSK_PROBE")) p.probe = atoi(pr);
  if (bx) {
    p.bx = bx;
    p.bmask = bmask;
    p.stats = stats;
    p.fold_reset = nsk::bn_fold_counter_bwd((cudaStream_t)stream);
  }
  if (splits > 1)
    return conv_split_run(p, ma, mb, splits, dsteps, dx, beta, stats, nparts, (cudaStream_t)stream);
  CUtensorMap mc;
  const char* red = getenv("NSK_TMA_REDUCE");
  const bool ts = ncls == 1 && (beta == 0.f || (beta == 1.f && (bx || !(red && red[0] == '0')))) &&
                  out_map(&mc, dx, p.M, d->C, d->C);
  if (bx) {  // the epilogue adds the pending gradient itself (it needs the sum for the statistics)
    p.bacc = beta == 1.f;
    p.beta = 0.f;
    p.tma_store = ts ? 1 : 0;
  } else {
    p.tma_store = ts ? (beta == 1.f ? 2 : 1) : 0;
    if (ts) p.beta = 0.f;  // the accumulation (if any) happens in the TMA reduce
  }
  if (bx) {
    rc = dispatch_bn<2, 2>(BN, ma, mb, p, (p.M + 127) / 128, (d->C + BN - 1) / BN, ncls_run,
                              (cudaStream_t)stream, nparts, ts ? &mc : nullptr);
    if (rc != NSK_ERR_UNSUPPORTED) return rc;
    // the statistics buffers do not fit beside this tile configuration: plain (accumulating) dgrad, no partials --
    // the caller then runs the BatchNorm backward's own reduction over the unmasked gradient
    *nparts = 0;
    return conv_dgrad(d, dy, w, dx, beta, nullptr, nullptr, nullptr, 0, nullptr, stream);
  }
  return dispatch_bn<2>(BN, ma, mb, p, (p.M + 127) / 128, (d->C + BN - 1) / BN, ncls_run, (cudaStream_t)stream,
                        nparts, ts ? &mc : nullptr);
}

}  // namespace

extern "C" {

// Grid cap for the weight-gradient kernels. side.py sets it to one CTA per SM while wgrads run on a side stream
// next to the rest of backward: two persistent CTAs per SM starve the compute stream (2.41 -> 2.35 ms/step).
int nsk_wgrad_grid_cap(int ctas) {
  g_wgrad_grid_cap = ctas < 0 ? 0 : ctas;
  return NSK_OK;
}

uint64_t nsk_conv2d_wgrad_workspace(const NskConvDesc* d) {
  if (wgrad_rr128_ok(d)) {  // three column-offset units per split, ~one unit per SM
    const int k_steps = (int)((long long)d->N * d->P * d->Q / 64);
    int splits = nsk::sm_count() / 3;
    if (splits > k_steps / 8) splits = k_steps / 8;
    return (uint64_t)(splits < 1 ? 1 : splits) * 1152 * 128 * sizeof(float);
  }
  if (wgrad_rr64_ok(d)) {  // one split per SM (wgrad_rr64_kernel): 640 x 64 fp32 partials each
    const long long pix = (long long)d->N * d->P * d->Q;
    const int k_steps = (int)(pix / 64);
    int splits = nsk::sm_count();
    if (splits > k_steps / 8) splits = k_steps / 8;
    return (uint64_t)(splits < 1 ? 1 : splits) * 640 * 64 * sizeof(float);
  }
  const int M = d->R * d->S * d->C;
  const int Mpad = ((M + 127) / 128) * 128;
  const long long pix = (long long)d->N * d->P * d->Q;
  const int k_steps = (int)((pix + 63) / 64);
  const int mt = Mpad / 128;
  const int BN = pick_bn(d->K);
  const int nt = (d->K + BN - 1) / BN;
  int target = nsk::sm_count() * (BN <= 128 ? 2 : 1);  // one persistent wave (2 CTAs per SM for BN <= 128)
  int splits = target / (mt * nt);
  if (splits < 1) splits = 1;
  int max_splits = k_steps / 8 > 0 ? k_steps / 8 : 1;
  if (splits > max_splits) splits = max_splits;
  return (uint64_t)splits * Mpad * d->K * sizeof(float);
}

// dw[k,r,s,c] (+)= sum_{n,p,q} dy[n,p,q,k] * x[n, p*st-pad+r, q*st-pad+s, c]   (fp32 out)
int nsk_conv2d_wgrad(const NskConvDesc* d, const void* x, const void* dy, float* dw, float beta, void* ws,
                     uint64_t ws_bytes, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (wgrad_rr128_ok(d)) {
    const long long npix = (long long)d->N * d->P * d->Q;
    const int k_steps = (int)(npix / 64);
    int splits = (int)(ws_bytes / (1152ull * 128 * sizeof(float)));
    if (splits > nsk::sm_count() / 3) splits = nsk::sm_count() / 3;
    if (splits > k_steps / 8) splits = k_steps / 8;
    if (splits >= 1) {
      const int per = (k_steps + splits - 1) / splits;
      splits = (k_steps + per - 1) / per;
      CUtensorMap mx, mdy;
      if ((rc = nhwc_map(&mx, x, d->N, d->H, d->W, 128, 64, 16, 6, 1, 1))) return rc;
      {  // dy as {64 outputs, pixels, 2 halves (128 B apart)}: both 64-wide N atoms in one box, 8 KB apart
        uint64_t dims[3] = {64, (uint64_t)npix, 2};
        uint64_t str[2] = {128 * 2, 128};
        uint32_t box[3] = {64, 64, 2};
        if ((rc = nsk::encode_tmap(&mdy, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dy, dims, str, box, nullptr,
                                   CU_TENSOR_MAP_SWIZZLE_128B)))
          return rc;
      }
      WgrrProb q{};
      q.k_steps = k_steps;
      q.per = per;
      q.units = 3 * splits;
      q.HW = d->H * d->W;
      q.Wimg = d->W;
      q.ws = (float*)ws;
      q.Mpad = 1152;
      const int smem = kWg128Stages * kWg128Stage + 1024 + 256;
      static bool configured = false;
      if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(wgrad_rr128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return nsk::cuda_status(e, "cudaFuncSetAttribute(wgrad_rr128)");
        configured = true;
      }
      int grid = q.units;
      if (grid > nsk::sm_count()) grid = nsk::sm_count();
      nsk::launch_pdl(wgrad_rr128_kernel, grid, 256, smem, (cudaStream_t)stream, mx, mdy, q);
      NSK_LAUNCH_CHECK("wgrad_rr128_kernel");
      const long long total = 1152LL * 128;
      if (((uintptr_t)dw & 15) || ((uintptr_t)ws & 15))
        return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d wgrad: dw and workspace must be 16-byte aligned");
      if (total / 4 < (long long)nsk::sm_count() * 512 && splits >= 16)
        nsk::launch_pdl(wgrad_reduce_kernel<8>, (unsigned)((total / 4 + 31) / 32), dim3(32, 8), 0,
                        (cudaStream_t)stream, (const float*)ws, splits, 1152, 1152, 128, dw, beta);
      else
        nsk::launch_pdl(wgrad_reduce_kernel<1>, (unsigned)((total / 4 + 255) / 256), dim3(256, 1), 0,
                        (cudaStream_t)stream, (const float*)ws, splits, 1152, 1152, 128, dw, beta);
      NSK_LAUNCH_CHECK("wgrad_reduce_kernel");
      return NSK_OK;
    }
  }
  if (wgrad_rr64_ok(d)) {
    const long long npix = (long long)d->N * d->P * d->Q;
    const int k_steps = (int)(npix / 64);
    int splits = (int)(ws_bytes / (640ull * 64 * sizeof(float)));
    if (splits > nsk::sm_count()) splits = nsk::sm_count();
    if (splits > k_steps / 8) splits = k_steps / 8;
    if (splits >= 1) {
      const int per = (k_steps + splits - 1) / splits;
      splits = (k_steps + per - 1) / per;
      CUtensorMap mx, mdy;
      if ((rc = nhwc_map(&mx, x, d->N, d->H, d->W, 64, 64, 32, 4, 1, 1))) return rc;
      {
        uint64_t dims[2] = {64, (uint64_t)npix};
        uint64_t str[1] = {64 * 2};
        uint32_t box[2] = {64, 64};
        if ((rc = nsk::encode_tmap(&mdy, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dy, dims, str, box, nullptr,
                                   CU_TENSOR_MAP_SWIZZLE_128B)))
          return rc;
      }
      WgrrProb q{};
      q.k_steps = k_steps;
      q.per = per;
      q.units = splits;
      q.HW = d->H * d->W;
      q.Wimg = d->W;
      q.ws = (float*)ws;
      q.Mpad = 640;
      const int smem = kWgrrStages * kWgrrStage + 1024 + 256;
      static bool configured = false;
      if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(wgrad_rr64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return nsk::cuda_status(e, "cudaFuncSetAttribute(wgrad_rr64)");
        configured = true;
      }
      int grid = splits;
      if (grid > nsk::sm_count()) grid = nsk::sm_count();
      nsk::launch_pdl(wgrad_rr64_kernel, grid, 256, smem, (cudaStream_t)stream, mx, mdy, q);
      NSK_LAUNCH_CHECK("wgrad_rr64_kernel");
      const long long total = 576LL * 64;
      if (((uintptr_t)dw & 15) || ((uintptr_t)ws & 15))
        return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d wgrad: dw and workspace must be 16-byte aligned");
      if (total / 4 < (long long)nsk::sm_count() * 512 && splits >= 16)
        nsk::launch_pdl(wgrad_reduce_kernel<8>, (unsigned)((total / 4 + 31) / 32), dim3(32, 8), 0,
                        (cudaStream_t)stream, (const float*)ws, splits, 640, 576, 64, dw, beta);
      else
        nsk::launch_pdl(wgrad_reduce_kernel<1>, (unsigned)((total / 4 + 255) / 256), dim3(256, 1), 0,
                        (cudaStream_t)stream, (const float*)ws, splits, 640, 576, 64, dw, beta);
      NSK_LAUNCH_CHECK("wgrad_reduce_kernel");
      return NSK_OK;
    }
  }
  const int P = d->P, Q = d->Q;
  int Wt = 0, Ht = 0, Nt = 0;
  const long long pix = (long long)d->N * P * Q;
  // the tiled path needs whole-row 64-pixel tiles; im2col mode walks any grid (the K tail past the last
  // pixel reads zeros on both operands)
  const bool i2c = !pixel_tile(Q, P, 64, &Wt, &Ht, &Nt) || (pix % 64) || force_i2c();
  const int RS = d->R * d->S;
  const int M = RS * d->C;
  const int Mpad = ((M + 127) / 128) * 128;
  const int k_steps = (int)((pix + 63) / 64);
  const int BN = pick_bn(d->K);
  const int mt = Mpad / 128, nt = (d->K + BN - 1) / BN;
  int splits = (int)(ws_bytes / ((uint64_t)Mpad * d->K * sizeof(float)));
  if (splits < 1) return nsk::set_error(NSK_ERR_SHAPE, "conv2d wgrad: workspace too small");
  uint64_t want = nsk_conv2d_wgrad_workspace(d) / ((uint64_t)Mpad * d->K * sizeof(float));
  if ((uint64_t)splits > want) splits = (int)want;
  const int per = (k_steps + splits - 1) / splits;
  splits = (k_steps + per - 1) / per;
  CUtensorMap ma, mb;
  if (!i2c && (rc = nhwc_map(&ma, x, d->N, d->H, d->W, d->C, 64, Wt, Ht, Nt, d->stride))) return rc;
  {
    uint64_t dims[2] = {(uint64_t)d->K, (uint64_t)pix};
    uint64_t str[1] = {(uint64_t)d->K * 2};
    uint32_t box[2] = {64, 64};
    if ((rc = nsk::encode_tmap(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dy, dims, str, box, nullptr,
                               CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
  }
  // B (dy, MN-major) for a BN-wide tile = BN/64 slabs of 64 channels: one 3-D box {64, 64 pixels, BN/64 slabs}
  // (slab stride 128 B) instead of BN/64 boxes
  int bslab = 0;
  if (BN > 64 && !(getenv("NSK_BSLAB") && getenv("NSK_BSLAB")[0] == '0')) {
    uint64_t dims[3] = {64, (uint64_t)pix, (uint64_t)d->K / 64};
    uint64_t str[2] = {(uint64_t)d->K * 2, 128};
    uint32_t box[3] = {64, 64, (uint32_t)BN / 64};
    CUtensorMap m3;
    if (nsk::encode_tmap(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dy, dims, str, box, nullptr,
                         CU_TENSOR_MAP_SWIZZLE_128B) == NSK_OK) {
      mb = m3;
      bslab = 1;
    }
  }
  UmmaProb p{};
  p.bslab = bslab;
  p.mode = MODE_WGRAD;
  p.a_mn = 1;
  p.b_mn = 1;
  p.M = M;
  p.N = d->K;
  p.k_steps = k_steps;
  p.k_per_split = per;
  p.Wt = Wt; p.Ht = Ht; p.Nt = Nt;
  p.Wo = Q; p.Ho = P;
  p.cs = d->stride;
  int t = 0;
  for (int r = 0; r < d->R; ++r)
    for (int s = 0; s < d->S; ++s, ++t) {
      p.tdh[0][t] = (signed char)(r - d->pad);
      p.tdw[0][t] = (signed char)(s - d->pad);
    }
  p.ntaps[0] = RS;
  if (i2c && (rc = i2c_map(p, &ma, x, d->N, d->H, d->W, d->C, P, Q, 1, 64))) return rc;
  p.atoms_total = M / 64;
  p.cin_atoms = d->C / 64;
  p.out = ws;
  p.ldc = d->K;
  p.out_f32 = 1;
  p.Mpad = Mpad;
  if (const char* pr = getenv("NSK_PROBE")) p.probe = atoi(pr);
  if ((rc = dispatch_bn<2>(BN, ma, mb, p, mt, nt, splits, (cudaStream_t)stream))) return rc;
  long long total = (long long)M * d->K;
  if (((uintptr_t)dw & 15) || ((uintptr_t)ws & 15))
    return nsk::set_error(NSK_ERR_UNSUPPORTED, "conv2d wgrad: dw and workspace must be 16-byte aligned");
  if (total / 4 < (long long)nsk::sm_count() * 512 && splits >= 16)
    nsk::launch_pdl(wgrad_reduce_kernel<8>, (unsigned)((total / 4 + 31) / 32), dim3(32, 8), 0, (cudaStream_t)stream,
                    (const float*)ws, splits, Mpad, M, d->K, dw, beta);
  else
    nsk::launch_pdl(wgrad_reduce_kernel<1>, (unsigned)((total / 4 + 255) / 256), dim3(256, 1), 0, (cudaStream_t)stream,
                    (const float*)ws, splits, Mpad, M, d->K, dw, beta);
  NSK_LAUNCH_CHECK("wgrad_reduce_kernel");
  return NSK_OK;
}

}  // extern "C"
