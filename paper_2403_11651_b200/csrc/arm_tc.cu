// arm_tc.cu -- ARM rate on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Same function as arm_rate.cu (PAPER.md:106-109 ARM f_psi, :120 R term of
// Eq. 1; Table 1 ARM column; readings #1-#8): for every latent the
// causal context c, the MLP z1 = ReLU(W0 c + b0), z_{k+1} = ReLU(W_k z_k + b_k
// [+ z_k]), (mu, s) = W_out z + b_out, then -log2 of the Laplace bin mass.
//
// The hidden layers are dense contractions over all latents at once -- [128
// latents x K] x [K x N] per MMA block -- so they run as tcgen05.mma kind::tf32
// with fp32 accumulators in TMEM:
//   * layer 0: A = the context rows, small integers (|y| <= 2^10), EXACT in
//     tf32, so only the weights are split: W = W_hi + W_lo (tf32 each) and
//     D = A.W_hi + A.W_lo.  The bias rides on a constant-1 input column.
//   * hidden layer k >= 1: the activations are arbitrary fp32, split per
//     element z = z_hi + z_lo (cvt.rna.tf32 + exact subtraction):
//     D = z_hi.W_hi + z_hi.W_lo + z_lo.W_hi ("3xTF32"): every product is exact
//     in fp32 and only the z_lo.W_lo term (~2^-22 relative) is dropped, so the
//     result is fp32-accurate (well inside the 1e-3-bit per-latent and 1e-4
//     total-rate tolerances).
//   * the 2-wide output layer, the Laplace bits and the reduction stay on the
//     CUDA cores (packed FFMA2, uniform weights), one latent per thread.
//
// CTA = 128 threads = one MMA block of M = 128 latents at a time: thread t
// owns latent t of the block, writes row t of the A operand and reads TMEM
// lane t of the accumulator (warp w <-> lanes 32w .. 32w+31).  A tile of the
// FFMA2 kernel's geometry (8 rows x 64 latents; same tile table, same window
// staging) is 4 blocks of 2 rows.  Operands are K-major, no-swizzle canonical
// layout in shared memory (8-row x 16-byte core matrices; LBO = 128 B between
// K-adjacent core matrices, SBO = K/4 x 128 B between 8-row groups; the encoding
// is validated by tools/microbench/tc_probe.cu).  Several CTAs per SM overlap
// one CTA's MMA wait with the others' CUDA-core work.
//
// Status (measured on B200): 142 us per 2K image vs 140 us for
// the FFMA2 kernel -- each 128-latent block pays two serialised MMA round trips
// and 4 CTAs per SM do not hide them; a variant with the A operands in TMEM
// (tcgen05.st, TS MMAs) measured 175 us.  Beating FFMA2 needs a warp-specialised
// multi-stage pipeline, so this path is opt-in (CCRD_ARM_PATH=tc) and
// parity-tested, not the default.
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "arm_math.cuh"
#include "ccrd_common.cuh"
#include "tcgen05.cuh"

namespace ccrd {

constexpr int TC_THREADS = 128;
constexpr int TC_M = 128;
constexpr int TC_CTAS_PER_SM = 4;

__host__ __device__ constexpr int rup(int x, int m) { return (x + m - 1) / m * m; }

template <int C, int NH, int NHL>
struct ArmTcShape {
  static constexpr int K0 = rup(C + 1, 8);                  // context + bias column
  static constexpr int NP = rup(NH, 16) < 16 ? 16 : rup(NH, 16);  // MMA N (M = 128 needs N % 16 == 0)
  static constexpr int K1 = rup(NH + 1, 8);                 // hidden + bias column
  static constexpr int NHID = NHL - 1;                      // NH -> NH layers on the tensor cores
  static constexpr int BW0 = NP * K0;                       // floats per weight matrix
  static constexpr int BW1 = NP * K1;
  static constexpr int A_FLOATS = TC_M * (K0 > 2 * K1 ? K0 : 2 * K1);  // A0 | (A_hi, A_lo)
  static constexpr int WIN = ARM_SH * ARM_SW;
  static constexpr int B_FLOATS = 2 * BW0 + 2 * NHID * BW1;
  static constexpr size_t SMEM = sizeof(float) * (size_t)(A_FLOATS + B_FLOATS + WIN) + 64;
  static_assert(NP <= 32, "one 32-column TMEM accumulator");
  static_assert(K0 % 8 == 0 && K1 % 8 == 0, "tcgen05 shape");
};

// K-major canonical offset (floats) of element (r, k) of an operand with K
// columns: core matrix (r/8, k/4), 8 rows x 4 floats each
__host__ __device__ constexpr int kmaj(int r, int k, int K) {
  return (r >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

template <int C, int NH, int NHL>
struct ArmTcParams {
  using S = ArmTcShape<C, NH, NHL>;
  ArmGeom g;
  const int16_t* lat;
  double* partial;  // [tiles][16]: one per (block, warp)
  float* mu;        // optional per-latent debug outputs
  float* scale;
  float* bits;
  // weights, pre-split on the host into tf32 (hi, lo) pairs, canonical layout
  float B0[2][S::BW0];                                    // [hi/lo] layer 0 (bias in column C)
  float B1[(S::NHID > 0) ? S::NHID : 1][2][S::BW1];       // [layer][hi/lo] (residual folded, bias in column NH)
  float2 wo[NH];                                          // output layer (mu, log-scale) per input
  float2 bo;
  float2 wm[NH / 2], wsl[NH / 2];                         // output layer as input pairs: mu, log-scale
  CUtensorMap tmap[CC_MAX_LEVELS];  // int16 grid l ([rows present][w]) for TMA window loads (arm_tcg_kernel, TMA)
};

// -log2 Laplace bin mass (identical to arm_rate.cu's; see there)
__device__ __forceinline__ float laplace_bits_tc(float y, float mu, float s, const ArmGeom& g) {
  constexpr float LOG2E = 1.4426950408889634f;
  s = fminf(fmaxf(s, g.lsmin), g.lsmax);
  const float ibl = exp2f_approx(-s * LOG2E) * LOG2E;
  const float a = fabsf(y - mu);
  const float am = fminf(a, 0.5f);
  const float e1 = exp2f_approx((am - 0.5f) * ibl);
  const float e2 = exp2f_approx(-(am + 0.5f) * ibl);
  const float p_in = 1.0f - 0.5f * (e1 + e2);
  const float bits_in = -log2f_approx(fmaxf(p_in, g.p_floor));
  const float bits_out = fmaf(a - 0.5f, ibl, 1.0f) - log2f_approx(1.0f - exp2f_approx(-ibl));
  return fminf(a < 0.5f ? bits_in : bits_out, g.bits_cap);
}

template <int C, int NH, int NHL>
__global__ void __launch_bounds__(TC_THREADS, TC_CTAS_PER_SM)
    arm_tc_kernel(const __grid_constant__ ArmTcParams<C, NH, NHL> p) {
  using S = ArmTcShape<C, NH, NHL>;
  constexpr int K0 = S::K0, NP = S::NP, K1 = S::K1;
  extern __shared__ __align__(1024) float tsm[];
  float* sA = tsm;                              // A0 [128 x K0] | A_hi, A_lo [128 x K1] each
  float* sB = tsm + S::A_FLOATS;                // B0 hi, lo, then B1 hi, lo per hidden layer
  float* win = sB + S::B_FLOATS;                // causal window of the tile (fp32)
  uint64_t* bar = reinterpret_cast<uint64_t*>(win + S::WIN + (S::WIN & 1));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // weights -> shared memory (canonical layout prepared on the host)
  {
    const float4* src0 = reinterpret_cast<const float4*>(&p.B0[0][0]);
    float4* dst = reinterpret_cast<float4*>(sB);
    for (int i = t; i < 2 * S::BW0 / 4; i += TC_THREADS) dst[i] = src0[i];
    if constexpr (S::NHID > 0) {
      const float4* src1 = reinterpret_cast<const float4*>(&p.B1[0][0][0]);
      for (int i = t; i < 2 * S::NHID * S::BW1 / 4; i += TC_THREADS) dst[2 * S::BW0 / 4 + i] = src1[i];
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
  const uint32_t sA_u = smem_u32(sA), sB_u = smem_u32(sB);
  uint32_t phase = 0;

  const int n_tiles = p.g.tile_begin[p.g.L];
#pragma unroll 1
  for (int b = blockIdx.x; b < n_tiles; b += gridDim.x) {
    // ---- (level, tile) and the causal window (zero outside the grid)
    int l = 0;
#pragma unroll 1
    while (l + 1 < p.g.L && b >= p.g.tile_begin[l + 1]) l++;
    const int tl = b - p.g.tile_begin[l];
    const int ty = tl / p.g.tiles_x[l];
    const int i0 = p.g.own_lo[l] + ty * ARM_TY, j0 = (tl - ty * p.g.tiles_x[l]) * ARM_TX;
    const int w = p.g.lv.w[l], rlo = p.g.lv.lo[l], rhi = p.g.lv.hi[l];
    const int16_t* __restrict__ grid = p.lat + p.g.lv.off[l];
    {
      constexpr int IT = (S::WIN + TC_THREADS - 1) / TC_THREADS;
      int16_t v[IT];
#pragma unroll
      for (int k = 0; k < IT; k++) {
        const int s = t + k * TC_THREADS;
        const int r = s / ARM_SW, c = s - r * ARM_SW;
        const int gi = i0 - ARM_HALO_TOP + r, gj = j0 - ARM_HALO_X + c;
        v[k] = (s < S::WIN && gi >= rlo && gi < rhi && gj >= 0 && gj < w) ? __ldg(grid + (int64_t)(gi - rlo) * w + gj)
                                                                        : (int16_t)0;
      }
      __syncthreads();  // the previous tile's readers of `win` are done
#pragma unroll
      for (int k = 0; k < IT; k++) {
        const int s = t + k * TC_THREADS;
        if (s < S::WIN) win[s] = (float)v[k];
      }
      __syncthreads();
    }

    // ---- four blocks of 2 rows x 64 latents
#pragma unroll 1
    for (int q = 0; q < ARM_TY / 2; q++) {
      const int ry = 2 * q + (t >> 6), cx = t & 63;  // this thread's latent in the tile
      const float* center = win + (ry + ARM_HALO_TOP) * ARM_SW + cx + ARM_HALO_X;
      const float y = center[0];
      // A0 row t: [context (C), 1 (bias), 0 ...]
      {
        float row[K0];
#pragma unroll
        for (int c = 0; c < C; c++) row[c] = center[p.g.ctx_off[c]];
        row[C] = 1.0f;
#pragma unroll
        for (int c = C + 1; c < K0; c++) row[c] = 0.0f;
#pragma unroll
        for (int c4 = 0; c4 < K0 / 4; c4++)
          *reinterpret_cast<float4*>(sA + kmaj(t, 4 * c4, K0)) =
              make_float4(row[4 * c4], row[4 * c4 + 1], row[4 * c4 + 2], row[4 * c4 + 3]);
      }
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      if (t == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int s = 0; s < K0 / 8; s++) {
          const uint64_t da = umma_desc(sA_u + s * 256, 128, (K0 / 4) * 128);
          mma_tf32(tmem, da, umma_desc(sB_u + s * 256, 128, (K0 / 4) * 128), IDESC, s > 0);
          mma_tf32(tmem, da, umma_desc(sB_u + S::BW0 * 4 + s * 256, 128, (K0 / 4) * 128), IDESC, 1);
        }
        mma_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      float z[NP];
      tmem_row<NP>(taddr, z);
#pragma unroll
      for (int n = 0; n < NH; n++) z[n] = fmaxf(z[n], 0.0f);

      // ---- hidden layers NH -> NH (3xTF32)
#pragma unroll 1
      for (int k = 0; k < S::NHID; k++) {
        float* aH = sA;
        float* aL = sA + TC_M * K1;
#pragma unroll
        for (int c4 = 0; c4 < K1 / 4; c4++) {
          float hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int c = 4 * c4 + e;
            const float x = (c < NH) ? z[c] : (c == NH ? 1.0f : 0.0f);
            hi[e] = tf32_rna(x);
            lo[e] = x - hi[e];
          }
          *reinterpret_cast<float4*>(aH + kmaj(t, 4 * c4, K1)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<float4*>(aL + kmaj(t, 4 * c4, K1)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (t == 0) {
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t bh = sB_u + 4 * (2 * S::BW0 + 2 * k * S::BW1), bl = bh + 4 * S::BW1;
          const uint32_t ah = sA_u, al = sA_u + 4 * TC_M * K1;
#pragma unroll
          for (int s = 0; s < K1 / 8; s++) {
            const uint64_t dah = umma_desc(ah + s * 256, 128, (K1 / 4) * 128);
            const uint64_t dal = umma_desc(al + s * 256, 128, (K1 / 4) * 128);
            const uint64_t dbh = umma_desc(bh + s * 256, 128, (K1 / 4) * 128);
            const uint64_t dbl = umma_desc(bl + s * 256, 128, (K1 / 4) * 128);
            mma_tf32(tmem, dah, dbh, IDESC, s > 0);
            mma_tf32(tmem, dah, dbl, IDESC, 1);
            mma_tf32(tmem, dal, dbh, IDESC, 1);
          }
          mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        tmem_row<NP>(taddr, z);
#pragma unroll
        for (int n = 0; n < NH; n++) z[n] = fmaxf(z[n], 0.0f);
      }

      // ---- output layer (mu, log-scale) on the CUDA cores, Laplace bits
      uint64_t o = ldp2(p.bo);
#pragma unroll
      for (int n = 0; n < NH; n++) o = ffma2(f2pack(z[n], z[n]), ldp2(p.wo[n]), o);
      const int i = i0 + ry, j = j0 + cx;
      float bits = 0.0f;
      if (i < p.g.own_hi[l] && j < w) {
        const float2 ms = f2unpack(o);
        bits = laplace_bits_tc(y, ms.x, ms.y, p.g);
        if (p.bits != nullptr) {
          const int64_t qi = p.g.lv.off[l] + (int64_t)(i - rlo) * w + j;
          p.bits[qi] = bits;
          if (p.mu) p.mu[qi] = ms.x;
          if (p.scale) p.scale[qi] = __expf(fminf(fmaxf(ms.y, p.g.lsmin), p.g.lsmax));
        }
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o2);
      if (lane == 0) p.partial[(int64_t)b * 16 + q * 4 + warp] = (double)bits;
      // the next block rewrites A and the accumulator: every thread's TMEM load
      // of this block is complete (wait::ld in tmem_row) before the barrier
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

// ---------------------------------------------------------------- warp-specialised pipeline
// The same arithmetic as arm_tc_kernel (exact context x [B_hi + B_lo], 3xTF32
// hidden layer, FFMA2 output layer, the same Laplace bits), pipelined over
// blocks of 128 latents with dedicated warps, two blocks in flight:
//   warps 0-3 (front): stage the tile's causal window, gather the contexts of
//             block b into A0[b % 2]; epilogue 0 of block b-1: TMEM D0 ->
//             ReLU -> hi / lo split into A1[(b-1) % 2];
//   warp 8:   allocates TMEM, issues MMA0(b) and MMA1(b-1) as their operands
//             arrive (mbarriers), commits to the waiting warps;
//   warps 4-7 (back): epilogue 1 of block b: TMEM D1 -> ReLU -> output layer
//             -> Laplace bits (y re-read from the int16 latents) -> partials.
// The serial version pays two MMA round trips per block on the same warps;
// here the front, back and tensor work of neighbouring blocks overlap.
constexpr int TW_THREADS = 288;  // 9 warps
#ifndef CCRD_TW_A1_SLOTS
#define CCRD_TW_A1_SLOTS 1
#endif
constexpr int TW_A1_SLOTS = CCRD_TW_A1_SLOTS;

template <int C, int NH, int NHL>
struct ArmTcwShape {
  using S = ArmTcShape<C, NH, NHL>;
  static constexpr int K0 = S::K0, K1 = S::K1, NP = S::NP;
  static constexpr int A0F = TC_M * K0;        // floats per A0 slot
  static constexpr int A1F = 2 * TC_M * K1;    // hi + lo per A1 slot
  static constexpr int OFF_B = 0;
  static constexpr int OFF_WIN = S::B_FLOATS;
  static constexpr int OFF_A0 = OFF_WIN + ((ARM_SH * ARM_SW + 31) / 32) * 32;
  static constexpr int A1S = TW_A1_SLOTS;  // A1 slots (1: smaller CTA, more CTAs per SM)
  static constexpr int OFF_A1 = OFF_A0 + 2 * A0F;
  static constexpr int FLOATS = OFF_A1 + A1S * A1F;
  static constexpr size_t SMEM = sizeof(float) * (size_t)FLOATS + 16 * 8 + 64;
  static_assert(S::NHID == 1, "one hidden NH -> NH layer");
};

__device__ __forceinline__ void tw_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void front_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int C, int NH, int NHL>
__global__ void __launch_bounds__(TW_THREADS, 1) arm_tcw_kernel(const __grid_constant__ ArmTcParams<C, NH, NHL> p) {
  using S = ArmTcShape<C, NH, NHL>;
  using W = ArmTcwShape<C, NH, NHL>;
  constexpr int K0 = S::K0, NP = S::NP, K1 = S::K1;
  extern __shared__ __align__(1024) float tsm[];
  float* sB = tsm + W::OFF_B;
  float* win = tsm + W::OFF_WIN;
  float* sA0 = tsm + W::OFF_A0;
  float* sA1 = tsm + W::OFF_A1;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tsm + W::FLOATS);
  uint64_t* a0_full = bars;       // [2] front -> MMA
  uint64_t* d0_full = bars + 2;   // [2] MMA0 commit
  uint64_t* a1_full = bars + 4;   // [2] front epilogue 0 -> MMA
  uint64_t* d1_full = bars + 6;   // [2] MMA1 commit
  uint64_t* d1_empty = bars + 8;  // [2] back done with D1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  {
    const float4* src0 = reinterpret_cast<const float4*>(&p.B0[0][0]);
    float4* dst = reinterpret_cast<float4*>(sB);
    for (int i = t; i < 2 * S::BW0 / 4; i += TW_THREADS) dst[i] = src0[i];
    const float4* src1 = reinterpret_cast<const float4*>(&p.B1[0][0][0]);
    for (int i = t; i < 2 * S::BW1 / 4; i += TW_THREADS) dst[2 * S::BW0 / 4 + i] = src1[i];
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int k = 0; k < 2; k++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(a0_full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d0_full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(a1_full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d1_full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(d1_empty + k)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;  // D0[0], D0[1], D1[0], D1[1]: NP columns each
  constexpr uint32_t IDESC =
      (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);

  const int n_tiles = p.g.tile_begin[p.g.L];
  const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nb = 4 * my_tiles;  // blocks of 128 latents (a tile = 8 rows x 64 = 4 blocks)
  auto tile_of = [&](int b) { return (int)blockIdx.x + (b >> 2) * (int)gridDim.x; };

  if (warp < 4) {
    // ======================= front: window, gather, epilogue 0
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    int l = 0, i0 = 0, j0 = 0;
#pragma unroll 1
    for (int b = 0; b <= nb; b++) {
      if (b < nb) {
        const int tile = tile_of(b), q = b & 3, s = b & 1;
        if (q == 0) {  // stage this tile's causal window (fp32, zero outside the grid)
          l = 0;
          while (l + 1 < p.g.L && tile >= p.g.tile_begin[l + 1]) l++;
          const int tl = tile - p.g.tile_begin[l];
          const int ty = tl / p.g.tiles_x[l];
          i0 = p.g.own_lo[l] + ty * ARM_TY;
          j0 = (tl - ty * p.g.tiles_x[l]) * ARM_TX;
          const int w = p.g.lv.w[l], rlo = p.g.lv.lo[l], rhi = p.g.lv.hi[l];
          const int16_t* __restrict__ grid = p.lat + p.g.lv.off[l];
          constexpr int IT = (S::WIN + 127) / 128;
          int16_t v[IT];
#pragma unroll
          for (int k = 0; k < IT; k++) {
            const int e = t + k * 128;
            const int r = e / ARM_SW, c = e - r * ARM_SW;
            const int gi = i0 - ARM_HALO_TOP + r, gj = j0 - ARM_HALO_X + c;
            v[k] = (e < S::WIN && gi >= rlo && gi < rhi && gj >= 0 && gj < w)
                       ? __ldg(grid + (int64_t)(gi - rlo) * w + gj) : (int16_t)0;
          }
          front_sync();  // every front thread is done with the previous tile's window
#pragma unroll
          for (int k = 0; k < IT; k++) {
            const int e = t + k * 128;
            if (e < S::WIN) win[e] = (float)v[k];
          }
          front_sync();
        }
        // A0 row t: [context (C), 1 (bias), 0 ...]   (A0[s] is free: MMA0(b-2) completed,
        // observed by this warp in epilogue 0 of block b-2)
        const int ry = 2 * q + (t >> 6), cx = t & 63;
        const float* center = win + (ry + ARM_HALO_TOP) * ARM_SW + cx + ARM_HALO_X;
        float row[K0];
#pragma unroll
        for (int c = 0; c < C; c++) row[c] = center[p.g.ctx_off[c]];
        row[C] = 1.0f;
#pragma unroll
        for (int c = C + 1; c < K0; c++) row[c] = 0.0f;
        float* A0 = sA0 + s * W::A0F;
#pragma unroll
        for (int c4 = 0; c4 < K0 / 4; c4++)
          *reinterpret_cast<float4*>(A0 + kmaj(t, 4 * c4, K0)) =
              make_float4(row[4 * c4], row[4 * c4 + 1], row[4 * c4 + 2], row[4 * c4 + 3]);
        asm volatile("fence.proxy.async.shared::cta;");
        __syncwarp();
        if (lane == 0) tw_arrive(a0_full + s);
      }
      if (b >= 1) {  // epilogue 0 of block b-1
        const int bb = b - 1, s = bb & 1;
        mbar_wait(d0_full + s, (bb >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        float z[NP];
        tmem_row<NP>(taddr + s * NP, z);
        // the A1 slot of block bb was last read by MMA1(bb - A1S)
        if (W::A1S == 2 && bb >= 2) mbar_wait(d1_full + s, ((bb >> 1) - 1) & 1);
        if (W::A1S == 1 && bb >= 1) mbar_wait(d1_full + ((bb - 1) & 1), ((bb - 1) >> 1) & 1);
        float* aH = sA1 + (W::A1S == 2 ? s : 0) * W::A1F;
        float* aL = aH + TC_M * K1;
#pragma unroll
        for (int c4 = 0; c4 < K1 / 4; c4++) {
          float hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int c = 4 * c4 + e;
            const float x = (c < NH) ? fmaxf(z[c], 0.0f) : (c == NH ? 1.0f : 0.0f);
            hi[e] = tf32_rna(x);
            lo[e] = x - hi[e];
          }
          *reinterpret_cast<float4*>(aH + kmaj(t, 4 * c4, K1)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<float4*>(aL + kmaj(t, 4 * c4, K1)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) tw_arrive(a1_full + s);
      }
    }
  } else if (warp < 8) {
    // ======================= back: epilogue 1, output layer, Laplace bits
    const int tb = t - 128;
    const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
#pragma unroll 1
    for (int b = 0; b < nb; b++) {
      const int tile = tile_of(b), q = b & 3, s = b & 1;
      mbar_wait(d1_full + s, (b >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      float z[NP];
      tmem_row<NP>(taddr + 2 * NP + s * NP, z);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) tw_arrive(d1_empty + s);  // D1[s] may be overwritten
      uint64_t o = ldp2(p.bo);
#pragma unroll
      for (int n = 0; n < NH; n++) {
        const float zn = fmaxf(z[n], 0.0f);
        o = ffma2(f2pack(zn, zn), ldp2(p.wo[n]), o);
      }
      int l = 0;
      while (l + 1 < p.g.L && tile >= p.g.tile_begin[l + 1]) l++;
      const int tl = tile - p.g.tile_begin[l];
      const int ty = tl / p.g.tiles_x[l];
      const int i = p.g.own_lo[l] + ty * ARM_TY + 2 * q + (tb >> 6);
      const int j = (tl - ty * p.g.tiles_x[l]) * ARM_TX + (tb & 63);
      const int w = p.g.lv.w[l], rlo = p.g.lv.lo[l];
      float bits = 0.0f;
      if (i < p.g.own_hi[l] && j < w) {
        const int64_t qi = p.g.lv.off[l] + (int64_t)(i - rlo) * w + j;
        const float y = (float)__ldg(p.lat + qi);
        const float2 ms = f2unpack(o);
        bits = laplace_bits_tc(y, ms.x, ms.y, p.g);
        if (p.bits != nullptr) {
          p.bits[qi] = bits;
          if (p.mu) p.mu[qi] = ms.x;
          if (p.scale) p.scale[qi] = __expf(fminf(fmaxf(ms.y, p.g.lsmin), p.g.lsmax));
        }
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o2);
      if (lane == 0) p.partial[(int64_t)tile * 16 + q * 4 + (warp & 3)] = (double)bits;
    }
  } else if (lane == 0) {
    // ======================= MMA issue
    const uint32_t sB_u = smem_u32(sB), sA0_u = smem_u32(sA0), sA1_u = smem_u32(sA1);
    auto mma0 = [&](int b) {
      const int s = b & 1;
      mbar_wait(a0_full + s, (b >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_u = sA0_u + 4 * s * W::A0F, d = tmem + s * NP;
#pragma unroll
      for (int k = 0; k < K0 / 8; k++) {
        const uint64_t da = umma_desc(a_u + k * 256, 128, (K0 / 4) * 128);
        mma_tf32(d, da, umma_desc(sB_u + k * 256, 128, (K0 / 4) * 128), IDESC, k > 0);
        mma_tf32(d, da, umma_desc(sB_u + S::BW0 * 4 + k * 256, 128, (K0 / 4) * 128), IDESC, 1);
      }
      mma_commit(d0_full + s);
    };
    auto mma1 = [&](int b) {
      const int s = b & 1;
      mbar_wait(a1_full + s, (b >> 1) & 1);
      if (b >= 2) mbar_wait(d1_empty + s, ((b >> 1) - 1) & 1);  // back done with D1[s] of block b-2
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ah = sA1_u + 4 * (W::A1S == 2 ? s : 0) * W::A1F, al = ah + 4 * TC_M * K1, d = tmem + 2 * NP + s * NP;
      const uint32_t bh = sB_u + 4 * (2 * S::BW0), bl = bh + 4 * S::BW1;
#pragma unroll
      for (int k = 0; k < K1 / 8; k++) {
        const uint64_t dah = umma_desc(ah + k * 256, 128, (K1 / 4) * 128);
        const uint64_t dal = umma_desc(al + k * 256, 128, (K1 / 4) * 128);
        const uint64_t dbh = umma_desc(bh + k * 256, 128, (K1 / 4) * 128);
        const uint64_t dbl = umma_desc(bl + k * 256, 128, (K1 / 4) * 128);
        mma_tf32(d, dah, dbh, IDESC, k > 0);
        mma_tf32(d, dah, dbl, IDESC, 1);
        mma_tf32(d, dal, dbh, IDESC, 1);
      }
      mma_commit(d1_full + s);
    };
#pragma unroll 1
    for (int b = 0; b < nb; b++) {
      mma0(b);
      if (b >= 1) mma1(b - 1);
    }
    if (nb >= 1) mma1(nb - 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}


// ---------------------------------------------------------------- warpgroup pipelines (the default TC ARM)
// Measured constraints (tools/microbench/tc_bench.cu, B200): one issuing thread
// sustains one tcgen05.mma per ~25 cycles (A in TMEM) whatever N is, while two
// or more issuers per SM reach the tensor pipe's floor of 128 N / 256 cycles
// per MMA (12 at N = 24); A operands read from shared memory cost ~41 cycles
// per K = 8 MMA (the 4 KB A tile), from TMEM ~25; a TMEM load waited on alone
// costs ~90 cycles, several in flight ~10.  Hence:
//   * NWG independent warpgroups per CTA (one persistent CTA per SM); every
//     warpgroup runs the whole chain for its own blocks of 128 latents and
//     issues its own MMAs (NWG issuers per SM; while one warpgroup waits for
//     its MMAs the others compute);
//   * every operand that changes per block lives in TMEM (TS MMAs): thread t
//     of the warpgroup owns latent t of the block = TMEM lane t for all three
//     stages, so the centre value y and the partial sums stay in registers;
//   * per warpgroup 3 column groups, reused in place:
//       X: A0 = [context, 1, 0..] (K0), then A1_lo (NH)
//       Y: D0 (NH) -> A1_hi in place; columns NH .. K1-1 hold the constant
//          bias input [1, 0, ..] written once (MMA0 has N = NH: never touched)
//       D: D1 (NH)
//   * stage order per block: gather -> tcgen05.st A0 -> barrier -> MMA0 ->
//     epilogue 0 (ReLU, hi/lo split, tcgen05.st) -> barrier -> MMA1 ->
//     epilogue 1 (ReLU, output layer on the CUDA cores with constant-bank
//     weights, Laplace bits, per-warp partial).
// The arithmetic is arm_tc_kernel's (exact context x [W_hi + W_lo], 3xTF32
// hidden layer with a truncated hi part -- exact split whatever rounding the
// tensor core applies to an already-tf32 value).
template <int C, int NH>
struct ArmTcgShape {
  static constexpr int K0 = rup(C + 1, 8), K1 = rup(NH + 1, 8);
  static constexpr int XC = K0 > NH ? K0 : NH;
  static constexpr int YC = K1, DC = NH;
  static constexpr int SLOT = XC + YC + DC;  // TMEM columns per warpgroup
  static constexpr int NWG = (512 / SLOT) < 6 ? (512 / SLOT) : 6;
  static constexpr int THREADS = NWG * 128;
  static constexpr int WIN = ARM_SH * ARM_SW;
  static constexpr int WINP = (WIN + 31) / 32 * 32;
  // TMA box: 80 x 11 int16 from column j0 - 8 (the innermost start coordinate
  // must be 16-byte aligned -- a box at j0 - 4 faults with "illegal
  // instruction", tools/microbench/tma_probe.cu); the window is columns 4 .. 75
  static constexpr int RAWW = ARM_SW + 8;
  static constexpr int RAWB = (RAWW * ARM_SH * 2 + 127) / 128 * 128;  // bytes per raw buffer, 128-aligned
  static constexpr size_t smem_bytes(int b_floats, bool tma) {
    return sizeof(float) * ((size_t)b_floats + (size_t)NWG * WINP) + (tma ? (size_t)NWG * 2 * RAWB : 0) +
           8 * 3 * NWG + 16;
  }
  static_assert(NH % 8 == 0 && C % 8 == 0, "MMA N and K steps of 8");
  static_assert(ARM_TX % 8 == 0 && ARM_HALO_X == 4, "TMA box origin j0 - 8 is 16-byte aligned");
  static_assert(K1 - NH == 8 && K0 - C == 8, "one 8-column bias block");
};

// predicated 16-bit load (0 when !ok): a PTX predicate, so ptxas keeps every
// load of a batch in flight instead of branching around each one
__device__ __forceinline__ int16_t ldg_s16_pred(const int16_t* ptr, bool ok) {
  int16_t v;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\tmov.b16 %0, 0;\n\t@p ld.global.nc.b16 %0, [%1];\n\t}"
               : "=h"(v)
               : "l"(ptr), "r"((int)ok));
  return v;
}

__device__ __forceinline__ void wg_sync(int g) { asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory"); }

// The context template of reading #4 (SPEC.md:256's nearest-causal list) as
// compile-time shared-memory offsets dy * ARM_SW + dx: the gather becomes
// plain LDS [R + imm].  Descriptors with another template run STD = false.
constexpr int kStdCtx[24][2] = {{0, -1},  {0, -2},  {-1, 0},  {-1, -1}, {-1, 1},  {-1, -2}, {-1, 2},  {0, -3},
                                {-2, 0},  {-2, -1}, {-2, 1},  {-1, -3}, {-1, 3},  {-2, -2}, {-2, 2},  {-2, -3},
                                {-2, 3},  {-3, 0},  {-3, -1}, {-3, 1},  {-3, -2}, {-3, 2},  {0, -4},  {-1, -4}};
__host__ __device__ constexpr int std_ctx_dy(int c) {
  return c == 0 || c == 1 || c == 7 || c == 22 ? 0 : (c <= 6 || c == 11 || c == 12 || c == 23) ? -1 : c <= 16 ? -2 : -3;
}
__host__ __device__ constexpr int std_ctx_dx(int c) {
  constexpr int dx[24] = {-1, -2, 0, -1, 1, -2, 2, -3, 0, -1, 1, -3, 3, -2, 2, -3, 3, 0, -1, 1, -2, 2, -4, -4};
  return dx[c];
}
static bool is_std_ctx(const cc_model_desc& d) {
  if (d.n_ctx > 24) return false;
  for (int c = 0; c < d.n_ctx; c++)
    if (d.ctx_dy[c] != kStdCtx[c][0] || d.ctx_dx[c] != kStdCtx[c][1] || std_ctx_dy(c) != kStdCtx[c][0] ||
        std_ctx_dx(c) != kStdCtx[c][1])
      return false;
  return true;
}

template <int C, int NH, int NHL, bool STD, bool TMA>
__global__ void __launch_bounds__(ArmTcgShape<C, NH>::THREADS, 1)
    arm_tcg_kernel(const __grid_constant__ ArmTcParams<C, NH, NHL> p) {
  using S = ArmTcShape<C, NH, NHL>;
  using G = ArmTcgShape<C, NH>;
  constexpr int K0 = S::K0, K1 = S::K1, NWG = G::NWG;
  static_assert(K0 == G::K0 && K1 == G::K1, "shapes");
  extern __shared__ __align__(1024) float tsm[];
  float* sB = tsm;                      // B0 hi, lo | B1 hi, lo (canonical K-major)
  float* wins = tsm + S::B_FLOATS;      // one causal window per warpgroup (fp32)
  int16_t* raws = reinterpret_cast<int16_t*>(wins + NWG * G::WINP);  // TMA: 2 int16 windows per warpgroup
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(raws) + (TMA ? NWG * 2 * G::RAWB : 0));
  uint64_t* tbars = bars + NWG;         // TMA: 2 per warpgroup
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tbars + 2 * NWG);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int g = warp >> 2, qd = warp & 3, tw = t & 127;  // warpgroup, lane quadrant, latent of the block
  {
    const float4* src0 = reinterpret_cast<const float4*>(&p.B0[0][0]);
    float4* dst = reinterpret_cast<float4*>(sB);
    for (int i = t; i < 2 * S::BW0 / 4; i += G::THREADS) dst[i] = src0[i];
    const float4* src1 = reinterpret_cast<const float4*>(&p.B1[0][0][0]);
    for (int i = t; i < 2 * S::BW1 / 4; i += G::THREADS) dst[2 * S::BW0 / 4 + i] = src1[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t < 3 * NWG) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + t)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);  // this warp's lanes
  const uint32_t cX = (uint32_t)(g * G::SLOT), cY = cX + G::XC, cD = cY + G::YC;
  // the constant bias input of A1_hi (Y columns NH .. K1-1), written once
  {
    float cst[8] = {1.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    tmem_st_cols<8>(tl + cY + NH, cst);
    tmem_wait_st();
  }
  float* win = wins + g * G::WINP;
  uint64_t* bar = bars + g;
  uint32_t phase = 0;
  constexpr uint32_t IDESC =
      (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NH >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
  const uint32_t sB_u = smem_u32(sB);
  // B descriptors of k-step 0 (hi); lo = hi + LO (address units of 16 bytes)
  const uint64_t dB0 = umma_desc(sB_u, 128, (K0 / 4) * 128);
  const uint64_t dB1 = umma_desc(sB_u + 8 * S::BW0, 128, (K1 / 4) * 128);
  constexpr uint32_t LO0 = (4 * S::BW0) >> 4, LO1 = (4 * S::BW1) >> 4;

  const int n_tiles = p.g.tile_begin[p.g.L];
  const int stride = (int)gridDim.x * NWG;
  // (level, i0, j0) of a tile
  auto locate = [&](int tile, int& l, int& i0, int& j0) {
    l = 0;
#pragma unroll 1
    while (l + 1 < p.g.L && tile >= p.g.tile_begin[l + 1]) l++;
    const int tt = tile - p.g.tile_begin[l];
    const int ty = tt / p.g.tiles_x[l];
    i0 = p.g.own_lo[l] + ty * ARM_TY;
    j0 = (tt - ty * p.g.tiles_x[l]) * ARM_TX;
  };
  // TMA: one elected thread loads a tile's int16 window (zero fill outside
  // the grid = reading #5's padding) into raw buffer b, completing tbars[2g+b]
  int16_t* raw = raws + g * G::RAWB;  // [2][RAWB / 2]
  auto tma_window = [&](int tile, int b) {
    int tl, ti0, tj0;
    locate(tile, tl, ti0, tj0);
    uint64_t* tb = tbars + 2 * g + b;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(tb)), "r"(2 * G::RAWW * ARM_SH)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(raw + b * (G::RAWB / 2))),
        "l"(reinterpret_cast<uint64_t>(&p.tmap[tl])), "r"(smem_u32(tb)), "r"(tj0 - ARM_HALO_X - 4),
        "r"(ti0 - ARM_HALO_TOP - p.g.lv.lo[tl])
        : "memory");
  };
  if (TMA && tw == 0 && (int)blockIdx.x * NWG + g < n_tiles) tma_window((int)blockIdx.x * NWG + g, 0);
  int it = 0;
#pragma unroll 1
  for (int tile = (int)blockIdx.x * NWG + g; tile < n_tiles; tile += stride, it++) {
    int l, i0, j0;
    locate(tile, l, i0, j0);
    const int w = p.g.lv.w[l], rlo = p.g.lv.lo[l], rhi = p.g.lv.hi[l];
    if constexpr (TMA) {
      // prefetch the next tile's window into the other buffer (its previous
      // contents were converted before this warpgroup's last staging barrier)
      if (tw == 0 && tile + stride < n_tiles) tma_window(tile + stride, (it + 1) & 1);
      mbar_wait(tbars + 2 * g + (it & 1), (it >> 1) & 1);
      // int16 -> fp32, 4 elements per step (a window row = 18 groups of 4 =
      // raw columns 4 .. 75 of the 80-column box)
      const int16_t* rb = raw + (it & 1) * (G::RAWB / 2);
      for (int u = tw; u < G::WIN / 4; u += 128) {
        const int rr = u / (ARM_SW / 4), kk = u - rr * (ARM_SW / 4);
        const uint2 q = *reinterpret_cast<const uint2*>(rb + rr * G::RAWW + 4 + 4 * kk);
        float4 f;
        f.x = (float)(int16_t)(q.x & 0xFFFFu);
        f.y = (float)(int16_t)(q.x >> 16);
        f.z = (float)(int16_t)(q.y & 0xFFFFu);
        f.w = (float)(int16_t)(q.y >> 16);
        *reinterpret_cast<float4*>(win + 4 * u) = f;
      }
      wg_sync(g);
    } else
    {  // causal window of the tile (fp32, zero outside the grid); every
       // thread of this warpgroup passed the previous tile's last pre-MMA
       // barrier, so the previous window has no reader left.  Element e =
       // (r, c) of the 11 x 72 window, e = tw + 128 k: 32-bit offsets from
       // the window origin, bounds checks only on edge tiles.
      const int16_t* __restrict__ base = p.lat + p.g.lv.off[l] + (int64_t)(i0 - ARM_HALO_TOP - rlo) * w + (j0 - ARM_HALO_X);
      const bool inner = i0 - ARM_HALO_TOP >= rlo && i0 + ARM_TY <= rhi && j0 - ARM_HALO_X >= 0 && j0 + ARM_TX + ARM_HALO_X <= w;
      constexpr int IT = (G::WIN + 127) / 128;
      int16_t v[IT];
      int off[IT];
      bool ok[IT];
      int r = tw / ARM_SW, c = tw - (tw / ARM_SW) * ARM_SW;
#pragma unroll
      for (int k = 0; k < IT; k++) {  // offsets and predicates first (no branches) ...
        const int gi = i0 - ARM_HALO_TOP + r, gj = j0 - ARM_HALO_X + c;
        ok[k] = ((k < IT - 1) || (tw + 128 * k < G::WIN)) &&
                (inner || (gi >= rlo && gi < rhi && gj >= 0 && gj < w));
        off[k] = r * w + c;
        c += 128 - ARM_SW;  // + 128 elements = + 1 row + 56 columns, at most one wrap
        const bool wrap = c >= ARM_SW;
        c -= wrap ? ARM_SW : 0;
        r += wrap ? 2 : 1;
      }
#pragma unroll
      for (int k = 0; k < IT; k++) v[k] = ldg_s16_pred(base + off[k], ok[k]);  // ... then every load in flight
#pragma unroll
      for (int k = 0; k < IT; k++) {
        const int e = tw + k * 128;
        if ((k < IT - 1) || e < G::WIN) win[e] = (float)v[k];
      }
      wg_sync(g);
    }
    float tbits = 0.0f;  // this thread's bits over the tile's 4 blocks
#pragma unroll 1
    for (int q = 0; q < ARM_TY / 2; q++) {
      const int ry = 2 * q + (tw >> 6), cx = tw & 63;
      const float* center = win + (ry + ARM_HALO_TOP) * ARM_SW + cx + ARM_HALO_X;
      const float y = center[0];
      {  // A0 row: [context (C), 1, 0 x 7]
        float row[C], tail[8] = {1.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c = 0; c < C; c++) row[c] = center[STD ? std_ctx_dy(c) * ARM_SW + std_ctx_dx(c) : p.g.ctx_off[c]];
        tmem_st_cols<C>(tl + cX, row);
        tmem_st_cols<8>(tl + cX + C, tail);
        tmem_wait_st();
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      wg_sync(g);
      if (qd == (q & 3)) {  // MMA0: D0 = A0 B0_hi + A0 B0_lo (one elected lane; the issuing warp rotates)
        asm volatile("tcgen05.fence::after_thread_sync;");
        mma_batch_hilo<K0 / 8>(tmem + cY, tmem + cX, dB0, IDESC, bar, LO0);
      }
      mbar_wait_sleep(bar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      {  // epilogue 0: ReLU, z = hi + lo (hi = z truncated to tf32: exact split)
        float z[NH], lo[NH];
        tmem_ld_cols<NH>(tl + cY, z);
#pragma unroll
        for (int n = 0; n < NH; n += 2) {
          const float r0 = fmaxf(z[n], 0.0f), r1 = fmaxf(z[n + 1], 0.0f);
          z[n] = __uint_as_float(__float_as_uint(r0) & 0xFFFFE000u);
          z[n + 1] = __uint_as_float(__float_as_uint(r1) & 0xFFFFE000u);
          const float2 d = f2unpack(fsub2(f2pack(r0, r1), f2pack(z[n], z[n + 1])));  // exact
          lo[n] = d.x;
          lo[n + 1] = d.y;
        }
        tmem_st_cols<NH>(tl + cY, z);
        tmem_st_cols<NH>(tl + cX, lo);
        tmem_wait_st();
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      wg_sync(g);
      if (qd == (q & 3)) {  // MMA1: D1 = A1_hi B1_hi + A1_hi B1_lo + A1_lo B1_hi
        asm volatile("tcgen05.fence::after_thread_sync;");
        mma_batch_3x<K1 / 8, NH / 8>(tmem + cD, tmem + cY, tmem + cX, dB1, IDESC, bar, LO1);
      }
      mbar_wait_sleep(bar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      // epilogue 1: ReLU, output layer (mu, log-scale), Laplace bits
      float z[NH];
      tmem_ld_cols<NH>(tl + cD, z);
      // output layer over input pairs (two FFMA2 per pair of hidden units)
      uint64_t am = f2pack(p.bo.x, 0.0f), as = f2pack(p.bo.y, 0.0f);
#pragma unroll
      for (int n = 0; n < NH; n += 2) {
        const uint64_t r2 = f2pack(fmaxf(z[n], 0.0f), fmaxf(z[n + 1], 0.0f));
        am = ffma2(r2, ldp2(p.wm[n / 2]), am);
        as = ffma2(r2, ldp2(p.wsl[n / 2]), as);
      }
      const float2 m2 = f2unpack(am), s2 = f2unpack(as);
      const float mu = m2.x + m2.y, ls = s2.x + s2.y;
      const int i = i0 + ry, j = j0 + cx;
      if (i < p.g.own_hi[l] && j < w) {
        const float bits = laplace_bits(y, mu, ls, p.g);
        tbits += bits;
        if (p.bits != nullptr) {
          const int64_t qi = p.g.lv.off[l] + (int64_t)(i - rlo) * w + j;
          p.bits[qi] = bits;
          if (p.mu) p.mu[qi] = mu;
          if (p.scale) p.scale[qi] = __expf(fminf(fmaxf(ls, p.g.lsmin), p.g.lsmax));
        }
      }
      // D1 / X / Y are rewritten by the next block only after the next
      // pre-MMA barriers, which every thread reaches after its loads here
      asm volatile("tcgen05.fence::before_thread_sync;");
    }
    // one fp64 partial per warp and tile (fixed order: deterministic)
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) tbits += __shfl_xor_sync(0xffffffffu, tbits, o2);
    if (lane == 0) p.partial[(int64_t)tile * 4 + qd] = (double)tbits;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- host launcher
typedef CUresult (*ArmEncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static ArmEncodeTiledFn arm_encode_tiled() {
  static ArmEncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<ArmEncodeTiledFn>(ptr);
    cudaGetLastError();
  }
  return fn;
}

// One 2-D 16-bit tensor map per grid (UINT16: the bits are reinterpreted as int16) (rows present in the buffer x w), box =
// the 11 x 72 causal window; zero fill outside = reading #5's zero padding.
// False (LDG staging instead) when a grid's rows are not 16-byte strided /
// aligned (TMA's requirement) or the encoder is unavailable.
static bool arm_tma_maps(const ArmGeom& g, const int16_t* lat, CUtensorMap* maps) {
  static const bool off = getenv("CCRD_ARM_NO_TMA") && getenv("CCRD_ARM_NO_TMA")[0] == '1';
  if (off) return false;
  ArmEncodeTiledFn enc = arm_encode_tiled();
  if (!enc) return false;
  for (int l = 0; l < g.L; l++) {
    const int64_t w = g.lv.w[l], rows = g.lv.hi[l] - g.lv.lo[l];
    const uintptr_t a = reinterpret_cast<uintptr_t>(lat + g.lv.off[l]);
    if (rows < 1 || (w * 2) % 16 != 0 || a % 16 != 0) return false;
  }
  for (int l = 0; l < g.L; l++) {
    const cuuint64_t dims[2] = {(cuuint64_t)g.lv.w[l], (cuuint64_t)(g.lv.hi[l] - g.lv.lo[l])};
    const cuuint64_t strides[1] = {(cuuint64_t)g.lv.w[l] * 2};
    const cuuint32_t box[2] = {(cuuint32_t)(ARM_SW + 8), (cuuint32_t)ARM_SH};  // from column j0 - 8 (16-byte aligned)
    const cuuint32_t es[2] = {1, 1};
    if (enc(&maps[l], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)(lat + g.lv.off[l]), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

// tf32 round-to-nearest (ties away, like cvt.rna) of a finite float
static float tf32_rna_host(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

template <int C, int NH, int NHL>
static int launch_arm_tc(const ArmGeom& g, const cc_model_desc& d, const float* arm_w, const int16_t* lat,
                         double* partial, float* mu, float* scale, float* bits, cudaStream_t stream) {
  using S = ArmTcShape<C, NH, NHL>;
  using P = ArmTcParams<C, NH, NHL>;
  static_assert(sizeof(P) <= 32 * 1024 - 16, "kernel parameters exceed the 32 KB bank");
  P p;  // ~15 KB, copied into the launch's parameter bank
  memset(&p, 0, sizeof(p));
  p.g = g;
  p.lat = lat;
  p.partial = partial;
  p.mu = mu;
  p.scale = scale;
  p.bits = bits;
  auto res = [&](int k) { return (d.arm_residual_mask >> k) & 1u; };
  auto put = [](float* hi, float* lo, int n, int k, int K, float v) {
    const float h = tf32_rna_host(v);
    hi[kmaj(n, k, K)] = h;
    lo[kmaj(n, k, K)] = v - h;
  };
  // blob: per layer W[out][in] then b[out]
  const float* q = arm_w;
  for (int n = 0; n < NH; n++) {
    for (int i = 0; i < C; i++) put(p.B0[0], p.B0[1], n, i, S::K0, q[n * C + i] + ((res(0) && i == n) ? 1.0f : 0.0f));
    put(p.B0[0], p.B0[1], n, C, S::K0, q[C * NH + n]);
  }
  q += C * NH + NH;
  for (int k = 0; k < NHL - 1; k++) {
    for (int n = 0; n < NH; n++) {
      for (int i = 0; i < NH; i++)
        put(p.B1[k][0], p.B1[k][1], n, i, S::K1, q[n * NH + i] + ((res(k + 1) && i == n) ? 1.0f : 0.0f));
      put(p.B1[k][0], p.B1[k][1], n, NH, S::K1, q[NH * NH + n]);
    }
    q += NH * NH + NH;
  }
  for (int i = 0; i < NH; i++) p.wo[i] = make_float2(q[i], q[NH + i]);
  for (int i = 0; i < NH / 2; i++) {
    p.wm[i] = make_float2(q[2 * i], q[2 * i + 1]);
    p.wsl[i] = make_float2(q[NH + 2 * i], q[NH + 2 * i + 1]);
  }
  p.bo = make_float2(q[2 * NH], q[2 * NH + 1]);

  const int tiles = g.tile_begin[g.L];
  if (tiles == 0) return 0;
  static const bool ss = getenv("CCRD_ARM_TC_SS") && getenv("CCRD_ARM_TC_SS")[0] == '1';  // the serial version
  static const bool ws = getenv("CCRD_ARM_TC_WS") && getenv("CCRD_ARM_TC_WS")[0] == '1';  // warp-specialised
  if constexpr (NHL == 2) {
    if (!ss && !ws) {  // default: warpgroup pipelines
      using G = ArmTcgShape<C, NH>;
      constexpr size_t smem_t = G::smem_bytes(S::B_FLOATS, true), smem_n = G::smem_bytes(S::B_FLOATS, false);
      static bool attr_g = false;
      if (!attr_g) {
        cudaFuncSetAttribute(arm_tcg_kernel<C, NH, NHL, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
        cudaFuncSetAttribute(arm_tcg_kernel<C, NH, NHL, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
        cudaFuncSetAttribute(arm_tcg_kernel<C, NH, NHL, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_n);
        cudaFuncSetAttribute(arm_tcg_kernel<C, NH, NHL, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_n);
        attr_g = true;
      }
      const bool tma = arm_tma_maps(g, lat, p.tmap);
      const int need = (tiles + G::NWG - 1) / G::NWG, cap = device_sm_count();
      const bool sc = is_std_ctx(d);
      auto kern = tma ? (sc ? arm_tcg_kernel<C, NH, NHL, true, true> : arm_tcg_kernel<C, NH, NHL, false, true>)
                      : (sc ? arm_tcg_kernel<C, NH, NHL, true, false> : arm_tcg_kernel<C, NH, NHL, false, false>);
      kern<<<need < cap ? need : cap, G::THREADS, tma ? smem_t : smem_n, stream>>>(p);
      return 1;
    }
    if (!ss) {
      using W = ArmTcwShape<C, NH, NHL>;
      static bool attr_w = false;
      if (!attr_w) {
        cudaFuncSetAttribute(arm_tcw_kernel<C, NH, NHL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W::SMEM);
        attr_w = true;
      }
      const int per_sm = (int)((227u * 1024u) / W::SMEM) < 1 ? 1 : (int)((227u * 1024u) / W::SMEM);
      const int cap = per_sm * device_sm_count();
      arm_tcw_kernel<C, NH, NHL><<<tiles < cap ? tiles : cap, TW_THREADS, W::SMEM, stream>>>(p);
      return 1;
    }
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(arm_tc_kernel<C, NH, NHL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
    attr = true;
  }
  const int cap = TC_CTAS_PER_SM * device_sm_count();
  arm_tc_kernel<C, NH, NHL><<<tiles < cap ? tiles : cap, TC_THREADS, S::SMEM, stream>>>(p);
  return 1;
}

struct ArmTcEntry {
  int C, NH, NHL;
  ArmLaunchFn fn;
};

// Tensor-core ARM shapes: the ~2000 MAC/pixel config ([16,24,24,2]) and the
// Table 1 wider ARMs (A1079 [16,16,16,2], A2300 [24,24,24,2]).
static const ArmTcEntry kArmTc[] = {
    {16, 24, 2, launch_arm_tc<16, 24, 2>},
    {16, 16, 2, launch_arm_tc<16, 16, 2>},
    {24, 24, 2, launch_arm_tc<24, 24, 2>},
};

// rate partials per 8 x 64 tile written by the selected tensor-core kernel
int arm_tc_partials_per_tile() {
  static const bool ss = getenv("CCRD_ARM_TC_SS") && getenv("CCRD_ARM_TC_SS")[0] == '1';
  static const bool ws = getenv("CCRD_ARM_TC_WS") && getenv("CCRD_ARM_TC_WS")[0] == '1';
  return (ss || ws) ? 16 : 4;
}

ArmLaunchFn find_arm_tc_launcher(int C, int NH, int NHL) {
  for (const auto& e : kArmTc)
    if (e.C == C && e.NH == NH && e.NHL == NHL) return e.fn;
  return nullptr;
}

}  // namespace ccrd
