// synth.cu -- fused upsampling f_upsilon + synthesis f_theta + distortion.
//
// One CTA produces a 32 x 64 tile of x_hat ("upsample the
// latents to a dense representation and synthesize the decoded image";
// Table 1 upsampling / synthesis columns; Eq. 1 distortion):
//   1. last x2 upsampling step.  pyramid.cu has already carried grids 2..L-1
//      to level 1 (S_1); the tile stages grid 1 + S_1 over its level-1 window
//      (replicate padding = clamped reads) and runs the horizontal pass of the
//      separable stride-2 transposed conv into shared memory.
//   2. per PAIR of rows (2q, 2q+1) of the tile + halo: the last vertical step
//      (both phases share the K/2 + 1 source rows) and the L -> C_h -> 3 1x1
//      MLP for both pixels in registers (packed FFMA2, two neurons per
//      instruction, each uniform weight load feeding two pixels).
//   3. residual 3x3 layers: each thread owns a column segment of 8 rows and,
//      per input channel, loads its 10 x 3 window once; every uniform weight
//      feeds 8 outputs.  The halo ring of the non-last layers is recomputed,
//      never exchanged; replicate padding at the image border is index
//      clamping.
//   4. the last layer's output goes straight from registers to x_hat
//      (optional) and the (x - x_hat)^2 partial sum -> fp64 per CTA.
// The dense L x H x W tensor is never materialised in HBM.
#include <cstdlib>

#include "ccrd_common.cuh"

#ifndef CCRD_SYN_VSCALAR
#define CCRD_SYN_VSCALAR 0  // last vertical step on scalar FMAs (experiment)
#endif
#ifndef CCRD_SYN_MC
#define CCRD_SYN_MC 20  // hidden neurons per MLP chunk (live accumulators)
#endif


namespace ccrd {

#ifdef CCRD_SYN_TIMING
// experiment build: per-CTA phase timestamps [cta][8] (clock64), read back by
// cc_debug_syn_timing (tools/ only)
__device__ unsigned long long g_syn_timing[1 << 16][8];
#define SYN_MARK(k)                                                               \
  if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) {                                \
    unsigned long long t;                                                          \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));                              \
    g_syn_timing[blockIdx.x][k] = t;                                               \
  }
#else
#define SYN_MARK(k)
#endif

// Window sizes of the upsampling chain (compile time).  Level 0's window is the
// tile + an even halo RE; level j+1's window starts at ((lo_j >> 1) - K/4)
// rounded down to even and holds n_j/2 + K/2 + 1 entries rounded up to even --
// every source index the x2 step from level j+1 to level j touches.
template <int K>
__host__ __device__ constexpr int wnext(int n) {
  return ((n / 2 + K / 2 + 1) + 1) & ~1;
}
template <int K>
__host__ __device__ constexpr int wsize(int n0, int j) {
  return j == 0 ? n0 : wnext<K>(wsize<K>(n0, j - 1));
}

template <int L, int CH, int R, int K>
struct SynShape {
  static constexpr int RE = 2 * ((R + 1) / 2);   // even halo of the level-0 region
  static constexpr int RH0 = SYN_TH + 2 * RE;    // level-0 region rows
  static constexpr int RW0 = SYN_TW + 2 * RE;    // level-0 region cols
  static constexpr int NR1 = wsize<K>(RH0, 1);   // level-1 window (largest of levels >= 1)
  static constexpr int NC1 = wsize<K>(RW0, 1);
  static constexpr int NS = (L > 1) ? (L - 1) : 1;  // stack slots (levels 1..L-1)
  static constexpr int SLOT = NR1 * NC1;            // stack slot (floats)
  static constexpr int TSLOT = NR1 * RW0;           // tmph slot (floats)
  static constexpr int STACK = NS * SLOT;
  static constexpr int HBUF = 3 * RH0 * RW0;
  static constexpr int BUF_A = (STACK > HBUF) ? STACK : HBUF;  // stack | h (ping)
  static constexpr int TMPH = NS * TSLOT;
  static constexpr int BUF_B = (TMPH > HBUF) ? TMPH : HBUF;    // tmph  | h (pong)
  // int16 level-0 region [RH0][LP]: region column c at LO + c, so that the
  // TMA box origin RX - LO is 16-byte aligned (RX = X0 - RE, X0 a multiple of 8)
  static constexpr int LO = (-RE) & 7;
  static constexpr int LP = (LO + RW0 + 7) & ~7;
  static constexpr int LAT0 = ((RH0 * LP + 1) / 2);            // int16 level-0 region, in floats
  static constexpr size_t SMEM = sizeof(float) * (size_t)(BUF_A + BUF_B + LAT0);
  // ---- TMA-staged variant (synth_kernel<..., TMA = true>)
  // level-1 window origin lc = X0 / 2 + A1 (X0 / 2 a multiple of 8); S_1 (fp32)
  // boxes need lc 16-byte aligned, grid 1 (int16) is boxed from lc - G0
  static constexpr int A1 = (-(RE / 2) - K / 4) & ~1;
  static constexpr int G0 = A1 & 7;
  static constexpr int GP = (G0 + NC1 + 7) & ~7;  // grid-1 raw pitch (int16)
  static constexpr bool TMA_OK = (L >= 3) && (A1 & 3) == 0 && (NC1 % 4) == 0 && NC1 <= 256 && NR1 <= 256 &&
                                 LP <= 256 && RH0 <= 256 && SYN_TW % 16 == 0 && NR1 * GP * 2 <= 4 * BUF_B;
  static constexpr int al128(int b) { return (b + 127) & ~127; }
  // byte offsets from a 128-aligned base: bufA (= the stack) placed so that
  // stack slot 1 (the S_1 box) is 128-aligned, bufB (holds the grid-1 box until
  // the conversion into slot 0), lat0
  static constexpr int T_A = (128 - (SLOT * 4) % 128) % 128;
  static constexpr int T_B = al128(T_A + BUF_A * 4);
  static constexpr int T_L = al128(T_B + BUF_B * 4);
  static constexpr size_t SMEM_TMA = (size_t)T_L + (size_t)RH0 * LP * 2 + 128;  // + alignment slack
  static constexpr uint32_t TMA_BYTES = (uint32_t)((L - 2) * SLOT * 4 + NR1 * GP * 2 + RH0 * LP * 2);
  // MLP = 1: the 1x1 weights (A0t, a0, A1: contiguous in SynWeights) copied
  // once per CTA, so that each lane reads its MMA fragments without
  // lane-divergent constant-bank loads
  static constexpr int WRAW = L * CH + CH + 3 * CH;
  static constexpr size_t SMEM_MMA = SMEM + sizeof(float) * (size_t)WRAW;
  static constexpr int NWARPS = SYN_THREADS / 32;
  static constexpr int SEGS = SYN_THREADS / SYN_TW;            // column segments per tile column
  static constexpr int RS = SYN_TH / SEGS;                      // rows per segment
  static_assert(SYN_THREADS % SYN_TW == 0 && SYN_TH % SEGS == 0, "conv mapping");
  static_assert(SYN_TH % 2 == 0 && SYN_TW % 2 == 0, "even tiles");
};

struct SynCtx {
  float* stack;   // [slot][NR_j][NC_j]      (slot = level - 1)
  float* tmph;    // [slot][NR_{j+1}][NC_j]
  int* wlo_r;     // window origins (shared), per level
  int* wlo_c;
};

// Level-1 staging: slot 0 = grid 1 (int16 latents), slots 1 .. L-2 = S_1
// (grids 2 .. L-1 already upsampled to level 1 by pyramid.cu), each over the
// level-1 window, replicate-extended (clamped reads).  Every thread issues all
// of its loads before the first store.
template <int L, int CH, int R, int K>
struct LoadLevel1 {
  using S = SynShape<L, CH, R, K>;
  static constexpr int NR = S::NR1, NC = S::NC1;
  static constexpr int IT = (NR * NC + SYN_THREADS - 1) / SYN_THREADS;
  static __device__ __forceinline__ void run(const SynParams<L, CH, R, K>& p, const SynCtx& c) {
    const int gw = p.g.lv.w[1], blo = p.g.lv.lo[1], bhi = p.g.lv.hi[1];  // buffer window of level 1
    const int lr = c.wlo_r[1], lc = c.wlo_c[1];
    const int16_t* g1 = p.lat + p.g.lv.off[1];
    const int64_t plane = (int64_t)(bhi - blo) * gw;
    float v[L - 1][IT];
#pragma unroll
    for (int k = 0; k < IT; k++) {
      const int it = threadIdx.x + k * SYN_THREADS;
      const int rr = it / NC, cc = it - rr * NC;
      const int64_t gi = (int64_t)(clampi(lr + rr, blo, bhi - 1) - blo) * gw + clampi(lc + cc, 0, gw - 1);
      const bool ok = it < NR * NC;
      v[0][k] = ok ? (float)__ldg(g1 + gi) : 0.0f;
#pragma unroll
      for (int sl = 1; sl < L - 1; sl++) v[sl][k] = ok ? __ldg(p.s1 + (int64_t)(sl - 1) * plane + gi) : 0.0f;
    }
#pragma unroll
    for (int sl = 0; sl < L - 1; sl++)
#pragma unroll
      for (int k = 0; k < IT; k++) {
        const int it = threadIdx.x + k * SYN_THREADS;
        if (it < NR * NC) c.stack[sl * S::SLOT + it] = v[sl][k];
      }
  }
};

template <int L, int CH, int R, int K>
struct LoadLat0 {
  using S = SynShape<L, CH, R, K>;
  static constexpr int N = S::RH0 * S::RW0;
  static constexpr int IT = (N + SYN_THREADS - 1) / SYN_THREADS;
  static __device__ __forceinline__ void run(const SynParams<L, CH, R, K>& p, int16_t* lat0, int RY, int RX) {
    const int W = p.g.W, blo = p.g.lv.lo[0], bhi = p.g.lv.hi[0];  // buffer window of level 0
    int16_t v[IT];
#pragma unroll
    for (int k = 0; k < IT; k++) {
      const int it = threadIdx.x + k * SYN_THREADS;
      const int rr = it / S::RW0, cc = it - rr * S::RW0;
      v[k] = (it < N) ? __ldg(p.lat + (int64_t)(clampi(RY + rr, blo, bhi - 1) - blo) * W + clampi(RX + cc, 0, W - 1))
                      : 0;
    }
#pragma unroll
    for (int k = 0; k < IT; k++) {
      const int it = threadIdx.x + k * SYN_THREADS;
      const int rr = it / S::RW0, cc = it - rr * S::RW0;
      if (it < N) lat0[rr * S::LP + S::LO + cc] = v[k];
    }
  }
};

// Horizontal pass of the x2 step from level J+1 to level J (J = 0 here) for
// every grid l > J (stack slots J .. L-2); the vertical pass of the last step is
// done per pixel pair in phase 2.  out[2q + r] = sum_t k[2t + 1 - r] g[q + r + K/4 - 1 - t]
// (stride-2 transposed conv on the replicate-extended input, DESIGN.md readings
// #12-#13): the even and odd outputs share the K/2 + 1 sources
// g[q - K/4 .. q + K/4]; replicate padding = clamping the SOURCE index.
template <int L, int CH, int R, int K, int J>
struct ChainStep {
  using S = SynShape<L, CH, R, K>;
  static constexpr int NRs = wsize<K>(S::RH0, J + 1), NCs = wsize<K>(S::RW0, J + 1);  // source window
  static constexpr int NRd = wsize<K>(S::RH0, J), NCd = wsize<K>(S::RW0, J);          // dest window
  static constexpr int NSL = L - 1 - J;

  static __device__ __forceinline__ void run(const SynParams<L, CH, R, K>& p, const SynCtx& c) {
    const float* kk = p.w.k;
    // ---- horizontal: (rows of window J+1) x (cols of window J); each thread
    // owns PPT adjacent column pairs of a row (PPT = 2: 6 loads feed 4
    // outputs, one 16-byte store), the same FMA order per output
    {
      constexpr int NCP = NCd / 2;
      constexpr int PPT = (NCP % 2 == 0 && NCd % 4 == 0 && S::TSLOT % 4 == 0 && S::BUF_A % 4 == 0) ? 2 : 1;
      constexpr int NCQ = NCP / PPT;
      constexpr int NRG = SYN_THREADS / NCQ;
      constexpr int NSV = K / 2 + PPT;  // sources of PPT pairs
      const int cq = threadIdx.x % NCQ, rg = threadIdx.x / NCQ;
      if (rg < NRG) {
        const int q = (c.wlo_c[J] >> 1) + PPT * cq;  // (lo_c[J] + 2 PPT cq) / 2; lo_c[J] even
        const int ws = p.g.lv.w[J + 1], lo_s = c.wlo_c[J + 1];
        int off[NSV];
#pragma unroll
        for (int u = 0; u < NSV; u++) off[u] = clampi(q - K / 4 + u, 0, ws - 1) - lo_s;
#pragma unroll 2
        for (int k = rg; k < NSL * NRs; k += NRG) {
          const int sl = k / NRs, row = k - sl * NRs;
          const float* src = c.stack + (J + sl) * S::SLOT + row * NCs;
          float sv[NSV];
#pragma unroll
          for (int u = 0; u < NSV; u++) sv[u] = src[off[u]];
          float a[2 * PPT];
#pragma unroll
          for (int pr = 0; pr < PPT; pr++) {
            float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
            for (int t = 0; t < K / 2; t++) {
              a0 = fmaf(kk[2 * t + 1], sv[pr + K / 2 - 1 - t], a0);
              a1 = fmaf(kk[2 * t], sv[pr + K / 2 - t], a1);
            }
            a[2 * pr] = a0;
            a[2 * pr + 1] = a1;
          }
          float* dst = c.tmph + (J + sl) * S::TSLOT + row * NCd + 2 * PPT * cq;
          if constexpr (PPT == 2)
            *reinterpret_cast<float4*>(dst) = make_float4(a[0], a[1], a[2], a[3]);
          else
            *reinterpret_cast<float2*>(dst) = make_float2(a[0], a[1]);
        }
      }
    }
    __syncthreads();
  }
};

// 1x1 synthesis layers L -> CH (ReLU) -> 3 (ReLU unless R == 0: the module's
// last layer) for a PAIR of pixels (rows 2q, 2q+1) held in the two lanes of
// every FFMA2: v[i] = (pixel 0, pixel 1) of input channel i, and each weight
// is a broadcast uniform operand (UR.F32), so one instruction does one MAC of
// both pixels and 4 weights come per uniform load.  Per neuron: bias first,
// then the inputs in order (the oracle's summation order).
template <int L, int CH, int R, int K>
__device__ __forceinline__ void mlp_pair(const SynParams<L, CH, R, K>& p, const uint64_t (&v)[L], uint64_t (&out)[3]) {
  // hidden layer in chunks of MC neurons: fewer live accumulators (each chunk
  // adds its contribution to the three output pairs), same FMA count and the
  // same per-output summation order as one pass (bias, then hidden 0 .. CH-1)
  constexpr int MC = (CH % CCRD_SYN_MC == 0 && CH > CCRD_SYN_MC) ? CCRD_SYN_MC : CH;
  const uint64_t one = f2pack(1.0f, 1.0f);
  uint64_t o[3];
#pragma unroll
  for (int c = 0; c < 3; c++) o[c] = ffma2(one, f2pack(p.w.a1[c], p.w.a1[c]), 0ull);
#pragma unroll
  for (int n0 = 0; n0 < CH; n0 += MC) {
    uint64_t acc[MC];
    // the bias is the addend of the first input's FMA: fma(v0, w, b) equals
    // fma(v0, w, 0 + b) bit for bit and saves one FMA-pipe instruction (a
    // FADD2) per neuron -- the 1x1 stack is FMA-pipe bound (-2.2 % kernel time)
#pragma unroll
    for (int n = 0; n < MC; n++)
      acc[n] = ffma2(v[0], f2pack(p.w.A0t[0][n0 + n], p.w.A0t[0][n0 + n]), f2pack(p.w.a0[n0 + n], p.w.a0[n0 + n]));
#pragma unroll
    for (int i = 1; i < L; i++)
#pragma unroll
      for (int n = 0; n < MC; n++) acc[n] = ffma2(v[i], f2pack(p.w.A0t[i][n0 + n], p.w.A0t[i][n0 + n]), acc[n]);
#pragma unroll
    for (int n = 0; n < MC; n++) {
      const float2 h = f2unpack(acc[n]);
      acc[n] = f2pack(fmaxf(h.x, 0.0f), fmaxf(h.y, 0.0f));
    }
#pragma unroll
    for (int c = 0; c < 3; c++)
#pragma unroll
      for (int n = 0; n < MC; n++) o[c] = ffma2(acc[n], f2pack(p.w.A1[c][n0 + n], p.w.A1[c][n0 + n]), o[c]);
  }
#pragma unroll
  for (int c = 0; c < 3; c++) {
    if (R > 0) {
      const float2 h = f2unpack(o[c]);
      o[c] = f2pack(fmaxf(h.x, 0.0f), fmaxf(h.y, 0.0f));
    }
    out[c] = o[c];
  }
}

// x = v / 255 correctly rounded in fp32 without a division: q0 = v r
// (r = fp32(1/255)), one FMA residual correction.  Verified equal to the IEEE
// quotient float32(v) / float32(255) for all 256 values of v (exact rational
// check, reading 23); no slow-path call, no extra registers.
__device__ __forceinline__ float u8_to_x(uint32_t v) {
  const float fv = (float)v, r = 0.003921568859368562698364f;  // fp32(1/255)
  const float q0 = __fmul_rn(fv, r);
  return __fmaf_rn(__fmaf_rn(-q0, 255.0f, fv), r, q0);
}
// the target image x at plane offset i: fp32, or 8-bit (IMG8 = desc.image_u8)
template <bool IMG8, class P>
__device__ __forceinline__ float load_x(const P& p, int64_t i) {
  if constexpr (IMG8)
    return u8_to_x(__ldg(p.image8 + i));
  else
    return __ldg(p.image + i);
}

// ------------------------------------------- 1x1 layer 0 on the tensor cores
// Legacy warp MMA (mma.sync m16n8k8 tf32; HMMA.1688 on sm_100a, 1024 MACs per
// warp instruction, 512 MAC/clk/SM measured -- tools/microbench/hmma_probe.cu)
// needs no TMEM, so it coexists with the tensor-core ARM CTA that holds all of
// its SM's TMEM.  fp32 accuracy through the 3xTF32 split: x = hi + lo with hi
// = x rounded to tf32 and lo = x - hi (exact in fp32), D = lo_a hi_b + hi_a
// lo_b + hi_a hi_b (the dropped lo_a lo_b is < 2^-22 |a b|).
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t syn_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// N shared loads a, a + S, a + 2S, ... (32-bit shared addresses: no generic
// window arithmetic inside the loop)
template <int N, int S, int U = 0>
__device__ __forceinline__ void lds_col(uint32_t a, float (&v)[N]) {
  if constexpr (U < N) {
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v[U]) : "r"(a), "n"(U * S));
    lds_col<N, S, U + 1>(a, v);
  }
}
__device__ __forceinline__ int lds_s16(uint32_t a) {
  short v;
  asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
// the same rounding (to nearest, ties away from zero) in two integer ops, for
// finite x (the values here are finite fp32 sums)
__device__ __forceinline__ uint32_t tf32_round(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }
__device__ __forceinline__ void mma_tf32_1688(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ------------------------------------------------ TMA tile staging (TMA = true)
// One mbarrier per CTA; thread 0 arms it with the byte count of a tile's three
// boxes (S_1 slots, grid 1, level-0 region) and issues them; every thread waits
// on the phase parity.
__device__ __forceinline__ void syn_mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(syn_smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void syn_mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t b = syn_smem_u32(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void syn_tma_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          syn_smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(syn_smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void syn_tma_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          syn_smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(syn_smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---- thread-block cluster helpers (CLU: vertical tile pairs)
__device__ __forceinline__ void syn_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// MLP = 0: the 1x1 stack on packed FFMA2 (one thread per vertical pixel pair);
// MLP = 1: layer 0 as warp MMAs over m-tiles of 16 pixels, layer 1 on FFMA2
// (chain mode only, no debug outputs).
// TMA = true (S::TMA_OK shapes, chain mode, MLP = 0): a tile whose windows
// lie inside the latent buffers (no replicate clamping needed) is staged by
// three TMA boxes (S_1 slots, grid 1, level-0 region) that thread 0 issues at
// the CTA's start -- no per-element index math, clamps or register round trip;
// border tiles use the clamped LDG staging.  Both stage the same values, so
// the results are bit-identical.  (Persistent CTAs prefetching the next tile
// measured slower: DESIGN.md 7.4.)
template <int L, int CH, int R, int K, bool DENSE_IN, bool IMG8, int MLP, bool TMA, bool CLU = false>
__global__ void __launch_bounds__(SYN_THREADS, SYN_CTAS_PER_SM)
    synth_kernel(const __grid_constant__ SynParams<L, CH, R, K> p) {
  using S = SynShape<L, CH, R, K>;
  static_assert(!TMA || (S::TMA_OK && !DENSE_IN && MLP == 0), "TMA staging: chain mode, FFMA2 MLP");
  static_assert(!CLU || (TMA && S::RE == 2 && (R == 1 || R == 2)), "vertical pairs: one halo pair-row, one ring row");
  constexpr int RE = S::RE, RH0 = S::RH0, RW0 = S::RW0;
  constexpr int HP = RH0 * RW0;
  constexpr int LP = S::LP, LO = S::LO;
  extern __shared__ float smem[];
  float *bufA, *bufB;
  int16_t* lat0;
  if constexpr (TMA) {  // 128-byte aligned TMA destinations (SynShape T_*)
    char* b = reinterpret_cast<char*>(smem) + ((128u - (syn_smem_u32(smem) & 127u)) & 127u);
    bufA = reinterpret_cast<float*>(b + S::T_A);
    bufB = reinterpret_cast<float*>(b + S::T_B);
    lat0 = reinterpret_cast<int16_t*>(b + S::T_L);
  } else {
    bufA = smem;
    bufB = smem + S::BUF_A;
    lat0 = reinterpret_cast<int16_t*>(smem + S::BUF_A + S::BUF_B);  // [RH0][LP]
  }
  __shared__ int wlo_r[CC_MAX_LEVELS], wlo_c[CC_MAX_LEVELS];
  __shared__ double warp_buf[SYN_THREADS / 32];
  __shared__ uint64_t tbar;
  pdl_trigger();  // the next image's synthesis may be scheduled as this grid drains

  const int H = p.g.H, W = p.g.W;
  const int Ys = p.g.y0, Ye = p.g.y1;  // output rows (full image: 0 .. H); x_hat / image rows are Ys-relative
  // CLU: a cluster of two CTAs = two vertically adjacent tiles (rank 0 on top);
  // each computes the 1x1 stack and the first 3x3 layer for its own rows only
  // and reads the partner's rows it needs as halo through distributed shared
  // memory.  A rank-1 CTA past the last tile row (odd tile rows) only joins
  // the cluster barriers.
  int ty, tx, tile, rank = 0;
  bool partner = false;
  if constexpr (CLU) {
    const int tiles_y = p.g.n_tiles / p.g.tiles_x;
    rank = (int)(blockIdx.x & 1u);
    const int pr = (int)(blockIdx.x >> 1), py = pr / p.g.tiles_x;
    tx = pr - py * p.g.tiles_x;
    ty = 2 * py + rank;
    tile = ty * p.g.tiles_x + tx;
    partner = rank ? true : (ty + 1 < tiles_y);
    if (ty >= tiles_y) {  // ghost: the partner's cluster barriers (after the 1x1 stack, each non-last 3x3 layer, the end)
#pragma unroll
      for (int k = 0; k < R + 1; k++) syn_cluster_sync();
      return;
    }
  } else {
    ty = blockIdx.x / p.g.tiles_x;
    tx = blockIdx.x - ty * p.g.tiles_x;
    tile = blockIdx.x;
  }
  const int Y0 = Ys + ty * SYN_TH, X0 = tx * SYN_TW;
  const int RY = Y0 - RE, RX = X0 - RE;  // origin of the level-0 region (even)
  // CLU: the pair-row of the region the partner computes (-1: none)
  const int shared_rp = (CLU && partner) ? (rank ? 0 : RH0 / 2 - 1) : -1;

  bool staged = false;  // TMA: this tile's boxes are in flight
  if constexpr (TMA) {
    const int lr = ((RY >> 1) - K / 4) & ~1, lc = ((RX >> 1) - K / 4) & ~1;
    const int blo0 = p.g.lv.lo[0], blo1 = p.g.lv.lo[1];
    staged = RY >= blo0 && RY + RH0 <= p.g.lv.hi[0] && RX >= 0 && RX + RW0 <= W && lr >= blo1 &&
             lr + S::NR1 <= p.g.lv.hi[1] && lc >= 0 && lc + S::NC1 <= p.g.lv.w[1];
    if (threadIdx.x == 0) {
      syn_mbar_init(&tbar);
      if (staged) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(syn_smem_u32(&tbar)),
                     "r"(S::TMA_BYTES)
                     : "memory");
        syn_tma_3d(bufA + S::SLOT, &p.tm_s1, &tbar, lc, lr - blo1, 0);      // stack slots 1 .. L-2
        syn_tma_2d(bufB, &p.tm_g1, &tbar, lc - S::G0, lr - blo1);          // grid 1 (int16), in tmph's space
        syn_tma_2d(lat0, &p.tm_lat0, &tbar, RX - LO, RY - blo0);
      }
    }
  }

  float* wraw = smem + S::BUF_A + S::BUF_B + S::LAT0;  // MLP = 1 only: [WRAW]
  if constexpr (MLP == 1) {
    const float* wsrc = &p.w.A0t[0][0];
    for (int i = threadIdx.x; i < S::WRAW; i += SYN_THREADS) wraw[i] = wsrc[i];
  }
  if (threadIdx.x < 32) {
    int r = RY, cl = RX;
    for (int j = 0; j < L; j++) {
      if (threadIdx.x == j) {
        wlo_r[j] = r;
        wlo_c[j] = cl;
      }
      r = ((r >> 1) - K / 4) & ~1;  // arithmetic shift = floor division
      cl = ((cl >> 1) - K / 4) & ~1;
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- 1. chain
  if constexpr (!DENSE_IN) {
    // level 0's region (int16) and the level-1 stack (grid 1 + S_1): by TMA,
    // else all LDG loads in flight together (clamped reads = replicate padding)
    SYN_MARK(0);
    SynCtx c{bufA, bufB, wlo_r, wlo_c};
    if (TMA && staged) {
      syn_mbar_wait(&tbar, 0);
      // grid 1: int16 box -> fp32 slot 0 of the stack
      const int16_t* g1raw = reinterpret_cast<const int16_t*>(bufB);
#pragma unroll
      for (int k = 0; k < (S::NR1 * S::NC1 + SYN_THREADS - 1) / SYN_THREADS; k++) {
        const int i = threadIdx.x + k * SYN_THREADS;
        const int rr = i / S::NC1, cc = i - rr * S::NC1;
        if (i < S::NR1 * S::NC1) bufA[i] = (float)g1raw[rr * S::GP + S::G0 + cc];
      }
    } else {
      LoadLat0<L, CH, R, K>::run(p, lat0, RY, RX);
      if constexpr (L > 1) LoadLevel1<L, CH, R, K>::run(p, c);
    }
    __syncthreads();
    if constexpr (L > 1) {
      SYN_MARK(1);
#ifndef CCRD_SYN_EXP_NOCHAIN  // timing experiment only (wrong results): no horizontal pass
      ChainStep<L, CH, R, K, 0>::run(p, c);  // last step's horizontal pass
#endif
      SYN_MARK(2);
    }
  }

  // ------------------------------------- 2. last vertical step + 1x1 MLP
  // Items: pairs of rows (2q, 2q+1) x columns of the level-0 region.
  float* hA = bufA;  // [3][RH0][RW0] relative to (RY, RX)
  float* hB = bufB;
  {
    const int64_t P = (int64_t)H * W;
    const int64_t Pst = (int64_t)(Ye - Ys) * W;
    // level-1 rows are clamped to the buffer window (= [0, h_1) for a full image)
    const int b1lo = (L > 1) ? p.g.lv.lo[1] : 0, b1hi = (L > 1) ? p.g.lv.hi[1] : 1;
    const int lo1 = wlo_r[(L > 1) ? 1 : 0];
    constexpr int NPAIR = (RH0 / 2) * RW0;
    // one item = a pair of rows (2 rp, 2 rp + 1) at column cc: its L dense
    // values (FFMA2 lane pairs), then after the MLP its 3 outputs per pixel
    auto dense_of = [&](int rp, int cc, uint64_t (&v)[L]) {
      const int y0 = RY + 2 * rp, x = RX + cc;
      const bool has1 = (y0 + 1 < H);
      if constexpr (DENSE_IN) {
        // channel 0 straight from the int16 latents when given (the 2-D TConv
        // path: the pyramid fills channels 1 .. L-1), else from the dense tensor
        const int yc = clampi(y0, 0, H - 1), xc = clampi(x, 0, W - 1);
#pragma unroll
        for (int l = 0; l < L; l++) {
          if (l == 0 && p.lat != nullptr)
            v[0] = f2pack((float)__ldg(p.lat + (int64_t)yc * W + xc),
                          has1 ? (float)__ldg(p.lat + (int64_t)(yc + 1) * W + xc) : 0.0f);
          else
            v[l] = f2pack(__ldg(p.dense_in + l * P + (int64_t)yc * W + xc),
                          has1 ? __ldg(p.dense_in + l * P + (int64_t)(yc + 1) * W + xc) : 0.0f);
        }
      } else {
        v[0] = f2pack((float)lat0[2 * rp * LP + LO + cc], (float)lat0[(2 * rp + 1) * LP + LO + cc]);
        if constexpr (L > 1) {
          // last vertical x2 step, both phases in one FFMA2 lane pair:
          // (out[2q], out[2q+1]) = sum_u sv[u] (k[K-1-2u], k[K-2u]) over the
          // sources sv[u] = rows q - K/4 + u of window 1 (clamped)
          const int q = y0 >> 1;
          int ro[K / 2 + 1];
#pragma unroll
          for (int u = 0; u <= K / 2; u++) ro[u] = (clampi(q - K / 4 + u, b1lo, b1hi - 1) - lo1) * RW0 + cc;
#pragma unroll
          for (int l = 1; l < L; l++) {
            const float* src = bufB + (l - 1) * S::TSLOT;
#if CCRD_SYN_VSCALAR
            // scalar FMAs: K FMA-pipe cycles per channel instead of K + 2 (the
            // packed form multiplies the two phases' missing taps by zero)
            float sv[K / 2 + 1];
#pragma unroll
            for (int u = 0; u <= K / 2; u++) sv[u] = src[ro[u]];
            float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
            for (int u = K / 2 - 1; u >= 0; u--) a0 = fmaf(sv[u], p.w.kv[u].x, a0);
#pragma unroll
            for (int u = K / 2; u >= 1; u--) a1 = fmaf(sv[u], p.w.kv[u].y, a1);
            v[l] = f2pack(a0, a1);
#else
            uint64_t a = 0ull;
#pragma unroll
            for (int u = K / 2; u >= 0; u--) {
              const float sv = src[ro[u]];
              a = ffma2(f2pack(sv, sv), ldp2(p.w.kv[u]), a);
            }
            v[l] = a;
#endif
          }
        }
      }
    };
    auto needed = [&](int rp, int cc) {  // read by the convs (inside the image), not computed by the partner
      const int y0 = RY + 2 * rp, x = RX + cc;
      if (CLU && rp == shared_rp) return false;
#ifdef CCRD_SYN_EXP_NOHALO  // timing experiment only (wrong results): no MLP on the halo rows
      if (2 * rp < RE || 2 * rp >= RE + SYN_TH) return false;
#endif
      return !(x < 0 || x >= W || y0 + 1 < 0 || y0 >= H);
    };
    auto store = [&](int rp, int cc, const uint64_t (&v)[L], const uint64_t (&op)[3]) {
      const int y0 = RY + 2 * rp, x = RX + cc;
      const bool has1 = (y0 + 1 < H);
      const bool inx = (x >= X0 && x < X0 + SYN_TW);
      const bool in0 = inx && y0 >= Y0 && y0 < Y0 + SYN_TH;
      const bool in1 = inx && has1 && y0 + 1 >= Y0 && y0 + 1 < Y0 + SYN_TH;
      if (p.dense_out != nullptr) {
#pragma unroll
        for (int l = 0; l < L; l++) {
          const float2 d = f2unpack(v[l]);
          if (in0) p.dense_out[l * P + (int64_t)y0 * W + x] = d.x;
          if (in1) p.dense_out[l * P + (int64_t)(y0 + 1) * W + x] = d.y;
        }
      }
      float out0[3], out1[3];
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const float2 t = f2unpack(op[c]);
        out0[c] = t.x;
        out1[c] = t.y;
      }
      if (p.h1_out != nullptr) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
          if (in0 && y0 < Ye) p.h1_out[c * Pst + (int64_t)(y0 - Ys) * W + x] = out0[c];
          if (in1 && y0 + 1 < Ye) p.h1_out[c * Pst + (int64_t)(y0 + 1 - Ys) * W + x] = out1[c];
        }
      }
      const int o = 2 * rp * RW0 + cc;
#pragma unroll
      for (int c = 0; c < 3; c++) {
        hA[c * HP + o] = out0[c];
        hA[c * HP + o + RW0] = out1[c];
      }
    };
    if constexpr (MLP == 0) {
      // item = rp x RW0 + cc, advanced by SYN_THREADS without a division
      int rp = (int)threadIdx.x / RW0, cc = (int)threadIdx.x - rp * RW0;
#pragma unroll 1
      for (int item = threadIdx.x; item < NPAIR; item += SYN_THREADS) {
        if (needed(rp, cc)) {  // else never read by the convs
          uint64_t v[L], op[3];
          dense_of(rp, cc, v);
          mlp_pair<L, CH, R, K>(p, v, op);
          store(rp, cc, v, op);
        }
        cc += SYN_THREADS % RW0;
        rp += SYN_THREADS / RW0;
        if (cc >= RW0) {
          cc -= RW0;
          rp++;
        }
      }
    } else {
      // m-tile = 2 row pairs x 4 columns of the level-0 region: MMA row g
      // (0..7) = pixel (row 2 rp, column cc) and row g + 8 = (row 2 rp + 1, cc)
      // with rp = 2 rq + g / 4, cc = 4 cq + g % 4, so each thread's two rows
      // are a vertical pair -- the last upsampling step's FFMA2 lane pair.
      // K (= 8) positions: t -> channel t + 1 (t < 3) or 0 (t = 3); t + 4 ->
      // channel t + 4 (t < 3) or the constant 1 that carries the bias.  Lane
      // (g, t) computes exactly its fragment's dense values: t < 3 two
      // upsampled channels, t = 3 the level-0 latents and the constant.
      static_assert(!DENSE_IN && L <= 7 && CH % 8 == 0 && RW0 % 4 == 0 && (RH0 / 2) % 2 == 0, "mma MLP shape");
      constexpr int NJ = CH / 8;
      constexpr int CQ = RW0 / 4, NMT = (RH0 / 4) * CQ;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const int g = lane >> 2, t = lane & 3;
      const int chA = (t < 3) ? t + 1 : 0, chB = (t < 3) ? t + 4 : -1;  // chB = -1: the bias
      // B fragments (per lane, once per CTA, from the shared copy of the
      // weights): b0 = B[t][8j + g], b1 = B[t + 4][8j + g]
      const float* sA0t = wraw;             // [L][CH]
      const float* sa0 = wraw + L * CH;     // [CH]
      const float* sA1 = sa0 + CH;          // [3][CH]
      uint32_t bh[NJ][2], bl[NJ][2];
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        const int n = 8 * j + g;
        const float w0 = (chA < L) ? sA0t[chA * CH + n] : 0.0f;
        const float w1 = (chB < 0) ? sa0[n] : (chB < L) ? sA0t[chB * CH + n] : 0.0f;
        bh[j][0] = tf32_rna(w0);
        bh[j][1] = tf32_rna(w1);
        bl[j][0] = tf32_rna(w0 - __uint_as_float(bh[j][0]));
        bl[j][1] = tf32_rna(w1 - __uint_as_float(bh[j][1]));
      }
      // layer-1 weight pairs of this lane's hidden units (8 j + 2 t, 8 j + 2 t + 1)
      uint64_t w1p[3][NJ];
#pragma unroll
      for (int c = 0; c < 3; c++)
#pragma unroll
        for (int j = 0; j < NJ; j++)
          w1p[c][j] = *reinterpret_cast<const uint64_t*>(sA1 + c * CH + 8 * j + 2 * t);
      const float bias1 = p.w.a1[(t < 3) ? t : 2];
      // tmph row of source u = 0 for this lane's row pair (the window rows past
      // the image already hold the replicated edge rows: LoadLevel1 clamps)
      const int dr = g >> 2, dc = g & 3;
      const int srcT = (dr + (RY >> 1) - K / 4 - lo1) * RW0 + dc;
      const int latT = 2 * dr * RW0 + dc;            // in the level-0 region (hA)
      const int latTl = 2 * dr * LP + LO + dc;       // in the lat0 buffer
      // shared-window addresses, fixed per lane: t = 3 reads a valid slot too
      // (its values are discarded by the selects below), so every lane runs
      // the same branch-free instruction stream
      const int slotA = (t < 3 && chA < L) ? chA - 1 : 0;
      const int slotB = (t < 3 && chB < L) ? chB - 1 : 0;
      const uint32_t aA0 = syn_smem_u32(bufB) + 4u * (uint32_t)(slotA * S::TSLOT + srcT);
      const uint32_t aB0 = syn_smem_u32(bufB) + 4u * (uint32_t)(slotB * S::TSLOT + srcT);
      const uint32_t aL0 = syn_smem_u32(lat0) + 2u * (uint32_t)latTl;
      const bool okA = (t == 3) || chA < L, okB = (t == 3) || chB < L;
#pragma unroll 1
      for (int mt = warp; mt < NMT; mt += S::NWARPS) {
        const int rq = mt / CQ, cq = mt - rq * CQ;
        const int moff = 4 * rq * RW0 + 4 * cq;  // m-tile origin in the level-0 region
        const uint32_t so = 4u * (uint32_t)(2 * rq * RW0 + 4 * cq);
        uint64_t va = 0ull, vb = 0ull;  // (row 2 rp, row 2 rp + 1) of channels chA, chB
        if constexpr (L > 1) {
          float sa[K / 2 + 1], sb[K / 2 + 1];
          lds_col<K / 2 + 1, 4 * RW0>(aA0 + so, sa);
          lds_col<K / 2 + 1, 4 * RW0>(aB0 + so, sb);
#pragma unroll
          for (int u = K / 2; u >= 0; u--) {
            va = ffma2(f2pack(sa[u], sa[u]), ldp2(p.w.kv[u]), va);
            vb = ffma2(f2pack(sb[u], sb[u]), ldp2(p.w.kv[u]), vb);
          }
        }
        const uint32_t la = aL0 + 2u * (uint32_t)(4 * rq * LP + 4 * cq);
        const float l0 = (float)lds_s16(la), l1 = (float)lds_s16(la + 2u * LP);
        va = (t == 3) ? f2pack(l0, l1) : va;
        vb = (t == 3) ? f2pack(1.0f, 1.0f) : vb;
        va = okA ? va : 0ull;
        vb = okB ? vb : 0ull;
        const float2 fa = f2unpack(va), fb = f2unpack(vb);
        uint32_t ah[4], al[4];
        ah[0] = tf32_round(fa.x);
        ah[1] = tf32_round(fa.y);
        ah[2] = tf32_round(fb.x);
        ah[3] = tf32_round(fb.y);
        {
          const float2 la = f2unpack(fsub2(va, f2pack(__uint_as_float(ah[0]), __uint_as_float(ah[1]))));
          const float2 lb = f2unpack(fsub2(vb, f2pack(__uint_as_float(ah[2]), __uint_as_float(ah[3]))));
          al[0] = __float_as_uint(la.x);
          al[1] = __float_as_uint(la.y);
          al[2] = __float_as_uint(lb.x);
          al[3] = __float_as_uint(lb.y);
        }
        uint64_t o0[3], o1[3];  // layer-1 partials: pixel g / g + 8, lanes = (even, odd) hidden
#pragma unroll
        for (int c = 0; c < 3; c++) o0[c] = o1[c] = 0ull;
#pragma unroll
        for (int j = 0; j < NJ; j++) {
          float d[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          mma_tf32_1688(d, al, bh[j][0], bh[j][1]);
          mma_tf32_1688(d, ah, bl[j][0], bl[j][1]);
          mma_tf32_1688(d, ah, bh[j][0], bh[j][1]);
          const uint64_t h0 = f2pack(fmaxf(d[0], 0.0f), fmaxf(d[1], 0.0f));
          const uint64_t h1 = f2pack(fmaxf(d[2], 0.0f), fmaxf(d[3], 0.0f));
#pragma unroll
          for (int c = 0; c < 3; c++) {
            o0[c] = ffma2(h0, w1p[c][j], o0[c]);
            o1[c] = ffma2(h1, w1p[c][j], o1[c]);
          }
        }
        float s0[3], s1[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const float2 a = f2unpack(o0[c]), b = f2unpack(o1[c]);
          s0[c] = a.x + a.y;
          s1[c] = b.x + b.y;
        }
#pragma unroll
        for (int m = 1; m <= 2; m <<= 1)
#pragma unroll
          for (int c = 0; c < 3; c++) {
            s0[c] += __shfl_xor_sync(0xffffffffu, s0[c], m);
            s1[c] += __shfl_xor_sync(0xffffffffu, s1[c], m);
          }
        // lane t keeps output channel min(t, 2) (t = 3 stores the same value
        // as t = 2 to the same address)
        float x0 = s0[2], x1 = s1[2];
        x0 = (t == 1) ? s0[1] : x0;
        x1 = (t == 1) ? s1[1] : x1;
        x0 = (t == 0) ? s0[0] : x0;
        x1 = (t == 0) ? s1[0] : x1;
        x0 += bias1;
        x1 += bias1;
        if (R > 0) {
          x0 = fmaxf(x0, 0.0f);
          x1 = fmaxf(x1, 0.0f);
        }
        const int o = latT + moff;
        float* hc = hA + ((t < 3) ? t : 2) * HP + o;
        hc[0] = x0;
        hc[RW0] = x1;
      }
    }
  }
  __syncthreads();
  if constexpr (CLU) {  // the partner's 1x1 outputs of my shared pair-row
    syn_cluster_sync();
    if (partner) {
      const int src = rank ? RH0 - 4 : 2, dst = rank ? 0 : RH0 - 2;  // region rows (partner / mine)
      const uint32_t local = syn_smem_u32(bufA);
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank ^ 1));
      for (int i = threadIdx.x; i < 3 * 2 * RW0; i += SYN_THREADS) {
        const int c = i / (2 * RW0), rr = i - c * 2 * RW0;  // rr = row (0..1) x RW0 + column
        float v;
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote + 4u * (uint32_t)(c * HP + src * RW0 + rr)) : "memory");
        bufA[c * HP + dst * RW0 + rr] = v;
      }
    }
    __syncthreads();
  }

  SYN_MARK(3);
  // ------------------------------------------------- 3. residual 3x3 layers
  const int64_t Pimg = (int64_t)(Ye - Ys) * W;  // plane of image / x_hat (strip rows only)
  float sse = 0.0f;
  float* hin = hA;
  float* hout = hB;
  // conv output at (y, x) from hin (replicate padding = clamped reads); used
  // for the halo ring only
  auto conv_px = [&](int r, int y, int x, float (&o)[3]) {
    int ro[3], co[3];
#pragma unroll
    for (int d = 0; d < 3; d++) {
      ro[d] = (clampi(y + d - 1, 0, H - 1) - RY) * RW0;
      co[d] = clampi(x + d - 1, 0, W - 1) - RX;
    }
    const int ctr = (y - RY) * RW0 + (x - RX);
    // same operation order as the interior path (bias, then per input channel
    // its residual term and its 9 taps), so a pixel's value does not depend on
    // whether it falls in a tile's interior or its halo ring: strips and the
    // full image agree bit for bit
    uint64_t a01 = f2pack(p.w.g[r][0], p.w.g[r][1]);
    float a2 = p.w.g[r][2];
#pragma unroll
    for (int ci = 0; ci < 3; ci++) {
      const float c = hin[ci * HP + ctr];
      if (ci == 2) {
        a2 += c;
      } else {
        float2 t = f2unpack(a01);
        if (ci == 0) t.x += c;
        else t.y += c;
        a01 = f2pack(t.x, t.y);
      }
#pragma unroll
      for (int ky = 0; ky < 3; ky++)
#pragma unroll
        for (int kx = 0; kx < 3; kx++) {
          const float hv = hin[ci * HP + ro[ky] + co[kx]];
          a01 = ffma2(f2pack(hv, hv), ldp2(p.w.Gp[r][ci][ky][kx]), a01);
          a2 = fmaf(hv, p.w.Gs[r][ci][ky][kx], a2);
        }
    }
    const float2 a = f2unpack(a01);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = a2;
  };
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int e = R - 1 - r;  // halo this layer's output still needs
    const bool last = (r == R - 1);
    const int ylim = last ? Ye : H;  // non-last layers also feed the rows just past the strip
    // interior (the tile): each thread owns a column segment of RS rows; per
    // input channel it loads the (RS + 2) x 3 window once and every uniform
    // weight (pair) feeds RS outputs
    {
      constexpr int RS = S::RS;
      const int cc = threadIdx.x % SYN_TW, seg = threadIdx.x / SYN_TW;
      const int x = X0 + cc;
      const int yb = Y0 + seg * RS;
      if (x < W && yb < ylim) {
        int co[3];
#pragma unroll
        for (int d = 0; d < 3; d++) co[d] = clampi(x + d - 1, 0, W - 1) - RX;
        // x for the output rows, in flight during the math.  8-bit: the raw
        // bytes stay integers until the distortion below -- converted at the
        // load, every warp stalled on its loads before the math (the largest
        // single stall of the kernel)
        float img[RS][3];
        uint32_t img8[RS][3];
        if (last && (IMG8 ? p.image8 != nullptr : p.image != nullptr)) {
#pragma unroll
          for (int i = 0; i < RS; i++)
#pragma unroll
            for (int c = 0; c < 3; c++) {
              const int64_t gi = c * Pimg + (int64_t)(yb + i - Ys) * W + x;
              if constexpr (IMG8)
                img8[i][c] = (yb + i < Ye) ? (uint32_t)__ldg(p.image8 + gi) : 0u;
              else
                img[i][c] = (yb + i < Ye) ? __ldg(p.image + gi) : 0.0f;
            }
        }
        uint64_t a01[RS];
        float a2[RS];
#pragma unroll
        for (int i = 0; i < RS; i++) {
          a01[i] = f2pack(p.w.g[r][0], p.w.g[r][1]);
          a2[i] = p.w.g[r][2];
        }
#pragma unroll
        for (int ci = 0; ci < 3; ci++) {
          float in[RS + 2][3];  // rows yb-1 .. yb+RS (clamped) x cols x-1 .. x+1
#pragma unroll
          for (int d = 0; d < RS + 2; d++) {
            const int rof = ci * HP + (clampi(yb + d - 1, 0, H - 1) - RY) * RW0;
#pragma unroll
            for (int kx = 0; kx < 3; kx++) in[d][kx] = hin[rof + co[kx]];
          }
          // residual: output channel co = ci adds its own input
#pragma unroll
          for (int i = 0; i < RS; i++) {
            if (ci == 2) {
              a2[i] += in[i + 1][1];
            } else {
              float2 t = f2unpack(a01[i]);
              if (ci == 0) t.x += in[i + 1][1];
              else t.y += in[i + 1][1];
              a01[i] = f2pack(t.x, t.y);
            }
          }
#pragma unroll
          for (int ky = 0; ky < 3; ky++)
#pragma unroll
            for (int kx = 0; kx < 3; kx++) {
              const uint64_t w01 = ldp2(p.w.Gp[r][ci][ky][kx]);
              const float w2 = p.w.Gs[r][ci][ky][kx];
#pragma unroll
              for (int i = 0; i < RS; i++) {
                const float hv = in[i + ky][kx];
                a01[i] = ffma2(f2pack(hv, hv), w01, a01[i]);
                a2[i] = fmaf(hv, w2, a2[i]);
              }
            }
        }
#pragma unroll
        for (int i = 0; i < RS; i++) {
          const int y = yb + i;
          if (y >= ylim) break;
          const float2 a = f2unpack(a01[i]);
          const float o[3] = {a.x, a.y, a2[i]};
          if (!last) {
            const int ctr = (y - RY) * RW0 + (x - RX);
#pragma unroll
            for (int c = 0; c < 3; c++) hout[c * HP + ctr] = fmaxf(o[c], 0.0f);
          } else {
            if (p.out_u8 != nullptr || p.x_hat != nullptr) {  // optional outputs (uniform branch)
              const int64_t gi = (int64_t)(y - Ys) * W + x;
              if (p.out_u8 != nullptr) {  // decoder output: clamp to [0,1], 8-bit, ties to even (reading N3)
#pragma unroll
                for (int c = 0; c < 3; c++)
                  p.out_u8[gi * 3 + c] = (uint8_t)__float2uint_rn(255.0f * fminf(fmaxf(o[c], 0.0f), 1.0f));
              }
              if (p.x_hat != nullptr) {
#pragma unroll
                for (int c = 0; c < 3; c++) p.x_hat[c * Pimg + gi] = o[c];
              }
            }
            // 8-bit: min(v, late) == v (v <= 255 <= late) ties each byte's
            // conversion to this row's result, so the scheduler cannot hoist
            // it (with its load wait) above the convolution
            const uint32_t late = __float_as_uint(o[0]) | 255u;
#pragma unroll
            for (int c = 0; c < 3; c++) {
              if ((IMG8 ? p.image8 != nullptr : p.image != nullptr)) {
                float xv;
                if constexpr (IMG8)
                  xv = u8_to_x(min(img8[i][c], late));
                else
                  xv = img[i][c];
                const float ev = xv - o[c];
                sse = fmaf(ev, ev, sse);
              }
            }
          }
        }
      }
    }
    // halo ring of width e around the tile (non-last layers only), enumerated
    // directly: top / bottom rows, then left / right columns
#ifdef CCRD_SYN_EXP_NORING  // timing experiment only (wrong results): no conv halo ring
    if (false) {
#else
    if (e > 0) {
#endif
      const int NWr = SYN_TW + 2 * e;
      const int n_top = e * NWr, n_side = e * SYN_TH;
#pragma unroll 1
      for (int idx = threadIdx.x; idx < 2 * n_top + 2 * n_side; idx += SYN_THREADS) {
        int y, x;
        if (idx < 2 * n_top) {
          const int j = idx < n_top ? idx : idx - n_top;
          const int rr = j / NWr;
          y = (idx < n_top) ? Y0 - e + rr : Y0 + SYN_TH + rr;
          x = X0 - e + (j - rr * NWr);
        } else {
          const int j0 = idx - 2 * n_top;
          const int j = j0 < n_side ? j0 : j0 - n_side;
          const int rr = j / e;
          y = Y0 + rr;
          x = (j0 < n_side) ? X0 - e + (j - rr * e) : X0 + SYN_TW + (j - rr * e);
        }
        if (y < 0 || y >= H || x < 0 || x >= W) continue;
        if (CLU && partner && (rank ? y < Y0 : y >= Y0 + SYN_TH)) continue;  // the partner's interior row
        float o[3];
        conv_px(r, y, x, o);
        const int ctr = (y - RY) * RW0 + (x - RX);
#pragma unroll
        for (int c = 0; c < 3; c++) hout[c * HP + ctr] = fmaxf(o[c], 0.0f);
      }
    }
    if (!last) {
      __syncthreads();
      if constexpr (CLU) {  // the partner's first-layer outputs of my shared ring row (region columns 1 .. RW0-2)
        syn_cluster_sync();
        if (partner) {
          const int src = rank ? RH0 - 3 : 2, dst = rank ? 1 : RH0 - 2;
          const uint32_t local = syn_smem_u32(hout);
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank ^ 1));
          for (int i = threadIdx.x; i < 3 * (RW0 - 2); i += SYN_THREADS) {
            const int c = i / (RW0 - 2), cc = 1 + i - c * (RW0 - 2);
            float v;
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote + 4u * (uint32_t)(c * HP + src * RW0 + cc)) : "memory");
            hout[c * HP + dst * RW0 + cc] = v;
          }
        }
        __syncthreads();
      }
      SYN_MARK(4);
      float* t = hin;
      hin = hout;
      hout = t;
    }
  }

  // R == 0: the 1x1 stack's output is x_hat
  if constexpr (R == 0) {
#pragma unroll 1
    for (int item = threadIdx.x; item < SYN_TH * SYN_TW; item += SYN_THREADS) {
      const int rr = item / SYN_TW, cc = item - rr * SYN_TW;
      const int y = Y0 + rr, x = X0 + cc;
      if (y >= Ye || x >= W) continue;
      const int ctr = (y - RY) * RW0 + (x - RX);
      const int64_t gi = (int64_t)(y - Ys) * W + x;
      if (p.out_u8 != nullptr) {
#pragma unroll
        for (int c = 0; c < 3; c++)
          p.out_u8[gi * 3 + c] = (uint8_t)__float2uint_rn(255.0f * fminf(fmaxf(hin[c * HP + ctr], 0.0f), 1.0f));
      }
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const float xh = hin[c * HP + ctr];
        if (p.x_hat != nullptr) p.x_hat[c * Pimg + gi] = xh;
        if ((IMG8 ? p.image8 != nullptr : p.image != nullptr)) {
          const float ev = load_x<IMG8>(p, c * Pimg + gi) - xh;
          sse = fmaf(ev, ev, sse);
        }
      }
    }
  }

  // ------------------------------------------------------ 4. distortion
  const double s = block_sum<SYN_THREADS>(sse, warp_buf);
  if (threadIdx.x == 0 && p.partial != nullptr) p.partial[tile] = s;
  if constexpr (CLU) syn_cluster_sync();  // the partner has read my shared memory
  SYN_MARK(5);
#ifdef CCRD_SYN_TIMING
  if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) {
    unsigned int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_syn_timing[blockIdx.x][6] = sm;
  }
#endif
  pdl_wait();  // complete only after the previous kernel of the stream
}

#ifdef CCRD_SYN_TIMING
}  // namespace ccrd
extern "C" int cc_debug_syn_timing(unsigned long long* host, int n_cta) {
  return (int)cudaMemcpyFromSymbol(host, ccrd::g_syn_timing, sizeof(unsigned long long) * 8 * (size_t)n_cta);
}
namespace ccrd {
#endif

// ---------------------------------------------------------------- host launcher
// one kernel variant: opt in to its dynamic shared memory size once, launch
template <int L, int CH, int R, int K, bool DENSE_IN, bool IMG8, int MLP, bool TMA = false>
static void syn_go(const SynParams<L, CH, R, K>& p, int n_tiles, size_t smem, cudaStream_t stream) {
  static const bool attr = (cudaFuncSetAttribute(synth_kernel<L, CH, R, K, DENSE_IN, IMG8, MLP, TMA>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                            true);
  (void)attr;
  launch_ctl(synth_kernel<L, CH, R, K, DENSE_IN, IMG8, MLP, TMA>, (unsigned)n_tiles, SYN_THREADS, smem, stream, p);
}

// CLU: clusters of two vertically adjacent tiles, grid = 2 x tiles_x x
// ceil(tiles_y / 2) (a rank-1 CTA past the last tile row is a ghost)
template <int L, int CH, int R, int K, bool IMG8>
static void syn_go_pairs(const SynParams<L, CH, R, K>& p, size_t smem, cudaStream_t stream) {
  auto kern = synth_kernel<L, CH, R, K, false, IMG8, 0, true, true>;
  static const bool attr = (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), true);
  (void)attr;
  const int tiles_y = p.g.n_tiles / p.g.tiles_x;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * p.g.tiles_x * ((tiles_y + 1) / 2)));
  cfg.blockDim = dim3(SYN_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_launch_ctl.pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, p);
}
// Opt-in (CCRD_SYN_CLU=1, read per launch: tests toggle it): measured slower
// than one CTA per tile (108.0 vs 100.3 us per 2K image, path 1.742e10 vs
// 1.839e10 px/s) -- the three cluster barriers hold both CTAs of a pair in
// step and cost more than the 1x1 / 3x3 rows they save.
static bool syn_pairs_enabled() {
  const char* e = getenv("CCRD_SYN_CLU");
  return e && e[0] == '1';
}

// ---- tensor maps of the TMA staging (driver entry point, no -lcuda)
typedef CUresult (*SynEncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static SynEncodeTiledFn syn_encode_tiled() {
  static const SynEncodeTiledFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    SynEncodeTiledFn f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<SynEncodeTiledFn>(ptr);
    cudaGetLastError();
    return f;
  }();
  return fn;
}
// The three boxes of a tile (SynShape: S_1 [L-2][NR1][NC1] fp32, grid 1
// [NR1][GP] int16 from column lc - G0, level-0 region [RH0][LP] int16 from
// column RX - LO).  False (LDG staging) when a buffer is not 16-byte aligned /
// strided as TMA requires, or the encoder is unavailable.
template <int L, int CH, int R, int K>
static bool syn_tma_maps(SynParams<L, CH, R, K>& p) {
  using S = SynShape<L, CH, R, K>;
  if constexpr (!S::TMA_OK) {
    return false;
  } else {
    SynEncodeTiledFn enc = syn_encode_tiled();
    if (!enc || p.lat == nullptr || p.s1 == nullptr) return false;
    const LevelGeom& lv = p.g.lv;
    const int64_t W = p.g.W, w1 = lv.w[1], r0 = lv.hi[0] - lv.lo[0], r1 = lv.hi[1] - lv.lo[1];
    const int16_t* g1 = p.lat + lv.off[1];
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    if (r0 < 1 || r1 < 1 || (W * 2) % 16 || (w1 * 2) % 16 || !al16(p.lat) || !al16(g1) || !al16(p.s1)) return false;
    const cuuint32_t es[3] = {1, 1, 1};
    {
      const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)r0};
      const cuuint64_t str[1] = {(cuuint64_t)W * 2};
      const cuuint32_t box[2] = {(cuuint32_t)S::LP, (cuuint32_t)S::RH0};
      if (enc(&p.tm_lat0, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)p.lat, dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    }
    {
      const cuuint64_t dims[2] = {(cuuint64_t)w1, (cuuint64_t)r1};
      const cuuint64_t str[1] = {(cuuint64_t)w1 * 2};
      const cuuint32_t box[2] = {(cuuint32_t)S::GP, (cuuint32_t)S::NR1};
      if (enc(&p.tm_g1, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)g1, dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    }
    {
      const cuuint64_t dims[3] = {(cuuint64_t)w1, (cuuint64_t)r1, (cuuint64_t)(L - 2)};
      const cuuint64_t str[2] = {(cuuint64_t)w1 * 4, (cuuint64_t)(w1 * r1 * 4)};
      const cuuint32_t box[3] = {(cuuint32_t)S::NC1, (cuuint32_t)S::NR1, (cuuint32_t)(L - 2)};
      if (enc(&p.tm_s1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)p.s1, dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    }
    return true;
  }
}
template <int L, int CH, int R, int K>
static int launch_syn(const SynGeom& g, const cc_model_desc& d, const float* up_w,
                      const float* syn_w, const int16_t* lat, const float* s1, const float* dense_in,
                      const float* image, float* x_hat, float* dense_out, float* h1_out,
                      double* partial, cudaStream_t stream, uint8_t* out_u8) {
  SynParams<L, CH, R, K> p;
  p.g = g;
  p.lat = lat;
  p.s1 = s1;
  p.dense_in = dense_in;
  p.image = d.image_u8 ? nullptr : image;
  p.image8 = d.image_u8 ? reinterpret_cast<const uint8_t*>(image) : nullptr;
  p.x_hat = x_hat;
  p.dense_out = dense_out;
  p.h1_out = h1_out;
  p.partial = partial;
  p.out_u8 = out_u8;
  for (int t = 0; t < K; t++) p.w.k[t] = up_w ? up_w[t] : 0.0f;
  // last vertical step: (a0, a1) += sv[u] (k[K-1-2u], k[K-2u]), zero where a
  // phase has no tap (u = K/2 for a0, u = 0 for a1)
  for (int u = 0; u <= K / 2; u++)
    p.w.kv[u] = make_float2(u < K / 2 && up_w ? up_w[K - 1 - 2 * u] : 0.0f, u > 0 && up_w ? up_w[K - 2 * u] : 0.0f);
  const float* q = syn_w;
  for (int i = 0; i < L; i++)
    for (int n = 0; n < CH; n++) p.w.A0t[i][n] = q[n * L + i];
  for (int n = 0; n < CH; n++) p.w.a0[n] = q[L * CH + n];
  q += L * CH + CH;
  for (int c = 0; c < 3; c++)
    for (int n = 0; n < CH; n++) p.w.A1[c][n] = q[c * CH + n];
  for (int c = 0; c < 3; c++) p.w.a1[c] = q[3 * CH + c];
  q += 3 * CH + 3;
  for (int r = 0; r < R; r++) {
    for (int ci = 0; ci < 3; ci++)
      for (int ky = 0; ky < 3; ky++)
        for (int kx = 0; kx < 3; kx++) {
          auto G = [&](int co) { return q[((co * 3 + ci) * 3 + ky) * 3 + kx]; };
          p.w.Gp[r][ci][ky][kx] = make_float2(G(0), G(1));
          p.w.Gs[r][ci][ky][kx] = G(2);
        }
    for (int c = 0; c < 3; c++) p.w.g[r][c] = q[81 + c];
    q += 84;
  }
  using S = SynShape<L, CH, R, K>;
  // 1x1 layer 0 on warp MMAs (chain mode, no debug outputs) when selected
  // (cc_set_synth_path CC_SYN_MMA; measured slower)
  constexpr bool kMmaShape = L <= 7 && CH % 8 == 0 && S::RW0 % 4 == 0 && (S::RH0 / 2) % 2 == 0;
  const bool mma = kMmaShape && !dense_in && !dense_out && !h1_out && synth_path() == CC_SYN_MMA;
  const size_t smem = mma ? S::SMEM_MMA : S::SMEM;
  // TMA-staged tiles (cc_set_synth_path CC_SYN_TMA / AUTO)
  const int sp = synth_path();
  const bool tma = !dense_in && !dense_out && !h1_out && !mma && (sp == CC_SYN_TMA || sp == CC_SYN_AUTO) &&
                   syn_tma_maps(p);
  if (tma) {
    if constexpr (S::TMA_OK) {
      constexpr bool kPairs = S::RE == 2 && (R == 1 || R == 2);
      if (kPairs && syn_pairs_enabled() && g.n_tiles / g.tiles_x >= 2) {
        if constexpr (kPairs) {
          if (d.image_u8) syn_go_pairs<L, CH, R, K, true>(p, S::SMEM_TMA, stream);
          else syn_go_pairs<L, CH, R, K, false>(p, S::SMEM_TMA, stream);
        }
      } else if (d.image_u8) {
        syn_go<L, CH, R, K, false, true, 0, true>(p, g.n_tiles, S::SMEM_TMA, stream);
      } else {
        syn_go<L, CH, R, K, false, false, 0, true>(p, g.n_tiles, S::SMEM_TMA, stream);
      }
    }
  } else if (dense_in) {  // stage entry cc_synthesize: fp32 images only (checked by the API)
    syn_go<L, CH, R, K, true, false, 0>(p, g.n_tiles, smem, stream);
  } else if (mma) {
    if constexpr (kMmaShape) {
      if (d.image_u8) syn_go<L, CH, R, K, false, true, 1>(p, g.n_tiles, smem, stream);
      else syn_go<L, CH, R, K, false, false, 1>(p, g.n_tiles, smem, stream);
    }
  } else if (d.image_u8) {
    syn_go<L, CH, R, K, false, true, 0>(p, g.n_tiles, smem, stream);
  } else {
    syn_go<L, CH, R, K, false, false, 0>(p, g.n_tiles, smem, stream);
  }
  return 0;
}

struct SynEntry {
  int L, CH, R, K;
  SynLaunchFn fn;
};

// Compiled synthesis shapes: BASELINE.json configs (tiny [4,8,3]+1, low
// [7,16,3]+2, ref [7,40,3]+2; 8 taps), Table 1 (A300 [7,8,3]+1, A545/A1079
// [7,16,3]+2 with 4 taps, A2300 [7,40,3]+2 with 8 taps) and small L / other R
// for the edge-case tests.
static const SynEntry kSyn[] = {
    {4, 8, 1, 8, launch_syn<4, 8, 1, 8>},     {7, 16, 2, 8, launch_syn<7, 16, 2, 8>},
    {7, 40, 2, 8, launch_syn<7, 40, 2, 8>},   {7, 8, 1, 4, launch_syn<7, 8, 1, 4>},
    {7, 16, 2, 4, launch_syn<7, 16, 2, 4>},   {4, 8, 1, 4, launch_syn<4, 8, 1, 4>},
    {1, 8, 1, 8, launch_syn<1, 8, 1, 8>},     {5, 8, 1, 8, launch_syn<5, 8, 1, 8>},
    {5, 8, 1, 4, launch_syn<5, 8, 1, 4>},     {4, 8, 0, 8, launch_syn<4, 8, 0, 8>},
    {4, 8, 3, 8, launch_syn<4, 8, 3, 8>},     {2, 8, 1, 8, launch_syn<2, 8, 1, 8>},
    {3, 8, 1, 8, launch_syn<3, 8, 1, 8>},     {7, 40, 2, 4, launch_syn<7, 40, 2, 4>},
};

SynLaunchFn find_syn_launcher(int L, int CH, int R, int K) {
  for (const auto& e : kSyn)
    if (e.L == L && e.CH == CH && e.R == R && e.K == K) return e.fn;
  return nullptr;
}

}  // namespace ccrd
