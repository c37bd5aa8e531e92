// arm_tc.cu -- ARM rate on the 5th-generation tensor cores (tcgen05 + TMEM),
// the default ARM path for the shapes compiled here (cc_set_arm_path).
//
// Same function as arm_rate.cu (PAPER.md:106-109 ARM f_psi, :120 R term of
// Eq. 1; Table 1 ARM column; readings #1-#8): for every latent the
// causal context c, the MLP z1 = ReLU(W0 c + b0), z_{k+1} = ReLU(W_k z_k + b_k
// [+ z_k]), (mu, s) = W_out z + b_out, then -log2 of the Laplace bin mass.
//
// The hidden layers are dense contractions over blocks of 128 latents --
// [128 x K] x [K x NH] -- run as tcgen05.mma kind::tf32 (M = 128, N = NH) with
// fp32 accumulators in TMEM, fp32-accurate through a split:
//   * layer 0: the context is small integers, exact in tf32 (11 significant
//     bits) when |c| <= 2048, so only the weights are split, W = W_hi + W_lo
//     (tf32 each): D0 = A0 W_hi + A0 W_lo.  The bias rides on a constant-1
//     input column.  A window holding a latent outside +-2048 (detected while
//     staging it) splits the context too, c = c_hi + c_lo, and adds c_lo W;
//   * the hidden layer: the activations are split per element z = z_hi + z_lo
//     (z_hi = z truncated to tf32, z_lo = z - z_hi, exact) and
//     D1 = z_hi W_hi + z_hi W_lo + z_lo W_hi ("3xTF32"): only the z_lo W_lo term
//     (~2^-22 relative) is dropped;
//   * the 2-wide output layer, the Laplace bits and the reduction stay on the
//     CUDA cores (packed FFMA2 over input pairs, constant-bank weights).
//
// Every operand that changes per block lives in TMEM (TS MMAs: A from TMEM, B
// = the weights, K-major no-swizzle canonical layout in shared memory); thread
// t of a warpgroup owns latent t of a block = TMEM lane t through all stages.
// Measured constraints that shape the kernels (tools/microbench/tc_bench.cu):
// one issuing thread sustains one MMA per ~25 cycles, two or more issuers per
// SM reach the tensor pipe's N-floor; a 6 / 11-MMA batch + commit + wait takes
// 467 / 569 cycles alone; TMEM loads need several in flight.  Hence several
// warpgroups per SM, each issuing its own MMA batches (one asm statement per
// batch), and -- in arm_tcp_kernel, the default -- two blocks in flight per
// warpgroup so one block's MMA latency overlaps the other's CUDA-core stage.
// The causal window of each 8 x 64 tile arrives by TMA (zero fill = the zero
// padding of reading #5) where every grid's rows are 16-byte strided, by
// predicated LDG otherwise.  DESIGN.md 7.2 has the measurements.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "arm_math.cuh"
#include "ccrd_common.cuh"
#include "tcgen05.cuh"

namespace ccrd {

constexpr int TC_M = 128;  // latents per MMA block (TMEM lanes)

__host__ __device__ constexpr int rup(int x, int m) { return (x + m - 1) / m * m; }

template <int C, int NH, int NHL>
struct ArmTcShape {
  static constexpr int K0 = rup(C + 1, 8);                  // context + bias column
  static constexpr int NP = rup(NH, 16) < 16 ? 16 : rup(NH, 16);  // weight rows stored (the MMAs use N = NH)
  static constexpr int K1 = rup(NH + 1, 8);                 // hidden + bias column
  static constexpr int NHID = NHL - 1;                      // NH -> NH layers on the tensor cores
  static constexpr int BW0 = NP * K0;                       // floats per weight matrix
  static constexpr int BW1 = NP * K1;
  static constexpr int B_FLOATS = 2 * BW0 + 2 * NHID * BW1;
  static_assert(NP <= 32, "one 32-column TMEM accumulator");
  static_assert(K0 % 8 == 0 && K1 % 8 == 0, "tcgen05 shape");
};

// K-major canonical offset (floats) of element (r, k) of an operand with K
// columns: core matrix (r/8, k/4), 8 rows x 4 floats each
__host__ __device__ constexpr int kmaj(int r, int k, int K) {
  return (r >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

// host-side packing of the tensor-core ARM's B operands
template <int C, int NH, int NHL>
struct ArmTcB {
  using S = ArmTcShape<C, NH, NHL>;
  float B0[2][S::BW0];                               // [hi/lo] layer 0 (bias in column C)
  float B1[(S::NHID > 0) ? S::NHID : 1][2][S::BW1];  // [layer][hi/lo] (residual folded, bias in column NH)
};

template <int C, int NH, int NHL>
struct ArmTcParams {
  using S = ArmTcShape<C, NH, NHL>;
  ArmGeom g;
  const int16_t* lat;
  double* partial;  // [tiles][16]: one per (block, warp)
  float* mu;        // optional per-latent debug outputs
  float* scale;
  float* bits;
  float2 wo[NH];                                          // output layer (mu, log-scale) per input
  float2 bo;
  float2 wm[NH / 2], wsl[NH / 2];                         // output layer as input pairs: mu, log-scale
  const float* gB;  // the weights, pre-split on the host into tf32 (hi, lo) pairs in the canonical
                    // K-major layout (ArmTcB), in global memory: bulk-loaded into shared memory
  CUtensorMap tmap[CC_MAX_LEVELS];  // int16 grid l ([rows present][w]) for TMA window loads (arm_tcg_kernel, TMA)
};

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
#ifndef CCRD_TCG_NWG
#define CCRD_TCG_NWG 6  // warpgroups per SM (experiment knob; TMEM caps it at 512 / SLOT)
#endif
  static constexpr int NWG = (512 / SLOT) < CCRD_TCG_NWG ? (512 / SLOT) : CCRD_TCG_NWG;
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

#ifndef CCRD_TCG_SPIN
#define CCRD_TCG_SPIN 0  // 1: plain try_wait spin on the MMA barrier (experiment knob)
#endif
#if CCRD_TCG_SPIN
#define TCG_WAIT(b, ph) mbar_wait(b, ph)
#else
#define TCG_WAIT(b, ph) mbar_wait_sleep(b, ph)
#endif

#ifdef CCRD_TCG_TIMING
// experiment build: per-CTA sums of phase durations of warpgroup 0, warp 0
// (clock64), read back by cc_debug_tcg_timing (tools/ only)
__device__ unsigned long long g_tcg_timing[1024][12];
#define TCG_T(k)                                                     \
  if (tw == 0) {                                                     \
    unsigned long long t_;                                           \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));               \
    if (k > 0) tacc[k - 1] += t_ - tlast;                            \
    tlast = t_;                                                      \
  }
#else
#define TCG_T(k)
#endif

__device__ __forceinline__ void wg_sync(int g) { asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory"); }


// named barrier of warpgroup g with an OR over its threads' predicates
__device__ __forceinline__ bool wg_sync_or(int g, bool v) {
  uint32_t r;
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %2, 0;\n\tbar.red.or.pred q, %1, 128, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
               : "=r"(r)
               : "r"(g + 1), "r"((int)v)
               : "memory");
  return r != 0;
}

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

// Windows holding a latent outside +-2048: the context is split exactly,
// c = c_hi + c_lo (c_hi = c truncated to tf32, c_lo = c - c_hi, both exact in
// tf32), row <- c_hi and c_lo to TMEM at taddr; MMA0 then adds c_lo (B0_hi +
// B0_lo) (mma_batch_4t: with |c| up to 2^15 the c_lo B0_lo term is as large
// as fp32 rounding, so it is kept).
template <int C>
__device__ __forceinline__ void split_ctx(float (&row)[C], uint32_t taddr) {
  float lo[C];
#pragma unroll
  for (int c = 0; c < C; c++) {
    const float h = __uint_as_float(__float_as_uint(row[c]) & 0xFFFFE000u);
    lo[c] = row[c] - h;
    row[c] = h;
  }
  tmem_st_cols<C>(taddr, lo);
}

// LDG staging of a tile's fp32 window by the 128 threads of a warpgroup
// (zero outside the grid); returns whether a latent outside +-2048 is in it
template <int WIN>
__device__ __forceinline__ bool stage_window_ldg(const int16_t* lat, const ArmGeom& g, int l, int i0, int j0, float* win,
                                                 int tw) {
  const int w = g.lv.w[l], rlo = g.lv.lo[l], rhi = g.lv.hi[l];
  const int16_t* __restrict__ base = lat + g.lv.off[l] + (int64_t)(i0 - ARM_HALO_TOP - rlo) * w + (j0 - ARM_HALO_X);
  const bool inner = i0 - ARM_HALO_TOP >= rlo && i0 + ARM_TY <= rhi && j0 - ARM_HALO_X >= 0 && j0 + ARM_TX + ARM_HALO_X <= w;
  constexpr int IT = (WIN + 127) / 128;
  int16_t v[IT];
  int off[IT];
  bool ok[IT];
  int r = tw / ARM_SW, c = tw - (tw / ARM_SW) * ARM_SW;
#pragma unroll
  for (int k = 0; k < IT; k++) {  // offsets and predicates first (no branches) ...
    const int gi = i0 - ARM_HALO_TOP + r, gj = j0 - ARM_HALO_X + c;
    ok[k] = ((k < IT - 1) || (tw + 128 * k < WIN)) && (inner || (gi >= rlo && gi < rhi && gj >= 0 && gj < w));
    off[k] = r * w + c;
    c += 128 - ARM_SW;  // + 128 elements = + 1 row + 56 columns, at most one wrap
    const bool wrap = c >= ARM_SW;
    c -= wrap ? ARM_SW : 0;
    r += wrap ? 2 : 1;
  }
#pragma unroll
  for (int k = 0; k < IT; k++) v[k] = ldg_s16_pred(base + off[k], ok[k]);  // ... then every load in flight
  bool big = false;
#pragma unroll
  for (int k = 0; k < IT; k++) {
    const int e = tw + k * 128;
    if ((k < IT - 1) || e < WIN) win[e] = (float)v[k];
    big |= v[k] > 2048 || v[k] < -2048;
  }
  return big;
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
  __shared__ __align__(8) uint64_t wbar;  // the weights' bulk copy
  pdl_trigger();  // the next image's ARM may be scheduled as this grid drains
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t < 3 * NWG) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + t)));
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wbar)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // the split weights (B operands, ~14 KB) in one bulk copy from global memory
  // (a per-thread copy from the kernel-parameter bank serialises in the
  // constant cache: ~7 % of the kernel's stall samples)
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&wbar)), "r"(4 * S::B_FLOATS)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sB)),
                 "l"(p.gB), "r"(4 * S::B_FLOATS), "r"(smem_u32(&wbar))
                 : "memory");
  }
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
#ifdef CCRD_TCG_TIMING
  unsigned long long tacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tlast = 0, tstart = 0, ttile = 0;
  if (tw == 0) asm volatile("mov.u64 %0, %%clock64;" : "=l"(tstart));
#endif
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
    const int ty = tile_row(tt, p.g.tiles_x[l], p.g.tx_mul[l]);
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
  mbar_wait(&wbar, 0);  // the weights are in shared memory
  int it = 0;
#pragma unroll 1
  for (int tile = (int)blockIdx.x * NWG + g; tile < n_tiles; tile += stride, it++) {
#ifdef CCRD_TCG_TIMING
    if (tw == 0) asm volatile("mov.u64 %0, %%clock64;" : "=l"(ttile));
#endif
    int l, i0, j0;
    locate(tile, l, i0, j0);
    const int w = p.g.lv.w[l], rlo = p.g.lv.lo[l], rhi = p.g.lv.hi[l];
    bool big = false;
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
        big |= fmaxf(fmaxf(fabsf(f.x), fabsf(f.y)), fmaxf(fabsf(f.z), fabsf(f.w))) > 2048.0f;
      }
    } else
    {  // causal window of the tile (fp32, zero outside the grid); every
       // thread of this warpgroup passed the previous tile's last pre-MMA
       // barrier, so the previous window has no reader left
      big = stage_window_ldg<G::WIN>(p.lat, p.g, l, i0, j0, win, tw);
    }
    // a latent outside +-2048 in the window is not exact in tf32 (11
    // significant bits): this tile splits the context, c = c_hi + c_lo
    const bool split0 = wg_sync_or(g, big);
#ifdef CCRD_TCG_TIMING
    if (tw == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));
      tacc[8] += t_ - ttile;
      tacc[10] += 1;
    }
#endif
    float tbits = 0.0f;  // this thread's bits over the tile's 4 blocks
#pragma unroll 1
    for (int q = 0; q < ARM_TY / 2; q++) {
      const int ry = 2 * q + (tw >> 6), cx = tw & 63;
      const float* center = win + (ry + ARM_HALO_TOP) * ARM_SW + cx + ARM_HALO_X;
      const float y = center[0];
      TCG_T(0);
      {  // A0 row: [context (C), 1, 0 x 7]
        float row[C], tail[8] = {1.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c = 0; c < C; c++) row[c] = center[STD ? std_ctx_dy(c) * ARM_SW + std_ctx_dx(c) : p.g.ctx_off[c]];
        if (split0) split_ctx<C>(row, tl + cD);  // c_lo -> the D1 columns (free until MMA1)
        tmem_st_cols<C>(tl + cX, row);
        tmem_st_cols<8>(tl + cX + C, tail);
        tmem_wait_st();
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      TCG_T(1);
      wg_sync(g);
      TCG_T(2);
      if (qd == (q & 3)) {  // MMA0: D0 = A0 B0_hi + A0 B0_lo (one elected lane; the issuing warp rotates)
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (split0)  // + c_lo (B0_hi + B0_lo)
          mma_batch_4t<K0 / 8, C / 8>(tmem + cY, tmem + cX, tmem + cD, dB0, IDESC, bar, LO0);
        else
          mma_batch_hilo<K0 / 8>(tmem + cY, tmem + cX, dB0, IDESC, bar, LO0);
      }
      TCG_WAIT(bar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      TCG_T(3);
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
      TCG_T(4);
      wg_sync(g);
      TCG_T(5);
      if (qd == (q & 3)) {  // MMA1: D1 = A1_hi B1_hi + A1_hi B1_lo + A1_lo B1_hi
        asm volatile("tcgen05.fence::after_thread_sync;");
        mma_batch_3x<K1 / 8, NH / 8>(tmem + cD, tmem + cY, tmem + cX, dB1, IDESC, bar, LO1);
      }
      TCG_WAIT(bar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      TCG_T(6);
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
      TCG_T(7);
#ifdef CCRD_TCG_TIMING
      tacc[7] += 1;  // blocks
#endif
    }
    // one fp64 partial per warp and tile (fixed order: deterministic)
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) tbits += __shfl_xor_sync(0xffffffffu, tbits, o2);
    if (lane == 0) p.partial[(int64_t)tile * 4 + qd] = (double)tbits;
  }
#ifdef CCRD_TCG_TIMING
  if (tw == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));
    tacc[9] = t_ - tstart;
  }
  if (t == 0 && blockIdx.x < 1024)
    for (int k = 0; k < 12; k++) g_tcg_timing[blockIdx.x][k] = tacc[k];
#endif
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  pdl_wait();  // complete only after the previous kernel of the stream (TMEM already released)
}


// ---------------------------------------------------------------- ping-pong warpgroups
// arm_tcg_kernel's arithmetic with TWO blocks of 128 latents in flight per
// warpgroup (TMEM slot pair, one mbarrier each): a warpgroup's MMA latency
// (measured 467 / 569 cycles for the 6 / 11-MMA batches alone,
// tools/microbench/tc_bench.cu) overlaps the other block's stage instead of
// idling.  Per pair of blocks (A, B):
//   wait MMA0(A); epi0(A); MMA1(A) | wait MMA0(B); epi0(B); MMA1(B) |
//   wait MMA1(A); epi1(A); gather(A'); MMA0(A') | wait MMA1(B); epi1(B); gather(B'); MMA0(B')
// The blocks of a warpgroup are its tiles' 4 blocks in order (A = q 0 / 2, B =
// q 1 / 3), so a tile's window is staged before gather(q 0) and its last
// reader is gather(q 3).
template <int C, int NH>
struct ArmTcpShape {
  using G = ArmTcgShape<C, NH>;
  static constexpr int SLOT = G::SLOT;                       // TMEM columns per block in flight
#ifndef CCRD_TCP_NWG
#define CCRD_TCP_NWG 3
#endif
  static constexpr int NWG = (512 / (2 * SLOT)) < CCRD_TCP_NWG ? (512 / (2 * SLOT)) : CCRD_TCP_NWG;
  static constexpr int THREADS = NWG * 128;
  static constexpr int USED = NWG * 2 * SLOT;  // TMEM columns used; the allocation is the next power of two
  static constexpr int TMEM_COLS = USED <= 32 ? 32 : USED <= 64 ? 64 : USED <= 128 ? 128 : USED <= 256 ? 256 : 512;
  static constexpr size_t smem_bytes(int b_floats, bool tma) {
    return sizeof(float) * ((size_t)b_floats + (size_t)NWG * G::WINP) + (tma ? (size_t)NWG * 2 * G::RAWB : 0) +
           8 * 4 * NWG + 16;
  }
};

#ifndef CCRD_TCP_MAXREG
#define CCRD_TCP_MAXREG 104  // 384 x 104 + a synthesis CTA (256 x 96) fit one SM's 64 K registers
#endif
template <int C, int NH, int NHL, bool STD, bool TMA>
__global__ void __maxnreg__(CCRD_TCP_MAXREG)
    arm_tcp_kernel(const __grid_constant__ ArmTcParams<C, NH, NHL> p) {
  using S = ArmTcShape<C, NH, NHL>;
  using G = ArmTcgShape<C, NH>;
  using Q = ArmTcpShape<C, NH>;
  constexpr int K0 = S::K0, K1 = S::K1, NWG = Q::NWG;
  extern __shared__ __align__(1024) float tsm[];
  float* sB = tsm;
  float* wins = tsm + S::B_FLOATS;
  int16_t* raws = reinterpret_cast<int16_t*>(wins + NWG * G::WINP);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(raws) + (TMA ? NWG * 2 * G::RAWB : 0));
  uint64_t* tbars = bars + 2 * NWG;  // TMA: 2 per warpgroup
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tbars + 2 * NWG);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int g = warp >> 2, qd = warp & 3, tw = t & 127;
  __shared__ __align__(8) uint64_t wbar;  // the weights' bulk copy
  pdl_trigger();  // the next image's ARM may be scheduled as this grid drains
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(Q::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t < 4 * NWG) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + t)));
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wbar)));
  // operand-ready barriers [warpgroup][slot][A0 | A1]: each warp arrives after
  // its TMEM stores, only the issuing warp waits (the others go on)
  __shared__ __align__(8) uint64_t rbar[4][4];
  if (t < 4 * NWG) asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(&rbar[t >> 2][t & 3])));
  __shared__ uint32_t s_big[4];  // per warpgroup: some window held a latent outside +-2048
  if (t < 4) s_big[t] = 0;       // (before the CTA barrier below)
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // the split weights (B operands, ~14 KB) in one bulk copy from global memory
  // (a per-thread copy from the kernel-parameter bank serialises in the
  // constant cache: ~7 % of the kernel's stall samples)
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&wbar)), "r"(4 * S::B_FLOATS)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sB)),
                 "l"(p.gB), "r"(4 * S::B_FLOATS), "r"(smem_u32(&wbar))
                 : "memory");
  }
  const uint32_t tmem = *tmem_slot;
  const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
  uint32_t cX[2], cY[2], cD[2];
#pragma unroll
  for (int s = 0; s < 2; s++) {
    cX[s] = (uint32_t)((2 * g + s) * G::SLOT);
    cY[s] = cX[s] + G::XC;
    cD[s] = cY[s] + G::YC;
    float cst[8] = {1.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    tmem_st_cols<8>(tl + cY[s] + NH, cst);  // the constant bias input of A1_hi
  }
  tmem_wait_st();
  float* win = wins + g * G::WINP;
  uint64_t* bar = bars + 2 * g;  // one per slot
  uint32_t ph[2] = {0, 0};
  uint32_t rph = 0;  // phase bits of rbar[g][2 s + k]
  constexpr uint32_t IDESC =
      (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NH >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
  const uint32_t sB_u = smem_u32(sB);
  const uint64_t dB0 = umma_desc(sB_u, 128, (K0 / 4) * 128);
  const uint64_t dB1 = umma_desc(sB_u + 8 * S::BW0, 128, (K1 / 4) * 128);
  constexpr uint32_t LO0 = (4 * S::BW0) >> 4, LO1 = (4 * S::BW1) >> 4;

  const int n_tiles = p.g.tile_begin[p.g.L];
  const int stride = (int)gridDim.x * NWG;
  const int first = (int)blockIdx.x * NWG + g;
  const int my_tiles = first < n_tiles ? (n_tiles - 1 - first) / stride + 1 : 0;
  const int nb = 4 * my_tiles;
  auto locate = [&](int tile, int& l, int& i0, int& j0) {
    l = 0;
#pragma unroll 1
    while (l + 1 < p.g.L && tile >= p.g.tile_begin[l + 1]) l++;
    const int tt = tile - p.g.tile_begin[l];
    const int ty = tile_row(tt, p.g.tiles_x[l], p.g.tx_mul[l]);
    i0 = p.g.own_lo[l] + ty * ARM_TY;
    j0 = (tt - ty * p.g.tiles_x[l]) * ARM_TX;
  };
  int16_t* raw = raws + g * G::RAWB;
  auto tma_window = [&](int tile, int b) {
    int tl_, ti0, tj0;
    locate(tile, tl_, ti0, tj0);
    uint64_t* tb = tbars + 2 * g + b;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(tb)), "r"(2 * G::RAWW * ARM_SH)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(raw + b * (G::RAWB / 2))),
        "l"(reinterpret_cast<uint64_t>(&p.tmap[tl_])), "r"(smem_u32(tb)), "r"(tj0 - ARM_HALO_X - 4),
        "r"(ti0 - ARM_HALO_TOP - p.g.lv.lo[tl_])
        : "memory");
  };
  // current tile (the one whose window is staged)
  int c_l = 0, c_i0 = 0, c_j0 = 0, c_it = -1;
  int c_w = 0, c_oh = 0;  // the tile's grid width and owned-row end (per tile, not per block)
  auto stage = [&](int it) {  // stage the window of this warpgroup's it-th tile
    const int tile = first + it * stride;
    locate(tile, c_l, c_i0, c_j0);
    c_it = it;
    c_w = p.g.lv.w[c_l];
    c_oh = p.g.own_hi[c_l];
    const int w = p.g.lv.w[c_l], rlo = p.g.lv.lo[c_l], rhi = p.g.lv.hi[c_l];
    bool big = false;
    if constexpr (TMA) {
      if (tw == 0 && it + 1 < my_tiles) tma_window(tile + stride, (it + 1) & 1);
      mbar_wait(tbars + 2 * g + (it & 1), (it >> 1) & 1);
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
        big |= fmaxf(fmaxf(fabsf(f.x), fabsf(f.y)), fmaxf(fabsf(f.z), fabsf(f.w))) > 2048.0f;
      }
    } else {
      big = stage_window_ldg<G::WIN>(p.lat, p.g, c_l, c_i0, c_j0, win, tw);
    }
    // a latent outside +-2048 in the window is not exact in tf32 (11
    // significant bits): the tile is redone with a split context after the
    // main loop (no branch in the hot loop)
    if (big) s_big[g] = 1;
    wg_sync(g);
  };
  if (TMA && tw == 0 && my_tiles > 0) tma_window(first, 0);

  // per-slot state of the block in flight: centre value, validity, index
  float ys[2];
  bool valid[2];
  int64_t qidx[2] = {0, 0};
  float tbits = 0.0f;
  // block b (tile b / 4, q = b % 4) into slot s, then MMA0; SPLIT: the exact
  // path with the context split c = c_hi + c_lo (window staged by the caller)
  auto gather = [&](int b, int s, auto split_tag) {
    constexpr bool SPLIT = decltype(split_tag)::value;
    const int q = b & 3;
    if (!SPLIT && q == 0) stage(b >> 2);
    const int ry = 2 * q + (tw >> 6), cx = tw & 63;
    const float* center = win + (ry + ARM_HALO_TOP) * ARM_SW + cx + ARM_HALO_X;
    ys[s] = center[0];
    {
      float row[C], tail[8] = {1.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int c = 0; c < C; c++) row[c] = center[STD ? std_ctx_dy(c) * ARM_SW + std_ctx_dx(c) : p.g.ctx_off[c]];
      if constexpr (SPLIT) split_ctx<C>(row, tl + cD[s]);  // c_lo -> the D1 columns (free until MMA1)
      tmem_st_cols<C>(tl + cX[s], row);
      tmem_st_cols<8>(tl + cX[s] + C, tail);
    }
    const int i = c_i0 + ry, j = c_j0 + cx;
    valid[s] = i < c_oh && j < c_w;
    if (p.bits != nullptr) qidx[s] = p.g.lv.off[c_l] + (int64_t)(i - p.g.lv.lo[c_l]) * c_w + j;  // debug outputs only
    tmem_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rbar[g][2 * s])) : "memory");
    if (qd == (b & 3)) {
      if (b < 2) mbar_wait(&wbar, 0);  // the first use of the weights in shared memory
      mbar_wait(&rbar[g][2 * s], (rph >> (2 * s)) & 1u);  // every warp's A0 rows are in TMEM
      asm volatile("tcgen05.fence::after_thread_sync;");
      if constexpr (SPLIT)  // + c_lo (B0_hi + B0_lo)
        mma_batch_4t<K0 / 8, C / 8>(tmem + cY[s], tmem + cX[s], tmem + cD[s], dB0, IDESC, bar + s, LO0);
      else
        mma_batch_hilo<K0 / 8>(tmem + cY[s], tmem + cX[s], dB0, IDESC, bar + s, LO0);
    }
    rph ^= 1u << (2 * s);
  };
  auto epi0 = [&](int b, int s) {
    TCG_WAIT(bar + s, ph[s]);
    ph[s] ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    float z[NH], lo[NH];
    tmem_ld_cols<NH>(tl + cY[s], z);
#pragma unroll
    for (int n = 0; n < NH; n += 2) {
      const float r0 = fmaxf(z[n], 0.0f), r1 = fmaxf(z[n + 1], 0.0f);
      z[n] = __uint_as_float(__float_as_uint(r0) & 0xFFFFE000u);
      z[n + 1] = __uint_as_float(__float_as_uint(r1) & 0xFFFFE000u);
      const float2 d = f2unpack(fsub2(f2pack(r0, r1), f2pack(z[n], z[n + 1])));
      lo[n] = d.x;
      lo[n + 1] = d.y;
    }
    tmem_st_cols<NH>(tl + cY[s], z);
    tmem_st_cols<NH>(tl + cX[s], lo);
    tmem_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rbar[g][2 * s + 1])) : "memory");
    if (qd == (b & 3)) {
      mbar_wait(&rbar[g][2 * s + 1], (rph >> (2 * s + 1)) & 1u);  // every warp's A1 rows are in TMEM
      asm volatile("tcgen05.fence::after_thread_sync;");
      mma_batch_3x<K1 / 8, NH / 8>(tmem + cD[s], tmem + cY[s], tmem + cX[s], dB1, IDESC, bar + s, LO1);
    }
    rph ^= 1u << (2 * s + 1);
  };
  auto epi1 = [&](int b, int s) {
    TCG_WAIT(bar + s, ph[s]);
    ph[s] ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    float z[NH];
    tmem_ld_cols<NH>(tl + cD[s], z);
    // output layer: 4 independent FFMA2 chains (2 per output) over input pairs
    uint64_t am0 = f2pack(p.bo.x, 0.0f), as0 = f2pack(p.bo.y, 0.0f), am1 = 0ull, as1 = 0ull;
#pragma unroll
    for (int n = 0; n < NH; n += 4) {
      const uint64_t r2 = f2pack(fmaxf(z[n], 0.0f), fmaxf(z[n + 1], 0.0f));
      am0 = ffma2(r2, ldp2(p.wm[n / 2]), am0);
      as0 = ffma2(r2, ldp2(p.wsl[n / 2]), as0);
      if (n + 2 < NH) {
        const uint64_t r3 = f2pack(fmaxf(z[n + 2], 0.0f), fmaxf(z[n + 3], 0.0f));
        am1 = ffma2(r3, ldp2(p.wm[n / 2 + 1]), am1);
        as1 = ffma2(r3, ldp2(p.wsl[n / 2 + 1]), as1);
      }
    }
    const float2 m0 = f2unpack(am0), m1 = f2unpack(am1), s0 = f2unpack(as0), s1 = f2unpack(as1);
    const float mu = (m0.x + m1.x) + (m0.y + m1.y), ls = (s0.x + s1.x) + (s0.y + s1.y);
    {  // bits computed unconditionally (no branch around the MUFU chain), masked
      const float bits_v = laplace_bits(ys[s], mu, ls, p.g);
      const float bits = valid[s] ? bits_v : 0.0f;
      tbits += bits;
      if (valid[s] && p.bits != nullptr) {
        p.bits[qidx[s]] = bits;
        if (p.mu) p.mu[qidx[s]] = mu;
        if (p.scale) p.scale[qidx[s]] = __expf(fminf(fmaxf(ls, p.g.lsmin), p.g.lsmax));
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if ((b & 3) == 3) {  // the tile's last block: one fp64 partial per warp
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) tbits += __shfl_xor_sync(0xffffffffu, tbits, o2);
      if (lane == 0) p.partial[(int64_t)(first + (b >> 2) * stride) * 4 + qd] = (double)tbits;
      tbits = 0.0f;
    }
  };

  if (nb > 0) {
    const std::integral_constant<bool, false> fast;
    gather(0, 0, fast);
    gather(1, 1, fast);
#pragma unroll 1
    for (int b = 0; b < nb; b += 2) {
      epi0(b, 0);
      epi0(b + 1, 1);
      epi1(b, 0);
      if (b + 2 < nb) gather(b + 2, 0, fast);
      epi1(b + 1, 1);
      if (b + 3 < nb) gather(b + 3, 1, fast);
    }
  }
  // exact pass: every tile of this warpgroup whose window holds a latent
  // outside +-2048 again, context split, one block at a time in slot 0 (its
  // partials and per-latent outputs overwrite the main loop's)
  if (s_big[g]) {
    const std::integral_constant<bool, true> split;
#pragma unroll 1
    for (int it = 0; it < my_tiles; it++) {
      locate(first + it * stride, c_l, c_i0, c_j0);
      c_w = p.g.lv.w[c_l];
      c_oh = p.g.own_hi[c_l];
      const bool big = stage_window_ldg<G::WIN>(p.lat, p.g, c_l, c_i0, c_j0, win, tw);
      if (wg_sync_or(g, big)) {
#pragma unroll 1
        for (int q = 0; q < 4; q++) {
          gather(4 * it + q, 0, split);
          epi0(4 * it + q, 0);
          epi1(4 * it + q, 0);
        }
      }
      wg_sync(g);  // the window's readers are done before the next tile overwrites it
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Q::TMEM_COLS));
  pdl_wait();  // complete only after the previous kernel of the stream (TMEM already released)
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
  P p;  // ~2.5 KB, copied into the launch's parameter bank
  memset(&p, 0, sizeof(p));
  ArmTcB<C, NH, NHL> hb;  // the B operands, to global memory below
  memset(&hb, 0, sizeof(hb));
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
    for (int i = 0; i < C; i++) put(hb.B0[0], hb.B0[1], n, i, S::K0, q[n * C + i] + ((res(0) && i == n) ? 1.0f : 0.0f));
    put(hb.B0[0], hb.B0[1], n, C, S::K0, q[C * NH + n]);
  }
  q += C * NH + NH;
  for (int k = 0; k < NHL - 1; k++) {
    for (int n = 0; n < NH; n++) {
      for (int i = 0; i < NH; i++)
        put(hb.B1[k][0], hb.B1[k][1], n, i, S::K1, q[n * NH + i] + ((res(k + 1) && i == n) ? 1.0f : 0.0f));
      put(hb.B1[k][0], hb.B1[k][1], n, NH, S::K1, q[NH * NH + n]);
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
  // the B operands to global memory: the scratch after the 16 reserved partial
  // slots per tile (ARM_W_SCRATCH in ccrd_api.cu); pageable source, so the call
  // returns once the driver has staged it (p may go out of scope)
  float* gB = reinterpret_cast<float*>(partial + (size_t)tiles * 16);
  static_assert(4 * S::B_FLOATS <= 8 * ARM_W_SCRATCH_DOUBLES, "weight scratch");
  static_assert(sizeof(hb) == sizeof(float) * S::B_FLOATS, "packed B layout");
  // ARM_LAUNCH_ONLY: an earlier ARM_STAGE_ONLY call of this image staged gB
  // (a batch stages every image's weights before its first ARM kernel, so no
  // copy sits between two ARM kernels of the stream)
  if (g_launch_ctl.arm_stage != ARM_LAUNCH_ONLY &&
      cudaMemcpyAsync(gB, &hb, sizeof(hb), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return -1;
  if (g_launch_ctl.arm_stage == ARM_STAGE_ONLY) return 0;
  p.gB = gB;
  const bool tma = arm_tma_maps(g, lat, p.tmap);
  const bool sc = is_std_ctx(d);
  // default: ping-pong warpgroups (two blocks in flight each, arm_tcp_kernel);
  // CCRD_ARM_TC_PP=0 selects the one-block warpgroups (arm_tcg_kernel)
  static const bool pp = !(getenv("CCRD_ARM_TC_PP") && getenv("CCRD_ARM_TC_PP")[0] == '0');
  if (pp) {
    using Q = ArmTcpShape<C, NH>;
    constexpr size_t qs_t = Q::smem_bytes(S::B_FLOATS, true), qs_n = Q::smem_bytes(S::B_FLOATS, false);
    static bool attr_p = false;
    if (!attr_p) {
      cudaFuncSetAttribute(arm_tcp_kernel<C, NH, NHL, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qs_t);
      cudaFuncSetAttribute(arm_tcp_kernel<C, NH, NHL, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qs_t);
      cudaFuncSetAttribute(arm_tcp_kernel<C, NH, NHL, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qs_n);
      cudaFuncSetAttribute(arm_tcp_kernel<C, NH, NHL, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qs_n);
      attr_p = true;
    }
    const int need = (tiles + Q::NWG - 1) / Q::NWG, cap = device_sm_count() * (512 / Q::TMEM_COLS);
    auto kp = tma ? (sc ? arm_tcp_kernel<C, NH, NHL, true, true> : arm_tcp_kernel<C, NH, NHL, false, true>)
                  : (sc ? arm_tcp_kernel<C, NH, NHL, true, false> : arm_tcp_kernel<C, NH, NHL, false, false>);
    launch_ctl(kp, (unsigned)(need < cap ? need : cap), Q::THREADS, tma ? qs_t : qs_n, stream, p);
    return 1;
  }
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
  const int need = (tiles + G::NWG - 1) / G::NWG, cap = device_sm_count();
  auto kern = tma ? (sc ? arm_tcg_kernel<C, NH, NHL, true, true> : arm_tcg_kernel<C, NH, NHL, false, true>)
                  : (sc ? arm_tcg_kernel<C, NH, NHL, true, false> : arm_tcg_kernel<C, NH, NHL, false, false>);
  launch_ctl(kern, (unsigned)(need < cap ? need : cap), G::THREADS, tma ? smem_t : smem_n, stream, p);
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

// rate partials per 8 x 64 tile written by the tensor-core kernels (one per warp)
int arm_tc_partials_per_tile() { return 4; }

ArmLaunchFn find_arm_tc_launcher(int C, int NH, int NHL) {
  for (const auto& e : kArmTc)
    if (e.C == C && e.NH == NH && e.NHL == NHL) return e.fn;
  return nullptr;
}

}  // namespace ccrd

#ifdef CCRD_TCG_TIMING
extern "C" int cc_debug_tcg_timing(unsigned long long* host, int n_cta) {
  return (int)cudaMemcpyFromSymbol(host, ccrd::g_tcg_timing, sizeof(unsigned long long) * 12 * (size_t)n_cta);
}
#endif
