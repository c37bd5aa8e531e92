// arm_rate.cu -- ARM rate kernel: causal context gather, ARM MLP f_psi, Laplace
// bin probability and -log2, summed over every latent of every grid in ONE
// launch (PAPER.md:106-109 ARM, :120 R term of Eq. 1; Table 1 ARM column).
//
// Design (B200, FP32-FMA bound):
//   * one CTA = one tile of 8 rows x 64 latents of one grid; the tiles of all
//     L grids form one launch, mapped to (level, tile) through a prefix table;
//   * the causal window (3 rows above, 4 columns each side) is staged from the
//     int16 pyramid into shared memory as fp32, zero outside the grid;
//   * two latents per thread; the MLP weights live in the kernel-parameter
//     bank (uniform operands, no LSU traffic), every multiply-accumulate is a
//     packed FFMA2 producing two output neurons, and every uniform weight load
//     feeds both latents;
//   * stable Laplace -log2 P in fp32; bits -> warp shuffle -> one fp64 partial
//     per warp (fixed order; final sum in ccrd_api.cu).
#include "ccrd_common.cuh"

namespace ccrd {

// -log2 of the Laplace(mu, b) mass of the bin [y - 1/2, y + 1/2], floored at
// p_floor (readings #1-#3).  With a = |y - mu| and
// ib = 1/b:
//   a <  1/2 : P = 1 - (exp(-(1/2 - a) ib) + exp(-(1/2 + a) ib)) / 2
//   a >= 1/2 : -log2 P = 1 + (a - 1/2) ib log2(e) - log2(1 - exp(-ib))
// (the second form is log-domain, so far tails do not underflow).
// All exponentials / logarithms are single MUFU ops (ex2 / lg2): the worst
// case, 1 - exp(-ib) at b = 256, cancels to ~1e-4 bits per latent, inside the
// 1e-3-bit per-latent parity tolerance.
__device__ __forceinline__ float laplace_bits(float y, float mu, float s, const ArmGeom& g) {
  constexpr float LOG2E = 1.4426950408889634f;
  s = fminf(fmaxf(s, g.lsmin), g.lsmax);
  const float ibl = exp2f_approx(-s * LOG2E) * LOG2E;  // log2(e) / b
  const float a = fabsf(y - mu);
  const float am = fminf(a, 0.5f);
  const float e1 = exp2f_approx((am - 0.5f) * ibl);
  const float e2 = exp2f_approx(-(am + 0.5f) * ibl);
  const float p_in = 1.0f - 0.5f * (e1 + e2);
  const float bits_in = -log2f_approx(fmaxf(p_in, g.p_floor));
  const float bits_out = fmaf(a - 0.5f, ibl, 1.0f) - log2f_approx(1.0f - exp2f_approx(-ibl));
  return fminf(a < 0.5f ? bits_in : bits_out, g.bits_cap);
}

// One dense layer NIN -> 2*NO2 for NLAT latents with FFMA2 (two output neurons
// per instruction; each uniform weight pair feeds NLAT instructions).
template <int NLAT, int NIN, int NO2, bool RELU>
__device__ __forceinline__ void dense_ffma2(const float (&in)[NLAT][NIN], float (&out)[NLAT][2 * NO2],
                                            const float2 (&W)[NIN][NO2], const float2 (&B)[NO2]) {
  uint64_t acc[NLAT][NO2];
#pragma unroll
  for (int n = 0; n < NO2; n++) {
    const uint64_t b = ldp2(B[n]);
#pragma unroll
    for (int m = 0; m < NLAT; m++) acc[m][n] = b;
  }
  // latent-major inner order: one activation feeds NO2 consecutive FFMA2
  // (operand-reuse cache), the NO2 weight pairs stay in uniform registers
#pragma unroll
  for (int i = 0; i < NIN; i++) {
#pragma unroll
    for (int m = 0; m < NLAT; m++) {
      const uint64_t x = f2pack(in[m][i], in[m][i]);
#pragma unroll
      for (int n = 0; n < NO2; n++) acc[m][n] = ffma2(x, ldp2(W[i][n]), acc[m][n]);
    }
  }
#pragma unroll
  for (int m = 0; m < NLAT; m++)
#pragma unroll
    for (int n = 0; n < NO2; n++) {
      float2 v = f2unpack(acc[m][n]);
      out[m][2 * n] = RELU ? fmaxf(v.x, 0.0f) : v.x;
      out[m][2 * n + 1] = RELU ? fmaxf(v.y, 0.0f) : v.y;
    }
}

template <int C, int NH, int NHL>
__global__ void __launch_bounds__(ARM_THREADS, ARM_CTAS_PER_SM)
    arm_rate_kernel(const __grid_constant__ ArmParams<C, NH, NHL> p) {
  constexpr int M = ARM_LPT;
  constexpr int N = ARM_SH * ARM_SW;
  constexpr int IT = (N + ARM_THREADS - 1) / ARM_THREADS;
  __shared__ float tile[N];

  // (level, tile) of this CTA through the prefix table
  const int b = blockIdx.x;
  int l = 0;
#pragma unroll 1
  while (l + 1 < p.g.L && b >= p.g.tile_begin[l + 1]) l++;
  const int w = p.g.lv.w[l];
  const int rlo = p.g.lv.lo[l], rhi = p.g.lv.hi[l];  // buffer window (full image: 0 .. h)
  const int own_hi = p.g.own_hi[l];
  const int t = b - p.g.tile_begin[l];
  const int ty = t / p.g.tiles_x[l];
  const int i0 = p.g.own_lo[l] + ty * ARM_TY, j0 = (t - ty * p.g.tiles_x[l]) * ARM_TX;
  const int16_t* __restrict__ grid = p.lat + p.g.lv.off[l];

  // stage the causal window, fp32, zero outside the grid (reading #5; the
  // buffer window contains every row an owned latent's context reaches); every
  // load is issued before the first store
  {
    int16_t v[IT];
#pragma unroll
    for (int k = 0; k < IT; k++) {
      const int s = threadIdx.x + k * ARM_THREADS;
      const int r = s / ARM_SW, c = s - r * ARM_SW;
      const int gi = i0 - ARM_HALO_TOP + r, gj = j0 - ARM_HALO_X + c;
      v[k] = (s < N && gi >= rlo && gi < rhi && gj >= 0 && gj < w) ? __ldg(grid + (int64_t)(gi - rlo) * w + gj)
                                                                  : (int16_t)0;
    }
#pragma unroll
    for (int k = 0; k < IT; k++) {
      const int s = threadIdx.x + k * ARM_THREADS;
      if (s < N) tile[s] = (float)v[k];
    }
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int i = i0 + ly;

  // context gather (reading #4: offsets in template order)
  float z0[M][C], y[M];
#pragma unroll
  for (int m = 0; m < M; m++) {
    const float* center = tile + (ly + ARM_HALO_TOP) * ARM_SW + (lane + 32 * m + ARM_HALO_X);
#pragma unroll
    for (int c = 0; c < C; c++) z0[m][c] = center[p.g.ctx_off[c]];
    y[m] = center[0];
  }

  // ARM MLP: C -> NH (ReLU) -> [NH -> NH (ReLU)] x (NHL-1) -> 2
  float z[M][NH];
  dense_ffma2<M, C, NH / 2, true>(z0, z, p.w.w0, p.w.b0);
#pragma unroll
  for (int k = 0; k < NHL - 1; k++) {
    float zn[M][NH];
    dense_ffma2<M, NH, NH / 2, true>(z, zn, p.w.wh[k], p.w.bh[k]);
#pragma unroll
    for (int m = 0; m < M; m++)
#pragma unroll
      for (int n = 0; n < NH; n++) z[m][n] = zn[m][n];
  }
  uint64_t o[M];
#pragma unroll
  for (int m = 0; m < M; m++) o[m] = ldp2(p.w.bo);
#pragma unroll
  for (int n = 0; n < NH; n++) {
    const uint64_t wo = ldp2(p.w.wo[n]);
#pragma unroll
    for (int m = 0; m < M; m++) o[m] = ffma2(f2pack(z[m][n], z[m][n]), wo, o[m]);
  }

  float bits = 0.0f;
#pragma unroll
  for (int m = 0; m < M; m++) {
    const int j = j0 + lane + 32 * m;
    if (i < own_hi && j < w) {
      const float2 ms = f2unpack(o[m]);
      const float bm = laplace_bits(y[m], ms.x, ms.y, p.g);
      bits += bm;
      if (p.bits != nullptr) {
        const int64_t q = p.g.lv.off[l] + (int64_t)(i - rlo) * w + j;
        p.bits[q] = bm;
        if (p.mu) p.mu[q] = ms.x;
        if (p.scale) p.scale[q] = __expf(fminf(fmaxf(ms.y, p.g.lsmin), p.g.lsmax));
      }
    }
  }
  // one fp64 partial per warp (fixed order; no second CTA barrier)
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o2);
  if (lane == 0) p.partial[b * (ARM_THREADS / 32) + ly] = (double)bits;
}

// ---------------------------------------------------------------- host launcher
template <int C, int NH, int NHL>
static int launch_arm(const ArmGeom& g, const cc_model_desc& d, const float* arm_w,
                      const int16_t* lat, double* partial, float* mu, float* scale, float* bits,
                      cudaStream_t stream) {
  ArmParams<C, NH, NHL> p;
  p.g = g;
  p.lat = lat;
  p.partial = partial;
  p.mu = mu;
  p.scale = scale;
  p.bits = bits;
  // pack weights (blob: per layer W[out][in] then b[out]); fold residuals
  const float* q = arm_w;
  auto res = [&](int k) { return (d.arm_residual_mask >> k) & 1u; };
  for (int i = 0; i < C; i++)
    for (int n = 0; n < NH / 2; n++) {
      float a = q[(2 * n) * C + i], b = q[(2 * n + 1) * C + i];
      if (res(0)) {  // only legal when C == NH (validated)
        a += (i == 2 * n) ? 1.0f : 0.0f;
        b += (i == 2 * n + 1) ? 1.0f : 0.0f;
      }
      p.w.w0[i][n] = make_float2(a, b);
    }
  for (int n = 0; n < NH / 2; n++) p.w.b0[n] = make_float2(q[C * NH + 2 * n], q[C * NH + 2 * n + 1]);
  q += C * NH + NH;
  for (int k = 0; k < NHL - 1; k++) {
    for (int i = 0; i < NH; i++)
      for (int n = 0; n < NH / 2; n++) {
        float a = q[(2 * n) * NH + i], b = q[(2 * n + 1) * NH + i];
        if (res(k + 1)) {
          a += (i == 2 * n) ? 1.0f : 0.0f;
          b += (i == 2 * n + 1) ? 1.0f : 0.0f;
        }
        p.w.wh[k][i][n] = make_float2(a, b);
      }
    for (int n = 0; n < NH / 2; n++) p.w.bh[k][n] = make_float2(q[NH * NH + 2 * n], q[NH * NH + 2 * n + 1]);
    q += NH * NH + NH;
  }
  for (int i = 0; i < NH; i++) p.w.wo[i] = make_float2(q[i], q[NH + i]);
  p.w.bo = make_float2(q[2 * NH], q[2 * NH + 1]);

  arm_rate_kernel<C, NH, NHL><<<g.tile_begin[g.L], ARM_THREADS, 0, stream>>>(p);
  return 0;
}

struct ArmEntry {
  int C, NH, NHL;
  ArmLaunchFn fn;
};

// Compiled architectures: BASELINE.json configs ([8,8,8,2], [16,24,24,2]) and
// the Table 1 ARMs (A300 [8,8,2], A545 [8,8,8,2], A1079 [16,16,16,2],
// A2300 [24,24,24,2]).
static const ArmEntry kArm[] = {
    {8, 8, 1, launch_arm<8, 8, 1>},     {8, 8, 2, launch_arm<8, 8, 2>},
    {16, 16, 2, launch_arm<16, 16, 2>}, {16, 24, 2, launch_arm<16, 24, 2>},
    {24, 24, 2, launch_arm<24, 24, 2>},
};

ArmLaunchFn find_arm_launcher(int C, int NH, int NHL) {
  for (const auto& e : kArm)
    if (e.C == C && e.NH == NH && e.NHL == NHL) return e.fn;
  return nullptr;
}

}  // namespace ccrd
