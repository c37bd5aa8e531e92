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
#include "arm_math.cuh"
#include "ccrd_common.cuh"

namespace ccrd {

template <int C, int NH, int NHL>
__global__ void __launch_bounds__(ARM_THREADS, ARM_CTAS_PER_SM)
    arm_rate_kernel(const __grid_constant__ ArmParams<C, NH, NHL> p) {
  constexpr int M = ARM_LPT;
  constexpr int N = ARM_SH * ARM_SW;
  constexpr int IT = (N + ARM_THREADS - 1) / ARM_THREADS;
  __shared__ float tile[N];
  pdl_trigger();

  // (level, tile) of this CTA through the prefix table
  const int b = blockIdx.x;
  int l = 0;
#pragma unroll 1
  while (l + 1 < p.g.L && b >= p.g.tile_begin[l + 1]) l++;
  const int w = p.g.lv.w[l];
  const int rlo = p.g.lv.lo[l], rhi = p.g.lv.hi[l];  // buffer window (full image: 0 .. h)
  const int own_hi = p.g.own_hi[l];
  const int t = b - p.g.tile_begin[l];
  const int ty = tile_row(t, p.g.tiles_x[l], p.g.tx_mul[l]);
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
  pdl_wait();  // complete only after the previous kernel of the stream
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
  if (g_launch_ctl.arm_stage == ARM_STAGE_ONLY) return 0;  // weights travel in the parameters
  pack_arm_weights<C, NH, NHL>(d, arm_w, p.w);

  launch_ctl(arm_rate_kernel<C, NH, NHL>, (unsigned)g.tile_begin[g.L], ARM_THREADS, 0, stream, p);
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
