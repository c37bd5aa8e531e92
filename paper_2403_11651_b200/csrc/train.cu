// train.cu -- ONE Cool-chic encoder training iteration on the GPU (NEXT-2).
//
// PAPER.md:113-126 (Eq. 1): the encoder minimises J = D(x, x_hat) +
// lambda R(y_hat) / (H W) over the latents and psi, upsilon, theta through the
// continuous latents y and a differentiable proxy of Q; "One
// training iteration consists in one forward pass and one backward pass";
// Adam on every parameter.  Readings (T1-T3):
// noise proxy y_hat = y + u with u given as input (the random numbers are
// data), gradient passed unchanged to y; ReLU'(0) = 0, no gradient through the
// log-scale clamp outside its range or through the probability floor.
//
// Parameter vector (device fp32, the layout of include/ccrd.h):
//   [ y (N_lat, packed like the latents) | arm_w | up_w | syn_w ].
// The weights (arm | up | syn, <= 8 KB) are copied device-to-device into a
// __constant__ bank at the start of the step, so every kernel reads them as
// uniform operands with compile-time offsets.
//
// First version (correctness first): simple kernels, intermediates materialised
// in HBM, one output element / latent / pixel per thread.
//   1. proxy       y_hat = y + u
//   2. ARM         forward + backward per latent: rate, d/dy_hat (own + context,
//                  the latter gathered in a second kernel: deterministic),
//                  per-CTA partial weight gradients (shared-memory outer products)
//   3. upsampling  separable stride-2 transposed-conv steps level by level,
//                  every step's input kept (dense [L][H][W] at the end)
//   4. synthesis   1x1 layers, residual 3x3 layers, distortion; then their
//                  adjoints (3x3 adjoint in gather form over the clamped
//                  neighbourhood = replicate padding's adjoint), per-block
//                  partial weight gradients
//   5. upsampling adjoint, in gather form, tap-gradient partials
//   6. fp64 reduction of every partial into the gradient, Adam, cost.
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "ccrd_common.cuh"

namespace ccrd {

constexpr int TR_MAX_W = 2048;  // arm + up + syn weights (floats)
// TR_BANKS copies of the constant banks: up to TR_BANKS images train
// concurrently on different streams (a stream keeps a bank; a stream taking
// over another stream's bank waits for that stream's last use of it).  Every
// kernel addresses its bank through the offsets it is given (bank x size +
// the layer offset): the loads stay uniform (LDCU c[0x3][UR + imm]).
constexpr int TR_BANKS = 4;
// bank layout: ARM weights at 0, upsampling taps at TR_UP_OFF, synthesis at
// TR_SYN_OFF -- fixed offsets, so kernels templated on the bank read their
// weights at compile-time constant addresses (uniform LDCU)
constexpr int TR_UP_OFF = 1280, TR_SYN_OFF = 1344;
__constant__ float c_tw[TR_BANKS * TR_MAX_W];
// the ARM weights again, packed for FFMA2 in the forward: per layer k, for
// input i the pair (W[2n][i], W[2n+1][i]), then the bias pairs
constexpr int TR_MAX_ARMP = 768;  // float2 (A2300's ARM: 627 pairs)
__constant__ float2 c_tp[TR_BANKS * TR_MAX_ARMP];

__global__ void tr_pack_arm_kernel(const float* __restrict__ w, float2* __restrict__ out, int nl, int C, int NH) {
  // one thread per output pair; layer k: nin x (nout/2) weight pairs then nout/2 bias pairs
  int src = 0, dst = 0;
  for (int k = 0; k < nl; k++) {
    const int nin = (k == 0) ? C : NH, nout = (k == nl - 1) ? 2 : NH, n2 = nout / 2;
    for (int e = threadIdx.x; e < nin * n2 + n2; e += blockDim.x) {
      if (e < nin * n2) {
        const int i = e / n2, n = e - i * n2;
        out[dst + e] = make_float2(w[src + (2 * n) * nin + i], w[src + (2 * n + 1) * nin + i]);
      } else {
        const int n = e - nin * n2;
        out[dst + e] = make_float2(w[src + nin * nout + 2 * n], w[src + nin * nout + 2 * n + 1]);
      }
    }
    src += nin * nout + nout;
    dst += nin * n2 + n2;
  }
}

constexpr int TA_THREADS = 128;  // ARM: latents per CTA
constexpr int TS_THREADS = 128;  // synthesis 1x1 backward: pixels per CTA
constexpr int TB = 256;          // generic elementwise / stencil kernels
constexpr int TR_GRID_CAP = 592; // grid-stride reductions: 4 CTAs per SM
#ifndef CCRD_TR_TCONV_CAP
#define CCRD_TR_TCONV_CAP 256
#endif
constexpr int TR_TCONV_CAP = CCRD_TR_TCONV_CAP;  // transposed-conv adjoint: blocks per channel

struct TrainLevels {
  int32_t L, H, W;
  int32_t h[CC_MAX_LEVELS], w[CC_MAX_LEVELS];
  int64_t off[CC_MAX_LEVELS];
  int64_t n_lat;
};

// --------------------------------------------------------------- 1. proxy
__global__ void tr_proxy_kernel(const float* __restrict__ y, const float* __restrict__ u, float* __restrict__ yq,
                                int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    yq[i] = y[i] + u[i];
}

// --------------------------------------------------------------- 2. ARM
struct TrainArmParams {
  TrainLevels lv;
  int32_t n_ctx;
  int32_t dy[CC_MAX_CTX], dx[CC_MAX_CTX];
  uint32_t res_mask;
  float lsmin, lsmax, bits_cap, w_r;  // w_r = lambda / (H W)
  const float* yq;
  float* gown;     // [N_lat]      w_r d bits / d y_hat (own position)
  float* dctx;     // [C][N_lat]   d J / d context value c of this latent (coalesced stores / gathers)
  double* rate;    // [CTAs][4]    per-warp bits
  float* wpart;    // [CTAs][n_arm] partial weight gradients
  int32_t n_arm;
  int32_t tw0, tp0;  // this step's constant-bank base offsets (c_tw, c_tp)
};

// bits and d bits / d (y, mu, s) -- fp32, IEEE exp / log (the hybrid stable
// form of the forward kernel and its derivative)
__device__ __forceinline__ float tr_bits(float y, float mu, float s, const TrainArmParams& p, float& gy,
                                         float& gmu, float& gs) {
  constexpr float LN2 = 0.6931471805599453f;
  const bool inside = s > p.lsmin && s < p.lsmax;
  const float sc = fminf(fmaxf(s, p.lsmin), p.lsmax);
  const float b = expf(sc), ib = 1.0f / b;
  const float d = y - mu, a = fabsf(d), sg = d >= 0.0f ? 1.0f : -1.0f;
  float bits, dbda, dbdb;
  if (a >= 0.5f) {  // log domain: bits = 1 + (a - 1/2) / (b ln2) - log2(1 - e^{-1/b})
    const float em = expm1f(ib);  // e^{1/b} - 1
    bits = 1.0f + (a - 0.5f) * ib / LN2 - log2f(-expm1f(-ib));
    dbda = ib / LN2;
    dbdb = (ib * ib / LN2) * (1.0f / em - (a - 0.5f));
  } else {
    const float e1 = expf(-(0.5f - a) * ib), e2 = expf(-(0.5f + a) * ib);
    const float P = 1.0f - 0.5f * (e1 + e2);
    bits = -log2f(P);
    const float dPda = -(e1 - e2) * 0.5f * ib;
    const float dPdb = -0.5f * ib * ib * (e1 * (0.5f - a) + e2 * (0.5f + a));
    dbda = -dPda / (P * LN2);
    dbdb = -dPdb / (P * LN2);
  }
  if (bits >= p.bits_cap) {  // probability floor: constant
    gy = gmu = gs = 0.0f;
    return p.bits_cap;
  }
  gy = sg * dbda;
  gmu = -sg * dbda;
  gs = inside ? dbdb * b : 0.0f;
  return bits;
}

// Shared-memory record of one latent for the weight-gradient outer products:
// per layer k the input [z_k, 1, 0 ...] (KIN[k] = round4(nin + 1) floats) and
// the output gradient du_k (nout floats, even); 16-byte aligned.
template <int C, int NH, int NHL>
struct TrArmLayout {
  static constexpr int NL = NHL + 1;
  __host__ __device__ static constexpr int r4(int x) { return (x + 3) / 4 * 4; }
  __host__ __device__ static constexpr int kin(int k) { return r4((k == 0 ? C : NH) + 1); }
  __host__ __device__ static constexpr int nout(int k) { return k == NL - 1 ? 2 : NH; }
  __host__ __device__ static constexpr int zoff(int k) { return k == 0 ? 0 : zoff(k - 1) + kin(k - 1); }
  __host__ __device__ static constexpr int zend() { return zoff(NL - 1) + kin(NL - 1); }
  __host__ __device__ static constexpr int doff(int k) { return k == 0 ? zend() : doff(k - 1) + r4(nout(k - 1)); }
  __host__ __device__ static constexpr int woff(int k) {
    return k == 0 ? 0 : woff(k - 1) + (k - 1 == 0 ? C : NH) * nout(k - 1) + nout(k - 1);
  }
  // weight-gradient tiles of layer k (4 or 2 outputs x 4 inputs) and the
  // warps they take when each layer gets warps of its own
  __host__ __device__ static constexpr int ntile(int k) { return (kin(k) / 4) * (nout(k) % 4 == 0 ? nout(k) / 4 : nout(k) / 2); }
  __host__ __device__ static constexpr int nw(int k) { return (ntile(k) + 31) / 32; }
  __host__ __device__ static constexpr int wstart(int k) { return k == 0 ? 0 : wstart(k - 1) + nw(k - 1); }
  __host__ __device__ static constexpr int wsum() { return wstart(NL - 1) + nw(NL - 1); }
  static constexpr int VEC_RAW = doff(NL - 1) + r4(2);
  static constexpr int VEC = VEC_RAW + ((VEC_RAW / 4) % 2 == 0 ? 4 : 0);  // odd number of 16-byte words: bank spread
  static_assert(NL <= 4, "up to 3 hidden layers");
};

// Weight gradient of layer K over one CTA's latents, as a register-blocked
// outer product: the thread owns a TR (outputs: 4, or 2 for the output layer)
// x 4 (inputs; the input column nin is the constant 1 = the bias) tile with
// two interleaved partial sums, reading per latent one float4 (float2) of du
// and one float4 of z from the shared records; FFMA2 over input pairs (each
// lane its own fma chain: the same sums as scalar FMA).
template <int C, int NH, int NHL, int K>
__device__ __forceinline__ void tr_wgrad_tile(const float* tsm, const int tile, float* __restrict__ wp) {
  using LY = TrArmLayout<C, NH, NHL>;
  constexpr int NL = NHL + 1, VEC = LY::VEC;
  constexpr int nin = (K == 0) ? C : NH, nout = (K == NL - 1) ? 2 : NH;
  constexpr int tcols = LY::kin(K) / 4, TR = (nout % 4 == 0) ? 4 : 2;
  const int tr = tile / tcols, tc = tile - tr * tcols;
  const float* dp = tsm + LY::doff(K) + TR * tr;
  const float* zp = tsm + LY::zoff(K) + 4 * tc;
  uint64_t acc[2][TR][2];
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int a = 0; a < TR; a++) acc[h][a][0] = acc[h][a][1] = 0ull;
#pragma unroll 8
  for (int m = 0; m < TA_THREADS; m += 2) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      float dv[TR];
      if constexpr (TR == 4) {
        const float4 dd = *reinterpret_cast<const float4*>(dp + (m + h) * VEC);
        dv[0] = dd.x, dv[1] = dd.y, dv[2] = dd.z, dv[3] = dd.w;
      } else {
        const float2 dd = *reinterpret_cast<const float2*>(dp + (m + h) * VEC);
        dv[0] = dd.x, dv[1] = dd.y;
      }
      const ulonglong2 zz = *reinterpret_cast<const ulonglong2*>(zp + (m + h) * VEC);
#pragma unroll
      for (int a = 0; a < TR; a++) {
        const uint64_t d2 = f2pack(dv[a], dv[a]);
        acc[h][a][0] = ffma2(d2, zz.x, acc[h][a][0]);
        acc[h][a][1] = ffma2(d2, zz.y, acc[h][a][1]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < TR; a++)
#pragma unroll
    for (int bp = 0; bp < 2; bp++) {
      const float2 x0 = f2unpack(acc[0][a][bp]), x1 = f2unpack(acc[1][a][bp]);
      const float vv[2] = {x0.x + x1.x, x0.y + x1.y};
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int o = TR * tr + a, i2 = 4 * tc + 2 * bp + e;
        if (i2 < nin) wp[LY::woff(K) + o * nin + i2] = vv[e];                 // W[o][i]
        else if (i2 == nin) wp[LY::woff(K) + nin * nout + o] = vv[e];         // b[o]
      }
    }
}

// BANK: the constant bank this step's weights sit in, a template parameter so
// the weight reads keep their immediate constant offsets (uniform LDCU; a
// runtime bank base turns them into per-thread LDC, -9% per iteration)
template <int C, int NH, int NHL, int BANK>
__global__ void __launch_bounds__(TA_THREADS) tr_arm_kernel(const __grid_constant__ TrainArmParams p) {
  // per latent, in shared memory for the weight-gradient outer products:
  //   layer k input z_k (C or NH) and output gradient du_k (NH, or 2 for the last)
  constexpr int NL = NHL + 1;  // linear layers
  using LY = TrArmLayout<C, NH, NHL>;
  constexpr int VEC = LY::VEC;
  extern __shared__ __align__(16) float tsm[];
  float* vec = tsm + threadIdx.x * VEC;
  const int64_t q = blockIdx.x * (int64_t)TA_THREADS + threadIdx.x;
  const bool valid = q < p.lv.n_lat;
  float bits = 0.0f;
  if (valid) {
    int l = 0;
    while (l + 1 < p.lv.L && q >= p.lv.off[l + 1]) l++;
    const int h = p.lv.h[l], w = p.lv.w[l];
    const int64_t t = q - p.lv.off[l];
    const int t32 = (int)t;  // a grid's plane is < 2^31: 32-bit division
    const int i = t32 / w, j = t32 - i * w;
    const float* g = p.yq + p.lv.off[l];
    float z[NL][NH > C ? NH : C];  // z[k] = input of layer k
    float u[NL][NH];               // pre-activations of the hidden layers
#pragma unroll
    for (int c = 0; c < C; c++) {
      const int ii = i + p.dy[c], jj = j + p.dx[c];
      z[0][c] = (ii >= 0 && ii < h && jj >= 0 && jj < w) ? g[(int64_t)ii * w + jj] : 0.0f;
    }
    // forward, FFMA2: two output neurons per instruction (c_tp pairs)
    int offp = BANK * TR_MAX_ARMP;
    float mu = 0.0f, s = 0.0f;
#pragma unroll
    for (int k = 0; k < NL; k++) {
      const int nin = (k == 0) ? C : NH, nout = (k == NL - 1) ? 2 : NH, n2 = nout / 2;
      const bool res = (p.res_mask >> k) & 1u;
      uint64_t acc[(NH > 2 ? NH : 2) / 2];
#pragma unroll
      for (int n = 0; n < n2; n++) acc[n] = ldp2(c_tp[offp + nin * n2 + n]);
#pragma unroll
      for (int t2 = 0; t2 < nin; t2++) {
        const uint64_t x = f2pack(z[k][t2], z[k][t2]);
#pragma unroll
        for (int n = 0; n < n2; n++) acc[n] = ffma2(x, ldp2(c_tp[offp + t2 * n2 + n]), acc[n]);
      }
#pragma unroll
      for (int n = 0; n < n2; n++) {
        float2 a = f2unpack(acc[n]);
        if (res) {
          a.x += z[k][2 * n];
          a.y += z[k][2 * n + 1];
        }
        if (k < NL - 1) {
          u[k][2 * n] = a.x;
          u[k][2 * n + 1] = a.y;
          z[k + 1][2 * n] = fmaxf(a.x, 0.0f);
          z[k + 1][2 * n + 1] = fmaxf(a.y, 0.0f);
        } else {
          mu = a.x;
          s = a.y;
        }
      }
      offp += nin * n2 + n2;
    }
    float gy, gmu, gs;
    bits = tr_bits(g[t], mu, s, p, gy, gmu, gs);
    p.gown[q] = p.w_r * gy;
    // backward
    float du[NH > 2 ? NH : 2];
    du[0] = p.w_r * gmu;
    du[1] = p.w_r * gs;
    // stash the layer inputs [z_k, 1, 0 pad] and output gradients du_k
#pragma unroll
    for (int k = 0; k < NL; k++) {
      const int nin = (k == 0) ? C : NH;
#pragma unroll
      for (int t2 = 0; t2 < LY::kin(k); t2++) vec[LY::zoff(k) + t2] = t2 < nin ? z[k][t2] : (t2 == nin ? 1.0f : 0.0f);
    }
    vec[LY::doff(NL - 1) + 0] = du[0];
    vec[LY::doff(NL - 1) + 1] = du[1];
    int offk[NL];
    {
      int o2 = BANK * TR_MAX_W;
#pragma unroll
      for (int k = 0; k < NL; k++) {
        const int nin = (k == 0) ? C : NH, nout = (k == NL - 1) ? 2 : NH;
        offk[k] = o2;
        o2 += nin * nout + nout;
      }
    }
#pragma unroll
    for (int k = NL - 1; k >= 0; k--) {
      const int nin = (k == 0) ? C : NH, nout = (k == NL - 1) ? 2 : NH;
      const bool res = (p.res_mask >> k) & 1u;
      // dz[2m, 2m+1] = sum_o du[o] (W[o][2m], W[o][2m+1]) (+ du if residual): FFMA2
      float dz[NH > C ? NH : C];
      uint64_t dzp[(NH > C ? NH : C) / 2];
#pragma unroll
      for (int m = 0; m < nin / 2; m++) dzp[m] = res ? f2pack(du[2 * m], du[2 * m + 1]) : 0ull;
#pragma unroll
      for (int o = 0; o < nout; o++) {
        const uint64_t d2 = f2pack(du[o], du[o]);
#pragma unroll
        for (int m = 0; m < nin / 2; m++)
          dzp[m] = ffma2(d2, ldp2(*reinterpret_cast<const float2*>(&c_tw[offk[k] + o * nin + 2 * m])), dzp[m]);
      }
#pragma unroll
      for (int m = 0; m < nin / 2; m++) {
        const float2 v = f2unpack(dzp[m]);
        dz[2 * m] = v.x;
        dz[2 * m + 1] = v.y;
      }
      if (k > 0) {
#pragma unroll
        for (int n = 0; n < NH; n++) {
          du[n] = u[k - 1][n] > 0.0f ? dz[n] : 0.0f;
          vec[LY::doff(k - 1) + n] = du[n];
        }
      } else {
#pragma unroll
        for (int c = 0; c < C; c++) p.dctx[c * p.lv.n_lat + q] = dz[c];
      }
    }
  } else {
    for (int v = 0; v < VEC; v++) vec[v] = 0.0f;
  }
  // rate: one fp64 partial per warp
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o2);
  if ((threadIdx.x & 31) == 0) p.rate[blockIdx.x * (TA_THREADS / 32) + (threadIdx.x >> 5)] = (double)bits;
  __syncthreads();
  // per-CTA weight gradients, layer by layer (tr_wgrad_tile)
  if constexpr (LY::wsum() <= TA_THREADS / 32) {
    // each layer's tiles on warps of their own (no divergence between layers
    // inside a warp; every SM sub-partition busy)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* wp = p.wpart + (int64_t)blockIdx.x * p.n_arm;
    auto run = [&](auto kc) {
      constexpr int k = decltype(kc)::value;
      if (warp >= LY::wstart(k) && warp < LY::wstart(k) + LY::nw(k)) {
        const int tile = (warp - LY::wstart(k)) * 32 + lane;
        if (tile < LY::ntile(k)) tr_wgrad_tile<C, NH, NHL, k>(tsm, tile, wp);
      }
    };
    run(std::integral_constant<int, 0>{});
    run(std::integral_constant<int, 1>{});
    if constexpr (NL > 2) run(std::integral_constant<int, 2>{});
    if constexpr (NL > 3) run(std::integral_constant<int, 3>{});
  } else {
    float* wp = p.wpart + (int64_t)blockIdx.x * p.n_arm;
    int tile = threadIdx.x;
    auto run = [&](auto kc) {
      constexpr int k = decltype(kc)::value;
      for (; tile < LY::ntile(k); tile += TA_THREADS) tr_wgrad_tile<C, NH, NHL, k>(tsm, tile, wp);
      tile -= LY::ntile(k);
    };
    run(std::integral_constant<int, 0>{});
    run(std::integral_constant<int, 1>{});
    if constexpr (NL > 2) run(std::integral_constant<int, 2>{});
    if constexpr (NL > 3) run(std::integral_constant<int, 3>{});
  }
}

// gradient of J wrt y_hat from the rate: own term + the context terms of the
// latents that use this one (gather: deterministic)
struct TrainCtx {
  int32_t C;
  int32_t dy[CC_MAX_CTX], dx[CC_MAX_CTX];
};
__global__ void tr_arm_gather_kernel(TrainLevels lv, const __grid_constant__ TrainCtx cx, const float* __restrict__ gown,
                                     const float* __restrict__ dctx, float* __restrict__ gy) {
  const int C = cx.C;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= lv.n_lat) return;
  int l = 0;
  while (l + 1 < lv.L && q >= lv.off[l + 1]) l++;
  const int h = lv.h[l], w = lv.w[l];
  const int64_t t = q - lv.off[l];
  const int t32 = (int)t;  // 32-bit division
  const int i = t32 / w, j = t32 - i * w;
  float g = gown[q];
  const float* dl = dctx + lv.off[l];
  for (int c = 0; c < C; c++) {
    const int pi = i - cx.dy[c], pj = j - cx.dx[c];  // latent whose context c is (i, j)
    // channel plane c at a 64-bit offset (C x N_lat may exceed 2^31); 32-bit
    // offsets only inside one grid (< P < 2^31 elements)
    if (pi >= 0 && pi < h && pj >= 0 && pj < w) g += (dl + (int64_t)c * lv.n_lat)[pi * w + pj];
  }
  gy[q] = g;
}

// ------------------------------------------------ 3 / 5. one upsampling step
// Along one axis of `lines` lines: out[o] = sum_t k[2t+1-r] g[clamp(q+r+K/4-1-t)],
// o = 2q + r < m (the gather form of the stride-2 transposed conv on the
// replicate-extended input, reading #12).
template <int KT>  // KT > 0: the tap count at compile time (unrolled)
__global__ void tr_tconv_fwd_kernel(const float* __restrict__ g, float* __restrict__ out, int lines, int n, int m,
                                    int64_t g_ls, int64_t g_es, int64_t o_ls, int64_t o_es, int K_, int koff,
                                    int64_t g_cs, int64_t o_cs) {
  const int K = KT > 0 ? KT : K_;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)lines * m) return;
  g += blockIdx.y * g_cs;  // channel
  out += blockIdx.y * o_cs;
  // consecutive threads on consecutive addresses: along the line when its
  // elements are contiguous (x pass), across lines otherwise (y pass: columns)
  // 32-bit index math (a 64-bit division is a ~100-instruction call; the
  // planes here are < 2^31 elements)
  const int i32 = (int)idx;
  int line, o;
  if (g_es == 1) {
    line = i32 / m;
    o = i32 - line * m;
  } else {
    o = i32 / lines;
    line = i32 - o * lines;
  }
  const int q = o >> 1, r = o & 1;
  // 32-bit offsets within the channel plane (< 2^31 elements)
  const int gl = line * (int)g_ls, ge = (int)g_es;
  float acc = 0.0f;
#pragma unroll
  for (int t = 0; t < (KT > 0 ? KT / 2 : 4); t++) {
    if (KT == 0 && t >= K / 2) break;
    acc = fmaf(c_tw[koff + 2 * t + 1 - r], g[gl + clampi(q + r + K / 4 - 1 - t, 0, n - 1) * ge], acc);
  }
  out[line * (int)o_ls + o * (int)o_es] = acc;
}

// Adjoint: gg[s] = sum over extended positions i with clamp(i - E) = s of
// sum_j k[j] gout[2i + j - P]; tap gradient dk[j] = sum x_ext[i] gout[2i + j - P]
// (per-block partials [blocks][K]).
// KT > 0: the tap count as a compile-time constant (unrolled loops, the tap
// gradients in registers; with a runtime K they lived in local memory)
template <int KT>
__global__ void tr_tconv_bwd_kernel(const float* __restrict__ g, const float* __restrict__ gout, float* __restrict__ gg,
                                    int lines, int n, int m, int64_t g_ls, int64_t g_es, int64_t o_ls, int64_t o_es,
                                    int K_, int koff, float* __restrict__ kpart, int64_t g_cs, int64_t o_cs) {
  const int K = KT > 0 ? KT : K_;
  __shared__ float red[8][TB / 32];
  g += blockIdx.y * g_cs;  // channel (gg shares g's layout)
  gg += blockIdx.y * g_cs;
  gout += blockIdx.y * o_cs;
  kpart += (int64_t)blockIdx.y * gridDim.x * K;
  float dk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)lines * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int line, s;  // coalesced mapping (see tr_tconv_fwd_kernel); 32-bit index math
    const int i32 = (int)idx;
    if (g_es == 1) {
      line = i32 / n;
      s = i32 - line * n;
    } else {
      s = i32 / lines;
      line = i32 - s * lines;
    }
    const int E = K / 4, P = K / 2 - 1 + 2 * E;
    const float xs = g[line * (int)g_ls + s * (int)g_es];  // 32-bit plane offsets
    const int i_lo = (s == 0) ? 0 : s + E, i_hi = (s == n - 1) ? n - 1 + 2 * E : s + E;  // extended positions
    float acc = 0.0f;
    for (int i = i_lo; i <= i_hi; i++)
#pragma unroll
      for (int j = 0; j < (KT > 0 ? KT : 8); j++) {
        if (KT == 0 && j >= K) break;
        const int o = 2 * i + j - P;
        if (o >= 0 && o < m) {
          const float go = gout[line * (int)o_ls + o * (int)o_es];
          acc = fmaf(c_tw[koff + j], go, acc);
          dk[j] = fmaf(xs, go, dk[j]);
        }
      }
    gg[line * (int)g_ls + s * (int)g_es] = acc;
  }
  // block partial of the tap gradient
#pragma unroll
  for (int j = 0; j < (KT > 0 ? KT : 8); j++) {
    if (KT == 0 && j >= K) break;
    float v = dk[j];
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o2);
    if ((threadIdx.x & 31) == 0) red[j][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    float v = 0.0f;
    for (int w2 = 0; w2 < TB / 32; w2++) v += red[threadIdx.x][w2];
    kpart[(int64_t)blockIdx.x * K + threadIdx.x] = v;
  }
}

// ------------------------------------------------------------ 4. synthesis
struct TrainSynDims {
  int32_t H, W, L, CH, R;
  int64_t P;
  int32_t oA0, oa0, oA1, oa1, oG;  // offsets of the synthesis blocks in c_tw
  int32_t bank;                    // constant bank of this step
};

// 1x1 layers: u1 = A0 v + a0 (kept), h = A1 ReLU(u1) + a1 (pre kept), ReLU if R > 0
template <int L, int CH, int BANK>
__global__ void tr_syn1x1_fwd_kernel(TrainSynDims d, const float* __restrict__ dense, float* __restrict__ u1,
                                     float* __restrict__ us0, float* __restrict__ hs0) {
  constexpr int oA0 = BANK * TR_MAX_W + TR_SYN_OFF, oa0 = oA0 + L * CH, oA1 = oa0 + CH, oa1 = oA1 + 3 * CH;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= d.P) return;
  float v[L], o[3];
#pragma unroll
  for (int i = 0; i < L; i++) v[i] = dense[(int64_t)i * d.P + p];
#pragma unroll
  for (int c = 0; c < 3; c++) o[c] = c_tw[oa1 + c];
#pragma unroll 4
  for (int n = 0; n < CH; n++) {
    float a = c_tw[oa0 + n];
#pragma unroll
    for (int i = 0; i < L; i++) a = fmaf(c_tw[oA0 + n * L + i], v[i], a);
    if (u1 != nullptr) u1[(int64_t)n * d.P + p] = a;  // (the adjoint recomputes it: 160 B/px not stored)
    const float r = fmaxf(a, 0.0f);
#pragma unroll
    for (int c = 0; c < 3; c++) o[c] = fmaf(c_tw[oA1 + c * CH + n], r, o[c]);
  }
  for (int c = 0; c < 3; c++) {
    us0[c * d.P + p] = o[c];
    hs0[c * d.P + p] = d.R > 0 ? fmaxf(o[c], 0.0f) : o[c];
  }
}

// residual 3x3 layer r: us = hin + g + G * hin (replicate padding), hout = ReLU unless last
__global__ void tr_conv_fwd_kernel(TrainSynDims d, int r, const float* __restrict__ hin, float* __restrict__ us,
                                   float* __restrict__ hout) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= d.P) return;
  const int p32 = (int)p;  // 32-bit division (P < 2^31)
  const int y = p32 / d.W, x = p32 - y * d.W;
  const int oG = d.oG + 84 * r;
  // the 27 window values once (each feeds 3 outputs); channel planes at 64-bit
  // offsets (3 P may exceed 2^31), 32-bit offsets inside a plane (P < 2^31)
  const float* hc[3] = {hin, hin + d.P, hin + 2 * d.P};
  float* uc[3] = {us, us + d.P, us + 2 * d.P};
  float* oc[3] = {hout, hout + d.P, hout + 2 * d.P};
  int ro[3], cx[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    ro[k] = clampi(y + k - 1, 0, d.H - 1) * d.W;
    cx[k] = clampi(x + k - 1, 0, d.W - 1);
  }
  float v[3][3][3];
#pragma unroll
  for (int ci = 0; ci < 3; ci++)
#pragma unroll
    for (int ky = 0; ky < 3; ky++)
#pragma unroll
      for (int kx = 0; kx < 3; kx++) v[ci][ky][kx] = hc[ci][ro[ky] + cx[kx]];
#pragma unroll
  for (int co = 0; co < 3; co++) {
    float a = v[co][1][1] + c_tw[oG + 81 + co];  // residual (the centre tap is the pixel itself)
#pragma unroll
    for (int ci = 0; ci < 3; ci++)
#pragma unroll
      for (int ky = 0; ky < 3; ky++)
#pragma unroll
        for (int kx = 0; kx < 3; kx++) a = fmaf(c_tw[oG + ((co * 3 + ci) * 3 + ky) * 3 + kx], v[ci][ky][kx], a);
    uc[co][p32] = a;
    oc[co][p32] = (r < d.R - 1) ? fmaxf(a, 0.0f) : a;
  }
}

// distortion: dJ/dx_hat = -2 (x - x_hat) / (3 P); SSE per block (fp64)
__global__ void tr_loss_kernel(TrainSynDims d, const float* __restrict__ xh, const float* __restrict__ img,
                               float* __restrict__ gh, double* __restrict__ sse_part) {
  __shared__ double red[TB / 32];
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float e2 = 0.0f;
  if (t < 3 * d.P) {
    const float e = img[t] - xh[t];
    gh[t] = -2.0f * e / (3.0f * (float)d.P);
    e2 = e * e;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, o2);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = (double)e2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < TB / 32; w++) s += red[w];
    sse_part[blockIdx.x] = s;
  }
}

// adjoint of residual layer r: gpre = gh (x) ReLU'(us) (not on the last layer);
// gin = gpre (residual) + G^T-gather over the clamped neighbourhood;
// dG[co][ci][ky][kx] = sum gpre[co](p) hin[ci](clamp(p + tap)), dg[co] = sum gpre[co].
// Tiles of CT_Y x CT_X pixels (one per thread) with a 1-pixel halo of gpre and
// hin staged in shared memory; persistent CTAs accumulate dG in registers over
// their tiles and reduce once.
constexpr int CT_Y = 8, CT_X = 32;
// 4-byte global -> shared copy; src_bytes = 0 writes a zero (no read)
__device__ __forceinline__ void cp_async4(float* dst, const float* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__global__ void __launch_bounds__(CT_Y * CT_X)
    tr_conv_bwd_kernel(TrainSynDims d, int r, const float* __restrict__ hin, const float* __restrict__ us,
                       const float* __restrict__ gh, float* __restrict__ gin, float* __restrict__ gpart) {
  constexpr int SY = CT_Y + 2, SX = CT_X + 2, SN = 3 * SY * SX, NT = CT_Y * CT_X;
  // the persistent CTA's tiles are double-buffered: the raw gh / us / hin
  // windows of tile n+1 stream in (cp.async) while tile n computes
  __shared__ float rg[2][SN], ru[2][SN], rh[2][SN];
  __shared__ float sg[3][SY][SX];
  __shared__ float red[84][NT / 32];
  const int oG = d.oG + 84 * r;
  const bool relu = r < d.R - 1;
  const int tiles_x = (d.W + CT_X - 1) / CT_X, n_tiles = tiles_x * ((d.H + CT_Y - 1) / CT_Y);
  const int ty = threadIdx.x / CT_X, tx = threadIdx.x - ty * CT_X;
  auto issue = [&](int tile, int buf) {
    const int Y0 = (tile / tiles_x) * CT_Y, X0 = (tile % tiles_x) * CT_X;
    for (int k = threadIdx.x; k < SN; k += NT) {
      const int c = k / (SY * SX), rem = k - c * (SY * SX), yy = rem / SX, xx = rem - yy * SX;
      const int y = Y0 + yy - 1, x = X0 + xx - 1;
      const bool in = y >= 0 && y < d.H && x >= 0 && x < d.W;  // gpre exists only in the image
      const int64_t q = c * d.P + (int64_t)clampi(y, 0, d.H - 1) * d.W + clampi(x, 0, d.W - 1);
      cp_async4(&rg[buf][k], gh + q, in ? 4 : 0);
      if (relu) cp_async4(&ru[buf][k], us + q, in ? 4 : 0);
      cp_async4(&rh[buf][k], hin + q, 4);  // replicate padding
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float dG[84];
#pragma unroll
  for (int e = 0; e < 84; e++) dG[e] = 0.0f;
  int buf = 0;
  if ((int)blockIdx.x < n_tiles) issue(blockIdx.x, 0);
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, buf ^= 1) {
    const int Y0 = (tile / tiles_x) * CT_Y, X0 = (tile % tiles_x) * CT_X;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // this tile's window landed; the previous tile's readers are done
    if (tile + (int)gridDim.x < n_tiles) issue(tile + gridDim.x, buf ^ 1);
    for (int k = threadIdx.x; k < SN; k += NT) {
      float g = rg[buf][k];
      if (relu && !(ru[buf][k] > 0.0f)) g = 0.0f;
      (&sg[0][0][0])[k] = g;
    }
    __syncthreads();
    const float* sh = rh[buf];
#define SH(ci, yy, xx) sh[((ci) * SY + (yy)) * SX + (xx)]
    const int y = Y0 + ty, x = X0 + tx;
    if (y < d.H && x < d.W) {
      float gp[3];
#pragma unroll
      for (int co = 0; co < 3; co++) gp[co] = sg[co][ty + 1][tx + 1];
#pragma unroll
      for (int co = 0; co < 3; co++) {
        dG[81 + co] += gp[co];
#pragma unroll
        for (int ci = 0; ci < 3; ci++)
#pragma unroll
          for (int ky = 0; ky < 3; ky++)
#pragma unroll
            for (int kx = 0; kx < 3; kx++)
              dG[((co * 3 + ci) * 3 + ky) * 3 + kx] =
                  fmaf(gp[co], SH(ci, ty + ky, tx + kx), dG[((co * 3 + ci) * 3 + ky) * 3 + kx]);
      }
#undef SH
      const bool interior = y >= 1 && y <= d.H - 2 && x >= 1 && x <= d.W - 2;
#pragma unroll
      for (int ci = 0; ci < 3; ci++) {
        float a = gp[ci];  // residual
        if (interior) {
#pragma unroll
          for (int ky = 0; ky < 3; ky++)
#pragma unroll
            for (int kx = 0; kx < 3; kx++)
#pragma unroll
              for (int co = 0; co < 3; co++)
                a = fmaf(c_tw[oG + ((co * 3 + ci) * 3 + ky) * 3 + kx], sg[co][ty + 2 - ky][tx + 2 - kx], a);
        } else {  // every output q in the neighbourhood and tap whose clamped source is p
          for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++) {
              const int qy = y + dy, qx = x + dx;
              if (qy < 0 || qy >= d.H || qx < 0 || qx >= d.W) continue;
              for (int ky = 0; ky < 3; ky++)
                for (int kx = 0; kx < 3; kx++)
                  if (clampi(qy + ky - 1, 0, d.H - 1) == y && clampi(qx + kx - 1, 0, d.W - 1) == x)
                    for (int co = 0; co < 3; co++)
                      a = fmaf(c_tw[oG + ((co * 3 + ci) * 3 + ky) * 3 + kx], sg[co][ty + 1 + dy][tx + 1 + dx], a);
            }
        }
        gin[ci * d.P + (int64_t)y * d.W + x] = a;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 84; e++) {
    float v = dG[e];
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o2);
    if ((threadIdx.x & 31) == 0) red[e][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 84; e += CT_Y * CT_X) {
    float v = 0.0f;
    for (int w2 = 0; w2 < CT_Y * CT_X / 32; w2++) v += red[e][w2];
    gpart[(int64_t)blockIdx.x * 84 + e] = v;
  }
}

// adjoint of the 1x1 layers per pixel, dense gradient, per-CTA weight-gradient
// partials: register-tiled (4 x 4) outer products over the CTA's pixels, work
// items = (tile, 32-pixel chunk), chunk partials summed in a fixed order
template <int L, int CH>
struct TrSyn1x1Layout {
  __host__ __device__ static constexpr int r4(int x) { return (x + 3) / 4 * 4; }
  static constexpr int D2 = 0;                   // [d2 (3), 0]
  static constexpr int V1 = 4;                   // [relu(u1) (CH), 1, 0 ...]
  static constexpr int D1 = V1 + r4(CH + 1);     // d1 (CH)
  static constexpr int DN = D1 + r4(CH);         // [dense (L), 1, 0 ...]
  static constexpr int RAW = DN + r4(L + 1);
  static constexpr int VEC = RAW + ((RAW / 4) % 2 == 0 ? 4 : 0);  // odd count of 16-byte words
  static constexpr int T0 = (CH / 4) * (r4(L + 1) / 4);          // dA0 | da0 tiles
  static constexpr int T1 = r4(CH + 1) / 4;                      // dA1 | da1 tiles (rows: d2)
  static constexpr int NW = L * CH + CH + 3 * CH + 3;
  static_assert(CH % 4 == 0, "hidden width multiple of 4");
};

template <int L, int CH, int BANK>
__global__ void __launch_bounds__(TS_THREADS)
    tr_syn1x1_bwd_kernel(TrainSynDims d, const float* __restrict__ dense, const float* __restrict__ u1,
                         const float* __restrict__ us0, const float* __restrict__ gh, float* __restrict__ gdense,
                         float* __restrict__ wpart, int n_w) {
  constexpr int oA0 = BANK * TR_MAX_W + TR_SYN_OFF, oa0 = oA0 + L * CH, oA1 = oa0 + CH, oa1 = oA1 + 3 * CH;
  using LY = TrSyn1x1Layout<L, CH>;
  constexpr int VEC = LY::VEC;
  extern __shared__ __align__(16) float ssm[];
  float* vec = ssm + threadIdx.x * VEC;
  const int64_t p = blockIdx.x * (int64_t)TS_THREADS + threadIdx.x;
  for (int v = 0; v < VEC; v++) vec[v] = 0.0f;
  if (p < d.P) {
    float d2[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      float g = gh[c * d.P + p];
      if (d.R > 0 && !(us0[c * d.P + p] > 0.0f)) g = 0.0f;
      d2[c] = g;
      vec[LY::D2 + c] = g;
    }
#pragma unroll
    for (int i = 0; i < L; i++) vec[LY::DN + i] = dense[(int64_t)i * d.P + p];
    vec[LY::DN + L] = 1.0f;
    vec[LY::V1 + CH] = 1.0f;
    float gd[L];
#pragma unroll
    for (int i = 0; i < L; i++) gd[i] = 0.0f;
    // the CH pre-activations recomputed from the dense input in the forward's
    // exact order (bias, then inputs 0 .. L-1): bit-identical, and 160 B/px of
    // HBM traffic each way saved against storing them
    float ua[CH];
    {
      float v[L];
#pragma unroll
      for (int i = 0; i < L; i++) v[i] = dense[(int64_t)i * d.P + p];
#pragma unroll
      for (int n = 0; n < CH; n++) {
        float a = c_tw[oa0 + n];
#pragma unroll
        for (int i = 0; i < L; i++) a = fmaf(c_tw[oA0 + n * L + i], v[i], a);
        ua[n] = a;
      }
    }
#pragma unroll
    for (int n = 0; n < CH; n++) {
      const float a = ua[n];
      vec[LY::V1 + n] = fmaxf(a, 0.0f);
      float g = 0.0f;
#pragma unroll
      for (int c = 0; c < 3; c++) g = fmaf(c_tw[oA1 + c * CH + n], d2[c], g);
      g = a > 0.0f ? g : 0.0f;
      vec[LY::D1 + n] = g;
#pragma unroll
      for (int i = 0; i < L; i++) gd[i] = fmaf(c_tw[oA0 + n * L + i], g, gd[i]);
    }
#pragma unroll
    for (int i = 0; i < L; i++) gdense[(int64_t)i * d.P + p] = gd[i];
  }
  __syncthreads();
  // Weight gradients over the CTA's pixels as two small split-K products,
  // G0 = D1^T [CH x P] . [dense, 1] [P x NC0] (dA0 | da0) and
  // G1 = D2^T [4 x P] . [relu(u1), 1] [P x 8 T1] (dA1 | da1): warps 0-1 take
  // G0's 8 x NC0 tiles, warps 2-3 G1's 4 x 8 tiles, each over one K-chunk of
  // pixels, FFMA2 over column pairs with the row value a register broadcast
  // (16 floats read per 64 MACs: the 4 x 4 tiles read 8 per 16 and were
  // shared-memory bound); chunk partials then go through shared memory (over
  // the records) and are summed in a fixed order (deterministic).
  constexpr int NC0 = LY::r4(L + 1);                        // G0 columns (dense + bias, padded)
  constexpr int T0n = CH / 8, T1n = (LY::r4(CH + 1) + 7) / 8;  // tiles
  constexpr int K0 = (64 / T0n) < 32 ? (64 / T0n) : 32, K1 = (64 / T1n) < 32 ? (64 / T1n) : 32;  // K-chunks
  constexpr int PX0 = (TS_THREADS + K0 - 1) / K0, PX1 = (TS_THREADS + K1 - 1) / K1;  // pixels per chunk
  constexpr int G0F = CH * NC0, G1W = 8 * T1n, G1F = 4 * G1W;   // floats per chunk partial
  static_assert(CH % 8 == 0 && (NC0 == 4 || NC0 == 8), "tile shapes");
  static_assert(K0 * G0F + K1 * G1F <= TS_THREADS * VEC, "partials fit over the records");
  const int t = threadIdx.x;
  uint64_t acc0[8][NC0 / 2];
  uint64_t acc1[4][4];
  int tile = -1, kc = 0;
  if (t < 64) {
    if (t < T0n * K0) {
      tile = t / K0;
      kc = t - tile * K0;
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int c = 0; c < NC0 / 2; c++) acc0[r][c] = 0ull;
      const int m1 = (kc + 1) * PX0 < TS_THREADS ? (kc + 1) * PX0 : TS_THREADS;
      for (int m = kc * PX0; m < m1; m++) {
        const float* v = ssm + m * VEC;
        const float4 d0 = *reinterpret_cast<const float4*>(v + LY::D1 + 8 * tile);
        const float4 d1 = *reinterpret_cast<const float4*>(v + LY::D1 + 8 * tile + 4);
        const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        uint64_t z[NC0 / 2];
#pragma unroll
        for (int c4 = 0; c4 < NC0 / 4; c4++) {
          const ulonglong2 zz = *reinterpret_cast<const ulonglong2*>(v + LY::DN + 4 * c4);
          z[2 * c4] = zz.x;
          z[2 * c4 + 1] = zz.y;
        }
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint64_t d2 = f2pack(dv[r], dv[r]);
#pragma unroll
          for (int c = 0; c < NC0 / 2; c++) acc0[r][c] = ffma2(d2, z[c], acc0[r][c]);
        }
      }
    }
  } else {
    const int u = t - 64;
    if (u < T1n * K1) {
      tile = u / K1;
      kc = u - tile * K1;
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc1[r][c] = 0ull;
      const int m1 = (kc + 1) * PX1 < TS_THREADS ? (kc + 1) * PX1 : TS_THREADS;
      for (int m = kc * PX1; m < m1; m++) {
        const float* v = ssm + m * VEC;
        const float4 dd = *reinterpret_cast<const float4*>(v + LY::D2);
        const float dv[4] = {dd.x, dd.y, dd.z, dd.w};
        const ulonglong2 za = *reinterpret_cast<const ulonglong2*>(v + LY::V1 + 8 * tile);
        const ulonglong2 zb = *reinterpret_cast<const ulonglong2*>(v + LY::V1 + 8 * tile + 4);
        const uint64_t z[4] = {za.x, za.y, zb.x, zb.y};
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const uint64_t d2 = f2pack(dv[r], dv[r]);
#pragma unroll
          for (int c = 0; c < 4; c++) acc1[r][c] = ffma2(d2, z[c], acc1[r][c]);
        }
      }
    }
  }
  __syncthreads();  // every record read: the partials go over them
  float* P0 = ssm;              // [K0][CH][NC0]
  float* P1 = ssm + K0 * G0F;   // [K1][4][G1W]
  if (tile >= 0) {
    if (t < 64) {
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int c = 0; c < NC0 / 2; c++) {
          const float2 x = f2unpack(acc0[r][c]);
          *reinterpret_cast<float2*>(P0 + kc * G0F + (8 * tile + r) * NC0 + 2 * c) = x;
        }
    } else {
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const float2 x = f2unpack(acc1[r][c]);
          *reinterpret_cast<float2*>(P1 + kc * G1F + r * G1W + 8 * tile + 2 * c) = x;
        }
    }
  }
  __syncthreads();
  for (int e = t; e < n_w; e += TS_THREADS) {
    const float* src;
    int stride, nk;
    if (e < CH * L) {  // A0[n][i]
      const int n = e / L, i = e - n * L;
      src = P0 + n * NC0 + i, stride = G0F, nk = K0;
    } else if (e < CH * L + CH) {  // a0[n]: the bias column
      src = P0 + (e - CH * L) * NC0 + L, stride = G0F, nk = K0;
    } else if (e < CH * L + CH + 3 * CH) {  // A1[c][n]
      const int q = e - CH * L - CH, c = q / CH, n = q - c * CH;
      src = P1 + c * G1W + n, stride = G1F, nk = K1;
    } else {  // a1[c]: the bias column
      src = P1 + (e - CH * L - CH - 3 * CH) * G1W + CH, stride = G1F, nk = K1;
    }
    float v = 0.0f;
    for (int k = 0; k < nk; k++) v += src[k * stride];
    wpart[(int64_t)blockIdx.x * n_w + e] = v;
  }
}

// ------------------------------------------------------------ 6. reduction
// Two-stage fp64 reduction of partial rows part[b * stride + e], b < blocks,
// e < n: stage 1 sums row chunks (blockIdx.y) with one thread per entry
// (coalesced across the warp), stage 2 sums the chunks into grad[e].
constexpr int TR_RCHUNK = 128;
__global__ void tr_reduce1_kernel(const float* __restrict__ part, int64_t blocks, int64_t stride, int n,
                                  double* __restrict__ tmp) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t per = (blocks + gridDim.y - 1) / gridDim.y;
  const int64_t b0 = blockIdx.y * per, b1 = b0 + per < blocks ? b0 + per : blocks;
  double s = 0.0;
#pragma unroll 4
  for (int64_t b = b0; b < b1; b++) s += (double)part[b * stride + e];
  tmp[(int64_t)blockIdx.y * n + e] = s;
}
// Narrow partial rows (n <= 128): the block's threads are (row slot, element)
// pairs striding over the chunk's rows (n_pad = next power of two >= n), then a
// fixed-order tree over the row slots -- all threads busy instead of n of them
// walking every row serially (deterministic: fixed assignment and order).
__global__ void __launch_bounds__(256) tr_reduce1_narrow_kernel(const float* __restrict__ part, int64_t blocks,
                                                                int64_t stride, int n, int n_pad,
                                                                double* __restrict__ tmp) {
  __shared__ double red[256];
  const int e = threadIdx.x & (n_pad - 1), slot = threadIdx.x / n_pad, slots = 256 / n_pad;
  const int64_t per = (blocks + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < blocks ? b0 + per : blocks;
  double s = 0.0;
  if (e < n) {
#pragma unroll 4
    for (int64_t b = b0 + slot; b < b1; b += slots) s += (double)part[b * stride + e];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int half = slots / 2; half > 0; half >>= 1) {
    if (slot < half) red[threadIdx.x] += red[threadIdx.x + half * n_pad];
    __syncthreads();
  }
  if (slot == 0 && e < n) tmp[(int64_t)blockIdx.x * n + e] = red[threadIdx.x];
}
// one warp per element: lanes stride over the chunks, fixed-order shuffle tree
__global__ void tr_reduce2_kernel(const double* __restrict__ tmp, int chunks, int n, float* __restrict__ grad) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (e >= n) return;
  double s = 0.0;
  for (int c = lane; c < chunks; c += 32) s += tmp[(int64_t)c * n + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) grad[e] = (float)s;
}

constexpr int TR_RES_THREADS = 1024;  // one CTA: short serial chains per thread
__global__ void __launch_bounds__(TR_RES_THREADS) tr_result_kernel(const double* __restrict__ rate_part, int64_t n_rate,
                                                                  const double* __restrict__ sse_part, int64_t n_sse,
                                                                  double inv_3p, double lambda_over_p,
                                                                  cc_rd_result* out) {
  __shared__ double ra[TR_RES_THREADS], sa[TR_RES_THREADS];
  double r = 0.0, s = 0.0;
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < n_rate; i += TR_RES_THREADS) r += rate_part[i];
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < n_sse; i += TR_RES_THREADS) s += sse_part[i];
  ra[threadIdx.x] = r;
  sa[threadIdx.x] = s;
  __syncthreads();
  for (int o = TR_RES_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      ra[threadIdx.x] += ra[threadIdx.x + o];
      sa[threadIdx.x] += sa[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cc_rd_result res;
    res.rate_bits = ra[0];
    res.sse = sa[0];
    res.mse = sa[0] * inv_3p;
    res.cost = res.mse + lambda_over_p * ra[0];
    *out = res;
  }
}

// Adam (Kingma & Ba): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// p -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
__global__ void tr_adam_kernel(float* __restrict__ par, const float* __restrict__ g, float* __restrict__ m,
                               float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float c1,
                               float c2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.0f - b1) * gi;
    const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    par[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}

// ============================================================== host side
struct TrainPlan {
  TrainLevels lv;
  int64_t n_arm, n_up, n_syn, n_par;
  // workspace offsets (bytes)
  size_t o_yq, o_gown, o_dctx, o_rate, o_wpart_arm, o_chain, o_dense, o_u1, o_us, o_hs, o_gh0, o_gh1, o_gdense,
      o_g0, o_g1, o_kpart, o_cpart, o_spart, o_sse, o_grad_tmp, total;
  int64_t arm_ctas, p_blocks, s_blocks, kpart_rows;
  std::vector<int64_t> chain_off;  // per (l, j): output of step j for grid l; mid after the x pass
  std::vector<int64_t> mid_off;
};

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

static void make_plan(const cc_model_desc& d, TrainPlan& pl) {
  TrainLevels& lv = pl.lv;
  memset(&lv, 0, sizeof(lv));
  lv.L = d.L;
  lv.H = d.H;
  lv.W = d.W;
  int64_t off = 0;
  for (int l = 0; l < d.L; l++) {
    lv.h[l] = (int32_t)((d.H + (1 << l) - 1) >> l);
    lv.w[l] = (int32_t)((d.W + (1 << l) - 1) >> l);
    lv.off[l] = off;
    off += (int64_t)lv.h[l] * lv.w[l];
  }
  lv.n_lat = off;
  pl.n_arm = 0;
  for (int k = 0; k < d.arm_n_layers; k++) pl.n_arm += (int64_t)d.arm_widths[k] * d.arm_widths[k + 1] + d.arm_widths[k + 1];
  pl.n_up = d.up_taps;
  const int CH = d.syn_widths[1];
  pl.n_syn = (int64_t)d.L * CH + CH + 3 * CH + 3 + 84 * (int64_t)d.syn_n_res;
  pl.n_par = lv.n_lat + pl.n_arm + pl.n_up + pl.n_syn;
  const int64_t P = (int64_t)d.H * d.W;
  pl.arm_ctas = (lv.n_lat + TA_THREADS - 1) / TA_THREADS;
  pl.p_blocks = (P + TB - 1) / TB < TR_GRID_CAP ? (P + TB - 1) / TB : TR_GRID_CAP;  // grid-stride conv adjoint
  pl.s_blocks = (P + TS_THREADS - 1) / TS_THREADS;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += a256(bytes);
    return r;
  };
  pl.o_yq = take(4 * lv.n_lat);
  pl.o_gown = take(4 * lv.n_lat);
  pl.o_dctx = take(4 * lv.n_lat * d.n_ctx);
  pl.o_rate = take(8 * pl.arm_ctas * (TA_THREADS / 32));
  pl.o_wpart_arm = take(4 * pl.arm_ctas * pl.n_arm);
  // upsampling stacks T_j = [y_hat_j, S_j] (L - j channels at level j; T_0 is
  // the dense tensor) and the x-pass intermediates mid_j ((L-1-j) channels of
  // h_{j+1} x w_j), offsets in floats; tap-gradient partial rows per adjoint
  pl.chain_off.assign(CC_MAX_LEVELS * CC_MAX_LEVELS, -1);
  pl.mid_off.assign(CC_MAX_LEVELS * CC_MAX_LEVELS, -1);
  int64_t c = 0, kp = 0;
  for (int j = 1; j < d.L; j++) {  // T_0 lives in the dense buffer
    pl.chain_off[j] = c;
    c += (int64_t)(d.L - j) * lv.h[j] * lv.w[j];
  }
  for (int j = 0; j + 1 < d.L; j++) {
    const int nch = d.L - 1 - j;
    pl.mid_off[j] = c;
    c += (int64_t)nch * lv.h[j + 1] * lv.w[j];
    auto capb = [](int64_t n) { const int64_t b = (n + TB - 1) / TB; return b < TR_TCONV_CAP ? b : (int64_t)TR_TCONV_CAP; };
    kp += (int64_t)nch * (capb((int64_t)lv.h[j + 1] * lv.w[j]) + capb((int64_t)lv.h[j + 1] * lv.w[j + 1]));
  }
  pl.kpart_rows = kp > 0 ? kp : 1;
  pl.o_chain = take(4 * (c > 0 ? c : 1));
  pl.o_dense = take(4 * (size_t)d.L * P);
  pl.o_u1 = take(0);  // hidden pre-activations: recomputed by the 1x1 adjoint, not stored
  pl.o_us = take(4 * (size_t)(d.syn_n_res + 1) * 3 * P);
  pl.o_hs = take(4 * (size_t)(d.syn_n_res + 1) * 3 * P);
  pl.o_gh0 = take(4 * 3 * (size_t)P);
  pl.o_gh1 = take(4 * 3 * (size_t)P);
  pl.o_gdense = take(4 * (size_t)d.L * P);
  pl.o_g0 = take(4 * (size_t)d.L * P);  // gradient stacks gT_j (ping)
  pl.o_g1 = take(4 * (size_t)d.L * P);  // gmid / gT_j (pong)
  pl.o_kpart = take(4 * (size_t)pl.kpart_rows * d.up_taps);
  pl.o_cpart = take(4 * (size_t)(d.syn_n_res > 0 ? d.syn_n_res : 1) * pl.p_blocks * 84);
  pl.o_spart = take(4 * (size_t)pl.s_blocks * (d.L * CH + CH + 3 * CH + 3));
  pl.o_sse = take(8 * (size_t)((3 * P + TB - 1) / TB));
  pl.o_grad_tmp = take(8 * (size_t)TR_RCHUNK * TR_MAX_W);  // stage-1 reduction chunks (fp64)
  pl.total = o;
}

int64_t train_param_count(const cc_model_desc& d) {
  TrainPlan pl;
  make_plan(d, pl);
  return pl.n_par;
}
size_t train_workspace_bytes(const cc_model_desc& d) {
  TrainPlan pl;
  make_plan(d, pl);
  return pl.total;
}

typedef void (*TrArmFn)(dim3, int, size_t, cudaStream_t, const TrainArmParams&);
template <int C, int NH, int NHL>
static void tr_arm_launch(dim3 g, int t, size_t smem, cudaStream_t s, const TrainArmParams& p) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tr_arm_kernel<C, NH, NHL, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(tr_arm_kernel<C, NH, NHL, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(tr_arm_kernel<C, NH, NHL, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(tr_arm_kernel<C, NH, NHL, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  static_assert(TR_BANKS == 4, "one instantiation per bank");
  switch (p.tp0 / TR_MAX_ARMP) {
    case 0: tr_arm_kernel<C, NH, NHL, 0><<<g, t, smem, s>>>(p); break;
    case 1: tr_arm_kernel<C, NH, NHL, 1><<<g, t, smem, s>>>(p); break;
    case 2: tr_arm_kernel<C, NH, NHL, 2><<<g, t, smem, s>>>(p); break;
    default: tr_arm_kernel<C, NH, NHL, 3><<<g, t, smem, s>>>(p); break;
  }
}
struct TrArmEntry {
  int C, NH, NHL;
  TrArmFn fn;
  int vec;  // floats per latent record in shared memory
};
#define TR_ARM(C, NH, NHL) {C, NH, NHL, tr_arm_launch<C, NH, NHL>, TrArmLayout<C, NH, NHL>::VEC}
static const TrArmEntry kTrArm[] = {
    TR_ARM(16, 24, 2), TR_ARM(8, 8, 2), TR_ARM(8, 8, 1), TR_ARM(16, 16, 2), TR_ARM(24, 24, 2),
};

typedef void (*TrSynFwdFn)(int, int, cudaStream_t, const TrainSynDims&, const float*, float*, float*, float*);
typedef void (*TrSynBwdFn)(int, int, size_t, cudaStream_t, const TrainSynDims&, const float*, const float*,
                           const float*, const float*, float*, float*, int);
template <int L, int CH>
static void tr_syn_fwd_launch(int g, int t, cudaStream_t s, const TrainSynDims& d, const float* dense, float* u1,
                              float* us0, float* hs0) {
  switch (d.bank) {  // one instantiation per constant bank (compile-time weight addresses)
    case 0: tr_syn1x1_fwd_kernel<L, CH, 0><<<g, t, 0, s>>>(d, dense, u1, us0, hs0); break;
    case 1: tr_syn1x1_fwd_kernel<L, CH, 1><<<g, t, 0, s>>>(d, dense, u1, us0, hs0); break;
    case 2: tr_syn1x1_fwd_kernel<L, CH, 2><<<g, t, 0, s>>>(d, dense, u1, us0, hs0); break;
    default: tr_syn1x1_fwd_kernel<L, CH, 3><<<g, t, 0, s>>>(d, dense, u1, us0, hs0); break;
  }
}
template <int L, int CH>
static void tr_syn_bwd_launch(int g, int t, size_t smem, cudaStream_t s, const TrainSynDims& d, const float* dense,
                              const float* u1, const float* us0, const float* gh, float* gdense, float* wpart, int n_w) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tr_syn1x1_bwd_kernel<L, CH, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(tr_syn1x1_bwd_kernel<L, CH, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(tr_syn1x1_bwd_kernel<L, CH, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(tr_syn1x1_bwd_kernel<L, CH, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  switch (d.bank) {
    case 0: tr_syn1x1_bwd_kernel<L, CH, 0><<<g, t, smem, s>>>(d, dense, u1, us0, gh, gdense, wpart, n_w); break;
    case 1: tr_syn1x1_bwd_kernel<L, CH, 1><<<g, t, smem, s>>>(d, dense, u1, us0, gh, gdense, wpart, n_w); break;
    case 2: tr_syn1x1_bwd_kernel<L, CH, 2><<<g, t, smem, s>>>(d, dense, u1, us0, gh, gdense, wpart, n_w); break;
    default: tr_syn1x1_bwd_kernel<L, CH, 3><<<g, t, smem, s>>>(d, dense, u1, us0, gh, gdense, wpart, n_w); break;
  }
}
struct TrSynEntry {
  int L, CH;
  TrSynFwdFn fwd;
  TrSynBwdFn bwd;
  int vec;  // floats per pixel record of the 1x1 adjoint
};
#define TR_SYN(L, CH) {L, CH, tr_syn_fwd_launch<L, CH>, tr_syn_bwd_launch<L, CH>, TrSyn1x1Layout<L, CH>::VEC}
static const TrSynEntry kTrSyn[] = {TR_SYN(7, 40), TR_SYN(7, 16), TR_SYN(7, 8), TR_SYN(4, 8)};
static const TrSynEntry* find_tr_syn(const cc_model_desc& d) {
  for (const auto& e : kTrSyn)
    if (e.L == d.L && e.CH == d.syn_widths[1]) return &e;
  return nullptr;
}

int train_supported(const cc_model_desc& d) {
  if (d.up_2d || !find_tr_syn(d)) return 0;
  // the kernels use 32-bit offsets inside one plane (a grid, a channel of the
  // image): P must stay below 2^31 (cc_validate admits exactly 2^31)
  if ((int64_t)d.H * d.W >= ((int64_t)1 << 31)) return 0;
  for (const auto& e : kTrArm)
    if (e.C == d.n_ctx && e.NH == d.arm_widths[1] && e.NHL == d.arm_n_layers - 1) return 1;
  return 0;
}

// sum of partial rows into grad[0 .. n): fp64, two coalesced stages
static int reduce_partials(const float* part, int64_t blocks, int64_t stride, int n, float* grad, double* tmp,
                           cudaStream_t s) {
  const int chunks = (int)(blocks < TR_RCHUNK ? (blocks > 0 ? blocks : 1) : TR_RCHUNK);
  if (n <= 128) {
    int n_pad = 1;
    while (n_pad < n) n_pad <<= 1;
    tr_reduce1_narrow_kernel<<<chunks, 256, 0, s>>>(part, blocks, stride, n, n_pad, tmp);
  } else {
    tr_reduce1_kernel<<<dim3((n + TB - 1) / TB, chunks), TB, 0, s>>>(part, blocks, stride, n, tmp);
  }
  tr_reduce2_kernel<<<(n + 7) / 8, 256, 0, s>>>(tmp, chunks, n, grad);
  return 2;
}

static int blocks_for(int64_t n) { return (int)((n + TB - 1) / TB); }

#define TCONV_BWD(K) ((K) == 8 ? tr_tconv_bwd_kernel<8> : (K) == 4 ? tr_tconv_bwd_kernel<4> : tr_tconv_bwd_kernel<0>)
#define TCONV_FWD(K) ((K) == 8 ? tr_tconv_fwd_kernel<8> : (K) == 4 ? tr_tconv_fwd_kernel<4> : tr_tconv_fwd_kernel<0>)

// The small levels' steps of the upsampling chain (forward or adjoint) in ONE
// single-CTA launch: each of them is a few thousand elements, so as separate
// launches they cost launch latency, not work.  Passes run in order with a
// CTA barrier between them (a pass reads the previous one's output).
constexpr int TCH_THREADS = 1024;
constexpr int TCH_MAX_PASSES = 4 * CC_MAX_LEVELS;
struct TrChainPass {
  int32_t kind;  // 0 tconv forward, 1 tconv adjoint (+ tap partial rows), 2 add dst = a + b, 3 copy dst = a
  int32_t lines, n, m, nch;
  int64_t g_ls, g_es, o_ls, o_es, g_cs, o_cs;
  const float* a;  // kind 0/1: g (input), 2/3: a
  const float* b;  // kind 1: gout; 2: b
  float* dst;      // kind 0: out, 1: gg, 2/3: dst
  float* kpart;    // kind 1: nch rows of K
  int64_t count;   // kind 2/3: elements
};
struct TrChain {
  int32_t np, K, koff;
  TrChainPass p[TCH_MAX_PASSES];
};
template <int KT>
__global__ void __launch_bounds__(TCH_THREADS) tr_chain_kernel(const __grid_constant__ TrChain c) {
  __shared__ float red[8][TCH_THREADS / 32];
  const int K = KT;
  for (int pi = 0; pi < c.np; pi++) {
    const TrChainPass& P = c.p[pi];
    if (P.kind >= 2) {
      for (int64_t e = threadIdx.x; e < P.count; e += TCH_THREADS)
        P.dst[e] = P.kind == 2 ? P.a[e] + P.b[e] : P.a[e];
    } else if (P.kind == 0) {
      const int64_t per = (int64_t)P.lines * P.m;
      for (int64_t e = threadIdx.x; e < per * P.nch; e += TCH_THREADS) {
        const int ch = (int)e / (int)per;  // the small levels: 32-bit index math
        const int idx = (int)e - ch * (int)per;
        const float* g = P.a + ch * P.g_cs;
        int line, o;
        if (P.g_es == 1) {
          line = idx / P.m;
          o = idx - line * P.m;
        } else {
          o = idx / P.lines;
          line = idx - o * P.lines;
        }
        const int q = o >> 1, r = o & 1;
        float acc = 0.0f;
#pragma unroll
        for (int t = 0; t < K / 2; t++)
          acc = fmaf(c_tw[c.koff + 2 * t + 1 - r], g[line * P.g_ls + (int64_t)clampi(q + r + K / 4 - 1 - t, 0, P.n - 1) * P.g_es], acc);
        P.dst[ch * P.o_cs + line * P.o_ls + (int64_t)o * P.o_es] = acc;
      }
    } else {  // adjoint, one channel at a time (one tap-partial row each)
      for (int ch = 0; ch < P.nch; ch++) {
        const float* g = P.a + ch * P.g_cs;
        const float* gout = P.b + ch * P.o_cs;
        float* gg = P.dst + ch * P.g_cs;
        float dk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t idx = threadIdx.x; idx < (int64_t)P.lines * P.n; idx += TCH_THREADS) {
          int line, s2;
          if (P.g_es == 1) {
            line = (int)idx / P.n;
            s2 = (int)idx - line * P.n;
          } else {
            s2 = (int)idx / P.lines;
            line = (int)idx - s2 * P.lines;
          }
          const int E = K / 4, PP = K / 2 - 1 + 2 * E;
          const float xs = g[line * P.g_ls + (int64_t)s2 * P.g_es];
          const int i_lo = (s2 == 0) ? 0 : s2 + E, i_hi = (s2 == P.n - 1) ? P.n - 1 + 2 * E : s2 + E;
          float acc = 0.0f;
          for (int i = i_lo; i <= i_hi; i++)
#pragma unroll
            for (int j = 0; j < K; j++) {
              const int o = 2 * i + j - PP;
              if (o >= 0 && o < P.m) {
                const float go = gout[line * P.o_ls + (int64_t)o * P.o_es];
                acc = fmaf(c_tw[c.koff + j], go, acc);
                dk[j] = fmaf(xs, go, dk[j]);
              }
            }
          gg[line * P.g_ls + (int64_t)s2 * P.g_es] = acc;
        }
#pragma unroll
        for (int j = 0; j < K; j++) {
          float v = dk[j];
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o2);
          if ((threadIdx.x & 31) == 0) red[j][threadIdx.x >> 5] = v;
        }
        __syncthreads();
        if (threadIdx.x < K) {
          float v = 0.0f;
          for (int w2 = 0; w2 < TCH_THREADS / 32; w2++) v += red[threadIdx.x][w2];
          P.kpart[(int64_t)ch * K + threadIdx.x] = v;
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}
// a level step goes to the chain when its largest pass is this small
constexpr int64_t TCH_SMALL = 8192;
static void launch_chain(const TrChain& c, cudaStream_t s) {
  if (c.np == 0) return;
  if (c.K == 8) tr_chain_kernel<8><<<1, TCH_THREADS, 0, s>>>(c);
  else tr_chain_kernel<4><<<1, TCH_THREADS, 0, s>>>(c);
}

// ---------------------------------------------------------------- constant-bank ownership
// A bank is BUSY from acquire_bank (before its weights are copied in) to
// release_bank (after the step's last kernel is enqueued): a busy bank is never
// handed to another caller, so no copy into c_tw / c_tp can be enqueued while
// another host thread is still enqueuing kernels that read that bank.  A free
// bank remembers its last owner stream and an event recorded by that owner at
// release (while it still owned the bank), so a new owner's stream waits for
// every kernel of the previous owner's last step before overwriting it.  When
// every bank is busy the caller BLOCKS on the host until one is released.
// State is per device (one bank table per device; __constant__ memory is
// per-device), the events are created on their device and reused.
constexpr int TR_MAX_DEVICES = 64;
struct TrBank {
  cudaStream_t owner = nullptr;
  bool used = false;  // has had an owner (last_use recorded)
  bool busy = false;  // held by a caller between acquire and release
  cudaEvent_t last_use = nullptr;
  uint64_t tick = 0;
};
struct TrBankSet {
  TrBank b[TR_BANKS];
  bool init = false;
};
static TrBankSet g_banks[TR_MAX_DEVICES];
static std::mutex g_bank_mu;
static std::condition_variable g_bank_cv;
static uint64_t g_bank_tick = 0;

// the bank stream s trains with on the current device (blocks while all are
// busy); -1 if the device index is out of range or an event cannot be created
static int acquire_bank(cudaStream_t s, int* dev_out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= TR_MAX_DEVICES) return -1;
  std::unique_lock<std::mutex> lk(g_bank_mu);
  TrBankSet& set = g_banks[dev];
  if (!set.init) {
    for (auto& b : set.b)
      if (cudaEventCreateWithFlags(&b.last_use, cudaEventDisableTiming) != cudaSuccess) return -1;
    set.init = true;
  }
  int k = -1;
  for (;;) {
    // the bank this stream used last, if free; else the least recently used free bank
    for (int i = 0; i < TR_BANKS; i++)
      if (!set.b[i].busy && set.b[i].used && set.b[i].owner == s) k = i;
    if (k < 0)
      for (int i = 0; i < TR_BANKS; i++)
        if (!set.b[i].busy && (k < 0 || set.b[i].tick < set.b[k].tick)) k = i;
    if (k >= 0) break;
    g_bank_cv.wait(lk);
  }
  TrBank& b = set.b[k];
  if (b.used && b.owner != s) cudaStreamWaitEvent(s, b.last_use, 0);  // previous owner's last step
  b.owner = s;
  b.used = true;
  b.busy = true;
  b.tick = ++g_bank_tick;
  *dev_out = dev;
  return k;
}
static void release_bank(int dev, int k, cudaStream_t s) {
  {
    std::lock_guard<std::mutex> lk(g_bank_mu);
    TrBank& b = g_banks[dev].b[k];
    cudaEventRecord(b.last_use, s);  // still the owner: nobody else can hold a busy bank
    b.busy = false;
  }
  g_bank_cv.notify_all();
}
// releases the bank on every exit path of train_step_impl
struct TrBankGuard {
  int dev, k;
  cudaStream_t s;
  ~TrBankGuard() {
    if (k >= 0) release_bank(dev, k, s);
  }
};

// The iteration.  Returns the number of kernel launches (>= 0) or -1 if a
// CUDA call failed (the caller checks cudaGetLastError).
int train_step_impl(const cc_model_desc& d, float* par, const float* noise, const float* image, float* am, float* av,
                    const cc_adam* opt, cc_rd_result* result, float* grad, void* ws, cudaStream_t s) {
  TrainPlan pl;
  make_plan(d, pl);
  char* W = (char*)ws;
  auto F = [&](size_t o) { return (float*)(W + o); };
  const TrainLevels& lv = pl.lv;
  const int64_t P = (int64_t)d.H * d.W;
  const int L = d.L, K = d.up_taps, CH = d.syn_widths[1], R = d.syn_n_res;
  int launches = 0;
  // weights -> constant bank (arm | up | syn), device to device
  const int64_t nw = pl.n_arm + pl.n_up + pl.n_syn;
  (void)nw;
  if (pl.n_arm > TR_UP_OFF || pl.n_up > TR_SYN_OFF - TR_UP_OFF || pl.n_syn > TR_MAX_W - TR_SYN_OFF ||
      pl.n_arm / 2 + 2 > TR_MAX_ARMP)
    return -2;
  int bank_dev = 0;
  const int bank = acquire_bank(s, &bank_dev);
  if (bank < 0) return -1;
  TrBankGuard bank_guard{bank_dev, bank, s};  // released after the last enqueue, on every path
  const int tw0 = bank * TR_MAX_W, tp0 = bank * TR_MAX_ARMP;
  const float* pw = par + lv.n_lat;  // [arm | up | syn] -> the bank's fixed slots
  cudaMemcpyToSymbolAsync(c_tw, pw, sizeof(float) * (size_t)pl.n_arm, sizeof(float) * (size_t)tw0,
                          cudaMemcpyDeviceToDevice, s);
  cudaMemcpyToSymbolAsync(c_tw, pw + pl.n_arm, sizeof(float) * (size_t)pl.n_up, sizeof(float) * (size_t)(tw0 + TR_UP_OFF),
                          cudaMemcpyDeviceToDevice, s);
  cudaMemcpyToSymbolAsync(c_tw, pw + pl.n_arm + pl.n_up, sizeof(float) * (size_t)pl.n_syn,
                          sizeof(float) * (size_t)(tw0 + TR_SYN_OFF), cudaMemcpyDeviceToDevice, s);
  {  // FFMA2-packed ARM weights (forward) through a workspace buffer
    float2* packed = (float2*)(W + pl.o_grad_tmp);  // free until the first reduction
    tr_pack_arm_kernel<<<1, 256, 0, s>>>(par + lv.n_lat, packed, d.arm_n_layers, d.n_ctx, d.arm_widths[1]);
    cudaMemcpyToSymbolAsync(c_tp, packed, sizeof(float2) * (size_t)(pl.n_arm / 2 + 2), sizeof(float2) * (size_t)tp0,
                            cudaMemcpyDeviceToDevice, s);
    launches++;
  }
  const int koff = tw0 + TR_UP_OFF;  // taps in c_tw
  TrainSynDims sd;
  sd.H = d.H;
  sd.W = d.W;
  sd.L = L;
  sd.CH = CH;
  sd.R = R;
  sd.P = P;
  sd.oA0 = tw0 + TR_SYN_OFF;
  sd.bank = bank;
  sd.oa0 = sd.oA0 + L * CH;
  sd.oA1 = sd.oa0 + CH;
  sd.oa1 = sd.oA1 + 3 * CH;
  sd.oG = sd.oa1 + 3;
  float* g_lat = grad;                     // gradient layout = parameter layout
  float* g_arm = grad + lv.n_lat;
  float* g_up = g_arm + pl.n_arm;
  float* g_syn = g_up + pl.n_up;

  // 1. proxy
  tr_proxy_kernel<<<blocks_for(lv.n_lat), TB, 0, s>>>(par, noise, F(pl.o_yq), lv.n_lat);
  launches++;
  // 2. ARM forward + backward, gather, weight-gradient reduction
  {
    TrainArmParams ap;
    memset(&ap, 0, sizeof(ap));
    ap.lv = lv;
    ap.n_ctx = d.n_ctx;
    for (int c = 0; c < d.n_ctx; c++) {
      ap.dy[c] = d.ctx_dy[c];
      ap.dx[c] = d.ctx_dx[c];
    }
    ap.res_mask = d.arm_residual_mask;
    ap.lsmin = d.logscale_min;
    ap.lsmax = d.logscale_max;
    ap.bits_cap = (float)(-log2((double)d.p_floor));
    ap.w_r = (float)(d.lambda / (double)P);
    ap.yq = F(pl.o_yq);
    ap.gown = F(pl.o_gown);
    ap.dctx = F(pl.o_dctx);
    ap.rate = (double*)(W + pl.o_rate);
    ap.wpart = F(pl.o_wpart_arm);
    ap.n_arm = (int)pl.n_arm;
    ap.tw0 = tw0;
    ap.tp0 = tp0;
    const int C = d.n_ctx, NH = d.arm_widths[1], NL = d.arm_n_layers;
    const TrArmEntry* ae = nullptr;
    for (const auto& e : kTrArm)
      if (e.C == C && e.NH == NH && e.NHL == NL - 1) ae = &e;
    if (!ae) return -3;
    ae->fn(dim3((unsigned)pl.arm_ctas), TA_THREADS, sizeof(float) * (size_t)TA_THREADS * ae->vec, s, ap);
    launches++;
  }
  {
    TrainCtx cx;
    memset(&cx, 0, sizeof(cx));
    cx.C = d.n_ctx;
    for (int c = 0; c < d.n_ctx; c++) {
      cx.dy[c] = d.ctx_dy[c];
      cx.dx[c] = d.ctx_dx[c];
    }
    tr_arm_gather_kernel<<<blocks_for(lv.n_lat), TB, 0, s>>>(lv, cx, F(pl.o_gown), F(pl.o_dctx), g_lat);
    launches++;
    launches += reduce_partials(F(pl.o_wpart_arm), pl.arm_ctas, pl.n_arm, (int)pl.n_arm, g_arm,
                                (double*)(W + pl.o_grad_tmp), s);
  }
  // 3. upsampling forward on stacks: T_{L-1} = [y_hat_{L-1}]; step j takes
  //    T_{j+1} (L-1-j channels) through one x2 step into T_j[1..]; T_j[0] = y_hat_j
  float* dense = F(pl.o_dense);
  float* chain = F(pl.o_chain);
  auto Tj = [&](int j) { return j == 0 ? dense : chain + pl.chain_off[j]; };
  // small levels (the coarse end of the chain) go to one single-CTA launch
  const bool chain_ok = (K == 8 || K == 4);
  auto small = [&](int j) { return chain_ok && (int64_t)lv.h[j] * lv.w[j] * (L - 1 - j) <= TCH_SMALL; };
  TrChain fc;
  fc.np = 0, fc.K = K, fc.koff = koff;
  for (int j = 0; j < L; j++) {
    if (j >= 1 && small(j - 1)) {  // T_j[0] = y_hat_j feeds only small steps: copy inside the chain
      TrChainPass& c = fc.p[fc.np++];
      c = TrChainPass{};
      c.kind = 3, c.a = F(pl.o_yq) + lv.off[j], c.dst = Tj(j), c.count = (int64_t)lv.h[j] * lv.w[j];
    } else {
      cudaMemcpyAsync(Tj(j), F(pl.o_yq) + lv.off[j], sizeof(float) * (size_t)lv.h[j] * lv.w[j],
                      cudaMemcpyDeviceToDevice, s);
    }
  }
  for (int j = L - 2; j >= 0; j--) {
    const int nch = L - 1 - j;
    const int hs = lv.h[j + 1], ws2 = lv.w[j + 1], wd = lv.w[j], hd = lv.h[j];
    float* mid = chain + pl.mid_off[j];
    if (small(j)) {
      TrChainPass& x = fc.p[fc.np++];
      x = TrChainPass{};
      x.kind = 0, x.a = Tj(j + 1), x.dst = mid, x.lines = hs, x.n = ws2, x.m = wd, x.nch = nch;
      x.g_ls = ws2, x.g_es = 1, x.o_ls = wd, x.o_es = 1, x.g_cs = (int64_t)hs * ws2, x.o_cs = (int64_t)hs * wd;
      TrChainPass& y = fc.p[fc.np++];
      y = TrChainPass{};
      y.kind = 0, y.a = mid, y.dst = Tj(j) + (int64_t)hd * wd, y.lines = wd, y.n = hs, y.m = hd, y.nch = nch;
      y.g_ls = 1, y.g_es = wd, y.o_ls = 1, y.o_es = wd, y.g_cs = (int64_t)hs * wd, y.o_cs = (int64_t)hd * wd;
      if (j == 0 || !small(j - 1)) {
        launch_chain(fc, s);
        launches++;
        fc.np = 0;
      }
      continue;
    }
    // x pass: per channel, lines = rows (hs), n = ws2 -> m = wd
    TCONV_FWD(K)<<<dim3(blocks_for((int64_t)hs * wd), nch), TB, 0, s>>>(
        Tj(j + 1), mid, hs, ws2, wd, ws2, 1, wd, 1, K, koff, (int64_t)hs * ws2, (int64_t)hs * wd);
    // y pass: per channel, lines = columns (wd), n = hs -> m = hd, into T_j channels 1..
    TCONV_FWD(K)<<<dim3(blocks_for((int64_t)wd * hd), nch), TB, 0, s>>>(
        mid, Tj(j) + (int64_t)hd * wd, wd, hs, hd, 1, wd, 1, wd, K, koff, (int64_t)hs * wd, (int64_t)hd * wd);
    launches += 2;
  }
  // 4. synthesis forward, distortion, synthesis adjoint
  float* us = F(pl.o_us);
  float* hsb = F(pl.o_hs);
  const TrSynEntry* se = find_tr_syn(d);
  if (!se) return -4;
  se->fwd(blocks_for(P), TB, s, sd, dense, nullptr, us, hsb);  // u1 is recomputed by the adjoint
  launches++;
  for (int r = 0; r < R; r++) {
    tr_conv_fwd_kernel<<<blocks_for(P), TB, 0, s>>>(sd, r, hsb + (int64_t)r * 3 * P, us + (int64_t)(r + 1) * 3 * P,
                                                  hsb + (int64_t)(r + 1) * 3 * P);
    launches++;
  }
  float* gh = F(pl.o_gh0);
  float* gh2 = F(pl.o_gh1);
  const int64_t n_sse = (3 * P + TB - 1) / TB;
  tr_loss_kernel<<<(int)n_sse, TB, 0, s>>>(sd, hsb + (int64_t)R * 3 * P, image, gh, (double*)(W + pl.o_sse));
  launches++;
  for (int r = R - 1; r >= 0; r--) {
    float* cpart = F(pl.o_cpart) + (int64_t)r * pl.p_blocks * 84;
    tr_conv_bwd_kernel<<<(int)pl.p_blocks, CT_Y * CT_X, 0, s>>>(sd, r, hsb + (int64_t)r * 3 * P,
                                                              us + (int64_t)(r + 1) * 3 * P, gh, gh2, cpart);
    launches++;
    launches += reduce_partials(cpart, pl.p_blocks, 84, 84, g_syn + (sd.oG - sd.oA0) + 84 * r,
                                (double*)(W + pl.o_grad_tmp), s);
    float* t = gh;
    gh = gh2;
    gh2 = t;
  }
  {
    const int n_w = L * CH + CH + 3 * CH + 3;
    const size_t smem = sizeof(float) * (size_t)TS_THREADS * se->vec;  // records, then the chunk partials over them
    se->bwd((int)pl.s_blocks, TS_THREADS, smem, s, sd, dense, nullptr, us, gh, F(pl.o_gdense), F(pl.o_spart), n_w);
    launches++;
    launches += reduce_partials(F(pl.o_spart), pl.s_blocks, n_w, n_w, g_syn, (double*)(W + pl.o_grad_tmp), s);
  }
  // 5. upsampling adjoint on the stacks: gT_0 = gdense; gy_hat_j += gT_j[0];
  //    gT_{j+1} = Up^T(gT_j[1..]) (y adjoint then x adjoint), tap partials
  float* gdense = F(pl.o_gdense);
  float* kpart = F(pl.o_kpart);
  int64_t krow = 0;
  const float* gT = gdense;
  TrChain bc;  // the small levels' adjoint steps (from the first small one to the coarsest level)
  bc.np = 0, bc.K = K, bc.koff = koff;
  for (int j = 0; j < L; j++) {
    const bool sm = L >= 2 && small(j < L - 1 ? j : L - 2);
    if (sm) {
      TrChainPass& a = bc.p[bc.np++];
      a = TrChainPass{};
      a.kind = 2, a.a = g_lat + lv.off[j], a.b = gT, a.dst = g_lat + lv.off[j], a.count = (int64_t)lv.h[j] * lv.w[j];
    } else {
      tr_proxy_kernel<<<blocks_for((int64_t)lv.h[j] * lv.w[j]), TB, 0, s>>>(g_lat + lv.off[j], gT, g_lat + lv.off[j],
                                                                          (int64_t)lv.h[j] * lv.w[j]);
      launches++;
    }
    if (j + 1 >= L) break;
    const int nch = L - 1 - j;
    const int hs = lv.h[j + 1], ws2 = lv.w[j + 1], wd = lv.w[j], hd = lv.h[j];
    const float* mid = chain + pl.mid_off[j];
    float* gmid = F(pl.o_g1);
    float* gnext = (gT == F(pl.o_g0)) ? F(pl.o_g1) + (int64_t)nch * hs * wd : F(pl.o_g0);  // not aliasing gT / gmid
    if (sm) {
      TrChainPass& y = bc.p[bc.np++];
      y = TrChainPass{};
      y.kind = 1, y.a = mid, y.b = gT + (int64_t)hd * wd, y.dst = gmid, y.lines = wd, y.n = hs, y.m = hd, y.nch = nch;
      y.g_ls = 1, y.g_es = wd, y.o_ls = 1, y.o_es = wd, y.g_cs = (int64_t)hs * wd, y.o_cs = (int64_t)hd * wd;
      y.kpart = kpart + krow * K;
      krow += nch;
      TrChainPass& x = bc.p[bc.np++];
      x = TrChainPass{};
      x.kind = 1, x.a = Tj(j + 1), x.b = gmid, x.dst = gnext, x.lines = hs, x.n = ws2, x.m = wd, x.nch = nch;
      x.g_ls = ws2, x.g_es = 1, x.o_ls = wd, x.o_es = 1, x.g_cs = (int64_t)hs * ws2, x.o_cs = (int64_t)hs * wd;
      x.kpart = kpart + krow * K;
      krow += nch;
      gT = gnext;
      continue;
    }
    // y adjoint: inputs mid (per channel: lines = columns wd, n = hs), outputs gT_j[1..] (m = hd)
    const int64_t b1 = blocks_for((int64_t)wd * hs) < TR_TCONV_CAP ? blocks_for((int64_t)wd * hs) : TR_TCONV_CAP;
    TCONV_BWD(K)<<<dim3((unsigned)b1, nch), TB, 0, s>>>(mid, gT + (int64_t)hd * wd, gmid, wd, hs, hd, 1, wd, 1,
                                                               wd, K, koff, kpart + krow * K, (int64_t)hs * wd,
                                                               (int64_t)hd * wd);
    krow += b1 * nch;
    // x adjoint: inputs T_{j+1} (lines = rows hs, n = ws2), outputs gmid (m = wd)
    const int64_t b2 = blocks_for((int64_t)hs * ws2) < TR_TCONV_CAP ? blocks_for((int64_t)hs * ws2) : TR_TCONV_CAP;
    TCONV_BWD(K)<<<dim3((unsigned)b2, nch), TB, 0, s>>>(Tj(j + 1), gmid, gnext, hs, ws2, wd, ws2, 1, wd, 1, K,
                                                               koff, kpart + krow * K, (int64_t)hs * ws2,
                                                               (int64_t)hs * wd);
    krow += b2 * nch;
    launches += 2;
    gT = gnext;
  }
  if (bc.np > 0) {
    launch_chain(bc, s);
    launches++;
  }
  if (krow > 0) {
    launches += reduce_partials(kpart, krow, K, K, g_up, (double*)(W + pl.o_grad_tmp), s);
  } else {
    cudaMemsetAsync(g_up, 0, sizeof(float) * (size_t)K, s);
  }
  // 6. cost of this forward, then Adam on every parameter
  tr_result_kernel<<<1, TR_RES_THREADS, 0, s>>>((double*)(W + pl.o_rate), pl.arm_ctas * (TA_THREADS / 32), (double*)(W + pl.o_sse),
                                    n_sse, 1.0 / (3.0 * (double)P), d.lambda / (double)P, result);
  launches++;
  if (opt) {
    const float c1 = (float)(1.0 - pow((double)opt->beta1, opt->t)), c2 = (float)(1.0 - pow((double)opt->beta2, opt->t));
    tr_adam_kernel<<<blocks_for(pl.n_par) < 4096 ? blocks_for(pl.n_par) : 4096, TB, 0, s>>>(
        par, grad, am, av, pl.n_par, opt->lr, opt->beta1, opt->beta2, opt->eps, c1, c2);
    launches++;
  }
  return launches;  // bank_guard records this stream's last use of the bank
}

}  // namespace ccrd
