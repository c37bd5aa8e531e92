// arm_math.cuh -- the ARM arithmetic shared by the encoder's rate kernel
// (arm_rate.cu) and the wavefront decoder (arm_decode.cu), so both compute
// bit-identical (mu, log-scale, bits) for every latent: the Laplace bin
// -log2 P, the FFMA2 dense layers and the host-side weight packing.
#pragma once
#include "ccrd_common.cuh"

namespace ccrd {

// -log2 of the Laplace(mu, b) mass of the bin [y - 1/2, y + 1/2], floored at
// p_floor (readings #1-#3).  With a = |y - mu|,
// ib = 1/b, t1 = exp(-|a - 1/2| ib) and t2 = exp(-(min(a, 1/2) + 1/2) ib):
//   a <  1/2 : P = 1 - (t1 + t2) / 2            (t1, t2 = the two tail masses x 2)
//   a >= 1/2 : P = t1 (1 - t2) / 2              (t2 = exp(-ib): the bin's far edge)
// -- three MUFU ex2 and one lg2.  The far tails need no log-domain form: a P
// below p_floor is floored, and t1 flushes to zero only below 2^-126 (then P
// is floored too; a subnormal p_floor -- validated only as (0, 1) -- is
// reached there as bits_cap).
// The worst case, 1 - exp(-ib) at b = 256, cancels to ~1e-4 bits per latent,
// inside the 1e-3-bit per-latent parity tolerance.
__device__ __forceinline__ float laplace_bits(float y, float mu, float s, const ArmGeom& g) {
  constexpr float LOG2E = 1.4426950408889634f;
  s = fminf(fmaxf(s, g.lsmin), g.lsmax);
  const float ibl = exp2f_approx(-s * LOG2E) * LOG2E;  // log2(e) / b
  const float a = fabsf(y - mu);
  const float am = fminf(a, 0.5f);
  const float t1 = exp2f_approx(-fabsf(a - 0.5f) * ibl);
  const float t2 = exp2f_approx(-(am + 0.5f) * ibl);
  const float p_in = 1.0f - 0.5f * (t1 + t2);
  const float p_out = 0.5f * t1 * (1.0f - t2);
  const float pr = a < 0.5f ? p_in : p_out;
  return fminf(-log2f_approx(fmaxf(pr, g.p_floor)), g.bits_cap);
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

// Host: pack one image's ARM blob (per layer W[out][in] then b[out],
// PAPER.md:106-109; Table 1 "LinR" residuals folded as W' = W + I).
template <int C, int NH, int NHL>
static inline void pack_arm_weights(const cc_model_desc& d, const float* arm_w, ArmWeights<C, NH, NHL>& w) {
  const float* q = arm_w;
  auto res = [&](int k) { return (d.arm_residual_mask >> k) & 1u; };
  for (int i = 0; i < C; i++)
    for (int n = 0; n < NH / 2; n++) {
      float a = q[(2 * n) * C + i], b = q[(2 * n + 1) * C + i];
      if (res(0)) {  // only legal when C == NH (validated)
        a += (i == 2 * n) ? 1.0f : 0.0f;
        b += (i == 2 * n + 1) ? 1.0f : 0.0f;
      }
      w.w0[i][n] = make_float2(a, b);
    }
  for (int n = 0; n < NH / 2; n++) w.b0[n] = make_float2(q[C * NH + 2 * n], q[C * NH + 2 * n + 1]);
  q += C * NH + NH;
  for (int k = 0; k < NHL - 1; k++) {
    for (int i = 0; i < NH; i++)
      for (int n = 0; n < NH / 2; n++) {
        float a = q[(2 * n) * NH + i], b = q[(2 * n + 1) * NH + i];
        if (res(k + 1)) {
          a += (i == 2 * n) ? 1.0f : 0.0f;
          b += (i == 2 * n + 1) ? 1.0f : 0.0f;
        }
        w.wh[k][i][n] = make_float2(a, b);
      }
    for (int n = 0; n < NH / 2; n++) w.bh[k][n] = make_float2(q[NH * NH + 2 * n], q[NH * NH + 2 * n + 1]);
    q += NH * NH + NH;
  }
  for (int i = 0; i < NH; i++) w.wo[i] = make_float2(q[i], q[NH + i]);
  w.bo = make_float2(q[2 * NH], q[2 * NH + 1]);

}

}  // namespace ccrd
