/*
 * cctrain.c -- plain fp64 CPU oracle of ONE Cool-chic encoder training
 * iteration (NEXT-2): forward on the quantisation proxy, backward, Adam.
 *
 * TEST INFRASTRUCTURE ONLY (same rule as ccoracle.c): loaded by tests/ and
 * bench.py's baseline legs, never by the CUDA product path; shares no code
 * with it.
 *
 * What it computes, in the paper's order:
 *   PAPER.md:113-124 (Eq. 1): the encoder minimises
 *       J = D(x, x_hat) + lambda R(y_hat) / (H W)      (cost as in the RD forward)
 *   over the latents and psi, upsilon, theta, "through the continuous version
 *   y, using ... a differentiable proxy for the quantization Q" (PAPER.md:
 *   124-126).  Reading T1: the proxy is additive uniform noise,
 *   y_hat = y + u, u ~ U(-1/2, 1/2) given as an INPUT (the random numbers are
 *   data), with gradient passing unchanged to y.
 *   "One training iteration consists in one forward pass and
 *   one backward pass" -- here the exact gradient of J by the chain rule,
 *   layer by layer (every layer: gradient wrt its weights and wrt its input).
 *   SPEC.md:89-92 / PAPER.md (Adam, kingma2014adam): one Adam step on every
 *   parameter (latents y, ARM psi, upsampling taps upsilon, synthesis theta)
 *   with the same learning rate:
 *       m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g^2;
 *       p -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps).
 *
 * Forward definitions are those of ccoracle.c (readings #1-#22) evaluated on
 * real-valued y_hat: the Laplace bin mass P = F(y+1/2) - F(y-1/2) with the
 * continuous y; -log2 max(P, p_floor); the log-scale clamp.  Derivatives of the
 * non-smooth points (reading T2): ReLU'(0) = 0, the clamp passes no gradient
 * outside (lsmin, lsmax), the floor passes none when P < p_floor, and
 * replicate padding / zero context padding route gradients to the clamped /
 * no source.
 *
 * Parameter vector layout (shared with the ABI only as a documented layout,
 * not code): [ y (N_lat, packed like the latents) | arm_w | up_w | syn_w ].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ccoracle.h"

static int clampi_t(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

typedef struct {
  double lr, beta1, beta2, eps;
  int32_t t; /* step number, >= 1 */
} orc_adam;

int64_t orc_train_param_count(const orc_model* m) {
  int32_t h[ORC_MAX_LEVELS], w[ORC_MAX_LEVELS];
  int64_t n = orc_level_dims(m, h, w);
  for (int k = 0; k < m->arm_n_layers; k++) n += (int64_t)m->arm_widths[k] * m->arm_widths[k + 1] + m->arm_widths[k + 1];
  n += m->up_2d ? (int64_t)m->up_taps * m->up_taps : m->up_taps;
  for (int k = 0; k < m->syn_n_1x1; k++) n += (int64_t)m->syn_widths[k] * m->syn_widths[k + 1] + m->syn_widths[k + 1];
  n += 84 * (int64_t)m->syn_n_res;
  return n;
}

/* ---------------------------------------------------------------- Laplace */
static double lap_F(double t, double mu, double b) {
  return t < mu ? 0.5 * exp((t - mu) / b) : 1.0 - 0.5 * exp(-(t - mu) / b);
}
static double lap_f(double t, double mu, double b) { return exp(-fabs(t - mu) / b) / (2.0 * b); }

/* bits and its partial derivatives wrt y, mu and s (the pre-clamp log-scale) */
static double bits_and_grad(const orc_model* m, double y, double mu, double s, double* dy, double* dmu,
                            double* ds) {
  const double sc = s < m->logscale_min ? m->logscale_min : (s > m->logscale_max ? m->logscale_max : s);
  const double b = exp(sc);
  const double P = lap_F(y + 0.5, mu, b) - lap_F(y - 0.5, mu, b);
  if (!(P >= m->p_floor)) { /* floored: constant */
    *dy = *dmu = *ds = 0.0;
    return -log2(m->p_floor);
  }
  const double fu = lap_f(y + 0.5, mu, b), fl = lap_f(y - 0.5, mu, b);
  const double dPdy = fu - fl, dPdmu = -(fu - fl);
  /* dF(t)/db = -(t - mu) f(t) / b */
  const double dPdb = -((y + 0.5 - mu) * fu - (y - 0.5 - mu) * fl) / b;
  const double dbits_dP = -1.0 / (P * log(2.0));
  *dy = dbits_dP * dPdy;
  *dmu = dbits_dP * dPdmu;
  *ds = (s > m->logscale_min && s < m->logscale_max) ? dbits_dP * dPdb * b : 0.0;
  return -log2(P);
}

/* -------------------------------------------------- ARM forward + backward */
/* For latent (i, j) of grid g (h x w, doubles): accumulates the rate, adds
 * w_r * d bits / d y_hat into gy (own position and the context positions) and
 * w_r * d bits / d psi into garm. */
static double arm_latent(const orc_model* m, const double* g, int h, int w, int i, int j, const float* arm_w,
                         double w_r, double* gy, double* garm) {
  const int K = m->arm_n_layers;
  double z[ORC_MAX_LAYERS + 1][64], u[ORC_MAX_LAYERS][64];
  const int C = m->n_ctx;
  for (int c = 0; c < C; c++) {
    const int ii = i + m->ctx_dy[c], jj = j + m->ctx_dx[c];
    z[0][c] = (ii >= 0 && ii < h && jj >= 0 && jj < w) ? g[(int64_t)ii * w + jj] : 0.0;
  }
  /* forward, layer by layer (weights W_k[out][in] then b_k[out]) */
  const float* q = arm_w;
  const float* Wk[ORC_MAX_LAYERS];
  for (int k = 0; k < K; k++) {
    const int nin = m->arm_widths[k], nout = m->arm_widths[k + 1];
    Wk[k] = q;
    for (int o = 0; o < nout; o++) {
      double a = (double)q[nin * nout + o];
      for (int t = 0; t < nin; t++) a += (double)q[o * nin + t] * z[k][t];
      if (m->arm_residual[k]) a += z[k][o];
      u[k][o] = a;
      z[k + 1][o] = (k < K - 1) ? (a > 0.0 ? a : 0.0) : a;
    }
    q += nin * nout + nout;
  }
  const double mu = z[K][0], s = z[K][1];
  const double y = g[(int64_t)i * w + j];
  double dy, dmu, ds;
  const double bits = bits_and_grad(m, y, mu, s, &dy, &dmu, &ds);
  gy[(int64_t)i * w + j] += w_r * dy;
  /* backward */
  double dz[64], du[64];
  du[0] = w_r * dmu;
  du[1] = w_r * ds;
  int64_t goff = 0;
  int64_t off[ORC_MAX_LAYERS];
  for (int k = 0; k < K; k++) {
    off[k] = goff;
    goff += (int64_t)m->arm_widths[k] * m->arm_widths[k + 1] + m->arm_widths[k + 1];
  }
  for (int k = K - 1; k >= 0; k--) {
    const int nin = m->arm_widths[k], nout = m->arm_widths[k + 1];
    for (int o = 0; o < nout; o++) {
      for (int t = 0; t < nin; t++) garm[off[k] + o * nin + t] += du[o] * z[k][t];
      garm[off[k] + (int64_t)nin * nout + o] += du[o];
    }
    for (int t = 0; t < nin; t++) {
      double a = m->arm_residual[k] ? du[t] : 0.0;
      for (int o = 0; o < nout; o++) a += (double)Wk[k][o * nin + t] * du[o];
      dz[t] = a;
    }
    if (k > 0)
      for (int t = 0; t < nin; t++) du[t] = u[k - 1][t] > 0.0 ? dz[t] : 0.0;
  }
  for (int c = 0; c < C; c++) {
    const int ii = i + m->ctx_dy[c], jj = j + m->ctx_dx[c];
    if (ii >= 0 && ii < h && jj >= 0 && jj < w) gy[(int64_t)ii * w + jj] += dz[c];
  }
  return bits;
}

/* ------------------------------------------- upsampling (one stride-2 step) */
/* forward along one axis: the scatter definition of ccoracle.c's tconv_1d */
static void tconv1(const double* g, int n, int64_t gs, const float* k, int K, double* out, int mlen, int64_t os) {
  const int E = K / 4, P = K / 2 - 1 + 2 * E;
  for (int o = 0; o < mlen; o++) out[o * os] = 0.0;
  for (int i = 0; i < n + 2 * E; i++) {
    const double xi = g[clampi_t(i - E, 0, n - 1) * gs];
    for (int j = 0; j < K; j++) {
      const int o = 2 * i + j - P;
      if (o >= 0 && o < mlen) out[o * os] += xi * (double)k[j];
    }
  }
}
/* its adjoint: gg += T^T gout, gk += d<gout, T g>/dk */
static void tconv1_bwd(const double* g, int n, int64_t gs, const float* k, int K, const double* gout, int mlen,
                       int64_t os, double* gg, double* gk) {
  const int E = K / 4, P = K / 2 - 1 + 2 * E;
  for (int i = 0; i < n + 2 * E; i++) {
    const int src = clampi_t(i - E, 0, n - 1);
    const double xi = g[src * gs];
    double acc = 0.0;
    for (int j = 0; j < K; j++) {
      const int o = 2 * i + j - P;
      if (o >= 0 && o < mlen) {
        acc += (double)k[j] * gout[o * os];
        gk[j] += xi * gout[o * os];
      }
    }
    gg[src * gs] += acc;
  }
}
/* 2-D (Table 1) step and adjoint */
static void tconv2(const double* g, int n, int nw, const float* k2, int K, double* out, int mh, int mw) {
  const int E = K / 4, P = K / 2 - 1 + 2 * E;
  for (int64_t t = 0; t < (int64_t)mh * mw; t++) out[t] = 0.0;
  for (int i = 0; i < n + 2 * E; i++)
    for (int i2 = 0; i2 < nw + 2 * E; i2++) {
      const double xi = g[(int64_t)clampi_t(i - E, 0, n - 1) * nw + clampi_t(i2 - E, 0, nw - 1)];
      for (int a = 0; a < K; a++) {
        const int o = 2 * i + a - P;
        if (o < 0 || o >= mh) continue;
        for (int b = 0; b < K; b++) {
          const int o2 = 2 * i2 + b - P;
          if (o2 >= 0 && o2 < mw) out[(int64_t)o * mw + o2] += xi * (double)k2[a * K + b];
        }
      }
    }
}
static void tconv2_bwd(const double* g, int n, int nw, const float* k2, int K, const double* gout, int mh, int mw,
                       double* gg, double* gk) {
  const int E = K / 4, P = K / 2 - 1 + 2 * E;
  for (int i = 0; i < n + 2 * E; i++)
    for (int i2 = 0; i2 < nw + 2 * E; i2++) {
      const int64_t src = (int64_t)clampi_t(i - E, 0, n - 1) * nw + clampi_t(i2 - E, 0, nw - 1);
      const double xi = g[src];
      double acc = 0.0;
      for (int a = 0; a < K; a++) {
        const int o = 2 * i + a - P;
        if (o < 0 || o >= mh) continue;
        for (int b = 0; b < K; b++) {
          const int o2 = 2 * i2 + b - P;
          if (o2 >= 0 && o2 < mw) {
            const double go = gout[(int64_t)o * mw + o2];
            acc += (double)k2[a * K + b] * go;
            gk[a * K + b] += xi * go;
          }
        }
      }
      gg[src] += acc;
    }
}

/* ---------------------------------------------------------- the iteration */
/* Gradient of J at (y_hat = y + u, params) and J's components.
 * params: [y | arm_w | up_w | syn_w] (fp32).  grad: same layout (fp64).
 * out[4] = {rate_bits, sse, mse, cost} of this forward. */
int orc_train_grad(const orc_model* m, const float* params, const float* noise, const float* image, double* out,
                   double* grad) {
  int32_t h[ORC_MAX_LEVELS], w[ORC_MAX_LEVELS];
  const int64_t n_lat = orc_level_dims(m, h, w);
  const int64_t n_par = orc_train_param_count(m);
  const int L = m->L, H = m->H, W = m->W, K = m->up_taps;
  const int64_t P = (int64_t)H * W;
  const float* arm_w = params + n_lat;
  int64_t n_arm = 0;
  for (int k = 0; k < m->arm_n_layers; k++) n_arm += (int64_t)m->arm_widths[k] * m->arm_widths[k + 1] + m->arm_widths[k + 1];
  const float* up_w = arm_w + n_arm;
  const int n_up = m->up_2d ? K * K : K;
  const float* syn_w = up_w + n_up;
  for (int64_t t = 0; t < n_par; t++) grad[t] = 0.0;
  double* gy = grad;
  double* garm = grad + n_lat;
  double* gup = garm + n_arm;
  double* gsyn = gup + n_up;
  if (m->syn_n_1x1 != 2) return -1;

  /* proxy latents y_hat = y + u (fp64) */
  double* yq = (double*)malloc(sizeof(double) * (size_t)n_lat);
  for (int64_t t = 0; t < n_lat; t++) yq[t] = (double)params[t] + (double)noise[t];
  int64_t loff[ORC_MAX_LEVELS];
  {
    int64_t o = 0;
    for (int l = 0; l < L; l++) {
      loff[l] = o;
      o += (int64_t)h[l] * w[l];
    }
  }
  const double w_r = m->lambda / (double)P;

  /* rate and its gradient (ARM) */
  double R = 0.0;
  for (int l = 0; l < L; l++)
    for (int i = 0; i < h[l]; i++)
      for (int j = 0; j < w[l]; j++)
        R += arm_latent(m, yq + loff[l], h[l], w[l], i, j, arm_w, w_r, gy + loff[l], garm);

  /* upsampling forward, keeping every step's input for the backward */
  double* dense = (double*)malloc(sizeof(double) * (size_t)L * P);
  double* chain[ORC_MAX_LEVELS][ORC_MAX_LEVELS]; /* chain[l][j]: grid l carried to level j (j <= l) */
  double* mid[ORC_MAX_LEVELS][ORC_MAX_LEVELS];   /* separable: after the x pass of step j */
  memset(chain, 0, sizeof(chain));
  memset(mid, 0, sizeof(mid));
  for (int l = 0; l < L; l++) {
    chain[l][l] = (double*)malloc(sizeof(double) * (size_t)h[l] * w[l]);
    memcpy(chain[l][l], yq + loff[l], sizeof(double) * (size_t)h[l] * w[l]);
    for (int j = l - 1; j >= 0; j--) {
      const double* g = chain[l][j + 1];
      double* t2 = (double*)malloc(sizeof(double) * (size_t)h[j] * w[j]);
      if (m->up_2d) {
        tconv2(g, h[j + 1], w[j + 1], up_w, K, t2, h[j], w[j]);
      } else {
        double* t1 = (double*)malloc(sizeof(double) * (size_t)h[j + 1] * w[j]);
        for (int r = 0; r < h[j + 1]; r++) tconv1(g + (int64_t)r * w[j + 1], w[j + 1], 1, up_w, K, t1 + (int64_t)r * w[j], w[j], 1);
        for (int c = 0; c < w[j]; c++) tconv1(t1 + c, h[j + 1], w[j], up_w, K, t2 + c, h[j], w[j]);
        mid[l][j] = t1;
      }
      chain[l][j] = t2;
    }
    memcpy(dense + (int64_t)l * P, chain[l][0], sizeof(double) * (size_t)P);
  }

  /* synthesis forward with the activations kept */
  const int CH = m->syn_widths[1], RN = m->syn_n_res;
  const float* A0 = syn_w;
  const float* a0 = A0 + L * CH;
  const float* A1 = a0 + CH;
  const float* a1 = A1 + CH * 3;
  const float* Gr = a1 + 3;
  double* u1 = (double*)malloc(sizeof(double) * (size_t)CH * P);  /* layer-0 pre-activation */
  double* hs[8];                                                  /* hs[0] = 1x1 output (post ReLU), hs[r+1] = res layer r out */
  double* us[8];                                                  /* pre-activations (1x1 layer 1 and each res layer) */
  for (int r = 0; r <= RN; r++) {
    hs[r] = (double*)malloc(sizeof(double) * 3 * (size_t)P);
    us[r] = (double*)malloc(sizeof(double) * 3 * (size_t)P);
  }
  for (int64_t p = 0; p < P; p++) {
    double v1[64];
    for (int n = 0; n < CH; n++) {
      double a = (double)a0[n];
      for (int i = 0; i < L; i++) a += (double)A0[n * L + i] * dense[(int64_t)i * P + p];
      u1[(int64_t)n * P + p] = a;
      v1[n] = a > 0.0 ? a : 0.0;
    }
    for (int c = 0; c < 3; c++) {
      double a = (double)a1[c];
      for (int n = 0; n < CH; n++) a += (double)A1[c * CH + n] * v1[n];
      us[0][(int64_t)c * P + p] = a;
      hs[0][(int64_t)c * P + p] = (RN > 0) ? (a > 0.0 ? a : 0.0) : a;  /* ReLU unless it is the last layer */
    }
  }
  for (int r = 0; r < RN; r++) {
    const float* G = Gr + 84 * r;
    const float* gb = G + 81;
    for (int y = 0; y < H; y++)
      for (int x = 0; x < W; x++)
        for (int co = 0; co < 3; co++) {
          double a = hs[r][(int64_t)co * P + (int64_t)y * W + x] + (double)gb[co];
          for (int ci = 0; ci < 3; ci++)
            for (int ky = 0; ky < 3; ky++)
              for (int kx = 0; kx < 3; kx++)
                a += (double)G[((co * 3 + ci) * 3 + ky) * 3 + kx] *
                     hs[r][(int64_t)ci * P + (int64_t)clampi_t(y + ky - 1, 0, H - 1) * W + clampi_t(x + kx - 1, 0, W - 1)];
          us[r + 1][(int64_t)co * P + (int64_t)y * W + x] = a;
          hs[r + 1][(int64_t)co * P + (int64_t)y * W + x] = (r < RN - 1) ? (a > 0.0 ? a : 0.0) : a;
        }
  }
  const double* xh = hs[RN];
  double sse = 0.0;
  for (int64_t t = 0; t < 3 * P; t++) {
    const double e = (double)image[t] - xh[t];
    sse += e * e;
  }
  const double mse = sse / (3.0 * (double)P);
  out[0] = R;
  out[1] = sse;
  out[2] = mse;
  out[3] = mse + m->lambda * R / (double)P;

  /* backward: synthesis */
  double* gh = (double*)malloc(sizeof(double) * 3 * (size_t)P);  /* dJ / d(current layer output) */
  for (int64_t t = 0; t < 3 * P; t++) gh[t] = -2.0 * ((double)image[t] - xh[t]) / (3.0 * (double)P);
  double* gin = (double*)malloc(sizeof(double) * 3 * (size_t)P);
  for (int r = RN - 1; r >= 0; r--) {
    const float* G = Gr + 84 * r;
    double* gG = gsyn + (int64_t)(L * CH + CH + CH * 3 + 3) + 84 * r;
    /* through the ReLU of this layer (none on the last) */
    for (int64_t t = 0; t < 3 * P; t++)
      if (r < RN - 1 && !(us[r + 1][t] > 0.0)) gh[t] = 0.0;
    for (int64_t t = 0; t < 3 * P; t++) gin[t] = gh[t]; /* residual */
    for (int y = 0; y < H; y++)
      for (int x = 0; x < W; x++)
        for (int co = 0; co < 3; co++) {
          const double d = gh[(int64_t)co * P + (int64_t)y * W + x];
          gG[81 + co] += d;
          for (int ci = 0; ci < 3; ci++)
            for (int ky = 0; ky < 3; ky++)
              for (int kx = 0; kx < 3; kx++) {
                const int64_t src = (int64_t)ci * P + (int64_t)clampi_t(y + ky - 1, 0, H - 1) * W + clampi_t(x + kx - 1, 0, W - 1);
                gG[((co * 3 + ci) * 3 + ky) * 3 + kx] += d * hs[r][src];
                gin[src] += (double)G[((co * 3 + ci) * 3 + ky) * 3 + kx] * d;
              }
        }
    double* tswap = gh;
    gh = gin;
    gin = tswap;
  }
  /* 1x1 layer 1 (L->CH->3): through its ReLU when residual layers follow */
  double* gdense = (double*)calloc((size_t)L * P, sizeof(double));
  {
    double* gA0 = gsyn;
    double* ga0 = gA0 + L * CH;
    double* gA1 = ga0 + CH;
    double* ga1 = gA1 + CH * 3;
    for (int64_t p = 0; p < P; p++) {
      double d2[3], v1[64], d1[64];
      for (int c = 0; c < 3; c++) {
        double d = gh[(int64_t)c * P + p];
        if (RN > 0 && !(us[0][(int64_t)c * P + p] > 0.0)) d = 0.0;
        d2[c] = d;
      }
      for (int n = 0; n < CH; n++) {
        const double a = u1[(int64_t)n * P + p];
        v1[n] = a > 0.0 ? a : 0.0;
      }
      for (int c = 0; c < 3; c++) {
        ga1[c] += d2[c];
        for (int n = 0; n < CH; n++) gA1[c * CH + n] += d2[c] * v1[n];
      }
      for (int n = 0; n < CH; n++) {
        double a = 0.0;
        for (int c = 0; c < 3; c++) a += (double)A1[c * CH + n] * d2[c];
        d1[n] = u1[(int64_t)n * P + p] > 0.0 ? a : 0.0;
      }
      for (int n = 0; n < CH; n++) {
        ga0[n] += d1[n];
        for (int i = 0; i < L; i++) gA0[n * L + i] += d1[n] * dense[(int64_t)i * P + p];
      }
      for (int i = 0; i < L; i++) {
        double a = 0.0;
        for (int n = 0; n < CH; n++) a += (double)A0[n * L + i] * d1[n];
        gdense[(int64_t)i * P + p] = a;
      }
    }
  }
  /* backward: upsampling, level by level (adjoint of every step, reverse order) */
  for (int64_t t = 0; t < (int64_t)h[0] * w[0]; t++) gy[loff[0] + t] += gdense[t];
  for (int l = 1; l < L; l++) {
    double* gcur = (double*)malloc(sizeof(double) * (size_t)P);
    memcpy(gcur, gdense + (int64_t)l * P, sizeof(double) * (size_t)P);
    for (int j = 0; j < l; j++) {
      /* step j maps chain[l][j+1] (h_{j+1} x w_{j+1}) -> chain[l][j] (h_j x w_j) */
      double* gprev = (double*)calloc((size_t)h[j + 1] * w[j + 1], sizeof(double));
      if (m->up_2d) {
        tconv2_bwd(chain[l][j + 1], h[j + 1], w[j + 1], up_w, K, gcur, h[j], w[j], gprev, gup);
      } else {
        double* gmid = (double*)calloc((size_t)h[j + 1] * w[j], sizeof(double));
        for (int c = 0; c < w[j]; c++)
          tconv1_bwd(mid[l][j] + c, h[j + 1], w[j], up_w, K, gcur + c, h[j], w[j], gmid + c, gup);
        for (int r = 0; r < h[j + 1]; r++)
          tconv1_bwd(chain[l][j + 1] + (int64_t)r * w[j + 1], w[j + 1], 1, up_w, K, gmid + (int64_t)r * w[j], w[j], 1,
                     gprev + (int64_t)r * w[j + 1], gup);
        free(gmid);
      }
      free(gcur);
      gcur = gprev;
    }
    for (int64_t t = 0; t < (int64_t)h[l] * w[l]; t++) gy[loff[l] + t] += gcur[t];
    free(gcur);
  }

  for (int l = 0; l < L; l++)
    for (int j = 0; j <= l; j++) {
      free(chain[l][j]);
      free(mid[l][j]);
    }
  for (int r = 0; r <= RN; r++) {
    free(hs[r]);
    free(us[r]);
  }
  free(u1);
  free(gh);
  free(gin);
  free(gdense);
  free(dense);
  free(yq);
  return 0;
}

/* One Adam step (Kingma & Ba) on every parameter; m, v are the moments. */
void orc_adam_step(int64_t n, float* params, const double* grad, double* mom1, double* mom2, const orc_adam* o) {
  const double c1 = 1.0 - pow(o->beta1, o->t), c2 = 1.0 - pow(o->beta2, o->t);
  for (int64_t i = 0; i < n; i++) {
    mom1[i] = o->beta1 * mom1[i] + (1.0 - o->beta1) * grad[i];
    mom2[i] = o->beta2 * mom2[i] + (1.0 - o->beta2) * grad[i] * grad[i];
    params[i] = (float)((double)params[i] - o->lr * (mom1[i] / c1) / (sqrt(mom2[i] / c2) + o->eps));
  }
}

/* The whole iteration: gradient at the current point, then Adam. */
int orc_train_step(const orc_model* m, float* params, const float* noise, const float* image, double* mom1,
                   double* mom2, const orc_adam* o, double* out, double* grad) {
  const int rc = orc_train_grad(m, params, noise, image, out, grad);
  if (rc) return rc;
  orc_adam_step(orc_train_param_count(m), params, grad, mom1, mom2, o);
  return 0;
}
