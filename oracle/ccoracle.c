/*
 * ccoracle.c -- plain fp64 CPU oracle of the Cool-chic RD forward.
 *
 * TEST INFRASTRUCTURE ONLY (see ccoracle.h).  Written from the paper
 * (/root/reference/PAPER.md, "Overfitted image coding at reduced complexity")
 * and the readings in DESIGN.md; no blocking, fusion or reordering beyond the
 * definitions.  Every function cites the passage it follows.
 *
 * Pins (tests/test_oracle_*.py, `-m "not gpu"`): closed-form Laplace bits,
 * telescoping normalisation, closed-form rate of constant latents,
 * torch conv_transpose2d / bilinear / conv2d cross-checks, causality,
 * constant preservation, zero-network closed forms, MAC counters == closed form.
 */
#include "ccoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 1;

void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int orc_get_threads(void) { return g_threads; }

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ---- step 1: dims ("y_l in Z^{H/2^l x W/2^l}"; SPEC.md:135
 *      reads the division as a ceiling for odd sizes) ---------------------- */
int64_t orc_level_dims(const orc_model* m, int32_t* h, int32_t* w) {
  int64_t n = 0;
  for (int l = 0; l < m->L; l++) {
    int64_t d = (int64_t)1 << l;
    h[l] = (int32_t)((m->H + d - 1) / d);
    w[l] = (int32_t)((m->W + d - 1) / d);
    n += (int64_t)h[l] * w[l];
  }
  return n;
}

/* ---- step 5: discrete Laplace bin probability (R = -log2 p_psi;
 *      reading #1: Laplace(mu, b) integrated over [y - 1/2, y + 1/2]) -------- */
static double laplace_cdf(double t, double mu, double b) {
  if (t < mu) return 0.5 * exp((t - mu) / b);
  return 1.0 - 0.5 * exp(-(t - mu) / b);
}

double orc_laplace_prob(double y, double mu, double b) {
  return laplace_cdf(y + 0.5, mu, b) - laplace_cdf(y - 0.5, mu, b);
}

/* reading #3: floor the probability before the log, no renormalisation */
double orc_laplace_bits(double y, double mu, double b, double p_floor) {
  double p = orc_laplace_prob(y, mu, b);
  if (p < p_floor) p = p_floor;
  return -log2(p);
}

/* ---- step 2: causal context ("conditioned on neighbouring
 *      values"; reading #4 template, #5 same grid, 0 outside) -------------- */
void orc_context(const orc_model* m, const int16_t* grid, int32_t h, int32_t w,
                 int32_t i, int32_t j, double* ctx) {
  for (int c = 0; c < m->n_ctx; c++) {
    int ii = i + m->ctx_dy[c], jj = j + m->ctx_dx[c];
    ctx[c] = (ii >= 0 && ii < h && jj >= 0 && jj < w) ? (double)grid[(int64_t)ii * w + jj] : 0.0;
  }
}

/* ---- steps 3-4: ARM MLP f_psi (Table 1 ARM column, caption
 *      315-317 "All layers are followed by a ReLU non linearity except for the
 *      last one of each module", "R stands for residual").  Reading #8:
 *      u = W z + b; u += z on residual layers; z = ReLU(u) except last.
 *      Outputs: mu = z[0], b = exp(clamp(z[1], logscale_min, logscale_max))
 *      (reading #2). ------------------------------------------------------- */
void orc_arm_mlp(const orc_model* m, const double* ctx, const float* arm_w,
                 double* mu, double* b, int64_t* macs) {
  double z[64], u[64];
  int nin = m->arm_widths[0];
  for (int c = 0; c < nin; c++) z[c] = ctx[c];
  const float* p = arm_w;
  for (int k = 0; k < m->arm_n_layers; k++) {
    int in = m->arm_widths[k], out = m->arm_widths[k + 1];
    const float* Wk = p;            /* W_k[out][in] */
    const float* bk = p + in * out; /* b_k[out]     */
    for (int o = 0; o < out; o++) {
      double s = (double)bk[o];
      for (int q = 0; q < in; q++) s += (double)Wk[o * in + q] * z[q];
      u[o] = s;
    }
    if (macs) *macs += (int64_t)in * out;
    if (m->arm_residual[k])
      for (int o = 0; o < out; o++) u[o] += z[o];
    int last = (k == m->arm_n_layers - 1);
    for (int o = 0; o < out; o++) z[o] = (!last && u[o] < 0.0) ? 0.0 : u[o];
    p += in * out + out;
  }
  double s = z[1];
  if (s < m->logscale_min) s = m->logscale_min;
  if (s > m->logscale_max) s = m->logscale_max;
  *mu = z[0];
  *b = exp(s);
}

/* per-row worker shared by orc_rate and orc_rate_rows */
static double rate_row(const orc_model* m, const int16_t* grid, int32_t h, int32_t w, int32_t i,
                       const float* arm_w, double* mu_o, double* b_o, double* bits_o, int64_t* macs) {
  double row = 0.0, ctx[64];
  for (int j = 0; j < w; j++) {
    double mu, b;
    orc_context(m, grid, h, w, i, j, ctx);
    orc_arm_mlp(m, ctx, arm_w, &mu, &b, macs);
    double y = (double)grid[(int64_t)i * w + j];
    double bits = orc_laplace_bits(y, mu, b, m->p_floor);
    if (mu_o) mu_o[j] = mu;
    if (b_o) b_o[j] = b;
    if (bits_o) bits_o[j] = bits;
    row += bits;
  }
  return row;
}

/* ---- step 6 (R of Eq. 1): R = sum over all latents of all grids.
 *      One psi for every grid (reading #6). Rows are summed in a fixed order. */
double orc_rate(const orc_model* m, const int16_t* latents, const float* arm_w,
                double* mu, double* b, double* bits, orc_macs* macs) {
  int32_t h[ORC_MAX_LEVELS], w[ORC_MAX_LEVELS];
  orc_level_dims(m, h, w);
  double total = 0.0;
  int64_t off = 0, mac_total = 0;
  for (int l = 0; l < m->L; l++) {
    const int16_t* grid = latents + off;
    double* rows = (double*)calloc((size_t)h[l], sizeof(double));
    int64_t lmacs = 0;
#pragma omp parallel for schedule(dynamic, 4) num_threads(g_threads) reduction(+ : lmacs)
    for (int i = 0; i < h[l]; i++) {
      int64_t o = off + (int64_t)i * w[l];
      rows[i] = rate_row(m, grid, h[l], w[l], i, arm_w, mu ? mu + o : NULL, b ? b + o : NULL,
                         bits ? bits + o : NULL, &lmacs);
    }
    for (int i = 0; i < h[l]; i++) total += rows[i];
    free(rows);
    mac_total += lmacs;
    off += (int64_t)h[l] * w[l];
  }
  if (macs) macs->arm += mac_total;
  return total;
}

double orc_rate_rows(const orc_model* m, const int16_t* latents, const float* arm_w,
                     int32_t level, int32_t r0, int32_t r1, double* bits) {
  int32_t h[ORC_MAX_LEVELS], w[ORC_MAX_LEVELS];
  orc_level_dims(m, h, w);
  int64_t off = 0;
  for (int l = 0; l < level; l++) off += (int64_t)h[l] * w[l];
  double total = 0.0;
  int64_t macs = 0;
  for (int i = r0; i < r1; i++)
    total += rate_row(m, latents + off, h[level], w[level], i, arm_w, NULL, NULL,
                      bits ? bits + (int64_t)(i - r0) * w[level] : NULL, &macs);
  return total;
}

/* ---- NEXT-3 (decoder: the decoder recovers
 *      the latents one by one, the ARM conditioning each on already decoded
 *      neighbours).  The autoregressive decode of every grid in raster order.
 *      The entropy decoder (range coder) is out of scope: `truth` plays it --
 *      once the ARM has produced (mu, b) for latent (i, j), the decoded value
 *      truth[i][j] is revealed and written to `decoded`.  Contexts are read
 *      from the DECODED grid only; a position not yet decoded is poison:
 *      returns -1 if one is ever read (the template would not be causal), 0
 *      otherwise.  Outputs (optional) per latent, packed like the latents:
 *      mu, b, bits; *rate = their sum (rows in fixed order). -------------- */
int orc_arm_decode(const orc_model* m, const int16_t* truth, const float* arm_w, int16_t* decoded,
                   double* mu, double* b, double* bits, double* rate) {
  int32_t h[ORC_MAX_LEVELS], w[ORC_MAX_LEVELS];
  const int64_t n = orc_level_dims(m, h, w);
  unsigned char* known = (unsigned char*)calloc((size_t)n, 1);
  double total = 0.0, ctx[64];
  int64_t off = 0;
  int bad = 0;
  for (int l = 0; l < m->L && !bad; l++) {
    for (int i = 0; i < h[l] && !bad; i++)
      for (int j = 0; j < w[l]; j++) {
        for (int c = 0; c < m->n_ctx; c++) {
          const int ii = i + m->ctx_dy[c], jj = j + m->ctx_dx[c];
          if (ii >= 0 && ii < h[l] && jj >= 0 && jj < w[l]) {
            const int64_t q = off + (int64_t)ii * w[l] + jj;
            if (!known[q]) bad = 1;
            ctx[c] = (double)decoded[q];
          } else {
            ctx[c] = 0.0;
          }
        }
        if (bad) break;
        double mu_, b_;
        orc_arm_mlp(m, ctx, arm_w, &mu_, &b_, NULL);
        const int64_t q = off + (int64_t)i * w[l] + j;
        const double bt = orc_laplace_bits((double)truth[q], mu_, b_, m->p_floor);
        if (mu) mu[q] = mu_;
        if (b) b[q] = b_;
        if (bits) bits[q] = bt;
        total += bt;
        decoded[q] = truth[q]; /* the entropy decoder's answer */
        known[q] = 1;
      }
    off += (int64_t)h[l] * w[l];
  }
  free(known);
  if (rate) *rate = total;
  return bad ? -1 : 0;
}

/* ---- step 7: one stride-2 transposed convolution along one axis
 *      (Table 1 "1-1-TConv-K", caption "Transpose convolutions use a stride of
 *      2"; readings #11-#13).  Definition of a transposed convolution with
 *      stride 2 and padding P applied to the replicate-extended input
 *      x_ext[i] = g[clamp(i - E, 0, n - 1)], i = 0 .. n + 2E - 1, E = K/4:
 *          out[o] = sum over (i, j) with 2 i + j - P == o of x_ext[i] k[j],
 *      P = K/2 - 1 + 2E, keeping the first m outputs (crop).  Written as the
 *      scatter of each input sample through the kernel. ------------------ */
static void tconv_1d(const double* g, int n, int64_t gs, const float* k, int K,
                     double* out, int mlen, int64_t os, int64_t* macs) {
  int E = K / 4, P = K / 2 - 1 + 2 * E;
  for (int o = 0; o < mlen; o++) out[o * os] = 0.0;
  for (int i = 0; i < n + 2 * E; i++) {
    double xi = g[clampi(i - E, 0, n - 1) * gs];
    for (int j = 0; j < K; j++) {
      int o = 2 * i + j - P;
      if (o >= 0 && o < mlen) {
        out[o * os] += xi * (double)k[j];
        (*macs)++;
      }
    }
  }
}

/* ---- step 7 (Table 1 exact architectures, NEXT-1): one stride-2 transposed
 *      convolution with a non-separable K x K kernel (Table 1 "1-1-TConv-4" /
 *      "TConv-8": 16 / 64 parameters), the 2-D form of
 *      tconv_1d's definition on the input replicate-extended along both axes
 *      (x_ext[i][i'] = g[clamp(i - E)][clamp(i' - E)]):
 *          out[o][o'] = sum over (i, a, i', b) with 2 i + a - P == o and
 *                       2 i' + b - P == o' of x_ext[i][i'] k2[a][b],
 *      cropped to (mh x mw).  Scatter of each extended input sample. ------ */
static void tconv_2d(const double* g, int n, int nw, const float* k2, int K, double* out, int mh, int mw,
                     int64_t* macs) {
  int E = K / 4, P = K / 2 - 1 + 2 * E;
  for (int64_t t = 0; t < (int64_t)mh * mw; t++) out[t] = 0.0;
  int64_t mc = 0;
  for (int i = 0; i < n + 2 * E; i++)
    for (int i2 = 0; i2 < nw + 2 * E; i2++) {
      double xi = g[(int64_t)clampi(i - E, 0, n - 1) * nw + clampi(i2 - E, 0, nw - 1)];
      for (int a = 0; a < K; a++) {
        int o = 2 * i + a - P;
        if (o < 0 || o >= mh) continue;
        for (int b = 0; b < K; b++) {
          int o2 = 2 * i2 + b - P;
          if (o2 >= 0 && o2 < mw) {
            out[(int64_t)o * mw + o2] += xi * (double)k2[a * K + b];
            mc++;
          }
        }
      }
    }
  *macs += mc;
}

/* ---- step 7: upsampling f_upsilon ("The linear upsampling
 *      ... upsample the latents to a dense representation").  Channel 0 is
 *      y_0; grid l >= 1 goes through l successive x2 steps with the shared
 *      separable filter k (x) k (BASELINE.json configs[0]), each step a
 *      transposed conv along x to width w_j then along y to height h_j
 *      (reading #14), j = l-1 .. 0. ----------------------------------------- */
void orc_upsample(const orc_model* m, const int16_t* latents, const float* up_w,
                  double* dense, orc_macs* macs) {
  int32_t h[ORC_MAX_LEVELS], w[ORC_MAX_LEVELS];
  orc_level_dims(m, h, w);
  const int64_t P = (int64_t)m->H * m->W;
  int64_t off = 0, up_macs = 0;
  for (int l = 0; l < m->L; l++) {
    /* g = y_l as doubles */
    double* g = (double*)malloc(sizeof(double) * (size_t)h[l] * w[l]);
    for (int64_t t = 0; t < (int64_t)h[l] * w[l]; t++) g[t] = (double)latents[off + t];
    int gh = h[l], gw = w[l];
    for (int j = l - 1; j >= 0; j--) {
      if (m->up_2d) { /* Table 1 2-D TConv-K: (gh x gw) -> (h_j x w_j) in one step */
        double* t2 = (double*)malloc(sizeof(double) * (size_t)h[j] * w[j]);
        tconv_2d(g, gh, gw, up_w, m->up_taps, t2, h[j], w[j], &up_macs);
        free(g);
        g = t2;
        gh = h[j];
        gw = w[j];
        continue;
      }
      /* along x: (gh x gw) -> (gh x w_j) */
      double* t1 = (double*)malloc(sizeof(double) * (size_t)gh * w[j]);
      int64_t mx = 0;
#pragma omp parallel for num_threads(g_threads) reduction(+ : mx)
      for (int r = 0; r < gh; r++)
        tconv_1d(g + (int64_t)r * gw, gw, 1, up_w, m->up_taps, t1 + (int64_t)r * w[j], w[j], 1, &mx);
      /* along y: (gh x w_j) -> (h_j x w_j) */
      double* t2 = (double*)malloc(sizeof(double) * (size_t)h[j] * w[j]);
      int64_t my = 0;
#pragma omp parallel for num_threads(g_threads) reduction(+ : my)
      for (int c = 0; c < w[j]; c++)
        tconv_1d(t1 + c, gh, w[j], up_w, m->up_taps, t2 + c, h[j], w[j], &my);
      up_macs += mx + my;
      free(t1);
      free(g);
      g = t2;
      gh = h[j];
      gw = w[j];
    }
    memcpy(dense + (int64_t)l * P, g, sizeof(double) * (size_t)P);
    free(g);
    off += (int64_t)h[l] * w[l];
  }
  if (macs) macs->up += up_macs;
}

/* ---- steps 8-9: synthesis f_theta (Table 1 synthesis column,
 *      "7-40-Conv-1, 40-3-Conv-1, 3-3-ConvR-3, 3-3-ConvR-3"; caption: ReLU after
 *      every layer but the module's last; readings #9, #15).  1x1 layers per
 *      pixel: v = ReLU(A v + a).  Residual 3x3 layers on replicate-padded input
 *      (cross-correlation G[co][ci][ky][kx]):
 *          v'_co = v_co + g_co + sum G[co][ci][ky][kx] v_ci(clamp(y+ky-1), clamp(x+kx-1))
 *      then ReLU except after the last layer.  No output clamp (reading #16). */
void orc_synthesis(const orc_model* m, const double* dense, const float* syn_w,
                   double* x_hat, double* h_1x1, orc_macs* macs) {
  const int H = m->H, W = m->W;
  const int64_t P = (int64_t)H * W;
  const int n1 = m->syn_n_1x1, R = m->syn_n_res;
  const int cout = m->syn_widths[n1];
  double* v = (double*)malloc(sizeof(double) * (size_t)cout * P);
  int64_t syn_macs = 0;
  /* 1x1 stack */
#pragma omp parallel for num_threads(g_threads) reduction(+ : syn_macs)
  for (int y = 0; y < H; y++) {
    double a[64], b[64];
    for (int x = 0; x < W; x++) {
      int64_t px = (int64_t)y * W + x;
      int in = m->syn_widths[0];
      for (int c = 0; c < in; c++) a[c] = dense[c * P + px];
      const float* p = syn_w;
      for (int k = 0; k < n1; k++) {
        in = m->syn_widths[k];
        int out = m->syn_widths[k + 1];
        const float* A = p;
        const float* bias = p + in * out;
        for (int o = 0; o < out; o++) {
          double s = (double)bias[o];
          for (int q = 0; q < in; q++) s += (double)A[o * in + q] * a[q];
          b[o] = s;
        }
        syn_macs += (int64_t)in * out;
        int last = (k == n1 - 1) && (R == 0);
        for (int o = 0; o < out; o++) a[o] = (!last && b[o] < 0.0) ? 0.0 : b[o];
        p += in * out + out;
      }
      for (int o = 0; o < cout; o++) v[o * P + px] = a[o];
    }
  }
  if (h_1x1) memcpy(h_1x1, v, sizeof(double) * (size_t)cout * P);
  /* residual 3x3 stack */
  const float* p = syn_w;
  for (int k = 0; k < n1; k++) p += m->syn_widths[k] * m->syn_widths[k + 1] + m->syn_widths[k + 1];
  double* nv = (double*)malloc(sizeof(double) * (size_t)3 * P);
  for (int r = 0; r < R; r++) {
    const float* G = p;          /* [3][3][3][3] */
    const float* gb = p + 81;    /* [3]          */
    int last = (r == R - 1);
#pragma omp parallel for num_threads(g_threads) reduction(+ : syn_macs)
    for (int y = 0; y < H; y++) {
      for (int x = 0; x < W; x++) {
        for (int co = 0; co < 3; co++) {
          double s = v[co * P + (int64_t)y * W + x] + (double)gb[co];
          for (int ci = 0; ci < 3; ci++)
            for (int ky = 0; ky < 3; ky++)
              for (int kx = 0; kx < 3; kx++) {
                int yy = clampi(y + ky - 1, 0, H - 1), xx = clampi(x + kx - 1, 0, W - 1);
                s += (double)G[((co * 3 + ci) * 3 + ky) * 3 + kx] * v[ci * P + (int64_t)yy * W + xx];
              }
          if (!last && s < 0.0) s = 0.0;
          nv[co * P + (int64_t)y * W + x] = s;
        }
        syn_macs += 81;
      }
    }
    memcpy(v, nv, sizeof(double) * (size_t)3 * P);
    p += 84;
  }
  memcpy(x_hat, v, sizeof(double) * (size_t)3 * P);
  free(nv);
  free(v);
  if (macs) macs->syn += syn_macs;
}

/* ---- Eq. 1: D = MSE over 3HW ("here the mean-squared
 *      error", reading #17); cost = MSE + lambda R / (H W) (reading #18). ---- */
int orc_rd_forward(const orc_model* m, const int16_t* latents, const float* arm_w,
                   const float* up_w, const float* syn_w, const float* image,
                   double* out, double* x_hat, double* dense, orc_macs* macs) {
  if (m->L < 1 || m->L > ORC_MAX_LEVELS || m->H < 1 || m->W < 1) return -1;
  const int64_t P = (int64_t)m->H * m->W;
  double* d = dense ? dense : (double*)malloc(sizeof(double) * (size_t)m->L * P);
  double* xh = x_hat ? x_hat : (double*)malloc(sizeof(double) * (size_t)3 * P);
  double R = orc_rate(m, latents, arm_w, NULL, NULL, NULL, macs);
  orc_upsample(m, latents, up_w, d, macs);
  orc_synthesis(m, d, syn_w, xh, NULL, macs);
  double* rows = (double*)calloc((size_t)m->H, sizeof(double));
#pragma omp parallel for num_threads(g_threads)
  for (int y = 0; y < m->H; y++) {
    double s = 0.0;
    for (int c = 0; c < 3; c++)
      for (int x = 0; x < m->W; x++) {
        int64_t t = c * P + (int64_t)y * m->W + x;
        double e = (double)image[t] - xh[t];
        s += e * e;
      }
    rows[y] = s;
  }
  double sse = 0.0;
  for (int y = 0; y < m->H; y++) sse += rows[y];
  free(rows);
  double mse = sse / (3.0 * (double)P);
  out[0] = R;
  out[1] = sse;
  out[2] = mse;
  out[3] = mse + m->lambda * R / (double)P;
  if (!dense) free(d);
  if (!x_hat) free(xh);
  return 0;
}

/* ---- decoder output (NEXT-3): clamp to [0,1], 8-bit = 255 x
 *      rounded to nearest, ties to even (reading N3),
 *      interleaved RGB. ------------------------------------------------------ */
void orc_decode_u8(const orc_model* m, const double* x_hat, uint8_t* out) {
  const int64_t P = (int64_t)m->H * m->W;
  for (int64_t p = 0; p < P; p++)
    for (int c = 0; c < 3; c++) {
      double v = x_hat[(int64_t)c * P + p];
      v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
      out[p * 3 + c] = (uint8_t)rint(255.0 * v);
    }
}
