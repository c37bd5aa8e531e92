/*
 * ccanalysis.c -- plain fp64 CPU oracle of the N-O Cool-chic analysis
 * transform y = f_alpha(x) (NEXT-4; Eq. 3).
 *
 * TEST INFRASTRUCTURE ONLY (same rule as ccoracle.c): shares no code with
 * the CUDA path.
 *
 * Fig. 4 (the architecture) is missing from PAPER.md; the text fixes: L = 7
 * grids, C = 64 features, "a series of L residual blocks progressively
 * downsample the input", "after each downsampling step, a simple 1x1
 * convolution merges the C = 64 features into the l-th latent", ConvNeXt
 * blocks, downsampling blocks whose identity branch is "a stride-2 2x2 average
 * pooling and a 1x1 convolution", "the first residual block does not
 * downsample", "additional residual blocks are stacked after each
 * downsampling".  Readings (A1-A7), after
 * SPEC.md:535-576's reconstruction:
 *   A1 stem: 1x1 conv 3 -> C with bias.
 *   A2 block (stride 1): y = x + W2 ReLU(W1 dw(x) + b1) + b2, dw = depth-wise
 *      7x7 conv with bias, zero padding 3; expansion 4C (no norm, ReLU).
 *   A3 downsampling block: main branch dw 7x7 stride 2 (zero pad 3) -> W1 ->
 *      ReLU -> W2 (+b2); identity branch 2x2 average pool stride 2 (ceil
 *      mode, mean over the in-image samples) -> 1x1 conv C -> C with bias;
 *      y = main + identity.
 *   A4 three blocks per level (level 0: three stride-1 blocks; level l >= 1:
 *      one downsampling block + two stride-1 blocks; ELIC stacks 3).
 *   A5 after level l's blocks: latent l = 1x1 conv C -> 1 with bias (kept
 *      continuous; rounding belongs to the coder).
 *   A6 grid l has ceil(H/2^l) x ceil(W/2^l) samples (== the decoder's dims).
 * Parameter blob (fp32): stem W[C][3], b[C]; per level, per block: dw k[C][7][7],
 * dw b[C], W1[4C][C], b1[4C], W2[C][4C], b2[C], then (downsampling blocks
 * only) Wid[C][C], bid[C]; after the level's blocks: Wm[C], bm.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t H, W, L, C, blocks;  /* blocks per level */
} orc_analysis;

static int64_t blk_params(int C, int down) {
  int64_t n = (int64_t)C * 49 + C + (int64_t)4 * C * C + 4 * C + (int64_t)4 * C * C + C;
  if (down) n += (int64_t)C * C + C;
  return n;
}

int64_t orc_analysis_param_count(const orc_analysis* a) {
  int64_t n = (int64_t)a->C * 3 + a->C;
  for (int l = 0; l < a->L; l++) {
    for (int b = 0; b < a->blocks; b++) n += blk_params(a->C, l > 0 && b == 0);
    n += a->C + 1;
  }
  return n;
}

/* depth-wise 7x7, stride s, zero padding 3: in [C][h][w] -> out [C][ho][wo] */
static void dwconv(const double* in, int C, int h, int w, int s, const float* k, const float* kb, double* out, int ho,
                   int wo, int64_t* macs) {
#pragma omp parallel for  /* independent channels */
  for (int c = 0; c < C; c++)
    for (int y = 0; y < ho; y++)
      for (int x = 0; x < wo; x++) {
        double a = (double)kb[c];
        for (int ky = 0; ky < 7; ky++)
          for (int kx = 0; kx < 7; kx++) {
            const int iy = s * y + ky - 3, ix = s * x + kx - 3;
            if (iy >= 0 && iy < h && ix >= 0 && ix < w) a += (double)k[(c * 7 + ky) * 7 + kx] * in[((int64_t)c * h + iy) * w + ix];
          }
        out[((int64_t)c * ho + y) * wo + x] = a;
      }
  *macs += (int64_t)C * 49 * ho * wo;
}

/* out[n][p] = b[n] + sum_k W[n][k] in[k][p] (+ relu) */
static void pointwise(const double* in, int K, int64_t P, const float* Wt, const float* b, int N, int relu, double* out,
                      int64_t* macs) {
#pragma omp parallel for  /* independent output channels */
  for (int n = 0; n < N; n++)
    for (int64_t p = 0; p < P; p++) {
      double a = (double)b[n];
      for (int k = 0; k < K; k++) a += (double)Wt[(int64_t)n * K + k] * in[(int64_t)k * P + p];
      out[(int64_t)n * P + p] = (relu && a < 0.0) ? 0.0 : a;
    }
  *macs += (int64_t)N * K * P;
}

/* The analysis transform: image [3][H][W] (fp32) -> latents packed level after
 * level (fp64, ceil dims).  macs (optional): multiply count. */
int orc_analysis_forward(const orc_analysis* a, const float* image, const float* w, double* latents, int64_t* macs) {
  const int C = a->C, L = a->L;
  int64_t mc = 0;
  int h = a->H, wd = a->W;
  int64_t P = (int64_t)h * wd;
  double* x = (double*)malloc(sizeof(double) * (size_t)C * P);
  const float* q = w;
  /* A1 stem */
  {
    double* img = (double*)malloc(sizeof(double) * 3 * (size_t)P);
    for (int64_t t = 0; t < 3 * P; t++) img[t] = (double)image[t];
    pointwise(img, 3, P, q, q + C * 3, C, 0, x, &mc);
    q += C * 3 + C;
    free(img);
  }
  int64_t loff = 0;
  for (int l = 0; l < L; l++) {
    for (int b = 0; b < a->blocks; b++) {
      const int down = (l > 0 && b == 0);
      const int ho = down ? (h + 1) / 2 : h, wo = down ? (wd + 1) / 2 : wd;
      const int64_t Po = (int64_t)ho * wo;
      const float* k = q;
      const float* kb = k + C * 49;
      const float* W1 = kb + C;
      const float* b1 = W1 + 4 * C * C;
      const float* W2 = b1 + 4 * C;
      const float* b2 = W2 + 4 * C * C;
      double* t0 = (double*)malloc(sizeof(double) * (size_t)C * Po);
      double* t1 = (double*)malloc(sizeof(double) * (size_t)4 * C * Po);
      double* y = (double*)malloc(sizeof(double) * (size_t)C * Po);
      dwconv(x, C, h, wd, down ? 2 : 1, k, kb, t0, ho, wo, &mc);
      pointwise(t0, C, Po, W1, b1, 4 * C, 1, t1, &mc);
      pointwise(t1, 4 * C, Po, W2, b2, C, 0, y, &mc);
      q = b2 + C;
      if (!down) {
        for (int64_t t = 0; t < (int64_t)C * Po; t++) y[t] += x[t];
      } else {
        /* identity branch: 2x2 average pool (ceil mode, in-image samples) -> 1x1 */
        double* pool = (double*)malloc(sizeof(double) * (size_t)C * Po);
        for (int c = 0; c < C; c++)
          for (int yy = 0; yy < ho; yy++)
            for (int xx = 0; xx < wo; xx++) {
              double s = 0.0;
              int n = 0;
              for (int dy = 0; dy < 2; dy++)
                for (int dx = 0; dx < 2; dx++) {
                  const int iy = 2 * yy + dy, ix = 2 * xx + dx;
                  if (iy < h && ix < wd) {
                    s += x[((int64_t)c * h + iy) * wd + ix];
                    n++;
                  }
                }
              pool[((int64_t)c * ho + yy) * wo + xx] = s / n;
            }
        const float* Wid = q;
        const float* bid = Wid + C * C;
        double* idn = (double*)malloc(sizeof(double) * (size_t)C * Po);
        pointwise(pool, C, Po, Wid, bid, C, 0, idn, &mc);
        for (int64_t t = 0; t < (int64_t)C * Po; t++) y[t] += idn[t];
        q = bid + C;
        free(pool);
        free(idn);
      }
      free(t0);
      free(t1);
      free(x);
      x = y;
      h = ho;
      wd = wo;
      P = Po;
    }
    /* A5 merge C -> 1 */
    {
      const float* Wm = q;
      const float* bm = Wm + C;
      for (int64_t p = 0; p < P; p++) {
        double s = (double)bm[0];
        for (int c = 0; c < C; c++) s += (double)Wm[c] * x[(int64_t)c * P + p];
        latents[loff + p] = s;
      }
      mc += (int64_t)C * P;
      q = bm + 1;
    }
    loff += P;
  }
  free(x);
  if (macs) *macs = mc;
  return (q - w == orc_analysis_param_count(a)) ? 0 : -1;
}
