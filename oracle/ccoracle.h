/*
 * ccoracle.h -- plain fp64 CPU oracle of the Cool-chic rate-distortion forward.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no
 * code, header, table or constant with the CUDA product path
 * (paper_2403_11651_b200/, include/ccrd.h) and neither includes the other.
 *
 * What it computes (Eq. 1):
 *     cost = D(x, x_hat) + lambda * R(y_hat) / (H W)
 *     D    = mean-squared error over the 3 H W RGB values
 *     R    = sum over every latent of -log2 p_psi(y_hat)          (rate, bits)
 *     x_hat = f_theta(f_upsilon(y_hat))
 * with the readings listed in DESIGN.md ("Readings of the paper").
 *
 * Everything is evaluated in double precision from the fp32 parameters and the
 * int16 latents, with plain loops (OpenMP over independent rows only).
 */
#ifndef CCORACLE_H
#define CCORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_LEVELS 12
#define ORC_MAX_LAYERS 8

typedef struct {
  int32_t H, W, L;                       /* image size, number of latent grids          */
  int32_t n_ctx;                         /* number of causal context offsets            */
  int32_t ctx_dy[32], ctx_dx[32];        /* offsets (dy, dx), in order                  */
  int32_t arm_n_layers;                  /* number of ARM linear layers                 */
  int32_t arm_widths[ORC_MAX_LAYERS + 1];/* [n_ctx, hidden..., 2]                       */
  int32_t arm_residual[ORC_MAX_LAYERS];  /* 1 = "LinR" layer (u += z)                   */
  int32_t up_taps;                       /* K: 4 or 8                                   */
  int32_t up_2d;                         /* 0: separable k (x) k, up_w = k[K] (BASELINE)  */
                                         /* 1: 2-D K x K kernel, up_w = k2[K][K] row-major */
                                         /*    (Table 1 "TConv-K", 16 / 64 params; NEXT-1) */
  int32_t syn_n_1x1;                     /* number of 1x1 layers                        */
  int32_t syn_widths[ORC_MAX_LAYERS + 1];/* [L, C_h..., 3]                              */
  int32_t syn_n_res;                     /* residual 3x3 3->3 layers                    */
  double logscale_min, logscale_max;     /* clamp of the log-scale output               */
  double p_floor;                        /* probability floor before -log2              */
  double lambda;                         /* Lagrange multiplier (Eq. 1)                 */
} orc_model;

typedef struct { int64_t arm, up, syn; } orc_macs;

/* Grid sizes ceil(H/2^l) x ceil(W/2^l).  Returns N_lat. */
int64_t orc_level_dims(const orc_model* m, int32_t* h, int32_t* w);

/* Discrete Laplace bin probability P = F(y+1/2) - F(y-1/2) and its -log2 with
 * the floor (R term of Eq. 1; reading #1, #3). */
double orc_laplace_prob(double y, double mu, double b);
double orc_laplace_bits(double y, double mu, double b, double p_floor);

/* ARM forward for one context vector -> (mu, b) (Table 1 ARM). */
void orc_arm_mlp(const orc_model* m, const double* ctx, const float* arm_w,
                 double* mu, double* b, int64_t* macs);

/* Context of latent (i, j) of one grid (h x w), 0 outside (reading #4, #5). */
void orc_context(const orc_model* m, const int16_t* grid, int32_t h, int32_t w,
                 int32_t i, int32_t j, double* ctx);

/* Rate over every latent of every grid.  Optional per-latent outputs (packed
 * like the latents): mu, b, bits.  Returns R in bits. */
double orc_rate(const orc_model* m, const int16_t* latents, const float* arm_w,
                double* mu, double* b, double* bits, orc_macs* macs);

/* Upsampling f_upsilon: dense [L][H][W] (reading #11-#14;
 * up_2d: Table 1's non-separable 2-D TConv-K). */
void orc_upsample(const orc_model* m, const int16_t* latents, const float* up_w,
                  double* dense, orc_macs* macs);

/* Synthesis f_theta: dense [L][H][W] -> x_hat [3][H][W]  (Table 1 synthesis).
 * Optional h_1x1: output of the 1x1 stack [3][H][W]. */
void orc_synthesis(const orc_model* m, const double* dense, const float* syn_w,
                   double* x_hat, double* h_1x1, orc_macs* macs);

/* The whole RD forward.  out[4] = {rate_bits, sse, mse, cost}.
 * x_hat (optional) [3][H][W]; dense (optional) [L][H][W]. */
int orc_rd_forward(const orc_model* m, const int16_t* latents, const float* arm_w,
                   const float* up_w, const float* syn_w, const float* image,
                   double* out, double* x_hat, double* dense, orc_macs* macs);

/* Decoder output (NEXT-3; "final output clamped to [0,1]";
 * 8-bit RGB, pixel = 255 x): out[(y W + x) 3 + c] =
 * rint(255 clamp(x_hat[c][y][x], 0, 1)) (round half to even; reading N3). */
/* NEXT-3: autoregressive decode in raster order (entropy decoder played by
 * `truth`); 0, or -1 if a context read an undecoded latent. */
int orc_arm_decode(const orc_model* m, const int16_t* truth, const float* arm_w, int16_t* decoded,
                   double* mu, double* b, double* bits, double* rate);
void orc_decode_u8(const orc_model* m, const double* x_hat, uint8_t* out);

/* Rate and per-latent outputs for the latents of rows [r0, r1) of level l only
 * (bounded samples at full size; same arithmetic as orc_rate). */
double orc_rate_rows(const orc_model* m, const int16_t* latents, const float* arm_w,
                     int32_t level, int32_t r0, int32_t r1, double* bits);

void orc_set_threads(int n);
int orc_get_threads(void);

#ifdef __cplusplus
}
#endif
#endif
