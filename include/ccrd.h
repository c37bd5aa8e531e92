/*
 * ccrd.h -- C ABI of the B200-native Cool-chic rate-distortion forward.
 *
 * Computes, for each image, Eq. 1 (lines 117-124):
 *
 *     cost = D(x, x_hat) + lambda * R(y_hat) / (H W)
 *     R(y_hat) = sum over every latent of every grid of -log2 p_psi(y_hat)
 *     x_hat    = f_theta(f_upsilon(y_hat))       (Table 1)
 *     D        = mean-squared error over the 3 H W values ("here the
 *                mean-squared error")
 *
 * with the readings of DESIGN.md ("Readings of the paper"): Laplace(mu, b)
 * integrated over the unit bin, b = exp(clamp(out1, logscale_min,
 * logscale_max)), probability floored at p_floor before -log2, shared separable
 * stride-2 transposed-conv upsampling with replicate padding, synthesis 1x1
 * layers then residual 3x3 layers with replicate padding, ReLU after every layer
 * except the last of each module (Table 1 caption).
 *
 * Every step runs in CUDA kernels compiled for sm_100a.  There is no CPU
 * fallback: if no CUDA device is present every compute entry returns CC_ECUDA.
 *
 * Conventions
 *   - All functions return 0 (CC_OK) or a negative CC_E* code; nothing aborts,
 *     prints or throws across the ABI.  cc_last_error() gives a thread-local
 *     human-readable detail of the last failure on the calling thread.
 *   - The caller owns every buffer.  The library allocates nothing on the
 *     device, keeps no pointer after return, and is reentrant.  Device buffers
 *     must stay alive until the work queued on `stream` completes (CUDA stream
 *     semantics).  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream).
 *   - Weight blobs are HOST pointers (<= 8 KB per image); they are packed into
 *     kernel parameters at call time, so no device->host synchronisation is
 *     needed and the host memory may be reused as soon as the call returns.
 *   - Latents: int16, device, levels 0..L-1 packed one after the other, each
 *     row-major with h_l = ceil(H / 2^l) rows and w_l = ceil(W / 2^l) columns
 *     (PAPER.md:103-105 writes H/2^l; SPEC.md:135 gives the ceiling).
 *   - Images and x_hat: fp32, device, planar [3][H][W].
 */
#ifndef CCRD_H
#define CCRD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_OK 0
#define CC_EINVAL (-1)      /* null pointer, bad size, inconsistent widths, non-causal offset */
#define CC_ENOTSUP (-2)     /* valid per the paper but not compiled in (see cc_model_desc)     */
#define CC_EWORKSPACE (-3)  /* workspace missing or smaller than cc_workspace_bytes()         */
#define CC_ECUDA (-4)       /* CUDA launch / runtime error (detail in cc_last_error)          */
#define CC_ENONFINITE (-5)  /* non-finite result (opt-in check)                                */

#define CC_MAX_LEVELS 12
#define CC_MAX_CTX 32
#define CC_MAX_LAYERS 8

/* Model descriptor (by value; validated on every call).
 *
 * ARM f_psi (Table 1 ARM column): arm_widths = [n_ctx,
 *   hidden..., 2]; layer k is "LinR" (u = W z + b + z) when bit k of
 *   arm_residual_mask is set (requires in == out and k not last); ReLU after
 *   every layer except the last; outputs (mu, log-scale).
 *   Compiled: n_ctx in {8, 16, 24}, 1..3 hidden layers of equal width in
 *   {8, 16, 24, 32}.
 * Context: n_ctx strictly causal offsets (dy < 0, or dy == 0 and dx < 0) with
 *   -3 <= dy <= 0 and |dx| <= 4; neighbours outside the grid read 0.
 * Upsampling f_upsilon (Table 1 "1-1-TConv-K"): one shared
 *   stride-2 transposed conv, K = up_taps in {4, 8}, no bias: separable
 *   k (x) k (up_2d = 0, BASELINE.json) or a non-separable K x K kernel
 *   (up_2d = 1, Table 1's exact architectures; not available for strips).
 * Synthesis f_theta (Table 1 synthesis column): syn_widths = [L, C_h, 3]
 *   (syn_n_1x1 = 2) then syn_n_res residual 3x3 3->3 layers.
 *   Compiled: L in 1..8 with C_h in {8, 16, 24, 32, 40, 48}; syn_n_res in 0..3.
 */
typedef struct {
  int32_t H, W, L;                     /* image size; 1 <= L <= 12                     */
  int32_t n_ctx;                       /* context size C                               */
  int8_t ctx_dy[CC_MAX_CTX];           /* offsets, in the order they feed layer 0      */
  int8_t ctx_dx[CC_MAX_CTX];
  int32_t arm_n_layers;                /* number of ARM linear layers                  */
  int32_t arm_widths[CC_MAX_LAYERS + 1];
  uint32_t arm_residual_mask;
  int32_t up_taps;                     /* K                                            */
  int32_t up_2d;                       /* 0: separable k (x) k, up_w = k[K] (BASELINE)   */
                                       /* 1: 2-D K x K kernel, up_w = k2[K][K] row-major */
                                       /*    (Table 1 "TConv-K", 16 / 64 params)          */
  int32_t syn_n_1x1;                   /* number of 1x1 layers (2 supported)           */
  int32_t syn_widths[CC_MAX_LAYERS + 1];
  int32_t syn_n_res;                   /* residual 3x3 layers                          */
  float logscale_min, logscale_max;    /* clamp of the ARM log-scale output            */
  float p_floor;                       /* probability floor before -log2               */
  double lambda;                       /* Lagrange multiplier of Eq. 1                 */
  int32_t image_u8;                    /* 0: images are fp32 planar [3][H][W] in [0,1]; */
                                       /* 1: uint8 planar [3][H][W], x = v / 255 (the  */
                                       /*    paper's 8-bit RGB sources; fp32 IEEE       */
                                       /*    division).  x_hat stays fp32.  Applies to  */
                                       /*    every `image` argument taking this desc    */
                                       /*    except cc_train_step / cc_synthesize       */
                                       /*    (fp32 only: CC_ENOTSUP).                   */
  int32_t latents_i8;                  /* cc_rd_forward_host only: 1 = io.latents are  */
                                       /*    int8 host arrays (every value in           */
                                       /*    [-128, 127]; the caller's guarantee),      */
                                       /*    uploaded at 1 byte per latent and widened  */
                                       /*    to int16 on the device.  Device entry      */
                                       /*    points need 0 (else CC_ENOTSUP).            */
} cc_model_desc;

/* Per-image result, written to DEVICE memory (so it can be all-reduced
 * without a host synchronisation). */
typedef struct {
  double rate_bits;  /* R, bits                          */
  double sse;        /* sum over 3HW of (x - x_hat)^2    */
  double mse;        /* sse / (3 H W)                    */
  double cost;       /* mse + lambda * rate_bits / (H W) */
} cc_rd_result;

/* One image.  Blob layouts (fp32, row-major):
 *   arm_w: per layer k: W_k[out][in], then b_k[out].
 *   up_w : k[K] (separable), or k2[a][b] row-major (up_2d; a = vertical tap,
 *          b = horizontal): out[2q+r][2p+s] = sum_{t,u} k2[2t+1-r][2u+1-s]
 *          g[q+r+K/4-1-t][p+s+K/4-1-u] on the replicate-extended grid.
 *   syn_w: per 1x1 layer: A_m[out][in], a_m[out]; then per residual 3x3 layer
 *          G_r[co][ci][ky][kx] (cross-correlation, replicate padding), g_r[3]. */
typedef struct {
  const int16_t* latents;  /* device, packed pyramid                     */
  const float* arm_w;      /* HOST                                        */
  const float* up_w;       /* HOST                                        */
  const float* syn_w;      /* HOST                                        */
  const float* image;      /* device [3][H][W] (may be NULL: sse = 0)     */
  float* x_hat;            /* device [3][H][W] or NULL (not written)      */
} cc_image_io;

/* Workspace (device) needed by cc_rd_forward for n_img images; 0 on error. */
size_t cc_workspace_bytes(const cc_model_desc* desc, int32_t n_img);

/* The full RD forward for n_img images that share one descriptor (each image
 * has its own latents, weights and image).  results: DEVICE array [n_img].
 * Work is queued on `stream`; the call does not synchronise. */
int cc_rd_forward(const cc_model_desc* desc, const cc_image_io* io, int32_t n_img,
                  cc_rd_result* results, void* workspace, size_t workspace_bytes,
                  void* stream);

/* Same computation from HOST buffers (end-to-end path): io[i].latents,
 * io[i].image and io[i].x_hat (optional) are host pointers (pinned memory
 * recommended); results is a HOST array [n_img].  The call copies inputs to
 * the device workspace (double-buffered, overlapped with compute), runs the
 * forward, copies the results (and x_hat if requested) back and synchronises
 * `stream` before returning.  Workspace: cc_workspace_bytes_host(). */
size_t cc_workspace_bytes_host(const cc_model_desc* desc, int32_t n_img);
int cc_rd_forward_host(const cc_model_desc* desc, const cc_image_io* io, int32_t n_img,
                       cc_rd_result* results, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ------------------------------------------------------------------ strips
 * One image split into horizontal strips of pixel rows (the
 * BASELINE.json configs[4] single 4320x7680 image across 1/2/4/8 GPUs).  A
 * strip owns pixel rows [r0, r1) and, at every level l, latent rows
 * own_lo[l] = ceil(r0 / 2^l) .. own_hi[l] = ceil(r1 / 2^l) (so the strips of a
 * partition own every latent exactly once).  Its latent BUFFER holds global rows
 * [lo[l], hi[l]) of each grid: the owned rows plus a halo copied from the
 * neighbouring strips (the halo exchange).  cc_strip_window() computes the
 * smallest window from the receptive field of the forward:
 *   level 0: rows r0 - R .. r1 + R (R residual 3x3 layers);
 *   level j+1: rows floor(a/2) - K/4 .. floor(b/2) + K/4 for level j's rows a..b
 *              (one x2 stride-2 transposed-conv step, reading #12);
 *   and, for the ARM, the context rows above the owned rows
 *   (max -dy of the template);
 * clipped to the grid.  Inside it the kernels compute exactly what the full
 * image computes for the owned rows (replicate padding only at true image
 * borders), so the strips' x_hat are bit-identical to the full image's rows.
 */
typedef struct {
  int32_t r0, r1;                      /* owned pixel rows; 0 <= r0 < r1 <= H, r0 even */
  int32_t own_lo[CC_MAX_LEVELS];       /* owned latent rows of grid l                   */
  int32_t own_hi[CC_MAX_LEVELS];
  int32_t lo[CC_MAX_LEVELS];           /* rows present in the latent buffer (window)    */
  int32_t hi[CC_MAX_LEVELS];
} cc_strip;

/* Fills *out with the owned rows and the minimal window of pixel rows
 * [r0, r1) (host only; no device).  CC_EINVAL on a bad descriptor or range
 * (r0 odd, r0 >= r1, r1 > H). */
int cc_strip_window(const cc_model_desc* desc, int32_t r0, int32_t r1, cc_strip* out);

/* Number of int16 latents in a strip's window buffer: sum_l (hi_l - lo_l) w_l;
 * grid l starts at sum_{m<l} (hi_m - lo_m) w_m.  -1 on error. */
int64_t cc_strip_latent_count(const cc_model_desc* desc, const cc_strip* strip);

/* Workspace (device) of cc_rd_forward_strip; 0 on error. */
size_t cc_workspace_bytes_strip(const cc_model_desc* desc, const cc_strip* strip);

/* The RD forward of one strip.  io->latents: DEVICE window buffer (above);
 * io->image / io->x_hat: DEVICE [3][r1 - r0][W] (strip rows only; image may be
 * NULL, x_hat may be NULL).  *result (DEVICE) receives the strip's ADDITIVE
 * share: rate_bits over the owned latents, sse over the owned pixels,
 * mse = sse / (3 H W) and cost = mse + lambda rate_bits / (H W) with the FULL
 * image's H W -- summing the four fields over the strips of a partition (one
 * all-reduce) gives the full image's result.  The window must contain the one
 * cc_strip_window() returns for (r0, r1) (CC_EINVAL otherwise). */
int cc_rd_forward_strip(const cc_model_desc* desc, const cc_strip* strip, const cc_image_io* io,
                        cc_rd_result* result, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------- training (NEXT-2)
 * ONE encoder training iteration (Eq. 1 "simultaneously
 * learning the latent and the different neural networks"
 * "one forward pass and one backward pass"; SPEC.md:476-479 Adam on every
 * parameter): forward on the proxy latents y_hat = y + u, the exact gradient
 * of J = MSE + lambda R / (H W) wrt every parameter, then one Adam step.
 * Readings (T1-T3): u ~ U(-1/2, 1/2) is an INPUT (`noise`, packed
 * like the latents), its gradient passes unchanged to y; ReLU'(0) = 0; no
 * gradient through the log-scale clamp outside (logscale_min, logscale_max) or
 * through the probability floor.  Separable upsampling only (up_2d = 0).
 *
 * params: DEVICE fp32 [cc_train_param_count()] = [ y (N_lat, packed like the
 * latents) | arm_w | up_w | syn_w ] (blob layouts as in cc_image_io), updated
 * in place.  adam_m, adam_v: DEVICE fp32, same length (zero before step t = 1).
 * grad: DEVICE fp32, same length: receives the gradient at the input point.
 * opt: HOST; NULL = gradient only (no update).  result: DEVICE, the cost of
 * this forward (rate_bits, sse, mse, cost).  image: DEVICE [3][H][W].
 * Concurrency: weights are staged into one of 4 per-device __constant__ banks
 * per call.  Calls may run concurrently on different streams AND from
 * different host threads: a bank is held exclusively from the start of a call
 * to the end of its enqueue, a stream taking over a bank waits (on the GPU)
 * for the previous owner's last step, and a caller finding all 4 banks held
 * blocks on the host until one is released.  Results are bit-identical to
 * the same steps run one at a time.  Shapes with H W >= 2^31 are CC_ENOTSUP
 * (32-bit offsets inside a plane). */
typedef struct {
  float lr, beta1, beta2, eps;
  int32_t t;  /* Adam step number, >= 1 */
} cc_adam;
int64_t cc_train_param_count(const cc_model_desc* desc);   /* -1 on error */
size_t cc_train_workspace_bytes(const cc_model_desc* desc);
int cc_train_step(const cc_model_desc* desc, float* params, const float* noise, const float* image,
                  float* adam_m, float* adam_v, const cc_adam* opt, cc_rd_result* result, float* grad,
                  void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------ decode (NEXT-3)
 * The decoder's data-parallel output stage ("upsample the
 * latents to a dense representation and synthesize the decoded image";
 * SPEC.md:309-312 "final output clamped to [0,1]"; SPEC.md:332, 624-625 8-bit
 * output, pixel = 255 x): from the decoded latents (DEVICE, packed pyramid) to
 * out_rgb8 (DEVICE, interleaved [H][W][3] uint8) = rint(255 clamp(x_hat, 0, 1))
 * (ties to even, reading N3).  The autoregressive entropy decoding of the
 * latents themselves is sequential and out of scope.  Same kernels as
 * cc_rd_forward without the ARM and the distortion.  Workspace:
 * cc_workspace_bytes(desc, 1). */
int cc_decode(const cc_model_desc* desc, const int16_t* latents, const float* up_w, const float* syn_w,
              uint8_t* out_rgb8, void* workspace, size_t workspace_bytes, void* stream);

/* --------------------------------------------- N-O analysis (NEXT-4)
 * The non-overfitted Cool-chic analysis transform y_hat = f_alpha(x)
 * (Eq. 3): C-channel ConvNeXt-style blocks (depth-wise 7x7,
 * point-wise C -> 4C -> C with ReLU, residual), `blocks` per level, a stride-2
 * downsampling block opening each level l >= 1 (identity branch: 2x2 average
 * pooling + 1x1 conv), a 1x1 C -> 1 merge giving latent grid l after each
 * level.  Fig. 4 is missing from the paper: every structural choice is a
 * reading (A1-A7).  Weight blob: stem W[C][3], b[C]; per level, per
 * block: dw k[C][7][7], dw b[C], W1[4C][C], b1[4C], W2[C][4C], b2[C], then
 * (downsampling blocks only) Wid[C][C], bid[C]; per level: Wm[C], bm.
 * N images share the one network (N-O: the same f_alpha for every image,
 * PAPER.md:426-429).  image: DEVICE [N][3][H][W] fp32; weights: DEVICE blob;
 * latents: DEVICE fp32 [N][n_lat], each image's grids packed level after
 * level (the decoder's ceil dims), continuous (rounding belongs to the coder).
 * C: a multiple of 4 in [4, 512].  tf32 selects the arithmetic of the
 * point-wise layers: 0 = fp32 (cuBLASLt GEMMs, CUBLAS_COMPUTE_32F); 1 = TF32
 * on the tcgen05 tensor cores, each block ONE fused kernel when C == 64
 * (depth-wise conv, both point-wise layers with the hidden layer kept in TMEM,
 * residual and merge; analysis_tc.cu), else cuBLASLt TF32; 2 = TF32 cuBLASLt
 * GEMMs unfused (the library baseline); 3 = as 1 with FP16 tensor-core
 * operands (the same 10-bit mantissa as TF32, 5-bit exponent: |values| <
 * 65504): stride-1 blocks with a TMA-staged depth-wise stage,
 * downsampling blocks warp-specialised with the stride-2 depth-wise + pool
 * read from global memory -- the fast path.  Operands of the TF32 /
 * FP16 products are rounded to 10-bit mantissas, accumulation is fp32. */
typedef struct {
  int32_t H, W, L, C, blocks, tf32;
  int32_t N; /* images per call, >= 1 */
} cc_analysis_desc;
int64_t cc_analysis_param_count(const cc_analysis_desc* a);     /* -1 on error */
size_t cc_analysis_workspace_bytes(const cc_analysis_desc* a);  /* 0 on error  */
int cc_analysis_forward(const cc_analysis_desc* a, const float* image, const float* weights, float* latents,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------ NEXT-3: ARM decode
 * The decoder's autoregressive ARM (the latents
 * are decoded one by one, the ARM conditioning each on already decoded
 * neighbours) as a wavefront over the anti-diagonals t = a i + j of every
 * grid, a = 1 + max over the template's dy < 0 of floor(dx / -dy) (so every
 * context of (i, j) lies on an earlier t); all images and grids at once.  The
 * entropy decoder (range coder) is out of scope: it is played by
 * io[i].latents (DEVICE int16, packed like the latents) -- a latent's value
 * is revealed only after its (mu, b) were computed from the latents decoded
 * before it; contexts are read from the decoded values only, and a read of a
 * not-yet-decoded latent is counted in *poison_reads.  io[i].arm_w: HOST
 * blob; the other io fields are ignored.  Outputs: decoded[i] (DEVICE int16,
 * packed), rate (DEVICE double [n_img], sum of -log2 P per image), optional
 * per-latent mu / scale / bits (host arrays of DEVICE pointers, or NULL),
 * poison_reads (DEVICE int32 [1] or NULL; accumulated, the caller zeroes it).
 * Per-latent (mu, scale, bits) are bit-identical to cc_arm_rate's.  Latent
 * values must not be -32768 (the undecoded marker).  Test hook: env
 * CCRD_DEC_SKEW overrides a (a too small skew must produce poison reads). */
size_t cc_arm_decode_workspace_bytes(const cc_model_desc* desc, int32_t n_img); /* 0 on error */
int cc_arm_decode(const cc_model_desc* desc, const cc_image_io* io, int32_t n_img, int16_t* const* decoded,
                  double* rate, float* const* mu, float* const* scale, float* const* bits, int32_t* poison_reads,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Stage entry: ARM rate only (PAPER.md:120 R term).  rate: DEVICE double [1].
 * Optional DEVICE float arrays (packed like the latents, NULL to skip):
 * mu, scale (= b), bits (per latent -log2 P).  Workspace as cc_rd_forward(1). */
int cc_arm_rate(const cc_model_desc* desc, const int16_t* latents, const float* arm_w,
                double* rate, float* mu, float* scale, float* bits,
                void* workspace, size_t workspace_bytes, void* stream);

/* Stage entry: upsampling only -- DEVICE dense [L][H][W] fp32 (PAPER.md:109-111,
 * "upsample the latents to a dense representation").  Runs the same kernels as
 * cc_rd_forward (coarse pyramid + fused last step) with the dense output of
 * the synthesis kernel enabled.  Workspace: cc_workspace_bytes(desc, 1). */
int cc_upsample(const cc_model_desc* desc, const int16_t* latents, const float* up_w,
                float* dense, void* workspace, size_t workspace_bytes, void* stream);

/* Stage entry: synthesis from a DEVICE dense [L][H][W] fp32 tensor to x_hat
 * [3][H][W] (device) and sse (device double [1], needs image; NULL to skip).
 * h_1x1 (optional, device [3][H][W]): output of the 1x1 stack. */
int cc_synthesize(const cc_model_desc* desc, const float* dense, const float* syn_w,
                  const float* image, float* x_hat, double* sse, float* h_1x1,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Closed-form multiply-accumulates per output pixel (host only, no device). */
typedef struct {
  double arm, up, syn, total;  /* per pixel                         */
  int64_t arm_macs, up_macs, syn_macs;  /* per image (exact integers)  */
  int64_t n_latents;
} cc_mac_breakdown;
double cc_mac_per_pixel(const cc_model_desc* desc, cc_mac_breakdown* out);

/* Validates a descriptor (host only).  0 or a negative code. */
int cc_validate(const cc_model_desc* desc);

const char* cc_strerror(int code);
const char* cc_last_error(void);
const char* cc_version(void);

/* Number of kernels the last cc_rd_forward / cc_rd_forward_host call on this
 * thread launched (bench bookkeeping). */
int64_t cc_last_launch_count(void);

/* ARM rate path (process-wide; host only, no device needed).  The ARM MLP
 * (Table 1 ARM column) is computed either by
 *   CC_ARM_FFMA2: packed FP32 FMAs on the CUDA cores (arm_rate.cu), every
 *                 compiled ARM shape; the decoder's wavefront ARM uses the
 *                 same arithmetic, so per-latent outputs are bit-identical
 *                 to cc_arm_decode's;
 *   CC_ARM_TC:    tcgen05 kind::tf32 MMAs with a 3xTF32 split (fp32-accurate,
 *                 DESIGN.md 7.2) for the shapes it is compiled for
 *                 ([16,24,24,2], [16,16,16,2], [24,24,24,2]), FFMA2 otherwise;
 *   CC_ARM_AUTO:  (default) the measured-faster path per shape: CC_ARM_TC
 *                 for the [16,24,24,2] ARM (BASELINE's ~2000 MAC/px config),
 *                 CC_ARM_FFMA2 for the others.
 * The initial value comes from the environment (CCRD_ARM_PATH = ffma2 | tc).
 * Workspace sizes do not depend on the path.  cc_set_arm_path: CC_EINVAL for
 * an unknown value.  cc_arm_path_for: the path a descriptor runs on now
 * (CC_ARM_FFMA2 or CC_ARM_TC), -1 for an invalid descriptor. */
#define CC_ARM_AUTO 0
#define CC_ARM_FFMA2 1
#define CC_ARM_TC 2
int cc_set_arm_path(int32_t path);
int32_t cc_get_arm_path(void);
int32_t cc_arm_path_for(const cc_model_desc* desc);

/* Synthesis 1x1 path (process-wide; host only).  Layer 0 of the per-pixel
 * 1x1 MLP (Table 1 synthesis column) is computed either by
 *   CC_SYN_FFMA2: packed FP32 FMAs, one thread per vertical pixel pair;
 *   CC_SYN_MMA:   warp MMAs (mma.sync m16n8k8 tf32, 3xTF32 split,
 *                 fp32-accurate), layer 1 still on FFMA2;
 *                 only where it applies (L <= 7, C_h a multiple of 8, the
 *                 latent-chain entries without debug outputs), FFMA2 otherwise;
 *   CC_SYN_TMA:   CC_SYN_FFMA2's arithmetic in persistent CTAs whose tiles
 *                 are staged by TMA one tile ahead; where it
 *                 applies (L >= 3, 8-tap chains, latent rows and S_1 rows
 *                 16-byte strided / aligned, no debug outputs), CC_SYN_FFMA2
 *                 otherwise.  Bit-identical to CC_SYN_FFMA2;
 *   CC_SYN_AUTO:  (default) CC_SYN_TMA where it applies, else CC_SYN_FFMA2
 *                 (the warp-MMA form is issue-bound: 127 vs 109 us per 2K
 *                 image).
 * The initial value comes from the environment (CCRD_SYN_PATH = ffma2 | mma
 * | tma).  cc_set_synth_path: CC_EINVAL for an unknown value. */
#define CC_SYN_AUTO 0
#define CC_SYN_FFMA2 1
#define CC_SYN_MMA 2
#define CC_SYN_TMA 3
int cc_set_synth_path(int32_t path);
int32_t cc_get_synth_path(void);

/* Per-kernel timing (bench.py roofline): between cc_profile_begin() and
 * cc_profile_end(), every kernel the calling thread launches through this
 * library is bracketed by CUDA events recorded on its own stream.
 * cc_profile_end() synchronises those events and returns the summed device
 * time per kernel kind.  Events only; no extra synchronisation in between. */
typedef struct {
  double arm_ms, syn_ms, reduce_ms, pyr_ms;   /* summed event time per kind */
  int64_t arm_launches, syn_launches, reduce_launches, pyr_launches;
} cc_profile_summary;
int cc_profile_begin(void);
int cc_profile_end(cc_profile_summary* out);

#ifdef __cplusplus
}
#endif
#endif /* CCRD_H */
