// ccrd_common.cuh -- shared device helpers and launch-parameter records of the
// CUDA product path.  Nothing here is shared with oracle/ (independent code).
#pragma once

#include <cuda.h>  // CUtensorMap (TMA descriptors in kernel parameters)
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ccrd.h"

namespace ccrd {

// ---------------------------------------------------------------- FFMA2 helpers
// sm_100a has a packed fp32 FMA (PTX fma.rn.f32x2, SASS FFMA2): one warp
// instruction performs 64 FMAs and occupies the FMA pipe for two cycles, so the
// issue slot it frees carries the loads, ReLUs and index math.  Measured on the
// B200 (tools/microbench/ffma_probe.cu): 126.9 FMA/clk/SM with FFMA2 vs 111-124
// with scalar FFMA.  Rounding is identical to fmaf (round-to-nearest, fused).
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
// 64-bit view of a float2 stored in the kernel parameter bank
__device__ __forceinline__ uint64_t ldp2(const float2& v) {
  return *reinterpret_cast<const uint64_t*>(&v);
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// tile row of tile tt in a level with `tx` tiles per row (ArmGeom::tx_mul)
__device__ __forceinline__ int tile_row(int tt, int tx, uint32_t mul) {
  return mul ? (int)__umulhi((uint32_t)tt, mul) : tt / tx;
}

// Single-MUFU base-2 exponential / logarithm (PTX ex2.approx / lg2.approx).
__device__ __forceinline__ float exp2f_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float log2f_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Block-wide deterministic sum of one fp32 value per thread -> fp64 (thread 0).
template <int NT>
__device__ __forceinline__ double block_sum(float v, double* warp_buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_buf[wid] = (double)v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < NT / 32; w++) s += warp_buf[w];
  }
  return s;
}

// ------------------------------------------------------------------ geometry
// Level dimensions and the latent-buffer window.  Full image: lo = 0, hi = h.
// Strip (cc_rd_forward_strip): the buffer holds only global rows
// [lo_l, hi_l) of grid l; every latent read clamps its row to that window (at
// a true image border the window edge IS the border, so this is the replicate
// padding; at an interior window edge it only feeds rows that are discarded).
struct LevelGeom {
  int32_t h[CC_MAX_LEVELS];    // global grid height ceil(H / 2^l)
  int32_t w[CC_MAX_LEVELS];
  int32_t lo[CC_MAX_LEVELS];   // first global row present in the buffer
  int32_t hi[CC_MAX_LEVELS];   // one past the last row present
  int64_t off[CC_MAX_LEVELS];  // element offset of level l in the packed (windowed) buffer
};

// ARM tiling: one CTA = 8 rows x 64 latents of one grid; warp w owns row w,
// lane t the latents at columns t and t + 32 (two latents per thread, so every
// uniform weight load feeds two FFMA2).
#ifndef CCRD_ARM_LPT  // experiment knobs (tools/ variants); the defaults are the measured best
#define CCRD_ARM_LPT 2
#endif
#ifndef CCRD_ARM_TY
#define CCRD_ARM_TY 8
#endif
#ifndef CCRD_ARM_CPS
#define CCRD_ARM_CPS 2
#endif
constexpr int ARM_LPT = CCRD_ARM_LPT;      // latents per thread
constexpr int ARM_TX = 32 * ARM_LPT;
constexpr int ARM_TY = CCRD_ARM_TY;
constexpr int ARM_THREADS = 32 * ARM_TY;
constexpr int ARM_CTAS_PER_SM = CCRD_ARM_CPS;
constexpr int ARM_HALO_TOP = 3;  // dy >= -3
constexpr int ARM_HALO_X = 4;    // |dx| <= 4
constexpr int ARM_SW = ARM_TX + 2 * ARM_HALO_X;
constexpr int ARM_SH = ARM_TY + ARM_HALO_TOP;

struct ArmGeom {
  LevelGeom lv;
  int32_t L;
  int32_t tiles_x[CC_MAX_LEVELS];
  // ceil(2^32 / tiles_x): tile row = umulhi(t, tx_mul) for every tile t of
  // the level (exact while tiles x tiles_x < 2^32, checked on the host; 0 =
  // use the division)
  uint32_t tx_mul[CC_MAX_LEVELS];
  int32_t tile_begin[CC_MAX_LEVELS + 1];  // prefix over levels; [L] = total CTAs
  int32_t own_lo[CC_MAX_LEVELS];          // latent rows whose rate this launch counts
  int32_t own_hi[CC_MAX_LEVELS];          //   (full image: 0 .. h)
  int32_t ctx_off[CC_MAX_CTX];            // dy * ARM_SW + dx (shared-memory offsets)
  float lsmin, lsmax;                     // log-scale clamp
  float p_floor;                          // probability floor
  float bits_cap;                         // -log2(p_floor)
};

// ARM weights packed for FFMA2: for input i, the pair (out 2n, out 2n+1).
// Residual layers are folded on the host (W' = W + I: LinR computes
// ReLU(W z + b + z) = ReLU(W' z + b)).
template <int C, int NH, int NHL>
struct ArmWeights {
  float2 w0[C][NH / 2];
  float2 b0[NH / 2];
  float2 wh[(NHL > 1) ? (NHL - 1) : 1][NH][NH / 2];
  float2 bh[(NHL > 1) ? (NHL - 1) : 1][NH / 2];
  float2 wo[NH];  // (mu, log-scale) pair per input
  float2 bo;
};

template <int C, int NH, int NHL>
struct ArmParams {
  ArmGeom g;
  const int16_t* lat;
  double* partial;  // [CTAs x warps] per-warp rate partial sums
  float* mu;        // optional per-latent debug outputs
  float* scale;
  float* bits;
  ArmWeights<C, NH, NHL> w;
};

// Synthesis tiling: one CTA = 32 x 64 output pixels, 256 threads.
#ifndef CCRD_SYN_THREADS
#define CCRD_SYN_THREADS 256
#endif
#ifndef CCRD_SYN_CPS
#define CCRD_SYN_CPS 2
#endif
#ifndef CCRD_SYN_TH
#define CCRD_SYN_TH 32
#endif
#ifndef CCRD_SYN_TW
#define CCRD_SYN_TW 64
#endif
constexpr int SYN_TH = CCRD_SYN_TH;
constexpr int SYN_TW = CCRD_SYN_TW;
constexpr int SYN_THREADS = CCRD_SYN_THREADS;
constexpr int SYN_CTAS_PER_SM = CCRD_SYN_CPS;

template <int L, int CH, int R, int K>
struct SynWeights {
  float k[K];                 // upsampling taps
  float2 kv[K / 2 + 1];       // last vertical step, both phases: (a0, a1) += sv[u] x kv[u]
  float A0t[L][CH];           // 1x1 layer 0, input-major (4 consecutive outputs per uniform load)
  float a0[CH];
  float A1[3][CH];            // 1x1 layer 1
  float a1[3];
  float2 Gp[(R > 0) ? R : 1][3][3][3];  // residual 3x3: (co 0, co 1) per [ci][ky][kx]
  float Gs[(R > 0) ? R : 1][3][3][3];   // co 2
  float g[(R > 0) ? R : 1][3];
};

struct SynGeom {
  LevelGeom lv;
  int32_t H, W;
  int32_t y0, y1;  // output pixel rows [y0, y1) (full image: 0 .. H); y0 even
  int32_t tiles_x, n_tiles;
};

template <int L, int CH, int R, int K>
struct SynParams {
  SynGeom g;
  const int16_t* lat;      // latents (chain mode)
  const float* s1;         // S_1 = grids 2..L-1 upsampled to level 1, [L-2][h1][w1] (pyramid.cu)
  const float* dense_in;   // [L][H][W] (synthesize-from-dense mode) or null
  const float* image;      // [3][H][W] fp32 or null
  const uint8_t* image8;   // [3][H][W] 8-bit (x = v / 255, desc.image_u8) or null
  float* x_hat;            // [3][H][W] or null
  float* dense_out;        // debug [L][H][W] or null
  float* h1_out;           // debug [3][H][W] or null
  double* partial;         // [n tiles] per-CTA SSE partial sums
  uint8_t* out_u8;         // decode: interleaved 8-bit RGB [H][W][3] of clamp(x_hat) or null
  SynWeights<L, CH, R, K> w;
  // TMA staging (synth_kernel<..., TMA = true> only): level-0 latents (int16,
  // 2-D), grid 1 (int16, 2-D), S_1 (fp32, 3-D [L-2][rows][w_1]) over the
  // buffer windows
  CUtensorMap tm_lat0, tm_g1, tm_s1;
};

// Coarse upsampling pyramid (pyramid.cu): S_j = grids j+1 .. L-1 at level j.
constexpr int PYR_TH = 32;
constexpr int PYR_TW = 64;
#ifndef CCRD_PYR_THREADS
#define CCRD_PYR_THREADS 256
#endif
constexpr int PYR_THREADS = CCRD_PYR_THREADS;
constexpr int PYR_MAX_IMG = 64;  // images per launch (kernel-parameter batch)

struct PyrImage {
  const int16_t* lat;  // packed latents of this image
  float* S;            // this image's pyramid buffer (S_j at S + s_off[j])
  float k[8];          // upsampling taps
};

struct PyrGeom {
  LevelGeom lv;
  int32_t L;
  int64_t s_off[CC_MAX_LEVELS];  // float offset of S_j; S_j = [L-1-j][hi_j - lo_j][w_j]
  int64_t s_floats;              // total floats per image
};

template <int K>
struct PyrParams {
  LevelGeom lv;
  int32_t L, j, tiles_x, y_base;  // tiles cover rows y_base + PYR_TH * ty (y_base = lo_j rounded down to even)
  int64_t s_off[CC_MAX_LEVELS];
  PyrImage img[PYR_MAX_IMG];
};

int launch_pyramid(const PyrGeom& g, int K, const PyrImage* imgs, int n_img, cudaStream_t s);
int pyramid_launch_count(const PyrGeom& g, int n_img);

// Table 1 2-D TConv-K (up_2d): the pyramid runs every level down to level 0,
// whose L-1 upsampled grids go to a dense [L][H][W] buffer (channels 1..L-1)
// that the synthesis kernel reads in its dense-input mode.
struct Pyr2dImage {
  const int16_t* lat;  // packed latents
  float* S;            // S_j for j >= 1 (workspace, PyrGeom offsets)
  float* dense;        // [L][H][W]: S_0 = channels 1 .. L-1
  float k2[64];        // K x K taps, row-major (a = vertical, b = horizontal)
};
int launch_pyramid2d(const PyrGeom& g, int K, const Pyr2dImage* imgs, int n_img, cudaStream_t s);
int pyramid2d_launch_count(const PyrGeom& g, int n_img);
int launch_lat0_to_dense(const int16_t* lat, float* dense, int64_t n, cudaStream_t s);

// Reduction of per-CTA partials into per-image results (deterministic, fp64).
struct ReduceJob {
  const double* arm_partial;
  int32_t n_arm;
  const double* syn_partial;
  int32_t n_syn;
  double inv_3p, lambda_over_p;
};

// ------------------------------------------------ programmatic dependent launch
// Consecutive per-image ARM (or synthesis) kernels of one stream are
// independent, but stream order would hold kernel i + 1 until kernel i's last
// CTA exits, leaving SMs idle in every tail.  With programmatic stream
// serialization (PDL) kernel i + 1 may start once every CTA of kernel i has
// started (pdl_trigger at each CTA's start); every CTA then waits for kernel
// i's completion at its END (pdl_wait), so kernel i + 1 still completes after
// kernel i and anything ordered after the last kernel sees every image.  Both
// are no-ops in a kernel launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Per-thread launch controls, set by the batched forward (ccrd_api.cu) around
// one launcher call through LaunchCtlScope:
//   pdl:       launch with programmatic stream serialization (the previous
//              operation in the stream must be an independent kernel);
//   arm_stage: ARM launchers only -- ARM_STAGE_ONLY copies the packed weights
//              to the image's scratch and returns, ARM_LAUNCH_ONLY launches
//              with weights staged by an earlier call, 0 does both.
enum { ARM_STAGE_ONLY = 1, ARM_LAUNCH_ONLY = 2 };
struct LaunchCtl {
  bool pdl = false;
  int arm_stage = 0;
};
extern thread_local LaunchCtl g_launch_ctl;
struct LaunchCtlScope {
  LaunchCtl saved;
  LaunchCtlScope(bool pdl, int arm_stage) : saved(g_launch_ctl) { g_launch_ctl = LaunchCtl{pdl, arm_stage}; }
  ~LaunchCtlScope() { g_launch_ctl = saved; }
};
bool pdl_enabled();  // CCRD_PDL=0 disables programmatic dependent launches (experiments)

// launch `kern` on `s`, with programmatic stream serialization when g_launch_ctl.pdl
template <typename P>
static inline cudaError_t launch_ctl(void (*kern)(P), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                                     const P& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_launch_ctl.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

// Host-side launchers (defined in arm_rate.cu / synth.cu).
typedef int (*ArmLaunchFn)(const ArmGeom& g, const cc_model_desc& d, const float* arm_w,
                           const int16_t* lat, double* partial, float* mu, float* scale,
                           float* bits, cudaStream_t s);
typedef int (*SynLaunchFn)(const SynGeom& g, const cc_model_desc& d, const float* up_w,
                           const float* syn_w, const int16_t* lat, const float* s1, const float* dense_in,
                           const float* image, float* x_hat, float* dense_out, float* h1_out,
                           double* partial, cudaStream_t s, uint8_t* out_u8);

ArmLaunchFn find_arm_launcher(int C, int NH, int NHL);     // FFMA2 path (arm_rate.cu)
ArmLaunchFn find_arm_tc_launcher(int C, int NH, int NHL);  // tensor-core path (arm_tc.cu)
int arm_tc_partials_per_tile();                            // rate partials per tile of that path
// per image, after the ARM's 16 partial slots per tile: the tensor-core ARM's
// packed weights (global copy, bulk-loaded into shared memory by each CTA)
constexpr int ARM_W_SCRATCH_DOUBLES = 2560;
int device_sm_count();  // current device's SMs (lazily cached; 148 without a device)

// N-O analysis transform (analysis.cu, NEXT-4)
int64_t analysis_param_count(const cc_analysis_desc& a);
size_t analysis_workspace_bytes(const cc_analysis_desc& a);
// NEXT-3 wavefront ARM decode (arm_decode.cu)
int dec_skew(const cc_model_desc& d);
size_t dec_workspace_bytes(const cc_model_desc& d, int n_img);
int arm_decode_impl(const cc_model_desc& d, const ArmGeom& g, int a_override, int n_img, const int16_t* const* truth,
                    const float* const* arm_w, int16_t* const* decoded, float* const* mu, float* const* scale,
                    float* const* bits, double* rate, int32_t* poison, void* ws, cudaStream_t s);
int analysis_block_tc(int mode, bool down, const float* in, float* out, const float* blk, const float* wm, float* lat,
                      int h, int w, int ho, int wo, int n_img, int64_t lat_img, int sm_count, cudaStream_t s);
int analysis_forward_impl(const cc_analysis_desc& a, const float* image, const float* w, float* lat, void* ws,
                          cudaStream_t s);

// training iteration (train.cu, NEXT-2)
int64_t train_param_count(const cc_model_desc& d);
size_t train_workspace_bytes(const cc_model_desc& d);
int train_supported(const cc_model_desc& d);
int train_step_impl(const cc_model_desc& d, float* par, const float* noise, const float* image, float* am, float* av,
                    const cc_adam* opt, cc_rd_result* result, float* grad, void* ws, cudaStream_t s);
SynLaunchFn find_syn_launcher(int L, int CH, int R, int K);
// synthesis 1x1 path (cc_set_synth_path; ccrd_api.cu): CC_SYN_AUTO / FFMA2 / MMA
int synth_path();

}  // namespace ccrd
