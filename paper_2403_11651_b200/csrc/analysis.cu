// analysis.cu -- the N-O Cool-chic analysis transform y = f_alpha(x) on the
// GPU (NEXT-4; Eq. 3; readings A1-A7 of DESIGN.md, the same
// as oracle/ccanalysis.c documents -- the two share no code).
//
// Activations are NHWC fp32 ([pixels][C]).  The depth-wise 7x7 convolutions,
// the stem, the 2x2 average pooling and the 1x1 C -> 1 merges are kernels here;
// the point-wise layers are dense GEMMs over all pixels ([P x C] x [C x 4C] ->
// ReLU -> [P x 4C] x [4C x C]) and run on cuBLASLt ("plain library GEMMs")
// with their epilogues fused: bias + ReLU on the expansion, bias + the
// residual (or the downsampling block's main branch) through the C operand
// (beta = 1) on the projection.  `tf32` selects fp32 or TF32 tensor-core math
// for the GEMMs (CUBLAS_COMPUTE_32F vs CUBLAS_COMPUTE_32F_FAST_TF32).
#include <cublasLt.h>

#include <cstring>

#include "ccrd_common.cuh"

namespace ccrd {

constexpr int AN_TB = 256;

// grid-stride over pixels: threadIdx.x = 4 channels (blockDim.x = C / 4),
// threadIdx.y = pixel within the block's group; a thread's 4 weights rows stay
// in registers across its pixels (the stem writes C floats per pixel: HBM-bound)
__global__ void an_stem_kernel(const float* __restrict__ img, const float* __restrict__ w, float* __restrict__ x,
                               int64_t P, int C) {
  const int c = 4 * threadIdx.x;
  float wr[4][3], bb[4];
#pragma unroll
  for (int e = 0; e < 4; e++) {
    bb[e] = __ldg(w + C * 3 + c + e);
#pragma unroll
    for (int i = 0; i < 3; i++) wr[e][i] = __ldg(w + (c + e) * 3 + i);
  }
  for (int64_t p = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; p < P; p += (int64_t)gridDim.x * blockDim.y) {
    const float i0 = __ldg(img + p), i1 = __ldg(img + P + p), i2 = __ldg(img + 2 * P + p);
    float o[4];
#pragma unroll
    for (int e = 0; e < 4; e++) o[e] = fmaf(wr[e][2], i2, fmaf(wr[e][1], i1, fmaf(wr[e][0], i0, bb[e])));
    *reinterpret_cast<float4*>(x + p * C + c) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// depth-wise 7x7, stride s, zero padding 3; NHWC, one output (pixel, channel)
// per thread, channels fastest (a warp reads 32 consecutive channels per tap)
__global__ void an_dw_kernel(const float* __restrict__ in, const float* __restrict__ k, const float* __restrict__ kb,
                             float* __restrict__ out, int h, int w, int ho, int wo, int s, int C) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)ho * wo * C) return;
  const int64_t p = idx / C;
  const int c = (int)(idx - p * C);
  const int y = (int)(p / wo), x = (int)(p - (int64_t)y * wo);
  float a = kb[c];
  const float* kc = k + c * 49;
#pragma unroll
  for (int ky = 0; ky < 7; ky++) {
    const int iy = s * y + ky - 3;
    if (iy < 0 || iy >= h) continue;
#pragma unroll
    for (int kx = 0; kx < 7; kx++) {
      const int ix = s * x + kx - 3;
      if (ix >= 0 && ix < w) a = fmaf(kc[ky * 7 + kx], in[((int64_t)iy * w + ix) * C + c], a);
    }
  }
  out[idx] = a;
}

// 2x2 average pooling, stride 2, ceil mode, mean over the in-image samples
__global__ void an_pool_kernel(const float* __restrict__ in, float* __restrict__ out, int h, int w, int ho, int wo, int C) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)ho * wo * C) return;
  const int64_t p = idx / C;
  const int c = (int)(idx - p * C);
  const int y = (int)(p / wo), x = (int)(p - (int64_t)y * wo);
  float sum = 0.0f;
  int n = 0;
  for (int dy = 0; dy < 2; dy++)
    for (int dx = 0; dx < 2; dx++) {
      const int iy = 2 * y + dy, ix = 2 * x + dx;
      if (iy < h && ix < w) {
        sum += in[((int64_t)iy * w + ix) * C + c];
        n++;
      }
    }
  out[idx] = sum / (float)n;
}

// latent = bm + sum_c Wm[c] x[p][c]
__global__ void an_merge_kernel(const float* __restrict__ x, const float* __restrict__ wm, float* __restrict__ lat,
                                int64_t P, int C) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  float a = wm[C];
  for (int c = 0; c < C; c++) a = fmaf(wm[c], x[p * C + c], a);
  lat[p] = a;
}

// ---------------------------------------------------------------- cuBLASLt
struct LtState {
  cublasLtHandle_t h = nullptr;
};
static thread_local LtState g_lt;

// D (m x n col-major, ld m) = op(A) B + beta C + bias (m), epilogue relu?
//   A: weights row-major [m][k] == col-major k x m, used transposed
//   B, C, D: NHWC activations == col-major (channels) x (pixels)
static int lt_gemm(int m, int64_t n, int k, const float* A, const float* B, const float* Cm, float* D, const float* bias,
                   bool relu, bool tf32, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (!g_lt.h && cublasLtCreate(&g_lt.h) != CUBLAS_STATUS_SUCCESS) return -1;
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr, ld = nullptr;
  cublasStatus_t st = cublasLtMatmulDescCreate(&op, tf32 ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F, CUDA_R_32F);
  const cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof(tA));
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof(tB));
  const cublasLtEpilogue_t epi = relu ? CUBLASLT_EPILOGUE_RELU_BIAS : CUBLASLT_EPILOGUE_BIAS;
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi));
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
  cublasLtMatrixLayoutCreate(&la, CUDA_R_32F, k, m, k);
  cublasLtMatrixLayoutCreate(&lb, CUDA_R_32F, k, n, k);
  cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, m, n, m);
  cublasLtMatrixLayoutCreate(&ld, CUDA_R_32F, m, n, m);
  cublasLtMatmulPreference_t pref = nullptr;
  cublasLtMatmulPreferenceCreate(&pref);
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof(ws_bytes));
  cublasLtMatmulHeuristicResult_t heur;
  int found = 0;
  st = cublasLtMatmulAlgoGetHeuristic(g_lt.h, op, la, lb, lc, ld, pref, 1, &heur, &found);
  const float alpha = 1.0f, beta = Cm ? 1.0f : 0.0f;
  if (st == CUBLAS_STATUS_SUCCESS && found > 0)
    st = cublasLtMatmul(g_lt.h, op, &alpha, A, la, B, lb, &beta, Cm ? Cm : D, lc, D, ld, &heur.algo, ws, ws_bytes, s);
  else if (st == CUBLAS_STATUS_SUCCESS)
    st = CUBLAS_STATUS_NOT_SUPPORTED;
  cublasLtMatmulPreferenceDestroy(pref);
  cublasLtMatrixLayoutDestroy(la);
  cublasLtMatrixLayoutDestroy(lb);
  cublasLtMatrixLayoutDestroy(lc);
  cublasLtMatrixLayoutDestroy(ld);
  cublasLtMatmulDescDestroy(op);
  return st == CUBLAS_STATUS_SUCCESS ? 0 : -(int)st - 100;
}

// ---------------------------------------------------------------- plan
struct AnPlan {
  int64_t P0, n_params, n_lat;  // n_lat: latents per image
  size_t o_x, o_y, o_t, o_h, o_pool, o_lt, total;
  size_t lt_bytes;
};

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

// x, y: the N images' activations (ping-pong); t0, h1, pool, cuBLASLt
// workspace: one image at a time (unfused modes)
static void an_plan(const cc_analysis_desc& a, AnPlan& pl) {
  const int C = a.C;
  const int N = a.N;
  pl.P0 = (int64_t)a.H * a.W;
  pl.n_params = (int64_t)C * 3 + C;
  pl.n_lat = 0;
  for (int l = 0; l < a.L; l++) {
    for (int b = 0; b < a.blocks; b++) {
      pl.n_params += (int64_t)C * 49 + C + 8LL * C * C + 4 * C + C;
      if (l > 0 && b == 0) pl.n_params += (int64_t)C * C + C;
    }
    pl.n_params += C + 1;
    pl.n_lat += (int64_t)((a.H + (1 << l) - 1) >> l) * ((a.W + (1 << l) - 1) >> l);
  }
  const bool fused = (a.tf32 == 1 || a.tf32 == 3) && C == 64;
  pl.lt_bytes = fused ? 0 : (32u << 20);
  size_t o = 0;
  auto take = [&](size_t b) {
    const size_t r = o;
    o += a256(b);
    return r;
  };
  pl.o_x = take(4 * (size_t)pl.P0 * C * N);
  pl.o_y = take(4 * (size_t)pl.P0 * C * N);
  pl.o_t = take(fused ? 0 : 4 * (size_t)pl.P0 * C);
  pl.o_h = take(fused ? 0 : 4 * (size_t)pl.P0 * 4 * C);
  pl.o_pool = take(fused ? 0 : 4 * (size_t)((pl.P0 + 3) / 4 + a.W + a.H + 1) * C);
  pl.o_lt = take(pl.lt_bytes);
  pl.total = o;
}

int64_t analysis_param_count(const cc_analysis_desc& a) {
  AnPlan pl;
  an_plan(a, pl);
  return pl.n_params;
}
size_t analysis_workspace_bytes(const cc_analysis_desc& a) {
  AnPlan pl;
  an_plan(a, pl);
  return pl.total;
}

static int blocks_of(int64_t n) { return (int)((n + AN_TB - 1) / AN_TB); }

static void launch_stem(const float* image, const float* w, float* x, int64_t P, int C, cudaStream_t s) {
  const dim3 tb(C / 4, AN_TB / (C / 4));  // C % 4 == 0 (validated), C / 4 <= AN_TB
  const int64_t need = (P + tb.y - 1) / tb.y;
  const int64_t cap = (int64_t)device_sm_count() * 8;
  an_stem_kernel<<<(unsigned)(need < cap ? need : cap), tb, 0, s>>>(image, w, x, P, C);
}

// One image through the unfused path (dw kernels + cuBLASLt GEMMs); x holds
// the stem output.  Returns launches or a negative code.
static int unfused_one(const cc_analysis_desc& a, const AnPlan& pl, const float* w, float* lat, float* x, float* y,
                       char* W, cudaStream_t s) {
  float* t0 = (float*)(W + pl.o_t);
  float* h1 = (float*)(W + pl.o_h);
  float* pool = (float*)(W + pl.o_pool);
  void* ltws = W + pl.o_lt;
  const int C = a.C;
  const bool tf32 = a.tf32 != 0;  // 1 / 3 (C != 64) or 2: TF32 cuBLASLt
  int launches = 0, rc;
  int h = a.H, wd = a.W;
  int64_t P = pl.P0;
  const float* q = w + C * 3 + C;
  int64_t loff = 0;
  for (int l = 0; l < a.L; l++) {
    for (int b = 0; b < a.blocks; b++) {
      const bool down = l > 0 && b == 0;
      const int ho = down ? (h + 1) / 2 : h, wo = down ? (wd + 1) / 2 : wd;
      const int64_t Po = (int64_t)ho * wo;
      const float* k = q;
      const float* kb = k + C * 49;
      const float* W1 = kb + C;
      const float* b1 = W1 + 4 * C * C;
      const float* W2 = b1 + 4 * C;
      const float* b2 = W2 + 4 * C * C;
      q = b2 + C;
      an_dw_kernel<<<blocks_of(Po * C), AN_TB, 0, s>>>(x, k, kb, t0, h, wd, ho, wo, down ? 2 : 1, C);
      launches++;
      // expansion: h1 = ReLU(W1 t0 + b1)
      if ((rc = lt_gemm(4 * C, Po, C, W1, t0, nullptr, h1, b1, true, tf32, ltws, pl.lt_bytes, s))) return rc;
      launches++;
      if (!down) {
        // projection + residual: y = W2 h1 + b2 + x
        if ((rc = lt_gemm(C, Po, 4 * C, W2, h1, x, y, b2, false, tf32, ltws, pl.lt_bytes, s))) return rc;
        launches++;
      } else {
        // main branch y = W2 h1 + b2; identity branch: y += Wid pool(x) + bid
        const float* Wid = q;
        const float* bid = Wid + C * C;
        q = bid + C;
        if ((rc = lt_gemm(C, Po, 4 * C, W2, h1, nullptr, y, b2, false, tf32, ltws, pl.lt_bytes, s))) return rc;
        an_pool_kernel<<<blocks_of(Po * C), AN_TB, 0, s>>>(x, pool, h, wd, ho, wo, C);
        if ((rc = lt_gemm(C, Po, C, Wid, pool, y, y, bid, false, tf32, ltws, pl.lt_bytes, s))) return rc;
        launches += 3;
      }
      float* tmp = x;
      x = y;
      y = tmp;
      h = ho;
      wd = wo;
      P = Po;
    }
    an_merge_kernel<<<blocks_of(P), AN_TB, 0, s>>>(x, q, lat + loff, P, C);
    launches++;
    q += C + 1;
    loff += P;
  }
  return launches;
}

// Returns launches (>= 0) or a negative code (< -100: cuBLASLt status).
int analysis_forward_impl(const cc_analysis_desc& a, const float* image, const float* w, float* lat, void* ws,
                          cudaStream_t s) {
  AnPlan pl;
  an_plan(a, pl);
  char* W = (char*)ws;
  float* x = (float*)(W + pl.o_x);
  float* y = (float*)(W + pl.o_y);
  const int C = a.C, N = a.N;
  const int64_t P0 = pl.P0;
  int launches = 0;
  if (!((a.tf32 == 1 || a.tf32 == 3) && C == 64)) {
    for (int n = 0; n < N; n++) {
      launch_stem(image + n * 3 * P0, w, x, P0, C, s);
      const int r = unfused_one(a, pl, w, lat + n * pl.n_lat, x, y, W, s);
      if (r < 0) return r;
      launches += 1 + r;
    }
    return launches;
  }
  // fused tensor-core blocks (analysis_tc.cu), all N images per launch; the
  // merge rides on each level's last block
  for (int n = 0; n < N; n++) launch_stem(image + n * 3 * P0, w, x + n * P0 * C, P0, C, s);
  launches += N;
  const int sms = device_sm_count();
  const float* q = w + C * 3 + C;
  int h = a.H, wd = a.W;
  int64_t loff = 0;
  for (int l = 0; l < a.L; l++) {
    for (int b = 0; b < a.blocks; b++) {
      const bool down = l > 0 && b == 0;
      const int ho = down ? (h + 1) / 2 : h, wo = down ? (wd + 1) / 2 : wd;
      const float* blk = q;
      q += (int64_t)C * 49 + C + 8LL * C * C + 4 * C + C + (down ? (int64_t)C * C + C : 0);
      const bool last = b == a.blocks - 1;
      if (analysis_block_tc(a.tf32, down, x, y, blk, last ? q : nullptr, last ? lat + loff : nullptr, h, wd, ho, wo, N,
                            pl.n_lat, sms, s))
        return -1;
      launches++;
      float* tmp = x;
      x = y;
      y = tmp;
      h = ho;
      wd = wo;
    }
    q += C + 1;
    loff += (int64_t)h * wd;
  }
  return launches;
}

}  // namespace ccrd
