// pyramid.cu -- the coarse part of the upsampling f_upsilon (
// Table 1 "1-1-TConv-K"; readings #11-#14), batched over images.
//
// S_j[k] = grid (j + 1 + k) upsampled to level j's resolution (h_j x w_j),
// k = 0 .. L-2-j:   S_j[0] = Up(y_{j+1}),  S_j[k] = Up(S_{j+1}[k-1]).
// One launch per level j = L-2 .. 1 for all images (per-image filters and
// pointers in the parameter bank).  Up() is one x2 step: a stride-2 transposed
// conv along x (width w_j) then along y (height h_j) on the replicate-extended
// input (clamped source index), cropped to the level's size:
//   out[2q + r] = sum_t k[2t + 1 - r] g[q + r + K/4 - 1 - t].
// The last step (S_1 and y_1 -> level 0) is fused into synth_kernel, so the
// full-resolution dense tensor never exists in memory.  The FMA order per
// output matches synth_kernel's ChainStep exactly.
#include <cstring>

#include "ccrd_common.cuh"

namespace ccrd {

template <int K>
__global__ void __launch_bounds__(PYR_THREADS)
    pyramid_kernel(const __grid_constant__ PyrParams<K> p) {
  constexpr int SR = PYR_TH / 2 + K / 2;  // source rows of a tile
  constexpr int SC = PYR_TW / 2 + K / 2;  // source cols
  extern __shared__ float psm[];
  const PyrImage& im = p.img[blockIdx.y];
  const int j = p.j;
  const int nch = p.L - 1 - j;
  float* sw = psm;                       // [nch][SR][SC]
  float* tmp = psm + nch * SR * SC;      // [nch][SR][PYR_TW]
  // level j rows [lo_j, hi_j) are produced (buffer row = global row - lo_j);
  // level j+1 sources are read clamped to ITS window [lo_{j+1}, hi_{j+1})
  const int wj = p.lv.w[j], loj = p.lv.lo[j], hij = p.lv.hi[j], nj = hij - loj;
  const int ws = p.lv.w[j + 1], los = p.lv.lo[j + 1], his = p.lv.hi[j + 1], ns = his - los;
  const int ty = blockIdx.x / p.tiles_x;
  const int Y0 = p.y_base + ty * PYR_TH, X0 = (blockIdx.x - ty * p.tiles_x) * PYR_TW;
  const int r0 = (Y0 >> 1) - K / 4, c0 = (X0 >> 1) - K / 4;  // source window origin
  float* Sj = im.S + p.s_off[j];
  const float* Sn = im.S + p.s_off[j + 1];  // S_{j+1}, nch - 1 channels
  const int16_t* lat = im.lat + p.lv.off[j + 1];

  // source windows of every channel, replicate-extended (clamped): a thread
  // owns one window column (its clamped source column computed once) and
  // walks rows; grid j+1 (int16) first, then the S_{j+1} channels (fp32) ----
  {
    constexpr int RPI = PYR_THREADS / SC;  // rows per pass
    const int cc = threadIdx.x % SC, rsub = threadIdx.x / SC;
    if (rsub < RPI) {
      const int gc = clampi(c0 + cc, 0, ws - 1);
      const int64_t plane = (int64_t)ns * ws;
      if (r0 >= los && r0 + SR <= his) {  // no row clamping: pointer walks
        const int64_t step = (int64_t)RPI * ws, first = (int64_t)(r0 + rsub - los) * ws + gc;
        const int16_t* lp = lat + first;
#pragma unroll 3
        for (int rr = rsub; rr < SR; rr += RPI, lp += step) sw[rr * SC + cc] = (float)__ldg(lp);
#pragma unroll 1
        for (int k1 = 0; k1 < nch - 1; k1++) {
          const float* sp = Sn + k1 * plane + first;
          float* d = sw + (SR + k1 * SR) * SC + cc;
#pragma unroll 3
          for (int rr = rsub; rr < SR; rr += RPI, sp += step) d[rr * SC] = __ldg(sp);
        }
      } else {
#pragma unroll 4
        for (int rr = rsub; rr < SR; rr += RPI)
          sw[rr * SC + cc] = (float)__ldg(lat + (int64_t)(clampi(r0 + rr, los, his - 1) - los) * ws + gc);
#pragma unroll 4
        for (int row = rsub; row < (nch - 1) * SR; row += RPI) {  // row = (k - 1) * SR + rr
          const int k1 = row / SR, rr = row - k1 * SR;
          sw[(SR + row) * SC + cc] =
              __ldg(Sn + k1 * plane + (int64_t)(clampi(r0 + rr, los, his - 1) - los) * ws + gc);
        }
      }
    }
  }
  __syncthreads();
  // horizontal: column pairs (2q, 2q+1) share sources q - K/4 .. q + K/4; a
  // thread takes two adjacent pairs (6 loads feed 4 outputs, one 16-byte store)
#pragma unroll 2
  for (int it = threadIdx.x; it < nch * SR * (PYR_TW / 4); it += PYR_THREADS) {
    const int row = it / (PYR_TW / 4), cq = it - row * (PYR_TW / 4);  // row = k * SR + rr
    const float* src = sw + row * SC + 2 * cq;
    float s[K / 2 + 2];
#pragma unroll
    for (int u = 0; u < K / 2 + 2; u++) s[u] = src[u];
    float a[4];
#pragma unroll
    for (int pr = 0; pr < 2; pr++) {
      float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
      for (int t = 0; t < K / 2; t++) {
        a0 = fmaf(im.k[2 * t + 1], s[pr + K / 2 - 1 - t], a0);
        a1 = fmaf(im.k[2 * t], s[pr + K / 2 - t], a1);
      }
      a[2 * pr] = a0;
      a[2 * pr + 1] = a1;
    }
    *reinterpret_cast<float4*>(tmp + row * PYR_TW + 4 * cq) = make_float4(a[0], a[1], a[2], a[3]);
  }
  __syncthreads();
  // vertical: row pairs, stored (cropped) to S_j[k]; a thread takes four
  // adjacent columns of one row pair: 16-byte shared loads, FFMA2 over column
  // pairs (each output keeps its FMA order), 16-byte stores where the level's
  // rows are 16-byte aligned ---------------------------------------------------
  const bool vec = (wj & 3) == 0 && (reinterpret_cast<uintptr_t>(Sj) & 15) == 0;
#pragma unroll 1
  for (int it = threadIdx.x; it < nch * (PYR_TH / 2) * (PYR_TW / 4); it += PYR_THREADS) {
    const int kr = it / (PYR_TW / 4), cq = it - kr * (PYR_TW / 4);
    const int k = kr / (PYR_TH / 2), rp = kr - k * (PYR_TH / 2);
    const float* src = tmp + (k * SR + rp) * PYR_TW + 4 * cq;
    uint64_t s01[K / 2 + 1], s23[K / 2 + 1];  // source row u, columns (0, 1) and (2, 3)
#pragma unroll
    for (int u = 0; u <= K / 2; u++) {
      const float4 f = *reinterpret_cast<const float4*>(src + u * PYR_TW);
      s01[u] = f2pack(f.x, f.y);
      s23[u] = f2pack(f.z, f.w);
    }
    uint64_t e01 = 0ull, e23 = 0ull, d01 = 0ull, d23 = 0ull;  // even / odd output row
#pragma unroll
    for (int t = 0; t < K / 2; t++) {
      const uint64_t k1 = f2pack(im.k[2 * t + 1], im.k[2 * t + 1]), k0 = f2pack(im.k[2 * t], im.k[2 * t]);
      e01 = ffma2(k1, s01[K / 2 - 1 - t], e01);
      e23 = ffma2(k1, s23[K / 2 - 1 - t], e23);
      d01 = ffma2(k0, s01[K / 2 - t], d01);
      d23 = ffma2(k0, s23[K / 2 - t], d23);
    }
    const int x = X0 + 4 * cq;
    const int yb = Y0 + 2 * rp - loj;  // buffer row of the even output
    float* dst = Sj + (int64_t)k * nj * wj + (int64_t)yb * wj + x;
    const float2 e0 = f2unpack(e01), e1 = f2unpack(e23), o0 = f2unpack(d01), o1 = f2unpack(d23);
    const float ev[4] = {e0.x, e0.y, e1.x, e1.y}, od[4] = {o0.x, o0.y, o1.x, o1.y};
#pragma unroll
    for (int r = 0; r < 2; r++) {
      if ((unsigned)(yb + r) >= (unsigned)nj) continue;  // rows [lo_j, hi_j) only
      const float* v = r ? od : ev;
      float* d = dst + r * wj;
      if (vec && x + 3 < wj) {
        *reinterpret_cast<float4*>(d) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; c++)
          if (x + c < wj) d[c] = v[c];
      }
    }
  }
}

template <int K>
static int launch_pyr(const PyrGeom& g, const PyrImage* imgs, int n_img, cudaStream_t s) {
  PyrParams<K> p;
  p.lv = g.lv;
  p.L = g.L;
  for (int l = 0; l < CC_MAX_LEVELS; l++) p.s_off[l] = g.s_off[l];
  for (int j = g.L - 2; j >= 1; j--) {
    p.j = j;
    p.tiles_x = (g.lv.w[j] + PYR_TW - 1) / PYR_TW;
    p.y_base = g.lv.lo[j] & ~1;
    const int tiles = p.tiles_x * ((g.lv.hi[j] - p.y_base + PYR_TH - 1) / PYR_TH);
    if (tiles == 0) continue;
    for (int b = 0; b < n_img; b += PYR_MAX_IMG) {
      const int m = (n_img - b < PYR_MAX_IMG) ? n_img - b : PYR_MAX_IMG;
      for (int i = 0; i < m; i++) p.img[i] = imgs[b + i];
      constexpr int SR = PYR_TH / 2 + K / 2, SC = PYR_TW / 2 + K / 2;
      const size_t smem = sizeof(float) * (size_t)(g.L - 1 - j) * SR * (SC + PYR_TW);
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(pyramid_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      pyramid_kernel<K><<<dim3(tiles, m), PYR_THREADS, smem, s>>>(p);
    }
  }
  return 0;
}

int launch_pyramid(const PyrGeom& g, int K, const PyrImage* imgs, int n_img, cudaStream_t s) {
  if (g.L < 3) return 0;  // S_1 is empty: the synthesis kernel reads y_1 directly
  return K == 4 ? launch_pyr<4>(g, imgs, n_img, s) : launch_pyr<8>(g, imgs, n_img, s);
}

int pyramid_launch_count(const PyrGeom& g, int n_img) {
  if (g.L < 3) return 0;
  int lv = 0;
  for (int j = g.L - 2; j >= 1; j--) lv += (g.lv.hi[j] > g.lv.lo[j]) ? 1 : 0;
  return lv * ((n_img + PYR_MAX_IMG - 1) / PYR_MAX_IMG);
}

// ------------------------------------------------------------------ 2-D TConv
// Table 1 "1-1-TConv-K" as a non-separable K x K kernel (
// NEXT-1): out[2q+r][2p+s] = sum_{t,u} k2[2t+1-r][2u+1-s] g[q+r+K/4-1-t][p+s+K/4-1-u]
// on the replicate-extended input (clamped source rows / columns), cropped.
// One launch per level j = L-2 .. 0 for all images; a thread produces a 2x2
// output block from the (K/2+1)^2 shared sources around (q, p).
constexpr int PYR2D_MAX_IMG = 32;  // images per launch (k2 in the parameter bank)

template <int K>
struct Pyr2dParams {
  LevelGeom lv;
  int32_t L, j, tiles_x;
  int64_t s_off[CC_MAX_LEVELS];
  int64_t plane0;  // H * W (level-0 channel stride of the dense buffer)
  Pyr2dImage img[PYR2D_MAX_IMG];
};

template <int K>
__global__ void __launch_bounds__(PYR_THREADS)
    pyramid2d_kernel(const __grid_constant__ Pyr2dParams<K> p) {
  constexpr int SR = PYR_TH / 2 + K / 2;  // source rows of a tile
  constexpr int SC = PYR_TW / 2 + K / 2;  // source cols
  constexpr int H2 = K / 2;
  extern __shared__ float psm[];
  const Pyr2dImage& im = p.img[blockIdx.y];
  const int j = p.j;
  const int nch = p.L - 1 - j;
  float* sw = psm;  // [nch][SR][SC]
  const int hj = p.lv.h[j], wj = p.lv.w[j];
  const int hs = p.lv.h[j + 1], ws = p.lv.w[j + 1];
  const int ty = blockIdx.x / p.tiles_x;
  const int Y0 = ty * PYR_TH, X0 = (blockIdx.x - ty * p.tiles_x) * PYR_TW;
  const int r0 = (Y0 >> 1) - K / 4, c0 = (X0 >> 1) - K / 4;  // source window origin
  const float* Sn = im.S + p.s_off[j + 1];                    // S_{j+1}, nch - 1 channels
  const int16_t* lat = im.lat + p.lv.off[j + 1];
  float* Sj = (j == 0) ? im.dense + p.plane0 : im.S + p.s_off[j];
  const int64_t plane_j = (int64_t)hj * wj;

#pragma unroll 4
  for (int it = threadIdx.x; it < nch * SR * SC; it += PYR_THREADS) {
    const int k = it / (SR * SC), rem = it - k * (SR * SC);
    const int rr = rem / SC, cc = rem - rr * SC;
    const int64_t gi = (int64_t)clampi(r0 + rr, 0, hs - 1) * ws + clampi(c0 + cc, 0, ws - 1);
    sw[it] = (k == 0) ? (float)__ldg(lat + gi) : __ldg(Sn + (int64_t)(k - 1) * hs * ws + gi);
  }
  __syncthreads();
#pragma unroll 1
  for (int it = threadIdx.x; it < nch * (PYR_TH / 2) * (PYR_TW / 2); it += PYR_THREADS) {
    const int k = it / ((PYR_TH / 2) * (PYR_TW / 2)), rem = it - k * ((PYR_TH / 2) * (PYR_TW / 2));
    const int qq = rem / (PYR_TW / 2), pp = rem - qq * (PYR_TW / 2);
    // sources rho, sigma = 0 .. K/2 <-> rows q - K/4 + rho, columns p - K/4 + sigma
    const float* src = sw + (k * SR + qq) * SC + pp;
    float g[H2 + 1][H2 + 1];
#pragma unroll
    for (int a = 0; a <= H2; a++)
#pragma unroll
      for (int b = 0; b <= H2; b++) g[a][b] = src[a * SC + b];
    float o[2][2];
#pragma unroll
    for (int r = 0; r < 2; r++)
#pragma unroll
      for (int s = 0; s < 2; s++) {
        float acc = 0.0f;
#pragma unroll
        for (int t = 0; t < H2; t++)
#pragma unroll
          for (int u = 0; u < H2; u++)
            acc = fmaf(im.k2[(2 * t + 1 - r) * K + (2 * u + 1 - s)], g[r + H2 - 1 - t][s + H2 - 1 - u], acc);
        o[r][s] = acc;
      }
    const int y = Y0 + 2 * qq, x = X0 + 2 * pp;
    float* dst = Sj + (int64_t)k * plane_j;
#pragma unroll
    for (int r = 0; r < 2; r++)
#pragma unroll
      for (int s = 0; s < 2; s++)
        if (y + r < hj && x + s < wj) dst[(int64_t)(y + r) * wj + x + s] = o[r][s];
  }
}

template <int K>
static int launch_pyr2d(const PyrGeom& g, const Pyr2dImage* imgs, int n_img, cudaStream_t s) {
  Pyr2dParams<K> p;  // ~9 KB, copied into the launch's parameter bank
  memset(&p, 0, sizeof(p));
  p.lv = g.lv;
  p.L = g.L;
  p.plane0 = (int64_t)g.lv.h[0] * g.lv.w[0];
  for (int l = 0; l < CC_MAX_LEVELS; l++) p.s_off[l] = g.s_off[l];
  for (int j = g.L - 2; j >= 0; j--) {
    p.j = j;
    p.tiles_x = (g.lv.w[j] + PYR_TW - 1) / PYR_TW;
    const int tiles = p.tiles_x * ((g.lv.h[j] + PYR_TH - 1) / PYR_TH);
    constexpr int SR = PYR_TH / 2 + K / 2, SC = PYR_TW / 2 + K / 2;
    const size_t smem = sizeof(float) * (size_t)(g.L - 1 - j) * SR * SC;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(pyramid2d_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int b = 0; b < n_img; b += PYR2D_MAX_IMG) {
      const int m = (n_img - b < PYR2D_MAX_IMG) ? n_img - b : PYR2D_MAX_IMG;
      for (int i = 0; i < m; i++) p.img[i] = imgs[b + i];
      pyramid2d_kernel<K><<<dim3(tiles, m), PYR_THREADS, smem, s>>>(p);
    }
  }
  return 0;
}

int launch_pyramid2d(const PyrGeom& g, int K, const Pyr2dImage* imgs, int n_img, cudaStream_t s) {
  if (g.L < 2) return 0;
  return K == 4 ? launch_pyr2d<4>(g, imgs, n_img, s) : launch_pyr2d<8>(g, imgs, n_img, s);
}

int pyramid2d_launch_count(const PyrGeom& g, int n_img) {
  if (g.L < 2) return 0;
  return (g.L - 1) * ((n_img + PYR2D_MAX_IMG - 1) / PYR2D_MAX_IMG);
}

__global__ void lat0_to_dense_kernel(const int16_t* __restrict__ lat, float* __restrict__ dense, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dense[i] = (float)lat[i];
}

int launch_lat0_to_dense(const int16_t* lat, float* dense, int64_t n, cudaStream_t s) {
  const int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  lat0_to_dense_kernel<<<blocks, 256, 0, s>>>(lat, dense, n);
  return 0;
}

}  // namespace ccrd
