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

  // source windows of every channel, replicate-extended (clamped) ------------
#pragma unroll 4
  for (int it = threadIdx.x; it < nch * SR * SC; it += PYR_THREADS) {
    const int k = it / (SR * SC), rem = it - k * (SR * SC);
    const int rr = rem / SC, cc = rem - rr * SC;
    const int64_t gi = (int64_t)(clampi(r0 + rr, los, his - 1) - los) * ws + clampi(c0 + cc, 0, ws - 1);
    sw[it] = (k == 0) ? (float)__ldg(lat + gi) : __ldg(Sn + (int64_t)(k - 1) * ns * ws + gi);
  }
  __syncthreads();
  // horizontal: column pairs (2q, 2q+1) share sources q - K/4 .. q + K/4 ----
#pragma unroll 2
  for (int it = threadIdx.x; it < nch * SR * (PYR_TW / 2); it += PYR_THREADS) {
    const int row = it / (PYR_TW / 2), cp = it - row * (PYR_TW / 2);  // row = k * SR + rr
    const float* src = sw + row * SC + cp;
    float s[K / 2 + 1];
#pragma unroll
    for (int u = 0; u <= K / 2; u++) s[u] = src[u];
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int t = 0; t < K / 2; t++) {
      a0 = fmaf(im.k[2 * t + 1], s[K / 2 - 1 - t], a0);
      a1 = fmaf(im.k[2 * t], s[K / 2 - t], a1);
    }
    *reinterpret_cast<float2*>(tmp + row * PYR_TW + 2 * cp) = make_float2(a0, a1);
  }
  __syncthreads();
  // vertical: row pairs, stored (cropped) to S_j[k] ----------------------------
#pragma unroll 2
  for (int it = threadIdx.x; it < nch * (PYR_TH / 2) * PYR_TW; it += PYR_THREADS) {
    const int kr = it / PYR_TW, cc = it - kr * PYR_TW;
    const int k = kr / (PYR_TH / 2), rp = kr - k * (PYR_TH / 2);
    const float* src = tmp + (k * SR + rp) * PYR_TW + cc;
    float s[K / 2 + 1];
#pragma unroll
    for (int u = 0; u <= K / 2; u++) s[u] = src[u * PYR_TW];
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int t = 0; t < K / 2; t++) {
      a0 = fmaf(im.k[2 * t + 1], s[K / 2 - 1 - t], a0);
      a1 = fmaf(im.k[2 * t], s[K / 2 - t], a1);
    }
    const int y = Y0 + 2 * rp, x = X0 + cc;
    if (x < wj) {
      float* dst = Sj + (int64_t)k * nj * wj + (int64_t)(y - loj) * wj + x;
      if (y >= loj && y < hij) dst[0] = a0;
      if (y + 1 >= loj && y + 1 < hij) dst[wj] = a1;
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

}  // namespace ccrd
