// synth.cu -- fused upsampling f_upsilon + synthesis f_theta + distortion.
//
// One CTA produces a 32 x 64 tile of x_hat ("upsample the
// latents to a dense representation and synthesize the decoded image";
// Table 1 upsampling / synthesis columns; Eq. 1 distortion):
//   1. upsampling chain in shared memory, coarse to fine: the stack of grids
//      l >= j is carried at resolution j over the window the tile needs, each
//      x2 step a separable stride-2 transposed conv (horizontal pass, then
//      vertical pass; replicate padding = index clamping, crop = never
//      computing past the next level's size);
//   2. per pixel of the tile + R-pixel halo: the last vertical step and the
//      L -> C_h -> 3 1x1 MLP in registers (packed FFMA2, two neurons per
//      instruction), result to shared memory;
//   3. R residual 3x3 layers on shared memory (replicate padding at the image
//      border; the halo is recomputed, never exchanged);
//   4. x_hat store (optional) and (x - x_hat)^2 partial sums -> fp64 per CTA.
// The dense L x H x W tensor is never materialised in HBM.
#include "ccrd_common.cuh"

namespace ccrd {

template <int L, int CH, int R, int K>
struct SynShape {
  static constexpr int RH0 = SYN_TH + 2 * R;  // rows of the level-0 region (tile + halo)
  static constexpr int RW0 = SYN_TW + 2 * R;
  static constexpr int MR1 = RH0 / 2 + 6;     // bound on window rows at levels >= 1
  static constexpr int MC1 = RW0 / 2 + 6;
  static constexpr int NS = (L > 1) ? (L - 1) : 1;  // stack slots (levels 1..L-1)
  static constexpr int STACK = NS * MR1 * MC1;
  static constexpr int HBUF = 3 * RH0 * RW0;
  static constexpr int BUF_A = (STACK > HBUF) ? STACK : HBUF;          // stack | h (ping)
  static constexpr int TMPH = NS * MR1 * RW0;
  static constexpr int BUF_B = (TMPH > HBUF) ? TMPH : HBUF;            // tmpH | h (pong)
  static constexpr size_t SMEM = sizeof(float) * (size_t)(BUF_A + BUF_B);
};

struct Win {
  int r_lo, r_hi, c_lo, c_hi;  // inclusive window of a level
};

// out[2q + r] = sum_t k[2t + 1 - r] * g[clamp(q + r + K/4 - 1 - t)]
// (stride-2 transposed conv on the replicate-extended input, DESIGN.md
//  readings #12-#13; the oracle evaluates the same definition as a scatter).
template <int K>
__device__ __forceinline__ float up_tap(const float* __restrict__ kk, const float* src, int stride,
                                        int o, int n_src, int lo_src) {
  const int q = o >> 1, par = o & 1;
  float acc = 0.0f;
#pragma unroll
  for (int t = 0; t < K / 2; t++) {
    const int idx = clampi(q + par + K / 4 - 1 - t, 0, n_src - 1) - lo_src;
    acc = fmaf(kk[2 * t + 1 - par], src[idx * stride], acc);
  }
  return acc;
}

template <int L, int CH, int R, int K, bool DENSE_IN>
__global__ void __launch_bounds__(SYN_THREADS, 2)
    synth_kernel(const __grid_constant__ SynParams<L, CH, R, K> p) {
  using S = SynShape<L, CH, R, K>;
  extern __shared__ float smem[];
  float* bufA = smem;
  float* bufB = smem + S::BUF_A;
  __shared__ Win win[CC_MAX_LEVELS];
  __shared__ double warp_buf[SYN_THREADS / 32];

  const int H = p.g.H, W = p.g.W;
  const int ty = blockIdx.x / p.g.tiles_x;
  const int tx = blockIdx.x - ty * p.g.tiles_x;
  const int Y0 = ty * SYN_TH, X0 = tx * SYN_TW;
  const int Y1 = min(H, Y0 + SYN_TH), X1 = min(W, X0 + SYN_TW);
  // level-0 region: tile + R halo, clamped to the image
  const int r0 = max(0, Y0 - R), r1 = min(H, Y1 + R);
  const int c0 = max(0, X0 - R), c1 = min(W, X1 + R);
  const int nr0 = r1 - r0, nc0 = c1 - c0;

  if (threadIdx.x == 0) {
    Win v{r0, r1 - 1, c0, c1 - 1};
    win[0] = v;
    for (int j = 1; j < L; j++) {
      v.r_lo = max(0, (v.r_lo >> 1) - K / 4);
      v.r_hi = min(p.g.lv.h[j] - 1, (v.r_hi >> 1) + K / 4);
      v.c_lo = max(0, (v.c_lo >> 1) - K / 4);
      v.c_hi = min(p.g.lv.w[j] - 1, (v.c_hi >> 1) + K / 4);
      win[j] = v;
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- 1. chain
  if constexpr (!DENSE_IN && L > 1) {
    constexpr int MR1 = S::MR1, MC1 = S::MC1, RW0 = S::RW0;
    float* stack = bufA;  // [slot][MR1][MC1], slot = level - 1
    float* tmph = bufB;   // [slot][MR1][RW0]
    auto load_level = [&](int lev) {
      const Win v = win[lev];
      const int nr = v.r_hi - v.r_lo + 1, nc = v.c_hi - v.c_lo + 1;
      const int16_t* g = p.lat + p.g.lv.off[lev];
      const int gw = p.g.lv.w[lev];
      float* dst = stack + (lev - 1) * MR1 * MC1;
#pragma unroll 1
      for (int s = threadIdx.x; s < nr * nc; s += SYN_THREADS) {
        const int rr = s / nc, cc = s - rr * nc;
        dst[rr * MC1 + cc] = (float)__ldg(g + (int64_t)(v.r_lo + rr) * gw + v.c_lo + cc);
      }
    };
    load_level(L - 1);
    __syncthreads();
#pragma unroll 1
    for (int j = L - 1; j >= 1; j--) {
      // horizontal pass: level j (window j) -> columns of window j-1, for grids j..L-1
      const Win vs = win[j], vd = win[j - 1];
      const int nrs = vs.r_hi - vs.r_lo + 1;
      const int ncd = vd.c_hi - vd.c_lo + 1;
      const int nslots = L - j;  // slots j-1 .. L-2
      const int per = nrs * ncd;
      const int tstride = (j == 1) ? RW0 : MC1;
#pragma unroll 1
      for (int s = threadIdx.x; s < nslots * per; s += SYN_THREADS) {
        const int sl = s / per, rem = s - sl * per;
        const int rr = rem / ncd, cc = rem - rr * ncd;
        const int slot = j - 1 + sl;
        const float* src = stack + slot * MR1 * MC1 + rr * MC1;
        tmph[slot * MR1 * RW0 + rr * tstride + cc] =
            up_tap<K>(p.w.k, src, 1, vd.c_lo + cc, p.g.lv.w[j], vs.c_lo);
      }
      __syncthreads();
      if (j == 1) break;  // the last vertical step is done per pixel in phase 2
      // vertical pass: rows of window j-1
      const int nrd = vd.r_hi - vd.r_lo + 1;
      const int per2 = nrd * ncd;
#pragma unroll 1
      for (int s = threadIdx.x; s < nslots * per2; s += SYN_THREADS) {
        const int sl = s / per2, rem = s - sl * per2;
        const int rr = rem / ncd, cc = rem - rr * ncd;
        const int slot = j - 1 + sl;
        const float* src = tmph + slot * MR1 * RW0 + cc;
        stack[slot * MR1 * MC1 + rr * MC1 + cc] =
            up_tap<K>(p.w.k, src, MC1, vd.r_lo + rr, p.g.lv.h[j], vs.r_lo);
      }
      // grid j-1 joins the stack (slot j-2) at its own resolution
      if (j - 1 >= 1) load_level(j - 1);
      __syncthreads();
    }
  }

  // ------------------------------------------------- 2. last step + 1x1 MLP
  float* hA = bufA;  // [3][RH0][RW0], indexed relative to (r0, c0)
  float* hB = bufB;
  constexpr int RH0 = S::RH0, RW0 = S::RW0;
  constexpr int HP = RH0 * RW0;
  {
    const Win v1 = win[(L > 1) ? 1 : 0];
    const int16_t* g0 = p.lat;
    const int64_t P = (int64_t)H * W;
#pragma unroll 1
    for (int s = threadIdx.x; s < nr0 * nc0; s += SYN_THREADS) {
      const int rr = s / nc0, cc = s - rr * nc0;
      const int y = r0 + rr, x = c0 + cc;
      float v[L];
      if constexpr (DENSE_IN) {
#pragma unroll
        for (int l = 0; l < L; l++) v[l] = __ldg(p.dense_in + l * P + (int64_t)y * W + x);
      } else {
        v[0] = (float)__ldg(g0 + (int64_t)y * W + x);
#pragma unroll
        for (int l = 1; l < L; l++) {
          const float* src = bufB + (l - 1) * S::MR1 * RW0 + cc;
          v[l] = up_tap<K>(p.w.k, src, RW0, y, p.g.lv.h[1], v1.r_lo);
        }
      }
      const bool inner = (y >= Y0 && y < Y1 && x >= X0 && x < X1);
      if (p.dense_out != nullptr && inner) {
#pragma unroll
        for (int l = 0; l < L; l++) p.dense_out[l * P + (int64_t)y * W + x] = v[l];
      }
      // layer 0: L -> CH, ReLU
      uint64_t acc[CH / 2];
#pragma unroll
      for (int n = 0; n < CH / 2; n++) acc[n] = ldp2(p.w.a0[n]);
#pragma unroll
      for (int i = 0; i < L; i++) {
        const uint64_t xi = f2pack(v[i], v[i]);
#pragma unroll
        for (int n = 0; n < CH / 2; n++) acc[n] = ffma2(xi, ldp2(p.w.A0[i][n]), acc[n]);
      }
      // layer 1: CH -> 3 (ReLU unless it is the module's last layer, i.e. R == 0)
      uint64_t o01a = f2pack(p.w.a1[0], p.w.a1[1]), o01b = f2pack(0.0f, 0.0f);
      float o2a = p.w.a1[2], o2b = 0.0f;
#pragma unroll
      for (int n = 0; n < CH / 2; n++) {
        const float2 hv = f2unpack(acc[n]);
        const float h0 = fmaxf(hv.x, 0.0f), h1 = fmaxf(hv.y, 0.0f);
        o01a = ffma2(f2pack(h0, h0), ldp2(p.w.A1p[2 * n]), o01a);
        o2a = fmaf(h0, p.w.A1s[2 * n], o2a);
        o01b = ffma2(f2pack(h1, h1), ldp2(p.w.A1p[2 * n + 1]), o01b);
        o2b = fmaf(h1, p.w.A1s[2 * n + 1], o2b);
      }
      const float2 oa = f2unpack(o01a), ob = f2unpack(o01b);
      float o[3] = {oa.x + ob.x, oa.y + ob.y, o2a + o2b};
      if (R > 0) {
#pragma unroll
        for (int c = 0; c < 3; c++) o[c] = fmaxf(o[c], 0.0f);
      }
      if (p.h1_out != nullptr && inner) {
#pragma unroll
        for (int c = 0; c < 3; c++) p.h1_out[c * P + (int64_t)y * W + x] = o[c];
      }
#pragma unroll
      for (int c = 0; c < 3; c++) hA[c * HP + rr * RW0 + cc] = o[c];
    }
  }
  __syncthreads();

  // ------------------------------------------------- 3. residual 3x3 layers
  float* hin = hA;
  float* hout = hB;
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int e = R - 1 - r;  // remaining halo after this layer
    const int yr0 = max(0, Y0 - e), yr1 = min(H, Y1 + e);
    const int xr0 = max(0, X0 - e), xr1 = min(W, X1 + e);
    const int nr = yr1 - yr0, nc = xr1 - xr0;
    const bool last = (r == R - 1);
#pragma unroll 1
    for (int s = threadIdx.x; s < nr * nc; s += SYN_THREADS) {
      const int rr = s / nc, cc = s - rr * nc;
      const int y = yr0 + rr, x = xr0 + cc;
      int ro[3], co[3];
#pragma unroll
      for (int d = 0; d < 3; d++) {
        ro[d] = (clampi(y + d - 1, 0, H - 1) - r0) * RW0;
        co[d] = clampi(x + d - 1, 0, W - 1) - c0;
      }
      const int ctr = (y - r0) * RW0 + (x - c0);
      uint64_t a01 = f2pack(hin[ctr] + p.w.g[r][0], hin[HP + ctr] + p.w.g[r][1]);
      float a2 = hin[2 * HP + ctr] + p.w.g[r][2];
#pragma unroll
      for (int ci = 0; ci < 3; ci++)
#pragma unroll
        for (int ky = 0; ky < 3; ky++)
#pragma unroll
          for (int kx = 0; kx < 3; kx++) {
            const float hv = hin[ci * HP + ro[ky] + co[kx]];
            a01 = ffma2(f2pack(hv, hv), ldp2(p.w.Gp[r][ci][ky][kx]), a01);
            a2 = fmaf(hv, p.w.Gs[r][ci][ky][kx], a2);
          }
      const float2 a = f2unpack(a01);
      float o[3] = {a.x, a.y, a2};
      if (!last) {
#pragma unroll
        for (int c = 0; c < 3; c++) o[c] = fmaxf(o[c], 0.0f);
      }
#pragma unroll
      for (int c = 0; c < 3; c++) hout[c * HP + ctr] = o[c];
    }
    __syncthreads();
    float* t = hin;
    hin = hout;
    hout = t;
  }

  // --------------------------------------------- 4. x_hat + distortion (Eq. 1)
  float sse = 0.0f;
  {
    const int64_t P = (int64_t)H * W;
    const int nr = Y1 - Y0, nc = X1 - X0;
#pragma unroll 1
    for (int s = threadIdx.x; s < nr * nc; s += SYN_THREADS) {
      const int rr = s / nc, cc = s - rr * nc;
      const int y = Y0 + rr, x = X0 + cc;
      const int ctr = (y - r0) * RW0 + (x - c0);
      const int64_t gidx = (int64_t)y * W + x;
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const float xh = hin[c * HP + ctr];
        if (p.x_hat != nullptr) p.x_hat[c * P + gidx] = xh;
        if (p.image != nullptr) {
          const float e = __ldg(p.image + c * P + gidx) - xh;
          sse = fmaf(e, e, sse);
        }
      }
    }
  }
  const double s = block_sum<SYN_THREADS>(sse, warp_buf);
  if (threadIdx.x == 0 && p.partial != nullptr) p.partial[blockIdx.x] = s;
}

// ---------------------------------------------------------------- host launcher
template <int L, int CH, int R, int K>
static int launch_syn(const SynGeom& g, const cc_model_desc& d, const float* up_w,
                      const float* syn_w, const int16_t* lat, const float* dense_in,
                      const float* image, float* x_hat, float* dense_out, float* h1_out,
                      double* partial, cudaStream_t stream) {
  (void)d;
  SynParams<L, CH, R, K> p;
  p.g = g;
  p.lat = lat;
  p.dense_in = dense_in;
  p.image = image;
  p.x_hat = x_hat;
  p.dense_out = dense_out;
  p.h1_out = h1_out;
  p.partial = partial;
  for (int t = 0; t < K; t++) p.w.k[t] = up_w ? up_w[t] : 0.0f;
  const float* q = syn_w;
  for (int i = 0; i < L; i++)
    for (int n = 0; n < CH / 2; n++) p.w.A0[i][n] = make_float2(q[(2 * n) * L + i], q[(2 * n + 1) * L + i]);
  for (int n = 0; n < CH / 2; n++) p.w.a0[n] = make_float2(q[L * CH + 2 * n], q[L * CH + 2 * n + 1]);
  q += L * CH + CH;
  for (int i = 0; i < CH; i++) {
    p.w.A1p[i] = make_float2(q[i], q[CH + i]);
    p.w.A1s[i] = q[2 * CH + i];
  }
  for (int c = 0; c < 3; c++) p.w.a1[c] = q[3 * CH + c];
  q += 3 * CH + 3;
  for (int r = 0; r < R; r++) {
    for (int ci = 0; ci < 3; ci++)
      for (int ky = 0; ky < 3; ky++)
        for (int kx = 0; kx < 3; kx++) {
          auto G = [&](int co) { return q[((co * 3 + ci) * 3 + ky) * 3 + kx]; };
          p.w.Gp[r][ci][ky][kx] = make_float2(G(0), G(1));
          p.w.Gs[r][ci][ky][kx] = G(2);
        }
    for (int c = 0; c < 3; c++) p.w.g[r][c] = q[81 + c];
    q += 84;
  }
  using S = SynShape<L, CH, R, K>;
  static bool attr_set[2] = {false, false};
  const size_t smem = S::SMEM;
  if (dense_in) {
    if (!attr_set[1]) {
      cudaFuncSetAttribute(synth_kernel<L, CH, R, K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      attr_set[1] = true;
    }
    synth_kernel<L, CH, R, K, true><<<g.n_tiles, SYN_THREADS, smem, stream>>>(p);
  } else {
    if (!attr_set[0]) {
      cudaFuncSetAttribute(synth_kernel<L, CH, R, K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      attr_set[0] = true;
    }
    synth_kernel<L, CH, R, K, false><<<g.n_tiles, SYN_THREADS, smem, stream>>>(p);
  }
  return 0;
}

struct SynEntry {
  int L, CH, R, K;
  SynLaunchFn fn;
};

// Compiled synthesis shapes: BASELINE.json configs (tiny [4,8,3]+1, low
// [7,16,3]+2, ref [7,40,3]+2; 8 taps), Table 1 (A300 [7,8,3]+1, A545/A1079
// [7,16,3]+2 with 4 taps, A2300 [7,40,3]+2 with 8 taps) and small L for tests.
static const SynEntry kSyn[] = {
    {4, 8, 1, 8, launch_syn<4, 8, 1, 8>},     {7, 16, 2, 8, launch_syn<7, 16, 2, 8>},
    {7, 40, 2, 8, launch_syn<7, 40, 2, 8>},   {7, 8, 1, 4, launch_syn<7, 8, 1, 4>},
    {7, 16, 2, 4, launch_syn<7, 16, 2, 4>},   {4, 8, 1, 4, launch_syn<4, 8, 1, 4>},
    {1, 8, 1, 8, launch_syn<1, 8, 1, 8>},     {5, 8, 1, 8, launch_syn<5, 8, 1, 8>},
    {5, 8, 1, 4, launch_syn<5, 8, 1, 4>},     {4, 8, 0, 8, launch_syn<4, 8, 0, 8>},
    {4, 8, 3, 8, launch_syn<4, 8, 3, 8>},     {2, 8, 1, 8, launch_syn<2, 8, 1, 8>},
    {3, 8, 1, 8, launch_syn<3, 8, 1, 8>},     {7, 40, 2, 4, launch_syn<7, 40, 2, 4>},
};

SynLaunchFn find_syn_launcher(int L, int CH, int R, int K) {
  for (const auto& e : kSyn)
    if (e.L == L && e.CH == CH && e.R == R && e.K == K) return e.fn;
  return nullptr;
}

}  // namespace ccrd
