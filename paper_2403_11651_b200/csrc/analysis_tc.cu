// analysis_tc.cu -- one N-O ConvNeXt block of the analysis transform as ONE
// persistent tcgen05 kernel (NEXT-4, TF32 mode, C = 64; PAPER.md:432-447,
// readings A2/A3/A5 of DESIGN.md).
//
//   stride-1 block:      y = x + W2 ReLU(W1 dw(x) + b1) + b2
//   downsampling block:  y = W2 ReLU(W1 dw_s2(x) + b1) + b2 + Wid pool(x) + bid
//   (last block of a level, optional) latent = Wm . y + bm
//
// The unfused form (analysis.cu) streams t0 = dw(x) [P x C], the expansion
// h [P x 4C] and its read-back through HBM: ~3.3 KB per pixel per block.
// Here one CTA per SM keeps W1, W2 (and Wid) resident in shared memory and,
// per tile of 4 x 32 output pixels (M = 128, one TMEM lane per pixel):
//   1. depth-wise 7x7 on the CUDA cores (packed FFMA2, 2 channels x 8 pixels per thread;
//      for downsampling blocks also the 2x2 mean pool) -> A tile in shared
//      memory, K-major SWIZZLE_128B, rounded to TF32;
//   2. tcgen05.mma SS: D1[128 x 256] (TMEM) = A x W1^T;
//   3. epilogue in place: D1 <- tf32(ReLU(D1 + b1)) (tcgen05.ld / .st);
//   4. tcgen05.mma TS (A = the hidden layer straight from TMEM):
//      D2[128 x 64] = hidden x W2^T  (+ pool x Wid^T, SS, downsampling);
//   5. epilogue: y = D2 + b2 (+ bid) (+ x), stored NHWC, and the level's C -> 1
//      merge when requested.
// HBM traffic per block: read x (+ halo, mostly L2 hits) and write y, 0.5 KB
// per output pixel (2 KB/px in + 0.25 KB/px out for downsampling blocks).
#include <cuda.h>

#include <cstdlib>

#include "ccrd_common.cuh"
#include "tcgen05.cuh"

namespace ccrd {

constexpr int BT_THREADS = 512;  // 16 warps: latency hiding for the depth-wise loads
constexpr int BT_C = 64, BT_HID = 256;  // C = 64, expansion 4C (A2)
constexpr int BT_TY = 4, BT_TX = 32;    // output tile: 4 rows x 32 pixels = MMA M 128

struct BlockTcParams {
  const float* in;   // x, NHWC [h][w][64]
  float* out;        // y, NHWC [ho][wo][64]
  const float* blk;  // block parameters: dw k[64][49], kb[64], W1[256][64], b1, W2[64][256], b2, (Wid[64][64], bid)
  const float* wm;   // merge Wm[64], bm (nullable)
  float* lat;        // latent grid [ho][wo] (nullable)
  int h, w, ho, wo, tiles_x, n_tiles;
  int tpi;                           // tiles per image (n_tiles = tpi x images)
  int64_t in_img, out_img, lat_img;  // per-image strides (elements) of in, out, lat
};

// byte offset of element (r, k) of a K-major SWIZZLE_128B operand with R rows:
// K split in 32-float (128-byte) atom columns of R x 128 bytes each
__host__ __device__ constexpr uint32_t sw128(int r, int k, int R) {
  return (uint32_t)((k >> 5) * (R * 128) + (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) & 7) ^ (r & 7)) << 4) +
                    (k & 3) * 4);
}

constexpr int XS_LD = 68;  // padded row: quarter-warp float4 reads hit distinct banks

template <bool DOWN>
struct BtSmem {
  static constexpr uint32_t W1 = 0;                              // [256 x 64]
  static constexpr uint32_t W2 = W1 + BT_HID * BT_C * 4;         // [64 x 256]
  static constexpr uint32_t A1 = W2 + BT_C * BT_HID * 4;         // [128 x 64] dw output
  static constexpr uint32_t AP = A1 + 128 * BT_C * 4;            // [128 x 64] pool (downsampling)
  static constexpr uint32_t WID = AP + (DOWN ? 128 * BT_C * 4 : 0);  // [64 x 64]
  static constexpr uint32_t B1 = WID + (DOWN ? BT_C * BT_C * 4 : 0);
  static constexpr uint32_t B2 = B1 + BT_HID * 4;
  static constexpr uint32_t WM = B2 + BT_C * 4;
  static constexpr uint32_t MP = WM + BT_C * 4;                  // merge partials [4][128]
  static constexpr uint32_t WK = MP + 4 * 128 * 4;               // dw weights [49][32] channel pairs
  static constexpr uint32_t XS = WK + 49 * 32 * 8;               // residual x tile [128][68] (stride 1)
  static constexpr uint32_t BAR = XS + (DOWN ? 0 : 128 * XS_LD * 4);  // 2 mbarriers
  static constexpr uint32_t SLOT = BAR + 16;
  static constexpr uint32_t TOTAL = SLOT + 16 + 1024;            // + alignment slack
};

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128
__host__ __device__ constexpr uint32_t bt_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ uint64_t ldg_f2(const float* p) { return ldp2(__ldg(reinterpret_cast<const float2*>(p))); }

// 16 TMEM lanes x 8 NREP columns (16x256b, NREP repetitions): thread t gets
// lane t/4 (regs 4m, 4m+1) and lane t/4 + 8 (regs 4m+2, 4m+3), columns
// 8m + 2(t%4), +1 (CUTLASS SM100_TMEM_LOAD_16dp256b{2,4}x layouts)
template <int NREP>
__device__ __forceinline__ void tmem_ld16x256(uint32_t taddr, float (&v)[4 * NREP]);
template <>
__device__ __forceinline__ void tmem_ld16x256<4>(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 16; k++) v[k] = __uint_as_float(r[k]);
}
template <>
__device__ __forceinline__ void tmem_ld16x256<2>(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 8; k++) v[k] = __uint_as_float(r[k]);
}

// Epilogue of one warp: its lane quarter (= tile row oy) x channels c0 ..
// c0 + 8 NREP of D2 (TMEM address td2 = lane quarter + the column of c0):
// y = D2 + b2 (+ x from `res`, RES) stored NHWC.  With the 16x256b loads every
// global access of the warp covers 8 pixels x 32 contiguous bytes (the 32x32b
// thread-per-pixel form puts lanes 256 B apart: 4x the L1 wavefronts).
// partv[k] accumulates the merge partial (Wm . y over these channels) of
// pixel column 8k + t/4.
template <int NREP, bool RES>
__device__ __forceinline__ void epi2_rows(uint32_t td2, int c0, const float* res, float* out, int oy, int ho, int ox0,
                                          int wo, const float* b2s, const float* wms, float (&partv)[4], int lane) {
  const int t0 = lane & 3, t1 = lane >> 2;
#pragma unroll
  for (int g = 0; g < 2; g++) {  // 16-lane halves of the quarter (all lanes: .sync.aligned)
    float d[4 * NREP];
    tmem_ld16x256<NREP>(td2 + ((uint32_t)(16 * g) << 16), d);
#pragma unroll
    for (int rr = 0; rr < 2; rr++) {
      const int ox = ox0 + 16 * g + 8 * rr + t1;
      if (oy < ho && ox < wo) {
        const int64_t po = ((int64_t)oy * wo + ox) * BT_C + c0 + 2 * t0;
        float2 xv[NREP];
#pragma unroll
        for (int m = 0; m < NREP; m++)
          xv[m] = RES ? __ldg(reinterpret_cast<const float2*>(res + po + 8 * m)) : make_float2(0.0f, 0.0f);
#pragma unroll
        for (int m = 0; m < NREP; m++) {
          const int c = c0 + 8 * m + 2 * t0;
          const float2 y = make_float2(d[4 * m + 2 * rr] + b2s[c] + xv[m].x, d[4 * m + 2 * rr + 1] + b2s[c + 1] + xv[m].y);
          *reinterpret_cast<float2*>(out + po + 8 * m) = y;
          partv[2 * g + rr] = fmaf(wms[c], y.x, fmaf(wms[c + 1], y.y, partv[2 * g + rr]));
        }
      }
    }
  }
}

// Sum each pixel's partials over the 4 threads holding its channels and write
// them to mp[slot][pixel] (pixel = quarter * 32 + column).
__device__ __forceinline__ void epi2_partials(float (&partv)[4], float* mp, int slot, int quarter, int lane) {
#pragma unroll
  for (int k = 0; k < 4; k++) {
    partv[k] += __shfl_xor_sync(0xffffffffu, partv[k], 1);
    partv[k] += __shfl_xor_sync(0xffffffffu, partv[k], 2);
  }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int k = 0; k < 4; k++) mp[slot * 128 + quarter * 32 + 8 * k + (lane >> 2)] = partv[k];
  }
}

template <bool DOWN>
__global__ void __launch_bounds__(BT_THREADS, 1) an_block_tc_kernel(const __grid_constant__ BlockTcParams p) {
  using S = BtSmem<DOWN>;
  extern __shared__ uint8_t bt_raw[];
  uint8_t* sm = bt_raw + ((1024u - (smem_u32(bt_raw) & 1023u)) & 1023u);
  const uint32_t su = smem_u32(sm);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* b1s = reinterpret_cast<float*>(sm + S::B1);
  float* b2s = reinterpret_cast<float*>(sm + S::B2);
  float* wms = reinterpret_cast<float*>(sm + S::WM);
  float* mp = reinterpret_cast<float*>(sm + S::MP);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S::BAR);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + S::SLOT);

  const float* dk = p.blk;
  const float* dkb = dk + BT_C * 49;
  const float* W1 = dkb + BT_C;
  const float* b1 = W1 + BT_HID * BT_C;
  const float* W2 = b1 + BT_HID;
  const float* b2 = W2 + BT_C * BT_HID;
  const float* Wid = b2 + BT_C;
  const float* bid = Wid + BT_C * BT_C;

  // ---- resident operands: weights -> shared memory (TF32, swizzled), biases.
  // Unrolled loads, all of a thread's in flight at once; scalar because a
  // block's parameters are only 4-byte aligned in the blob (65-float merges).
  {
    constexpr int N1 = BT_HID * BT_C / 4 / BT_THREADS;  // 8 groups of 4 per thread per matrix
    float4 a[N1], b[N1];
#pragma unroll
    for (int u = 0; u < N1; u++) {
      const float* pa = W1 + 4 * (t + u * BT_THREADS);
      const float* pb = W2 + 4 * (t + u * BT_THREADS);
      a[u] = make_float4(__ldg(pa), __ldg(pa + 1), __ldg(pa + 2), __ldg(pa + 3));
      b[u] = make_float4(__ldg(pb), __ldg(pb + 1), __ldg(pb + 2), __ldg(pb + 3));
    }
#pragma unroll
    for (int u = 0; u < N1; u++) {
      const int i = 4 * (t + u * BT_THREADS);  // W1 [256][64], W2 [64][256]; k = i & .. is a multiple of 4
      *reinterpret_cast<float4*>(sm + S::W1 + sw128(i >> 6, i & 63, BT_HID)) =
          make_float4(tf32_rna(a[u].x), tf32_rna(a[u].y), tf32_rna(a[u].z), tf32_rna(a[u].w));
      *reinterpret_cast<float4*>(sm + S::W2 + sw128(i >> 8, i & 255, BT_C)) =
          make_float4(tf32_rna(b[u].x), tf32_rna(b[u].y), tf32_rna(b[u].z), tf32_rna(b[u].w));
    }
    if constexpr (DOWN) {
#pragma unroll
      for (int u = 0; u < BT_C * BT_C / 4 / BT_THREADS; u++) {
        const int i = 4 * (t + u * BT_THREADS);
        const float* pc = Wid + i;
        const float4 c = make_float4(__ldg(pc), __ldg(pc + 1), __ldg(pc + 2), __ldg(pc + 3));
        *reinterpret_cast<float4*>(sm + S::WID + sw128(i >> 6, i & 63, BT_C)) =
            make_float4(tf32_rna(c.x), tf32_rna(c.y), tf32_rna(c.z), tf32_rna(c.w));
      }
    }
  }
  // depth-wise weights, channel-pair interleaved: wks[tap][cp] = (k[2cp][tap], k[2cp+1][tap])
  float2* wks = reinterpret_cast<float2*>(sm + S::WK);
  for (int i = t; i < 49 * 32; i += BT_THREADS) {
    const int tap = i >> 5, c2 = i & 31;
    wks[i] = make_float2(__ldg(dk + (2 * c2) * 49 + tap), __ldg(dk + (2 * c2 + 1) * 49 + tap));
  }
  if (t < BT_HID) b1s[t] = __ldg(b1 + t);
  if (t < BT_C) {
    b2s[t] = __ldg(b2 + t) + (DOWN ? __ldg(bid + t) : 0.0f);
    wms[t] = p.wm ? __ldg(p.wm + t) : 0.0f;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 1)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;                                       // D1 / hidden: columns 0..255
  const uint32_t tmem_d2 = tmem + BT_HID;                            // D2: columns 256..319
  const uint32_t tlane = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's lane quarter

  // depth-wise mapping: channel pair cp = lane, output row ry, 8-pixel group xq
  const int cp = lane, ry = warp & 3, xq = warp >> 2;
  const uint64_t kb2 = f2pack(__ldg(dkb + 2 * cp), __ldg(dkb + 2 * cp + 1));
  const float bm = p.wm ? __ldg(p.wm + BT_C) : 0.0f;
  float* xs = reinterpret_cast<float*>(sm + S::XS);

  constexpr int STR = DOWN ? 2 : 1;
  constexpr int NX = STR * 7 + 7;  // input columns under 8 outputs (14 or 21)
  uint32_t ph = 0;
#pragma unroll 1
  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const int img = tile / p.tpi, tr = tile - img * p.tpi;
    const int ty = tr / p.tiles_x, tx = tr - ty * p.tiles_x;
    const int oy = ty * BT_TY + ry, ox0 = tx * BT_TX + xq * 8;
    const float* pin = p.in + img * p.in_img;
    float* pout = p.out + img * p.out_img;
    float* plat = p.lat ? p.lat + img * p.lat_img : nullptr;

    // ---- 1. depth-wise 7x7 (zero padding 3) of outputs (oy, ox0 .. ox0+7)
    uint64_t acc[8], ps[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      acc[j] = kb2;
      ps[j] = 0;
    }
    const int gx0 = STR * ox0 - 3;
    const bool interior = gx0 >= 0 && gx0 + NX <= p.w;  // warp-uniform: no column checks
#pragma unroll
    for (int ky = 0; ky < 7; ky++) {
      const int iy = STR * oy + ky - 3;
      if (iy < 0 || iy >= p.h) continue;  // zero padding rows (warp-uniform)
      const float* row = pin + ((int64_t)iy * p.w + gx0) * BT_C + 2 * cp;
      uint64_t v[NX];
      if (interior) {
#pragma unroll
        for (int ix = 0; ix < NX; ix++) v[ix] = ldg_f2(row + ix * BT_C);
      } else {
#pragma unroll
        for (int ix = 0; ix < NX; ix++) {
          v[ix] = 0ull;
          if (gx0 + ix >= 0 && gx0 + ix < p.w) v[ix] = ldg_f2(row + ix * BT_C);
        }
      }
      if constexpr (!DOWN) {
        if (ky == 3) {  // the centre row: this tile's residual x
#pragma unroll
          for (int j = 0; j < 8; j++)
            *reinterpret_cast<uint64_t*>(xs + (ry * 32 + xq * 8 + j) * XS_LD + 2 * cp) = v[j + 3];
        }
      } else {
        if (ky == 3 || ky == 4) {
#pragma unroll
          for (int j = 0; j < 8; j++) {
            ps[j] = ffma2(v[2 * j + 3], f2pack(1.0f, 1.0f), ps[j]);
            ps[j] = ffma2(v[2 * j + 4], f2pack(1.0f, 1.0f), ps[j]);
          }
        }
      }
#pragma unroll
      for (int kx = 0; kx < 7; kx++) {
        const uint64_t wv = ldp2(wks[(ky * 7 + kx) * 32 + cp]);
#pragma unroll
        for (int j = 0; j < 8; j++) acc[j] = ffma2(v[STR * j + kx], wv, acc[j]);
      }
    }
    if constexpr (!DOWN) {
      if (oy < 0 || oy >= p.h) {  // rows below the image: residual 0 (never stored)
#pragma unroll
        for (int j = 0; j < 8; j++) *reinterpret_cast<uint64_t*>(xs + (ry * 32 + xq * 8 + j) * XS_LD + 2 * cp) = 0ull;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int r = ry * 32 + xq * 8 + j;
      const float2 a = f2unpack(acc[j]);
      *reinterpret_cast<float2*>(sm + S::A1 + sw128(r, 2 * cp, 128)) = make_float2(tf32_rna(a.x), tf32_rna(a.y));
      if constexpr (DOWN) {
        // mean over the in-image samples of the 2x2 window (ceil mode, A3)
        const int ox = ox0 + j;
        const float inv = 1.0f / (float)(((2 * oy + 1 < p.h) ? 2 : 1) * ((2 * ox + 1 < p.w) ? 2 : 1));
        const float2 q = f2unpack(ps[j]);
        *reinterpret_cast<float2*>(sm + S::AP + sw128(r, 2 * cp, 128)) =
            make_float2(tf32_rna(q.x * inv), tf32_rna(q.y * inv));
      }
    }

    // ---- 2. D1 = A x W1^T   (M 128, N 256, K 64: 8 MMAs of K 8)
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int s = 0; s < 8; s++)
        mma_tf32(tmem, umma_desc_sw128(su + S::A1 + (s >> 2) * (128 * 128) + (s & 3) * 32),
                 umma_desc_sw128(su + S::W1 + (s >> 2) * (BT_HID * 128) + (s & 3) * 32), bt_idesc(BT_HID), s > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, ph);
    asm volatile("tcgen05.fence::after_thread_sync;");

    // ---- 3. hidden = tf32(ReLU(D1 + b1)), in place in TMEM
#pragma unroll 1
    for (int cc = 0; cc < 2; cc++) {
      const int col = (warp >> 2) * 64 + cc * 32;
      float v[32];
      tmem_row<32>(tlane + col, v);
#pragma unroll
      for (int j = 0; j < 32; j++) v[j] = tf32_rna(fmaxf(v[j] + b1s[col + j], 0.0f));
      tmem_st32(tlane + col, v);
    }
    tmem_wait_st();

    // ---- 4. D2 = hidden x W2^T (TS, K 256) (+ pool x Wid^T, SS, K 64)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int s = 0; s < 32; s++)
        mma_tf32_ts(tmem_d2, tmem + 8 * s, umma_desc_sw128(su + S::W2 + (s >> 2) * (BT_C * 128) + (s & 3) * 32),
                    bt_idesc(BT_C), s > 0);
      if constexpr (DOWN) {
#pragma unroll
        for (int s = 0; s < 8; s++)
          mma_tf32(tmem_d2, umma_desc_sw128(su + S::AP + (s >> 2) * (128 * 128) + (s & 3) * 32),
                   umma_desc_sw128(su + S::WID + (s >> 2) * (BT_C * 128) + (s & 3) * 32), bt_idesc(BT_C), 1);
      }
      mma_commit(bar + 1);
    }
    mbar_wait(bar + 1, ph);
    ph ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");

    // ---- 5. y = D2 + b2 (+ bid) (+ x); 16 channels per warp (quarter cq = warp >> 2)
    if constexpr (DOWN) {
      const int cq = warp >> 2;
      float partv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      epi2_rows<2, false>(tlane + BT_HID + cq * 16, cq * 16, nullptr, pout, ty * BT_TY + (warp & 3), p.ho, tx * BT_TX,
                          p.wo, b2s, wms, partv, lane);
      if (plat) epi2_partials(partv, mp, cq, warp & 3, lane);
    } else {
      const int cq = warp >> 2, r = (warp & 3) * 32 + lane;
      float d[16];
      tmem_row<16>(tlane + BT_HID + cq * 16, d);
      const int oy2 = ty * BT_TY + (warp & 3), ox2 = tx * BT_TX + lane;
      float part = 0.0f;
      if (oy2 < p.ho && ox2 < p.wo) {
        float4* o = reinterpret_cast<float4*>(pout + ((int64_t)oy2 * p.wo + ox2) * BT_C + cq * 16);
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int c = cq * 16 + 4 * i;
          float4 y = make_float4(d[4 * i] + b2s[c], d[4 * i + 1] + b2s[c + 1], d[4 * i + 2] + b2s[c + 2],
                                 d[4 * i + 3] + b2s[c + 3]);
          if constexpr (!DOWN) {
            const float4 x = *reinterpret_cast<const float4*>(xs + r * XS_LD + c);
            y.x += x.x;
            y.y += x.y;
            y.z += x.z;
            y.w += x.w;
          }
          o[i] = y;
          part = fmaf(wms[c], y.x, part);
          part = fmaf(wms[c + 1], y.y, part);
          part = fmaf(wms[c + 2], y.z, part);
          part = fmaf(wms[c + 3], y.w, part);
        }
      }
      if (plat) mp[cq * 128 + r] = part;
    }
    // TMEM D1/D2 and the A tiles are rewritten by the next tile
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (plat && t < 128) {
      const int oy2 = ty * BT_TY + (t >> 5), ox2 = tx * BT_TX + (t & 31);
      if (oy2 < p.ho && ox2 < p.wo) plat[(int64_t)oy2 * p.wo + ox2] = ((mp[t] + mp[128 + t]) + (mp[256 + t] + mp[384 + t])) + bm;
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- warp-specialised stride-1 block
// Same arithmetic as an_block_tc_kernel<false>, pipelined across tiles:
//   warps 0-7  (depth-wise): dw of tile i -> A[i % 2] (double buffer) -> arrive A_full
//   warps 8-15 (epilogue, one per TMEM lane quarter x column half); lane 0 of
//              warp 8 issues the MMAs:
//     MMA1(i) once A_full[i % 2] and MMA2(i-1) completed; commits D1_full and A_empty[i % 2]
//     epi2(i-1) (overlaps MMA1(i)), epi1(i), then MMA2(i) -> D2_full
// so the tensor cores and the epilogue run under the depth-wise work of the
// next tiles.  The residual x is re-read from L2 in epi2.
struct WsSmem {
  static constexpr uint32_t W1 = 0;
  static constexpr uint32_t W2 = W1 + BT_HID * BT_C * 4;
  static constexpr uint32_t A = W2 + BT_C * BT_HID * 4;  // 2 x [128 x 64]
  static constexpr uint32_t B1 = A + 2 * 128 * BT_C * 4;
  static constexpr uint32_t B2 = B1 + BT_HID * 4;
  static constexpr uint32_t WM = B2 + BT_C * 4;
  static constexpr uint32_t MP = WM + BT_C * 4;          // merge partials [2][128]
  static constexpr uint32_t WK = MP + 2 * 128 * 4;
  static constexpr uint32_t BAR = WK + 49 * 32 * 8;      // A_full[2], A_empty[2], D1_full, D2_full
  static constexpr uint32_t SLOT = BAR + 6 * 8;
  static constexpr uint32_t TOTAL = SLOT + 16 + 1024;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__global__ void __launch_bounds__(BT_THREADS, 1) an_block_ws_kernel(const __grid_constant__ BlockTcParams p) {
  using S = WsSmem;
  extern __shared__ uint8_t bt_raw[];
  uint8_t* sm = bt_raw + ((1024u - (smem_u32(bt_raw) & 1023u)) & 1023u);
  const uint32_t su = smem_u32(sm);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* b1s = reinterpret_cast<float*>(sm + S::B1);
  float* b2s = reinterpret_cast<float*>(sm + S::B2);
  float* wms = reinterpret_cast<float*>(sm + S::WM);
  float* mp = reinterpret_cast<float*>(sm + S::MP);
  float2* wks = reinterpret_cast<float2*>(sm + S::WK);
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sm + S::BAR);
  uint64_t* a_empty = a_full + 2;
  uint64_t* d1_full = a_full + 4;
  uint64_t* d2_full = a_full + 5;
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + S::SLOT);

  const float* dk = p.blk;
  const float* dkb = dk + BT_C * 49;
  const float* W1 = dkb + BT_C;
  const float* b1 = W1 + BT_HID * BT_C;
  const float* W2 = b1 + BT_HID;
  const float* b2 = W2 + BT_C * BT_HID;
  {
    constexpr int N1 = BT_HID * BT_C / 4 / BT_THREADS;
    float4 a[N1], b[N1];
#pragma unroll
    for (int u = 0; u < N1; u++) {
      const float* pa = W1 + 4 * (t + u * BT_THREADS);
      const float* pb = W2 + 4 * (t + u * BT_THREADS);
      a[u] = make_float4(__ldg(pa), __ldg(pa + 1), __ldg(pa + 2), __ldg(pa + 3));
      b[u] = make_float4(__ldg(pb), __ldg(pb + 1), __ldg(pb + 2), __ldg(pb + 3));
    }
#pragma unroll
    for (int u = 0; u < N1; u++) {
      const int i = 4 * (t + u * BT_THREADS);
      *reinterpret_cast<float4*>(sm + S::W1 + sw128(i >> 6, i & 63, BT_HID)) =
          make_float4(tf32_rna(a[u].x), tf32_rna(a[u].y), tf32_rna(a[u].z), tf32_rna(a[u].w));
      *reinterpret_cast<float4*>(sm + S::W2 + sw128(i >> 8, i & 255, BT_C)) =
          make_float4(tf32_rna(b[u].x), tf32_rna(b[u].y), tf32_rna(b[u].z), tf32_rna(b[u].w));
    }
  }
  for (int i = t; i < 49 * 32; i += BT_THREADS) {
    const int tap = i >> 5, c2 = i & 31;
    wks[i] = make_float2(__ldg(dk + (2 * c2) * 49 + tap), __ldg(dk + (2 * c2 + 1) * 49 + tap));
  }
  if (t < BT_HID) b1s[t] = __ldg(b1 + t);
  if (t < BT_C) {
    b2s[t] = __ldg(b2 + t);
    wms[t] = p.wm ? __ldg(p.wm + t) : 0.0f;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int k = 0; k < 2; k++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(a_full + k)));  // 8 dw warps
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(a_empty + k)));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d1_full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d2_full)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  const uint32_t tmem_d2 = tmem + BT_HID;
  const uint32_t tlane = tmem + ((uint32_t)((warp & 3) * 32) << 16);

  if (warp < 8) {
    // ================= depth-wise producers: channel pair lane, row warp&3, 16 pixels
    const int cp = lane, ry = warp & 3, xh = warp >> 2;
    const uint64_t kb2 = f2pack(__ldg(dkb + 2 * cp), __ldg(dkb + 2 * cp + 1));
    int i = 0;
#pragma unroll 1
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, i++) {
      const int b = i & 1;
      if (i >= 2) mbar_wait(a_empty + b, ((i >> 1) - 1) & 1);
      const int img = tile / p.tpi, tr = tile - img * p.tpi;
      const int ty = tr / p.tiles_x, tx = tr - ty * p.tiles_x;
      const int oy = ty * BT_TY + ry, ox0 = tx * BT_TX + xh * 16;
      const float* pin = p.in + img * p.in_img;
      uint64_t acc[16];
#pragma unroll
      for (int j = 0; j < 16; j++) acc[j] = kb2;
      const int gx0 = ox0 - 3;
      const bool interior = gx0 >= 0 && gx0 + 22 <= p.w;
#pragma unroll
      for (int ky = 0; ky < 7; ky++) {
        const int iy = oy + ky - 3;
        if (iy < 0 || iy >= p.h) continue;
        const float* row = pin + ((int64_t)iy * p.w + gx0) * BT_C + 2 * cp;
        uint64_t v[22];
        if (interior) {
#pragma unroll
          for (int ix = 0; ix < 22; ix++) v[ix] = ldg_f2(row + ix * BT_C);
        } else {
#pragma unroll
          for (int ix = 0; ix < 22; ix++) {
            v[ix] = 0ull;
            if (gx0 + ix >= 0 && gx0 + ix < p.w) v[ix] = ldg_f2(row + ix * BT_C);
          }
        }
#pragma unroll
        for (int kx = 0; kx < 7; kx++) {
          const uint64_t wv = ldp2(wks[(ky * 7 + kx) * 32 + cp]);
#pragma unroll
          for (int j = 0; j < 16; j++) acc[j] = ffma2(v[j + kx], wv, acc[j]);
        }
      }
      uint8_t* A = sm + S::A + b * (128 * BT_C * 4);
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const float2 a = f2unpack(acc[j]);
        *reinterpret_cast<float2*>(A + sw128(ry * 32 + xh * 16 + j, 2 * cp, 128)) =
            make_float2(tf32_rna(a.x), tf32_rna(a.y));
      }
      asm volatile("fence.proxy.async.shared::cta;");
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + b);
    }
  } else {
    // ================= MMA issue + epilogues
    const int e = warp - 8, hh = e >> 2, q = e & 3;
    const bool leader = (e == 0 && lane == 0);
    const float bm = p.wm ? __ldg(p.wm + BT_C) : 0.0f;
    int i = 0, prev = -1;
#pragma unroll 1
    for (int tile = blockIdx.x;; tile += gridDim.x, i++) {
      const bool has = tile < p.n_tiles;
      if (leader && has) {
        mbar_wait(a_full + (i & 1), (i >> 1) & 1);
        if (i >= 1) mbar_wait(d2_full, (i - 1) & 1);  // MMA2(i-1) consumed the hidden layer in D1
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_u = su + S::A + (i & 1) * (128 * BT_C * 4);
#pragma unroll
        for (int s = 0; s < 8; s++)
          mma_tf32(tmem, umma_desc_sw128(a_u + (s >> 2) * (128 * 128) + (s & 3) * 32),
                   umma_desc_sw128(su + S::W1 + (s >> 2) * (BT_HID * 128) + (s & 3) * 32), bt_idesc(BT_HID), s > 0);
        mma_commit(d1_full);
        mma_commit(a_empty + (i & 1));
      }
      __syncwarp();
      if (prev >= 0) {
        // ---- epi2(prev): y = D2 + b2 + x
        mbar_wait(d2_full, (i - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int pimg = prev / p.tpi, ptr = prev - pimg * p.tpi;
        const int pty = ptr / p.tiles_x, ptx = ptr - pty * p.tiles_x;
        const float* pin = p.in + pimg * p.in_img;
        float* pout = p.out + pimg * p.out_img;
        float* plat = p.lat ? p.lat + pimg * p.lat_img : nullptr;
        float partv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        epi2_rows<4, true>(tlane + BT_HID + hh * 32, hh * 32, pin, pout, pty * BT_TY + q, p.ho, ptx * BT_TX, p.wo, b2s,
                           wms, partv, lane);
        if (plat) {
          epi2_partials(partv, mp, hh, q, lane);
          epi_sync();
          const int te = e * 32 + lane;
          if (te < 128) {
            const int oy3 = pty * BT_TY + (te >> 5), ox3 = ptx * BT_TX + (te & 31);
            if (oy3 < p.ho && ox3 < p.wo) plat[(int64_t)oy3 * p.wo + ox3] = (mp[te] + mp[128 + te]) + bm;
          }
        }
      }
      if (!has) break;
      // ---- epi1(i): hidden = tf32(ReLU(D1 + b1)) in place
      mbar_wait(d1_full, i & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
      for (int cc = 0; cc < 4; cc++) {
        const int col = hh * 128 + cc * 32;
        float v[32];
        tmem_row<32>(tlane + col, v);
#pragma unroll
        for (int j = 0; j < 32; j++) v[j] = tf32_rna(fmaxf(v[j] + b1s[col + j], 0.0f));
        tmem_st32(tlane + col, v);
      }
      tmem_wait_st();
      asm volatile("tcgen05.fence::before_thread_sync;");
      epi_sync();  // also: every epi2(prev) read of D2 and of mp is done
      if (leader) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int s = 0; s < 32; s++)
          mma_tf32_ts(tmem_d2, tmem + 8 * s, umma_desc_sw128(su + S::W2 + (s >> 2) * (BT_C * 128) + (s & 3) * 32),
                      bt_idesc(BT_C), s > 0);
        mma_commit(d2_full);
      }
      __syncwarp();
      prev = tile;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- FP16-operand, TMA-staged stride-1 block (mode 3)
// The warp-specialised block with FP16 tensor-core operands (10-bit mantissa,
// like TF32; fp32 accumulation): W1, W2 and the A tiles take half the shared
// memory, which buys a double-buffered input stage.  One TMA per stage brings
// [10 rows][38 px][32 channels] of x (the tile + the 3-pixel halo; the TMA
// zero-fills out-of-image coordinates = the convolution's zero padding) into
// shared memory; the depth-wise warps read it in register sliding windows
// (8 pixels x 2 channels per thread, no bounds checks).  Two stages (channel
// halves) per tile.
constexpr int HS_ROWS = BT_TY + 6, HS_COLS = BT_TX + 6, HS_CH = 32;
constexpr uint32_t HS_STAGE = HS_ROWS * HS_COLS * HS_CH * 4;  // 48,640 bytes

struct H16Params {
  CUtensorMap tin;  // x as [n][h][w][64] fp32, box {32, 38, 10, 1}
  BlockTcParams p;
};

struct H16Smem {
  static constexpr uint32_t W1 = 0;                          // [256 x 64] f16
  static constexpr uint32_t W2 = W1 + BT_HID * BT_C * 2;     // [64 x 256] f16
  static constexpr uint32_t A = W2 + BT_C * BT_HID * 2;      // 2 x [128 x 64] f16
  static constexpr uint32_t ST = A + 2 * 128 * BT_C * 2;     // 2 input stages
  static constexpr uint32_t B1 = ST + 2 * HS_STAGE;
  static constexpr uint32_t B2 = B1 + BT_HID * 4;
  static constexpr uint32_t WM = B2 + BT_C * 4;
  static constexpr uint32_t MP = WM + BT_C * 4;
  static constexpr uint32_t WK = MP + 2 * 128 * 4;
  static constexpr uint32_t BAR = WK + 49 * 32 * 8;  // st_full[2], a_full[2], a_empty[2], d1_full, d2_full
  static constexpr uint32_t SLOT = BAR + 8 * 8;
  static constexpr uint32_t TOTAL = SLOT + 16 + 1024;
};

// K-major SWIZZLE_128B offset of 16-bit element (r, k): 64 elements per atom row
__host__ __device__ constexpr uint32_t sw128h(int r, int k, int R) {
  return (uint32_t)((k >> 6) * (R * 128) + (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) & 7) ^ (r & 7)) << 4) +
                    (k & 7) * 2);
}
// instruction descriptor kind::f16: D f32, A/B f16, K-major, M = 128
__host__ __device__ constexpr uint32_t h16_idesc(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
// {lo, hi} -> f16x2 (lo in the low half: the lower K index)
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void dw_sync() { asm volatile("bar.sync 2, 256;" ::: "memory"); }

__global__ void __launch_bounds__(BT_THREADS, 1) an_block_h16_kernel(const __grid_constant__ H16Params hp) {
  using S = H16Smem;
  const BlockTcParams& p = hp.p;
  extern __shared__ uint8_t bt_raw[];
  uint8_t* sm = bt_raw + ((1024u - (smem_u32(bt_raw) & 1023u)) & 1023u);
  const uint32_t su = smem_u32(sm);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* b1s = reinterpret_cast<float*>(sm + S::B1);
  float* b2s = reinterpret_cast<float*>(sm + S::B2);
  float* wms = reinterpret_cast<float*>(sm + S::WM);
  float* mp = reinterpret_cast<float*>(sm + S::MP);
  float2* wks = reinterpret_cast<float2*>(sm + S::WK);
  uint64_t* st_full = reinterpret_cast<uint64_t*>(sm + S::BAR);
  uint64_t* a_full = st_full + 2;
  uint64_t* a_empty = st_full + 4;
  uint64_t* d1_full = st_full + 6;
  uint64_t* d2_full = st_full + 7;
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + S::SLOT);

  const float* dk = p.blk;
  const float* dkb = dk + BT_C * 49;
  const float* W1 = dkb + BT_C;
  const float* b1 = W1 + BT_HID * BT_C;
  const float* W2 = b1 + BT_HID;
  const float* b2 = W2 + BT_C * BT_HID;
  {
    constexpr int N1 = BT_HID * BT_C / 4 / BT_THREADS;
#pragma unroll
    for (int u = 0; u < N1; u++) {
      const int i = 4 * (t + u * BT_THREADS);
      const float* pa = W1 + i;
      const float* pb = W2 + i;
      const float a0 = __ldg(pa), a1 = __ldg(pa + 1), a2 = __ldg(pa + 2), a3 = __ldg(pa + 3);
      const float c0 = __ldg(pb), c1 = __ldg(pb + 1), c2 = __ldg(pb + 2), c3 = __ldg(pb + 3);
      *reinterpret_cast<uint2*>(sm + S::W1 + sw128h(i >> 6, i & 63, BT_HID)) = make_uint2(pack_h2(a0, a1), pack_h2(a2, a3));
      *reinterpret_cast<uint2*>(sm + S::W2 + sw128h(i >> 8, i & 255, BT_C)) = make_uint2(pack_h2(c0, c1), pack_h2(c2, c3));
    }
  }
  for (int i = t; i < 49 * 32; i += BT_THREADS) {
    const int tap = i >> 5, c2 = i & 31;
    wks[i] = make_float2(__ldg(dk + (2 * c2) * 49 + tap), __ldg(dk + (2 * c2 + 1) * 49 + tap));
  }
  if (t < BT_HID) b1s[t] = __ldg(b1 + t);
  if (t < BT_C) {
    b2s[t] = __ldg(b2 + t);
    wms[t] = p.wm ? __ldg(p.wm + t) : 0.0f;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int k = 0; k < 2; k++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(st_full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(a_full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(a_empty + k)));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d1_full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d2_full)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;                 // D1: columns 0..255
  const uint32_t tmem_h = tmem + BT_HID;       // hidden, f16x2: 256..383
  const uint32_t tmem_d2 = tmem + BT_HID + 128;  // D2: 384..447
  const uint32_t tlane = tmem + ((uint32_t)((warp & 3) * 32) << 16);

  if (warp < 8) {
    // ================= depth-wise producers over the TMA stages
    const int n_my = (p.n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // tiles of this CTA
    const int n_st = 2 * n_my;
    auto issue = [&](int s) {  // stage s = (local tile s / 2, channel half s % 2) -> buffer s % 2
      const int tile = blockIdx.x + (s >> 1) * gridDim.x;
      const int img = tile / p.tpi, tr = tile - img * p.tpi;
      const int ty = tr / p.tiles_x, tx = tr - ty * p.tiles_x;
      mbar_expect_tx(st_full + (s & 1), HS_STAGE);
      tma_load_4d(sm + S::ST + (s & 1) * HS_STAGE, &hp.tin, st_full + (s & 1), (s & 1) * HS_CH, tx * BT_TX - 3,
                  ty * BT_TY - 3, img);
    };
    if (t == 0) {
      issue(0);
      if (n_st > 1) issue(1);
    }
    const int cp16 = lane & 15, ry = warp & 3, xg = ((warp >> 2) << 1) | (lane >> 4);
#pragma unroll 1
    for (int s = 0; s < n_st; s++) {
      const int i = s >> 1, hf = s & 1;
      const int cpair = hf * 16 + cp16;  // channel pair of this stage
      mbar_wait(st_full + (s & 1), (s >> 1) & 1);
      const float* stg = reinterpret_cast<const float*>(sm + S::ST + (s & 1) * HS_STAGE);
      uint64_t acc[8];
      {
        const uint64_t kb2 = f2pack(__ldg(dkb + 2 * cpair), __ldg(dkb + 2 * cpair + 1));
#pragma unroll
        for (int j = 0; j < 8; j++) acc[j] = kb2;
      }
#pragma unroll
      for (int ky = 0; ky < 7; ky++) {
        const float* row = stg + ((ry + ky) * HS_COLS + xg * 8) * HS_CH + 2 * cp16;
        uint64_t v[14];
#pragma unroll
        for (int ix = 0; ix < 14; ix++) v[ix] = *reinterpret_cast<const uint64_t*>(row + ix * HS_CH);
#pragma unroll
        for (int kx = 0; kx < 7; kx++) {
          const uint64_t wv = ldp2(wks[(ky * 7 + kx) * 32 + cpair]);
#pragma unroll
          for (int j = 0; j < 8; j++) acc[j] = ffma2(v[j + kx], wv, acc[j]);
        }
      }
      dw_sync();  // every depth-wise thread is done with this stage's buffer
      if (t == 0 && s + 2 < n_st) issue(s + 2);
      if (hf == 0 && i >= 2) mbar_wait(a_empty + (i & 1), ((i >> 1) - 1) & 1);
      uint8_t* A = sm + S::A + (i & 1) * (128 * BT_C * 2);
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const float2 a = f2unpack(acc[j]);
        *reinterpret_cast<uint32_t*>(A + sw128h(ry * 32 + xg * 8 + j, 2 * cpair, 128)) = pack_h2(a.x, a.y);
      }
      if (hf == 1) {
        asm volatile("fence.proxy.async.shared::cta;");
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full + (i & 1));
      }
    }
  } else {
    // ================= MMA issue + epilogues (as an_block_ws_kernel, f16 operands)
    const int e = warp - 8, hh = e >> 2, q = e & 3;
    const bool leader = (e == 0 && lane == 0);
    const float bm = p.wm ? __ldg(p.wm + BT_C) : 0.0f;
    int i = 0, prev = -1;
#pragma unroll 1
    for (int tile = blockIdx.x;; tile += gridDim.x, i++) {
      const bool has = tile < p.n_tiles;
      if (leader && has) {
        mbar_wait(a_full + (i & 1), (i >> 1) & 1);
        if (i >= 1) mbar_wait(d2_full, (i - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_u = su + S::A + (i & 1) * (128 * BT_C * 2);
#pragma unroll
        for (int k = 0; k < 4; k++)
          mma_f16(tmem, umma_desc_sw128(a_u + k * 32), umma_desc_sw128(su + S::W1 + k * 32), h16_idesc(BT_HID), k > 0);
        mma_commit(d1_full);
        mma_commit(a_empty + (i & 1));
      }
      __syncwarp();
      if (prev >= 0) {
        mbar_wait(d2_full, (i - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int pimg = prev / p.tpi, ptr = prev - pimg * p.tpi;
        const int pty = ptr / p.tiles_x, ptx = ptr - pty * p.tiles_x;
        const float* pin = p.in + pimg * p.in_img;
        float* pout = p.out + pimg * p.out_img;
        float* plat = p.lat ? p.lat + pimg * p.lat_img : nullptr;
        float partv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        epi2_rows<4, true>(tlane + BT_HID + 128 + hh * 32, hh * 32, pin, pout, pty * BT_TY + q, p.ho, ptx * BT_TX, p.wo,
                           b2s, wms, partv, lane);
        if (plat) {
          epi2_partials(partv, mp, hh, q, lane);
          epi_sync();
          const int te = e * 32 + lane;
          if (te < 128) {
            const int oy3 = pty * BT_TY + (te >> 5), ox3 = ptx * BT_TX + (te & 31);
            if (oy3 < p.ho && ox3 < p.wo) plat[(int64_t)oy3 * p.wo + ox3] = (mp[te] + mp[128 + te]) + bm;
          }
        }
      }
      if (!has) break;
      mbar_wait(d1_full, i & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
      for (int cc = 0; cc < 4; cc++) {
        const int col = hh * 128 + cc * 32;
        float v[32];
        tmem_row<32>(tlane + col, v);
        uint32_t hv[16];
#pragma unroll
        for (int j = 0; j < 16; j++)
          hv[j] = pack_h2(fmaxf(v[2 * j] + b1s[col + 2 * j], 0.0f), fmaxf(v[2 * j + 1] + b1s[col + 2 * j + 1], 0.0f));
        tmem_st16(tlane + BT_HID + (col >> 1), hv);
      }
      tmem_wait_st();
      asm volatile("tcgen05.fence::before_thread_sync;");
      epi_sync();
      if (leader) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int k = 0; k < 16; k++)
          mma_f16_ts(tmem_d2, tmem_h + 8 * k, umma_desc_sw128(su + S::W2 + (k >> 2) * (BT_C * 128) + (k & 3) * 32),
                     h16_idesc(BT_C), k > 0);
        mma_commit(d2_full);
      }
      __syncwarp();
      prev = tile;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- FP16 warp-specialised downsampling block
// The downsampling block (A3) in the mode-3 design: FP16 operands, warps 0-7
// compute the stride-2 depth-wise 7x7 AND the 2x2 mean pool straight from
// global memory (a stride-2 stage would need 115 KB) into double-buffered A /
// AP tiles; warps 8-15 run MMA1 (A x W1^T), the ReLU epilogue into TMEM, MMA2
// (hidden x W2^T, TS) + (pool x Wid^T, SS) and the output epilogue.  A slot is
// released after MMA2 (which still reads the pool tile).
struct H16dSmem {
  static constexpr uint32_t W1 = 0;                          // [256 x 64] f16
  static constexpr uint32_t W2 = W1 + BT_HID * BT_C * 2;     // [64 x 256] f16
  static constexpr uint32_t WID = W2 + BT_C * BT_HID * 2;    // [64 x 64] f16
  static constexpr uint32_t A = WID + BT_C * BT_C * 2;       // 2 x [128 x 64] f16 (dw)
  static constexpr uint32_t AP = A + 2 * 128 * BT_C * 2;     // 2 x [128 x 64] f16 (pool)
  static constexpr uint32_t B1 = AP + 2 * 128 * BT_C * 2;
  static constexpr uint32_t B2 = B1 + BT_HID * 4;
  static constexpr uint32_t WM = B2 + BT_C * 4;
  static constexpr uint32_t MP = WM + BT_C * 4;
  static constexpr uint32_t WK = MP + 2 * 128 * 4;
  static constexpr uint32_t BAR = WK + 49 * 32 * 8;  // a_full[2], a_empty[2], d1_full, d2_full
  static constexpr uint32_t SLOT = BAR + 6 * 8;
  static constexpr uint32_t TOTAL = SLOT + 16 + 1024;
};

__global__ void __launch_bounds__(BT_THREADS, 1) an_block_h16d_kernel(const __grid_constant__ BlockTcParams p) {
  using S = H16dSmem;
  extern __shared__ uint8_t bt_raw[];
  uint8_t* sm = bt_raw + ((1024u - (smem_u32(bt_raw) & 1023u)) & 1023u);
  const uint32_t su = smem_u32(sm);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* b1s = reinterpret_cast<float*>(sm + S::B1);
  float* b2s = reinterpret_cast<float*>(sm + S::B2);
  float* wms = reinterpret_cast<float*>(sm + S::WM);
  float* mp = reinterpret_cast<float*>(sm + S::MP);
  float2* wks = reinterpret_cast<float2*>(sm + S::WK);
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sm + S::BAR);
  uint64_t* a_empty = a_full + 2;
  uint64_t* d1_full = a_full + 4;
  uint64_t* d2_full = a_full + 5;
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + S::SLOT);

  const float* dk = p.blk;
  const float* dkb = dk + BT_C * 49;
  const float* W1 = dkb + BT_C;
  const float* b1 = W1 + BT_HID * BT_C;
  const float* W2 = b1 + BT_HID;
  const float* b2 = W2 + BT_C * BT_HID;
  const float* Wid = b2 + BT_C;
  const float* bid = Wid + BT_C * BT_C;
  {
    constexpr int N1 = BT_HID * BT_C / 4 / BT_THREADS;
#pragma unroll
    for (int u = 0; u < N1; u++) {
      const int i = 4 * (t + u * BT_THREADS);
      const float* pa = W1 + i;
      const float* pb = W2 + i;
      const float a0 = __ldg(pa), a1 = __ldg(pa + 1), a2 = __ldg(pa + 2), a3 = __ldg(pa + 3);
      const float c0 = __ldg(pb), c1 = __ldg(pb + 1), c2 = __ldg(pb + 2), c3 = __ldg(pb + 3);
      *reinterpret_cast<uint2*>(sm + S::W1 + sw128h(i >> 6, i & 63, BT_HID)) = make_uint2(pack_h2(a0, a1), pack_h2(a2, a3));
      *reinterpret_cast<uint2*>(sm + S::W2 + sw128h(i >> 8, i & 255, BT_C)) = make_uint2(pack_h2(c0, c1), pack_h2(c2, c3));
    }
#pragma unroll
    for (int u = 0; u < BT_C * BT_C / 4 / BT_THREADS; u++) {
      const int i = 4 * (t + u * BT_THREADS);
      const float* pc = Wid + i;
      *reinterpret_cast<uint2*>(sm + S::WID + sw128h(i >> 6, i & 63, BT_C)) =
          make_uint2(pack_h2(__ldg(pc), __ldg(pc + 1)), pack_h2(__ldg(pc + 2), __ldg(pc + 3)));
    }
  }
  for (int i = t; i < 49 * 32; i += BT_THREADS) {
    const int tap = i >> 5, c2 = i & 31;
    wks[i] = make_float2(__ldg(dk + (2 * c2) * 49 + tap), __ldg(dk + (2 * c2 + 1) * 49 + tap));
  }
  if (t < BT_HID) b1s[t] = __ldg(b1 + t);
  if (t < BT_C) {
    b2s[t] = __ldg(b2 + t) + __ldg(bid + t);
    wms[t] = p.wm ? __ldg(p.wm + t) : 0.0f;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int k = 0; k < 2; k++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(a_full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(a_empty + k)));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d1_full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(d2_full)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;                   // D1: columns 0..255
  const uint32_t tmem_h = tmem + BT_HID;         // hidden, f16x2: 256..383
  const uint32_t tmem_d2 = tmem + BT_HID + 128;  // D2: 384..447
  const uint32_t tlane = tmem + ((uint32_t)((warp & 3) * 32) << 16);

  if (warp < 8) {
    // ================= depth-wise (stride 2) + 2x2 pool producers
    const int cp = lane, ry = warp & 3, xh = warp >> 2;
    const uint64_t kb2 = f2pack(__ldg(dkb + 2 * cp), __ldg(dkb + 2 * cp + 1));
    int i = 0;
#pragma unroll 1
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, i++) {
      const int b = i & 1;
      if (i >= 2) mbar_wait(a_empty + b, ((i >> 1) - 1) & 1);
      const int img = tile / p.tpi, tr = tile - img * p.tpi;
      const int ty = tr / p.tiles_x, tx = tr - ty * p.tiles_x;
      const float* pin = p.in + img * p.in_img;
      const int oy = ty * BT_TY + ry;
      uint8_t* A = sm + S::A + b * (128 * BT_C * 2);
      uint8_t* AP = sm + S::AP + b * (128 * BT_C * 2);
#pragma unroll 1
      for (int half = 0; half < 2; half++) {  // 2 x 8 output pixels (register budget)
        const int ox0 = tx * BT_TX + xh * 16 + half * 8;
        uint64_t acc[8], ps[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
          acc[j] = kb2;
          ps[j] = 0ull;
        }
        const int gx0 = 2 * ox0 - 3;
        constexpr int NX = 21;  // input columns under 8 stride-2 outputs
        const bool interior = gx0 >= 0 && gx0 + NX <= p.w;
#pragma unroll
        for (int ky = 0; ky < 7; ky++) {
          const int iy = 2 * oy + ky - 3;
          if (iy < 0 || iy >= p.h) continue;
          const float* row = pin + ((int64_t)iy * p.w + gx0) * BT_C + 2 * cp;
          uint64_t v[NX];
          if (interior) {
#pragma unroll
            for (int ix = 0; ix < NX; ix++) v[ix] = ldg_f2(row + ix * BT_C);
          } else {
#pragma unroll
            for (int ix = 0; ix < NX; ix++) {
              v[ix] = 0ull;
              if (gx0 + ix >= 0 && gx0 + ix < p.w) v[ix] = ldg_f2(row + ix * BT_C);
            }
          }
          if (ky == 3 || ky == 4) {
#pragma unroll
            for (int j = 0; j < 8; j++) {
              ps[j] = ffma2(v[2 * j + 3], f2pack(1.0f, 1.0f), ps[j]);
              ps[j] = ffma2(v[2 * j + 4], f2pack(1.0f, 1.0f), ps[j]);
            }
          }
#pragma unroll
          for (int kx = 0; kx < 7; kx++) {
            const uint64_t wv = ldp2(wks[(ky * 7 + kx) * 32 + cp]);
#pragma unroll
            for (int j = 0; j < 8; j++) acc[j] = ffma2(v[2 * j + kx], wv, acc[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int r = ry * 32 + xh * 16 + half * 8 + j;
          const float2 a = f2unpack(acc[j]);
          *reinterpret_cast<uint32_t*>(A + sw128h(r, 2 * cp, 128)) = pack_h2(a.x, a.y);
          const int ox = ox0 + j;
          const float inv = 1.0f / (float)(((2 * oy + 1 < p.h) ? 2 : 1) * ((2 * ox + 1 < p.w) ? 2 : 1));
          const float2 q = f2unpack(ps[j]);
          *reinterpret_cast<uint32_t*>(AP + sw128h(r, 2 * cp, 128)) = pack_h2(q.x * inv, q.y * inv);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + b);
    }
  } else {
    // ================= MMA issue + epilogues
    const int e = warp - 8, hh = e >> 2, q = e & 3;
    const bool leader = (e == 0 && lane == 0);
    const float bm = p.wm ? __ldg(p.wm + BT_C) : 0.0f;
    int i = 0, prev = -1;
#pragma unroll 1
    for (int tile = blockIdx.x;; tile += gridDim.x, i++) {
      const bool has = tile < p.n_tiles;
      if (leader && has) {
        mbar_wait(a_full + (i & 1), (i >> 1) & 1);
        if (i >= 1) mbar_wait(d2_full, (i - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_u = su + S::A + (i & 1) * (128 * BT_C * 2);
#pragma unroll
        for (int k = 0; k < 4; k++)
          mma_f16(tmem, umma_desc_sw128(a_u + k * 32), umma_desc_sw128(su + S::W1 + k * 32), h16_idesc(BT_HID), k > 0);
        mma_commit(d1_full);
      }
      __syncwarp();
      if (prev >= 0) {
        mbar_wait(d2_full, (i - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int pimg = prev / p.tpi, ptr = prev - pimg * p.tpi;
        const int pty = ptr / p.tiles_x, ptx = ptr - pty * p.tiles_x;
        float* pout = p.out + pimg * p.out_img;
        float* plat = p.lat ? p.lat + pimg * p.lat_img : nullptr;
        float partv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        epi2_rows<4, false>(tlane + BT_HID + 128 + hh * 32, hh * 32, nullptr, pout, pty * BT_TY + q, p.ho, ptx * BT_TX,
                            p.wo, b2s, wms, partv, lane);
        if (plat) {
          epi2_partials(partv, mp, hh, q, lane);
          epi_sync();
          const int te = e * 32 + lane;
          if (te < 128) {
            const int oy3 = pty * BT_TY + (te >> 5), ox3 = ptx * BT_TX + (te & 31);
            if (oy3 < p.ho && ox3 < p.wo) plat[(int64_t)oy3 * p.wo + ox3] = (mp[te] + mp[128 + te]) + bm;
          }
        }
      }
      if (!has) break;
      mbar_wait(d1_full, i & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
      for (int cc = 0; cc < 4; cc++) {
        const int col = hh * 128 + cc * 32;
        float v[32];
        tmem_row<32>(tlane + col, v);
        uint32_t hv[16];
#pragma unroll
        for (int j = 0; j < 16; j++)
          hv[j] = pack_h2(fmaxf(v[2 * j] + b1s[col + 2 * j], 0.0f), fmaxf(v[2 * j + 1] + b1s[col + 2 * j + 1], 0.0f));
        tmem_st16(tlane + BT_HID + (col >> 1), hv);
      }
      tmem_wait_st();
      asm volatile("tcgen05.fence::before_thread_sync;");
      epi_sync();
      if (leader) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int k = 0; k < 16; k++)
          mma_f16_ts(tmem_d2, tmem_h + 8 * k, umma_desc_sw128(su + S::W2 + (k >> 2) * (BT_C * 128) + (k & 3) * 32),
                     h16_idesc(BT_C), k > 0);
        const uint32_t ap_u = su + S::AP + (i & 1) * (128 * BT_C * 2);
#pragma unroll
        for (int k = 0; k < 4; k++)  // identity branch: pool x Wid^T (K = 64)
          mma_f16(tmem_d2, umma_desc_sw128(ap_u + k * 32), umma_desc_sw128(su + S::WID + k * 32), h16_idesc(BT_C), 1);
        mma_commit(d2_full);
        mma_commit(a_empty + (i & 1));  // A and AP of this tile are consumed
      }
      __syncwarp();
      prev = tile;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static int launch_block_h16(const BlockTcParams& p, int n_img, int sm_count, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(an_block_h16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H16Smem::TOTAL) !=
        cudaSuccess)
      return -1;
    attr = true;
  }
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return -1;
  H16Params hp;
  hp.p = p;
  const cuuint64_t dims[4] = {(cuuint64_t)BT_C, (cuuint64_t)p.w, (cuuint64_t)p.h, (cuuint64_t)n_img};
  const cuuint64_t strides[3] = {(cuuint64_t)BT_C * 4, (cuuint64_t)p.w * BT_C * 4, (cuuint64_t)p.h * p.w * BT_C * 4};
  const cuuint32_t box[4] = {(cuuint32_t)HS_CH, (cuuint32_t)HS_COLS, (cuuint32_t)HS_ROWS, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  if (enc(&hp.tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(p.in), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  const int grid = p.n_tiles < sm_count ? p.n_tiles : sm_count;
  an_block_h16_kernel<<<grid, BT_THREADS, H16Smem::TOTAL, s>>>(hp);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------- launcher
template <bool DOWN>
static int launch_block_tc(const BlockTcParams& p, int sm_count, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(an_block_tc_kernel<DOWN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)BtSmem<DOWN>::TOTAL) != cudaSuccess)
      return -1;
    attr = true;
  }
  const int grid = p.n_tiles < sm_count ? p.n_tiles : sm_count;
  an_block_tc_kernel<DOWN><<<grid, BT_THREADS, BtSmem<DOWN>::TOTAL, s>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

int analysis_block_tc(int mode, bool down, const float* in, float* out, const float* blk, const float* wm, float* lat,
                      int h, int w, int ho, int wo, int n_img, int64_t lat_img, int sm_count, cudaStream_t s) {
  BlockTcParams p;
  p.in = in;
  p.out = out;
  p.blk = blk;
  p.wm = wm;
  p.lat = lat;
  p.h = h;
  p.w = w;
  p.ho = ho;
  p.wo = wo;
  p.tiles_x = (wo + BT_TX - 1) / BT_TX;
  p.tpi = p.tiles_x * ((ho + BT_TY - 1) / BT_TY);
  p.n_tiles = p.tpi * n_img;
  p.in_img = (int64_t)h * w * BT_C;
  p.out_img = (int64_t)ho * wo * BT_C;
  p.lat_img = lat_img;
  if (down && mode == 3) {
    static bool attr_d = false;
    if (!attr_d) {
      if (cudaFuncSetAttribute(an_block_h16d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H16dSmem::TOTAL) !=
          cudaSuccess)
        return -1;
      attr_d = true;
    }
    const int grid = p.n_tiles < sm_count ? p.n_tiles : sm_count;
    an_block_h16d_kernel<<<grid, BT_THREADS, H16dSmem::TOTAL, s>>>(p);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
  }
  if (down) return launch_block_tc<true>(p, sm_count, s);
  if (mode == 3) return launch_block_h16(p, n_img, sm_count, s);
  static const bool seq = getenv("CCRD_AN_SEQ") && getenv("CCRD_AN_SEQ")[0] == '1';  // A/B: sequential kernel
  if (seq) return launch_block_tc<false>(p, sm_count, s);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(an_block_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WsSmem::TOTAL) !=
        cudaSuccess)
      return -1;
    attr = true;
  }
  const int grid = p.n_tiles < sm_count ? p.n_tiles : sm_count;
  an_block_ws_kernel<<<grid, BT_THREADS, WsSmem::TOTAL, s>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace ccrd
