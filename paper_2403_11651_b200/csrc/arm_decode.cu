// arm_decode.cu -- NEXT-3: the decoder's autoregressive ARM as a wavefront on
// the GPU (the decoder recovers the latents one by
// one, the ARM conditioning each on already decoded neighbours; SURVEY.md
// 8(f) NEXT-3 "wavefront-parallel autoregressive ARM (anti-diagonal schedule
// over the causal template) emitting per-latent (mu, b)").
//
// Dependency: latent (i, j) of a grid needs the decoded latents at
// (i + dy, j + dx) for every context offset (dy < 0, or dy = 0 and dx < 0).
// With the skew a = 1 + max over dy < 0 of floor(dx / -dy), every context of
// (i, j) lies on an earlier step of t = a i + j, so the latents of one step
// are independent: step t evaluates all of them at once (anti-diagonal
// wavefront), T = a (h - 1) + w steps per grid instead of h w.
//
// One launch per image (its ARM weights in the parameter bank: uniform FFMA2
// operands), one CTA per grid; thread k owns the rows r = k (mod threads).  The
// decoded values of the last 32 columns of each live row sit in a shared-memory
// ring (row r at ring row r mod RR, RR >= w/a + 5: no live row aliases a
// context row; a row's newest column is at most 3a + 4 < 32 ahead of any
// column read from it, so no slot is overwritten while still needed).  The
// ring starts POISONED (INT16_MIN, never a valid latent here): a context read
// of a latent not decoded yet is counted and corrupts (mu, b), so the parity
// tests catch any schedule error.  With a counter (CHECK), each row re-poisons
// its ring row when it starts and keeps the 8 slots ahead of its newest column
// poisoned, so this holds for every row and column, not only the first RR rows
// and 32 columns.  The entropy decoder (range coder) is out of
// scope: it is played by `truth` -- after (mu, b) of a latent exist, its value
// is revealed and written to the ring and to `decoded`.
//
// Arithmetic: the encoder's own code (arm_math.cuh: FFMA2 dense layers, folded
// residuals, Laplace -log2 P), one latent per thread: every latent's (mu,
// log-scale, bits) is bit-identical to cc_arm_rate's.
#include <cstring>
#include <vector>

#include "arm_math.cuh"
#include "ccrd_common.cuh"

namespace ccrd {

constexpr int DEC_THREADS = 512;
constexpr int DEC_STREAMS = 128;  // per image two launches (level 0 / the rest) on separate halves of a pool
constexpr int DEC_RING = 32;  // columns kept per live row
constexpr int DEC_PAD = ARM_HALO_X;  // |dx| <= 4
constexpr int DEC_RW = DEC_RING + 2 * DEC_PAD;  // ring row: physical column p holds logical column (p - 4) & 31
                                                // (the 4 columns at either end duplicated), so a context read
                                                // is (row constant + dx + 4) + (j & 31), never wrapping
constexpr int16_t DEC_POISON = INT16_MIN;

// One launch = one image: its ARM weights live in the kernel-parameter bank, so
// every FFMA2 takes them as uniform operands (no shared-memory traffic), as in
// the encoder's arm_rate_kernel.
template <int C, int NH, int NHL>
struct DecParams {
  ArmGeom g;        // level dims, Laplace clamps / floor (laplace_bits)
  int32_t a;        // wavefront skew
  int32_t rr_mask;  // ring rows - 1 (power of two)
  int8_t dy[CC_MAX_CTX], dx[CC_MAX_CTX];
  const int16_t* truth;  // the entropy decoder's answers, packed like the latents
  int16_t* decoded;
  float* mu;             // optional per-latent outputs
  float* scale;
  float* bits;
  double* partial;        // [L] per-grid rate of this image
  int32_t l0;             // first grid of this launch (CTA b runs grid l0 + b)
  int32_t* poison_reads;  // optional counter
  ArmWeights<C, NH, NHL> w;
};

// CHECK: count context reads of not-yet-decoded latents (tests pass a counter)
template <int C, int NH, int NHL, bool CHECK>
__global__ void __launch_bounds__(DEC_THREADS, 1)
    arm_decode_kernel(const __grid_constant__ DecParams<C, NH, NHL> p) {
  extern __shared__ int16_t ring[];  // [RR][DEC_RW]
  __shared__ float wsum[DEC_THREADS / 32];
  const int l = p.l0 + (int)blockIdx.x;
  const int nring = (p.rr_mask + 1) * DEC_RW;
  for (int i = threadIdx.x; i < nring; i += DEC_THREADS) ring[i] = DEC_POISON;
  __syncthreads();

  const int h = p.g.lv.h[l], w = p.g.lv.w[l], a = p.a;
  const int64_t off = p.g.lv.off[l];
  const int16_t* __restrict__ truth = p.truth + off;
  int16_t* decoded = p.decoded + off;
  const int T = a * (h - 1) + w;
  float bsum = 0.0f;
  int poison = 0;
  // per context, for the thread's current row: ring offset of (r + dy, j + dx)
  // minus (j & 31) -- recomputed only when the thread's row changes
  int cached_r = -1;
  int roff[C];
#pragma unroll 1
  for (int s = 0; s < T; s++) {
    // rows on this step: 0 <= s - a r < w
    const int r_lo = s - w + 1 <= 0 ? 0 : (s - w + a) / a;
    const int r_hi = min(h - 1, s / a);
    int r = r_lo + (((int)threadIdx.x - r_lo) % DEC_THREADS + DEC_THREADS) % DEC_THREADS;
#pragma unroll 1
    for (; r <= r_hi; r += DEC_THREADS) {
      const int j = s - a * r;
      const int64_t q = (int64_t)r * w + j;
      // the entropy decoder's answer, loaded now (used only after (mu, b) exist)
      // so its memory latency hides under the MLP
      const int16_t yv = truth[q];
      float z0[1][C];
      if (r >= ARM_HALO_TOP && j >= ARM_HALO_X && j + ARM_HALO_X < w) {
        // interior (every context in the grid: no bounds checks)
        if (r != cached_r) {
#pragma unroll
          for (int c = 0; c < C; c++) roff[c] = ((r + p.dy[c]) & p.rr_mask) * DEC_RW + DEC_PAD + p.dx[c];
          cached_r = r;
        }
        const int16_t* rj = ring + (j & (DEC_RING - 1));
#pragma unroll
        for (int c = 0; c < C; c++) {
          const int16_t q = rj[roff[c]];
          if constexpr (CHECK) poison += (q == DEC_POISON);
          z0[0][c] = (float)q;
        }
      } else {
#pragma unroll
        for (int c = 0; c < C; c++) {
          const int rr = r + p.dy[c], jj = j + p.dx[c];
          float v = 0.0f;
          if (rr >= 0 && jj >= 0 && jj < w) {
            const int16_t q = ring[(rr & p.rr_mask) * DEC_RW + (jj & (DEC_RING - 1)) + DEC_PAD];
            if constexpr (CHECK) poison += (q == DEC_POISON);
            v = (float)q;
          }
          z0[0][c] = v;
        }
      }
      float z[1][NH];
      dense_ffma2<1, C, NH / 2, true>(z0, z, p.w.w0, p.w.b0);
#pragma unroll
      for (int k = 0; k < NHL - 1; k++) {
        float zn[1][NH];
        dense_ffma2<1, NH, NH / 2, true>(z, zn, p.w.wh[k], p.w.bh[k]);
#pragma unroll
        for (int n = 0; n < NH; n++) z[0][n] = zn[0][n];
      }
      uint64_t o = ldp2(p.w.bo);
#pragma unroll
      for (int n = 0; n < NH; n++) o = ffma2(f2pack(z[0][n], z[0][n]), ldp2(p.w.wo[n]), o);
      const float2 ms = f2unpack(o);
      const float bt = laplace_bits((float)yv, ms.x, ms.y, p.g);
      bsum += bt;
      {
        int16_t* row = ring + (r & p.rr_mask) * DEC_RW;
        if constexpr (CHECK) {
          // keep the poison meaningful past the first RR rows and 32 columns:
          // the ring row of row r last held row r - RR, dead once row r starts
          // (RR >= w/a + 6), so row r's first latent re-poisons all of it ...
          if (j == 0)
            for (int k = 0; k < DEC_RW; k++) row[k] = DEC_POISON;
        }
        const int lc = j & (DEC_RING - 1);
        int16_t* rw = row + lc + DEC_PAD;
        rw[0] = yv;
        if (lc >= DEC_RING - DEC_PAD) rw[-DEC_RING] = yv;  // left pad
        if (lc < DEC_PAD) rw[DEC_RING] = yv;               // right pad
        if constexpr (CHECK) {
          // ... and every latent poisons the slot 8 columns ahead (it holds
          // column j - 24; readers of this row are at columns >= j - 3a - 4 >
          // j - 24 for a <= 6), so columns j+1 .. j+8 of the row are always
          // poison until decoded: a premature read near the wavefront counts
          if (p.a <= 6) {
            const int pc = (j + 8) & (DEC_RING - 1);
            int16_t* pw = row + pc + DEC_PAD;
            pw[0] = DEC_POISON;
            if (pc >= DEC_RING - DEC_PAD) pw[-DEC_RING] = DEC_POISON;
            if (pc < DEC_PAD) pw[DEC_RING] = DEC_POISON;
          }
        }
      }
      decoded[q] = yv;
      if (p.bits) p.bits[off + q] = bt;
      if (p.mu) p.mu[off + q] = ms.x;
      if (p.scale) p.scale[off + q] = __expf(fminf(fmaxf(ms.y, p.g.lsmin), p.g.lsmax));
    }
    __syncthreads();  // step s's ring writes before step s + 1's reads
  }
  if (CHECK && p.poison_reads && poison) atomicAdd(p.poison_reads, poison);
  // CTA rate partial, fixed order
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o2);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = bsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < DEC_THREADS / 32; k++) t += (double)wsum[k];
    p.partial[l] = t;
  }
}

// rate[i] = sum over the grids of image i, level order
__global__ void dec_rate_kernel(const double* __restrict__ partial, int L, int n, double* __restrict__ rate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = 0.0;
  for (int l = 0; l < L; l++) t += partial[i * L + l];
  rate[i] = t;
}

// ---------------------------------------------------------------- host side
int dec_skew(const cc_model_desc& d) {
  int a = 1;
  for (int c = 0; c < d.n_ctx; c++)
    if (d.ctx_dy[c] < 0) {
      const int dy = -d.ctx_dy[c], dx = d.ctx_dx[c];
      const int need = (dx >= 0 ? dx / dy : -((-dx + dy - 1) / dy)) + 1;  // floor(dx / dy) + 1
      if (need > a) a = need;
    }
  return a;
}

static int ring_rows(const cc_model_desc& d, int a, int w0) {
  int rr = 1;
  while (rr < w0 / a + 6) rr <<= 1;
  (void)d;
  return rr;
}

size_t dec_workspace_bytes(const cc_model_desc& d, int n_img) {
  return (size_t)n_img * d.L * sizeof(double) + 256;  // per-grid rate partials
}

// a pool of streams for the per-image launches (joined back to the caller's)
struct DecStreams {
  cudaStream_t s[DEC_STREAMS] = {};
  cudaEvent_t ev[DEC_STREAMS + 1] = {};
  int device = -1;
};
static thread_local DecStreams g_dec;

static int dec_streams(DecStreams** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (g_dec.device != dev) {
    for (int k = 0; k < DEC_STREAMS; k++)
      if (cudaStreamCreateWithFlags(&g_dec.s[k], cudaStreamNonBlocking) != cudaSuccess) return -1;
    for (int k = 0; k <= DEC_STREAMS; k++)
      if (cudaEventCreateWithFlags(&g_dec.ev[k], cudaEventDisableTiming) != cudaSuccess) return -1;
    g_dec.device = dev;
  }
  *out = &g_dec;
  return 0;
}

template <int C, int NH, int NHL>
static int launch_dec(const cc_model_desc& d, const ArmGeom& g, int a_override, int n_img,
                      const int16_t* const* truth, const float* const* arm_w, int16_t* const* decoded,
                      float* const* mu, float* const* scale, float* const* bits, double* rate, int32_t* poison,
                      void* ws, cudaStream_t s) {
  DecParams<C, NH, NHL> p;
  memset(&p, 0, sizeof(p));
  p.g = g;
  p.a = a_override > 0 ? a_override : dec_skew(d);
  const int rr = ring_rows(d, p.a, g.lv.w[0]);
  p.rr_mask = rr - 1;
  for (int c = 0; c < d.n_ctx; c++) {
    p.dy[c] = d.ctx_dy[c];
    p.dx[c] = d.ctx_dx[c];
  }
  p.poison_reads = poison;
  const size_t smem = (size_t)rr * DEC_RW * sizeof(int16_t);
  if (smem > 200 * 1024) return -2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(arm_decode_kernel<C, NH, NHL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(arm_decode_kernel<C, NH, NHL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  DecStreams* ps = nullptr;
  if (dec_streams(&ps)) return -1;
  double* part = reinterpret_cast<double*>(ws);
  cudaEventRecord(ps->ev[DEC_STREAMS], s);  // fork after the caller's queued work
  const int half = DEC_STREAMS / 2;
  const int ns = n_img < half ? n_img : half;  // streams per pass
  for (int k = 0; k < ns; k++) {
    cudaStreamWaitEvent(ps->s[k], ps->ev[DEC_STREAMS], 0);
    cudaStreamWaitEvent(ps->s[half + k], ps->ev[DEC_STREAMS], 0);
  }
  // every image's level-0 grid first (the longest wavefront: T = a (h - 1) + w
  // steps on one SM), then the smaller grids fill the remaining SMs -- with
  // all of an image's grids in one launch the block scheduler interleaved them
  // and most level-0 grids started late (64 x 2K: 50 -> see DESIGN 8.3.1)
  for (int pass = 0; pass < 2; pass++) {
    if (pass == 1 && d.L < 2) break;
    for (int i = 0; i < n_img; i++) {
      pack_arm_weights<C, NH, NHL>(d, arm_w[i], p.w);
      p.truth = truth[i];
      p.decoded = decoded[i];
      p.mu = mu ? mu[i] : nullptr;
      p.scale = scale ? scale[i] : nullptr;
      p.bits = bits ? bits[i] : nullptr;
      p.partial = part + (size_t)i * d.L;
      p.l0 = pass == 0 ? 0 : 1;
      auto kern = poison ? arm_decode_kernel<C, NH, NHL, true> : arm_decode_kernel<C, NH, NHL, false>;
      kern<<<pass == 0 ? 1 : d.L - 1, DEC_THREADS, smem, ps->s[pass * half + i % ns]>>>(p);
    }
  }
  for (int k = 0; k < ns; k++) {  // join both passes' streams
    cudaEventRecord(ps->ev[k], ps->s[k]);
    cudaStreamWaitEvent(s, ps->ev[k], 0);
    cudaEventRecord(ps->ev[half + k], ps->s[half + k]);
    cudaStreamWaitEvent(s, ps->ev[half + k], 0);
  }
  dec_rate_kernel<<<(n_img + 127) / 128, 128, 0, s>>>(part, d.L, n_img, rate);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

typedef int (*DecLaunchFn)(const cc_model_desc&, const ArmGeom&, int, int, const int16_t* const*, const float* const*,
                           int16_t* const*, float* const*, float* const*, float* const*, double*, int32_t*, void*,
                           cudaStream_t);
struct DecEntry {
  int C, NH, NHL;
  DecLaunchFn fn;
};
static const DecEntry kDec[] = {
    {8, 8, 1, launch_dec<8, 8, 1>},     {8, 8, 2, launch_dec<8, 8, 2>},
    {16, 16, 2, launch_dec<16, 16, 2>}, {16, 24, 2, launch_dec<16, 24, 2>},
    {24, 24, 2, launch_dec<24, 24, 2>},
};

// Returns launches (n_img + 1) or a negative code (-3: ARM shape not compiled,
// -2: ring exceeds shared memory).
int arm_decode_impl(const cc_model_desc& d, const ArmGeom& g, int a_override, int n_img, const int16_t* const* truth,
                    const float* const* arm_w, int16_t* const* decoded, float* const* mu, float* const* scale,
                    float* const* bits, double* rate, int32_t* poison, void* ws, cudaStream_t s) {
  const int NH = d.arm_widths[1], NHL = d.arm_n_layers - 1;
  for (const auto& e : kDec)
    if (e.C == d.n_ctx && e.NH == NH && e.NHL == NHL) {
      const int rc = e.fn(d, g, a_override, n_img, truth, arm_w, decoded, mu, scale, bits, rate, poison, ws, s);
      return rc < 0 ? rc : (d.L > 1 ? 2 : 1) * n_img + 1;
    }
  return -3;
}

}  // namespace ccrd
