// ccrd_api.cu -- the C ABI (include/ccrd.h): validation, geometry, dispatch to
// the compiled kernel shapes, the deterministic fp64 reduction kernel, the
// host-buffer (end-to-end) path and the MAC closed form.
#include <cstdarg>
#include <cstdlib>
#include <vector>
#include <cstdio>
#include <atomic>
#include <cstring>

#include "ccrd_common.cuh"

namespace ccrd {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

// ---- optional per-kernel event timing (cc_profile_begin / cc_profile_end)
enum { PK_ARM = 0, PK_SYN = 1, PK_RED = 2, PK_PYR = 3 };
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};
struct ProfState {
  bool on = false;
  ProfRec* recs = nullptr;
  int n = 0, cap = 0;
  cudaEvent_t* pool = nullptr;  // reusable events
  int pool_n = 0, pool_used = 0;
};
static thread_local ProfState g_prof;

static cudaEvent_t prof_event() {
  ProfState& P = g_prof;
  if (P.pool_used == P.pool_n) {
    int nn = P.pool_n ? 2 * P.pool_n : 256;
    cudaEvent_t* np = new cudaEvent_t[nn];
    for (int i = 0; i < P.pool_n; i++) np[i] = P.pool[i];
    for (int i = P.pool_n; i < nn; i++) cudaEventCreate(&np[i]);
    delete[] P.pool;
    P.pool = np;
    P.pool_n = nn;
  }
  return P.pool[P.pool_used++];
}

// RAII bracket around one launch
struct ProfScope {
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(int k, cudaStream_t st) : kind(k), s(st) {
    if (g_prof.on) {
      a = prof_event();
      cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (!a) return;
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, s);
    ProfState& P = g_prof;
    if (P.n == P.cap) {
      int nc = P.cap ? 2 * P.cap : 256;
      ProfRec* nr = new ProfRec[nc];
      for (int i = 0; i < P.n; i++) nr[i] = P.recs[i];
      delete[] P.recs;
      P.recs = nr;
      P.cap = nc;
    }
    P.recs[P.n++] = ProfRec{kind, a, b};
  }
};

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

static int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CC_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return CC_OK;
}

// ------------------------------------------------------------- descriptor
static int32_t ceil_shift(int64_t v, int l) { return (int32_t)((v + ((int64_t)1 << l) - 1) >> l); }

// Level dimensions; `win` (a strip) sets the buffer window of every grid
// (nullptr: the full image, window = the whole grid).
static void level_dims(const cc_model_desc& d, const cc_strip* win, LevelGeom& g, int64_t* n_lat) {
  int64_t off = 0;
  for (int l = 0; l < CC_MAX_LEVELS; l++) {
    if (l < d.L) {
      g.h[l] = ceil_shift(d.H, l);
      g.w[l] = ceil_shift(d.W, l);
      g.lo[l] = win ? win->lo[l] : 0;
      g.hi[l] = win ? win->hi[l] : g.h[l];
      g.off[l] = off;
      off += (int64_t)(g.hi[l] - g.lo[l]) * g.w[l];
    } else {
      g.h[l] = g.w[l] = g.lo[l] = g.hi[l] = 0;
      g.off[l] = off;
    }
  }
  if (n_lat) *n_lat = off;
}
static void level_dims(const cc_model_desc& d, LevelGeom& g, int64_t* n_lat) { level_dims(d, nullptr, g, n_lat); }

// The strip of pixel rows [r0, r1): owned latent rows and the minimal buffer
// window (include/ccrd.h "strips").  Assumes a valid descriptor.
static void strip_window(const cc_model_desc& d, int r0, int r1, cc_strip& st) {
  memset(&st, 0, sizeof(st));
  st.r0 = r0;
  st.r1 = r1;
  int maxdy = 0;
  for (int c = 0; c < d.n_ctx; c++) maxdy = (-d.ctx_dy[c] > maxdy) ? -d.ctx_dy[c] : maxdy;
  // synthesis receptive field: R residual 3x3 layers at level 0, then one x2
  // step per level (sources floor(y/2) - K/4 .. floor(y/2) + K/4)
  int a = r0 - d.syn_n_res, b = r1 - 1 + d.syn_n_res;  // inclusive rows
  for (int l = 0; l < d.L; l++) {
    const int h = ceil_shift(d.H, l);
    if (l > 0) {
      a = (a >> 1) - d.up_taps / 4;  // arithmetic shift = floor
      b = (b >> 1) + d.up_taps / 4;
    }
    a = a < 0 ? 0 : a;
    b = b > h - 1 ? h - 1 : b;
    st.own_lo[l] = ceil_shift(r0, l);
    st.own_hi[l] = ceil_shift(r1, l);
    int lo = a, hi = b + 1;
    if (st.own_hi[l] > st.own_lo[l]) {  // ARM: the context rows above the owned rows
      const int alo = st.own_lo[l] - maxdy < 0 ? 0 : st.own_lo[l] - maxdy;
      lo = alo < lo ? alo : lo;
      hi = st.own_hi[l] > hi ? st.own_hi[l] : hi;
    }
    st.lo[l] = lo;
    st.hi[l] = hi;
  }
}

static void full_strip(const cc_model_desc& d, cc_strip& st) {
  memset(&st, 0, sizeof(st));
  st.r0 = 0;
  st.r1 = d.H;
  for (int l = 0; l < d.L; l++) {
    st.own_lo[l] = st.lo[l] = 0;
    st.own_hi[l] = st.hi[l] = ceil_shift(d.H, l);
  }
}

// SM count of the current device (lazily cached device attribute; 148 = B200
// when no device is visible).  Sizes the persistent grids.
int device_sm_count() {
  static thread_local int dev_cached = -2, sms = 148;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  if (dev != dev_cached) {
    int n = 0;
    if (dev < 0 || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cudaGetLastError();
    sms = n;
    dev_cached = dev;
  }
  return sms;
}

// ARM path (cc_set_arm_path; initial value from CCRD_ARM_PATH = ffma2 | tc):
// AUTO = the tensor-core kernel (arm_tc.cu) where it measured faster (below),
// the FFMA2 kernel (arm_rate.cu) elsewhere; FFMA2 / TC force a path (TC for
// the shapes it is compiled for).
static std::atomic<int> g_arm_path{-1};
static int arm_path() {
  int v = g_arm_path.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("CCRD_ARM_PATH");
    v = (e && strcmp(e, "ffma2") == 0) ? CC_ARM_FFMA2 : (e && strcmp(e, "tc") == 0) ? CC_ARM_TC : CC_ARM_AUTO;
    int expect = -1;
    g_arm_path.compare_exchange_strong(expect, v);
    v = g_arm_path.load();
  }
  return v;
}
static bool arm_use_tc(const cc_model_desc& d) {
  const int path = arm_path();
  if (path == CC_ARM_FFMA2 || find_arm_tc_launcher(d.n_ctx, d.arm_widths[1], d.arm_n_layers - 1) == nullptr)
    return false;
  // AUTO: where the tensor-core kernel measured faster -- the [16,24,24,2] ARM
  // (2K: 91 vs 140 us; 512x768: 28 vs 27 us with a faster two-stream path).
  // The Table 1 [16,16,16,2] / [24,24,24,2] ARMs on 512x768 images measured
  // slower on the tensor cores (path 8.7e9 vs 9.8e9, 6.5e9 vs 6.9e9 px/s).
  if (path == CC_ARM_AUTO) return d.n_ctx == 16 && d.arm_widths[1] == 24;
  return true;
}
// Synthesis path (cc_set_synth_path; initial value from CCRD_SYN_PATH =
// ffma2 | mma | tma): AUTO = TMA where it applies, else FFMA2 (the warp-MMA
// form measured slower); MMA = layer 0 on warp MMAs wherever
// synth.cu has that form; TMA = FFMA2 arithmetic, persistent CTAs with
// TMA-staged tiles.
static std::atomic<int> g_syn_path{-1};
int synth_path() {
  int v = g_syn_path.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("CCRD_SYN_PATH");
    v = (e && strcmp(e, "ffma2") == 0) ? CC_SYN_FFMA2
        : (e && strcmp(e, "mma") == 0) ? CC_SYN_MMA
        : (e && strcmp(e, "tma") == 0) ? CC_SYN_TMA
                                        : CC_SYN_AUTO;
    int expect = -1;
    g_syn_path.compare_exchange_strong(expect, v);
    v = g_syn_path.load();
  }
  return v;
}
thread_local LaunchCtl g_launch_ctl;
bool pdl_enabled() {
  static const bool on = !(getenv("CCRD_PDL") && getenv("CCRD_PDL")[0] == '0');
  return on;
}
static ArmLaunchFn arm_launcher(const cc_model_desc& d) {
  return arm_use_tc(d) ? find_arm_tc_launcher(d.n_ctx, d.arm_widths[1], d.arm_n_layers - 1)
                       : find_arm_launcher(d.n_ctx, d.arm_widths[1], d.arm_n_layers - 1);
}
static int arm_partials_per_tile(const cc_model_desc& d) { return arm_use_tc(d) ? arm_tc_partials_per_tile() : ARM_TY; }
constexpr int ARM_PARTIALS_CAP = 16;  // per tile, any path: the workspace layout does not depend on the path

static int validate(const cc_model_desc* dp) {
  if (!dp) return fail(CC_EINVAL, "null descriptor");
  const cc_model_desc& d = *dp;
  if (d.H < 1 || d.W < 1) return fail(CC_EINVAL, "H, W must be >= 1 (got %d x %d)", d.H, d.W);
  if ((int64_t)d.H * d.W > ((int64_t)1 << 31)) return fail(CC_ENOTSUP, "image larger than 2^31 pixels");
  if (d.L < 1 || d.L > CC_MAX_LEVELS) return fail(CC_EINVAL, "L must be in 1..%d (got %d)", CC_MAX_LEVELS, d.L);
  if (d.image_u8 != 0 && d.image_u8 != 1) return fail(CC_EINVAL, "image_u8 must be 0 or 1 (got %d)", d.image_u8);
  if (d.latents_i8 != 0 && d.latents_i8 != 1) return fail(CC_EINVAL, "latents_i8 must be 0 or 1 (got %d)", d.latents_i8);
  if (d.n_ctx < 1 || d.n_ctx > CC_MAX_CTX) return fail(CC_EINVAL, "n_ctx must be in 1..%d", CC_MAX_CTX);
  for (int c = 0; c < d.n_ctx; c++) {
    const int dy = d.ctx_dy[c], dx = d.ctx_dx[c];
    if (!(dy < 0 || (dy == 0 && dx < 0)))
      return fail(CC_EINVAL, "context offset %d (%d,%d) is not strictly causal", c, dy, dx);
    if (dy < -ARM_HALO_TOP || dx < -ARM_HALO_X || dx > ARM_HALO_X)
      return fail(CC_ENOTSUP, "context offset %d (%d,%d) outside the staged window (dy>=-3, |dx|<=4)", c, dy, dx);
    for (int e = 0; e < c; e++)
      if (d.ctx_dy[e] == dy && d.ctx_dx[e] == dx) return fail(CC_EINVAL, "duplicate context offset %d", c);
  }
  if (d.arm_n_layers < 2 || d.arm_n_layers > CC_MAX_LAYERS)
    return fail(CC_ENOTSUP, "arm_n_layers must be in 2..%d", CC_MAX_LAYERS);
  if (d.arm_widths[0] != d.n_ctx) return fail(CC_EINVAL, "arm_widths[0] (%d) != n_ctx (%d)", d.arm_widths[0], d.n_ctx);
  if (d.arm_widths[d.arm_n_layers] != 2) return fail(CC_EINVAL, "ARM must output 2 values (mu, log-scale)");
  for (int k = 0; k < d.arm_n_layers; k++) {
    if (d.arm_widths[k] < 1) return fail(CC_EINVAL, "ARM width %d < 1", k);
    if ((d.arm_residual_mask >> k) & 1u) {
      if (k == d.arm_n_layers - 1) return fail(CC_EINVAL, "residual on the last ARM layer");
      if (d.arm_widths[k] != d.arm_widths[k + 1]) return fail(CC_EINVAL, "residual ARM layer %d is not square", k);
    }
  }
  if (d.arm_residual_mask >> d.arm_n_layers) return fail(CC_EINVAL, "residual mask has bits past the last layer");
  for (int k = 2; k < d.arm_n_layers; k++)
    if (d.arm_widths[k] != d.arm_widths[1]) return fail(CC_ENOTSUP, "ARM hidden layers must share one width");
  if (d.up_taps != 4 && d.up_taps != 8) return fail(CC_ENOTSUP, "up_taps must be 4 or 8");
  if (d.up_2d != 0 && d.up_2d != 1) return fail(CC_EINVAL, "up_2d must be 0 or 1");
  if (d.syn_n_1x1 != 2) return fail(CC_ENOTSUP, "synthesis must have exactly two 1x1 layers");
  if (d.syn_widths[0] != d.L) return fail(CC_EINVAL, "syn_widths[0] (%d) != L (%d)", d.syn_widths[0], d.L);
  if (d.syn_widths[2] != 3) return fail(CC_EINVAL, "synthesis must output 3 channels");
  if (d.syn_widths[1] < 1) return fail(CC_EINVAL, "synthesis hidden width < 1");
  if (d.syn_n_res < 0 || d.syn_n_res > 3) return fail(CC_ENOTSUP, "syn_n_res must be in 0..3");
  if (!(d.logscale_min <= d.logscale_max)) return fail(CC_EINVAL, "logscale_min > logscale_max");
  if (!(d.p_floor > 0.0f && d.p_floor < 1.0f)) return fail(CC_EINVAL, "p_floor must be in (0, 1)");
  for (int l = 0; l < d.L; l++) {
    const int64_t s = (int64_t)1 << l;
    if ((d.H + s - 1) / s < 1 || (d.W + s - 1) / s < 1) return fail(CC_EINVAL, "level %d has zero size", l);
  }
  if (!find_arm_launcher(d.n_ctx, d.arm_widths[1], d.arm_n_layers - 1))
    return fail(CC_ENOTSUP, "ARM shape (C=%d, hidden=%d x %d) not compiled", d.n_ctx, d.arm_widths[1],
                d.arm_n_layers - 1);
  if (!find_syn_launcher(d.L, d.syn_widths[1], d.syn_n_res, d.up_taps))
    return fail(CC_ENOTSUP, "synthesis shape (L=%d, C_h=%d, R=%d, K=%d) not compiled", d.L, d.syn_widths[1],
                d.syn_n_res, d.up_taps);
  return CC_OK;
}

static void arm_geom(const cc_model_desc& d, const cc_strip* win, ArmGeom& g) {
  memset(&g, 0, sizeof(g));
  level_dims(d, win, g.lv, nullptr);
  g.L = d.L;
  int acc = 0;
  for (int l = 0; l < CC_MAX_LEVELS; l++) {
    g.tile_begin[l] = acc;
    if (l < d.L) {
      g.own_lo[l] = win ? win->own_lo[l] : 0;
      g.own_hi[l] = win ? win->own_hi[l] : g.lv.h[l];
      g.tiles_x[l] = (g.lv.w[l] + ARM_TX - 1) / ARM_TX;
      const int64_t nt = (int64_t)g.tiles_x[l] * ((g.own_hi[l] - g.own_lo[l] + ARM_TY - 1) / ARM_TY);
      // m = ceil(2^32 / d), e = m d - 2^32 < d: floor(n m / 2^32) = floor(n / d)
      // for n e < 2^32, which n < nt, nt d < 2^32 guarantees
      const uint64_t dx = (uint64_t)(g.tiles_x[l] > 0 ? g.tiles_x[l] : 1);
      g.tx_mul[l] = (dx > 1 && (uint64_t)nt * dx < (1ull << 32)) ? (uint32_t)(((1ull << 32) + dx - 1) / dx) : 0u;
      acc += (int)nt;
    }
  }
  g.tile_begin[CC_MAX_LEVELS] = acc;
  g.tile_begin[d.L] = acc;
  for (int c = 0; c < d.n_ctx; c++) g.ctx_off[c] = d.ctx_dy[c] * ARM_SW + d.ctx_dx[c];
  g.lsmin = d.logscale_min;
  g.lsmax = d.logscale_max;
  g.p_floor = d.p_floor;
  g.bits_cap = (float)(-log2((double)d.p_floor));
}

static void syn_geom(const cc_model_desc& d, const cc_strip* win, SynGeom& g) {
  memset(&g, 0, sizeof(g));
  level_dims(d, win, g.lv, nullptr);
  g.H = d.H;
  g.W = d.W;
  g.y0 = win ? win->r0 : 0;
  g.y1 = win ? win->r1 : d.H;
  g.tiles_x = (d.W + SYN_TW - 1) / SYN_TW;
  g.n_tiles = g.tiles_x * ((g.y1 - g.y0 + SYN_TH - 1) / SYN_TH);
}

static int n_arm_partials(const cc_model_desc& d, const cc_strip* win) {  // written by the current path
  ArmGeom g;
  arm_geom(d, win, g);
  return g.tile_begin[d.L] * arm_partials_per_tile(d);
}
static int n_arm_cap(const cc_model_desc& d, const cc_strip* win) {  // reserved (synthesis partials follow)
  ArmGeom g;
  arm_geom(d, win, g);
  return g.tile_begin[d.L] * ARM_PARTIALS_CAP + ARM_W_SCRATCH_DOUBLES;  // + the tensor-core ARM's weight scratch
}
static int n_syn_ctas(const cc_model_desc& d, const cc_strip* win) {
  SynGeom g;
  syn_geom(d, win, g);
  return g.n_tiles;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static void pyr_geom(const cc_model_desc& d, const cc_strip* win, PyrGeom& g) {
  memset(&g, 0, sizeof(g));
  level_dims(d, win, g.lv, nullptr);
  g.L = d.L;
  int64_t off = 0;
  for (int j = 1; j + 1 < d.L; j++) {  // S_j: grids j+1 .. L-1 at level j, over the window rows
    g.s_off[j] = off;
    off += (int64_t)(d.L - 1 - j) * (g.lv.hi[j] - g.lv.lo[j]) * g.lv.w[j];
    off = (off + 63) & ~(int64_t)63;
  }
  g.s_floats = off;
}

// Workspace per image: ARM partials + synthesis partials (fp64) + a result
// scratch slot used by the stage entries + the upsampling pyramid S_1..S_{L-2}
static size_t partial_bytes(const cc_model_desc& d, const cc_strip* win) {
  return align256(sizeof(double) * (size_t)(n_arm_cap(d, win) + n_syn_ctas(d, win))) +
         align256(sizeof(cc_rd_result));
}
// 2-D TConv (up_2d): the dense [L][H][W] level-0 tensor after the pyramid
static size_t dense_bytes(const cc_model_desc& d) {
  return d.up_2d ? align256(sizeof(float) * (size_t)d.L * d.H * d.W) : 0;
}
static size_t slice_bytes(const cc_model_desc& d, const cc_strip* win) {
  PyrGeom pg;
  pyr_geom(d, win, pg);
  return partial_bytes(d, win) + align256(sizeof(float) * (size_t)pg.s_floats) + dense_bytes(d);
}
static float* slice_dense(const cc_model_desc& d, const cc_strip* win, void* slice) {
  PyrGeom pg;
  pyr_geom(d, win, pg);
  return (float*)((char*)slice + partial_bytes(d, win) + align256(sizeof(float) * (size_t)pg.s_floats));
}
static float* slice_pyr(const cc_model_desc& d, const cc_strip* win, void* slice) {
  return (float*)((char*)slice + partial_bytes(d, win));
}

// ------------------------------------------------------------- reduction
// One CTA per image, fixed-order tree => bitwise deterministic.
// Kernel-parameter batch of reduction jobs (avoids a host->device copy).
constexpr int MAX_JOBS_PER_LAUNCH = 64;
struct ReduceBatch {
  ReduceJob j[MAX_JOBS_PER_LAUNCH];
};
// One job = one thread-block cluster of RED_CL CTAs on RED_CL SMs: CTA r sums
// the contiguous chunk r of the job's partials (thread t: elements t, t + 256,
// ... of the chunk, four loads in flight), a fixed-order tree in shared memory,
// then the leader adds the RED_CL chunk sums in rank order through distributed
// shared memory.  The grouping depends only on the partial counts, so the
// result is bitwise deterministic; one CTA per job (round 1) took 154 us for
// the 8K image's 377 K partials (7 % of its step), latency-bound on one SM.
constexpr int RED_CL = 8;
constexpr int RED_T = 256;
__device__ __forceinline__ double red_chunk(const double* __restrict__ v, int n, int r) {
  const int per = (n + RED_CL - 1) / RED_CL, lo = r * per, hi = min(n, lo + per);
  double a = 0.0;
  int i = lo + (int)threadIdx.x;
  for (; i + 3 * RED_T < hi; i += 4 * RED_T) {
    const double x0 = v[i], x1 = v[i + RED_T], x2 = v[i + 2 * RED_T], x3 = v[i + 3 * RED_T];
    a += x0;
    a += x1;
    a += x2;
    a += x3;
  }
  for (; i < hi; i += RED_T) a += v[i];
  return a;
}
__global__ void __cluster_dims__(RED_CL, 1, 1) __launch_bounds__(RED_T)
    reduce_batch_kernel(const __grid_constant__ ReduceBatch b, cc_rd_result* __restrict__ out) {
  __shared__ double sa[RED_T], ss[RED_T];
  const int job = blockIdx.x / RED_CL;
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  const ReduceJob& j = b.j[job];
  sa[threadIdx.x] = red_chunk(j.arm_partial, j.n_arm, (int)r);
  ss[threadIdx.x] = red_chunk(j.syn_partial, j.n_syn, (int)r);
  __syncthreads();
  for (int o = RED_T / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sa[threadIdx.x] += sa[threadIdx.x + o];
      ss[threadIdx.x] += ss[threadIdx.x + o];
    }
    __syncthreads();
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (r == 0 && threadIdx.x == 0) {
    double A = 0.0, S = 0.0;
    for (int k = 0; k < RED_CL; k++) {  // rank order
      uint32_t pa, ps;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(pa) : "r"((uint32_t)__cvta_generic_to_shared(sa)), "r"(k));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ps) : "r"((uint32_t)__cvta_generic_to_shared(ss)), "r"(k));
      double x, y;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(x) : "r"(pa));
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(y) : "r"(ps));
      A += x;
      S += y;
    }
    cc_rd_result res;
    res.rate_bits = A;
    res.sse = S;
    res.mse = S * j.inv_3p;
    res.cost = res.mse + j.lambda_over_p * A;
    out[job] = res;
  }
  // no CTA leaves while the leader reads its shared memory
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

static ReduceJob make_job(const cc_model_desc& d, const cc_strip* win, double* part) {
  ReduceJob j;
  j.n_arm = n_arm_partials(d, win);
  j.n_syn = n_syn_ctas(d, win);
  j.arm_partial = part;
  j.syn_partial = part + n_arm_cap(d, win);
  const double P = (double)d.H * (double)d.W;
  j.inv_3p = 1.0 / (3.0 * P);
  j.lambda_over_p = d.lambda / P;
  return j;
}

static int launch_reduce(const ReduceJob* jobs, int n, cc_rd_result* out, cudaStream_t s) {
  for (int b = 0; b < n; b += MAX_JOBS_PER_LAUNCH) {
    ReduceBatch rb;
    const int m = (n - b < MAX_JOBS_PER_LAUNCH) ? n - b : MAX_JOBS_PER_LAUNCH;
    for (int i = 0; i < m; i++) rb.j[i] = jobs[b + i];
    ProfScope ps(PK_RED, s);
    reduce_batch_kernel<<<m * RED_CL, RED_T, 0, s>>>(rb, out + b);
    g_launches++;
  }
  return cuda_check("reduce_batch_kernel");
}

static bool have_device(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

// ARM rate of one image (per-warp partials at the start of `part`)
static int arm_one(const cc_model_desc& d, const cc_strip* win, const int16_t* lat, const float* arm_w, double* part,
                   cudaStream_t s) {
  ArmGeom ag;
  arm_geom(d, win, ag);
  if (ag.tile_begin[d.L] == 0) return CC_OK;  // a strip owning no latent rows
  {
    ProfScope ps(PK_ARM, s);
    arm_launcher(d)(ag, d, arm_w, lat, part, nullptr, nullptr,
                                                                    nullptr, s);
  }
  g_launches++;
  return cuda_check("arm_rate_kernel");
}

// every image's ARM weights to its scratch before the batch's first ARM kernel
// (ARM_STAGE_ONLY), so the ARM kernels follow one another in the stream
static int arm_stage_all(const cc_model_desc& d, const cc_strip* win, const int16_t* const* lat,
                         const float* const* arm_w, char* slices, size_t per, int n, cudaStream_t s) {
  ArmGeom ag;
  arm_geom(d, win, ag);
  if (ag.tile_begin[d.L] == 0) return CC_OK;
  LaunchCtlScope lc(false, ARM_STAGE_ONLY);
  const ArmLaunchFn fn = arm_launcher(d);
  for (int i = 0; i < n; i++)
    if (fn(ag, d, arm_w[i], lat[i], (double*)(slices + per * (size_t)i), nullptr, nullptr, nullptr, s) < 0)
      return fail(CC_ECUDA, "ARM weight staging copy failed");
  return cuda_check("ARM weight staging");
}

// coarse upsampling pyramid of n images (batched launches)
static int pyr_many(const cc_model_desc& d, const cc_strip* win, const PyrImage* imgs, int n, cudaStream_t s) {
  PyrGeom pg;
  pyr_geom(d, win, pg);
  {
    ProfScope ps(PK_PYR, s);
    launch_pyramid(pg, d.up_taps, imgs, n, s);
  }
  g_launches += pyramid_launch_count(pg, n);
  return cuda_check("pyramid_kernel");
}

// fused last upsampling step + synthesis + distortion of one image
static int syn_one(const cc_model_desc& d, const cc_strip* win, const int16_t* lat, const float* s1,
                   const float* up_w, const float* syn_w, const float* image, float* x_hat, float* dense_out,
                   double* syn_part, cudaStream_t s, uint8_t* out_u8 = nullptr) {
  SynGeom sg;
  syn_geom(d, win, sg);
  {
    ProfScope ps(PK_SYN, s);
    find_syn_launcher(d.L, d.syn_widths[1], d.syn_n_res, d.up_taps)(sg, d, up_w, syn_w, lat, s1, nullptr, image,
                                                                    x_hat, dense_out, nullptr, syn_part, s, out_u8);
  }
  g_launches++;
  return cuda_check("synth_kernel");
}

static PyrImage pyr_image(const cc_model_desc& d, const int16_t* lat, const float* up_w, float* S) {
  PyrImage im;
  im.lat = lat;
  im.S = S;
  for (int t = 0; t < 8; t++) im.k[t] = t < d.up_taps ? up_w[t] : 0.0f;
  return im;
}

// Side stream for the upsampling pyramid (lazily created, one per host
// thread): the pyramid is latency-bound and independent of the ARM, so it runs
// concurrently with the ARM launches and is joined before the synthesis.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int device = -1;
};
static thread_local SideStream g_side;

static int side_stream(SideStream** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  if (g_side.s == nullptr || g_side.device != dev) {
    if (cudaStreamCreateWithFlags(&g_side.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_side.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_side.join, cudaEventDisableTiming) != cudaSuccess)
      return cuda_check("side stream");
    g_side.device = dev;
  }
  *out = &g_side;
  return CC_OK;
}

// ARM || (pyramid -> synthesis) on two streams (default, measured +10 % on
// the batched 2K workload); CCRD_SERIAL=1 runs everything on the caller's
// stream (per-kernel timing; read at every call)
static bool concurrent_streams() {
  const char* e = getenv("CCRD_SERIAL");
  return !(e && strcmp(e, "1") == 0);
}

// whole path for images [0, n): pyramid -> synthesis on a side stream || ARM
// (or all serial); per-image workspace slices of `per` bytes
static int forward_batch(const cc_model_desc& d, const cc_strip* win, const int16_t* const* lat,
                         const float* const* arm_w, const float* const* up_w, const float* const* syn_w,
                         const float* const* image, float* const* x_hat, char* slices, size_t per, int n,
                         cudaStream_t s, bool overlap, bool join = true, bool fork = true,
                         const cudaEvent_t* arm_wait = nullptr, const cudaEvent_t* syn_wait = nullptr) {
  PyrGeom pg;
  pyr_geom(d, win, pg);
  const int n_arm = n_arm_cap(d, win);  // synthesis partials start here
  // no programmatic launches while cc_profile_* brackets every launch with
  // events (each kernel's own duration is what those events measure)
  const bool pdl = pdl_enabled() && !g_prof.on;
  int rc;
  if (d.up_2d) {  // Table 1 2-D TConv: full pyramid -> dense, then synthesis from it
    static thread_local Pyr2dImage im2[MAX_JOBS_PER_LAUNCH];
    for (int i = 0; i < n; i++) {
      im2[i].lat = lat[i];
      im2[i].S = slice_pyr(d, win, slices + per * (size_t)i);
      im2[i].dense = slice_dense(d, win, slices + per * (size_t)i);
      for (int t = 0; t < 64; t++) im2[i].k2[t] = t < d.up_taps * d.up_taps ? up_w[i][t] : 0.0f;
    }
    {
      ProfScope ps(PK_PYR, s);
      launch_pyramid2d(pg, d.up_taps, im2, n, s);
    }
    g_launches += pyramid2d_launch_count(pg, n);
    if ((rc = cuda_check("pyramid2d_kernel"))) return rc;
    for (int i = 0; i < n; i++)
      if ((rc = arm_one(d, win, lat[i], arm_w[i], (double*)(slices + per * (size_t)i), s))) return rc;
    for (int i = 0; i < n; i++) {
      char* sl = slices + per * (size_t)i;
      SynGeom sg;
      syn_geom(d, win, sg);
      {
        ProfScope ps(PK_SYN, s);
        find_syn_launcher(d.L, d.syn_widths[1], d.syn_n_res, d.up_taps)(
            sg, d, nullptr, syn_w[i], lat[i], nullptr, slice_dense(d, win, sl), image[i], x_hat[i], nullptr, nullptr,
            (double*)sl + n_arm, s, nullptr);
      }
      g_launches++;
      if ((rc = cuda_check("synth_kernel(dense_in)"))) return rc;
    }
    return CC_OK;
  }
  PyrImage imgs[MAX_JOBS_PER_LAUNCH];
  for (int i = 0; i < n; i++)
    imgs[i] = pyr_image(d, lat[i], up_w[i], slice_pyr(d, win, slices + per * (size_t)i));
  if (overlap) {
    // concurrent: the ARM kernels on `s`, the pyramid + synthesis kernels on a
    // side stream (they do not depend on the ARM); an SM holds one ARM CTA
    // (FMA-bound) next to one synthesis CTA (latency phases), so each fills
    // the other's gaps.  Joined before the caller's next work on `s`.
    SideStream* side = nullptr;
    if ((rc = side_stream(&side))) return rc;
    if (fork) {  // else the caller has ordered the side stream after this batch's inputs
      cudaEventRecord(side->fork, s);
      cudaStreamWaitEvent(side->s, side->fork, 0);
    }
    if (arm_wait) cudaStreamWaitEvent(side->s, arm_wait[n - 1], 0);  // every latent of the batch landed
    auto syn_i = [&](int i) -> int {
      char* sl = slices + per * (size_t)i;
      const float* s1 = slice_pyr(d, win, sl) + pg.s_off[1];
      if (syn_wait) cudaStreamWaitEvent(side->s, syn_wait[i], 0);  // image i landed
      // synthesis i > 0 directly follows synthesis i - 1 in the side stream
      LaunchCtlScope lc(pdl && i > 0 && !syn_wait, 0);
      return syn_one(d, win, lat[i], s1, up_w[i], syn_w[i], image[i], x_hat[i], nullptr, (double*)sl + n_arm,
                     side->s);
    };
    auto arm_i = [&](int i) -> int {
      if (arm_wait) cudaStreamWaitEvent(s, arm_wait[i], 0);
      LaunchCtlScope lc(pdl && i > 0 && !arm_wait, ARM_LAUNCH_ONLY);
      return arm_one(d, win, lat[i], arm_w[i], (double*)(slices + per * (size_t)i), s);
    };
    if ((rc = pyr_many(d, win, imgs, n, side->s))) return rc;
    // both streams get work from the start: the ARM weights staged, then image
    // i's ARM and synthesis launches enqueued together (enqueueing all the
    // synthesis launches first left the ARM stream idle while the host
    // enqueued them: 1.8634e10 vs 1.8668e10 px/s)
    if ((rc = arm_stage_all(d, win, lat, arm_w, slices, per, n, s))) return rc;
    for (int i = 0; i < n; i++)
      if ((rc = arm_i(i)) || (rc = syn_i(i))) return rc;
    cudaEventRecord(side->join, side->s);
    if (join) cudaStreamWaitEvent(s, side->join, 0);  // else the caller orders on the side stream
    return CC_OK;
  }
  if ((rc = arm_stage_all(d, win, lat, arm_w, slices, per, n, s))) return rc;
  if ((rc = pyr_many(d, win, imgs, n, s))) return rc;
  for (int i = 0; i < n; i++) {
    LaunchCtlScope lc(pdl && i > 0, ARM_LAUNCH_ONLY);
    if ((rc = arm_one(d, win, lat[i], arm_w[i], (double*)(slices + per * (size_t)i), s))) return rc;
  }
  for (int i = 0; i < n; i++) {
    char* sl = slices + per * (size_t)i;
    const float* s1 = slice_pyr(d, win, sl) + pg.s_off[1];
    // the first synthesis reads the pyramid's output: ordered normally after the ARMs
    LaunchCtlScope lc(pdl && i > 0, 0);
    if ((rc = syn_one(d, win, lat[i], s1, up_w[i], syn_w[i], image[i], x_hat[i], nullptr, (double*)sl + n_arm, s)))
      return rc;
  }
  return CC_OK;
}

}  // namespace ccrd

using namespace ccrd;

extern "C" {

const char* cc_version(void) { return "ccrd 0.1 (sm_100a)"; }

const char* cc_strerror(int code) {
  switch (code) {
    case CC_OK: return "ok";
    case CC_EINVAL: return "invalid argument";
    case CC_ENOTSUP: return "not supported by the compiled kernels";
    case CC_EWORKSPACE: return "workspace missing or too small";
    case CC_ECUDA: return "CUDA error";
    case CC_ENONFINITE: return "non-finite value";
    default: return "unknown error";
  }
}

const char* cc_last_error(void) { return g_err; }

int cc_profile_begin(void) {
  g_prof.on = true;
  g_prof.n = 0;
  g_prof.pool_used = 0;
  return CC_OK;
}

int cc_profile_end(cc_profile_summary* out) {
  ProfState& P = g_prof;
  P.on = false;
  if (!out) return fail(CC_EINVAL, "null summary");
  memset(out, 0, sizeof(*out));
  for (int i = 0; i < P.n; i++) {
    if (cudaEventSynchronize(P.recs[i].b) != cudaSuccess) return cuda_check("cc_profile_end");
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, P.recs[i].a, P.recs[i].b);
    switch (P.recs[i].kind) {
      case PK_ARM: out->arm_ms += ms; out->arm_launches++; break;
      case PK_SYN: out->syn_ms += ms; out->syn_launches++; break;
      case PK_PYR: out->pyr_ms += ms; out->pyr_launches++; break;
      default: out->reduce_ms += ms; out->reduce_launches++; break;
    }
  }
  P.n = 0;
  P.pool_used = 0;
  return cuda_check("cc_profile_end");
}
int64_t cc_last_launch_count(void) { return g_launches; }

int cc_set_arm_path(int32_t path) {
  if (path != CC_ARM_AUTO && path != CC_ARM_FFMA2 && path != CC_ARM_TC)
    return fail(CC_EINVAL, "arm path must be CC_ARM_AUTO, CC_ARM_FFMA2 or CC_ARM_TC (got %d)", path);
  g_arm_path.store(path);
  return CC_OK;
}
int32_t cc_get_arm_path(void) { return arm_path(); }
int32_t cc_arm_path_for(const cc_model_desc* desc) {
  if (validate(desc) != CC_OK) return -1;
  return arm_use_tc(*desc) ? CC_ARM_TC : CC_ARM_FFMA2;
}

int cc_set_synth_path(int32_t path) {
  if (path != CC_SYN_AUTO && path != CC_SYN_FFMA2 && path != CC_SYN_MMA && path != CC_SYN_TMA)
    return fail(CC_EINVAL, "synthesis path must be CC_SYN_AUTO, CC_SYN_FFMA2, CC_SYN_MMA or CC_SYN_TMA (got %d)",
                path);
  g_syn_path.store(path);
  return CC_OK;
}
int32_t cc_get_synth_path(void) { return synth_path(); }

int cc_validate(const cc_model_desc* desc) { return validate(desc); }

// latents_i8 is a host-path transfer format; device entry points take int16
static int validate_device(const cc_model_desc* desc) {
  const int rc = validate(desc);
  if (rc) return rc;
  if (desc->latents_i8) return fail(CC_ENOTSUP, "latents_i8 applies to cc_rd_forward_host only (device latents are int16)");
  return CC_OK;
}

size_t cc_workspace_bytes(const cc_model_desc* desc, int32_t n_img) {
  if (validate(desc) != CC_OK || n_img < 1) return 0;
  return slice_bytes(*desc, nullptr) * (size_t)n_img;
}

int cc_rd_forward(const cc_model_desc* desc, const cc_image_io* io, int32_t n_img, cc_rd_result* results,
                  void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_device(desc);
  if (rc) return rc;
  if (!io || n_img < 1 || !results) return fail(CC_EINVAL, "io/results null or n_img < 1");
  const size_t per = slice_bytes(*desc, nullptr);
  const size_t need = per * (size_t)n_img;
  if (!workspace || workspace_bytes < need)
    return fail(CC_EWORKSPACE, "need %zu workspace bytes, got %zu", need, workspace_bytes);
  for (int i = 0; i < n_img; i++)
    if (!io[i].latents || !io[i].arm_w || !io[i].up_w || !io[i].syn_w)
      return fail(CC_EINVAL, "image %d: null latents or weights", i);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  char* slices = (char*)workspace;
  for (int b = 0; b < n_img; b += MAX_JOBS_PER_LAUNCH) {
    const int m = (n_img - b < MAX_JOBS_PER_LAUNCH) ? n_img - b : MAX_JOBS_PER_LAUNCH;
    const int16_t* lat[MAX_JOBS_PER_LAUNCH];
    const float *aw[MAX_JOBS_PER_LAUNCH], *uw[MAX_JOBS_PER_LAUNCH], *sw[MAX_JOBS_PER_LAUNCH],
        *img[MAX_JOBS_PER_LAUNCH];
    float* xh[MAX_JOBS_PER_LAUNCH];
    ReduceJob jobs[MAX_JOBS_PER_LAUNCH];
    for (int i = 0; i < m; i++) {
      const cc_image_io& x = io[b + i];
      lat[i] = x.latents;
      aw[i] = x.arm_w;
      uw[i] = x.up_w;
      sw[i] = x.syn_w;
      img[i] = x.image;
      xh[i] = x.x_hat;
      jobs[i] = make_job(*desc, nullptr, (double*)(slices + per * (size_t)(b + i)));
    }
    rc = forward_batch(*desc, nullptr, lat, aw, uw, sw, img, xh, slices + per * (size_t)b, per, m, s,
                       concurrent_streams());
    if (rc) return rc;
    rc = launch_reduce(jobs, m, results + b, s);
    if (rc) return rc;
  }
  return CC_OK;
}

// ---------------------------------------------------------------- host path
// Device workspace layout: [partials x n_img][results x n_img][2 staging slots:
// latents | image | x_hat].
static size_t stage_slot_bytes(const cc_model_desc& d) {
  int64_t n_lat = 0;
  LevelGeom g;
  level_dims(d, g, &n_lat);
  const size_t P = (size_t)d.H * d.W;
  // int16 latents | fp32-sized image | x_hat | int8 latent upload (latents_i8)
  return align256(sizeof(int16_t) * (size_t)n_lat) + 2 * align256(sizeof(float) * 3 * P) +
         (d.latents_i8 ? align256((size_t)n_lat) : 0);
}

__global__ void widen_i8_kernel(const int8_t* __restrict__ in, int16_t* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

// The host path stages CHUNKS of HOST_CHUNK images (one forward_batch call
// each: batched pyramid launch, ARM / synthesis kernels back to back) in
// HOST_SLOTS rotating slots: uploads run ahead of the compute by up to
// HOST_SLOTS - 1 chunks.  One image per call measured 23 % slower than batched.
constexpr int HOST_SLOTS_MAX = 4, HOST_CHUNK_MAX = 8;
// defaults 3 slots x 4 images (swept on B200, batched 2K: 2x1 9.42, 2x2 9.70,
// 2x4 9.54, 3x4 10.07, 4x4 10.06, 2x8 9.62 Gpx/s e2e); CCRD_HOST_SLOTS /
// CCRD_HOST_CHUNK (read per call) for experiments
static int host_env(const char* name, int def, int lo, int hi) {
  const char* v = getenv(name);
  const int x = v ? atoi(v) : def;
  return x < lo ? lo : (x > hi ? hi : x);
}

// the host path's upload / read-back streams and slot events, per thread and device
struct HostPool {
  cudaStream_t cs = nullptr, ds = nullptr;
  cudaStream_t wsm = nullptr;  // int8 -> int16 latent widening (keeps the upload stream copies-only)
  cudaEvent_t widened[HOST_SLOTS_MAX * HOST_CHUNK_MAX];  // per image: int16 latents ready
  cudaEvent_t copied[HOST_SLOTS_MAX], computed[HOST_SLOTS_MAX], computed_side[HOST_SLOTS_MAX],
      read_back[HOST_SLOTS_MAX];
  cudaEvent_t img_copied[HOST_SLOTS_MAX * HOST_CHUNK_MAX];  // per image: latents landed (its ARM may start)
  cudaEvent_t img_done[HOST_SLOTS_MAX * HOST_CHUNK_MAX];    // per image: image landed (its synthesis may start)
  int device = -1;
};
static thread_local HostPool g_host;

static int host_pool(HostPool** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  if (g_host.device != dev) {
    // the upload stream runs at the highest priority: its small kernels (the
    // int8 -> int16 latent widening) take the next free SM slots instead of
    // queueing behind the compute stream's blocks
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&g_host.cs, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&g_host.wsm, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithFlags(&g_host.ds, cudaStreamNonBlocking) != cudaSuccess)
      return cuda_check("stream create");
    for (int k = 0; k < HOST_SLOTS_MAX; k++)
      if (cudaEventCreateWithFlags(&g_host.copied[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&g_host.computed[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&g_host.computed_side[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&g_host.read_back[k], cudaEventDisableTiming) != cudaSuccess)
        return cuda_check("event create");
    for (int k = 0; k < HOST_SLOTS_MAX * HOST_CHUNK_MAX; k++)
      if (cudaEventCreateWithFlags(&g_host.img_copied[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&g_host.widened[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&g_host.img_done[k], cudaEventDisableTiming) != cudaSuccess)
        return cuda_check("event create");
    g_host.device = dev;
  }
  *out = &g_host;
  return CC_OK;
}

// staging slots x images per slot of the host pipeline (measured best 4 x 4;
// CCRD_HOST_SLOTS / CCRD_HOST_CHUNK override for experiments)
static int host_slots() { return host_env("CCRD_HOST_SLOTS", 4, 2, HOST_SLOTS_MAX); }
// images per staged chunk: 1 for megapixel images (the pipeline fills after one
// image's upload; 64 x 2K e2e: chunk 1 1.194e10, 2 1.188e10, 4 1.176e10 px/s),
// 4 for small ones, whose host path is enqueue-bound
static int host_chunk(const cc_model_desc& d) {
  return host_env("CCRD_HOST_CHUNK", (int64_t)d.H * d.W >= (1 << 20) ? 1 : 4, 1, HOST_CHUNK_MAX);
}

size_t cc_workspace_bytes_host(const cc_model_desc* desc, int32_t n_img) {
  if (validate(desc) != CC_OK || n_img < 1) return 0;
  return slice_bytes(*desc, nullptr) * (size_t)n_img +
         align256(sizeof(cc_rd_result) * (size_t)n_img) +
         (size_t)host_slots() * host_chunk(*desc) * stage_slot_bytes(*desc);
}

int cc_rd_forward_host(const cc_model_desc* desc, const cc_image_io* io, int32_t n_img, cc_rd_result* results,
                       void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate(desc);
  if (rc) return rc;
  if (!io || n_img < 1 || !results) return fail(CC_EINVAL, "io/results null or n_img < 1");
  const cc_model_desc& d = *desc;
  const size_t need = cc_workspace_bytes_host(desc, n_img);
  if (!workspace || workspace_bytes < need)
    return fail(CC_EWORKSPACE, "need %zu workspace bytes, got %zu", need, workspace_bytes);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  const size_t per = slice_bytes(d, nullptr);
  char* ws = (char*)workspace;
  cc_rd_result* dres = (cc_rd_result*)(ws + per * (size_t)n_img);
  char* stage = ws + per * (size_t)n_img + align256(sizeof(cc_rd_result) * (size_t)n_img);
  const size_t slot = stage_slot_bytes(d);
  const int HOST_SLOTS = host_slots();
  const int HOST_CHUNK = host_chunk(d);
  int64_t n_lat = 0;
  LevelGeom lg;
  level_dims(d, lg, &n_lat);
  const size_t P = (size_t)d.H * d.W;
  const size_t lat_b = sizeof(int16_t) * (size_t)n_lat, xh_b = sizeof(float) * 3 * P;
  const size_t img_b = (d.image_u8 ? 1 : sizeof(float)) * 3 * P;  // 8-bit images: 3 bytes per pixel

  cudaStream_t s = (cudaStream_t)stream;
  // copy stream + per-slot events: copies of image i+1 overlap compute of image i
  // three streams: uploads (cs), compute (s), readbacks (ds); PCIe is full
  // duplex, so image i+1's upload, image i's compute and image i-1's x_hat
  // readback overlap.  HOST_SLOTS staging slots of HOST_CHUNK images; events
  // guard their reuse.
  // streams and events live in a per-thread pool (creating and destroying 2
  // streams + 16 events per call cost more than a small batch's compute)
  HostPool* hp = nullptr;
  if ((rc = host_pool(&hp))) return rc;
  cudaStream_t cs = hp->cs, ds = hp->ds;
  // With concurrent streams the ARM (on s) and the pyramid + synthesis (on
  // the side stream) of consecutive images are not joined per image: each
  // stream runs image after image (as in cc_rd_forward's batch); a slot is
  // reused once both streams are done with it, x_hat is read back after the
  // side stream, and the reduction joins the side stream once.
  const bool conc = concurrent_streams();
  SideStream* side = nullptr;
  if (conc && (rc = side_stream(&side))) return rc;
  static const bool widen_stream = !(getenv("CCRD_WIDEN_STREAM") && getenv("CCRD_WIDEN_STREAM")[0] == '0');
  cudaEvent_t *copied = hp->copied, *computed = hp->computed, *computed_side = hp->computed_side,
              *read_back = hp->read_back;
  // start the side streams after whatever is already queued on s
  cudaEventRecord(computed[0], s);
  cudaStreamWaitEvent(cs, computed[0], 0);
  cudaStreamWaitEvent(ds, computed[0], 0);
  if (conc) cudaStreamWaitEvent(side->s, computed[0], 0);
  for (int k = 0; k < HOST_SLOTS; k++) {
    cudaEventRecord(computed[k], s);
    cudaEventRecord(computed_side[k], s);
    cudaEventRecord(read_back[k], s);
  }
  ReduceJob* jobs = new ReduceJob[n_img];
  for (int i0 = 0, c = 0; i0 < n_img && rc == CC_OK; i0 += HOST_CHUNK, c++) {
    const int k = c % HOST_SLOTS, m = n_img - i0 < HOST_CHUNK ? n_img - i0 : HOST_CHUNK;
    const int16_t* l1[HOST_CHUNK_MAX];
    const float *a1[HOST_CHUNK_MAX], *u1[HOST_CHUNK_MAX], *s1[HOST_CHUNK_MAX], *i1[HOST_CHUNK_MAX];
    float* x1[HOST_CHUNK_MAX];
    float* dxhs[HOST_CHUNK_MAX];
    cudaEvent_t lat_ev[HOST_CHUNK_MAX];  // per image: its int16 latents are on the device
    cudaEvent_t last_widened = nullptr;
    cudaStreamWaitEvent(cs, computed[k], 0);  // slot k's inputs were consumed by chunk c - HOST_SLOTS
    cudaStreamWaitEvent(cs, computed_side[k], 0);
    for (int j = 0; j < m && rc == CC_OK; j++) {
      char* base = stage + slot * (size_t)(k * HOST_CHUNK + j);
      int16_t* dlat = (int16_t*)base;
      int8_t* dlat8 = (int8_t*)(base + align256(lat_b) + 2 * align256(xh_b));
      float* dimg = (float*)(base + align256(lat_b));
      dxhs[j] = (float*)(base + align256(lat_b) + align256(xh_b));
      const cc_image_io& x = io[i0 + j];
      if (!x.latents || !x.arm_w || !x.up_w || !x.syn_w) {
        rc = fail(CC_EINVAL, "image %d: null latents or weights", i0 + j);
        break;
      }
      // the ARM needs only the latents: its event goes before the image (70 % of
      // the bytes; uploading all of a chunk's latents first measured slower)
      cudaEvent_t lat_ready = hp->img_copied[k * HOST_CHUNK_MAX + j];
      if (d.latents_i8) {  // 1 byte per latent over PCIe, widened to int16 on the device
        cudaMemcpyAsync(dlat8, x.latents, (size_t)n_lat, cudaMemcpyHostToDevice, cs);
        if (widen_stream) {  // on its own stream: the upload stream stays copies-only
          cudaEventRecord(lat_ready, cs);
          cudaStreamWaitEvent(hp->wsm, lat_ready, 0);
          widen_i8_kernel<<<(unsigned)((n_lat + 255) / 256), 256, 0, hp->wsm>>>(dlat8, dlat, n_lat);
          lat_ready = hp->widened[k * HOST_CHUNK_MAX + j];
          cudaEventRecord(lat_ready, hp->wsm);
          last_widened = lat_ready;
        } else {
          widen_i8_kernel<<<(unsigned)((n_lat + 255) / 256), 256, 0, cs>>>(dlat8, dlat, n_lat);
          cudaEventRecord(lat_ready, cs);
        }
        g_launches++;
      } else {
        cudaMemcpyAsync(dlat, x.latents, lat_b, cudaMemcpyHostToDevice, cs);
        cudaEventRecord(lat_ready, cs);
      }
      lat_ev[j] = lat_ready;
      if (x.image) cudaMemcpyAsync(dimg, x.image, img_b, cudaMemcpyHostToDevice, cs);
      cudaEventRecord(hp->img_done[k * HOST_CHUNK_MAX + j], cs);
      l1[j] = dlat;
      a1[j] = x.arm_w;
      u1[j] = x.up_w;
      s1[j] = x.syn_w;
      i1[j] = x.image ? dimg : nullptr;
      x1[j] = x.x_hat ? dxhs[j] : nullptr;
      jobs[i0 + j] = make_job(d, nullptr, (double*)(ws + per * (size_t)(i0 + j)));
    }
    if (rc) break;
    cudaEventRecord(copied[k], cs);
    if (!conc) {  // concurrent: the ARM waits per image (below)
      cudaStreamWaitEvent(s, copied[k], 0);
      if (last_widened) cudaStreamWaitEvent(s, last_widened, 0);
    }
    cudaStreamWaitEvent(s, read_back[k], 0);  // slot k's x_hat of chunk c - HOST_SLOTS is read back
    if (conc)  // the side stream waits for this chunk's own inputs (per image, below), not for the ARM stream
      cudaStreamWaitEvent(side->s, read_back[k], 0);
    rc = forward_batch(d, nullptr, l1, a1, u1, s1, i1, x1, ws + per * (size_t)i0, per, m, s, conc, /*join=*/false,
                       /*fork=*/!conc, conc ? lat_ev : nullptr,
                       conc ? hp->img_done + k * HOST_CHUNK_MAX : nullptr);
    if (rc) break;
    cudaEventRecord(computed[k], s);
    cudaEventRecord(computed_side[k], conc ? side->s : s);
    cudaStreamWaitEvent(ds, computed_side[k], 0);
    for (int j = 0; j < m; j++)
      if (io[i0 + j].x_hat) cudaMemcpyAsync(io[i0 + j].x_hat, dxhs[j], xh_b, cudaMemcpyDeviceToHost, ds);
    cudaEventRecord(read_back[k], ds);
  }
  if (conc) {  // the last images' synthesis
    cudaEventRecord(side->join, side->s);
    cudaStreamWaitEvent(s, side->join, 0);
  }
  if (rc == CC_OK) rc = launch_reduce(jobs, n_img, dres, s);
  if (rc == CC_OK) {
    cudaMemcpyAsync(results, dres, sizeof(cc_rd_result) * (size_t)n_img, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = cuda_check("cc_rd_forward_host sync");
  } else {
    cudaStreamSynchronize(s);
  }
  cudaStreamSynchronize(cs);
  cudaStreamSynchronize(hp->wsm);
  if (cudaStreamSynchronize(ds) != cudaSuccess && rc == CC_OK) rc = cuda_check("cc_rd_forward_host readback");
  delete[] jobs;
  if (rc == CC_OK) rc = cuda_check("cc_rd_forward_host");
  return rc;
}

// ---------------------------------------------------------------- strips
static int validate_strip(const cc_model_desc& d, const cc_strip* st) {
  if (!st) return fail(CC_EINVAL, "null strip");
  if (d.up_2d) return fail(CC_ENOTSUP, "strips are implemented for the separable upsampling only");
  if (st->r0 < 0 || st->r1 > d.H || st->r0 >= st->r1 || (st->r0 & 1))
    return fail(CC_EINVAL, "strip rows [%d, %d) must satisfy 0 <= r0 < r1 <= H (%d) with r0 even", st->r0, st->r1,
                d.H);
  cc_strip need;
  strip_window(d, st->r0, st->r1, need);
  for (int l = 0; l < d.L; l++) {
    if (st->own_lo[l] != need.own_lo[l] || st->own_hi[l] != need.own_hi[l])
      return fail(CC_EINVAL, "strip level %d: owned rows [%d, %d) != ceil(r/2^l) = [%d, %d)", l, st->own_lo[l],
                  st->own_hi[l], need.own_lo[l], need.own_hi[l]);
    if (st->lo[l] < 0 || st->hi[l] > ceil_shift(d.H, l) || st->lo[l] > need.lo[l] || st->hi[l] < need.hi[l])
      return fail(CC_EINVAL, "strip level %d: window [%d, %d) does not contain the receptive field [%d, %d)", l,
                  st->lo[l], st->hi[l], need.lo[l], need.hi[l]);
  }
  return CC_OK;
}

int cc_strip_window(const cc_model_desc* desc, int32_t r0, int32_t r1, cc_strip* out) {
  int rc = validate(desc);
  if (rc) return rc;
  if (!out) return fail(CC_EINVAL, "null strip");
  if (r0 < 0 || r1 > desc->H || r0 >= r1 || (r0 & 1))
    return fail(CC_EINVAL, "strip rows [%d, %d) must satisfy 0 <= r0 < r1 <= H (%d) with r0 even", r0, r1, desc->H);
  strip_window(*desc, r0, r1, *out);
  return CC_OK;
}

int64_t cc_strip_latent_count(const cc_model_desc* desc, const cc_strip* strip) {
  if (validate(desc) != CC_OK || validate_strip(*desc, strip) != CC_OK) return -1;
  LevelGeom g;
  int64_t n = 0;
  level_dims(*desc, strip, g, &n);
  return n;
}

size_t cc_workspace_bytes_strip(const cc_model_desc* desc, const cc_strip* strip) {
  if (validate(desc) != CC_OK || validate_strip(*desc, strip) != CC_OK) return 0;
  return slice_bytes(*desc, strip);
}

int cc_rd_forward_strip(const cc_model_desc* desc, const cc_strip* strip, const cc_image_io* io,
                        cc_rd_result* result, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_device(desc);
  if (rc) return rc;
  const cc_model_desc& d = *desc;
  if ((rc = validate_strip(d, strip))) return rc;
  if (!io || !result) return fail(CC_EINVAL, "io/result null");
  if (!io->latents || !io->arm_w || !io->up_w || !io->syn_w) return fail(CC_EINVAL, "null latents or weights");
  const size_t per = slice_bytes(d, strip);
  if (!workspace || workspace_bytes < per)
    return fail(CC_EWORKSPACE, "need %zu workspace bytes, got %zu", per, workspace_bytes);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  const int16_t* l1[1] = {io->latents};
  const float *a1[1] = {io->arm_w}, *u1[1] = {io->up_w}, *s1[1] = {io->syn_w}, *i1[1] = {io->image};
  float* x1[1] = {io->x_hat};
  if ((rc = forward_batch(d, strip, l1, a1, u1, s1, i1, x1, (char*)workspace, per, 1, s, concurrent_streams())))
    return rc;
  ReduceJob j = make_job(d, strip, (double*)workspace);
  return launch_reduce(&j, 1, result, s);
}

// ---------------------------------------------------------------- training
int64_t cc_train_param_count(const cc_model_desc* desc) {
  if (validate(desc) != CC_OK) return -1;
  return train_param_count(*desc);
}

size_t cc_train_workspace_bytes(const cc_model_desc* desc) {
  if (validate(desc) != CC_OK || !train_supported(*desc)) return 0;
  return train_workspace_bytes(*desc);
}

int cc_train_step(const cc_model_desc* desc, float* params, const float* noise, const float* image, float* adam_m,
                  float* adam_v, const cc_adam* opt, cc_rd_result* result, float* grad, void* workspace,
                  size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_device(desc);
  if (rc) return rc;
  const cc_model_desc& d = *desc;
  if (!train_supported(d)) return fail(CC_ENOTSUP, "training step not compiled for this shape (or up_2d)");
  if (d.image_u8) return fail(CC_ENOTSUP, "the training step takes an fp32 image (image_u8 = 0)");
  if (!params || !noise || !image || !result || !grad) return fail(CC_EINVAL, "null params / noise / image / result / grad");
  if (opt && (!adam_m || !adam_v || opt->t < 1)) return fail(CC_EINVAL, "Adam needs m, v and t >= 1");
  const size_t need = train_workspace_bytes(d);
  if (!workspace || workspace_bytes < need)
    return fail(CC_EWORKSPACE, "need %zu workspace bytes, got %zu", need, workspace_bytes);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  const int n = train_step_impl(d, params, noise, image, adam_m, adam_v, opt, result, grad, workspace,
                                (cudaStream_t)stream);
  if (n < 0) return fail(CC_ENOTSUP, "training step: unsupported shape (%d)", n);
  g_launches = n;
  return cuda_check("cc_train_step");
}

// ---------------------------------------------------------------- analysis
static int validate_analysis(const cc_analysis_desc* a) {
  if (!a) return fail(CC_EINVAL, "null analysis descriptor");
  if (a->H < 1 || a->W < 1 || a->L < 1 || a->L > CC_MAX_LEVELS || a->C < 4 || a->C > 512 || a->C % 4 || a->blocks < 1)
    return fail(CC_EINVAL, "bad analysis descriptor (H %d, W %d, L %d, C %d, blocks %d)", a->H, a->W, a->L, a->C,
                a->blocks);
  if (a->tf32 < 0 || a->tf32 > 3) return fail(CC_EINVAL, "tf32 must be 0, 1, 2 or 3");
  if (a->N < 1 || (int64_t)a->N * a->H * a->W > ((int64_t)1 << 31) / 4)
    return fail(CC_EINVAL, "bad analysis batch N %d (N H W must stay below 2^29)", a->N);
  return CC_OK;
}

int64_t cc_analysis_param_count(const cc_analysis_desc* a) {
  if (validate_analysis(a)) return -1;
  return analysis_param_count(*a);
}

size_t cc_analysis_workspace_bytes(const cc_analysis_desc* a) {
  if (validate_analysis(a)) return 0;
  return analysis_workspace_bytes(*a);
}

int cc_analysis_forward(const cc_analysis_desc* a, const float* image, const float* weights, float* latents,
                        void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_analysis(a);
  if (rc) return rc;
  if (!image || !weights || !latents) return fail(CC_EINVAL, "null image / weights / latents");
  const size_t need = analysis_workspace_bytes(*a);
  if (!workspace || workspace_bytes < need) return fail(CC_EWORKSPACE, "need %zu workspace bytes", need);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  const int n = analysis_forward_impl(*a, image, weights, latents, workspace, (cudaStream_t)stream);
  if (n < 0) return fail(CC_ECUDA, "cuBLASLt matmul failed (%d)", n);
  g_launches = n;
  return cuda_check("cc_analysis_forward");
}

// ---------------------------------------------------------------- ARM decode (NEXT-3)
size_t cc_arm_decode_workspace_bytes(const cc_model_desc* desc, int32_t n_img) {
  if (validate_device(desc) != CC_OK || n_img < 1) return 0;
  return dec_workspace_bytes(*desc, n_img);
}

int cc_arm_decode(const cc_model_desc* desc, const cc_image_io* io, int32_t n_img, int16_t* const* decoded,
                  double* rate, float* const* mu, float* const* scale, float* const* bits, int32_t* poison_reads,
                  void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_device(desc);
  if (rc) return rc;
  if (!io || n_img < 1 || !decoded || !rate) return fail(CC_EINVAL, "io / decoded / rate null or n_img < 1");
  const size_t need = dec_workspace_bytes(*desc, n_img);
  if (!workspace || workspace_bytes < need) return fail(CC_EWORKSPACE, "need %zu workspace bytes", need);
  std::vector<const int16_t*> truth(n_img);
  std::vector<const float*> aw(n_img);
  for (int i = 0; i < n_img; i++) {
    if (!io[i].latents || !io[i].arm_w || !decoded[i]) return fail(CC_EINVAL, "image %d: null latents / arm_w / decoded", i);
    truth[i] = io[i].latents;
    aw[i] = io[i].arm_w;
  }
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  ArmGeom g;
  arm_geom(*desc, nullptr, g);
  const char* sk = getenv("CCRD_DEC_SKEW");
  const int n = arm_decode_impl(*desc, g, sk ? atoi(sk) : 0, n_img, truth.data(), aw.data(), decoded, mu, scale, bits,
                                rate, poison_reads, workspace, (cudaStream_t)stream);
  if (n == -3) return fail(CC_ENOTSUP, "ARM shape not compiled for the decoder");
  if (n == -2) return fail(CC_ENOTSUP, "decoder ring exceeds shared memory (grid too wide)");
  if (n < 0) return cuda_check("cc_arm_decode launch");
  g_launches = n;
  return cuda_check("cc_arm_decode");
}

// ---------------------------------------------------------------- decode
int cc_decode(const cc_model_desc* desc, const int16_t* latents, const float* up_w, const float* syn_w,
              uint8_t* out_rgb8, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_device(desc);
  if (rc) return rc;
  if (!latents || !up_w || !syn_w || !out_rgb8) return fail(CC_EINVAL, "null latents / up_w / syn_w / out");
  const cc_model_desc& d = *desc;
  const size_t per = slice_bytes(d, nullptr);
  if (!workspace || workspace_bytes < per) return fail(CC_EWORKSPACE, "need %zu workspace bytes", per);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  PyrGeom pg;
  pyr_geom(d, nullptr, pg);
  if (d.up_2d) {
    Pyr2dImage im2;
    im2.lat = latents;
    im2.S = slice_pyr(d, nullptr, workspace);
    im2.dense = slice_dense(d, nullptr, workspace);
    for (int t = 0; t < 64; t++) im2.k2[t] = t < d.up_taps * d.up_taps ? up_w[t] : 0.0f;
    launch_pyramid2d(pg, d.up_taps, &im2, 1, s);
    g_launches += pyramid2d_launch_count(pg, 1);
    SynGeom sg;
    syn_geom(d, nullptr, sg);
    find_syn_launcher(d.L, d.syn_widths[1], d.syn_n_res, d.up_taps)(sg, d, nullptr, syn_w, latents, nullptr, im2.dense,
                                                                    nullptr, nullptr, nullptr, nullptr, nullptr, s,
                                                                    out_rgb8);
    g_launches++;
    return cuda_check("cc_decode(2d)");
  }
  float* S = slice_pyr(d, nullptr, workspace);
  PyrImage im = pyr_image(d, latents, up_w, S);
  if ((rc = pyr_many(d, nullptr, &im, 1, s))) return rc;
  return syn_one(d, nullptr, latents, S + pg.s_off[1], up_w, syn_w, nullptr, nullptr, nullptr, nullptr, s, out_rgb8);
}

// ---------------------------------------------------------------- stages
int cc_arm_rate(const cc_model_desc* desc, const int16_t* latents, const float* arm_w, double* rate, float* mu,
                float* scale, float* bits, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_device(desc);
  if (rc) return rc;
  if (!latents || !arm_w || !rate) return fail(CC_EINVAL, "null latents / arm_w / rate");
  const size_t per = partial_bytes(*desc, nullptr);
  if (!workspace || workspace_bytes < per)
    return fail(CC_EWORKSPACE, "need %zu workspace bytes", per);  // <= cc_workspace_bytes(desc, 1)
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  if ((mu || scale) && !bits) return fail(CC_EINVAL, "mu/scale debug outputs need bits != NULL");
  const cc_model_desc& d = *desc;
  cudaStream_t s = (cudaStream_t)stream;
  ArmGeom ag;
  arm_geom(d, nullptr, ag);
  double* part = (double*)workspace;
  arm_launcher(d)(ag, d, arm_w, latents, part, mu, scale, bits, s);
  g_launches++;
  if ((rc = cuda_check("arm_rate_kernel"))) return rc;
  // rate only: reduce with an empty synthesis partial set
  ReduceJob j = make_job(d, nullptr, part);
  j.n_syn = 0;
  cc_rd_result* tmp = (cc_rd_result*)((char*)workspace + per - align256(sizeof(cc_rd_result)));
  if ((rc = launch_reduce(&j, 1, tmp, s))) return rc;
  cudaMemcpyAsync(rate, &tmp->rate_bits, sizeof(double), cudaMemcpyDeviceToDevice, s);
  return cuda_check("cc_arm_rate");
}

int cc_upsample(const cc_model_desc* desc, const int16_t* latents, const float* up_w, float* dense,
                void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate_device(desc);
  if (rc) return rc;
  if (!latents || !up_w || !dense) return fail(CC_EINVAL, "null latents / up_w / dense");
  const cc_model_desc& d = *desc;
  const size_t per = slice_bytes(d, nullptr);
  if (!workspace || workspace_bytes < per) return fail(CC_EWORKSPACE, "need %zu workspace bytes", per);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  if (d.up_2d) {  // the production 2-D path: pyramid2d writes channels 1..L-1
    PyrGeom pg;
    pyr_geom(d, nullptr, pg);
    Pyr2dImage im2;
    im2.lat = latents;
    im2.S = slice_pyr(d, nullptr, workspace);
    im2.dense = dense;
    for (int t = 0; t < 64; t++) im2.k2[t] = t < d.up_taps * d.up_taps ? up_w[t] : 0.0f;
    launch_pyramid2d(pg, d.up_taps, &im2, 1, s);
    launch_lat0_to_dense(latents, dense, (int64_t)d.H * d.W, s);
    g_launches += pyramid2d_launch_count(pg, 1) + 1;
    return cuda_check("cc_upsample(2d)");
  }
  // the production path (pyramid + fused last step) with its dense output on;
  // synthesis weights are irrelevant here: zero blob of the right size
  PyrGeom pg;
  pyr_geom(d, nullptr, pg);
  float* S = slice_pyr(d, nullptr, workspace);
  PyrImage im = pyr_image(d, latents, up_w, S);
  if ((rc = pyr_many(d, nullptr, &im, 1, s))) return rc;
  const int CH = d.syn_widths[1];
  const int nsyn = d.L * CH + CH + CH * 3 + 3 + 84 * d.syn_n_res;
  float* zeros = new float[nsyn]();
  rc = syn_one(d, nullptr, latents, S + pg.s_off[1], up_w, zeros, nullptr, nullptr, dense, nullptr, s);
  delete[] zeros;
  return rc;
}

int cc_synthesize(const cc_model_desc* desc, const float* dense, const float* syn_w, const float* image,
                  float* x_hat, double* sse, float* h_1x1, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int rc = validate(desc);
  if (rc) return rc;
  if (!dense || !syn_w) return fail(CC_EINVAL, "null dense / syn_w");
  if (sse && !image) return fail(CC_EINVAL, "sse requested without image");
  if (image && desc->image_u8) return fail(CC_ENOTSUP, "cc_synthesize takes an fp32 image (image_u8 = 0)");
  const cc_model_desc& d = *desc;
  SynGeom sg;
  syn_geom(d, nullptr, sg);
  const size_t need = align256(sizeof(double) * (size_t)sg.n_tiles) + sizeof(cc_rd_result);
  if (sse && (!workspace || workspace_bytes < need)) return fail(CC_EWORKSPACE, "need %zu workspace bytes", need);
  if (!have_device()) return fail(CC_ECUDA, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  double* part = sse ? (double*)workspace : nullptr;
  find_syn_launcher(d.L, d.syn_widths[1], d.syn_n_res, d.up_taps)(sg, d, nullptr, syn_w, nullptr, nullptr, dense,
                                                                   image, x_hat, nullptr, h_1x1, part, s, nullptr);
  g_launches++;
  if ((rc = cuda_check("synth_kernel(dense_in)"))) return rc;
  if (sse) {
    ReduceJob j = make_job(d, nullptr, part);
    j.n_arm = 0;
    j.syn_partial = part;
    cc_rd_result* tmp = (cc_rd_result*)((char*)workspace + align256(sizeof(double) * (size_t)sg.n_tiles));
    if ((rc = launch_reduce(&j, 1, tmp, s))) return rc;
    cudaMemcpyAsync(sse, &tmp->sse, sizeof(double), cudaMemcpyDeviceToDevice, s);
  }
  return cuda_check("cc_synthesize");
}

// ---------------------------------------------------------------- MAC count
// Closed form: ARM sum_k in_k out_k per latent;
// upsampling (K/2) MAC per produced sample of every separable pass; synthesis
// sum in out + 81 R per pixel.  Biases and residual adds are free.
double cc_mac_per_pixel(const cc_model_desc* desc, cc_mac_breakdown* out) {
  if (validate(desc) != CC_OK) return -1.0;
  const cc_model_desc& d = *desc;
  LevelGeom g;
  int64_t n_lat = 0;
  level_dims(d, g, &n_lat);
  int64_t arm_pl = 0;
  for (int k = 0; k < d.arm_n_layers; k++) arm_pl += (int64_t)d.arm_widths[k] * d.arm_widths[k + 1];
  const int64_t arm = arm_pl * n_lat;
  int64_t up = 0;
  for (int l = 1; l < d.L; l++)
    for (int j = 0; j < l; j++)
      up += d.up_2d ? (int64_t)(d.up_taps / 2) * (d.up_taps / 2) * g.h[j] * g.w[j]  // (K/2)^2 per output
                    : (int64_t)(d.up_taps / 2) * ((int64_t)g.h[j + 1] * g.w[j] + (int64_t)g.h[j] * g.w[j]);
  int64_t syn_pp = 81 * (int64_t)d.syn_n_res;
  for (int k = 0; k < d.syn_n_1x1; k++) syn_pp += (int64_t)d.syn_widths[k] * d.syn_widths[k + 1];
  const int64_t P = (int64_t)d.H * d.W;
  const int64_t syn = syn_pp * P;
  const double tot = (double)(arm + up + syn) / (double)P;
  if (out) {
    out->arm = (double)arm / P;
    out->up = (double)up / P;
    out->syn = (double)syn / P;
    out->total = tot;
    out->arm_macs = arm;
    out->up_macs = up;
    out->syn_macs = syn;
    out->n_latents = n_lat;
  }
  return tot;
}

}  // extern "C"
