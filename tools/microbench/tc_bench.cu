// tcgen05 throughput probe (B200, sm_100a): the numbers the pipelined
// tensor-core ARM is designed against.
//   ldtm  : tcgen05.ld 32x32b.xN by W warps of one CTA per SM, bytes / cycle / SM
//   sttm  : tcgen05.st 32x32b.xN, bytes / cycle / SM
//   mma   : back-to-back tcgen05.mma kind::tf32, M = 128, N in {16, 24, 32, 48, 64},
//           K = 8, A from TMEM (TS) or shared memory (SS); cycles per MMA
//   n24   : correctness of an N = 24 MMA (steps of 8 legal at cta_group::1?)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_bench tc_bench.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(b), "r"(phase));
}

#define LD32(r, a)                                                                                              \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                        \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),       \
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),     \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),     \
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                          \
               : "r"(a))
#define ST32(a, r)                                                                                             \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
               "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),          \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), \
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),  \
               "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), \
               "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))

// mode 0: ldtm, 1: sttm, 2: ldtm with 2 loads in flight before the wait
__global__ void tmem_bw(int mode, int iters, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32 % 256);
  uint32_t r[32], q[32];
  for (int j = 0; j < 32; j++) r[j] = threadIdx.x * 32 + j;
  ST32(ta, r);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  float acc = 0.f;
  const unsigned long long t0 = clock64();
  if (mode == 0) {
    for (int it = 0; it < iters; it++) {
      LD32(r, ta);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += __uint_as_float(r[it & 31]);
    }
  } else if (mode == 1) {
    for (int it = 0; it < iters; it++) {
      r[it & 31] += 1;
      ST32(ta, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  } else {
    for (int it = 0; it < iters; it += 2) {
      LD32(r, ta);
      LD32(q, ta + 32 * 0);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += __uint_as_float(r[it & 31]) + __uint_as_float(q[(it + 1) & 31]);
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

// back-to-back MMAs issued by one thread; ts: A from TMEM
__global__ void mma_rate(int N, int ts, int n_mma, unsigned long long* cyc) {
  extern __shared__ __align__(1024) float sm[];
  float* sA = sm;               // 128 x 8
  float* sB = sm + 128 * 8;     // 64 x 8
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 8 + 64 * 8; i += blockDim.x) sm[i] = 0.0f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = sdesc(su32(sA), 128, 256), db = sdesc(su32(sB), 128, 256);
    const unsigned long long t0 = clock64();
    for (int k = 0; k < n_mma; k++) {
      if (ts)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tm), "r"(tm + 64), "l"(db), "r"(idesc), "r"(1));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    mbar_wait(su32(&bar), 0);
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}


// NC independent accumulators (D_c at column c * 64), issued round robin: is
// the ~96-cycle per-MMA cost a dependency on the accumulator or the issue?
__global__ void mma_chains(int N, int ts, int n_mma, int NC, int acc_mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) float sm[];
  float* sA = sm;
  float* sB = sm + 128 * 8;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 8 + 64 * 8; i += blockDim.x) sm[i] = 0.0f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = sdesc(su32(sA), 128, 256), db = sdesc(su32(sB), 128, 256);
    const unsigned long long t0 = clock64();
    for (int k = 0; k < n_mma; k += NC)
      for (int c = 0; c < NC; c++) {
        const uint32_t d = tm + c * 64;
        const uint32_t acc = acc_mode;
        if (ts)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(d), "r"(tm + 448), "l"(db), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    mbar_wait(su32(&bar), 0);
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}


// warp-wide issue: the whole warp runs the loop, elect.sync picks the issuing
// lane inside ONE asm block of 8 MMAs (no per-MMA branch / ELECT loop).
// sep: 8 different accumulators (columns 32 c) or one
__global__ void mma_burst(int N, int ts, int n_iter, int sep, unsigned long long* cyc, int small = 0) {
  extern __shared__ __align__(1024) float sm[];
  float* sA = sm;
  float* sB = sm + 128 * 8;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 8 + 64 * 8; i += blockDim.x) sm[i] = 0.0f;
  if (warp == 0) {
    if (small) asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
    else asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t db = sdesc(su32(sB), 128, 256);
    const uint64_t da = sdesc(su32(sA), 128, 256);
    const uint32_t st = sep ? (small ? 8 : 32) : 0;
    const uint32_t a_t = small ? tm + 96 : tm + 320;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < n_iter; it++) {
      if (ts)
        asm volatile(
            "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%4], [%1], %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%5], [%1], %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%6], [%1], %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%7], [%1], %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%8], [%1], %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%9], [%1], %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%10], [%1], %2, %3, 1;\n\t}"
            ::"r"(tm), "r"(a_t), "l"(db), "r"(idesc), "r"(tm + st), "r"(tm + 2 * st), "r"(tm + 3 * st), "r"(tm + 4 * st),
            "r"(tm + 5 * st), "r"(tm + 6 * st), "r"(tm + 7 * st));
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%4], %1, %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%5], %1, %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%6], %1, %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%7], %1, %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%8], %1, %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%9], %1, %2, %3, 1;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%10], %1, %2, %3, 1;\n\t}"
            ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(tm + st), "r"(tm + 2 * st), "r"(tm + 3 * st), "r"(tm + 4 * st),
            "r"(tm + 5 * st), "r"(tm + 6 * st), "r"(tm + 7 * st));
    }
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
                 "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar)));
    mbar_wait(su32(&bar), 0);
    const unsigned long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    if (small) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}


// latency of a batch of n dependent (same accumulator) TS MMAs + commit +
// mbarrier wait, issued by one elected lane of warp 0, averaged over reps
__global__ void mma_latency(int N, int n, int reps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) float sm[];
  float* sB = sm;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 64 * 8; i += blockDim.x) sm[i] = 0.0f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t db = sdesc(su32(sB), 128, 256);
    unsigned long long tot = 0;
    for (int r = 0; r < reps; r++) {
      const unsigned long long t0 = clock64();
      for (int k = 0; k < n; k++)
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
                     "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}"
                     ::"r"(tm), "r"(tm + 64), "l"(db), "r"(idesc));
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
                   "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar)));
      mbar_wait(su32(&bar), r & 1);
      tot += clock64() - t0;
    }
    if (t == 0) cyc[blockIdx.x] = tot / reps;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

// N = 24 correctness: D[128 x 24] = A[128 x 8] B[24 x 8]^T, integer operands
__global__ void n24(const float* A, const float* B, float* D, int N) {
  __shared__ __align__(1024) float sA[128 * 8];
  __shared__ __align__(1024) float sB[64 * 8];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  auto kmaj = [](int r, int k) { return (r >> 3) * 64 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3); };  // K = 8
  for (int i = t; i < 128 * 8; i += 128) sA[kmaj(i / 8, i % 8)] = A[i];
  for (int i = t; i < 64 * 8; i += 128) sB[kmaj(i / 8, i % 8)] = i < N * 8 ? B[i] : 0.0f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  // poison D's 64 columns
  {
    uint32_t r[32];
    for (int j = 0; j < 32; j++) r[j] = __float_as_uint(-999.0f);
    ST32(tm + ((uint32_t)(warp * 32) << 16), r);
    ST32(tm + ((uint32_t)(warp * 32) << 16) + 32, r);
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tm), "l"(sdesc(su32(sA), 128, 256)), "l"(sdesc(su32(sB), 128, 256)), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  mbar_wait(su32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[32], q[32];
  LD32(r, tm + ((uint32_t)(warp * 32) << 16));
  LD32(q, tm + ((uint32_t)(warp * 32) << 16) + 32);
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 32; j++) D[t * 64 + j] = __uint_as_float(r[j]);
  for (int j = 0; j < 32; j++) D[t * 64 + 32 + j] = __uint_as_float(q[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

int main(int argc, char** argv) {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, sizeof(unsigned long long) * 1024);
  cudaMalloc(&sink, sizeof(float) * 1024 * 1024);
  unsigned long long h[1024];

  if (argc > 1 && atoi(argv[1]) == 2) {
    for (int n : {1, 2, 6, 11, 22})
      for (int ctas : {1, 4}) {
        mma_latency<<<sms * ctas, 128, 4096>>>(24, n, 64, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("lat error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms * ctas, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < sms * ctas; i++) m += (double)h[i];
        printf("latency: %2d MMAs (N24) + commit + wait, %d CTA/SM: %6.0f cyc\n", n, ctas, m / (sms * ctas));
      }
    return 0;
  }
  const char* names[] = {"ldtm x32 (wait each)", "sttm x32", "ldtm x32 (2 in flight)"};
  for (int mode = 0; mode < 3; mode++)
    for (int warps : {4, 8, 16}) {
      const int iters = 4096;
      tmem_bw<<<sms, warps * 32>>>(mode, iters, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < sms; i++) m += (double)h[i];
      m /= sms;
      const double bytes = (double)iters * warps * 32 * 32 * 4;
      printf("%-24s warps %2d: %8.1f B/cyc/SM (%.1f cyc per warp-instr)\n", names[mode], warps, bytes / m,
             m / ((double)iters * warps / (mode == 2 ? 1 : 1)));
    }
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int ts = 0; ts < 2; ts++)
    for (int N : {16, 24, 32, 48, 64}) {
      const int n_mma = 2048;
      mma_rate<<<sms, 128, 64 * 1024>>>(N, ts, n_mma, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("mma N=%d error %s\n", N, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < sms; i++) m += (double)h[i];
      m /= sms;
      printf("mma tf32 %s M128 N%-3d K8: %6.2f cyc/MMA (floor 128N/256 = %5.1f) -> %6.0f MAC/cyc/SM\n", ts ? "TS" : "SS", N,
             m / n_mma, 128.0 * N / 256, 128.0 * N * 8 / (m / n_mma));
    }

  cudaFuncSetAttribute(mma_chains, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int ts = 0; ts < 2; ts++)
    for (int acc_mode = 1; acc_mode < 1; acc_mode++)
      for (int N : {24, 32, 64})
        for (int NC : {1, 2, 4, 7}) {
          const int n_mma = 2016;
          mma_chains<<<sms, 128, 64 * 1024>>>(N, ts, n_mma, NC, acc_mode, cyc);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("chains error %s\n", cudaGetErrorString(e));
            return 1;
          }
          cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
          double m = 0;
          for (int i = 0; i < sms; i++) m += (double)h[i];
          m /= sms;
          printf("chains %s acc=%d N%-3d NC %d: %6.2f cyc/MMA (floor %5.1f)\n", ts ? "TS" : "SS", acc_mode, N, NC,
                 m / n_mma, 128.0 * N / 256);
        }
  // several CTAs per SM, one chain each (independent issuers): 4 x 128 columns
  for (int ctas : {2, 4})
    for (int N : {24, 32}) {
      const int n_mma = 2016;
      cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 / ctas);
      mma_rate<<<sms * ctas, 128, 200 * 1024 / ctas>>>(N, 1, n_mma, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("multi-cta error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms * ctas, cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < sms * ctas; i++) m += (double)h[i];
      m /= sms * ctas;
      printf("%d CTAs/SM, one TS chain each, N%d: %6.2f cyc per MMA per CTA -> %.2f cyc/MMA per SM\n", ctas, N, m / n_mma,
             m / n_mma / ctas);
    }

  cudaFuncSetAttribute(mma_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int ts = 0; ts < 2; ts++)
    for (int sep = 0; sep < 2; sep++)
      for (int N : {24, 32, 64, 128}) {
        const int n_iter = 256;
        mma_burst<<<sms, 128, 64 * 1024>>>(N, ts, n_iter, sep, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("burst error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < sms; i++) m += (double)h[i];
        m /= sms;
        printf("burst %s sep=%d N%-3d: %6.2f cyc/MMA (floor %5.1f)\n", ts ? "TS" : "SS", sep, N, m / (8.0 * n_iter),
               128.0 * N / 256);
      }

  for (int ctas : {2, 4})
    for (int N : {24, 48}) {
      const int n_iter = 256;
      cudaFuncSetAttribute(mma_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 / ctas);
      mma_burst<<<sms * ctas, 128, 200 * 1024 / ctas>>>(N, 1, n_iter, 0, cyc, 1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("burst multi error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms * ctas, cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < sms * ctas; i++) m += (double)h[i];
      m /= sms * ctas;
      printf("burst TS %d CTAs/SM N%d: %6.2f cyc/MMA per CTA -> %.2f per SM\n", ctas, N, m / (8.0 * n_iter),
             m / (8.0 * n_iter) / ctas);
    }
  // N = 24 correctness
  float *A, *B, *D;
  cudaMallocManaged(&A, 128 * 8 * 4);
  cudaMallocManaged(&B, 64 * 8 * 4);
  cudaMallocManaged(&D, 128 * 64 * 4);
  for (int i = 0; i < 128 * 8; i++) A[i] = (float)(rand() % 9 - 4);
  for (int i = 0; i < 64 * 8; i++) B[i] = (float)(rand() % 9 - 4);
  for (int N : {24, 40}) {
    n24<<<1, 128>>>(A, B, D, N);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("n%d error %s\n", N, cudaGetErrorString(e));
      return 1;
    }
    int bad = 0, untouched = 0;
    for (int r = 0; r < 128; r++)
      for (int n = 0; n < 64; n++) {
        if (n < N) {
          float ref = 0;
          for (int k = 0; k < 8; k++) ref += A[r * 8 + k] * B[n * 8 + k];
          bad += D[r * 64 + n] != ref;
        } else {
          untouched += D[r * 64 + n] == -999.0f;
        }
      }
    printf("N=%d MMA: %d wrong of %d, %d of %d columns beyond N untouched\n", N, bad, 128 * N, untouched, 128 * (64 - N));
  }
  printf("sm clock attr %d kHz\n", clk);
  return 0;
}
