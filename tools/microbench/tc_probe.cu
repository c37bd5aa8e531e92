// tcgen05 tf32 probe (SS = both operands in shared memory; TS = A in TMEM,
// written with tcgen05.st 32x32b: lane = row, one tf32 per column): D[128 x 32] = A[128 x 24] . B[32 x 24]^T with K-major,
// no-swizzle canonical operands in shared memory, accumulated over 3 k=8
// MMAs, read back with tcgen05.ld 32x32b.  Validates the descriptor encodings
// used by the tensor-core ARM kernel.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tc_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 24;

// element (r, k) of a K-major operand with `rows` rows: core matrix (r/8, k/4)
// of 8 rows x 16 bytes; core matrices K-adjacent at LBO = 128 B, 8-row groups
// at SBO = (K/4) * 128 B
__host__ __device__ inline int kmaj_off(int r, int k) {
  return (r >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);  // in floats
}

__device__ inline uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (Blackwell)
  return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__global__ void probe(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) float sA[M * K];
  __shared__ __align__(1024) float sB[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < M * K; i += blockDim.x) sA[kmaj_off(i / K, i % K)] = A[i];
  for (int i = t; i < N * K; i += blockDim.x) sB[kmaj_off(i / K, i % K)] = B[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sA), b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int s = 0; s < K / 8; s++) {
      const uint64_t da = smem_desc(a0 + s * 256, 128, (K / 4) * 128);
      const uint64_t db = smem_desc(b0 + s * 256, 128, (K / 4) * 128);
      const uint32_t acc = s > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
  }
  // wait phase 0
  {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(b), "r"(0u));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 32; j++) D[t * N + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

__global__ void probe_ts(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) float sB[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < N * K; i += blockDim.x) sB[kmaj_off(i / K, i % K)] = B[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;               // D: columns 0..31, A: columns 32..32+K-1
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  {
    uint32_t a[K];
    for (int k = 0; k < K; k++) a[k] = __float_as_uint(A[t * K + k]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(tmem + lane_base + 32), "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]),
                 "r"(a[6]), "r"(a[7]), "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]),
                 "r"(a[15]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(tmem + lane_base + 48), "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]),
                 "r"(a[22]), "r"(a[23]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int s = 0; s < K / 8; s++) {
      const uint64_t db = smem_desc(b0 + s * 256, 128, (K / 4) * 128);
      const uint32_t acc = s > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
          "r"(tmem + 32 + 8 * s), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
  }
  {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(b), "r"(0u));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tmem + lane_base));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 32; j++) D[t * N + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}


int check(const char* name, const float* A, const float* B, const float* D) {
  int bad = 0;
  double maxerr = 0;
  for (int r = 0; r < M; r++)
    for (int n = 0; n < N; n++) {
      double ref = 0;
      for (int k = 0; k < K; k++) ref += (double)A[r * K + k] * B[n * K + k];
      const double err = fabs(ref - D[r * N + n]);
      maxerr = err > maxerr ? err : maxerr;
      if (err > 1e-6 && bad++ < 5) printf("%s mismatch r=%d n=%d got %f want %f\n", name, r, n, D[r * N + n], ref);
    }
  printf("tc_probe %s: %s (max err %g, %d bad)\n", name, bad ? "FAIL" : "OK", maxerr, bad);
  return bad;
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, sizeof(float) * M * K);
  cudaMallocManaged(&B, sizeof(float) * N * K);
  cudaMallocManaged(&D, sizeof(float) * M * N);
  srand(1);
  // integer-valued operands: tf32 products and sums are exact
  for (int i = 0; i < M * K; i++) A[i] = (float)(rand() % 17 - 8);
  for (int i = 0; i < N * K; i++) B[i] = (float)(rand() % 9 - 4) * 0.25f;
  probe<<<1, 128>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  int bad = check("SS", A, B, D);
  for (int i = 0; i < M * N; i++) D[i] = -1.0f;
  probe_ts<<<1, 128>>>(A, B, D);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error (TS) %s\n", cudaGetErrorString(e));
    return 1;
  }
  bad += check("TS", A, B, D);
  return bad != 0;
}
