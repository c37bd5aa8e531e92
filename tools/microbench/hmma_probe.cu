// Legacy mma.sync throughput on sm_100a (no TMEM): 8 independent accumulator
// chains per warp, W warps per SM.  Reports MAC/clk/SM for m16n8k8 tf32 and
// m16n8k16 f16 / bf16 (fp32 accumulators).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int iters, float* out, unsigned long long* cyc) {
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float d[8][4];
  for (int c = 0; c < 8; c++)
    for (int j = 0; j < 4; j++) d[c][j] = 0.f;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < 8; c++)
      if (MODE == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else if (MODE == 1)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const unsigned long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < 8; c++)
    for (int j = 0; j < 4; j++) s += d[c][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// latency: one dependent chain of m16n8k8 tf32 MMAs, one warp
__global__ void lat(int iters, float* out, unsigned long long* cyc) {
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  const unsigned long long t1 = clock64();
  out[threadIdx.x] = d[0] + d[1] + d[2] + d[3];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8 * 4096);
  for (int mode = 0; mode < 3; mode++)
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 2048;
    if (mode == 0) k<0><<<sms, warps * 32>>>(iters, out, cyc);
    if (mode == 1) k<1><<<sms, warps * 32>>>(iters, out, cyc);
    if (mode == 2) k<2><<<sms, warps * 32>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    unsigned long long h[1024];
    cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < sms; i++) m += h[i];
    m /= sms;
    const double macs = (double)iters * 8 * warps * 16 * 8 * (mode == 0 ? 8 : 16);
    printf("mma.sync %s, %2d warps/SM: %7.1f MAC/clk/SM (%.1f cyc per mma per warp)\n",
           mode == 0 ? "m16n8k8 tf32" : mode == 1 ? "m16n8k16 f16" : "m16n8k16 bf16", warps, macs / m,
           m / (iters * 8.0));
  }
  {
    lat<<<1, 32>>>(4096, out, cyc);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("mma.sync m16n8k8 tf32 dependent chain: %.1f cycles per mma\n", h / 4096.0);
  }
  return 0;
}
