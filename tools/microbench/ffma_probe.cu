// FFMA / FFMA2 throughput probe for sm_100a: decides the FP32 FMA roofline denominator
// (SURVEY.md §8d "Open: FFMA2") and the ARM kernel's operand-delivery strategy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NACC 16
#define ITERS 2048

__constant__ float cW[64];
struct PW { float w[64]; };

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}

// 1: all-register FFMA (x_i * y + acc_i)
__global__ void k_reg(float* out, float y0) {
  float acc[NACC]; float x[NACC];
  for (int i = 0; i < NACC; i++) { acc[i] = threadIdx.x * 1e-7f; x[i] = y0 + (threadIdx.x + i) * 1e-6f; }
  float y = y0 + threadIdx.x * 1e-9f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(x[i], y, acc[i]);
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}
// 2: weight from __constant__ (distinct per accumulator) -> c-bank or ureg operand
__global__ void k_const(float* out, float x0) {
  float acc[NACC];
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-7f;
  float x = x0 + threadIdx.x * 1e-9f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(x, cW[i], acc[i]);
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}
// 3: weight from kernel params
__global__ void k_param(float* out, float x0, PW p) {
  float acc[NACC];
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-7f;
  float x = x0 + threadIdx.x * 1e-9f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(x, p.w[i], acc[i]);
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}
// 4: FFMA2 all-register
__global__ void k_ffma2_reg(float* out, float y0) {
  unsigned long long acc[NACC / 2], x[NACC / 2];
  for (int i = 0; i < NACC / 2; i++) { acc[i] = pack2(threadIdx.x * 1e-7f, 0.f); x[i] = pack2(y0 + (threadIdx.x + i) * 1e-6f, y0 - (threadIdx.x + i) * 1e-6f); }
  float yy = y0 + threadIdx.x * 1e-9f;
  unsigned long long y = pack2(yy, yy * 1.5f);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) acc[i] = ffma2(x[i], y, acc[i]);
  }
  float s = 0; for (int i = 0; i < NACC / 2; i++) { float a, b; unpack2(acc[i], a, b); s += a + b; }
  if (s == 12345.f) out[0] = s;
}
// 5: FFMA2 with weight pairs from kernel params (two output neurons per instr)
__global__ void k_ffma2_param(float* out, float x0, PW p) {
  unsigned long long acc[NACC / 2];
  for (int i = 0; i < NACC / 2; i++) acc[i] = pack2(threadIdx.x * 1e-7f, 0.f);
  float xx = x0 + threadIdx.x * 1e-9f;
  unsigned long long x = pack2(xx, xx);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) acc[i] = ffma2(x, pack2(p.w[2 * i], p.w[2 * i + 1]), acc[i]);
  }
  float s = 0; for (int i = 0; i < NACC / 2; i++) { float a, b; unpack2(acc[i], a, b); s += a + b; }
  if (s == 12345.f) out[0] = s;
}
// 6: FFMA imm-form
__global__ void k_imm(float* out, float x0) {
  float acc[NACC];
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-7f;
  float x = x0 + threadIdx.x * 1e-9f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(x, 1.0001f + i * 0.001f, acc[i]);
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* d; cudaMalloc(&d, 64);
  float hw[64]; PW pw; for (int i = 0; i < 64; i++) { hw[i] = 1.0f + i * 1e-3f; pw.w[i] = hw[i]; }
  cudaMemcpyToSymbol(cW, hw, sizeof(hw));
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, clk);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int sms = prop.multiProcessorCount;
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads) * 4;
    double fmas = (double)blocks * threads * ITERS * NACC;
    auto run = [&](const char* name, auto launch) {
      for (int w = 0; w < 3; w++) launch();
      cudaEventRecord(a);
      for (int r = 0; r < 5; r++) launch();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
      double rate = fmas / (ms * 1e-3);
      printf("threads %4d %-12s %8.3f ms  %.3e FMA/s  = %.1f FMA/clk/SM @%.0f MHz nominal\n", threads, name, ms, rate,
             rate / sms / (clk * 1e3), clk / 1e3);
    };
    run("reg", [&] { k_reg<<<blocks, threads>>>(d, 1.0f); });
    run("const", [&] { k_const<<<blocks, threads>>>(d, 1.0f); });
    run("param", [&] { k_param<<<blocks, threads>>>(d, 1.0f, pw); });
    run("imm", [&] { k_imm<<<blocks, threads>>>(d, 1.0f); });
    run("ffma2_reg", [&] { k_ffma2_reg<<<blocks, threads>>>(d, 1.0f); });
    run("ffma2_param", [&] { k_ffma2_param<<<blocks, threads>>>(d, 1.0f, pw); });
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
