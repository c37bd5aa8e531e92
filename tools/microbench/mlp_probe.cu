// ARM-MLP operand-delivery probe: 16->24->24->2 FFMA2 MLP on synthetic
// activations, weights from (a) the kernel-parameter bank (LDCU -> uniform
// registers) or (b) shared memory (broadcast LDS), NLAT latents per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2pack(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float2 f2unpack(uint64_t v) { float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

struct W { float2 w0[16][12]; float2 b0[12]; float2 w1[24][12]; float2 b1[12]; float2 wo[24]; float2 bo; };

template <int M, int NIN, int NO2, class WT, class BT>
__device__ __forceinline__ void layer(const float (&in)[M][NIN], float (&out)[M][2 * NO2], const WT& Wm, const BT& B) {
  uint64_t acc[M][NO2];
#pragma unroll
  for (int n = 0; n < NO2; n++) { uint64_t b = *reinterpret_cast<const uint64_t*>(&B[n]);
#pragma unroll
    for (int m = 0; m < M; m++) acc[m][n] = b; }
#pragma unroll
  for (int i = 0; i < NIN; i++)
#pragma unroll
    for (int m = 0; m < M; m++) {
      uint64_t x = f2pack(in[m][i], in[m][i]);
#pragma unroll
      for (int n = 0; n < NO2; n++) acc[m][n] = ffma2(x, *reinterpret_cast<const uint64_t*>(&Wm[i][n]), acc[m][n]);
    }
#pragma unroll
  for (int m = 0; m < M; m++)
#pragma unroll
    for (int n = 0; n < NO2; n++) { float2 v = f2unpack(acc[m][n]); out[m][2*n] = fmaxf(v.x, 0.f); out[m][2*n+1] = fmaxf(v.y, 0.f); }
}

template <int M, bool SMEM>
__global__ void __launch_bounds__(256, 2) k(const __grid_constant__ W w, float* out, int iters) {
  __shared__ W ws;
  if (SMEM) { for (int i = threadIdx.x; i < (int)(sizeof(W) / 4); i += 256) reinterpret_cast<float*>(&ws)[i] = reinterpret_cast<const float*>(&w)[i]; __syncthreads(); }
  const W& ww = SMEM ? ws : w;
  float s = 0.f;
  for (int it = 0; it < iters; it++) {
    float z0[M][16];
#pragma unroll
    for (int m = 0; m < M; m++)
#pragma unroll
      for (int c = 0; c < 16; c++) z0[m][c] = (float)((threadIdx.x + c + m + it) & 7) - 3.f;
    float z1[M][24], z2[M][24];
    layer<M, 16, 12>(z0, z1, ww.w0, ww.b0);
    layer<M, 24, 12>(z1, z2, ww.w1, ww.b1);
#pragma unroll
    for (int m = 0; m < M; m++) {
      uint64_t o = *reinterpret_cast<const uint64_t*>(&ww.bo);
#pragma unroll
      for (int n = 0; n < 24; n++) o = ffma2(f2pack(z2[m][n], z2[m][n]), *reinterpret_cast<const uint64_t*>(&ww.wo[n]), o);
      float2 v = f2unpack(o); s += v.x + v.y;
    }
  }
  if (s == 1234.5f) out[0] = s;
}

int main() {
  W w; float* hw = reinterpret_cast<float*>(&w);
  for (int i = 0; i < (int)(sizeof(W) / 4); i++) hw[i] = 0.01f * ((i * 37) % 17 - 8);
  float* d; cudaMalloc(&d, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 2 * 8; int iters = 64;
  auto run = [&](const char* name, int M, auto launch) {
    for (int i = 0; i < 3; i++) launch();
    cudaEventRecord(a); for (int i = 0; i < 5; i++) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    double fma = (double)blocks * 256 * iters * M * 1008;
    printf("%-14s M=%d %.3f ms  %.1f TFLOP/s  %.1f%% of 74.45\n", name, M, ms, 2 * fma / ms / 1e9, 100 * 2 * fma / ms / 1e9 / 74.45);
  };
  run("param", 1, [&] { k<1, false><<<blocks, 256>>>(w, d, iters); });
  run("param", 2, [&] { k<2, false><<<blocks, 256>>>(w, d, iters); });

  iters = 4096;
  run("param-long", 2, [&] { k<2, false><<<blocks, 256>>>(w, d, iters); });
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
