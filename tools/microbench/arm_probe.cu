// Attribute the ARM kernel's loss vs the pure FFMA2 MLP: variants add the
// shared-memory context gather (runtime uniform offsets), the Laplace bits and
// the per-unit partial store on top of the mlp_probe loop.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2pack(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float2 f2unpack(uint64_t v) { float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

struct W { float2 w0[16][12]; float2 b0[12]; float2 w1[24][12]; float2 b1[12]; float2 wo[24]; float2 bo; int dy[16], dx[16]; };

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

__device__ __forceinline__ float laplace_bits(float y, float mu, float s) {
  s = fminf(fmaxf(s, -6.9f), 5.5f);
  const float ib = __expf(-s);
  const float a = fabsf(y - mu);
  const float am = fminf(a, 0.5f);
  const float e1 = __expf((am - 0.5f) * ib);
  const float e2 = __expf(-(am + 0.5f) * ib);
  const float p_in = 1.0f - 0.5f * (e1 + e2);
  const float bits_in = -__log2f(fmaxf(p_in, 1.5e-5f));
  const float bits_out = 1.0f + (a - 0.5f) * ib * 1.4426950408889634f - __log2f(-expm1f(-ib));
  return fminf(a < 0.5f ? bits_in : bits_out, 16.f);
}

// V bits: 1 = smem ctx gather, 2 = laplace, 4 = partial store
template <int V>
__global__ void __launch_bounds__(256, 2) k(const __grid_constant__ W w, double* out, int iters) {
  constexpr int M = 2;
  __shared__ float ring[8][4][72];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * 4 * 72; i += 256) (&ring[0][0][0])[i] = (float)((i * 7) % 9 - 4);
  __syncthreads();
  float s = 0.f;
  for (int it = 0; it < iters; it++) {
    float z0[M][16], y[M];
    if (V & 1) {
#pragma unroll
      for (int c = 0; c < 16; c++) {
        const float* rp = ring[warp][(it + w.dy[c]) & 3] + 4 + w.dx[c] + lane;
#pragma unroll
        for (int m = 0; m < M; m++) z0[m][c] = rp[32 * m];
      }
#pragma unroll
      for (int m = 0; m < M; m++) y[m] = ring[warp][it & 3][4 + lane + 32 * m];
    } else {
#pragma unroll
      for (int m = 0; m < M; m++) {
#pragma unroll
        for (int c = 0; c < 16; c++) z0[m][c] = (float)((threadIdx.x + c + m + it) & 7) - 3.f;
        y[m] = 1.f;
      }
    }
    float z1[M][24], z2[M][24];
    layer<M, 16, 12>(z0, z1, w.w0, w.b0);
    layer<M, 24, 12>(z1, z2, w.w1, w.b1);
    float bits = 0.f;
#pragma unroll
    for (int m = 0; m < M; m++) {
      uint64_t o = *reinterpret_cast<const uint64_t*>(&w.bo);
#pragma unroll
      for (int n = 0; n < 24; n++) o = ffma2(f2pack(z2[m][n], z2[m][n]), *reinterpret_cast<const uint64_t*>(&w.wo[n]), o);
      float2 v = f2unpack(o);
      bits += (V & 2) ? laplace_bits(y[m], v.x, v.y) : v.x + v.y;
    }
    if (V & 4) {
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o2);
      if (lane == 0) out[(blockIdx.x * 8 + warp) * iters + it] = bits;
    } else {
      s += bits;
    }
  }
  if (s == 1234.5f) out[0] = s;
}

int main() {
  W w; float* hw = reinterpret_cast<float*>(&w);
  for (int i = 0; i < (int)(sizeof(W) / 4) - 32; i++) hw[i] = 0.01f * ((i * 37) % 17 - 8);
  const int dy[16] = {0, 0, -1, -1, -1, -1, -1, 0, -2, -2, -2, -1, -1, -2, -2, -2};
  const int dx[16] = {-1, -2, 0, -1, 1, -2, 2, -3, 0, -1, 1, -3, 3, -2, 2, -3};
  for (int c = 0; c < 16; c++) { w.dy[c] = dy[c]; w.dx[c] = dx[c]; }
  const int blocks = 148 * 2 * 8, iters = 64;
  double* d; cudaMalloc(&d, sizeof(double) * blocks * 8 * iters);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; i++) launch();
    cudaEventRecord(a); for (int i = 0; i < 5; i++) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    double fma = (double)blocks * 256 * iters * 2 * 1008;
    printf("%-22s %.3f ms  %.1f TFLOP/s  %.1f%% of 74.45\n", name, ms, 2 * fma / ms / 1e9, 100 * 2 * fma / ms / 1e9 / 74.45);
  };
  run("mlp", [&] { k<0><<<blocks, 256>>>(w, d, iters); });
  run("+ctx", [&] { k<1><<<blocks, 256>>>(w, d, iters); });
  run("+laplace", [&] { k<2><<<blocks, 256>>>(w, d, iters); });
  run("+partial", [&] { k<4><<<blocks, 256>>>(w, d, iters); });
  run("+ctx+laplace", [&] { k<3><<<blocks, 256>>>(w, d, iters); });
  run("+ctx+laplace+partial", [&] { k<7><<<blocks, 256>>>(w, d, iters); });
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
