// 2-D 16-bit TMA window probe (the ARM kernel's staging): box 72 x 11 at
// (c0, c1) of an int16 [h][w] grid, zero fill outside.  Checks the result
// against a host gather.  Variants: map as a __grid_constant__ struct member
// indexed dynamically (as arm_tcg_kernel does) and as a plain parameter.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <cstring>

struct Maps {
  int pad[17];
  CUtensorMap m[4];
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ Maps mp, int which, int c0, int c1, int16_t* out, int bw, int mode) {
  __shared__ __align__(128) int16_t buf[72 * 11 + 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bw * 11 * 2) : "memory");
    if (mode == 2)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %5}], [%2];" ::"r"(
              su32(buf)),
          "l"(reinterpret_cast<uint64_t>(&mp.m[which])), "r"(su32(&bar)), "r"(c0), "r"(c1), "r"(0)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              su32(buf)),
          "l"(reinterpret_cast<uint64_t>(which == 0 ? &mp.m[0] : which == 1 ? &mp.m[1] : which == 2 ? &mp.m[2] : &mp.m[3])), "r"(su32(&bar)), "r"(mode == 1 ? c0 / 2 : c0), "r"(c1)
          : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(&bar)), "r"(0));
  for (int i = threadIdx.x; i < bw * 11; i += blockDim.x) out[i] = buf[i];
}


struct MapFirst {
  CUtensorMap m;
  int pad[17];
};
template <int V>
__global__ void probe_v(const __grid_constant__ CUtensorMap m0, const __grid_constant__ MapFirst mf, int c0, int c1,
                        int16_t* out, int bw) {
  __shared__ __align__(128) int16_t buf[72 * 11 + 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const CUtensorMap* mp = V == 0 ? &m0 : &mf.m;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bw * 11 * 2) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(buf)),
        "l"(reinterpret_cast<uint64_t>(mp)), "r"(su32(&bar)), "r"(c0), "r"(c1)
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(&bar)), "r"(0));
  for (int i = threadIdx.x; i < bw * 11; i += blockDim.x) out[i] = buf[i];
}


__global__ void probe_dyn(const __grid_constant__ CUtensorMap m0, int c0, int c1, int16_t* out, int bw) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  int16_t* buf = reinterpret_cast<int16_t*>(dsm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bw * 11 * 2) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(buf)),
        "l"(reinterpret_cast<uint64_t>(&m0)), "r"(su32(bar)), "r"(c0), "r"(c1)
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(bar)), "r"(0));
  for (int i = threadIdx.x; i < bw * 11; i += blockDim.x) out[i] = buf[i];
}


__global__ void probe_4d(const __grid_constant__ CUtensorMap m0, int16_t* out) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(32 * 4 * 4 * 4) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            su32(dsm)),
        "l"(reinterpret_cast<uint64_t>(&m0)), "r"(su32(bar)), "r"(0), "r"(1), "r"(2), "r"(0)
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(bar)), "r"(0));
  const int16_t* b = reinterpret_cast<const int16_t*>(dsm);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = b[i];
}


template <int RANK>
__global__ void probe_rank(const __grid_constant__ CUtensorMap m0, int16_t* out, int bytes, int a, int b, int c) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
    if (RANK == 4)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
              su32(dsm)),
          "l"(reinterpret_cast<uint64_t>(&m0)), "r"(su32(bar)), "r"(a), "r"(b), "r"(0), "r"(0)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              su32(dsm)),
          "l"(reinterpret_cast<uint64_t>(&m0)), "r"(su32(bar)), "r"(0), "r"(a), "r"(b)
          : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(bar)), "r"(0));
  const int16_t* bb = reinterpret_cast<const int16_t*>(dsm);
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = bb[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int BW = argc > 1 ? atoi(argv[1]) : 72;
  const int c0s = argc > 2 ? atoi(argv[2]) : -4;
  const int mode = argc > 3 ? atoi(argv[3]) : 0;  // 0 uint16 2d, 1 float32 2d (pairs), 2 uint16 4d
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  Enc enc = (Enc)ptr;
  const int h = 40, w = 512;
  std::vector<int16_t> hg(h * w);
  for (int i = 0; i < h * w; i++) hg[i] = (int16_t)((i * 7919) % 601 - 300);
  int16_t *dg, *dout;
  cudaMalloc(&dg, h * w * 2);
  cudaMalloc(&dout, 4096);
  cudaMemcpy(dg, hg.data(), h * w * 2, cudaMemcpyHostToDevice);
  Maps mp;
  memset(&mp, 0, sizeof(mp));
  for (int k = 0; k < 4; k++) {
    const cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)h};
    const cuuint64_t strides[1] = {(cuuint64_t)w * 2};
    const cuuint32_t box[2] = {(cuuint32_t)BW, 11}, es[2] = {1, 1};
    CUresult r;
    if (mode == 14) {  // uint16 4D {w, h, 1, 1} box {64, 11, 1, 1}
      const cuuint64_t d4[4] = {(cuuint64_t)w, (cuuint64_t)h, 1, 1};
      const cuuint64_t s4[3] = {(cuuint64_t)w * 2, (cuuint64_t)w * h * 2, (cuuint64_t)w * h * 2};
      const cuuint32_t b4[4] = {64, 11, 1, 1}, e4[4] = {1, 1, 1, 1};
      r = enc(&mp.m[k], CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, dg, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else if (mode == 15) {  // uint16 3D {8, w/8, h} box {8, 10, 11}
      const cuuint64_t d3[3] = {8, (cuuint64_t)w / 8, (cuuint64_t)h};
      const cuuint64_t s3[2] = {16, (cuuint64_t)w * 2};
      const cuuint32_t b3[3] = {8, 10, 11}, e3[3] = {1, 1, 1};
      r = enc(&mp.m[k], CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, dg, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else if (mode == 13) {  // analysis-identical: FLOAT32 4D [1][h][w/32][32] box {32, 11, 2, 1}
      const cuuint64_t d4[4] = {32, (cuuint64_t)w / 64, (cuuint64_t)h, 1};
      const cuuint64_t s4[3] = {128, (cuuint64_t)w * 2, (cuuint64_t)w * h * 2};
      const cuuint32_t b4[4] = {32, 4, 4, 1}, e4[4] = {1, 1, 1, 1};
      r = enc(&mp.m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dg, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else if (mode == 0 || mode >= 10)
      r = enc(&mp.m[k], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, dg, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    else if (mode == 1) {
      const cuuint64_t d2[2] = {(cuuint64_t)w / 2, (cuuint64_t)h};
      const cuuint32_t b2[2] = {(cuuint32_t)BW / 2, 11};
      r = enc(&mp.m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dg, d2, strides, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const cuuint64_t d4[4] = {(cuuint64_t)w, (cuuint64_t)h, 1, 1};
      const cuuint64_t s4[3] = {(cuuint64_t)w * 2, (cuuint64_t)w * h * 2, (cuuint64_t)w * h * 2};
      const cuuint32_t b4[4] = {(cuuint32_t)BW, 11, 1, 1}, e4[4] = {1, 1, 1, 1};
      r = enc(&mp.m[k], CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, dg, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }

  if (mode >= 10) {
    MapFirst mf;
    memcpy(&mf.m, &mp.m[0], sizeof(CUtensorMap));
    if (mode == 14 || mode == 15) {
      // window origin column c0s (mode 15: c0s / 8 chunks), row -3
      if (mode == 14) probe_rank<4><<<1, 128, 8192>>>(mp.m[0], dout, 64 * 11 * 2, c0s, -3, 0);
      else probe_rank<3><<<1, 128, 8192>>>(mp.m[0], dout, 80 * 11 * 2, c0s / 8, -3, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
      const int cw = mode == 14 ? 64 : 80;
      std::vector<int16_t> o(cw * 11);
      cudaMemcpy(o.data(), dout, cw * 11 * 2, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int r = 0; r < 11; r++)
        for (int c = 0; c < cw; c++) {
          const int gi = -3 + r, gj = (mode == 14 ? c0s : c0s / 8 * 8) + c;
          const int16_t want = (gi >= 0 && gi < h && gj >= 0 && gj < w) ? hg[gi * w + gj] : 0;
          bad += o[r * cw + c] != want;
        }
      printf("mode %d: %d wrong\n", mode, bad);
      return 0;
    }
    if (mode == 13) probe_4d<<<1, 128, 8192>>>(mp.m[0], dout);
    else if (mode == 12) probe_dyn<<<1, 128, 8192>>>(mp.m[0], c0s, 3, dout, BW);
    else if (mode == 10) probe_v<0><<<1, 128>>>(mp.m[0], mf, c0s, -3, dout, BW);
    else probe_v<1><<<1, 128>>>(mp.m[0], mf, c0s, -3, dout, BW);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", mode, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    return 0;
  }
  printf("sizeof(Maps) %zu offsetof m %zu\n", sizeof(Maps), offsetof(Maps, m));
  int bad_total = 0;
  const int coords[4][2] = {{c0s, -3}, {60, 5}, {470, 33}, {100, 20}};
  for (int t = 0; t < 4; t++) {
    probe<<<1, 128>>>(mp, t, coords[t][0], coords[t][1], dout, BW, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("case %d: %s\n", t, cudaGetErrorString(e)); return 1; }
    std::vector<int16_t> o(72 * 11);
    cudaMemcpy(o.data(), dout, 72 * 11 * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 11; r++)
      for (int c = 0; c < BW; c++) {
        const int gi = coords[t][1] + r, gj = coords[t][0] + c;
        const int16_t want = (gi >= 0 && gi < h && gj >= 0 && gj < w) ? hg[gi * w + gj] : 0;
        bad += o[r * BW + c] != want;
      }
    printf("case %d (%d, %d): %d wrong\n", t, coords[t][0], coords[t][1], bad);
    bad_total += bad;
  }
  return bad_total != 0;
}
