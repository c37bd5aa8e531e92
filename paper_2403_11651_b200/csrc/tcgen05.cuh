// tcgen05.cuh -- the 5th-generation tensor-core primitives shared by the
// tensor-core kernels (arm_tc.cu, analysis_tc.cu): shared-memory matrix
// descriptors, tcgen05.mma kind::tf32 (A from shared memory or from TMEM),
// commit / mbarrier wait, TMEM loads and stores.
#pragma once
#include <cstdint>

namespace ccrd {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // version 1, no swizzle
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(phase));
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// TMEM lane block of this warp -> NP fp32 registers (this thread's latent)
template <int NP>
__device__ __forceinline__ void tmem_row(uint32_t taddr, float (&v)[NP]);
template <>
__device__ __forceinline__ void tmem_row<32>(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; j++) v[j] = __uint_as_float(r[j]);
}
template <>
__device__ __forceinline__ void tmem_row<16>(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; j++) v[j] = __uint_as_float(r[j]);
}

// K-major SWIZZLE_128B descriptor (layout type 2): 8-row x 128-byte atoms,
// 1024-byte aligned, 16-byte chunks XOR-ed with the row (r & 7); SBO = 1024
// (next 8-row group), LBO unused (1).  A K step inside the atom advances the
// start address by its byte offset.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// D (TMEM) (+)= A (TMEM, M lanes x K columns) x B (shared memory)
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

// 32 columns of this warp's 32 TMEM lanes <- registers (no wait)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- no-wait TMEM shapes (issue several, then one tcgen05.wait): 32x32b.x8 / x16 / x32
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// N consecutive columns (N % 8 == 0) of this warp's lanes -> registers, one wait
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[N]) {
  static_assert(N % 8 == 0, "multiples of 8 columns");
  uint32_t r[N];
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16) tmem_ld16_nw(taddr + c, r + c);
  if constexpr (N % 16 == 8) tmem_ld8_nw(taddr + (N - 8), r + (N - 8));
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < N; c++) v[c] = __uint_as_float(r[c]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
// registers -> N consecutive columns (no wait)
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const float (&v)[N]) {
  static_assert(N % 8 == 0, "multiples of 8 columns");
  uint32_t r[N];
#pragma unroll
  for (int c = 0; c < N; c++) r[c] = __float_as_uint(v[c]);
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16) tmem_st16u(taddr + c, r + c);
  if constexpr (N % 16 == 8) tmem_st8(taddr + (N - 8), r + (N - 8));
}

// One elected lane of a CONVERGED warp issues the MMA (every lane executes the
// asm with warp-uniform operands, so ptxas emits a plain predicated UTCHMMA
// instead of a per-lane ELECT loop: measured ~25 vs ~96 cycles per MMA issue,
// tools/microbench/tc_bench.cu).  D (TMEM) (+)= A (TMEM) x B (shared memory).
__device__ __forceinline__ void mma_tf32_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                                  uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.b32 q, %4, 0;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, q;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)));
}

// mbarrier wait with a suspend-time hint: the thread sleeps in the barrier
// until the phase completes (or ~1 ms passes) instead of spinning through
// try_wait timeouts (measured: ~25 spin iterations per wait without a hint).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(phase), "n"(1000000));
}

// Whole MMA batches in ONE asm statement issued by one elected lane of a
// converged warp: the descriptors of consecutive K steps differ by 256 bytes
// (16 in the descriptor's address field), the lo operand by a constant; the
// batch ends with the commit to `bar`.  (Per-MMA asm statements cost ~28
// SASS instructions each -- ELECT / VOTEU / R2UR / descriptor rebuilds.)
#define CCRD_MMA_TS(D, A, B, ACC) "@p tcgen05.mma.cta_group::1.kind::tf32 [" D "], [" A "], " B ", %2, " ACC ";\n\t"
#define CCRD_ADVANCE "add.s64 bh, bh, 16;\n\tadd.s64 bl, bl, 16;\n\tadd.u32 a, a, 8;\n\t"
// D = A0 x (B_hi + B_lo) over KS k-steps; A in TMEM at columns a .. a + 8 KS
template <int KS>
__device__ __forceinline__ void mma_batch_hilo(uint32_t d, uint32_t a, uint64_t bh, uint32_t idesc, uint64_t* bar,
                                               uint32_t lo_off16);
template <>
__device__ __forceinline__ void mma_batch_hilo<3>(uint32_t d, uint32_t a, uint64_t bh, uint32_t idesc, uint64_t* bar,
                                                  uint32_t lo_off16) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bh, bl;\n\t.reg .b32 a;\n\t"
      "elect.sync _|p, 0xffffffff;\n\tmov.b64 bh, %3;\n\tcvt.u64.u32 bl, %5;\n\tadd.s64 bl, bh, bl;\n\tmov.b32 a, %1;\n\t"
      CCRD_MMA_TS("%0", "a", "bh", "0") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
      ::"r"(d), "r"(a), "r"(idesc), "l"(bh), "r"(smem_u32(bar)), "r"(lo_off16));
}
template <>
__device__ __forceinline__ void mma_batch_hilo<4>(uint32_t d, uint32_t a, uint64_t bh, uint32_t idesc, uint64_t* bar,
                                                  uint32_t lo_off16) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bh, bl;\n\t.reg .b32 a;\n\t"
      "elect.sync _|p, 0xffffffff;\n\tmov.b64 bh, %3;\n\tcvt.u64.u32 bl, %5;\n\tadd.s64 bl, bh, bl;\n\tmov.b32 a, %1;\n\t"
      CCRD_MMA_TS("%0", "a", "bh", "0") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
      ::"r"(d), "r"(a), "r"(idesc), "l"(bh), "r"(smem_u32(bar)), "r"(lo_off16));
}
// 3xTF32 hidden layer: D = A_hi (B_hi + B_lo) [KS1 k-steps, A_hi at ah] + A_lo B_hi [KSL k-steps, A_lo at al]
template <int KS1, int KSL>
__device__ __forceinline__ void mma_batch_3x(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint32_t idesc,
                                             uint64_t* bar, uint32_t lo_off16);
#define CCRD_3X_HEAD                                                                                         \
  "{\n\t.reg .pred p;\n\t.reg .b64 bh, bl, b0;\n\t.reg .b32 a;\n\t"                                          \
  "elect.sync _|p, 0xffffffff;\n\tmov.b64 bh, %3;\n\tmov.b64 b0, %3;\n\tcvt.u64.u32 bl, %6;\n\tadd.s64 bl, bh, bl;\n\t" \
  "mov.b32 a, %1;\n\t"
#define CCRD_3X_LO_HEAD "mov.b64 bh, b0;\n\tmov.b32 a, %5;\n\t"
#define CCRD_ADV_LO "add.s64 bh, bh, 16;\n\tadd.u32 a, a, 8;\n\t"
template <>
__device__ __forceinline__ void mma_batch_3x<4, 3>(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint32_t idesc,
                                                   uint64_t* bar, uint32_t lo_off16) {
  asm volatile(
      CCRD_3X_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "0") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      CCRD_3X_LO_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_ADV_LO
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_ADV_LO
      CCRD_MMA_TS("%0", "a", "bh", "1")
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
      ::"r"(d), "r"(ah), "r"(idesc), "l"(bh), "r"(smem_u32(bar)), "r"(al), "r"(lo_off16));
}
template <>
__device__ __forceinline__ void mma_batch_3x<3, 2>(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint32_t idesc,
                                                   uint64_t* bar, uint32_t lo_off16) {
  asm volatile(
      CCRD_3X_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "0") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      CCRD_3X_LO_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_ADV_LO
      CCRD_MMA_TS("%0", "a", "bh", "1")
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
      ::"r"(d), "r"(ah), "r"(idesc), "l"(bh), "r"(smem_u32(bar)), "r"(al), "r"(lo_off16));
}

// exact-context layer 0: D = A_hi (B_hi + B_lo) [KS1 k-steps] + A_lo (B_hi + B_lo) [KSL k-steps]
template <int KS1, int KSL>
__device__ __forceinline__ void mma_batch_4t(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint32_t idesc,
                                             uint64_t* bar, uint32_t lo_off16);
#define CCRD_4T_LO_HEAD "mov.b64 bh, b0;\n\tcvt.u64.u32 bl, %6;\n\tadd.s64 bl, bh, bl;\n\tmov.b32 a, %5;\n\t"
template <>
__device__ __forceinline__ void mma_batch_4t<3, 2>(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint32_t idesc,
                                                   uint64_t* bar, uint32_t lo_off16) {
  asm volatile(
      CCRD_3X_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "0") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      CCRD_4T_LO_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
      ::"r"(d), "r"(ah), "r"(idesc), "l"(bh), "r"(smem_u32(bar)), "r"(al), "r"(lo_off16));
}
template <>
__device__ __forceinline__ void mma_batch_4t<4, 3>(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint32_t idesc,
                                                   uint64_t* bar, uint32_t lo_off16) {
  asm volatile(
      CCRD_3X_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "0") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      CCRD_4T_LO_HEAD
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1") CCRD_ADVANCE
      CCRD_MMA_TS("%0", "a", "bh", "1") CCRD_MMA_TS("%0", "a", "bl", "1")
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
      ::"r"(d), "r"(ah), "r"(idesc), "l"(bh), "r"(smem_u32(bar)), "r"(al), "r"(lo_off16));
}

}  // namespace ccrd
