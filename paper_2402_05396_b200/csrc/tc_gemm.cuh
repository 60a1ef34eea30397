// 3xTF32 GEMM on the 5th-generation tensor cores (tcgen05, TMEM accumulators)
// for the f32 path of K7 (score.cu).
//
//   C[M, N] = epilogue( A'[M, K] @ W[K, N] ),   A' = A or LN(A) (fused)
//
// Precision: operands are split x = x_hi + x_lo + O(2^-23 x) with
// x_hi = rna_tf32(x), x_lo = rna_tf32(x - x_hi), and every product is
// a_hi*b_hi + (a_hi*b_lo + a_lo*b_hi) -- three kind::tf32 MMAs per K step
// (the dropped a_lo*b_lo is 2^-22 relative; measured: adding it changes
// nothing, the error is the tensor core's accumulator, see below).
//
// The hi*hi products accumulate in one TMEM accumulator, the two correction
// products in a second one (2^-11 smaller, so its own rounding is
// negligible); the epilogue adds them in IEEE fp32.  Folding the corrections
// into the main accumulator would triple the accumulator roundings and
// costs ~3x the error of an fp32 FFMA GEMM.
//
// CTA = 128 rows x one N tile (<= 128 columns, multiple of 16); TMEM holds
// both accumulators in 2*Nt <= 256 columns -> two CTAs per SM.
// Warp roles (192 threads):
//   warps 0-3  A producers: each thread owns one row, loads 8 K-elements per
//              stage (two float4, prefetched PF stages ahead in registers),
//              applies the fused LayerNorm, splits hi/lo and writes the
//              canonical K-major core-matrix layout; then the epilogue
//              (tcgen05.ld 32x32b: thread = row, 16 columns per load).
//   warp 4     lane 0: issues the 3 MMAs of a stage (single thread,
//              tcgen05.mma) and releases it with tcgen05.commit.
//   warp 5     lane 0: bulk-copies the pre-packed weight image of each stage
//              (cp.async.bulk, mbarrier complete_tx), running STAGES ahead.
// Stage = one MMA K-step (8 tf32): A hi|lo 2 x 4 KB, W hi|lo 2 x Nt*32 B.
#pragma once

#include "common.cuh"

namespace tg {
namespace tc {

constexpr int BM = 128;
constexpr int MAX_NT = 128;   // N per CTA (one instruction, N % 16 == 0)
constexpr int KSTEP = 8;      // tf32 elements per MMA
#ifndef TG_KPER
#define TG_KPER 2
#endif
constexpr int KPER = TG_KPER;  // K steps per pipeline stage (1 or 2)
static_assert(KPER == 1 || KPER == 2, "raw-A tile swizzle covers 32- and 64-byte rows");
constexpr int STAGES = 6;     // 6 x (16 KB A + 2 x 2 x Nt x 32 B W) <= 192 KB; 7 stages measured 20% slower
                              // (the larger carve-out leaves the epilogue's loads no L1)
constexpr int EPW = 16;                 // epilogue warps: 4 per TMEM lane quarter
constexpr int EPARTS = EPW / 4;         // column parts per row (one per warp of a quarter)
constexpr int THREADS = 64 + 32 * EPW;  // loader warp + MMA warp + epilogue
constexpr int CONV_WARPS = 4 * KPER;    // raw-A variant: converter warps per chunk (a K step per four)
#ifndef TG_CONV_GROUPS
#define TG_CONV_GROUPS 2
#endif
#ifndef TG_RA_EPW
#define TG_RA_EPW 8
#endif
constexpr int CONV_GROUPS = TG_CONV_GROUPS;  // raw-A variant: converter groups taking alternate chunks
constexpr int RA_EPW = TG_RA_EPW;            // raw-A variant: epilogue warps (a multiple of 4)
constexpr int RA_THREADS = 64 + 32 * (CONV_WARPS * CONV_GROUPS + RA_EPW);
#ifndef TG_DOT_GROUPS
#define TG_DOT_GROUPS 1
#endif
#ifndef TG_DOT_EPW
#define TG_DOT_EPW 16
#endif
constexpr int DOT_GROUPS = TG_DOT_GROUPS;  // dot epilogues (per-element row-vector loads): converter groups
constexpr int DOT_EPW = TG_DOT_EPW;        // ... and epilogue warps
constexpr int RA_THREADS_DOT = 64 + 32 * (CONV_WARPS * DOT_GROUPS + DOT_EPW);
#ifndef TG_RA_NST
#define TG_RA_NST 5
#endif
constexpr int RA_NST = TG_RA_NST;       // raw-A variant: stages (hi|lo A + W + raw A tile)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TG_DONE_%=;\n\t"
      "bra TG_WAIT_%=;\n"
      "TG_DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// the same wait with a nanosleep back-off between polls: for warps that wait
// long (the epilogue for a whole mainloop), so their spinning does not take
// issue slots from the converter warps on the same schedulers
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  while (!mbar_test(bar, phase)) __nanosleep(200);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Round to the nearest tf32, ties away from zero: the same bits as
// cvt.rna.tf32.f32 (which sm_100 runs as an ~7-instruction sequence with
// inf / NaN guards) in two integer ops -- adding half a tf32 ulp to the
// sign-magnitude bits rounds the magnitude, a carry moves into the
// exponent as it should, and inf stays inf (its mantissa is zero)
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// SMEM matrix descriptor, K-major, no swizzle: core matrix = 8 rows x 16 B
// contiguous; LBO = byte distance between the two K-halves (4 tf32 each),
// SBO = byte distance between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor: kind::tf32, f32 accumulate, A/B K-major.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Same MMA with the A operand kept in the tensor core's collector buffer
// (fill: read A from shared memory and keep it; lastuse: reuse the kept A
// and release it) -- the hi*hi and hi*lo products share A_hi, so the second
// one does not re-read its 4 KB from shared memory.
__device__ __forceinline__ void mma_tf32_afill(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_alast(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// ---- 2-CTA clusters: the weight stage is loaded half by each CTA and
// multicast to both; each CTA's MMA releases the stage in both CTAs.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// One K step of the 3xTF32 product in one asm block, issued by one elected
// lane of a full warp: hi*hi into the main accumulator (A_hi kept in the
// collector), hi*lo and lo*hi into the correction accumulator.  Descriptors
// are passed as 32-bit words (start-address words of A_hi, A_lo, B_hi, B_lo
// and the shared high word) so the loop's arithmetic stays 32-bit.
template <int CG>
__device__ __forceinline__ void mma3_tf32(uint32_t dmain, uint32_t dcorr, uint32_t ah, uint32_t al, uint32_t bh,
                                          uint32_t bl, uint32_t dhi, uint32_t idesc, uint32_t accumulate) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t.reg .b64 dah, dal, dbh, dbl;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %8, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "mov.b64 dah, {%2, %6};\n\tmov.b64 dal, {%3, %6};\n\tmov.b64 dbh, {%4, %6};\n\tmov.b64 dbl, {%5, %6};\n\t"
#ifndef TG_EXP_HIHI_ONLY
        "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], dah, dbh, %7, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%1], dah, dbl, %7, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], dal, dbh, %7, t;\n\t}" ::"r"(dmain),
#else  // timing experiment only (wrong results): the hi*hi product alone
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], dah, dbh, %7, p;\n\t}" ::"r"(dmain),
#endif
        "r"(dcorr), "r"(ah), "r"(al), "r"(bh), "r"(bl), "r"(dhi), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t.reg .b64 dah, dal, dbh, dbl;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %8, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "mov.b64 dah, {%2, %6};\n\tmov.b64 dal, {%3, %6};\n\tmov.b64 dbh, {%4, %6};\n\tmov.b64 dbl, {%5, %6};\n\t"
        "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::fill [%0], dah, dbh, %7, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::lastuse [%1], dah, dbl, %7, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], dal, dbh, %7, t;\n\t}" ::"r"(dmain),
        "r"(dcorr), "r"(ah), "r"(al), "r"(bh), "r"(bl), "r"(dhi), "r"(idesc), "r"(accumulate)
        : "memory");
}

// The MMA / commit helpers are executed by a whole warp and issue from one
// elected lane (elect.sync): warp-uniform operands stay in uniform registers,
// so consecutive MMAs do not serialise on per-lane R2UR broadcasts.
// ---- CTA pairs (cta_group::2): one 256 x N MMA over both SMs; each CTA
// holds its 128 rows of A and half (N/2 rows) of B; the leader issues.
__device__ __forceinline__ void mma_tf32_afill_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                    uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_alast_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                    uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// completion of the pair's MMAs -> the barrier at this offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
// arrive on the barrier at this offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// 16 TMEM columns of this warp's 32 lanes into registers (no wait: issue
// several, then tmem_wait_ld once)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  tmem_ld16_nowait(taddr, r);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// byte offset of (row, k) inside one K-step block of a K-major canonical tile
__device__ __forceinline__ uint32_t core_off(int row, int k) {
  return (uint32_t)((row >> 3) * 256 + (row & 7) * 16 + (k >> 2) * 128 + (k & 3) * 4);
}

}  // namespace tc
}  // namespace tg
