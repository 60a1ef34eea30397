// PCG64 stream arithmetic and numpy's float64 pairwise summation on the
// device, shared by K8 (wor.cu) and K9 (select.cu).
//
//  - numpy Generator.random(): state <- state * M + inc (128-bit LCG), output
//    XSL-RR 128/64, double = (out >> 11) * 2^-53.  Output k (0-based) of a
//    stream is the output of the state advanced k+1 steps (pcg_advance).
//  - numpy add.reduce over float64 (loops_utils.h pairwise_sum): blocks of
//    <= 128 with 8 strided accumulators; larger ranges split in halves at a
//    multiple of 8.
#pragma once

#include "common.cuh"

namespace tg {

struct u128 {
  uint64_t hi, lo;
};

__device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}
__device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

constexpr uint64_t PCG_MUL_HI = 0x2360ED051FC65DA4ull;
constexpr uint64_t PCG_MUL_LO = 0x4385DF649FCCF645ull;

// state advanced by `delta` LCG steps (standard square-and-multiply jump).
static __device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mul{0, 1}, acc_add{0, 0};
  u128 cur_mul{PCG_MUL_HI, PCG_MUL_LO}, cur_add = inc;
  while (delta) {
    if (delta & 1) {
      acc_mul = mul128(acc_mul, cur_mul);
      acc_add = add128(mul128(acc_add, cur_mul), cur_add);
    }
    cur_add = mul128(add128(cur_mul, u128{0, 1}), cur_add);
    cur_mul = mul128(cur_mul, cur_mul);
    delta >>= 1;
  }
  return add128(mul128(acc_mul, state), acc_add);
}

// XSL-RR 128/64 output of a state; double = (x >> 11) * 2^-53 (numpy random()).
__device__ __forceinline__ double pcg_double(u128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = static_cast<unsigned>(s.hi >> 58);
  const uint64_t o = (x >> rot) | (x << ((64u - rot) & 63u));
  return static_cast<double>(o >> 11) * (1.0 / 9007199254740992.0);
}

// numpy pairwise_sum for n <= 128 over a[i*stride] (loops_utils.h: n < 8 is a
// plain loop from 0., otherwise 8 strided accumulators then the tail).
__device__ __forceinline__ double pw_block(const double* a, int n, int stride) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[(i + j) * stride]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
  return res;
}

// numpy pairwise_sum for n <= 248 (one recursive split: n2 = n/2 - (n/2)%8).
__device__ __forceinline__ double pw_sum(const double* a, int n, int stride) {
  if (n <= 128) return pw_block(a, n, stride);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_block(a, n2, stride), pw_block(a + n2 * stride, n - n2, stride));
}

}  // namespace tg
