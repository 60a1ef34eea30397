// K8: policy sampling without replacement.  Replaces sampler.py:138-176.
//
// The reference runs n vectorised rounds over the whole (B, m) batch:
//   total = probs.sum(axis=1)            numpy pairwise sum (8 accumulators)
//   alive = total > 1e-12
//   u     = rng.random(B) * total        PCG64 output k*B + b for row b
//   pick  = min(#(cumsum(probs) < u), m-1);  probs[pick] = 0
// then sorts each row's picks ascending (stable, padding last) and gathers
// log q of the picks.  Every row only reads its own draw, so one thread owns
// one row: it jumps its PCG64 state to position b+1 (O(log b) 128-bit LCG
// squarings), then advances by B_global per round with the host-computed
// jump constants, reproducing the exact numpy draw.  probs live in shared
// memory laid out [slot][thread] (bank-conflict free); sums use numpy's
// association order so the selection is bit-identical given the same q.
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
__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
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

template <typename T>
__global__ void wor_kernel(const T* __restrict__ q, const T* __restrict__ lq, int64_t B, int m, int n, tg_pcg64 rng,
                           tg_rowmap rows, int64_t* __restrict__ selected, uint8_t* __restrict__ sel_mask,
                           T* __restrict__ sel_lq) {
  extern __shared__ double sm[];
  const int S = blockDim.x;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double* pr = sm + threadIdx.x;  // pr[j*S]
  for (int j = 0; j < m; ++j) pr[j * S] = static_cast<double>(q[b * m + j]);
  const int64_t gb = global_row(rows, b);
  const u128 inc{rng.inc_hi, rng.inc_lo};
  u128 st = pcg_advance(u128{rng.state_hi, rng.state_lo}, inc, static_cast<uint64_t>(gb) + 1);
  const u128 jm{rng.jmul_hi, rng.jmul_lo}, ja{rng.jadd_hi, rng.jadd_lo};
  int64_t* out = selected + b * n;
  int nsel = 0;
  for (int k = 0; k < n; ++k) {
    if (k > 0) st = add128(mul128(jm, st), ja);
    const double total = pw_sum(pr, m, S);
    if (!(total > 1e-12)) break;  // dead rows stay dead: later rounds pick nothing
    const double u = __dmul_rn(pcg_double(st), total);
    double cums = 0.0;
    int below = 0;
    for (int j = 0; j < m; ++j) {
      cums = j == 0 ? pr[0] : __dadd_rn(cums, pr[j * S]);
      below += cums < u;
    }
    const int pick = below < m - 1 ? below : m - 1;
    out[nsel++] = pick;
    pr[pick * S] = 0.0;
  }
  // ascending slot order (stable argsort of picks, padding last)
  for (int a = 1; a < nsel; ++a) {
    const int64_t key = out[a];
    int c = a - 1;
    while (c >= 0 && out[c] > key) {
      out[c + 1] = out[c];
      --c;
    }
    out[c + 1] = key;
  }
  for (int j = nsel; j < n; ++j) out[j] = -1;
  for (int j = 0; j < n; ++j) {
    const bool valid = j < nsel;
    sel_mask[b * n + j] = valid ? 1 : 0;
    if (sel_lq) {
      const int64_t s = valid ? out[j] : 0;
      sel_lq[b * n + j] = lq[b * m + s] * static_cast<T>(valid ? 1 : 0);
    }
  }
}

}  // namespace tg

using namespace tg;

extern "C" int tg_sample_wor(const void* q, const void* log_q, int32_t dtype, int64_t B, int32_t m, int32_t n,
                             const tg_pcg64* rng, tg_rowmap rows, int64_t* selected, uint8_t* sel_mask, void* sel_log_q,
                             void* stream) {
  if (m < 1 || n < 1) return fail(TG_ECONFIG, "need 1 <= n and m >= 1");
  if (m > 248) return fail(TG_EVALUE, "m=%d exceeds the device limit 248", m);
  if (B <= 0) return TG_OK;
  if (sel_log_q != nullptr && log_q == nullptr) return fail(TG_EVALUE, "sel_log_q needs log_q");
  const int threads = m <= 96 ? 64 : 32;
  const size_t smem = (size_t)threads * m * sizeof(double);
  const int grid = ceil_div(B, threads);
  const cudaStream_t st = as_stream(stream);
  if (dtype == 1) {
    if (smem > 48 * 1024)
      TG_CUDA(cudaFuncSetAttribute(wor_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    wor_kernel<double><<<grid, threads, smem, st>>>(static_cast<const double*>(q), static_cast<const double*>(log_q), B,
                                                    m, n, *rng, rows, selected, sel_mask,
                                                    static_cast<double*>(sel_log_q));
  } else if (dtype == 0) {
    if (smem > 48 * 1024)
      TG_CUDA(cudaFuncSetAttribute(wor_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    wor_kernel<float><<<grid, threads, smem, st>>>(static_cast<const float*>(q), static_cast<const float*>(log_q), B, m,
                                                   n, *rng, rows, selected, sel_mask, static_cast<float*>(sel_log_q));
  } else {
    return fail(TG_EVALUE, "dtype must be 0 (f32) or 1 (f64)");
  }
  TG_LAUNCHED();
  return TG_OK;
}
