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
#include "pcg.cuh"

namespace tg {

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
