// K10: the surrogate-loss head of the sampler update.
//
// The sampler is trained through a log-derivative surrogate whose per-pick
// coefficients are frozen functions of the aggregator's forward and of
// dL/dh (sampler.py:183-250, composed in training.py:409-436):
//
//   TGAT        c_j = (<dL/dh, V_j> tau_j / lam^3 - <dL/dh, mu> tau_j / lam^4) / n
//               lam = sum_j tau_j, mu = sum_j tau_j V_j over the picks
//                                                  (tgat_sample_coefficients :191-213)
//   GraphMixer  c_j = (1/n) sum_k dL/dh_k w'_jk mu_jk  (graphmixer_sample_coefficients :230-239)
//               with training.py's mu = msgs @ Wc1, w'_j = 1 + rowsum(Wt1 @ Wt2)_j
//
// and loss = sum c * selected_log_q.  Its gradient with respect to the
// scoring logits closes the head of the backward pass: index (:257-271 of
// autodiff.py) scatters c into the picked slots, log_softmax_masked's vjp
// (autodiff.py:447-464) gives  dlogits = g_m - q * sum(g_m).
//
// Layout: one block (or warp) per root row; reductions over the feature
// axis in f64 whatever the dtype (the reference's f32 mode promotes these
// to f64 through n_eff as well).  Reassociations, each exact up to
// rounding: <dL/dh, mu> = sum_j tau_j <dL/dh, V_j> (no [B, d] mu), and for
// the mixer sum_k dL_k mu_jk = msgs_j . (Wc1 dL) (no [B, n, d] mu).
#include <cuda_runtime.h>

#include "common.cuh"

namespace tg {

template <typename T>
__device__ __forceinline__ double ld64(const T* p, int64_t i) {
  return (double)p[i];
}

// TGAT coefficients: block per row, warps over picks j (lanes over d)
template <typename T>
__global__ void tgat_coeff_kernel(int64_t B, int n, int d, const T* __restrict__ dh, int64_t dh_ld,
                                  const T* __restrict__ tau, const T* __restrict__ V, const uint8_t* __restrict__ sel,
                                  const uint8_t* __restrict__ contrib, T* __restrict__ c, int* __restrict__ bad) {
  extern __shared__ double sm[];
  double* dot_v = sm;  // [n]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const T* g = dh + b * dh_ld;
    for (int j = warp; j < n; j += nw) {
      const T* v = V + (b * n + j) * (int64_t)d;
      double s = 0.0;
      for (int k = lane; k < d; k += 32) s = fma((double)g[k], (double)v[k], s);
      s = warp_sum(s);
      if (lane == 0) dot_v[j] = s;
    }
    __syncthreads();
    if (warp == 0) {
      double lam = 0.0, dmu = 0.0;
      int cnt = 0;
      for (int j = lane; j < n; j += 32) {
        const bool sj = sel[b * n + j] != 0;
        const double t = sj ? ld64(tau, b * n + j) : 0.0;
        lam += t;
        dmu = fma(t, dot_v[j], dmu);
        cnt += sj;
      }
      lam = warp_sum(lam);
      dmu = warp_sum(dmu);
      cnt = warp_sum(cnt);
      const bool active = contrib[b] != 0 && cnt > 0;
      if (active && lam <= 0.0 && lane == 0) atomicExch(bad, 1);
      const double ls = lam > 0.0 ? lam : 1.0;
      const double l3 = ls * ls * ls, l4 = l3 * ls;
      const double ne = (double)(cnt > 1 ? cnt : 1);
      for (int j = lane; j < n; j += 32) {
        const bool sj = sel[b * n + j] != 0;
        const double t = sj ? ld64(tau, b * n + j) : 0.0;
        const double cj = (dot_v[j] * t / l3 - dmu * t / l4) / ne;
        c[b * n + j] = (T)((sj && active) ? cj : 0.0);
      }
    }
    __syncthreads();
  }
}

// GraphMixer coefficients from the messages (training.py:423-431): block
// per row; v = Wc1 dL/dh (warps over the d_msg outputs), then warps over j
template <typename T>
__global__ void gmixer_coeff_kernel(int64_t B, int n, int dm, int d, int ht, const T* __restrict__ dh, int64_t dh_ld,
                                    const T* __restrict__ msgs, int64_t msg_ld, const T* __restrict__ Wc1,
                                    const T* __restrict__ Wt1, const T* __restrict__ Wt2,
                                    const uint8_t* __restrict__ sel, const uint8_t* __restrict__ contrib,
                                    T* __restrict__ c) {
  extern __shared__ double sm[];
  double* v = sm;           // [dm]
  double* wrow = v + dm;    // [n]
  double* rs = wrow + n;    // [ht]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // w'_j = 1 + sum_k (Wt1 Wt2)_jk = 1 + Wt1_j . rowsum(Wt2)   (row-independent)
  for (int l = warp; l < ht; l += nw) {
    double s = 0.0;
    for (int k = lane; k < n; k += 32) s += (double)Wt2[(int64_t)l * n + k];
    s = warp_sum(s);
    if (lane == 0) rs[l] = s;
  }
  __syncthreads();
  for (int j = warp; j < n; j += nw) {
    double s = 0.0;
    for (int l = lane; l < ht; l += 32) s = fma((double)Wt1[(int64_t)j * ht + l], rs[l], s);
    s = warp_sum(s);
    if (lane == 0) wrow[j] = 1.0 + s;
  }
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const T* g = dh + b * dh_ld;
    for (int i = warp; i < dm; i += nw) {
      const T* w = Wc1 + (int64_t)i * d;
      double s = 0.0;
      for (int k = lane; k < d; k += 32) s = fma((double)w[k], (double)g[k], s);
      s = warp_sum(s);
      if (lane == 0) v[i] = s;
    }
    __syncthreads();
    int cnt = 0;
    for (int j = 0; j < n; ++j) cnt += sel[b * n + j] != 0;
    const double ne = (double)(cnt > 1 ? cnt : 1);
    const bool cb = contrib[b] != 0;
    for (int j = warp; j < n; j += nw) {
      const T* mr = msgs + (b * n + j) * msg_ld;
      double s = 0.0;
      for (int i = lane; i < dm; i += 32) s = fma((double)mr[i], v[i], s);
      s = warp_sum(s);
      if (lane == 0) c[b * n + j] = (T)((cb && sel[b * n + j]) ? wrow[j] * s / ne : 0.0);
    }
    __syncthreads();
  }
}

// general mixer form (graphmixer_sample_coefficients): warp per (b, j);
// w' is [n, d] (wp_bstride 0) or [B, n, d]
template <typename T>
__global__ void mixer_coeff_general_kernel(int64_t B, int n, int d, const T* __restrict__ dh, int64_t dh_ld,
                                           const T* __restrict__ wp, int64_t wp_bstride, const T* __restrict__ mu,
                                           const uint8_t* __restrict__ sel, const uint8_t* __restrict__ contrib,
                                           T* __restrict__ c) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < B * n; w += nwarps) {
    const int64_t b = w / n;
    const int j = (int)(w - b * n);
    int cnt = 0;
    for (int jj = lane; jj < n; jj += 32) cnt += sel[b * n + jj] != 0;
    cnt = warp_sum(cnt);
    const T* g = dh + b * dh_ld;
    const T* wr = wp + b * wp_bstride + (int64_t)j * d;
    const T* mr = mu + (b * n + j) * (int64_t)d;
    double s = 0.0;
    for (int k = lane; k < d; k += 32) s = fma((double)g[k] * (double)wr[k], (double)mr[k], s);
    s = warp_sum(s);
    if (lane == 0) {
      const double ne = (double)(cnt > 1 ? cnt : 1);
      c[w] = (T)((contrib[b] && sel[w]) ? s / ne : 0.0);
    }
  }
}

// dlogits and the per-row loss: warp per row; lane owns slots lane + 32 t
constexpr int LQ_MAXM = 256;
template <typename T>
__global__ void logq_grad_kernel(int64_t B, int m, int n, const T* __restrict__ q, const T* __restrict__ log_q,
                                 const uint8_t* __restrict__ mask, const int64_t* __restrict__ selected,
                                 const uint8_t* __restrict__ sel, const T* __restrict__ c, T* __restrict__ dlogits,
                                 double* __restrict__ row_loss) {
  constexpr int PER = LQ_MAXM / 32;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < B; b += nwarps) {
    double g[PER];
#pragma unroll
    for (int t = 0; t < PER; ++t) g[t] = 0.0;
    double loss = 0.0;
    for (int j = 0; j < n; ++j) {
      if (!sel[b * n + j]) continue;
      const int64_t s = selected[b * n + j];
      const double cj = (double)c[b * n + j];
      const int si = (int)(s > 0 ? s : 0);
      if (lane == 0) loss = fma(cj, (double)log_q[b * m + si], loss);
#pragma unroll
      for (int t = 0; t < PER; ++t)
        if (lane + 32 * t == si) g[t] += cj;  // index vjp: scatter into the picked slot
    }
    double S = 0.0;
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int i = lane + 32 * t;
      if (i < m && mask[b * m + i]) S += g[t];
    }
    S = warp_sum(S);
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int i = lane + 32 * t;
      if (i < m) {
        const double gm = mask[b * m + i] ? g[t] : 0.0;
        dlogits[b * m + i] = (T)(gm - (double)q[b * m + i] * S);
      }
    }
    if (lane == 0 && row_loss != nullptr) row_loss[b] = loss;
  }
}

// deterministic total of the per-row losses: one block, fixed order
__global__ void sum_rows_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  __shared__ double part[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) part[threadIdx.x] += part[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

static int grid_rows(int64_t rows) {
  const int64_t cap = (int64_t)device_sms() * 8;
  return (int)(rows < cap ? (rows > 0 ? rows : 1) : cap);
}

}  // namespace tg

using namespace tg;

extern "C" int tg_tgat_sample_coeffs(int32_t dtype, int64_t B, int32_t n, int32_t d, const void* dL_dh, int64_t dh_ld,
                                     const void* tau, const void* V, const uint8_t* sel_mask,
                                     const uint8_t* contrib, void* c, void* stream) {
  if (dtype != 0 && dtype != 1) return fail(TG_EVALUE, "dtype must be 0 (f32) or 1 (f64)");
  if (n < 1 || d < 1 || dh_ld < d) return fail(TG_EVALUE, "bad shape n=%d d=%d ld=%lld", n, d, (long long)dh_ld);
  if (B <= 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  int* bad = nullptr;
  TG_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  TG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const size_t smem = (size_t)n * sizeof(double);
  if (smem > 48 * 1024) return fail(TG_EVALUE, "n=%d picks exceed the device limit", n);
  if (dtype == 1)
    tgat_coeff_kernel<double><<<grid_rows(B), 256, smem, st>>>(B, n, d, static_cast<const double*>(dL_dh), dh_ld,
                                                               static_cast<const double*>(tau),
                                                               static_cast<const double*>(V), sel_mask, contrib,
                                                               static_cast<double*>(c), bad);
  else
    tgat_coeff_kernel<float><<<grid_rows(B), 256, smem, st>>>(B, n, d, static_cast<const float*>(dL_dh), dh_ld,
                                                              static_cast<const float*>(tau),
                                                              static_cast<const float*>(V), sel_mask, contrib,
                                                              static_cast<float*>(c), bad);
  TG_LAUNCHED();
  int h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaFreeAsync(bad, st));
  TG_CUDA(cudaStreamSynchronize(st));
  if (h) return fail(TG_EFLOAT, "attention normalizer must be positive");
  return TG_OK;
}

extern "C" int tg_graphmixer_sample_coeffs(int32_t dtype, int64_t B, int32_t n, int32_t d_msg, int32_t d, int32_t ht,
                                           const void* dL_dh, int64_t dh_ld, const void* msgs, int64_t msg_ld,
                                           const void* Wc1, const void* Wt1, const void* Wt2,
                                           const uint8_t* sel_mask, const uint8_t* contrib, void* c, void* stream) {
  if (dtype != 0 && dtype != 1) return fail(TG_EVALUE, "dtype must be 0 (f32) or 1 (f64)");
  if (n < 1 || d_msg < 1 || d < 1 || ht < 1 || dh_ld < d || msg_ld < d_msg)
    return fail(TG_EVALUE, "bad shape n=%d d_msg=%d d=%d ht=%d", n, d_msg, d, ht);
  if (B <= 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  const size_t smem = (size_t)(d_msg + n + ht) * sizeof(double);
  if (smem > 227 * 1024) return fail(TG_EVALUE, "d_msg=%d exceeds the device limit", d_msg);
  if (dtype == 1) {
    auto k = gmixer_coeff_kernel<double>;
    if (smem > 48 * 1024) TG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid_rows(B), 256, smem, st>>>(B, n, d_msg, d, ht, static_cast<const double*>(dL_dh), dh_ld,
                                       static_cast<const double*>(msgs), msg_ld, static_cast<const double*>(Wc1),
                                       static_cast<const double*>(Wt1), static_cast<const double*>(Wt2), sel_mask,
                                       contrib, static_cast<double*>(c));
  } else {
    auto k = gmixer_coeff_kernel<float>;
    if (smem > 48 * 1024) TG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid_rows(B), 256, smem, st>>>(B, n, d_msg, d, ht, static_cast<const float*>(dL_dh), dh_ld,
                                       static_cast<const float*>(msgs), msg_ld, static_cast<const float*>(Wc1),
                                       static_cast<const float*>(Wt1), static_cast<const float*>(Wt2), sel_mask,
                                       contrib, static_cast<float*>(c));
  }
  TG_LAUNCHED();
  return TG_OK;
}

extern "C" int tg_mixer_sample_coeffs(int32_t dtype, int64_t B, int32_t n, int32_t d, const void* dL_dh, int64_t dh_ld,
                                      const void* w_prime, int64_t wp_bstride, const void* mu,
                                      const uint8_t* sel_mask, const uint8_t* contrib, void* c, void* stream) {
  if (dtype != 0 && dtype != 1) return fail(TG_EVALUE, "dtype must be 0 (f32) or 1 (f64)");
  if (n < 1 || d < 1 || dh_ld < d) return fail(TG_EVALUE, "bad shape n=%d d=%d", n, d);
  if (B <= 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  const int grid = grid_rows((B * n + 7) / 8);
  if (dtype == 1)
    mixer_coeff_general_kernel<double><<<grid, 256, 0, st>>>(B, n, d, static_cast<const double*>(dL_dh), dh_ld,
                                                             static_cast<const double*>(w_prime), wp_bstride,
                                                             static_cast<const double*>(mu), sel_mask, contrib,
                                                             static_cast<double*>(c));
  else
    mixer_coeff_general_kernel<float><<<grid, 256, 0, st>>>(B, n, d, static_cast<const float*>(dL_dh), dh_ld,
                                                            static_cast<const float*>(w_prime), wp_bstride,
                                                            static_cast<const float*>(mu), sel_mask, contrib,
                                                            static_cast<float*>(c));
  TG_LAUNCHED();
  return TG_OK;
}

extern "C" int tg_logq_surrogate_grad(int32_t dtype, int64_t B, int32_t m, int32_t n, const void* q,
                                      const void* log_q, const uint8_t* mask, const int64_t* selected,
                                      const uint8_t* sel_mask, const void* c, void* dlogits, double* row_loss,
                                      double* loss, void* stream) {
  if (dtype != 0 && dtype != 1) return fail(TG_EVALUE, "dtype must be 0 (f32) or 1 (f64)");
  if (m < 1 || n < 1) return fail(TG_EVALUE, "bad shape m=%d n=%d", m, n);
  if (m > LQ_MAXM) return fail(TG_EVALUE, "m=%d exceeds the device limit %d", m, LQ_MAXM);
  if (loss != nullptr && row_loss == nullptr) return fail(TG_EVALUE, "loss needs row_loss scratch");
  const cudaStream_t st = as_stream(stream);
  if (B > 0) {
    const int grid = grid_rows((B + 7) / 8);
    if (dtype == 1)
      logq_grad_kernel<double><<<grid, 256, 0, st>>>(B, m, n, static_cast<const double*>(q),
                                                     static_cast<const double*>(log_q), mask, selected, sel_mask,
                                                     static_cast<const double*>(c), static_cast<double*>(dlogits),
                                                     row_loss);
    else
      logq_grad_kernel<float><<<grid, 256, 0, st>>>(B, m, n, static_cast<const float*>(q),
                                                    static_cast<const float*>(log_q), mask, selected, sel_mask,
                                                    static_cast<const float*>(c), static_cast<float*>(dlogits),
                                                    row_loss);
    TG_LAUNCHED();
  }
  if (loss != nullptr) {
    sum_rows_kernel<<<1, 256, 0, st>>>(row_loss, B > 0 ? B : 0, loss);
    TG_LAUNCHED();
  }
  return TG_OK;
}

// ---- Adam step on the sampler's parameters (params.py:80-99, called by
// update_sampler, sampler.py:253-256).  One launch for every tensor of the
// store: grid.y = tensor.  Each operation is the reference's numpy
// operation in the same order and precision (explicit _rn intrinsics, no
// FMA contraction), so the update is bit-identical: python-float
// coefficients act in the parameter dtype (NumPy 2 weak scalars); a float64
// gradient for a float32 parameter makes the moment additions float64 and
// rounds the result to float32, as numpy's in-place `+=` does.
namespace tg {

struct AdamDev {
  void* p;
  const void* g;
  void* m;
  void* v;
  int64_t n;
  int32_t g_dtype;  // -1 none (zeros), 0 f32, 1 f64
};

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

template <typename T>
__global__ void adam_kernel(const AdamDev* __restrict__ ts, double lr, double beta1, double beta2, double eps,
                            double bc1, double bc2) {
  const AdamDev a = ts[blockIdx.y];
  T* p = static_cast<T*>(a.p);
  T* m = static_cast<T*>(a.m);
  T* v = static_cast<T*>(a.v);
  const T b1 = (T)beta1, b2 = (T)beta2, omb1 = (T)(1.0 - beta1), omb2 = (T)(1.0 - beta2);
  const T c1 = (T)bc1, c2 = (T)bc2, lr_t = (T)lr, eps_t = (T)eps;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    T mi = mul_rn(m[i], b1);  // m *= beta1
    T vi = mul_rn(v[i], b2);  // v *= beta2
    if (a.g_dtype == 1 && sizeof(T) == 4) {
      // float64 gradient into float32 moments: the += runs in float64
      const double g = static_cast<const double*>(a.g)[i];
      mi = (T)__dadd_rn((double)mi, __dmul_rn(1.0 - beta1, g));
      vi = (T)__dadd_rn((double)vi, __dmul_rn(__dmul_rn(1.0 - beta2, g), g));
    } else {
      T g = T(0);
      if (a.g_dtype == 0) g = (T) static_cast<const float*>(a.g)[i];
      else if (a.g_dtype == 1) g = (T) static_cast<const double*>(a.g)[i];
      mi = add_rn(mi, mul_rn(omb1, g));                // m += (1 - beta1) * g
      vi = add_rn(vi, mul_rn(mul_rn(omb2, g), g));     // v += (1 - beta2) * g * g
    }
    m[i] = mi;
    v[i] = vi;
    // p -= lr * (m / bc1) / (sqrt(v / bc2) + eps)
    p[i] = sub_rn(p[i], div_rn(mul_rn(lr_t, div_rn(mi, c1)), add_rn(sqrt_rn(div_rn(vi, c2)), eps_t)));
  }
}

}  // namespace tg

extern "C" int tg_adam_step(int32_t dtype, const tg_adam_tensor* tensors, int32_t count, double lr, double beta1,
                            double beta2, double eps, double bc1, double bc2, void* stream) {
  if (dtype != 0 && dtype != 1) return fail(TG_EVALUE, "dtype must be 0 (f32) or 1 (f64)");
  if (count < 0 || count > 65535) return fail(TG_EVALUE, "count=%d out of range", count);
  if (count == 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  int64_t nmax = 0;
  for (int i = 0; i < count; ++i) {
    if (tensors[i].n < 0) return fail(TG_EVALUE, "tensor %d has negative size", i);
    if (tensors[i].g_dtype < -1 || tensors[i].g_dtype > 1) return fail(TG_EVALUE, "tensor %d: bad g_dtype", i);
    if (dtype == 1 && tensors[i].g_dtype == 0) return fail(TG_EVALUE, "tensor %d: f32 gradient for f64 parameter", i);
    if (tensors[i].n > nmax) nmax = tensors[i].n;
  }
  if (nmax == 0) return TG_OK;
  static_assert(sizeof(tg_adam_tensor) == sizeof(AdamDev), "tg_adam_tensor layout");
  AdamDev* dt = nullptr;
  TG_CUDA(cudaMallocAsync(&dt, sizeof(AdamDev) * count, st));
  TG_CUDA(cudaMemcpyAsync(dt, tensors, sizeof(AdamDev) * count, cudaMemcpyHostToDevice, st));
  const int64_t blocks = (nmax + 255) / 256;
  const dim3 grid((unsigned)(blocks < 1024 ? blocks : 1024), (unsigned)count);
  if (dtype == 1)
    adam_kernel<double><<<grid, 256, 0, st>>>(dt, lr, beta1, beta2, eps, bc1, bc2);
  else
    adam_kernel<float><<<grid, 256, 0, st>>>(dt, lr, beta1, beta2, eps, bc1, bc2);
  TG_LAUNCHED();
  TG_CUDA(cudaFreeAsync(dt, st));
  // the host table may be freed when this returns
  TG_CUDA(cudaStreamSynchronize(st));
  return TG_OK;
}
