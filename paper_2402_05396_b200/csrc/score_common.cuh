// Device helpers shared by K7's forward (score.cu) and the sampler backward
// (score_bwd.cu): f32/f64 math overloads, the exact GeLU and leaky ReLU of
// autodiff.py:313-340, LayerNorm row statistics (autodiff.py:397-404) and the
// parameter-free encoder blocks (TE / FE / identity, encoders.py:171-200).
#pragma once

#include "common.cuh"

namespace tg {

enum Dec : int { DEC_LINEAR = 0, DEC_GAT = 1, DEC_GATV2 = 2, DEC_TRANS = 3 };

__device__ __forceinline__ float erf_t(float x) { return erff(x); }
__device__ __forceinline__ double erf_t(double x) { return erf(x); }
__device__ __forceinline__ float exp_t(float x) { return expf(x); }
__device__ __forceinline__ double exp_t(double x) { return exp(x); }
__device__ __forceinline__ float log_t(float x) { return logf(x); }
__device__ __forceinline__ double log_t(double x) { return log(x); }
__device__ __forceinline__ float sqrt_t(float x) { return sqrtf(x); }
__device__ __forceinline__ double sqrt_t(double x) { return sqrt(x); }

// exact (erf) GeLU, autodiff.py:313-319: x * (0.5 * (1 + erf(x / sqrt 2)))
template <typename T>
__device__ __forceinline__ T gelu(T x) {
  const T c = T(0.70710678118654752440);
  return x * (T(0.5) * (T(1) + erf_t(x * c)));
}
template <typename T>
__device__ __forceinline__ T leaky(T x, T s) {
  return x > T(0) ? x : s * x;
}

// ---- per-row LayerNorm statistics (autodiff.py:397-404): two-pass mean/var.
template <typename T>
__global__ void rowstats_kernel(const T* __restrict__ x, int64_t M, int d, int64_t ld, T eps, T* __restrict__ out) {
  // the row is read once: lane l keeps elements l, l + 32, ... (up to 16 of
  // them) in registers for the second pass; same per-lane order as the loop
  constexpr int PER = 16;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= M) return;
  const T* r = x + row * ld;
  T s = T(0);
  if constexpr (sizeof(T) == 4) {
    // f32 rows of a 16-B-pitched buffer: lane l keeps float4 units l, l+32,
    // ... (up to 512 columns), 4x fewer load instructions than one float per
    // lane per pass; columns past d are masked (the pad may hold anything)
    if (d <= 512 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      float4 e[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int c = 4 * (lane + 32 * t);
        e[t] = c < d ? *reinterpret_cast<const float4*>(r + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      auto val = [&](int t, int k) {
        const int c = 4 * (lane + 32 * t) + k;
        const float* f = reinterpret_cast<const float*>(&e[t]);
        return c < d ? f[k] : 0.f;
      };
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int k = 0; k < 4; ++k) s += val(t, k);
      s = warp_sum(s);
      const T mu = s / T(d);
      T v = T(0);
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * (lane + 32 * t) + k < d) {
            const T u = val(t, k) - mu;
            v = fma(u, u, v);
          }
      v = warp_sum(v);
      if (lane == 0) {
        out[2 * row] = mu;
        out[2 * row + 1] = T(1) / sqrt_t(v / T(d) + eps);
      }
      return;
    }
  }
  if (d <= 32 * PER) {
    T e[PER];
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int c = lane + 32 * t;
      e[t] = c < d ? r[c] : T(0);
    }
#pragma unroll
    for (int t = 0; t < PER; ++t)
      if (lane + 32 * t < d) s += e[t];
    s = warp_sum(s);
    const T mu = s / T(d);
    T v = T(0);
#pragma unroll
    for (int t = 0; t < PER; ++t)
      if (lane + 32 * t < d) {
        const T u = e[t] - mu;
        v = fma(u, u, v);
      }
    v = warp_sum(v);
    if (lane == 0) {
      out[2 * row] = mu;
      out[2 * row + 1] = T(1) / sqrt_t(v / T(d) + eps);
    }
    return;
  }
  for (int c = lane; c < d; c += 32) s += r[c];
  s = warp_sum(s);
  const T mu = s / T(d);
  T v = T(0);
  for (int c = lane; c < d; c += 32) {
    const T t = r[c] - mu;
    v = fma(t, t, v);
  }
  v = warp_sum(v);
  if (lane == 0) {
    out[2 * row] = mu;
    out[2 * row + 1] = T(1) / sqrt_t(v / T(d) + eps);
  }
}

// cos(x) of the time encoding (encoders.py:67), x = dt * omega formed in f64
// like the reference.  f64 mode: libdevice cos.  f32 mode (the reference's
// float32 precision casts the f64 cosine): Cody-Waite reduction by 2*pi in
// f64, then cosf of the reduced argument -- within 1 f32 ulp of the cast,
// at a fraction of the f64 cost (x reaches 1e6 rad).
template <typename T>
__device__ __forceinline__ T time_cos(double x);
template <>
__device__ __forceinline__ double time_cos<double>(double x) {
  return cos(x);
}
template <>
__device__ __forceinline__ float time_cos<float>(double x) {
  const double k = rint(x * 0.15915494309189535);  // 1 / (2 pi)
  double r = fma(-k, 6.283185307179586, x);         // 2 pi, high part
  r = fma(-k, 2.4492935982947064e-16, r);           // 2 pi, low part
  return cosf(static_cast<float>(r));
}

// ---- TE / FE / identity blocks of z_raw, masked (encoders.py:171-183).
template <typename T>
__global__ void encode_misc_kernel(const int64_t* __restrict__ ids, const double* __restrict__ dts,
                                   const uint8_t* __restrict__ mask, int64_t B, int m, int F, int te_off,
                                   const double* __restrict__ omega, const double* __restrict__ fe_table, T* z,
                                   int64_t ld) {
  extern __shared__ int64_t sh[];
  int64_t* sid = sh;                                  // [m]
  double* sdt = reinterpret_cast<double*>(sid + m);   // [m]
  int* sfreq = reinterpret_cast<int*>(sdt + m);       // [m]
  uint8_t* smask = reinterpret_cast<uint8_t*>(sfreq + m);
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      sid[j] = ids[b * m + j];
      sdt[j] = dts[b * m + j];
      smask[j] = mask[b * m + j];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      int f = 0;
      if (smask[j])
        for (int q = 0; q < m; ++q) f += (smask[q] && sid[q] == sid[j]);
      sfreq[j] = f;
    }
    __syncthreads();
    // thread = output column, one loop per column kind (no per-element
    // branching on the kind), rows in turn; masked slots are 0
    const int W = 2 * F + m;
    T* zb = z + (b * m) * ld + te_off;
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
      T* zc = zb + c;
      if (c < F) {  // TE: cos(dt * omega_c)
        const double om = omega[c];
        for (int j = 0; j < m; ++j) zc[j * ld] = smask[j] ? time_cos<T>(sdt[j] * om) : T(0);
      } else if (c < 2 * F) {  // FE: the frequency table row of the slot's count
        const double* fe = fe_table + (c - F);
        for (int j = 0; j < m; ++j) zc[j * ld] = smask[j] ? static_cast<T>(fe[(int64_t)sfreq[j] * F]) : T(0);
      } else {  // identity: slot q holds the same node as slot j
        const int q = c - 2 * F;
        const bool mq = smask[q] != 0;
        const int64_t idq = sid[q];
        for (int j = 0; j < m; ++j) zc[j * ld] = (smask[j] && mq && sid[j] == idq) ? T(1) : T(0);
      }
    }
  }
}

// ---- target rows: [proj_v | 0_e | TE(0) | FE(1) | 0_m] (padded, sampler.py:75-88)
// or [proj_v | TE(0) | FE(1)] (trans, encoders.py:186-200).  proj_v is written
// by a GEMM into columns [0, F) beforehand.
template <typename T>
__global__ void target_misc_kernel(int64_t B, int F, int m, int has_v, int has_e, int padded,
                                   const double* __restrict__ fe_table, T* zt, int64_t ld) {
  const int off = (has_v ? F : 0);
  const int W = padded ? (has_e ? F : 0) + 2 * F + m : 2 * F;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < B * W; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / W;
    const int c = (int)(e - b * W);
    T v = T(0);
    int cc = c;
    if (padded && has_e) {
      if (cc < F) {
        zt[b * ld + off + c] = T(0);
        continue;
      }
      cc -= F;
    }
    if (cc < F)
      v = T(1);  // cos(0 * omega) (encoders.py:196)
    else if (cc < 2 * F)
      v = static_cast<T>(fe_table[F + (cc - F)]);  // FE(1) (encoders.py:198)
    zt[b * ld + off + c] = v;
  }
}

// ---- masked softmax + log-softmax per root (autodiff.py:421-464).
// logit[r] = sum_p partial[r, p] (+ rowterm[b]); gat: leaky; trans: *1/sqrt(count).
template <typename T>
__global__ void softmax_kernel(const T* __restrict__ partial, int P, const T* __restrict__ rowterm,
                               const uint8_t* __restrict__ mask, int64_t B, int m, int dec, T slope,
                               T* __restrict__ q, T* __restrict__ lq) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); b < B;
       b += (int64_t)gridDim.x * (blockDim.x / 32)) {
    int cnt = 0;
    for (int j = lane; j < m; j += 32) cnt += mask[b * m + j] != 0;
    cnt = warp_sum(cnt);
    const T scale = T(1) / sqrt_t(static_cast<T>(cnt > 1 ? cnt : 1));
    T mx = -INFINITY;
    for (int j = lane; j < m; j += 32) {
      const int64_t r = b * m + j;
      if (mask[r]) {
        T l = T(0);
        for (int pp = 0; pp < P; ++pp) l += partial[r * P + pp];
        if (dec == DEC_GAT) l = leaky(l + rowterm[b], slope);
        if (dec == DEC_TRANS) l = l * scale;
        mx = l > mx ? l : mx;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T other = __shfl_xor_sync(FULL, mx, o);
      mx = other > mx ? other : mx;
    }
    if (cnt == 0) mx = T(0);
    T z = T(0);
    for (int j = lane; j < m; j += 32) {
      const int64_t r = b * m + j;
      if (mask[r]) {
        T l = T(0);
        for (int pp = 0; pp < P; ++pp) l += partial[r * P + pp];
        if (dec == DEC_GAT) l = leaky(l + rowterm[b], slope);
        if (dec == DEC_TRANS) l = l * scale;
        z += exp_t(l - mx);
      }
    }
    z = warp_sum(z);
    const T lse = z > T(0) ? log_t(z) + mx : T(0);
    for (int j = lane; j < m; j += 32) {
      const int64_t r = b * m + j;
      T qq = T(0), ll = T(-1e30);
      if (mask[r]) {
        T l = T(0);
        for (int pp = 0; pp < P; ++pp) l += partial[r * P + pp];
        if (dec == DEC_GAT) l = leaky(l + rowterm[b], slope);
        if (dec == DEC_TRANS) l = l * scale;
        qq = exp_t(l - mx) / z;
        ll = l - lse;
      }
      q[r] = qq;
      lq[r] = ll;
    }
  }
}

}  // namespace tg
