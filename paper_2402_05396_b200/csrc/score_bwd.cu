// Sampler backward: the scoring network's parameter gradients from
// d loss / d logits (second half).
//
// The reference's update_sampler (sampler.py:253-256) runs ad.backward
// (autodiff.py:495) from the surrogate loss through index + log-softmax
// (K10 gives dlogits) and then through the network K7 evaluates:
// decode_policy (sampler.py:91-135) -> mixer_transform (sampler.py:69-72,
// mixer.py:31-51) -> encode_neighborhood_batch / encode_target_batch
// (encoders.py:152-200), accumulating into every sampler parameter's .grad.
// This file is that chain on the device: the forward intermediates the
// vjps need (pre-activations, LayerNorm statistics, the mixer's hidden
// layers) are recomputed into a workspace, then each reference vjp
// (autodiff.py: affine/matmul, gelu :313-323, leaky_relu :333-341,
// layer_norm :397-418, the mixer's transposes and residuals) runs as a
// hand-written row / tile kernel or, for the plain matrix products, a cuBLAS
// GEMM (dW = X^T dY over up to 300k rows, dX = dY W^T).  Parameter gradients
// ACCUMULATE (+=), as .grad does across a loss with several layers
// (training.py:411-436); the caller zeroes them per update.
//
// Layout: rows r = b*m + j (B roots x m candidate slots), row stride ld =
// round_up(d_enc, 4) in T (f64: the reference's default precision; f32).
// Column sums (bias / LayerNorm-affine gradients) are X^T 1 GEMVs, so every
// reduction is deterministic.
#include <cublas_v2.h>

#include <mutex>

#include "score_common.cuh"

namespace tg {
namespace {

// d/dx [x Phi(x)] = Phi(x) + x phi(x)  (autodiff.py:321-323)
template <typename T>
__device__ __forceinline__ T gelu_grad(T x) {
  const T cdf = T(0.5) * (T(1) + erf_t(x * T(0.70710678118654752440)));
  const T pdf = T(0.39894228040143267794) * exp_t(T(-0.5) * x * x);
  return cdf + x * pdf;
}

// ---------------------------------------------------------------- cuBLAS
struct Blas {
  cublasHandle_t h = nullptr;
  int dev = -1;
};

cublasHandle_t blas(cudaStream_t st) {
  thread_local Blas b;
  int dev = 0;
  cudaGetDevice(&dev);
  if (b.h == nullptr || b.dev != dev) {
    if (b.h) cublasDestroy(b.h);
    b.h = nullptr;
    if (cublasCreate(&b.h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    cublasSetMathMode(b.h, CUBLAS_PEDANTIC_MATH);  // plain FP32 / FP64, no TF32
    b.dev = dev;
  }
  cublasSetStream(b.h, st);
  return b.h;
}

// Row-major C[M,N] = alpha op(A) op(B) + beta C, op(A) [M,K], op(B) [K,N].
// A is stored [M,K] (ta false) or [K,M] (ta true), row stride lda; B alike.
// (col-major view: C^T = op(B)^T op(A)^T.)
template <typename T>
int gemm_rm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, T alpha, const T* A, int64_t lda,
            const T* B, int64_t ldb, T beta, T* C, int64_t ldc) {
  if (M == 0 || N == 0) return TG_OK;
  cublasHandle_t h = blas(st);
  if (!h) return fail(TG_ECUDA, "cublasCreate failed");
  const cublasOperation_t oa = ta ? CUBLAS_OP_T : CUBLAS_OP_N, ob = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasStatus_t s;
  if constexpr (sizeof(T) == 8)
    s = cublasDgemm(h, ob, oa, (int)N, (int)M, (int)K, reinterpret_cast<const double*>(&alpha),
                    reinterpret_cast<const double*>(B), (int)ldb, reinterpret_cast<const double*>(A), (int)lda,
                    reinterpret_cast<const double*>(&beta), reinterpret_cast<double*>(C), (int)ldc);
  else
    s = cublasSgemm(h, ob, oa, (int)N, (int)M, (int)K, reinterpret_cast<const float*>(&alpha),
                    reinterpret_cast<const float*>(B), (int)ldb, reinterpret_cast<const float*>(A), (int)lda,
                    reinterpret_cast<const float*>(&beta), reinterpret_cast<float*>(C), (int)ldc);
  if (s != CUBLAS_STATUS_SUCCESS) return fail(TG_ECUDA, "cublas gemm failed (%d)", (int)s);
  return TG_OK;
}

// out[N] += sum over the M rows of X [M,N] (row stride ld)   (bias grads)
template <typename T>
int colsum_acc(cudaStream_t st, const T* X, int64_t M, int64_t N, int64_t ld, const T* ones, T* out) {
  if (!out) return TG_OK;
  return gemm_rm<T>(st, true, false, N, 1, M, T(1), X, ld, ones, 1, T(1), out, 1);
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 1 << 16) {
  const int64_t g = (n + threads - 1) / threads;
  return (unsigned)(g < 1 ? 1 : (g < cap ? g : cap));
}

// ---------------------------------------------------------------- elementwise kernels
template <typename T>
__global__ void fill_kernel(T* x, int64_t n, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

// f32 feature rows -> T, dense [M, d]
template <typename T>
__global__ void rows_to_t_kernel(const float* __restrict__ x, int64_t ldx, int64_t M, int d, T* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * d; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d;
    y[i] = static_cast<T>(x[r * ldx + (i - r * d)]);
  }
}

// z[r, col + c] = mask ? gelu(P[r, c]) : 0   (encoders.py:162-169, 183)
template <typename T>
__global__ void gelu_cols_kernel(const T* __restrict__ P, int64_t M, int F, const uint8_t* __restrict__ mask, T* z,
                                 int64_t ld, int col) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * F; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int c = (int)(i - r * F);
    const T v = gelu(P[i]);
    z[r * ld + col + c] = (mask == nullptr || mask[r]) ? v : T(0);
  }
}

// dP[r, c] = (mask ? dz[r, col + c] : 0) * gelu'(P[r, c])
template <typename T>
__global__ void gelu_cols_grad_kernel(const T* __restrict__ dz, int64_t ld, int col, const T* __restrict__ P,
                                      int64_t M, int F, const uint8_t* __restrict__ mask, T* __restrict__ dP) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * F; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int c = (int)(i - r * F);
    const T g = (mask == nullptr || mask[r]) ? dz[r * ld + col + c] : T(0);
    dP[i] = g * gelu_grad(P[i]);
  }
}

// out = gamma * ((x - mu) * inv) + beta   (autodiff.py:397-405)
template <typename T>
__global__ void ln_apply_kernel(const T* __restrict__ x, int64_t M, int d, int64_t ld, const T* __restrict__ stats,
                                const T* __restrict__ g, const T* __restrict__ b, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * d; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d;
    const int c = (int)(i - r * d);
    const T xhat = (x[r * ld + c] - stats[2 * r]) * stats[2 * r + 1];
    out[r * ld + c] = g[c] * xhat + b[c];
  }
}

// U += bias (kept: the pre-activation), H = gelu(U)
template <typename T>
__global__ void bias_gelu_kernel(T* U, int64_t M, int N, int64_t ld, const T* __restrict__ bias, T* __restrict__ H) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N;
    const int c = (int)(i - r * N);
    const T u = U[r * ld + c] + bias[c];
    U[r * ld + c] = u;
    H[r * ld + c] = gelu(u);
  }
}

// y = R + (y + bias)   (the residual of mixer.py:46-47)
template <typename T>
__global__ void bias_resid_kernel(T* y, int64_t M, int N, int64_t ld, const T* __restrict__ bias,
                                  const T* __restrict__ R) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N;
    const int c = (int)(i - r * N);
    y[r * ld + c] = R[r * ld + c] + (y[r * ld + c] + bias[c]);
  }
}

// dU = dH * gelu'(U), in place on dH
template <typename T>
__global__ void gelu_grad_kernel(T* dH, const T* __restrict__ U, int64_t M, int N, int64_t ld) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N;
    const int c = (int)(i - r * N);
    dH[r * ld + c] *= gelu_grad(U[r * ld + c]);
  }
}

// out[r, k] = s[r] * v[k] (+ out when acc)  -- rank-1 vjps of the dot decoders
template <typename T>
__global__ void outer_kernel(const T* __restrict__ s, int64_t M, const T* __restrict__ v, int N, T* out, int64_t ld,
                             int acc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N;
    const int c = (int)(i - r * N);
    const T x = s[r] * v[c];
    out[r * ld + c] = acc ? out[r * ld + c] + x : x;
  }
}

// out[b, k] = sum_s X[b*m + s, k]  (gradient of a per-root row broadcast to m slots)
template <typename T>
__global__ void slot_sum_kernel(const T* __restrict__ X, int64_t ldx, int64_t B, int m, int N, T* __restrict__ out,
                                int64_t ldo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / N;
    const int c = (int)(i - b * N);
    T s = T(0);
    for (int j = 0; j < m; ++j) s += X[(b * m + j) * ldx + c];
    out[b * ldo + c] = s;
  }
}

// gatv2 (sampler.py:116-122): Q[r] = z W_top + R[b] (in place, the
// pre-activation), H[r] = leaky(Q[r])
template <typename T>
__global__ void gatv2_fwd_kernel(T* Q, const T* __restrict__ R, int64_t M, int m, int N, int64_t ld, T slope,
                                 T* __restrict__ H) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N;
    const int c = (int)(i - r * N);
    const T q = Q[r * ld + c] + R[(r / m) * ld + c];
    Q[r * ld + c] = q;
    H[r * ld + c] = leaky(q, slope);
  }
}

// gatv2 vjp: dQ[r, k] = G[r] a[k] leaky'(Q[r, k])   (autodiff.py:333-341)
template <typename T>
__global__ void gatv2_bwd_kernel(const T* __restrict__ G, const T* __restrict__ a, const T* __restrict__ Q, int64_t M,
                                 int N, int64_t ld, T slope, T* __restrict__ dQ) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N;
    const int c = (int)(i - r * N);
    dQ[r * ld + c] = (G[r] * a[c]) * (Q[r * ld + c] > T(0) ? T(1) : slope);
  }
}

// gat (sampler.py:104-115): raw[r] = pu[r].a_u + pv[b].a_v, draw = G leaky'(raw);
// dsum[b] = sum over the root's slots of draw.  One warp per root.
template <typename T>
__global__ void gat_bwd_kernel(const T* __restrict__ pu, const T* __restrict__ pv, int64_t ld, const T* __restrict__ a,
                               const T* __restrict__ G, int64_t B, int m, int d, T slope, T* __restrict__ draw,
                               T* __restrict__ dsum) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); b < B;
       b += (int64_t)gridDim.x * (blockDim.x / 32)) {
    T sv = T(0);
    for (int c = lane; c < d; c += 32) sv += pv[b * ld + c] * a[d + c];
    sv = warp_sum(sv);
    T acc = T(0);
    for (int j = 0; j < m; ++j) {
      const int64_t r = b * m + j;
      T su = T(0);
      for (int c = lane; c < d; c += 32) su += pu[r * ld + c] * a[c];
      su = warp_sum(su);
      const T raw = su + sv;
      const T g = G[r] * (raw > T(0) ? T(1) : slope);
      if (lane == 0) draw[r] = g;
      acc += g;
    }
    if (lane == 0) dsum[b] = acc;
  }
}

// trans (sampler.py:123-129): logits = (qt[b] . kn[r]) / sqrt(max(valid, 1));
// draw = G / sqrt(count); dqt[b] = sum_s draw kn[r]; dkn[r] = draw qt[b].
// One block per root, threads over channels.
template <typename T>
__global__ void trans_bwd_kernel(const T* __restrict__ qt, const T* __restrict__ kn, int64_t ld,
                                 const T* __restrict__ G, const uint8_t* __restrict__ mask, int64_t B, int m, int d,
                                 T* __restrict__ dqt, T* __restrict__ dkn) {
  __shared__ double sdraw[64];
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int cnt = 0;
      for (int j = 0; j < m; ++j) cnt += mask[b * m + j] != 0;
      const double inv = 1.0 / sqrt(static_cast<double>(cnt > 1 ? cnt : 1));
      for (int j = 0; j < m; ++j) sdraw[j] = static_cast<double>(G[b * m + j] * static_cast<T>(inv));
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      T s = T(0);
      const T q = qt[b * ld + c];
      for (int j = 0; j < m; ++j) {
        const T g = static_cast<T>(sdraw[j]);
        s += g * kn[(b * m + j) * ld + c];
        dkn[(b * m + j) * ld + c] = g * q;
      }
      dqt[b * ld + c] = s;
    }
  }
}

// ---- token MLP (mixer.py:40-51) forward / backward, one CTA per root.
// Thread t owns channel c = c0 + t of a chunk of CH channels; per-slot
// vectors of its channel live in shared-memory tiles [m][CH] (column
// access, conflict-free), the m x m token weights are broadcast reads.
//   a2  = LN2(y) column      Ut = a2^T Wt1 + bt1    Ht = gelu(Ut)
//   out = Ht Wt2 + bt2        z_mixed = (y + out) * mask
// backward (dzm = d loss / d z_mixed):
//   dO = dzm * mask   dHt = Wt2 dO   dUt = dHt gelu'(Ut)   da2 = Wt1 dUt
// and the per-(root, channel) rows the weight gradients need are written
// (b*d + c)-major for the GEMMs dWt1 = A2^T dUt, dWt2 = Ht^T dO.
template <typename T, bool BWD>
__global__ void token_kernel(const T* __restrict__ y, int64_t ld, const T* __restrict__ st2, int64_t B, int m, int d,
                             const T* __restrict__ g2, const T* __restrict__ b2, const T* __restrict__ Wt1,
                             const T* __restrict__ bt1, const T* __restrict__ Wt2, const T* __restrict__ bt2,
                             const uint8_t* __restrict__ mask, T* __restrict__ zmix, const T* __restrict__ dzm,
                             T* __restrict__ dy, T* __restrict__ da2, T* __restrict__ A2t, T* __restrict__ Htt,
                             T* __restrict__ dOt, T* __restrict__ dUtt) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sw1 = reinterpret_cast<T*>(smem_raw);  // [m][m]
  T* sw2 = sw1 + m * m;                     // [m][m]
  T* sb1 = sw2 + m * m;                     // [m]
  T* sb2 = sb1 + m;                         // [m]
  T* smu = sb2 + m;                         // [m]
  T* sinv = smu + m;                        // [m]
  T* sa = sinv + m;                         // [m][CH] a2
  const int CH = blockDim.x;
  T* su = sa + m * CH;   // [m][CH] Ut
  T* sd = su + m * CH;   // [m][CH] dO
  T* sg = sd + m * CH;   // [m][CH] dUt
  __shared__ uint8_t smask[64];
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
    sw1[i] = Wt1[i];
    sw2[i] = Wt2[i];
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    sb1[i] = bt1[i];
    sb2[i] = bt2[i];
  }
  const int t = threadIdx.x;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      smu[j] = st2[2 * (b * m + j)];
      sinv[j] = st2[2 * (b * m + j) + 1];
      smask[j] = mask[b * m + j];
    }
    __syncthreads();
    for (int c0 = 0; c0 < d; c0 += CH) {
      const int c = c0 + t;
      if (c < d) {
        const T gc = g2[c], bc = b2[c];
        for (int s = 0; s < m; ++s) {
          const T xhat = (y[(b * m + s) * ld + c] - smu[s]) * sinv[s];
          sa[s * CH + t] = gc * xhat + bc;
        }
        for (int j = 0; j < m; ++j) {
          T u = T(0);
          for (int i = 0; i < m; ++i) u += sa[i * CH + t] * sw1[i * m + j];
          su[j * CH + t] = u + sb1[j];
        }
        if (!BWD) {
          for (int s = 0; s < m; ++s) {
            T o = T(0);
            for (int j = 0; j < m; ++j) o += gelu(su[j * CH + t]) * sw2[j * m + s];
            const T zo = y[(b * m + s) * ld + c] + (o + sb2[s]);
            zmix[(b * m + s) * ld + c] = zo * (smask[s] ? T(1) : T(0));
          }
        } else {
          const int64_t row = (b * d + c) * m;
          for (int s = 0; s < m; ++s) {
            const T g = smask[s] ? dzm[(b * m + s) * ld + c] : T(0);
            sd[s * CH + t] = g;
            dy[(b * m + s) * ld + c] = g;  // residual branch of z = y + token(LN2(y))
            dOt[row + s] = g;
            A2t[row + s] = sa[s * CH + t];
          }
          for (int j = 0; j < m; ++j) {
            T h = T(0);
            for (int s = 0; s < m; ++s) h += sw2[j * m + s] * sd[s * CH + t];
            const T u = su[j * CH + t];
            Htt[row + j] = gelu(u);
            const T gu = h * gelu_grad(u);
            sg[j * CH + t] = gu;
            dUtt[row + j] = gu;
          }
          for (int i = 0; i < m; ++i) {
            T a = T(0);
            for (int j = 0; j < m; ++j) a += sw1[i * m + j] * sg[j * CH + t];
            da2[(b * m + i) * ld + c] = a;
          }
        }
      }
    }
  }
}

// LayerNorm vjp (autodiff.py:407-416), one warp per row:
//   gx = g * xhat; dxhat = g * gamma; m1 = mean(dxhat); m2 = mean(gx * gamma)
//   dx += inv * (dxhat - m1 - xhat * m2);  gx is written for d gamma.
template <typename T>
__global__ void ln_bwd_kernel(const T* __restrict__ g, const T* __restrict__ x, int64_t ld,
                              const T* __restrict__ stats, const T* __restrict__ gamma, int64_t M, int d, T* dx,
                              T* __restrict__ gx) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < M;
       r += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const T mu = stats[2 * r], inv = stats[2 * r + 1];
    T s1 = T(0), s2 = T(0);
    for (int c = lane; c < d; c += 32) {
      const T gg = g[r * ld + c];
      const T xh = (x[r * ld + c] - mu) * inv;
      s1 += gg * gamma[c];
      s2 += (gg * xh) * gamma[c];
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const T m1 = s1 / T(d), m2 = s2 / T(d);
    for (int c = lane; c < d; c += 32) {
      const T gg = g[r * ld + c];
      const T xh = (x[r * ld + c] - mu) * inv;
      dx[r * ld + c] += inv * ((gg * gamma[c] - m1) - xh * m2);
      gx[r * ld + c] = gg * xh;
    }
  }
}

// ---------------------------------------------------------------- workspace
inline int64_t r4(int64_t x) { return (x + 3) & ~int64_t(3); }

struct Bump {
  size_t bytes = 0;
  size_t take(size_t n) {
    const size_t o = bytes;
    bytes += (n + 255) & ~size_t(255);
    return o;
  }
};

struct BwdLayout {
  int64_t ld, M, B;
  size_t ones, Xv, Xe, Xt, Pv, Pe, Pt, z, dz, zt, dzt, st1, st2, a1, U, H, y, zmix, dzm, dy, T1, T2, T3, T4, bvec1,
      bvec2, bvec3, mvec, total;
};

BwdLayout bwd_layout(const tg_score_model& s, int64_t B, size_t esz) {
  BwdLayout L{};
  const int d = s.d_enc, F = s.F, m = s.m;
  L.ld = r4(d);
  L.B = B;
  L.M = B * m;
  const int64_t M = L.M, ld = L.ld;
  const bool f64 = esz == 8;
  const bool mixer = s.decoder == DEC_LINEAR || s.decoder == DEC_TRANS;
  const bool need_t = s.decoder != DEC_LINEAR && s.d_v > 0;
  Bump w;
  const int64_t nones = M > B * (int64_t)d ? M : B * (int64_t)d;
  L.ones = w.take(nones * esz);
  if (s.d_v && f64) L.Xv = w.take(M * s.d_v * esz);
  if (s.d_e && f64) L.Xe = w.take(M * s.d_e * esz);
  if (need_t && f64) L.Xt = w.take(B * s.d_v * esz);
  if (s.d_v) L.Pv = w.take(M * F * esz);
  if (s.d_e) L.Pe = w.take(M * F * esz);
  if (need_t) L.Pt = w.take(B * F * esz);
  L.z = w.take(M * ld * esz);
  L.dz = w.take(M * ld * esz);
  L.zt = w.take(B * ld * esz);
  L.dzt = w.take(B * ld * esz);
  if (mixer) {
    L.st1 = w.take(2 * M * esz);
    L.st2 = w.take(2 * M * esz);
    L.a1 = w.take(M * ld * esz);
    L.U = w.take(M * ld * esz);
    L.H = w.take(M * ld * esz);
    L.y = w.take(M * ld * esz);
    L.zmix = w.take(M * ld * esz);
    L.dzm = w.take(M * ld * esz);
    L.dy = w.take(M * ld * esz);
  }
  // T1..T4: [M, ld] or [B*d, m] scratch (token rows / decoder products)
  const int64_t tsz = (M * ld > B * (int64_t)d * m ? M * ld : B * (int64_t)d * m) * esz;
  L.T1 = w.take(tsz);
  L.T2 = w.take(tsz);
  if (mixer) {
    L.T3 = w.take(tsz);
    L.T4 = w.take(tsz);
  }
  L.bvec1 = w.take(B * ld * esz);
  L.bvec2 = w.take(B * ld * esz);
  L.bvec3 = w.take(B * ld * esz);
  L.mvec = w.take(M * esz);
  L.total = w.bytes;
  return L;
}

int validate_bwd(const tg_score_model* s) {
  if (!s) return fail(TG_EVALUE, "null score model");
  if (s->dtype != 0 && s->dtype != 1) return fail(TG_EVALUE, "score dtype must be 0 (f32) or 1 (f64)");
  if (s->decoder < 0 || s->decoder > 3) return fail(TG_ECONFIG, "unknown decoder %d", s->decoder);
  if (s->m < 1 || s->m > 64) return fail(TG_EVALUE, "scoring supports 1 <= m <= 64 (got %d)", s->m);
  const int d_enc = (s->d_v ? s->F : 0) + (s->d_e ? s->F : 0) + 2 * s->F + s->m;
  if (s->d_enc != d_enc) return fail(TG_EVALUE, "d_enc %d != encoded width %d", s->d_enc, d_enc);
  if (s->d_tv != (s->d_v ? s->F : 0) + 2 * s->F) return fail(TG_EVALUE, "bad target width %d", s->d_tv);
  return TG_OK;
}


// gat forward terms (sampler.py:104-115): lu[r] = pu[r].a_u, lv[b] = pv[b].a_v
// (the softmax kernel applies leaky(lu + lv)).  One warp per root.
template <typename T>
__global__ void gat_terms_kernel(const T* __restrict__ pu, const T* __restrict__ pv, int64_t ld,
                                 const T* __restrict__ a, int64_t B, int m, int d, T* __restrict__ lu,
                                 T* __restrict__ lv) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); b < B;
       b += (int64_t)gridDim.x * (blockDim.x / 32)) {
    T sv = T(0);
    for (int c = lane; c < d; c += 32) sv += pv[b * ld + c] * a[d + c];
    sv = warp_sum(sv);
    if (lane == 0) lv[b] = sv;
    for (int j = 0; j < m; ++j) {
      T su = T(0);
      for (int c = lane; c < d; c += 32) su += pu[(b * m + j) * ld + c] * a[c];
      su = warp_sum(su);
      if (lane == 0) lu[b * m + j] = su;
    }
  }
}

// trans forward (sampler.py:123-129): raw[r] = qt[b] . kn[r] (the softmax
// kernel applies 1/sqrt(count)).  One warp per row.
template <typename T>
__global__ void trans_raw_kernel(const T* __restrict__ qt, const T* __restrict__ kn, int64_t ld, int64_t M, int m,
                                 int d, T* __restrict__ raw) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < M;
       r += (int64_t)gridDim.x * (blockDim.x / 32)) {
    T s = T(0);
    for (int c = lane; c < d; c += 32) s += qt[(r / m) * ld + c] * kn[r * ld + c];
    s = warp_sum(s);
    if (lane == 0) raw[r] = s;
  }
}

// encode_target_batch's [proj_v | TE(0) | FE(1)] -> the neighbor row layout
// [proj_v | 0_e | TE(0) | FE(1) | 0_m] (pad_target_to_neighbor_layout,
// sampler.py:75-88)
template <typename T>
__global__ void pad_target_kernel(const T* __restrict__ zt, int64_t ldt, int64_t B, int F, int m, int has_v,
                                  int has_e, T* __restrict__ out, int64_t ldo) {
  const int d = (has_v ? F : 0) + (has_e ? F : 0) + 2 * F + m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B * d; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / d;
    int c = (int)(i - b * d);
    T v = T(0);
    const int pv = has_v ? F : 0;
    if (c < pv) {
      v = zt[b * ldt + c];
    } else {
      c -= pv;
      if (has_e) c -= F;
      if (c >= 0 && c < 2 * F) v = zt[b * ldt + pv + c];
    }
    out[b * ldo + (i - b * d)] = v;
  }
}

#define LAUNCH(kern, n, ...)                                                   \
  do {                                                                         \
    kern<<<grid_for((n), 256), 256, 0, st>>>(__VA_ARGS__);                     \
    TG_LAUNCHED();                                                             \
  } while (0)
#define RC(x)              \
  do {                     \
    int _rc = (x);         \
    if (_rc) return _rc;   \
  } while (0)

// One call's view of the model, its sizes and the workspace carve-up.
template <typename T>
struct Ctx {
  const tg_score_model& s;
  int64_t B, M, ld;
  int m, F, d;
  bool has_v, has_e;
  cudaStream_t st;
  unsigned char* ws;
  BwdLayout L;
  Ctx(const tg_score_model& s_, int64_t B_, unsigned char* ws_, cudaStream_t st_)
      : s(s_), B(B_), st(st_), ws(ws_), L(bwd_layout(s_, B_, sizeof(T))) {
    M = L.M, ld = L.ld, m = s.m, F = s.F, d = s.d_enc, has_v = s.d_v > 0, has_e = s.d_e > 0;
  }
  T* P(size_t off) const { return reinterpret_cast<T*>(ws + off); }
  static const T* W(const void* p) { return static_cast<const T*>(p); }
};

// Feature rows as the GEMM operand type: f32 rows are used in place for f32
// models and widened into the workspace for f64 ones.
template <typename T>
int prep_rows(Ctx<T>& c, const float* rows, int64_t ld_in, int64_t n, int w, size_t off, const T** out,
              int64_t* ld_out) {
  const cudaStream_t st = c.st;
  if (w == 0 || n == 0 || rows == nullptr) {
    *out = nullptr;
    *ld_out = w;
    return TG_OK;
  }
  if constexpr (sizeof(T) == 8) {
    LAUNCH(rows_to_t_kernel<T>, n * w, rows, ld_in, n, w, c.P(off));
    *out = c.P(off);
    *ld_out = w;
  } else {
    *out = reinterpret_cast<const T*>(rows);
    *ld_out = ld_in;
  }
  return TG_OK;
}

// encode_neighborhood_batch (encoders.py:152-183) into z [M, ld]; keeps the
// projections' pre-activations Pv / Pe.
template <typename T>
int enc_fwd(Ctx<T>& c, const int64_t* ids, const double* dts, const uint8_t* mask, const T* Xv, int64_t ldxv,
            const T* Xe, int64_t ldxe, T* z) {
  const cudaStream_t st = c.st;
  const auto& s = c.s;
  int col = 0;
  if (c.has_v) {
    RC(gemm_rm<T>(st, false, false, c.M, c.F, s.d_v, T(1), Xv, ldxv, c.W(s.W_node), c.F, T(0), c.P(c.L.Pv), c.F));
    LAUNCH(gelu_cols_kernel<T>, c.M * c.F, c.P(c.L.Pv), c.M, c.F, mask, z, c.ld, col);
    col += c.F;
  }
  if (c.has_e) {
    RC(gemm_rm<T>(st, false, false, c.M, c.F, s.d_e, T(1), Xe, ldxe, c.W(s.W_edge), c.F, T(0), c.P(c.L.Pe), c.F));
    LAUNCH(gelu_cols_kernel<T>, c.M * c.F, c.P(c.L.Pe), c.M, c.F, mask, z, c.ld, col);
  }
  const int te_off = (c.has_v ? c.F : 0) + (c.has_e ? c.F : 0);
  const size_t sm = (size_t)c.m * (sizeof(int64_t) + sizeof(double) + sizeof(int) + 1) + 16;
  encode_misc_kernel<T><<<(unsigned)(c.B < 65535 ? c.B : 65535), 256, sm, st>>>(ids, dts, mask, c.B, c.m, c.F, te_off,
                                                                                 s.omega, s.fe_table, z, c.ld);
  TG_LAUNCHED();
  return TG_OK;
}

// encode_target_batch (encoders.py:186-200) into zt [B, ld], padded into the
// neighbor layout (gat / gatv2) or not (trans); keeps Pt.
template <typename T>
int tgt_fwd(Ctx<T>& c, const T* Xt, int64_t ldxt, bool padded, T* zt) {
  const cudaStream_t st = c.st;
  if (c.has_v) {
    RC(gemm_rm<T>(st, false, false, c.B, c.F, c.s.d_v, T(1), Xt, ldxt, c.W(c.s.W_node), c.F, T(0), c.P(c.L.Pt),
                  c.F));
    LAUNCH(gelu_cols_kernel<T>, c.B * c.F, c.P(c.L.Pt), c.B, c.F, (const uint8_t*)nullptr, zt, c.ld, 0);
  }
  const int Wd = padded ? (c.has_e ? c.F : 0) + 2 * c.F + c.m : 2 * c.F;
  LAUNCH(target_misc_kernel<T>, c.B * Wd, c.B, c.F, c.m, (int)c.has_v, (int)c.has_e, (int)padded, c.s.fe_table, zt,
         c.ld);
  return TG_OK;
}

template <typename T>
int token_chunk(const Ctx<T>& c, size_t* smem) {
  int CH = 128;  // channels per chunk: the widest whose tiles fit 200 KB
  while (CH > 32 && (size_t)(2 * c.m * c.m + 4 * c.m + 4 * c.m * CH) * sizeof(T) > 200 * 1024) CH /= 2;
  *smem = (size_t)(2 * c.m * c.m + 4 * c.m + 4 * c.m * CH) * sizeof(T);
  return CH;
}

// mixer_transform (sampler.py:69-72 -> mixer.py:31-51) of z into zmix,
// keeping LN1 / LN2 statistics, LN1(z), U (pre-GeLU), H and y.
template <typename T>
int mix_fwd(Ctx<T>& c, const T* z, const uint8_t* mask, T* zmix) {
  const cudaStream_t st = c.st;
  const auto& s = c.s;
  const int64_t M = c.M, ld = c.ld;
  const int d = c.d;
  const T eps = T(1e-5);
  T *st1 = c.P(c.L.st1), *st2 = c.P(c.L.st2), *a1 = c.P(c.L.a1), *U = c.P(c.L.U), *H = c.P(c.L.H), *y = c.P(c.L.y);
  rowstats_kernel<T><<<(unsigned)((M + 7) / 8), 256, 0, st>>>(z, M, d, ld, eps, st1);
  TG_LAUNCHED();
  LAUNCH(ln_apply_kernel<T>, M * d, z, M, d, ld, st1, c.W(s.ln1_g), c.W(s.ln1_b), a1);
  RC(gemm_rm<T>(st, false, false, M, d, d, T(1), a1, ld, c.W(s.Wc1), d, T(0), U, ld));
  LAUNCH(bias_gelu_kernel<T>, M * d, U, M, d, ld, c.W(s.bc1), H);
  RC(gemm_rm<T>(st, false, false, M, d, d, T(1), H, ld, c.W(s.Wc2), d, T(0), y, ld));
  LAUNCH(bias_resid_kernel<T>, M * d, y, M, d, ld, c.W(s.bc2), z);
  rowstats_kernel<T><<<(unsigned)((M + 7) / 8), 256, 0, st>>>(y, M, d, ld, eps, st2);
  TG_LAUNCHED();
  size_t tsm = 0;
  const int CH = token_chunk(c, &tsm);
  const unsigned tgrid = (unsigned)(c.B < (int64_t)device_sms() * 8 ? c.B : (int64_t)device_sms() * 8);
  auto kf = token_kernel<T, false>;
  TG_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
  kf<<<tgrid, CH, tsm, st>>>(y, ld, st2, c.B, c.m, d, c.W(s.ln2_g), c.W(s.ln2_b), c.W(s.Wt1), c.W(s.bt1),
                             c.W(s.Wt2), c.W(s.bt2), mask, zmix, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                             nullptr);
  TG_LAUNCHED();
  return TG_OK;
}

// decode_policy (sampler.py:91-135): logits from z_raw / z_mixed / the
// (padded for gat / gatv2) target rows, then the masked softmax and
// log-softmax (autodiff.py:429-464).
template <typename T>
int dec_fwd(Ctx<T>& c, const T* z, const T* zmix, const T* zt, const uint8_t* mask, T* q, T* lq) {
  const cudaStream_t st = c.st;
  const auto& s = c.s;
  const int64_t M = c.M, B = c.B, ld = c.ld;
  const int d = c.d, m = c.m;
  T* logits = c.P(c.L.mvec);
  T* rowterm = c.P(c.L.bvec3);
  if (s.decoder == DEC_LINEAR) {
    RC(gemm_rm<T>(st, false, false, M, 1, d, T(1), zmix, ld, c.W(s.w_linear), 1, T(0), logits, 1));
  } else if (s.decoder == DEC_TRANS) {
    T* qt = c.P(c.L.bvec1);
    T* kn = c.P(c.L.T1);
    RC(gemm_rm<T>(st, false, false, B, d, s.d_tv, T(1), zt, ld, c.W(s.W_trans_target), d, T(0), qt, ld));
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), zmix, ld, c.W(s.W_trans_nbr), d, T(0), kn, ld));
    trans_raw_kernel<T><<<grid_for(M * 32, 256), 256, 0, st>>>(qt, kn, ld, M, m, d, logits);
    TG_LAUNCHED();
  } else if (s.decoder == DEC_GAT) {
    T* pu = c.P(c.L.T1);
    T* pv = c.P(c.L.bvec1);
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), z, ld, c.W(s.W_gat), d, T(0), pu, ld));
    RC(gemm_rm<T>(st, false, false, B, d, d, T(1), zt, ld, c.W(s.W_gat), d, T(0), pv, ld));
    gat_terms_kernel<T><<<grid_for(B * 32, 256), 256, 0, st>>>(pu, pv, ld, c.W(s.a_gat), B, m, d, logits, rowterm);
    TG_LAUNCHED();
  } else {
    const T* Wtop = c.W(s.W_gatv2);
    T* Q = c.P(c.L.T1);
    T* Hh = c.P(c.L.T2);
    T* R = c.P(c.L.bvec1);
    RC(gemm_rm<T>(st, false, false, B, d, d, T(1), zt, ld, Wtop + (int64_t)d * d, d, T(0), R, ld));
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), z, ld, Wtop, d, T(0), Q, ld));
    LAUNCH(gatv2_fwd_kernel<T>, M * d, Q, R, M, m, d, ld, static_cast<T>(s.slope), Hh);
    RC(gemm_rm<T>(st, false, false, M, 1, d, T(1), Hh, ld, c.W(s.a_gatv2), 1, T(0), logits, 1));
  }
  softmax_kernel<T><<<grid_for(B * 32, 256), 256, 0, st>>>(logits, 1, rowterm, mask, B, m, s.decoder,
                                                            static_cast<T>(s.slope), q, lq);
  TG_LAUNCHED();
  return TG_OK;
}

template <typename T>
int run_backward(const tg_score_model& s, const int64_t* ids, const double* dts, const uint8_t* mask,
                 const float* node_rows, int64_t node_ld, const float* edge_rows, int64_t edge_ld,
                 const float* tgt_rows, int64_t tgt_ld, int64_t B, const T* G, const tg_score_grads& gr,
                 unsigned char* ws, cudaStream_t st) {
  Ctx<T> c(s, B, ws, st);
  const BwdLayout& L = c.L;
  const int m = s.m, F = s.F, d = s.d_enc;
  const int64_t M = L.M, ld = L.ld;
  const bool has_v = c.has_v, has_e = c.has_e;
  const bool mixer = s.decoder == DEC_LINEAR || s.decoder == DEC_TRANS;
  const bool need_t = s.decoder != DEC_LINEAR;
  const bool padded = s.decoder == DEC_GAT || s.decoder == DEC_GATV2;
  const T slope = static_cast<T>(s.slope);
  auto P = [&](size_t off) { return c.P(off); };
  auto W = [](const void* p) { return static_cast<const T*>(p); };
  auto Gp = [](void* p) { return static_cast<T*>(p); };
  T* ones = P(L.ones);
  {
    const int64_t n = M > B * (int64_t)d ? M : B * (int64_t)d;
    LAUNCH(fill_kernel<T>, n, ones, n, T(1));
  }
  // ---- forward recompute
  const T *Xv, *Xe, *Xt = nullptr;
  int64_t ldxv, ldxe, ldxt = s.d_v;
  RC(prep_rows(c, node_rows, node_ld, M, s.d_v, L.Xv, &Xv, &ldxv));
  RC(prep_rows(c, edge_rows, edge_ld, M, s.d_e, L.Xe, &Xe, &ldxe));
  if (need_t) RC(prep_rows(c, tgt_rows, tgt_ld, B, s.d_v, L.Xt, &Xt, &ldxt));
  T* z = P(L.z);
  RC(enc_fwd(c, ids, dts, mask, Xv, ldxv, Xe, ldxe, z));
  T* zt = P(L.zt);
  if (need_t) RC(tgt_fwd(c, Xt, ldxt, padded, zt));
  T* zmix = nullptr;
  if (mixer) {
    zmix = P(L.zmix);
    RC(mix_fwd(c, z, mask, zmix));
  }
  size_t tsm = 0;
  const int CH = token_chunk(c, &tsm);
  const unsigned tgrid = (unsigned)(B < (int64_t)device_sms() * 8 ? B : (int64_t)device_sms() * 8);

  // ---- decoder vjps (sampler.py:100-129) -> dz (raw path) / dzm (mixed path) / dzt
  T* dz = P(L.dz);
  T* dzt = P(L.dzt);
  T* dzm = mixer ? P(L.dzm) : nullptr;
  bool dz_set = false;
  if (s.decoder == DEC_LINEAR) {
    // logits = z_mixed . w: dw += z_mixed^T G, dz_mixed = G w^T
    if (gr.w_linear) RC(gemm_rm<T>(st, true, false, d, 1, M, T(1), zmix, ld, G, 1, T(1), Gp(gr.w_linear), 1));
    LAUNCH(outer_kernel<T>, M * d, G, M, W(s.w_linear), d, dzm, ld, 0);
  } else if (s.decoder == DEC_TRANS) {
    T* qt = P(L.bvec1);
    T* dqt = P(L.bvec2);
    T* kn = P(L.T1);
    T* dkn = P(L.T2);
    RC(gemm_rm<T>(st, false, false, B, d, s.d_tv, T(1), zt, ld, W(s.W_trans_target), d, T(0), qt, ld));
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), zmix, ld, W(s.W_trans_nbr), d, T(0), kn, ld));
    trans_bwd_kernel<T><<<(unsigned)(B < 65535 ? B : 65535), 128, 0, st>>>(qt, kn, ld, G, mask, B, m, d, dqt, dkn);
    TG_LAUNCHED();
    if (gr.W_trans_target)
      RC(gemm_rm<T>(st, true, false, s.d_tv, d, B, T(1), zt, ld, dqt, ld, T(1), Gp(gr.W_trans_target), d));
    RC(gemm_rm<T>(st, false, true, B, s.d_tv, d, T(1), dqt, ld, W(s.W_trans_target), d, T(0), dzt, ld));
    if (gr.W_trans_nbr) RC(gemm_rm<T>(st, true, false, d, d, M, T(1), zmix, ld, dkn, ld, T(1), Gp(gr.W_trans_nbr), d));
    RC(gemm_rm<T>(st, false, true, M, d, d, T(1), dkn, ld, W(s.W_trans_nbr), d, T(0), dzm, ld));
  } else if (s.decoder == DEC_GAT) {
    const T* Wg = W(s.W_gat);
    const T* ag = W(s.a_gat);
    T* pu = P(L.T1);
    T* dpu = P(L.T2);
    T* pv = P(L.bvec1);
    T* dpv = P(L.bvec2);
    T* draw = P(L.mvec);
    T* dsum = P(L.bvec3);
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), z, ld, Wg, d, T(0), pu, ld));
    RC(gemm_rm<T>(st, false, false, B, d, d, T(1), zt, ld, Wg, d, T(0), pv, ld));
    gat_bwd_kernel<T><<<grid_for(B * 32, 256), 256, 0, st>>>(pu, pv, ld, ag, G, B, m, d, slope, draw, dsum);
    TG_LAUNCHED();
    if (gr.a_gat) {
      RC(gemm_rm<T>(st, true, false, d, 1, M, T(1), pu, ld, draw, 1, T(1), Gp(gr.a_gat), 1));
      RC(gemm_rm<T>(st, true, false, d, 1, B, T(1), pv, ld, dsum, 1, T(1), Gp(gr.a_gat) + d, 1));
    }
    LAUNCH(outer_kernel<T>, M * d, draw, M, ag, d, dpu, ld, 0);
    LAUNCH(outer_kernel<T>, B * d, dsum, B, ag + d, d, dpv, ld, 0);
    if (gr.W_gat) {
      RC(gemm_rm<T>(st, true, false, d, d, M, T(1), z, ld, dpu, ld, T(1), Gp(gr.W_gat), d));
      RC(gemm_rm<T>(st, true, false, d, d, B, T(1), zt, ld, dpv, ld, T(1), Gp(gr.W_gat), d));
    }
    RC(gemm_rm<T>(st, false, true, M, d, d, T(1), dpu, ld, Wg, d, T(0), dz, ld));
    RC(gemm_rm<T>(st, false, true, B, d, d, T(1), dpv, ld, Wg, d, T(0), dzt, ld));
    dz_set = true;
  } else {  // gatv2
    const T* Wtop = W(s.W_gatv2);
    const T* Wbot = Wtop + (int64_t)d * d;
    const T* av = W(s.a_gatv2);
    T* Q = P(L.T1);
    T* Hh = P(L.T2);
    T* R = P(L.bvec1);
    T* dQs = P(L.bvec2);
    RC(gemm_rm<T>(st, false, false, B, d, d, T(1), zt, ld, Wbot, d, T(0), R, ld));
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), z, ld, Wtop, d, T(0), Q, ld));
    LAUNCH(gatv2_fwd_kernel<T>, M * d, Q, R, M, m, d, ld, slope, Hh);
    if (gr.a_gatv2) RC(gemm_rm<T>(st, true, false, d, 1, M, T(1), Hh, ld, G, 1, T(1), Gp(gr.a_gatv2), 1));
    T* dQ = Hh;  // hidden no longer needed
    LAUNCH(gatv2_bwd_kernel<T>, M * d, G, av, Q, M, d, ld, slope, dQ);
    LAUNCH(slot_sum_kernel<T>, B * d, dQ, ld, B, m, d, dQs, ld);
    if (gr.W_gatv2) {
      RC(gemm_rm<T>(st, true, false, d, d, M, T(1), z, ld, dQ, ld, T(1), Gp(gr.W_gatv2), d));
      RC(gemm_rm<T>(st, true, false, d, d, B, T(1), zt, ld, dQs, ld, T(1), Gp(gr.W_gatv2) + (int64_t)d * d, d));
    }
    RC(gemm_rm<T>(st, false, true, M, d, d, T(1), dQ, ld, Wtop, d, T(0), dz, ld));
    RC(gemm_rm<T>(st, false, true, B, d, d, T(1), dQs, ld, Wbot, d, T(0), dzt, ld));
    dz_set = true;
  }

  // ---- mixer vjp (mixer.py:31-51 through mixer_transform's mask)
  if (mixer) {
    T *st1 = P(L.st1), *st2 = P(L.st2), *a1 = P(L.a1), *U = P(L.U), *H = P(L.H), *y = P(L.y);
    T* dy = P(L.dy);
    T* da2 = zmix;  // z_mixed consumed by the decoder vjp above
    T *A2t = P(L.T1), *Htt = P(L.T2), *dOt = P(L.T3), *dUt = P(L.T4);
    auto kb = token_kernel<T, true>;
    TG_CUDA(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    kb<<<tgrid, CH, tsm, st>>>(y, ld, st2, B, m, d, W(s.ln2_g), W(s.ln2_b), W(s.Wt1), W(s.bt1), W(s.Wt2), W(s.bt2),
                               mask, nullptr, dzm, dy, da2, A2t, Htt, dOt, dUt);
    TG_LAUNCHED();
    const int64_t BD = B * (int64_t)d;
    if (gr.Wt1) RC(gemm_rm<T>(st, true, false, m, m, BD, T(1), A2t, m, dUt, m, T(1), Gp(gr.Wt1), m));
    if (gr.Wt2) RC(gemm_rm<T>(st, true, false, m, m, BD, T(1), Htt, m, dOt, m, T(1), Gp(gr.Wt2), m));
    RC(colsum_acc<T>(st, dUt, BD, m, m, ones, Gp(gr.bt1)));
    RC(colsum_acc<T>(st, dOt, BD, m, m, ones, Gp(gr.bt2)));
    // LN2: dy += vjp(da2); gx2 -> d ln2_gamma
    T* gx = P(L.T1);
    ln_bwd_kernel<T><<<grid_for(M * 32, 256), 256, 0, st>>>(da2, y, ld, st2, W(s.ln2_g), M, d, dy, gx);
    TG_LAUNCHED();
    RC(colsum_acc<T>(st, gx, M, d, ld, ones, Gp(gr.ln2_g)));
    RC(colsum_acc<T>(st, da2, M, d, ld, ones, Gp(gr.ln2_b)));
    // channel MLP: y = z + (H Wc2 + bc2), H = gelu(U), U = LN1(z) Wc1 + bc1
    RC(colsum_acc<T>(st, dy, M, d, ld, ones, Gp(gr.bc2)));
    if (gr.Wc2) RC(gemm_rm<T>(st, true, false, d, d, M, T(1), H, ld, dy, ld, T(1), Gp(gr.Wc2), d));
    T* dH = dzm;
    RC(gemm_rm<T>(st, false, true, M, d, d, T(1), dy, ld, W(s.Wc2), d, T(0), dH, ld));
    LAUNCH(gelu_grad_kernel<T>, M * d, dH, U, M, d, ld);
    RC(colsum_acc<T>(st, dH, M, d, ld, ones, Gp(gr.bc1)));
    if (gr.Wc1) RC(gemm_rm<T>(st, true, false, d, d, M, T(1), a1, ld, dH, ld, T(1), Gp(gr.Wc1), d));
    T* da1 = P(L.T2);
    RC(gemm_rm<T>(st, false, true, M, d, d, T(1), dH, ld, W(s.Wc1), d, T(0), da1, ld));
    // dz = dy (residual) + LN1 vjp(da1)
    TG_CUDA(cudaMemcpyAsync(dz, dy, (size_t)M * ld * sizeof(T), cudaMemcpyDeviceToDevice, st));
    T* gx1 = P(L.T3);
    ln_bwd_kernel<T><<<grid_for(M * 32, 256), 256, 0, st>>>(da1, z, ld, st1, W(s.ln1_g), M, d, dz, gx1);
    TG_LAUNCHED();
    RC(colsum_acc<T>(st, gx1, M, d, ld, ones, Gp(gr.ln1_g)));
    RC(colsum_acc<T>(st, da1, M, d, ld, ones, Gp(gr.ln1_b)));
    dz_set = true;
  }
  (void)dz_set;

  // ---- encoder vjps: W_node (neighbors + targets), W_edge
  if (has_v && gr.W_node) {
    T* dP = P(mixer ? L.T4 : L.T2);
    LAUNCH(gelu_cols_grad_kernel<T>, M * F, dz, ld, 0, P(L.Pv), M, F, mask, dP);
    RC(gemm_rm<T>(st, true, false, s.d_v, F, M, T(1), Xv, ldxv, dP, F, T(1), Gp(gr.W_node), F));
    if (need_t) {
      T* dPt = P(L.bvec3);
      LAUNCH(gelu_cols_grad_kernel<T>, B * F, dzt, ld, 0, P(L.Pt), B, F, (const uint8_t*)nullptr, dPt);
      RC(gemm_rm<T>(st, true, false, s.d_v, F, B, T(1), Xt, ldxt, dPt, F, T(1), Gp(gr.W_node), F));
    }
  }
  if (has_e && gr.W_edge) {
    T* dP = P(mixer ? L.T4 : L.T2);
    LAUNCH(gelu_cols_grad_kernel<T>, M * F, dz, ld, has_v ? F : 0, P(L.Pe), M, F, mask, dP);
    RC(gemm_rm<T>(st, true, false, s.d_e, F, M, T(1), Xe, ldxe, dP, F, T(1), Gp(gr.W_edge), F));
  }
  return TG_OK;
}

// ---- the staged forward (reference-signature drop-ins, encoders.py /
// sampler.py): each stage reads the caller's tensors (their own row
// strides), runs on the internal [rows, ld] layout and writes the caller's.
template <typename T>
int copy_in(const Ctx<T>& c, const void* src, int64_t lds, int64_t rows, int w, T* dst) {
  TG_CUDA(cudaMemcpy2DAsync(dst, c.ld * sizeof(T), src, lds * sizeof(T), (size_t)w * sizeof(T), rows,
                            cudaMemcpyDeviceToDevice, c.st));
  return TG_OK;
}
template <typename T>
int copy_out(const Ctx<T>& c, const T* src, int64_t rows, int w, void* dst, int64_t ldd) {
  TG_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(T), src, c.ld * sizeof(T), (size_t)w * sizeof(T), rows,
                            cudaMemcpyDeviceToDevice, c.st));
  return TG_OK;
}

template <typename T>
int stage_encode(const tg_score_model& s, const int64_t* ids, const double* dts, const uint8_t* mask,
                 const float* node_rows, int64_t node_ld, const float* edge_rows, int64_t edge_ld, int64_t B,
                 void* out, int64_t ldo, unsigned char* ws, cudaStream_t st) {
  Ctx<T> c(s, B, ws, st);
  const T *Xv, *Xe;
  int64_t ldxv, ldxe;
  RC(prep_rows(c, node_rows, node_ld, c.M, s.d_v, c.L.Xv, &Xv, &ldxv));
  RC(prep_rows(c, edge_rows, edge_ld, c.M, s.d_e, c.L.Xe, &Xe, &ldxe));
  RC(enc_fwd(c, ids, dts, mask, Xv, ldxv, Xe, ldxe, c.P(c.L.z)));
  return copy_out(c, c.P(c.L.z), c.M, c.d, out, ldo);
}

template <typename T>
int stage_target(const tg_score_model& s, const float* tgt_rows, int64_t tgt_ld, int64_t B, void* out, int64_t ldo,
                 unsigned char* ws, cudaStream_t st) {
  Ctx<T> c(s, B, ws, st);
  const T* Xt;
  int64_t ldxt;
  RC(prep_rows(c, tgt_rows, tgt_ld, B, s.d_v, c.L.Xt, &Xt, &ldxt));
  RC(tgt_fwd(c, Xt, ldxt, false, c.P(c.L.zt)));
  return copy_out(c, c.P(c.L.zt), B, s.d_tv, out, ldo);
}

template <typename T>
int stage_mixer(const tg_score_model& s, const void* z, int64_t ldz, const uint8_t* mask, int64_t B, void* out,
                int64_t ldo, unsigned char* ws, cudaStream_t st) {
  Ctx<T> c(s, B, ws, st);
  RC(copy_in(c, z, ldz, c.M, c.d, c.P(c.L.z)));
  RC(mix_fwd(c, c.P(c.L.z), mask, c.P(c.L.zmix)));
  return copy_out(c, c.P(c.L.zmix), c.M, c.d, out, ldo);
}

template <typename T>
int stage_decode(const tg_score_model& s, const void* z_raw, int64_t ldr, const void* z_mixed, int64_t ldm,
                 const void* z_target, int64_t ldt, const uint8_t* mask, int64_t B, void* q, void* lq,
                 unsigned char* ws, cudaStream_t st) {
  Ctx<T> c(s, B, ws, st);
  T* z = nullptr;
  T* zmix = nullptr;
  T* zt = nullptr;
  if (s.decoder == DEC_GAT || s.decoder == DEC_GATV2) {
    RC(copy_in(c, z_raw, ldr, c.M, c.d, c.P(c.L.z)));
    z = c.P(c.L.z);
    zt = c.P(c.L.zt);
    pad_target_kernel<T><<<grid_for(B * c.d, 256), 256, 0, st>>>(static_cast<const T*>(z_target), ldt, B, c.F, c.m,
                                                                 (int)c.has_v, (int)c.has_e, zt, c.ld);
    TG_LAUNCHED();
  } else {
    RC(copy_in(c, z_mixed, ldm, c.M, c.d, c.P(c.L.zmix)));
    zmix = c.P(c.L.zmix);
    if (s.decoder == DEC_TRANS) {
      RC(copy_in(c, z_target, ldt, B, s.d_tv, c.P(c.L.zt)));
      zt = c.P(c.L.zt);
    }
  }
  return dec_fwd(c, z, zmix, zt, mask, static_cast<T*>(q), static_cast<T*>(lq));
}

}  // namespace
}  // namespace tg

using namespace tg;

extern "C" int tg_score_backward_workspace(const tg_score_model* s, int64_t B, size_t* bytes) {
  int rc = validate_bwd(s);
  if (rc) return rc;
  if (!bytes) return fail(TG_EVALUE, "null bytes");
  *bytes = bwd_layout(*s, B, s->dtype ? 8 : 4).total;
  return TG_OK;
}

extern "C" int tg_score_backward(const tg_score_model* s, const int64_t* ids, const double* dts,
                                 const uint8_t* mask, const float* node_rows, int64_t node_ld,
                                 const float* edge_rows, int64_t edge_ld, const float* tgt_rows, int64_t tgt_ld,
                                 int64_t B, const void* dlogits, const tg_score_grads* grads, void* workspace,
                                 size_t ws_bytes, void* stream) {
  int rc = validate_bwd(s);
  if (rc) return rc;
  if (!grads) return fail(TG_EVALUE, "null gradient table");
  if (B < 0) return fail(TG_EVALUE, "negative batch");
  if (B == 0) return TG_OK;
  if (!dlogits || !ids || !dts || !mask) return fail(TG_EVALUE, "null input");
  if (s->d_v && (!node_rows || (s->decoder != 0 && !tgt_rows)))
    return fail(TG_EVALUE, "node feature rows required (d_v=%d)", s->d_v);
  if (s->d_e && !edge_rows) return fail(TG_EVALUE, "edge feature rows required (d_e=%d)", s->d_e);
  const size_t need = bwd_layout(*s, B, s->dtype ? 8 : 4).total;
  if (ws_bytes < need) return fail(TG_EVALUE, "backward workspace too small: %zu < %zu", ws_bytes, need);
  const cudaStream_t st = as_stream(stream);
  auto* ws = static_cast<unsigned char*>(workspace);
  if (s->dtype == 1)
    return run_backward<double>(*s, ids, dts, mask, node_rows, node_ld, edge_rows, edge_ld, tgt_rows, tgt_ld, B,
                                static_cast<const double*>(dlogits), *grads, ws, st);
  return run_backward<float>(*s, ids, dts, mask, node_rows, node_ld, edge_rows, edge_ld, tgt_rows, tgt_ld, B,
                             static_cast<const float*>(dlogits), *grads, ws, st);
}

extern "C" int tg_score_stage_workspace(const tg_score_model* s, int64_t B, size_t* bytes) {
  return tg_score_backward_workspace(s, B, bytes);
}

#define TG_STAGE_CHECK(s, B, ws_bytes)                                                         \
  do {                                                                                         \
    int _rc = validate_bwd(s);                                                                 \
    if (_rc) return _rc;                                                                       \
    if ((B) < 0) return fail(TG_EVALUE, "negative batch");                                     \
    if ((B) == 0) return TG_OK;                                                                \
    const size_t _need = bwd_layout(*(s), (B), (s)->dtype ? 8 : 4).total;                      \
    if ((ws_bytes) < _need) return fail(TG_EVALUE, "stage workspace too small: %zu < %zu", (size_t)(ws_bytes), _need); \
  } while (0)

extern "C" int tg_encode_neighborhood(const tg_score_model* s, const int64_t* ids, const double* dts,
                                      const uint8_t* mask, const float* node_rows, int64_t node_ld,
                                      const float* edge_rows, int64_t edge_ld, int64_t B, void* z, int64_t ldz,
                                      void* workspace, size_t ws_bytes, void* stream) {
  TG_STAGE_CHECK(s, B, ws_bytes);
  if (s->d_v && !node_rows) return fail(TG_EVALUE, "node feature rows required (d_v=%d)", s->d_v);
  if (s->d_e && !edge_rows) return fail(TG_EVALUE, "edge feature rows required (d_e=%d)", s->d_e);
  auto* ws = static_cast<unsigned char*>(workspace);
  if (s->dtype == 1)
    return stage_encode<double>(*s, ids, dts, mask, node_rows, node_ld, edge_rows, edge_ld, B, z, ldz, ws,
                                as_stream(stream));
  return stage_encode<float>(*s, ids, dts, mask, node_rows, node_ld, edge_rows, edge_ld, B, z, ldz, ws,
                             as_stream(stream));
}

extern "C" int tg_encode_target(const tg_score_model* s, const float* tgt_rows, int64_t tgt_ld, int64_t B, void* zt,
                                int64_t ldt, void* workspace, size_t ws_bytes, void* stream) {
  TG_STAGE_CHECK(s, B, ws_bytes);
  if (s->d_v && !tgt_rows) return fail(TG_EVALUE, "target node rows required (d_v=%d)", s->d_v);
  auto* ws = static_cast<unsigned char*>(workspace);
  if (s->dtype == 1) return stage_target<double>(*s, tgt_rows, tgt_ld, B, zt, ldt, ws, as_stream(stream));
  return stage_target<float>(*s, tgt_rows, tgt_ld, B, zt, ldt, ws, as_stream(stream));
}

extern "C" int tg_mixer_transform(const tg_score_model* s, const void* z, int64_t ldz, const uint8_t* mask, int64_t B,
                                  void* out, int64_t ldo, void* workspace, size_t ws_bytes, void* stream) {
  TG_STAGE_CHECK(s, B, ws_bytes);
  auto* ws = static_cast<unsigned char*>(workspace);
  if (s->dtype == 1) return stage_mixer<double>(*s, z, ldz, mask, B, out, ldo, ws, as_stream(stream));
  return stage_mixer<float>(*s, z, ldz, mask, B, out, ldo, ws, as_stream(stream));
}

extern "C" int tg_decode_policy(const tg_score_model* s, const void* z_raw, int64_t ldr, const void* z_mixed,
                                int64_t ldm, const void* z_target, int64_t ldt, const uint8_t* mask, int64_t B,
                                void* q, void* log_q, void* workspace, size_t ws_bytes, void* stream) {
  TG_STAGE_CHECK(s, B, ws_bytes);
  const bool raw = s->decoder == 1 || s->decoder == 2;
  if (raw && !z_raw) return fail(TG_EVALUE, "the %s decoder reads z_raw", s->decoder == 1 ? "gat" : "gatv2");
  if (!raw && !z_mixed) return fail(TG_EVALUE, "the linear / trans decoders read z_mixed");
  if (s->decoder != 0 && !z_target) return fail(TG_EVALUE, "this decoder reads z_target");
  auto* ws = static_cast<unsigned char*>(workspace);
  if (s->dtype == 1)
    return stage_decode<double>(*s, z_raw, ldr, z_mixed, ldm, z_target, ldt, mask, B, q, log_q, ws,
                                as_stream(stream));
  return stage_decode<float>(*s, z_raw, ldr, z_mixed, ldm, z_target, ldt, mask, B, q, log_q, ws, as_stream(stream));
}
