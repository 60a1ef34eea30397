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

constexpr int DEC_LINEAR = 0, DEC_GAT = 1, DEC_GATV2 = 2, DEC_TRANS = 3;

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

template <typename T>
int run_backward(const tg_score_model& s, const int64_t* ids, const double* dts, const uint8_t* mask,
                 const float* node_rows, int64_t node_ld, const float* edge_rows, int64_t edge_ld,
                 const float* tgt_rows, int64_t tgt_ld, int64_t B, const T* G, const tg_score_grads& gr,
                 unsigned char* ws, cudaStream_t st) {
  const BwdLayout L = bwd_layout(s, B, sizeof(T));
  const int m = s.m, F = s.F, d = s.d_enc;
  const int64_t M = L.M, ld = L.ld;
  const bool has_v = s.d_v > 0, has_e = s.d_e > 0;
  const bool mixer = s.decoder == DEC_LINEAR || s.decoder == DEC_TRANS;
  const bool need_t = s.decoder != DEC_LINEAR;
  const bool padded = s.decoder == DEC_GAT || s.decoder == DEC_GATV2;
  const T slope = static_cast<T>(s.slope);
  const T eps = T(1e-5);
  auto P = [&](size_t off) { return reinterpret_cast<T*>(ws + off); };
  auto W = [](const void* p) { return static_cast<const T*>(p); };
  auto Gp = [](void* p) { return static_cast<T*>(p); };
  T* ones = P(L.ones);
  {
    const int64_t n = M > B * (int64_t)d ? M : B * (int64_t)d;
    LAUNCH(fill_kernel<T>, n, ones, n, T(1));
  }
  // ---- forward recompute: encoders (encoders.py:152-200)
  const T* Xv = nullptr;
  const T* Xe = nullptr;
  const T* Xt = nullptr;
  int64_t ldxv = s.d_v, ldxe = s.d_e, ldxt = s.d_v;
  if constexpr (sizeof(T) == 8) {
    if (has_v) {
      LAUNCH(rows_to_t_kernel<T>, M * s.d_v, node_rows, node_ld, M, s.d_v, P(L.Xv));
      Xv = P(L.Xv);
    }
    if (has_e) {
      LAUNCH(rows_to_t_kernel<T>, M * s.d_e, edge_rows, edge_ld, M, s.d_e, P(L.Xe));
      Xe = P(L.Xe);
    }
    if (has_v && need_t) {
      LAUNCH(rows_to_t_kernel<T>, B * s.d_v, tgt_rows, tgt_ld, B, s.d_v, P(L.Xt));
      Xt = P(L.Xt);
    }
  } else {
    Xv = reinterpret_cast<const T*>(node_rows), ldxv = node_ld;
    Xe = reinterpret_cast<const T*>(edge_rows), ldxe = edge_ld;
    Xt = reinterpret_cast<const T*>(tgt_rows), ldxt = tgt_ld;
  }
  T* z = P(L.z);
  int col = 0;
  if (has_v) {
    RC(gemm_rm<T>(st, false, false, M, F, s.d_v, T(1), Xv, ldxv, W(s.W_node), F, T(0), P(L.Pv), F));
    LAUNCH(gelu_cols_kernel<T>, M * F, P(L.Pv), M, F, mask, z, ld, col);
    col += F;
  }
  if (has_e) {
    RC(gemm_rm<T>(st, false, false, M, F, s.d_e, T(1), Xe, ldxe, W(s.W_edge), F, T(0), P(L.Pe), F));
    LAUNCH(gelu_cols_kernel<T>, M * F, P(L.Pe), M, F, mask, z, ld, col);
  }
  const int te_off = (has_v ? F : 0) + (has_e ? F : 0);
  {
    const size_t sm = (size_t)m * (sizeof(int64_t) + sizeof(double) + sizeof(int) + 1) + 16;
    encode_misc_kernel<T><<<(unsigned)(B < 65535 ? B : 65535), 256, sm, st>>>(ids, dts, mask, B, m, F, te_off,
                                                                               s.omega, s.fe_table, z, ld);
    TG_LAUNCHED();
  }
  // target embedding: padded into the neighbor layout (gat / gatv2,
  // sampler.py:75-88) or as encode_target_batch returns it (trans)
  T* zt = P(L.zt);
  if (need_t) {
    if (has_v) {
      RC(gemm_rm<T>(st, false, false, B, F, s.d_v, T(1), Xt, ldxt, W(s.W_node), F, T(0), P(L.Pt), F));
      LAUNCH(gelu_cols_kernel<T>, B * F, P(L.Pt), B, F, (const uint8_t*)nullptr, zt, ld, 0);
    }
    const int Wd = padded ? (has_e ? F : 0) + 2 * F + m : 2 * F;
    LAUNCH(target_misc_kernel<T>, B * Wd, B, F, m, (int)has_v, (int)has_e, (int)padded, s.fe_table, zt, ld);
  }
  // ---- mixer forward (linear / trans read z_mixed)
  T* zmix = nullptr;
  if (mixer) {
    T *st1 = P(L.st1), *st2 = P(L.st2), *a1 = P(L.a1), *U = P(L.U), *H = P(L.H), *y = P(L.y);
    zmix = P(L.zmix);
    rowstats_kernel<T><<<(unsigned)((M + 7) / 8), 256, 0, st>>>(z, M, d, ld, eps, st1);
    TG_LAUNCHED();
    LAUNCH(ln_apply_kernel<T>, M * d, z, M, d, ld, st1, W(s.ln1_g), W(s.ln1_b), a1);
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), a1, ld, W(s.Wc1), d, T(0), U, ld));
    LAUNCH(bias_gelu_kernel<T>, M * d, U, M, d, ld, W(s.bc1), H);
    RC(gemm_rm<T>(st, false, false, M, d, d, T(1), H, ld, W(s.Wc2), d, T(0), y, ld));
    LAUNCH(bias_resid_kernel<T>, M * d, y, M, d, ld, W(s.bc2), z);
    rowstats_kernel<T><<<(unsigned)((M + 7) / 8), 256, 0, st>>>(y, M, d, ld, eps, st2);
    TG_LAUNCHED();
  }
  int CH = 128;  // channels per chunk: the widest whose tiles fit 200 KB
  while (CH > 32 && (size_t)(2 * m * m + 4 * m + 4 * m * CH) * sizeof(T) > 200 * 1024) CH /= 2;
  const size_t tsm = (size_t)(2 * m * m + 4 * m + 4 * m * CH) * sizeof(T);
  const unsigned tgrid = (unsigned)(B < (int64_t)device_sms() * 8 ? B : (int64_t)device_sms() * 8);
  if (mixer) {
    auto kf = token_kernel<T, false>;
    TG_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    kf<<<tgrid, CH, tsm, st>>>(P(L.y), ld, P(L.st2), B, m, d, W(s.ln2_g), W(s.ln2_b), W(s.Wt1), W(s.bt1), W(s.Wt2),
                               W(s.bt2), mask, zmix, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    TG_LAUNCHED();
  }

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
