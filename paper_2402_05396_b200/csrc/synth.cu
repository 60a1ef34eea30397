// Synthetic shape generator (bench inputs).  Every value is a
// pure function of (seed, stream, counter) through splitmix64 and exact IEEE
// f64 arithmetic (explicit _rn intrinsics, no contraction), so
// oracle/shapes.py regenerates bit-identical graphs and feature rows on the
// host for the parity checks.  GDELT-sized tables (191M x 186 f32) are
// written straight into HBM.
#include "common.cuh"

namespace tg {

__device__ __forceinline__ uint64_t hstream(uint64_t seed, uint64_t stream, uint64_t c) {
  return mix64(mix64(seed ^ (stream * STREAM)) + (c + 1) * GOLDEN);
}
__device__ __forceinline__ double unit(uint64_t z) {
  return static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void synth_events_kernel(int64_t e0, int64_t n, int64_t E, int64_t V, uint64_t seed,
                                    const double* __restrict__ cdf, const int64_t* __restrict__ node_at_rank,
                                    int ts_mode, double span, int64_t* __restrict__ src, int64_t* __restrict__ dst,
                                    double* __restrict__ ts) {
  const double step = span / static_cast<double>(E);
  const double tie_scale = static_cast<double>(E / 8 > 0 ? E / 8 : 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e0 + i;
    const double u1 = unit(hstream(seed, 1, e));
    int64_t lo = 0, hi = V;  // first rank with cdf >= u1 (np.searchsorted side='left')
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] < u1) lo = mid + 1;
      else hi = mid;
    }
    if (lo >= V) lo = V - 1;
    src[i] = node_at_rank[lo];
    dst[i] = static_cast<int64_t>(hstream(seed, 2, e) % static_cast<uint64_t>(V));
    double t;
    if (ts_mode == 0) {
      t = __dmul_rn(__dadd_rn(static_cast<double>(e), unit(hstream(seed, 3, e))), step);
    } else if (ts_mode == 1) {
      t = floor(__dmul_rn(unit(hstream(seed, 4, e)), tie_scale));
    } else {
      t = static_cast<double>(e + 1);
    }
    ts[i] = t;
  }
}

__global__ void synth_features_kernel(int64_t r0, int64_t n, int d, uint64_t seed, float* __restrict__ out,
                                      int64_t ld) {
  const int64_t total = n * (int64_t)d;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = w / d;
    const int j = static_cast<int>(w - i * d);
    const uint64_t z = mix64(mix64(seed ^ (static_cast<uint64_t>(r0 + i + 1) * STREAM)) + (uint64_t)(j + 1) * GOLDEN);
    out[i * ld + j] = static_cast<float>(static_cast<int32_t>(z >> 40) - 8388608) * (1.0f / 8388608.0f);
  }
}

static int grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  const int64_t cap = (int64_t)device_sms() * 32;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace tg

using namespace tg;

extern "C" int tg_synth_events(int64_t e0, int64_t n, int64_t E, int64_t V, uint64_t seed, const double* zipf_cdf,
                               const int64_t* node_at_rank, int32_t ts_mode, double span, int64_t* src, int64_t* dst,
                               double* ts, void* stream) {
  if (n <= 0) return TG_OK;
  if (V <= 0) return fail(TG_EVALUE, "need V >= 1");
  synth_events_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(e0, n, E, V, seed, zipf_cdf, node_at_rank, ts_mode,
                                                                  span, src, dst, ts);
  TG_LAUNCHED();
  return TG_OK;
}

extern "C" int tg_synth_features(int64_t r0, int64_t n, int32_t d, uint64_t seed, float* out, int64_t ld,
                                 void* stream) {
  if (n <= 0 || d <= 0) return TG_OK;
  synth_features_kernel<<<grid_for(n * (int64_t)d), 256, 0, as_stream(stream)>>>(r0, n, d, seed, out, ld);
  TG_LAUNCHED();
  return TG_OK;
}
