// Warp-cooperative feature-row movement shared by the fused finder (find.cu)
// and the standalone feature slice (gather.cu).
//
// A warp moves a GROUP of up to 32 rows.  Lane j owns row j of the group: it
// resolves that row's source pointer (tier lookup) and its mode, then the
// whole warp streams the group's rows as one flat sequence of VEC-float units
// so consecutive lanes touch consecutive 8/16-byte words (coalesced loads of
// each 688/744-byte row, fully coalesced stores of the contiguous output
// block).  U units per lane are issued before any store so each warp keeps
// U*32*VEC*4 bytes in flight.
#pragma once

#include "common.cuh"

namespace tg {

enum RowMode : int { ROW_COPY = 0, ROW_ZERO = 1, ROW_TIMES_ZERO = 2 };

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  using T = float;
};
template <>
struct VecT<2> {
  using T = float2;
};
template <>
struct VecT<4> {
  using T = float4;
};

__device__ __forceinline__ float ld_stream(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];"
               : "=f"(r.x), "=f"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float zero_like(float) { return 0.0f; }
__device__ __forceinline__ float2 zero_like(float2) { return make_float2(0.0f, 0.0f); }
__device__ __forceinline__ float4 zero_like(float4) { return make_float4(0.0f, 0.0f, 0.0f, 0.0f); }
__device__ __forceinline__ float times_zero(float a) { return a * 0.0f; }
__device__ __forceinline__ float2 times_zero(float2 a) { return make_float2(a.x * 0.0f, a.y * 0.0f); }
__device__ __forceinline__ float4 times_zero(float4 a) {
  return make_float4(a.x * 0.0f, a.y * 0.0f, a.z * 0.0f, a.w * 0.0f);
}

// Source row of logical row r (eid or node id) given its cache slot.
__device__ __forceinline__ const float* row_source(const tg_feat_store& s, int64_t r, int32_t slot) {
  if (s.hot != nullptr && slot >= 0) return s.hot + (int64_t)slot * s.hot_ld;
  if (s.n_peers > 0) {
    int64_t p = r / s.shard_rows;
    return s.peers[p] + (r - p * s.shard_rows) * s.ld;
  }
  return s.table + r * s.ld;
}

// Copy `nrows` (<= 32) rows; lane j supplies (src, mode) of row j.
// dst0 is the first output row; rows are out_ld floats apart.
template <int VEC, int U>
__device__ __forceinline__ void warp_move_rows(const float* src_lane, int mode_lane, int nrows,
                                               float* dst0, int64_t out_ld, int d, int lane) {
  using V = typename VecT<VEC>::T;
  const int nv = d / VEC;
  const int total = nrows * nv;
  // (row, col) of this lane's current unit; advanced by 32 units per step.
  int row = lane / nv;
  int col = lane - row * nv;
  for (int base = 0; base < total; base += 32 * U) {
    V v[U];
    int rr[U], cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rr[u] = row;
      cc[u] = col;
      col += 32;
      while (col >= nv) {
        col -= nv;
        ++row;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int w = base + u * 32 + lane;
      const int srow = rr[u] < 32 ? rr[u] : 31;
      const float* s = reinterpret_cast<const float*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(src_lane), srow));
      const int md = __shfl_sync(FULL, mode_lane, srow);
      V x = zero_like(V());
      if (w < total && md != ROW_ZERO) {
        x = ld_stream(reinterpret_cast<const V*>(s) + cc[u]);
        if (md == ROW_TIMES_ZERO) x = times_zero(x);
      }
      v[u] = x;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int w = base + u * 32 + lane;
      if (w < total) reinterpret_cast<V*>(dst0 + (int64_t)rr[u] * out_ld)[cc[u]] = v[u];
    }
  }
}

// Flattened row gather (gather.cu): out[i, :] = row(ids[i]) for valid i
// (mask == NULL or mask[i]); invalid rows are +0.0 (ROW_ZERO) or
// row(ids[i]) * 0.0 (ROW_TIMES_ZERO).  slot_of (may be NULL) routes resident
// rows to the hot tier when the store has one.
int launch_row_gather(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store& fs,
                      const int32_t* slot_of, int invalid_mode, float* out, int64_t out_ld, cudaStream_t st);

// Widest vector that divides the row width and keeps every row aligned.
inline int pick_vec(int d, int64_t ld_a, int64_t ld_b, const void* p_a, const void* p_b,
                    const void* p_c = nullptr, int64_t ld_c = 0) {
  auto ok = [&](int v) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p_a), b = reinterpret_cast<uintptr_t>(p_b),
                    c = reinterpret_cast<uintptr_t>(p_c);
    const uintptr_t bytes = 4u * v;
    return d % v == 0 && ld_a % v == 0 && ld_b % v == 0 && ld_c % v == 0 && a % bytes == 0 &&
           b % bytes == 0 && c % bytes == 0;
  };
  if (ok(4)) return 4;
  if (ok(2)) return 2;
  return 1;
}

}  // namespace tg
