// Shared device/host helpers for libtaser_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "taser_b200.h"

namespace tg {

// ---- error plumbing --------------------------------------------------------
std::string& last_error();
std::atomic<unsigned long long>& launch_counter();

inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

#define TG_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return ::tg::fail(TG_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,         \
                        cudaGetErrorString(_e));                                   \
  } while (0)

// Check a launch and count it (the bench reports how many of OUR kernels ran).
#define TG_LAUNCHED()                                                              \
  do {                                                                             \
    ::tg::launch_counter().fetch_add(1, std::memory_order_relaxed);                \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess)                                                         \
      return ::tg::fail(TG_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__,           \
                        cudaGetErrorString(_e));                                   \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr unsigned FULL = 0xffffffffu;

// ---- splitmix64 (finder.py:29-33, 56-66) ------------------------------------
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t MIX2 = 0x94D049BB133111EBull;
constexpr uint64_t STREAM = 0xA24BAED4963EE407ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}

// Draw k (1-based) of row stream `state` = mix(state + k*GOLDEN): the k-th
// call of finder.py:_next without carrying the running state.
__device__ __forceinline__ uint64_t draw(uint64_t state, uint64_t k) {
  return mix64(state + k * GOLDEN);
}

__device__ __forceinline__ int64_t global_row(const tg_rowmap& r, int64_t i) {
  return i < r.split ? r.base0 + i : r.base1 + (i - r.split);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

int device_sms();

}  // namespace tg
