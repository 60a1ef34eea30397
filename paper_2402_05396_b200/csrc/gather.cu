// K4 + K5: feature slice through the HBM cache.
//
// Replaces training.py:207-221 (_edge_feature_rows: rows of the valid slots
// in a zero buffer, looked up through the cache in train mode),
// training.py:223-230 (_node_feature_rows: node rows times the mask, i.e.
// signed zeros on padded slots) and cache.py:72-86 (lookup: count every
// access, report residency).
//
// A warp takes 32 consecutive slots: lane j resolves slot j (cache slot,
// counter increment, tier), then the warp streams the 32 rows with
// 8/16-byte vector loads (rows.cuh).  Hit/miss totals are warp-aggregated
// with __ballot_sync and added once per block.
#include "rows.cuh"

namespace tg {

constexpr int kGatherWarps = 8;

template <int VEC>
__global__ void __launch_bounds__(kGatherWarps * 32)
    gather_kernel(const int64_t* __restrict__ ids, const uint8_t* __restrict__ mask, int64_t n,
                  tg_feat_store fs, tg_cache_dev cache, int has_cache, int mask_mode, float* out,
                  int64_t out_ld, uint8_t* hits_out) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned long long hits = 0, misses = 0;
  const int64_t groups = (n + 31) / 32;
  for (int64_t grp = (int64_t)blockIdx.x * kGatherWarps + warp; grp < groups;
       grp += (int64_t)gridDim.x * kGatherWarps) {
    const int64_t i = grp * 32 + lane;
    const bool in_range = i < n;
    const bool valid = in_range && (mask == nullptr || mask[i] != 0);
    int64_t r = 0;
    if (in_range) r = ids[i];
    int32_t slot = -1;
    if (has_cache && valid) {
      slot = cache.slot_of[r];
      atomicAdd(cache.counters + r, 1);
    }
    if (has_cache) {
      hits += __popc(__ballot_sync(FULL, valid && slot >= 0));
      misses += __popc(__ballot_sync(FULL, valid && slot < 0));
    }
    if (hits_out && in_range) hits_out[i] = slot >= 0 ? 1 : 0;
    if (out != nullptr) {
      int mode = ROW_ZERO;
      const float* src = nullptr;
      if (valid) {
        mode = ROW_COPY;
        src = row_source(fs, r, slot);
      } else if (in_range && mask_mode == 1) {
        mode = ROW_TIMES_ZERO;  // node rows: row(ids[i]) * 0.0
        src = row_source(fs, r, -1);
      }
      const int64_t left = n - grp * 32;
      const int nrows = left < 32 ? (int)left : 32;
      warp_move_rows<VEC, (VEC == 4 ? 8 : 16)>(src, mode, nrows, out + grp * 32 * out_ld, out_ld,
                                                fs.d, lane);
    }
  }
  if (has_cache) {
    __shared__ unsigned long long red[2];
    if (threadIdx.x < 2) red[threadIdx.x] = 0;
    __syncthreads();
    if (lane == 0) {
      atomicAdd(&red[0], hits);
      atomicAdd(&red[1], misses);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (red[0]) atomicAdd(cache.stats + 0, red[0]);
      if (red[1]) atomicAdd(cache.stats + 1, red[1]);
    }
  }
}

static int launch_gather(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store* store,
                         const tg_cache_dev* cache, int mask_mode, float* out, int64_t out_ld,
                         uint8_t* hits, cudaStream_t st) {
  if (n < 0) return fail(TG_EVALUE, "negative row count");
  if (n == 0) return TG_OK;
  tg_feat_store fs{};
  if (store) fs = *store;
  if (out != nullptr && (store == nullptr || fs.d <= 0)) out = nullptr;
  tg_cache_dev cd{};
  const int has_cache = cache != nullptr && cache->slot_of != nullptr;
  if (has_cache) cd = *cache;
  if (out == nullptr && !has_cache && hits == nullptr) return TG_OK;
  const int vec = out ? pick_vec(fs.d, fs.ld, out_ld, fs.table, out, fs.hot, fs.hot ? fs.hot_ld : 0) : 4;
  const int64_t groups = (n + 31) / 32;
  const int64_t want = (groups + kGatherWarps - 1) / kGatherWarps;
  const int64_t cap = (int64_t)device_sms() * 8;
  const int grid = (int)(want < cap ? want : cap);
  const int threads = kGatherWarps * 32;
  if (vec == 4)
    gather_kernel<4><<<grid, threads, 0, st>>>(ids, mask, n, fs, cd, has_cache, mask_mode, out, out_ld, hits);
  else if (vec == 2)
    gather_kernel<2><<<grid, threads, 0, st>>>(ids, mask, n, fs, cd, has_cache, mask_mode, out, out_ld, hits);
  else
    gather_kernel<1><<<grid, threads, 0, st>>>(ids, mask, n, fs, cd, has_cache, mask_mode, out, out_ld, hits);
  TG_LAUNCHED();
  return TG_OK;
}

__global__ void range_kernel(const int64_t* __restrict__ ids, int64_t n, int64_t limit, int* bad) {
  int local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = ids[i];
    local |= (x < 0) | (x >= limit);
  }
  if (__any_sync(FULL, local) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

__global__ void gather_rows_kernel(const float* __restrict__ in, int64_t in_ld, const int64_t* __restrict__ order,
                                   int64_t n, int d, float* __restrict__ out, int64_t out_ld) {
  const int64_t total = n * (int64_t)d;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = w / d;
    const int c = (int)(w - r * d);
    out[r * out_ld + c] = in[order[r] * in_ld + c];
  }
}

}  // namespace tg

using namespace tg;

extern "C" int tg_lookup_gather(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store* store,
                                const tg_cache_dev* cache, int32_t mask_mode, float* out, int64_t out_ld,
                                void* stream) {
  if (mask_mode != 0 && mask_mode != 1) return fail(TG_EVALUE, "mask_mode must be 0 or 1");
  return launch_gather(ids, mask, n, store, cache, mask_mode, out, out_ld, nullptr, as_stream(stream));
}

extern "C" int tg_cache_lookup(const int64_t* ids, int64_t n, const tg_cache_dev* cache, uint8_t* hits,
                               const tg_feat_store* store, float* feat_out, int64_t out_ld, void* stream) {
  if (cache == nullptr || cache->slot_of == nullptr) return fail(TG_EVALUE, "cache state required");
  return launch_gather(ids, nullptr, n, store, cache, 0, feat_out, out_ld, hits, as_stream(stream));
}

extern "C" int tg_check_range(const int64_t* ids, int64_t n, int64_t limit, void* stream) {
  if (n <= 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  int* bad = nullptr;
  TG_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  TG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const int64_t want = (n + 255) / 256;
  const int grid = (int)(want < 4096 ? want : 4096);
  range_kernel<<<grid, 256, 0, st>>>(ids, n, limit, bad);
  TG_LAUNCHED();
  int h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaFreeAsync(bad, st));
  TG_CUDA(cudaStreamSynchronize(st));
  if (h) return fail(TG_EINDEX, "edge id out of range [0, %lld)", (long long)limit);
  return TG_OK;
}

extern "C" int tg_gather_rows_f32(const float* in, int64_t in_ld, const int64_t* order, int64_t n, int32_t d,
                                  float* out, int64_t out_ld, void* stream) {
  if (n <= 0 || d <= 0) return TG_OK;
  const int64_t total = n * (int64_t)d;
  const int64_t want = (total + 255) / 256;
  const int grid = (int)(want < 65535 ? want : 65535);
  gather_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(in, in_ld, order, n, d, out, out_ld);
  TG_LAUNCHED();
  return TG_OK;
}
