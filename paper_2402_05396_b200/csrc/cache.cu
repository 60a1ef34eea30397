// K6: epoch-boundary cache replacement.  Replaces cache.py:89-118
// (_topk_edges + maybe_replace) and the top-k used by oracle_cache
// (cache.py:121-136).
//
// The reference ranks touched edges by the composite key count*E - eid
// (count descending, eid ascending) and keeps the k largest.  On device the
// same order is the uint64 key (count << 32) | ~eid, which is unique per
// edge, so "top k" is exactly {key >= T} for T the k-th largest key.  T is
// found by an MSB-first radix select: eight 8-bit digit passes, each a
// shared-memory histogram of the keys that match the digits fixed so far,
// followed by a one-block scan that fixes the next digit -- no sort of the
// (up to 191M) counters and no host round trip between passes.
#include <cub/cub.cuh>

#include "rows.cuh"

namespace tg {

struct SelectState {
  unsigned long long prefix;  // digits fixed so far
  unsigned long long fixed;   // mask of fixed digits
  long long k_rem;            // rank still to find inside the prefix
  unsigned long long hist[256];
};

__device__ __forceinline__ unsigned long long edge_key(const int32_t* counts, int64_t e) {
  const int32_t c = counts[e];
  return c > 0 ? (static_cast<unsigned long long>(c) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(e))
               : 0ull;
}

__global__ void touched_kernel(const int32_t* __restrict__ counts, int64_t E, unsigned long long* out) {
  unsigned long long local = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    local += counts[e] > 0;
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

__global__ void hist_kernel(const int32_t* __restrict__ counts, int64_t E, int shift, SelectState* s) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned long long prefix = s->prefix, fixed = s->fixed;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = edge_key(counts, e);
    if (k != 0 && (k & fixed) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&s->hist[i], (unsigned long long)h[i]);
}

__global__ void pick_digit_kernel(int shift, SelectState* s) {
  // one thread: walk digits from 255 down (largest keys first)
  if (threadIdx.x != 0) return;
  long long above = 0;
  int d = 255;
  for (; d > 0; --d) {
    const long long c = (long long)s->hist[d];
    if (above + c >= s->k_rem) break;
    above += c;
  }
  s->prefix |= (unsigned long long)d << shift;
  s->fixed |= 255ull << shift;
  s->k_rem -= above;
  for (int i = 0; i < 256; ++i) s->hist[i] = 0;
}

__global__ void overlap_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ slot_of, int64_t E,
                               const SelectState* s, int use_threshold, unsigned long long* out,
                               uint8_t* __restrict__ sel_mask) {
  const unsigned long long T = use_threshold ? s->prefix : 1ull;
  unsigned long long ov = 0, sel = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = edge_key(counts, e);
    const bool in = k != 0 && k >= T;
    sel += in;
    if (slot_of) ov += in && slot_of[e] >= 0;
    if (sel_mask) sel_mask[e] = in ? 1 : 0;
  }
  ov = warp_sum(ov);
  sel = warp_sum(sel);
  if ((threadIdx.x & 31) == 0) {
    if (ov) atomicAdd(out + 0, ov);
    if (sel) atomicAdd(out + 1, sel);
  }
}

__global__ void flag_kernel(const uint8_t* __restrict__ sel, int64_t E, int32_t* __restrict__ flags) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    flags[e] = sel[e];
}

__global__ void assign_kernel(const uint8_t* __restrict__ sel, const int32_t* __restrict__ scan, int64_t E,
                              int32_t* __restrict__ slot_of) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    slot_of[e] = sel[e] ? scan[e] : -1;
}

// hot[slot_of[e]] = cold row(e) for the newly resident set (warp per row).
__global__ void refill_kernel(const int32_t* __restrict__ slot_of, int64_t E, tg_feat_store fs, float* hot,
                              int64_t hot_ld) {
  const int lane = threadIdx.x & 31;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < E;
       e += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t s = slot_of[e];
    if (s < 0) continue;
    const float* src = row_source(fs, e, -1);
    for (int j = lane; j < fs.d; j += 32) hot[(int64_t)s * hot_ld + j] = src[j];
  }
}

static int grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  const int64_t cap = (int64_t)device_sms() * 8;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

// Fills sel_mask (may be NULL) with the top-k touched edges; returns
// (overlap with slot_of, selected count) in host_ov.
static int select_topk(const int32_t* counts, const int32_t* slot_of, int64_t E, int64_t k, uint8_t* sel_mask,
                       unsigned long long host_ov[2], cudaStream_t st) {
  unsigned long long* dev = nullptr;
  SelectState* s = nullptr;
  TG_CUDA(cudaMallocAsync(&dev, 3 * sizeof(unsigned long long), st));
  TG_CUDA(cudaMallocAsync(&s, sizeof(SelectState), st));
  TG_CUDA(cudaMemsetAsync(dev, 0, 3 * sizeof(unsigned long long), st));
  TG_CUDA(cudaMemsetAsync(s, 0, sizeof(SelectState), st));
  touched_kernel<<<grid_for(E), 256, 0, st>>>(counts, E, dev + 2);
  TG_LAUNCHED();
  unsigned long long touched = 0;
  TG_CUDA(cudaMemcpyAsync(&touched, dev + 2, sizeof(touched), cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaStreamSynchronize(st));
  int use_threshold = 0;
  if (k <= 0 || touched == 0) {
    // empty top-k: nothing selected
    if (sel_mask) TG_CUDA(cudaMemsetAsync(sel_mask, 0, E, st));
    host_ov[0] = host_ov[1] = 0;
    TG_CUDA(cudaFreeAsync(dev, st));
    TG_CUDA(cudaFreeAsync(s, st));
    return TG_OK;
  }
  if ((long long)touched > k) {
    use_threshold = 1;
    const long long kr = k;
    TG_CUDA(cudaMemcpyAsync(&s->k_rem, &kr, sizeof(kr), cudaMemcpyHostToDevice, st));
    for (int shift = 56; shift >= 0; shift -= 8) {
      hist_kernel<<<grid_for(E), 256, 0, st>>>(counts, E, shift, s);
      TG_LAUNCHED();
      pick_digit_kernel<<<1, 32, 0, st>>>(shift, s);
      TG_LAUNCHED();
    }
  }
  overlap_kernel<<<grid_for(E), 256, 0, st>>>(counts, slot_of, E, s, use_threshold, dev, sel_mask);
  TG_LAUNCHED();
  TG_CUDA(cudaMemcpyAsync(host_ov, dev, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaFreeAsync(dev, st));
  TG_CUDA(cudaFreeAsync(s, st));
  TG_CUDA(cudaStreamSynchronize(st));
  return TG_OK;
}

}  // namespace tg

using namespace tg;

extern "C" int tg_cache_replace(const tg_cache_dev* cache, int64_t k, int64_t epsilon, const tg_feat_store* store,
                                float* hot, int64_t hot_ld, int64_t* host_out, void* stream) {
  if (cache == nullptr || cache->slot_of == nullptr || cache->counters == nullptr)
    return fail(TG_EVALUE, "cache state required");
  const int64_t E = cache->num_edges;
  const cudaStream_t st = as_stream(stream);
  uint8_t* sel = nullptr;
  if (E > 0) TG_CUDA(cudaMallocAsync(&sel, E, st));
  unsigned long long ov[2] = {0, 0};
  if (E > 0) {
    const int rc = select_topk(cache->counters, cache->slot_of, E, k, sel, ov, st);
    if (rc != TG_OK) return rc;
  }
  const bool replaced = (long long)ov[0] < epsilon;
  if (replaced && E > 0) {
    int32_t *flags = nullptr, *scan = nullptr;
    TG_CUDA(cudaMallocAsync(&flags, E * sizeof(int32_t), st));
    TG_CUDA(cudaMallocAsync(&scan, E * sizeof(int32_t), st));
    flag_kernel<<<grid_for(E), 256, 0, st>>>(sel, E, flags);
    TG_LAUNCHED();
    size_t tmp_bytes = 0;
    TG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags, scan, E, st));
    void* tmp = nullptr;
    TG_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    TG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags, scan, E, st));
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    assign_kernel<<<grid_for(E), 256, 0, st>>>(sel, scan, E, cache->slot_of);
    TG_LAUNCHED();
    TG_CUDA(cudaFreeAsync(tmp, st));
    TG_CUDA(cudaFreeAsync(flags, st));
    TG_CUDA(cudaFreeAsync(scan, st));
    if (hot != nullptr && store != nullptr && store->d > 0) {
      refill_kernel<<<grid_for(E * 32), 256, 0, st>>>(cache->slot_of, E, *store, hot, hot_ld);
      TG_LAUNCHED();
    }
  }
  if (sel) TG_CUDA(cudaFreeAsync(sel, st));
  if (E > 0) TG_CUDA(cudaMemsetAsync(cache->counters, 0, E * sizeof(int32_t), st));
  if (cache->stats) TG_CUDA(cudaMemsetAsync(cache->stats, 0, 2 * sizeof(unsigned long long), st));
  TG_CUDA(cudaStreamSynchronize(st));
  host_out[0] = replaced ? 1 : 0;
  host_out[1] = (int64_t)ov[0];
  host_out[2] = 0;
  host_out[3] = (int64_t)ov[1];
  return TG_OK;
}

extern "C" int tg_topk_mask(const int32_t* counts, int64_t E, int64_t k, uint8_t* topk_mask, int64_t* host_selected,
                            void* stream) {
  unsigned long long ov[2] = {0, 0};
  if (E > 0) {
    const int rc = select_topk(counts, nullptr, E, k, topk_mask, ov, as_stream(stream));
    if (rc != TG_OK) return rc;
  }
  *host_selected = (int64_t)ov[1];
  return TG_OK;
}
