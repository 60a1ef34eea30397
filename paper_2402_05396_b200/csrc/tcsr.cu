// K1: device T-CSR construction.  Replaces graph.py:94-152 (build_graph).
//
// Reference: stable argsort of the events by ts (graph.py:112), eids
// reassigned in that order (graph.py:131), every event duplicated into both
// endpoints' lists and np.lexsort((eid, ts, node)) (graph.py:133-137),
// offsets = cumsum(bincount(node)) (graph.py:139-141).
//
// Device plan:
//   1. ts keys -> order-preserving uint64 (ts >= 0 after validation, -0.0
//      canonicalised to +0.0 so it ties with +0.0 like np.argsort), stable
//      LSD radix sort of (key, index) -> `order` (skipped when ts is already
//      non-decreasing: the stable order is then the identity).
//   2. events gathered into eid order.
//   3. entry k = 2*eid + side (side 0: src list, 1: dst list) keyed by its
//      node; a stable radix sort over ceil(log2 V) bits puts each node's
//      entries in eid order.  Because eids follow the stable ts order,
//      (eid) order == (ts, eid) order, which is the reference lexsort; the
//      only (node, ts, eid) ties are the two copies of a self-loop, and they
//      are identical.
//   4. offsets[v] = first sorted position with node >= v, written by one
//      pass over the sorted keys (no histogram atomics: a Zipf hub would
//      serialise them).
#include <cub/cub.cuh>

#include "common.cuh"

namespace tg {

__global__ void check_kernel(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                             const double* __restrict__ ts, int64_t E, unsigned long long* info) {
  // info[0] flags: 1 non-finite ts, 2 negative ts, 4 negative node, 8 unsorted
  // info[1] max node (as unsigned, nodes >= 0 when flag 4 is clear)
  unsigned flags = 0;
  long long mx = -1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = ts[i];
    if (!isfinite(t)) flags |= 1;
    if (t < 0.0) flags |= 2;
    const int64_t s = src[i], d = dst[i];
    if (s < 0 || d < 0) flags |= 4;
    mx = max(mx, (long long)max(s, d));
    if (i + 1 < E && !(ts[i + 1] >= t)) flags |= 8;
  }
  for (int o = 16; o > 0; o >>= 1) {
    flags |= __shfl_xor_sync(FULL, flags, o);
    mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (flags) atomicOr(reinterpret_cast<unsigned*>(info), flags);
    if (mx >= 0) atomicMax(reinterpret_cast<long long*>(info + 1), mx);
  }
}

__global__ void ts_keys_kernel(const double* __restrict__ ts, int64_t E, unsigned long long* __restrict__ keys,
                               int64_t* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = ts[i];
    keys[i] = t == 0.0 ? 0ull : static_cast<unsigned long long>(__double_as_longlong(t));
    idx[i] = i;
  }
}

__global__ void iota_kernel(int64_t* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

__global__ void permute_events_kernel(const int64_t* __restrict__ order, const int64_t* __restrict__ src,
                                      const int64_t* __restrict__ dst, const double* __restrict__ ts, int64_t E,
                                      int64_t* __restrict__ src_s, int64_t* __restrict__ dst_s,
                                      double* __restrict__ ts_s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = order ? order[i] : i;
    src_s[i] = src[o];
    dst_s[i] = dst[o];
    ts_s[i] = ts[o];
  }
}

__global__ void entry_keys_kernel(const int64_t* __restrict__ src_s, const int64_t* __restrict__ dst_s, int64_t E,
                                  uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t n = 2 * E;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = k >> 1;
    keys[k] = static_cast<uint32_t>((k & 1) ? dst_s[e] : src_s[e]);
    vals[k] = static_cast<int32_t>(k);
  }
}

__global__ void fill_adj_kernel(const int32_t* __restrict__ vals, const int64_t* __restrict__ src_s,
                                const int64_t* __restrict__ dst_s, const double* __restrict__ ts_s, int64_t n,
                                int32_t* __restrict__ nbr, double* __restrict__ adj_ts, int32_t* __restrict__ adj_eid) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = vals[p];
    const int64_t e = k >> 1;
    nbr[p] = static_cast<int32_t>((k & 1) ? src_s[e] : dst_s[e]);
    adj_ts[p] = ts_s[e];
    adj_eid[p] = static_cast<int32_t>(e);
  }
}

__global__ void offsets_kernel(const uint32_t* __restrict__ keys, int64_t n, int64_t V, int64_t* __restrict__ offsets) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = p > 0 ? (int64_t)keys[p - 1] : -1;
    const int64_t cur = p < n ? (int64_t)keys[p] : V;
    for (int64_t v = prev + 1; v <= cur; ++v) offsets[v] = p;
  }
}

static int grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  const int64_t cap = (int64_t)device_sms() * 16;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace tg

using namespace tg;

extern "C" int tg_tcsr_check(const int64_t* src, const int64_t* dst, const double* ts, int64_t E, int64_t* host_info,
                             void* stream) {
  if (E < 0) return fail(TG_EVALUE, "negative event count");
  host_info[0] = -1;
  host_info[1] = 1;
  if (E == 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  unsigned long long* info = nullptr;
  TG_CUDA(cudaMallocAsync(&info, 2 * sizeof(unsigned long long), st));
  const unsigned long long init[2] = {0ull, static_cast<unsigned long long>(-1ll)};
  TG_CUDA(cudaMemcpyAsync(info, init, sizeof(init), cudaMemcpyHostToDevice, st));
  check_kernel<<<grid_for(E), 256, 0, st>>>(src, dst, ts, E, info);
  TG_LAUNCHED();
  unsigned long long h[2];
  TG_CUDA(cudaMemcpyAsync(h, info, sizeof(h), cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaFreeAsync(info, st));
  TG_CUDA(cudaStreamSynchronize(st));
  const unsigned flags = static_cast<unsigned>(h[0]);
  if (flags & 1) return fail(TG_EDATA, "non-finite timestamp");
  if (flags & 2) return fail(TG_EDATA, "negative timestamp");
  if (flags & 4) return fail(TG_EDATA, "negative node id");
  host_info[0] = static_cast<int64_t>(h[1]);
  host_info[1] = (flags & 8) ? 0 : 1;
  return TG_OK;
}

extern "C" int tg_tcsr_build(const int64_t* src, const int64_t* dst, const double* ts, int64_t E, int64_t V,
                              int32_t ts_sorted, int64_t* order, int64_t* src_s, int64_t* dst_s, double* ts_s,
                              int64_t* offsets, int32_t* nbr, double* adj_ts, int32_t* adj_eid, void* stream) {
  if (E < 0 || V < 0) return fail(TG_EVALUE, "negative sizes");
  if (2 * E >= (int64_t)INT32_MAX) return fail(TG_EVALUE, "2E=%lld exceeds the int32 adjacency index", (long long)(2 * E));
  if (V >= (int64_t)INT32_MAX) return fail(TG_EVALUE, "V exceeds int32 node ids");
  const cudaStream_t st = as_stream(stream);
  const int64_t n = 2 * E;
  // 1. stable ts order
  int64_t* ord = order;
  bool own_order = false;
  if (E > 0 && !ts_sorted) {
    if (ord == nullptr) {
      TG_CUDA(cudaMallocAsync(&ord, E * sizeof(int64_t), st));
      own_order = true;
    }
    unsigned long long *k_in = nullptr, *k_out = nullptr;
    int64_t* v_in = nullptr;
    TG_CUDA(cudaMallocAsync(&k_in, E * sizeof(unsigned long long), st));
    TG_CUDA(cudaMallocAsync(&k_out, E * sizeof(unsigned long long), st));
    TG_CUDA(cudaMallocAsync(&v_in, E * sizeof(int64_t), st));
    ts_keys_kernel<<<grid_for(E), 256, 0, st>>>(ts, E, k_in, v_in);
    TG_LAUNCHED();
    size_t tmp_bytes = 0;
    TG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, v_in, ord, E, 0, 64, st));
    void* tmp = nullptr;
    TG_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    TG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, v_in, ord, E, 0, 64, st));
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    TG_CUDA(cudaFreeAsync(tmp, st));
    TG_CUDA(cudaFreeAsync(k_in, st));
    TG_CUDA(cudaFreeAsync(k_out, st));
    TG_CUDA(cudaFreeAsync(v_in, st));
  } else if (order != nullptr && E > 0) {
    iota_kernel<<<grid_for(E), 256, 0, st>>>(order, E);
    TG_LAUNCHED();
    ord = nullptr;  // identity
  } else {
    ord = nullptr;
  }
  // 2. events in eid order
  if (E > 0) {
    permute_events_kernel<<<grid_for(E), 256, 0, st>>>(ord, src, dst, ts, E, src_s, dst_s, ts_s);
    TG_LAUNCHED();
  }
  if (own_order) TG_CUDA(cudaFreeAsync(ord, st));
  // 3. stable node sort of the 2E entries
  uint32_t *kk = nullptr, *kk_out = nullptr;
  int32_t *vv = nullptr, *vv_out = nullptr;
  if (n > 0) {
    TG_CUDA(cudaMallocAsync(&kk, n * sizeof(uint32_t), st));
    TG_CUDA(cudaMallocAsync(&kk_out, n * sizeof(uint32_t), st));
    TG_CUDA(cudaMallocAsync(&vv, n * sizeof(int32_t), st));
    TG_CUDA(cudaMallocAsync(&vv_out, n * sizeof(int32_t), st));
    entry_keys_kernel<<<grid_for(n), 256, 0, st>>>(src_s, dst_s, E, kk, vv);
    TG_LAUNCHED();
    int bits = 1;
    while (bits < 32 && ((int64_t)1 << bits) < V) ++bits;
    size_t tmp_bytes = 0;
    TG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kk, kk_out, vv, vv_out, n, 0, bits, st));
    void* tmp = nullptr;
    TG_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    TG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kk, kk_out, vv, vv_out, n, 0, bits, st));
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    TG_CUDA(cudaFreeAsync(tmp, st));
    fill_adj_kernel<<<grid_for(n), 256, 0, st>>>(vv_out, src_s, dst_s, ts_s, n, nbr, adj_ts, adj_eid);
    TG_LAUNCHED();
  }
  // 4. offsets
  offsets_kernel<<<grid_for(n + 1), 256, 0, st>>>(kk_out, n, V, offsets);
  TG_LAUNCHED();
  if (n > 0) {
    TG_CUDA(cudaFreeAsync(kk, st));
    TG_CUDA(cudaFreeAsync(kk_out, st));
    TG_CUDA(cudaFreeAsync(vv, st));
    TG_CUDA(cudaFreeAsync(vv_out, st));
  }
  return TG_OK;
}

// ---- coarse time index (tg_graph.coarse_*): every 2^shift-th timestamp of
// each node's adjacency list.  For GDELT (382.6M entries, shift 6) it is
// 6M doubles = 48 MB -- L2-resident -- so a hub's pivot search probes L2
// and then sweeps one 64-entry block in HBM (find.cu).
namespace tg {

__global__ void __launch_bounds__(1024) coarse_off_kernel(const int64_t* __restrict__ off, int64_t V, int shift,
                                                          int64_t* __restrict__ coff) {
  // single block: per-thread contiguous node ranges, block-wide exclusive scan
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (V + 1023) / 1024;
  const int64_t a = t * per < V ? t * per : V, b = (t + 1) * per < V ? (t + 1) * per : V;
  const int64_t mask = (int64_t(1) << shift) - 1;
  int64_t s = 0;
  for (int64_t v = a; v < b; ++v) s += (off[v + 1] - off[v] + mask) >> shift;
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t x = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += x;
    __syncthreads();
  }
  int64_t run = part[t] - s;  // exclusive prefix of this thread's range
  for (int64_t v = a; v < b; ++v) {
    coff[v] = run;
    run += (off[v + 1] - off[v] + mask) >> shift;
  }
  if (t == 1023) coff[V] = part[1023];
}

__global__ void coarse_fill_kernel(const int64_t* __restrict__ off, const double* __restrict__ ts, int64_t V,
                                   int shift, const int64_t* __restrict__ coff, double* __restrict__ cts) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < V; v += warps) {
    const int64_t lo = off[v], c0 = coff[v], nb = coff[v + 1] - c0;
    for (int64_t i = lane; i < nb; i += 32) cts[c0 + i] = ts[lo + (i << shift)];
  }
}

}  // namespace tg

extern "C" int tg_tcsr_coarse(const tg_graph* g, int32_t shift, int64_t* coarse_off, double* coarse_ts,
                              void* stream) {
  using namespace tg;
  if (g == nullptr || coarse_off == nullptr || coarse_ts == nullptr) return fail(TG_EVALUE, "tg_tcsr_coarse: null");
  if (shift < 1 || shift > 16) return fail(TG_EVALUE, "coarse shift %d outside [1, 16]", shift);
  const cudaStream_t st = as_stream(stream);
  coarse_off_kernel<<<1, 1024, 0, st>>>(g->offsets, g->num_nodes, shift, coarse_off);
  TG_LAUNCHED();
  const int64_t want = (g->num_nodes * 32 + 255) / 256;
  const int grid = (int)(want < 65535 ? (want > 0 ? want : 1) : 65535);
  coarse_fill_kernel<<<grid, 256, 0, st>>>(g->offsets, g->adj_ts, g->num_nodes, shift, coarse_off, coarse_ts);
  TG_LAUNCHED();
  return TG_OK;
}
