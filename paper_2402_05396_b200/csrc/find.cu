// K2 + K3 (+ K4/K5): temporal neighbor finding fused with materialisation,
// hop expansion and the cached edge-feature slice.
//
// Replaces finder.py:85-149 (_batch_kernel), finder.py:162-179
// (batch_find_arrays), training.py:246-252 (materialise ids/ts/eids/dts),
// training.py:311-314 (next-hop queries) and training.py:207-221 +
// cache.py:72-86 (feature rows through the cache).
//
// One warp per query.  The pivot (count of entries with ts < t,
// finder.py:69-77) is found by a 32-ary search: the 32 lanes probe 32 evenly
// spaced timestamps, __ballot_sync gives the prefix of probes below t, and
// the range shrinks 33x per round; once it is <= 128 entries one coalesced
// sweep counts the rest.  A 22,934-entry window (GDELT mean degree) takes two
// probe rounds + one sweep instead of 15 dependent binary-search loads.
//
// Uniform selection reproduces the reference's sequential rejection sampler
// bit-for-bit: draw k of row i is splitmix64(mix(seed ^ i*STREAM) + k*GOLDEN)
// (finder.py:99-105); the warp evaluates draws k..k+31 at once and accepts,
// in draw order, the first ones that are new (ballot + popc prefix), so the
// accepted set equals the sequential one.
#include "rows.cuh"

namespace tg {

constexpr int kFindWarps = 8;  // warps per block

// #{i in [lo, hi) : ts[i] < t} over the warp, U loads per lane issued
// together per pass (one memory latency per 32*U entries)
template <int U>
__device__ __forceinline__ int64_t warp_count_below(const double* __restrict__ ts, int64_t lo, int64_t hi, double t,
                                                    int lane) {
  int below = 0;
  for (int64_t base = lo; base < hi; base += 32 * U) {
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + lane + 32 * u;
      x[u] = i < hi ? ts[i] : t;  // past the range: not below
    }
#pragma unroll
    for (int u = 0; u < U; ++u) below += x[u] < t;
  }
  return warp_sum(below);
}

// First index in [lo, hi) whose ts is not < t (numpy/finder strict-< pivot).
__device__ __forceinline__ int64_t warp_pivot(const double* __restrict__ ts, int64_t lo, int64_t hi,
                                              double t, int lane) {
  while (hi - lo > 128) {
    const int64_t n = hi - lo;
    const int64_t pos = lo + (n * (lane + 1)) / 33;
    const bool below = ts[pos] < t;
    const int c = __popc(__ballot_sync(FULL, below));  // probes 0..c-1 are < t
    const int64_t nlo = c > 0 ? lo + (n * c) / 33 + 1 : lo;
    const int64_t nhi = c < 32 ? lo + (n * (c + 1)) / 33 : hi;
    lo = nlo;
    hi = nhi;
  }
  return lo + warp_count_below<4>(ts, lo, hi, t, lane);
}

// `target` distinct offsets in [0, win) in the reference's acceptance order
// (finder.py:100-113 / 122-137).  acc is this warp's shared scratch.
__device__ __forceinline__ void draw_distinct(uint64_t state, uint64_t win, int target,
                                              int32_t* acc, int lane) {
  int cnt = 0;
  uint64_t k0 = 0;
  while (cnt < target) {
    const uint64_t z = draw(state, k0 + lane + 1);
    const int32_t r = static_cast<int32_t>(z % win);
    bool dup = false;
    for (int j = 0; j < cnt; ++j) dup |= acc[j] == r;
#pragma unroll
    for (int s = 1; s < 32; ++s) {
      const int32_t o = __shfl_up_sync(FULL, r, s);
      dup |= (lane >= s) & (o == r);
    }
    const unsigned fresh = __ballot_sync(FULL, !dup);
    const int rank = __popc(fresh & ((1u << lane) - 1u));
    const int need = target - cnt;
    if (!dup && rank < need) acc[cnt + rank] = r;
    cnt += min(__popc(fresh), need);
    k0 += 32;
    __syncwarp();
  }
}

#ifndef TG_FIND_MINB
#define TG_FIND_MINB 6  // resident blocks per SM for the recent policy
#endif
// Up to kMaxFindBatch query batches of one layer (same m / policy) in one
// launch: several mini-batches' finders become one grid instead of a chain
// of small, latency-bound launches (a 1/8 root shard of a GDELT batch is
// only 225 + 2,475 queries).  Query gi belongs to batch b with q0[b] <= gi
// < q0[b+1] and is row gi - q0[b] of that batch's arguments.
constexpr int kMaxFindBatch = 16;
struct FindBatch {
  tg_find_args a[kMaxFindBatch];
  int64_t q0[kMaxFindBatch + 1];
  int nb;
};

#ifndef TG_FIND_MINB_U
#define TG_FIND_MINB_U 4  // resident blocks per SM for the uniform policy
#endif
template <bool UNIFORM>
__global__ void __launch_bounds__(kFindWarps * 32, UNIFORM ? TG_FIND_MINB_U : TG_FIND_MINB)
    find_kernel(tg_graph g, const __grid_constant__ FindBatch fb, tg_cache_dev cache, int has_cache) {
  extern __shared__ int32_t smem[];
  __shared__ unsigned long long red_valid[kMaxFindBatch];
  if (threadIdx.x < kMaxFindBatch) red_valid[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // through a lane-0 shuffle: provably warp-uniform, so the query loop and the
  // ballots / shuffles in it compile without divergence (WARPSYNC) fallbacks
  const int warp = __shfl_sync(FULL, (int)(threadIdx.x >> 5), 0);
  const int m = fb.a[0].m;
  int32_t* acc = smem + warp * 2 * m;  // draws (uniform)
  int32_t* out = acc + m;              // sorted selection (uniform)

  unsigned long long hits = 0, misses = 0;
  const int64_t total = fb.q0[fb.nb];

  for (int64_t gi = (int64_t)blockIdx.x * kFindWarps + warp; gi < total;
       gi += (int64_t)gridDim.x * kFindWarps) {
    int bi = 0;
    while (bi + 1 < fb.nb && gi >= fb.q0[bi + 1]) ++bi;
    const tg_find_args& a = fb.a[bi];
    const int64_t i = gi - fb.q0[bi];
    const uint64_t seed = a.seed_ptr ? *a.seed_ptr : a.seed;
    const int64_t v = a.qv[i];
    const double t = a.qt[i];
    int64_t lo = 0, hi = 0, c0 = 0, c1 = 0;
    if (v >= 0 && v < g.num_nodes) {  // the list bounds and the coarse bounds in one round
      lo = g.offsets[v];
      hi = g.offsets[v + 1];
      if (g.coarse_ts != nullptr) {
        c0 = g.coarse_off[v];
        c1 = g.coarse_off[v + 1];
      }
    }
    int64_t p;
    if (g.coarse_ts != nullptr && hi - lo > 128) {
      // coarse index: c = #{i : ts[lo + (i << s)] < t} (L2: one counting pass
      // for up to 512 coarse entries, i.e. windows up to 32k), then the pivot
      // lies in (lo + ((c-1) << s), lo + (c << s)]: one sweep of < 2^s HBM
      // entries.  Same strict-< count as the plain search.
      const int64_t c = c1 - c0 <= 512 ? warp_count_below<16>(g.coarse_ts, c0, c1, t, lane)
                                        : warp_pivot(g.coarse_ts, c0, c1, t, lane) - c0;
      if (c == 0) {
        p = lo;
      } else {
        const int64_t a = lo + ((c - 1) << g.coarse_shift) + 1;
        const int64_t b = lo + (c << g.coarse_shift) < hi ? lo + (c << g.coarse_shift) : hi;
        p = warp_pivot(g.adj_ts, a, b, t, lane);
      }
    } else {
      p = warp_pivot(g.adj_ts, lo, hi, t, lane);
    }
    const int64_t win = p - lo;
    int cnt;
    bool sorted_in_smem = false;
    if (!UNIFORM || win <= m) {
      cnt = static_cast<int>(win < m ? win : m);
    } else {
      cnt = m;
      sorted_in_smem = true;
      const uint64_t state = mix64(seed ^ (static_cast<uint64_t>(global_row(a.rows, i)) * STREAM));
      if (2 * static_cast<int64_t>(m) <= win) {
        draw_distinct(state, static_cast<uint64_t>(win), m, acc, lane);
        // insertion sort descending (finder.py:115-121) == rank by larger count
        for (int j = lane; j < m; j += 32) {
          const int32_t x = acc[j];
          int rank = 0;
          for (int q = 0; q < m; ++q) rank += acc[q] > x;
          out[rank] = x;
        }
      } else {
        const int nex = static_cast<int>(win) - m;
        draw_distinct(state, static_cast<uint64_t>(win), nex, acc, lane);
        // emit the window descending, skipping exclusions (finder.py:138-147)
        int k = 0;
        for (int64_t c0 = 0; c0 < win; c0 += 32) {
          const int64_t r = win - 1 - (c0 + lane);
          bool keep = r >= 0;
          if (keep)
            for (int q = 0; q < nex; ++q) keep &= acc[q] != static_cast<int32_t>(r);
          const unsigned km = __ballot_sync(FULL, keep);
          if (keep) out[k + __popc(km & ((1u << lane) - 1u))] = static_cast<int32_t>(r);
          k += __popc(km);
        }
      }
      __syncwarp();
    }
    if (lane == 0) atomicAdd(&red_valid[bi], (unsigned long long)cnt);

    // materialise slots lane, lane+32, ... (training.py:246-252) and the
    // next-hop queries (training.py:311-314); count cache accesses
    for (int g0 = 0; g0 < m; g0 += 32) {
      const int j = g0 + lane;
      const bool in_row = j < m;
      const bool valid = j < cnt;
      int64_t pos = -1;
      if (valid) pos = sorted_in_smem ? lo + out[j] : p - 1 - j;
      int64_t nb = 0, e = 0;
      double ets = 0.0, dt = 0.0;
      if (valid) {
        nb = g.nbr[pos];
        ets = g.adj_ts[pos];
        e = g.adj_eid[pos];
        dt = __dsub_rn(t, ets);
      }
      const int64_t o = i * m + j;
      if (in_row) {
        if (a.idx) a.idx[o] = pos;
        if (a.ids) a.ids[o] = nb;
        if (a.eids) a.eids[o] = e;
        if (a.dts) a.dts[o] = dt;
        if (a.tss) a.tss[o] = ets;
        if (a.mask) a.mask[o] = valid ? 1 : 0;
        if (a.next_v) {
          a.next_v[a.B + o] = nb;
          a.next_t[a.B + o] = __dsub_rn(t, dt);
        }
      }
      if (has_cache) {
        int32_t slot = -1;
        if (valid) {
          slot = cache.slot_of[e];
          atomicAdd(cache.counters + e, 1);
        }
        hits += __popc(__ballot_sync(FULL, valid && slot >= 0));
        misses += __popc(__ballot_sync(FULL, valid && slot < 0));
      }
    }
    if (lane == 0) {
      if (a.cnt) a.cnt[i] = cnt;
      if (a.window) a.window[i] = win;
      if (a.next_v) {
        a.next_v[i] = v;
        a.next_t[i] = t;
      }
    }
    __syncwarp();
  }

  // block-aggregate the counters, then one atomic per block (and batch)
  __shared__ unsigned long long red[2];
  if (threadIdx.x < 2) red[threadIdx.x] = 0;
  __syncthreads();
  if (lane == 0 && has_cache) {
    atomicAdd(&red[0], hits);
    atomicAdd(&red[1], misses);
  }
  __syncthreads();
  if (threadIdx.x == 0 && has_cache) {
    if (red[0]) atomicAdd(cache.stats + 0, red[0]);
    if (red[1]) atomicAdd(cache.stats + 1, red[1]);
  }
  if (threadIdx.x < fb.nb && fb.a[threadIdx.x].valid_count && red_valid[threadIdx.x])
    atomicAdd(fb.a[threadIdx.x].valid_count, red_valid[threadIdx.x]);
}

template <bool UNIFORM>
static int launch_find(const tg_graph& g, const FindBatch& fb, const tg_cache_dev& cache, int has_cache,
                       cudaStream_t st) {
  const size_t smem = UNIFORM ? (size_t)kFindWarps * 2 * fb.a[0].m * sizeof(int32_t) : 0;
  auto kern = find_kernel<UNIFORM>;
  if (smem > 48 * 1024) TG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // the same shared-memory carveout as the K5 gathers that run beside it, so
  // its CTAs can join SMs holding gather CTAs instead of waiting for a
  // differently configured SM (measured: the uniform finder waited out
  // whole gathers on B)
  static const bool carve = getenv("TG_FIND_NO_CARVEOUT") == nullptr;
  if (carve) TG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          (int)cudaSharedmemCarveoutMaxShared));
  const int64_t total = fb.q0[fb.nb];
  const int64_t want = (total + kFindWarps - 1) / kFindWarps;
  const int64_t cap = (int64_t)device_sms() * 16;
  const int grid = (int)(want < cap ? want : cap);
  kern<<<grid, kFindWarps * 32, smem, st>>>(g, fb, cache, has_cache);
  TG_LAUNCHED();
  return TG_OK;
}

static int check_find_args(const tg_find_args* a) {
  if (a->m < 1) return fail(TG_EVALUE, "budget m must be >= 1");
  if (a->m > 2048) return fail(TG_EVALUE, "budget m=%d exceeds the device limit 2048", a->m);
  if (a->policy != TG_RECENT && a->policy != TG_UNIFORM) return fail(TG_EVALUE, "unknown policy %d", a->policy);
  if (a->B < 0) return fail(TG_EVALUE, "negative batch");
  if ((a->next_v == nullptr) != (a->next_t == nullptr)) return fail(TG_EVALUE, "next_v/next_t must be given together");
  return TG_OK;
}

}  // namespace tg

using namespace tg;

extern "C" int tg_find(const tg_graph* g, const tg_find_args* a, const tg_feat_store* store,
                       const tg_cache_dev* cache, void* stream) {
  if (!g || !a) return fail(TG_EVALUE, "tg_find: null graph/args");
  if (a->m < 1) return fail(TG_EVALUE, "budget m must be >= 1");
  if (a->m > 2048) return fail(TG_EVALUE, "budget m=%d exceeds the device limit 2048", a->m);
  if (a->policy != TG_RECENT && a->policy != TG_UNIFORM)
    return fail(TG_EVALUE, "unknown policy %d", a->policy);
  if (a->B < 0) return fail(TG_EVALUE, "negative batch");
  if ((a->next_v == nullptr) != (a->next_t == nullptr))
    return fail(TG_EVALUE, "next_v/next_t must be given together");
  if (a->feat_out != nullptr && store == nullptr) return fail(TG_EVALUE, "feat_out needs a store");
  if (a->B == 0) return TG_OK;
  const int has_feat = a->feat_out != nullptr && store->d > 0;
  tg_cache_dev cd{};
  const int has_cache = cache != nullptr && cache->slot_of != nullptr;
  if (has_cache) cd = *cache;
  const cudaStream_t st = as_stream(stream);
  tg_find_args args = *a;
  // the feature slice reads eids + mask back: keep them in temporaries when
  // the caller did not ask for them
  int64_t* tmp_eids = nullptr;
  uint8_t* tmp_mask = nullptr;
  if (has_feat && args.eids == nullptr) {
    TG_CUDA(cudaMallocAsync(&tmp_eids, (size_t)args.B * args.m * sizeof(int64_t), st));
    args.eids = tmp_eids;
  }
  if (has_feat && args.mask == nullptr) {
    TG_CUDA(cudaMallocAsync(&tmp_mask, (size_t)args.B * args.m, st));
    args.mask = tmp_mask;
  }
  FindBatch fb{};
  fb.a[0] = args;
  fb.q0[0] = 0;
  fb.q0[1] = args.B;
  fb.nb = 1;
  int rc = args.policy == TG_UNIFORM ? launch_find<true>(*g, fb, cd, has_cache, st)
                                     : launch_find<false>(*g, fb, cd, has_cache, st);
  if (rc == TG_OK && has_feat)
    rc = launch_row_gather(args.eids, args.mask, args.B * args.m, *store, has_cache ? cd.slot_of : nullptr,
                           ROW_ZERO, args.feat_out, args.feat_ld, st);
  if (tmp_eids) TG_CUDA(cudaFreeAsync(tmp_eids, st));
  if (tmp_mask) TG_CUDA(cudaFreeAsync(tmp_mask, st));
  return rc;
}

extern "C" int tg_find_batch(const tg_graph* g, const tg_find_args* args, int32_t nb, const tg_cache_dev* cache,
                             void* stream) {
  if (!g || (nb > 0 && !args)) return fail(TG_EVALUE, "tg_find_batch: null graph/args");
  if (nb < 0) return fail(TG_EVALUE, "negative batch count");
  const cudaStream_t st = as_stream(stream);
  tg_cache_dev cd{};
  const int has_cache = cache != nullptr && cache->slot_of != nullptr;
  if (has_cache) cd = *cache;
  for (int b = 0; b < nb; ++b) {
    const int rc = check_find_args(args + b);
    if (rc != TG_OK) return rc;
    if (args[b].feat_out != nullptr) return fail(TG_EVALUE, "tg_find_batch: feat_out is not supported (use K5)");
    if (args[b].m != args[0].m || args[b].policy != args[0].policy)
      return fail(TG_EVALUE, "tg_find_batch: every batch needs the same m and policy");
  }
  for (int b0 = 0; b0 < nb; b0 += kMaxFindBatch) {
    FindBatch fb{};
    fb.q0[0] = 0;
    for (int k = 0; k < kMaxFindBatch && b0 + k < nb; ++k) {
      fb.a[fb.nb] = args[b0 + k];
      fb.q0[fb.nb + 1] = fb.q0[fb.nb] + args[b0 + k].B;
      ++fb.nb;
    }
    if (fb.q0[fb.nb] == 0) continue;
    const int rc = args[0].policy == TG_UNIFORM ? launch_find<true>(*g, fb, cd, has_cache, st)
                                                : launch_find<false>(*g, fb, cd, has_cache, st);
    if (rc != TG_OK) return rc;
  }
  return TG_OK;
}
