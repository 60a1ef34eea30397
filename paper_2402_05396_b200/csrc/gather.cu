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
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rows.cuh"
#include "tc_gemm.cuh"

namespace tg {

// ---- per-slot cache accounting (cache.py:78-82): counters, hits/misses.
__global__ void count_kernel(const int64_t* __restrict__ ids, const uint8_t* __restrict__ mask, int64_t n,
                             tg_cache_dev cache, uint8_t* __restrict__ hits_out) {
  unsigned long long hits = 0, misses = 0;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool in_range = i < n;
    const bool valid = in_range && (mask == nullptr || mask[i] != 0);
    int32_t slot = -1;
    if (valid) {
      const int64_t r = ids[i];
      slot = cache.slot_of[r];
      atomicAdd(cache.counters + r, 1);
    }
    if (hits_out && in_range) hits_out[i] = slot >= 0 ? 1 : 0;
    hits += __popc(__ballot_sync(FULL, valid && slot >= 0));
    misses += __popc(__ballot_sync(FULL, valid && slot < 0));
  }
  __shared__ unsigned long long red[2];
  if (threadIdx.x < 2) red[threadIdx.x] = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&red[0], hits);
    atomicAdd(&red[1], misses);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (red[0]) atomicAdd(cache.stats + 0, red[0]);
    if (red[1]) atomicAdd(cache.stats + 1, red[1]);
  }
}

// ---- row gather (K5).  A block takes a tile of ROWS rows: ROWS threads
// resolve the rows' sources once (mask, id, cache slot -> tier pointer) into
// shared memory, then all 256 threads stream the tile as a flat sequence of
// VEC-float units (unit u = row u/nv, column u%nv), so consecutive threads
// touch consecutive 8/16-byte words of each 688/744-byte source row and the
// output block is written contiguously.  Each thread issues UNR loads before
// its first store.  Per-unit cost is one smem read, a reciprocal-multiply
// division and the load/store pair -- the per-row work is hoisted.
template <int VEC, int ROWS, int UNR>
__global__ void __launch_bounds__(256) row_gather_kernel(const int64_t* __restrict__ ids,
                                                         const uint8_t* __restrict__ mask, int64_t n, int nv,
                                                         float inv_nv, tg_feat_store fs,
                                                         const int32_t* __restrict__ slot_of, int invalid_mode,
                                                         float* __restrict__ out, int64_t out_ld) {
  using V = typename VecT<VEC>::T;
  // double-buffered tile metadata: tile i+1's (id, mask) loads are issued
  // before tile i's rows are streamed, so their latency hides behind the copy
  __shared__ const V* s_src[2][ROWS];
  __shared__ int s_mode[2][ROWS];
  const int t = threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * ROWS;
  int64_t r0 = (int64_t)blockIdx.x * ROWS;
  int64_t nid = 0;
  int nvalid = 0;
  auto fetch = [&](int64_t base) {
    const int64_t r = base + t;
    if (t < ROWS && r < n) {
      nid = ids[r];
      nvalid = mask == nullptr ? 1 : mask[r];
    }
  };
  fetch(r0);
  for (int buf = 0; r0 < n; r0 += step, buf ^= 1) {
    const int rows = n - r0 < ROWS ? (int)(n - r0) : ROWS;
    if (t < rows) {
      const bool valid = nvalid != 0;
      const V* src = nullptr;
      int mode = ROW_ZERO;
      if (valid || invalid_mode == ROW_TIMES_ZERO) {
        const int32_t slot = (valid && slot_of != nullptr && fs.hot != nullptr) ? slot_of[nid] : -1;
        src = reinterpret_cast<const V*>(row_source(fs, nid, slot));
        mode = valid ? ROW_COPY : ROW_TIMES_ZERO;
      }
      s_src[buf][t] = src;
      s_mode[buf][t] = mode;
    }
    __syncthreads();
    fetch(r0 + step);
    const int units = rows * nv;
    float* dst0 = out + r0 * out_ld;
    for (int u0 = t; u0 < units; u0 += 256 * UNR) {
      V v[UNR];
      int rr[UNR], cc[UNR];
#pragma unroll
      for (int k = 0; k < UNR; ++k) {
        const int u = u0 + k * 256;
        int r = __float2int_rz(__int2float_rn(u) * inv_nv);
        r -= r * nv > u;
        r += (r + 1) * nv <= u;
        rr[k] = u < units ? r : -1;
        cc[k] = u - r * nv;
        v[k] = zero_like(V());
        if (u < units) {
          const int md = s_mode[buf][r];
          if (md != ROW_ZERO) {
            const V x = ld_stream(s_src[buf][r] + cc[k]);
            v[k] = md == ROW_COPY ? x : times_zero(x);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < UNR; ++k)
        if (rr[k] >= 0) reinterpret_cast<V*>(dst0 + (int64_t)rr[k] * out_ld)[cc[k]] = v[k];
    }
  }
}

template <int VEC>
static int launch_row_gather_v(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store& fs, int cw,
                               const int32_t* slot_of, int invalid_mode, float* out, int64_t out_ld, cudaStream_t st) {
  constexpr int ROWS = 64, UNR = 4;
  const int nv = cw / VEC;
  const int64_t tiles = (n + ROWS - 1) / ROWS;
  const int64_t cap = (int64_t)device_sms() * 8;
  const int grid = (int)(tiles < cap ? tiles : cap);
  row_gather_kernel<VEC, ROWS, UNR><<<grid, 256, 0, st>>>(ids, mask, n, nv, 1.0f / (float)nv, fs, slot_of, invalid_mode,
                                                         out, out_ld);
  TG_LAUNCHED();
  return TG_OK;
}

// ---- K5 on the bulk-copy (TMA) engine.  When source and output rows share
// one 16-byte-multiple pitch (the padded layout), a tile of ROWS output rows
// is one contiguous block: lane i bulk-copies source row i (cp.async.bulk
// global->shared, mbarrier complete_tx) -- or zero-fills it for a padded
// slot -- and one bulk store (shared->global) writes the whole tile.  One
// warp per CTA keeps STAGES tiles in flight; the copy engine, not the
// register file, provides the memory-level parallelism.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// Up to kMaxSegs row lists (e.g. every layer of a mini-batch) in ONE launch:
// tile t belongs to the segment whose tile range holds it, so one grid of
// persistent CTAs streams all layers' rows back to back instead of a small
// launch per layer competing with the big one for SM slots.
constexpr int kMaxSegs = 32;  // e.g. 2 layers x 16 mini-batches of one captured step group
struct GatherSegs {
  const int64_t* ids[kMaxSegs];
  const uint8_t* mask[kMaxSegs];
  float* out[kMaxSegs];
  int64_t n[kMaxSegs];
  int64_t tile0[kMaxSegs + 1];  // first tile of each segment; tile0[nseg] = total
  int nseg;
};

template <int ROWS, int STAGES>
__global__ void __launch_bounds__(32) row_gather_bulk_kernel(GatherSegs sg, tg_feat_store fs,
                                                             const int32_t* __restrict__ slot_of, uint32_t rowbytes) {
  extern __shared__ __align__(128) unsigned char sbuf[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sbuf + (size_t)STAGES * ROWS * rowbytes);
  const int lane = threadIdx.x;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) tc::mbar_init(bar + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t ntiles = sg.tile0[sg.nseg];
  const int64_t first = blockIdx.x, step = gridDim.x;
  const int64_t mine = first < ntiles ? (ntiles - first + step - 1) / step : 0;
  // segment and first row of global tile t
  auto locate = [&](int64_t t, int& seg, int64_t& r0) {
    seg = 0;
    while (seg + 1 < sg.nseg && t >= sg.tile0[seg + 1]) ++seg;
    r0 = (t - sg.tile0[seg]) * ROWS;
  };
  auto issue = [&](int64_t k) {  // loads of my k-th tile into stage k % STAGES
    const int stage = (int)(k % STAGES);
    int seg;
    int64_t r0;
    locate(first + k * step, seg, r0);
    const int64_t n = sg.n[seg];
    const uint8_t* mask = sg.mask[seg];
    unsigned char* sb = sbuf + (size_t)stage * ROWS * rowbytes;
    const int64_t r = r0 + lane;
    const bool in = lane < ROWS && r < n;
    const bool valid = in && (mask == nullptr || mask[r] != 0);
    const unsigned vm = __ballot_sync(FULL, valid);
    if (lane == 0) tc::mbar_arrive_expect_tx(bar + stage, (uint32_t)__popc(vm) * rowbytes);
    __syncwarp();
    if (valid) {
      const int64_t id = sg.ids[seg][r];
      const int32_t slot = (slot_of != nullptr && fs.hot != nullptr) ? slot_of[id] : -1;
      tc::bulk_g2s(sb + (size_t)lane * rowbytes, row_source(fs, id, slot), rowbytes, bar + stage);
    } else if (in) {
      float4* z = reinterpret_cast<float4*>(sb + (size_t)lane * rowbytes);
      for (uint32_t i = 0; i < rowbytes / 16; ++i) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  for (int64_t k = 0; k < mine && k < STAGES - 1; ++k) issue(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int stage = (int)(k % STAGES);
    tc::mbar_wait(bar + stage, (uint32_t)((k / STAGES) & 1));
    tc::fence_proxy_async();  // zero-filled rows (generic stores) -> bulk store
    __syncwarp();
    if (lane == 0) {
      int seg;
      int64_t r0;
      locate(first + k * step, seg, r0);
      const int64_t n = sg.n[seg];
      const int rows = n - r0 < ROWS ? (int)(n - r0) : ROWS;
      bulk_s2g(reinterpret_cast<unsigned char*>(sg.out[seg]) + r0 * rowbytes, sbuf + (size_t)stage * ROWS * rowbytes,
               (uint32_t)rows * rowbytes);
      bulk_commit();
    }
    if (k + STAGES - 1 < mine) {
      // refill the stage of tile k-1: its bulk store (the second most recent
      // group) must have finished reading shared memory
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      issue(k + STAGES - 1);
    }
  }
  if (lane == 0) bulk_wait_read<0>();
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// K5 on the tensor engine's row gather (sm_100 `tile::gather4`): one TMA
// instruction moves FOUR table rows, named by their row indices, into shared
// memory, so a 32-row tile is 8 loads instead of 32 -- the engine's per-
// request cost, not bytes, bounded the bulk-copy version (halving the rows
// per request at constant bytes in flight halved its throughput).  Padded
// slots name a row past the table (TMA zero-fills out-of-bounds rows, which
// is the reference's zero row, training.py:218).  Groups of four rows land
// 128-B aligned; a tile is written back with one bulk store per group.
//
// TS (default when every segment fits kMaxTsSegs): the shared tile keeps a
// 128-B-aligned row pitch (the load box is that wide; columns past the row
// read as zero), so each tile goes back with ONE tensor store through a
// per-segment 2-D map of the output (rows past the segment and the pad
// columns are clipped) -- 8 loads + 1 store per 32 rows.
constexpr int G4_ROWS = 32, G4_GROUPS = G4_ROWS / 4;
constexpr int kMaxTsSegs = 8;
struct OutMaps {
  CUtensorMap m[kMaxTsSegs];
};
template <int STAGES, bool TS, int ROWS = G4_ROWS>
__global__ void __launch_bounds__(32) row_gather_g4_kernel(GatherSegs sg, const __grid_constant__ CUtensorMap tm,
                                                           const __grid_constant__ OutMaps om, int32_t oob_row,
                                                           uint32_t rowbytes, uint32_t gstride, int tz, int sh) {
  extern __shared__ __align__(128) unsigned char sbuf[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sbuf + (size_t)STAGES * (ROWS / 4) * gstride);
  const int lane = threadIdx.x;
  uint64_t pol = 0;
  if (sh) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) tc::mbar_init(bar + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t ntiles = sg.tile0[sg.nseg];
  const int64_t first = blockIdx.x, step = gridDim.x;
  const int64_t mine = first < ntiles ? (ntiles - first + step - 1) / step : 0;
  auto locate = [&](int64_t t, int& seg, int64_t& r0) {
    seg = 0;
    while (seg + 1 < sg.nseg && t >= sg.tile0[seg + 1]) ++seg;
    r0 = (t - sg.tile0[seg]) * ROWS;
  };
  auto issue = [&](int64_t k) {
    const int stage = (int)(k % STAGES);
    int seg;
    int64_t r0;
    locate(first + k * step, seg, r0);
    const int64_t n = sg.n[seg];
    const int rows = n - r0 < ROWS ? (int)(n - r0) : ROWS;
    const int64_t r = r0 + lane;
    const uint8_t* mask = sg.mask[seg];
    const bool valid = lane < rows && (mask == nullptr || mask[r] != 0);
    // tz (node rows, training.py:227-229): a padded slot still loads its
    // id's row, made row * 0.0 (signed zeros) in shared memory below
    const int32_t row = (valid || (tz && lane < rows)) ? (int32_t)sg.ids[seg][r] : oob_row;
    const int groups = (rows + 3) >> 2;
    // (TS: a box row is the padded pitch, gstride / 4 bytes)
    if (lane == 0) tc::mbar_arrive_expect_tx(bar + stage, (uint32_t)groups * (TS ? gstride : 4u * rowbytes));
    __syncwarp();
    const int32_t q0 = __shfl_sync(FULL, row, (4 * lane) & 31), q1 = __shfl_sync(FULL, row, (4 * lane + 1) & 31);
    const int32_t q2 = __shfl_sync(FULL, row, (4 * lane + 2) & 31), q3 = __shfl_sync(FULL, row, (4 * lane + 3) & 31);
    if (lane < groups) {
      unsigned char* dst = sbuf + ((size_t)stage * (ROWS / 4) + lane) * gstride;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
          "%3, %4, %5, %6}], [%7];" ::"r"(tc::smem_u32(dst)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(q0), "r"(q1), "r"(q2), "r"(q3),
          "r"(tc::smem_u32(bar + stage))
          : "memory");
    }
  };
  for (int64_t k = 0; k < mine && k < STAGES - 1; ++k) issue(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int stage = (int)(k % STAGES);
    tc::mbar_wait(bar + stage, (uint32_t)((k / STAGES) & 1));
    int seg;
    int64_t r0;
    locate(first + k * step, seg, r0);
    const int64_t n = sg.n[seg];
    const int rows = n - r0 < ROWS ? (int)(n - r0) : ROWS;
    const int groups = (rows + 3) >> 2;
    if (tz) {
      const uint8_t* mask = sg.mask[seg];
      const bool pad = lane < rows && mask != nullptr && mask[r0 + lane] == 0;
      unsigned pm = __ballot_sync(FULL, pad);
      if (pm) {
        unsigned char* sb = sbuf + (size_t)stage * (ROWS / 4) * gstride;
        while (pm) {
          const int j = __ffs(pm) - 1;
          pm &= pm - 1;
          float* w = reinterpret_cast<float*>(
              sb + (TS ? (size_t)j * (gstride / 4) : (size_t)(j >> 2) * gstride + (size_t)(j & 3) * rowbytes));
          for (uint32_t q = lane; q < rowbytes / 4; q += 32) w[q] = w[q] * 0.0f;  // IEEE x * 0.0 (signs, inf, NaN)
        }
        tc::fence_proxy_async();  // generic smem writes -> the store's async-proxy reads
        __syncwarp();
      }
    }
    if constexpr (TS) {
      if (lane == 0) {
        if (sh) {  // the mini-batch rows stream out: evict them first, keep the table's hot rows in L2
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                  reinterpret_cast<uint64_t>(&om.m[seg])),
              "r"(0), "r"((int)r0), "r"(tc::smem_u32(sbuf + (size_t)stage * (ROWS / 4) * gstride)), "l"(pol)
              : "memory");
        } else {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                           reinterpret_cast<uint64_t>(&om.m[seg])),
                       "r"(0), "r"((int)r0), "r"(tc::smem_u32(sbuf + (size_t)stage * (ROWS / 4) * gstride))
                       : "memory");
        }
      }
    } else if (lane < groups) {
      const int nr = rows - 4 * lane < 4 ? rows - 4 * lane : 4;
      bulk_s2g(reinterpret_cast<unsigned char*>(sg.out[seg]) + (r0 + 4 * lane) * rowbytes,
               sbuf + ((size_t)stage * (ROWS / 4) + lane) * gstride, (uint32_t)nr * rowbytes);
    }
    bulk_commit();  // per lane: its own bulk group
    if (k + STAGES - 1 < mine) {
      bulk_wait_read<1>();  // this lane's store of tile k-1 has read its group
      __syncwarp();
      issue(k + STAGES - 1);
    }
  }
  bulk_wait_read<0>();
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

using EncodeTiledG4 = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// gather4 K5 over segments; *handled false when the layout does not allow it
static int launch_g4_segs(const GatherSegs& sg, const tg_feat_store& fs, int tz, int trows, cudaStream_t st,
                          bool* handled) {
  *handled = false;
  static EncodeTiledG4 enc = nullptr;
  if (enc == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      cudaGetLastError();
      return TG_OK;
    }
    enc = reinterpret_cast<EncodeTiledG4>(fn);
  }
  // the rows as 8-byte elements (the copy is bit-for-bit; the type only
  // sizes the box): a box is <= 256 elements, so rows up to 2 KB -- every
  // pitched width up to 512 floats (GDELT 188, MovieLens 268)
  const int64_t rows_total = fs.num_rows > 0 ? fs.num_rows : 0;
  if (rows_total <= 0 || rows_total >= ((int64_t)1 << 31) - 1 || (fs.ld & 1) || fs.ld / 2 > 256) return TG_OK;
  const uint32_t rowbytes = (uint32_t)(fs.ld * 4);
  const uint32_t pitch = (rowbytes + 127) & ~127u;  // TS: smem row pitch
  bool ts = sg.nseg <= kMaxTsSegs && pitch / 8 <= 256 && getenv("TG_K5_G4_BULKSTORE") == nullptr;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  const cuuint32_t estr[2] = {1, 1};
  for (int i = 0; ts && i < sg.nseg; ++i) {
    const cuuint64_t odims[2] = {(cuuint64_t)(fs.ld / 2), (cuuint64_t)sg.n[i]};
    const cuuint64_t ostr[1] = {(cuuint64_t)fs.ld * 4};
    const cuuint32_t obox[2] = {pitch / 8, (cuuint32_t)trows};
    ts = enc(&om.m[i], CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, sg.out[i], odims, ostr, obox, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  CUtensorMap tm;
  // L2 sector promotion of the row loads (TG_K5_G4_PROMO: 0 none, 1 64 B =
  // default, 2 128 B, 3 256 B; read per call: sweeps).  64 B: E's K5 53.1 ->
  // 51.5 us per launch (0.926 -> 0.955 of the copy peak) against 256 B --
  // a 752-B row starting mid-granule drags in up to 504 B it does not use
  // (profiles/r02s5_k5_promotion.md)
  // (A's L2-sized table: 6.3 us per step at 64 B, 6.4 at 256 B -- same box)
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
  if (const char* e = getenv("TG_K5_G4_PROMO")) {
    const int v = atoi(e);
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
            : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
            : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                     : CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)(fs.ld / 2), (cuuint64_t)rows_total};
  const cuuint64_t strides[1] = {(cuuint64_t)fs.ld * 4};
  cuuint32_t box[2] = {ts ? pitch / 8 : (cuuint32_t)(fs.ld / 2), 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<float*>(fs.table), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    if (!ts) return TG_OK;
    ts = false;  // the padded box was refused: per-group stores with the exact box
    box[0] = (cuuint32_t)(fs.ld / 2);
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<float*>(fs.table), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return TG_OK;
  }
  const uint32_t gstride = ts ? 4 * pitch : (4 * rowbytes + 127) & ~127u;
  // tiles per CTA ring: three CTAs per SM beat deeper rings (GDELT rows,
  // profiles/r02s5_k5_stages.md: 3 tiles x 3 CTAs 53.3 us per launch, 4 x 2
  // 56.3, 2 x 4 55.4, 6 x 1 83), so the ring is 3 tiles when three such
  // CTAs fit in shared memory and 2 otherwise (TG_K5_G4_STAGES: 2, 3, 4, 6)
  const int tgroups = trows / 4;
  int g4_stages = 3 * ((size_t)3 * G4_GROUPS * gstride + 24 + 1024) <= 228 * 1024 ? 3 : 2;
  if (const char* e = getenv("TG_K5_G4_STAGES")) {
    const int v = atoi(e);
    if (v == 2 || v == 3 || v == 4 || v == 6) g4_stages = v;
  }
  const size_t smem = (size_t)g4_stages * tgroups * gstride + g4_stages * 8;
  if (smem > 200 * 1024) return TG_OK;
  auto pick = [&](auto st) {
    constexpr int S = decltype(st)::value;
    if (trows == 16) return ts ? row_gather_g4_kernel<S, true, 16> : row_gather_g4_kernel<S, false, 16>;
    return ts ? row_gather_g4_kernel<S, true> : row_gather_g4_kernel<S, false>;
  };
  auto kern = g4_stages == 2   ? pick(std::integral_constant<int, 2>{})
              : g4_stages == 3 ? pick(std::integral_constant<int, 3>{})
              : g4_stages == 6 ? pick(std::integral_constant<int, 6>{})
                               : pick(std::integral_constant<int, 4>{});
  TG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int per_sm = (int)((228 * 1024) / (smem + 1024));
  const int64_t cap = (int64_t)device_sms() * (per_sm > 0 ? per_sm : 1);
  const int64_t t0 = sg.tile0[sg.nseg];
  const int grid = (int)(t0 < cap ? t0 : cap);
  // evict-first tensor stores (TG_K5_STORE_HINT=1, read per call): measured
  // +-0 (E: DRAM reads 116.7 -> 111.8 MB per launch, 53.1 -> 53.0 us; B 50.0
  // -> 50.2 us; profiles/r02s5_k5_store_hint.md), so off by default
  const char* she = getenv("TG_K5_STORE_HINT");
  const int sh = she ? atoi(she) : 0;
  kern<<<grid, 32, smem, st>>>(sg, tm, om, (int32_t)rows_total, rowbytes, gstride, tz, sh);
  TG_LAUNCHED();
  *handled = true;
  return TG_OK;
}

static bool bulk_ok(const tg_feat_store& fs, const int32_t* slot_of, int invalid_mode, const float* out, int64_t out_ld) {
  const int64_t pitch = fs.ld;
  // peer shards (fs.peers) share the pitch and 16-B alignment by contract
  // (taser_b200.h); the bulk engine reads peer-mapped rows over NVLink
  if (invalid_mode != ROW_ZERO) return false;
  if (out_ld != pitch || (pitch * 4) % 16 != 0 || pitch < fs.d) return false;
  if (fs.hot != nullptr && slot_of != nullptr && fs.hot_ld != pitch) return false;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return al(fs.table) && al(out) && (fs.hot == nullptr || al(fs.hot));
}

// Bulk-engine gather of up to kMaxSegs row lists in one launch; *handled is
// false when the layout does not allow it (the caller takes the register path)
static int launch_bulk_segs(const tg_gather_seg* segs, int nseg, const tg_feat_store& fs, const int32_t* slot_of,
                            int invalid_mode, int64_t out_ld, cudaStream_t st, bool* handled) {
  *handled = false;
  if (nseg < 1 || nseg > kMaxSegs || fs.d <= 0 || getenv("TG_K5_REGISTER_PATH") != nullptr) return TG_OK;
  int64_t n = 0;
  // gather4 pays for tables that live in HBM (random rows: the per-request
  // cost bounds the per-row copies -- A's 108 MB, B's 462 MB, C, D's edges,
  // E); a small, L2-resident one (D's 5 MB node table) is faster per row
  // through the per-row paths (measured: D's node-row gathers 61 -> 82 us)
  const char* g4env = getenv("TG_K5_G4_MIN_MB");  // read per call: tests force either path
  const double g4_min = g4env ? atof(g4env) * 1e6 : 32e6;
  bool bulk = true, g4ok = fs.n_peers == 0 && (fs.hot == nullptr || slot_of == nullptr) && fs.table != nullptr &&
                        getenv("TG_K5_NO_G4") == nullptr && (double)fs.num_rows * fs.ld * 4 >= g4_min;
  for (int i = 0; i < nseg; ++i) {
    if (segs[i].n > 0 && !bulk_ok(fs, slot_of, invalid_mode, segs[i].out, out_ld)) bulk = false;
    // gather4 also covers node rows (ROW_TIMES_ZERO): the layout test of the
    // bulk path with the mode check left out
    if (segs[i].n > 0 && !bulk_ok(fs, slot_of, ROW_ZERO, segs[i].out, out_ld)) g4ok = false;
    n += segs[i].n;
  }
  if (n == 0) {
    *handled = true;
    return TG_OK;
  }
  if (!bulk && !(g4ok && invalid_mode == ROW_TIMES_ZERO)) return TG_OK;
  const uint32_t rowbytes = (uint32_t)(fs.ld * 4);
  // the tensor engine's 4-row gather: one table (no hot tier, no peer shards)
  if (g4ok) {
    GatherSegs g4{};
    int64_t tt = 0;
    // rows per tile (TG_K5_G4_ROWS: 16 or 32; read per call: sweeps and tests)
    const char* g4r = getenv("TG_K5_G4_ROWS");
    const int g4_rows = (g4r && atoi(g4r) == 16) ? 16 : G4_ROWS;
    for (int i = 0; i < nseg; ++i) {
      if (segs[i].n <= 0) continue;
      const int k = g4.nseg++;
      g4.ids[k] = segs[i].ids;
      g4.mask[k] = segs[i].mask;
      g4.out[k] = segs[i].out;
      g4.n[k] = segs[i].n;
      g4.tile0[k] = tt;
      tt += (segs[i].n + g4_rows - 1) / g4_rows;
    }
    g4.tile0[g4.nseg] = tt;
    const int rc = launch_g4_segs(g4, fs, invalid_mode == ROW_TIMES_ZERO, g4_rows, st, handled);
    if (rc != TG_OK || *handled) return rc;
  }
  if (!bulk) return TG_OK;
  // 32-row tiles x 4 stages for the big layers; a batch too small to give
  // every resident CTA several of them (GDELT hop 1 alone: 18k rows) uses
  // 8-row tiles on 4x the CTAs, so more rows are in flight at once.
  // TG_K5_TILE=<rows>x<stages> (32x4, 16x8, 8x16, 16x6, 8x4) overrides.
  int ROWS = 32, STAGES = 4;
  const int64_t big_cap = (int64_t)device_sms() * (int)((228 * 1024) / ((size_t)4 * 32 * rowbytes + 1056));
  if ((n + 31) / 32 < 3 * big_cap && getenv("TG_K5_TILE32") == nullptr) ROWS = 8;
  if (const char* e = getenv("TG_K5_TILE")) sscanf(e, "%dx%d", &ROWS, &STAGES);
  const size_t smem = (size_t)STAGES * ROWS * rowbytes + STAGES * 8;
  if (smem > 200 * 1024) return TG_OK;
  GatherSegs sg{};
  sg.nseg = 0;
  int64_t t0 = 0;
  for (int i = 0; i < nseg; ++i) {
    if (segs[i].n <= 0) continue;
    const int k = sg.nseg++;
    sg.ids[k] = segs[i].ids;
    sg.mask[k] = segs[i].mask;
    sg.out[k] = segs[i].out;
    sg.n[k] = segs[i].n;
    sg.tile0[k] = t0;
    t0 += (segs[i].n + ROWS - 1) / ROWS;
  }
  sg.tile0[sg.nseg] = t0;
  auto kern = row_gather_bulk_kernel<32, 4>;
  if (ROWS == 8 && STAGES == 4) kern = row_gather_bulk_kernel<8, 4>;
  else if (ROWS == 16 && STAGES == 8) kern = row_gather_bulk_kernel<16, 8>;
  else if (ROWS == 8 && STAGES == 16) kern = row_gather_bulk_kernel<8, 16>;
  else if (ROWS == 16 && STAGES == 6) kern = row_gather_bulk_kernel<16, 6>;
  else if (!(ROWS == 32 && STAGES == 4)) return fail(TG_EVALUE, "TG_K5_TILE %dx%d not built", ROWS, STAGES);
  TG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int per_sm = (int)((228 * 1024) / (smem + 1024));
  const int64_t cap = (int64_t)device_sms() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(t0 < cap ? t0 : cap);
  kern<<<grid, 32, smem, st>>>(sg, fs, slot_of, rowbytes);
  TG_LAUNCHED();
  *handled = true;
  return TG_OK;
}

int launch_row_gather(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store& fs,
                      const int32_t* slot_of, int invalid_mode, float* out, int64_t out_ld, cudaStream_t st) {
  if (n > 0 && fs.d > 0 && out != nullptr) {
    const tg_gather_seg seg{ids, mask, n, out};
    bool handled = false;
    const int rc = launch_bulk_segs(&seg, 1, fs, slot_of, invalid_mode, out_ld, st, &handled);
    if (rc != TG_OK || handled) return rc;
  }
  if (n <= 0 || fs.d <= 0 || out == nullptr) return TG_OK;
  // copy width: rows padded to 16 B on both sides
  // are moved whole, pad columns included, with 16-byte units
  int cw = fs.d;
  const int r4 = (fs.d + 3) & ~3;
  if (fs.ld >= r4 && out_ld >= r4 && (fs.hot == nullptr || fs.hot_ld >= r4)) cw = r4;
  const int vec = pick_vec(cw, fs.ld, out_ld, fs.table, out, fs.hot, fs.hot ? fs.hot_ld : 0);
  if (vec == 4) return launch_row_gather_v<4>(ids, mask, n, fs, cw, slot_of, invalid_mode, out, out_ld, st);
  if (vec == 2) return launch_row_gather_v<2>(ids, mask, n, fs, cw, slot_of, invalid_mode, out, out_ld, st);
  return launch_row_gather_v<1>(ids, mask, n, fs, cw, slot_of, invalid_mode, out, out_ld, st);
}

static int launch_gather(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store* store,
                         const tg_cache_dev* cache, int mask_mode, float* out, int64_t out_ld,
                         uint8_t* hits, cudaStream_t st) {
  if (n < 0) return fail(TG_EVALUE, "negative row count");
  if (n == 0) return TG_OK;
  const int has_cache = cache != nullptr && cache->slot_of != nullptr;
  if (has_cache || hits != nullptr) {
    if (!has_cache) return fail(TG_EVALUE, "hit flags need a cache");
    const int64_t want = (n + 255) / 256;
    const int64_t cap = (int64_t)device_sms() * 16;
    count_kernel<<<(int)(want < cap ? want : cap), 256, 0, st>>>(ids, mask, n, *cache, hits);
    TG_LAUNCHED();
  }
  if (out != nullptr && store != nullptr && store->d > 0)
    return launch_row_gather(ids, mask, n, *store, has_cache ? cache->slot_of : nullptr,
                             mask_mode == 1 ? ROW_TIMES_ZERO : ROW_ZERO, out, out_ld, st);
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

// Selection gather + hop expansion after the adaptive sampler
// (training.py:281-291 and :311-314): sel_x[b, k] = x[b, selected[b, k]]
// where selected, 0 / 0.0 on padded picks; children of root b at
// next[B + b*n + k] = (sel_id, t_b - sel_dt), targets at next[b].
__global__ void select_expand_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ eids,
                                     const double* __restrict__ dts, const int64_t* __restrict__ selected,
                                     const uint8_t* __restrict__ smask, const int64_t* __restrict__ qv,
                                     const double* __restrict__ qt, int64_t B, int m, int n, int64_t* sel_ids,
                                     int64_t* sel_eids, double* sel_dts, int64_t* next_v, double* next_t) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < B * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / n;
    const bool v = smask[e] != 0;
    const int64_t s = v ? selected[e] : 0;
    const int64_t src = b * m + s;
    const int64_t id = v ? ids[src] : 0;
    const double dt = v ? dts[src] : 0.0;
    if (sel_ids) sel_ids[e] = id;
    if (sel_eids) sel_eids[e] = v ? eids[src] : 0;
    if (sel_dts) sel_dts[e] = dt;
    if (next_v) {
      next_v[B + e] = id;
      next_t[B + e] = __dsub_rn(qt[b], dt);
      if (e - b * n == 0) {
        next_v[b] = qv[b];
        next_t[b] = qt[b];
      }
    }
  }
}

}  // namespace tg

using namespace tg;

extern "C" int tg_select_expand(const int64_t* ids, const int64_t* eids, const double* dts, const int64_t* selected,
                                const uint8_t* sel_mask, const int64_t* qv, const double* qt, int64_t B, int32_t m,
                                int32_t n, int64_t* sel_ids, int64_t* sel_eids, double* sel_dts, int64_t* next_v,
                                double* next_t, void* stream) {
  if (m < 1 || n < 1) return fail(TG_EVALUE, "need m, n >= 1");
  if ((next_v == nullptr) != (next_t == nullptr)) return fail(TG_EVALUE, "next_v/next_t must be given together");
  if (B <= 0) return TG_OK;
  const int64_t total = B * n;
  const int64_t want = (total + 255) / 256;
  const int grid = (int)(want < 65535 ? want : 65535);
  select_expand_kernel<<<grid, 256, 0, as_stream(stream)>>>(ids, eids, dts, selected, sel_mask, qv, qt, B, m, n,
                                                            sel_ids, sel_eids, sel_dts, next_v, next_t);
  TG_LAUNCHED();
  return TG_OK;
}

extern "C" int tg_lookup_gather(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store* store,
                                const tg_cache_dev* cache, int32_t mask_mode, float* out, int64_t out_ld,
                                void* stream) {
  if (mask_mode != 0 && mask_mode != 1) return fail(TG_EVALUE, "mask_mode must be 0 or 1");
  return launch_gather(ids, mask, n, store, cache, mask_mode, out, out_ld, nullptr, as_stream(stream));
}

extern "C" int tg_gather_rows(const int64_t* ids, const uint8_t* mask, int64_t n, const tg_feat_store* store,
                              const int32_t* slot_of, int32_t mask_mode, float* out, int64_t out_ld, void* stream) {
  if (mask_mode != 0 && mask_mode != 1) return fail(TG_EVALUE, "mask_mode must be 0 or 1");
  if (n < 0) return fail(TG_EVALUE, "negative row count");
  if (store == nullptr) return fail(TG_EVALUE, "tg_gather_rows needs a store");
  return launch_row_gather(ids, mask, n, *store, slot_of, mask_mode == 1 ? ROW_TIMES_ZERO : ROW_ZERO, out, out_ld,
                           as_stream(stream));
}

extern "C" int tg_gather_rows_multi(const tg_gather_seg* segs, int32_t nseg, const tg_feat_store* store,
                                    const int32_t* slot_of, int32_t mask_mode, int64_t out_ld, void* stream) {
  if (mask_mode != 0 && mask_mode != 1) return fail(TG_EVALUE, "mask_mode must be 0 or 1");
  if (nseg < 0 || (nseg > 0 && segs == nullptr)) return fail(TG_EVALUE, "bad segment list");
  if (store == nullptr) return fail(TG_EVALUE, "tg_gather_rows_multi needs a store");
  for (int i = 0; i < nseg; ++i)
    if (segs[i].n < 0) return fail(TG_EVALUE, "negative row count in segment %d", i);
  const int mode = mask_mode == 1 ? ROW_TIMES_ZERO : ROW_ZERO;
  const cudaStream_t st = as_stream(stream);
  for (int i0 = 0; i0 < nseg; i0 += kMaxSegs) {
    const int k = nseg - i0 < kMaxSegs ? nseg - i0 : kMaxSegs;
    bool handled = false;
    int rc = launch_bulk_segs(segs + i0, k, *store, slot_of, mode, out_ld, st, &handled);
    if (rc != TG_OK) return rc;
    if (handled) continue;
    for (int i = i0; i < i0 + k; ++i) {  // register path, one launch per segment
      rc = launch_row_gather(segs[i].ids, segs[i].mask, segs[i].n, *store, slot_of, mode, segs[i].out, out_ld, st);
      if (rc != TG_OK) return rc;
    }
  }
  return TG_OK;
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
