// K9: importance-weighted mini-batch selection.
//
// Replaces selector.py:46-53 select_batch -- p = scores / scores.sum(),
// rng.choice(n, b, replace=False, p=p), sorted + base_eid -- and
// selector.py:56-61 update_scores (Eq. 10: scores[e] = sigmoid(logit) +
// gamma), called from training.py:364-367 / :403-404.
//
// numpy's choice(replace=False, p) runs rounds: draw size-n_uniq doubles,
// zero p at the indices found so far, cdf = cumsum(p), cdf /= cdf[-1],
// searchsorted(x, 'right'), keep first occurrences.  Every step is
// reproduced bit for bit:
//
//   * scores.sum(): numpy's pairwise tree (pcg.cuh pw_block leaves, the
//     same split points), evaluated leaves-in-parallel then level by level;
//   * the draws: PCG64 outputs off .. off+k-1 of the Trainer's S_BATCH
//     substream (each thread jumps to its position);
//   * cumsum: a SEQUENTIAL f64 prefix sum, s_k = fl(s_{k-1} + p_k).  It is
//     not reassociable, but inside one binade [2^E, 2^(E+1)) every partial
//     sum is a multiple of u = 2^(E-52), so fl(s + p) = s + rne(p/u)*u
//     unless p/u ends in exactly .5 (a tie, decided by the parity of s/u).
//     Chunks of CH elements whose whole range stays inside one binade (with
//     a 2^-20 margin, checked against an approximate parallel prefix) and
//     hold no tie advance s by an exact integer D * u computed in parallel;
//     the few chunks that cross a binade or hold a tie (and the first chunk,
//     where s starts at 0) are summed element by element.  One warp walks
//     the chunk chain 32 chunks per step with an integer warp scan, so the
//     exact start of every chunk is known;
//   * searchsorted: binary search over the exact chunk ends, then a
//     sequential walk inside the one chunk that holds the crossing.
//
// Cost per round: ~3 streaming passes over p (8 B/row) + O(#chunks) serial
// steps -- HBM-bound, versus numpy's single-threaded cumsum.
#include <cmath>

#include "pcg.cuh"

namespace tg {

constexpr int SEL_CH = 2048;          // elements per chunk
constexpr double SEL_MARGIN = 0x1p-20;  // relative guard band around binade edges

// ---- pairwise total (numpy add.reduce order) --------------------------------
// Node of the recursion at depth `level` reached by the top bits of q.
struct PwNode {
  int64_t lo, n;
  int leaf_level;  // depth at which the path met a leaf (n <= 128), or -1
};

__device__ __forceinline__ PwNode pw_descend(int64_t n, int depth, int64_t q, int levels) {
  PwNode r{0, n, -1};
  for (int lvl = 0; lvl < levels; ++lvl) {
    if (r.n <= 128) {
      r.leaf_level = lvl;
      return r;
    }
    int64_t n2 = r.n / 2;
    n2 -= n2 % 8;
    if ((q >> (depth - 1 - lvl)) & 1) {
      r.lo += n2;
      r.n -= n2;
    } else {
      r.n = n2;
    }
  }
  if (r.n <= 128) r.leaf_level = levels;
  return r;
}

// leaves: thread q (of 2^depth) owns the leaf whose leftmost depth-`depth`
// position is q; its value goes to val[q]
__global__ void pw_leaf_kernel(const double* __restrict__ a, int64_t n, int depth, double* __restrict__ val) {
  const int64_t Q = (int64_t)1 << depth;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Q; q += (int64_t)gridDim.x * blockDim.x) {
    const PwNode nd = pw_descend(n, depth, q, depth);
    if (nd.leaf_level < 0) continue;  // cannot happen when depth is deep enough
    const int low_bits = depth - nd.leaf_level;
    if (low_bits > 0 && (q & (((int64_t)1 << low_bits) - 1)) != 0) continue;  // not the leaf's representative
    val[q] = pw_block(a + nd.lo, (int)nd.n, 1);
  }
}

// internal nodes at `level`: val[pos] = val[pos] + val[pos + half] in numpy's order
__global__ void pw_combine_kernel(int64_t n, int depth, int level, double* __restrict__ val) {
  const int64_t nodes = (int64_t)1 << level;
  const int64_t span = (int64_t)1 << (depth - level);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nodes; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = j * span;
    const PwNode nd = pw_descend(n, depth, pos, level);
    if (nd.leaf_level >= 0) continue;  // a leaf at or above this level: value already in place / node absent
    val[pos] = __dadd_rn(val[pos], val[pos + span / 2]);
  }
}

// depth at which every node of the recursion is a leaf (host mirror of the
// split; a level holds only a handful of distinct sizes)
static int pw_depth(int64_t n) {
  int64_t sizes[64];
  int ns = 1, d = 0;
  sizes[0] = n;
  for (;;) {
    int64_t next[64];
    int nn = 0;
    bool any = false;
    for (int i = 0; i < ns; ++i) {
      if (sizes[i] <= 128) continue;
      any = true;
      int64_t n2 = sizes[i] / 2;
      n2 -= n2 % 8;
      const int64_t kids[2] = {n2, sizes[i] - n2};
      for (int64_t kv : kids) {
        bool seen = false;
        for (int j = 0; j < nn; ++j) seen |= next[j] == kv;
        if (!seen && nn < 64) next[nn++] = kv;
      }
    }
    if (!any) return d;
    for (int i = 0; i < nn; ++i) sizes[i] = next[i];
    ns = nn;
    ++d;
  }
}

// ---- p = scores / total, validity flags (numpy choice's checks) -------------
__global__ void normalize_kernel(const double* __restrict__ s, int64_t n, const double* __restrict__ total,
                                 double* __restrict__ p, unsigned long long* __restrict__ nonzero,
                                 int* __restrict__ bad) {
  const double T = *total;
  unsigned long long nz = 0;
  int b = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = __ddiv_rn(s[i], T);
    p[i] = v;
    nz += v > 0.0;
    b |= (v < 0.0) ? 1 : 0;
    b |= (v != v) ? 2 : 0;
  }
  nz = warp_sum(nz);
  b = __reduce_or_sync(FULL, b);
  if ((threadIdx.x & 31) == 0) {
    if (nz) atomicAdd(nonzero, nz);
    if (b) atomicOr(bad, b);
  }
}

// ---- per-chunk approximate sums (any order) ----------------------------------
__global__ void chunk_sum_kernel(const double* __restrict__ p, int64_t n, int64_t nch, double* __restrict__ csum) {
  __shared__ double red[32];
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int64_t lo = c * SEL_CH, hi = lo + SEL_CH < n ? lo + SEL_CH : n;
    double s = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += p[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
      v = warp_sum(v);
      if (threadIdx.x == 0) csum[c] = v;
    }
    __syncthreads();
  }
}

// exclusive scan of the chunk sums (one block; approximate starts)
__global__ void chunk_scan_kernel(const double* __restrict__ csum, int64_t nch, double* __restrict__ astart) {
  __shared__ double part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (nch + T - 1) / T;
  const int64_t lo = t * per, hi = lo + per < nch ? lo + per : nch;
  double s = 0.0;
  for (int64_t c = lo; c < hi; ++c) s += csum[c];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    double acc = 0.0;
    for (int i = 0; i < T; ++i) {
      const double v = part[i];
      part[i] = acc;
      acc += v;
    }
  }
  __syncthreads();
  double acc = part[t];
  for (int64_t c = lo; c < hi; ++c) {
    astart[c] = acc;
    acc += csum[c];
  }
}

// binade exponent E of a positive double: 2^E <= v < 2^(E+1)
__device__ __forceinline__ int binade(double v) {
  int e;
  frexp(v, &e);
  return e - 1;
}

// fast-path classification + exact integer advance of each chunk
__global__ void chunk_classify_kernel(const double* __restrict__ p, int64_t n, int64_t nch,
                                      const double* __restrict__ astart, const double* __restrict__ csum,
                                      long long* __restrict__ dinc, int* __restrict__ ebin) {
  __shared__ int s_ok;
  __shared__ long long s_d[32];
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const double a0 = astart[c], a1 = a0 + csum[c];
    int E = 0;
    bool ok = a0 > 0.0;
    if (ok) {
      E = binade(a0);
      ok = a0 >= ldexp(1.0, E) * (1.0 + SEL_MARGIN) && a1 <= ldexp(1.0, E + 1) * (1.0 - SEL_MARGIN);
    }
    if (threadIdx.x == 0) s_ok = ok ? 1 : 0;
    __syncthreads();
    long long d = 0;
    int tie = 0;
    if (ok) {
      const int64_t lo = c * SEL_CH, hi = lo + SEL_CH < n ? lo + SEL_CH : n;
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double q = ldexp(p[i], 52 - E);  // p / u, exact (power-of-two scale)
        const double f = floor(q);
        tie |= (q - f) == 0.5;
        d += (long long)rint(q);
      }
    }
    d = warp_sum(d);
    tie = __reduce_or_sync(FULL, tie);
    if ((threadIdx.x & 31) == 0) {
      s_d[threadIdx.x >> 5] = d;
      if (tie) s_ok = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long D = 0;
      for (int w = 0; w < (int)blockDim.x / 32; ++w) D += s_d[w];
      dinc[c] = D;
      ebin[c] = s_ok ? E : INT32_MIN;
    }
    __syncthreads();
  }
}

// Exact chunk starts.  One warp: 32 chunks per step when they all take the
// fast path from the current exact s, else one chunk summed sequentially.
__global__ void chunk_walk_kernel(const double* __restrict__ p, int64_t n, int64_t nch,
                                  const long long* __restrict__ dinc, const int* __restrict__ ebin,
                                  double* __restrict__ sstart) {
  __shared__ double s_chunk[SEL_CH];
  const int lane = threadIdx.x;
  double s = 0.0;
  int64_t c = 0;
  while (c < nch) {
    const int64_t cc = c + lane;
    const bool in = cc < nch;
    const long long D = in ? dinc[cc] : 0;
    const int E = in ? ebin[cc] : INT32_MIN;
    // inclusive warp scan of D
    long long incl = D;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const int Es = s > 0.0 ? binade(s) : INT32_MIN;
    bool good = in && E != INT32_MIN && E == Es;
    if (good) {
      const double u = ldexp(1.0, E - 52);
      good = __dadd_rn(s, __dmul_rn((double)incl, u)) < ldexp(1.0, E + 1);
    }
    const unsigned bad = __ballot_sync(FULL, !good);
    const int f = bad ? __ffs(bad) - 1 : 32;  // leading run of fast chunks
    if (f > 0) {
      const double u = ldexp(1.0, Es - 52);
      if (lane < f) sstart[cc] = __dadd_rn(s, __dmul_rn((double)(incl - D), u));
      const long long tot = __shfl_sync(FULL, incl, f - 1);
      s = __dadd_rn(s, __dmul_rn((double)tot, u));
      c += f;
      continue;
    }
    // chunk c by the sequential definition: the warp stages it in shared
    // memory (coalesced), lane 0 adds in order, the result is broadcast
    {
      const int64_t lo = c * SEL_CH, hi = lo + SEL_CH < n ? lo + SEL_CH : n;
      for (int64_t i = lo + lane; i < hi; i += 32) s_chunk[i - lo] = p[i];
      __syncwarp();
      if (lane == 0) {
        sstart[c] = s;
        const int cnt = (int)(hi - lo);
#pragma unroll 8
        for (int i = 0; i < cnt; ++i) s = __dadd_rn(s, s_chunk[i]);
      }
      __syncwarp();
      s = __shfl_sync(FULL, s, 0);
    }
    ++c;
  }
  if (lane == 0) sstart[nch] = s;
}

// draws x_i = PCG64 output (off + i) and their searchsorted positions
__global__ void draw_search_kernel(const double* __restrict__ p, int64_t n, int64_t nch,
                                   const double* __restrict__ sstart, tg_pcg64 rng, uint64_t off, int64_t k,
                                   int64_t* __restrict__ newidx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const u128 st = pcg_advance(u128{rng.state_hi, rng.state_lo}, u128{rng.inc_hi, rng.inc_lo}, off + (uint64_t)i + 1);
  const double x = pcg_double(st);
  const double L = sstart[nch];
  // first chunk whose end (= next chunk's start) normalises above x
  int64_t lo = 0, hi = nch - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (__ddiv_rn(sstart[mid + 1], L) > x)
      hi = mid;
    else
      lo = mid + 1;
  }
  double s = sstart[lo];
  const int64_t a = lo * SEL_CH, b = a + SEL_CH < n ? a + SEL_CH : n;
  int64_t j = b - 1;
  // sequential walk in blocks of 8 (loads issued ahead of the dependent adds)
  for (int64_t q0 = a; q0 < b; q0 += 8) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = q0 + r < b ? p[q0 + r] : 0.0;
    int hit = -1;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (hit < 0 && q0 + r < b) {
        s = __dadd_rn(s, v[r]);
        if (__ddiv_rn(s, L) > x) hit = r;
      }
    }
    if (hit >= 0) {
      j = q0 + hit;
      break;
    }
  }
  newidx[i] = j;
}

// keep first occurrences (np.unique return_index, sorted), append to found
__global__ void dedup_append_kernel(const int64_t* __restrict__ newidx, int64_t k, int64_t* __restrict__ found,
                                    int64_t n_uniq, double* __restrict__ p, long long* __restrict__ count) {
  __shared__ int s_cnt;
  extern __shared__ int64_t s_new[];  // k candidates when they fit (else read from global)
  const bool staged = k <= 6144;
  if (threadIdx.x == 0) s_cnt = 0;
  if (staged)
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) s_new[i] = newidx[i];
  __syncthreads();
  const int64_t* cand = staged ? s_new : newidx;
  // ordered compaction: each pass handles blockDim.x candidates
  for (int64_t base = 0; base < k; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool keep = false;
    int64_t v = 0;
    if (i < k) {
      v = cand[i];
      keep = true;
      for (int64_t j = 0; j < i; ++j)
        if (cand[j] == v) {
          keep = false;
          break;
        }
    }
    // block-wide exclusive scan of keep (warp ballots + shared prefix)
    __shared__ int wsum[32];
    const unsigned m = __ballot_sync(FULL, keep);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    int before = 0;
    for (int q = 0; q < w; ++q) before += wsum[q];
    const int rank = s_cnt + before + __popc(m & ((1u << lane) - 1));
    if (keep) {
      found[n_uniq + rank] = v;
      p[v] = 0.0;  // numpy zeroes p[found] before the next round's cumsum
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int q = 0; q < (int)blockDim.x / 32; ++q) tot += wsum[q];
      s_cnt += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = s_cnt;
}

// out = sort(found) + base (distinct values: rank by counting)
__global__ void rank_sort_kernel(const int64_t* __restrict__ found, int64_t b, int64_t base, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = found[i];
    int64_t r = 0;
    for (int64_t j = 0; j < b; ++j) r += found[j] < v;
    out[r] = v + base;
  }
}

// ---- update_scores (selector.py:56-61) ---------------------------------------
__global__ void update_scores_kernel(double* __restrict__ scores, int64_t n, const int64_t* __restrict__ eids,
                                     int64_t b, int64_t base, const double* __restrict__ logits, double gamma) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = eids[i];
    bool last = true;  // numpy fancy assignment: the last duplicate wins
    for (int64_t j = i + 1; j < b; ++j)
      if (eids[j] == e) {
        last = false;
        break;
      }
    if (!last) continue;
    const double x = logits[i];
    const double ex = exp(-fabs(x));
    const double sg = x >= 0.0 ? 1.0 / (1.0 + ex) : ex / (1.0 + ex);
    scores[e - base] = sg + gamma;
  }
}

__global__ void eid_range_kernel(const int64_t* __restrict__ e, int64_t b, int64_t lo, int64_t hi, int* bad) {
  int x = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x)
    x |= (e[i] < lo) | (e[i] >= hi);
  if (__any_sync(FULL, x) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

static int grid_for(int64_t work, int threads = 256) {
  const int64_t g = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)device_sms() * 16;
  return (int)(g < 1 ? 1 : (g < cap ? g : cap));
}

}  // namespace tg

using namespace tg;

extern "C" int tg_select_batch(const double* scores, int64_t n, int64_t b, const tg_pcg64* rng, int64_t base,
                               int64_t* out, int64_t* host_draws, void* stream) {
  if (host_draws) *host_draws = 0;
  if (n < 1) return fail(TG_EVALUE, "need at least one training edge");
  if (b < 0) return fail(TG_EVALUE, "negative batch size");
  if (b > n) return fail(TG_EVALUE, "batch size %lld exceeds %lld training edges", (long long)b, (long long)n);
  if (b == 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  const int64_t nch = (n + SEL_CH - 1) / SEL_CH;
  const int depth = pw_depth(n);
  const int64_t Q = (int64_t)1 << depth;
  // one stream-ordered workspace
  const size_t bytes = (size_t)n * 8 + (size_t)Q * 8 + (size_t)nch * (8 + 8 + 8 + 4) + (size_t)(nch + 1) * 8 +
                       (size_t)b * 8 * 2 + 32 + 16 * 16;  // + alignment slack of the 11 sub-buffers
  unsigned char* ws = nullptr;
  TG_CUDA(cudaMallocAsync(&ws, bytes, st));
  unsigned char* q = ws;
  auto take = [&](size_t sz) {
    unsigned char* r = q;
    q += (sz + 15) & ~size_t(15);
    return r;
  };
  double* p = reinterpret_cast<double*>(take((size_t)n * 8));
  double* val = reinterpret_cast<double*>(take((size_t)Q * 8));
  double* csum = reinterpret_cast<double*>(take((size_t)nch * 8));
  double* astart = reinterpret_cast<double*>(take((size_t)nch * 8));
  long long* dinc = reinterpret_cast<long long*>(take((size_t)nch * 8));
  int* ebin = reinterpret_cast<int*>(take((size_t)nch * 4));
  double* sstart = reinterpret_cast<double*>(take((size_t)(nch + 1) * 8));
  int64_t* found = reinterpret_cast<int64_t*>(take((size_t)b * 8));
  int64_t* newidx = reinterpret_cast<int64_t*>(take((size_t)b * 8));
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(take(32));  // nonzero, bad, count
  int rc = TG_OK;
  auto done = [&](int r) {
    cudaFreeAsync(ws, st);
    return r;
  };
  // total = scores.sum() in numpy's pairwise order
  pw_leaf_kernel<<<grid_for(Q), 256, 0, st>>>(scores, n, depth, val);
  TG_LAUNCHED();
  for (int lvl = depth - 1; lvl >= 0; --lvl) {
    pw_combine_kernel<<<grid_for((int64_t)1 << lvl), 256, 0, st>>>(n, depth, lvl, val);
    TG_LAUNCHED();
  }
  TG_CUDA(cudaMemsetAsync(flags, 0, 32, st));
  normalize_kernel<<<grid_for(n), 256, 0, st>>>(scores, n, val, p, flags, reinterpret_cast<int*>(flags + 1));
  TG_LAUNCHED();
  unsigned long long hf[2] = {0, 0};
  TG_CUDA(cudaMemcpyAsync(hf, flags, 16, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaStreamSynchronize(st));
  if (hf[1] & 2) return done(fail(TG_EVALUE, "probabilities contain NaN"));
  if (hf[1] & 1) return done(fail(TG_EVALUE, "probabilities are not non-negative"));
  if ((int64_t)hf[0] < b) return done(fail(TG_EVALUE, "Fewer non-zero entries in p than size"));
  int64_t n_uniq = 0;
  uint64_t off = 0;
  const int sms = device_sms();
  while (n_uniq < b) {
    const int64_t k = b - n_uniq;
    const int cg = (int)(nch < (int64_t)sms * 8 ? nch : (int64_t)sms * 8);
    chunk_sum_kernel<<<cg, 256, 0, st>>>(p, n, nch, csum);
    TG_LAUNCHED();
    chunk_scan_kernel<<<1, 1024, 0, st>>>(csum, nch, astart);
    TG_LAUNCHED();
    chunk_classify_kernel<<<cg, 256, 0, st>>>(p, n, nch, astart, csum, dinc, ebin);
    TG_LAUNCHED();
    chunk_walk_kernel<<<1, 32, 0, st>>>(p, n, nch, dinc, ebin, sstart);
    TG_LAUNCHED();
    draw_search_kernel<<<(unsigned)((k + 127) / 128), 128, 0, st>>>(p, n, nch, sstart, *rng, off, k, newidx);
    TG_LAUNCHED();
    dedup_append_kernel<<<1, 1024, k <= 6144 ? (size_t)k * 8 : 0, st>>>(newidx, k, found, n_uniq, p,
                                                                      reinterpret_cast<long long*>(flags + 2));
    TG_LAUNCHED();
    long long cnt = 0;
    TG_CUDA(cudaMemcpyAsync(&cnt, flags + 2, 8, cudaMemcpyDeviceToHost, st));
    TG_CUDA(cudaStreamSynchronize(st));
    off += (uint64_t)k;
    n_uniq += cnt;
    if (cnt <= 0) {
      rc = fail(TG_ECUDA, "selection round made no progress");
      break;
    }
  }
  if (host_draws) *host_draws = (int64_t)off;
  if (rc == TG_OK) {
    rank_sort_kernel<<<grid_for(b), 256, 0, st>>>(found, b, base, out);
    TG_LAUNCHED();
  }
  return done(rc);
}

extern "C" int tg_update_scores(double* scores, int64_t n, const int64_t* eids, int64_t b, int64_t base,
                                const double* logits, double gamma, void* stream) {
  if (b <= 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  int* bad = nullptr;
  TG_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  TG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  eid_range_kernel<<<grid_for(b), 256, 0, st>>>(eids, b, base, base + n, bad);
  TG_LAUNCHED();
  int h = 0;
  TG_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaFreeAsync(bad, st));
  TG_CUDA(cudaStreamSynchronize(st));
  if (h) return fail(TG_EINDEX, "eid outside the training range");
  update_scores_kernel<<<grid_for(b), 256, 0, st>>>(scores, n, eids, b, base, logits, gamma);
  TG_LAUNCHED();
  return TG_OK;
}
