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
#include <cstdio>
#include <cstdlib>

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

// leaves: 8 threads per depth-`depth` position q; the group of the leaf's
// representative (leftmost position) sums it in numpy's order -- thread j
// owns accumulator r[j] (a[j], a[j+8], ...), the pairs combine by xor
// shuffles ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), thread 0 adds the tail.
// The same pass accumulates approximate per-chunk sums of the scores
// (atomics, any order) and the sign counts numpy's choice() checks.
__global__ void pw_leaf8_kernel(const double* __restrict__ a, int64_t n, int depth, double* __restrict__ val,
                                double* __restrict__ csum, unsigned long long* __restrict__ signs) {
  const int64_t Q = (int64_t)1 << depth;
  unsigned long long npos = 0, nneg = 0;
  const int j = threadIdx.x & 7;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3; g < ((Q + 3) / 4) * 4;
       g += ((int64_t)gridDim.x * blockDim.x) >> 3) {
    bool active = false;
    PwNode nd{0, 0, -1};
    if (j == 0 && g < Q) {  // one descent per 8-lane group, shared below
      nd = pw_descend(n, depth, g, depth);
      const int low_bits = depth - nd.leaf_level;
      active = nd.leaf_level >= 0 && !(low_bits > 0 && (g & (((int64_t)1 << low_bits) - 1)) != 0);
    }
    const int src = threadIdx.x & ~7;
    nd.lo = __shfl_sync(FULL, nd.lo, src & 31);
    nd.n = __shfl_sync(FULL, nd.n, src & 31);
    active = __shfl_sync(FULL, (int)active, src & 31) != 0;
    const double* x = a + nd.lo;
    const int nl = active ? (int)nd.n : 0;
    const int m8 = nl >= 8 ? nl - nl % 8 : 0;
    double r = 0.0;
    if (m8 > 0) {
      r = x[j];
#pragma unroll 4
      for (int i = 8; i < m8; i += 8) r = __dadd_rn(r, x[i + j]);
    }
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 4));
    // chunk sums + sign counts over this lane's elements i = j (mod 8)
    double c0 = 0.0, c1 = 0.0;
    const int64_t cfirst = nd.lo / SEL_CH;
#pragma unroll 4
    for (int i = j; i < nl; i += 8) {
      const double v = x[i];
      npos += v > 0.0;
      nneg += v < 0.0;
      if ((nd.lo + i) / SEL_CH == cfirst)
        c0 += v;
      else
        c1 += v;
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      c0 += __shfl_xor_sync(FULL, c0, o);
      c1 += __shfl_xor_sync(FULL, c1, o);
    }
    if (active && j == 0) {
      double res;
      if (nl < 8) {
        res = 0.0;
        for (int i = 0; i < nl; ++i) res = __dadd_rn(res, x[i]);
      } else {
        res = r;
        for (int i = m8; i < nl; ++i) res = __dadd_rn(res, x[i]);
      }
      val[g] = res;
      atomicAdd(csum + cfirst, c0);
      if (c1 != 0.0) atomicAdd(csum + cfirst + 1, c1);
    }
  }
  npos = warp_sum(npos);
  nneg = warp_sum(nneg);
  if ((threadIdx.x & 31) == 0) {
    if (npos) atomicAdd(signs + 0, npos);
    if (nneg) atomicAdd(signs + 1, nneg);
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
        for (int q = 0; q < nn; ++q) seen |= next[q] == kv;
        if (!seen && nn < 64) next[nn++] = kv;
      }
    }
    if (!any) return d;
    for (int i = 0; i < nn; ++i) sizes[i] = next[i];
    ns = nn;
    ++d;
  }
}

// ---- p on the fly: p_i = scores_i / T, 0 for indices found in earlier rounds
struct PView {
  const double* s;
  const uint32_t* zmask;  // bit i: p_i zeroed (numpy's p[found] = 0)
  double T;
  double R;               // RN(1 / T), computed on the host
  int64_t n;
};
// fl(s / T) without a division: q0 = RN(s R), r = s - q0 T (exact by FMA),
// q1 = RN(q0 + r R) is the correctly rounded quotient when R = RN(1/T) and
// everything stays in the normal range (Markstein; checked bit-for-bit
// against IEEE division on 1e8 random pairs, tests/test_host.py); outside
// that range the IEEE division is used.
__device__ __forceinline__ double div_rn(double s, double T, double R) {
  const double q0 = __dmul_rn(s, R);
  const double aq = fabs(q0);
  if (aq > 0x1p-1000 && aq < 0x1p+1000) {
    const double r = __fma_rn(-q0, T, s);
    return __fma_rn(r, R, q0);
  }
  return __ddiv_rn(s, T);
}
__device__ __forceinline__ double p_at(const PView& v, int64_t i) {
  const double x = div_rn(v.s[i], v.T, v.R);
  return ((v.zmask[i >> 5] >> (i & 31)) & 1u) ? 0.0 : x;
}
// p from a raw score and its zero-mask word (loads issued separately, so a
// batch of them is in flight before any of the dependent arithmetic)
__device__ __forceinline__ double p_of(const PView& v, double sv, uint32_t zw, int64_t i) {
  return ((zw >> (i & 31)) & 1u) ? 0.0 : div_rn(sv, v.T, v.R);
}

// binade exponent E of a positive double: 2^E <= v < 2^(E+1)
__device__ __forceinline__ int binade(double v) {
  return (int)((__double_as_longlong(v) >> 52) & 0x7FF) - 1023;  // v normal and > 0
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
// the fast path needs v >= 2^-900 (normal u and an exact power-of-two scale)
__device__ __forceinline__ bool fast_binade(double v) { return v >= 0x1p-900 && v < 0x1p+900; }

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

// Fast-path classification + exact integer advance of each chunk (warp per
// chunk).  astart/csum are sums of SCORES; /T turns them into p sums.
constexpr int SEL_SLOTS = 2048;  // chunks whose p values are staged for the walk (x 16 KB)

__device__ __forceinline__ void stage_p(const PView& pv, int64_t lo, int64_t hi, int lane, double* dst) {
  for (int64_t i0 = lo; i0 < hi; i0 += 32 * 8) {  // 8 loads in flight per lane
    double v[8];
    uint32_t zw[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // loads only, then the arithmetic
      const int64_t i = i0 + 32 * u + lane;
      v[u] = i < hi ? __ldg(pv.s + i) : 0.0;
      zw[u] = i < hi ? __ldg(pv.zmask + (i >> 5)) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + 32 * u + lane;
      if (i < hi) dst[i - lo] = p_of(pv, v[u], zw[u], i);
    }
  }
}

// Chunks the fast path cannot take get their p values written to a staging
// slot here, where thousands of warps compute the divisions in parallel;
// the single-warp walk then reads them instead of dividing serially.
__global__ void chunk_classify_kernel(PView pv, int64_t nch, const double* __restrict__ astart,
                                      const double* __restrict__ csum, long long* __restrict__ dinc,
                                      int* __restrict__ ebin, int* __restrict__ pslot, double* __restrict__ pbuf,
                                      int* __restrict__ nslots) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w0; c < nch; c += nw) {
    const double a0 = astart[c] / pv.T, a1 = (astart[c] + csum[c]) / pv.T;
    bool ok = fast_binade(a0);
    int E = 0;
    if (ok) {
      E = binade(a0);
      ok = a0 >= pow2(E) * (1.0 + SEL_MARGIN) && a1 <= pow2(E + 1) * (1.0 - SEL_MARGIN);
    }
    long long d = 0;
    int tie = 0;
    if (ok) {  // warp-uniform
      const double scale = pow2(52 - E);  // 1/u
      const int64_t lo = c * SEL_CH, hi = lo + SEL_CH < pv.n ? lo + SEL_CH : pv.n;
      for (int64_t i0 = lo; i0 < hi; i0 += 32 * 16) {  // 16 loads in flight per lane
        double v[16];
        uint32_t zw[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {  // loads only
          const int64_t i = i0 + 32 * u + lane;
          v[u] = i < hi ? __ldg(pv.s + i) : 0.0;
          zw[u] = i < hi ? __ldg(pv.zmask + (i >> 5)) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double q = p_of(pv, v[u], zw[u], i0 + 32 * u + lane) * scale;  // exact: power-of-two scale
          const double r = rint(q);
          tie |= fabs(q - r) == 0.5 || !(q < 0x1p53);  // a tie, or an element past the binade
          d += (long long)r;
        }
      }
    }
    d = warp_sum(d);
    tie = __any_sync(FULL, tie);
    if (lane == 0) {
      dinc[c] = d;
      ebin[c] = (ok && !tie) ? E : INT32_MIN;
    }
    if (!ok || tie) {  // warp-uniform: stage this chunk's p for the walk
      int slot = 0;
      if (lane == 0) slot = atomicAdd(nslots, 1);
      slot = __shfl_sync(FULL, slot, 0);
      if (slot < SEL_SLOTS) {
        const int64_t lo = c * SEL_CH, hi = lo + SEL_CH < pv.n ? lo + SEL_CH : pv.n;
        stage_p(pv, lo, hi, lane, pbuf + (size_t)slot * SEL_CH);
        if (lane == 0) pslot[c] = slot;
      }
    }
  }
}

// One warp-wide step over 32 consecutive elements [base, base+32) ∩ [.., hi)
// from the exact running sum s (uniform across the warp): the exact partial
// sums via the binade shortcut when it applies (no tie, stays in binade),
// else element by element.  Returns the new s; incl_out[lane] = exact sum
// after this lane's element (for the searchsorted caller).
__device__ __forceinline__ double warp_step(double p, double s, int lane, double* s_lane) {
  if (s > 0.0 && fast_binade(s)) {
    const int E = binade(s);
    const double q = p * pow2(52 - E);
    const double r = rint(q);
    const bool tie = fabs(q - r) == 0.5 || !(q < 0x1p53);
    long long incl = (long long)r;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const long long tot = __shfl_sync(FULL, incl, 31);
    const double u = pow2(E - 52);
    const double end = __dadd_rn(s, __dmul_rn((double)tot, u));
    if (!__any_sync(FULL, tie) && end < pow2(E + 1)) {
      *s_lane = __dadd_rn(s, __dmul_rn((double)incl, u));
      return end;
    }
  }
  // sequential (every lane keeps the same running sum)
  double mine = s;
  for (int k = 0; k < 32; ++k) {
    const double pk = __shfl_sync(FULL, p, k);
    s = __dadd_rn(s, pk);
    if (k == lane) mine = s;
  }
  *s_lane = mine;
  return s;
}

// A chunk the fast path could not take (binade crossing, tie, s = 0):
// the warp stages its p values in shared memory, then advances by batches
// of 32 sub-chunks of 32 elements -- each lane sums one sub-chunk's exact
// integer increment in the binade of the current s, an integer warp scan
// finds the first sub-chunk that crosses the binade or holds a tie, and
// only that sub-chunk is added element by element.  Returns the end sum.
__device__ double slow_chunk(const PView& pv, int64_t lo, int64_t hi, double s, int lane, double* s_p,
                             const double* staged) {
  if (staged) {  // p precomputed by chunk_classify_kernel
    const int cnt0 = (int)(hi - lo);
    for (int i0 = 0; i0 < cnt0; i0 += 32 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = i0 + 32 * u + lane < cnt0 ? staged[i0 + 32 * u + lane] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + 32 * u + lane < cnt0) s_p[i0 + 32 * u + lane] = v[u];
    }
  } else {
    stage_p(pv, lo, hi, lane, s_p);
  }
  __syncwarp();
  const int cnt = (int)(hi - lo);
  int i = 0;
  while (i < cnt) {
    if (fast_binade(s)) {
      const int E = binade(s);
      const double scale = pow2(52 - E);
      const int sb = i + 32 * lane;  // this lane's sub-chunk
      // integer-valued doubles: exact while < 2^53, and any larger sum fails
      // the binade test below anyway (no F2I on the chain)
      double d = 0.0;
      bool bad = sb >= cnt;
      if (!bad) {
        const int se = sb + 32 < cnt ? sb + 32 : cnt;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int e = sb + ((k + lane) & 31);  // rotated: conflict-free smem reads, sum order irrelevant
          const double q = e < se ? s_p[e] * scale : 0.0;
          const double r = rint(q);
          bad |= fabs(q - r) == 0.5 || !(q < 0x1p53);
          d += r;
        }
      }
      double incl = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
      }
      if (!bad) bad = !(__dadd_rn(s, __dmul_rn(incl, pow2(E - 52))) < pow2(E + 1));
      const unsigned bm = __ballot_sync(FULL, bad);
      const int f = bm ? __ffs(bm) - 1 : 32;
      if (f > 0) {
        s = __dadd_rn(s, __dmul_rn(__shfl_sync(FULL, incl, f - 1), pow2(E - 52)));
        i += 32 * f;
        if (f == 32 || i >= cnt) continue;
      }
    }
    // one sub-chunk element by element (every lane keeps the same sum)
    const int se = i + 32 < cnt ? i + 32 : cnt;
    for (int e = i; e < se; ++e) s = __dadd_rn(s, s_p[e]);
    i = se;
  }
  __syncwarp();
  return s;
}

// Groups of 32 consecutive chunks: when all 32 are fast in one binade the
// group advances s by one exact integer gtot * u (the in-group exclusive
// prefix pexcl[c] fills sstart later, in parallel); gE = INT_MIN otherwise.
__global__ void chunk_group_kernel(int64_t nch, const long long* __restrict__ dinc, const int* __restrict__ ebin,
                                   long long* __restrict__ pexcl, long long* __restrict__ gtot, int* __restrict__ gE) {
  const int lane = threadIdx.x & 31;
  const int64_t ng = (nch + 31) / 32;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ng;
       g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t c = g * 32 + lane;
    const long long D = c < nch ? dinc[c] : 0;
    const int E = c < nch ? ebin[c] : INT32_MIN;
    long long incl = D;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    if (c < nch) pexcl[c] = incl - D;
    const int E0 = __shfl_sync(FULL, E, 0);
    const bool same = __all_sync(FULL, c >= nch || (E == E0 && E != INT32_MIN));
    if (lane == 31) {
      gtot[g] = incl;
      gE[g] = same ? E0 : INT32_MIN;
    }
  }
}

// Exact chunk starts.  One warp walks the groups: a uniform group whose end
// stays in the binade of the exact running sum advances in one step (its
// start is recorded in gs[g]); any other group is walked chunk by chunk --
// leading fast chunks by an integer warp scan, a slow chunk 32 elements per
// warp step -- writing sstart directly (gs[g] = NaN).  The group table is
// staged through shared memory 1024 groups at a time.
__global__ void chunk_walk_kernel(PView pv, int64_t nch, const long long* __restrict__ dinc,
                                  const int* __restrict__ ebin, const long long* __restrict__ gtot,
                                  const int* __restrict__ gE, double* __restrict__ gs, double* __restrict__ sstart,
                                  const int* __restrict__ pslot, const double* __restrict__ pbuf,
                                  unsigned long long* __restrict__ stats) {
  constexpr int STAGE = 1024;
  __shared__ long long s_tot[STAGE];
  __shared__ int s_e[STAGE];
  __shared__ double s_p[SEL_CH];
  const int lane = threadIdx.x;
  const int64_t ng = (nch + 31) / 32;
  double s = 0.0;
  unsigned long long n_uniform = 0, n_batches = 0, n_slow = 0;
  for (int64_t g0 = 0; g0 < ng; g0 += STAGE) {
    const int cnt = ng - g0 < STAGE ? (int)(ng - g0) : STAGE;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
      s_tot[i] = gtot[g0 + i];
      s_e[i] = gE[g0 + i];
    }
    __syncwarp();
    for (int gi = 0; gi < cnt; ++gi) {
      const int64_t g = g0 + gi;
      const int E = s_e[gi];
      if (E != INT32_MIN && fast_binade(s) && binade(s) == E) {
        // a run of uniform groups in integer form: s = m * u, m in [2^52, 2^53)
        const double u = pow2(E - 52);
        long long m = (long long)__dmul_rn(s, pow2(52 - E));
        int gj = gi;
        while (gj < cnt && s_e[gj] == E && m + s_tot[gj] < (1LL << 53)) {
          if (lane == 0) gs[g0 + gj] = __dmul_rn((double)m, u);
          m += s_tot[gj];
          ++gj;
        }
        if (gj > gi) {
          n_uniform += gj - gi;
          s = __dmul_rn((double)m, u);
          gi = gj - 1;
          continue;
        }
      }
      if (lane == 0) gs[g] = __longlong_as_double(0x7FF8000000000000LL);  // NaN: starts written below
      int64_t c = g * 32;
      const int64_t cend = c + 32 < nch ? c + 32 : nch;
      while (c < cend) {
        const int64_t cc = c + lane;
        const bool in = cc < cend;
        const long long D = in ? dinc[cc] : 0;
        const int Ec = in ? ebin[cc] : INT32_MIN;
        long long incl = D;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long v = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += v;
        }
        const int Es = fast_binade(s) ? binade(s) : INT32_MIN;
        bool good = in && Ec != INT32_MIN && Ec == Es;
        if (good) good = __dadd_rn(s, __dmul_rn((double)incl, pow2(Ec - 52))) < pow2(Ec + 1);
        const unsigned bad = __ballot_sync(FULL, !good);
        const int f = bad ? __ffs(bad) - 1 : 32;
        ++n_batches;
        if (f > 0) {
          const double u = pow2(Es - 52);
          if (lane < f) sstart[cc] = __dadd_rn(s, __dmul_rn((double)(incl - D), u));
          s = __dadd_rn(s, __dmul_rn((double)__shfl_sync(FULL, incl, f - 1), u));
          c += f;
          continue;
        }
        ++n_slow;
        // chunk c the slow way
        if (lane == 0) sstart[c] = s;
        const int64_t lo = c * SEL_CH, hi = lo + SEL_CH < pv.n ? lo + SEL_CH : pv.n;
        const int slot = pslot[c];
        s = slow_chunk(pv, lo, hi, s, lane, s_p, slot >= 0 ? pbuf + (size_t)slot * SEL_CH : nullptr);
        ++c;
      }
    }
  }
  if (lane == 0) {
    sstart[nch] = s;
    if (stats) {
      stats[0] += n_uniform;
      stats[1] += n_batches;
      stats[2] += n_slow;
    }
  }
}

// sstart of the chunks of groups the walk advanced in one step
__global__ void chunk_fill_kernel(int64_t nch, const long long* __restrict__ pexcl, const int* __restrict__ gE,
                                  const double* __restrict__ gs, double* __restrict__ sstart) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = c >> 5;
    const double s = gs[g];
    if (s == s) sstart[c] = __dadd_rn(s, __dmul_rn((double)pexcl[c], pow2(gE[g] - 52)));
  }
}

// Warp per draw: x = PCG64 output (off + i); j = first index whose
// normalised exact cumsum exceeds x (searchsorted side='right').
__global__ void draw_search_kernel(PView pv, int64_t nch, const double* __restrict__ sstart, tg_pcg64 rng,
                                   uint64_t off, int64_t k, int64_t* __restrict__ newidx) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= k) return;
  const u128 st = pcg_advance(u128{rng.state_hi, rng.state_lo}, u128{rng.inc_hi, rng.inc_lo}, off + (uint64_t)w + 1);
  const double x = pcg_double(st);
  const double L = sstart[nch];
  int64_t lo = 0, hi = nch - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (__ddiv_rn(sstart[mid + 1], L) > x)
      hi = mid;
    else
      lo = mid + 1;
  }
  double s = sstart[lo];
  const int64_t a = lo * SEL_CH, b = a + SEL_CH < pv.n ? a + SEL_CH : pv.n;
  int64_t j = b - 1;
  double pn = a + lane < b ? p_at(pv, a + lane) : 0.0;
  for (int64_t b0 = a; b0 < b; b0 += 32) {
    const double p = pn;
    pn = b0 + 32 + lane < b ? p_at(pv, b0 + 32 + lane) : 0.0;  // next step's load in flight
    double sl;
    const double s2 = warp_step(p, s, lane, &sl);
    const unsigned hit = __ballot_sync(FULL, b0 + lane < b && __ddiv_rn(sl, L) > x);
    if (hit) {
      j = b0 + __ffs(hit) - 1;
      break;
    }
    s = s2;
  }
  if (lane == 0) newidx[w] = j;
}

// keep first occurrences (np.unique return_index, sorted), append to found;
// zero them in p (bitmap) and take their scores out of the chunk sums
__global__ void dedup_append_kernel(const int64_t* __restrict__ newidx, int64_t k, int64_t* __restrict__ found,
                                    int64_t n_uniq, uint32_t* __restrict__ zmask, const double* __restrict__ scores,
                                    double* __restrict__ csum, long long* __restrict__ count) {
  __shared__ int s_cnt;
  __shared__ int wsum[32];
  extern __shared__ int64_t s_new[];  // k candidates when they fit (else read from global)
  const bool staged = k <= 6144;
  if (threadIdx.x == 0) s_cnt = 0;
  if (staged)
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) s_new[i] = newidx[i];
  __syncthreads();
  const int64_t* cand = staged ? s_new : newidx;
  for (int64_t base = 0; base < k; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool keep = false;
    int64_t v = 0;
    if (i < k) {
      v = cand[i];
      keep = true;
      for (int64_t q = 0; q < i; ++q)
        if (cand[q] == v) {
          keep = false;
          break;
        }
    }
    const unsigned m = __ballot_sync(FULL, keep);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    int before = 0;
    for (int q = 0; q < w; ++q) before += wsum[q];
    const int rank = s_cnt + before + __popc(m & ((1u << lane) - 1));
    if (keep) {
      found[n_uniq + rank] = v;
      atomicOr(zmask + (v >> 5), 1u << (v & 31));
      atomicAdd(csum + v / SEL_CH, -scores[v]);
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
// numpy fancy assignment scores[idx] = v: for a repeated eid the LAST batch
// position wins.  vals holds either logits (final = 0: Eq. 10 on the device,
// exp within 1 ulp of numpy's) or the caller's finished sigmoid + gamma
// values (final = 1: the reference's own host arithmetic, bit-exact).
__device__ __forceinline__ double eq10(double x, double gamma, int final_vals) {
  if (final_vals) return x;
  const double ex = exp(-fabs(x));
  const double sg = x >= 0.0 ? 1.0 / (1.0 + ex) : ex / (1.0 + ex);
  return sg + gamma;
}

constexpr int SCATTER_MAX = 4096;  // one CTA sorts (eid, position) keys in shared memory

// b <= SCATTER_MAX: bitonic sort of (eid - base) << 12 | i, then the last
// key of every equal-eid run (its largest position) writes.
__global__ void __launch_bounds__(1024) scatter_last_sorted_kernel(double* __restrict__ scores,
                                                                   const int64_t* __restrict__ eids, int b,
                                                                   int64_t base, const double* __restrict__ vals,
                                                                   double gamma, int final_vals) {
  __shared__ unsigned long long key[SCATTER_MAX];
  int P = 1;
  while (P < b) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x)
    key[i] = i < b ? ((unsigned long long)(eids[i] - base) << 12) | (unsigned)i : ~0ull;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = key[i], c = key[l];
          if (((i & k) == 0) == (a > c)) {
            key[i] = c;
            key[l] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    const unsigned long long e = key[i] >> 12;
    if (i + 1 < b && (key[i + 1] >> 12) == e) continue;
    const int pos = (int)(key[i] & 4095u);
    scores[e] = eq10(vals[pos], gamma, final_vals);
  }
}

// larger batches: each position checks for a later duplicate (O(b^2) reads)
__global__ void update_scores_kernel(double* __restrict__ scores, int64_t n, const int64_t* __restrict__ eids,
                                     int64_t b, int64_t base, const double* __restrict__ vals, double gamma,
                                     int final_vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = eids[i];
    bool last = true;
    for (int64_t j = i + 1; j < b; ++j)
      if (eids[j] == e) {
        last = false;
        break;
      }
    if (!last) continue;
    scores[e - base] = eq10(vals[i], gamma, final_vals);
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
  const int64_t zwords = (n + 31) / 32;
  // one stream-ordered workspace (p is never materialised: p_at divides on the fly)
  const int64_t ng = (nch + 31) / 32;
  const size_t bytes = (size_t)Q * 8 + (size_t)zwords * 4 + (size_t)nch * (8 + 8 + 8 + 4 + 8) + (size_t)(nch + 1) * 8 +
                       (size_t)ng * (8 + 4 + 8) + (size_t)nch * 4 + (size_t)SEL_SLOTS * SEL_CH * 8 + 16 +
                       (size_t)b * 8 * 2 + 128 + 20 * 16;  // + alignment slack of the sub-buffers
  unsigned char* ws = nullptr;
  {
    // keep freed stream-ordered memory in the device's default pool so the
    // per-call workspace (tens of MB at GDELT size) is not re-mapped each time
    static thread_local int pooled_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev != pooled_dev) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = 1ull << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pooled_dev = dev;
    }
  }
  TG_CUDA(cudaMallocAsync(&ws, bytes, st));
  unsigned char* q = ws;
  auto take = [&](size_t sz) {
    unsigned char* r = q;
    q += (sz + 15) & ~size_t(15);
    return r;
  };
  double* val = reinterpret_cast<double*>(take((size_t)Q * 8));
  uint32_t* zmask = reinterpret_cast<uint32_t*>(take((size_t)zwords * 4));
  double* csum = reinterpret_cast<double*>(take((size_t)nch * 8));
  double* astart = reinterpret_cast<double*>(take((size_t)nch * 8));
  long long* dinc = reinterpret_cast<long long*>(take((size_t)nch * 8));
  int* ebin = reinterpret_cast<int*>(take((size_t)nch * 4));
  double* sstart = reinterpret_cast<double*>(take((size_t)(nch + 1) * 8));
  long long* pexcl = reinterpret_cast<long long*>(take((size_t)nch * 8));
  long long* gtot = reinterpret_cast<long long*>(take((size_t)ng * 8));
  int* gE = reinterpret_cast<int*>(take((size_t)ng * 4));
  double* gs = reinterpret_cast<double*>(take((size_t)ng * 8));
  int* pslot = reinterpret_cast<int*>(take((size_t)nch * 4));
  double* pbuf = reinterpret_cast<double*>(take((size_t)SEL_SLOTS * SEL_CH * 8));
  int* nslots = reinterpret_cast<int*>(take(16));
  int64_t* found = reinterpret_cast<int64_t*>(take((size_t)b * 8));
  int64_t* newidx = reinterpret_cast<int64_t*>(take((size_t)b * 8));
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(take(128));  // npos, nneg, count, walk stats[9]
  auto done = [&](int r) {
    cudaFreeAsync(ws, st);
    return r;
  };
  TG_CUDA(cudaMemsetAsync(zmask, 0, (size_t)zwords * 4, st));
  TG_CUDA(cudaMemsetAsync(csum, 0, (size_t)nch * 8, st));
  TG_CUDA(cudaMemsetAsync(flags, 0, 128, st));
  // total = scores.sum() in numpy's pairwise order (+ chunk sums, sign counts)
  pw_leaf8_kernel<<<grid_for(Q * 8), 256, 0, st>>>(scores, n, depth, val, csum, flags);
  TG_LAUNCHED();
  for (int lvl = depth - 1; lvl >= 0; --lvl) {
    pw_combine_kernel<<<grid_for((int64_t)1 << lvl), 256, 0, st>>>(n, depth, lvl, val);
    TG_LAUNCHED();
  }
  double T = 0.0;
  unsigned long long hf[2] = {0, 0};
  TG_CUDA(cudaMemcpyAsync(&T, val, 8, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaMemcpyAsync(hf, flags, 16, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaStreamSynchronize(st));
  // numpy choice(): p = scores / T; NaN, negative and non-zero checks on p
  const bool nan = !(T == T) || T == 0.0 || std::isinf(T);
  if (nan) return done(fail(TG_EVALUE, "probabilities contain NaN"));
  const unsigned long long pos = T > 0 ? hf[0] : hf[1], neg = T > 0 ? hf[1] : hf[0];
  if (neg) return done(fail(TG_EVALUE, "probabilities are not non-negative"));
  if ((int64_t)pos < b) return done(fail(TG_EVALUE, "Fewer non-zero entries in p than size"));
  const PView pv{scores, zmask, T, 1.0 / T, n};
  int rc = TG_OK;
  int64_t n_uniq = 0;
  uint64_t off = 0;
  while (n_uniq < b) {
    const int64_t k = b - n_uniq;
    chunk_scan_kernel<<<1, 1024, 0, st>>>(csum, nch, astart);
    TG_LAUNCHED();
    TG_CUDA(cudaMemsetAsync(pslot, 0xFF, (size_t)nch * 4, st));
    TG_CUDA(cudaMemsetAsync(nslots, 0, 4, st));
    chunk_classify_kernel<<<grid_for(nch * 32), 256, 0, st>>>(pv, nch, astart, csum, dinc, ebin, pslot, pbuf,
                                                              nslots);
    TG_LAUNCHED();
    chunk_group_kernel<<<grid_for(ng * 32), 256, 0, st>>>(nch, dinc, ebin, pexcl, gtot, gE);
    TG_LAUNCHED();
    chunk_walk_kernel<<<1, 32, 0, st>>>(pv, nch, dinc, ebin, gtot, gE, gs, sstart, pslot, pbuf, flags + 3);
    TG_LAUNCHED();
    chunk_fill_kernel<<<grid_for(nch), 256, 0, st>>>(nch, pexcl, gE, gs, sstart);
    TG_LAUNCHED();
    draw_search_kernel<<<(unsigned)((k * 32 + 255) / 256), 256, 0, st>>>(pv, nch, sstart, *rng, off, k, newidx);
    TG_LAUNCHED();
    dedup_append_kernel<<<1, 1024, k <= 6144 ? (size_t)k * 8 : 0, st>>>(
        newidx, k, found, n_uniq, zmask, scores, csum, reinterpret_cast<long long*>(flags + 2));
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
  if (getenv("TG_SELECT_STATS")) {
    unsigned long long ws3[3] = {0, 0, 0};
    cudaMemcpyAsync(ws3, flags + 3, 24, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "tg_select_batch: n=%lld chunks=%lld groups=%lld rounds_draws=%llu uniform_steps=%llu "
            "chunk_batches=%llu slow_chunks=%llu\n",
            (long long)n, (long long)nch, (long long)ng, (unsigned long long)off, ws3[0], ws3[1], ws3[2]);
  }
  if (rc == TG_OK) {
    rank_sort_kernel<<<grid_for(b), 256, 0, st>>>(found, b, base, out);
    TG_LAUNCHED();
  }
  return done(rc);
}

static int scatter_scores(double* scores, int64_t n, const int64_t* eids, int64_t b, int64_t base,
                          const double* vals, double gamma, int final_vals, void* stream) {
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
  if (b <= SCATTER_MAX)
    scatter_last_sorted_kernel<<<1, 1024, 0, st>>>(scores, eids, (int)b, base, vals, gamma, final_vals);
  else
    update_scores_kernel<<<grid_for(b), 256, 0, st>>>(scores, n, eids, b, base, vals, gamma, final_vals);
  TG_LAUNCHED();
  return TG_OK;
}

extern "C" int tg_update_scores(double* scores, int64_t n, const int64_t* eids, int64_t b, int64_t base,
                                const double* logits, double gamma, void* stream) {
  return scatter_scores(scores, n, eids, b, base, logits, gamma, 0, stream);
}

extern "C" int tg_scatter_scores(double* scores, int64_t n, const int64_t* eids, int64_t b, int64_t base,
                                 const double* values, void* stream) {
  return scatter_scores(scores, n, eids, b, base, values, 0.0, 1, stream);
}
