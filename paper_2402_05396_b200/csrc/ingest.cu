// Event-file ingest on the device: graph.py:159-205
// ingest_events reads "src,dst,ts[,f1..fde]" lines one by one in Python --
// hours for a GDELT-sized file.  Here the raw bytes go to HBM once and:
//
//   1. line terminators are found in parallel (Python text mode: "\n",
//      "\r\n" and a lone "\r" all end a line) and compacted in order;
//   2. a warp per line strips it, skips blank / '#' lines, and counts
//      fields; the data lines get their output row by a prefix sum;
//   3. a warp per data line splits the fields (comma ballots over 32-byte
//      windows) and its lanes parse them with CPython's int()/float()
//      semantics (decimal.cuh: correctly rounded Eisel-Lemire), narrowing
//      feature values to f32 like np.array(feats, dtype=np.float32).
//
// The first failing line (in file order) and the first failing check in
// Python's order -- field count, int, int, float, features left to right,
// finite timestamp, feature width -- are reported, so the host can raise
// the reference's DataError text for that line.
#include <cub/cub.cuh>

#include "common.cuh"
#include "decimal.cuh"

namespace tg {

constexpr int ING_BYTES = 4096;  // bytes per block in the terminator scan

__device__ __forceinline__ bool is_term(const char* t, int64_t n, int64_t i) {
  const char c = t[i];
  return c == '\n' || (c == '\r' && (i + 1 >= n || t[i + 1] != '\n'));
}

__global__ void term_count_kernel(const char* __restrict__ t, int64_t n, int64_t* __restrict__ cnt) {
  const int64_t lo = (int64_t)blockIdx.x * ING_BYTES;
  int c = 0;
  for (int64_t i = lo + threadIdx.x; i < lo + ING_BYTES && i < n; i += blockDim.x) c += is_term(t, n, i);
  typedef cub::BlockReduce<int, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const int tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

// line ends in order: block b writes its terminators after the exclusive prefix
__global__ void term_write_kernel(const char* __restrict__ t, int64_t n, const int64_t* __restrict__ base,
                                  int64_t* __restrict__ ends) {
  const int64_t lo = (int64_t)blockIdx.x * ING_BYTES;
  typedef cub::BlockScan<int, 256> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t run;
  if (threadIdx.x == 0) run = base[blockIdx.x];
  __syncthreads();
  for (int64_t i0 = lo; i0 < lo + ING_BYTES && i0 < n; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const int f = (i < n && i < lo + ING_BYTES) ? is_term(t, n, i) : 0;
    int pos, tot;
    BS(tmp).ExclusiveSum(f, pos, tot);
    if (f) ends[run + pos] = i;
    __syncthreads();
    if (threadIdx.x == 0) run += tot;
    __syncthreads();
  }
}

struct LineSpan {
  int64_t a, b;  // stripped [a, b)
};

__device__ __forceinline__ LineSpan line_span(const char* t, int64_t n, const int64_t* ends, int64_t nterm, int64_t l) {
  int64_t a = l == 0 ? 0 : ends[l - 1] + 1;
  int64_t b = l < nterm ? ends[l] : n;
  while (a < b && dec::is_space(t[a])) ++a;
  while (b > a && dec::is_space(t[b - 1])) --b;
  return {a, b};
}

// warp per line: data flag, field count; first data line for the width
__global__ void line_classify_kernel(const char* __restrict__ t, int64_t n, const int64_t* __restrict__ ends,
                                     int64_t nterm, int64_t nlines, int* __restrict__ isdata, int* __restrict__ nf,
                                     unsigned long long* __restrict__ first_data) {
  const int lane = threadIdx.x & 31;
  for (int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < nlines;
       l += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const LineSpan sp = line_span(t, n, ends, nterm, l);
    const bool data = sp.b > sp.a && t[sp.a] != '#';
    int commas = 0;
    if (data)
      for (int64_t i = sp.a + lane; i < sp.b; i += 32) commas += t[i] == ',';
    commas = warp_sum(commas);
    if (lane == 0) {
      isdata[l] = data ? 1 : 0;
      nf[l] = data ? commas + 1 : 0;
      if (data) atomicMin(first_data, (unsigned long long)l);
    }
  }
}

// warp per data line: split + parse.  err: min over lines of
// (line << 16) | check, check = field index for parse errors (Python's
// left-to-right order), 0xFFF0 non-finite ts, 0xFFF1 width, 0xFFF2 too few
// fields (checked first), 0xFFF3 > 19-digit value the fast path cannot
// decide, 0xFFF4 int out of int64 range.
constexpr int ERR_FEW = 0xFFEF, ERR_NONFINITE = 0xFFF0, ERR_WIDTH = 0xFFF1, ERR_UNSUP = 0xFFF3, ERR_RANGE = 0xFFF4;

__global__ void line_parse_kernel(const char* __restrict__ t, int64_t n, const int64_t* __restrict__ ends,
                                  int64_t nterm, int64_t nlines, const int* __restrict__ isdata,
                                  const int* __restrict__ nf, const int* __restrict__ row, int width,
                                  int64_t* __restrict__ src, int64_t* __restrict__ dst, double* __restrict__ ts,
                                  float* __restrict__ feats, int64_t feat_ld, unsigned long long* __restrict__ err,
                                  int64_t* __restrict__ unsup, int64_t unsup_cap,
                                  unsigned long long* __restrict__ n_unsup) {
  constexpr int MAXF = 1024;  // fields per line held in shared memory per warp
  __shared__ int s_start[8][MAXF + 1];  // field starts relative to the stripped line
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int* fs = s_start[wib];
  for (int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < nlines;
       l += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (!isdata[l]) continue;
    const int nfl = nf[l];
    const LineSpan sp = line_span(t, n, ends, nterm, l);
    auto report = [&](int check) {
      atomicMin(err, ((unsigned long long)l << 16) | (unsigned)check);
    };
    if (nfl < 3) {
      if (lane == 0) report(ERR_FEW);
      continue;
    }
    if (nfl > MAXF) {  // more fields than the staging holds: treat as a width error
      if (lane == 0) report(ERR_WIDTH);
      continue;
    }
    // field starts: position after each comma, in order (ballot per 32 bytes)
    if (lane == 0) fs[0] = 0;
    int k = 1;
    for (int64_t i0 = sp.a; i0 < sp.b; i0 += 32) {
      const int64_t i = i0 + lane;
      const bool c = i < sp.b && t[i] == ',';
      const unsigned m = __ballot_sync(FULL, c);
      if (c) fs[k + __popc(m & ((1u << lane) - 1))] = (int)(i + 1 - sp.a);
      k += __popc(m);
    }
    if (lane == 0) fs[nfl] = (int)(sp.b - sp.a) + 1;  // sentinel: the end of the last field + 1
    __syncwarp();
    const int r = row[l];
    int bad = 0x7FFFFFFF;  // this lane's first failing check
    bool undecided = false;  // a > 19-digit value whose rounding the fast path cannot settle
    for (int f = lane; f < nfl; f += 32) {
      const char* p = t + sp.a + fs[f];
      const int len = fs[f + 1] - 1 - fs[f];
      if (f < 2) {
        int64_t v = 0;
        const int st = dec::parse_int(p, len, v);
        if (st == dec::OK) {
          if (f == 0) src[r] = v;
          else dst[r] = v;
        } else {
          bad = min(bad, st == dec::RANGE ? ERR_RANGE : f);
        }
      } else {
        uint64_t bits = 0;
        const int st = dec::parse_float(p, len, bits);
        if (st == dec::OK) {
          const double v = __longlong_as_double((long long)bits);
          if (f == 2) {
            ts[r] = v;
            if (!isfinite(v)) bad = min(bad, ERR_NONFINITE);
          } else if (f - 3 < width) {
            feats[(int64_t)r * feat_ld + (f - 3)] = __double2float_rn(v);
          }
        } else if (st == dec::UNSUPPORTED) {
          undecided = true;  // Python parses it: the host re-parses this line
        } else {
          bad = min(bad, f);
        }
      }
    }
    if (__any_sync(FULL, undecided) && lane == 0) {
      const unsigned long long k = atomicAdd(n_unsup, 1ull);
      if ((int64_t)k < unsup_cap) unsup[k] = l;
    }
    // Python parses every field before the finiteness and width checks
    int first = bad;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(FULL, first, o));
    if (lane == 0) {
      int check = first;  // a field's parse error (Python raises at the first), else:
      if (check == 0x7FFFFFFF && nfl - 3 != width) check = ERR_WIDTH;  // finite ts, then the width
      if (check != 0x7FFFFFFF) report(check);
    }
    __syncwarp();
  }
}

}  // namespace tg

using namespace tg;

extern "C" int tg_ingest_lines(const char* text, int64_t nbytes, int64_t* ends, int64_t* host_info, void* stream) {
  // host_info[0] = terminators, [1] = lines (terminated or a trailing
  // partial line); ends (may be NULL to only count) receives the terminator
  // offsets in order.
  host_info[0] = host_info[1] = 0;
  if (nbytes <= 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  const int64_t nb = (nbytes + ING_BYTES - 1) / ING_BYTES;
  int64_t* cnt = nullptr;
  TG_CUDA(cudaMallocAsync(&cnt, (size_t)(nb + 1) * 8 * 2, st));
  int64_t* base = cnt + nb + 1;
  term_count_kernel<<<(unsigned)nb, 256, 0, st>>>(text, nbytes, cnt);
  TG_LAUNCHED();
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, base, (int)nb + 1, st);
  void* tmp = nullptr;
  TG_CUDA(cudaMemsetAsync(cnt + nb, 0, 8, st));
  TG_CUDA(cudaMallocAsync(&tmp, tb, st));
  TG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, base, (int)nb + 1, st));
  int64_t total = 0;
  TG_CUDA(cudaMemcpyAsync(&total, base + nb, 8, cudaMemcpyDeviceToHost, st));
  if (ends) {
    term_write_kernel<<<(unsigned)nb, 256, 0, st>>>(text, nbytes, base, ends);
    TG_LAUNCHED();
  }
  char last = 0;
  TG_CUDA(cudaMemcpyAsync(&last, text + nbytes - 1, 1, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaFreeAsync(tmp, st));
  TG_CUDA(cudaFreeAsync(cnt, st));
  TG_CUDA(cudaStreamSynchronize(st));
  host_info[0] = total;
  host_info[1] = total + ((last == '\n' || last == '\r') ? 0 : 1);
  return TG_OK;
}

extern "C" int tg_ingest_classify(const char* text, int64_t nbytes, const int64_t* ends, int64_t nterm,
                                  int64_t nlines, int* isdata, int* nf, int* row, int64_t* host_info, void* stream) {
  // host_info[0] = data lines, [1] = first data line (-1 if none), [2] = its field count
  host_info[0] = 0;
  host_info[1] = -1;
  host_info[2] = 0;
  if (nlines <= 0) return TG_OK;
  const cudaStream_t st = as_stream(stream);
  unsigned long long* fd = nullptr;
  TG_CUDA(cudaMallocAsync(&fd, 16, st));
  TG_CUDA(cudaMemsetAsync(fd, 0xFF, 8, st));
  const int64_t warps = nlines;
  const int64_t want = (warps * 32 + 255) / 256;
  const int grid = (int)(want < (int64_t)device_sms() * 64 ? want : (int64_t)device_sms() * 64);
  line_classify_kernel<<<grid, 256, 0, st>>>(text, nbytes, ends, nterm, nlines, isdata, nf, fd);
  TG_LAUNCHED();
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, isdata, row, (int)nlines, st);
  void* tmp = nullptr;
  TG_CUDA(cudaMallocAsync(&tmp, tb, st));
  TG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, isdata, row, (int)nlines, st));
  int last_row = 0, last_data = 0;
  unsigned long long first = 0;
  TG_CUDA(cudaMemcpyAsync(&last_row, row + nlines - 1, 4, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaMemcpyAsync(&last_data, isdata + nlines - 1, 4, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaMemcpyAsync(&first, fd, 8, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaStreamSynchronize(st));
  host_info[0] = (int64_t)last_row + last_data;
  if (first != ~0ull) {
    host_info[1] = (int64_t)first;
    int nf0 = 0;
    TG_CUDA(cudaMemcpyAsync(&nf0, nf + first, 4, cudaMemcpyDeviceToHost, st));
    TG_CUDA(cudaStreamSynchronize(st));
    host_info[2] = nf0;
  }
  TG_CUDA(cudaFreeAsync(tmp, st));
  TG_CUDA(cudaFreeAsync(fd, st));
  TG_CUDA(cudaStreamSynchronize(st));
  return TG_OK;
}

extern "C" int tg_ingest_parse(const char* text, int64_t nbytes, const int64_t* ends, int64_t nterm, int64_t nlines,
                               const int* isdata, const int* nf, const int* row, int32_t width, int64_t* src,
                               int64_t* dst, double* ts, float* feats, int64_t feat_ld, int64_t* unsup,
                               int64_t unsup_cap, int64_t* host_err, void* stream) {
  // host_err[0] = first failing line (0-based) or -1, [1] = its check code,
  // [2] = lines with an undecidable value (their indices in unsup[0..cap))
  host_err[0] = -1;
  host_err[1] = 0;
  host_err[2] = 0;
  if (nlines <= 0) return TG_OK;
  if (width > 0 && feats == nullptr) return fail(TG_EVALUE, "feature buffer required (width %d)", width);
  const cudaStream_t st = as_stream(stream);
  unsigned long long* err = nullptr;
  TG_CUDA(cudaMallocAsync(&err, 16, st));
  TG_CUDA(cudaMemsetAsync(err, 0xFF, 8, st));
  TG_CUDA(cudaMemsetAsync(err + 1, 0, 8, st));
  const int64_t want = (nlines * 32 + 255) / 256;
  const int grid = (int)(want < (int64_t)device_sms() * 32 ? want : (int64_t)device_sms() * 32);
  line_parse_kernel<<<grid, 256, 0, st>>>(text, nbytes, ends, nterm, nlines, isdata, nf, row, width, src, dst, ts,
                                          feats, feat_ld, err, unsup, unsup ? unsup_cap : 0, err + 1);
  TG_LAUNCHED();
  unsigned long long h = 0, hu = 0;
  TG_CUDA(cudaMemcpyAsync(&h, err, 8, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaMemcpyAsync(&hu, err + 1, 8, cudaMemcpyDeviceToHost, st));
  TG_CUDA(cudaFreeAsync(err, st));
  TG_CUDA(cudaStreamSynchronize(st));
  if (h != ~0ull) {
    host_err[0] = (int64_t)(h >> 16);
    host_err[1] = (int64_t)(h & 0xFFFF);
  }
  host_err[2] = (int64_t)hu;
  return TG_OK;
}
