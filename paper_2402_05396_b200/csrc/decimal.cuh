// Decimal text -> binary64 exactly as CPython's float() / int() read the
// fields of an event file (graph.py:159-205 ingest_events).  Host + device.
//
// float(): optional whitespace, sign, "inf"/"infinity"/"nan" (any case), or
// digits with single underscores between digits, optional fraction and
// exponent.  The value is rounded correctly (ties to even) with the
// Eisel-Lemire algorithm: the 19-digit significand w times a 128-bit
// power of five (pow5_table.inc) -- a 128-bit product is always sufficient
// for w < 10^19 (Mushtak & Lemire 2023).  Inputs with more than 19
// significant digits are decided by evaluating the truncated significand
// w and w + 1; when those disagree the field is reported as unsupported
// (TG_EVALUE) instead of guessed -- shortest-repr text (what save_dataset
// writes, graph.py:231-236) never has more than 17 digits.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD inline
#endif

namespace tg {
namespace dec {

enum Status : int { OK = 0, BAD = 1, UNSUPPORTED = 2, RANGE = 3 };

#ifdef __CUDACC__
__constant__ uint64_t kPow5[] = {
#include "pow5_table.inc"
};
#else
static const uint64_t kPow5[] = {
#include "pow5_table.inc"
};
#endif

TG_HD uint64_t pow5_word(int i) {
#ifdef __CUDA_ARCH__
  return kPow5[i];
#else
  return kPow5[i];
#endif
}

TG_HD void mul128(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

TG_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

TG_HD bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }
TG_HD char lower(char c) { return (c >= 'A' && c <= 'Z') ? (char)(c + 32) : c; }

// Eisel-Lemire: w * 10^q (w != 0) -> IEEE bits (without sign)
TG_HD uint64_t eisel_lemire(uint64_t w, int64_t q) {
  if (w == 0 || q < -342) return 0;
  if (q > 308) return 0x7FF0000000000000ull;
  const int lz = clz64(w);
  w <<= lz;
  const int idx = 2 * (int)(q + 342);
  uint64_t hi, lo;
  mul128(w, pow5_word(idx), hi, lo);
  const uint64_t mask = 0xFFFFFFFFFFFFFFFFull >> (52 + 3);
  if ((hi & mask) == mask) {
    uint64_t h2, l2;
    mul128(w, pow5_word(idx + 1), h2, l2);
    lo += h2;
    if (h2 > lo) ++hi;
  }
  const int upper = (int)(hi >> 63);
  const int shift = upper + 64 - 52 - 3;
  uint64_t mant = hi >> shift;
  int32_t p2 = (int32_t)((((152170 + 65536) * q) >> 16) + 63) + upper - lz + 1023;
  if (p2 <= 0) {  // subnormal
    if (-p2 + 1 >= 64) return 0;
    mant >>= -p2 + 1;
    mant += (mant & 1);
    mant >>= 1;
    p2 = (mant < (1ull << 52)) ? 0 : 1;
    return ((uint64_t)p2 << 52) | (mant & ((1ull << 52) - 1));
  }
  if (lo <= 1 && q >= -4 && q <= 23 && (mant & 3) == 1) {  // exactly halfway: round to even
    if ((mant << shift) == hi) mant &= ~1ull;
  }
  mant += (mant & 1);
  mant >>= 1;
  if (mant >= (2ull << 52)) {
    mant = 1ull << 52;
    ++p2;
  }
  mant &= ~(1ull << 52);
  if (p2 >= 0x7FF) return 0x7FF0000000000000ull;
  return ((uint64_t)p2 << 52) | mant;
}

TG_HD bool match_word(const char* p, int n, const char* w) {
  int i = 0;
  for (; w[i]; ++i)
    if (i >= n || lower(p[i]) != w[i]) return false;
  return i == n;
}

// Python float(text[0:n]) -> bits.  Returns Status.
TG_HD int parse_float(const char* s, int n, uint64_t& bits) {
  int i = 0, e = n;
  while (i < e && is_space(s[i])) ++i;
  while (e > i && is_space(s[e - 1])) --e;
  if (i >= e) return BAD;
  uint64_t sign = 0;
  if (s[i] == '+' || s[i] == '-') {
    sign = s[i] == '-' ? (1ull << 63) : 0;
    ++i;
  }
  if (i >= e) return BAD;
  const char c0 = lower(s[i]);
  if (c0 == 'i' || c0 == 'n') {
    if (match_word(s + i, e - i, "inf") || match_word(s + i, e - i, "infinity")) {
      bits = sign | 0x7FF0000000000000ull;
      return OK;
    }
    if (match_word(s + i, e - i, "nan")) {
      bits = sign | 0x7FF8000000000000ull;
      return OK;
    }
    return BAD;
  }
  uint64_t w = 0;
  int nd = 0;          // significant digits consumed into w (<= 19)
  bool more = false;   // a non-zero digit beyond the 19th
  int64_t dexp = 0;    // decimal exponent adjustment
  int ndigits = 0;     // all digits seen (integer + fraction)
  bool prev_digit = false;
  // integer part
  while (i < e) {
    const char c = s[i];
    if (c >= '0' && c <= '9') {
      ++ndigits;
      if (nd < 19) {
        if (w || c != '0') {
          w = w * 10 + (uint64_t)(c - '0');
          ++nd;
        }
      } else {
        ++dexp;
        more |= c != '0';
      }
      prev_digit = true;
      ++i;
    } else if (c == '_') {
      if (!prev_digit || i + 1 >= e || s[i + 1] < '0' || s[i + 1] > '9') return BAD;
      prev_digit = false;
      ++i;
    } else {
      break;
    }
  }
  if (i < e && s[i] == '.') {
    ++i;
    prev_digit = false;
    bool first = true;
    while (i < e) {
      const char c = s[i];
      if (c >= '0' && c <= '9') {
        ++ndigits;
        if (nd < 19) {
          if (w || c != '0') {
            w = w * 10 + (uint64_t)(c - '0');
            ++nd;
          }
          --dexp;
        } else {
          more |= c != '0';
        }
        prev_digit = true;
        first = false;
        ++i;
      } else if (c == '_') {
        if (first || !prev_digit || i + 1 >= e || s[i + 1] < '0' || s[i + 1] > '9') return BAD;
        prev_digit = false;
        ++i;
      } else {
        break;
      }
    }
  }
  if (ndigits == 0) return BAD;
  if (i < e && (s[i] == 'e' || s[i] == 'E')) {
    ++i;
    bool eneg = false;
    if (i < e && (s[i] == '+' || s[i] == '-')) {
      eneg = s[i] == '-';
      ++i;
    }
    if (i >= e || s[i] < '0' || s[i] > '9') return BAD;
    int64_t ev = 0;
    bool pd = false;
    while (i < e) {
      const char c = s[i];
      if (c >= '0' && c <= '9') {
        if (ev < 100000000) ev = ev * 10 + (c - '0');
        pd = true;
        ++i;
      } else if (c == '_') {
        if (!pd || i + 1 >= e || s[i + 1] < '0' || s[i + 1] > '9') return BAD;
        pd = false;
        ++i;
      } else {
        break;
      }
    }
    dexp += eneg ? -ev : ev;
  }
  if (i != e) return BAD;
  if (w == 0) {
    bits = sign;
    return OK;
  }
  const uint64_t b0 = eisel_lemire(w, dexp);
  if (more) {  // truncated significand: w and w + 1 must round alike
    const uint64_t w1 = w + 1;
    const uint64_t b1 = (w1 == 10000000000000000000ull) ? eisel_lemire(1000000000000000000ull, dexp + 1)
                                                       : eisel_lemire(w1, dexp);
    if (b0 != b1) return UNSUPPORTED;
  }
  bits = sign | b0;
  return OK;
}

// Python int(text[0:n]) (base 10) into int64.  Returns Status.
TG_HD int parse_int(const char* s, int n, int64_t& out) {
  int i = 0, e = n;
  while (i < e && is_space(s[i])) ++i;
  while (e > i && is_space(s[e - 1])) --e;
  if (i >= e) return BAD;
  bool neg = false;
  if (s[i] == '+' || s[i] == '-') {
    neg = s[i] == '-';
    ++i;
  }
  if (i >= e) return BAD;
  uint64_t v = 0;
  bool prev_digit = false, any = false, over = false;
  while (i < e) {
    const char c = s[i];
    if (c >= '0' && c <= '9') {
      if (v > (0xFFFFFFFFFFFFFFFFull - 9) / 10) over = true;
      v = v * 10 + (uint64_t)(c - '0');
      prev_digit = any = true;
    } else if (c == '_') {
      if (!prev_digit || i + 1 >= e || s[i + 1] < '0' || s[i + 1] > '9') return BAD;
      prev_digit = false;
    } else {
      return BAD;
    }
    ++i;
  }
  if (!any) return BAD;
  if (over || v > (neg ? 0x8000000000000000ull : 0x7FFFFFFFFFFFFFFFull)) return RANGE;
  out = neg ? (int64_t)(0 - v) : (int64_t)v;
  return OK;
}

}  // namespace dec
}  // namespace tg
