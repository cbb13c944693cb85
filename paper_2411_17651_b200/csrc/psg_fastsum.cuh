// psg_fastsum.cuh — exact closed form of repeated FP64 additions.
//
// A decode-only run adds the same per-iteration cost to the clock / energy /
// flops / bytes accumulators k times (simulator.cpp:125-133 over the
// iterations of one batch, batching.cpp:78-93).  The reference performs k
// sequential round-to-nearest additions; this header reproduces their result
// bit for bit in O(binade crossings) instead of O(k):
//
//   Let acc = m * u with u = ulp(acc) and m in [2^52, 2^53) (acc positive,
//   normal) and inc > 0 with s = inc / u (exact: a power-of-two scaling).
//   While the exact sum stays inside the binade, fl(acc + inc) = (m + R) * u
//   with R = round-to-nearest(s) — independent of m unless s is exactly a
//   half-integer (a tie, where round-half-even looks at m's parity: from an
//   even m every tied step adds R0 rounded up to even).  So t additions are
//   m + t*R as long as m + t*R + 1 < 2^53; the step that leaves the binade, a
//   tie from an odd m, zero/negative/subnormal operands and non-finite values
//   fall back to one plain addition.
//
// The simulation kernel caches segment_key() — R and the tie flag depend only
// on the increment and acc's exponent — per (batch size, accumulator) and
// runs a decode run as compose(m + t*R) with the arrival step from
// floor_div(); add_n() / advance_until() are the general multi-binade forms
// (tests, tools).  Host and device share this code so the CPU test
// (tests/test_cpu_fastsum.py) checks it against sequential stepping.
#pragma once
#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define PSG_HD __host__ __device__ __forceinline__
#else
#define PSG_HD inline
#include <string.h>
#endif

namespace psg {
namespace fastsum {

PSG_HD double add_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}

PSG_HD int64_t bits_of(double x) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(x);
#else
  int64_t b;
  memcpy(&b, &x, sizeof b);
  return b;
#endif
}

PSG_HD double of_bits(int64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(b);
#else
  double x;
  memcpy(&x, &b, sizeof x);
  return x;
#endif
}

constexpr int64_t kHidden = int64_t(1) << 52;
constexpr int64_t kTop = int64_t(1) << 53;

// One binade segment of acc += inc.  On success returns true with
// m = mantissa integer of acc (acc = m * 2^(ebits - 1075)) and R = the
// per-step mantissa increment; steps stay exact while m + t*R <= 2^53 - 2.
struct Segment {
  int64_t m, R, ebits;
};

PSG_HD bool segment(double acc, double inc, Segment& g) {
  const int64_t b = bits_of(acc);
  const int64_t eb = (b >> 52) & 0x7ff;
  if (b < 0 || eb == 0 || eb == 0x7ff) return false;  // negative / zero / subnormal / inf / nan
  const int64_t ib = bits_of(inc);
  const int64_t ie = (ib >> 52) & 0x7ff;
  if (ib <= 0 || ie == 0 || ie == 0x7ff) return false;  // inc <= 0 / subnormal / inf / nan
  // s = inc / u = inc * 2^(1075 - eb); compare exponents first so the scaling
  // never overflows or lands in the subnormal range with lost bits
  const int64_t shift = 1075 - eb;  // s = inc * 2^shift
  if (ie + shift >= 1023 + 52) return false;  // s >= 2^52: leaves the binade at once
  g.m = (b & (kHidden - 1)) | kHidden;
  g.ebits = eb;
  if (ie + shift < 1023 - 2) {  // s < 1/4: every addition rounds back to acc
    g.R = 0;
    return true;
  }
  const double s = of_bits(ib + shift * kHidden);  // exact power-of-two scaling (normal result)
  const double fl = floor(s);
  const double frac = s - fl;  // exact
  if (frac == 0.5) {
    // tie (s = R0 + 1/2): round-half-even makes the result even, and from an
    // even m every step adds R0 rounded up to even; an odd m takes one plain
    // step first
    if (g.m & 1) return false;
    const int64_t R0 = int64_t(fl);
    g.R = R0 + (R0 & 1);
    return true;
  }
  g.R = int64_t(frac > 0.5 ? fl + 1.0 : fl);  // exact: s < 2^52
  return true;
}

// The mantissa-independent part of segment(): for acc's binade (exponent
// field eb, normal positive acc) and inc, the per-step increment R and
// whether s = inc / ulp is a tie (then R holds only from an even mantissa).
// Cacheable per (inc, eb).  Returns false where segment() never applies.
PSG_HD bool segment_key(double acc, double inc, int64_t& eb, int64_t& R, bool& tie) {
  const int64_t b = bits_of(acc);
  eb = (b >> 52) & 0x7ff;
  if (b < 0 || eb == 0 || eb == 0x7ff) return false;
  tie = false;
  if (inc == 0.0 && bits_of(inc) == 0) {  // +0: every addition leaves acc as it is
    R = 0;
    return true;
  }
  const int64_t ib = bits_of(inc);
  const int64_t ie = (ib >> 52) & 0x7ff;
  if (ib <= 0 || ie == 0 || ie == 0x7ff) return false;
  const int64_t shift = 1075 - eb;
  if (ie + shift >= 1023 + 52) return false;
  if (ie + shift < 1023 - 2) {
    R = 0;
    return true;
  }
  const double s = of_bits(ib + shift * kHidden);
  const double fl = floor(s);
  const double frac = s - fl;
  const int64_t R0 = int64_t(fl);
  tie = frac == 0.5;
  R = tie ? R0 + (R0 & 1) : int64_t(frac > 0.5 ? fl + 1.0 : fl);
  return true;
}

PSG_HD double compose(int64_t m, int64_t ebits) {
  return of_bits((ebits << 52) | (m - kHidden));
}

// floor(a / b) for 0 <= a < 2^53, 1 <= b < 2^53.  Device: three rounds of
// an FP32-reciprocal quotient on the exact integer remainder (each round
// shrinks the error by ~2^-21), then an exact +-1 fix-up — no FP64 divide.
PSG_HD int64_t floor_div(int64_t a, int64_t b) {
#if defined(__CUDA_ARCH__)
  const float rf = __frcp_rn(float(b));
  int64_t q = int64_t(float(a) * rf);
  int64_t r = a - q * b;
  q += int64_t(float(r) * rf);
  r = a - q * b;
  q += int64_t(float(r) * rf);
  r = a - q * b;
  while (r < 0) { --q; r += b; }
  while (r >= b) { ++q; r -= b; }
  return q;
#else
  return a / b;
#endif
}

// t * R <= lim without overflow (t >= 0, R >= 1, -1 <= lim < 2^53).
PSG_HD bool fits(int64_t t, int64_t R, int64_t lim) {
  if (lim < 0) return false;
#if defined(__CUDA_ARCH__)
  if (__umul64hi(uint64_t(t), uint64_t(R)) != 0) return false;
#else
  if ((unsigned __int128)(uint64_t(t)) * uint64_t(R) >> 64) return false;
#endif
  return uint64_t(t) * uint64_t(R) <= uint64_t(lim);
}

// acc after k sequential additions of inc.
PSG_HD double add_n(double acc, double inc, int64_t k) {
  while (k > 0) {
    Segment g;
    if (segment(acc, inc, g)) {
      if (g.R == 0) return acc;
      const int64_t lim = kTop - 2 - g.m;
      if (fits(k, g.R, lim)) return compose(g.m + k * g.R, g.ebits);
      const int64_t t = lim > 0 ? floor_div(lim, g.R) : 0;
      if (t > 0) {
        acc = compose(g.m + t * g.R, g.ebits);
        k -= t;
        continue;
      }
    } else if (inc == 0.0 && !(acc != acc)) {
      return add_rn(acc, inc);  // one step reaches the fixed point (-0 + 0 = +0)
    }
    acc = add_rn(acc, inc);
    --k;
  }
  return acc;
}

// The clock of a decode run: runs iterations j = 0, 1, ... while j < kmax and
// the iteration's start clock is < a; returns the number of iterations run,
// clock advanced accordingly.
PSG_HD int64_t advance_until(double& clock, double d, int64_t kmax, double a) {
  int64_t j = 0;
  double c = clock;
  while (j < kmax && c < a) {
    Segment g;
    if (segment(c, d, g)) {
      if (g.R == 0) {  // the clock never moves again; c < a stays true
        clock = c;
        return kmax;
      }
      const int64_t lim = kTop - 2 - g.m;
      int64_t t = kmax - j;
      if (!fits(t, g.R, lim)) t = lim > 0 ? floor_div(lim, g.R) : 0;
      // a inside this binade: a = M * u exactly (a > c >= 2^e, same ulp);
      // stop at the first step with m + jR >= M
      const int64_t ab = bits_of(a);
      if (t > 0 && ((ab >> 52) & 0x7ff) == g.ebits) {
        const int64_t gap = ((ab & (kHidden - 1)) | kHidden) - g.m;  // > 0
        if (t * g.R >= gap) t = floor_div(gap - 1, g.R) + 1;
      }
      if (t > 0) {
        c = compose(g.m + t * g.R, g.ebits);
        j += t;
        continue;
      }
    }
    c = add_rn(c, d);
    ++j;
  }
  clock = c;
  return j;
}

}  // namespace fastsum
}  // namespace psg
