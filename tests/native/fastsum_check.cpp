// CPU check of psg_fastsum.cuh against sequential round-to-nearest additions
// (tests/test_cpu_fastsum.py builds and runs this).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "psg_fastsum.cuh"

using psg::fastsum::add_n;
using psg::fastsum::advance_until;

// segment_key (the kernel's per-(inc, binade) cache of R) must reproduce
// segment(): same R wherever segment() applies, and a tie flag exactly where
// segment() refuses an odd mantissa.
// The simulation kernel's closed-form decode run (psg_sim.cu, cached segment
// keys): iterations j = 0.. while j < kmax and the start clock is below a,
// the clock advanced in one multiply-add; false where the kernel steps
// serially instead.
static bool kernel_closed_form(double clock, double d, long kmax, double a, double& out, long& j) {
  int64_t eb = 0, R = 0;
  bool tie = false;
  if (!psg::fastsum::segment_key(clock, d, eb, R, tie) || R >= (int64_t(1) << 52)) return false;
  int64_t bits;
  std::memcpy(&bits, &clock, sizeof bits);
  const int64_t m = (bits & (psg::fastsum::kHidden - 1)) | psg::fastsum::kHidden;
  if (tie && (m & 1)) return false;
  if (R > 0 && !psg::fastsum::fits(kmax, R, psg::fastsum::kTop - 2 - m)) return false;
  long t = kmax;
  if (!(clock < a)) {
    t = 0;
  } else if (R > 0) {
    int64_t ab;
    std::memcpy(&ab, &a, sizeof ab);
    if ((ab >> 52) == (bits >> 52)) {
      const int64_t gap = ((ab & (psg::fastsum::kHidden - 1)) | psg::fastsum::kHidden) - m;
      const int64_t ta = psg::fastsum::floor_div(gap - 1, R) + 1;
      t = ta < t ? long(ta) : t;
    }
  }
  j = t;
  out = R > 0 ? psg::fastsum::compose(m + t * R, eb) : clock;
  return true;
}

static bool key_agrees(double acc, double inc) {
  psg::fastsum::Segment g{0, 0, 0};
  const bool ok = psg::fastsum::segment(acc, inc, g);
  int64_t eb = 0, R = 0;
  bool tie = false;
  const bool kok = psg::fastsum::segment_key(acc, inc, eb, R, tie);
  if (inc == 0.0 && !std::signbit(inc) && acc > 0 && std::isnormal(acc)) return kok && R == 0 && !tie;
  if (!kok) return !ok;
  int64_t bits;
  std::memcpy(&bits, &acc, sizeof bits);
  const bool odd = bits & 1;
  if (tie && odd) return !ok;
  return ok && g.R == R && g.ebits == eb;
}

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

int main(int argc, char** argv) {
  const long cases = argc > 1 ? std::atol(argv[1]) : 20000;
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  long bad = 0, fast_steps = 0, kernel_cf = 0;
  auto pick = [&](double lo_exp, double hi_exp) {
    double v = std::ldexp(1.0 + U(rng), int(lo_exp + (hi_exp - lo_exp) * U(rng)));
    switch (rng() % 8) {
      case 0: v = std::ldexp(std::floor(v * 1024) / 1024, 0); break;  // few mantissa bits: ties
      case 1: v = std::ldexp(1.0, int(lo_exp + (hi_exp - lo_exp) * U(rng))); break;
      default: break;
    }
    return v;
  };
  for (long c = 0; c < cases; ++c) {
    double acc = (rng() % 10 == 0) ? 0.0 : pick(-30, 60);
    double inc = (rng() % 20 == 0) ? 0.0 : pick(-40, 40);
    if (rng() % 4 == 0) {  // integer-valued accumulators (flops / bytes): frequent ties
      acc = std::floor(std::ldexp(1.0 + U(rng), 40 + int(rng() % 25)));
      inc = std::ldexp(double(1 + rng() % 4096), int(rng() % 20));
    }
    if (rng() % 50 == 0) inc = -inc;
    const long k = long(rng() % 5000);
    if (!key_agrees(acc, inc) || !key_agrees(inc, acc)) {
      if (bad < 10) std::printf("segment_key acc=%a inc=%a\n", acc, inc);
      ++bad;
    }
    // add_n
    double ref = acc;
    for (long i = 0; i < k; ++i) ref = ref + inc;
    const double got = add_n(acc, inc, k);
    if (!same(ref, got)) {
      if (bad < 10) std::printf("add_n acc=%a inc=%a k=%ld ref=%a got=%a\n", acc, inc, k, ref, got);
      ++bad;
    }
    fast_steps += k;
    // advance_until with an arrival
    if (inc >= 0) {
      double a;
      switch (rng() % 4) {
        case 0: a = INFINITY; break;
        case 1: a = ref; break;                   // exactly a reachable clock value
        case 2: a = acc + (ref - acc) * U(rng); break;
        default: a = std::nextafter(ref, 0.0); break;
      }
      double rc = acc;
      long rj = 0;
      while (rj < k && rc < a) { rc = rc + inc; ++rj; }
      double kc = 0.0;
      long kj = 0;
      const bool kok = acc > 0 && kernel_closed_form(acc, inc, k, a, kc, kj);
      kernel_cf += kok;
      if (kok && (kj != rj || !same(kc, rc))) {
        if (bad < 10)
          std::printf("kernel closed form acc=%a d=%a k=%ld a=%a ref=(%ld,%a) got=(%ld,%a)\n", acc, inc, k, a,
                      rj, rc, kj, kc);
        ++bad;
      }
      double gc = acc;
      const long gj = long(advance_until(gc, inc, k, a));
      if (gj != rj || !same(gc, rc)) {
        if (bad < 10)
          std::printf("advance acc=%a d=%a k=%ld a=%a ref=(%ld,%a) got=(%ld,%a)\n", acc, inc, k, a, rj,
                      rc, gj, gc);
        ++bad;
      }
    }
  }
  // targeted ties / half-ulp increments / binade edges
  const double accs[] = {1.0, 1.0 + 0x1p-52, 1.5, 2.0 - 0x1p-52, 0x1p30 - 1.0, 3.0};
  const double incs[] = {0x1p-53, 3 * 0x1p-53, 0x1p-54, 1.5 * 0x1p-52, 0x1p-52, 0.25, 1.0 / 3, 0x1p-60};
  for (double a0 : accs)
    for (double d : incs)
      for (int sh = -70; sh <= 70; ++sh)
        for (double a1 : {a0, std::nextafter(a0, 4 * a0)})  // both mantissa parities
          if (!key_agrees(std::ldexp(a1, sh), d)) {
            if (bad < 20) std::printf("edge segment_key acc=%a inc=%a\n", std::ldexp(a1, sh), d);
            ++bad;
          }
  for (double a0 : accs)
    for (double d : incs)
      for (long k = 0; k < 3000; k += 1 + k / 7) {
        double ref = a0;
        for (long i = 0; i < k; ++i) ref = ref + d;
        const double got = add_n(a0, d, k);
        if (!same(ref, got)) {
          if (bad < 20) std::printf("edge add_n acc=%a inc=%a k=%ld ref=%a got=%a\n", a0, d, k, ref, got);
          ++bad;
        }
        double gc = a0;
        const long gj = long(advance_until(gc, d, k, ref));
        double rc = a0;
        long rj = 0;
        while (rj < k && rc < ref) { rc = rc + d; ++rj; }
        if (gj != rj || !same(gc, rc)) {
          if (bad < 20) std::printf("edge advance acc=%a d=%a k=%ld\n", a0, d, k);
          ++bad;
        }
      }
  std::printf("cases=%ld steps=%ld kernel_closed_form=%ld bad=%ld\n", cases, fast_steps, kernel_cf, bad);
  return bad ? 1 : 0;
}
