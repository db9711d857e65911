// flop_count.h -- host-only counting scalar used to report the algorithmic FP64
// operation count of the device formulation (gks_flux.cuh instantiated with T = CD).
// Counting rules: + - * / count 1, fma counts 2, sqrt 1,
// each special function (exp, expm1, erfc, rsqrt) 1 and is also tallied separately.
// Operations whose operands are compile-time constants of the device code (literal
// values, multiplication by an exact 1 or 0, addition of an exact 0) are folded by
// the compiler and are not counted.
#pragma once
#include <cmath>

namespace cgks {
namespace fc {

struct Tally {
  double flops = 0, adds = 0, muls = 0, divs = 0, fmas = 0, special = 0, sqrts = 0;
};
inline Tally& tally() {
  static thread_local Tally t;
  return t;
}

struct CD {
  double v;
  bool k;  // known at compile time
  CD() : v(0.0), k(true) {}
  CD(double x) : v(x), k(true) {}
  static CD run(double x) {
    CD c(x);
    c.k = false;
    return c;
  }
};

inline CD add_(const CD& a, const CD& b, double r) {
  if (a.k && b.k) return CD(r);
  if (a.k && a.v == 0.0) return b.k ? CD(r) : CD::run(r);
  if (b.k && b.v == 0.0) return a.k ? CD(r) : CD::run(r);
  tally().adds += 1;
  tally().flops += 1;
  return CD::run(r);
}
inline CD operator+(const CD& a, const CD& b) { return add_(a, b, a.v + b.v); }
inline CD operator-(const CD& a, const CD& b) { return add_(a, b, a.v - b.v); }
inline CD operator-(const CD& a) { return a.k ? CD(-a.v) : CD::run(-a.v); }
inline CD operator*(const CD& a, const CD& b) {
  double r = a.v * b.v;
  if (a.k && b.k) return CD(r);
  if ((a.k && a.v == 0.0) || (b.k && b.v == 0.0)) return CD(0.0);
  if (a.k && (a.v == 1.0 || a.v == -1.0)) return CD::run(r);
  if (b.k && (b.v == 1.0 || b.v == -1.0)) return CD::run(r);
  tally().muls += 1;
  tally().flops += 1;
  return CD::run(r);
}
inline CD operator/(const CD& a, const CD& b) {
  double r = a.v / b.v;
  if (a.k && b.k) return CD(r);
  if (b.k && b.v == 1.0) return CD::run(r);
  tally().divs += 1;
  tally().flops += 1;
  return CD::run(r);
}
inline CD& operator+=(CD& a, const CD& b) { return a = a + b; }
inline CD& operator-=(CD& a, const CD& b) { return a = a - b; }
inline CD& operator*=(CD& a, const CD& b) { return a = a * b; }
inline bool operator>(const CD& a, const CD& b) { return a.v > b.v; }
inline bool operator<(const CD& a, const CD& b) { return a.v < b.v; }
inline bool operator!=(const CD& a, const CD& b) { return a.v != b.v; }
inline CD special_(double r) {
  tally().special += 1;
  tally().flops += 1;
  return CD::run(r);
}
inline CD exp(const CD& a) { return a.k ? CD(std::exp(a.v)) : special_(std::exp(a.v)); }
inline CD expm1(const CD& a) { return a.k ? CD(std::expm1(a.v)) : special_(std::expm1(a.v)); }
inline CD erfc(const CD& a) { return a.k ? CD(std::erfc(a.v)) : special_(std::erfc(a.v)); }
// erfc with the shared exp(-z^2) (gks_flux.cuh: erfc_e) counts as one special function
inline CD erfc_e(const CD& z, const CD& e) { return z.k ? CD(std::erfc(z.v)) : special_(std::erfc(z.v)); }
inline CD rsqrt_(const CD& a) { return a.k ? CD(1.0 / std::sqrt(a.v)) : special_(1.0 / std::sqrt(a.v)); }
inline CD sqrt(const CD& a) {
  if (a.k) return CD(std::sqrt(a.v));
  tally().sqrts += 1;
  tally().flops += 1;
  return CD::run(std::sqrt(a.v));
}
inline CD fmax(const CD& a, const CD& b) {  // a comparison: not counted
  return (a.k && b.k) ? CD(std::fmax(a.v, b.v)) : CD::run(std::fmax(a.v, b.v));
}
inline CD fabs(const CD& a) { return a.k ? CD(std::fabs(a.v)) : CD::run(std::fabs(a.v)); }
inline CD fma(const CD& a, const CD& b, const CD& c) { return a * b + c; }

}  // namespace fc
}  // namespace cgks
