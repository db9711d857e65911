// per-phase algorithmic flop tally of one flux point (host only; nvcc exp/flop_phases.cu)
#include <cstdio>
#include "../paper_2508_19911_b200/csrc/flop_count.h"
#include "../paper_2508_19911_b200/csrc/gks_flux.cuh"
using namespace cgks;
struct XM { fc::CD operator()(const fc::CD& x) const { return x; } bool flag(bool b) const { return b; } };
struct PH { fc::CD* s; double* m; void put(int i, const fc::CD& v) const { s[i] = v; } fc::CD get(int i) const { return s[i]; }
  void mark(int k) const { m[k] = fc::tally().flops; } };
int main() {
  using fc::CD;
  FluxConst f{1.4, 2.0, 1e-3, 0.72, 0.05, 10.0, 10.0, 1 / 0.72 - 1, 0.0};
  CD W[5], dW[3][5];
  const double w0[5] = {1.0, 0.3, -0.2, 0.1, 2.7};
  for (int i = 0; i < 5; ++i) { W[i] = CD::run(w0[i]); for (int d = 0; d < 3; ++d) dW[d][i] = CD::run(0.01 * (i + 1) * (d + 1)); }
  GPOutT<CD> o; CD slots[40]; double marks[6] = {0};
  fc::tally() = fc::Tally();
  gks_flux_side<true>(0, W, dW, CD::run(1e-3), CD::run(1e3), f, XM(), PH{slots, marks}, o);
  auto t = fc::tally();
  printf("S phase %.0f  G phase %.0f  relax %.0f  total %.0f (fma %.0f add %.0f mul %.0f div %.0f special %.0f sqrt %.0f)\n",
         marks[1], marks[5] - marks[1], t.flops - marks[5], t.flops, t.fmas, t.adds, t.muls, t.divs, t.special, t.sqrts);
}
