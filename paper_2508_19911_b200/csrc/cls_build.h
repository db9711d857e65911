// cls_build.h -- host tables of the CGKS-5th reconstruction (product path).
#pragma once
#include <cstdio>

namespace cgks {

constexpr int MAXB = 34;   // quartic basis size in 3-D
constexpr int MAXC = 18;   // face + edge neighbours in 3-D
constexpr int MAXL = 45;   // least-squares rows in 3-D
constexpr int MAXD = 63;   // data vector length in 3-D

struct ClsTables {
  int dim, nb, nc, nface, nl, nd;
  int expo[MAXB][3];        // basis exponents d
  int nbr[MAXC][3];         // neighbour offsets (faces first)
  int lsrow_cell[MAXL];     // LS row -> neighbour index (-1 = own cell)
  double lsrow_dir[MAXL][3];
  double R[MAXB * MAXD];    // coefficients = R . data   (row-major nb x nd)
  double avg0[MAXB];        // own-cell average of delta^d/d!
  double cond_estimate;
};

bool build_cls(int dim, ClsTables& T, char* err, int errlen);
void basis_at(const ClsTables& T, const double x[3], double* val, double* der);

}  // namespace cgks
