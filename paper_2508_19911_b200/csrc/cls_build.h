// cls_build.h -- host tables of the CGKS-5th reconstruction (product path).
#pragma once
#include <cstdio>

namespace cgks {

constexpr int MAXB = 34;   // quartic basis size in 3-D
constexpr int MAXC = 18;   // face + edge neighbours in 3-D
constexpr int MAXL = 54;   // least-squares rows in 3-D (45; 54 with the 12 own-cell line rows)
constexpr int MAXD = 72;   // data vector length in 3-D (63; 72 with line DOFs)

struct ClsTables {
  int dim, nb, nc, nface, nl, nd;
  int expo[MAXB][3];        // basis exponents d
  int nbr[MAXC][3];         // neighbour offsets (faces first)
  int lsrow_cell[MAXL];     // LS row -> neighbour index (-1 = own cell)
  double lsrow_dir[MAXL][3];
  int lsrow_line[MAXL];     // >= 0: own-cell line-averaged derivative l (line DOFs), direction axis
  int lsrow_axis[MAXL];
  double lsrow_t[MAXL][3];  // transverse position of the line (reference units)
  int lines;                // 1: line-DOF variant
  double R[MAXB * MAXD];    // coefficients = R . data   (row-major nb x nd)
  double avg0[MAXB];        // own-cell average of delta^d/d!
  double cond_estimate;
};

// lines = 1: the own cell's line-averaged derivatives (at the transverse face Gauss points) replace its
// gradient as LS data
bool build_cls(int dim, ClsTables& T, char* err, int errlen, int lines = 0);
void basis_at(const ClsTables& T, const double x[3], double* val, double* der);

}  // namespace cgks
