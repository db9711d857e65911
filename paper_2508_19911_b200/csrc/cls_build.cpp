// cls_build.cpp -- host-side construction of the CGKS-5th reconstruction tables
// (product path; independent of oracle/).
//
// The compact quartic P^4 = Q_0 + sum_{1<=|d|<=4} a_d p_d is the
// constrained least-squares solution of Eq. (compact-big-5): the
// averages of the face and edge neighbours are matched exactly, the neighbour
// gradient data in the least-squares sense.  On a uniform mesh the map
// data -> coefficients is one matrix for all cells (reference cell).
// Here it is computed by the null-space method with Householder QR in long
// double (readings R1-R5 of DESIGN.md):
//   C a = d_c (exact rows), min |A a - d_a| (least-squares rows)
//   C^T = [Q1 Q2] [R1; 0],  a = Q1 R1^{-T} d_c + Q2 z,  z = (A Q2)^+ (d_a - A Q1 R1^{-T} d_c).
// Also builds the basis value/derivative tables at the face Gauss points.
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "cls_build.h"

namespace cgks {

namespace {

typedef long double ld;

ld fact(int k) {
  ld f = 1;
  for (int i = 2; i <= k; ++i) f *= i;
  return f;
}

// average over [o-1/2, o+1/2] of x^k
ld avg1(int o, int k) {
  ld a = o - 0.5L, b = o + 0.5L;
  ld pa = 1, pb = 1;
  for (int i = 0; i <= k; ++i) {
    pa *= a;
    pb *= b;
  }
  return (pb - pa) / (k + 1);
}

// average over the unit cell at offset o of delta^e / e!
ld mavg(const int o[3], const int e[3]) {
  ld r = 1;
  for (int a = 0; a < 3; ++a) r *= avg1(o[a], e[a]) / fact(e[a]);
  return r;
}

ld ipow(ld x, int k) {
  ld r = 1;
  for (int i = 0; i < k; ++i) r *= x;
  return r;
}

// Householder QR of an m x n matrix (column-major in a vector of vectors: M[col][row]).
// Returns the full orthogonal Q (m x m, Q[col][row]) and R (n columns of length m).
void householder_qr(int m, int n, std::vector<std::vector<ld>>& M, std::vector<std::vector<ld>>& Q) {
  Q.assign(m, std::vector<ld>(m, 0));
  for (int i = 0; i < m; ++i) Q[i][i] = 1;
  for (int k = 0; k < n && k < m; ++k) {
    ld nrm = 0;
    for (int i = k; i < m; ++i) nrm += M[k][i] * M[k][i];
    nrm = std::sqrt(nrm);
    if (nrm == 0) continue;
    ld alpha = M[k][k] > 0 ? -nrm : nrm;
    std::vector<ld> v(m, 0);
    for (int i = k; i < m; ++i) v[i] = M[k][i];
    v[k] -= alpha;
    ld vn = 0;
    for (int i = k; i < m; ++i) vn += v[i] * v[i];
    if (vn == 0) continue;
    // apply H = I - 2 v v^T / (v^T v) to remaining columns of M and accumulate Q = Q H
    for (int j = k; j < n; ++j) {
      ld s = 0;
      for (int i = k; i < m; ++i) s += v[i] * M[j][i];
      s = 2 * s / vn;
      for (int i = k; i < m; ++i) M[j][i] -= s * v[i];
    }
    for (int r = 0; r < m; ++r) {  // rows of Q: (Q H)[r][.]
      ld s = 0;
      for (int i = k; i < m; ++i) s += Q[i][r] * v[i];
      s = 2 * s / vn;
      for (int i = k; i < m; ++i) Q[i][r] -= s * v[i];
    }
  }
}

}  // namespace

bool build_cls(int dim, ClsTables& T, char* err, int errlen, int lines) {
  std::memset(&T, 0, sizeof(T));
  T.dim = dim;
  T.lines = lines;
  // basis multi-indices, degree 1..4 over the active axes
  int nb = 0;
  for (int s = 1; s <= 4; ++s)
    for (int i = s; i >= 0; --i)
      for (int j = s - i; j >= 0; --j) {
        int k = s - i - j;
        if ((dim < 2 && j) || (dim < 3 && k)) continue;
        T.expo[nb][0] = i;
        T.expo[nb][1] = j;
        T.expo[nb][2] = k;
        ++nb;
      }
  T.nb = nb;
  // neighbours: faces (-a, +a), then edges (pairs a<b, signs)
  int nc = 0;
  for (int a = 0; a < dim; ++a)
    for (int s = -1; s <= 1; s += 2) {
      T.nbr[nc][0] = T.nbr[nc][1] = T.nbr[nc][2] = 0;
      T.nbr[nc][a] = s;
      ++nc;
    }
  T.nface = nc;
  for (int a = 0; a < dim; ++a)
    for (int b = a + 1; b < dim; ++b)
      for (int sa = -1; sa <= 1; sa += 2)
        for (int sb = -1; sb <= 1; sb += 2) {
          T.nbr[nc][0] = T.nbr[nc][1] = T.nbr[nc][2] = 0;
          T.nbr[nc][a] = sa;
          T.nbr[nc][b] = sb;
          ++nc;
        }
  T.nc = nc;
  // least-squares rows: (cell index or -1 for own, reference direction)
  int nl = 0;
  auto add_row = [&](int cell, double d0, double d1, double d2) {
    T.lsrow_cell[nl] = cell;
    T.lsrow_dir[nl][0] = d0;
    T.lsrow_dir[nl][1] = d1;
    T.lsrow_dir[nl][2] = d2;
    T.lsrow_line[nl] = -1;
    ++nl;
  };
  for (int m = 0; m < T.nface; ++m)
    for (int a = 0; a < dim; ++a) add_row(m, a == 0, a == 1, a == 2);
  const double r2 = 1.0 / std::sqrt(2.0);
  for (int n = T.nface; n < nc; ++n) {
    const int* o = T.nbr[n];
    if (dim == 2) {
      add_row(n, 1, 0, 0);
      add_row(n, 0, 1, 0);
    } else {
      int t = (o[0] == 0) ? 0 : (o[1] == 0 ? 1 : 2);
      add_row(n, t == 0, t == 1, t == 2);                   // along the shared edge (R2)
      add_row(n, o[0] * r2, o[1] * r2, o[2] * r2);         // towards the target centroid (R2)
    }
  }
  if (!lines) {
    for (int a = 0; a < dim; ++a) add_row(-1, a == 0, a == 1, a == 2);  // own gradient (R1)
  } else {
    // own-cell line-averaged derivatives: per axis a, lines at the transverse Gauss points
    // g = p * n2 + q (p: sign along t1 = (a+1)%3, q: along t2 = (a+2)%3, active axes only)
    const double gq = 0.5 / std::sqrt(3.0);
    int l = 0;
    for (int a = 0; a < dim; ++a) {
      const int t1 = (a + 1) % 3, t2 = (a + 2) % 3;
      const int n1 = t1 < dim ? 2 : 1, n2 = t2 < dim ? 2 : 1;
      for (int p = 0; p < n1; ++p)
        for (int q = 0; q < n2; ++q, ++l) {
          add_row(-1, 0, 0, 0);
          T.lsrow_line[nl - 1] = l;
          T.lsrow_axis[nl - 1] = a;
          T.lsrow_t[nl - 1][0] = T.lsrow_t[nl - 1][1] = T.lsrow_t[nl - 1][2] = 0.0;
          if (t1 < dim) T.lsrow_t[nl - 1][t1] = p == 0 ? -gq : gq;
          if (t2 < dim) T.lsrow_t[nl - 1][t2] = q == 0 ? -gq : gq;
        }
    }
  }
  T.nl = nl;
  T.nd = nc + nl;

  const int zero[3] = {0, 0, 0};
  // C: nc x nb; A: nl x nb
  std::vector<std::vector<ld>> C(nc, std::vector<ld>(nb)), A(nl, std::vector<ld>(nb));
  for (int r = 0; r < nc; ++r)
    for (int k = 0; k < nb; ++k) C[r][k] = mavg(T.nbr[r], T.expo[k]) - mavg(zero, T.expo[k]);
  for (int r = 0; r < nl; ++r) {
    if (T.lsrow_line[r] >= 0) {
      // (1/|l|) int_l dp/dl dl in reference units: p at the line's end minus p at its start
      const int a = T.lsrow_axis[r];
      for (int k = 0; k < nb; ++k) {
        ld vp = 1, vm = 1;
        for (int b = 0; b < 3; ++b) {
          const ld xp = (ld)T.lsrow_t[r][b] + (b == a ? 0.5L : 0.0L);
          const ld xm = (ld)T.lsrow_t[r][b] - (b == a ? 0.5L : 0.0L);
          ld fp = 1, fm = 1, fa = 1;
          for (int e = 1; e <= T.expo[k][b]; ++e) {
            fp *= xp;
            fm *= xm;
            fa *= e;
          }
          vp *= fp / fa;
          vm *= fm / fa;
        }
        A[r][k] = vp - vm;
      }
      continue;
    }
    int o[3] = {0, 0, 0};
    if (T.lsrow_cell[r] >= 0)
      for (int a = 0; a < 3; ++a) o[a] = T.nbr[T.lsrow_cell[r]][a];
    for (int k = 0; k < nb; ++k) {
      ld s = 0;
      for (int a = 0; a < 3; ++a) {
        if (T.lsrow_dir[r][a] == 0.0 || T.expo[k][a] == 0) continue;
        int e[3] = {T.expo[k][0], T.expo[k][1], T.expo[k][2]};
        e[a] -= 1;
        s += (ld)T.lsrow_dir[r][a] * mavg(o, e);
      }
      A[r][k] = s;
    }
  }
  // QR of C^T (nb x nc), column-major: M[col r][row k] = C[r][k]
  std::vector<std::vector<ld>> M(nc, std::vector<ld>(nb)), Qf;
  for (int r = 0; r < nc; ++r)
    for (int k = 0; k < nb; ++k) M[r][k] = C[r][k];
  householder_qr(nb, nc, M, Qf);
  ld dmax = 0, dmin = 1e300L;
  for (int r = 0; r < nc; ++r) {
    dmax = std::max(dmax, std::fabs(M[r][r]));
    dmin = std::min(dmin, std::fabs(M[r][r]));
  }
  if (!(dmin > 1e-12L * dmax)) {
    std::snprintf(err, errlen, "CLS: exact-constraint matrix is rank deficient (dim %d)", dim);
    return false;
  }
  int nz = nb - nc;
  // P = Q1 R1^{-T} (nb x nc): solve R1^T Y = I, then P = Q1 Y
  std::vector<std::vector<ld>> Y(nc, std::vector<ld>(nc, 0));  // Y[row][col]
  for (int col = 0; col < nc; ++col)
    for (int row = 0; row < nc; ++row) {  // forward substitution: R1^T lower triangular, R1[i][j] = M[j][i]
      ld s = (row == col) ? 1 : 0;
      for (int q = 0; q < row; ++q) s -= M[row][q] * Y[q][col];  // (R1^T)[row][q] = R1[q][row] = M[row][q]
      Y[row][col] = s / M[row][row];
    }
  std::vector<std::vector<ld>> Pm(nb, std::vector<ld>(nc, 0));
  for (int i = 0; i < nb; ++i)
    for (int col = 0; col < nc; ++col) {
      ld s = 0;
      for (int q = 0; q < nc; ++q) s += Qf[q][i] * Y[q][col];  // Q1[i][q] = Qf[q][i]
      Pm[i][col] = s;
    }
  // B = A Q2 (nl x nz), QR of B
  std::vector<std::vector<ld>> Bc(nz, std::vector<ld>(nl, 0)), Qb;  // column-major
  for (int c = 0; c < nz; ++c)
    for (int r = 0; r < nl; ++r) {
      ld s = 0;
      for (int k = 0; k < nb; ++k) s += A[r][k] * Qf[nc + c][k];
      Bc[c][r] = s;
    }
  householder_qr(nl, nz, Bc, Qb);
  dmax = 0;
  dmin = 1e300L;
  for (int c = 0; c < nz; ++c) {
    dmax = std::max(dmax, std::fabs(Bc[c][c]));
    dmin = std::min(dmin, std::fabs(Bc[c][c]));
  }
  if (!(dmin > 1e-12L * dmax)) {
    std::snprintf(err, errlen, "CLS: least-squares part is rank deficient after constraint elimination (dim %d)", dim);
    return false;
  }
  T.cond_estimate = (double)(dmax / dmin);
  // K = Rb^{-1} Qb1^T (nz x nl)
  std::vector<std::vector<ld>> K(nz, std::vector<ld>(nl, 0));
  for (int r = 0; r < nl; ++r) {
    // solve Rb x = Qb1^T e_r  -> column r of K
    std::vector<ld> rhs(nz);
    for (int c = 0; c < nz; ++c) rhs[c] = Qb[c][r];  // Qb1[r][c] = Qb[c][r]
    for (int c = nz - 1; c >= 0; --c) {
      ld s = rhs[c];
      for (int q = c + 1; q < nz; ++q) s -= Bc[q][c] * K[q][r];  // Rb[c][q] = Bc[q][c]
      K[c][r] = s / Bc[c][c];
    }
  }
  // S = Q2 K (nb x nl);  R = [(I - S A) P, S]
  std::vector<std::vector<ld>> S(nb, std::vector<ld>(nl, 0));
  for (int i = 0; i < nb; ++i)
    for (int r = 0; r < nl; ++r) {
      ld s = 0;
      for (int c = 0; c < nz; ++c) s += Qf[nc + c][i] * K[c][r];
      S[i][r] = s;
    }
  for (int i = 0; i < nb; ++i) {
    for (int col = 0; col < nc; ++col) {
      ld s = Pm[i][col];
      for (int r = 0; r < nl; ++r) {
        ld ap = 0;
        for (int k = 0; k < nb; ++k) ap += A[r][k] * Pm[k][col];
        s -= S[i][r] * ap;
      }
      T.R[i * T.nd + col] = (double)s;
    }
    for (int r = 0; r < nl; ++r) T.R[i * T.nd + nc + r] = (double)S[i][r];
  }
  // basis averages over the own cell (for the zero-mean basis) and Gauss-point tables
  for (int k = 0; k < nb; ++k) T.avg0[k] = (double)mavg(zero, T.expo[k]);
  return true;
}

// values and reference derivatives of p_d at reference point x
void basis_at(const ClsTables& T, const double x[3], double* val, double* der /* [3][nb] */) {
  const int zero[3] = {0, 0, 0};
  for (int k = 0; k < T.nb; ++k) {
    const int* e = T.expo[k];
    ld v = 1;
    for (int a = 0; a < 3; ++a) v *= ipow((ld)x[a], e[a]) / fact(e[a]);
    val[k] = (double)(v - mavg(zero, e));
    for (int a = 0; a < 3; ++a) {
      if (e[a] == 0) {
        der[a * T.nb + k] = 0.0;
        continue;
      }
      int f[3] = {e[0], e[1], e[2]};
      f[a] -= 1;
      ld d = 1;
      for (int b = 0; b < 3; ++b) d *= ipow((ld)x[b], f[b]) / fact(f[b]);
      der[a * T.nb + k] = (double)d;
    }
  }
}

}  // namespace cgks
