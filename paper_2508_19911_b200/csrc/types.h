// types.h -- plain structs shared by host and device code (no device symbols).
#pragma once
#include <stdint.h>

#include "gks_flux.cuh"

namespace cgks {

// ---------------------------------------------------------------------------
// constant geometry / parameters
// ---------------------------------------------------------------------------
struct Geo {
  int n[3];          // local cells
  int dim;
  int bounded[3];    // axis has non-periodic boundaries, or is a decomposed axis (ghost storage)
  int halo[3];       // axis is decomposed: ghost cells are stored (filled by the halo exchange)
  int zoff;          // storage offset of z-plane 0 (2 ghost planes when z is decomposed)
  int yoff;          // storage offset of y-row 0 (2 ghost rows when y is decomposed: pencils, 2-D y-slabs)
  int elo[3];        // extended (reconstruction) range start: -1 on bounded axes
  int en[3];         // extended counts
  int fn[3][3];      // face-grid dims for faces normal to axis a: fn[a][b]
  long long plane;   // n0*n1 (cells of a z-plane)
  long long splane;  // n0*(n1 + 2 yoff): storage stride of one field of a z-plane
  long long eplane;  // en0*en1
  double h[3], ih[3];
  int bc[3][2];
  double bc_state[3][2][5];
  double cfl, fixed_dt, mu, gamma;
  double k_venkat, chi_c, eps_venkat2;
  double chi_is;  // 1 / chi_scale (GENO)
  double suth;  // Sutherland constant S (0: constant mu)
  int lines;    // CGKS-5th line-DOF variant
  int ngl;      // lines per axis (transverse face Gauss points: 4 / 2 / 1)
  int nfr;      // fields of a face record (30, plus 2 x ngl x 10 per-Gauss-point values with lines)
  // stretched tensor-product mesh (NEXT-4, R37): per-axis cell widths and their inverses, indexed
  // cell + 2 for cells -2 .. n+1 (ghost widths: periodic image or boundary cell)
  int stretched;
  const double* hw[3];
  const double* ihw[3];
};

struct ErrState {
  int code;        // 0 ok, 3 positivity, 4 numerical
  int stage;       // 1, 2
  long long step;  // global step index at failure
  int cell[3];
  int kernel;      // 1 flux, 2 update, 3 dt
};

struct TimeState {
  double t;
  long long steps;
  double dt;
  unsigned long long dtmin_bits;
  int pad;
  double idt;  // 1/dt, written with dt
};

}  // namespace cgks
