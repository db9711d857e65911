// gks_flux.cuh -- FP64 device code of the gas-kinetic interface solver at one
// Gauss point, written for sm_100a.
//
// Everything is register resident: Maxwellian moment recursions, closed-form
// micro-slopes, 5x5 moment matrices <X psi_i psi_j> assembled from the normal-velocity
// moments and a 19-entry tangential table per Maxwellian, and the cancellation-free combined
// time coefficients alpha_i, beta_i of F^n = sum alpha_i M_i and
// F_t^n = sum beta_i M_i (derived from the time integrals of Eq. (flux) with
// E2 = exp(-dt/(2 tau)), E1 = E2^2, so one exp per Gauss point).
// Independent of oracle/ (different formulation of the same mathematics).
//
// The functions are templated on the scalar type T: T = double on the device; the
// host instantiates them with a counting type (flop_count.h) to report the
// algorithmic FP64 operation count of this formulation.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include <type_traits>

#define HD __host__ __device__ __forceinline__

namespace cgks {

HD double rsqrt_(double x) {
#ifdef __CUDA_ARCH__
  return rsqrt(x);
#else
  return 1.0 / sqrt(x);
#endif
}

struct FluxConst {
  double gamma, N, mu, Pr, tau_eps, tau_C, relax_C;
  double pfix;  // 1/Pr - 1
  double suth;  // Sutherland constant S: mu(T) = mu (1 + S) T^{3/2} / (T + S); 0 = constant mu
};

// Complementary error function given e = exp(-z^2), which the caller shares with the half-range
// moment seed: Chebyshev series of (1 + 2a) exp(a^2) erfc(a) in t = (a - K) / (a + K), a = |z|,
// K = 3.75, 25 terms (Shepherd-Laframboise form; coefficients computed by tools/erfc_fit.py),
// erfc(-a) = 2 - erfc(a).  Branch-free; one reciprocal.  Max relative error (tools/erfc_fit.py):
// 1.2e-15 for |z| <= 3, 6e-14 at |z| = 26 (the rounding of z^2 inside exp).
// Chebyshev coefficients of erfc_e (tools/erfc_fit.py); on the device a __constant__ table, so the
// FMAs take them as constant-bank operands instead of materialising 64-bit immediates
#define CGKS_ERFC_COEFS 2.3551578691348034, -0.004590054580646478, -0.08424913336651792, 0.05920993999819189, -0.026658668435305753, 0.009074997670705265, -0.002413163540417608, 0.0004907758365258086, -6.916973302501207e-05, 4.13902798607301e-06, 7.74038306619849e-07, -2.1886401049234397e-07, 1.076499946567091e-08, 4.521959811218287e-09, -7.754400208831351e-10, -6.318088340886684e-11, 2.86879501093067e-11, 1.9455868545777347e-13, -9.65469674843344e-13, 3.25254814814874e-14, 3.3478119482868056e-14, -1.864562880419313e-15, -1.2507950530688648e-15, 7.418235256624044e-17, 5.0681489047961116e-17
static __constant__ double c_erfc[25] = {CGKS_ERFC_COEFS};

// erf(z) / z as a series in z^2 for |z| < 1/2 (12 terms of 2/sqrt(pi) sum (-z^2)^n / (n! (2n+1)), relative
// error of 1 - z S below 3e-16 there); the device takes it for |z| < 1/2
#define CGKS_ERF_SMALL 1.1283791670955126, -0.37612638903183754, 0.11283791670955126, -0.026866170645131252, 0.005223977625442188, -0.0008548327023450852, 0.00012055332981789664, -1.492565035840625e-05, 1.6462114365889246e-06, -1.6365844691234924e-07, 1.4807192815879218e-08, -1.2290555301717926e-09
static __constant__ double c_erf_small[12] = {CGKS_ERF_SMALL};

template <typename T>
HD T erfc_e(T z, T e) {
  constexpr double K = 3.75;
#ifdef __CUDA_ARCH__
  const double* c = c_erf_small;
  const double* C = c_erfc;
#else
  constexpr double c[12] = {CGKS_ERF_SMALL};
  constexpr double C[25] = {CGKS_ERFC_COEFS};
#endif
  // per lane (not per warp): the value of a face must not depend on which faces share its warp,
  // so that decomposed runs stay bit-identical; at low Mach the branch is uniform anyway.  (The host
  // flop count instantiates this with a counting type and takes the branch the sample data takes.)
  if (fabs(z) < 0.5) {
    // Estrin form (dependency depth 5 instead of Horner's 11): pairs in x, quads in x^2, x^4, x^8
    const T x = z * z, x2 = x * x, x4 = x2 * x2, x8 = x4 * x4;
    const T p0 = fma(T(c[1]), x, T(c[0])), p1 = fma(T(c[3]), x, T(c[2])), p2 = fma(T(c[5]), x, T(c[4]));
    const T p3 = fma(T(c[7]), x, T(c[6])), p4 = fma(T(c[9]), x, T(c[8])), p5 = fma(T(c[11]), x, T(c[10]));
    const T q0 = fma(p1, x2, p0), q1 = fma(p3, x2, p2), q2 = fma(p5, x2, p4);
    const T s = fma(q2, x8, fma(q1, x4, q0));
    return fma(-z, s, T(1.0));
  }
  const T a = fabs(z);
  const T q = 1.0 + 2.0 * a;
  const T r = 1.0 / ((a + K) * q);
  const T t = (a - K) * q * r;
  const T t2 = 2.0 * t;
  T b1 = C[24], b2 = 0.0;  // Clenshaw
#pragma unroll
  for (int j = 23; j >= 1; --j) {
    const T b0 = C[j] + t2 * b1 - b2;
    b2 = b1;
    b1 = b0;
  }
  const T f = 0.5 * C[0] + t * b1 - b2;
  const T y = e * f * ((a + K) * r);
  return z < 0.0 ? 2.0 - y : y;
}

// half-range moments over u>0 (side=+1) or u<0 (side=-1)
template <typename T>
HD void half_moments(T U, T lam, T r, double side, T* M) {  // r = 1/(2 lam)
  const T rl = rsqrt_(lam);
  const T sl = lam * rl;  // sqrt(lam)
  const T e = exp(-lam * U * U);
  const T g = (0.5 * 0.56418958354775628695) * e * rl;  // exp(-lam U^2) / (2 sqrt(pi lam))
  M[0] = 0.5 * erfc_e(-side * sl * U, e);
  M[1] = U * M[0] + side * g;
#pragma unroll
  for (int k = 0; k < 5; ++k) M[k + 2] = U * M[k + 1] + (k + 1) * r * M[k];
}


// ---------------------------------------------------------------------------
// Half-range moment vectors and their directional derivatives.
// c_X = <X psi> for X = u^p v^q w^r (q + r <= 1), psi = (1, u, v, w, (u^2 + eta)/2), eta =
// v^2 + w^2 + xi^2, of a Maxwellian restricted to u > 0 or u < 0: the normal factor is a
// half-range moment M_k = <u^k>, the transverse factor one of 8 full-Gaussian expectations.
// Because the micro-slope of a perturbation dW is the first-order expansion of the Maxwellian
// on any fixed velocity domain, rho <X a psi>_half = D[rho c_X](W) dW: every half-range term
// of Eq. (flux) with a micro-slope is a directional derivative of rho c_X (no 5x5 solves).
// ---------------------------------------------------------------------------
template <typename T>
struct Tg {
  T V, W, V2, W2, VW, e1, ve, we;  // <v>, <w>, <v^2>, <w^2>, <vw>, <eta>, <v eta>, <w eta>
  T Z;                             // V^2 + W^2 + (4 + N) s (for the derivatives)
};

template <typename T>
HD void tg_value(T V, T W, T s, double N, Tg<T>& t) {
  const T VV = V * V, WW = W * W;
  const T Z = VV + WW + (4.0 + N) * s;
  t.Z = Z;
  t.V = V;
  t.W = W;
  t.V2 = VV + s;
  t.W2 = WW + s;
  t.VW = V * W;
  t.e1 = VV + WW + (2.0 + N) * s;
  t.ve = V * Z;
  t.we = W * Z;
}

// derivative of the transverse expectations along (dV, dW, ds); Z = V^2 + W^2 + (4 + N) s (per side)
template <typename T>
HD void tg_deriv(T V, T W, T Z, double N, T dV, T dW, T ds, Tg<T>& d) {
  const T dZ = 2.0 * (V * dV + W * dW) + (4.0 + N) * ds;
  d.V = dV;
  d.W = dW;
  d.V2 = 2.0 * V * dV + ds;
  d.W2 = 2.0 * W * dW + ds;
  d.VW = V * dW + W * dV;
  d.e1 = 2.0 * (V * dV + W * dW) + (2.0 + N) * ds;
  d.ve = dV * Z + V * dZ;
  d.we = dW * Z + W * dZ;
}

template <int q, int r, typename T>
HD void tg_pick(const Tg<T>& t, T& g000, T& g100, T& g010, T& g001, bool deriv) {
  if (q == 0 && r == 0) {
    g000 = deriv ? T(0.0) : T(1.0);
    g100 = t.V;
    g010 = t.W;
    g001 = t.e1;
  } else if (q == 1) {
    g000 = t.V;
    g100 = t.V2;
    g010 = t.VW;
    g001 = t.ve;
  } else {
    g000 = t.W;
    g100 = t.VW;
    g010 = t.W2;
    g001 = t.we;
  }
}

// rho-weighted transverse factors of one pick (q, r): value G_j = rho g_j, derivative
// H_j = rho h_j + drho g_j (j = 000, 100, 010, 001), with the halves of the 000 and 001 entries
// that enter the energy component (psi_4 = (u^2 + eta) / 2)
template <typename T>
struct RW {
  T x0, x1, x2, x3, x0h, x3h;
};

template <int q, int r, typename T>
HD RW<T> rw_value(const Tg<T>& t, T rho) {
  T g000, g100, g010, g001;
  tg_pick<q, r>(t, g000, g100, g010, g001, false);
  RW<T> w;
  w.x0 = (q == 0 && r == 0) ? rho : rho * g000;
  w.x1 = rho * g100;
  w.x2 = rho * g010;
  w.x3 = rho * g001;
  w.x0h = 0.5 * w.x0;
  w.x3h = 0.5 * w.x3;
  return w;
}

template <int q, int r, typename T>
HD RW<T> rw_deriv(const Tg<T>& t, const Tg<T>& dt, T rho, T drho) {
  T g000, g100, g010, g001, h000, h100, h010, h001;
  tg_pick<q, r>(t, g000, g100, g010, g001, false);
  tg_pick<q, r>(dt, h000, h100, h010, h001, true);
  RW<T> w;
  w.x0 = (q == 0 && r == 0) ? drho : rho * h000 + drho * g000;
  w.x1 = rho * h100 + drho * g100;
  w.x2 = rho * h010 + drho * g010;
  w.x3 = rho * h001 + drho * g001;
  w.x0h = 0.5 * w.x0;
  w.x3h = 0.5 * w.x3;
  return w;
}

// c += rho c_X (value), X = u^p v^q w^r with G = rw_value<q, r>
template <int p, typename T>
HD void col_value(const T* M, const RW<T>& G, T* c) {
  c[0] = fma(M[p], G.x0, c[0]);
  c[1] = fma(M[p + 1], G.x0, c[1]);
  c[2] = fma(M[p], G.x1, c[2]);
  c[3] = fma(M[p], G.x2, c[3]);
  c[4] = fma(M[p + 2], G.x0h, fma(M[p], G.x3h, c[4]));
}

// c += D[rho c_X] = rho dc_X + drho c_X: directional derivative, with the normal moments' derivative
// dM and the pick's rho-weighted value G and derivative H
template <int p, typename T>
HD void col_deriv(const T* M, const T* dM, const RW<T>& G, const RW<T>& H, T* c) {
  c[0] = fma(dM[p], G.x0, fma(M[p], H.x0, c[0]));
  c[1] = fma(dM[p + 1], G.x0, fma(M[p + 1], H.x0, c[1]));
  c[2] = fma(dM[p], G.x1, fma(M[p], H.x1, c[2]));
  c[3] = fma(dM[p], G.x2, fma(M[p], H.x2, c[3]));
  c[4] = fma(dM[p + 2], G.x0h, fma(M[p + 2], H.x0h, fma(dM[p], G.x3h, fma(M[p], H.x3h, c[4]))));
}

// derivative of the normal moments M_0..M_4 along (dU, dlam):
// dM_k/dU = 2 lam (M_{k+1} - U M_k) = 2 lam A_k, dM_k/dlam = s M_k - (M_{k+2} - 2 U M_{k+1} + U^2 M_k) = B_k;
// A_k and B_k do not depend on the direction: formed once per side (moments_ab), then 2 flops per k and
// direction (the formulation the flop count instantiates is the one executed: no repeated subexpressions)
template <typename T>
HD void moments_ab(const T* M, T U, T s, T* A, T* B) {
  const T U2 = 2.0 * U, UU = U * U;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    A[k] = M[k + 1] - U * M[k];
    B[k] = s * M[k] - (M[k + 2] - U2 * M[k + 1] + UU * M[k]);
  }
}
template <typename T>
HD void moments_deriv(const T* A, const T* B, T lam, T dU, T dlam, T* dM) {
  const T tl = 2.0 * lam * dU;
#pragma unroll
  for (int k = 0; k < 5; ++k) dM[k] = tl * A[k] + dlam * B[k];
}

// heat-flux functional of a flux-moment vector about U0 (R20):
// qF(v) = v_E - U0 . v_mom + |U0|^2/2 v_rho; a state vector Q contributes -U0n qF(Q)
template <typename T>
HD T qF(const T* v, T U0, T V0, T W0, T uu2) {
  return fma(uu2, v[0], fma(-U0, v[1], fma(-V0, v[2], fma(-W0, v[3], v[4]))));
}

// ---------------------------------------------------------------------------
// Full-Maxwellian contractions as Jacobian-vector products.  The micro-slope a of a
// perturbation dW is the first-order expansion of the Maxwellian, g(W + e dW) = g(W)(1 + e a.psi),
// so rho <X a psi> = D[rho <X psi>](W) dW for any velocity weight X.  With X = u_al this is the
// Euler-flux Jacobian, with X = u_n u_al the Jacobian of H_al = rho <u_n u_al psi>; both have
// closed forms (BGK gas with N internal degrees of freedom, N + 3 = 2/(gamma-1)).
// ---------------------------------------------------------------------------
template <typename T>
struct Dprim {
  T dr, du[3], dp, udu;
};

// primitive perturbation (d rho, dU, dp) of a conservative perturbation d at (rho, U)
template <typename T>
HD Dprim<T> dprim(T ir, const T* U, T uu2, double gm1, const T* d) {
  Dprim<T> q;
  q.dr = d[0];
#pragma unroll
  for (int i = 0; i < 3; ++i) q.du[i] = (d[1 + i] - U[i] * d[0]) * ir;
  q.dp = gm1 * fma(uu2, d[0], fma(-U[0], d[1], fma(-U[1], d[2], fma(-U[2], d[3], d[4]))));
  q.udu = U[0] * q.du[0] + U[1] * q.du[1] + U[2] * q.du[2];
  return q;
}

// acc += s DF_al(W) d, F_al = (m_al, m_al U + p e_al, U_al (E + p)) the Euler flux along al
template <int AL, typename T, typename S>
HD void jvp_flux(T rho, const T* U, T p, T E, const T* d, const Dprim<T>& q, S s, T* acc) {
  // s = +-1 (a sign, folded into the FMAs): acc += s * DF d as FMA chains into the accumulators
  const T smA = s * (rho * U[AL]), sd = s * d[1 + AL];
  acc[0] += sd;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const T a = b == AL ? acc[1 + b] + s * q.dp : acc[1 + b];
    acc[1 + b] = fma(sd, U[b], fma(smA, q.du[b], a));
  }
  acc[4] = fma(s * q.du[AL], E + p, fma(s * U[AL], d[4] + q.dp, acc[4]));
}

// acc += DH_al(W) d, H_al = rho <u_n u_al psi> (n = 0, the face normal):
//   H[0] = rho U_n U_al + p d_{n al}
//   H[b] = rho U_n U_al U_b + p (d_{n al} U_b + d_{n b} U_al + d_{al b} U_n)
//   H[4] = ((rho |U|^2 + (N+7) p) U_n U_al + (p |U|^2 + (N+5) p^2/rho) d_{n al}) / 2
template <int AL, typename T>
HD void jvp_flux2(T rho, T ir, const T* U, T p, T uu, double K5, double K7, const Dprim<T>& q, T* acc) {
  const T UnUa = U[0] * U[AL];
  const T dUnUa = q.du[0] * U[AL] + U[0] * q.du[AL];
  const T cU = q.dr * UnUa + rho * dUnUa;  // D(rho U_n U_al)
  const T rU = rho * UnUa;
  acc[0] += AL == 0 ? cU + q.dp : cU;
#pragma unroll
  for (int b = 0; b < 3; ++b) {  // FMA chains into the accumulators
    T a = acc[1 + b];
    if (AL == 0) a = fma(q.dp, U[b], fma(p, q.du[b], a));
    if (b == 0) a = fma(q.dp, U[AL], fma(p, q.du[AL], a));
    if (AL == b) a = fma(q.dp, U[0], fma(p, q.du[0], a));
    acc[1 + b] = fma(cU, U[b], fma(rU, q.du[b], a));
  }
  const T c1 = rho * uu + K7 * p;
  const T dc1 = q.dr * uu + 2.0 * rho * q.udu + K7 * q.dp;
  T v4 = dc1 * UnUa + c1 * dUnUa;
  if (AL == 0) v4 += q.dp * uu + 2.0 * p * q.udu + K5 * p * ir * (2.0 * q.dp - p * ir * q.dr);
  acc[4] = fma(0.5, v4, acc[4]);
}

// ---------------------------------------------------------------------------
// The interface solver at one Gauss point, run by one lane (k_flux1):
//   (S) side_terms, once per side: all half-range terms of Eq. (flux) of that side (W0 and dW0 parts,
//       MF3..MF5, MQ4, MQ5) as values and directional derivatives of half-range moment vectors,
//       accumulated into x1[0..44]: 0-4 W0 part (R13), 5-19 dW0 parts (R14), 20-24 MF3 =
//       rho <u psi>, 25-29 MF4 = rho <u (a.u) psi>, 30-34 MF5 = rho <u A psi>, 35-39 MQ4 =
//       rho <(a.u) psi>, 40-44 MQ5 = rho <A psi> (half ranges); also the side's pressure, positivity
//       and Euler time derivative dW/dt (R23, for the side relaxation);
//   (G) interface_terms, once: interface equilibrium g0, collision time and combined time
//       coefficients, equilibrium terms as Jacobian-vector products, everything folded into F^n,
//       F_t^n, Q^n, Q_t^n and the heat-flux scalars of the Prandtl fix;
//   then the side relaxation (relax_ee) of both sides.
// All in the normal frame (normal = first axis; dW[dir][var], dir 0 = normal).
// ---------------------------------------------------------------------------
template <typename T>
HD bool side_terms(double sgn, const T* W, const T (*dW)[5], const FluxConst& fc, T* x1, T& p_out, T* dtw) {
  const T gm1 = fc.gamma - 1.0;
  const T rho = W[0], ir = 1.0 / rho;
  const T U = W[1] * ir, V = W[2] * ir, Ww = W[3] * ir;
  const T uu2s = 0.5 * (U * U + V * V + Ww * Ww);
  const T p = gm1 * (W[4] - rho * uu2s);
  const bool ok = (rho > 0.0) && (p > 0.0);
  const T ip = ok ? T(1.0) / p : T(1.0);
  const T lam = ok ? T(0.5) * rho * ip : T(1.0);
  const T sv = ok ? p * ir : T(0.5);  // variance 1/(2 lam)
  const T Uv[3] = {U, V, Ww};
  p_out = p;
#pragma unroll
  for (int i = 0; i < 5; ++i) dtw[i] = 0.0;
  // primitive perturbations of the three slopes: used by dW/dt and by the slope directions below
  const Dprim<T> qs[3] = {dprim(ir, Uv, uu2s, fc.gamma - 1.0, dW[0]), dprim(ir, Uv, uu2s, fc.gamma - 1.0, dW[1]),
                          dprim(ir, Uv, uu2s, fc.gamma - 1.0, dW[2])};
  jvp_flux<0>(rho, Uv, p, W[4], dW[0], qs[0], -1.0, dtw);
  jvp_flux<1>(rho, Uv, p, W[4], dW[1], qs[1], -1.0, dtw);
  jvp_flux<2>(rho, Uv, p, W[4], dW[2], qs[2], -1.0, dtw);
  T M[7];
  half_moments(U, lam, sv, sgn, M);  // H(u) or 1-H(u)
  T MA[5], MB[5];
  moments_ab(M, U, sv, MA, MB);
  Tg<T> tg;
  tg_value(V, Ww, sv, fc.N, tg);
  const RW<T> G00 = rw_value<0, 0>(tg, rho), G10 = rw_value<1, 0>(tg, rho), G01 = rw_value<0, 1>(tg, rho);
  col_value<0>(M, G00, x1 + 0);
  col_value<1>(M, G00, x1 + 20);
#pragma unroll
  for (int dir = 0; dir < 4; ++dir) {
    const Dprim<T> q = dir < 3 ? qs[dir] : dprim(ir, Uv, uu2s, fc.gamma - 1.0, dtw);
    const T dlam = lam * (q.dr * ir - q.dp * ip);
    const T ds = -2.0 * sv * sv * dlam;
    T dM[5];
    moments_deriv(MA, MB, lam, q.du[0], dlam, dM);
    Tg<T> dt;
    tg_deriv(V, Ww, tg.Z, fc.N, q.du[1], q.du[2], ds, dt);
    const RW<T> H00 = rw_deriv<0, 0>(tg, dt, rho, q.dr);
    if (dir == 0) {
      col_deriv<0>(M, dM, G00, H00, x1 + 5);
      col_deriv<1>(M, dM, G00, H00, x1 + 35);
      col_deriv<2>(M, dM, G00, H00, x1 + 25);
    } else if (dir == 1) {
      const RW<T> H10 = rw_deriv<1, 0>(tg, dt, rho, q.dr);
      col_deriv<0>(M, dM, G00, H00, x1 + 10);
      col_deriv<0>(M, dM, G10, H10, x1 + 35);
      col_deriv<1>(M, dM, G10, H10, x1 + 25);
    } else if (dir == 2) {
      const RW<T> H01 = rw_deriv<0, 1>(tg, dt, rho, q.dr);
      col_deriv<0>(M, dM, G00, H00, x1 + 15);
      col_deriv<0>(M, dM, G01, H01, x1 + 35);
      col_deriv<1>(M, dM, G01, H01, x1 + 25);
    } else {
      col_deriv<0>(M, dM, G00, H00, x1 + 40);
      col_deriv<1>(M, dM, G00, H00, x1 + 30);
    }
  }
  return ok;
}

// Interface phase (G) from the summed half-range terms: x1[0..19] in registers, the
// half-range vectors x1[20..44] in parking slots 0..24 (get(i)).  Writes acc[0..9] = F^n, F_t^n
// (Prandtl fix applied) and acc[10..19] = Q^n, Q_t^n of the interface, and the relative pressure jump
// |pL - pR| / (pL + pR) for the side relaxation.  Returns the positivity of the equilibrium state.
// TONLY (the second stage of S2O4, which needs only the time derivatives): only F_t^n and Q_t^n
// (acc[5..9], acc[15..19]) are formed; acc[0..4] and acc[10..14] are left unset.
template <typename T, typename P, bool TONLY = false>
HD bool interface_terms(const T* x1, T pL, T pR, T dt, T idt, const FluxConst& fc, const P& park, T* acc, T& jump_out) {
  const T gm1 = fc.gamma - 1.0;
  const T r0 = x1[0], i0 = 1.0 / r0;
  const T U0 = x1[1] * i0, V0 = x1[2] * i0, Ww0 = x1[3] * i0;
  const T uu2 = 0.5 * (U0 * U0 + V0 * V0 + Ww0 * Ww0);
  const T p0 = gm1 * (x1[4] - r0 * uu2);
  const bool good = (r0 > 0.0) && (p0 > 0.0);
  const T rpp = 1.0 / (p0 * (pL + pR));
  const T jump = fabs(pL - pR) * (p0 * rpp);
  jump_out = jump;
  T mu_p0 = fc.mu * ((pL + pR) * rpp);
  if (fc.suth > 0.0) {
    const T T0 = p0 * i0;
    mu_p0 = fc.mu * (1.0 + fc.suth) * sqrt(T0) * i0 / (T0 + fc.suth);
  }
  const T tau = (fc.mu > 0.0) ? (mu_p0 + fc.tau_C * jump * dt) : (fc.tau_eps + fc.tau_C * jump) * dt;
  T al[6], be[6];
  T a20, a21;  // heat-flux scalars of the Prandtl fix (R20)
  {
    const T U0v[3] = {U0, V0, Ww0};
    const T uu0 = 2.0 * uu2;
    const double K5 = fc.N + 5.0, K7 = fc.N + 7.0;
    T MQa[5], MF1[5], MF2[5], MF0[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) MQa[i] = MF1[i] = MF2[i] = 0.0;
    {
      const T* d0 = x1 + 5;
      const Dprim<T> q0 = dprim(i0, U0v, uu2, fc.gamma - 1.0, d0);
      jvp_flux<0>(r0, U0v, p0, x1[4], d0, q0, 1.0, MQa);
      jvp_flux2<0>(r0, i0, U0v, p0, uu0, K5, K7, q0, MF1);
      const T* d1 = x1 + 10;
      const Dprim<T> q1 = dprim(i0, U0v, uu2, fc.gamma - 1.0, d1);
      jvp_flux<1>(r0, U0v, p0, x1[4], d1, q1, 1.0, MQa);
      jvp_flux2<1>(r0, i0, U0v, p0, uu0, K5, K7, q1, MF1);
      const T* d2 = x1 + 15;
      const Dprim<T> q2 = dprim(i0, U0v, uu2, fc.gamma - 1.0, d2);
      jvp_flux<2>(r0, U0v, p0, x1[4], d2, q2, 1.0, MQa);
      jvp_flux2<2>(r0, i0, U0v, p0, uu0, K5, K7, q2, MF1);
      const Dprim<T> qa = dprim(i0, U0v, uu2, fc.gamma - 1.0, MQa);
      jvp_flux<0>(r0, U0v, p0, x1[4], MQa, qa, -1.0, MF2);
    }
    {
      const T m2 = -expm1(-0.5 * dt / tau);  // 1 - E2 without cancellation
      const T E2 = 1.0 - m2;
      const T qq = 4.0 * tau * m2 * m2 * idt * idt;
      be[0] = qq;
      be[1] = 4.0 * tau * m2 * (dt * E2 - 2.0 * tau * m2) * idt * idt;
      be[2] = 1.0 - tau * qq;
      be[3] = -qq;
      be[4] = -be[1];
      be[5] = tau * qq;
      if (!TONLY) {
        const T c3 = tau * m2 * (3.0 - E2) * idt;
        al[0] = 1.0 - c3;
        al[1] = 2.0 * tau * c3 - tau * (1.0 + 2.0 * E2 - E2 * E2);
        al[2] = -tau + tau * c3;
        al[3] = c3;
        al[4] = -2.0 * tau * c3 + tau * E2 * (2.0 - E2);
        al[5] = -tau * c3;
      }
    }
    MF0[0] = r0 * U0;
    MF0[1] = r0 * U0 * U0 + p0;
    MF0[2] = r0 * U0 * V0;
    MF0[3] = r0 * U0 * Ww0;
    MF0[4] = U0 * (x1[4] + p0);
    const T sMF0 = qF(MF0, U0, V0, Ww0, uu2), sMF1 = qF(MF1, U0, V0, Ww0, uu2), sMF2 = qF(MF2, U0, V0, Ww0, uu2),
            sMQa = qF(MQa, U0, V0, Ww0, uu2);
    const T sW = qF(x1, U0, V0, Ww0, uu2);  // qF(W0); MQ0 = MQ3 = W0
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const T mf0 = MF0[i], mf1 = MF1[i], mf2 = MF2[i], mqa = MQa[i];
      if (!TONLY) {
        acc[i] = al[0] * mf0 + al[1] * mf1 + al[2] * mf2;
        acc[10 + i] = (al[0] + al[3]) * x1[i] + (al[1] - al[2]) * mqa;  // MQ1 = MQa, MQ2 = -MQa (compatibility)
      }
      acc[5 + i] = be[0] * mf0 + be[1] * mf1 + be[2] * mf2;
      acc[15 + i] = (be[0] + be[3]) * x1[i] + (be[1] - be[2]) * mqa;
    }
    if (!TONLY)
      a20 = -U0 * sW * (al[0] - 1.0 + al[3]) + (al[0] - 1.0) * sMF0 + al[1] * (sMF1 - U0 * sMQa) +
            al[2] * (sMF2 + U0 * sMQa);
    a21 = -U0 * sW * (be[0] + be[3]) + be[0] * sMF0 + be[1] * (sMF1 - U0 * sMQa) + (be[2] - 1.0) * (sMF2 + U0 * sMQa);
  }
  {
    T v3[5], v4[5], v5[5], q4[5], q5[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      v3[i] = park.get(i);
      v4[i] = park.get(5 + i);
      v5[i] = park.get(10 + i);
      q4[i] = park.get(15 + i);
      q5[i] = park.get(20 + i);
    }
    const T s3 = qF(v3, U0, V0, Ww0, uu2);
    const T s4 = qF(v4, U0, V0, Ww0, uu2) - U0 * qF(q4, U0, V0, Ww0, uu2);
    const T s5 = qF(v5, U0, V0, Ww0, uu2) - U0 * qF(q5, U0, V0, Ww0, uu2);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      if (!TONLY) {
        acc[i] = fma(al[3], v3[i], fma(al[4], v4[i], fma(al[5], v5[i], acc[i])));
        acc[10 + i] = fma(al[4], q4[i], fma(al[5], q5[i], acc[10 + i]));
      }
      acc[5 + i] = fma(be[3], v3[i], fma(be[4], v4[i], fma(be[5], v5[i], acc[5 + i])));
      acc[15 + i] = fma(be[4], q4[i], fma(be[5], q5[i], acc[15 + i]));
    }
    if (!TONLY) a20 = fma(al[3], s3, fma(al[4], s4, fma(al[5], s5, a20)));
    a21 = fma(be[3], s3, fma(be[4], s4, fma(be[5], s5, a21)));
  }
  if (fc.Pr != 1.0) {  // Prandtl fix (R20)
    if (!TONLY) acc[4] = fma(fc.pfix, a20, acc[4]);
    acc[9] = fma(fc.pfix, a21, acc[9]);
  }
  return good;
}

// side-state relaxation weight (R23): ee = exp(-dt / tau0), tau0 = C |pL - pR| / (pL + pR) dt,
// which is below 1e-304 for C jump < 1/700 (smooth regions) and is then taken as 0: the reciprocal is only
// formed in its safe range (no division slow path for tau0 -> 0)
template <typename T>
HD T relax_ee(T jump, const FluxConst& fc) {
  const T rC = fc.relax_C * jump;
  return (rC > 1.0 / 700.0) ? exp(-1.0 / fmax(rC, T(1.0 / 700.0))) : T(0.0);
}

}  // namespace cgks
