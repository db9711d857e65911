// gks_flux.cuh -- FP64 device code of the gas-kinetic interface solver at one
// Gauss point, written for sm_100a.
//
// Everything is register resident: Maxwellian moment recursions, closed-form
// micro-slopes, moment contractions with compile-time indices (the compiler
// folds <u^0> = 1 and common products), and the cancellation-free combined
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
};

// moments of a Maxwellian: u (normal, possibly half range), v, w (full), xi^2
template <typename T>
struct MomT {
  T u[7], v[7], w[7], x2, x4;
};

template <typename T>
HD void full_moments(T U, T lam, T* M) {
  const T r = 0.5 / lam;
  M[0] = 1.0;
  M[1] = U;
#pragma unroll
  for (int k = 0; k < 5; ++k) M[k + 2] = U * M[k + 1] + (k + 1) * r * M[k];
}

// half-range moments over u>0 (side=+1) or u<0 (side=-1)
template <typename T>
HD void half_moments(T U, T lam, double side, T* M) {
  const T r = 0.5 / lam;
  const T sl = sqrt(lam);
  const T g = 0.5 * exp(-lam * U * U) * rsqrt_(lam * 3.14159265358979323846);
  M[0] = 0.5 * erfc(-side * sl * U);
  M[1] = U * M[0] + side * g;
#pragma unroll
  for (int k = 0; k < 5; ++k) M[k + 2] = U * M[k + 1] + (k + 1) * r * M[k];
}

// <u^a v^b w^c (xi^2)^d psi>, psi = (1,u,v,w,(u^2+v^2+w^2+xi^2)/2)
template <int a, int b, int c, int d, typename T>
HD void psi_m(const MomT<T>& m, T* o) {
  const T xd = (d == 0) ? T(1.0) : m.x2;
  const T xd1 = (d == 0) ? m.x2 : m.x4;
  const T vw = m.v[b] * m.w[c];
  const T base = m.u[a] * vw;
  o[0] = base * xd;
  o[1] = m.u[a + 1] * vw * xd;
  o[2] = m.u[a] * m.v[b + 1] * m.w[c] * xd;
  o[3] = m.u[a] * m.v[b] * m.w[c + 1] * xd;
  o[4] = 0.5 * ((m.u[a + 2] * vw + m.u[a] * (m.v[b + 2] * m.w[c] + m.v[b] * m.w[c + 2])) * xd + base * xd1);
}

// acc += s * <u^a v^b w^c (sum_j k_j psi_j) psi>
template <int a, int b, int c, typename T, typename S>
HD void apsi_acc(const MomT<T>& m, const T* k, S s, T* acc) {
  T t[5];
  T o[5];
  psi_m<a, b, c, 0>(m, o);
#pragma unroll
  for (int i = 0; i < 5; ++i) t[i] = k[0] * o[i];
  psi_m<a + 1, b, c, 0>(m, o);
#pragma unroll
  for (int i = 0; i < 5; ++i) t[i] += k[1] * o[i];
  psi_m<a, b + 1, c, 0>(m, o);
#pragma unroll
  for (int i = 0; i < 5; ++i) t[i] += k[2] * o[i];
  psi_m<a, b, c + 1, 0>(m, o);
#pragma unroll
  for (int i = 0; i < 5; ++i) t[i] += k[3] * o[i];
  T e[5];
  psi_m<a + 2, b, c, 0>(m, e);
  psi_m<a, b + 2, c, 0>(m, o);
#pragma unroll
  for (int i = 0; i < 5; ++i) e[i] += o[i];
  psi_m<a, b, c + 2, 0>(m, o);
#pragma unroll
  for (int i = 0; i < 5; ++i) e[i] += o[i];
  psi_m<a, b, c, 1>(m, o);
  const T h = 0.5 * k[4];
#pragma unroll
  for (int i = 0; i < 5; ++i) acc[i] += s * (t[i] + h * (e[i] + o[i]));
}

// micro-slope: the unique a = sum_j a_j psi_j with <a psi>_full = b, closed form for a
// Maxwellian (U, V, W, lam) with N internal degrees of freedom
template <typename T>
HD void micro_slope(T U, T V, T W, T lam, double N, const T* b, T* a) {
  const T uu = U * U + V * V + W * W;
  const T K3 = (N + 3.0) / (2.0 * lam);
  a[4] = (4.0 * lam * lam / (N + 3.0)) * (2.0 * b[4] - 2.0 * (U * b[1] + V * b[2] + W * b[3]) + (uu - K3) * b[0]);
  const T tl = 2.0 * lam;
  a[1] = tl * (b[1] - U * b[0]) - U * a[4];
  a[2] = tl * (b[2] - V * b[0]) - V * a[4];
  a[3] = tl * (b[3] - W * b[0]) - W * a[4];
  a[0] = b[0] - U * a[1] - V * a[2] - W * a[3] - 0.5 * a[4] * (uu + K3);
}

// outputs of one Gauss point, normal frame
template <typename T>
struct GPOutT {
  T Fn[5], Ft[5];
  T QLn[5], QLt[5], QRn[5], QRt[5];
};
typedef GPOutT<double> GPOut;

// Returns false when a side (or the interface equilibrium) is not positive.
// W*: conservative states; dW*[dir][var]: physical derivatives (dir 0 = normal).
template <bool COMPACT, typename T>
HD bool gks_flux_point(const T* WL, const T (*dWL)[5], const T* WR, const T (*dWR)[5], T dt, const FluxConst& fc,
                       GPOutT<T>& o) {
  typedef MomT<T> Mom;
  const T gm1 = fc.gamma - 1.0;
  // ---- primitives of the two sides
  const T rL = WL[0], rR = WR[0];
  const T iL = 1.0 / rL, iR = 1.0 / rR;
  const T UL = WL[1] * iL, VL = WL[2] * iL, WwL = WL[3] * iL;
  const T UR = WR[1] * iR, VR = WR[2] * iR, WwR = WR[3] * iR;
  const T pL = gm1 * (WL[4] - 0.5 * rL * (UL * UL + VL * VL + WwL * WwL));
  const T pR = gm1 * (WR[4] - 0.5 * rR * (UR * UR + VR * VR + WwR * WwR));
  if (!(rL > 0.0) || !(rR > 0.0) || !(pL > 0.0) || !(pR > 0.0)) return false;
  const T lL = 0.5 * rL / pL, lR = 0.5 * rR / pR;

  Mom hL, hR;  // g_l restricted to u>0, g_r restricted to u<0 (H(u))
  half_moments(UL, lL, 1.0, hL.u);
  full_moments(VL, lL, hL.v);
  full_moments(WwL, lL, hL.w);
  hL.x2 = 0.5 * fc.N / lL;
  hL.x4 = fc.N * (fc.N + 2.0) * 0.25 / (lL * lL);
  half_moments(UR, lR, -1.0, hR.u);
  full_moments(VR, lR, hR.v);
  full_moments(WwR, lR, hR.w);
  hR.x2 = 0.5 * fc.N / lR;
  hR.x4 = fc.N * (fc.N + 2.0) * 0.25 / (lR * lR);

  // ---- interface equilibrium W0 = rho_l <psi>_{+,l} + rho_r <psi>_{-,r}   (R13)
  T W0[5];
  {
    T a[5], b[5];
    psi_m<0, 0, 0, 0>(hL, a);
    psi_m<0, 0, 0, 0>(hR, b);
#pragma unroll
    for (int i = 0; i < 5; ++i) W0[i] = rL * a[i] + rR * b[i];
  }
  const T r0 = W0[0], i0 = 1.0 / r0;
  const T U0 = W0[1] * i0, V0 = W0[2] * i0, Ww0 = W0[3] * i0;
  const T p0 = gm1 * (W0[4] - 0.5 * r0 * (U0 * U0 + V0 * V0 + Ww0 * Ww0));
  if (!(r0 > 0.0) || !(p0 > 0.0)) return false;
  const T l0 = 0.5 * r0 / p0;
  Mom f0;
  full_moments(U0, l0, f0.u);
  full_moments(V0, l0, f0.v);
  full_moments(Ww0, l0, f0.w);
  f0.x2 = 0.5 * fc.N / l0;
  f0.x4 = fc.N * (fc.N + 2.0) * 0.25 / (l0 * l0);

  // ---- micro-slopes of the sides (R15) and of the equilibrium (R14)
  T aL[3][5], aR[3][5], ab[3][5];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    T b[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) b[i] = dWL[d][i] * iL;
    micro_slope(UL, VL, WwL, lL, fc.N, b, aL[d]);
#pragma unroll
    for (int i = 0; i < 5; ++i) b[i] = dWR[d][i] * iR;
    micro_slope(UR, VR, WwR, lR, fc.N, b, aR[d]);
    T s[5] = {0, 0, 0, 0, 0};
    apsi_acc<0, 0, 0>(hL, aL[d], rL, s);
    apsi_acc<0, 0, 0>(hR, aR[d], rR, s);
#pragma unroll
    for (int i = 0; i < 5; ++i) s[i] *= i0;
    micro_slope(U0, V0, Ww0, l0, fc.N, s, ab[d]);
  }

  // ---- time coefficients A from compatibility <(a.u + A) psi> = 0 (R16), full moments.
  // dWdt_s = rho_s <A_s psi> = -rho_s <(a_s.u) psi> is the Euler time derivative of side s (R23).
  T AL[5], AR[5], Ab[5];
  T dtWL[5], dtWR[5];
  {
    Mom fL;
    full_moments(UL, lL, fL.u);
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      fL.v[k] = hL.v[k];
      fL.w[k] = hL.w[k];
    }
    fL.x2 = hL.x2;
    fL.x4 = hL.x4;
    T b[5] = {0, 0, 0, 0, 0};
    apsi_acc<1, 0, 0>(fL, aL[0], -1.0, b);
    apsi_acc<0, 1, 0>(fL, aL[1], -1.0, b);
    apsi_acc<0, 0, 1>(fL, aL[2], -1.0, b);
    micro_slope(UL, VL, WwL, lL, fc.N, b, AL);
#pragma unroll
    for (int i = 0; i < 5; ++i) dtWL[i] = rL * b[i];
  }
  {
    Mom fR;
    full_moments(UR, lR, fR.u);
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      fR.v[k] = hR.v[k];
      fR.w[k] = hR.w[k];
    }
    fR.x2 = hR.x2;
    fR.x4 = hR.x4;
    T b[5] = {0, 0, 0, 0, 0};
    apsi_acc<1, 0, 0>(fR, aR[0], -1.0, b);
    apsi_acc<0, 1, 0>(fR, aR[1], -1.0, b);
    apsi_acc<0, 0, 1>(fR, aR[2], -1.0, b);
    micro_slope(UR, VR, WwR, lR, fc.N, b, AR);
#pragma unroll
    for (int i = 0; i < 5; ++i) dtWR[i] = rR * b[i];
  }
  // equilibrium: keep MQa = rho0 <(abar.u) psi> (state moment), Abar from -MQa
  T MQa[5] = {0, 0, 0, 0, 0};
  apsi_acc<1, 0, 0>(f0, ab[0], r0, MQa);
  apsi_acc<0, 1, 0>(f0, ab[1], r0, MQa);
  apsi_acc<0, 0, 1>(f0, ab[2], r0, MQa);
  {
    T b[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) b[i] = -MQa[i] * i0;
    micro_slope(U0, V0, Ww0, l0, fc.N, b, Ab);
  }

  // ---- collision time (R17)
  const T jump = fabs((pL - pR) / (pL + pR));
  const T tau = (fc.mu > 0.0) ? (fc.mu / p0 + fc.tau_C * jump * dt) : (fc.tau_eps + fc.tau_C * jump) * dt;

  // ---- flux moment vectors (u psi) of the six terms of Eq. (flux)
  T MF[6][5];
  psi_m<1, 0, 0, 0>(f0, MF[0]);
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    MF[0][i] *= r0;
    MF[1][i] = 0.0;
    MF[2][i] = 0.0;
  }
  apsi_acc<2, 0, 0>(f0, ab[0], r0, MF[1]);
  apsi_acc<1, 1, 0>(f0, ab[1], r0, MF[1]);
  apsi_acc<1, 0, 1>(f0, ab[2], r0, MF[1]);
  apsi_acc<1, 0, 0>(f0, Ab, r0, MF[2]);
  {
    T a[5], b[5];
    psi_m<1, 0, 0, 0>(hL, a);
    psi_m<1, 0, 0, 0>(hR, b);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      MF[3][i] = rL * a[i] + rR * b[i];
      MF[4][i] = 0.0;
      MF[5][i] = 0.0;
    }
  }
  apsi_acc<2, 0, 0>(hL, aL[0], rL, MF[4]);
  apsi_acc<1, 1, 0>(hL, aL[1], rL, MF[4]);
  apsi_acc<1, 0, 1>(hL, aL[2], rL, MF[4]);
  apsi_acc<2, 0, 0>(hR, aR[0], rR, MF[4]);
  apsi_acc<1, 1, 0>(hR, aR[1], rR, MF[4]);
  apsi_acc<1, 0, 1>(hR, aR[2], rR, MF[4]);
  apsi_acc<1, 0, 0>(hL, AL, rL, MF[5]);
  apsi_acc<1, 0, 0>(hR, AR, rR, MF[5]);

  // ---- combined time coefficients: F^n = sum alpha_i MF_i, F_t^n = sum beta_i MF_i
  // (E2 = e^{-dt/(2tau)}, m2 = 1-E2; tau == 0 gives E2 = 0 and the Euler limits)
  const T idt = 1.0 / dt;
  const T E2 = exp(-0.5 * dt / tau);
  const T m2 = -expm1(-0.5 * dt / tau);
  const T c3 = tau * m2 * (3.0 - E2) * idt;  // tau m2 (3-E2)/dt
  const T q = 4.0 * tau * m2 * m2 * idt * idt;  // 4 tau m2^2/dt^2
  T al[6], be[6];
  al[0] = 1.0 - c3;
  be[0] = q;
  al[1] = 2.0 * tau * c3 - tau * (1.0 + 2.0 * E2 - E2 * E2);
  be[1] = 4.0 * tau * m2 * (dt * E2 - 2.0 * tau * m2) * idt * idt;
  al[2] = -tau + tau * c3;
  be[2] = 1.0 - tau * q;
  al[3] = c3;
  be[3] = -q;
  al[4] = -2.0 * tau * c3 + tau * E2 * (2.0 - E2);
  be[4] = -be[1];
  al[5] = -tau * c3;
  be[5] = tau * q;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    T fn = 0.0, ft = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      fn += al[k] * MF[k][i];
      ft += be[k] * MF[k][i];
    }
    o.Fn[i] = fn;
    o.Ft[i] = ft;
  }

  const bool need_state = COMPACT || (fc.Pr != 1.0);
  if (need_state) {
    // state moment vectors (psi) of the six terms
    T MQ[6][5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      MQ[0][i] = W0[i];
      MQ[1][i] = MQa[i];
      MQ[2][i] = -MQa[i];  // rho0 <Abar psi> = -rho0 <(abar.u) psi> by compatibility
      MQ[3][i] = W0[i];    // rho_l <psi>_{+} + rho_r <psi>_{-} = W0
      MQ[4][i] = 0.0;
      MQ[5][i] = 0.0;
    }
    apsi_acc<1, 0, 0>(hL, aL[0], rL, MQ[4]);
    apsi_acc<0, 1, 0>(hL, aL[1], rL, MQ[4]);
    apsi_acc<0, 0, 1>(hL, aL[2], rL, MQ[4]);
    apsi_acc<1, 0, 0>(hR, aR[0], rR, MQ[4]);
    apsi_acc<0, 1, 0>(hR, aR[1], rR, MQ[4]);
    apsi_acc<0, 0, 1>(hR, aR[2], rR, MQ[4]);
    apsi_acc<0, 0, 0>(hL, AL, rL, MQ[5]);
    apsi_acc<0, 0, 0>(hR, AR, rR, MQ[5]);

    T Qn[5], Qt[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      T qn = 0.0, qt = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        qn += al[k] * MQ[k][i];
        qt += be[k] * MQ[k][i];
      }
      Qn[i] = qn;
      Qt[i] = qt;
    }
    if (fc.Pr != 1.0) {
      // Prandtl fix (R20) on the non-equilibrium part: coefficients of C1 - T and C3 - T^2/2
      // combine to (alpha_1 - 1, beta_1) and (alpha_3, beta_3 - 1).
      T Fna[5], Fta[5], Qna[5], Qta[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        Fna[i] = o.Fn[i] - MF[0][i];
        Fta[i] = o.Ft[i] - MF[2][i];
        Qna[i] = Qn[i] - MQ[0][i];
        Qta[i] = Qt[i] - MQ[2][i];
      }
      const T uu = U0 * U0 + V0 * V0 + Ww0 * Ww0;
      const T qn = (Fna[4] - (U0 * Fna[1] + V0 * Fna[2] + Ww0 * Fna[3]) + 0.5 * uu * Fna[0]) -
                        U0 * (Qna[4] - (U0 * Qna[1] + V0 * Qna[2] + Ww0 * Qna[3]) + 0.5 * uu * Qna[0]);
      const T qt = (Fta[4] - (U0 * Fta[1] + V0 * Fta[2] + Ww0 * Fta[3]) + 0.5 * uu * Fta[0]) -
                        U0 * (Qta[4] - (U0 * Qta[1] + V0 * Qta[2] + Ww0 * Qta[3]) + 0.5 * uu * Qta[0]);
      const T pf = 1.0 / fc.Pr - 1.0;
      o.Fn[4] += pf * qn;
      o.Ft[4] += pf * qt;
    }
    if (COMPACT) {
      // side-state relaxation (R23)
      const T tau0 = fc.relax_C * jump * dt;
      const T e = (tau0 > 0.0) ? exp(-dt / tau0) : 0.0;
      const T w = 1.0 - e;
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        o.QLn[i] = w * Qn[i] + e * WL[i];
        o.QLt[i] = w * Qt[i] + e * dtWL[i];
        o.QRn[i] = w * Qn[i] + e * WR[i];
        o.QRt[i] = w * Qt[i] + e * dtWR[i];
      }
    }
  }
  return true;
}

}  // namespace cgks
