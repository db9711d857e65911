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

// ---------------------------------------------------------------------------
// Tangential moment table of a Maxwellian: t(a,b,c) = <v^a w^b eta^c>, eta = v^2 + w^2 + xi^2
// (v, w and xi are full-range Gaussians, so every psi_i psi_j moment factorises into a
// normal-velocity moment U_k times one of these 19 numbers).
// ---------------------------------------------------------------------------
template <typename T>
struct Tang {
  T v1, w1, e1, v2, vw, w2, ve, we, e2, v3, v2w, vw2, v2e, vwe, ve2, w3, w2e, we2;
};

template <typename T>
HD void tang_table(T V, T W, T lam, double N, Tang<T>& t) {
  const T s = 0.5 / lam;  // variance 1/(2 lam)
  // full 1-D moments
  const T V2 = V * V + s, W2 = W * W + s;
  const T V3 = V * V2 + 2.0 * s * V, W3 = W * W2 + 2.0 * s * W;
  const T V4 = V * V3 + 3.0 * s * V2, W4 = W * W3 + 3.0 * s * W2;
  const T V5 = V * V4 + 4.0 * s * V3, W5 = W * W4 + 4.0 * s * W3;
  const T X1 = N * s, X2 = N * (N + 2.0) * s * s;  // <xi^2>, <xi^4>
  t.v1 = V;
  t.w1 = W;
  t.v2 = V2;
  t.w2 = W2;
  t.vw = V * W;
  t.v3 = V3;
  t.w3 = W3;
  t.v2w = V2 * W;
  t.vw2 = V * W2;
  t.e1 = V2 + W2 + X1;
  t.ve = V3 + V * (W2 + X1);
  t.we = W3 + W * (V2 + X1);
  t.v2e = V4 + V2 * (W2 + X1);
  t.vwe = W * V3 + V * W3 + t.vw * X1;
  t.w2e = W4 + W2 * (V2 + X1);
  t.e2 = V4 + W4 + X2 + 2.0 * (V2 * W2 + X1 * (V2 + W2));
  t.ve2 = V5 + V * (W4 + X2) + 2.0 * (V3 * W2 + X1 * (V3 + V * W2));
  t.we2 = W5 + W * (V4 + X2) + 2.0 * (W3 * V2 + X1 * (W3 + W * V2));
}

// Entries of the symmetric moment matrix M_ij = <X psi_i psi_j>, X = u^p v^q w^r (q + r <= 1),
// psi_4 = (u^2 + eta)/2; upper entries e = 0..14 in the order (00,01,02,03,04,11,12,13,14,22,
// 23,24,33,34,44).  Entries are produced one at a time and applied to several vectors at
// once (sym_mv), so a matrix never occupies 15 registers.
__host__ __device__ constexpr int sym_i(int e) {
  return e < 5 ? 0 : (e < 9 ? 1 : (e < 12 ? 2 : (e < 14 ? 3 : 4)));
}
__host__ __device__ constexpr int sym_j(int e) {
  return e < 5 ? e : (e < 9 ? e - 4 : (e < 12 ? e - 7 : (e < 14 ? e - 9 : 4)));
}

template <int p, int q, int r, typename T>
HD T sym_entry(int e, const T* U, const Tang<T>& t) {
  // tangential factors g(a,b,c) = <v^(q+a) w^(r+b) eta^c> of this X
  const T g000 = (q == 0 && r == 0) ? T(1.0) : (q == 1 ? t.v1 : t.w1);
  const T g100 = (q == 0 && r == 0) ? t.v1 : (q == 1 ? t.v2 : t.vw);
  const T g010 = (q == 0 && r == 0) ? t.w1 : (q == 1 ? t.vw : t.w2);
  const T g001 = (q == 0 && r == 0) ? t.e1 : (q == 1 ? t.ve : t.we);
  const T g200 = (q == 0 && r == 0) ? t.v2 : (q == 1 ? t.v3 : t.v2w);
  const T g110 = (q == 0 && r == 0) ? t.vw : (q == 1 ? t.v2w : t.vw2);
  const T g101 = (q == 0 && r == 0) ? t.ve : (q == 1 ? t.v2e : t.vwe);
  const T g020 = (q == 0 && r == 0) ? t.w2 : (q == 1 ? t.vw2 : t.w3);
  const T g011 = (q == 0 && r == 0) ? t.we : (q == 1 ? t.vwe : t.w2e);
  const T g002 = (q == 0 && r == 0) ? t.e2 : (q == 1 ? t.ve2 : t.we2);
  switch (e) {
    case 0: return U[p] * g000;
    case 1: return U[p + 1] * g000;
    case 2: return U[p] * g100;
    case 3: return U[p] * g010;
    case 4: return 0.5 * (U[p + 2] * g000 + U[p] * g001);
    case 5: return U[p + 2] * g000;
    case 6: return U[p + 1] * g100;
    case 7: return U[p + 1] * g010;
    case 8: return 0.5 * (U[p + 3] * g000 + U[p + 1] * g001);
    case 9: return U[p] * g200;
    case 10: return U[p] * g110;
    case 11: return 0.5 * (U[p + 2] * g100 + U[p] * g101);
    case 12: return U[p] * g020;
    case 13: return 0.5 * (U[p + 2] * g010 + U[p] * g011);
    default: return 0.25 * (U[p + 4] * g000 + 2.0 * U[p + 2] * g001 + U[p] * g002);
  }
}

// out[v] += M a[v] for NV vectors; with COL0 also col0 += M e_0 (= <X psi>)
template <int p, int q, int r, int NV, bool COL0, typename T>
HD void sym_mv(const T* U, const Tang<T>& t, const T (*a)[5], T (*out)[5], T* col0) {
#pragma unroll
  for (int e = 0; e < 15; ++e) {
    const int i = sym_i(e), j = sym_j(e);
    const T m = sym_entry<p, q, r>(e, U, t);
    if (COL0 && i == 0) col0[j] += m;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      out[v][i] += m * a[v][j];
      if (i != j) out[v][j] += m * a[v][i];
    }
  }
}

// heat-flux functional of a flux-moment vector about U0 (R20):
// qF(v) = v_E - U0 . v_mom + |U0|^2/2 v_rho; a state vector Q contributes -U0n qF(Q)
template <typename T>
HD T qF(const T* v, T U0, T V0, T W0, T uu2) {
  return v[4] - (U0 * v[1] + V0 * v[2] + W0 * v[3]) + uu2 * v[0];
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
  q.dp = gm1 * (d[4] - (U[0] * d[1] + U[1] * d[2] + U[2] * d[3]) + uu2 * d[0]);
  q.udu = U[0] * q.du[0] + U[1] * q.du[1] + U[2] * q.du[2];
  return q;
}

// acc += s DF_al(W) d, F_al = (m_al, m_al U + p e_al, U_al (E + p)) the Euler flux along al
template <int AL, typename T, typename S>
HD void jvp_flux(T rho, const T* U, T p, T E, const T* d, const Dprim<T>& q, S s, T* acc) {
  const T mA = rho * U[AL];
  acc[0] += s * d[1 + AL];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    T v = d[1 + AL] * U[b] + mA * q.du[b];
    if (b == AL) v += q.dp;
    acc[1 + b] += s * v;
  }
  acc[4] += s * (q.du[AL] * (E + p) + U[AL] * (d[4] + q.dp));
}

// acc += DH_al(W) d, H_al = rho <u_n u_al psi> (n = 0, the face normal):
//   H[0] = rho U_n U_al + p d_{n al}
//   H[b] = rho U_n U_al U_b + p (d_{n al} U_b + d_{n b} U_al + d_{al b} U_n)
//   H[4] = ((rho |U|^2 + (N+7) p) U_n U_al + (p |U|^2 + (N+5) p^2/rho) d_{n al}) / 2
template <int AL, typename T>
HD void jvp_flux2(T rho, T ir, const T* U, T p, T uu, double K5, double K7, const Dprim<T>& q, T* acc) {
  const T UnUa = U[0] * U[AL];
  const T dUnUa = q.du[0] * U[AL] + U[0] * q.du[AL];
  acc[0] += q.dr * UnUa + rho * dUnUa;
  if (AL == 0) acc[0] += q.dp;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    T v = q.dr * UnUa * U[b] + rho * (dUnUa * U[b] + UnUa * q.du[b]);
    if (AL == 0) v += q.dp * U[b] + p * q.du[b];
    if (b == 0) v += q.dp * U[AL] + p * q.du[AL];
    if (AL == b) v += q.dp * U[0] + p * q.du[0];
    acc[1 + b] += v;
  }
  const T c1 = rho * uu + K7 * p;
  const T dc1 = q.dr * uu + 2.0 * rho * q.udu + K7 * q.dp;
  T v4 = dc1 * UnUa + c1 * dUnUa;
  if (AL == 0) v4 += q.dp * uu + 2.0 * p * q.udu + K5 * p * ir * (2.0 * q.dp - p * ir * q.dr);
  acc[4] += 0.5 * v4;
}

// per-lane parking slots (shared memory on the device) for values that live across phases
struct ParkDev {
  double* base;  // base + slot * 128 + lane
  __device__ __forceinline__ void put(int s, double v) const { base[s * 128] = v; }
  __device__ __forceinline__ double get(int s) const { return base[s * 128]; }
  __device__ __forceinline__ void mark(int) const {}  // phase markers (used by the host flop count)
};

// ---------------------------------------------------------------------------
// One side of the interface solver at one Gauss point (two cooperating lanes per Gauss
// point: side 0 = left state restricted to u > 0, side 1 = right state restricted to u < 0).
// Phases: (A1) own half-range contributions to W0 and dW0 -> exchange (lane xor 1) ->
// (G) interface equilibrium g0, collision time and combined time coefficients, equilibrium
// terms of Eq. (flux) folded into F^n, F_t^n, Q^n, Q_t^n and the heat-flux scalars ->
// (A2) own compatibility coefficients A and own half-range flux/state terms -> exchange ->
// Prandtl fix and own side relaxation.  Both lanes run the same instruction stream.
// Inputs in the normal frame: W (5) conservative state of this side, dW[dir][var] physical
// derivatives (dir 0 = normal).  Outputs (normal frame): side 0 holds Fn, Ft, QLn, QLt;
// side 1 holds Fn, Ft and its QRn, QRt in the QLn/QLt slots.  Returns false if a state
// (own, other, or the equilibrium) is not positive.
// ---------------------------------------------------------------------------
template <bool COMPACT, typename T, typename X, typename P>
HD bool gks_flux_side(int side, const T* W, const T (*dW)[5], T dt, const FluxConst& fc, const X& xchg,
                      const P& park, GPOutT<T>& o) {
  const T gm1 = fc.gamma - 1.0;
  const double sgn = side == 0 ? 1.0 : -1.0;
  // ---- (A1) primitives, moments and micro-slopes of this side (R15)
  const T rho = W[0], ir = 1.0 / rho;
  const T U = W[1] * ir, V = W[2] * ir, Ww = W[3] * ir;
  const T p = gm1 * (W[4] - 0.5 * rho * (U * U + V * V + Ww * Ww));
  const bool ok = (rho > 0.0) && (p > 0.0);
  const T lam = ok ? T(0.5) * rho / p : T(1.0);
  T a[3][5];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    T b[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) b[i] = dW[d][i] * ir;
    micro_slope(U, V, Ww, lam, fc.N, b, a[d]);
  }
  T x1[21];
  {
    T Uh[7];
    half_moments(U, lam, sgn, Uh);  // H(u) or 1-H(u)
    Tang<T> tg;
    tang_table(V, Ww, lam, fc.N, tg);
    T dw0[3][5], w0[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      w0[i] = 0.0;
      dw0[0][i] = dw0[1][i] = dw0[2][i] = 0.0;
    }
    sym_mv<0, 0, 0, 3, true>(Uh, tg, a, dw0, w0);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      x1[i] = rho * w0[i];  // W0 part (R13)
#pragma unroll
      for (int d = 0; d < 3; ++d) x1[5 + 5 * d + i] = rho * dw0[d][i];  // dW0 part (R14)
    }
  }
  x1[20] = p;
  // Euler time derivative of this side (R23): dW/dt = rho <A psi> = -sum_al DF_al(W) dW_al (full
  // moments, compatibility R16), as Jacobian-vector products
  {
    const T Uv[3] = {U, V, Ww};
    const T uu2s = 0.5 * (U * U + V * V + Ww * Ww);
    T dtw[5] = {0, 0, 0, 0, 0};
    const Dprim<T> q0 = dprim(ir, Uv, uu2s, fc.gamma - 1.0, dW[0]);
    jvp_flux<0>(rho, Uv, p, W[4], dW[0], q0, -1.0, dtw);
    const Dprim<T> q1 = dprim(ir, Uv, uu2s, fc.gamma - 1.0, dW[1]);
    jvp_flux<1>(rho, Uv, p, W[4], dW[1], q1, -1.0, dtw);
    const Dprim<T> q2 = dprim(ir, Uv, uu2s, fc.gamma - 1.0, dW[2]);
    jvp_flux<2>(rho, Uv, p, W[4], dW[2], q2, -1.0, dtw);
#pragma unroll
    for (int i = 0; i < 5; ++i) park.put(15 + i, dtw[i]);
  }
  // park what the own-side phase A2 needs (a, dW/dt): frees registers during the equilibrium phase
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int i = 0; i < 5; ++i) park.put(5 * d + i, a[d][i]);
  // ---- exchange 1: W0, dW0 = sum of the two half-range contributions
  const bool ok_other = xchg.flag(ok);
  T other_p;
  {
#pragma unroll
    for (int i = 0; i < 21; ++i) {
      const T y = xchg(x1[i]);
      if (i < 20)
        x1[i] += y;
      else
        other_p = y;
    }
  }
  bool good = ok && ok_other;
  park.mark(1);  // start of the equilibrium phase (identical in both lanes)
  const T pL = side == 0 ? p : other_p, pR = side == 0 ? other_p : p;
  // ---- (G) interface equilibrium g0 (R13, R14)
  const T r0 = x1[0], i0 = 1.0 / r0;
  const T U0 = x1[1] * i0, V0 = x1[2] * i0, Ww0 = x1[3] * i0;
  const T uu2 = 0.5 * (U0 * U0 + V0 * V0 + Ww0 * Ww0);
  const T p0 = gm1 * (x1[4] - r0 * uu2);
  good = good && (r0 > 0.0) && (p0 > 0.0);
  const T l0 = good ? T(0.5) * r0 / p0 : T(1.0);
  // collision time (R17) and combined time coefficients:
  // F^n = sum alpha_k MF_k, F_t^n = sum beta_k MF_k (E2 = e^{-dt/(2tau)}, tau = 0 -> Euler limit)
  const T jump = fabs((pL - pR) / (pL + pR));
  const T tau = (fc.mu > 0.0) ? (fc.mu / p0 + fc.tau_C * jump * dt) : (fc.tau_eps + fc.tau_C * jump) * dt;
  T al[6], be[6];
  {
    const T idt = 1.0 / dt;
    const T E2 = exp(-0.5 * dt / tau);
    const T m2 = -expm1(-0.5 * dt / tau);
    const T c3 = tau * m2 * (3.0 - E2) * idt;
    const T qq = 4.0 * tau * m2 * m2 * idt * idt;
    al[0] = 1.0 - c3;
    be[0] = qq;
    al[1] = 2.0 * tau * c3 - tau * (1.0 + 2.0 * E2 - E2 * E2);
    be[1] = 4.0 * tau * m2 * (dt * E2 - 2.0 * tau * m2) * idt * idt;
    al[2] = -tau + tau * c3;
    be[2] = 1.0 - tau * qq;
    al[3] = c3;
    be[3] = -qq;
    al[4] = -2.0 * tau * c3 + tau * E2 * (2.0 - E2);
    be[4] = -be[1];
    al[5] = -tau * c3;
    be[5] = tau * qq;
  }
  // accumulators: Fn, Ft, Qn, Qt, and the heat-flux scalars qn, qt of the Prandtl fix (R20):
  // q = sum_k alpha'_k s_k with s_k = qF(MF_k) - U0n qF(MQ_k), alpha'_0 = alpha_0 - 1,
  // beta'_2 = beta_2 - 1 (non-equilibrium part f - (T g0 + T^2/2 Abar g0))
  T acc[22];
  {
    const T sW = qF(x1, U0, V0, Ww0, uu2);  // qF(W0); MQ0 = MQ3 = W0
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      acc[i] = 0.0;
      acc[5 + i] = 0.0;
      acc[10 + i] = (al[0] + al[3]) * x1[i];
      acc[15 + i] = (be[0] + be[3]) * x1[i];
    }
    acc[20] = -U0 * sW * (al[0] - 1.0 + al[3]);
    acc[21] = -U0 * sW * (be[0] + be[3]);
  }
  {
    // equilibrium terms (full Maxwellian g0): MF0 = F_n(W0), MQa = rho0 <(abar.u) psi> =
    // sum_al DF_al(W0) dW0_al, MF1 = rho0 <u (abar.u) psi> = sum_al DH_al(W0) dW0_al,
    // MF2 = rho0 <u Abar psi> = DF_n(W0) (rho0 <Abar psi>) = -DF_n(W0) MQa (compatibility R16)
    const T U0v[3] = {U0, V0, Ww0};
    const T uu0 = 2.0 * uu2;
    const double K5 = fc.N + 5.0, K7 = fc.N + 7.0;
    T MQa[1][5], MF1[1][5], MF2[1][5], MF0[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) MQa[0][i] = MF1[0][i] = MF2[0][i] = 0.0;
    {
      const T* d0 = x1 + 5;
      const Dprim<T> q0 = dprim(i0, U0v, uu2, fc.gamma - 1.0, d0);
      jvp_flux<0>(r0, U0v, p0, x1[4], d0, q0, 1.0, MQa[0]);
      jvp_flux2<0>(r0, i0, U0v, p0, uu0, K5, K7, q0, MF1[0]);
      const T* d1 = x1 + 10;
      const Dprim<T> q1 = dprim(i0, U0v, uu2, fc.gamma - 1.0, d1);
      jvp_flux<1>(r0, U0v, p0, x1[4], d1, q1, 1.0, MQa[0]);
      jvp_flux2<1>(r0, i0, U0v, p0, uu0, K5, K7, q1, MF1[0]);
      const T* d2 = x1 + 15;
      const Dprim<T> q2 = dprim(i0, U0v, uu2, fc.gamma - 1.0, d2);
      jvp_flux<2>(r0, U0v, p0, x1[4], d2, q2, 1.0, MQa[0]);
      jvp_flux2<2>(r0, i0, U0v, p0, uu0, K5, K7, q2, MF1[0]);
      const Dprim<T> qa = dprim(i0, U0v, uu2, fc.gamma - 1.0, MQa[0]);
      jvp_flux<0>(r0, U0v, p0, x1[4], MQa[0], qa, -1.0, MF2[0]);
    }
    MF0[0] = r0 * U0;
    MF0[1] = r0 * U0 * U0 + p0;
    MF0[2] = r0 * U0 * V0;
    MF0[3] = r0 * U0 * Ww0;
    MF0[4] = U0 * (x1[4] + p0);
    const T sMF0 = qF(MF0, U0, V0, Ww0, uu2), sMF1 = qF(MF1[0], U0, V0, Ww0, uu2),
            sMF2 = qF(MF2[0], U0, V0, Ww0, uu2), sMQa = qF(MQa[0], U0, V0, Ww0, uu2);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const T mf0 = MF0[i], mf1 = MF1[0][i], mf2 = MF2[0][i], mqa = MQa[0][i];
      acc[i] += al[0] * mf0 + al[1] * mf1 + al[2] * mf2;
      acc[5 + i] += be[0] * mf0 + be[1] * mf1 + be[2] * mf2;
      acc[10 + i] += (al[1] - al[2]) * mqa;  // MQ1 = MQa, MQ2 = -MQa (compatibility)
      acc[15 + i] += (be[1] - be[2]) * mqa;
    }
    // s0 = qF(MF0) - U0n qF(W0) (W0 part added above), s1 = qF(MF1) - U0n qF(MQa), s2 = qF(MF2) + U0n qF(MQa)
    acc[20] += (al[0] - 1.0) * sMF0 + al[1] * (sMF1 - U0 * sMQa) + al[2] * (sMF2 + U0 * sMQa);
    acc[21] += be[0] * sMF0 + be[1] * (sMF1 - U0 * sMQa) + (be[2] - 1.0) * (sMF2 + U0 * sMQa);
  }
  // the whole equilibrium phase is executed identically by both lanes (counted once)
  park.mark(2);
  park.mark(3);
  park.mark(4);
  // ---- (A2) own side: compatibility coefficients A (R16), Euler time derivative (R23),
  // half-range flux and state terms of this side
  T sacc[22];
  T dtW[5];
  {
    T a2[3][5];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int i = 0; i < 5; ++i) a2[d][i] = park.get(5 * d + i);
    Tang<T> tg;
    tang_table(V, Ww, lam, fc.N, tg);
    T A[1][5];
    {
      T b[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        dtW[i] = park.get(15 + i);
        b[i] = dtW[i] * ir;
      }
      micro_slope(U, V, Ww, lam, fc.N, b, A[0]);  // A = M^{-1}(-<(a.u) psi>) (R16)
    }
    T Uh[7];
    half_moments(U, lam, sgn, Uh);
    // MF3 = <u psi>, MF5 = <u A psi>, MQ4 = <(a.u) psi>, MF4 = <u (a.u) psi>, MQ5 = <A psi> (x rho)
    T MF3[5], MF5[1][5], MQ4[1][5], MF4[1][5], MQ5[1][5];
#pragma unroll
    for (int i = 0; i < 5; ++i) MF3[i] = MF5[0][i] = MQ4[0][i] = MF4[0][i] = MQ5[0][i] = 0.0;
    {
      T vv[2][5], oo[2][5];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        vv[0][i] = A[0][i];
        vv[1][i] = a2[0][i];
        oo[0][i] = oo[1][i] = 0.0;
      }
      sym_mv<1, 0, 0, 2, true>(Uh, tg, vv, oo, MF3);
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        MF5[0][i] = oo[0][i];
        MQ4[0][i] = oo[1][i];
      }
    }
    sym_mv<0, 1, 0, 1, false>(Uh, tg, &a2[1], MQ4, (T*)nullptr);
    sym_mv<0, 0, 1, 1, false>(Uh, tg, &a2[2], MQ4, (T*)nullptr);
    sym_mv<2, 0, 0, 1, false>(Uh, tg, &a2[0], MF4, (T*)nullptr);
    sym_mv<1, 1, 0, 1, false>(Uh, tg, &a2[1], MF4, (T*)nullptr);
    sym_mv<1, 0, 1, 1, false>(Uh, tg, &a2[2], MF4, (T*)nullptr);
    sym_mv<0, 0, 0, 1, false>(Uh, tg, A, MQ5, (T*)nullptr);
    const T s3 = rho * qF(MF3, U0, V0, Ww0, uu2);
    const T s4 = rho * (qF(MF4[0], U0, V0, Ww0, uu2) - U0 * qF(MQ4[0], U0, V0, Ww0, uu2));
    const T s5 = rho * (qF(MF5[0], U0, V0, Ww0, uu2) - U0 * qF(MQ5[0], U0, V0, Ww0, uu2));
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const T mf3 = rho * MF3[i], mf4 = rho * MF4[0][i], mf5 = rho * MF5[0][i];
      const T mq4 = rho * MQ4[0][i], mq5 = rho * MQ5[0][i];
      sacc[i] = al[3] * mf3 + al[4] * mf4 + al[5] * mf5;
      sacc[5 + i] = be[3] * mf3 + be[4] * mf4 + be[5] * mf5;
      sacc[10 + i] = al[4] * mq4 + al[5] * mq5;
      sacc[15 + i] = be[4] * mq4 + be[5] * mq5;
    }
    sacc[20] = al[3] * s3 + al[4] * s4 + al[5] * s5;
    sacc[21] = be[3] * s3 + be[4] * s4 + be[5] * s5;
  }
  // ---- exchange 2: add the other side's half-range terms
#pragma unroll
  for (int i = 0; i < 22; ++i) acc[i] += sacc[i] + xchg(sacc[i]);
  // ---- Prandtl fix (R20) and outputs
  if (fc.Pr != 1.0) {
    const double pf = 1.0 / fc.Pr - 1.0;
    acc[4] += pf * acc[20];
    acc[9] += pf * acc[21];
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    o.Fn[i] = acc[i];
    o.Ft[i] = acc[5 + i];
  }
  if (COMPACT) {
    // side-state relaxation of this side (R23)
    const T tau0 = fc.relax_C * jump * dt;
    const T ee = (tau0 > 0.0) ? exp(-dt / tau0) : T(0.0);
    const T w = 1.0 - ee;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      o.QLn[i] = w * acc[10 + i] + ee * W[i];
      o.QLt[i] = w * acc[15 + i] + ee * dtW[i];
    }
  }
  return good;
}

}  // namespace cgks
