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
  // park what the own-side phase A2 needs (a, W): frees registers during the equilibrium phase
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
    T U0f[7];
    full_moments(U0, l0, U0f);
    Tang<T> t0;
    tang_table(V0, Ww0, l0, fc.N, t0);
    T ab[3][5];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      T b[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) b[i] = x1[5 + 5 * d + i] * i0;
      micro_slope(U0, V0, Ww0, l0, fc.N, b, ab[d]);
    }
    park.mark(2);  // end of the first duplicated block
    // MQa = rho0 <(abar.u) psi> (lane side 0) and MF1 = rho0 <u (abar.u) psi> (lane side 1) are the same
    // three contractions with the normal-velocity moments shifted by one order: one code path,
    // moments shifted by `side`, then one exchange
    T MQa[1][5], MF1[1][5];
    {
      T U0s[6];
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) U0s[kk] = side ? U0f[kk + 1] : U0f[kk];
      T Xs[1][5];
#pragma unroll
      for (int i = 0; i < 5; ++i) Xs[0][i] = 0.0;
      sym_mv<1, 0, 0, 1, false>(U0s, t0, &ab[0], Xs, (T*)nullptr);
      sym_mv<0, 1, 0, 1, false>(U0s, t0, &ab[1], Xs, (T*)nullptr);
      sym_mv<0, 0, 1, 1, false>(U0s, t0, &ab[2], Xs, (T*)nullptr);
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const T y = xchg(Xs[0][i]);
        MQa[0][i] = side ? y : Xs[0][i];
        MF1[0][i] = side ? Xs[0][i] : y;
      }
    }
    park.mark(3);  // start of the second duplicated block
    // Abar from compatibility (R16): <(abar.u + Abar) psi> = 0
    T Ab[1][5];
    {
      T b[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) b[i] = -MQa[0][i];
      micro_slope(U0, V0, Ww0, l0, fc.N, b, Ab[0]);
    }
    // MF0 = rho0 <u psi>, MF2 = rho0 <u Abar psi>
    T MF2[1][5], MF0[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) MF2[0][i] = MF0[i] = 0.0;
    sym_mv<1, 0, 0, 1, true>(U0f, t0, Ab, MF2, MF0);
    const T sMF0 = r0 * qF(MF0, U0, V0, Ww0, uu2), sMF1 = r0 * qF(MF1[0], U0, V0, Ww0, uu2),
            sMF2 = r0 * qF(MF2[0], U0, V0, Ww0, uu2), sMQa = r0 * qF(MQa[0], U0, V0, Ww0, uu2);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const T mf0 = r0 * MF0[i], mf1 = r0 * MF1[0][i], mf2 = r0 * MF2[0][i], mqa = r0 * MQa[0][i];
      acc[i] += al[0] * mf0 + al[1] * mf1 + al[2] * mf2;
      acc[5 + i] += be[0] * mf0 + be[1] * mf1 + be[2] * mf2;
      acc[10 + i] += (al[1] - al[2]) * mqa;  // MQ1 = MQa, MQ2 = -MQa (compatibility)
      acc[15 + i] += (be[1] - be[2]) * mqa;
    }
    // s0 = qF(MF0) - U0n qF(W0) (W0 part added above), s1 = qF(MF1) - U0n qF(MQa), s2 = qF(MF2) + U0n qF(MQa)
    acc[20] += (al[0] - 1.0) * sMF0 + al[1] * (sMF1 - U0 * sMQa) + al[2] * (sMF2 + U0 * sMQa);
    acc[21] += be[0] * sMF0 + be[1] * (sMF1 - U0 * sMQa) + (be[2] - 1.0) * (sMF2 + U0 * sMQa);
  }
  park.mark(4);  // end of the equilibrium phase
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
      T Uf[7];
      full_moments(U, lam, Uf);
      T b[1][5];
#pragma unroll
      for (int i = 0; i < 5; ++i) b[0][i] = 0.0;
      sym_mv<1, 0, 0, 1, false>(Uf, tg, &a2[0], b, (T*)nullptr);
      sym_mv<0, 1, 0, 1, false>(Uf, tg, &a2[1], b, (T*)nullptr);
      sym_mv<0, 0, 1, 1, false>(Uf, tg, &a2[2], b, (T*)nullptr);
#pragma unroll
      for (int i = 0; i < 5; ++i) b[0][i] = -b[0][i];
      micro_slope(U, V, Ww, lam, fc.N, b[0], A[0]);
#pragma unroll
      for (int i = 0; i < 5; ++i) dtW[i] = rho * b[0][i];
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
