// flux_ws.cuh -- warp-specialised CGKS-5th interface-flux kernel for 3-D grids (sm_100a).
//
// The generic k_flux runs the interface part of the gas-kinetic solver (equilibrium g0, collision
// time, time coefficients, Jacobian-vector products, fold, Prandtl fix) in both lanes of a Gauss
// point to stay convergent.  Here a block has 2 "side" warps and 1 "interface" warp:
//   side warps (64 lanes = 8 faces x 4 Gauss points x 2 sides): TMA tile staging, face-plane
//     evaluation of both cells' quartics, the half-range terms of each side (side_terms), one
//     shuffle sums the two sides, and the sums plus each side's W, dW/dt go to a shared handoff;
//   interface warp (32 lanes = one per Gauss point): interface_terms once per Gauss point, the
//     relaxation of both sides, the 2x2 Gauss-point sum and the face record stores.
// Named barriers hand the buffer over (1 = full, 2 = empty, 3 = side warps only); the next tile's
// TMA is issued as soon as the evaluation has consumed the current one, so it lands while the side
// terms are computed.  Blocks are persistent over batches of 8 faces (P:93-129, P:142-150,
// P:324-354; same arithmetic as k_flux, ~20 % fewer instructions per Gauss point).
#pragma once

namespace cgks {

template <int AX>
struct FluxWS {
  static constexpr int NG = 4;                           // Gauss points per face
  static constexpr int FPB = 8;                          // faces per batch
  static constexpr int FY = AX == 0 ? 1 : 2;             // faces along the normal axis
  static constexpr int FX = FPB / FY;                    // faces along x
  static constexpr int NT = AX == 0 ? FX + 2 : FX * (FY + 1);  // tile cells (x: from the even cell i0 - 2)
  static constexpr int TX = AX == 0 ? NT : FX;
  static constexpr int TN = AX == 0 ? 1 : FY + 1;
  static constexpr int NB = 34;
  static constexpr int NREC = NB * 5;
  static constexpr int NQ = 4;
  static constexpr int TS = NB + 1;
  static constexpr int FS = AX == 2 ? FX : NT;           // field stride of the tile
  __host__ __device__ static constexpr int cbase(int c, int nfield) {
    return AX == 2 ? (c / FX) * nfield * FX + c % FX : c;
  }
  static constexpr int STILE = (NREC * NT + 15) / 16 * 16;
  static constexpr int TILE = STILE + 5 * NT;
  static constexpr int TAB = 2 * NQ * TS;
  static constexpr int NS = 64;                          // side lanes
  static constexpr int XS = 20 * NS;                     // evaluation scatter slots
  static constexpr int NH = 68;                          // handoff values per Gauss point
  static constexpr int HAND = NH * 32;
  static constexpr int OFF_TAB = (TILE + 15) / 16 * 16;
  static constexpr int OFF_XS = OFF_TAB + TAB;
  static constexpr int OFF_HAND = OFF_XS + XS;
  static constexpr int OFF_BAR = OFF_HAND + HAND;
  static constexpr size_t smem_bytes() { return sizeof(double) * (size_t)OFF_BAR + 16; }
};

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// batch b -> face origin (i0, j0, k0); grid order x fastest, then the normal axis, then the other
template <int AX>
__device__ __forceinline__ void ws_batch(long long b, int& i0, int& j0, int& k0) {
  using FT = FluxWS<AX>;
  const int nbx = (c_geo.fn[AX][0] + FT::FX - 1) / FT::FX;
  const int ib = (int)(b % nbx);
  const long long r = b / nbx;
  i0 = ib * FT::FX;
  if (AX == 0) {
    j0 = (int)(r % c_geo.fn[0][1]);
    k0 = (int)(r / c_geo.fn[0][1]);
  } else if (AX == 1) {
    const int nby = (c_geo.fn[1][1] + FT::FY - 1) / FT::FY;
    j0 = (int)(r % nby) * FT::FY;
    k0 = (int)(r / nby);
  } else {
    const int nbz = (c_geo.fn[2][2] + FT::FY - 1) / FT::FY;
    k0 = (int)(r % nbz) * FT::FY;
    j0 = (int)(r / nbz);
  }
}

template <int AX>
__device__ __forceinline__ long long ws_nbatch() {
  using FT = FluxWS<AX>;
  const long long nbx = (c_geo.fn[AX][0] + FT::FX - 1) / FT::FX;
  if (AX == 0) return nbx * c_geo.fn[0][1] * c_geo.fn[0][2];
  if (AX == 1) return nbx * ((c_geo.fn[1][1] + FT::FY - 1) / FT::FY) * c_geo.fn[1][2];
  return nbx * ((c_geo.fn[2][2] + FT::FY - 1) / FT::FY) * c_geo.fn[2][1];
}

// stage the tile of the batch at face origin (i0, j0, k0): TMA when it needs no periodic wrap
// (returns true: completion on the mbarrier), otherwise cp.async by the 64 side lanes
template <int AX>
__device__ __forceinline__ bool ws_stage(const double* __restrict__ U, const double* __restrict__ rec, double* tile,
                                         uint64_t* bar, const CUtensorMap* tm_rec, const CUtensorMap* tm_U, int i0,
                                         int j0, int k0, int t) {
  using FT = FluxWS<AX>;
  constexpr int NT = FT::NT, FX = FT::FX;
  const int x0 = AX == 0 ? i0 - 2 : i0, y0 = AX == 1 ? j0 - 1 : j0, z0 = AX == 2 ? k0 - 1 : k0;
  const bool wraps = (AX == 0 && x0 < 0 && !c_geo.bounded[0]) || (AX == 1 && y0 < 0 && !c_geo.bounded[1]) ||
                     (AX == 2 && z0 < 0 && !c_geo.bounded[2]);
  if (!wraps) {
    if (t == 0) {
      mbar_expect_tx(bar, (unsigned)(sizeof(double) * (FT::NREC + 5) * NT));
      tma_load_4d(tile, tm_rec, bar, x0 - c_geo.elo[0], y0 - c_geo.elo[1], 0, z0 - c_geo.elo[2]);
      tma_load_4d(tile + FT::STILE, tm_U, bar, x0, y0, 0, z0 + c_geo.zoff);
    }
    return true;
  }
  constexpr int TPC = FT::NS / NT;  // side lanes per tile cell
  const int c = t % NT, fsub = t / NT;
  if (fsub < TPC) {
    int ci, cj = j0, ck = k0;
    if (AX == 0) {
      ci = i0 - 2 + c;
      if (c_geo.bounded[0] && ci < -1) ci = -1;
    } else {
      ci = i0 + c % FX;
      if (AX == 1) cj += c / FX - 1;
      if (AX == 2) ck += c / FX - 1;
    }
    const int imax = c_geo.n[0] - 1 + (c_geo.bounded[0] ? 1 : 0);
    if (ci > imax) ci = imax;
    if (AX == 1) {
      const int jmax = c_geo.n[1] - 1 + (c_geo.bounded[1] ? 1 : 0);
      if (cj > jmax) cj = jmax;
    }
    if (AX == 2) {
      const int kmax = c_geo.n[2] - 1 + (c_geo.bounded[2] ? 1 : 0);
      if (ck > kmax) ck = kmax;
    }
    const long long st = c_geo.eplane;
    const double* src = rec + eidx(FT::NREC, 0, ci, cj, ck) + fsub * st;
    unsigned dst = (unsigned)__cvta_generic_to_shared(tile + FT::cbase(c, FT::NREC) + fsub * FT::FS);
    for (int fld = fsub; fld < FT::NREC; fld += TPC) {
      cp_async8s(dst, src);
      src += TPC * st;
      dst += TPC * FT::FS * (unsigned)sizeof(double);
    }
    const double* ub = U + sidx(20, 0, wrap_ax(0, ci), wrap_ax(1, cj), wrap_ax(2, ck));
    double* sdst = tile + FT::STILE + FT::cbase(c, 5);
    for (int v = fsub; v < 5; v += TPC) cp_async8(sdst + v * FT::FS, ub + v * c_geo.plane);
  }
  return false;
}

template <int AX>
__global__ void __launch_bounds__(96, 4) k_flux_ws(const double* __restrict__ U, const double* __restrict__ rec,
                                                   const double* __restrict__ gtab, double* __restrict__ face,
                                                   const TimeState* __restrict__ ts, ErrState* __restrict__ err,
                                                   int stage, const __grid_constant__ CUtensorMap tm_rec,
                                                   const __grid_constant__ CUtensorMap tm_U) {
  using FT = FluxWS<AX>;
  constexpr int NT = FT::NT, NB = FT::NB, FX = FT::FX, NQ = FT::NQ, NS = FT::NS;
  constexpr int NF = 30;
  extern __shared__ __align__(128) double smem[];
  double* tile = smem;
  double* tab = smem + FT::OFF_TAB;
  double* xs = smem + FT::OFF_XS;      // [q*5 + v][64]
  double* hand = smem + FT::OFF_HAND;  // [value][32]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FT::OFF_BAR);
  if (err->code) return;
  const int t = threadIdx.x;
  const long long nb = ws_nbatch<AX>();
  const double dt = ts->dt, idt = ts->idt;
  constexpr int P0 = AX, P1 = (AX + 1) % 3, P2 = (AX + 2) % 3;
  if (t < NS) {
    // =========================== side warps ===========================
    const int side = t & 1, gp = (t >> 1) & 3, fl = t >> 3;
    const int fx = fl % FX, fy = fl / FX;
    if (t == 0) mbar_init(bar, 1);
    for (int q = t; q < 2 * NQ * FT::TS; q += NS) cp_async8(tab + q, gtab + q);
    nbar_sync(3, NS);  // barrier initialised
    unsigned phase = 0;
    long long b = blockIdx.x;
    int i0 = 0, j0 = 0, k0 = 0;
    bool tma_cur = false;
    if (b < nb) {
      ws_batch<AX>(b, i0, j0, k0);
      tma_cur = ws_stage<AX>(U, rec, tile, bar, &tm_rec, &tm_U, i0, j0, k0, t);
    }
    bool first = true;
    for (; b < nb; b += gridDim.x) {
      // ---- this batch's tile has landed
      cp_async_wait_all();
      if (tma_cur) {
        mbar_wait(bar, phase);
        phase ^= 1;
      }
      nbar_sync(3, NS);
      // ---- evaluation of this side's quartic at the face Gauss points (face-plane parity form)
      const int c = AX == 0 ? fl + side + 1 : (fy + side) * FX + fx;
      const double* tc = tile + FT::cbase(c, FT::NREC);
      const double* sc = tile + FT::STILE + FT::cbase(c, 5);
      constexpr int TA = P1, TB = P2;
      {
        const double* T = tab + (side * NQ + gp) * FT::TS;
        double S[5][4];
#pragma unroll
        for (int v = 0; v < 5; ++v)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) S[v][cc] = 0.0;
#pragma unroll
        for (int kk = 0; kk < NB; ++kk) {
          const int cls = (ReconGen<3>::expo(kk, TA) & 1) | ((ReconGen<3>::expo(kk, TB) & 1) << 1);
          const double tt = T[kk];
#pragma unroll
          for (int v = 0; v < 5; ++v) S[v][cls] = fma(tc[(kk * 5 + v) * FT::FS], tt, S[v][cls]);
        }
        const int flip = gp == 2 ? 1 : (gp == 3 ? 2 : 0);
#pragma unroll
        for (int g2 = 0; g2 < 4; ++g2) {
          const double sA = (g2 & 1) ? 1.0 : -1.0, sB = (g2 & 2) ? 1.0 : -1.0;
          const double chi = ((flip & 1) ? sA : 1.0) * ((flip & 2) ? sB : 1.0);
          double* dst = xs + (t - 2 * gp + 2 * g2);
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            double val = S[v][0];
            val = fma(sA, S[v][1], val);
            val = fma(sB, S[v][2], fma(sA * sB, S[v][3], val));
            dst[(gp * 5 + v) * NS] = chi * val;
          }
        }
      }
      double Wc[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) Wc[v] = sc[v * FT::FS];
      // the tile is consumed: prefetch the next batch's tile while this batch's side terms run
      nbar_sync(3, NS);
      const long long bn = b + gridDim.x;
      int ni0 = 0, nj0 = 0, nk0 = 0;
      bool tma_next = false;
      if (bn < nb) {
        ws_batch<AX>(bn, ni0, nj0, nk0);
        tma_next = ws_stage<AX>(U, rec, tile, bar, &tm_rec, &tm_U, ni0, nj0, nk0, t);
      }
      double wn[5], dn[3][5];
      {
        double W[5], g[3][5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          W[v] = Wc[v] + xs[v * NS + t];
          g[AX][v] = xs[(5 + v) * NS + t] * c_geo.ih[AX];
          g[TA][v] = xs[(10 + v) * NS + t] * c_geo.ih[TA];
          g[TB][v] = xs[(15 + v) * NS + t] * c_geo.ih[TB];
        }
        wn[0] = W[0]; wn[1] = W[1 + P0]; wn[2] = W[1 + P1]; wn[3] = W[1 + P2]; wn[4] = W[4];
        const int pp[3] = {P0, P1, P2};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          dn[d][0] = g[pp[d]][0];
          dn[d][1] = g[pp[d]][1 + P0];
          dn[d][2] = g[pp[d]][1 + P1];
          dn[d][3] = g[pp[d]][1 + P2];
          dn[d][4] = g[pp[d]][4];
        }
      }
      __syncwarp();  // xs is rewritten by the next batch's evaluation only after the next tile wait
      // ---- half-range terms of this side, summed with the other side's by one exchange
      double x1[46], dtw[5];
      const bool ok = side_terms(side, wn, dn, c_fc, x1, dtw);
      const bool ok_other = __shfl_xor_sync(0xffffffffu, (int)ok, 1) != 0;
      double other_p = 0.0;
#pragma unroll
      for (int q = 0; q < 46; ++q) {
        const double y = __shfl_xor_sync(0xffffffffu, x1[q], 1);
        if (q < 45)
          x1[q] += y;
        else
          other_p = y;
      }
      // ---- hand over to the interface warp
      if (!first) nbar_sync(2, 96);  // the interface warp has read the previous batch
      first = false;
      double* h = hand + fl * 4 + gp;
      if (side == 0) {
#pragma unroll
        for (int q = 0; q < 45; ++q) h[q * 32] = x1[q];
        h[45 * 32] = x1[45];  // pL
        h[46 * 32] = other_p;  // pR
        h[67 * 32] = (ok && ok_other) ? 1.0 : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        h[(47 + side * 10 + q) * 32] = wn[q];
        h[(52 + side * 10 + q) * 32] = dtw[q];
      }
      nbar_arrive(1, 96);
      i0 = ni0;
      j0 = nj0;
      k0 = nk0;
      tma_cur = tma_next;
    }
    if (!first) nbar_sync(2, 96);  // consume the interface warp's last release
  } else {
    // ========================= interface warp =========================
    const int u = t - NS;
    const int fl = u >> 2, gp = u & 3;
    const int fx = fl % FX, fy = fl / FX;
    const double* h = hand + u;
    const int fn0 = c_geo.fn[AX][0], fn1 = c_geo.fn[AX][1];
    const long long fpl = (long long)fn0 * fn1;
    for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
      int i0, j0, k0;
      ws_batch<AX>(b, i0, j0, k0);
      const int i = i0 + fx, j = AX == 1 ? j0 + fy : j0, k = AX == 2 ? k0 + fy : k0;
      const bool valid = i < fn0 && (AX != 1 || j < c_geo.fn[1][1]) && (AX != 2 || k < c_geo.fn[2][2]);
      nbar_sync(1, 96);  // handoff full
      double x1[20];
#pragma unroll
      for (int q = 0; q < 20; ++q) x1[q] = h[q * 32];
      struct HandSV {
        const double* h;
        __device__ double operator()(int q) const { return h[(20 + q) * 32]; }
        // W_s at 47 + 10 s, dW_s/dt at 52 + 10 s
        __device__ double rel(int r, int q) const { return h[(47 + 10 * r + q) * 32]; }
      };
      struct NoPark {
        __device__ void mark(int) const {}
      };
      IfaceOut<double, 2> io;  // relaxation of both sides (R23)
      const bool good =
          interface_terms(x1, HandSV{h}, h[45 * 32], h[46 * 32], dt, idt, c_fc, NoPark{}, io) && h[67 * 32] != 0.0;
      double y[32];
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        y[q] = io.Fn[q];
        y[5 + q] = io.Ft[q];
        y[10 + q] = io.Qs[0][q];
        y[15 + q] = io.Qs[0][5 + q];
        y[20 + q] = io.Qs[1][q];
        y[25 + q] = io.Qs[1][5 + q];
      }
      y[30] = y[31] = 0.0;
      nbar_arrive(2, 96);  // handoff empty
      if (valid && !good) flag_error(err, 3, 1, stage, ts->steps, i, j, k);
      // back to the global frame (bit-exact component permutation)
      double z[32];
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        z[s * 5 + 0] = y[s * 5 + 0];
        z[s * 5 + 1 + P0] = y[s * 5 + 1];
        z[s * 5 + 1 + P1] = y[s * 5 + 2];
        z[s * 5 + 1 + P2] = y[s * 5 + 3];
        z[s * 5 + 4] = y[s * 5 + 4];
      }
      z[30] = z[31] = 0.0;
      // Gauss-point sum over the face's 4 lanes by a reduce-scatter ((g0 + g1) + (g2 + g3)), weight 1/4
      const bool up = gp & 1, up2 = gp & 2;
      double r1[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double send = up ? z[q] : z[16 + q];
        const double keep = up ? z[16 + q] : z[q];
        r1[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      double r2[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double send = up2 ? r1[q] : r1[8 + q];
        const double keep = up2 ? r1[8 + q] : r1[q];
        r2[q] = 0.25 * (keep + __shfl_xor_sync(0xffffffffu, send, 2));
      }
      if (valid) {
        const int o0 = (up ? 16 : 0) + (up2 ? 8 : 0);
        double* dst = face + (long long)k * NF * fpl + (long long)j * fn0 + i + (long long)o0 * fpl;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (o0 + q < NF) dst[q * fpl] = r2[q];
      }
    }
  }
}

}  // namespace cgks
