// flux1.cuh -- K2 with one lane per (face, Gauss point) (included by kernels.cuh).
//
// The lane evaluates the reconstructions of BOTH cells of its face at its Gauss point and runs the
// whole gas-kinetic solver of P:93-129 for it: the two half-range sides one after the other into the
// same accumulators (side_terms), then the interface phase once (interface_terms).  Against k_flux
// (two lanes per Gauss point, one per side, one lane exchange, the interface phase computed by both
// lanes) this executes no lane exchange and no duplicated interface work: ~3000 instead of
// 2 x 2450 instructions per Gauss point.  A block of 128 threads serves 128 / NG faces, so the staged
// tile is twice k_flux's per block; the face-plane parity evaluation results are parked in
// registers across one block barrier and then scattered through the dead tile (no separate scratch),
// which keeps the shared memory at ~50 KB per block (3 blocks = 12 warps per SM, as k_flux).
#pragma once

namespace cgks {

#ifndef CGKS_RPAD
#define CGKS_RPAD 2
#endif
#ifndef CGKS_TMA_SPLIT
#define CGKS_TMA_SPLIT 1
#endif
#ifndef CGKS_EVAL_SQ
#define CGKS_EVAL_SQ 1
#endif
#ifndef CGKS_SPECIAL_RS
#define CGKS_SPECIAL_RS 1  // full-record kernels: the specialised 30-value Gauss-point reduce-scatter (0: the generic
                           // one, measured 1.398 / 1.389 / 1.387 -> 1.429 / 1.406 / 1.408 ms per launch)
#endif
#ifndef CGKS_EVAL_REMAP
#define CGKS_EVAL_REMAP 1
#endif
#ifndef CGKS_FY1
#define CGKS_FY1 4  // faces of a y- / z-face patch along the normal axis (x extent = faces per block / FY1).
                    // 64-thread blocks: 4 x 4 patches (tile of 4 x 5 cells, 64-byte TMA rows; the two sides of a face
                    // sit 64 bytes apart modulo 128, so the evaluation's 16-byte loads are conflict-free, and the
                    // block's 31 KB leave the SM 60 KB of L1): y / z 1.380 / 1.385 ms, stage 2 1.363 / 1.360, against
                    // 8 x 2 patches (8 x 3 cells, 128-byte rows, 2-way conflicts between the sides): 1.431 / 1.424,
                    // 1.379 / 1.396.  (128-thread blocks, round 2 earlier: 16 x 2 1.611, 8 x 4 1.622, 4 x 8 1.66)
#endif

template <int DIM, int AX, bool COMPACT>
struct FluxTile1 {
  static constexpr int NG = COMPACT ? Sten<DIM>::NG : 1;
  static constexpr int NTHR = AX == 0 ? CGKS_FLUX_NTHR_X : CGKS_FLUX_NTHR_YZ;  // threads per block (one per Gauss point)
  static constexpr int MINB = (AX == 0 ? CGKS_FLUX_WARPS_X : CGKS_FLUX_WARPS_YZ) * 32 / NTHR;  // resident blocks per SM
  static constexpr int FPB = NTHR / NG;                      // faces per block
  static constexpr int FY = AX == 0 ? 1 : CGKS_FY1;          // faces along the normal axis
  static constexpr int FX = FPB / FY;                        // faces along x
  static constexpr int NT = AX == 0 ? FPB + 2 : FX * (FY + 1);
  static constexpr int TX = AX == 0 ? NT : FX;
  static constexpr int TN = AX == 0 ? 1 : FY + 1;
  static constexpr int NB = Sten<DIM>::NB;
  static constexpr int NREC = COMPACT ? NB * 5 : 15;
  static constexpr int NQ = DIM + 1;                         // value + DIM derivatives
  static constexpr int QPL = COMPACT ? (NQ + NG - 1) / NG : 0;  // quantities evaluated per lane and side
  static constexpr int XR = COMPACT ? 2 * NQ * 5 : 0;        // evaluation result rows [side][q][v]
  static constexpr int TS = ((NB / 2) % 2 == 1) ? NB : NB + 2;
  static constexpr int TAB = COMPACT ? 2 * NQ * TS : 0;
  static constexpr int FS = AX == 0 ? NT : FX;
  // the reconstruction fields arrive in NSPL parts of NRH fields (TMA boxes on their own mbarriers, so the
  // evaluation of the first basis functions overlaps the load of the rest): tile layout [part][plane][field
  // of the part][x]; field f of tile cell c at cbase(c, NRH) + faddr(f)
  static constexpr int NSPL = COMPACT ? CGKS_TMA_SPLIT : 1;
  static constexpr int NRH = NREC / NSPL;
  static_assert(NREC % NSPL == 0 && NRH % 5 == 0, "parts of whole basis functions");
  static constexpr int KH = NRH / 5;  // basis functions per part
  static constexpr int PSTR = (NRH * NT + 15) / 16 * 16;  // 128-byte aligned parts (bulk-tensor destinations)
  __host__ __device__ static constexpr int faddr(int f) { return (f / NRH) * PSTR + (f % NRH) * FS; }
  __host__ __device__ static constexpr int cbase(int c, int nfield) {
    return AX == 0 ? c : (c / FX) * nfield * FX + c % FX;
  }
  // CGKS-5th: the coefficient pairs of the global layout (cidx) arrive as they are: tile row r (one x-row of
  // FS cells) holds [pair p][cell x][2], so coefficient kk of component v of tile cell c is at
  // pbase(c) + coef(kk, v); GKS-2nd keeps one field per TMA row (faddr / cbase)
  static_assert(!COMPACT || NSPL == 1, "coefficient pairs: one TMA part");
  __host__ __device__ static constexpr int pbase(int c) { return AX == 0 ? 2 * c : (c / FX) * NREC * FX + 2 * (c % FX); }
  __host__ __device__ static constexpr int coef(int kk, int v) { return ((kk >> 1) * 5 + v) * 2 * FS + (kk & 1); }
  static constexpr int FSU = AX == 2 ? FX : NT;
  __host__ __device__ static constexpr int cbaseU(int c) { return AX == 2 ? (c / FX) * 5 * FX + c % FX : c; }
  static constexpr int STILE = NSPL * PSTR;
  // Per-lane rows (row r of lane l at r * NTHR + l): CGKS-5th uses the dead tile -- the evaluation
  // results [side][q][v] (XR rows), each side's dW/dt parked over its consumed d/dn rows, and 25 slots
  // for the half-range vectors x1[20..44]; GKS-2nd parks those 25 behind its (small) tile.
  static constexpr int FREE0 = COMPACT ? NQ * 5 - 10 : 0;  // rows 10 .. NQ*5-1: free once side 0 is read
  static constexpr int PROWS = COMPACT ? XR + 25 - FREE0 : 25;
  // row stride of the lanes' rows: NTHR + CGKS_RPAD (even) moves the rows of the 4 quantities (5 rows apart)
  // onto different banks, so the scatter of the evaluation results (a face's 4 lanes write 4 rows, STS.128)
  // is no longer 4-way conflicted; lanes read their own column (conflict-free at any stride).  Measured
  // per launch (x / y / z, ms): pad 0: 1.78 / 1.75 / 1.74; 2: 1.62 / 1.62 / 1.62; 4: 1.63 / 1.62 / 1.62;
  // 6, 10: 1.65 / 1.62 / 1.62; 18, 26: x 1.95 (shared memory then caps x-face blocks at 5 per SM)
  static constexpr int RS = COMPACT ? NTHR + CGKS_RPAD : NTHR;
  static constexpr int PARK0 = COMPACT ? 0 : (STILE + 5 * NT + NTHR - 1) / NTHR * NTHR;
  static constexpr int TILE = COMPACT ? (STILE + 5 * NT > PROWS * RS ? STILE + 5 * NT : PROWS * RS)
                                      : PARK0 + PROWS * NTHR;
  static_assert(CGKS_RPAD % 2 == 0, "the evaluation tables behind the rows are read as double2");
  static constexpr size_t smem_bytes() { return sizeof(double) * ((size_t)TILE + TAB) + 8 * NSPL; }
  // parking slot j (0..24, the half-range vectors x1[20..44]) -> row: free of both sides' W and dW/dt
  // rows and of side 1's unread rows
  __host__ __device__ static constexpr int park_row(int j) {
    return !COMPACT ? j : (j < FREE0 ? 10 + j : XR + (j - FREE0));
  }
};

template <int DIM, int AX, bool COMPACT>
struct ParkDev1 {
  double* col;
  __device__ __forceinline__ void put(int s, double v) const {
    col[FluxTile1<DIM, AX, COMPACT>::park_row(s) * FluxTile1<DIM, AX, COMPACT>::RS] = v;
  }
  __device__ __forceinline__ double get(int s) const {
    return col[FluxTile1<DIM, AX, COMPACT>::park_row(s) * FluxTile1<DIM, AX, COMPACT>::RS];
  }
};

// TONLY: the second stage of S2O4 uses only the time derivatives F_t^n, Q_t^n of the stage-1
// state; the kernel then forms and stores only those (half of the face record; k_update<MODE 1> reads
// nothing else)
template <int DIM, int AX, bool COMPACT, bool BOX, bool LINES = false, bool STR = false, bool TONLY = false>
__global__ void
#ifdef CGKS_FLUX_MAXNREG
__maxnreg__(CGKS_FLUX_MAXNREG)
#elif defined(CGKS_FLUX_MAXNREG_X)
__maxnreg__(AX == 0 ? CGKS_FLUX_MAXNREG_X : CGKS_FLUX_MAXNREG_YZ)
#else
__launch_bounds__(FluxTile1<DIM, AX, COMPACT>::NTHR, FluxTile1<DIM, AX, COMPACT>::MINB)
#endif
k_flux1(const double* __restrict__ U, const double* __restrict__ rec,
                                                const double* __restrict__ gtab, double* __restrict__ face,
                                                const TimeState* __restrict__ ts, ErrState* __restrict__ err,
                                                int stage, const __grid_constant__ CUtensorMap tm_rec,
                                                const __grid_constant__ CUtensorMap tm_U, int use_tma, int kb,
                                                int ke, int kofs) {
  // face planes [kb, ke) along z (a z-chunk of the stage, or all); face records of plane k at
  // face + k * NFR * fpl (the caller shifts chunk buffers); reconstruction plane of cell k at extended
  // plane k - elo[2] - kofs of rec (TMA coordinates; the pointer is shifted likewise)
  using FT = FluxTile1<DIM, AX, COMPACT>;
  constexpr int NG = FT::NG, NB = FT::NB, NT = FT::NT, NQ = FT::NQ;
  constexpr int NV = COMPACT ? 20 : 5;
  extern __shared__ __align__(128) double smem[];
  double* tile = smem;              // reconstruction fields, then Q (TMA box layout); later the lane rows
  double* tab = smem + FT::TILE;    // [side][quantity][TS] face evaluation tables
  uint64_t* bar = reinterpret_cast<uint64_t*>(tab + FT::TAB);
  constexpr int FX = FT::FX, FY = FT::FY;
  const int fn0 = c_geo.fn[AX][0];
  const int i0 = blockIdx.x * FX;
  const int j0 = AX == 1 ? blockIdx.y * FY : (AX == 2 ? blockIdx.z : blockIdx.y);
  const int k0 = kb + (AX == 2 ? blockIdx.y * FY : blockIdx.z);
  // ---- stage the tile (as k_flux): TMA boxes when no periodic wrap, else cp.async per element
  const int x0 = AX == 0 ? i0 - 2 : i0, y0 = AX == 1 ? j0 - 1 : j0, z0 = AX == 2 ? k0 - 1 : k0;
  const bool wraps = (AX == 0 && x0 < 0 && !c_geo.bounded[0]) || (AX == 1 && y0 < 0 && !c_geo.bounded[1]) ||
                     (AX == 2 && z0 < 0 && !c_geo.bounded[2]);
  const bool tma = !BOX && use_tma && !wraps;
  if (tma) {
    if (threadIdx.x == 0) {
      // the first part of the reconstruction fields, Q and the evaluation tables (one 1-D bulk copy) complete
      // on mbarrier 0, part p > 0 on mbarrier p
#pragma unroll
      for (int p = 0; p < FT::NSPL; ++p) mbar_init(bar + p, 1);
      mbar_expect_tx(bar, (unsigned)(sizeof(double) * ((FT::NRH + 5) * NT + FT::TAB)));
#pragma unroll
      for (int p = 1; p < FT::NSPL; ++p) mbar_expect_tx(bar + p, (unsigned)(sizeof(double) * FT::NRH * NT));
#pragma unroll
      for (int p = 0; p < FT::NSPL; ++p)
        tma_load_4d(tile + p * FT::PSTR, &tm_rec, bar + p, COMPACT ? 2 * (x0 - c_geo.elo[0]) : x0 - c_geo.elo[0],
                    COMPACT ? 0 : p * FT::NRH, y0 - c_geo.elo[1], z0 - c_geo.elo[2] - kofs);
      tma_load_4d(tile + FT::STILE, &tm_U, bar, x0, y0 + c_geo.yoff, 0, z0 + c_geo.zoff);
      if (COMPACT) bulk_load(tab, gtab, (unsigned)(sizeof(double) * FT::TAB), bar);
    }
  } else {
    // cp.async: TPC threads per tile cell (index math once per cell), a strided subset of its fields each
    constexpr int TPC = FT::NTHR / NT > 0 ? FT::NTHR / NT : 1;
    for (int w = threadIdx.x; w < NT * TPC; w += blockDim.x) {
      const int c = w % NT, fsub = w / NT;
      int ci, cj = j0, ck = k0;
      if (AX == 0) {
        ci = i0 - 2 + c;
        if (c_geo.bounded[0] && ci < -1) ci = -1;  // column 0 feeds no face
      } else {
        ci = i0 + c % FX;
        if (AX == 1) cj += c / FX - 1;
        if (AX == 2) ck += c / FX - 1;
      }
      // clamp the ragged tails (those cells only feed faces that are not stored)
      const int imax = c_geo.n[0] - 1 + (c_geo.bounded[0] ? 1 : 0);
      if (ci > imax) ci = imax;
      if (AX == 1) {
        const int jmax = c_geo.n[1] - 1 + (c_geo.bounded[1] ? 1 : 0);
        if (cj > jmax) cj = jmax;
      }
      if (AX == 2) {
        const int kmax = min(c_geo.n[2] - 1 + (c_geo.bounded[2] ? 1 : 0), ke - 1);  // (chunk: its last cell)
        if (ck > kmax) ck = kmax;
      }
      const long long st = c_geo.en[0];  // field stride of the reconstruction array
      if (COMPACT) {  // 16-byte coefficient pairs (cidx layout)
        const double* src = rec + cidx(FT::NREC, 0, 0, ci, cj, ck) + fsub * 2 * st;
        const unsigned dst0 = (unsigned)__cvta_generic_to_shared(tile + FT::pbase(c));
#pragma unroll 4
        for (int pr = fsub; pr < FT::NREC / 2; pr += TPC) {
          cp_async16s(dst0 + pr * 2 * FT::FS * (unsigned)sizeof(double), src);
          src += TPC * 2 * st;
        }
      } else {
        const double* src = rec + eidx(FT::NREC, 0, ci, cj, ck) + fsub * st;
        const unsigned dst0 = (unsigned)__cvta_generic_to_shared(tile + FT::cbase(c, FT::NRH));
#pragma unroll 4
        for (int fld = fsub; fld < FT::NREC; fld += TPC) {
          cp_async8s(dst0 + FT::faddr(fld) * (unsigned)sizeof(double), src);
          src += TPC * st;
        }
      }
      double* sdst = tile + FT::STILE + FT::cbaseU(c);
      if (BOX) {
        for (int v = fsub; v < 5; v += TPC) sdst[v * FT::FSU] = ld_state<BOX>(U, NV, v, ci, cj, ck);
      } else {
        const double* ub = U + sidx(NV, 0, wrap_ax(0, ci), wrap_ax(1, cj), wrap_ax(2, ck));
        for (int v = fsub; v < 5; v += TPC) cp_async8(sdst + v * FT::FSU, ub + v * c_geo.splane);
      }
    }
  }
  if (COMPACT && !tma)
    for (int q = threadIdx.x; q < FT::TAB; q += blockDim.x) cp_async8(tab + q, gtab + q);
  const bool stop = __syncthreads_or(err->code != 0);
  CGKS_JIT(5);
  cp_async_wait_all();
  if (tma) mbar_wait(bar, 0);
  if (stop) {
    if (tma)
#pragma unroll
      for (int p = 1; p < FT::NSPL; ++p) mbar_wait(bar + p, 0);  // no bulk copy may land after the exit
    return;
  }
  __syncthreads();

  const double dt = ts->dt;
  const int lane = threadIdx.x;
  const int gp = lane % NG;
  const int fl = lane / NG;  // face within the block
  const int fx = fl % FX, fy = fl / FX;
  const int i = i0 + fx, j = AX == 1 ? j0 + fy : j0, k = AX == 2 ? k0 + fy : k0;
  const bool valid = i < fn0 && (AX != 1 || j < c_geo.fn[1][1]) && k < ke;
  // tile columns of the two cells (left = side 0, right = side 1)
  const int cL = AX == 0 ? fl + 1 : fy * FX + fx;
  const int cR = AX == 0 ? fl + 2 : (fy + 1) * FX + fx;
  CGKS_BOUND(cR, NT, "flux tile cell");
  static_assert(!COMPACT || FT::PROWS * FT::RS <= FT::TILE, "lane rows inside the tile region");
  static_assert(FT::STILE + 5 * NT <= FT::TILE, "tile inside its region");
  constexpr int P0 = AX, P1 = (AX + 1) % 3, P2 = (AX + 2) % 3;
  double ihL[3], ihR[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) ihL[a] = ihR[a] = a < DIM ? c_geo.ih[a] : 0.0;
  if (STR) {
    const int cc[3] = {i, j, k};
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      if (a == AX) {
        ihL[a] = icw(a, min(cc[a] - 1, c_geo.n[a] + 1));
        ihR[a] = icw(a, min(cc[a], c_geo.n[a] + 1));
      } else {
        ihL[a] = ihR[a] = icw(a, min(cc[a], c_geo.n[a] + 1));
      }
    }
  }
  constexpr int RS = FT::RS;                // row stride of the lanes' rows
  double* col = tile + lane;                // this lane's rows in the dead tile: row r at col[r * RS]
  const ParkDev1<DIM, AX, COMPACT> park{tile + FT::PARK0 + lane};
  // global-frame W (5) and physical derivatives (3 x 5) of side s -> normal frame
  auto to_normal = [&](const double* W, const double (*g)[5], double* wn, double (*dn)[5]) {
    wn[0] = W[0];
    wn[1] = W[1 + P0];
    wn[2] = W[1 + P1];
    wn[3] = W[1 + P2];
    wn[4] = W[4];
    const int pp[3] = {P0, P1, P2};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      dn[d][0] = g[pp[d]][0];
      dn[d][1] = g[pp[d]][1 + P0];
      dn[d][2] = g[pp[d]][1 + P1];
      dn[d][3] = g[pp[d]][1 + P2];
      dn[d][4] = g[pp[d]][4];
    }
  };
  constexpr int TA = DIM == 3 ? P1 : (DIM == 2 ? 1 - AX : 0);  // active transverse axes
  constexpr int TB = DIM == 3 ? P2 : 0;
#if CGKS_EVAL_SQ
  constexpr bool SQ = COMPACT && DIM == 3 && NG == 4;
#else
  constexpr bool SQ = false;
#endif
  if constexpr (SQ) {
    // Face-plane parity evaluation, one side per lane: lane gp of a face evaluates side s = gp & 1 for the
    // quantities qa = gp >> 1 (value or d/dn) and qa + 2 (d/dtA or d/dtB) at all 4 Gauss points, so every
    // coefficient it loads feeds two FMAs (170 shared-memory loads per lane instead of 340 for both sides);
    // the results wait in registers for the block barrier (tile dead), then go to their lanes' columns.
    // x-faces: the lane works for its own face (sides cL, cL + 1 are adjacent 16-byte pairs).  y- / z-faces: the
    // two sides are tile rows a multiple of 128 bytes apart, so lanes of one quarter-warp reading both sides of a
    // face hit the same banks (ncu: 49 M LDS bank conflicts per launch against 3 M for x-faces); there lane Lw of
    // a warp (one row of 8 faces) takes face Lw & 7, side (Lw >> 3) & 1, quantity pair Lw >> 4: every quarter-warp
    // reads 8 consecutive pairs of one tile row (conflict-free) and shares its table entries.  Results bitwise
    // equal.  Measured per launch with 8 x 2 patches (y / z, ms): stage-2 kernels 1.403 / 1.412 -> 1.378 / 1.396,
    // full-record kernels 1.431 / 1.424 -> 1.450 / 1.446 (ptxas then spills 48 instead of 32 bytes), so only the
    // former used it; the default 4 x 4 patches are conflict-free as they are (FX = 4: not remapped)
    constexpr bool REMAP = AX != 0 && FX == 8 && (CGKS_EVAL_REMAP == 2 || (CGKS_EVAL_REMAP == 1 && TONLY));
    const int lw = lane & 31;
    const int sd = REMAP ? (lw >> 3) & 1 : gp & 1, qa = REMAP ? lw >> 4 : gp >> 1;
    const int ef = REMAP ? (lane >> 5) * 8 + (lw & 7) : fl;  // the face (of the block) this lane evaluates
    const int ecol = ef * NG;                                // its lanes' columns
    const int cs = REMAP ? ((ef / FX) + sd) * FX + ef % FX : (sd ? cR : cL);
    const double* tc = tile + FT::pbase(cs);
    const double* sc = tile + FT::STILE + FT::cbaseU(cs);
    const double* Ta = tab + (sd * NQ + qa) * FT::TS;
    const double* Tb = Ta + 2 * FT::TS;
    double Sa[5][4], Sb[5][4];
#pragma unroll
    for (int v = 0; v < 5; ++v)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        Sa[v][cc] = (cc == 0 && qa == 0) ? sc[v * FT::FSU] : 0.0;  // the value's sums start from the average
        Sb[v][cc] = 0.0;
      }
#pragma unroll
    for (int k2 = 0; k2 < NB; k2 += 2) {
      const double2 ta = *reinterpret_cast<const double2*>(Ta + k2);
      const double2 tb = *reinterpret_cast<const double2*>(Tb + k2);
      const int cls0 = (ReconGen<DIM>::expo(k2, TA) & 1) | ((ReconGen<DIM>::expo(k2, TB) & 1) << 1);
      const int cls1 = (ReconGen<DIM>::expo(k2 + 1, TA) & 1) | ((ReconGen<DIM>::expo(k2 + 1, TB) & 1) << 1);
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double2 c = *reinterpret_cast<const double2*>(tc + FT::coef(k2, v));  // coefficients k2, k2 + 1
        Sa[v][cls0] = fma(c.x, ta.x, Sa[v][cls0]);
        Sb[v][cls0] = fma(c.x, tb.x, Sb[v][cls0]);
        Sa[v][cls1] = fma(c.y, ta.y, Sa[v][cls1]);
        Sb[v][cls1] = fma(c.y, tb.y, Sb[v][cls1]);
      }
    }
    // Gauss point g (bit 0: + along tA, bit 1: + along tB) = sum over the parity classes with signs; a
    // tangential derivative (quantity qa + 2: flip 1 for d/dtA, 2 for d/dtB) lowers one parity (sign of
    // the points on the - side of that axis)
    const int flipb = qa == 0 ? 1 : 2;
    double R[2][5][4];
#pragma unroll
    for (int v = 0; v < 5; ++v)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const double* S = w ? Sb[v] : Sa[v];
        const double ap = S[0] + S[1], am = S[0] - S[1];
        const double bp = S[2] + S[3], bm = S[2] - S[3];
        const double r[4] = {am - bm, ap - bp, am + bm, ap + bp};
#pragma unroll
        for (int g2 = 0; g2 < 4; ++g2) {
          const unsigned neg = w ? ((((flipb & 1) && !(g2 & 1)) ? 1u : 0u) ^ (((flipb & 2) && !(g2 & 2)) ? 1u : 0u)) : 0u;
          R[w][v][g2] = __longlong_as_double(__double_as_longlong(r[g2]) ^ ((long long)neg << 63));
        }
      }
    CGKS_JIT(3);
    __syncthreads();  // the tile is dead: its space holds the lanes' rows from here on
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int v = 0; v < 5; ++v)
#pragma unroll
        for (int g2 = 0; g2 < 4; ++g2) {
          CGKS_BOUND(((sd * NQ + qa + 2 * w) * 5 + v) * RS + (ecol + g2), FT::TILE, "flux eval scatter");
          tile[((sd * NQ + qa + 2 * w) * 5 + v) * RS + (ecol + g2)] = R[w][v][g2];
        }
    CGKS_JIT(4);
    __syncwarp();
  } else if (COMPACT) {
    // Face-plane parity evaluation (as k_flux): lane gp computes quantity q = gp (+ NG ...) of both
    // sides at all NG Gauss points; the results wait in registers for the block barrier (tile dead),
    // then go to their destination lanes' columns.
    double R[2][FT::QPL > 0 ? FT::QPL : 1][5][NG];
    // x-faces: one code copy for both sides (rolled loop; the results move into the side's register set by
    // selects); y- / z-faces: both sides unrolled -- the faster variant per axis, measured (flux_x 1.83 vs
    // 1.86 ms, flux_y / z 1.75 vs 1.81 ms)
    constexpr bool ROLLED = AX == 0;
    auto eval_side = [&](const int s) {
      const int cs = s ? cR : cL;
      const double* tc = tile + FT::pbase(cs);
      const double* sc = tile + FT::STILE + FT::cbaseU(cs);
      const double* Tb = tab + s * NQ * FT::TS;
#pragma unroll
      for (int qi = 0; qi < FT::QPL; ++qi) {
        const int q = gp + qi * NG;
        if (q >= NQ) break;
        const double* T = Tb + q * FT::TS;
        // S[v][0] enters every Gauss point with sign +1 (and flip = 0 for the value): the value's sums start
        // from the cell average
        double S[5][NG];
#pragma unroll
        for (int v = 0; v < 5; ++v)
#pragma unroll
          for (int cc = 0; cc < NG; ++cc) S[v][cc] = (cc == 0 && q == 0) ? sc[v * FT::FSU] : 0.0;
#pragma unroll
        for (int k2 = 0; k2 < NB; k2 += 2) {
          const double2 tt = *reinterpret_cast<const double2*>(T + k2);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kk = k2 + h;
            if (kk >= NB) break;
            const int cls = DIM == 3 ? ((ReconGen<DIM>::expo(kk, TA) & 1) | ((ReconGen<DIM>::expo(kk, TB) & 1) << 1))
                                     : (DIM == 2 ? (ReconGen<DIM>::expo(kk, TA) & 1) : 0);
            const double t = h ? tt.y : tt.x;
#pragma unroll
            for (int v = 0; v < 5; ++v) S[v][cls] = fma(tc[FT::coef(kk, v)], t, S[v][cls]);
          }
        }
        const int flip = q == 2 ? 1 : (q == 3 ? 2 : 0);
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          double r[NG];
          if constexpr (NG == 1) {
            r[0] = S[v][0];
          } else {
            const double ap = S[v][0] + S[v][1], am = S[v][0] - S[v][1];
            if constexpr (NG == 2) {
              r[0] = am;
              r[1] = ap;
            } else {
              const double bp = S[v][2] + S[v][3], bm = S[v][2] - S[v][3];
              r[0] = am - bm;
              r[1] = ap - bp;
              r[2] = am + bm;
              r[3] = ap + bp;
            }
          }
#pragma unroll
          for (int g2 = 0; g2 < NG; ++g2) {
            const unsigned neg = (((flip & 1) && !(g2 & 1)) ? 1u : 0u) ^ (((flip & 2) && !(g2 & 2)) ? 1u : 0u);
            const long long bits = __double_as_longlong(r[g2]) ^ ((long long)neg << 63);
            // (rolled: 0.0 + x measured 15 % faster per flux launch than the plain value -- ptxas then places
            // the results in their registers without moves)
            const double val = ROLLED ? 0.0 + __longlong_as_double(bits) : __longlong_as_double(bits);
            R[0][qi][v][g2] = s ? R[0][qi][v][g2] : val;
            R[1][qi][v][g2] = s ? val : R[1][qi][v][g2];
          }
        }
      }
    };
    if constexpr (ROLLED) {
#pragma unroll 1
      for (int s = 0; s < 2; ++s) eval_side(s);
    } else {
      eval_side(0);
      eval_side(1);
    }
    CGKS_JIT(3);
    __syncthreads();  // the tile is dead: its space holds the lanes' rows from here on
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int qi = 0; qi < FT::QPL; ++qi) {
        const int q = gp + qi * NG;
        if (q >= NQ) break;
#pragma unroll
        for (int v = 0; v < 5; ++v)
#pragma unroll
          for (int g2 = 0; g2 < NG; ++g2) {
            CGKS_BOUND(((s * NQ + q) * 5 + v) * RS + (lane - gp + g2), FT::TILE, "flux eval scatter");
            tile[((s * NQ + q) * 5 + v) * RS + (lane - gp + g2)] = R[s][qi][v][g2];
          }
      }
    CGKS_JIT(4);
    __syncwarp();
  }
  // side s of this lane's Gauss point in the normal frame
  auto load_side = [&](int s, double* wn, double (*dn)[5]) {
    double W[5], g[3][5];
    const double* ih = s ? ihR : ihL;
    if (COMPACT) {
      const double* rb = col + s * NQ * 5 * RS;
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        W[v] = rb[v * RS];
        g[0][v] = g[1][v] = g[2][v] = 0.0;
        // physical derivatives: 1/h is in the evaluation table on a uniform mesh, per cell on a stretched one
        g[AX][v] = STR ? rb[(5 + v) * RS] * ih[AX] : rb[(5 + v) * RS];
        if (DIM > 1) g[TA][v] = STR ? rb[((2 % NQ) * 5 + v) * RS] * ih[TA] : rb[((2 % NQ) * 5 + v) * RS];
        if (DIM > 2) g[TB][v] = STR ? rb[((3 % NQ) * 5 + v) * RS] * ih[TB] : rb[((3 % NQ) * 5 + v) * RS];
      }
    } else {
      const int cs = s ? cR : cL;
      const double* tc = tile + FT::cbase(cs, FT::NRH);
      const double* sc = tile + FT::STILE + FT::cbaseU(cs);
      const double hs = s ? -0.5 : 0.5;
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        W[v] = sc[v * FT::FSU] + hs * tc[(AX * 5 + v) * FT::FS];
#pragma unroll
        for (int a = 0; a < 3; ++a) g[a][v] = tc[(a * 5 + v) * FT::FS] * (a < DIM ? ih[a] : 0.0);
      }
    }
    to_normal(W, g, wn, dn);
  };
  // the two sides' half-range terms: side 0 into x1, its vectors x1[20..44] parked (so that they are
  // not live across side 1), side 1 into fresh accumulators for them, then the sums parked
  double x1[45];
#pragma unroll
  for (int q = 0; q < 45; ++q) x1[q] = 0.0;
  double pLR[2];
  int okLR = 1;
#pragma unroll 1
  for (int s = 0; s < 2; ++s) {  // rolled: one code copy of the side phase (instruction cache)
    double wn[5], dn[3][5], dtw[5], ps;
    load_side(s, wn, dn);
    const bool oks = side_terms(s ? -1.0 : 1.0, wn, dn, c_fc, x1, ps, dtw);
    pLR[0] = s ? pLR[0] : ps;
    pLR[1] = s ? ps : pLR[1];
    okLR &= oks ? 1 : 0;
    if (COMPACT)
#pragma unroll
      for (int v = 0; v < 5; ++v) col[(s * NQ * 5 + 5 + v) * RS] = dtw[v];  // over the side's consumed d/dn rows
    asm volatile("" ::: "memory");  // the parked side-0 vectors stay out of registers during side 1
#pragma unroll
    for (int q = 0; q < 25; ++q) {
      park.put(q, (s ? park.get(q) : 0.0) + x1[20 + q]);
      x1[20 + q] = 0.0;
    }
  }
  const double pL = pLR[0], pR = pLR[1];
  double acc[20], jump;
  const bool good =
      interface_terms<double, ParkDev1<DIM, AX, COMPACT>, TONLY>(x1, pL, pR, dt, ts->idt, c_fc, park, acc, jump) &&
      okLR;
  if (valid && !good) flag_error(err, 3, 1, stage, ts->steps, i, j, k);
  // outputs of this Gauss point in the global frame: y = Fn Ft QLn QLt QRn QRt (face record order)
  constexpr int NR = COMPACT ? 30 : 10;
  double y[NR];
  auto gidx = [](int cc) { return cc == 0 ? 0 : (cc == 4 ? 4 : 1 + (cc == 1 ? P0 : (cc == 2 ? P1 : P2))); };
#pragma unroll
  for (int cc = 0; cc < 5; ++cc) {
    y[gidx(cc)] = acc[cc];
    y[5 + gidx(cc)] = acc[5 + cc];
  }
  if (COMPACT) {
    // side-state relaxation of both sides (R23): Q^s = w Q^n + (1 - w) W_s, Q^s_t likewise
    const double ee = relax_ee(jump, c_fc);
    if (__all_sync(0xffffffffu, ee == 0.0)) {  // smooth flow in the whole warp
#pragma unroll
      for (int cc = 0; cc < 5; ++cc) {
        y[10 + gidx(cc)] = y[20 + gidx(cc)] = acc[10 + cc];
        y[15 + gidx(cc)] = y[25 + gidx(cc)] = acc[15 + cc];
      }
    } else {
      const double w = 1.0 - ee;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        // W_s (global frame, rows s*NQ*5 + 0..4) and dW_s/dt (normal frame, rows s*NQ*5 + 5..9)
        const double* rb = col + s * NQ * 5 * RS;
        double Wg[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) Wg[v] = rb[v * RS];
        const double Wn[5] = {Wg[0], Wg[1 + P0], Wg[1 + P1], Wg[1 + P2], Wg[4]};
#pragma unroll
        for (int cc = 0; cc < 5; ++cc) {
          if (!TONLY) y[10 + 10 * s + gidx(cc)] = w * acc[10 + cc] + ee * Wn[cc];
          y[15 + 10 * s + gidx(cc)] = w * acc[15 + cc] + ee * rb[(5 + cc) * RS];
        }
      }
    }
  }
  const int fn1 = c_geo.fn[AX][1];
  const long long fpl = (long long)fn0 * fn1;
  constexpr int NGL_ = DIM == 3 ? 4 : (DIM == 2 ? 2 : 1);
  constexpr int NFR = COMPACT ? (LINES ? 30 + 2 * NGL_ * 10 : 30) : 10;
  const long long base = (long long)k * NFR * fpl + (long long)j * fn0 + i;
  if (valid) {  // face records of planes [kb, ke) (the caller shifts a chunk's buffer)
    CGKS_BOUND(i, fn0, "flux face i");
    CGKS_BOUND(j, fn1, "flux face j");
    CGKS_BOUND(k - kb, ke - kb, "flux face k");
  }
  if (COMPACT && LINES && valid) {
    // line DOFs: both sides' relaxed values at this Gauss point, line order g = p * n2 + q
    const int gcan = NG == 4 ? 2 * (gp & 1) + ((gp >> 1) & 1) : gp;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      double* dst = face + base + (long long)(30 + (s * NG + gcan) * 10) * fpl;
#pragma unroll
      for (int q = TONLY ? 5 : 0; q < 10; ++q) dst[q * fpl] = y[10 + 10 * s + q];
    }
  }
  if constexpr (!TONLY && CGKS_SPECIAL_RS) {
    if constexpr (NG == 1) {
      if (valid)
#pragma unroll
        for (int q = 0; q < NR; ++q) face[base + q * fpl] = y[q];
    } else {
      // Gauss-point sum by a reduce-scatter over the face's NG lanes: round 1 (partner gp ^ 1) halves
      // the 30 values, round 2 (gp ^ 2, NG = 4) splits the 15 into 8 + 7; every sum is
      // (g0 + g1) + (g2 + g3) whichever lane forms it (deterministic); weight 1/NG after the sum
      // (a sum through the lanes' shared-memory rows instead: 3 % slower per step, measured)
      constexpr int H = NR / 2;  // 15
      const bool up = gp & 1;
      double z[16];
#pragma unroll
      for (int q = 0; q < H; ++q) {
        const double send = up ? y[q] : y[H + q];
        const double keep = up ? y[H + q] : y[q];
        z[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      z[15] = 0.0;
      const double wgt = 1.0 / NG;
      if constexpr (NG == 2) {
        if (valid) {
          double* dst = face + base + (long long)(up ? H : 0) * fpl;
#pragma unroll
          for (int q = 0; q < H; ++q) dst[q * fpl] = wgt * z[q];
        }
      } else {
        const bool up2 = gp & 2;
        double zz[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double send = up2 ? z[q] : z[8 + q];
          const double keep = up2 ? z[8 + q] : z[q];
          zz[q] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        if (valid) {
          const int o0 = (up ? H : 0) + (up2 ? 8 : 0);
          const int cnt = up2 ? H - 8 : 8;
          double* dst = face + base + (long long)o0 * fpl;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < cnt) dst[q * fpl] = wgt * zz[q];
        }
      }
    }
  } else {
  // the record fields this launch writes: all NR, or (TONLY) F_t, Q^L_t, Q^R_t (CGKS-5th) / F_t (GKS-2nd)
    constexpr int NO = TONLY ? (COMPACT ? 15 : 5) : NR;
    auto fld = [](int o) { return !TONLY ? o : (o < 5 ? 5 + o : (o < 10 ? 15 + (o - 5) : 25 + (o - 10))); };
    double yo[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) yo[o] = y[fld(o)];
    if constexpr (NG == 1) {
      if (valid)
#pragma unroll
        for (int o = 0; o < NO; ++o) face[base + fld(o) * fpl] = yo[o];
    } else {
      // Gauss-point sum by a reduce-scatter over the face's NG lanes: round 1 (partner gp ^ 1) splits the NO
      // outputs into H1 + (NO - H1), round 2 (gp ^ 2, NG = 4) each half into H2 + rest; every sum is
      // (g0 + g1) + (g2 + g3) whichever lane forms it (deterministic); weight 1/NG after the sum
      // (a sum through the lanes' shared-memory rows instead: slower, measured twice)
      constexpr int H1 = (NO + 1) / 2, H2 = (H1 + 1) / 2;
      const bool up = gp & 1;
      double z[H1];
#pragma unroll
      for (int q = 0; q < H1; ++q) {
        const double hi = H1 + q < NO ? yo[H1 + q < NO ? H1 + q : 0] : 0.0;
        const double send = up ? yo[q] : hi;
        const double keep = up ? hi : yo[q];
        z[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      const double wgt = 1.0 / NG;
      const int lim = up ? NO : H1;  // end of this lane's half
      if constexpr (NG == 2) {
        if (valid) {
          const int o0 = up ? H1 : 0;
#pragma unroll
          for (int q = 0; q < H1; ++q)
            if (o0 + q < lim) face[base + fld(o0 + q) * fpl] = wgt * z[q];
        }
      } else {
        const bool up2 = gp & 2;
        double zz[H2];
#pragma unroll
        for (int q = 0; q < H2; ++q) {
          const double hi = H2 + q < H1 ? z[H2 + q < H1 ? H2 + q : 0] : 0.0;
          const double send = up2 ? z[q] : hi;
          const double keep = up2 ? hi : z[q];
          zz[q] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        if (valid) {
          const int o0 = (up ? H1 : 0) + (up2 ? H2 : 0);
          const int lim2 = up2 ? lim : (up ? H1 : 0) + H2;
#pragma unroll
          for (int q = 0; q < H2; ++q)
            if (o0 + q < lim2) face[base + fld(o0 + q) * fpl] = wgt * zz[q];
        }
      }
    }
  }
}

}  // namespace cgks
