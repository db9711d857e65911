// stage_impl.cuh -- launch sequence of one stage for dimension CGKS_DIM (included once per
// translation unit stage_d<D>.cu).
#pragma once
#ifndef CGKS_DIM
#error "define CGKS_DIM before including stage_impl.cuh"
#endif
#include <cstdio>

#include "driver.h"
#include "kernels.cuh"

namespace cgks {
namespace {

template <typename... KArgs, typename... Args>
int launch(LaunchEnv& env, const char* name, void (*kern)(KArgs...), long long nthreads, int block, Args... args) {
  if (nthreads <= 0) return 0;
  const long long nblk = (nthreads + block - 1) / block;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (env.prof) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, env.stream);
  }
  kern<<<(unsigned)nblk, block, 0, env.stream>>>(args...);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (env.msg) std::snprintf(env.msg, env.msglen, "launch of %s failed: %s", name, cudaGetErrorString(e));
    return 5;
  }
  if (env.prof) {
    cudaEventRecord(e1, env.stream);
    env.pending->push_back({name, {e0, e1}});
  }
  return 0;
}

#define LAUNCH(name, kern, n, blk, ...)                                 \
  do {                                                                  \
    int rc_ = launch(env, name, kern, (long long)(n), blk, __VA_ARGS__); \
    if (rc_) return rc_;                                                \
  } while (0)

constexpr int D = CGKS_DIM;

// reconstruction: one block per TX x TY x TZ cells of the extended range, shared-memory halo tile
template <bool NONLIN, bool BOX, bool LINES = false, bool STR = false>
int recon5_launch(LaunchEnv& env, const StageArgs& a) {
  using RT = ReconTile<D>;
  auto kern = k_recon5<D, NONLIN, BOX, LINES, STR>;
  static bool attr = false;
  const size_t smem = RT::smem_bytes();
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 5;
    attr = true;
  }
  // extended z planes [z0, z1): all, a part (halo overlap), or a z-chunk's cells and their two
  // neighbour planes (chunked stage: rec holds extended planes ck0 .. ck0 + cn + 1 from its start)
  int z0 = a.rz1 < 0 ? 0 : a.rz0, z1 = a.rz1 < 0 ? a.en[2] : a.rz1;
  double* rec = a.rec;
  if (a.cn >= 0) {
    z0 = a.ck0;
    z1 = a.ck0 + a.cn + 2;
    rec = a.rec - (long long)a.ck0 * a.en[0] * a.en[1] * (5 * Sten<D>::NB);
  }
  if (z1 <= z0) return 0;
  const dim3 grid((unsigned)((a.en[0] + RT::TX - 1) / RT::TX), (unsigned)((a.en[1] + RT::TY - 1) / RT::TY),
                  (unsigned)((z1 - z0 + RT::TZ - 1) / RT::TZ));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (env.prof) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, env.stream);
  }
  kern<<<grid, RT::NTH, smem, env.stream>>>(a.Uin, rec, a.err, a.Lin, z0, z1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (env.msg) std::snprintf(env.msg, env.msglen, "launch of recon5 failed: %s", cudaGetErrorString(e));
    return 5;
  }
  if (env.prof) {
    cudaEventRecord(e1, env.stream);
    env.pending->push_back({"recon5", {e0, e1}});
  }
  return 0;
}

// flux kernel: one block per FPB faces of an x-row, dynamic shared memory tile
template <int AX, bool COMPACT>
using FluxTileSel = FluxTile1<D, AX, COMPACT>;

template <bool COMPACT, bool BOX, int AX, bool LINES = false, bool STR = false, bool TONLY = false>
int flux_launch(LaunchEnv& env, const char* name, const StageArgs& a, int stage) {
  using FT = FluxTileSel<AX, COMPACT>;
  auto kern = k_flux1<D, AX, COMPACT, BOX, LINES, STR, TONLY>;
  static bool attr = false;
  const size_t smem = FT::smem_bytes();
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 5;
    attr = true;
  }
  // face planes [kb, ke) along z: all of them, or those of the z-chunk a.ck0 .. a.ck0 + a.cn (chunked
  // stage; z-faces: cn + 1 planes); the chunk's face records and reconstruction planes start at kb
  const int kb = a.cn < 0 ? 0 : a.ck0;
  const int ke = a.cn < 0 ? a.fn[AX][2] : a.ck0 + a.cn + (AX == 2 ? 1 : 0);
  if (ke <= kb) return 0;
  constexpr int NGL_ = D == 3 ? 4 : (D == 2 ? 2 : 1);
  constexpr int NFR = COMPACT ? (LINES ? 30 + 2 * NGL_ * 10 : 30) : 10;
  double* face = a.face[AX] - (long long)kb * NFR * a.fn[AX][0] * a.fn[AX][1];
  const double* rec = a.rec - (long long)kb * a.en[0] * a.en[1] * (COMPACT ? 5 * Sten<D>::NB : 15);
  const unsigned gy = (unsigned)(AX == 1 ? (a.fn[AX][1] + FT::FY - 1) / FT::FY : a.fn[AX][1]);
  const unsigned gz = (unsigned)(AX == 2 ? (ke - kb + FT::FY - 1) / FT::FY : ke - kb);
  const unsigned gx = (unsigned)((a.fn[AX][0] + FT::FX - 1) / FT::FX);
  const dim3 grid = AX == 2 ? dim3(gx, gz, gy) : dim3(gx, gy, gz);  // z-faces: (x, z, y) order
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (env.prof) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, env.stream);
  }
  static const CUtensorMap none{};
  kern<<<grid, FT::NTHR, smem, env.stream>>>(a.Uin, rec, a.gtab[AX], face, a.ts, a.err, stage,
                                        a.use_tma ? a.tm_rec[AX] : none, a.use_tma ? a.tm_U[AX] : none,
                                        a.use_tma && !BOX ? 1 : 0, kb, ke, a.cn < 0 ? 0 : kb);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (env.msg) std::snprintf(env.msg, env.msglen, "launch of %s failed: %s", name, cudaGetErrorString(e));
    return 5;
  }
  if (env.prof) {
    cudaEventRecord(e1, env.stream);
    env.pending->push_back({name, {e0, e1}});
  }
  return 0;
}

template <bool COMPACT, bool NONLIN, bool BOX, bool LINES = false, bool STR = false>
int stage_t(LaunchEnv& env, const StageArgs& a, int mode, int stage) {
  if (a.part != 3) {
    if (COMPACT) {
      int rc = recon5_launch<NONLIN, BOX, LINES, STR>(env, a);
      if (rc) return rc;
    } else {
      int z0 = a.rz1 < 0 ? 0 : a.rz0, z1 = a.rz1 < 0 ? a.en[2] : a.rz1;
      double* rec = a.rec;
      if (a.cn >= 0) {  // z-chunk (see recon5_launch)
        z0 = a.ck0;
        z1 = a.ck0 + a.cn + 2;
        rec = a.rec - (long long)a.ck0 * a.en[0] * a.en[1] * 15;
      }
      if (z1 > z0)
        LAUNCH("recon2", (k_recon2<D, NONLIN, BOX>), (long long)a.en[0] * a.en[1] * (z1 - z0), 256, a.Uin, rec,
               a.err, z0, z1);
    }
    if (a.part == 1) return 0;
  }
  if (COMPACT && mode == 1) {
    // second stage of S2O4: the update uses only the time derivatives (flux kernels "flux_*_t")
    int rc = flux_launch<COMPACT, BOX, 0, LINES, STR, true>(env, "flux_x_t", a, stage);
    if (!rc && D > 1) rc = flux_launch<COMPACT, BOX, (D > 1 ? 1 : 0), LINES, STR, true>(env, "flux_y_t", a, stage);
    if (!rc && D > 2) rc = flux_launch<COMPACT, BOX, (D > 2 ? 2 : 0), LINES, STR, true>(env, "flux_z_t", a, stage);
    if (rc) return rc;
  } else {
    int rc = flux_launch<COMPACT, BOX, 0, LINES, STR>(env, "flux_x", a, stage);
    if (!rc && D > 1) rc = flux_launch<COMPACT, BOX, (D > 1 ? 1 : 0), LINES, STR>(env, "flux_y", a, stage);
    if (!rc && D > 2) rc = flux_launch<COMPACT, BOX, (D > 2 ? 2 : 0), LINES, STR>(env, "flux_z", a, stage);
    if (rc) return rc;
  }
  {
    // cells of the planes [kc0, kc1): all, or the z-chunk; chunk face records start at plane kc0
    const int kc0 = a.cn < 0 ? 0 : a.ck0, kc1 = a.cn < 0 ? a.nz : a.ck0 + a.cn;
    constexpr int NGL_ = D == 3 ? 4 : (D == 2 ? 2 : 1);
    constexpr int NFR = COMPACT ? (LINES ? 30 + 2 * NGL_ * 10 : 30) : 10;
    double* fc[3];
    for (int d = 0; d < 3; ++d)
      fc[d] = a.face[d] ? a.face[d] - (long long)kc0 * NFR * a.fn[d][0] * a.fn[d][1] : nullptr;
    const long long ncl = (long long)(kc1 - kc0) * (a.ncell / a.nz);
    if (mode == 0)
      LAUNCH("update", (k_update<D, COMPACT, 0, LINES>), ncl, 256, a.Uin, fc[0], fc[1], fc[2], a.Uout, a.carry,
             a.ts, a.err, a.Lout, a.Lcarry, kc0, kc1);
    else if (mode == 1)
      LAUNCH("update", (k_update<D, COMPACT, 1, LINES>), ncl, 256, a.Uin, fc[0], fc[1], fc[2], a.Uout, a.carry,
             a.ts, a.err, a.Lout, a.Lcarry, kc0, kc1);
    else
      LAUNCH("update", (k_update<D, COMPACT, 2, LINES>), ncl, 256, a.Uin, fc[0], fc[1], fc[2], a.Uout, a.carry,
             a.ts, a.err, a.Lout, a.Lcarry, kc0, kc1);
  }
  return 0;
}

int stage_fn(LaunchEnv& env, const StageArgs& a, int mode, int stage) {
  const bool c = a.scheme == 1, nl = a.nonlinear != 0, b = a.box != 0;
  if (a.stretched) {  // stretched tensor-product mesh (NEXT-4)
    if (c && a.lines) {  // with line DOFs (NEXT-1)
      if (!nl && !b) return stage_t<true, false, false, true, true>(env, a, mode, stage);
      if (nl && !b) return stage_t<true, true, false, true, true>(env, a, mode, stage);
      if (!nl && b) return stage_t<true, false, true, true, true>(env, a, mode, stage);
      return stage_t<true, true, true, true, true>(env, a, mode, stage);
    }
    if (c && !nl && !b) return stage_t<true, false, false, false, true>(env, a, mode, stage);
    if (c && nl && !b) return stage_t<true, true, false, false, true>(env, a, mode, stage);
    if (c && !nl && b) return stage_t<true, false, true, false, true>(env, a, mode, stage);
    if (c && nl && b) return stage_t<true, true, true, false, true>(env, a, mode, stage);
    if (!c && !nl && !b) return stage_t<false, false, false, false, true>(env, a, mode, stage);
    if (!c && nl && !b) return stage_t<false, true, false, false, true>(env, a, mode, stage);
    if (!c && !nl && b) return stage_t<false, false, true, false, true>(env, a, mode, stage);
    return stage_t<false, true, true, false, true>(env, a, mode, stage);
  }
  if (c && a.lines) {  // CGKS-5th with line DOFs (NEXT-1)
    if (!nl && !b) return stage_t<true, false, false, true>(env, a, mode, stage);
    if (nl && !b) return stage_t<true, true, false, true>(env, a, mode, stage);
    if (!nl && b) return stage_t<true, false, true, true>(env, a, mode, stage);
    return stage_t<true, true, true, true>(env, a, mode, stage);
  }
  if (c && !nl && !b) return stage_t<true, false, false>(env, a, mode, stage);
  if (c && nl && !b) return stage_t<true, true, false>(env, a, mode, stage);
  if (c && !nl && b) return stage_t<true, false, true>(env, a, mode, stage);
  if (c && nl && b) return stage_t<true, true, true>(env, a, mode, stage);
  if (!c && !nl && !b) return stage_t<false, false, false>(env, a, mode, stage);
  if (!c && nl && !b) return stage_t<false, true, false>(env, a, mode, stage);
  if (!c && !nl && b) return stage_t<false, false, true>(env, a, mode, stage);
  return stage_t<false, true, true>(env, a, mode, stage);
}

// diagnostics: reconstruction of the state a.Uin, then quadrature per (cell, node); returns the number of
// block partials written to part (4 doubles each)
// the reconstruction of a.Uin in the context's variant (line DOFs, stretched mesh), for the diagnostics
template <bool COMPACT, bool NONLIN, bool BOX>
int recon_any(LaunchEnv& env, const StageArgs& a) {
  if (COMPACT) {
    if (a.lines && a.stretched) return recon5_launch<NONLIN, BOX, true, true>(env, a);
    if (a.lines) return recon5_launch<NONLIN, BOX, true, false>(env, a);
    if (a.stretched) return recon5_launch<NONLIN, BOX, false, true>(env, a);
    return recon5_launch<NONLIN, BOX>(env, a);
  }
  LAUNCH("recon2", (k_recon2<D, NONLIN, BOX>), a.necell, 256, a.Uin, a.rec, a.err, 0, 1 << 30);
  return 0;
}

template <bool COMPACT, bool NONLIN, bool BOX>
int diag_t(LaunchEnv& env, const StageArgs& a, const double* wtab, double* part, long long* nblk) {
  {
    int rc = recon_any<COMPACT, NONLIN, BOX>(env, a);
    if (rc) return rc;
  }
  constexpr int NP = DiagQuad<D>::NP;
  *nblk = (a.ncell * NP + 255) / 256;
  LAUNCH("diag", (k_diag<D, COMPACT>), a.ncell * NP, 256, (const double*)a.Uin, (const double*)a.rec, wtab, part);
  return 0;
}

// Q-criterion of a.Uin at the cell centroids into out[ncell] (reconstruction first)
template <bool COMPACT, bool NONLIN, bool BOX>
int qcrit_t(LaunchEnv& env, const StageArgs& a, const double* wc, double* out) {
  {
    int rc = recon_any<COMPACT, NONLIN, BOX>(env, a);
    if (rc) return rc;
  }
  LAUNCH("qcrit", (k_qcrit<D, COMPACT>), a.ncell, 256, (const double*)a.Uin, (const double*)a.rec, wc, out);
  return 0;
}

int qcrit_fn(LaunchEnv& env, const StageArgs& a, const double* wc, double* out) {
  const bool c = a.scheme == 1, nl = a.nonlinear != 0, b = a.box != 0;
  if (c && !nl && !b) return qcrit_t<true, false, false>(env, a, wc, out);
  if (c && nl && !b) return qcrit_t<true, true, false>(env, a, wc, out);
  if (c && !nl && b) return qcrit_t<true, false, true>(env, a, wc, out);
  if (c && nl && b) return qcrit_t<true, true, true>(env, a, wc, out);
  if (!c && !nl && !b) return qcrit_t<false, false, false>(env, a, wc, out);
  if (!c && nl && !b) return qcrit_t<false, true, false>(env, a, wc, out);
  if (!c && !nl && b) return qcrit_t<false, false, true>(env, a, wc, out);
  return qcrit_t<false, true, true>(env, a, wc, out);
}

int diag_fn(LaunchEnv& env, const StageArgs& a, const double* wtab, double* part, long long* nblk) {
  const bool c = a.scheme == 1, nl = a.nonlinear != 0, b = a.box != 0;
  if (c && !nl && !b) return diag_t<true, false, false>(env, a, wtab, part, nblk);
  if (c && nl && !b) return diag_t<true, true, false>(env, a, wtab, part, nblk);
  if (c && !nl && b) return diag_t<true, false, true>(env, a, wtab, part, nblk);
  if (c && nl && b) return diag_t<true, true, true>(env, a, wtab, part, nblk);
  if (!c && !nl && !b) return diag_t<false, false, false>(env, a, wtab, part, nblk);
  if (!c && nl && !b) return diag_t<false, true, false>(env, a, wtab, part, nblk);
  if (!c && !nl && b) return diag_t<false, false, true>(env, a, wtab, part, nblk);
  return diag_t<false, true, true>(env, a, wtab, part, nblk);
}

template <bool C>
void flux_tile_t(int ax, int* tx, int* tn, int* nfbox) {
  if (ax == 0) {
    *tx = FluxTileSel<0, C>::TX;
    *tn = FluxTileSel<0, C>::TN;
    *nfbox = FluxTileSel<0, C>::NRH;
  } else if (ax == 1) {
    *tx = FluxTileSel<(D > 1 ? 1 : 0), C>::TX;
    *tn = FluxTileSel<(D > 1 ? 1 : 0), C>::TN;
    *nfbox = FluxTileSel<(D > 1 ? 1 : 0), C>::NRH;
  } else {
    *tx = FluxTileSel<(D > 2 ? 2 : 0), C>::TX;
    *tn = FluxTileSel<(D > 2 ? 2 : 0), C>::TN;
    *nfbox = FluxTileSel<(D > 2 ? 2 : 0), C>::NRH;
  }
}

void flux_tile_fn(int ax, int compact, int* tx, int* tn, int* nfbox) {
  if (compact)
    flux_tile_t<true>(ax, tx, tn, nfbox);
  else
    flux_tile_t<false>(ax, tx, tn, nfbox);
}

int lines_init_fn(cudaStream_t s, const double* U, double* Lb, long long ncell) {
  k_lines_from_grad<D><<<(unsigned)((ncell + 255) / 256), 256, 0, s>>>(U, Lb);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

int upload_fn(const Geo& g, const FluxConst& fc, const double* Rp, int nnz, cudaStream_t s) {
  if (cudaMemcpyToSymbolAsync(c_geo, &g, sizeof(Geo), 0, cudaMemcpyHostToDevice, s) != cudaSuccess) return 5;
  if (cudaMemcpyToSymbolAsync(c_fc, &fc, sizeof(FluxConst), 0, cudaMemcpyHostToDevice, s) != cudaSuccess) return 5;
  if (nnz > 0 && cudaMemcpyToSymbolAsync(c_Rp, Rp, sizeof(double) * nnz, 0, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return 5;
  return 0;
}

int dt_fn(LaunchEnv& env, const double* U, int NV, TimeState* ts, ErrState* err, long long ncell) {
  LAUNCH("dt", k_dt<D>, ncell, 256, U, NV, ts, err);
  return 0;
}

int dt_final_fn(LaunchEnv& env, TimeState* ts, ErrState* err) {
  LAUNCH("dt_finalize", k_dt_finalize, 1, 32, ts, err);
  return 0;
}

int step_end_fn(LaunchEnv& env, TimeState* ts, ErrState* err) {
  LAUNCH("step_end", k_step_end, 1, 32, ts, err);
  return 0;
}

int err_poison_fn(LaunchEnv& env, TimeState* ts, ErrState* err, long long test_step) {
  LAUNCH("err_poison", k_err_poison, 1, 32, ts, (const ErrState*)err, test_step);
  return 0;
}

int pack_fn(cudaStream_t s, const double* src, double* dst, int NV, int f0, int nf, long long ncell) {
  const long long n = ncell * nf;
  k_pack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, dst, NV, f0, nf);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

int unpack_fn(cudaStream_t s, const double* src, double* dst, int NV, int f0, int nf, long long ncell) {
  const long long n = ncell * nf;
  k_unpack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, dst, NV, f0, nf);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

}  // namespace
}  // namespace cgks
