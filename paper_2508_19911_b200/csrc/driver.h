// driver.h -- host-side interface between the C ABI (cgks_api.cu) and the per-dimension
// translation units (stage_d1.cu, stage_d2.cu, stage_d3.cu) that hold the kernels.
// Each dimension is compiled separately (parallel builds); each owns its constant memory,
// so the ABI uploads the context's parameters through every unit it uses.
#pragma once
#include <cuda.h>  // CUtensorMap
#include <cuda_runtime.h>

#include <string>
#include <utility>
#include <vector>

#include "types.h"

namespace cgks {

struct LaunchEnv {
  cudaStream_t stream = nullptr;
  bool prof = false;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>>* pending = nullptr;
  char* msg = nullptr;
  int msglen = 0;
};

struct StageArgs {
  const double* Uin;
  double* Uout;
  double* carry;
  double* rec;
  double* face[3];
  const double* gtab[3];
  TimeState* ts;
  ErrState* err;
  long long ncell, necell;
  long long nface[3];
  int fn[3][3];   // face-grid dims per normal axis
  int en[3];      // extended (reconstruction) range per axis
  int scheme;     // 0 GKS-2nd, 1 CGKS-5th
  int nonlinear;
  int box;
  // line DOFs (CGKS-5th, NEXT-1): lines of Uin, of Uout, and the stage carry ([z][l*5+v][y][x])
  const double* Lin = nullptr;
  double* Lout = nullptr;
  double* Lcarry = nullptr;
  int lines = 0;
  int stretched = 0;  // stretched tensor-product mesh (NEXT-4)
  // TMA descriptors of the flux tiles per normal axis (reconstruction fields; cell averages of Uin)
  const CUtensorMap* tm_rec = nullptr;
  const CUtensorMap* tm_U = nullptr;
  int use_tma = 0;
  // stage parts (halo overlap of z-slab ranks): 0 = the whole stage; 1 = the reconstruction of the
  // extended z planes [rz0, rz1) only (offsets from the first extended plane); 3 = fluxes + update only
  int part = 0;
  int rz0 = 0, rz1 = -1;
  // z-chunked stage (large grids): cells of the planes [ck0, ck0 + cn) with the chunk's own
  // reconstruction (planes ck0 - 1 .. ck0 + cn) and face buffers; cn < 0: the whole slab
  int ck0 = 0, cn = -1;
  int nz = 1;  // local cell planes
};

struct DimOps {
  int (*upload)(const Geo& g, const FluxConst& fc, const double* Rp, int nnz, cudaStream_t s);
  // mode 0: S2O4 stage 1, 1: S2O4 stage 2, 2: S1O2
  int (*stage)(LaunchEnv& env, const StageArgs& a, int mode, int stage);
  int (*dt)(LaunchEnv& env, const double* U, int NV, TimeState* ts, ErrState* err, long long ncell);  // local min
  int (*dt_final)(LaunchEnv& env, TimeState* ts, ErrState* err);  // dt = CFL * (global) min
  // end of a step: t, steps += 1 and the next dt from the final update's fused CFL min (rank-reduced)
  int (*step_end)(LaunchEnv& env, TimeState* ts, ErrState* err);
  // NCCL slab runs: a failing rank posts its error code into the dt min before the allreduce
  // (test_step >= 0: test hook emulating a peer rank's failure in that step, CGKS_TEST_PEER_FAIL_STEP)
  int (*err_poison)(LaunchEnv& env, TimeState* ts, ErrState* err, long long test_step);
  int (*pack)(cudaStream_t s, const double* src, double* dst, int NV, int f0, int nf, long long ncell);
  int (*unpack)(cudaStream_t s, const double* src, double* dst, int NV, int f0, int nf, long long ncell);
  // flow diagnostics of a.Uin (reconstruction + quadrature); *nblk = number of 4-double block partials
  int (*diag)(LaunchEnv& env, const StageArgs& a, const double* wtab, double* part, long long* nblk);
  // flux tile extent (cells along x, cells along the normal axis) for the TMA boxes, CGKS-5th
  void (*flux_tile)(int ax, int compact, int* tx, int* tn, int* nfbox);  // flux tile extents, fields per TMA box
  // Q-criterion of a.Uin at the cell centroids (reconstruction + k_qcrit) into out[ncell]
  int (*qcrit)(LaunchEnv& env, const StageArgs& a, const double* wc, double* out);
  // line DOFs initialised from the gradients of U
  int (*lines_init)(cudaStream_t s, const double* U, double* Lb, long long ncell);
};

extern const DimOps kOps1, kOps2, kOps3;

}  // namespace cgks
