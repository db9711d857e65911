// kernels.cuh -- sm_100a FP64 kernels of one CGKS-5th / GKS-2nd stage.
//
//   k_recon5   compact CLS quartic coefficients per cell, GENO folded in
//   k_recon2   GKS-2nd least-squares slopes with Venkatakrishnan limiting
//   k_flux1    one thread per (face, Gauss point): evaluate both sides, gas-kinetic
//              flux + interface values, 2x2 Gauss face average by warp
//              shuffles, one face record per face (flux1.cuh)
//   k_update   residual L, dL/dt, Gauss-theorem gradients and the
//              S2O4 / S1O2 stage combinations
//   k_dt       CFL candidate per cell, warp-shuffle + block min, atomicMin
//
// Layout of every cell field: [z][field][y][x], x fastest (coalesced along x).
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors; no driver-API calls on the device)
#include <cuda_runtime.h>
#include <stdint.h>

#include "gks_flux.cuh"
#include "types.h"

namespace cgks {
template <int DIM>
struct ReconGen;
template <int DIM>
struct ReconGenL;  // line-DOF variant
}
#include "recon_gen.cuh"

namespace cgks {

constexpr int NBmax = 34;

// per translation unit (one per dimension, see stage_impl.cuh): internal linkage
static __constant__ Geo c_geo;
static __constant__ FluxConst c_fc;
constexpr int kMaxNNZ = ReconGen<3>::NNZ > ReconGenL<3>::NNZ ? ReconGen<3>::NNZ : ReconGenL<3>::NNZ;
static __constant__ double c_Rp[kMaxNNZ];  // parity-blocked CLS matrix (gen_recon.py), packed

// ---------------------------------------------------------------------------
// compile-time stencil tables (match cls_build.cpp ordering)
// ---------------------------------------------------------------------------
template <int DIM>
struct Sten {
  static constexpr int NB = DIM == 3 ? 34 : (DIM == 2 ? 14 : 4);
  static constexpr int NFACE = 2 * DIM;
  static constexpr int NEDGE = DIM == 3 ? 12 : (DIM == 2 ? 4 : 0);
  static constexpr int NC = NFACE + NEDGE;
  static constexpr int NL = NFACE * DIM + (DIM == 3 ? 2 * NEDGE : DIM * NEDGE) + DIM;
  static constexpr int ND = NC + NL;
  static constexpr int NG = DIM == 3 ? 4 : (DIM == 2 ? 2 : 1);  // face Gauss points (K)
};

// offset component `ax` of neighbour n (faces (-a,+a) per axis, then edges for axis pairs a<b)
template <int DIM>
__host__ __device__ constexpr int nbr_off(int n, int ax) {
  if (n < 2 * DIM) return (n / 2 == ax) ? ((n % 2) ? 1 : -1) : 0;
  int e = n - 2 * DIM;
  int pair = e / 4, sgn = e % 4;
  int a = 0, b = 1;
  if (DIM == 3) {
    if (pair == 0) { a = 0; b = 1; }
    if (pair == 1) { a = 0; b = 2; }
    if (pair == 2) { a = 1; b = 2; }
  }
  int sa = (sgn / 2) ? 1 : -1, sb = (sgn % 2) ? 1 : -1;
  if (ax == a) return sa;
  if (ax == b) return sb;
  return 0;
}

// ---------------------------------------------------------------------------
// state access with periodic wrap or box ghost rules (R29)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

__device__ __forceinline__ long long sidx(int NV, int f, int i, int j, int k) {
  return ((long long)(k + c_geo.zoff) * NV + f) * c_geo.splane + (long long)(j + c_geo.yoff) * c_geo.n[0] + i;
}

// periodic wrap, except on decomposed axes whose ghost cells are stored
__device__ __forceinline__ int wrap_ax(int a, int i) { return c_geo.halo[a] ? i : wrapi(i, c_geo.n[a]); }
// the same with the passed index clamped to the 2 stored ghost layers: the ragged tail of a reconstruction tile
// reaches further (its values feed no cell, but the read must stay inside the buffer)
__device__ __forceinline__ int wrap_ax_c(int a, int i) {
  return c_geo.halo[a] ? min(max(i, -2), c_geo.n[a] + 1) : wrapi(i, c_geo.n[a]);
}

// value of field f (0-4 Q, 5-19 gradient [axis][var]) of cell (i,j,k), any integer index
template <bool BOX>
__device__ __forceinline__ double ld_state(const double* __restrict__ U, int NV, int f, int i, int j, int k) {
  int idx[3] = {i, j, k};
  if (BOX) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (c_geo.bounded[a] && !c_geo.halo[a] && (idx[a] < 0 || idx[a] >= c_geo.n[a])) {
        int side = idx[a] < 0 ? 0 : 1;
        if (c_geo.bc[a][side] == 1) return f < 5 ? c_geo.bc_state[a][side][f] : 0.0;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (c_geo.halo[a]) {  // stored ghosts (the ragged tail of a reconstruction tile stays inside the buffer)
        idx[a] = min(max(idx[a], -2), c_geo.n[a] + 1);
        continue;
      }
      if (c_geo.bounded[a]) {
        idx[a] = idx[a] < 0 ? 0 : (idx[a] >= c_geo.n[a] ? c_geo.n[a] - 1 : idx[a]);
      } else {
        idx[a] = wrapi(idx[a], c_geo.n[a]);
      }
    }
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) idx[a] = wrap_ax(a, idx[a]);
  }
  return __ldg(U + sidx(NV, f, idx[0], idx[1], idx[2]));
}

// index into an extended-range per-cell buffer (coefficients / slopes), layout [z][y][field][x]:
// the NF fields of one x-row are contiguous (field stride en0), so a tile of a few rows spans a few
// contiguous blocks instead of one memory page per field and plane
__device__ __forceinline__ long long eidx(int NF, int f, int i, int j, int k) {
  // periodic axes wrap; bounded axes are stored from elo = -1
  int ii = c_geo.bounded[0] ? i : wrapi(i, c_geo.n[0]);
  int jj = c_geo.bounded[1] ? j : wrapi(j, c_geo.n[1]);
  int kk = c_geo.bounded[2] ? k : wrapi(k, c_geo.n[2]);
  ii -= c_geo.elo[0];
  jj -= c_geo.elo[1];
  kk -= c_geo.elo[2];
  return (((long long)kk * c_geo.en[1] + jj) * NF + f) * c_geo.en[0] + ii;
}

// CGKS-5th reconstruction coefficients (5 NB per cell): layout [z][y][pair][x][2] with pair p = (kk / 2) * 5 + v,
// i.e. the coefficients kk and kk + 1 (kk even) of component v of one cell side by side: one 16-byte store in
// the reconstruction, one 16-byte shared-memory load in the flux evaluation, and TMA rows of 2 x the tile
// width (half as many rows as one field per row)
__device__ __forceinline__ long long cidx(int NCO, int kk, int v, int i, int j, int k) {
  int ii = c_geo.bounded[0] ? i : wrapi(i, c_geo.n[0]);
  int jj = c_geo.bounded[1] ? j : wrapi(j, c_geo.n[1]);
  int kz = c_geo.bounded[2] ? k : wrapi(k, c_geo.n[2]);
  ii -= c_geo.elo[0];
  jj -= c_geo.elo[1];
  kz -= c_geo.elo[2];
  return ((long long)kz * c_geo.en[1] + jj) * NCO * c_geo.en[0] + (long long)((kk >> 1) * 5 + v) * 2 * c_geo.en[0] +
         2 * ii + (kk & 1);
}

// stretched meshes (R37): width / inverse width of cell index c along a (c in -2 .. n+1)
__device__ __forceinline__ double cw(int a, int c) { return __ldg(c_geo.hw[a] + c + 2); }
__device__ __forceinline__ double icw(int a, int c) { return __ldg(c_geo.ihw[a] + c + 2); }

// 8-byte asynchronous global -> shared copy (cp.async.ca, LDGSTS) and the matching wait
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async8s(unsigned smem_addr, const double* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16s(unsigned smem_addr, const double* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// TMA (cp.async.bulk.tensor) tile load completing on an mbarrier, and the mbarrier primitives
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b)
      : "memory");
}

// 1-D bulk copy global -> shared (bytes a multiple of 16, both addresses 16-byte aligned) on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}

// Debug bounds checks (build with CGKS_NVCC_DEFS=-DCGKS_CHECK; the pool has no compute-sanitizer): an index
// outside its buffer prints the site and traps (the context then reports CGKS_ERR_CUDA)
#ifdef CGKS_CHECK
#define CGKS_BOUND(i, n, what)                                                                              \
  do {                                                                                                      \
    if ((long long)(i) < 0 || (long long)(i) >= (long long)(n)) {                                           \
      printf("CGKS_CHECK %s: index %lld outside [0, %lld) at %s:%d block (%d,%d,%d) thread %d\n", what,     \
             (long long)(i), (long long)(n), __FILE__, __LINE__, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x); \
      __trap();                                                                                             \
    }                                                                                                       \
  } while (0)
#else
#define CGKS_BOUND(i, n, what) \
  do {                         \
  } while (0)
#endif

// Schedule perturbation (build with -DCGKS_JITTER): each warp sleeps a pseudo-random 0-4 us before the
// synchronisation points of the flux and reconstruction kernels, so that a missing barrier shows up as a
// run-to-run difference against the unperturbed build (results must stay bitwise equal)
#ifdef CGKS_JITTER
__device__ __forceinline__ void cgks_jitter(unsigned salt) {
  unsigned h = (blockIdx.x * 2654435761u) ^ (blockIdx.y * 40503u) ^ (blockIdx.z * 69069u) ^ ((threadIdx.x >> 5) * 97u) ^
               (salt * 2246822519u);
  h ^= h >> 13;
  h *= 3266489917u;
  h ^= h >> 16;
#ifdef CGKS_JITTER_ZERO
  __nanosleep(h & 1u);
#else
  __nanosleep(h & 4095u);
#endif
}
#ifndef CGKS_JIT_MASK
#define CGKS_JIT_MASK 0xff
#endif
#define CGKS_JIT(salt)                                    \
  do {                                                    \
    if ((CGKS_JIT_MASK >> (salt)) & 1) cgks_jitter(salt); \
  } while (0)
#else
#define CGKS_JIT(salt) \
  do {                 \
  } while (0)
#endif

__device__ __forceinline__ void flag_error(ErrState* err, int code, int kernel, int stage, long long step, int i,
                                           int j, int k) {
  if (atomicCAS(&err->code, 0, code) == 0) {
    err->kernel = kernel;
    err->stage = stage;
    err->step = step;
    err->cell[0] = i;
    err->cell[1] = j;
    err->cell[2] = k;
  }
}

// ---------------------------------------------------------------------------
// K1: CGKS-5th reconstruction (coefficients of P^4 on the reference cell, GENO folded)
// ---------------------------------------------------------------------------
// Block tile of the reconstruction: TX x TY x TZ cells, stencil data of one component
// (Q_v and the three gradient components) staged with a one-cell halo in shared memory by
// cp.async, double-buffered over the five components.
// reconstruction block tile (3-D): 32 x TY x TZ cells; measured per launch: 32x4x2 (2 blocks per SM)
// 0.624 ms, 32x8x1: 0.660, 32x8x2 (1 block): 0.736
#ifndef CGKS_RECON_TY
#define CGKS_RECON_TY 4
#endif
#ifndef CGKS_RECON_TZ
#define CGKS_RECON_TZ 2
#endif
#ifndef CGKS_RECON_MINB
#define CGKS_RECON_MINB 2  // resident reconstruction blocks per SM (register cap 128)
#endif
template <int DIM>
struct ReconTile {
  static constexpr int TX = 32;
  static constexpr int TY = DIM == 3 ? CGKS_RECON_TY : (DIM == 2 ? 8 : 1);
  static constexpr int TZ = DIM == 3 ? CGKS_RECON_TZ : 1;
  static constexpr int NTH = TX * TY * TZ;
  static constexpr int HX = TX + 2, HY = DIM >= 2 ? TY + 2 : 1, HZ = DIM == 3 ? TZ + 2 : 1;
  static constexpr int HALO = HX * HY * HZ;
  static constexpr int NFS = 1 + DIM;  // staged fields per component: Q_v, dQ_v/dx_a
  // two component buffers + the per-position staging offsets (ReconStageMap)
  static constexpr size_t smem_bytes() { return sizeof(double) * 2 * NFS * HALO + sizeof(unsigned) * HALO; }
};

template <int DIM, bool STR = false>
struct Recon5TileLoader {
  const double* __restrict__ s;  // staged fields of this component, at this thread's cell
  double q0, h0, h1, h2;
  double w[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // STR: widths of the cells at offsets -1, 0, +1 per axis
  const double* __restrict__ lv = nullptr;  // line DOFs: line 0 of this component at this cell (field stride plane)
  long long lstride = 0;                    // 5 * plane: next line
  double lmask = 1.0;                       // 0 for the ghost cell of an inflow boundary (no lines)
  static constexpr int HALO = ReconTile<DIM>::HALO;
  static constexpr int SY = ReconTile<DIM>::HX, SZ = ReconTile<DIM>::HX * ReconTile<DIM>::HY;
  __device__ __forceinline__ double at(int f, int ox, int oy, int oz) const {
    return s[f * HALO + oz * SZ + oy * SY + ox];
  }
  __device__ __forceinline__ double q(int ox, int oy, int oz) const { return at(0, ox, oy, oz) - q0; }
  __device__ __forceinline__ double g(int a, int ox, int oy, int oz) const {
    if (STR)  // each cell in its own reference units (R37)
      return w[a][(a == 0 ? ox : (a == 1 ? oy : oz)) + 1] * at(1 + a, ox, oy, oz);
    return (a == 0 ? h0 : (a == 1 ? h1 : h2)) * at(1 + a, ox, oy, oz);
  }
  // own-cell line-averaged derivative l in reference units (h_a (d_l Q)_l, a = l / lines per axis)
  __device__ __forceinline__ double line(int l) const {
    constexpr int NGL = DIM == 3 ? 4 : (DIM == 2 ? 2 : 1);
    const int a = l / NGL;
    if (STR) return lmask * w[a][1] * __ldg(lv + l * lstride);  // the own width (R37)
    return lmask * (a == 0 ? h0 : (a == 1 ? h1 : h2)) * __ldg(lv + l * lstride);
  }
};

// Halo-tile staging of the reconstruction.  The global offset of each tile position (index arithmetic,
// periodic wrap) is computed once per block into a shared table; field f of component v of that position
// sits at offset + (fld(f) + v) * plane in the [z][field][y][x] layout, so staging a component is one
// table load per position and one address add + cp.async per element.
template <int DIM>
struct ReconStageMap {
  using RT = ReconTile<DIM>;
  unsigned* off;  // [HALO] in shared memory
  __device__ __forceinline__ void init(int x0, int y0, int z0) const {
    for (int h = threadIdx.x; h < RT::HALO; h += RT::NTH) {
      const int hx = h % RT::HX, hy = (h / RT::HX) % RT::HY, hz = h / (RT::HX * RT::HY);
      const int i = x0 - 1 + hx, j = DIM >= 2 ? y0 - 1 + hy : 0, kk = DIM == 3 ? z0 - 1 + hz : 0;
      off[h] = (unsigned)sidx(20, 0, wrap_ax_c(0, i), wrap_ax_c(1, j), wrap_ax_c(2, kk));
    }
  }
};

// stage fields (Q_v, G_{a,v}) of the block's halo tile into buf ([field][position])
template <int DIM, bool BOX>
__device__ __forceinline__ void recon_stage(const double* __restrict__ U, double* buf, int v, int x0, int y0,
                                            int z0, const ReconStageMap<DIM>& map) {
  using RT = ReconTile<DIM>;
  if (BOX) {
    for (int idx = threadIdx.x; idx < RT::NFS * RT::HALO; idx += RT::NTH) {
      const int f = idx / RT::HALO, h = idx % RT::HALO;
      const int hx = h % RT::HX, hy = (h / RT::HX) % RT::HY, hz = h / (RT::HX * RT::HY);
      const int i = x0 - 1 + hx, j = DIM >= 2 ? y0 - 1 + hy : 0, kk = DIM == 3 ? z0 - 1 + hz : 0;
      const int fld = f == 0 ? v : 5 + (f - 1) * 5 + v;
      buf[idx] = ld_state<true>(U, 20, fld, i, j, kk);
    }
  } else {
    const double* Uv = U + (long long)v * c_geo.splane;
#pragma unroll 1
    for (int h = threadIdx.x; h < RT::HALO; h += RT::NTH) {
      {
        const double* src = Uv + map.off[h];
#pragma unroll
        for (int f = 0; f < RT::NFS; ++f)
          cp_async8(buf + f * RT::HALO + h, src + (f == 0 ? 0 : 5 + (f - 1) * 5) * c_geo.splane);
      }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int DIM, bool NONLIN, bool BOX, bool LINES = false, bool STR = false>
__global__ void __launch_bounds__(ReconTile<DIM>::NTH, CGKS_RECON_MINB) k_recon5(const double* __restrict__ U,
                                                                    double* __restrict__ coef,
                                                                    const ErrState* __restrict__ err,
                                                                    const double* __restrict__ Lin = nullptr,
                                                                    int zb = 0, int ze = 1 << 30) {
  using S = Sten<DIM>;
  using RT = ReconTile<DIM>;
  constexpr int NCO = S::NB * 5;
  extern __shared__ double rsm[];
  if (__syncthreads_or(err->code != 0)) return;  // block-uniform (the staging pipeline synchronises)
  const int tx = threadIdx.x % RT::TX, ty = (threadIdx.x / RT::TX) % RT::TY, tz = threadIdx.x / (RT::TX * RT::TY);
  // block origin in the extended (reconstruction) index range
  const int x0 = blockIdx.x * RT::TX + c_geo.elo[0];
  const int y0 = blockIdx.y * RT::TY + c_geo.elo[1];
  // (z planes [zb, ze) of the extended range: a part of it when the halo exchange is overlapped)
  const int z0 = zb + blockIdx.z * RT::TZ + c_geo.elo[2];
  const int i = x0 + tx, j = y0 + ty, k = z0 + tz;
  const bool valid = (i < c_geo.elo[0] + c_geo.en[0]) && (j < c_geo.elo[1] + c_geo.en[1]) &&
                     (k < c_geo.elo[2] + min(c_geo.en[2], ze));
  const int own = (DIM == 3 ? (tz + 1) * RT::HX * RT::HY : 0) + (DIM >= 2 ? (ty + 1) * RT::HX : 0) + tx + 1;
  // the stencil reads own +- one cell per axis of the halo tile
  CGKS_BOUND(own - 1 - (DIM >= 2 ? RT::HX : 0) - (DIM == 3 ? RT::HX * RT::HY : 0), RT::HALO, "recon halo low");
  CGKS_BOUND(own + 1 + (DIM >= 2 ? RT::HX : 0) + (DIM == 3 ? RT::HX * RT::HY : 0), RT::HALO, "recon halo high");
  const ReconStageMap<DIM> map{reinterpret_cast<unsigned*>(rsm + 2 * RT::NFS * RT::HALO)};
  if (!BOX) {
    map.init(x0, y0, z0);
    __syncthreads();
  }
  // coefficients (q, q + 1) (q even) of component v at cb[((q / 2) * 5 + v) * 2 * en0 + {0, 1}] (cidx)
  double* cb = coef + (valid ? cidx(NCO, 0, 0, i, j, k) : 0);
  if (valid) {  // the extended range of this launch (zb .. ze planes of the buffer)
    CGKS_BOUND(i - c_geo.elo[0], c_geo.en[0], "recon i");
    CGKS_BOUND(j - c_geo.elo[1], c_geo.en[1], "recon j");
  }
  const long long ep = c_geo.en[0];  // field stride
  recon_stage<DIM, BOX>(U, rsm, 0, x0, y0, z0, map);
#pragma unroll 1
  for (int v = 0; v < 5; ++v) {
    double* cur = rsm + (v & 1) * RT::NFS * RT::HALO;
    if (v < 4) {
      recon_stage<DIM, BOX>(U, rsm + ((v + 1) & 1) * RT::NFS * RT::HALO, v + 1, x0, y0, z0, map);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    CGKS_JIT(1);
    __syncthreads();
    Recon5TileLoader<DIM, STR> L{cur + own, 0.0, c_geo.h[0], c_geo.h[1], c_geo.h[2]};
    L.q0 = L.at(0, 0, 0, 0);
    if (STR) {
      const int ci[3] = {i, j, k};
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int o = -1; o <= 1; ++o) L.w[a][o + 1] = cw(a, min(max(ci[a] + o, -2), c_geo.n[a] + 1));
    }
    if (LINES) {  // own-cell lines, [z][l*5+v][y][x] (valid cells only; ragged threads read cell 0)
      constexpr int NLF = 5 * (DIM == 3 ? 12 : (DIM == 2 ? 4 : 1));
      int li[3] = {i, j, k};
      if (BOX) {  // box ghost cells: the boundary cell's lines (outflow), none (inflow), as ld_state
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (c_geo.halo[a]) continue;
          if (c_geo.bounded[a]) {
            if (li[a] < 0 || li[a] >= c_geo.n[a]) {
              if (c_geo.bc[a][li[a] < 0 ? 0 : 1] == 1) L.lmask = 0.0;
              li[a] = li[a] < 0 ? 0 : c_geo.n[a] - 1;
            }
          } else {
            li[a] = wrapi(li[a], c_geo.n[a]);
          }
        }
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) li[a] = wrap_ax(a, li[a]);
      }
      L.lv = Lin + (valid ? sidx(NLF, v, li[0], li[1], li[2]) : 0);
      L.lstride = 5 * c_geo.splane;
    }
    double acc[S::NB];
#pragma unroll
    for (int q = 0; q < S::NB; ++q) acc[q] = 0.0;
    // parity-blocked constrained least squares: data in difference form, so a
    // uniform field gives exactly zero coefficients
    if (LINES)
      ReconGenL<DIM>::matvec(L, c_Rp, acc);
    else
      ReconGen<DIM>::matvec(L, c_Rp, acc);
    if (NONLIN) {
      // GENO: sub-stencil linears P_m (R6), IS (R7), weights (R9), chi (R8);
      // Eq. (weno-new) folded into the coefficients (shared zero-mean basis, sum omega = 1)
      double IS[S::NFACE], bm[S::NFACE][3], gown[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        if (LINES) {  // the selected line derivatives: the lines along a, averaged (SPEC)
          constexpr int NGL = DIM == 3 ? 4 : (DIM == 2 ? 2 : 1);
          double sum = 0.0;
#pragma unroll
          for (int g = 0; g < NGL; ++g) sum += L.line(a * NGL + g);
          gown[a] = sum * (1.0 / NGL);
        } else {
          gown[a] = L.g(a, 0, 0, 0);
        }
      }
#pragma unroll
      for (int m = 0; m < S::NFACE; ++m) {
        const int ax = m / 2;
        const double s = (m % 2) ? 1.0 : -1.0;
        const double dface = L.q(ax == 0 ? (int)s : 0, ax == 1 ? (int)s : 0, ax == 2 ? (int)s : 0);
#pragma unroll
        for (int a = 0; a < 3; ++a) bm[m][a] = (a < DIM && a != ax) ? gown[a] : 0.0;
        bm[m][ax] = s * dface;
        IS[m] = bm[m][0] * bm[m][0] + bm[m][1] * bm[m][1] + bm[m][2] * bm[m][2];
      }
      const double eps = 1e-15;
      double ismax = IS[0], ismin = IS[0];
#pragma unroll
      for (int m = 1; m < S::NFACE; ++m) {
        ismax = fmax(ismax, IS[m]);
        ismin = fmin(ismin, IS[m]);
      }
      double lin[3] = {0.0, 0.0, 0.0};
      // omega_m = (IS_m + eps)^-5 / sum_k (IS_k + eps)^-5 (R9): with eps = 1e-15 every term is
      // at most 1e75, so the normalised form cannot overflow (6 reciprocals, no ratio table)
      double w5[S::NFACE], s5 = 0.0;
#pragma unroll
      for (int kk = 0; kk < S::NFACE; ++kk) {
        const double iv = 1.0 / (IS[kk] + eps);
        const double i2 = iv * iv;
        w5[kk] = i2 * i2 * iv;
        s5 += w5[kk];
      }
      const double is5 = 1.0 / s5;
#pragma unroll
      for (int m = 0; m < S::NFACE; ++m) {
        const double w = w5[m] * is5;
#pragma unroll
        for (int a = 0; a < DIM; ++a) lin[a] = fma(w, bm[m][a], lin[a]);
      }
      const double zeta = (ismax - ismin) / (ismin + eps + c_geo.chi_c * ismax) * c_geo.chi_is;
      const double z2 = zeta * zeta;
      const double chi = 1.0 / (1.0 + z2 * z2);
#pragma unroll
      for (int q = 0; q < S::NB; ++q) acc[q] *= chi;
#pragma unroll
      for (int a = 0; a < DIM; ++a) acc[a] = fma(1.0 - chi, lin[a], acc[a]);
    }
    if (valid) {
      double2* cv = reinterpret_cast<double2*>(cb + v * 2 * ep);
      static_assert(S::NB % 2 == 0, "coefficient pairs");
#pragma unroll
      for (int q = 0; q < S::NB; q += 2) {
        // streaming 16-byte store (evict-first: the coefficients are read back from HBM by the sweeps anyway);
        // running pointer, no per-coefficient index arithmetic
        __stcs(cv, make_double2(acc[q], acc[q + 1]));
        cv += 5 * ep;  // next pair of this component: 5 pairs of 2 x en0 doubles on
      }
    }
    CGKS_JIT(2);
    __syncthreads();  // this buffer is refilled by the prefetch two components ahead
  }
}

// ---------------------------------------------------------------------------
// K1': GKS-2nd slopes (reference units), limited
// ---------------------------------------------------------------------------
template <int DIM, bool NONLIN, bool BOX>
__global__ void __launch_bounds__(256) k_recon2(const double* __restrict__ U, double* __restrict__ slope,
                                                 const ErrState* __restrict__ err, int zb = 0, int ze = 1 << 30) {
  constexpr int NV = 5;
  if (err->code) return;
  // extended z planes [zb, ze) (a part of the range when the halo exchange is overlapped)
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x + (long long)zb * c_geo.en[0] * c_geo.en[1];
  const long long ntot = (long long)c_geo.en[0] * c_geo.en[1] * min(c_geo.en[2], ze);
  if (t >= ntot) return;
  const int i = (int)(t % c_geo.en[0]) + c_geo.elo[0];
  const int j = (int)((t / c_geo.en[0]) % c_geo.en[1]) + c_geo.elo[1];
  const int k = (int)(t / ((long long)c_geo.en[0] * c_geo.en[1])) + c_geo.elo[2];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const double q0 = ld_state<BOX>(U, NV, v, i, j, k);
    double qm[3], qp[3], b[3];
    double qmax = q0, qmin = q0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      qm[a] = ld_state<BOX>(U, NV, v, i - (a == 0), j - (a == 1), k - (a == 2));
      qp[a] = ld_state<BOX>(U, NV, v, i + (a == 0), j + (a == 1), k + (a == 2));
      b[a] = 0.5 * (qp[a] - qm[a]);  // least-squares slope on the uniform stencil (R12)
      qmax = fmax(qmax, fmax(qm[a], qp[a]));
      qmin = fmin(qmin, fmin(qm[a], qp[a]));
    }
    double phi = 1.0;
    if (NONLIN) {  // Venkatakrishnan (R11)
      double e2 = c_geo.eps_venkat2;
      if (c_geo.stretched) {  // (K h_g)^3 with the cell's own geometric-mean width (R37)
        double hp = 1.0;
        for (int a = 0; a < DIM; ++a) hp *= cw(a, a == 0 ? i : (a == 1 ? j : k));
        const double kv = c_geo.k_venkat;
        e2 = kv * kv * kv * (DIM == 3 ? hp : (DIM == 2 ? hp * sqrt(hp) : hp * hp * hp));
      }
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
#pragma unroll
        for (int s = -1; s <= 1; s += 2) {
          const double d2 = 0.5 * s * b[a];
          double ph = 1.0;
          if (d2 != 0.0) {
            const double d1 = d2 > 0.0 ? qmax - q0 : qmin - q0;
            ph = (d1 * d1 + e2 + 2.0 * d1 * d2) / (d1 * d1 + 2.0 * d2 * d2 + d1 * d2 + e2);
          }
          phi = fmin(phi, ph);
        }
      }
      phi = fmax(0.0, fmin(1.0, phi));
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) slope[eidx(15, a * 5 + v, i, j, k)] = (a < DIM) ? phi * b[a] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// K2: interface flux, one lane per (face, Gauss point): flux1.cuh (k_flux1).
// Face record (per face, normal axis AX): Fn[5] Ft[5] (+ QLn QLt QRn QRt for CGKS-5th).
// The face between cells (idx - e_AX) and idx carries the index idx (0..n, n+1 faces if bounded).
// ---------------------------------------------------------------------------
// threads per flux block (= Gauss points per block) per normal axis: 64 (16 faces: an x-run of 16, or a
// 4 x 4 y-/z-face patch, CGKS_FY1 in flux1.cuh), 6 blocks = 12 warps per SM (168 registers).  Measured per
// launch before the 4 x 4 patches (ms, x / y / z):
// x-faces 64 threads 1.535 vs 128: 1.71, 32: 1.92; y/z-faces 64 threads (8 x 2) 1.539 / 1.530 vs 128 (16 x 2)
// 1.542 / 1.545, 128 (8 x 4) 1.62 / 1.62 (round-2 kernel); 16 warps per SM (128 registers) spill and lose
// ~35 %
#ifndef CGKS_FLUX_NTHR_X
#define CGKS_FLUX_NTHR_X 64
#endif
#ifndef CGKS_FLUX_NTHR_YZ
#define CGKS_FLUX_NTHR_YZ 64
#endif
// resident warps per SM the flux kernels are compiled for (register cap = 65536 / (32 x warps))
#ifndef CGKS_FLUX_WARPS_X
#define CGKS_FLUX_WARPS_X 12
#endif
#ifndef CGKS_FLUX_WARPS_YZ
#define CGKS_FLUX_WARPS_YZ 12
#endif

}  // namespace cgks
#include "flux1.cuh"

namespace cgks {
// ---------------------------------------------------------------------------
// K3: residual, Gauss-theorem gradients and stage update
//   MODE 0: S2O4 stage 1  (Uin = U^n -> Uout = U*, carry)
//   MODE 1: S2O4 stage 2  (carry -> Uout = U^{n+1})
//   MODE 2: S1O2          (Uin = U^n -> Uout = U^{n+1})
// ---------------------------------------------------------------------------
// per-cell CFL candidate (R25): CFL-free min over the active axes of min(h_a / (|U_a| + c), h_a^2 / (3 nu));
// ok = false if the state is not positive (the candidate is then 1e300)
template <int DIM>
__device__ __forceinline__ double cfl_candidate(const double* q, int i, int j, int k, bool& ok) {
  const double ir = 1.0 / q[0];
  const double u[3] = {q[1] * ir, q[2] * ir, q[3] * ir};
  const double p = (c_geo.gamma - 1.0) * (q[4] - 0.5 * q[0] * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]));
  ok = (q[0] > 0.0) && (p > 0.0);
  double cand = 1e300;
  if (ok) {
    const double c = sqrt(c_geo.gamma * p * ir);
    double mu_T = c_geo.mu;
    if (c_geo.suth > 0.0) {  // Sutherland law, T = p / rho
      const double Tc = p * ir;
      mu_T = c_geo.mu * (1.0 + c_geo.suth) * Tc * sqrt(Tc) / (Tc + c_geo.suth);
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const double ha = c_geo.stretched ? cw(a, a == 0 ? i : (a == 1 ? j : k)) : c_geo.h[a];
      double d = ha / (fabs(u[a]) + c);
      if (c_geo.mu > 0.0) d = fmin(d, ha * ha / (3.0 * mu_T * ir));  // nu = mu(T) / rho (R25)
      cand = fmin(cand, d);
    }
  }
  return cand;
}

// block min of a candidate (all threads of the block call it), atomicMin of the bit pattern by thread 0
// (order-preserving for positive doubles; NaN bits are above every finite positive value)
__device__ __forceinline__ void block_min_atomic(double cand, unsigned long long* dst) {
  __shared__ double red[32];
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) cand = fmin(cand, __shfl_xor_sync(0xffffffffu, cand, m));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = cand;
  __syncthreads();
  if (w == 0) {
    cand = l < (int)(blockDim.x >> 5) ? red[l] : 1e300;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) cand = fmin(cand, __shfl_xor_sync(0xffffffffu, cand, m));
    if (l == 0) atomicMin(dst, (unsigned long long)__double_as_longlong(cand));
  }
}

template <int DIM, bool COMPACT, int MODE, bool LINES = false>
__global__ void __launch_bounds__(256) k_update(const double* __restrict__ Uin, const double* __restrict__ fx,
                                                 const double* __restrict__ fy, const double* __restrict__ fz,
                                                 double* __restrict__ Uout, double* __restrict__ carry,
                                                 TimeState* __restrict__ ts, ErrState* __restrict__ err,
                                                 double* __restrict__ Lout, double* __restrict__ Lcarry,
                                                 int kc0, int kc1) {
  constexpr int NV = COMPACT ? 20 : 5;
  constexpr int NF = COMPACT ? (LINES ? 30 + 2 * (DIM == 3 ? 4 : (DIM == 2 ? 2 : 1)) * 10 : 30) : 10;
  // the final update of a step (MODE 1, 2) also forms the next step's CFL candidates (fused):
  // block min, atomicMin into ts->dtmin_bits; k_step_end turns the (global) min into dt
  constexpr bool DT = MODE != 0;
  if (__syncthreads_or(err->code != 0)) return;  // block-uniform (block reduction below)
  // cells of the planes [kc0, kc1) (a z-chunk, or all); face records of plane k at F[a] + k * NF * fpl
  // (the caller shifts chunk buffers)
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x + (long long)kc0 * c_geo.plane;
  const long long nc = (long long)kc1 * c_geo.plane;
  double cand = 1e300;
  if (t < nc) {
  const int i = (int)(t % c_geo.n[0]);
  const int j = (int)((t / c_geo.n[0]) % c_geo.n[1]);
  const int k = (int)(t / c_geo.plane);
  const double dt = ts->dt;
  double L[5] = {0, 0, 0, 0, 0}, Lt[5] = {0, 0, 0, 0, 0};
  double Gn[3][5], Gt[3][5];
  const double* F[3] = {fx, fy, fz};
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int fn0 = c_geo.fn[a][0], fn1 = c_geo.fn[a][1];
    const long long fpl = (long long)fn0 * fn1;
    const int hi_i = i + (a == 0), hi_j = j + (a == 1), hi_k = k + (a == 2);
    // periodic axes wrap the high face; bounded axes have n+1 faces
    const int wi = c_geo.bounded[0] ? hi_i : wrapi(hi_i, c_geo.n[0]);
    const int wj = c_geo.bounded[1] ? hi_j : wrapi(hi_j, c_geo.n[1]);
    const int wk = c_geo.bounded[2] ? hi_k : wrapi(hi_k, c_geo.n[2]);
    const long long lo = (long long)k * NF * fpl + (long long)j * fn0 + i;
    const long long hi = (long long)wk * NF * fpl + (long long)wj * fn0 + wi;
    // own width (box cells: equal face areas on both sides, R37)
    const double ih = c_geo.stretched ? icw(a, a == 0 ? i : (a == 1 ? j : k)) : c_geo.ih[a];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      L[v] += (__ldg(F[a] + lo + v * fpl) - __ldg(F[a] + hi + v * fpl)) * ih;
      Lt[v] += (__ldg(F[a] + lo + (5 + v) * fpl) - __ldg(F[a] + hi + (5 + v) * fpl)) * ih;
      if (COMPACT) {
        // own side: left-side value at i+1/2, right-side value at i-1/2 (R24)
        Gn[a][v] = (__ldg(F[a] + hi + (10 + v) * fpl) - __ldg(F[a] + lo + (20 + v) * fpl)) * ih;
        Gt[a][v] = (__ldg(F[a] + hi + (15 + v) * fpl) - __ldg(F[a] + lo + (25 + v) * fpl)) * ih;
      }
    }
  }
  double Qo[5];
  if (MODE == 0) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double q = __ldg(Uin + sidx(NV, v, i, j, k));
      Qo[v] = q + 0.5 * dt * L[v] + 0.125 * dt * dt * Lt[v];
      carry[sidx(NV, v, i, j, k)] = q + dt * L[v] + (dt * dt / 6.0) * Lt[v];
      Uout[sidx(NV, v, i, j, k)] = Qo[v];
    }
    if (COMPACT) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          const double gn = a < DIM ? Gn[a][v] : 0.0, gt = a < DIM ? Gt[a][v] : 0.0;
          Uout[sidx(NV, 5 + a * 5 + v, i, j, k)] = gn + 0.5 * dt * gt;
          carry[sidx(NV, 5 + a * 5 + v, i, j, k)] = gn;
        }
    }
  } else if (MODE == 1) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      Qo[v] = __ldg(carry + sidx(NV, v, i, j, k)) + (dt * dt / 3.0) * Lt[v];
      Uout[sidx(NV, v, i, j, k)] = Qo[v];
    }
    if (COMPACT) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          const double gt = a < DIM ? Gt[a][v] : 0.0;
          Uout[sidx(NV, 5 + a * 5 + v, i, j, k)] = __ldg(carry + sidx(NV, 5 + a * 5 + v, i, j, k)) + dt * gt;
        }
    }
  } else {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      Qo[v] = __ldg(Uin + sidx(NV, v, i, j, k)) + dt * L[v] + 0.5 * dt * dt * Lt[v];
      Uout[sidx(NV, v, i, j, k)] = Qo[v];
    }
    if (COMPACT) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          const double gn = a < DIM ? Gn[a][v] : 0.0, gt = a < DIM ? Gt[a][v] : 0.0;
          Uout[sidx(NV, 5 + a * 5 + v, i, j, k)] = gn + dt * gt;
        }
    }
  }
  if (COMPACT && LINES) {
    // line-averaged derivatives: per axis a and line g, the own-side relaxed values at
    // Gauss point g of the faces i+1/2 (left side) and i-1/2 (right side), with the gradients'
    // two-stage rule (R24); layout [z][l*5+v][y][x]
    constexpr int NGL = DIM == 3 ? 4 : (DIM == 2 ? 2 : 1);
    constexpr int NLF = 5 * DIM * NGL;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int fn0 = c_geo.fn[a][0], fn1 = c_geo.fn[a][1];
      const long long fpl = (long long)fn0 * fn1;
      const int wi = c_geo.bounded[0] ? i + (a == 0) : wrapi(i + (a == 0), c_geo.n[0]);
      const int wj = c_geo.bounded[1] ? j + (a == 1) : wrapi(j + (a == 1), c_geo.n[1]);
      const int wk = c_geo.bounded[2] ? k + (a == 2) : wrapi(k + (a == 2), c_geo.n[2]);
      const double* flo = F[a] + (long long)k * NF * fpl + (long long)j * fn0 + i;
      const double* fhi = F[a] + (long long)wk * NF * fpl + (long long)wj * fn0 + wi;
      const double ih = c_geo.stretched ? icw(a, a == 0 ? i : (a == 1 ? j : k)) : c_geo.ih[a];  // own width (R37)
#pragma unroll
      for (int g = 0; g < NGL; ++g)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          const double ln = (__ldg(fhi + (30 + g * 10 + v) * fpl) - __ldg(flo + (30 + (NGL + g) * 10 + v) * fpl)) * ih;
          const double lt =
              (__ldg(fhi + (35 + g * 10 + v) * fpl) - __ldg(flo + (35 + (NGL + g) * 10 + v) * fpl)) * ih;
          const long long o = sidx(NLF, (a * NGL + g) * 5 + v, i, j, k);
          if (MODE == 0) {
            Lout[o] = ln + 0.5 * dt * lt;
            Lcarry[o] = ln;
          } else if (MODE == 1) {
            Lout[o] = Lcarry[o] + dt * lt;
          } else {
            Lout[o] = ln + dt * lt;
          }
        }
    }
  }
  // positivity of the updated state (R30)
  const double ke = 0.5 * (Qo[1] * Qo[1] + Qo[2] * Qo[2] + Qo[3] * Qo[3]) / Qo[0];
  const double p = (c_geo.gamma - 1.0) * (Qo[4] - ke);
  if (!(Qo[0] > 0.0) || !(p > 0.0)) flag_error(err, 3, 2, MODE == 0 ? 1 : 2, ts->steps, i, j, k);
  if (DT) {
    bool ok;
    cand = cfl_candidate<DIM>(Qo, i, j, k, ok);
    if (ok && !(cand == cand)) flag_error(err, 4, 2, 2, ts->steps, i, j, k);
  }
  }
  if (DT) block_min_atomic(cand, &ts->dtmin_bits);
}

// ---------------------------------------------------------------------------
// K4: CFL time step (R25): per-cell candidate, warp-shuffle min, block min, atomicMin on the
// bit pattern (order-preserving for positive doubles); NaN -> numerical error
// ---------------------------------------------------------------------------
template <int DIM>
__global__ void __launch_bounds__(256) k_dt(const double* __restrict__ U, int NV, TimeState* __restrict__ ts,
                                             ErrState* __restrict__ err) {
  if (__syncthreads_or(err->code != 0)) return;  // block-uniform (block reduction below)
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nc = (long long)c_geo.n[0] * c_geo.n[1] * c_geo.n[2];
  double cand = 1e300;
  if (t < nc) {
    const int i = (int)(t % c_geo.n[0]);
    const int j = (int)((t / c_geo.n[0]) % c_geo.n[1]);
    const int k = (int)(t / c_geo.plane);
    double q[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) q[v] = __ldg(U + sidx(NV, v, i, j, k));
    bool ok;
    cand = cfl_candidate<DIM>(q, i, j, k, ok);
    if (!ok)
      flag_error(err, 3, 3, 0, ts->steps, i, j, k);
    else if (!(cand == cand))
      flag_error(err, 4, 3, 0, ts->steps, i, j, k);
  }
  block_min_atomic(cand, &ts->dtmin_bits);
}

// dt of the first step of a cgks_step call from the k_dt min (rank-reduced; poison as in k_step_end)
static __global__ void k_dt_finalize(TimeState* ts, ErrState* err) {
  if (err->code) return;
  if (ts->dtmin_bits < 16ull) {
    flag_error(err, (int)ts->dtmin_bits, 4, 0, ts->steps, -1, -1, -1);
    return;
  }
  const double m = __longlong_as_double((long long)ts->dtmin_bits);
  const double dt = c_geo.fixed_dt > 0.0 ? c_geo.fixed_dt : c_geo.cfl * m;
  ts->dt = dt;
  ts->idt = 1.0 / dt;
  ts->dtmin_bits = (unsigned long long)__double_as_longlong(1e300);
}

// end of a step: advance t and the step count, and turn the (rank-reduced) min of the final update's
// CFL candidates into the next dt.  A bit pattern below 16 is an error code posted by a failing rank
// (k_err_poison) through the allreduce-min: this rank then fails the same step with the same code
// (kernel 4 = peer), so that every rank stops at the same step with the same state.
static __global__ void k_step_end(TimeState* ts, ErrState* err) {
  if (err->code) return;
  const unsigned long long b = ts->dtmin_bits;
  if (b < 16ull) {
    flag_error(err, (int)b, 4, 2, ts->steps, -1, -1, -1);
    return;
  }
  ts->t += ts->dt;
  ts->steps += 1;
  const double m = __longlong_as_double((long long)b);
  const double dt = c_geo.fixed_dt > 0.0 ? c_geo.fixed_dt : c_geo.cfl * m;
  ts->dt = dt;
  ts->idt = 1.0 / dt;
  ts->dtmin_bits = (unsigned long long)__double_as_longlong(1e300);
}

// a failing rank posts its error code as its dt candidate bits (below every positive double) before the
// allreduce-min of the NCCL slab runs, so that every rank sees it (k_step_end, k_dt_finalize)
// (test_step >= 0: test hook of tests/test_gpu_nccl_self.py -- a peer rank's positivity failure in that step)
static __global__ void k_err_poison(TimeState* ts, const ErrState* err, long long test_step) {
  if (err->code) ts->dtmin_bits = (unsigned long long)err->code;
  else if (test_step >= 0 && ts->steps == test_step) ts->dtmin_bits = 3ull;
}

// user layout [f][z][y][x]  <->  internal [z][f][y][x]
static __global__ void k_pack(const double* __restrict__ src, double* __restrict__ dst, int NV, int f0, int nf) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nc = (long long)c_geo.n[0] * c_geo.n[1] * c_geo.n[2];
  if (t >= nc * nf) return;
  const int f = (int)(t / nc);
  const long long c = t % nc;
  const int k = (int)(c / c_geo.plane);
  const long long r = c % c_geo.plane + (long long)c_geo.yoff * c_geo.n[0];  // rows are contiguous behind the y ghosts
  dst[((long long)(k + c_geo.zoff) * NV + f0 + f) * c_geo.splane + r] = src ? src[t] : 0.0;
}

static __global__ void k_unpack(const double* __restrict__ src, double* __restrict__ dst, int NV, int f0, int nf) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nc = (long long)c_geo.n[0] * c_geo.n[1] * c_geo.n[2];
  if (t >= nc * nf) return;
  const int f = (int)(t / nc);
  const long long c = t % nc;
  const int k = (int)(c / c_geo.plane);
  const long long r = c % c_geo.plane + (long long)c_geo.yoff * c_geo.n[0];
  dst[t] = src[((long long)(k + c_geo.zoff) * NV + f0 + f) * c_geo.splane + r];
}

// ---------------------------------------------------------------------------
// Flow diagnostics (reading R35): quadrature of each cell's
// reconstruction at the 3-point Gauss-Legendre nodes per active axis.  One thread per (cell, node);
// per block: sums of 1/2 rho |U|^2, mu(T) |curl U|^2, 4/3 mu(T) (div U)^2, rho (times weight and cell
// volume) in a fixed shuffle / shared-memory order, written to part[block][4].
// wtab (CGKS-5th): [node][value, d/dxi_0, d/dxi_1, d/dxi_2][NB] basis weights in reference units.
// ---------------------------------------------------------------------------
template <int DIM>
struct DiagQuad {
  static constexpr int NP = DIM == 3 ? 27 : (DIM == 2 ? 9 : 3);
  static constexpr int BLOCK = 256;
};

template <int DIM, bool COMPACT>
__global__ void __launch_bounds__(256) k_diag(const double* __restrict__ U, const double* __restrict__ rec,
                                               const double* __restrict__ wtab, double* __restrict__ part) {
  constexpr int NP = DiagQuad<DIM>::NP;
  constexpr int NB = Sten<DIM>::NB;
  constexpr int NV = COMPACT ? 20 : 5;
  constexpr int NW = COMPACT ? NP * 4 * NB : 1;
  __shared__ double wt[NW];
  __shared__ double red[8][4];
  if (COMPACT)
    for (int q = threadIdx.x; q < NW; q += blockDim.x) wt[q] = wtab[q];
  __syncthreads();
  const long long nc = (long long)c_geo.n[0] * c_geo.n[1] * c_geo.n[2];
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long cell = t / NP;
  const int p = (int)(t % NP);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (cell < nc) {
    const int i = (int)(cell % c_geo.n[0]);
    const int j = (int)((cell / c_geo.n[0]) % c_geo.n[1]);
    const int k = (int)(cell / c_geo.plane);
    // Gauss-Legendre node of this thread (3 per active axis on [-1/2, 1/2]) and its weight
    const double gx[3] = {-0.38729833462074168852, 0.0, 0.38729833462074168852};  // sqrt(3/5)/2
    const double gw[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
    const int pi = p % 3, pj = (p / 3) % 3, pk = p / 9;
    const double xi[3] = {gx[pi], DIM >= 2 ? gx[pj] : 0.0, DIM >= 3 ? gx[pk] : 0.0};
    // cell widths (stretched meshes: the cell's own, R37)
    double hc[3] = {c_geo.h[0], c_geo.h[1], c_geo.h[2]}, ihc[3] = {c_geo.ih[0], c_geo.ih[1], c_geo.ih[2]};
    if (c_geo.stretched) {
      const int ci[3] = {i, j, k};
      for (int a = 0; a < DIM; ++a) {
        hc[a] = cw(a, ci[a]);
        ihc[a] = icw(a, ci[a]);
      }
    }
    const double w = gw[pi] * (DIM >= 2 ? gw[pj] : 1.0) * (DIM >= 3 ? gw[pk] : 1.0) * hc[0] * hc[1] * hc[2];
    double W[5], dW[3][5];
    if (COMPACT) {
      const double* cb = rec + cidx(NB * 5, 0, 0, i, j, k);
      const long long ep = c_geo.en[0];  // pair stride / 2
      const double* wv = wt + p * 4 * NB;
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        double val = __ldg(U + sidx(NV, v, i, j, k)), d0 = 0.0, d1 = 0.0, d2 = 0.0;
        for (int kk = 0; kk < NB; ++kk) {
          const double c = __ldg(cb + (long long)((kk >> 1) * 5 + v) * 2 * ep + (kk & 1));
          val = fma(c, wv[kk], val);
          d0 = fma(c, wv[NB + kk], d0);
          d1 = fma(c, wv[2 * NB + kk], d1);
          d2 = fma(c, wv[3 * NB + kk], d2);
        }
        W[v] = val;
        dW[0][v] = d0 * ihc[0];
        dW[1][v] = d1 * ihc[1];
        dW[2][v] = d2 * ihc[2];
      }
    } else {
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        W[v] = __ldg(U + sidx(NV, v, i, j, k));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double sl = __ldg(rec + eidx(15, a * 5 + v, i, j, k));  // limited slope, reference units
          W[v] = fma(sl, xi[a], W[v]);
          dW[a][v] = sl * ihc[a];
        }
      }
    }
    const double ir = 1.0 / W[0];
    double Uv[3], dU[3][3];  // dU[a][b] = d U_b / d x_a
#pragma unroll
    for (int b = 0; b < 3; ++b) Uv[b] = W[1 + b] * ir;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) dU[a][b] = (dW[a][1 + b] - Uv[b] * dW[a][0]) * ir;
    const double ke = 0.5 * W[0] * (Uv[0] * Uv[0] + Uv[1] * Uv[1] + Uv[2] * Uv[2]);
    const double pr = (c_geo.gamma - 1.0) * (W[4] - ke);
    double mu = c_geo.mu;
    if (c_geo.suth > 0.0) {  // Sutherland law
      const double T = pr * ir;
      mu = c_geo.mu * (1.0 + c_geo.suth) * T * sqrt(T) / (T + c_geo.suth);
    }
    const double o0 = dU[1][2] - dU[2][1], o1 = dU[2][0] - dU[0][2], o2 = dU[0][1] - dU[1][0];
    const double dv = dU[0][0] + dU[1][1] + dU[2][2];
    acc[0] = w * ke;
    acc[1] = w * mu * (o0 * o0 + o1 * o1 + o2 * o2);
    acc[2] = w * (4.0 / 3.0) * mu * dv * dv;
    acc[3] = w * W[0];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], m);
  const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
#pragma unroll
    for (int q = 0; q < 4; ++q) red[wp][q] = acc[q];
  __syncthreads();
  if (threadIdx.x < 4) {
    double sum = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) sum += red[q][threadIdx.x];
    part[(long long)blockIdx.x * 4 + threadIdx.x] = sum;
  }
}

// ---------------------------------------------------------------------------
// Q-criterion at each cell centroid (reading R35): Q = -1/2 sum_ab dU_b/dx_a
// dU_a/dx_b from the cell's reconstruction at xi = 0: the value is Q0 + sum_k a_k p_k(0) (wc = p_k(0)
// = -avg0_k), the derivative along a only sees the linear basis function e_a (coefficient index a).
// out: [nz][ny][nx] (x fastest), one thread per cell.
// ---------------------------------------------------------------------------
template <int DIM, bool COMPACT>
__global__ void __launch_bounds__(256) k_qcrit(const double* __restrict__ U, const double* __restrict__ rec,
                                                const double* __restrict__ wc, double* __restrict__ out) {
  constexpr int NB = Sten<DIM>::NB;
  constexpr int NV = COMPACT ? 20 : 5;
  const long long nc = (long long)c_geo.n[0] * c_geo.n[1] * c_geo.n[2];
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc) return;
  const int i = (int)(t % c_geo.n[0]);
  const int j = (int)((t / c_geo.n[0]) % c_geo.n[1]);
  const int k = (int)(t / c_geo.plane);
  double ihc[3] = {c_geo.ih[0], c_geo.ih[1], c_geo.ih[2]};
  if (c_geo.stretched) {
    const int ci[3] = {i, j, k};
    for (int a = 0; a < DIM; ++a) ihc[a] = icw(a, ci[a]);
  }
  double W[5], dW[3][5];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    W[v] = __ldg(U + sidx(NV, v, i, j, k));
#pragma unroll
    for (int a = 0; a < 3; ++a) dW[a][v] = 0.0;
    if (COMPACT) {
      for (int kk = 0; kk < NB; ++kk) W[v] = fma(__ldg(rec + cidx(NB * 5, kk, v, i, j, k)), wc[kk], W[v]);
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        static_assert(ReconGen<DIM>::expo(0, 0) == 1, "linear basis functions first");
        dW[a][v] = __ldg(rec + cidx(NB * 5, a, v, i, j, k)) * ihc[a];
      }
    } else {
#pragma unroll
      for (int a = 0; a < DIM; ++a) dW[a][v] = __ldg(rec + eidx(15, a * 5 + v, i, j, k)) * ihc[a];
    }
  }
  const double ir = 1.0 / W[0];
  double Uv[3], dU[3][3];
#pragma unroll
  for (int b = 0; b < 3; ++b) Uv[b] = W[1 + b] * ir;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) dU[a][b] = (dW[a][1 + b] - Uv[b] * dW[a][0]) * ir;
  double q = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) q -= 0.5 * dU[a][b] * dU[b][a];
  out[t] = q;
}

// line DOFs from the cell-averaged gradients (each line along a starts as dQ/dx_a), [z][l*5+v][y][x]
template <int DIM>
__global__ void k_lines_from_grad(const double* __restrict__ U, double* __restrict__ Lb) {
  constexpr int NGL = DIM == 3 ? 4 : (DIM == 2 ? 2 : 1);
  constexpr int NLF = 5 * DIM * NGL;
  const long long nc = (long long)c_geo.n[0] * c_geo.n[1] * c_geo.n[2];
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc) return;
  const int i = (int)(t % c_geo.n[0]);
  const int j = (int)((t / c_geo.n[0]) % c_geo.n[1]);
  const int k = (int)(t / c_geo.plane);
  for (int a = 0; a < DIM; ++a)
    for (int g = 0; g < NGL; ++g)
      for (int v = 0; v < 5; ++v)
        Lb[sidx(NLF, (a * NGL + g) * 5 + v, i, j, k)] = U[sidx(20, 5 + a * 5 + v, i, j, k)];
}

}  // namespace cgks
