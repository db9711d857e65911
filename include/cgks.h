/*
 * cgks.h -- C ABI of the B200 (sm_100a) FP64 hot path of the fifth-order compact
 * gas-kinetic scheme CGKS-5th and the second-order GKS-2nd (arXiv 2508.19911).
 *
 * One call of cgks_step advances the cell averages Q and (CGKS-5th) the
 * cell-averaged gradients grad Q by whole time steps:
 *   - compact reconstruction at cell interfaces,
 *   - the time-dependent gas-kinetic interface flux and interface values
 *     (P:93-129),
 *   - the simultaneous update of averages and gradients with the two-stage
 *     fourth-order S2O4 or the one-stage S1O2,
 *   - the CFL time step, a global min-reduction.
 * Readings of points the paper leaves open are numbered R1-R34 in DESIGN.md.
 *
 * Conventions for every entry point
 *   - Return value: CGKS_OK (0) or one of the CGKS_ERR_* codes below; no
 *     exceptions cross the ABI.  cgks_last_error() gives a message.
 *   - All calls are synchronous with respect to the host on return.
 *   - Array arguments may be host or device pointers (detected with
 *     cudaPointerGetAttributes); the library copies and never retains them;
 *     the caller owns them.
 *   - User layout (rank-local block, x fastest):
 *       Q     : double[5][nz][ny][nx]      (rho, rho U, rho V, rho W, rho E)
 *       gradQ : double[3][5][nz][ny][nx]   (physical d/dx, d/dy, d/dz of each Q)
 *   - A context is bound to one CUDA device (the current device at create) and
 *     one rank, and is not thread-safe.
 */
#ifndef CGKS_H
#define CGKS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (2/3/4 mirror the exit codes of SPEC S:646) */
enum {
  CGKS_OK = 0,
  CGKS_ERR_CONFIG = 2,     /* invalid sizes, gamma not in (1,5/3], mu<0, Pr<=0, bc/decomposition, CLS rank check */
  CGKS_ERR_POSITIVITY = 3, /* rho<=0 or p<=0 in a state or reconstructed value (R30); state = last completed step */
  CGKS_ERR_NUMERICAL = 4,  /* NaN / non-finite time step */
  CGKS_ERR_CUDA = 5,       /* CUDA runtime failure */
  CGKS_ERR_COMM = 6        /* inter-GPU exchange failure */
};

/* boundary kinds per axis side (R29) */
enum { CGKS_BC_PERIODIC = 0, CGKS_BC_INFLOW = 1, CGKS_BC_OUTFLOW = 2 };

/* scheme ids and time schemes */
enum { CGKS_GKS2 = 0, CGKS_CGKS5 = 1 };
enum { CGKS_TIME_DEFAULT = 0, CGKS_TIME_S1O2 = 1, CGKS_TIME_S2O4 = 2 };

typedef struct cgks_ctx cgks_ctx; /* opaque; owns all device memory */

typedef struct {
  int64_t n[3];              /* global cells per axis; active axes are the leading ones with n>1
                                (n[2]==1: 2-D run; n[1]==n[2]==1: 1-D run)                          */
  double lo[3], hi[3];       /* box; uniform spacing h[a] = (hi[a]-lo[a])/n[a]                      */
  int bc[3][2];              /* CGKS_BC_* per axis (low, high side)                                */
  double bc_state[3][2][5];  /* conservative state for CGKS_BC_INFLOW sides                        */
  int nproc[3];              /* ranks per axis (1,Py,Pz), rank = ry + Py rz: (1,1,P) = z-slabs, Py > 1 =
                                pencils (3-D) or y-slabs (2-D; Pz = 1).  {1,1,1} or zeros = one rank  */
  int rank;                  /* this process' rank in [0, nproc product)                           */
  const void* nccl_id;       /* 128-byte ncclUniqueId, or NULL when there is one rank              */
  void* stream;              /* cudaStream_t to run on, or NULL for a library-owned stream         */
  const double* nodes[3];    /* stretched tensor-product mesh (DESIGN R37):
                                per axis the n[a]+1 increasing node coordinates (host pointer, copied
                                at create; global mesh), or NULL for the uniform spacing from lo/hi   */
} cgks_grid;

typedef struct {
  int id;           /* CGKS_GKS2 or CGKS_CGKS5                                                     */
  int nonlinear;    /* 0 = linear (chi == 1 / phi == 1), 1 = GENO / Venkatakrishnan   */
  int time_scheme;  /* CGKS_TIME_*: default S2O4 for CGKS-5th, S1O2 for GKS-2nd (R22)  */
  double cfl;       /* CFL number of the time step (R25)                               */
  double fixed_dt;  /* > 0 overrides the CFL time step                                            */
  double tau_eps;   /* inviscid collision time epsilon, paper 0.05                        */
  double tau_C;     /* pressure-jump constant C, paper 10                          */
  double relax_C;   /* tau0 jump constant of the side-state relaxation (R23), 10       */
  double k_venkat;  /* Venkatakrishnan K (R11), 0.3                                               */
  double chi_c;     /* GENO chi constant (R8), 0.01                                               */
  double sutherland_S; /* viscosity law: 0 = constant mu (R19, default); S > 0 = Sutherland law       */
                       /* mu(T) = mu (1 + S) T^{3/2} / (T + S), T = p / rho, with mu the value at T = 1 */
                       /* (S = 0.4042); used in the collision time and the viscous dt bound */
  int lines;           /* CGKS-5th: 1 = line-averaged derivatives of the own cell as reconstruction data  */
                       /* (SURVEY 8(f) NEXT-1), carried as extra DOFs per cell;    */
                       /* 0 = the cell-averaged gradient (R1, default).                                  */
  double chi_scale;    /* GENO: zeta of R8 divided by chi_scale before chi = 1/(1 + zeta^4); 1 = R8 as    */
                       /* read (default); larger values keep the quartic at larger sub-stencil contrasts  */
                       /* (the paper defers chi to its references; DESIGN.md section 8 measures 1 / 4 / 8) */
} cgks_scheme;

/* Fill a cgks_scheme with the paper defaults for scheme id (CGKS_GKS2 / CGKS_CGKS5). */
void cgks_scheme_defaults(int id, cgks_scheme* s);

/*
 * Create a context.  gamma in (1, 5/3]; mu >= 0 is the constant dynamic viscosity
 * (mu == 0: inviscid collision time P:344); Pr > 0 the Prandtl number (R20).
 * Builds the CGKS-5th constrained-least-squares matrix (R1-R4) on the
 * host in long double and checks its rank (CGKS_ERR_CONFIG when deficient).
 * Allocates all device memory on the current device, which the context keeps: every later call
 * on it makes that device current for its duration (and restores the caller's), so contexts on
 * different GPUs can be used from one thread.  *out is NULL on failure.
 */
int cgks_create(const cgks_grid* grid, double gamma, double mu, double Pr, const cgks_scheme* scheme,
                cgks_ctx** out);

/* Offset and size of this rank's block in the global grid. */
int cgks_local_extent(const cgks_ctx* ctx, int64_t off[3], int64_t n[3]);

/* Pure host function (no CUDA): the z-slab decomposition used by cgks_create.  For a global
 * grid n and nproc = (1,1,P), rank r owns planes [off[2], off[2] + nloc[2]) with
 * nloc[2] = n[2]/P; nbr = (lower, upper) neighbour ranks (periodic in z).  Returns
 * CGKS_ERR_CONFIG for unsupported layouts (nproc[0|1] > 1, P not dividing n[2], bad rank). */
int cgks_decompose(const int64_t n[3], const int nproc[3], int rank, int64_t off[3], int64_t nloc[3], int nbr[2]);

/* Pure host function (no CUDA): the pencil / y-slab decomposition used by cgks_create (north_star: "slab/pencil
 * decomposition"; pencils (1,Py,Pz), 2-D grids split along y).  nproc = (1,Py,Pz), rank =
 * ry + Py rz owns rows [off[1], off[1] + n[1]/Py) and planes [off[2], off[2] + n[2]/Pz); nbr = (y lower, y upper,
 * z lower, z upper) neighbour ranks (periodic).  CGKS_ERR_CONFIG for nproc[0] > 1, indivisible extents, bad rank. */
int cgks_decompose_pencil(const int64_t n[3], const int nproc[3], int rank, int64_t off[3], int64_t nloc[3],
                          int nbr[4]);

/* Writes a fresh 128-byte ncclUniqueId into out128 (rank 0 creates it and broadcasts it to
 * the other ranks, e.g. with torch.distributed, before cgks_create).  Loads libnccl.so.2 at
 * run time (CGKS_NCCL_LIB overrides the name).  CGKS_ERR_COMM if NCCL is unavailable. */
int cgks_nccl_unique_id(void* out128);

/* Pencils and y-slabs (grid.nproc = (1,Py,Pz), Py > 1; y periodic, >= 4 rows and planes per rank): the state
 * also stores 2 ghost rows per side along y.  Every stage first exchanges the y halos of the rank's own planes
 * (2-row strips of every field, packed into dense staging by pitched device copies, ncclSend/ncclRecv with the
 * two y neighbours), then the z halos as for slabs -- whole planes including the fresh y ghost rows, so the
 * edge-neighbour (corner) ghosts of the compact stencil arrive without a third exchange.  The in-process
 * group copies the strips directly between the members' buffers.  A 2-D grid with grid.nccl_id and one rank
 * runs the y path with the rank as its own neighbour (as the z path on a 3-D grid).
 *
 * Multi-rank contexts (grid.nproc = (1,1,P), P > 1):
 *   - with grid.nccl_id set, each process owns one rank; cgks_step exchanges a 2-plane halo
 *     of all fields (and line DOFs) with the z neighbours (ncclSend/ncclRecv, one group per
 *     stage, on a second stream overlapped with the interior reconstruction; CGKS_NO_OVERLAP=1
 *     serialises it) and reduces dt with ncclAllReduce(min).  P = 1 with grid.nccl_id set runs
 *     the same slab path with the rank as its own neighbour (bitwise equal to the plain context);
 *   - with grid.nccl_id == NULL the P contexts of one process (same device) form an
 *     in-process decomposition advanced in lock-step by cgks_step_group (halo copies,
 *     shared time state); cgks_step refuses such contexts.
 * ctxs[r] must be rank r (0..n-1) of the same decomposition.  Results equal the undecomposed
 * run bit for bit (same per-cell arithmetic, same global dt). */
int cgks_step_group(cgks_ctx** ctxs, int n, int nsteps);

/* The context's decomposition as its communicator reports it: *rank and *nranks (for NCCL
 * contexts from ncclCommUserRank / ncclCommCount of the live communicator, else the create-time
 * values), *backend = 0 single context, 1 NCCL, 2 in-process group.  Host only; any pointer may be
 * NULL.  CGKS_ERR_COMM if the NCCL queries fail. */
int cgks_comm_info(const cgks_ctx* ctx, int* rank, int* nranks, int* backend);

/* Planes per z-chunk of the stage driver: 0 = each stage passes over the whole (slab) grid; C > 0 =
 * the stages pass over z-chunks of C planes with chunk-sized reconstruction and face buffers (chosen
 * at create when the whole-grid buffers do not fit in the free device memory, or forced by the
 * environment variable CGKS_CHUNK=C; same results bit for bit).  -1 for a NULL context. */
int cgks_z_chunk(const cgks_ctx* ctx);

/* Set the state (user layout, rank-local block).  gradQ may be NULL (zero gradients;
 * not recommended for CGKS-5th, R26; ignored by GKS-2nd).  Resets t and the step count. */
int cgks_set_state(cgks_ctx* ctx, const double* Q, const double* gradQ);

/* Line DOFs (scheme.lines = 1): set / get the line-averaged derivatives, user layout
 * L[nl][5][nz][ny][nx] with nl = 12 / 4 / 1 (3-D / 2-D / 1-D): line l = a * ngl + g runs along axis a
 * through the cell at the transverse Gauss point g = p * n2 + q of the faces (p: sign -, + along
 * (a+1)%3, q along (a+2)%3, active axes only; offsets +-h/(2 sqrt 3)), value (Q(end) - Q(start)) / h_a.
 * cgks_set_state initialises every line along a with dQ/dx_a; call cgks_set_lines after it to set
 * exact line data.  Rank-local block on decomposed contexts (their 2-plane z halos travel with the
 * state's, cgks_step_group / NCCL).  Host or device pointers; CGKS_ERR_CONFIG without line DOFs. */
int cgks_set_lines(cgks_ctx* ctx, const double* L);
int cgks_get_lines(const cgks_ctx* ctx, double* L);

/* Advance nsteps time steps (each: dt min-reduction, then one S2O4 or S1O2 step).
 * On CGKS_ERR_POSITIVITY / CGKS_ERR_NUMERICAL the state is the last completed step. */
int cgks_step(cgks_ctx* ctx, int nsteps);

/* Copy the state out (user layout).  gradQ may be NULL. */
int cgks_get_state(const cgks_ctx* ctx, double* Q, double* gradQ);

/* Asynchronous variants (pipelined host I/O): they enqueue and return.  set_state_async copies host
 * inputs on an input copy stream into a staging buffer and converts them on the compute stream;
 * get_state_async converts on the compute stream and copies out on an output copy stream; both
 * wait for the previous use of their staging buffer, so set_state_async(n+1) overlaps step(n) and
 * get_state_async(n) overlaps step(n+1).  Host buffers must stay valid and unmodified (inputs) or
 * unread (outputs) until cgks_sync; pinned host memory makes the copies truly asynchronous.
 * cgks_step_async defers its error check to cgks_sync, which waits for everything enqueued and
 * returns what cgks_step would have returned (the state is then the last completed step).  Every
 * synchronous call first performs cgks_sync.  The staging buffers (2 x 160 B per cell) are
 * allocated on first use; CGKS_ERR_CUDA if they do not fit. */
int cgks_set_state_async(cgks_ctx* ctx, const double* Q, const double* gradQ);
int cgks_step_async(cgks_ctx* ctx, int nsteps);
int cgks_get_state_async(const cgks_ctx* ctx, double* Q, double* gradQ);
int cgks_sync(cgks_ctx* ctx);

/* Simulated time, completed steps, and the last time step used. */
int cgks_get_time(const cgks_ctx* ctx, double* t, int64_t* steps, double* last_dt);

/* Flow diagnostics of the current state (DESIGN R35):
 *   out[0] = int 1/2 rho |U|^2 dV            (kinetic energy)
 *   out[1] = int mu(T) |curl U|^2 dV        (solenoidal / enstrophy dissipation)
 *   out[2] = int 4/3 mu(T) (div U)^2 dV     (dilatational dissipation)
 *   out[3] = int rho dV                      (mass)
 * over the domain, by 3-point Gauss-Legendre quadrature per active axis of every cell's own
 * reconstruction (CGKS-5th quartic with GENO when nonlinear; GKS-2nd limited linear), mu(T) by the
 * context's viscosity law.  Unnormalised: divide by rho0 U0^2 |Omega| for the paper's E_k and eps.
 * out: host array of 4 doubles, caller-owned.  Synchronous; does not change the state.  Reuses the
 * reconstruction buffer.  CGKS_ERR_CONFIG for decomposed contexts (nproc > 1) in this version;
 * CGKS_ERR_NUMERICAL if a result is not finite. */
int cgks_diagnostics(cgks_ctx* ctx, double out[4]);

/* Q-criterion Q = (|Omega|^2 - |S|^2)/2 = -1/2 sum_ab dU_b/dx_a dU_a/dx_b at every cell centroid,
 * from the cell's reconstruction of the current state (the paper's TGV
 * iso-surfaces; DESIGN R35).  out: ncell doubles [nz][ny][nx] (x fastest, rank-local), host
 * or device pointer, caller-owned.  Synchronous; reuses the reconstruction buffer; does not change
 * the state.  CGKS_ERR_CONFIG for decomposed contexts in this version. */
int cgks_qcriterion(cgks_ctx* ctx, double* out);

/* Message of the last error (includes cell (i,j,k) and stage for positivity failures). */
const char* cgks_last_error(const cgks_ctx* ctx);

/* Number of library kernel launches per time step (for launch accounting). */
int cgks_launches_per_step(const cgks_ctx* ctx);

/* Per-kernel timing: run nsteps steps with a CUDA event pair around every launch on the
 * library stream; fills up to max entries of names (64 chars each), total ms and launch
 * counts; *n_out = number of distinct kernels.  Intended for the roofline report. */
int cgks_profile(cgks_ctx* ctx, int nsteps, int max, char* names, double* total_ms, int64_t* launches,
                 int* n_out);

/* Algorithmic FP64 operation count of this context's formulation, per launch of each
 * kernel (names as in cgks_profile; up to max entries of 64 chars) and per cell-update
 * (one full time step of one cell).  Counting rules: + - * / = 1, fma = 2, sqrt and each
 * special function (exp, expm1, erfc, rsqrt) = 1; compile-time constant folding excluded.
 * The flux point count comes from running the device formulation with a counting type. */
int cgks_algorithmic_flops(const cgks_ctx* ctx, int max, char* names, double* flops_per_launch,
                           double* flops_per_cell_step, int* n_out);

/* FP64 FMA throughput probe: runs a DFMA-bound kernel on all SMs of the current device
 * and returns the achieved FP64 TFLOP/s (2 flops per FMA) and the kernel time in ms. */
int cgks_fp64_peak(double* tflops, double* ms);

/* Release all resources.  Safe on NULL. */
void cgks_destroy(cgks_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* CGKS_H */
