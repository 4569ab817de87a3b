/*
 * kroncg.h -- C ABI of the B200 (sm_100a, fp64) Krylov solver for the Kronecker-structured
 * posterior-mean system of arxiv 2204.08057 (Bayesian CMB source separation).
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, "P:Lnnn" = line):
 *   (Q + B^T C B) mu = B^T C Y                                   Eq.(Axb), Eq.(mu*) P:L78-82
 *   B = A (x) I_N,  C = T (x) N_h,  Q = P (x) Q0
 * per HEALPix base face ("patch", App. A) of N = 4^level pixels on a 2^level x 2^level
 * grid with free boundary (reading R2).  In matrix form, with X = reshape(mu, N, k):
 *   G vec(X) = vec( N_h X M + Q0 X P ),   M = A^T T A,   P = diag(prior_scale),
 *   b        = vec( N_h Y T A ),
 *   Q0 = kappa2 I + L  (KCG_PRIOR_LAPLACIAN; BASELINE configs, reading R3/R24) or
 *   Q0 = D^2 + kappa2 I (KCG_PRIOR_D2; the paper's phi D^2),
 *   L  = graph Laplacian of the 4-neighbour face grid = -D of P:L100-106.
 *
 * Routes:
 *   kron_cg_solve    -- CG applied directly to G (Sec. 3.2), single-pass variant.
 *   sylvester_solve  -- Sylvester reformulation (Sec. 3.3), small factor diagonalised
 *                       once (Lemma 2): (Q0 + rho_i N_h) xt_i = ft_i, Ft = F W,
 *                       X = Xt W^T, all k shifted systems of all patches in ONE batched launch.
 *
 * Conventions (all entry points):
 *   - "_dev" pointers are CUDA device pointers, "_host" pointers are host memory.  Every buffer,
 *     including the workspace, is owned by the caller; the library never allocates device memory.
 *   - Layouts are C-contiguous, fp64:
 *       A_host            [P][n][k]   (A[p][f][c] = mixing of component c into map f)
 *       noise_prec_host   [P][n]      (T = 1/sigma^2, > 0)
 *       prior_scale_host  [P][k]      (paper phi_l = config tau_i, > 0)
 *       kappa2_host       [P]         (>= 0; kappa2 = 0 with hits = 1 still gives SPD G as M SPD)
 *       hits_dev          [P][side][side] (finite, > 0: checked on the device at create ->
 *                         KCG_E_ARG) or NULL for all ones; row slabs: see kcg_slab below
 *       Y                 [P][n][side][side]   row-major pixels idx = y*side + x (reading R1)
 *       mu / x / y        [P][k][side][side]
 *   - Calls are stream-ordered on the stream given at create and BLOCKING: they return after the
 *     report is on the host.  One solve at a time per context (not thread-safe).
 *   - x0 = 0; a system stops after the first iteration j with ||r_j||_2 <= tol ||b||_2 on the
 *     recursively updated residual (reading R8); iterations = number of x-updates.
 *     ||b|| = 0 gives mu = 0 after 0 iterations.  Y is never modified.
 *   - Errors: KCG_E_ARG (null pointer, tol <= 0, max_iter < 0, non-positive T/phi/hits,
 *     kappa2 < 0, non-finite scalars), KCG_E_SHAPE / KCG_E_CONFIG (descriptor out of range,
 *     workspace too small, unsupported combination), KCG_NOT_CONVERGED (max_iter reached: mu
 *     holds the last iterate; not fatal), KCG_E_BREAKDOWN (p^T G p <= 0 -- G not SPD),
 *     KCG_E_NONFINITE (NaN/Inf met during the iteration), KCG_E_CUDA (a CUDA call failed;
 *     kcg_last_error() has the text).
 */
#ifndef KRONCG_H
#define KRONCG_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define KCG_API __attribute__((visibility("default")))
#else
#define KCG_API
#endif

typedef struct kcg_ctx kcg_ctx;

typedef enum {
  KCG_OK = 0,
  KCG_NOT_CONVERGED = 1,
  KCG_E_ARG = 2,
  KCG_E_SHAPE = 3,
  KCG_E_CONFIG = 4,
  KCG_E_NONFINITE = 5,
  KCG_E_BREAKDOWN = 6,
  KCG_E_CUDA = 7,
  /* 8 is unassigned: the row-slab exchange uses peer memory, not NCCL (reading R35) */
  KCG_E_STATE = 9
} kcg_status;

enum { KCG_PRIOR_LAPLACIAN = 0, KCG_PRIOR_D2 = 1 };
enum { KCG_LAYOUT_ROW_MAJOR = 0, KCG_LAYOUT_NESTED = 1 };
enum { KCG_PRECOND_NONE = 0, KCG_PRECOND_BLOCK_JACOBI = 1 };
/* CG variant ("two variants of the conjugate gradient approach", reading R9): the
 * single-pass Chronopoulos-Gear form with recomputation (default: one grid-wide reduction and
 * 48 K N bytes per iteration) or the textbook Hestenes-Stiefel form of Alg. CG (P:L225-241:
 * two reductions, 72 K N bytes per iteration).  Same iterates in exact arithmetic.             */
enum { KCG_CG_SINGLE_PASS = 0, KCG_CG_HS = 1 };

/* Problem descriptor (fixed for the life of a context). */
typedef struct {
  int level;        /* face grid 2^level x 2^level, N = 4^level; 0 <= level <= 12 (App. A)  */
  int n_freq;       /* n, number of frequency maps; 1 <= n <= 64                                  */
  int n_comp;       /* k (paper m), number of sources; 1 <= k <= 8 and k <= n                      */
  int n_patches;    /* independent faces in this context (1..64)                                  */
  int prior;        /* KCG_PRIOR_LAPLACIAN: Q0 = kappa2 I + L (configs); KCG_PRIOR_D2: Q0 = D^2 +   */
                    /* kappa2 I (the paper's phi D^2; n_comp <= 4, no row slabs)        */
  int layout;       /* KCG_LAYOUT_ROW_MAJOR (y*side + x) or KCG_LAYOUT_NESTED (HEALPix NESTED      */
                    /* within the face; Y, mu, hits, apply/rhs arguments; no row slabs)            */
  int precond;      /* KCG_PRECOND_NONE (the paper's CG) or KCG_PRECOND_BLOCK_JACOBI (pixel */
                    /* k x k blocks of G, reading R10; n_comp <= 7; any level incl. 0)              */
  int host_staging; /* 1: workspace also holds Y / mu staging for the *_host entry points; 2: two   */
                    /* staging pairs (also kron_cg_solve_host_many, the pipelined entry point)     */
  int history_cap;  /* per-iteration max relative residual recorded on device (0 = off)            */
  int lanczos_cap;  /* block-Lanczos route (sylvester_lanczos_solve): 0 = not provisioned; else the   */
                    /* most Lanczos steps a solve may take (coefficients H_i, B_i, eliminations kept  */
                    /* on device: ~(5k^2 + k^3) * 8 bytes per step and patch); either prior (D2: k <= 4), */
                    /* no row slabs                                                                    */
  int lanczos_store;/* 1: keep the whole Lanczos basis V_1..V_cap in HBM (P*k*N*8*(lanczos_cap + 1)     */
                    /* bytes) and assemble M in one streaming pass; 0: the paper's memory-lean second  */
                    /* Lanczos pass, four block slots                                      */
  int cg_variant;   /* KCG_CG_SINGLE_PASS (0, default) or KCG_CG_HS; applies to the CG-based routes      */
                    /* (kron_cg_solve*, sylvester_solve*, kohler, solve_b, posterior_variance); KCG_CG_HS */
                    /* is not combined with row slabs (KCG_E_CONFIG)                                      */
} kcg_desc;

/* Solve report, filled on return (host memory). */
typedef struct {
  int status;              /* kcg_status of the solve                                        */
  int converged;           /* 1 if every system converged                                    */
  int iterations;          /* max over systems                                               */
  int n_systems;           /* patches (kron) or patches*k (sylvester)                        */
  int* iterations_per;     /* optional caller array [n_systems] (NULL = skip)                */
  double rel_residual;     /* max over systems of recursive ||r||/||b||                      */
  double rel_residual_true;/* max over patches of ||b - G mu||/||b||, recomputed at exit     */
  double wall_time_s;      /* device time of the whole solve (CUDA events, launching stream)  */
  double loop_time_s;      /* device time of the persistent CG kernel alone                  */
  long long system_iterations; /* sum over systems of iterations (+1 start pass each)        */
  double loop_bytes;       /* algorithmic HBM bytes of the CG kernel: per system-pass read +   */
                           /* write of r and p (32*K*N), plus x read + write (16*K*N) on the   */
                           /* passes that update x (every other pass: x += a_{q-1} p_{q-1} +   */
                           /* a_q p_q; a pending half-step is added after the loop)          */
  size_t peak_mem_bytes;   /* workspace bytes                                                */
  double* history;         /* optional caller array [history_cap] (NULL = skip)               */
  int history_len;
  long long kernel_launches; /* launches of the library's own kernels by this call (counted on */
                             /* the host at each launch; memsets and copies not included)     */
} kcg_report;

/* Bytes of device workspace needed for desc (256-byte aligned sub-buffers). 0 on bad desc. */
KCG_API size_t kron_cg_workspace_size(const kcg_desc* desc);

/* Validate, copy the small parameters to the device, diagonalise M = A^T T A against P
 * (Lemma 2: eigh(M, P), ascending rho, W^T P W = I, largest-|.| entry of each column positive)
 * and build the TMA descriptors.  stream: a cudaStream_t (NULL = legacy default stream).     */
KCG_API kcg_status kron_cg_create(const kcg_desc* desc, const double* A_host, const double* noise_prec_host,
                          const double* prior_scale_host, const double* kappa2_host,
                          const double* hits_dev, void* workspace_dev, size_t ws_bytes,
                          void* stream, kcg_ctx** out);

/* Kronecker route: CG on G (Sec. 3.2).  Y_dev [P][n][N] -> mu_dev [P][k][N].  Every device mu_dev
 * (all routes) must be 16-byte aligned (cudaMalloc / torch give 256): the kernels store the
 * solution as pixel pairs -- KCG_E_ARG otherwise.                                               */
KCG_API kcg_status kron_cg_solve(kcg_ctx* ctx, const double* Y_dev, double* mu_dev, double tol,
                         int max_iter, kcg_report* report);

/* Sylvester route (Sec. 3.3, Lemma 2): k shifted systems per patch, batched.  Per-column stop
 * ||rt_i|| <= tol ||ft_i|| (reading R15).  report->iterations_per is [P*k].                   */
KCG_API kcg_status sylvester_solve(kcg_ctx* ctx, const double* Y_dev, double* mu_dev, double tol,
                           int max_iter, kcg_report* report);

/* Block-Lanczos Sylvester solver -- the paper's Alg. SylvSolver: block Lanczos on
 * N_h^{-1} Q0 in the N_h inner product (Alg. Lanczos, Lemma 1) started from
 * Y^ = Y T A P^{-1} = V_1 B_0, Galerkin projection T_i Z + Z S^ = E_1 B_0 (Eq.(Sylv-small)) with
 * S^ = M P^{-1} = U R U^{-1} (Lemma 2), stop after the first step i with sqrt(gamma_i) <= tol ||B_0||_F
 * (gamma = the paper's residual estimate), Z from Eq.(soln-constr) P:L484-486 and
 * M = sum_j V_j G_j (Eq.(soln-darstellung)) written to mu_dev [P][k][N].  One context may run it
 * only if desc.lanczos_cap > 0 (KCG_E_CONFIG otherwise); max_iter is capped at lanczos_cap.
 * report->iterations_per is [P] (Lanczos steps per patch), report->rel_residual the max over
 * patches of sqrt(gamma)/||B_0||_F, report->rel_residual_true ||b - G mu||/||b|| as for CG.
 * A rank-deficient block (the Krylov space stops growing before convergence, e.g. 4^level < 2k)
 * gives KCG_E_BREAKDOWN; an exhausted space (W = V H to rounding) is an exact projection and
 * converges.                                                                                    */
KCG_API kcg_status sylvester_lanczos_solve(kcg_ctx* ctx, const double* Y_dev, double* mu_dev, double tol,
                                   int max_iter, kcg_report* report);
KCG_API kcg_status sylvester_lanczos_solve_host(kcg_ctx* ctx, const double* Y_host, double* mu_host, double tol,
                                        int max_iter, kcg_report* report);

/* Alg. Kohler (Kohler's sparse-dense Sylvester solver, the paper's comparison method):
 * real Schur factor S^ = A^T T A P^{-1} = W R W^T (canonical: ascending eigenvalues on R's diagonal,
 * W = orthonormalised Lemma-2 eigenvectors), F^ = Y^ W, then for i = 1..k one batched CG solve of
 * (Q0 + R_ii N_h) X^_i = N_h (F^_i - sum_{j<i} R_ji X^_j) over all patches, X = X^ W^T.  Per-column
 * stop ||r_i|| <= tol ||rhs_i||; report->iterations_per is [P*k] (patch-major).  No row slabs.     */
KCG_API kcg_status sylvester_kohler_solve(kcg_ctx* ctx, const double* Y_dev, double* mu_dev, double tol,
                                  int max_iter, kcg_report* report);

/* Many right-hand sides / parameter sweeps: G x = b for a GIVEN b_dev
 * [P][k][N] (user layout; each patch of the context is one system -- P copies of one parameter set
 * make P right-hand sides of one operator, P parameter sets one sweep), CG route, x0 = 0, stop on
 * ||r|| <= tol ||b||.  x_dev [P][k][N].  No row slabs (KCG_E_CONFIG).                          */
KCG_API kcg_status kron_cg_solve_b(kcg_ctx* ctx, const double* b_dev, double* x_dev, double tol, int max_iter,
                           kcg_report* report);

/* Warm start (reading R37; SURVEY 5 "warm start"): kron_cg_solve from a given initial guess
 * x0_dev [P][k][N] (user layout; may alias mu_dev) instead of 0 -- r_0 = b - G x_0 (one apply and
 * one residual pass before the CG kernel), stop on ||r_j|| <= tol ||b|| as usual (||r_0|| when
 * b = 0); a x_0 that already satisfies the rule returns after 0 iterations.  Kronecker route,
 * single-pass variant, no row slabs (KCG_E_CONFIG otherwise); the D2 prior, hits, NESTED and
 * block-Jacobi are supported.                                                                  */
KCG_API kcg_status kron_cg_solve_x0(kcg_ctx* ctx, const double* Y_dev, const double* x0_dev, double* mu_dev,
                                    double tol, int max_iter, kcg_report* report);

/* Posterior variances diag(Q^{-1}) = diag(G^{-1}) ("of most importance ... the main
 * diagonal") by Hutchinson's estimator with n_probes Rademacher probes:
 *   var = (1/s) sum_i z_i (.) G^{-1} z_i,   z_i[p][c][j] = +1 or -1 = sign bit of
 *   splitmix64(splitmix64(seed) + ((i P + p) k + c) N + j)   (j = the pixel's user-layout index)
 * -- an unbiased estimate; Var(var_j) = (1/s) sum_{l != j} (G^{-1})_{jl}^2.  Each probe is one batched
 * CG solve (kron_cg_solve_b) of all patches to tol.  var_dev [P][k][N]; scratch_dev 2 P k N doubles
 * (caller-owned).  report aggregates the probes (iterations = max, times and bytes summed;
 * iterations_per[p] = the most CG iterations patch p needed over the probes, n_systems = P).     */
KCG_API kcg_status posterior_variance(kcg_ctx* ctx, int n_probes, unsigned long long seed, double* var_dev,
                              double* scratch_dev, double tol, int max_iter, kcg_report* report);

/* Same as above with HOST buffers: copies Y in and mu out through the context's staging buffers
 * (desc.host_staging = 1), copies included in report->wall_time_s.                            */
KCG_API kcg_status kron_cg_solve_host(kcg_ctx* ctx, const double* Y_host, double* mu_host, double tol,
                              int max_iter, kcg_report* report);
KCG_API kcg_status sylvester_solve_host(kcg_ctx* ctx, const double* Y_host, double* mu_host, double tol,
                                int max_iter, kcg_report* report);

/* Pipelined host entry point for a stream of data sets (e.g. Monte-Carlo simulations of the maps):
 * nbatch Kronecker-route solves, batch i reading Y_host[i] [P][n][N] and writing mu_host[i]
 * [P][k][N] (pinned host memory for overlap; the pointers may repeat).  Needs desc.host_staging = 2
 * (two staging pairs in the workspace) and no row slabs (KCG_E_CONFIG).  The H2D copy of batch i+1
 * and the D2H copy of batch i-1 run on two copy streams while batch i is solved on the context's
 * stream; returns after the last copy.  reports: NULL or [nbatch] (each filled as by kron_cg_solve;
 * iterations_per / history pointers per report as usual).  Status: the worst over the batches;
 * an error stops the pipeline after the failing batch.                                           */
KCG_API kcg_status kron_cg_solve_host_many(kcg_ctx* ctx, int nbatch, const double* const* Y_host,
                                   double* const* mu_host, double tol, int max_iter, kcg_report* reports);

/* y = G x for all patches (Alg.MatvecQ + Alg.MatvecBCBT fused).  x_dev, y_dev
 * [P][k][N], must not alias.                                                                  */
KCG_API kcg_status kron_cg_apply(kcg_ctx* ctx, const double* x_dev, double* y_dev);

/* b = vec(N_h Y T A) for all patches (Eq.(mu*) right-hand side).  b_dev [P][k][N].            */
KCG_API kcg_status kron_cg_rhs(kcg_ctx* ctx, const double* Y_dev, double* b_dev);

/* The small-factor eigendecomposition computed at create: rho_host [P][k] ascending,
 * W_host [P][k][k] (W[p][c][i] = entry c of eigenvector i).                                    */
KCG_API kcg_status sylvester_factor(kcg_ctx* ctx, double* rho_host, double* W_host);

/* Text of the last error on ctx (never NULL). */
KCG_API const char* kcg_last_error(const kcg_ctx* ctx);
/* Name of a status code (static string). */
KCG_API const char* kcg_status_string(int status);

/* ---------------------------------------------------------------- row-slab decomposition
 * One face split into G row slabs: rank r holds the rows
 * [r side/G, (r+1) side/G) of every face of the context and exchanges two halo rows of r and p
 * with each neighbour every iteration -- stored by the CG kernel straight into the neighbour's
 * ghost rows (peer memory over NVLink, or the same GPU when emulated) -- plus one cross-rank sum
 * of the CG scalars per iteration (per-rank slots + system-scope flags, rank-ordered sum: every
 * rank computes identical scalars).  A context drives `nlocal` ranks: 1 (one process per GPU) or
 * all G (every rank emulated on this GPU in one cooperative launch, one CTA group per rank).
 * Layouts for a slab context: Y [nlocal][P][n][rows][side], mu [nlocal][P][k][rows][side],
 * hits [nlocal][P][rows + 4][side] -- GHOSTED: local rank j's plane p holds the face rows
 * [row0 - 2, row0 + rows + 2) of patch p (row0 = (rank0 + j) rows), i.e. its own rows plus the two
 * rows of the slab above and below, zeros beyond the face edge (kroncg.py ghost_rows() builds it
 * from a full face); rows = side / G.  Its own rows must be finite and > 0 (KCG_E_ARG otherwise).  All ranks must create their contexts before
 * any of them solves, and must issue the same sequence of solve / apply calls.              */
typedef struct {
  int nranks;            /* G: ranks sharing every face, 1..8; side % G == 0, side / G >= 4       */
  int rank0;             /* first (global) rank handled by this context                          */
  int nlocal;            /* 1 or nranks (emulation)                                               */
  void* peer_ws[8];      /* workspace of every rank [0, nranks), device addresses valid in this   */
                         /* process (own ranks' allocations; peers' through kcg_ipc_import); each */
                         /* kron_cg_workspace_size_slab bytes, 256-byte aligned, caller-owned     */
} kcg_slab;

/* Bytes of workspace per rank for a slab context of `nranks` ranks (0 on bad input). */
KCG_API size_t kron_cg_workspace_size_slab(const kcg_desc* desc, int nranks);

/* As kron_cg_create, for ranks [slab->rank0, slab->rank0 + slab->nlocal).  ws_bytes = the size of
 * each rank's workspace.  KCG_E_SHAPE if side is not divisible into >= 4-row slabs.             */
KCG_API kcg_status kron_cg_create_slab(const kcg_desc* desc, const kcg_slab* slab, const double* A_host,
                               const double* noise_prec_host, const double* prior_scale_host,
                               const double* kappa2_host, const double* hits_dev, size_t ws_bytes,
                               void* stream, kcg_ctx** out);

/* CUDA IPC for the slab peers: export the allocation holding dev_ptr (64-byte handle + the
 * pointer's offset inside it); import a peer's handle (returns the mapped pointer and the mapping
 * base to close with kcg_ipc_close after the context is destroyed).                            */
KCG_API kcg_status kcg_ipc_export(const void* dev_ptr, unsigned char handle[64], size_t* offset);
KCG_API kcg_status kcg_ipc_import(const unsigned char handle[64], size_t offset, void** dev_ptr, void** base);
KCG_API kcg_status kcg_ipc_close(void* base);

/* Release host-side state.  Does not free the caller's workspace. */
/* Row-slab plumbing check (diagnostic; no kernel waits on another rank, so several ranks may share
 * one GPU): kcg_slab_probe_put stores value + rank into slot [rank] of every rank's workspace
 * (peer stores through the kcg_ipc_import mappings) and synchronises the stream; after a host-side
 * barrier of all ranks, kcg_slab_probe_get copies this process's first local rank's nranks slots
 * to out_host (double[nranks]).  KCG_E_STATE on a non-slab context.  The slots are scratch of the
 * true-residual sum: call between solves only.                                                  */
KCG_API kcg_status kcg_slab_probe_put(kcg_ctx* ctx, double value);
KCG_API kcg_status kcg_slab_probe_get(kcg_ctx* ctx, double* out_host);

KCG_API void kron_cg_destroy(kcg_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* KRONCG_H */
