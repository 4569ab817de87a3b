// Internal declarations shared by the host runtime (kcg_host.cu) and the kernels (kcg_kernels.cu).
// Not part of the ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define KCG_KMAX 8
#define KCG_GMAX 8          // ranks sharing one face in row-slab mode
#define KCG_TX 64           // tile width (pixels) of the CG kernel
#define KCG_HALO 2          // single-pass recompute halo for a radius-1 stencil

namespace kcg {

// Compile-time tile height of the persistent kernel for K component planes per system.
// Tile geometry / threads per CTA of the CTA-tile CG kernel, per K (component planes per system).
// Each stage holds the r and p boxes (tile + 2-pixel halo) and, with x-TMA, the tile's x block.
#ifndef KCG_TY1
#define KCG_TY1 32          // tile rows, K = 1 (Sylvester columns)
#endif
#ifndef KCG_TY4
#define KCG_TY4 16          // tile rows, K = 4
#endif
#ifndef KCG_NT4
#define KCG_NT4 256         // threads, K = 4 (warps must divide the tile rows; 256: no spills)
#endif
#ifndef KCG_XTMA_MAXK
#define KCG_XTMA_MAXK 3     // x block TMA-staged with the boxes for K <= this (K=4: measured slower)
#endif
#ifndef KCG_TRACE
#define KCG_TRACE 0         // 1: record per-iteration phase timestamps (diagnostic builds only)
#endif
#define KCG_TRACE_ITERS 1024
#define KCG_TRACE_COLS 160  // [it][0..2] = CTA 0 start / after grid.sync / after reduction, [it][3+b] = CTA b tiles done
#ifndef KCG_SERP
#define KCG_SERP 1          // serpentine tile order across passes (L2 reuse when the state fits)
#endif
#ifndef KCG_RED_MAX
#define KCG_RED_MAX 4096    // redundant per-CTA reduction when active systems x tiles <= this
#endif
#ifndef KCG_DYN
#define KCG_DYN 1           // dynamic tile claiming after each CTA's first two tiles
#endif
#ifndef KCG_XPF
#define KCG_XPF 1           // prefetch the next tile's x block into L2 (TMA prefetch) when not staged
#endif
#ifndef KCG_ROWMAP
#define KCG_ROWMAP 1        // warp w owns tile rows w RPW .. w RPW + RPW - 1 (consecutive: shared up / down rows)
#endif
#ifndef KCG_PREC_SMEM_A
#define KCG_PREC_SMEM_A 0   // 1: PCG phase A reads the block-Jacobi inverses from shared memory (extra barrier)
#endif
#ifndef KCG_X2
#define KCG_X2 1            // update x every other pass (x += a_{q-1} p_{q-1} + a_q p_q): 40kN B/iter
#endif
#ifndef KCG_FUSEAB
#define KCG_FUSEAB 1        // tile kernel without a preconditioner: phases A and B fused (no barrier between)
#endif
// the fused tile phases (cg_fuse, after the tile geometry below): no preconditioner, the r_new box must
// fit next to the two stages (K <= 6), and K = 1 keeps its two CTAs per SM (the box would cost one)
#ifndef KCG_FUSE1
#define KCG_FUSE1 0         // also fuse K = 1 (then one CTA per SM: use with KCG_NT1 = 512, KCG_MINB1 = 1)
#endif

#ifndef KCG_MFENCE
#define KCG_MFENCE 0        // D2 row march: async-proxy fence before every stage refill (only WAR: not needed)
#endif
#ifndef KCG_XEARLY
#define KCG_XEARLY 0        // tile kernel, x from L2: rows of x requested before the phase-B barrier (1: row 0, 2: all)
#endif
#ifndef KCG_XMIX
#define KCG_XMIX 0          // 1 / 2: X2 with the x updates of tile class 1 (index / row parity) on the odd passes (measured slower)
#endif
// X2 schedule of the tile CG kernel: a tile of class (tile & 1) (KCG_XMIX; else class 0) updates x on
// the passes q >= 1 with (q & 1) == class, q >= 2 for class 0, so each pass carries half of the x
// traffic instead of every other pass carrying all of it.  After the last pass q = iters, a tile's
// pending alpha_q p_q is the one of a pass that was not its x pass (xfix_kernel).
// tile class: KCG_XMIX 1 = tile index parity, 2 = tile-row parity, 0 = class 0 everywhere
__host__ __device__ constexpr int cg_xclass(int ty, int tx, int tiles_x) {
  return KCG_XMIX == 1 ? ((ty * tiles_x + tx) & 1) : KCG_XMIX == 2 ? (ty & 1) : 0;
}
__host__ __device__ constexpr bool cg_xpass(int q, int cls) {
  return KCG_X2 ? (cls ? (q & 1) == 1 : (q >= 2 && (q & 1) == 0)) : q >= 1;
}
__host__ __device__ constexpr bool cg_xpending(int iters, int cls) {
  return KCG_X2 && iters > 0 && !cg_xpass(iters, cls);
}
#ifndef KCG_TY23
#define KCG_TY23 16         // tile rows, K = 2, 3 (two rows per warp; profiles/r02/ab_k23_tile_geometry.txt)
#endif
#ifndef KCG_NT23
#define KCG_NT23 256        // threads, K = 2, 3
#endif
__host__ __device__ constexpr int cg_tile_y(int K) { return K == 1 ? KCG_TY1 : (K <= 3 ? KCG_TY23 : (K == 4 ? KCG_TY4 : 8)); }
#ifndef KCG_NT1
#define KCG_NT1 256         // threads, K = 1
#endif
#ifndef KCG_MINB1
#define KCG_MINB1 2         // resident CTAs per SM, K = 1
#endif
__host__ __device__ constexpr int cg_threads(int K) { return K == 1 ? KCG_NT1 : (K <= 3 ? KCG_NT23 : (K == 4 ? KCG_NT4 : 256)); }
__host__ __device__ constexpr int cg_stages(int K) { return 2; }
#ifndef KCG_MINB4
#define KCG_MINB4 1         // resident CTAs per SM, K = 4
#endif
__host__ __device__ constexpr int cg_min_blocks(int K) { return K == 1 ? KCG_MINB1 : (K == 4 ? KCG_MINB4 : 1); }
// fused phases only with two or more rows per warp (one row per warp, k >= 5: the two recomputed
// neighbour rows triple the p_new work -- stress 2.66 vs 2.82 solves/s)
__host__ __device__ constexpr bool cg_fuse(int K, bool prec) {
  return KCG_FUSEAB && !prec && (K >= 2 || KCG_FUSE1) && K <= 6 && cg_tile_y(K) >= 2 * (cg_threads(K) / 32);
}
__host__ __device__ constexpr bool cg_xtma(int K) { return K <= KCG_XTMA_MAXK && K <= 6; }  // K>=7: smem
// Bytes of the x block staged with a tile.
__host__ __device__ constexpr int cg_xstage_bytes(int K) { return cg_xtma(K) ? K * cg_tile_y(K) * KCG_TX * 8 : 0; }
// Bytes of the preconditioner's u box (tile + 1-pixel ring, K planes, row pitch TX + 4).
__host__ __device__ constexpr int cg_ubox_bytes(int K) { return K * (cg_tile_y(K) + 2) * (KCG_TX + 2 * KCG_HALO) * 8; }
// Bytes of one pipeline stage (r and p boxes with halo, K planes, + x block).
__host__ __device__ constexpr int cg_stage_bytes(int K) {
  return 2 * K * (cg_tile_y(K) + 2 * KCG_HALO) * (KCG_TX + 2 * KCG_HALO) * 8 + cg_xstage_bytes(K);
}

// ---- D2 prior: the row-march CG kernel (kcg_march.cuh).  A GROUP of warps (m_kp(K) component
// planes per warp) marches a strip of m_out(K) output columns (32 lanes x m_cp(K) columns = the strip
// + a 4-column halo each side) down a segment of rows; rows of r, p, x, hits are TMA-staged one row per stage into a
// per-group ring of m_stages(K) stages; the planes meet only in the k x k mixing (shared rows).
#define KCG_MHALO 4
#define KCG_MCH 1           // rows per TMA stage
#define KCG_MPB 16          // rows per partial-sum block (fixed reduction order)
#define KCG_MSEGTAB 64      // per-pass segment plans for 1 .. 64 running systems (the last one: all n_sys)
// K = 4 (round 2): two face columns per lane (64-column boxes, 56 output columns: 12.5 % halo lanes
// instead of 25 %); without hits one plane per warp in 3 groups of 4 warps (fullsky-d2 63.1 vs 73.0 us per
// face-pass), with hits two planes per warp in 4 groups of 2 warps (the hits ring would spill the
// one-plane warp: paper workload 38.3 vs 45.0 ms) -- profiles/r02/ab_march_k4_columns_per_lane.txt.
// The geometry therefore depends on HITS (H) for K = 4; the strip width (m_cp) does not.
#ifndef KCG_MKP4
#define KCG_MKP4 1          // K = 4 without hits: component planes per warp
#endif
#ifndef KCG_MKP4H
#define KCG_MKP4H 2         // K = 4 with hits: component planes per warp
#endif
#ifndef KCG_MCP1
#define KCG_MCP1 2          // K = 1: face columns per lane (a 64-column box, 56 output columns)
#endif
#ifndef KCG_MCP4
#define KCG_MCP4 2          // K = 4: face columns per lane
#endif
__host__ __device__ constexpr int m_kp(int K, bool H) { return K == 4 ? (H ? KCG_MKP4H : KCG_MKP4) : 1; }  // planes per warp
__host__ __device__ constexpr int m_gw(int K, bool H) { return K / m_kp(K, H); }                           // warps per group
__host__ __device__ constexpr int m_cp(int K) { return K == 1 ? KCG_MCP1 : (K == 4 ? KCG_MCP4 : 1); }  // columns per lane
__host__ __device__ constexpr int m_out(int K) { return 32 * m_cp(K) - 2 * KCG_MHALO; }  // output columns
#ifndef KCG_MG4
#define KCG_MG4 4           // K = 4 (two planes per warp): groups per CTA
#endif
#ifndef KCG_MG4W
#define KCG_MG4W 3          // K = 4 (one plane per warp): groups per CTA
#endif
#ifndef KCG_MINT
#define KCG_MINT 0          // 1: interior work units (no face border in reach) run a step without border masks
#endif
#ifndef KCG_MG4Q
#define KCG_MG4Q 8          // K = 4 (all four planes in one warp, no group barrier): groups (= warps) per CTA
#endif
#ifndef KCG_MST4
#define KCG_MST4 4          // K = 4: TMA row stages per group (power of 2)
#endif
#ifndef KCG_MG1
#define KCG_MG1 12          // K = 1 (two columns per lane): groups per CTA
#endif
#ifndef KCG_MST1
#define KCG_MST1 4          // K = 1 (two columns per lane): TMA row stages per group (power of 2)
#endif
__host__ __device__ constexpr int m_groups(int K, bool H) {
  return K == 1 ? (m_cp(K) == 2 ? KCG_MG1 : 16)
                : (K == 2 ? 8 : (K == 3 ? 5 : (m_kp(K, H) == 1 ? (m_cp(K) == 2 ? KCG_MG4W : 4) : (m_kp(K, H) == 2 ? KCG_MG4 : KCG_MG4Q))));
}
__host__ __device__ constexpr int m_threads(int K, bool H) { return m_groups(K, H) * m_gw(K, H) * 32; }
__host__ __device__ constexpr int m_stages(int K, bool H) {  // (shared memory)
  return K == 4 && (m_kp(K, H) >= 2 || m_cp(K) == 2) ? KCG_MST4 : (m_cp(K) == 2 ? KCG_MST1 : 8);
}
__host__ __device__ constexpr int m_stage_doubles(int K) { return (3 * K + 1) * 32 * m_cp(K); }
// doubles of one group's shared memory: the stage ring + 3 exchange rings [4 rows][K][32 cp]
__host__ __device__ constexpr int m_group_doubles(int K, bool prec, bool H) {  // (u_new ring with block-Jacobi only)
  return m_stages(K, H) * m_stage_doubles(K) + (prec ? 3 : 2) * 4 * K * 32 * m_cp(K);
}
__host__ __device__ constexpr int m_strips(int side, int K) { return (side + m_out(K) - 1) / m_out(K); }
// rows per work unit (a multiple of KCG_MPB) minimising the estimated pass time
// ceil(units / groups) * (seg + 8 warm-up rows + ~4 rows of pipeline fill) for n_sys active systems;
// the host plans it for every possible number of running systems (CgArgs::seg_tab), the march
// kernel picks the plan of each pass
__host__ __device__ inline int m_seg_model(int side, int strips, int n_sys, int groups) {
  if (side <= KCG_MPB) return KCG_MPB;
  int best = side;
  long long bt = -1;
  for (int seg = KCG_MPB; seg < side + KCG_MPB; seg += KCG_MPB) {
    const long long units = (long long)n_sys * strips * ((side + seg - 1) / seg);
    const long long g = groups > 0 ? groups : 1;
    const long long t = (units + g - 1) / g * ((seg < side ? seg : side) + 2 * KCG_MHALO + 4);
    if (bt < 0 || t < bt) { bt = t; best = seg; }
  }
  return best;
}
__host__ __device__ constexpr int m_blocks(int side) { return (side + KCG_MPB - 1) / KCG_MPB; }
// partial slots per system: strips x 16-row blocks x warps of a group
__host__ __device__ constexpr int m_slots(int side, int K, bool H) { return m_strips(side, K) * m_blocks(side) * m_gw(K, H); }


// Per-system constant parameters of the operator  q_c = h sum_d M[c][d] p_d + tau_c (kappa2 p_c + (L p_c)).
// Kronecker route: one system per patch, K = k, M = A^T T A, tau = prior scales.
// Sylvester route: one system per (patch, column i), K = 1, M = [rho_i], tau = [1].
struct SysParams {
  double M[KCG_KMAX * KCG_KMAX];  // row-major K x K (compact)
  double tau[KCG_KMAX];
  double kappa2;
  double hits_plane;              // index of the hits plane (patch) as a double (exact)
  // pixel-block Jacobi (hits = 1): inverses of M + diag(Q0)_d diag(tau) for degree d = 2, 3, 4 and
  // d = 0 (the single pixel of a level-0 face), each row-major K x K, stored compactly one after the
  // other (Kinv[0][0 .. 4 K K)); slot of degree d: kinv_slot(d)
  double Kinv[4][KCG_KMAX * KCG_KMAX];
};

__host__ __device__ inline int kinv_slot(int deg) { return deg >= 2 ? deg - 2 : 3; }

// Per-system iteration state (kept redundantly in every CTA's shared memory).
enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXIT = 2, ST_BREAKDOWN = 3, ST_NONFINITE = 4 };
struct SysState {
  double bnorm2;   // ||b||^2
  double gamma;    // (r, r) of the current residual
  double alpha;    // step of the next pass
  double beta;     // p-update coefficient of the next pass
  double rel;      // last recursive ||r|| / ||b||
  int iters;       // completed iterations
  int status;
  int parity;      // which ping-pong buffer holds the current r, p
  int pad;
  double alpha_last;  // alpha used by the last completed pass (X2: its alpha p_new is pending in x
                      // when `iters` is odd -- added by the next x pass or by the fix-up kernel)
};

struct CgMaps {              // TMA descriptors of rbuf[0..1], pbuf[0..1] (box = {TX+4, TY+4, K})
  CUtensorMap r[2];
  CUtensorMap p[2];
  CUtensorMap x;             // the solution buffer, box = {TX, TY, K}; re-encoded per solve
  CUtensorMap h;             // D2 march kernel: the hits planes [P][side][side], box = {32, KCG_MCH, 1}
};

struct CgArgs {
  const SysParams* params;   // [n_sys]
  double* x;                 // user solution planes [n_sys*K][side][side]
  double* rbuf[2];           // internal ping-pong r planes, row pitch `pitch`
  double* pbuf[2];           // internal ping-pong p planes
  double* partials;          // [2][n_sys][tiles_per_sys][2]
  SysState* state_out;       // [n_sys]
  double* history;           // [history_cap]
  const double* hits;        // [P][side][side] or nullptr
  int history_cap;
  int side, pitch;
  int rows, row0, ghost;     // local slab rows, global face row of local row 0, ghost rows of r/p
                             // buffers above and below (row-slab mode; else side, 0, 0)
  int n_sys, tiles_x, tiles_y, tiles_per_sys;
  int max_iter;
  const double* bnorm2;      // warm start (reading R37): (||b - G x0||^2, ||b||^2) per system, else nullptr
  int x_tma;                 // 1: CgMaps::x describes `x` (TMA needs side >= 2): staged (K <= 3) or L2-prefetched
  int h_tma;                 // D2 march kernel: 1 = CgMaps::h describes the hits planes (side >= 2)
  int seg;                   // D2 march kernel: rows per work unit (a multiple of KCG_MPB); 0 = per pass from seg_tab
  unsigned short seg_tab[KCG_MSEGTAB];  // D2 march kernel, seg == 0: rows per unit with nact systems running
                             // = seg_tab[min(nact, KCG_MSEGTAB) - 1] (host-planned, kcg::m_seg_model)
  long long* trace;          // KCG_TRACE builds only: per-iteration %globaltimer stamps
  unsigned* sync;            // [2..3] tile-claim counters of the two pass parities (zeroed per launch)
  double tol2;
  // ---- row-slab mode (cg_slab_kernel only) ----
  int rank, nranks;          // this rank, ranks sharing every face (slab r holds rows [r rows, (r+1) rows))
  double* nb_r[2][2];        // [0 up / 1 down neighbour][buffer] its ghosted r buffers (nullptr: face end)
  double* nb_p[2][2];        // same for p
  double* slots[KCG_GMAX];   // every rank's cross-rank sums [2 parities][n_sys][nranks][NP]
  unsigned long long* flags[KCG_GMAX];  // every rank's flag array [nranks]
  unsigned long long* my_flags;          // == flags[rank]
  const double* my_slots;                // == slots[rank]
  unsigned* group;           // [0] barrier counter of this rank's CTA group (zeroed per launch)
  unsigned long long tag0;   // solve tag (solve number << 32); pass q (start pass 0) releases tag0 + q + 1
};

// One launch of the slab kernel: `nlocal` ranks (1 = one process per GPU; nranks = every rank
// emulated on one GPU in one cooperative launch), `ctas` CTAs per rank.
struct CgSlabLaunch {
  CgArgs a[KCG_GMAX];
  CgMaps m[KCG_GMAX];
  int nlocal, ctas;
};


// Small cross-rank operations of the slab runtime (by value: plain pointers valid in this process).
struct XrankPut {            // dst[g][rank * count + i] = src[i] for every rank g
  double* dst[KCG_GMAX];
  const double* src;
  int count, rank, nranks;
};
struct XrankSync {           // local ranks [rank0, rank0 + nlocal) meet every rank on `tag`
  unsigned long long* flags[KCG_GMAX];
  int nranks, rank0, nlocal;
  unsigned long long tag;
};
// Geometry of one rank's data: a face of side x side, `rows` local rows from global row `row0`,
// r/p buffers with row pitch `pitch` and `ghost` ghost rows above and below (0 without slabs).
struct SlabGeom {
  int side, rows, row0, pitch, ghost;
  int hits_ghost;            // ghost rows of the hits planes (= ghost, except for the dense rhs output)
  int nested;                // 1: the data maps Y are in HEALPix NESTED order inside the face (reading R1)
  int d2;                    // 1: prior Q0 = D^2 + kappa2 I (radius-2 operator)
};

// ---- textbook (HS) CG variant (kcg_hs.cuh; desc.cg_variant = KCG_CG_HS, reading R9)
#define KCG_HS_GRID_MAX 1024  // CTA partial rows per system in the workspace (>= the cooperative grid)
__host__ __device__ constexpr int hs_tile_y(int K) { return K <= 2 ? 16 : (K <= 4 ? 8 : 4); }
cudaError_t hs_kernel_config(int K, bool hits, bool prec, bool d2, int n_sys, int* max_grid, size_t* smem);
// q: a [n_sys K][side][pitch] scratch vector; part: [2][KCG_HS_GRID_MAX][n_sys][3] doubles
cudaError_t launch_cg_hs(int K, bool prec, bool d2, cudaStream_t s, const CgArgs& a, double* q, double* part,
                         int grid, size_t smem);
cudaError_t launch_hs_xfix(int K, cudaStream_t s, const SysState* st, const double* p0, const double* p1, double* x,
                           int n_sys, int side, int pitch);

// ---- small-problem regime: CG state resident in shared memory (kcg_res.cuh)
#define KCG_RES_CTA_MAX 1024  // CTA partial rows in the workspace [2][KCG_RES_CTA_MAX][3]
size_t res_smem(int K, int RS, int side, bool hits, bool prec, int n_sys);  // dynamic smem for RS-row strips
cudaError_t res_kernel_config(int K, bool hits, bool prec, size_t smem, int* blocks_per_sm);
// a.tiles_per_sys = strips per system (side / RS); grid = n_sys * strips; part: [2][grid][3] doubles
cudaError_t launch_cg_resident(int K, bool prec, cudaStream_t s, const CgArgs& a, double* part, int grid, size_t smem);

// ---- block-Lanczos Sylvester solver (Alg. SylvSolver)
#define KCG_LZ_GRID_MAX 512  // partial-sum rows per face in the workspace (>= the cooperative grid)
struct LzFace {              // per-face constants, host-computed at create (Lemma 2)
  double rho[KCG_KMAX];      // ascending eigenvalues of S^ = M P^{-1}
  double W[KCG_KMAX * KCG_KMAX];  // W[c*K + j]: eigenvector j (W^T P W = I); U = P W, U^{-1} = W^T
  double phi[KCG_KMAX];      // P = diag(phi)
  double kappa2;
};
struct LzState {             // per-face state, written by the face's reducer CTA
  int iters;                 // completed Lanczos steps i
  int status;                // ST_*
  double bnorm;              // ||B_0||_F
  double rel;                // sqrt(gamma_i) / ||B_0||_F (the paper's residual estimate)
};
struct LzArgs {
  const LzFace* prm;         // [P]
  const double* hits;        // [P][side][side] or nullptr (N_h = I)
  double* V;                 // block slots [nslots][P][K][side][pitch]: slot 0 = Y^ = Y T A P^{-1}
  double* Mx;                // solution M [P][K][side][side] (row-major pixels)
  double* part;              // per-CTA Gram partials [P][KCG_LZ_GRID_MAX][NPART]
  LzState* st;               // [P]
  double* Hs;                // H_i          [P][cap][K*K]
  double* Rs;                // B_0, B_2, .. [P][cap+1][K*K]  (Rs[a] normalises V_{a+1}: V_{a+1} Rs[a] = W_a)
  double* Ri;                // Rs^{-1}      [P][cap+1][K*K]
  double* Sinv;              // per shift j: Schur complement inverses of T_i + rho_j I  [P][cap][K][K*K]
  double* gv;                // per shift j: eliminated right-hand sides                 [P][cap][K][K]
  double* Zs;                // coefficients G_i of M = sum V_i G_i (Eq.(soln-darstellung)) [P][cap][K*K]
  int P, side, pitch, tiles_x, tiles_y, tps, cap, max_iter, store;
  double tol;
  long long* trace;          // KCG_TRACE builds: [pass][5 + CTA] %globaltimer stamps (else nullptr)
};
// V slot of block q: the HBM-resident basis (store) keeps every block; the paper's memory-lean
// two-pass mode rotates three slots after Y^.
__host__ __device__ inline int lz_slot(int store, int q) { return store ? q : (q == 0 ? 0 : 1 + (q - 1) % 3); }
__host__ __device__ constexpr int lz_tile_y(int K, bool d2) { return d2 ? 8 : (K <= 4 ? 16 : 8); }
__host__ __device__ constexpr int lz_npart(int K) {  // Gram partial per CTA and face
  return K <= 4 ? K * (2 * K + 1) : ((2 * K + 3) / 4) * ((2 * K + 3) / 4 + 1) / 2 * 16;
}

// ---------------------------------------------------------------- launchers (kcg_kernels.cu)
// All return cudaError_t of the launch.
cudaError_t launch_rhs(int K, cudaStream_t s, const double* Y, const double* E, const double* hits,
                       double* r0, double* p0, double* x, int P, int n, const SlabGeom& g);
cudaError_t launch_cg(int K, bool prec, bool d2, cudaStream_t s, const CgArgs& a, const CgMaps& m, int grid,
                      size_t smem);
cudaError_t cg_kernel_config(int K, bool hits, bool prec, bool slab, bool d2, int n_sys, int* max_grid,
                             size_t* smem);
cudaError_t launch_cg_slab(int K, bool prec, cudaStream_t s, const CgSlabLaunch& L, size_t smem);
cudaError_t launch_apply(int K, cudaStream_t s, const SysParams* params, const double* x, double* y,
                         const double* hits, int n_sys, const SlabGeom& g, const double* xg_top,
                         const double* xg_bot);
cudaError_t launch_resid(int K, cudaStream_t s, const SysParams* params, const double* x,
                         const double* Y, const double* E, const double* hits, double* partials,
                         double* out, int n_sys, int n, const SlabGeom& g, const double* xg_top,
                         const double* xg_bot);
cudaError_t launch_xfix(int K, int tile_y, cudaStream_t s, const SysState* st, const double* p0, const double* p1, double* x,
                        int n_sys, const SlabGeom& g);
cudaError_t launch_backtransform(int K, cudaStream_t s, const double* W, double* x, int P, size_t N);
cudaError_t launch_sub_pitched(cudaStream_t s, double* r, const double* v, size_t planes, int side, int pitch);
cudaError_t launch_ghost_fill(cudaStream_t s, const double* r0, const double* p0, double* up_r, double* up_p,
                              double* dn_r, double* dn_p, int planes, const SlabGeom& g);
cudaError_t launch_xghost(cudaStream_t s, const double* x, double* up_xg_bot, double* dn_xg_top, int planes,
                          const SlabGeom& g);
cudaError_t launch_put(cudaStream_t s, const XrankPut& P);
cudaError_t launch_xrank_sync(cudaStream_t s, const XrankSync& X);
// dst[plane][nest(x,y)] = src[plane][y side + x] (to_nested) or the inverse gather.
cudaError_t launch_permute(cudaStream_t s, const double* src, double* dst, size_t planes, int side, bool to_nested);
int apply_tiles_per_sys(int rows, int side, bool d2);
// Posterior variances (Hutchinson): z[p][c][pixel] = Rademacher(seed, probe, p, c, j) in the working
// row-major layout, j = the pixel's index in the user layout; var (=|+=) z * x, times scale.
cudaError_t launch_probe(cudaStream_t s, double* z, int P, int K, int side, bool nested, unsigned long long seed,
                         int probe);
// Alg. Kohler: rhs of column i (F^_i minus the Schur coupling, times N_h) and the column copy.
cudaError_t launch_kohler_rhs(int K, cudaStream_t s, const double* Y, const double* E, const double* Rk,
                              const double* Xh, const double* hits, double* r0, double* p0, double* x, int P, int n,
                              int i, int side, int pitch, bool nested);
cudaError_t launch_column_copy(cudaStream_t s, const double* src, double* dst, int P, int K, int i, size_t N);
// bad += number of entries of v[0..n) that are not finite and > 0 (hits validation at create)
cudaError_t launch_count_nonpositive(cudaStream_t s, const double* v, size_t n, unsigned* bad);
cudaError_t launch_var_accum(cudaStream_t s, const double* z, const double* x, double* var, size_t n, bool first,
                             double scale);
// block-Lanczos (kcg_lanczos_*.cu): one cooperative launch runs the Lanczos passes, the residual
// estimate, the coefficients and (two-pass mode) the replay that assembles M; store mode follows it
// with lz_assemble.
cudaError_t lz_kernel_config(int K, bool hits, bool d2, int* max_grid, size_t* smem);
cudaError_t launch_lanczos(int K, bool hits, bool d2, cudaStream_t s, const LzArgs& a, const CUtensorMap& vmap,
                           int grid, size_t smem);
__host__ __device__ constexpr int lz_halo(bool d2) { return d2 ? 4 : 2; }
cudaError_t launch_lz_assemble(int K, cudaStream_t s, const LzArgs& a);
template <int K>
struct LzEntry {  // defined in kcg_lanczos.cuh, instantiated per K in kcg_lanczos_{a,b}.cu
  static cudaError_t config(bool hits, bool d2, int* max_grid, size_t* smem);
  static cudaError_t launch(bool hits, bool d2, cudaStream_t s, const LzArgs& a, const CUtensorMap& vmap, int grid,
                            size_t smem);
  static cudaError_t assemble(cudaStream_t s, const LzArgs& a);
};

}  // namespace kcg
