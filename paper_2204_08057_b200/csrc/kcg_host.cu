// Host runtime and C ABI of libkroncg (see include/kroncg.h for the contract).
//
// Responsibilities: descriptor/argument validation, workspace carving (caller-owned device memory,
// no allocation after create), the small dense algebra of setup step a1 (M = A^T T A, E = T A,
// Lemma 2's eigh(M, P) by a cyclic Jacobi eigensolver, pixel-block Jacobi inverses), TMA
// descriptor encoding, stream-ordered kernel launches, CUDA-event timing and the solve report.
//
// Row-slab mode: every face is split into G row slabs, one per rank;
// a context drives `nlocal` ranks -- 1 (one process per GPU, peers reached through IPC-mapped
// workspaces) or all G (every rank emulated on this GPU: one cooperative launch, one CTA group per
// rank).  Each rank's state lives in its own workspace (RankState); the non-slab context is the
// one-rank case with no ghost rows.
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>  // header-only (NVTX3): ranges cost nothing without a profiler attached

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/kroncg.h"
#include "kcg_internal.h"

using kcg::CgArgs;
using kcg::CgMaps;
using kcg::CgSlabLaunch;
using kcg::SlabGeom;
using kcg::SysParams;
using kcg::SysState;

namespace {

// NVTX range over a host-side scope (the entry points and the phases of a solve), for nsys / ncu
// timelines: "kcg:<route>" around a call, "kcg:rhs" / "kcg:cg" / "kcg:post" inside.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

const size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
const unsigned long long kPostTag = 1ull << 31;  // tags of the post-CG rendezvous of a solve

// Per-rank workspace carving.
struct Layout {
  size_t r0, r1, p0, p1, partials, state, history, sync, group, resid_partials, resid_out, params_kron, params_syl,
      E_kron, E_syl, W, Y_stage, mu_stage, trace, slots, flags, xg_top, xg_bot, rslots, x_rm, y_rm, hits_rm,
      lz_V, lz_part, lz_st, lz_H, lz_R, lz_Ri, lz_Sinv, lz_g, lz_Z, lz_prm, E_lz, params_koh, E_koh, R_koh, W_koh,
      hs_part, res_part, Y_stage2, mu_stage2, total;
  int lz_slots;
  size_t vec_doubles, partial_doubles;
};

// Work geometry of the single-pass CG kernels: CTA tiles (Laplacian prior) or, for the D2 prior, the
// row-march kernel's strips (x) and 16-row partial-sum blocks (y).
int tiles_x(int side, int K, bool d2 = false) { return d2 ? kcg::m_strips(side, K) : (side + KCG_TX - 1) / KCG_TX; }
int tiles_y(int rows, int K, bool d2 = false) {
  return d2 ? kcg::m_blocks(rows) : (rows + kcg::cg_tile_y(K) - 1) / kcg::cg_tile_y(K);
}

// D2 row-march kernel: rows per work unit, planned for every number of running systems (seg = 0 and
// the table: the kernel picks each pass's plan; entry KCG_MSEGTAB - 1 serves every nact >= KCG_MSEGTAB
// and is planned for all n_sys); KCG_MSEG (diagnostics) fixes it.
void march_seg(kcg::CgArgs* a, int side, int K, int n_sys, int groups) {
  a->seg = 0;
  if (const char* ev = std::getenv("KCG_MSEG"))
    a->seg = std::max(KCG_MPB, (std::atoi(ev) + KCG_MPB - 1) / KCG_MPB * KCG_MPB);
  const int strips = kcg::m_strips(side, K);
  for (int i = 0; i < KCG_MSEGTAB; ++i) {
    const int n = i + 1 < KCG_MSEGTAB ? std::min(i + 1, n_sys) : std::max(n_sys, KCG_MSEGTAB);
    a->seg_tab[i] = (unsigned short)kcg::m_seg_model(side, strips, n, groups);
  }
}

// One rank's layout: `rows` local rows (side / nranks), r/p buffers with `ghost` ghost rows.
Layout layout_of(const kcg_desc* d, int nranks) {
  Layout L{};
  const int side = 1 << d->level;
  const int rows = side / nranks;
  const int ghost = nranks > 1 ? KCG_HALO : 0;
  const int pitch = side < 2 ? 2 : side;  // TMA global strides must be multiples of 16 bytes
  const size_t N = (size_t)rows * side;
  const size_t P = d->n_patches, n = d->n_freq, k = d->n_comp;
  L.vec_doubles = P * k * (size_t)pitch * (rows + 2 * ghost);
  const bool d2 = d->prior == KCG_PRIOR_D2;
  const size_t tk = (size_t)tiles_x(side, (int)k, d2) * tiles_y(rows, (int)k, d2) * (d2 ? k : 1);  // (D2: <= per plane)
  const size_t ts = (size_t)tiles_x(side, 1, d2) * tiles_y(rows, 1, d2);
  L.partial_doubles = 2 * std::max(P * tk, P * k * ts) * 3;  // [2 parities][systems][tiles][<= 3]
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align_up(bytes); return o; };
  L.r0 = take(L.vec_doubles * 8);
  L.r1 = take(L.vec_doubles * 8);
  L.p0 = take(L.vec_doubles * 8);
  L.p1 = take(L.vec_doubles * 8);
  L.partials = take(L.partial_doubles * 8);
  L.state = take(P * k * sizeof(SysState));
  L.history = take((size_t)std::max(d->history_cap, 1) * 8);
  L.sync = take(4 * sizeof(unsigned));
  L.group = take(4 * sizeof(unsigned));
  L.resid_partials = take(P * (size_t)kcg::apply_tiles_per_sys(rows, side, d2) * 2 * 8);
  L.resid_out = take(P * 2 * 8);
  L.params_kron = take(P * sizeof(SysParams));
  L.params_syl = take(P * k * sizeof(SysParams));
  L.E_kron = take(P * n * k * 8);
  L.E_syl = take(P * n * k * 8);
  L.W = take(P * k * k * 8);
  L.params_koh = take(P * k * sizeof(SysParams));  // Alg. Kohler: [column][patch]
  L.E_koh = take(P * n * k * 8);
  L.R_koh = take(P * k * k * 8);
  L.W_koh = take(P * k * k * 8);
  L.trace = KCG_TRACE ? take((size_t)KCG_TRACE_ITERS * KCG_TRACE_COLS * 8) : 0;
  if (d->host_staging) {
    L.Y_stage = take(P * n * N * 8);
    L.mu_stage = take(P * k * N * 8);
  }
  if (d->host_staging == 2 && nranks == 1) {  // second staging pair: kron_cg_solve_host_many's pipeline
    L.Y_stage2 = take(P * n * N * 8);
    L.mu_stage2 = take(P * k * N * 8);
  }
  // cross-rank areas (written by peers)
  L.slots = take(2 * P * k * (size_t)nranks * 3 * 8);
  L.flags = take(KCG_GMAX * sizeof(unsigned long long));
  L.xg_top = take(P * k * (size_t)side * 8);
  L.xg_bot = take(P * k * (size_t)side * 8);
  L.rslots = take((size_t)nranks * P * 2 * 8);
  if (d->layout == KCG_LAYOUT_NESTED) {  // row-major working copies (the kernels' layout)
    L.x_rm = take(P * k * N * 8);
    L.y_rm = take(P * k * N * 8);
    L.hits_rm = take(P * N * 8);
  }
  if (d->lanczos_cap > 0 && nranks == 1) {  // block-Lanczos route (Alg. SylvSolver)
    const size_t cap = (size_t)d->lanczos_cap, kk = k * k;
    L.lz_slots = d->lanczos_store ? d->lanczos_cap + 1 : 4;
    L.lz_V = take((size_t)L.lz_slots * P * k * pitch * rows * 8);
    L.lz_part = take(P * (size_t)KCG_LZ_GRID_MAX * kcg::lz_npart((int)k) * 8);
    L.lz_st = take(P * sizeof(kcg::LzState));
    L.lz_H = take(P * cap * kk * 8);
    L.lz_R = take(P * (cap + 1) * kk * 8);
    L.lz_Ri = take(P * (cap + 1) * kk * 8);
    L.lz_Sinv = take(P * cap * k * kk * 8);
    L.lz_g = take(P * cap * k * k * 8);
    L.lz_Z = take(P * cap * kk * 8);
    L.lz_prm = take(P * sizeof(kcg::LzFace));
    L.E_lz = take(P * n * k * 8);
  }
  L.res_part = take(2 * (size_t)KCG_RES_CTA_MAX * 3 * 8);  // resident kernel: CTA partials [2][grid][3]
  if (d->cg_variant == KCG_CG_HS)  // CTA partial sums of the HS variant [2][grid][systems][3]
    L.hs_part = take(2 * (size_t)KCG_HS_GRID_MAX * P * k * 3 * 8);
  L.total = off;
  return L;
}

// One rank's device state (pointers into its workspace) and TMA descriptors.
struct RankState {
  int rank = 0, row0 = 0;
  char* ws = nullptr;
  double* r[2] = {nullptr, nullptr};
  double* p[2] = {nullptr, nullptr};
  double *partials = nullptr, *history = nullptr, *resid_partials = nullptr, *resid_out = nullptr;
  SysState* state = nullptr;
  unsigned *sync = nullptr, *group = nullptr;
  SysParams *params_kron = nullptr, *params_syl = nullptr, *params_koh = nullptr;
  double *E_koh = nullptr, *R_koh = nullptr, *W_koh = nullptr;
  double *E_kron = nullptr, *E_syl = nullptr, *W_dev = nullptr, *Y_stage = nullptr, *mu_stage = nullptr;
  double *Y_stage2 = nullptr, *mu_stage2 = nullptr;  // host_staging == 2
  long long* trace = nullptr;
  double *slots = nullptr, *xg_top = nullptr, *xg_bot = nullptr, *rslots = nullptr;
  double *x_rm = nullptr, *y_rm = nullptr, *hits_rm = nullptr;  // NESTED layout only
  double* hs_part = nullptr;                                      // KCG_CG_HS only
  double* res_part = nullptr;                                     // resident kernel partials
  unsigned long long* flags = nullptr;
  const double* hits = nullptr;
  CgMaps maps_kron, maps_syl;
  // block-Lanczos route
  double *lz_V = nullptr, *lz_part = nullptr, *lz_H = nullptr, *lz_R = nullptr, *lz_Ri = nullptr,
         *lz_Sinv = nullptr, *lz_g = nullptr, *lz_Z = nullptr, *E_lz = nullptr;
  kcg::LzState* lz_st = nullptr;
  kcg::LzFace* lz_prm = nullptr;
  CUtensorMap lz_map;
};

RankState carve(char* ws, const Layout& L, int rank, int rows, bool staging, bool nested) {
  RankState R;
  R.rank = rank;
  R.row0 = rank * rows;
  R.ws = ws;
  R.r[0] = reinterpret_cast<double*>(ws + L.r0);
  R.r[1] = reinterpret_cast<double*>(ws + L.r1);
  R.p[0] = reinterpret_cast<double*>(ws + L.p0);
  R.p[1] = reinterpret_cast<double*>(ws + L.p1);
  R.partials = reinterpret_cast<double*>(ws + L.partials);
  R.state = reinterpret_cast<SysState*>(ws + L.state);
  R.history = reinterpret_cast<double*>(ws + L.history);
  R.sync = reinterpret_cast<unsigned*>(ws + L.sync);
  R.group = reinterpret_cast<unsigned*>(ws + L.group);
  R.resid_partials = reinterpret_cast<double*>(ws + L.resid_partials);
  R.resid_out = reinterpret_cast<double*>(ws + L.resid_out);
  R.params_kron = reinterpret_cast<SysParams*>(ws + L.params_kron);
  R.params_syl = reinterpret_cast<SysParams*>(ws + L.params_syl);
  R.params_koh = reinterpret_cast<SysParams*>(ws + L.params_koh);
  R.E_koh = reinterpret_cast<double*>(ws + L.E_koh);
  R.R_koh = reinterpret_cast<double*>(ws + L.R_koh);
  R.W_koh = reinterpret_cast<double*>(ws + L.W_koh);
  R.E_kron = reinterpret_cast<double*>(ws + L.E_kron);
  R.E_syl = reinterpret_cast<double*>(ws + L.E_syl);
  R.W_dev = reinterpret_cast<double*>(ws + L.W);
  if (KCG_TRACE) R.trace = reinterpret_cast<long long*>(ws + L.trace);
  if (staging) {
    R.Y_stage = reinterpret_cast<double*>(ws + L.Y_stage);
    R.mu_stage = reinterpret_cast<double*>(ws + L.mu_stage);
  }
  if (L.Y_stage2) {
    R.Y_stage2 = reinterpret_cast<double*>(ws + L.Y_stage2);
    R.mu_stage2 = reinterpret_cast<double*>(ws + L.mu_stage2);
  }
  R.slots = reinterpret_cast<double*>(ws + L.slots);
  R.flags = reinterpret_cast<unsigned long long*>(ws + L.flags);
  R.xg_top = reinterpret_cast<double*>(ws + L.xg_top);
  R.xg_bot = reinterpret_cast<double*>(ws + L.xg_bot);
  R.rslots = reinterpret_cast<double*>(ws + L.rslots);
  if (L.lz_slots > 0) {
    R.lz_V = reinterpret_cast<double*>(ws + L.lz_V);
    R.lz_part = reinterpret_cast<double*>(ws + L.lz_part);
    R.lz_st = reinterpret_cast<kcg::LzState*>(ws + L.lz_st);
    R.lz_H = reinterpret_cast<double*>(ws + L.lz_H);
    R.lz_R = reinterpret_cast<double*>(ws + L.lz_R);
    R.lz_Ri = reinterpret_cast<double*>(ws + L.lz_Ri);
    R.lz_Sinv = reinterpret_cast<double*>(ws + L.lz_Sinv);
    R.lz_g = reinterpret_cast<double*>(ws + L.lz_g);
    R.lz_Z = reinterpret_cast<double*>(ws + L.lz_Z);
    R.lz_prm = reinterpret_cast<kcg::LzFace*>(ws + L.lz_prm);
    R.E_lz = reinterpret_cast<double*>(ws + L.E_lz);
  }
  if (L.hs_part) R.hs_part = reinterpret_cast<double*>(ws + L.hs_part);
  R.res_part = reinterpret_cast<double*>(ws + L.res_part);
  if (nested) {
    R.x_rm = reinterpret_cast<double*>(ws + L.x_rm);
    R.y_rm = reinterpret_cast<double*>(ws + L.y_rm);
    R.hits_rm = reinterpret_cast<double*>(ws + L.hits_rm);
  }
  return R;
}

}  // namespace

// Small-problem regime (kcg_res.cuh): the CG state of a route kept in shared memory, strips of
// side / nstrip rows, grid = systems * nstrip CTAs (off: the streaming persistent kernel).
struct ResPlan {
  bool on = false;
  int nstrip = 0, grid = 0;
  size_t smem = 0;
};

struct kcg_ctx {
  kcg_desc d;
  ResPlan res_kron, res_syl, res_koh;
  cudaStream_t stream = nullptr;
  int side = 0, pitch = 0, P = 0, n = 0, k = 0;
  int nranks = 1, rank0 = 0, nlocal = 1, rows = 0, ghost = 0;
  size_t N = 0;  // local pixels per plane (rows * side)
  size_t ws_bytes = 0, ws_need = 0;
  bool slab = false;
  std::vector<RankState> R;            // local ranks
  std::vector<char*> peer_ws;          // every rank's workspace (slab mode)
  Layout L;
  std::vector<double> rho, W;          // host copies [P][k], [P][k][k]
  int tiles_x_kron = 0, tiles_y_kron = 0, tiles_x_syl = 0, tiles_y_syl = 0;
  int grid_kron = 0, grid_syl = 0;     // CTAs (per rank in slab mode)
  size_t smem_kron = 0, smem_syl = 0;
  int grid_lz = 0, tiles_x_lz = 0, tiles_y_lz = 0;  // block-Lanczos kernel
  size_t smem_lz = 0;
  std::vector<kcg::LzState> lz_host;
  unsigned long long solve_id = 0;     // cross-rank operations so far (identical on every rank)
  long long nlaunch = 0;               // library kernel launches since the current entry point began
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // kron_cg_solve_host_many: copy streams and their events (created on first use)
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr}, ev_solved[2] = {nullptr, nullptr};
  std::vector<SysState> st_host;
  std::vector<double> resid_host;
  std::string err;
};

namespace {

bool desc_ok(const kcg_desc* d, std::string* why) {
  char buf[256];
  if (!d) { *why = "desc is NULL"; return false; }
  if (d->level < 0 || d->level > 12) { snprintf(buf, sizeof buf, "level %d outside [0,12]", d->level); *why = buf; return false; }
  if (d->n_freq < 1 || d->n_freq > 64) { *why = "n_freq outside [1,64]"; return false; }
  if (d->n_comp < 1 || d->n_comp > KCG_KMAX) { *why = "n_comp outside [1,8]"; return false; }
  if (d->n_comp > d->n_freq) { *why = "n_comp > n_freq (A cannot have full column rank)"; return false; }
  if (d->n_patches < 1 || d->n_patches > 64) { *why = "n_patches outside [1,64]"; return false; }
  if (d->history_cap < 0) { *why = "history_cap < 0"; return false; }
  if (d->host_staging < 0 || d->host_staging > 2) { *why = "host_staging outside [0,2]"; return false; }
  if (d->lanczos_cap < 0 || d->lanczos_cap > 1000000) { *why = "lanczos_cap outside [0, 1e6]"; return false; }
  if (d->lanczos_store != 0 && d->lanczos_store != 1) { *why = "lanczos_store must be 0 or 1"; return false; }
  if (d->cg_variant != KCG_CG_SINGLE_PASS && d->cg_variant != KCG_CG_HS) { *why = "unknown cg_variant"; return false; }
  return true;
}

bool config_ok(const kcg_desc* d, std::string* why) {
  if (d->prior != KCG_PRIOR_LAPLACIAN && d->prior != KCG_PRIOR_D2) { *why = "unknown prior"; return false; }
  if (d->prior == KCG_PRIOR_D2 && d->n_comp > 4) {
    *why = "KCG_PRIOR_D2 is built for n_comp <= 4 (halo-4 boxes in shared memory)";
    return false;
  }
  if (d->layout != KCG_LAYOUT_ROW_MAJOR && d->layout != KCG_LAYOUT_NESTED) { *why = "unknown layout"; return false; }
  if (d->lanczos_cap > 0 && d->prior == KCG_PRIOR_D2 && d->n_comp > 4) {
    *why = "the block-Lanczos route with KCG_PRIOR_D2 is built for n_comp <= 4 (halo-4 boxes)";
    return false;
  }
  if (d->precond != KCG_PRECOND_NONE && d->precond != KCG_PRECOND_BLOCK_JACOBI) { *why = "unknown precond"; return false; }
  if (d->precond == KCG_PRECOND_BLOCK_JACOBI && d->n_comp > 7) {
    *why = "KCG_PRECOND_BLOCK_JACOBI is built for n_comp <= 7 (shared-memory budget)";
    return false;
  }
  return true;
}

bool slab_ok(const kcg_desc* d, int nranks, std::string* why) {
  if (nranks < 1 || nranks > KCG_GMAX) { *why = "nranks outside [1,8]"; return false; }
  const int side = 1 << d->level;
  if (nranks > 1 && (side % nranks != 0 || side / nranks < 2 * KCG_HALO)) {
    *why = "row slabs need side % nranks == 0 and side / nranks >= 4";
    return false;
  }
  return true;
}

// Symmetric eigendecomposition C = V diag(lam) V^T by cyclic Jacobi rotations (k <= 8).
void jacobi_eig(int k, std::vector<double> C, std::vector<double>* lam, std::vector<double>* V) {
  V->assign((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) (*V)[i * k + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) (i == j ? dia : off) += C[i * k + j] * C[i * k + j];
    if (off <= 1e-34 * dia || off == 0.0) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double apq = C[p * k + q];
        if (apq == 0.0) continue;
        const double theta = (C[q * k + q] - C[p * k + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int i = 0; i < k; ++i) {  // columns p, q
          const double cip = C[i * k + p], ciq = C[i * k + q];
          C[i * k + p] = c * cip - s * ciq;
          C[i * k + q] = s * cip + c * ciq;
        }
        for (int j = 0; j < k; ++j) {  // rows p, q
          const double cpj = C[p * k + j], cqj = C[q * k + j];
          C[p * k + j] = c * cpj - s * cqj;
          C[q * k + j] = s * cpj + c * cqj;
        }
        for (int i = 0; i < k; ++i) {
          const double vip = (*V)[i * k + p], viq = (*V)[i * k + q];
          (*V)[i * k + p] = c * vip - s * viq;
          (*V)[i * k + q] = s * vip + c * viq;
        }
      }
  }
  lam->resize(k);
  for (int i = 0; i < k; ++i) (*lam)[i] = C[i * k + i];
}

// Inverse of a small SPD matrix (Gauss-Jordan with partial pivoting; k <= 8).
void small_inverse(int k, const double* A, double* Ainv) {
  std::vector<double> T((size_t)k * 2 * k, 0.0);
  for (int i = 0; i < k; ++i) {
    for (int j = 0; j < k; ++j) T[i * 2 * k + j] = A[i * k + j];
    T[i * 2 * k + k + i] = 1.0;
  }
  for (int c = 0; c < k; ++c) {
    int piv = c;
    for (int i = c + 1; i < k; ++i)
      if (std::fabs(T[i * 2 * k + c]) > std::fabs(T[piv * 2 * k + c])) piv = i;
    if (piv != c)
      for (int j = 0; j < 2 * k; ++j) std::swap(T[c * 2 * k + j], T[piv * 2 * k + j]);
    const double inv = 1.0 / T[c * 2 * k + c];
    for (int j = 0; j < 2 * k; ++j) T[c * 2 * k + j] *= inv;
    for (int i = 0; i < k; ++i)
      if (i != c) {
        const double f = T[i * 2 * k + c];
        for (int j = 0; j < 2 * k; ++j) T[i * 2 * k + j] -= f * T[c * 2 * k + j];
      }
  }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) Ainv[i * k + j] = T[i * 2 * k + k + j];
}

// Pixel-block Jacobi blocks for hits = 1 (reading R10): Kinv_d = (M + diag(Q0)_d diag(tau))^{-1} for
// degree d = 2, 3, 4 and 0 (level 0: one pixel, no neighbours), with diag(Q0)_d = kappa2 + d
// (Laplacian) or kappa2 + d^2 + d (D^2), stored compactly (K x K each) in sp.Kinv, slot kinv_slot(d).
void set_block_jacobi(int K, const double* M, const double* tau, double kappa2, SysParams* sp, bool d2) {
  std::vector<double> A((size_t)K * K), Ai((size_t)K * K);
  double* out = &sp->Kinv[0][0];
  for (int d : {2, 3, 4, 0}) {
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j) A[i * K + j] = M[i * K + j] + (i == j ? (kappa2 + (d2 ? d * d + d : d)) * tau[i] : 0.0);
    small_inverse(K, A.data(), Ai.data());
    for (int e = 0; e < K * K; ++e) out[kcg::kinv_slot(d) * K * K + e] = Ai[e];
  }
}

// Lemma 2: M W = P W diag(rho), W^T P W = I, rho ascending, largest-|.| entry of each
// column positive.  P = diag(phi) > 0, so with C = P^{-1/2} M P^{-1/2} = V diag(rho) V^T, W = P^{-1/2} V.
void eigh_MP(int k, const double* M, const double* phi, double* rho, double* W) {
  std::vector<double> C((size_t)k * k), lam, V;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) C[i * k + j] = M[i * k + j] / std::sqrt(phi[i] * phi[j]);
  jacobi_eig(k, C, &lam, &V);
  std::vector<int> ord(k);
  for (int i = 0; i < k; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return lam[a] < lam[b]; });
  for (int ii = 0; ii < k; ++ii) {
    const int i = ord[ii];
    rho[ii] = lam[i];
    int arg = 0;
    double best = -1.0;
    for (int c = 0; c < k; ++c) {
      const double v = V[c * k + i] / std::sqrt(phi[c]);
      if (std::fabs(v) > best) { best = std::fabs(v); arg = c; }
    }
    const double sgn = (V[arg * k + i] < 0) ? -1.0 : 1.0;
    for (int c = 0; c < k; ++c) W[c * k + ii] = sgn * V[c * k + i] / std::sqrt(phi[c]);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool encode_map(CUtensorMap* m, double* base, int side, int buf_rows, int pitch, size_t planes, int K, bool d2,
                std::string* why) {
  // box: the CTA tile + halo, or (D2) one row-march stage of 32 m_cp(K) columns x KCG_MCH rows
  const int bx = d2 ? 32 * kcg::m_cp(K) : KCG_TX + 2 * KCG_HALO;
  const int by = d2 ? KCG_MCH : kcg::cg_tile_y(K) + 2 * KCG_HALO;
  auto enc = get_encode();
  if (!enc) { *why = "cuTensorMapEncodeTiled unavailable"; return false; }
  cuuint64_t dims[3] = {(cuuint64_t)side, (cuuint64_t)buf_rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * buf_rows * 8};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)K};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    *why = buf;
    return false;
  }
  return true;
}

// TMA descriptor of the solution buffer x [planes][side][side] with box {64, TY(K), K} (CTA kernel).
bool encode_xmap(CUtensorMap* m, double* base, int side, int rows, size_t planes, int K, bool d2, std::string* why) {
  auto enc = get_encode();
  if (!enc) { *why = "cuTensorMapEncodeTiled unavailable"; return false; }
  cuuint64_t dims[3] = {(cuuint64_t)side, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)side * 8, (cuuint64_t)side * rows * 8};
  cuuint32_t box[3] = {(cuuint32_t)(d2 ? 32 * kcg::m_cp(K) : KCG_TX), (cuuint32_t)(d2 ? KCG_MCH : kcg::cg_tile_y(K)),
                       (cuuint32_t)K};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled (x) failed (%d)", (int)r);
    *why = buf;
    return false;
  }
  return true;
}

// TMA descriptor of the hits planes [planes][side][side] for the D2 row-march kernel: box {32 cp, 1, 1}.
bool encode_hmap(CUtensorMap* m, const double* base, int side, size_t planes, int cp, std::string* why) {
  auto enc = get_encode();
  if (!enc) { *why = "cuTensorMapEncodeTiled unavailable"; return false; }
  cuuint64_t dims[3] = {(cuuint64_t)side, (cuuint64_t)side, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)side * 8, (cuuint64_t)side * side * 8};
  cuuint32_t box[3] = {(cuuint32_t)(32 * cp), (cuuint32_t)KCG_MCH, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled (hits) failed (%d)", (int)r);
    *why = buf;
    return false;
  }
  return true;
}

// TMA descriptor of the block-Lanczos slots [planes][side][pitch], box {64 + 4, TY + 4, K}.
bool encode_lzmap(CUtensorMap* m, double* base, int side, int pitch, size_t planes, int K, bool d2, std::string* why) {
  auto enc = get_encode();
  if (!enc) { *why = "cuTensorMapEncodeTiled unavailable"; return false; }
  cuuint64_t dims[3] = {(cuuint64_t)side, (cuuint64_t)side, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * side * 8};
  const int hb = kcg::lz_halo(d2);
  cuuint32_t box[3] = {(cuuint32_t)(KCG_TX + 2 * hb), (cuuint32_t)(kcg::lz_tile_y(K, d2) + 2 * hb), (cuuint32_t)K};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled (lanczos) failed (%d)", (int)r);
    *why = buf;
    return false;
  }
  return true;
}

bool finite_all(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

kcg_status cuda_fail(kcg_ctx* c, cudaError_t e, const char* what) {
  c->err = std::string(what) + ": " + cudaGetErrorString(e);
  return KCG_E_CUDA;
}

#define CK(call, what)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(c, _e, what); \
  } while (0)
// a launch of one of the library's kernels (counted for report->kernel_launches)
#define CKL(call, what) \
  do {                  \
    ++c->nlaunch;       \
    CK(call, what);     \
  } while (0)

enum Route { ROUTE_KRON = 0, ROUTE_SYL = 1 };

// fraction of a system's tiles in x class 1 (kcg::cg_xclass)
static double kcg_xclass1_frac(int tiles_x, int tiles_y) {
  long long n1 = 0;
  for (int ty = 0; ty < tiles_y; ++ty)
    for (int tx = 0; tx < tiles_x; ++tx) n1 += kcg::cg_xclass(ty, tx, tiles_x);
  return tiles_x * tiles_y > 0 ? (double)n1 / ((double)tiles_x * tiles_y) : 0.0;
}

SlabGeom geom_of(const kcg_ctx* c, const RankState& R) {
  return SlabGeom{c->side, c->rows, R.row0, c->pitch, c->ghost, c->ghost, c->d.layout == KCG_LAYOUT_NESTED,
                  c->d.prior == KCG_PRIOR_D2};
}

// Device pointer of `field` in rank g's workspace (same layout on every rank).
template <typename T>
T* peer_ptr(const kcg_ctx* c, int g, size_t off) { return reinterpret_cast<T*>(c->peer_ws[g] + off); }

kcg::XrankSync xsync_of(const kcg_ctx* c, unsigned long long tag) {
  kcg::XrankSync X{};
  for (int g = 0; g < c->nranks; ++g) X.flags[g] = peer_ptr<unsigned long long>(c, g, c->L.flags);
  X.nranks = c->nranks;
  X.rank0 = c->rank0;
  X.nlocal = c->nlocal;
  X.tag = tag;
  return X;
}

// Fill the slab fields of a rank's CgArgs (peers' ghosted buffers, slots, flags).
void fill_slab_args(const kcg_ctx* c, const RankState& R, CgArgs* a) {
  a->rank = R.rank;
  a->nranks = c->nranks;
  for (int dir = 0; dir < 2; ++dir) {
    const int g = R.rank + (dir == 0 ? -1 : 1);
    for (int b = 0; b < 2; ++b) {
      const bool ok = g >= 0 && g < c->nranks;
      a->nb_r[dir][b] = ok ? peer_ptr<double>(c, g, b ? c->L.r1 : c->L.r0) : nullptr;
      a->nb_p[dir][b] = ok ? peer_ptr<double>(c, g, b ? c->L.p1 : c->L.p0) : nullptr;
    }
  }
  for (int g = 0; g < KCG_GMAX; ++g) {
    a->slots[g] = g < c->nranks ? peer_ptr<double>(c, g, c->L.slots) : nullptr;
    a->flags[g] = g < c->nranks ? peer_ptr<unsigned long long>(c, g, c->L.flags) : nullptr;
  }
  a->my_flags = R.flags;
  a->my_slots = R.slots;
  a->group = R.group;
}

// x boundary rows of every local rank into its neighbours' xg_top / xg_bot, then a rendezvous.
kcg_status exchange_x_rows(kcg_ctx* c, const double* x_all, size_t x_rank_stride, unsigned long long tag) {
  cudaStream_t s = c->stream;
  for (int j = 0; j < c->nlocal; ++j) {
    const RankState& R = c->R[j];
    double* up = R.rank > 0 ? peer_ptr<double>(c, R.rank - 1, c->L.xg_bot) : nullptr;
    double* dn = R.rank + 1 < c->nranks ? peer_ptr<double>(c, R.rank + 1, c->L.xg_top) : nullptr;
    CKL(kcg::launch_xghost(s, x_all + j * x_rank_stride, up, dn, c->P * c->k, geom_of(c, R)), "x ghost kernel");
  }
  CKL(kcg::launch_xrank_sync(s, xsync_of(c, tag)), "rendezvous kernel");
  return KCG_OK;
}

// Right-hand side given as the data Y (IN_Y), as b = G mu itself in the user's layout (IN_B_USER,
// kron_cg_solve_b), or as b in the kernels' row-major working layout with mu returned in that
// layout too (IN_B_WORK: the posterior-variance probes).
enum InputMode { IN_Y = 0, IN_B_USER = 1, IN_B_WORK = 2 };

kcg_status solve_impl(kcg_ctx* c, Route route, const double* Y_in, double* mu_out, bool host_io, double tol,
                      int max_iter, kcg_report* rep, InputMode inmode = IN_Y, const double* x0 = nullptr,
                      const std::function<kcg_status()>* after_launch = nullptr) {
  Nvtx nv_(route == ROUTE_KRON ? "kcg:kron_cg_solve" : "kcg:sylvester_solve");
  if (!c) return KCG_E_ARG;
  if (x0 && (route != ROUTE_KRON || host_io || c->slab || inmode != IN_Y || c->d.cg_variant != KCG_CG_SINGLE_PASS)) {
    c->err = "warm start: Kronecker route, device buffers, single-pass CG, no row slabs";
    return KCG_E_CONFIG;
  }
  if (inmode != IN_Y && (route != ROUTE_KRON || host_io || c->slab)) {
    c->err = "a given right-hand side b needs the Kronecker route, device buffers and no row slabs";
    return KCG_E_CONFIG;
  }
  if (!Y_in || !mu_out) { c->err = "null Y or mu"; return KCG_E_ARG; }
  if (!host_io && (reinterpret_cast<uintptr_t>(mu_out) & 15)) {  // the kernels store x as double2
    c->err = "mu must be 16-byte aligned";
    return KCG_E_ARG;
  }
  if (!(tol > 0.0) || !std::isfinite(tol)) { c->err = "tol must be finite and > 0"; return KCG_E_ARG; }
  if (max_iter < 0) { c->err = "max_iter < 0"; return KCG_E_ARG; }
  if (host_io && !c->d.host_staging) { c->err = "host entry point needs desc.host_staging = 1"; return KCG_E_CONFIG; }
  cudaStream_t s = c->stream;
  const int P = c->P, n = c->n, k = c->k;
  const size_t N = c->N;
  const size_t y_stride = (size_t)P * n * N, mu_stride = (size_t)P * k * N;  // per local rank
  const bool kron = route == ROUTE_KRON;
  const int Kk = kron ? k : 1;
  const int n_sys = kron ? P : P * k;
  const bool prec = c->d.precond == KCG_PRECOND_BLOCK_JACOBI;
  const unsigned long long tag0 = (++c->solve_id) << 32;
  const bool bgiven = inmode != IN_Y;
  auto Yr = [&](int j) -> const double* {
    if (bgiven) return (inmode == IN_B_USER && c->R[j].y_rm) ? c->R[j].y_rm : Y_in;  // b, working layout
    return host_io ? c->R[j].Y_stage : Y_in + j * y_stride;
  };
  auto muu = [&](int j) -> double* { return host_io ? c->R[j].mu_stage : mu_out + j * mu_stride; };
  // the kernels' solution buffer: the user's mu, or the row-major copy for a NESTED layout
  auto mur = [&](int j) -> double* { return (c->R[j].x_rm && inmode != IN_B_WORK) ? c->R[j].x_rm : muu(j); };
  // geometry of the data / b reads: b is in the working layout (no NESTED gather)
  auto gin = [&](const RankState& R) { SlabGeom g = geom_of(c, R); if (bgiven) g.nested = 0; return g; };
  const int nin = bgiven ? k : n;  // planes per patch of the rhs input

  CK(cudaEventRecord(c->ev[0], s), "event");
  for (int j = 0; j < c->nlocal; ++j) {
    RankState& R = c->R[j];
    if (host_io) CK(cudaMemcpyAsync(R.Y_stage, Y_in + j * y_stride, y_stride * 8, cudaMemcpyHostToDevice, s), "H2D Y");
    if (inmode == IN_B_USER && R.y_rm)
      CKL(kcg::launch_permute(s, Y_in, R.y_rm, (size_t)P * k, c->side, false), "permute b");
    // (warm start: x is not zeroed -- x_0 may alias mu; it is copied in below)
    CKL(kcg::launch_rhs(k, s, Yr(j), bgiven ? nullptr : (kron ? R.E_kron : R.E_syl), R.hits, R.r[0], R.p[0],
                       x0 ? nullptr : mur(j), P, nin, gin(R)),
       "rhs kernel");
    if (x0) {  // warm start (reading R37): x = x_0, r_0 = b - G x_0, (||r_0||^2, ||b||^2) per system
      if (R.x_rm) CKL(kcg::launch_permute(s, x0, R.x_rm, (size_t)P * k, c->side, false), "permute x0");
      else if (x0 != mur(j)) CK(cudaMemcpyAsync(mur(j), x0, mu_stride * 8, cudaMemcpyDeviceToDevice, s), "D2D x0");
      CKL(kcg::launch_resid(k, s, R.params_kron, mur(j), Yr(j), R.E_kron, R.hits, R.resid_partials, R.resid_out, P, n,
                           gin(R), nullptr, nullptr),
         "residual kernel (x0)");
      CKL(kcg::launch_apply(k, s, R.params_kron, mur(j), R.r[1], R.hits, P, geom_of(c, R), nullptr, nullptr),
         "apply kernel (x0)");
      CKL(kcg::launch_sub_pitched(s, R.r[0], R.r[1], (size_t)P * k, c->side, c->pitch), "r0 = b - G x0");
    }
  }
  if (c->slab)
    for (int j = 0; j < c->nlocal; ++j) {
      const RankState& R = c->R[j];
      double *ur = nullptr, *up = nullptr, *dr = nullptr, *dp = nullptr;
      if (R.rank > 0) { ur = peer_ptr<double>(c, R.rank - 1, c->L.r0); up = peer_ptr<double>(c, R.rank - 1, c->L.p0); }
      if (R.rank + 1 < c->nranks) { dr = peer_ptr<double>(c, R.rank + 1, c->L.r0); dp = peer_ptr<double>(c, R.rank + 1, c->L.p0); }
      CKL(kcg::launch_ghost_fill(s, R.r[0], R.p[0], ur, up, dr, dp, P * k, geom_of(c, R)), "ghost fill kernel");
    }
  CK(cudaEventRecord(c->ev[1], s), "event");

  CgSlabLaunch* Lp = new CgSlabLaunch();  // large (TMA maps of every rank): heap, not stack
  std::unique_ptr<CgSlabLaunch> L_owner(Lp);
  CgSlabLaunch& Lx = *Lp;
  const ResPlan res = c->slab ? ResPlan{} : (kron ? c->res_kron : c->res_syl);
  for (int j = 0; j < c->nlocal; ++j) {
    RankState& R = c->R[j];
    CgArgs& a = Lx.a[j];
    a = CgArgs{};
    a.params = kron ? R.params_kron : R.params_syl;
    a.x = mur(j);
    a.rbuf[0] = R.r[0]; a.rbuf[1] = R.r[1];
    a.pbuf[0] = R.p[0]; a.pbuf[1] = R.p[1];
    a.partials = R.partials;
    a.state_out = R.state;
    a.history = R.history;
    a.history_cap = c->d.history_cap;
    a.hits = R.hits;
    a.side = c->side;
    a.pitch = c->pitch;
    a.rows = c->rows;
    a.row0 = R.row0;
    a.ghost = c->ghost;
    a.n_sys = n_sys;
    a.tiles_x = kron ? c->tiles_x_kron : c->tiles_x_syl;
    a.tiles_y = kron ? c->tiles_y_kron : c->tiles_y_syl;
    const bool march = c->d.prior == KCG_PRIOR_D2 && c->d.cg_variant == KCG_CG_SINGLE_PASS;
    a.tiles_per_sys = a.tiles_x * a.tiles_y * (march ? kcg::m_gw(Kk, R.hits != nullptr) : 1);  // row-march: partials per group warp
    a.max_iter = max_iter;
    a.tol2 = tol * tol;
    a.bnorm2 = x0 ? R.resid_out : nullptr;
    a.trace = R.trace;
    a.sync = R.sync;
    a.tag0 = tag0;
    if (c->slab) fill_slab_args(c, R, &a);
    CgMaps& maps = kron ? R.maps_kron : R.maps_syl;
    a.x_tma = 0;
    if (c->side >= 2 && (reinterpret_cast<uintptr_t>(a.x) % 16) == 0) {
      std::string why;
      if (!encode_xmap(&maps.x, a.x, c->side, c->rows, (size_t)P * k, Kk, c->d.prior == KCG_PRIOR_D2, &why)) {
        c->err = why;
        return KCG_E_CUDA;
      }
      a.x_tma = 1;
    }
    if (march) {  // row-march kernel: segment rows, hits by TMA
      a.h_tma = (R.hits && c->side >= 2) ? 1 : 0;
      march_seg(&a, c->side, Kk, n_sys, (kron ? c->grid_kron : c->grid_syl) * kcg::m_groups(Kk, R.hits != nullptr));
    }
    Lx.m[j] = maps;
    CK(cudaMemsetAsync(R.sync, 0, 4 * sizeof(unsigned), s), "memset sync");
    CK(cudaMemsetAsync(R.group, 0, 4 * sizeof(unsigned), s), "memset group");
  }
  if (c->slab) {
    Lx.nlocal = c->nlocal;
    Lx.ctas = kron ? c->grid_kron : c->grid_syl;
    CKL(kcg::launch_cg_slab(Kk, prec, s, Lx, kron ? c->smem_kron : c->smem_syl), "cg slab kernel");
  } else if (res.on) {
    CgArgs& a = Lx.a[0];
    a.tiles_per_sys = res.nstrip;
    if (c->d.history_cap > 0) CK(cudaMemsetAsync(a.history, 0, (size_t)c->d.history_cap * 8, s), "memset history");
    CKL(kcg::launch_cg_resident(Kk, prec, s, a, c->R[0].res_part, res.grid, res.smem), "cg kernel (resident)");
  } else if (c->d.cg_variant == KCG_CG_HS) {
    CKL(kcg::launch_cg_hs(Kk, prec, c->d.prior == KCG_PRIOR_D2, s, Lx.a[0], c->R[0].r[1], c->R[0].hs_part,
                         kron ? c->grid_kron : c->grid_syl, kron ? c->smem_kron : c->smem_syl),
       "cg kernel (HS variant)");
  } else {
    CKL(kcg::launch_cg(Kk, prec, c->d.prior == KCG_PRIOR_D2, s, Lx.a[0], Lx.m[0], kron ? c->grid_kron : c->grid_syl,
                      kron ? c->smem_kron : c->smem_syl),
       "cg kernel");
  }
  CK(cudaEventRecord(c->ev[2], s), "event");
  for (int j = 0; j < c->nlocal; ++j) {
    RankState& R = c->R[j];
    if (res.on) {  // x written whole by the resident kernel
    } else if (c->d.cg_variant == KCG_CG_HS)
      CKL(kcg::launch_hs_xfix(Kk, s, R.state, R.p[0], R.p[1], mur(j), n_sys, c->side, c->pitch), "x fix-up kernel");
    else if (KCG_X2)
      CKL(kcg::launch_xfix(Kk, c->d.prior == KCG_PRIOR_D2 ? 0 : kcg::cg_tile_y(Kk), s, R.state, R.p[0], R.p[1],
                           mur(j), n_sys, geom_of(c, R)),
          "x fix-up kernel");
    if (!kron) CKL(kcg::launch_backtransform(k, s, R.W_dev, mur(j), P, N), "backtransform kernel");
  }
  // true residual ||b - G x|| / ||b|| (one apply pass; x boundary rows exchanged in slab mode)
  if (c->slab) {
    for (int j = 0; j < c->nlocal; ++j) {
      const RankState& R = c->R[j];
      double* up = R.rank > 0 ? peer_ptr<double>(c, R.rank - 1, c->L.xg_bot) : nullptr;
      double* dn = R.rank + 1 < c->nranks ? peer_ptr<double>(c, R.rank + 1, c->L.xg_top) : nullptr;
      CKL(kcg::launch_xghost(s, mur(j), up, dn, P * k, geom_of(c, R)), "x ghost kernel");
    }
    CKL(kcg::launch_xrank_sync(s, xsync_of(c, tag0 + kPostTag + 1)), "rendezvous kernel");
  }
  for (int j = 0; j < c->nlocal; ++j) {
    RankState& R = c->R[j];
    CKL(kcg::launch_resid(k, s, R.params_kron, mur(j), Yr(j), bgiven ? nullptr : R.E_kron, R.hits, R.resid_partials,
                         R.resid_out, P, nin, gin(R), c->slab ? R.xg_top : nullptr, c->slab ? R.xg_bot : nullptr),
       "residual kernel");
    if (c->slab) {
      kcg::XrankPut Pt{};
      for (int g = 0; g < c->nranks; ++g) Pt.dst[g] = peer_ptr<double>(c, g, c->L.rslots);
      Pt.src = R.resid_out;
      Pt.count = P * 2;
      Pt.rank = R.rank;
      Pt.nranks = c->nranks;
      CKL(kcg::launch_put(s, Pt), "put kernel");
    }
  }
  if (c->slab) CKL(kcg::launch_xrank_sync(s, xsync_of(c, tag0 + kPostTag + 2)), "rendezvous kernel");
  for (int j = 0; j < c->nlocal; ++j)
    if (c->R[j].x_rm && inmode != IN_B_WORK)
      CKL(kcg::launch_permute(s, c->R[j].x_rm, muu(j), (size_t)P * k, c->side, true), "permute mu");
  // the solve's device work is queued: the caller's hook (kron_cg_solve_host_many: the next batch's H2D
  // and the previous batch's D2H) goes in now, so a host-blocking copy call cannot delay these kernels
  if (after_launch) {
    const kcg_status e = (*after_launch)();
    if (e != KCG_OK) return e;
  }
  c->st_host.resize(n_sys);
  const int nr = c->slab ? c->nranks : 1;
  c->resid_host.resize((size_t)nr * P * 2);
  CK(cudaMemcpyAsync(c->st_host.data(), c->R[0].state, n_sys * sizeof(SysState), cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaMemcpyAsync(c->resid_host.data(), c->slab ? c->R[0].rslots : c->R[0].resid_out, (size_t)nr * P * 2 * 8,
                     cudaMemcpyDeviceToHost, s),
     "D2H");
  if (host_io)
    for (int j = 0; j < c->nlocal; ++j)
      CK(cudaMemcpyAsync(mu_out + j * mu_stride, c->R[j].mu_stage, mu_stride * 8, cudaMemcpyDeviceToHost, s), "D2H mu");
  CK(cudaEventRecord(c->ev[3], s), "event");
  CK(cudaStreamSynchronize(s), "solve");

  // report (every rank holds the same scalars; residual sums added over ranks in rank order)
  int worst = KCG_OK, maxit = 0, allconv = 1;
  long long sumit = 0, passes = 0;
  double xpasses = 0.0;
  // tiles of class 1 (odd index) of the tile kernel's mixed x schedule (KCG_XMIX), per system
  const bool xmix = KCG_X2 && KCG_XMIX && c->d.prior != KCG_PRIOR_D2;
  const double frac1 = xmix ? kcg_xclass1_frac(kron ? c->tiles_x_kron : c->tiles_x_syl,
                                               kron ? c->tiles_y_kron : c->tiles_y_syl) : 0.0;
  double maxrel = 0.0;
  for (int i = 0; i < n_sys; ++i) {
    const SysState& z = c->st_host[i];
    maxit = std::max(maxit, z.iters);
    sumit += z.iters;
    passes += z.iters + 1;
    // x passes: class 0 the even q in [2, iters], class 1 the odd q in [1, iters]
    xpasses += KCG_X2 ? (1.0 - frac1) * (z.iters / 2) + frac1 * ((z.iters + 1) / 2) : (double)z.iters;
    maxrel = std::max(maxrel, z.rel);
    if (z.status != kcg::ST_CONVERGED) allconv = 0;
    int code = KCG_OK;
    if (z.status == kcg::ST_NONFINITE) code = KCG_E_NONFINITE;
    else if (z.status == kcg::ST_BREAKDOWN) code = KCG_E_BREAKDOWN;
    else if (z.status == kcg::ST_MAXIT) code = KCG_NOT_CONVERGED;
    auto rank = [](int cd) { return cd == KCG_E_NONFINITE ? 3 : cd == KCG_E_BREAKDOWN ? 2 : cd == KCG_NOT_CONVERGED ? 1 : 0; };
    if (rank(code) > rank(worst)) worst = code;
  }
  double maxtrue = 0.0;
  for (int p = 0; p < P; ++p) {
    double r2 = 0.0, b2 = 0.0;
    for (int g = 0; g < nr; ++g) {
      r2 += c->resid_host[((size_t)g * P + p) * 2];
      b2 += c->resid_host[((size_t)g * P + p) * 2 + 1];
    }
    maxtrue = std::max(maxtrue, b2 > 0 ? std::sqrt(r2 / b2) : std::sqrt(r2));
  }
  if (rep) {
    float t03 = 0.f, t12 = 0.f;
    cudaEventElapsedTime(&t03, c->ev[0], c->ev[3]);
    cudaEventElapsedTime(&t12, c->ev[1], c->ev[2]);
    rep->status = worst;
    rep->converged = allconv;
    rep->iterations = maxit;
    rep->n_systems = n_sys;
    if (rep->iterations_per)
      for (int i = 0; i < n_sys; ++i) rep->iterations_per[i] = c->st_host[i].iters;
    rep->rel_residual = maxrel;
    rep->rel_residual_true = maxtrue;
    rep->wall_time_s = t03 * 1e-3;
    rep->loop_time_s = t12 * 1e-3;
    rep->system_iterations = sumit;
    // per pass: read + write r and p (32 B per pixel and plane); x passes also read + write x.
    // Local bytes of this context's ranks (slab mode: the local rows of each local rank).
    rep->loop_bytes = (32.0 * (double)passes + 16.0 * (double)xpasses) * Kk * (double)N * c->nlocal;
    if (c->d.cg_variant == KCG_CG_HS)  // per iteration: pass A 4 vectors (+ x read + write from the 2nd), pass B 3
      rep->loop_bytes = (56.0 * (double)sumit + 16.0 * (double)std::max(0LL, sumit - n_sys)) * Kk * (double)N;
    if (res.on) {  // global bytes of the resident kernel: b in, x out, per pass the strips' halo rows
      const int rs = c->side / res.nstrip;
      rep->loop_bytes = 16.0 * Kk * (double)N * n_sys;
      if (res.nstrip > 1)
        rep->loop_bytes += (double)passes * res.nstrip * (std::min(4, rs) + 4) * c->side * Kk * 16.0;
    }
    rep->peak_mem_bytes = c->ws_need;
    rep->kernel_launches = c->nlaunch;
    rep->history_len = std::min(maxit, c->d.history_cap);
    if (rep->history && rep->history_len > 0) {
      cudaError_t e = cudaMemcpy(rep->history, c->R[0].history, (size_t)rep->history_len * 8, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(c, e, "D2H history");
    }
  }
  c->err.clear();
  return (kcg_status)worst;
}


// Block-Lanczos Sylvester solve (Alg. SylvSolver): rhs kernel (Y^ = Y T A P^{-1} into
// slot 0), one cooperative launch (Lanczos passes + gamma + coefficients + replay), store mode:
// the assembly kernel; then the true residual of G mu = b as for CG.
kcg_status lanczos_impl(kcg_ctx* c, const double* Y_in, double* mu_out, bool host_io, double tol, int max_iter,
                        kcg_report* rep) {
  Nvtx nv_("kcg:sylvester_lanczos_solve");
  if (!c) return KCG_E_ARG;
  if (c->L.lz_slots <= 0 || c->slab) {
    c->err = c->slab ? "block-Lanczos route: no row slabs" : "block-Lanczos route needs desc.lanczos_cap > 0";
    return KCG_E_CONFIG;
  }
  if (!Y_in || !mu_out) { c->err = "null Y or mu"; return KCG_E_ARG; }
  if (!host_io && (reinterpret_cast<uintptr_t>(mu_out) & 15)) {  // the kernels store x as double2
    c->err = "mu must be 16-byte aligned";
    return KCG_E_ARG;
  }
  if (!(tol > 0.0) || !std::isfinite(tol)) { c->err = "tol must be finite and > 0"; return KCG_E_ARG; }
  if (max_iter < 0) { c->err = "max_iter < 0"; return KCG_E_ARG; }
  if (host_io && !c->d.host_staging) { c->err = "host entry point needs desc.host_staging = 1"; return KCG_E_CONFIG; }
  cudaStream_t s = c->stream;
  const int P = c->P, n = c->n, k = c->k;
  const size_t N = c->N;
  RankState& R = c->R[0];
  const double* Yr = host_io ? R.Y_stage : Y_in;
  double* muu = host_io ? R.mu_stage : mu_out;
  double* mur = R.x_rm ? R.x_rm : muu;
  const int cap = c->d.lanczos_cap;
  const int mit = std::min(max_iter, cap);

  CK(cudaEventRecord(c->ev[0], s), "event");
  if (host_io) CK(cudaMemcpyAsync(R.Y_stage, Y_in, (size_t)P * n * N * 8, cudaMemcpyHostToDevice, s), "H2D Y");
  SlabGeom g{c->side, c->side, 0, c->pitch, 0, 0, c->d.layout == KCG_LAYOUT_NESTED, c->d.prior == KCG_PRIOR_D2};
  CKL(kcg::launch_rhs(k, s, Yr, R.E_lz, nullptr, R.lz_V, nullptr, nullptr, P, n, g), "lanczos rhs kernel");
  CK(cudaMemsetAsync(R.lz_st, 0, P * sizeof(kcg::LzState), s), "memset lanczos state");
  CK(cudaEventRecord(c->ev[1], s), "event");
  kcg::LzArgs a{};
  a.prm = R.lz_prm;
  a.hits = R.hits;
  a.V = R.lz_V;
  a.Mx = mur;
  a.part = R.lz_part;
  a.st = R.lz_st;
  a.Hs = R.lz_H;
  a.Rs = R.lz_R;
  a.Ri = R.lz_Ri;
  a.Sinv = R.lz_Sinv;
  a.gv = R.lz_g;
  a.Zs = R.lz_Z;
  a.P = P;
  a.side = c->side;
  a.pitch = c->pitch;
  a.tiles_x = c->tiles_x_lz;
  a.tiles_y = c->tiles_y_lz;
  a.tps = a.tiles_x * a.tiles_y;
  a.cap = cap;
  a.max_iter = mit;
  a.store = c->d.lanczos_store;
  a.tol = tol;
  a.trace = R.trace;
  CKL(kcg::launch_lanczos(k, R.hits != nullptr, c->d.prior == KCG_PRIOR_D2, s, a, R.lz_map, c->grid_lz, c->smem_lz),
     "lanczos kernel");
  if (a.store) CKL(kcg::launch_lz_assemble(k, s, a), "lanczos assembly kernel");
  CK(cudaEventRecord(c->ev[2], s), "event");
  CKL(kcg::launch_resid(k, s, R.params_kron, mur, Yr, R.E_kron, R.hits, R.resid_partials, R.resid_out, P, n,
                       geom_of(c, R), nullptr, nullptr),
     "residual kernel");
  if (R.x_rm) CKL(kcg::launch_permute(s, R.x_rm, muu, (size_t)P * k, c->side, true), "permute mu");
  c->lz_host.resize(P);
  c->resid_host.resize((size_t)P * 2);
  CK(cudaMemcpyAsync(c->lz_host.data(), R.lz_st, P * sizeof(kcg::LzState), cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaMemcpyAsync(c->resid_host.data(), R.resid_out, (size_t)P * 2 * 8, cudaMemcpyDeviceToHost, s), "D2H");
  if (host_io) CK(cudaMemcpyAsync(mu_out, R.mu_stage, (size_t)P * k * N * 8, cudaMemcpyDeviceToHost, s), "D2H mu");
  CK(cudaEventRecord(c->ev[3], s), "event");
  CK(cudaStreamSynchronize(s), "lanczos solve");

  int worst = KCG_OK, maxit = 0, allconv = 1;
  long long sumit = 0;
  double maxrel = 0.0, bytes = 0.0;
  const double vec = 8.0 * k * (double)N;  // one block vector of a patch
  for (int p = 0; p < P; ++p) {
    const kcg::LzState& z = c->lz_host[p];
    maxit = std::max(maxit, z.iters);
    sumit += z.iters;
    maxrel = std::max(maxrel, z.rel);
    if (z.status != kcg::ST_CONVERGED) allconv = 0;
    int code = KCG_OK;
    if (z.status == kcg::ST_NONFINITE) code = KCG_E_NONFINITE;
    else if (z.status == kcg::ST_BREAKDOWN) code = KCG_E_BREAKDOWN;
    else if (z.status == kcg::ST_MAXIT || z.status == kcg::ST_RUNNING) code = KCG_NOT_CONVERGED;
    auto rank = [](int cd) { return cd == KCG_E_NONFINITE ? 3 : cd == KCG_E_BREAKDOWN ? 2 : cd == KCG_NOT_CONVERGED ? 1 : 0; };
    if (rank(code) > rank(worst)) worst = code;
    // algorithmic bytes: Gram pass reads Y^; step 1 reads Y^ and writes V_1; step i >= 2 reads V_{i-1}
    // (and V_{i-2} from i = 3) and writes V_i; assembly reads V_1..V_i and writes M (store) or replays
    // the steps with M read + written (M only written on the first replay step)
    const int i = z.iters;
    double b = vec;  // Gram of Y^
    if (i >= 1) b += 2 * vec;
    if (i >= 2) b += (2.0 + 3.0 * (i - 2)) * vec;
    if (c->d.lanczos_store) b += (i > 0 ? (double)i + 1.0 : 1.0) * vec;
    else if (c->d.prior != KCG_PRIOR_D2 && k <= 4)  // pair-mapped replay: M every other pass
      b += (i >= 2 ? 3.0 * i - 3.0 + 2.0 * ((i + 1) / 2) - 1.0 : i == 1 ? 2.0 : 1.0) * vec;
    else b += (i >= 2 ? 5.0 * i - 4.0 : i == 1 ? 2.0 : 1.0) * vec;  // V reads/writes 3i-3, M 2i-1
    bytes += b;
  }
  double maxtrue = 0.0;
  for (int p = 0; p < P; ++p) {
    const double r2 = c->resid_host[(size_t)p * 2], b2 = c->resid_host[(size_t)p * 2 + 1];
    maxtrue = std::max(maxtrue, b2 > 0 ? std::sqrt(r2 / b2) : std::sqrt(r2));
  }
  if (rep) {
    float t03 = 0.f, t12 = 0.f;
    cudaEventElapsedTime(&t03, c->ev[0], c->ev[3]);
    cudaEventElapsedTime(&t12, c->ev[1], c->ev[2]);
    rep->status = worst;
    rep->converged = allconv;
    rep->iterations = maxit;
    rep->n_systems = P;
    if (rep->iterations_per)
      for (int p = 0; p < P; ++p) rep->iterations_per[p] = c->lz_host[p].iters;
    rep->rel_residual = maxrel;
    rep->rel_residual_true = maxtrue;
    rep->wall_time_s = t03 * 1e-3;
    rep->loop_time_s = t12 * 1e-3;
    rep->system_iterations = sumit;
    rep->loop_bytes = bytes;
    rep->peak_mem_bytes = c->ws_need;
    rep->kernel_launches = c->nlaunch;
    rep->history_len = 0;
  }
  c->err.clear();
  return (kcg_status)worst;
}

// Alg. Kohler (reading R33): the k columns of every patch solved one after the other,
// column i's right-hand side carrying the Schur coupling to the columns already solved; each column
// is one batched launch of the CG kernel over the P patches (K = 1 systems, shift R_ii).
kcg_status kohler_impl(kcg_ctx* c, const double* Y_in, double* mu_out, double tol, int max_iter, kcg_report* rep) {
  Nvtx nv_("kcg:sylvester_kohler_solve");
  if (!c) return KCG_E_ARG;
  if (c->slab) { c->err = "Alg. Kohler route: no row slabs"; return KCG_E_CONFIG; }
  if (!Y_in || !mu_out) { c->err = "null Y or mu"; return KCG_E_ARG; }
  if ((reinterpret_cast<uintptr_t>(mu_out) & 15)) {  // the kernels store x as double2
    c->err = "mu must be 16-byte aligned";
    return KCG_E_ARG;
  }
  if (!(tol > 0.0) || !std::isfinite(tol)) { c->err = "tol must be finite and > 0"; return KCG_E_ARG; }
  if (max_iter < 0) { c->err = "max_iter < 0"; return KCG_E_ARG; }
  cudaStream_t s = c->stream;
  const int P = c->P, n = c->n, k = c->k;
  const size_t N = c->N;
  RankState& R = c->R[0];
  double* mur = R.x_rm ? R.x_rm : mu_out;            // X^ (working layout), then X in place
  double* xcol = k > 1 ? R.r[1] + (size_t)P * c->pitch * c->side : mur;  // spare planes of r[1]
  const bool nested = c->d.layout == KCG_LAYOUT_NESTED, d2 = c->d.prior == KCG_PRIOR_D2;
  const bool prec = c->d.precond == KCG_PRECOND_BLOCK_JACOBI;
  std::vector<SysState> st((size_t)k * P);
  CK(cudaEventRecord(c->ev[0], s), "event");
  CK(cudaEventRecord(c->ev[1], s), "event");
  CgSlabLaunch* Lp = new CgSlabLaunch();
  std::unique_ptr<CgSlabLaunch> L_owner(Lp);
  for (int i = 0; i < k; ++i) {
    CKL(kcg::launch_kohler_rhs(k, s, Y_in, R.E_koh, R.R_koh, mur, R.hits, R.r[0], R.p[0], xcol, P, n, i, c->side,
                              c->pitch, nested),
       "kohler rhs kernel");
    CgArgs& a = Lp->a[0];
    a = CgArgs{};
    a.params = R.params_koh + (size_t)i * P;
    a.x = xcol;
    a.rbuf[0] = R.r[0]; a.rbuf[1] = R.r[1];
    a.pbuf[0] = R.p[0]; a.pbuf[1] = R.p[1];
    a.partials = R.partials;
    a.state_out = R.state;
    a.history = R.history;
    a.history_cap = 0;
    a.hits = R.hits;
    a.side = c->side;
    a.pitch = c->pitch;
    a.rows = c->rows;
    a.row0 = 0;
    a.ghost = 0;
    a.n_sys = P;
    a.tiles_x = c->tiles_x_syl;
    a.tiles_y = c->tiles_y_syl;
    a.tiles_per_sys = a.tiles_x * a.tiles_y;
    a.max_iter = max_iter;
    a.tol2 = tol * tol;
    a.trace = nullptr;
    a.sync = R.sync;
    CgMaps maps = R.maps_syl;
    a.x_tma = 0;
    if (c->side >= 2 && (reinterpret_cast<uintptr_t>(a.x) % 16) == 0) {
      std::string why;
      if (!encode_xmap(&maps.x, a.x, c->side, c->rows, (size_t)P, 1, d2, &why)) { c->err = why; return KCG_E_CUDA; }
      a.x_tma = 1;
    }
    CK(cudaMemsetAsync(R.sync, 0, 4 * sizeof(unsigned), s), "memset sync");
    const int grid = std::max(1, std::min(c->grid_syl, P * a.tiles_per_sys));
    if (d2) {
      a.h_tma = (R.hits && c->side >= 2) ? 1 : 0;
      march_seg(&a, c->side, 1, P, grid * kcg::m_groups(1, R.hits != nullptr));
    }
    if (c->res_koh.on) {
      a.tiles_per_sys = c->res_koh.nstrip;
      CKL(kcg::launch_cg_resident(1, prec, s, a, R.res_part, c->res_koh.grid, c->res_koh.smem),
         "cg kernel (kohler column, resident)");
    } else if (c->d.cg_variant == KCG_CG_HS) {
      CKL(kcg::launch_cg_hs(1, prec, d2, s, a, R.r[1], R.hs_part, grid, c->smem_syl), "cg kernel (kohler column, HS)");
      CKL(kcg::launch_hs_xfix(1, s, R.state, R.p[0], R.p[1], xcol, P, c->side, c->pitch), "x fix-up kernel");
    } else {
      CKL(kcg::launch_cg(1, prec, d2, s, a, maps, grid, c->smem_syl), "cg kernel (kohler column)");
      if (KCG_X2)
        CKL(kcg::launch_xfix(1, d2 ? 0 : kcg::cg_tile_y(1), s, R.state, R.p[0], R.p[1], xcol, P, geom_of(c, R)),
            "x fix-up kernel");
    }
    if (k > 1) CKL(kcg::launch_column_copy(s, xcol, mur, P, k, i, N), "column copy kernel");
    CK(cudaMemcpyAsync(st.data() + (size_t)i * P, R.state, P * sizeof(SysState), cudaMemcpyDeviceToHost, s), "D2H");
  }
  CKL(kcg::launch_backtransform(k, s, R.W_koh, mur, P, N), "backtransform kernel");
  CK(cudaEventRecord(c->ev[2], s), "event");
  CKL(kcg::launch_resid(k, s, R.params_kron, mur, Y_in, R.E_kron, R.hits, R.resid_partials, R.resid_out, P, n,
                       geom_of(c, R), nullptr, nullptr),
     "residual kernel");
  if (R.x_rm) CKL(kcg::launch_permute(s, R.x_rm, mu_out, (size_t)P * k, c->side, true), "permute mu");
  c->resid_host.resize((size_t)P * 2);
  CK(cudaMemcpyAsync(c->resid_host.data(), R.resid_out, (size_t)P * 2 * 8, cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaEventRecord(c->ev[3], s), "event");
  CK(cudaStreamSynchronize(s), "kohler solve");
  int worst = KCG_OK, maxit = 0, allconv = 1;
  long long sumit = 0, passes = 0;
  double xpasses = 0.0;
  const double frac1 = KCG_X2 && KCG_XMIX && !d2 ? kcg_xclass1_frac(c->tiles_x_syl, c->tiles_y_syl) : 0.0;  // K = 1
  double maxrel = 0.0;
  for (const SysState& z : st) {
    maxit = std::max(maxit, z.iters);
    sumit += z.iters;
    passes += z.iters + 1;
    xpasses += KCG_X2 ? (1.0 - frac1) * (z.iters / 2) + frac1 * ((z.iters + 1) / 2) : (double)z.iters;
    maxrel = std::max(maxrel, z.rel);
    if (z.status != kcg::ST_CONVERGED) allconv = 0;
    int code = KCG_OK;
    if (z.status == kcg::ST_NONFINITE) code = KCG_E_NONFINITE;
    else if (z.status == kcg::ST_BREAKDOWN) code = KCG_E_BREAKDOWN;
    else if (z.status == kcg::ST_MAXIT) code = KCG_NOT_CONVERGED;
    auto rank = [](int cd) { return cd == KCG_E_NONFINITE ? 3 : cd == KCG_E_BREAKDOWN ? 2 : cd == KCG_NOT_CONVERGED ? 1 : 0; };
    if (rank(code) > rank(worst)) worst = code;
  }
  double maxtrue = 0.0;
  for (int p = 0; p < P; ++p) {
    const double r2 = c->resid_host[(size_t)p * 2], b2 = c->resid_host[(size_t)p * 2 + 1];
    maxtrue = std::max(maxtrue, b2 > 0 ? std::sqrt(r2 / b2) : std::sqrt(r2));
  }
  if (rep) {
    float t03 = 0.f, t12 = 0.f;
    cudaEventElapsedTime(&t03, c->ev[0], c->ev[3]);
    cudaEventElapsedTime(&t12, c->ev[1], c->ev[2]);
    rep->status = worst;
    rep->converged = allconv;
    rep->iterations = maxit;
    rep->n_systems = P * k;
    if (rep->iterations_per)
      for (int p = 0; p < P; ++p)
        for (int i = 0; i < k; ++i) rep->iterations_per[p * k + i] = st[(size_t)i * P + p].iters;
    rep->rel_residual = maxrel;
    rep->rel_residual_true = maxtrue;
    rep->wall_time_s = t03 * 1e-3;
    rep->loop_time_s = t12 * 1e-3;
    rep->system_iterations = sumit;
    rep->loop_bytes = (32.0 * (double)passes + 16.0 * (double)xpasses) * (double)N;
    rep->peak_mem_bytes = c->ws_need;
    rep->kernel_launches = c->nlaunch;
    rep->history_len = 0;
  }
  c->err.clear();
  return (kcg_status)worst;
}
}  // namespace

namespace {

// Plan the shared-memory-resident CG kernel for systems of K planes on a side x side face: one CTA per
// system ("single": the face's K N values are few) or strips of RS >= 2 rows, at most one CTA per SM.
ResPlan plan_resident(int K, int side, int n_sys, bool hits, bool prec, int nsm) {
  ResPlan P;
  // KCG_RESIDENT: 0 = never, 2 = also the row-strip (grid-barrier) mode.  Default: single-CTA faces
  // only -- the strip mode measured slower than the streaming kernel (medium, L = 8, K = 3: 9.8 vs
  // 7.6 us per iteration; profiles/r02/res_trace_medium.txt), so it is an opt-in experiment.
  int mode = 1;
  if (const char* ev = std::getenv("KCG_RESIDENT")) mode = std::atoi(ev);
  if (mode == 0) return P;
  if (prec && K > 7) return P;
  const size_t lim = 220 * 1024;  // dynamic smem budget (static: ~3 KB)
  int best_rs = 0;
  if ((size_t)K * side * side <= 8192 && kcg::res_smem(K, side, side, hits, prec, n_sys) <= lim && n_sys <= nsm)
    best_rs = side;
  int rs0 = 2;  // experiments: KCG_RES_RS = the smallest strip height to consider
  if (const char* ev = std::getenv("KCG_RES_RS")) rs0 = std::max(2, std::atoi(ev));
  for (int rs = rs0; mode == 2 && !best_rs && rs <= side; rs *= 2) {
    const long long grid = (long long)n_sys * (side / rs);
    if (grid <= nsm && grid <= KCG_RES_CTA_MAX && kcg::res_smem(K, rs, side, hits, prec, n_sys) <= lim) best_rs = rs;
  }
  if (!best_rs) return P;
  P.nstrip = side / best_rs;
  P.grid = n_sys * P.nstrip;
  P.smem = kcg::res_smem(K, best_rs, side, hits, prec, n_sys);
  int nb = 0;
  if (kcg::res_kernel_config(K, hits, prec, P.smem, &nb) != cudaSuccess || nb < 1 || (long long)nb * nsm < P.grid) {
    cudaGetLastError();
    return ResPlan{};
  }
  P.on = true;
  return P;
}

// Shared body of kron_cg_create / kron_cg_create_slab.
kcg_status create_impl(const kcg_desc* d, const kcg_slab* sl, const double* A_host, const double* T_host,
                       const double* phi_host, const double* kappa2_host, const double* hits_dev, void* workspace_dev,
                       size_t ws_bytes, void* stream, kcg_ctx** out) {
  Nvtx nv_("kcg:create");
  if (!out) return KCG_E_ARG;
  *out = nullptr;
  kcg_ctx* c = new kcg_ctx();
  std::string why;
  auto fail = [&](kcg_status st, const std::string& msg) {
    c->err = msg;
    *out = c;  // hand back the ctx so the caller can read kcg_last_error, then destroy
    return st;
  };
  if (!desc_ok(d, &why)) return fail(KCG_E_SHAPE, why);
  c->d = *d;
  if (!config_ok(d, &why)) return fail(KCG_E_CONFIG, why);
  const int G = sl ? sl->nranks : 1;
  if (!slab_ok(d, G, &why)) return fail(KCG_E_SHAPE, why);
  if (sl && d->prior == KCG_PRIOR_D2) return fail(KCG_E_CONFIG, "row slabs are built for KCG_PRIOR_LAPLACIAN");
  if (sl && d->cg_variant == KCG_CG_HS) return fail(KCG_E_CONFIG, "row slabs run the single-pass CG variant only");
  if (sl && d->layout == KCG_LAYOUT_NESTED)
    return fail(KCG_E_CONFIG, "row slabs need KCG_LAYOUT_ROW_MAJOR (a NESTED face is not split into row slabs)");
  if (sl && (sl->rank0 < 0 || sl->nlocal < 1 || sl->rank0 + sl->nlocal > G || (sl->nlocal != 1 && sl->nlocal != G)))
    return fail(KCG_E_CONFIG, "slab: need 0 <= rank0, rank0 + nlocal <= nranks and nlocal in {1, nranks}");
  if (!A_host || !T_host || !phi_host || !kappa2_host) return fail(KCG_E_ARG, "null parameter pointer");
  const int P = d->n_patches, n = d->n_freq, k = d->n_comp;
  if (!finite_all(A_host, (size_t)P * n * k) || !finite_all(T_host, (size_t)P * n) ||
      !finite_all(phi_host, (size_t)P * k) || !finite_all(kappa2_host, P))
    return fail(KCG_E_NONFINITE, "non-finite A, noise_prec, prior_scale or kappa2");
  for (int i = 0; i < P * n; ++i)
    if (!(T_host[i] > 0)) return fail(KCG_E_ARG, "noise_prec must be > 0");
  for (int i = 0; i < P * k; ++i)
    if (!(phi_host[i] > 0)) return fail(KCG_E_ARG, "prior_scale must be > 0");
  for (int i = 0; i < P; ++i)
    if (!(kappa2_host[i] >= 0)) return fail(KCG_E_ARG, "kappa2 must be >= 0");

  const bool d2 = d->prior == KCG_PRIOR_D2;
  c->slab = sl != nullptr;
  c->nranks = G;
  c->rank0 = sl ? sl->rank0 : 0;
  c->nlocal = sl ? sl->nlocal : 1;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  c->side = 1 << d->level;
  c->rows = c->side / G;
  c->ghost = c->slab ? KCG_HALO : 0;
  c->pitch = c->side < 2 ? 2 : c->side;
  c->N = (size_t)c->rows * c->side;
  c->P = P; c->n = n; c->k = k;
  c->L = layout_of(d, G);
  c->ws_need = c->L.total;
  c->ws_bytes = ws_bytes;
  if (ws_bytes < c->L.total) return fail(KCG_E_SHAPE, "workspace too small (kron_cg_workspace_size)");
  if (c->slab) {
    c->peer_ws.resize(G);
    for (int g = 0; g < G; ++g) {
      c->peer_ws[g] = reinterpret_cast<char*>(sl->peer_ws[g]);
      if (!c->peer_ws[g]) return fail(KCG_E_ARG, "slab: null peer workspace");
      if (reinterpret_cast<uintptr_t>(c->peer_ws[g]) % kAlign) return fail(KCG_E_ARG, "workspace not 256-byte aligned");
    }
  } else {
    if (!workspace_dev) return fail(KCG_E_ARG, "null workspace");
    if (reinterpret_cast<uintptr_t>(workspace_dev) % kAlign) return fail(KCG_E_ARG, "workspace not 256-byte aligned");
    c->peer_ws.assign(1, reinterpret_cast<char*>(workspace_dev));
  }
  for (int j = 0; j < c->nlocal; ++j) {
    c->R.push_back(carve(c->peer_ws[c->rank0 + j], c->L, c->rank0 + j, c->rows, d->host_staging != 0,
                         d->layout == KCG_LAYOUT_NESTED));
    // hits [nlocal][P][rows + 2 ghost][side] (ghost rows = the face's rows beyond the slab, 0 outside)
    c->R.back().hits = hits_dev ? hits_dev + (size_t)j * P * (c->rows + 2 * c->ghost) * c->side : nullptr;
  }

  // setup step a1 (host, once): M = A^T T A, E = T A, eigh(M, P), E_syl = T A W, block-Jacobi inverses
  std::vector<SysParams> pk(P), ps((size_t)P * k);
  std::vector<double> Ek((size_t)P * n * k), Es((size_t)P * n * k);
  c->rho.assign((size_t)P * k, 0.0);
  c->W.assign((size_t)P * k * k, 0.0);
  for (int p = 0; p < P; ++p) {
    const double* A = A_host + (size_t)p * n * k;
    const double* T = T_host + (size_t)p * n;
    const double* phi = phi_host + (size_t)p * k;
    std::vector<double> M((size_t)k * k, 0.0);
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        double v = 0.0;
        for (int f = 0; f < n; ++f) v += A[f * k + a] * T[f] * A[f * k + b];
        M[a * k + b] = v;
      }
    for (int f = 0; f < n; ++f)
      for (int a = 0; a < k; ++a) Ek[((size_t)p * n + f) * k + a] = T[f] * A[f * k + a];
    double* rho = &c->rho[(size_t)p * k];
    double* W = &c->W[(size_t)p * k * k];
    eigh_MP(k, M.data(), phi, rho, W);
    for (int f = 0; f < n; ++f)
      for (int i = 0; i < k; ++i) {
        double v = 0.0;
        for (int a = 0; a < k; ++a) v += Ek[((size_t)p * n + f) * k + a] * W[a * k + i];
        Es[((size_t)p * n + f) * k + i] = v;
      }
    SysParams& sk = pk[p];
    std::memset(&sk, 0, sizeof sk);
    for (int e = 0; e < k * k; ++e) sk.M[e] = M[e];
    for (int a = 0; a < k; ++a) sk.tau[a] = phi[a];
    sk.kappa2 = kappa2_host[p];
    sk.hits_plane = p;
    set_block_jacobi(k, M.data(), phi, kappa2_host[p], &sk, d2);
    for (int i = 0; i < k; ++i) {
      SysParams& sy = ps[(size_t)p * k + i];
      std::memset(&sy, 0, sizeof sy);
      sy.M[0] = rho[i];
      sy.tau[0] = 1.0;
      sy.kappa2 = kappa2_host[p];
      sy.hits_plane = p;
      set_block_jacobi(1, sy.M, sy.tau, sy.kappa2, &sy, d2);
    }
  }
  // Alg. Kohler (reading R33): canonical real Schur factor S^ = W R W^T of S^ = M P^{-1}:
  // W = Q factor (modified Gram-Schmidt, positive diagonal) of the Lemma-2 eigenvectors U = P W_eig
  // (ascending rho), R = W^T S^ W upper triangular; E = T A P^{-1} W so that F^ = Y^ W = Y E.
  std::vector<SysParams> pko((size_t)P * k);
  std::vector<double> Eko((size_t)P * n * k), Rko((size_t)P * k * k), Wko((size_t)P * k * k);
  for (int p = 0; p < P; ++p) {
    const double* A = A_host + (size_t)p * n * k;
    const double* T = T_host + (size_t)p * n;
    const double* phi = phi_host + (size_t)p * k;
    const double* We = &c->W[(size_t)p * k * k];
    std::vector<double> M((size_t)k * k, 0.0), Q((size_t)k * k, 0.0);
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        double v = 0.0;
        for (int f = 0; f < n; ++f) v += A[f * k + a] * T[f] * A[f * k + b];
        M[a * k + b] = v;
      }
    for (int i = 0; i < k; ++i) {  // modified Gram-Schmidt on u_i = P w_i
      std::vector<double> v(k);
      for (int a = 0; a < k; ++a) v[a] = phi[a] * We[a * k + i];
      for (int j = 0; j < i; ++j) {
        double d = 0.0;
        for (int a = 0; a < k; ++a) d += Q[a * k + j] * v[a];
        for (int a = 0; a < k; ++a) v[a] -= d * Q[a * k + j];
      }
      double nr = 0.0;
      for (int a = 0; a < k; ++a) nr += v[a] * v[a];
      nr = std::sqrt(nr);
      for (int a = 0; a < k; ++a) Q[a * k + i] = v[a] / nr;
    }
    double* Rp = &Rko[(size_t)p * k * k];
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) {  // R = Q^T (M P^{-1}) Q
        double v = 0.0;
        for (int a = 0; a < k; ++a)
          for (int b = 0; b < k; ++b) v += Q[a * k + i] * M[a * k + b] / phi[b] * Q[b * k + j];
        Rp[i * k + j] = v;
      }
    for (int e = 0; e < k * k; ++e) Wko[(size_t)p * k * k + e] = Q[e];
    for (int f = 0; f < n; ++f)
      for (int i = 0; i < k; ++i) {
        double v = 0.0;
        for (int a = 0; a < k; ++a) v += T[f] * A[f * k + a] / phi[a] * Q[a * k + i];
        Eko[((size_t)p * n + f) * k + i] = v;
      }
    for (int i = 0; i < k; ++i) {
      SysParams& sy = pko[(size_t)i * P + p];
      std::memset(&sy, 0, sizeof sy);
      sy.M[0] = Rp[i * k + i];
      sy.tau[0] = 1.0;
      sy.kappa2 = kappa2_host[p];
      sy.hits_plane = p;
      set_block_jacobi(1, sy.M, sy.tau, sy.kappa2, &sy, d2);
    }
  }
  kcg_status st;
#define CKC(call, what)                              \
  do {                                               \
    cudaError_t _e = (call);                         \
    if (_e != cudaSuccess) {                         \
      st = cuda_fail(c, _e, what);                   \
      *out = c;                                      \
      return st;                                     \
    }                                                \
  } while (0)
  const size_t planes = (size_t)P * k;
  const int buf_rows = c->rows + 2 * c->ghost;
  for (RankState& R : c->R) {
    if (R.hits_rm && R.hits) {  // NESTED hits -> the kernels' row-major copy
      CKC(kcg::launch_permute(c->stream, R.hits, R.hits_rm, (size_t)P, c->side, false), "permute hits");
      R.hits = R.hits_rm;
    }
    CKC(cudaMemcpyAsync(R.params_kron, pk.data(), P * sizeof(SysParams), cudaMemcpyHostToDevice, c->stream), "H2D");
    CKC(cudaMemcpyAsync(R.params_syl, ps.data(), (size_t)P * k * sizeof(SysParams), cudaMemcpyHostToDevice, c->stream),
        "H2D");
    CKC(cudaMemcpyAsync(R.E_kron, Ek.data(), Ek.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    CKC(cudaMemcpyAsync(R.E_syl, Es.data(), Es.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    CKC(cudaMemcpyAsync(R.W_dev, c->W.data(), c->W.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    CKC(cudaMemcpyAsync(R.params_koh, pko.data(), pko.size() * sizeof(SysParams), cudaMemcpyHostToDevice, c->stream),
        "H2D");
    CKC(cudaMemcpyAsync(R.E_koh, Eko.data(), Eko.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    CKC(cudaMemcpyAsync(R.R_koh, Rko.data(), Rko.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    CKC(cudaMemcpyAsync(R.W_koh, Wko.data(), Wko.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    if (c->slab) {  // ghost rows at the face ends stay zero; flags start at 0 (peers only raise them)
      for (int b = 0; b < 2; ++b) {
        CKC(cudaMemsetAsync(R.r[b], 0, c->L.vec_doubles * 8, c->stream), "memset r");
        CKC(cudaMemsetAsync(R.p[b], 0, c->L.vec_doubles * 8, c->stream), "memset p");
      }
      CKC(cudaMemsetAsync(R.flags, 0, KCG_GMAX * sizeof(unsigned long long), c->stream), "memset flags");
      CKC(cudaMemsetAsync(R.xg_top, 0, planes * c->side * 8, c->stream), "memset xg");
      CKC(cudaMemsetAsync(R.xg_bot, 0, planes * c->side * 8, c->stream), "memset xg");
    }
    // TMA descriptors: Kron boxes span K = k planes, Sylvester boxes one plane.
    for (int i = 0; i < 2; ++i) {
      if (!encode_map(&R.maps_kron.r[i], R.r[i], c->side, buf_rows, c->pitch, planes, k, d2, &why) ||
          !encode_map(&R.maps_kron.p[i], R.p[i], c->side, buf_rows, c->pitch, planes, k, d2, &why) ||
          !encode_map(&R.maps_syl.r[i], R.r[i], c->side, buf_rows, c->pitch, planes, 1, d2, &why) ||
          !encode_map(&R.maps_syl.p[i], R.p[i], c->side, buf_rows, c->pitch, planes, 1, d2, &why))
        return fail(KCG_E_CUDA, why);
    }
    // D2 row-march kernel: the hits planes [P][side][side], one chunk of 32 x KCG_MCH per box
    if (d2 && R.hits && c->side >= 2) {  // box {32 m_cp(K), 1, 1}: the Kronecker and the K = 1 strips differ
      if (!encode_hmap(&R.maps_kron.h, R.hits, c->side, (size_t)P, kcg::m_cp(k), &why) ||
          !encode_hmap(&R.maps_syl.h, R.hits, c->side, (size_t)P, kcg::m_cp(1), &why))
        return fail(KCG_E_CUDA, why);
    }
  }
  if (c->L.lz_slots > 0) {  // block-Lanczos constants: Lemma 2 factor, E = T A P^{-1} (Y^ = Y E)
    std::vector<kcg::LzFace> lf(P);
    std::vector<double> El((size_t)P * n * k);
    for (int p = 0; p < P; ++p) {
      kcg::LzFace& F = lf[p];
      std::memset(&F, 0, sizeof F);
      for (int i = 0; i < k; ++i) {
        F.rho[i] = c->rho[(size_t)p * k + i];
        F.phi[i] = phi_host[(size_t)p * k + i];
        for (int cc = 0; cc < k; ++cc) F.W[cc * k + i] = c->W[((size_t)p * k + cc) * k + i];
      }
      F.kappa2 = kappa2_host[p];
      for (int f = 0; f < n; ++f)
        for (int a = 0; a < k; ++a)
          El[((size_t)p * n + f) * k + a] = T_host[(size_t)p * n + f] * A_host[((size_t)p * n + f) * k + a] / phi_host[(size_t)p * k + a];
    }
    RankState& R = c->R[0];
    CKC(cudaMemcpyAsync(R.lz_prm, lf.data(), P * sizeof(kcg::LzFace), cudaMemcpyHostToDevice, c->stream), "H2D");
    CKC(cudaMemcpyAsync(R.E_lz, El.data(), El.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
    if (!encode_lzmap(&R.lz_map, R.lz_V, c->side, c->pitch, (size_t)c->L.lz_slots * P * k, k, d2, &why))
      return fail(KCG_E_CUDA, why);
    int mgl = 0;
    CKC(kcg::lz_kernel_config(k, hits_dev != nullptr, d2, &mgl, &c->smem_lz), "lanczos kernel config");
    c->grid_lz = std::max(1, mgl);
    if (const char* ev = std::getenv("KCG_LZ_GRID")) c->grid_lz = std::max(1, std::min(c->grid_lz, std::atoi(ev)));  // diagnostics
    c->tiles_x_lz = (c->side + KCG_TX - 1) / KCG_TX;
    c->tiles_y_lz = (c->side + kcg::lz_tile_y(k, d2) - 1) / kcg::lz_tile_y(k, d2);
  }
  if (hits_dev) {  // hit counts must be finite and > 0 (G is SPD only then)
    for (RankState& R : c->R) {
      CKC(cudaMemsetAsync(R.sync, 0, sizeof(unsigned), c->stream), "memset");
      for (int p = 0; p < P; ++p)  // the slab's own rows (ghost rows at the face ends are zero)
        CKC(kcg::launch_count_nonpositive(c->stream, hits_dev + (size_t)(&R - &c->R[0]) * P * buf_rows * c->side +
                                                         ((size_t)p * buf_rows + c->ghost) * c->side,
                                          (size_t)c->rows * c->side, R.sync),
            "hits check kernel");
      unsigned bad = 0;
      CKC(cudaMemcpyAsync(&bad, R.sync, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream), "D2H");
      CKC(cudaStreamSynchronize(c->stream), "hits check");
      if (bad) return fail(KCG_E_ARG, "hits must be finite and > 0 (" + std::to_string(bad) + " entries are not)");
    }
  }
  CKC(cudaStreamSynchronize(c->stream), "create sync");
  c->tiles_x_kron = tiles_x(c->side, k, d2);
  c->tiles_y_kron = tiles_y(c->rows, k, d2);
  c->tiles_x_syl = tiles_x(c->side, 1, d2);
  c->tiles_y_syl = tiles_y(c->rows, 1, d2);
  int mg = 0;
  const bool prec = d->precond == KCG_PRECOND_BLOCK_JACOBI;
  if (!c->slab && !d2 && d->cg_variant == KCG_CG_SINGLE_PASS) {  // small-problem regime (state in smem)
    int dev = 0, nsm = 0;
    CKC(cudaGetDevice(&dev), "device");
    CKC(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "device attribute");
    c->res_kron = plan_resident(k, c->side, P, hits_dev != nullptr, prec, nsm);
    c->res_syl = plan_resident(1, c->side, P * k, hits_dev != nullptr, prec, nsm);
    c->res_koh = plan_resident(1, c->side, P, hits_dev != nullptr, prec, nsm);
  }
  if (d->cg_variant == KCG_CG_HS) {  // textbook CG variant: its own tile geometry and grid
    c->tiles_x_kron = c->tiles_x_syl = tiles_x(c->side, 1);
    c->tiles_y_kron = (c->rows + kcg::hs_tile_y(k) - 1) / kcg::hs_tile_y(k);
    c->tiles_y_syl = (c->rows + kcg::hs_tile_y(1) - 1) / kcg::hs_tile_y(1);
    CKC(kcg::hs_kernel_config(k, hits_dev != nullptr, prec, d2, P, &mg, &c->smem_kron), "hs kernel config (kron)");
    c->grid_kron = std::max(1, std::min({mg, KCG_HS_GRID_MAX, P * c->tiles_x_kron * c->tiles_y_kron}));
    CKC(kcg::hs_kernel_config(1, hits_dev != nullptr, prec, d2, P * k, &mg, &c->smem_syl), "hs kernel config (sylvester)");
    c->grid_syl = std::max(1, std::min({mg, KCG_HS_GRID_MAX, P * k * c->tiles_x_syl * c->tiles_y_syl}));
    for (int i = 0; i < 4; ++i) CKC(cudaEventCreate(&c->ev[i]), "event create");
    *out = c;
    return KCG_OK;
  }
  CKC(kcg::cg_kernel_config(k, hits_dev != nullptr, prec, c->slab, d2, P, &mg, &c->smem_kron), "cg kernel config (kron)");
  // (D2 row-march kernel: m_groups(K, hits) warp groups per CTA, each a work unit of >= one strip x 16 rows)
  const int wdk = d2 ? kcg::m_groups(k, hits_dev != nullptr) : 1, wds = d2 ? kcg::m_groups(1, hits_dev != nullptr) : 1;
  c->grid_kron = std::max(1, std::min(mg / c->nlocal, (P * c->tiles_x_kron * c->tiles_y_kron + wdk - 1) / wdk));
  CKC(kcg::cg_kernel_config(1, hits_dev != nullptr, prec, c->slab, d2, P * k, &mg, &c->smem_syl),
      "cg kernel config (sylvester)");
  c->grid_syl = std::max(1, std::min(mg / c->nlocal, (P * k * c->tiles_x_syl * c->tiles_y_syl + wds - 1) / wds));
  if (mg < c->nlocal) return fail(KCG_E_CONFIG, "slab: more emulated ranks than co-resident CTAs");
  for (int i = 0; i < 4; ++i) CKC(cudaEventCreate(&c->ev[i]), "event create");
#undef CKC
  *out = c;
  return KCG_OK;
}

}  // namespace

extern "C" {

size_t kron_cg_workspace_size(const kcg_desc* d) {
  std::string why;
  if (!desc_ok(d, &why)) return 0;
  return layout_of(d, 1).total;
}

size_t kron_cg_workspace_size_slab(const kcg_desc* d, int nranks) {
  std::string why;
  if (!desc_ok(d, &why) || !slab_ok(d, nranks, &why)) return 0;
  return layout_of(d, nranks).total;
}

kcg_status kron_cg_create(const kcg_desc* d, const double* A_host, const double* T_host, const double* phi_host,
                          const double* kappa2_host, const double* hits_dev, void* workspace_dev, size_t ws_bytes,
                          void* stream, kcg_ctx** out) {
  return create_impl(d, nullptr, A_host, T_host, phi_host, kappa2_host, hits_dev, workspace_dev, ws_bytes, stream,
                     out);
}

kcg_status kron_cg_create_slab(const kcg_desc* d, const kcg_slab* slab, const double* A_host, const double* T_host,
                               const double* phi_host, const double* kappa2_host, const double* hits_dev,
                               size_t ws_bytes, void* stream, kcg_ctx** out) {
  if (!slab) {
    if (out) *out = nullptr;
    return KCG_E_ARG;
  }
  return create_impl(d, slab, A_host, T_host, phi_host, kappa2_host, hits_dev, nullptr, ws_bytes, stream, out);
}

kcg_status kron_cg_solve(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter, kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return solve_impl(c, ROUTE_KRON, Y, mu, false, tol, max_iter, rep);
}
kcg_status sylvester_solve(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter, kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return solve_impl(c, ROUTE_SYL, Y, mu, false, tol, max_iter, rep);
}
kcg_status sylvester_kohler_solve(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter,
                                  kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return kohler_impl(c, Y, mu, tol, max_iter, rep);
}

kcg_status kron_cg_solve_x0(kcg_ctx* c, const double* Y, const double* x0, double* mu, double tol, int max_iter,
                            kcg_report* rep) {
  if (c) c->nlaunch = 0;
  if (c && !x0) { c->err = "null x0"; return KCG_E_ARG; }
  return solve_impl(c, ROUTE_KRON, Y, mu, false, tol, max_iter, rep, IN_Y, x0);
}

kcg_status kron_cg_solve_b(kcg_ctx* c, const double* b, double* x, double tol, int max_iter, kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return solve_impl(c, ROUTE_KRON, b, x, false, tol, max_iter, rep, IN_B_USER);
}

kcg_status posterior_variance(kcg_ctx* c, int n_probes, unsigned long long seed, double* var, double* scratch,
                              double tol, int max_iter, kcg_report* rep) {
  Nvtx nv_("kcg:posterior_variance");
  if (!c) return KCG_E_ARG;
  c->nlaunch = 0;
  if (!var || !scratch) { c->err = "null var or scratch"; return KCG_E_ARG; }
  if (n_probes < 1) { c->err = "n_probes < 1"; return KCG_E_ARG; }
  if (c->slab) { c->err = "posterior_variance: no row slabs"; return KCG_E_CONFIG; }
  cudaStream_t s = c->stream;
  const RankState& R = c->R[0];
  const size_t planes = (size_t)c->P * c->k, tot = planes * c->N;
  double* z = scratch;
  double* x = scratch + tot;
  double* acc = R.y_rm ? R.y_rm : var;  // row-major accumulator (NESTED: scattered at the end)
  kcg_report sub{}, all{};
  int worst = KCG_OK, maxit = 0;
  double wall = 0.0, loop = 0.0, bytes = 0.0, maxrel = 0.0, maxtrue = 0.0;
  long long sumit = 0;
  std::vector<int> its_probe(c->P), its_max(c->P, 0);  // per-patch iterations: max over the probes
  for (int i = 0; i < n_probes; ++i) {
    CKL(kcg::launch_probe(s, z, c->P, c->k, c->side, c->d.layout == KCG_LAYOUT_NESTED, seed, i), "probe kernel");
    sub = kcg_report{};
    sub.iterations_per = its_probe.data();
    const kcg_status st = solve_impl(c, ROUTE_KRON, z, x, false, tol, max_iter, &sub, IN_B_WORK);
    if (st != KCG_OK && st != KCG_NOT_CONVERGED) return st;
    if (st == KCG_NOT_CONVERGED) worst = KCG_NOT_CONVERGED;
    CKL(kcg::launch_var_accum(s, z, x, acc, tot, i == 0, i == n_probes - 1 ? 1.0 / n_probes : 1.0), "accumulate kernel");
    wall += sub.wall_time_s; loop += sub.loop_time_s; bytes += sub.loop_bytes;
    maxit = std::max(maxit, sub.iterations); sumit += sub.system_iterations;
    maxrel = std::max(maxrel, sub.rel_residual); maxtrue = std::max(maxtrue, sub.rel_residual_true);
    for (int p = 0; p < c->P; ++p) its_max[p] = std::max(its_max[p], its_probe[p]);
  }
  if (R.y_rm) CKL(kcg::launch_permute(s, R.y_rm, var, planes, c->side, true), "permute var");
  CK(cudaStreamSynchronize(s), "posterior variance");
  if (rep) {
    all = sub;
    all.status = worst; all.iterations = maxit; all.system_iterations = sumit;
    all.rel_residual = maxrel; all.rel_residual_true = maxtrue;
    all.wall_time_s = wall; all.loop_time_s = loop; all.loop_bytes = bytes;
    all.iterations_per = rep->iterations_per; all.history = rep->history; all.history_len = 0;
    all.n_systems = c->P;
    all.kernel_launches = c->nlaunch;
    if (all.iterations_per)
      for (int p = 0; p < c->P; ++p) all.iterations_per[p] = its_max[p];
    *rep = all;
  }
  c->err.clear();
  return (kcg_status)worst;
}

kcg_status sylvester_lanczos_solve(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter,
                                   kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return lanczos_impl(c, Y, mu, false, tol, max_iter, rep);
}
kcg_status sylvester_lanczos_solve_host(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter,
                                        kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return lanczos_impl(c, Y, mu, true, tol, max_iter, rep);
}
// Pipelined host entry point: batch i's solve overlaps the H2D copy of batch i+1 and the D2H copy of
// batch i-1 (two staging pairs, two copy streams; the solves themselves stay stream-ordered on the
// context's stream).
kcg_status kron_cg_solve_host_many(kcg_ctx* c, int nbatch, const double* const* Y_host, double* const* mu_host,
                                   double tol, int max_iter, kcg_report* reports) {
  Nvtx nv_("kcg:kron_cg_solve_host_many");
  if (!c) return KCG_E_ARG;
  c->nlaunch = 0;
  if (c->slab || c->d.host_staging != 2) {
    c->err = "kron_cg_solve_host_many needs desc.host_staging = 2 and no row slabs";
    return KCG_E_CONFIG;
  }
  if (nbatch < 1 || !Y_host || !mu_host) { c->err = "nbatch < 1 or null pointer array"; return KCG_E_ARG; }
  for (int i = 0; i < nbatch; ++i)
    if (!Y_host[i] || !mu_host[i]) { c->err = "null Y or mu"; return KCG_E_ARG; }
  RankState& R = c->R[0];
  if (!c->h2d_stream) {
    CK(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking), "stream create");
    CK(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking), "stream create");
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&c->ev_h2d[b], cudaEventDisableTiming), "event create");
      CK(cudaEventCreateWithFlags(&c->ev_d2h[b], cudaEventDisableTiming), "event create");
      CK(cudaEventCreateWithFlags(&c->ev_solved[b], cudaEventDisableTiming), "event create");
    }
  }
  double* Ys[2] = {R.Y_stage, R.Y_stage2};
  double* Ms[2] = {R.mu_stage, R.mu_stage2};
  const size_t yb = (size_t)c->P * c->n * c->N * 8, mb = (size_t)c->P * c->k * c->N * 8;
  cudaStream_t s = c->stream;
  CK(cudaEventRecord(c->ev_solved[1], s), "event");  // the context's stream is past earlier work
  CK(cudaStreamWaitEvent(c->h2d_stream, c->ev_solved[1], 0), "wait");
  CK(cudaMemcpyAsync(Ys[0], Y_host[0], yb, cudaMemcpyHostToDevice, c->h2d_stream), "H2D Y");
  CK(cudaEventRecord(c->ev_h2d[0], c->h2d_stream), "event");
  kcg_status worst = KCG_OK;
  // D2H of batch j's mu on the copy stream, after its solve (event ev_solved[j & 1])
  auto d2h = [&](int j) -> kcg_status {
    CK(cudaStreamWaitEvent(c->d2h_stream, c->ev_solved[j & 1], 0), "wait");
    CK(cudaMemcpyAsync(mu_host[j], Ms[j & 1], mb, cudaMemcpyDeviceToHost, c->d2h_stream), "D2H mu");
    CK(cudaEventRecord(c->ev_d2h[j & 1], c->d2h_stream), "event");
    return KCG_OK;
  };
  for (int i = 0; i < nbatch; ++i) {
    const int b = i & 1;
    CK(cudaStreamWaitEvent(s, c->ev_h2d[b], 0), "wait");
    if (i >= 2) CK(cudaStreamWaitEvent(s, c->ev_d2h[b], 0), "wait");  // mu of batch i-2 copied out
    kcg_report tmp{};
    kcg_report* rp = reports ? reports + i : &tmp;
    c->nlaunch = 0;  // per batch: rp->kernel_launches counts this solve's launches
    // once solve i is queued: batch i-1's D2H, then batch i+1's H2D into staging buffer b^1 (read by
    // solve i-1, which has returned)
    const std::function<kcg_status()> hook = [&]() -> kcg_status {
      if (i >= 1) {
        const kcg_status e = d2h(i - 1);
        if (e != KCG_OK) return e;
      }
      if (i + 1 < nbatch) {
        CK(cudaMemcpyAsync(Ys[b ^ 1], Y_host[i + 1], yb, cudaMemcpyHostToDevice, c->h2d_stream), "H2D Y");
        CK(cudaEventRecord(c->ev_h2d[b ^ 1], c->h2d_stream), "event");
      }
      return KCG_OK;
    };
    const kcg_status st = solve_impl(c, ROUTE_KRON, Ys[b], Ms[b], false, tol, max_iter, rp, IN_Y, nullptr, &hook);
    if (st != KCG_OK && st != KCG_NOT_CONVERGED) {
      cudaStreamSynchronize(c->h2d_stream);
      cudaStreamSynchronize(c->d2h_stream);
      return st;
    }
    if (st == KCG_NOT_CONVERGED) worst = st;
    CK(cudaEventRecord(c->ev_solved[b], s), "event");
  }
  {
    const kcg_status e = d2h(nbatch - 1);
    if (e != KCG_OK) return e;
  }
  CK(cudaStreamSynchronize(c->d2h_stream), "D2H");
  CK(cudaStreamSynchronize(c->h2d_stream), "H2D");
  c->err.clear();
  return worst;
}

kcg_status kron_cg_solve_host(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter, kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return solve_impl(c, ROUTE_KRON, Y, mu, true, tol, max_iter, rep);
}
kcg_status sylvester_solve_host(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter,
                                kcg_report* rep) {
  if (c) c->nlaunch = 0;
  return solve_impl(c, ROUTE_SYL, Y, mu, true, tol, max_iter, rep);
}

kcg_status kron_cg_apply(kcg_ctx* c, const double* x, double* y) {
  Nvtx nv_("kcg:kron_cg_apply");
  if (!c) return KCG_E_ARG;
  if (!x || !y) { c->err = "null x or y"; return KCG_E_ARG; }
  if (x == y) { c->err = "x and y must not alias"; return KCG_E_ARG; }
  const size_t stride = (size_t)c->P * c->k * c->N;
  if (c->slab) {
    const unsigned long long tag0 = (++c->solve_id) << 32;
    const kcg_status e = exchange_x_rows(c, x, stride, tag0 + kPostTag);
    if (e != KCG_OK) return e;
  }
  for (int j = 0; j < c->nlocal; ++j) {
    const RankState& R = c->R[j];
    const double* xi = x + j * stride;
    double* yo = y + j * stride;
    if (R.x_rm) {  // NESTED: gather, apply in row-major, scatter
      CKL(kcg::launch_permute(c->stream, xi, R.x_rm, (size_t)c->P * c->k, c->side, false), "permute x");
      xi = R.x_rm;
      yo = R.y_rm;
    }
    CKL(kcg::launch_apply(c->k, c->stream, R.params_kron, xi, yo, R.hits, c->P, geom_of(c, R),
                         c->slab ? R.xg_top : nullptr, c->slab ? R.xg_bot : nullptr),
       "apply kernel");
    if (R.x_rm) CKL(kcg::launch_permute(c->stream, R.y_rm, y + j * stride, (size_t)c->P * c->k, c->side, true), "permute y");
  }
  if (c->slab) {  // nobody rewrites a neighbour's xg_* before everyone is done reading it
    const unsigned long long tag0 = c->solve_id << 32;
    CKL(kcg::launch_xrank_sync(c->stream, xsync_of(c, tag0 + kPostTag + 1)), "rendezvous kernel");
  }
  CK(cudaStreamSynchronize(c->stream), "apply");
  return KCG_OK;
}

kcg_status kron_cg_rhs(kcg_ctx* c, const double* Y, double* b) {
  if (!c) return KCG_E_ARG;
  if (!Y || !b) { c->err = "null Y or b"; return KCG_E_ARG; }
  for (int j = 0; j < c->nlocal; ++j) {
    const RankState& R = c->R[j];
    SlabGeom g{c->side, c->rows, R.row0, c->side, 0, c->ghost, c->d.layout == KCG_LAYOUT_NESTED,
               c->d.prior == KCG_PRIOR_D2};  // dense b
    double* bo = R.y_rm ? R.y_rm : b + j * (size_t)c->P * c->k * c->N;
    CKL(kcg::launch_rhs(c->k, c->stream, Y + j * (size_t)c->P * c->n * c->N, R.E_kron, R.hits, bo, nullptr, nullptr,
                       c->P, c->n, g),
       "rhs kernel");
    if (R.y_rm) CKL(kcg::launch_permute(c->stream, R.y_rm, b + j * (size_t)c->P * c->k * c->N, (size_t)c->P * c->k,
                                       c->side, true), "permute b");
  }
  CK(cudaStreamSynchronize(c->stream), "rhs");
  return KCG_OK;
}

kcg_status sylvester_factor(kcg_ctx* c, double* rho, double* W) {
  if (!c) return KCG_E_ARG;
  if (!rho || !W) { c->err = "null output"; return KCG_E_ARG; }
  std::memcpy(rho, c->rho.data(), c->rho.size() * 8);
  std::memcpy(W, c->W.data(), c->W.size() * 8);
  return KCG_OK;
}

kcg_status kcg_ipc_export(const void* dev_ptr, unsigned char handle[64], size_t* offset) {
  if (!dev_ptr || !handle || !offset) return KCG_E_ARG;
  CUdeviceptr base = 0;
  size_t size = 0;
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return KCG_E_CUDA;
    range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  }
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) return KCG_E_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return KCG_E_CUDA;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::memcpy(handle, &h, 64);
  *offset = reinterpret_cast<uintptr_t>(dev_ptr) - static_cast<uintptr_t>(base);
  return KCG_OK;
}

kcg_status kcg_ipc_import(const unsigned char handle[64], size_t offset, void** dev_ptr, void** base_out) {
  if (!handle || !dev_ptr || !base_out) return KCG_E_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return KCG_E_CUDA;
  *base_out = base;
  *dev_ptr = static_cast<char*>(base) + offset;
  return KCG_OK;
}

kcg_status kcg_ipc_close(void* base) {
  if (!base) return KCG_E_ARG;
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? KCG_OK : KCG_E_CUDA;
}

const char* kcg_last_error(const kcg_ctx* c) { return c ? c->err.c_str() : "null context"; }

const char* kcg_status_string(int s) {
  switch (s) {
    case KCG_OK: return "KCG_OK";
    case KCG_NOT_CONVERGED: return "KCG_NOT_CONVERGED";
    case KCG_E_ARG: return "KCG_E_ARG";
    case KCG_E_SHAPE: return "KCG_E_SHAPE";
    case KCG_E_CONFIG: return "KCG_E_CONFIG";
    case KCG_E_NONFINITE: return "KCG_E_NONFINITE";
    case KCG_E_BREAKDOWN: return "KCG_E_BREAKDOWN";
    case KCG_E_CUDA: return "KCG_E_CUDA";
    case KCG_E_STATE: return "KCG_E_STATE";
    default: return "KCG_UNKNOWN";
  }
}

// Diagnostic (not part of the ABI header): the per-system CG state after the last solve, as
// doubles {bnorm2, gamma, alpha, beta, rel, iters, status, parity, alpha_last} per system.
KCG_API int kcg_debug_state(const kcg_ctx* c, double* out, int max_sys) {
  if (!c || !out) return 0;
  const int n = std::min(max_sys, (int)c->st_host.size());
  for (int i = 0; i < n; ++i) {
    const SysState& z = c->st_host[i];
    double* o = out + 9 * i;
    o[0] = z.bnorm2; o[1] = z.gamma; o[2] = z.alpha; o[3] = z.beta; o[4] = z.rel;
    o[5] = z.iters; o[6] = z.status; o[7] = z.parity; o[8] = z.alpha_last;
  }
  return n;
}

// Diagnostic (not part of the ABI header): launch configuration of the CG kernel per route:
// out = {grid_kron, grid_syl, smem_kron, smem_syl, sm_count, resident strips kron / syl / kohler}
// (grids per rank in slab mode).
KCG_API int kcg_debug_config(const kcg_ctx* c, long long* out) {
  if (!c || !out) return 0;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  out[0] = c->grid_kron; out[1] = c->grid_syl; out[2] = (long long)c->smem_kron; out[3] = (long long)c->smem_syl;
  out[4] = nsm;
  // the shared-memory-resident plans (small-problem regime): strips per system, 0 = streaming kernel
  out[5] = c->res_kron.on ? c->res_kron.nstrip : 0;
  out[6] = c->res_syl.on ? c->res_syl.nstrip : 0;
  out[7] = c->res_koh.on ? c->res_koh.nstrip : 0;
  return 8;
}

// Row-slab plumbing check without any waiting kernel (safe with several ranks on one GPU): each
// local rank stores value + rank into slot [rank] of EVERY rank's rslots area (peer stores through
// the IPC-mapped workspaces), then -- after the caller's host barrier -- kcg_slab_probe_get copies
// this process's first local rank's slots [0, nranks) to the host.
kcg_status kcg_slab_probe_put(kcg_ctx* c, double value) {
  if (!c || !c->slab) return KCG_E_STATE;
  cudaStream_t s = c->stream;
  std::vector<double> v(c->nlocal);
  for (int j = 0; j < c->nlocal; ++j) {
    RankState& R = c->R[j];
    v[j] = value + R.rank;
    CK(cudaMemcpyAsync(R.resid_out, &v[j], 8, cudaMemcpyHostToDevice, s), "H2D");
    kcg::XrankPut Pt{};
    for (int g = 0; g < c->nranks; ++g) Pt.dst[g] = peer_ptr<double>(c, g, c->L.rslots);
    Pt.src = R.resid_out;
    Pt.count = 1;
    Pt.rank = R.rank;
    Pt.nranks = c->nranks;
    CKL(kcg::launch_put(s, Pt), "put kernel");
  }
  CK(cudaStreamSynchronize(s), "probe sync");
  return KCG_OK;
}

kcg_status kcg_slab_probe_get(kcg_ctx* c, double* out_host) {
  if (!c || !c->slab || !out_host) return KCG_E_STATE;
  CK(cudaMemcpy(out_host, c->R[0].rslots, (size_t)c->nranks * 8, cudaMemcpyDeviceToHost), "D2H");
  return KCG_OK;
}

// Diagnostic (not part of the ABI header): copy the phase trace of the last solve (KCG_TRACE builds).
KCG_API int kcg_debug_trace(kcg_ctx* c, long long* out, int max_iters) {
  if (!c || !c->R[0].trace || !out) return 0;
  const int n = std::min(max_iters, KCG_TRACE_ITERS);
  cudaMemcpy(out, c->R[0].trace, (size_t)n * KCG_TRACE_COLS * 8, cudaMemcpyDeviceToHost);
  return KCG_TRACE_COLS;
}

void kron_cg_destroy(kcg_ctx* c) {
  if (!c) return;
  for (int i = 0; i < 4; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
    if (c->ev_d2h[i]) cudaEventDestroy(c->ev_d2h[i]);
    if (c->ev_solved[i]) cudaEventDestroy(c->ev_solved[i]);
  }
  if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  delete c;
}

}  // extern "C"
