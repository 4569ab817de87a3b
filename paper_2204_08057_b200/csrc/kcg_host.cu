// Host runtime and C ABI of libkroncg (see include/kroncg.h for the contract).
//
// Responsibilities: descriptor/argument validation, workspace carving (caller-owned device memory,
// no allocation after create), the small dense algebra of setup step a1 (M = A^T T A, E = T A,
// Lemma 2's eigh(M, P) by a cyclic Jacobi eigensolver), TMA descriptor encoding, stream-ordered
// kernel launches, CUDA-event timing and the solve report.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/kroncg.h"
#include "kcg_internal.h"

using kcg::CgArgs;
using kcg::CgMaps;
using kcg::SysParams;
using kcg::SysState;

struct kcg_ctx {
  kcg_desc d;
  cudaStream_t stream = nullptr;
  int side = 0, pitch = 0, P = 0, n = 0, k = 0;
  size_t N = 0;
  char* ws = nullptr;
  size_t ws_bytes = 0, ws_need = 0;
  double* r[2] = {nullptr, nullptr};
  double* p[2] = {nullptr, nullptr};
  double* partials = nullptr;
  SysState* state = nullptr;
  double* history = nullptr;
  double* resid_partials = nullptr;
  double* resid_out = nullptr;
  SysParams* params_kron = nullptr;
  SysParams* params_syl = nullptr;
  double* E_kron = nullptr;
  double* E_syl = nullptr;
  double* W_dev = nullptr;
  long long* trace = nullptr;
  unsigned* sync = nullptr;
  double* Y_stage = nullptr;
  double* mu_stage = nullptr;
  const double* hits = nullptr;
  std::vector<double> rho, W;  // host copies [P][k], [P][k][k]
  CgMaps maps_kron, maps_syl;
  int tiles_x_kron = 0, tiles_y_kron = 0, tiles_x_syl = 0, tiles_y_syl = 0;
  int grid_kron = 0, grid_syl = 0;
  size_t smem_kron = 0, smem_syl = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<SysState> st_host;
  std::vector<double> resid_host;
  std::string err;
};

namespace {

const size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {
  size_t r0, r1, p0, p1, partials, state, history, resid_partials, resid_out, params_kron, params_syl, E_kron,
      E_syl, W, Y_stage, mu_stage, trace, sync, total;
  size_t vec_doubles, partial_doubles;
};

bool desc_ok(const kcg_desc* d, std::string* why) {
  char buf[256];
  if (!d) { *why = "desc is NULL"; return false; }
  if (d->level < 0 || d->level > 12) { snprintf(buf, sizeof buf, "level %d outside [0,12]", d->level); *why = buf; return false; }
  if (d->n_freq < 1 || d->n_freq > 64) { *why = "n_freq outside [1,64]"; return false; }
  if (d->n_comp < 1 || d->n_comp > KCG_KMAX) { *why = "n_comp outside [1,8]"; return false; }
  if (d->n_comp > d->n_freq) { *why = "n_comp > n_freq (A cannot have full column rank)"; return false; }
  if (d->n_patches < 1 || d->n_patches > 64) { *why = "n_patches outside [1,64]"; return false; }
  if (d->history_cap < 0) { *why = "history_cap < 0"; return false; }
  return true;
}

bool config_ok(const kcg_desc* d, std::string* why) {
  if (d->prior != KCG_PRIOR_LAPLACIAN) { *why = "only KCG_PRIOR_LAPLACIAN is built"; return false; }
  if (d->layout != KCG_LAYOUT_ROW_MAJOR) { *why = "only KCG_LAYOUT_ROW_MAJOR is built"; return false; }
  if (d->precond != KCG_PRECOND_NONE && d->precond != KCG_PRECOND_BLOCK_JACOBI) { *why = "unknown precond"; return false; }
  if (d->precond == KCG_PRECOND_BLOCK_JACOBI && d->n_comp > 7) {
    *why = "KCG_PRECOND_BLOCK_JACOBI is built for n_comp <= 7 (shared-memory budget)";
    return false;
  }
  return true;
}

// Tile grid of the CG kernel (64 x cg_tile_y(K) tiles).
int tiles_x(int side, int K) { return (side + KCG_TX - 1) / KCG_TX; }
int tiles_y(int side, int K) { return (side + kcg::cg_tile_y(K) - 1) / kcg::cg_tile_y(K); }

Layout layout_of(const kcg_desc* d) {
  Layout L{};
  const int side = 1 << d->level;
  const int pitch = side < 2 ? 2 : side;  // TMA global strides must be multiples of 16 bytes
  const size_t N = (size_t)side * side;
  const size_t P = d->n_patches, n = d->n_freq, k = d->n_comp;
  L.vec_doubles = P * k * (size_t)pitch * side;
  const size_t tk = (size_t)tiles_x(side, (int)k) * tiles_y(side, (int)k);
  const size_t ts = (size_t)tiles_x(side, 1) * tiles_y(side, 1);
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
  L.resid_partials = take(P * (size_t)kcg::apply_tiles_per_sys(side) * 2 * 8);
  L.resid_out = take(P * 2 * 8);
  L.params_kron = take(P * sizeof(SysParams));
  L.params_syl = take(P * k * sizeof(SysParams));
  L.E_kron = take(P * n * k * 8);
  L.E_syl = take(P * n * k * 8);
  L.W = take(P * k * k * 8);
  L.trace = KCG_TRACE ? take((size_t)KCG_TRACE_ITERS * KCG_TRACE_COLS * 8) : 0;
  if (d->host_staging) {
    L.Y_stage = take(P * n * N * 8);
    L.mu_stage = take(P * k * N * 8);
  } else {
    L.Y_stage = L.mu_stage = 0;
  }
  L.total = off;
  return L;
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

// Pixel-block Jacobi blocks for hits = 1 (reading R10): Kinv_d = (M + (kappa2 + d) diag(tau))^{-1},
// d = 2, 3, 4, stored compactly (K x K each) in sp.Kinv.
void set_block_jacobi(int K, const double* M, const double* tau, double kappa2, SysParams* sp) {
  std::vector<double> A((size_t)K * K), Ai((size_t)K * K);
  double* out = &sp->Kinv[0][0];
  for (int d = 2; d <= 4; ++d) {
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j) A[i * K + j] = M[i * K + j] + (i == j ? (kappa2 + d) * tau[i] : 0.0);
    small_inverse(K, A.data(), Ai.data());
    for (int e = 0; e < K * K; ++e) out[(d - 2) * K * K + e] = Ai[e];
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

bool encode_map(CUtensorMap* m, double* base, int side, int pitch, size_t planes, int K, std::string* why) {
  const int bx = KCG_TX + 2 * KCG_HALO;
  const int by = kcg::cg_tile_y(K) + 2 * KCG_HALO;
  auto enc = get_encode();
  if (!enc) { *why = "cuTensorMapEncodeTiled unavailable"; return false; }
  cuuint64_t dims[3] = {(cuuint64_t)side, (cuuint64_t)side, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * side * 8};
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
bool encode_xmap(CUtensorMap* m, double* base, int side, size_t planes, int K, std::string* why) {
  auto enc = get_encode();
  if (!enc) { *why = "cuTensorMapEncodeTiled unavailable"; return false; }
  cuuint64_t dims[3] = {(cuuint64_t)side, (cuuint64_t)side, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)side * 8, (cuuint64_t)side * side * 8};
  cuuint32_t box[3] = {(cuuint32_t)KCG_TX, (cuuint32_t)kcg::cg_tile_y(K), (cuuint32_t)K};
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

enum Route { ROUTE_KRON = 0, ROUTE_SYL = 1 };

kcg_status solve_impl(kcg_ctx* c, Route route, const double* Y_in, double* mu_out, bool host_io, double tol,
                      int max_iter, kcg_report* rep) {
  if (!c) return KCG_E_ARG;
  if (!Y_in || !mu_out) { c->err = "null Y or mu"; return KCG_E_ARG; }
  if (!(tol > 0.0) || !std::isfinite(tol)) { c->err = "tol must be finite and > 0"; return KCG_E_ARG; }
  if (max_iter < 0) { c->err = "max_iter < 0"; return KCG_E_ARG; }
  if (host_io && !c->d.host_staging) { c->err = "host entry point needs desc.host_staging = 1"; return KCG_E_CONFIG; }
  cudaStream_t s = c->stream;
  const int P = c->P, n = c->n, k = c->k, side = c->side;
  const size_t N = c->N;
  const double* Y = host_io ? c->Y_stage : Y_in;
  double* mu = host_io ? c->mu_stage : mu_out;

  CK(cudaEventRecord(c->ev[0], s), "event");
  if (host_io) CK(cudaMemcpyAsync(c->Y_stage, Y_in, (size_t)P * n * N * 8, cudaMemcpyHostToDevice, s), "H2D Y");
  const bool kron = route == ROUTE_KRON;
  CK(kcg::launch_rhs(k, s, Y, kron ? c->E_kron : c->E_syl, c->hits, c->r[0], c->p[0], mu, P, n, side, c->pitch),
     "rhs kernel");
  CK(cudaEventRecord(c->ev[1], s), "event");

  CgArgs a;
  a.params = kron ? c->params_kron : c->params_syl;
  a.x = mu;
  a.rbuf[0] = c->r[0]; a.rbuf[1] = c->r[1];
  a.pbuf[0] = c->p[0]; a.pbuf[1] = c->p[1];
  a.partials = c->partials;
  a.state_out = c->state;
  a.history = c->history;
  a.history_cap = c->d.history_cap;
  a.hits = c->hits;
  a.side = side;
  a.pitch = c->pitch;
  a.rows = side;
  a.row0 = 0;
  a.ghost = 0;
  a.n_sys = kron ? P : P * k;
  a.tiles_x = kron ? c->tiles_x_kron : c->tiles_x_syl;
  a.tiles_y = kron ? c->tiles_y_kron : c->tiles_y_syl;
  a.tiles_per_sys = a.tiles_x * a.tiles_y;
  a.max_iter = max_iter;
  a.tol2 = tol * tol;
  a.trace = c->trace;
  a.sync = c->sync;
  CK(cudaMemsetAsync(c->sync, 0, 4 * sizeof(unsigned), s), "memset sync");
  const int Kk = kron ? k : 1;
  CgMaps& maps = kron ? c->maps_kron : c->maps_syl;
  a.x_tma = 0;
  if (side >= 2 && (reinterpret_cast<uintptr_t>(mu) % 16) == 0) {
    std::string why;
    if (!encode_xmap(&maps.x, mu, side, (size_t)P * k, Kk, &why)) { c->err = why; return KCG_E_CUDA; }
    a.x_tma = 1;
  }
  CK(kcg::launch_cg(Kk, c->d.precond == KCG_PRECOND_BLOCK_JACOBI, s, a, maps, kron ? c->grid_kron : c->grid_syl,
                    kron ? c->smem_kron : c->smem_syl),
     "cg kernel");
  CK(cudaEventRecord(c->ev[2], s), "event");
  if (KCG_X2) CK(kcg::launch_xfix(Kk, s, c->state, c->p[0], c->p[1], mu, a.n_sys, side, c->pitch), "x fix-up kernel");
  if (!kron) CK(kcg::launch_backtransform(k, s, c->W_dev, mu, P, side), "backtransform kernel");
  CK(kcg::launch_resid(k, s, c->params_kron, mu, Y, c->E_kron, c->hits, c->resid_partials, c->resid_out, P, n, side),
     "residual kernel");
  c->st_host.resize(a.n_sys);
  c->resid_host.resize((size_t)P * 2);
  CK(cudaMemcpyAsync(c->st_host.data(), c->state, a.n_sys * sizeof(SysState), cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaMemcpyAsync(c->resid_host.data(), c->resid_out, (size_t)P * 2 * 8, cudaMemcpyDeviceToHost, s), "D2H");
  if (host_io) CK(cudaMemcpyAsync(mu_out, c->mu_stage, (size_t)P * k * N * 8, cudaMemcpyDeviceToHost, s), "D2H mu");
  CK(cudaEventRecord(c->ev[3], s), "event");
  CK(cudaStreamSynchronize(s), "solve");

  // report
  int worst = KCG_OK, maxit = 0, allconv = 1;
  long long sumit = 0, passes = 0, xpasses = 0;
  double maxrel = 0.0;
  for (int i = 0; i < a.n_sys; ++i) {
    const SysState& z = c->st_host[i];
    maxit = std::max(maxit, z.iters);
    sumit += z.iters;
    passes += z.iters + 1;
    xpasses += KCG_X2 ? z.iters / 2 : z.iters;
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
    const double r2 = c->resid_host[2 * p], b2 = c->resid_host[2 * p + 1];
    maxtrue = std::max(maxtrue, b2 > 0 ? std::sqrt(r2 / b2) : std::sqrt(r2));
  }
  if (rep) {
    float t03 = 0.f, t12 = 0.f;
    cudaEventElapsedTime(&t03, c->ev[0], c->ev[3]);
    cudaEventElapsedTime(&t12, c->ev[1], c->ev[2]);
    rep->status = worst;
    rep->converged = allconv;
    rep->iterations = maxit;
    rep->n_systems = a.n_sys;
    if (rep->iterations_per)
      for (int i = 0; i < a.n_sys; ++i) rep->iterations_per[i] = c->st_host[i].iters;
    rep->rel_residual = maxrel;
    rep->rel_residual_true = maxtrue;
    rep->wall_time_s = t03 * 1e-3;
    rep->loop_time_s = t12 * 1e-3;
    rep->system_iterations = sumit;
    // per pass: read + write r and p (32 B per pixel and plane); x passes also read + write x
    rep->loop_bytes = (32.0 * (double)passes + 16.0 * (double)xpasses) * (kron ? k : 1) * (double)N;
    rep->peak_mem_bytes = c->ws_need;
    rep->history_len = std::min(maxit, c->d.history_cap);
    if (rep->history && rep->history_len > 0) {
      cudaError_t e = cudaMemcpy(rep->history, c->history, (size_t)rep->history_len * 8, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(c, e, "D2H history");
    }
  }
  c->err.clear();
  return (kcg_status)worst;
}

}  // namespace

extern "C" {

size_t kron_cg_workspace_size(const kcg_desc* d) {
  std::string why;
  if (!desc_ok(d, &why)) return 0;
  return layout_of(d).total;
}

kcg_status kron_cg_create(const kcg_desc* d, const double* A_host, const double* T_host, const double* phi_host,
                          const double* kappa2_host, const double* hits_dev, void* workspace_dev, size_t ws_bytes,
                          void* stream, kcg_ctx** out) {
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
  if (!A_host || !T_host || !phi_host || !kappa2_host) return fail(KCG_E_ARG, "null parameter pointer");
  if (!workspace_dev) return fail(KCG_E_ARG, "null workspace");
  if (reinterpret_cast<uintptr_t>(workspace_dev) % kAlign) return fail(KCG_E_ARG, "workspace not 256-byte aligned");
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
  Layout L = layout_of(d);
  if (ws_bytes < L.total) return fail(KCG_E_SHAPE, "workspace too small (kron_cg_workspace_size)");

  c->stream = reinterpret_cast<cudaStream_t>(stream);
  c->side = 1 << d->level;
  c->pitch = c->side < 2 ? 2 : c->side;
  c->N = (size_t)c->side * c->side;
  c->P = P; c->n = n; c->k = k;
  c->ws = reinterpret_cast<char*>(workspace_dev);
  c->ws_bytes = ws_bytes;
  c->ws_need = L.total;
  c->r[0] = reinterpret_cast<double*>(c->ws + L.r0);
  c->r[1] = reinterpret_cast<double*>(c->ws + L.r1);
  c->p[0] = reinterpret_cast<double*>(c->ws + L.p0);
  c->p[1] = reinterpret_cast<double*>(c->ws + L.p1);
  c->partials = reinterpret_cast<double*>(c->ws + L.partials);
  c->state = reinterpret_cast<SysState*>(c->ws + L.state);
  c->history = reinterpret_cast<double*>(c->ws + L.history);
  c->resid_partials = reinterpret_cast<double*>(c->ws + L.resid_partials);
  c->resid_out = reinterpret_cast<double*>(c->ws + L.resid_out);
  c->params_kron = reinterpret_cast<SysParams*>(c->ws + L.params_kron);
  c->params_syl = reinterpret_cast<SysParams*>(c->ws + L.params_syl);
  c->E_kron = reinterpret_cast<double*>(c->ws + L.E_kron);
  c->E_syl = reinterpret_cast<double*>(c->ws + L.E_syl);
  c->W_dev = reinterpret_cast<double*>(c->ws + L.W);
  if (KCG_TRACE) c->trace = reinterpret_cast<long long*>(c->ws + L.trace);
  c->sync = reinterpret_cast<unsigned*>(c->ws + L.sync);
  if (d->host_staging) {
    c->Y_stage = reinterpret_cast<double*>(c->ws + L.Y_stage);
    c->mu_stage = reinterpret_cast<double*>(c->ws + L.mu_stage);
  }
  c->hits = hits_dev;

  // setup step a1 (host, once): M = A^T T A, E = T A, eigh(M, P), E_syl = T A W
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
    set_block_jacobi(k, M.data(), phi, kappa2_host[p], &sk);
    for (int i = 0; i < k; ++i) {
      SysParams& sy = ps[(size_t)p * k + i];
      std::memset(&sy, 0, sizeof sy);
      sy.M[0] = rho[i];
      sy.tau[0] = 1.0;
      sy.kappa2 = kappa2_host[p];
      sy.hits_plane = p;
      set_block_jacobi(1, sy.M, sy.tau, sy.kappa2, &sy);
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
  CKC(cudaMemcpyAsync(c->params_kron, pk.data(), P * sizeof(SysParams), cudaMemcpyHostToDevice, c->stream), "H2D");
  CKC(cudaMemcpyAsync(c->params_syl, ps.data(), (size_t)P * k * sizeof(SysParams), cudaMemcpyHostToDevice, c->stream),
      "H2D");
  CKC(cudaMemcpyAsync(c->E_kron, Ek.data(), Ek.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
  CKC(cudaMemcpyAsync(c->E_syl, Es.data(), Es.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
  CKC(cudaMemcpyAsync(c->W_dev, c->W.data(), c->W.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
  CKC(cudaStreamSynchronize(c->stream), "create sync");

  // TMA descriptors: Kron boxes span K = k planes, Sylvester boxes one plane.
  const size_t planes = (size_t)P * k;
  for (int i = 0; i < 2; ++i) {
    if (!encode_map(&c->maps_kron.r[i], c->r[i], c->side, c->pitch, planes, k, &why) ||
        !encode_map(&c->maps_kron.p[i], c->p[i], c->side, c->pitch, planes, k, &why) ||
        !encode_map(&c->maps_syl.r[i], c->r[i], c->side, c->pitch, planes, 1, &why) ||
        !encode_map(&c->maps_syl.p[i], c->p[i], c->side, c->pitch, planes, 1, &why))
      return fail(KCG_E_CUDA, why);
  }
  c->tiles_x_kron = tiles_x(c->side, k);
  c->tiles_y_kron = tiles_y(c->side, k);
  c->tiles_x_syl = tiles_x(c->side, 1);
  c->tiles_y_syl = tiles_y(c->side, 1);
  int mg = 0;
  const bool prec = d->precond == KCG_PRECOND_BLOCK_JACOBI;
  CKC(kcg::cg_kernel_config(k, hits_dev != nullptr, prec, P, &mg, &c->smem_kron),
      "cg kernel config (kron)");
  c->grid_kron = std::max(1, std::min(mg, P * c->tiles_x_kron * c->tiles_y_kron));
  CKC(kcg::cg_kernel_config(1, hits_dev != nullptr, prec, P * k, &mg, &c->smem_syl),
      "cg kernel config (sylvester)");
  c->grid_syl = std::max(1, std::min(mg, P * k * c->tiles_x_syl * c->tiles_y_syl));
  for (int i = 0; i < 4; ++i) CKC(cudaEventCreate(&c->ev[i]), "event create");
#undef CKC
  *out = c;
  return KCG_OK;
}

kcg_status kron_cg_solve(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter, kcg_report* rep) {
  return solve_impl(c, ROUTE_KRON, Y, mu, false, tol, max_iter, rep);
}
kcg_status sylvester_solve(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter, kcg_report* rep) {
  return solve_impl(c, ROUTE_SYL, Y, mu, false, tol, max_iter, rep);
}
kcg_status kron_cg_solve_host(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter, kcg_report* rep) {
  return solve_impl(c, ROUTE_KRON, Y, mu, true, tol, max_iter, rep);
}
kcg_status sylvester_solve_host(kcg_ctx* c, const double* Y, double* mu, double tol, int max_iter,
                                kcg_report* rep) {
  return solve_impl(c, ROUTE_SYL, Y, mu, true, tol, max_iter, rep);
}

kcg_status kron_cg_apply(kcg_ctx* c, const double* x, double* y) {
  if (!c) return KCG_E_ARG;
  if (!x || !y) { c->err = "null x or y"; return KCG_E_ARG; }
  if (x == y) { c->err = "x and y must not alias"; return KCG_E_ARG; }
  CK(kcg::launch_apply(c->k, c->stream, c->params_kron, x, y, c->hits, c->P, c->side), "apply kernel");
  CK(cudaStreamSynchronize(c->stream), "apply");
  return KCG_OK;
}

kcg_status kron_cg_rhs(kcg_ctx* c, const double* Y, double* b) {
  if (!c) return KCG_E_ARG;
  if (!Y || !b) { c->err = "null Y or b"; return KCG_E_ARG; }
  CK(kcg::launch_rhs(c->k, c->stream, Y, c->E_kron, c->hits, b, nullptr, nullptr, c->P, c->n, c->side, c->side),
     "rhs kernel");
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
    case KCG_E_NCCL: return "KCG_E_NCCL";
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

// Diagnostic (not part of the ABI header): copy the device SysParams array of a route (0 kron,
// 1 sylvester) into out (at most max_bytes); returns sizeof(SysParams).
KCG_API int kcg_debug_params(const kcg_ctx* c, int route, void* out, size_t max_bytes) {
  if (!c || !out) return 0;
  const size_t n = route == 0 ? (size_t)c->P : (size_t)c->P * c->k;
  cudaMemcpy(out, route == 0 ? c->params_kron : c->params_syl, std::min(max_bytes, n * sizeof(SysParams)),
             cudaMemcpyDeviceToHost);
  return (int)sizeof(SysParams);
}

// Diagnostic (not part of the ABI header): launch configuration of the CG kernel per route:
// out = {grid_kron, grid_syl, smem_kron, smem_syl, sm_count}.
KCG_API int kcg_debug_config(const kcg_ctx* c, long long* out) {
  if (!c || !out) return 0;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  out[0] = c->grid_kron; out[1] = c->grid_syl; out[2] = (long long)c->smem_kron; out[3] = (long long)c->smem_syl;
  out[4] = nsm;
  return 5;
}

// Diagnostic (not part of the ABI header): copy the phase trace of the last solve (KCG_TRACE builds).
KCG_API int kcg_debug_trace(kcg_ctx* c, long long* out, int max_iters) {
  if (!c || !c->trace || !out) return 0;
  const int n = std::min(max_iters, KCG_TRACE_ITERS);
  cudaMemcpy(out, c->trace, (size_t)n * KCG_TRACE_COLS * 8, cudaMemcpyDeviceToHost);
  return KCG_TRACE_COLS;
}

void kron_cg_destroy(kcg_ctx* c) {
  if (!c) return;
  for (int i = 0; i < 4; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  delete c;
}

}  // extern "C"
