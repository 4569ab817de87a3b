#pragma once
// sm_100a fp64 block-Lanczos Sylvester solver -- the paper's Alg. SylvSolver for
//   N_h^{-1} Q0 M + M S^ = Y^,   S^ = A^T T A P^{-1},  Y^ = Y T A P^{-1}     (Eq.(Axb-Sylv))
// with the block Lanczos process in the N_h inner product (Alg. Lanczos, Lemma 1
// P:L317-327), the Galerkin projection T_i Z + Z S^ = E_1 B_0 (Eq.(Sylv-small)), S^ = U R U^{-1}
// (Lemma 2), the residual estimate gamma and M = sum_i V_i G_i
// (Eq.(soln-darstellung)) assembled by rerunning Lanczos or, with the basis
// kept in HBM, by one streaming pass.
//
// B200 formulation (readings R25-R30):
//  * One pass per Lanczos step reads V_{i-1} (tile + 2-pixel halo) and V_{i-2} and writes V_i:
//    W_{i-1} = N^{-1} Q0 V_{i-1} - V_{i-2} B_{i-1}^T and V_i = (W_{i-1} - V_{i-1} H_{i-1}) B_i^{-1} are
//    RECOMPUTED on the tile + 1 ring (never stored), then W_i = N^{-1} Q0 V_i - V_{i-1} B_i^T on the
//    tile: 3 block-vectors of HBM traffic per step (24 K N bytes) instead of the textbook 7+.
//  * ONE reduction per step: the N-weighted Gram of [V_i, W_i] gives H_i = V_i^T N W_i,
//    Gv = V_i^T N V_i and C0 = W_i^T N W_i, and the Cholesky-QR Gram of W_i - V_i H_i follows as
//    C = C0 - 2 H^T H + H^T Gv H (exact algebra; Gv keeps it accurate as orthogonality decays).
//  * gamma by block forward elimination of (T_i + rho_j I) f = E_1 B_0 u_j, one shift per warp,
//    O(m^3) per step per shift (the "only the needed entries" idea the paper cites) --
//    the same quantity as the paper's eigendecomposition formula; the coefficients Z come from the
//    stored eliminations by back substitution.
//  * Deterministic: static contiguous tile chunks per CTA, fixed-order sums.
#include "kcg_cg.cuh"

namespace kcg {

template <int K, bool D2 = false>
struct LzCfg {
  static constexpr int TX = KCG_TX;
  static constexpr int TY = lz_tile_y(K, D2);
  static constexpr int HB = D2 ? 4 : 2;                // box halo: V_{i-1} is needed on the tile + 2 RR ring
  static constexpr int RR = D2 ? 2 : 1;                // ring of V_i (the operator's radius)
  static constexpr int BW = TX + 2 * HB, BH = TY + 2 * HB;
  // K <= 4 Laplacian: pixel-pair mapping, the V_i region spans the box columns (16-byte aligned pairs)
  static constexpr bool PAIRS = !D2 && K <= 4;
  static constexpr int RW = PAIRS ? BW : TX + 2 * RR, RH = TY + 2 * RR, RN = RW * RH;  // V_i region
  static constexpr int BOX = K * BH * BW;
  static constexpr int STAGES = D2 ? 2 : (K <= 2 ? 3 : (K <= 5 ? 2 : 1));  // TMA tiles in flight
  static constexpr int KP = (2 * K + 3) / 4 * 4;      // Gram rows [V, W] padded to 4
  static constexpr int NB4 = KP / 4;
  static constexpr int NJOB = NB4 * (NB4 + 1) / 2;    // upper-triangle 4x4 blocks of the Gram
  static constexpr bool REGG = K <= 4;                 // Gram accumulated in registers in step B
  static constexpr int NPART = REGG ? K * (2 * K + 1) : NJOB * 16;
  static constexpr int NACC = REGG ? K * (2 * K + 1) : 16;
#ifndef KCG_LZ_WIDE
#define KCG_LZ_WIDE 0
#endif
  // KCG_LZ_WIDE: 512 threads (16 warps, <= 128 registers, step matrices in shared memory) for the
  // pair-mapped K <= 4 Laplacian kernel instead of 256 threads with register-resident matrices
  static constexpr int NT = (PAIRS && KCG_LZ_WIDE) ? 512 : 256;
  static constexpr bool REGM = !(PAIRS && KCG_LZ_WIDE);
  static constexpr int SL = NT / NJOB;                // pixel slices per Gram block
  static constexpr int NPIX = TX * TY;
  static constexpr int UPL = REGG ? K : KP;           // U = [V_i; (K > 4: W_i; 0 pad)] on the V_i region
  static constexpr int DW = TX + 6, DH = TY + 6;      // D2: D V on the tile + 3 ring (step A), + 1 (step B)
  static constexpr int DVN = D2 ? K * DW * DH : 0;
  static constexpr int OFF_U = STAGES * 2 * BOX;
  static constexpr int OFF_HS = OFF_U + UPL * RN;     // hits of the tile (K > 4)
  static constexpr int OFF_DV = OFF_HS + (REGG ? 0 : NPIX);
  static constexpr int OFF_MAT = OFF_DV + DVN;        // P1, P2, Ri, Bc, Z (K x K each)
  static constexpr int OFF_RED = OFF_MAT + 5 * K * K; // flush scratch [NT][4]
  static constexpr int DOUBLES = OFF_RED + (REGG ? (NT / 32) * NACC : NT * 4);
  static constexpr size_t SMEM = (size_t)DOUBLES * 8 + 64;  // + mbarriers
  // reducer scratch (in the box area, idle between passes)
  static constexpr int SC_GAM = 0;                          // raw Gram [NPART]
  static constexpr int SC_GRP = SC_GAM + NPART;              // group sums [NT]
  static constexpr int SC_M = SC_GRP + NT;                   // Gv, H, C0, T1, C, R, X(Rinv), B0 [8][K*K]
  static constexpr int SC_W = SC_M + 8 * K * K;              // per-shift warp scratch [K][9 K*K]
  static constexpr int SC_RES = SC_W + K * 9 * K * K;        // residual per shift [K] + flags
  static constexpr int SC_PRE = SC_RES + 2 * K + 8;         // prefetched B_0, rho, u_j = phi (.) w_j
  static constexpr int SC_END = SC_PRE + 2 * K * K + K;
  static_assert(SC_END <= OFF_U, "reducer scratch exceeds the box area");
  static_assert(SMEM + 6 * 1024 <= 227 * 1024, "shared memory budget (dynamic + static)");
};

enum { LZ_GRAM0 = 0, LZ_STEP = 1, LZ_REPLAY = 2 };

// ------------------------------------------------------------------------- small dense algebra
// Warp-cooperative on K x K row-major matrices in shared memory (K <= 8); lanes own entries.
template <int K>
__device__ __forceinline__ void w_matmul(const double* A, const double* B, double* Cm, bool transB = false) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < K * K; e += 32) {
    const int r = e / K, c = e - r * K;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) s = fma(A[r * K + k], transB ? B[c * K + k] : B[k * K + c], s);
    Cm[e] = s;
  }
  __syncwarp();
}
// Upper Cholesky C = R^T R (reads the upper triangle of C).  Returns false on a non-positive pivot.
template <int K>
__device__ __forceinline__ bool w_chol(const double* Cm, double* R) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  for (int e = lane; e < K * K; e += 32) R[e] = 0.0;
  __syncwarp();
  for (int j = 0; j < K; ++j) {
    double d = Cm[j * K + j];
    for (int k = 0; k < j; ++k) d = fma(-R[k * K + j], R[k * K + j], d);
    ok = ok && (d > 0.0) && isfinite(d);
    const double rjj = sqrt(d > 0.0 ? d : 0.0);
    if (lane > j && lane < K) {
      double v = Cm[j * K + lane];
      for (int k = 0; k < j; ++k) v = fma(-R[k * K + j], R[k * K + lane], v);
      R[j * K + lane] = v / rjj;
    }
    if (lane == 0) R[j * K + j] = rjj;
    __syncwarp();
  }
  return ok;
}
// X = R^{-1} for upper-triangular R (lane l owns column l).
template <int K>
__device__ __forceinline__ void w_triinv(const double* R, double* X) {
  const int lane = threadIdx.x & 31;
  if (lane < K) {
    const int l = lane;
    for (int j = K - 1; j > l; --j) X[j * K + l] = 0.0;
    X[l * K + l] = 1.0 / R[l * K + l];
    for (int j = l - 1; j >= 0; --j) {
      double s = 0.0;
      for (int k = j + 1; k <= l; ++k) s = fma(R[j * K + k], X[k * K + l], s);
      X[j * K + l] = -s / R[j * K + j];
    }
  }
  __syncwarp();
}
// Sinv = S^{-1} for SPD S via S = R^T R: S^{-1} = X X^T with X = R^{-1}.
template <int K>
__device__ __forceinline__ bool w_spdinv(const double* S, double* R, double* X, double* Sinv) {
  const bool ok = w_chol<K>(S, R);
  w_triinv<K>(R, X);
  w_matmul<K>(X, X, Sinv, true);
  return ok;
}

// Single-thread register versions for K <= 4 (the reduction's critical path: no warp barriers).
template <int K>
__device__ __forceinline__ bool r_chol(const double (&Cm)[K][K], double (&R)[K][K]) {  // C = R^T R, R upper
  bool ok = true;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double d = Cm[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d = fma(-R[k][j], R[k][j], d);
    ok = ok && (d > 0.0) && isfinite(d);
    const double rjj = sqrt(d > 0.0 ? d : 0.0);
    R[j][j] = rjj;
#pragma unroll
    for (int l = 0; l < K; ++l) {
      if (l < j) R[j][l] = 0.0;
      if (l > j) {
        double v = Cm[j][l];
#pragma unroll
        for (int k = 0; k < j; ++k) v = fma(-R[k][j], R[k][l], v);
        R[j][l] = v / rjj;
      }
    }
  }
  return ok;
}
template <int K>
__device__ __forceinline__ void r_triinv(const double (&R)[K][K], double (&X)[K][K]) {  // X = R^{-1}, upper
#pragma unroll
  for (int l = 0; l < K; ++l) {
#pragma unroll
    for (int j = 0; j < K; ++j) X[j][l] = 0.0;
    X[l][l] = 1.0 / R[l][l];
#pragma unroll
    for (int j = l - 1; j >= 0; --j) {
      double v = 0.0;
#pragma unroll
      for (int k = j + 1; k <= l; ++k) v = fma(R[j][k], X[k][l], v);
      X[j][l] = -v / R[j][j];
    }
  }
}

__device__ __forceinline__ int lz_deg(int gy, int gx, int side) {
  return 4 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1);
}

// ------------------------------------------------------------------------- partial flush
// Per-thread Gram accumulators -> the CTA's partial of face f (fixed slice order).
template <int K, bool D2>
__device__ __forceinline__ void lz_flush(const LzArgs& a, int f, double (&acc)[LzCfg<K, D2>::NACC], double* sm) {
  using C = LzCfg<K, D2>;  // the layout of THIS kernel's shared memory (OFF_RED differs per prior)
  const int tid = threadIdx.x;
  double* red = sm + C::OFF_RED;
  double* dst = a.part + ((size_t)f * KCG_LZ_GRID_MAX + blockIdx.x) * C::NPART;
  if constexpr (C::REGG) {
    // xor-shuffle tree per warp, then the warps in order (fixed order: deterministic)
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int e = 0; e < C::NACC; ++e) {
      const double v = warp_sum(acc[e]);
      if (lane == 0) red[warp * C::NACC + e] = v;
    }
    __syncthreads();
    if (tid < C::NACC) {
      double s = 0.0;
      for (int w = 0; w < C::NT / 32; ++w) s += red[w * C::NACC + tid];
      dst[tid] = s;
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int rd = 0; rd < 4; ++rd) {
#pragma unroll
      for (int j = 0; j < 4; ++j) red[tid * 4 + j] = acc[rd * 4 + j];
      __syncthreads();
      if (tid < C::NJOB * 4) {
        const int job = tid >> 2, j = tid & 3;
        double s = 0.0;
        for (int sl = 0; sl < C::SL; ++sl) s += red[(sl * C::NJOB + job) * 4 + j];
        dst[job * 16 + rd * 4 + j] = s;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------------- one pass over the tiles
// mode LZ_GRAM0 (q = 0): Gram of Y^.  LZ_STEP (q = i >= 1): Lanczos step i.  LZ_REPLAY (q >= 1):
// rebuild V_q and accumulate M += V_q G_q.  The active faces act[0..nact) are split into contiguous
// tile chunks, one per CTA.
template <int K, bool HITS, bool D2>
__device__ __forceinline__ void lz_pass(const LzArgs& a, const CUtensorMap* vmap, int q, int mode, const int* act,
                                        const int* its, int nact, double* sm, uint64_t* bar, uint32_t& phbits) {
  using C = LzCfg<K, D2>;
  double* Dv = sm + C::OFF_DV;  // D2 scratch
  const int tid = threadIdx.x, cta = blockIdx.x, ncta = gridDim.x;
  const long long T = (long long)nact * a.tps;
  const long long t0 = T * cta / ncta, t1 = T * (cta + 1) / ncta;
  if (t0 >= t1) return;
  const int side = a.side;
  const size_t pstride = (size_t)a.pitch * side;
  const int slot1 = q == 0 ? 0 : lz_slot(a.store, q - 1);
  const int slot2 = q >= 3 ? lz_slot(a.store, q - 2) : 0;
  const int slotq = lz_slot(a.store, q);
  const int nbox = q >= 3 ? 2 : 1;
  double* U = sm + C::OFF_U;
  double* hs = sm + C::OFF_HS;
  double* mats = sm + C::OFF_MAT;
  const double* P1m = mats;           // Hp Ri   (after the face prologue)
  const double* P2m = mats + K * K;   // Bp^T Ri
  const double* Ri = mats + 2 * K * K;
  const double* Bc = mats + 3 * K * K;
  const double* Zm = mats + 4 * K * K;

  auto issue = [&](long long t, int s) {
    const int ti = (int)t;
    const int f = act[ti / a.tps];
    const int lt = ti - (ti / a.tps) * a.tps;
    const int ty = lt / a.tiles_x, tx = lt - ty * a.tiles_x;
    double* b1 = sm + s * 2 * C::BOX;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bar[s], nbox * C::BOX * 8);
    tma_load_3d(b1, vmap, &bar[s], tx * C::TX - C::HB, ty * C::TY - C::HB, (slot1 * a.P + f) * K);
    if (nbox == 2) tma_load_3d(b1 + C::BOX, vmap, &bar[s], tx * C::TX - C::HB, ty * C::TY - C::HB, (slot2 * a.P + f) * K);
  };
  if (tid == 0)
    for (int s = 0; s < C::STAGES && t0 + s < t1; ++s) issue(t0 + s, s);

  double acc[C::NACC];  // Gram accumulators: packed upper triangle of [V, W] (K <= 4) or a 4x4 block
#pragma unroll
  for (int j = 0; j < C::NACC; ++j) acc[j] = 0.0;
  int cur = -1, its_f = 0;
  double kap = 0.0;
  const double* hp = nullptr;
  for (long long t = t0; t < t1; ++t) {
    const int s = C::STAGES == 1 ? 0 : (int)((t - t0) % C::STAGES);
    const int ai = (int)t / a.tps;
    const int f = act[ai];
    const int lt = (int)t - ai * a.tps;
    const int y0 = (lt / a.tiles_x) * C::TY, x0 = (lt % a.tiles_x) * C::TX;
    if (f != cur) {
      if (cur >= 0 && mode != LZ_REPLAY) lz_flush<K, D2>(a, cur, acc, sm);
#pragma unroll
      for (int j = 0; j < C::NACC; ++j) acc[j] = 0.0;
      cur = f;
      its_f = its[ai];
      kap = a.prm[f].kappa2;
      hp = HITS ? a.hits + (size_t)f * side * side : nullptr;
      if (mode != LZ_GRAM0) {
        const size_t fc = (size_t)f * a.cap, fr = (size_t)f * (a.cap + 1);
        for (int e = tid; e < K * K; e += C::NT) {
          mats[e] = q >= 2 ? __ldcg(a.Hs + (fc + q - 2) * K * K + e) : 0.0;
          mats[K * K + e] = q >= 2 ? __ldcg(a.Rs + (fr + q - 2) * K * K + e) : 0.0;
          mats[2 * K * K + e] = __ldcg(a.Ri + (fr + q - 1) * K * K + e);
          // Bc (steps) -- or, in the pair-mapped replay, G_{q-1} (M updated every other pass)
          mats[3 * K * K + e] = (mode == LZ_REPLAY && C::PAIRS) ? (q >= 2 ? __ldcg(a.Zs + (fc + q - 2) * K * K + e) : 0.0)
                                                                : __ldcg(a.Rs + (fr + q - 1) * K * K + e);
          mats[4 * K * K + e] = mode == LZ_REPLAY ? __ldcg(a.Zs + (fc + q - 1) * K * K + e) : 0.0;
        }
        __syncthreads();
        // fold the step-A products: V_q = w Ri - V_{q-2} (Bp^T Ri) - V_{q-1} (Hp Ri)
        double p1 = 0.0, p2 = 0.0;
        if (tid < K * K) {
          const int d = tid / K, c = tid - d * K;
          for (int e2 = 0; e2 < K; ++e2) {
            p1 = fma(mats[d * K + e2], mats[2 * K * K + e2 * K + c], p1);
            p2 = fma(mats[K * K + e2 * K + d], mats[2 * K * K + e2 * K + c], p2);
          }
        }
        __syncthreads();
        if (tid < K * K) { mats[tid] = p1; mats[K * K + tid] = p2; }
      }
      __syncthreads();
    }
    mbar_wait(&bar[s], (phbits >> s) & 1u);
    phbits ^= 1u << s;
    const double* B1 = sm + s * 2 * C::BOX;
    const double* B2 = B1 + C::BOX;

    if constexpr (C::PAIRS) {
      // ---- step A (pairs): V_q on box columns [0, BW) x ring rows; U col = box col, U row = box row - 1
      {
        constexpr int NRM = C::REGM ? K * K : 1;
        double rrr[NRM], r1r[NRM], r2r[NRM];
        if constexpr (C::REGM) {
#pragma unroll
          for (int e2 = 0; e2 < K * K; ++e2) { rrr[e2] = Ri[e2]; r1r[e2] = P1m[e2]; r2r[e2] = P2m[e2]; }
        }
        auto rrv = [&](int i2) { if constexpr (C::REGM) return rrr[i2]; else return Ri[i2]; };
        auto r1v = [&](int i2) { if constexpr (C::REGM) return r1r[i2]; else return P1m[i2]; };
        auto r2v = [&](int i2) { if constexpr (C::REGM) return r2r[i2]; else return P2m[i2]; };
        constexpr int NPR = C::BW / 2;  // pairs per row
        for (int e = tid; e < C::RH * NPR; e += C::NT) {
          const int ry = e / NPR, bc = 2 * (e - ry * NPR);
          const int gy = y0 - 1 + ry, gx = x0 - C::HB + bc;
          const int bi = (ry + 1) * C::BW + bc;
          const bool rowin = gy >= 0 && gy < side;
          // the outermost box columns have no outer neighbour; their V_q is not needed
          const bool f0 = rowin && bc > 0 && gx >= 0 && gx < side;
          const bool f1 = rowin && bc + 2 < C::BW && gx + 1 >= 0 && gx + 1 < side;
          double2 v[K];
          if (!f0 && !f1) {
#pragma unroll
            for (int c = 0; c < K; ++c) v[c] = make_double2(0.0, 0.0);
          } else if (mode == LZ_GRAM0) {
#pragma unroll
            for (int c = 0; c < K; ++c) {
              const double2 b = *reinterpret_cast<const double2*>(B1 + c * C::BH * C::BW + bi);
              v[c] = make_double2(f0 ? b.x : 0.0, f1 ? b.y : 0.0);
            }
          } else {
            double2 w[K], v1[K];
#pragma unroll
            for (int c = 0; c < K; ++c) v1[c] = *reinterpret_cast<const double2*>(B1 + c * C::BH * C::BW + bi);
            if (q == 1) {
#pragma unroll
              for (int c = 0; c < K; ++c) w[c] = v1[c];
            } else {
              const double kd0 = kap + (double)lz_deg(gy, gx, side), kd1 = kap + (double)lz_deg(gy, gx + 1, side);
              const double h0 = HITS && f0 ? __ldg(hp + (size_t)gy * side + gx) : 1.0;
              const double h1 = HITS && f1 ? __ldg(hp + (size_t)gy * side + gx + 1) : 1.0;
#pragma unroll
              for (int c = 0; c < K; ++c) {
                const double* p = B1 + c * C::BH * C::BW + bi;
                const double2 up = *reinterpret_cast<const double2*>(p - C::BW);
                const double2 dn = *reinterpret_cast<const double2*>(p + C::BW);
                const double l = f0 ? p[-1] : 0.0, r = f1 ? p[2] : 0.0;
                const double s0 = fma(kd0, v1[c].x, -(((up.x + dn.x) + l) + v1[c].y));
                const double s1 = fma(kd1, v1[c].y, -(((up.y + dn.y) + v1[c].x) + r));
                w[c] = make_double2(HITS ? s0 / h0 : s0, HITS ? s1 / h1 : s1);
              }
            }
            double2 v2[K];
#pragma unroll
            for (int d = 0; d < K; ++d)
              v2[d] = q >= 3 ? *reinterpret_cast<const double2*>(B2 + d * C::BH * C::BW + bi) : make_double2(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < K; ++c) {
              double sx = 0.0, sy = 0.0;
#pragma unroll
              for (int d = 0; d < K; ++d) { const double m2 = rrv(d * K + c); sx = fma(w[d].x, m2, sx); sy = fma(w[d].y, m2, sy); }
              if (q >= 2) {
#pragma unroll
                for (int d = 0; d < K; ++d) { const double m2 = r1v(d * K + c); sx = fma(-v1[d].x, m2, sx); sy = fma(-v1[d].y, m2, sy); }
              }
              if (q >= 3) {
#pragma unroll
                for (int d = 0; d < K; ++d) { const double m2 = r2v(d * K + c); sx = fma(-v2[d].x, m2, sx); sy = fma(-v2[d].y, m2, sy); }
              }
              v[c] = make_double2(f0 ? sx : 0.0, f1 ? sy : 0.0);
            }
          }
#pragma unroll
          for (int c = 0; c < K; ++c) *reinterpret_cast<double2*>(U + c * C::RN + ry * C::RW + bc) = v[c];
        }
      }
      __syncthreads();
      // ---- step B (pairs): W_q on the tile, store V_q, Gram in registers (or the replay's M update)
      {
        constexpr int NRB = C::REGM ? K * K : 1;
        double rbr[NRB];
        const double* rbs = mode == LZ_REPLAY ? Zm : Bc;
        if constexpr (C::REGM) {
#pragma unroll
          for (int e2 = 0; e2 < K * K; ++e2) rbr[e2] = rbs[e2];
        }
        auto rbv = [&](int i2) { if constexpr (C::REGM) return rbr[i2]; else return rbs[i2]; };
        constexpr int NPT = C::TX / 2;
        const size_t N = (size_t)side * side;
        for (int e = tid; e < C::TY * NPT; e += C::NT) {
          const int ly = e / NPT, lx = 2 * (e - ly * NPT);
          const int gy = y0 + ly, gx = x0 + lx;
          const int ri = (ly + 1) * C::RW + lx + C::HB;
          const int bi = (ly + C::HB) * C::BW + lx + C::HB;
          const bool in0 = gy < side && gx < side, in1 = gy < side && gx + 1 < side;
          double2 vq[K];
#pragma unroll
          for (int c = 0; c < K; ++c) vq[c] = *reinterpret_cast<const double2*>(U + c * C::RN + ri);
          if (mode == LZ_REPLAY) {
            // M is read and written every other pass: on even q it gains V_{q-1} G_{q-1} (V_{q-1} is in
            // the box) and V_q G_q; an odd last pass adds V_q G_q alone -- the assembly's q-major order
            const bool upd = (q & 1) == 0 || q == its_f;
            if (in0) {
              const size_t px = (size_t)gy * side + gx;
              double2 vo[K];
              if (upd && (q & 1) == 0) {
#pragma unroll
                for (int d = 0; d < K; ++d) vo[d] = *reinterpret_cast<const double2*>(B1 + d * C::BH * C::BW + bi);
              }
#pragma unroll
              for (int c = 0; c < K; ++c) {
                if (upd) {
                  double* mp = a.Mx + ((size_t)f * K + c) * N + px;
                  double mx = q > 2 ? mp[0] : 0.0, my = (q > 2 && in1) ? mp[1] : 0.0;
                  if ((q & 1) == 0) {
#pragma unroll
                    for (int d = 0; d < K; ++d) {
                      const double m1 = Bc[d * K + c];  // G_{q-1}
                      mx = fma(vo[d].x, m1, mx);
                      my = fma(vo[d].y, m1, my);
                    }
                  }
#pragma unroll
                  for (int d = 0; d < K; ++d) { const double m2 = rbv(d * K + c); mx = fma(vq[d].x, m2, mx); my = fma(vq[d].y, m2, my); }
                  mp[0] = mx;
                  if (in1) mp[1] = my;
                }
                if (q < its_f) {
                  double* vp = a.V + ((size_t)(slotq * a.P + f) * K + c) * pstride + (size_t)gy * a.pitch + gx;
                  vp[0] = vq[c].x;
                  if (in1) vp[1] = vq[c].y;
                }
              }
            }
            continue;
          }
          double2 w[K];
          double h0 = 1.0, h1 = 1.0;
          if (mode == LZ_GRAM0) {
            if (HITS) { h0 = in0 ? __ldg(hp + (size_t)gy * side + gx) : 0.0; h1 = in1 ? __ldg(hp + (size_t)gy * side + gx + 1) : 0.0; }
#pragma unroll
            for (int c = 0; c < K; ++c) w[c] = make_double2(0.0, 0.0);
          } else {
            const double kd0 = kap + (double)lz_deg(gy, gx, side), kd1 = kap + (double)lz_deg(gy, gx + 1, side);
            if (HITS) { h0 = in0 ? __ldg(hp + (size_t)gy * side + gx) : 1.0; h1 = in1 ? __ldg(hp + (size_t)gy * side + gx + 1) : 1.0; }
#pragma unroll
            for (int c = 0; c < K; ++c) {
              const double* p = U + c * C::RN + ri;
              const double2 up = *reinterpret_cast<const double2*>(p - C::RW);
              const double2 dn = *reinterpret_cast<const double2*>(p + C::RW);
              const double s0 = fma(kd0, vq[c].x, -(((up.x + dn.x) + p[-1]) + vq[c].y));
              const double s1 = fma(kd1, vq[c].y, -(((up.y + dn.y) + vq[c].x) + p[2]));
              w[c] = make_double2(HITS ? s0 / h0 : s0, HITS ? s1 / h1 : s1);
            }
            if (q >= 2) {
              double2 vo[K];
#pragma unroll
              for (int d = 0; d < K; ++d) vo[d] = *reinterpret_cast<const double2*>(B1 + d * C::BH * C::BW + bi);
#pragma unroll
              for (int c = 0; c < K; ++c)
#pragma unroll
                for (int d = 0; d < K; ++d) {
                  const double m2 = rbv(c * K + d);
                  w[c].x = fma(-vo[d].x, m2, w[c].x);
                  w[c].y = fma(-vo[d].y, m2, w[c].y);
                }
            }
            if (in0) {
#pragma unroll
              for (int c = 0; c < K; ++c) {
                double* vp = a.V + ((size_t)(slotq * a.P + f) * K + c) * pstride + (size_t)gy * a.pitch + gx;
                if (in1) *reinterpret_cast<double2*>(vp) = vq[c];
                else vp[0] = vq[c].x;
              }
            }
          }
          if (!in0) { h0 = 0.0; }
          if (!in1) { h1 = 0.0; }
          // N-weighted Gram of u = [V_q, W_q] at both pixels (h = 0 outside the face)
          {
            double u0[2 * K], u1[2 * K];
#pragma unroll
            for (int c = 0; c < K; ++c) { u0[c] = vq[c].x; u0[K + c] = w[c].x; u1[c] = vq[c].y; u1[K + c] = w[c].y; }
            int idx = 0;
#pragma unroll
            for (int i = 0; i < 2 * K; ++i) {
              const double a0 = h0 * u0[i], a1 = h1 * u1[i];
#pragma unroll
              for (int j = i; j < 2 * K; ++j) { acc[idx] = fma(a1, u1[j], fma(a0, u0[j], acc[idx])); ++idx; }
            }
          }
        }
      }
    } else {
    // ---- D2: D V_{q-1} on the tile + 3 ring (D v := 0 outside the face; D = -L)
      if constexpr (D2) {
        if (mode != LZ_GRAM0 && q >= 2) {
          for (int e = tid; e < K * C::DW * C::DH; e += C::NT) {
            const int c = e / (C::DW * C::DH), r = e - c * (C::DW * C::DH);
            const int dy = r / C::DW, dx = r - dy * C::DW;
            const int gy = y0 - 3 + dy, gx = x0 - 3 + dx;
            double d = 0.0;
            if (gy >= 0 && gy < side && gx >= 0 && gx < side) {
              const double* p = B1 + c * C::BH * C::BW + (dy + C::HB - 3) * C::BW + dx + C::HB - 3;
              d = (p[-C::BW] + p[C::BW] + p[-1] + p[1]) - (double)lz_deg(gy, gx, side) * p[0];
            }
            Dv[e] = d;
          }
          __syncthreads();
        }
      }
      // ---- step A: V_q on the tile + RR ring (zero outside the face: free boundary, reading R2)
      {
        // this tile's step-A matrices: registers for K <= 4, shared memory (broadcast) above
        constexpr int NR = C::REGG ? K * K : 1;
        double r1v[NR], r2v[NR], rrv[NR];
        if constexpr (C::REGG) {
  #pragma unroll
          for (int e2 = 0; e2 < K * K; ++e2) { rrv[e2] = Ri[e2]; r1v[e2] = P1m[e2]; r2v[e2] = P2m[e2]; }
        }
        auto rr = [&](int i) { if constexpr (C::REGG) return rrv[i]; else return Ri[i]; };
        auto r1 = [&](int i) { if constexpr (C::REGG) return r1v[i]; else return P1m[i]; };
        auto r2 = [&](int i) { if constexpr (C::REGG) return r2v[i]; else return P2m[i]; };
        for (int e = tid; e < C::RN; e += C::NT) {
          const int ry = e / C::RW, rx = e - ry * C::RW;
          const int gy = y0 - C::RR + ry, gx = x0 - C::RR + rx;
          const int bi = (ry + C::HB - C::RR) * C::BW + rx + C::HB - C::RR;
          double v[K];
          if (gy < 0 || gy >= side || gx < 0 || gx >= side) {
  #pragma unroll
            for (int c = 0; c < K; ++c) v[c] = 0.0;
          } else if (mode == LZ_GRAM0) {
  #pragma unroll
            for (int c = 0; c < K; ++c) v[c] = B1[c * C::BH * C::BW + bi];
          } else {
            double w[K], v1[K];
  #pragma unroll
            for (int c = 0; c < K; ++c) v1[c] = B1[c * C::BH * C::BW + bi];
            if (q == 1) {
  #pragma unroll
              for (int c = 0; c < K; ++c) w[c] = v1[c];
            } else {
              const double kd = kap + (double)lz_deg(gy, gx, side);
              const double h = HITS ? __ldg(hp + (size_t)gy * side + gx) : 1.0;
  #pragma unroll
              for (int c = 0; c < K; ++c) {
                double s2;
                if constexpr (D2) {  // Q0 v = D (D v) + kappa2 v
                  const double* d = Dv + c * C::DW * C::DH + (ry + 3 - C::RR) * C::DW + rx + 3 - C::RR;
                  s2 = fma(kap, v1[c], (d[-C::DW] + d[C::DW] + d[-1] + d[1]) - (kd - kap) * d[0]);
                } else {             // Q0 v = (kappa2 + deg) v - sum_nbr v
                  const double* p = B1 + c * C::BH * C::BW + bi;
                  s2 = fma(kd, v1[c], -(p[-C::BW] + p[C::BW] + p[-1] + p[1]));
                }
                w[c] = HITS ? s2 / h : s2;
              }
            }
            double v2[K];  // V_{q-2} at the pixel, loaded once (not once per output component)
  #pragma unroll
            for (int d = 0; d < K; ++d) v2[d] = q >= 3 ? B2[d * C::BH * C::BW + bi] : 0.0;
            if constexpr (C::REGG) {  // K <= 4: one chain per component (register-bound)
  #pragma unroll
              for (int c = 0; c < K; ++c) {
                double s2 = 0.0;
  #pragma unroll
                for (int d = 0; d < K; ++d) s2 = fma(w[d], rr(d * K + c), s2);
                if (q >= 2) {
  #pragma unroll
                  for (int d = 0; d < K; ++d) s2 = fma(-v1[d], r1(d * K + c), s2);
                }
                if (q >= 3) {
  #pragma unroll
                  for (int d = 0; d < K; ++d) s2 = fma(-v2[d], r2(d * K + c), s2);
                }
                v[c] = s2;
              }
            } else {  // K > 4: three independent product chains per component (latency-bound)
  #pragma unroll
              for (int c = 0; c < K; ++c) {
                double sa = 0.0, sb = 0.0, sc = 0.0;
  #pragma unroll
                for (int d = 0; d < K; ++d) {
                  sa = fma(w[d], rr(d * K + c), sa);
                  sb = fma(v1[d], r1(d * K + c), sb);
                  sc = fma(v2[d], r2(d * K + c), sc);
                }
                v[c] = q >= 3 ? sa - (sb + sc) : (q >= 2 ? sa - sb : sa);
              }
            }
          }
  #pragma unroll
          for (int c = 0; c < K; ++c) U[c * C::RN + e] = v[c];
        }
      }
      __syncthreads();
  
      // ---- D2: D V_q on the tile + 1 ring
      if constexpr (D2) {
        if (mode == LZ_STEP) {
          constexpr int W1 = C::TX + 2, H1 = C::TY + 2;
          for (int e = tid; e < K * W1 * H1; e += C::NT) {
            const int c = e / (W1 * H1), r = e - c * (W1 * H1);
            const int dy = r / W1, dx = r - dy * W1;
            const int gy = y0 - 1 + dy, gx = x0 - 1 + dx;
            double d = 0.0;
            if (gy >= 0 && gy < side && gx >= 0 && gx < side) {
              const double* p = U + c * C::RN + (dy + C::RR - 1) * C::RW + dx + C::RR - 1;
              d = (p[-C::RW] + p[C::RW] + p[-1] + p[1]) - (double)lz_deg(gy, gx, side) * p[0];
            }
            Dv[e] = d;
          }
          __syncthreads();
        }
      }
      // ---- step B: W_q on the tile (or the replay's M update); store V_q; Gram (K <= 4: in registers)
      {
        constexpr int NRB = C::REGG ? K * K : 1;
        double rbv[NRB];
        const double* rbs = mode == LZ_REPLAY ? Zm : Bc;
        if constexpr (C::REGG) {
  #pragma unroll
          for (int e2 = 0; e2 < K * K; ++e2) rbv[e2] = rbs[e2];
        }
        auto rb = [&](int i) { if constexpr (C::REGG) return rbv[i]; else return rbs[i]; };
        for (int e = tid; e < C::NPIX; e += C::NT) {
          const int ly = e / C::TX, lx = e - ly * C::TX;
          const int gy = y0 + ly, gx = x0 + lx;
          const int ri = (ly + C::RR) * C::RW + lx + C::RR;
          const int bi = (ly + C::HB) * C::BW + lx + C::HB;
          const bool in = gy < side && gx < side;
          if (mode == LZ_REPLAY) {
            if (in) {
              const size_t px = (size_t)gy * side + gx;
              const size_t N = (size_t)side * side;
  #pragma unroll
              for (int c = 0; c < K; ++c) {
                double m = q > 1 ? a.Mx[((size_t)f * K + c) * N + px] : 0.0;
  #pragma unroll
                for (int d = 0; d < K; ++d) m = fma(U[d * C::RN + ri], rb(d * K + c), m);
                a.Mx[((size_t)f * K + c) * N + px] = m;
              }
              if (q < its_f) {
  #pragma unroll
                for (int c = 0; c < K; ++c)
                  a.V[((size_t)(slotq * a.P + f) * K + c) * pstride + (size_t)gy * a.pitch + gx] = U[c * C::RN + ri];
              }
            }
            continue;
          }
          double w[K], vq[K];
          double h = 1.0;
  #pragma unroll
          for (int c = 0; c < K; ++c) vq[c] = U[c * C::RN + ri];
          if (!in) {
            h = 0.0;
  #pragma unroll
            for (int c = 0; c < K; ++c) w[c] = 0.0;
          } else if (mode == LZ_GRAM0) {
            if (HITS) h = __ldg(hp + (size_t)gy * side + gx);
  #pragma unroll
            for (int c = 0; c < K; ++c) w[c] = 0.0;
          } else {
            const double kd = kap + (double)lz_deg(gy, gx, side);
            if (HITS) h = __ldg(hp + (size_t)gy * side + gx);
  #pragma unroll
            for (int c = 0; c < K; ++c) {
              double s2;
              if constexpr (D2) {
                constexpr int W1 = C::TX + 2, H1 = C::TY + 2;
                const double* d = Dv + c * W1 * H1 + (ly + 1) * W1 + lx + 1;
                s2 = fma(kap, vq[c], (d[-W1] + d[W1] + d[-1] + d[1]) - (kd - kap) * d[0]);
              } else {
                const double* p = U + c * C::RN + ri;
                s2 = fma(kd, vq[c], -(p[-C::RW] + p[C::RW] + p[-1] + p[1]));
              }
              w[c] = HITS ? s2 / h : s2;
            }
            if (q >= 2) {
              double vo[K];  // V_{q-1} at the pixel
  #pragma unroll
              for (int d = 0; d < K; ++d) vo[d] = B1[d * C::BH * C::BW + bi];
  #pragma unroll
              for (int c = 0; c < K; ++c) {
                if constexpr (C::REGG) {
  #pragma unroll
                  for (int d = 0; d < K; ++d) w[c] = fma(-vo[d], rb(c * K + d), w[c]);
                } else {
                  double t2 = 0.0;
  #pragma unroll
                  for (int d = 0; d < K; ++d) t2 = fma(vo[d], rb(c * K + d), t2);
                  w[c] -= t2;
                }
              }
            }
  #pragma unroll
            for (int c = 0; c < K; ++c)
              a.V[((size_t)(slotq * a.P + f) * K + c) * pstride + (size_t)gy * a.pitch + gx] = vq[c];
          }
          if constexpr (C::REGG) {
            // N-weighted Gram of u = [V_q, W_q] at this pixel, packed upper triangle
            double u[2 * K];
  #pragma unroll
            for (int c = 0; c < K; ++c) { u[c] = vq[c]; u[K + c] = w[c]; }
            int idx = 0;
  #pragma unroll
            for (int i = 0; i < 2 * K; ++i) {
              const double hu = HITS ? h * u[i] : u[i];
  #pragma unroll
              for (int j = i; j < 2 * K; ++j) { acc[idx] = fma(hu, u[j], acc[idx]); ++idx; }
            }
          } else {
  #pragma unroll
            for (int c = 0; c < K; ++c) U[(K + c) * C::RN + ri] = w[c];
            if (HITS) hs[e] = h;
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0 && t + C::STAGES < t1) issue(t + C::STAGES, s);  // the stage's boxes are free

    // ---- K > 4: N-weighted Gram of [V_q, W_q] (upper-triangle 4x4 blocks, one per thread group)
    if constexpr (!C::REGG) {
      if (mode != LZ_REPLAY) {
        const int job = tid % C::NJOB, sl = tid / C::NJOB;
        if (sl < C::SL) {
          int bi = 0, r = job;
          while (r >= C::NB4 - bi) { r -= C::NB4 - bi; ++bi; }
          const int bj = bi + r;
          const double* ua = U + bi * 4 * C::RN;
          const double* ub = U + bj * 4 * C::RN;
          for (int px = sl; px < C::NPIX; px += C::SL) {
            const int ly = px / C::TX, lx = px - ly * C::TX;
            const int ri = (ly + C::RR) * C::RW + lx + C::RR;
            double xa[4], yb[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) { xa[j] = ua[j * C::RN + ri]; yb[j] = ub[j * C::RN + ri]; }
            if (HITS) {
              const double h = hs[px];
#pragma unroll
              for (int j = 0; j < 4; ++j) xa[j] *= h;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fma(xa[i], yb[j], acc[i * 4 + j]);
          }
        }
      }
      __syncthreads();  // U is free
    }
  }
  if (mode != LZ_REPLAY && cur >= 0) lz_flush<K, D2>(a, cur, acc, sm);
}

// ------------------------------------------------------------------------- per-face reduction
// Reducer CTA of face act[ai] after pass q: sums the CTA partials (fixed order), then
//   q = 0: B_0 = chol(Y^T N Y^);  q = i >= 1: H_i, C = W^T N W (Cholesky-QR Gram), B_{i+1} = chol(C),
//   per shift j: T_i + rho_j I eliminated by one more block row, gamma_j = ||B_{i+1} f_last||^2;
//   stop when sqrt(gamma) <= tol ||B_0||_F (Alg. SylvSolver).
// KCG_TRACE builds: sub-phase stamps of the reduction on CTA 0 (columns 153..157 of the pass row)
__device__ __forceinline__ void lz_stamp(const LzArgs& a, int q, int col) {
  if (KCG_TRACE && a.trace && blockIdx.x == 0 && threadIdx.x == 0 && q < KCG_TRACE_ITERS)
    a.trace[(size_t)q * KCG_TRACE_COLS + col] = globaltimer();
}

template <int K, bool D2>
__device__ void lz_reduce(const LzArgs& a, int q, const int* act, int nact, int ai, double* sm) {
  using C = LzCfg<K, D2>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, ncta = gridDim.x;
  const int f = act[ai];
  const long long T = (long long)nact * a.tps;
  const long long f0 = (long long)ai * a.tps, f1 = f0 + a.tps;
  const size_t fc = (size_t)f * a.cap, fr = (size_t)f * (a.cap + 1);
  // constants of the face and B_0 (L2 reads, issued before the partial sums)
  __shared__ LzState zpre;
  if (q >= 1 && tid == 0) zpre = a.st[f];
  if (q >= 1) {
    double* pre = sm + C::SC_PRE;
    const LzFace& pf0 = a.prm[f];
    for (int e = tid; e < K * K; e += C::NT) {
      pre[e] = __ldcg(a.Rs + fr * K * K + e);                        // B_0
      pre[K * K + K + e] = pf0.phi[e / K] * pf0.W[e];                 // U = P W: u_j = column j
    }
    if (tid < K) pre[K * K + tid] = pf0.rho[tid];
  }
  // the previous step's elimination of every shift does not depend on this pass: fetch it first
  // (overlaps the L2 latency with the partial sums below)
  if (q >= 2 && warp < K) {
    double* Sp = sm + C::SC_W + warp * 9 * K * K + K * K;
    double* Bs = Sp + K * K;
    double* gp = Bs + 6 * K * K;  // past Si: the 9th K x K slot of the warp
    const double* spg = a.Sinv + ((fc + q - 2) * K + warp) * K * K;
    for (int e = lane; e < K * K; e += 32) {
      Sp[e] = __ldcg(spg + e);
      Bs[e] = __ldcg(a.Rs + (fr + q - 1) * K * K + e);  // sub-diagonal block between blocks q-2, q-1
    }
    if (lane < K) gp[lane] = __ldcg(a.gv + ((fc + q - 2) * K + warp) * K + lane);
  }
  // CTAs whose chunk [T b / ncta, T (b+1) / ncta) holds the face's first / last tile, and the chunk
  // starts in between (empty chunks hold no partial)
  const int b_lo = (int)(((f0 + 1) * ncta + T - 1) / T) - 1;
  const int b_hi = (int)((f1 * ncta + T - 1) / T) - 1;
  __shared__ long long cst[KCG_LZ_GRID_MAX + 1];
  for (int b = b_lo + tid; b <= b_hi + 1; b += C::NT) cst[b - b_lo] = T * b / ncta;
  __syncthreads();
  double* gam = sm + C::SC_GAM;
  double* grp = sm + C::SC_GRP;
  constexpr int NG = C::NT / C::NPART;
  {
    const int g = tid / C::NPART, e = tid - g * C::NPART;
    if (g < NG) {
      // loads issued 8 at a time (memory-level parallelism), added in CTA order
      double s = 0.0;
      const double* src = a.part + (size_t)f * KCG_LZ_GRID_MAX * C::NPART + e;
      constexpr int UNR = 8;   // loads in flight per thread (24: measured slower)
      for (int b0 = b_lo + g; b0 <= b_hi; b0 += UNR * NG) {
        double v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          // clamped index: the compiler may issue the loads before the predicate is known
          const int b = min(b0 + u * NG, b_hi);
          const bool ok = b0 + u * NG <= b_hi && cst[b + 1 - b_lo] > cst[b - b_lo];
          const double pv = __ldcg(src + (size_t)b * C::NPART);
          v[u] = ok ? pv : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) s += v[u];
      }
      grp[g * C::NPART + e] = s;
    }
  }
  __syncthreads();
  if (tid < C::NPART) {
    double s = 0.0;
    for (int g = 0; g < NG; ++g) s += grp[g * C::NPART + tid];
    gam[tid] = s;
  }
  __syncthreads();
  lz_stamp(a, q, 153);
  double* Gv = sm + C::SC_M;
  double* H = Gv + K * K;
  double* C0 = H + K * K;
  double* T1 = C0 + K * K;
  double* Cm = T1 + K * K;
  double* R = Cm + K * K;
  double* X = R + K * K;
  double* res = sm + C::SC_RES;
  int* flag = reinterpret_cast<int*>(res + K);
  auto G = [&](int i, int j) {  // symmetric Gram entry (packed upper triangle, or 4x4 blocks)
    if (i > j) { const int t = i; i = j; j = t; }
    if constexpr (C::REGG) return gam[i * (2 * K) - i * (i - 1) / 2 + (j - i)];
    const int bi = i >> 2, bj = j >> 2;
    const int job = bi * C::NB4 - bi * (bi - 1) / 2 + (bj - bi);
    return gam[job * 16 + (i & 3) * 4 + (j & 3)];
  };
  for (int e = tid; e < K * K; e += C::NT) {
    const int r = e / K, c = e - r * K;
    Gv[e] = G(r, c);
    H[e] = G(r, K + c);
    C0[e] = G(K + r, K + c);
  }
  __syncthreads();
  if (q == 0) {
    if (warp == 0) {
      const bool ok = w_chol<K>(Gv, R);
      w_triinv<K>(R, X);
      if (lane == 0) {
        double tr = 0.0, fro = 0.0;
        for (int e = 0; e < K * K; ++e) fro += R[e] * R[e];
        for (int c = 0; c < K; ++c) tr += Gv[c * K + c];
        LzState z{};
        z.iters = 0;
        z.bnorm = sqrt(fro);
        z.rel = 1.0;
        if (!isfinite(tr)) z.status = ST_NONFINITE;
        else if (tr == 0.0) { z.status = ST_CONVERGED; z.bnorm = 0.0; z.rel = 0.0; }
        else if (!ok) z.status = ST_BREAKDOWN;
        else if (a.max_iter <= 0) z.status = ST_MAXIT;
        else z.status = ST_RUNNING;
        a.st[f] = z;
      }
      for (int e = lane; e < K * K; e += 32) {
        a.Rs[fr * K * K + e] = R[e];
        a.Ri[fr * K * K + e] = X[e];
      }
    }
    return;
  }
  // C = C0 - 2 H^T H + H^T Gv H   (Gram of W - V H given V^T N W = H).  One warp (a spare one when
  // K < 8) runs the Cholesky QR while the shift warps run their eliminations; only gamma needs both.
  const int cwarp = K < 8 ? K : 0;
  const int blk = q - 1;  // block index of H_i in T_i
  __shared__ double gvec[KCG_KMAX][KCG_KMAX], fvec[KCG_KMAX][KCG_KMAX];
  if constexpr (K <= 4) {
    // one thread for the Cholesky QR (lane 0 of warp K), one per shift j (lane 0 of warp j), all in
    // registers and concurrent
    if (lane == 0 && warp == K) {
      double Hr[K][K], Gr[K][K], Cr[K][K], Rr[K][K], Xr[K][K];
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) { Hr[r][c] = H[r * K + c]; Gr[r][c] = Gv[r * K + c]; }
      double cmax = 0.0, c0max = 0.0;
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) {
          double t1[K];
#pragma unroll
          for (int k = 0; k < K; ++k) {  // (Gv H)[k][c]
            double v = 0.0;
#pragma unroll
            for (int l = 0; l < K; ++l) v = fma(Gr[k][l], Hr[l][c], v);
            t1[k] = v;
          }
          double v = C0[r * K + c];
#pragma unroll
          for (int k = 0; k < K; ++k) v = fma(Hr[k][r], fma(-2.0, Hr[k][c], t1[k]), v);
          Cr[r][c] = v;
          Cm[r * K + c] = v;
          cmax = fmax(cmax, fabs(v));
          c0max = fmax(c0max, fabs(C0[r * K + c]));
        }
      const bool ok = r_chol<K>(Cr, Rr);
      const int fl = ok ? 1 : (cmax <= 1e-14 * c0max ? 2 : 0);
      if (ok) r_triinv<K>(Rr, Xr);
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) {
          R[r * K + c] = fl == 2 ? 0.0 : Rr[r][c];
          X[r * K + c] = (fl == 2 || !ok) ? 0.0 : Xr[r][c];
        }
      flag[0] = fl;
    }
    if (lane == 0 && warp < K) {
      const int j = warp;
      const double rho = sm[C::SC_PRE + K * K + j];
      double S[K][K], g[K];
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) S[r][c] = (r >= c ? H[r * K + c] : H[c * K + r]) + (r == c ? rho : 0.0);
      if (blk == 0) {
#pragma unroll
        for (int r = 0; r < K; ++r) {  // g = B_0 u_j
          double v = 0.0;
#pragma unroll
          for (int c = 0; c < K; ++c) v = fma(sm[C::SC_PRE + r * K + c], sm[C::SC_PRE + K * K + K + c * K + j], v);
          g[r] = v;
        }
      } else {
        const double* Sp = sm + C::SC_W + j * 9 * K * K + K * K;
        const double* Bs = Sp + K * K;
        double Xm[K][K];
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
          for (int c = 0; c < K; ++c) {  // X = B S_{blk-1}^{-1}
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k) v = fma(Bs[r * K + k], Sp[k * K + c], v);
            Xm[r][c] = v;
          }
#pragma unroll
        for (int r = 0; r < K; ++r) {
#pragma unroll
          for (int c = 0; c < K; ++c) {  // S = D - X B^T
            double v = S[r][c];
#pragma unroll
            for (int k = 0; k < K; ++k) v = fma(-Xm[r][k], Bs[c * K + k], v);
            S[r][c] = v;
          }
          double v = 0.0;  // g = -X g_prev
#pragma unroll
          for (int c = 0; c < K; ++c) v = fma(-Xm[r][c], Bs[6 * K * K + c], v);
          g[r] = v;
        }
      }
      double Rs2[K][K], Xs[K][K], Si[K][K];
      r_chol<K>(S, Rs2);
      r_triinv<K>(Rs2, Xs);
      double* so = a.Sinv + ((fc + blk) * K + j) * K * K;
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) {  // S^{-1} = X X^T
          double v = 0.0;
#pragma unroll
          for (int k = 0; k < K; ++k) v = fma(Xs[r][k], Xs[c][k], v);
          Si[r][c] = v;
          so[r * K + c] = v;
        }
#pragma unroll
      for (int r = 0; r < K; ++r) {
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c) v = fma(Si[r][c], g[c], v);
        fvec[j][r] = v;
        gvec[j][r] = g[r];
        a.gv[((fc + blk) * K + j) * K + r] = g[r];
      }
    }
  } else {
  if (warp == cwarp) {
    w_matmul<K>(Gv, H, T1);
    for (int e = lane; e < K * K; e += 32) {
      const int r = e / K, c = e - r * K;
      double s = C0[e];
      for (int k = 0; k < K; ++k) s = fma(H[k * K + r], fma(-2.0, H[k * K + c], T1[k * K + c]), s);
      Cm[e] = s;
    }
    __syncwarp();
    const bool ok = w_chol<K>(Cm, R);
    if (ok) w_triinv<K>(R, X);
    if (lane == 0) {
      // Krylov space exhausted (W - V H = 0 up to rounding): B_{i+1} = 0, the projection is exact
      double cmax = 0.0, c0max = 0.0;
      for (int e = 0; e < K * K; ++e) { cmax = fmax(cmax, fabs(Cm[e])); c0max = fmax(c0max, fabs(C0[e])); }
      flag[0] = ok ? 1 : (cmax <= 1e-14 * c0max ? 2 : 0);
    }
    __syncwarp();
    if (flag[0] == 2)
      for (int e = lane; e < K * K; e += 32) { R[e] = 0.0; X[e] = 0.0; }
  }
  // per shift j (one warp each): block forward elimination of (T_i + rho_j I) f = E_1 B_0 u_j
  if (warp < K) {
    const int j = warp;
    double* D = sm + C::SC_W + j * 9 * K * K;
    double* Sp = D + K * K;
    double* Bs = Sp + K * K;
    double* Xm = Bs + K * K;
    double* S = Xm + K * K;
    double* Rw = S + K * K;
    double* Xw = Rw + K * K;
    double* Si = Xw + K * K;
    const double rho = sm[C::SC_PRE + K * K + j];
    for (int e = lane; e < K * K; e += 32) {
      const int r = e / K, c = e - r * K;
      D[e] = (r >= c ? H[e] : H[c * K + r]) + (r == c ? rho : 0.0);  // lower triangle of H (reading R29)
    }
    __syncwarp();
    if (blk == 0) {
      for (int e = lane; e < K * K; e += 32) S[e] = D[e];
      if (lane < K) {  // g = B_0 u_j, u_j = P w_j
        double s = 0.0;
        for (int c = 0; c < K; ++c) s = fma(sm[C::SC_PRE + lane * K + c], sm[C::SC_PRE + K * K + K + c * K + j], s);
        gvec[j][lane] = s;
      }
      __syncwarp();
    } else {
      const double gp = lane < K ? Bs[6 * K * K + lane] : 0.0;  // prefetched at entry
      w_matmul<K>(Bs, Sp, Xm);                 // X = B S_{blk-1}^{-1}
      for (int e = lane; e < K * K; e += 32) {  // S = D - X B^T
        const int r = e / K, c = e - r * K;
        double s = D[e];
        for (int k = 0; k < K; ++k) s = fma(-Xm[r * K + k], Bs[c * K + k], s);
        S[e] = s;
      }
      if (lane < K) fvec[j][lane] = gp;
      __syncwarp();
      if (lane < K) {  // g = -X g_prev
        double s = 0.0;
        for (int c = 0; c < K; ++c) s = fma(-Xm[lane * K + c], fvec[j][c], s);
        gvec[j][lane] = s;
      }
      __syncwarp();
    }
    w_spdinv<K>(S, Rw, Xw, Si);
    if (lane < K) {  // f = S^{-1} g
      double s = 0.0;
      for (int c = 0; c < K; ++c) s = fma(Si[lane * K + c], gvec[j][c], s);
      fvec[j][lane] = s;
    }
    __syncwarp();
    double* so = a.Sinv + ((fc + blk) * K + j) * K * K;
    for (int e = lane; e < K * K; e += 32) so[e] = Si[e];
    if (lane < K) a.gv[((fc + blk) * K + j) * K + lane] = gvec[j][lane];
  }
  }  // K > 4
  lz_stamp(a, q, 154);
  __syncthreads();  // R (Cholesky warp) and every shift's f_last are ready
  if (tid < K) {    // gamma_j = ||B_{i+1} f_last||^2
    double g2 = 0.0;
    for (int r = 0; r < K; ++r) {
      double s2 = 0.0;
      for (int c = 0; c < K; ++c) s2 = fma(R[r * K + c], fvec[tid][c], s2);
      g2 = fma(s2, s2, g2);
    }
    res[tid] = g2;
  }
  __syncthreads();
  lz_stamp(a, q, 155);
  if (tid == 0) {
    LzState z = zpre;
    double gam2 = 0.0;
    for (int j = 0; j < K; ++j) gam2 += res[j];
    z.iters = q;
    z.rel = z.bnorm > 0.0 ? sqrt(gam2) / z.bnorm : 0.0;
    bool fin = isfinite(gam2);
    for (int e = 0; e < K * K; ++e) fin = fin && isfinite(Cm[e]) && isfinite(H[e]);
    if (!fin) z.status = ST_NONFINITE;
    else if (flag[0] == 0) z.status = ST_BREAKDOWN;
    else if (flag[0] == 2 || sqrt(gam2) <= a.tol * z.bnorm) z.status = ST_CONVERGED;
    else if (q >= a.max_iter || q >= a.cap) z.status = ST_MAXIT;
    else z.status = ST_RUNNING;
    a.st[f] = z;
  }
  for (int e = tid; e < K * K; e += C::NT) {
    a.Hs[(fc + blk) * K * K + e] = H[e];
    if (q + 1 <= a.cap) {
      a.Rs[(fr + q) * K * K + e] = R[e];
      a.Ri[(fr + q) * K * K + e] = X[e];
    }
  }
}

// ------------------------------------------------------------------------- coefficients Z
// Back substitution of the stored eliminations per shift j gives column j of Q F (Eq.(soln-constr)),
// then Z = (Q F) U^{-1} = (Q F) W^T (reading R27), block by block: G_a = Z[a].
template <int K, bool D2>
__device__ void lz_coeffs(const LzArgs& a, int f, double* sm) {
  using C = LzCfg<K, D2>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = __ldcg(&a.st[f].iters);
  if (i <= 0) return;
  const size_t fc = (size_t)f * a.cap, fr = (size_t)f * (a.cap + 1);
  if (warp < K) {
    const int j = warp;
    double fv = 0.0;  // lane r holds f_a[r]
    for (int blk = i - 1; blk >= 0; --blk) {
      const double* Si = a.Sinv + ((fc + blk) * K + j) * K * K;
      double rhs = lane < K ? __ldcg(a.gv + ((fc + blk) * K + j) * K + lane) : 0.0;
      if (blk < i - 1) {  // rhs -= B_{blk+1}^T f_{blk+1}
        const double* Bn = a.Rs + (fr + blk + 1) * K * K;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c) s = fma(lane < K ? __ldcg(Bn + c * K + lane) : 0.0, __shfl_sync(0xffffffffu, fv, c), s);
        rhs -= s;
      }
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c) s = fma(lane < K ? __ldcg(Si + lane * K + c) : 0.0, __shfl_sync(0xffffffffu, rhs, c), s);
      fv = s;
      if (lane < K) a.Zs[(fc + blk) * K * K + lane * K + j] = fv;  // F[blk][r][j]
    }
  }
  __syncthreads();
  const LzFace& pf = a.prm[f];
  for (int rr = tid; rr < i * K; rr += C::NT) {  // Z[a][r][:] = F[a][r][:] W^T
    double* z = a.Zs + fc * K * K + (size_t)rr * K;
    double Fr[K];
#pragma unroll
    for (int j = 0; j < K; ++j) Fr[j] = z[j];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) s = fma(Fr[j], pf.W[c * K + j], s);
      z[c] = s;
    }
  }
}

// ------------------------------------------------------------------------- the persistent kernel
template <int K, bool HITS, bool D2>
__global__ void __launch_bounds__(LzCfg<K, D2>::NT, 1)
    lanczos_kernel(const __grid_constant__ LzArgs a, const __grid_constant__ CUtensorMap vmap) {
  using C = LzCfg<K, D2>;
  extern __shared__ __align__(128) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::DOUBLES);  // [STAGES]
  __shared__ int act[64], its[64];
  __shared__ int nact_s, qmax_s;
  const int tid = threadIdx.x, cta = blockIdx.x, ncta = gridDim.x;
  cg::grid_group grid = cg::this_grid();
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  if constexpr (!C::REGG)
    for (int e = tid; e < (C::KP - 2 * K) * C::RN; e += C::NT) sm[C::OFF_U + 2 * K * C::RN + e] = 0.0;
  __syncthreads();
  uint32_t phbits = 0;  // mbarrier phase parity per stage

  // Lanczos passes (q = 0: B_0), one grid barrier before and one after the per-face reductions
  for (int q = 0;; ++q) {
    if (tid == 0) {
      int n = 0;
      for (int f = 0; f < a.P; ++f)
        if (q == 0 || __ldcg(&a.st[f].status) == ST_RUNNING) { its[n] = 0; act[n++] = f; }
      nact_s = n;
    }
    __syncthreads();
    const int nact = nact_s;
    if (nact == 0) break;
    long long* tr = (KCG_TRACE && a.trace && q < KCG_TRACE_ITERS) ? a.trace + (size_t)q * KCG_TRACE_COLS : nullptr;
    if (tr && cta == 0 && tid == 0) tr[0] = globaltimer();
    lz_pass<K, HITS, D2>(a, &vmap, q, q == 0 ? LZ_GRAM0 : LZ_STEP, act, its, nact, sm, bar, phbits);
    if (tr && tid == 0 && 5 + cta < KCG_TRACE_COLS) tr[5 + cta] = globaltimer();
    fence_proxy_async_global();
    __threadfence();
    grid.sync();
    if (tr && cta == 0 && tid == 0) tr[2] = globaltimer();
    for (int ai = cta; ai < nact; ai += ncta) {
      lz_reduce<K, D2>(a, q, act, nact, ai, sm);
      __syncthreads();
    }
    if (tr && cta == 0 && tid == 0) tr[3] = globaltimer();
    __threadfence();
    grid.sync();
    if (tr && cta == 0 && tid == 0) tr[4] = globaltimer();
  }
  // coefficients
  for (int f = cta; f < a.P; f += ncta) {
    lz_coeffs<K, D2>(a, f, sm);
    __syncthreads();
  }
  __threadfence();
  grid.sync();
  if (a.store) return;  // lz_assemble_kernel streams the stored basis
  // replay (the paper's second Lanczos pass): rebuild V_q and add V_q G_q
  const size_t N = (size_t)a.side * a.side;
  for (int f = 0; f < a.P; ++f)
    if (__ldcg(&a.st[f].iters) == 0)
      for (size_t e = (size_t)cta * C::NT + tid; e < (size_t)K * N; e += (size_t)ncta * C::NT) a.Mx[(size_t)f * K * N + e] = 0.0;
  if (tid == 0) {
    int m = 0;
    for (int f = 0; f < a.P; ++f) m = max(m, __ldcg(&a.st[f].iters));
    qmax_s = m;
  }
  __syncthreads();
  const int qmax = qmax_s;
  for (int q = 1; q <= qmax; ++q) {
    if (tid == 0) {
      int n = 0;
      for (int f = 0; f < a.P; ++f) {
        const int it = __ldcg(&a.st[f].iters);
        if (it >= q) { its[n] = it; act[n++] = f; }
      }
      nact_s = n;
    }
    __syncthreads();
    lz_pass<K, HITS, D2>(a, &vmap, q, LZ_REPLAY, act, its, nact_s, sm, bar, phbits);
    fence_proxy_async_global();
    __threadfence();
    grid.sync();
  }
}

// M = sum_q V_q G_q from the HBM-resident basis (store mode): one streaming pass over the blocks.
// Work units = (face, 512-pixel chunk), faces interleaved so every CTA gets a mix of step counts;
// a thread owns a pixel pair (double2), four blocks q in flight; G_q of the unit's face staged in
// shared memory.  Per pixel the sum runs q-major, d-minor -- the replay's order (bitwise equal M).
#define LZ_ASM_ZMAX 2048  // doubles of G_q staged per unit (longer bases stream from L1/L2)
template <int K>
__global__ void __launch_bounds__(256) lz_assemble_kernel(const LzArgs a) {
  __shared__ double zs[LZ_ASM_ZMAX];
  const size_t N = (size_t)a.side * a.side, pstride = (size_t)a.pitch * a.side;
  const bool pairs = (a.side & 1) == 0;
  const size_t per = pairs ? 512 : 256;
  const size_t nch = (N + per - 1) / per;
  for (size_t u = blockIdx.x; u < (size_t)a.P * nch; u += gridDim.x) {
    const int f = (int)(u % a.P);
    const size_t ch = u / a.P;
    const int it = __ldcg(&a.st[f].iters);
    const double* Zg = a.Zs + (size_t)f * a.cap * K * K;
    const int nz = min(it * K * K, LZ_ASM_ZMAX);
    __syncthreads();
    for (int e = threadIdx.x; e < nz; e += blockDim.x) zs[e] = __ldcg(Zg + e);
    __syncthreads();
    // G_q from shared memory when the unit's coefficients fit (block-uniform), else from L1/L2
    auto pair_body = [&](auto zload) {
      auto Z = [&](int q, int e) { return zload((q - 1) * K * K + e); };
      const size_t px = ch * per + 2 * threadIdx.x;
      if (px >= N) return;
      const size_t gy = px / a.side, gx = px - gy * a.side;
      const size_t off = gy * a.pitch + gx;
      double2 m[K];
#pragma unroll
      for (int c = 0; c < K; ++c) m[c] = make_double2(0.0, 0.0);
      int q = 1;
      for (; q + 3 <= it; q += 4) {
        double2 v[4][K];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double* b = a.V + ((size_t)((q + r) * a.P + f) * K) * pstride + off;
#pragma unroll
          for (int d = 0; d < K; ++d) v[r][d] = __ldcs(reinterpret_cast<const double2*>(b + d * pstride));
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < K; ++c)
#pragma unroll
            for (int d = 0; d < K; ++d) {
              const double z = Z(q + r, d * K + c);
              m[c].x = fma(v[r][d].x, z, m[c].x);
              m[c].y = fma(v[r][d].y, z, m[c].y);
            }
      }
      for (; q <= it; ++q) {
        const double* b = a.V + ((size_t)(q * a.P + f) * K) * pstride + off;
        double2 v[K];
#pragma unroll
        for (int d = 0; d < K; ++d) v[d] = __ldcs(reinterpret_cast<const double2*>(b + d * pstride));
#pragma unroll
        for (int c = 0; c < K; ++c)
#pragma unroll
          for (int d = 0; d < K; ++d) {
            const double z = Z(q, d * K + c);
            m[c].x = fma(v[d].x, z, m[c].x);
            m[c].y = fma(v[d].y, z, m[c].y);
          }
      }
#pragma unroll
      for (int c = 0; c < K; ++c) *reinterpret_cast<double2*>(a.Mx + ((size_t)f * K + c) * N + px) = m[c];
    };
    if (pairs) {
      if (it * K * K <= LZ_ASM_ZMAX) pair_body([&](int o) { return zs[o]; });
      else pair_body([&](int o) { return __ldg(Zg + o); });
      continue;
    } else {  // side == 1
      auto Z = [&](int q, int e) { const int o = (q - 1) * K * K + e; return o < LZ_ASM_ZMAX ? zs[o] : __ldg(Zg + o); };
      const size_t px = ch * per + threadIdx.x;
      if (px >= N) continue;
      const size_t gy = px / a.side, gx = px - gy * a.side;
      const size_t off = gy * a.pitch + gx;
      double m[K];
#pragma unroll
      for (int c = 0; c < K; ++c) m[c] = 0.0;
      for (int q = 1; q <= it; ++q) {
        const double* b = a.V + ((size_t)(q * a.P + f) * K) * pstride + off;
        double v[K];
#pragma unroll
        for (int d = 0; d < K; ++d) v[d] = b[d * pstride];
#pragma unroll
        for (int c = 0; c < K; ++c)
#pragma unroll
          for (int d = 0; d < K; ++d) m[c] = fma(v[d], Z(q, d * K + c), m[c]);
      }
#pragma unroll
      for (int c = 0; c < K; ++c) a.Mx[((size_t)f * K + c) * N + px] = m[c];
    }
  }
}

// ------------------------------------------------------------------------- host entry points
template <int K, bool D2>
const void* lz_kernel_ptr(bool hits) {
  return hits ? (const void*)lanczos_kernel<K, true, D2> : (const void*)lanczos_kernel<K, false, D2>;
}
template <int K>
const void* lz_kernel_sel(bool hits, bool d2) {
  if constexpr (K <= 4) {
    if (d2) return lz_kernel_ptr<K, true>(hits);
  }
  return d2 ? nullptr : lz_kernel_ptr<K, false>(hits);
}

template <int K>
cudaError_t LzEntry<K>::config(bool hits, bool d2, int* max_grid, size_t* smem) {
  const void* f = lz_kernel_sel<K>(hits, d2);
  if (!f) return cudaErrorInvalidValue;  // D2 is built for K <= 4
  const size_t sm = d2 ? LzCfg<K, (K <= 4)>::SMEM : LzCfg<K, false>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, per = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  const int nt = d2 ? LzCfg<K, (K <= 4)>::NT : LzCfg<K, false>::NT;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, nt, sm)) != cudaSuccess) return e;
  *max_grid = std::min(per * nsm, KCG_LZ_GRID_MAX);
  *smem = sm;
  return cudaSuccess;
}

template <int K>
cudaError_t LzEntry<K>::launch(bool hits, bool d2, cudaStream_t s, const LzArgs& a, const CUtensorMap& vmap, int grid,
                               size_t smem) {
  void* args[2] = {(void*)&a, (void*)&vmap};
  const void* f = lz_kernel_sel<K>(hits, d2);
  if (!f) return cudaErrorInvalidValue;
  const int nt = d2 ? LzCfg<K, (K <= 4)>::NT : LzCfg<K, false>::NT;
  return cudaLaunchCooperativeKernel(f, dim3(grid), dim3(nt), args, smem, s);
}

template <int K>
cudaError_t LzEntry<K>::assemble(cudaStream_t s, const LzArgs& a) {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t N = (size_t)a.side * a.side;
  const size_t units = (size_t)a.P * ((N + 511) / 512);
  const int bx = (int)std::max<size_t>(1, std::min<size_t>(units, (size_t)nsm * 8));
  lz_assemble_kernel<K><<<bx, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace kcg
