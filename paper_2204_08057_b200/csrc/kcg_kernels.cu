// sm_100a fp64 kernels of the Kronecker CG / Sylvester hot path (arxiv 2204.08057).
//
// The operator, per system with K component planes on the 2^L x 2^L face grid:
//   q_c(j) = h_j sum_d M[c][d] p_d(j) + tau_c ( kappa2 p_c(j) + deg(j) p_c(j) - sum_{nbr} p_c(nbr) )
// which is G = M (x) N_h + P (x) (kappa2 I + L)  (Eq.(Q*) P:L75, B^T C B by Eq.(7) P:L182-196,
// Q = P (x) Q0 P:L140-148, D = -L P:L100-106, Alg.MatvecD P:L128-138 evaluated out of place).
//
// Kernels:
//   rhs_kernel            b = vec(N_h Y E) with E = T A (Kron) or T A W (Sylvester, fused F W);
//                         also zeroes x and p  -- Eq.(mu*) P:L80, Alg.MatvecBCBT P:L188-196.
//   cg_persistent_kernel  the whole CG iteration, single-pass (Chronopoulos-Gear) with
//                         recomputation, ONE grid-wide reduction per iteration, tiles staged by
//                         TMA with a 2-pixel halo (zero-filled outside the face), 2-stage mbarrier
//                         pipeline, deterministic per-system reductions, converged systems frozen.
//   apply_kernel          y = G x (parity/diagnostics) or the true residual ||b - G x||^2.
//   backtransform_kernel  X = Xt W^T per pixel (Sylvester route, reading R13).
#include "kcg_internal.h"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace kcg {

// --------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// Bounded wait: a TMA transaction that never completes (a descriptor bug) traps after ~4 s
// instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  if (mbar_try_wait(bar, phase)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, phase)) {
    if (clock64() - t0 > (1LL << 33)) __trap();
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// --------------------------------------------------------------------------- rhs
// b[p][c][j] = h_j sum_f Y[p][f][j] E[p][f][c];  r0 = b (internal pitch), p0 = 0, x = 0.
template <int K>
__global__ void __launch_bounds__(256) rhs_kernel(const double* __restrict__ Y, const double* __restrict__ E,
                                                  const double* __restrict__ hits, double* __restrict__ r0,
                                                  double* __restrict__ p0, double* __restrict__ x, int n,
                                                  int side, int pitch) {
  extern __shared__ double Es[];  // [n][K]
  const int p = blockIdx.y;
  for (int e = threadIdx.x; e < n * K; e += blockDim.x) Es[e] = E[(size_t)p * n * K + e];
  __syncthreads();
  const size_t N = (size_t)side * side;
  const size_t ps = (size_t)pitch * side;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x) {
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    const double* yp = Y + (size_t)p * n * N + j;
    for (int f = 0; f < n; ++f) {
      const double y = __ldg(yp + (size_t)f * N);
#pragma unroll
      for (int c = 0; c < K; ++c) acc[c] = fma(y, Es[f * K + c], acc[c]);
    }
    const double h = hits ? __ldg(hits + (size_t)p * N + j) : 1.0;
    const size_t gy = j / side, gx = j - gy * side;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const size_t plane = (size_t)p * K + c;
      r0[plane * ps + gy * pitch + gx] = h * acc[c];
      if (p0) p0[plane * ps + gy * pitch + gx] = 0.0;
      if (x) x[plane * N + j] = 0.0;
    }
  }
}

// --------------------------------------------------------------------------- CG scalar update
// One CG scalar step for a system from its reduced partials (r,r) and (w,r) (Chronopoulos-Gear):
// the start pass (it < 0) gives ||b||^2 and alpha_0 = (b,b)/(Gb,b); afterwards
// beta = gamma'/gamma, alpha = gamma'/(delta - beta gamma'/alpha); stop on ||r|| <= tol ||b||.
__device__ __forceinline__ SysState cg_update(SysState z, double rr, double wr, int it, const CgArgs& a) {
  if (it < 0) {
    z.bnorm2 = rr;
    z.gamma = rr;
    z.rel = rr > 0.0 ? 1.0 : 0.0;
    if (!isfinite(rr) || !isfinite(wr)) z.status = ST_NONFINITE;
    else if (rr == 0.0) z.status = ST_CONVERGED;
    else if (!(wr > 0.0)) z.status = ST_BREAKDOWN;
    else if (a.max_iter <= 0) z.status = ST_MAXIT;
    else { z.alpha = rr / wr; z.beta = 0.0; }
  } else {
    z.iters = it + 1;
    z.rel = sqrt(rr / z.bnorm2);
    if (!isfinite(rr) || !isfinite(wr)) z.status = ST_NONFINITE;
    else if (rr <= a.tol2 * z.bnorm2) z.status = ST_CONVERGED;
    else if (z.iters >= a.max_iter) z.status = ST_MAXIT;
    else {
      const double beta = rr / z.gamma;
      const double den = wr - beta * rr / z.alpha;
      if (!(den > 0.0)) z.status = ST_BREAKDOWN;
      else { z.beta = beta; z.alpha = rr / den; z.gamma = rr; }
    }
  }
  z.parity ^= 1;
  return z;
}

// After the iteration's grid barrier: CTA b reduces the tile partials of active systems b, b+grid,...
// with all its threads (one round of independent loads; thread t sums tiles t, t+NT, ... in order,
// then a fixed warp/CTA tree -> deterministic, independent of grid size and batch composition),
// publishes the new state in a.state_out; a second grid barrier; every CTA pulls the states.
template <int NT>
__device__ __forceinline__ void reduce_update_systems(const CgArgs& a, SysState* st, const int* act, int nact,
                                                      int par_out, int it, double (*red)[32]) {
  constexpr int NW = NT / 32, U = 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tps = a.tiles_per_sys;
  for (int ii = blockIdx.x; ii < nact; ii += gridDim.x) {
    const int s = act[ii];
    const double2* base = reinterpret_cast<const double2*>(a.partials + ((size_t)par_out * a.n_sys + s) * tps * 2);
    double rr = 0.0, wr = 0.0;
    for (int t0 = tid; t0 < tps; t0 += U * NT) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int tl = t0 + u * NT;
        v[u] = tl < tps ? __ldcg(base + tl) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        rr += v[u].x;
        wr += v[u].y;
      }
    }
    rr = warp_sum(rr);
    wr = warp_sum(wr);
    if (lane == 0) { red[0][warp] = rr; red[1][warp] = wr; }
    __syncthreads();
    if (tid == 0) {
      double r2 = 0.0, w2 = 0.0;
      for (int w = 0; w < NW; ++w) { r2 += red[0][w]; w2 += red[1][w]; }
      a.state_out[s] = cg_update(st[s], r2, w2, it, a);
    }
    __syncthreads();
  }
  __threadfence();
  cg::this_grid().sync();
  for (int ii = tid; ii < nact; ii += NT) {
    const int s = act[ii];
    const SysState* g = a.state_out + s;
    SysState z;
    z.bnorm2 = __ldcg(&g->bnorm2);
    z.gamma = __ldcg(&g->gamma);
    z.alpha = __ldcg(&g->alpha);
    z.beta = __ldcg(&g->beta);
    z.rel = __ldcg(&g->rel);
    z.iters = __ldcg(&g->iters);
    z.status = __ldcg(&g->status);
    z.parity = __ldcg(&g->parity);
    z.pad = 0;
    st[s] = z;
  }
  __syncthreads();
}

// --------------------------------------------------------------------------- persistent CG
// One tile of one system: box = tile + 2-pixel halo, K planes of r and p staged by TMA (zero fill
// outside the face).  Warp w owns T rows w, w+NW, ...; lane l owns the pixel PAIR at tile columns
// 2l, 2l+1 (double2 in shared and global memory); horizontal neighbours come from shuffles.
//   Phase A  p_new = r + beta p                    whole box (elementwise)
//   Phase B  q = G p_new, r_new = r - alpha q      T rows (pairs) + the 1-pixel ring (scalars)
//   Phase C  w = G r_new on T; (r,r), (w,r); x += alpha p_new
// x: with XTMA the tile's x block (64 x TY x K) is TMA-loaded into shared memory at the start of the
// tile (consumed in phase C, so its latency hides behind phases A and B); x, r_new, p_new are
// written back with coalesced 16-byte vector stores.
// EDGE = the box touches the face border (bounds checks, degree 2/3); interior tiles skip both.
struct TileCtx {
  double* R;          // r box (stage)
  double* Pp;         // p box (stage)
  double* xs;         // x block of the tile in the stage [K][TY][TX] (XTMA)
  const double* Ms;   // M (K*K) then tau (K) of this tile's system, shared
  int s, y0, x0, par;
  double alpha, beta, kappa2;
  const double* hp;   // hits plane or nullptr
  uint64_t* bar;      // stage mbarrier
  uint32_t phase;
  double* part_out;
};

template <int K, bool EDGE, bool HITS, bool XTMA>
__device__ __forceinline__ void cg_tile(const CgArgs& a, const TileCtx& tc, double (*red)[32]) {
  constexpr int TY = cg_tile_y(K), TX = KCG_TX, H = KCG_HALO;
  constexpr int BW = TX + 2 * H, BH = TY + 2 * H, PLANE = BW * BH, FIELD = K * PLANE;
  constexpr int NT = cg_threads(K), NW = NT / 32, RPW = TY / NW;
  constexpr int RP = 2 * (TX + 2) + 2 * TY;  // ring points
  static_assert(TX == 64 && RPW * NW == TY, "pair mapping needs TX = 64 and NW | TY");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int side = a.side;
  const size_t N = (size_t)side * side;
  const size_t ps = (size_t)a.pitch * side;
  double* __restrict__ R = tc.R;
  double* __restrict__ Pp = tc.Pp;
  const int s = tc.s, y0 = tc.y0, x0 = tc.x0;
  const double alpha = tc.alpha, beta = tc.beta, kappa2 = tc.kappa2;
  const int gx = x0 + 2 * lane;

  mbar_wait(tc.bar, tc.phase);

  // Phase A
  {
    double2* P2 = reinterpret_cast<double2*>(Pp);
    const double2* R2 = reinterpret_cast<const double2*>(R);
    if (beta == 0.0) {
      for (int e = tid; e < FIELD / 2; e += NT) P2[e] = R2[e];
    } else {
      for (int e = tid; e < FIELD / 2; e += NT) {
        const double2 r = R2[e];
        double2 p = P2[e];
        p.x = fma(beta, p.x, r.x);
        p.y = fma(beta, p.y, r.y);
        P2[e] = p;
      }
    }
  }
  __syncthreads();

#if KCG_M_IN_REGS
  double M[K * K];
#pragma unroll
  for (int e = 0; e < K * K; ++e) M[e] = tc.Ms[e];
#else
  const double* M = tc.Ms;
#endif
  double tau[K];
#pragma unroll
  for (int c = 0; c < K; ++c) tau[c] = tc.Ms[K * K + c];

  // Phase B1: T rows, pairs
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    const int gy = y0 + warp + j * NW;
    const int ly = gy - y0 + H;
    bool in0 = true, in1 = true;
    double kd0 = kappa2 + 4.0, kd1 = kappa2 + 4.0;
    if (EDGE) {
      in0 = gy < side && gx < side;
      in1 = gy < side && gx + 1 < side;
      const double dy = (gy == 0) + (gy == side - 1);
      kd0 = kappa2 + (4.0 - dy - (gx == 0) - (gx == side - 1));
      kd1 = kappa2 + (4.0 - dy - (gx + 1 == 0) - (gx + 1 == side - 1));
    }
    double h0 = 1.0, h1 = 1.0;
    if (HITS) {
      if (in0) h0 = __ldg(tc.hp + (size_t)gy * side + gx);
      if (in1) h1 = __ldg(tc.hp + (size_t)gy * side + gx + 1);
    }
    double2 pc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) pc[c] = reinterpret_cast<const double2*>(Pp + c * PLANE + ly * BW)[1 + lane];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double* row = Pp + c * PLANE + ly * BW;
      const double2 up = reinterpret_cast<const double2*>(row - BW)[1 + lane];
      const double2 dn = reinterpret_cast<const double2*>(row + BW)[1 + lane];
      const double el = row[H - 1], er = row[H + TX];  // broadcast loads, no branch
      double left = __shfl_up_sync(0xffffffffu, pc[c].y, 1);
      double right = __shfl_down_sync(0xffffffffu, pc[c].x, 1);
      left = lane == 0 ? el : left;
      right = lane == 31 ? er : right;
      const double nb0 = (up.x + dn.x) + (left + pc[c].y);
      const double nb1 = (up.y + dn.y) + (pc[c].x + right);
      double mix0 = 0.0, mix1 = 0.0;
#pragma unroll
      for (int d = 0; d < K; ++d) {
        mix0 = fma(M[c * K + d], pc[d].x, mix0);
        mix1 = fma(M[c * K + d], pc[d].y, mix1);
      }
      const double q0 = HITS ? fma(h0, mix0, tau[c] * fma(kd0, pc[c].x, -nb0)) : fma(tau[c], fma(kd0, pc[c].x, -nb0), mix0);
      const double q1 = HITS ? fma(h1, mix1, tau[c] * fma(kd1, pc[c].y, -nb1)) : fma(tau[c], fma(kd1, pc[c].y, -nb1), mix1);
      double2* rp = reinterpret_cast<double2*>(R + c * PLANE + ly * BW) + 1 + lane;
      double2 rv = *rp;
      if (in0) rv.x = fma(-alpha, q0, rv.x);
      if (in1) rv.y = fma(-alpha, q1, rv.y);
      *rp = rv;
    }
  }
  // Phase B2: the 1-pixel ring around T (scalars)
  for (int t = tid; t < RP; t += NT) {
    int ly, lx;
    if (t < TX + 2) { ly = H - 1; lx = H - 1 + t; }
    else if (t < 2 * (TX + 2)) { ly = H + TY; lx = H - 1 + (t - (TX + 2)); }
    else { const int u = t - 2 * (TX + 2); ly = H + (u >> 1); lx = (u & 1) ? H + TX : H - 1; }
    const int gyr = y0 - H + ly, gxr = x0 - H + lx;
    double kd = kappa2 + 4.0;
    if (EDGE) {
      if (gyr < 0 || gyr >= side || gxr < 0 || gxr >= side) continue;
      kd = kappa2 + (4.0 - (gyr == 0) - (gyr == side - 1) - (gxr == 0) - (gxr == side - 1));
    }
    const double h = HITS ? __ldg(tc.hp + (size_t)gyr * side + gxr) : 1.0;
    const int o = ly * BW + lx;
    double pcs[K];
#pragma unroll
    for (int c = 0; c < K; ++c) pcs[c] = Pp[c * PLANE + o];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double* pl = Pp + c * PLANE + o;
      const double nb = (pl[-BW] + pl[BW]) + (pl[-1] + pl[1]);
      double mix = 0.0;
#pragma unroll
      for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], pcs[d], mix);
      const double q = HITS ? fma(h, mix, tau[c] * fma(kd, pcs[c], -nb)) : fma(tau[c], fma(kd, pcs[c], -nb), mix);
      R[c * PLANE + o] = fma(-alpha, q, R[c * PLANE + o]);
    }
  }
  __syncthreads();

  // Phase C
  double rr = 0.0, wr = 0.0;
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    const int gy = y0 + warp + j * NW;
    const int ly = gy - y0 + H;
    bool in0 = true, in1 = true;
    double kd0 = kappa2 + 4.0, kd1 = kappa2 + 4.0;
    if (EDGE) {
      in0 = gy < side && gx < side;
      in1 = gy < side && gx + 1 < side;
      const double dy = (gy == 0) + (gy == side - 1);
      kd0 = kappa2 + (4.0 - dy - (gx == 0) - (gx == side - 1));
      kd1 = kappa2 + (4.0 - dy - (gx + 1 == 0) - (gx + 1 == side - 1));
    }
    double h0 = 1.0, h1 = 1.0;
    if (HITS) {
      if (in0) h0 = __ldg(tc.hp + (size_t)gy * side + gx);
      if (in1) h1 = __ldg(tc.hp + (size_t)gy * side + gx + 1);
    }
    double* xp = a.x + ((size_t)s * K * side + gy) * side + gx;
    double2 xj[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      if (XTMA) {
        xj[c] = reinterpret_cast<const double2*>(tc.xs + ((size_t)c * TY + (gy - y0)) * TX)[lane];
      } else if (!EDGE || (in0 && in1)) {
        xj[c] = __ldcg(reinterpret_cast<const double2*>(xp + c * N));
      } else {
        xj[c].x = in0 ? __ldcg(xp + c * N) : 0.0;
        xj[c].y = in1 ? __ldcg(xp + c * N + 1) : 0.0;
      }
    }
    double2 rc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) rc[c] = reinterpret_cast<const double2*>(R + c * PLANE + ly * BW)[1 + lane];
    const size_t ro = ((size_t)s * K) * ps + (size_t)gy * a.pitch + gx;
    double* rout = (tc.par ? a.rbuf[0] : a.rbuf[1]) + ro;  // select, not a dynamic param index
    double* pout = (tc.par ? a.pbuf[0] : a.pbuf[1]) + ro;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double* row = R + c * PLANE + ly * BW;
      const double2 up = reinterpret_cast<const double2*>(row - BW)[1 + lane];
      const double2 dn = reinterpret_cast<const double2*>(row + BW)[1 + lane];
      const double el = row[H - 1], er = row[H + TX];
      double left = __shfl_up_sync(0xffffffffu, rc[c].y, 1);
      double right = __shfl_down_sync(0xffffffffu, rc[c].x, 1);
      left = lane == 0 ? el : left;
      right = lane == 31 ? er : right;
      const double nb0 = (up.x + dn.x) + (left + rc[c].y);
      const double nb1 = (up.y + dn.y) + (rc[c].x + right);
      double mix0 = 0.0, mix1 = 0.0;
#pragma unroll
      for (int d = 0; d < K; ++d) {
        mix0 = fma(M[c * K + d], rc[d].x, mix0);
        mix1 = fma(M[c * K + d], rc[d].y, mix1);
      }
      const double w0 = HITS ? fma(h0, mix0, tau[c] * fma(kd0, rc[c].x, -nb0)) : fma(tau[c], fma(kd0, rc[c].x, -nb0), mix0);
      const double w1 = HITS ? fma(h1, mix1, tau[c] * fma(kd1, rc[c].y, -nb1)) : fma(tau[c], fma(kd1, rc[c].y, -nb1), mix1);
      const double2 pn = reinterpret_cast<const double2*>(Pp + c * PLANE + ly * BW)[1 + lane];
      double2 xn;
      xn.x = fma(alpha, pn.x, xj[c].x);
      xn.y = fma(alpha, pn.y, xj[c].y);
      if (!EDGE || (in0 && in1)) {
        rr = fma(rc[c].x, rc[c].x, rr);
        wr = fma(w0, rc[c].x, wr);
        rr = fma(rc[c].y, rc[c].y, rr);
        wr = fma(w1, rc[c].y, wr);
        *reinterpret_cast<double2*>(xp + c * N) = xn;
        *reinterpret_cast<double2*>(rout + c * ps) = rc[c];
        *reinterpret_cast<double2*>(pout + c * ps) = pn;
      } else {
        if (in0) {
          rr = fma(rc[c].x, rc[c].x, rr);
          wr = fma(w0, rc[c].x, wr);
          xp[c * N] = xn.x;
          rout[c * ps] = rc[c].x;
          pout[c * ps] = pn.x;
        }
        if (in1) {
          rr = fma(rc[c].y, rc[c].y, rr);
          wr = fma(w1, rc[c].y, wr);
          xp[c * N + 1] = xn.y;
          rout[c * ps + 1] = rc[c].y;
          pout[c * ps + 1] = pn.y;
        }
      }
    }
  }
  rr = warp_sum(rr);
  wr = warp_sum(wr);
  if (lane == 0) { red[0][warp] = rr; red[1][warp] = wr; }
  __syncthreads();
  if (warp == 0) {
    double v0 = lane < NW ? red[0][lane] : 0.0;
    double v1 = lane < NW ? red[1][lane] : 0.0;
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    if (lane == 0) { tc.part_out[0] = v0; tc.part_out[1] = v1; }
  }
}

template <int K, bool HITS>
__global__ void __launch_bounds__(cg_threads(K), cg_min_blocks(K)) cg_persistent_kernel(const CgArgs a, const __grid_constant__ CgMaps maps) {
  constexpr int TY = cg_tile_y(K), TX = KCG_TX, H = KCG_HALO;
  constexpr int BW = TX + 2 * H, BH = TY + 2 * H;
  constexpr int FIELD = K * BW * BH;  // doubles of one field box
  constexpr int XBYTES = cg_xstage_bytes(K);  // x block, TMA-staged with the boxes (0 if disabled)
  constexpr int STAGE_BYTES = 2 * FIELD * 8 + XBYTES;
  constexpr int NT = cg_threads(K), NW = NT / 32, NS = cg_stages(K);
  static_assert(STAGE_BYTES == cg_stage_bytes(K), "stage size");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  SysState* st = reinterpret_cast<SysState*>(smem_raw + NS * STAGE_BYTES);
  int* act = reinterpret_cast<int*>(st + a.n_sys);
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double red[2][32];
  __shared__ double Ms[KCG_KMAX * KCG_KMAX + KCG_KMAX];
  __shared__ int s_nact;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tps = a.tiles_per_sys;
  const bool xtma = cg_xtma(K) && a.x_tma != 0;
  cg::grid_group grid = cg::this_grid();

  for (int s = tid; s < a.n_sys; s += NT) {
    SysState z;
    z.bnorm2 = 0.0; z.gamma = 0.0; z.alpha = 0.0; z.beta = 0.0; z.rel = 1.0;
    z.iters = 0; z.status = ST_RUNNING; z.parity = 0; z.pad = 0;
    st[s] = z;
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint32_t phase0 = 0, phase1 = 0;
  int it = -1;  // -1 = start pass (alpha = beta = 0): r, p <- b and (b, b), (G b, b)

  // TMA of tile t (index into the active-tile list) into stage sidx; parity flip for speculation
  auto issue = [&](int t, int sidx, int flip) {
    const int s = act[t / tps];
    const int tile = t - (t / tps) * tps;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int par = st[s].parity ^ flip;
    double* dst = reinterpret_cast<double*>(smem_raw + sidx * STAGE_BYTES);
    mbar_arrive_expect_tx(&mbar[sidx], xtma ? STAGE_BYTES : 2 * FIELD * 8);
    if (xtma) tma_load_3d(dst + 2 * FIELD, &maps.x, &mbar[sidx], tx * TX, ty * TY, s * K);
    tma_load_3d(dst, &maps.r[par], &mbar[sidx], tx * TX - H, ty * TY - H, s * K);
    tma_load_3d(dst + FIELD, &maps.p[par], &mbar[sidx], tx * TX - H, ty * TY - H, s * K);
  };

  int nact_prev = -1;
  bool spec = false;  // a speculative first TMA of this iteration is in flight in stage 0
  while (true) {
    if (tid == 0) {
      int n = 0;
      for (int s = 0; s < a.n_sys; ++s)
        if (st[s].status == ST_RUNNING) act[n++] = s;
      s_nact = n;
    }
    __syncthreads();
    const int nact = s_nact;
    if (spec && nact != nact_prev) {  // mis-speculated: drain the stale load before reusing stage 0
      mbar_wait(&mbar[0], phase0);
      phase0 ^= 1u;
      spec = false;
    }
    if (nact == 0) break;
    const int ntiles = nact * tps;
    const int par_out = (it + 1) & 1;
    const bool tr = KCG_TRACE && a.trace && it + 1 < KCG_TRACE_ITERS;
    if (tr && blockIdx.x == 0 && tid == 0) a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 0] = globaltimer();

    if (!spec && (int)blockIdx.x < ntiles && tid == 0) issue(blockIdx.x, 0, 0);
    spec = false;
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int sidx = NS == 2 ? (i & 1) : 0;
      const int tn = t + gridDim.x;
      __syncthreads();
      if (tid == 0) {
        if (NS == 2 && tn < ntiles) {
          fence_proxy_async_smem();
          issue(tn, sidx ^ 1, 0);
        } else if (NS == 1 && i > 0) {
          fence_proxy_async_smem();
          issue(t, 0, 0);
        }
      }
      const int s = act[t / tps];
      const int tile = t - (t / tps) * tps;
      const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
      const SysParams* sp = a.params + s;
      if (tid < K * K) Ms[tid] = __ldg(&sp->M[tid]);
      else if (tid < K * K + K) Ms[tid] = __ldg(&sp->tau[tid - K * K]);
      TileCtx tc;
      tc.R = reinterpret_cast<double*>(smem_raw + sidx * STAGE_BYTES);
      tc.Pp = tc.R + FIELD;
      tc.xs = tc.R + 2 * FIELD;
      tc.Ms = Ms;
      tc.s = s;
      tc.y0 = ty * TY;
      tc.x0 = tx * TX;
      tc.par = st[s].parity;
      tc.alpha = st[s].alpha;
      tc.beta = st[s].beta;
      tc.kappa2 = __ldg(&sp->kappa2);
      tc.hp = HITS ? a.hits + (size_t)__ldg(&sp->hits_plane) * ((size_t)a.side * a.side) : nullptr;
      tc.bar = &mbar[sidx];
      tc.phase = sidx ? phase1 : phase0;
      tc.part_out = a.partials + (((size_t)par_out * a.n_sys + s) * tps + tile) * 2;
      const bool interior = tc.x0 >= H && tc.x0 + TX + H <= a.side && tc.y0 >= H && tc.y0 + TY + H <= a.side;
      if (cg_xtma(K) && xtma) {
        if (interior) cg_tile<K, false, HITS, cg_xtma(K)>(a, tc, red);
        else cg_tile<K, true, HITS, cg_xtma(K)>(a, tc, red);
      } else {
        if (interior) cg_tile<K, false, HITS, false>(a, tc, red);
        else cg_tile<K, true, HITS, false>(a, tc, red);
      }
      if (sidx) phase1 ^= 1u; else phase0 ^= 1u;
    }

    if (tr && tid == 0 && blockIdx.x < KCG_TRACE_COLS - 3)
      a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 3 + blockIdx.x] = globaltimer();
    fence_proxy_async_global();
    grid.sync();
    fence_proxy_async_global();
    if (tr && blockIdx.x == 0 && tid == 0) a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 1] = globaltimer();
    // speculative first load of the next iteration (same active set, flipped parity) overlaps the
    // reduction below; verified against the new active count at the top of the loop
    if (it >= 0 && (int)blockIdx.x < ntiles && tid == 0) issue(blockIdx.x, 0, 1);
    spec = it >= 0 && (int)blockIdx.x < ntiles;
    nact_prev = nact;

    reduce_update_systems<NT>(a, st, act, nact, par_out, it, red);
    if (tr && blockIdx.x == 0 && tid == 0) a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 2] = globaltimer();
    if (blockIdx.x == 0 && tid == 0 && it >= 0 && it < a.history_cap) {
      double m = 0.0;
      for (int ii = 0; ii < nact; ++ii) m = fmax(m, st[act[ii]].rel);
      a.history[it] = m;
    }
    ++it;
  }
  if (blockIdx.x == 0)
    for (int s = tid; s < a.n_sys; s += NT) a.state_out[s] = st[s];
}

// --------------------------------------------------------------------------- warp-marching CG
// The production CG kernel.  Same single-pass Chronopoulos-Gear iteration, same per-tile partials
// and per-system reductions as cg_persistent_kernel, but each WARP owns a 60 x 16 output tile and
// marches down its 64-wide box (2-pixel halo) row by row:
//   box rows arrive through a per-warp ring of TMA chunks (CR rows x 64 cols x K planes, r and p,
//   zero-filled outside the face); per lane a PAIR of columns (32 lanes x 2 = the 64 box columns,
//   so the halo needs no special lanes); horizontal neighbours by shuffles; vertical neighbours
//   from a 3-row register window of p_new and r_new:
//     step b:  p_new(b) = r(b) + beta p(b)
//              r_new(b-1) = r(b-1) - alpha G p_new(b-1)          (rows b-2..b of p_new)
//              w(b-2) = G r_new(b-2); (r,r), (w,r); x += alpha p_new; store x, r_new, p_new (b-2)
// No block-level barrier inside an iteration; shared memory only receives the TMA data and is read
// once per element.  Columns 0/63 of the box produce garbage that no output uses.
__device__ __forceinline__ double2 shfl_up2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

template <int K, bool EDGE, bool HITS>
__device__ __forceinline__ void march_apply(const double2 (&up)[K], const double2 (&ctr)[K], const double2 (&dn)[K],
                                            const double* __restrict__ M, const double* __restrict__ tau, double kd0,
                                            double kd1, double h0, double h1, int lane, double2 (&out)[K]) {
  double mix0[K], mix1[K];
#pragma unroll
  for (int c = 0; c < K; ++c) {
    mix0[c] = 0.0;
    mix1[c] = 0.0;
#pragma unroll
    for (int d = 0; d < K; ++d) {
      mix0[c] = fma(M[c * K + d], ctr[d].x, mix0[c]);
      mix1[c] = fma(M[c * K + d], ctr[d].y, mix1[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < K; ++c) {
    double left = __shfl_up_sync(0xffffffffu, ctr[c].y, 1);
    double right = __shfl_down_sync(0xffffffffu, ctr[c].x, 1);
    left = lane == 0 ? 0.0 : left;
    right = lane == 31 ? 0.0 : right;
    const double nb0 = (up[c].x + dn[c].x) + (left + ctr[c].y);
    const double nb1 = (up[c].y + dn[c].y) + (ctr[c].x + right);
    if (HITS) {
      out[c].x = fma(h0, mix0[c], tau[c] * fma(kd0, ctr[c].x, -nb0));
      out[c].y = fma(h1, mix1[c], tau[c] * fma(kd1, ctr[c].y, -nb1));
    } else {
      out[c].x = fma(tau[c], fma(kd0, ctr[c].x, -nb0), mix0[c]);
      out[c].y = fma(tau[c], fma(kd1, ctr[c].y, -nb1), mix1[c]);
    }
  }
}

struct MarchWarp {
  uint64_t* bar;       // NB mbarriers of this warp
  double* ring;        // NB chunks of this warp
  long long seq;       // chunks consumed by this warp since kernel start (mbarrier phases)
};

template <int K, bool EDGE, bool HITS>
__device__ __forceinline__ void march_tile(const CgArgs& a, const CgMaps& maps, MarchWarp& mw,
                                           const double* __restrict__ Ms, int s, int y0, int x0, int par,
                                           double alpha, double beta, double kappa2, const double* __restrict__ hp,
                                           double* part_out, int lane, int& issued, int total_chunks, int q0,
                                           const int* act, const SysState* st, int tps, int gwarp,
                                           int nwarps_total) {
  constexpr int BW = 64, TY = MARCH_TY, BR = TY + 4, CR = march_cr(K), NB = march_nb(K);
  constexpr int NCH = BR / CR;
  constexpr int CHUNK = 2 * K * CR * BW;  // doubles: r [K][CR][64] then p [K][CR][64]
  static_assert(BR % CR == 0, "chunk rows");
  const int side = a.side;
  const size_t N = (size_t)side * side;
  const size_t ps = (size_t)a.pitch * side;
  double M[K * K], tau[K];
#pragma unroll
  for (int e = 0; e < K * K; ++e) M[e] = Ms[e];
#pragma unroll
  for (int c = 0; c < K; ++c) tau[c] = Ms[K * K + c];
  const int gx = x0 - 2 + 2 * lane;  // global column of .x
  const bool out_lane = lane >= 1 && lane <= 30;
  double* rout = (par ? a.rbuf[0] : a.rbuf[1]) + (size_t)s * K * ps;
  double* pout = (par ? a.pbuf[0] : a.pbuf[1]) + (size_t)s * K * ps;
  double* xbase = a.x + (size_t)s * K * N;

  // column masks / degrees that do not depend on the row
  bool cin0 = true, cin1 = true;
  double dx0 = 0.0, dx1 = 0.0;
  if (EDGE) {
    cin0 = gx >= 0 && gx < side;
    cin1 = gx + 1 >= 0 && gx + 1 < side;
    dx0 = (gx == 0) + (gx == side - 1);
    dx1 = (gx + 1 == 0) + (gx + 1 == side - 1);
  }

  double2 pnA[K], pnB[K], pnC[K], rnA[K], rnB[K], rnC[K], rprev[K], xa[K];
  double rr = 0.0, wr = 0.0;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    pnA[c] = pnB[c] = rnA[c] = rnB[c] = rprev[c] = xa[c] = make_double2(0.0, 0.0);
  }

  auto load_x = [&](double2 (&xr)[K], int o) {  // x of output box row o (o in [2, TY+1])
    const int gy = y0 - 2 + o;
    const bool ok = out_lane && (!EDGE || (gy < side && cin0 && cin1));
#pragma unroll
    for (int c = 0; c < K; ++c) {
      if (ok) xr[c] = __ldcg(reinterpret_cast<const double2*>(xbase + ((size_t)c * side + gy) * side + gx));
      else if (EDGE && out_lane && gy < side && (cin0 || cin1)) {
        xr[c].x = cin0 ? __ldcg(xbase + ((size_t)c * side + gy) * side + gx) : 0.0;
        xr[c].y = cin1 ? __ldcg(xbase + ((size_t)c * side + gy) * side + gx + 1) : 0.0;
      } else xr[c] = make_double2(0.0, 0.0);
    }
  };
  for (int b = 0; b < BR; ++b) {
    const int ch = b / CR, rb = b - ch * CR;
    const long long g = mw.seq + q0 + ch;  // global chunk sequence number
    const int slot = (int)(g % NB);
    if (rb == 0) {
      // keep NB-1 chunks in flight along this warp's chunk stream (may run into its next tile)
      const int want = min(q0 + ch + NB, total_chunks);
      __syncwarp();  // every lane is done reading the slot about to be refilled
      if (lane == 0) {
        while (issued < want) {
          const int qi = issued;
          const int ti = qi / NCH, ci = qi - ti * NCH;
          const int t = gwarp + ti * nwarps_total;
          const int si = act[t / tps];
          const int tile = t - (t / tps) * tps;
          const int tyi = tile / a.tiles_x, txi = tile - tyi * a.tiles_x;
          const long long gi = mw.seq + qi;
          const int sl = (int)(gi % NB);
          // the slot's previous chunk (gi - NB) was fully read by this warp before this point
          fence_proxy_async_smem();
          double* dst = mw.ring + (size_t)sl * CHUNK;
          mbar_arrive_expect_tx(&mw.bar[sl], CHUNK * 8);
          const int pi = st[si].parity;
          tma_load_3d(dst, &maps.r[pi], &mw.bar[sl], txi * MARCH_TX - 2, tyi * TY - 2 + ci * CR, si * K);
          tma_load_3d(dst + K * CR * BW, &maps.p[pi], &mw.bar[sl], txi * MARCH_TX - 2, tyi * TY - 2 + ci * CR, si * K);
          ++issued;
        }
      }
      issued = __shfl_sync(0xffffffffu, issued, 0);
      mbar_wait(&mw.bar[slot], (uint32_t)((g / NB) & 1));
    }
    if (b >= 4) load_x(xa, b - 2);  // x of this step's output row; used at the end of the step
    const double* rrow = mw.ring + (size_t)slot * CHUNK + rb * BW;
    const double* prow = rrow + K * CR * BW;
    double2 rcur[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      rcur[c] = reinterpret_cast<const double2*>(rrow + c * CR * BW)[lane];
      const double2 pv = reinterpret_cast<const double2*>(prow + c * CR * BW)[lane];
      pnC[c].x = fma(beta, pv.x, rcur[c].x);
      pnC[c].y = fma(beta, pv.y, rcur[c].y);
    }
    if (b >= 2) {  // r_new of box row m = b - 1
      const int gy = y0 - 2 + (b - 1);
      double kd0 = kappa2 + 4.0, kd1 = kappa2 + 4.0;
      bool in0 = true, in1 = true;
      if (EDGE) {
        const bool rin = gy >= 0 && gy < side;
        in0 = rin && cin0;
        in1 = rin && cin1;
        const double dy = (gy == 0) + (gy == side - 1);
        kd0 = kappa2 + (4.0 - dy - dx0);
        kd1 = kappa2 + (4.0 - dy - dx1);
      }
      double h0 = 1.0, h1 = 1.0;
      if (HITS) {
        if (in0) h0 = __ldg(hp + (size_t)gy * side + gx);
        if (in1) h1 = __ldg(hp + (size_t)gy * side + gx + 1);
      }
      double2 q[K];
      march_apply<K, EDGE, HITS>(pnA, pnB, pnC, M, tau, kd0, kd1, h0, h1, lane, q);
#pragma unroll
      for (int c = 0; c < K; ++c) {
        rnC[c].x = in0 ? fma(-alpha, q[c].x, rprev[c].x) : 0.0;
        rnC[c].y = in1 ? fma(-alpha, q[c].y, rprev[c].y) : 0.0;
      }
      if (b >= 4) {  // outputs of box row o = b - 2
        const int o = b - 2;
        const int gyo = y0 - 2 + o;
        double kdo0 = kappa2 + 4.0, kdo1 = kappa2 + 4.0;
        bool on0 = out_lane, on1 = out_lane;
        if (EDGE) {
          const bool rin = gyo < side;
          on0 = on0 && rin && cin0;
          on1 = on1 && rin && cin1;
          const double dy = (gyo == 0) + (gyo == side - 1);
          kdo0 = kappa2 + (4.0 - dy - dx0);
          kdo1 = kappa2 + (4.0 - dy - dx1);
        }
        double ho0 = 1.0, ho1 = 1.0;
        if (HITS) {
          if (on0) ho0 = __ldg(hp + (size_t)gyo * side + gx);
          if (on1) ho1 = __ldg(hp + (size_t)gyo * side + gx + 1);
        }
        double2 w[K];
        march_apply<K, EDGE, HITS>(rnA, rnB, rnC, M, tau, kdo0, kdo1, ho0, ho1, lane, w);
        const size_t xo = (size_t)gyo * side + gx;
        const size_t ro = (size_t)gyo * a.pitch + gx;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          double2 xn;
          xn.x = fma(alpha, pnA[c].x, xa[c].x);
          xn.y = fma(alpha, pnA[c].y, xa[c].y);
          if (!EDGE || (on0 && on1)) {
            if (out_lane) {
              rr = fma(rnB[c].x, rnB[c].x, rr);
              rr = fma(rnB[c].y, rnB[c].y, rr);
              wr = fma(w[c].x, rnB[c].x, wr);
              wr = fma(w[c].y, rnB[c].y, wr);
              *reinterpret_cast<double2*>(xbase + c * N + xo) = xn;
              *reinterpret_cast<double2*>(rout + c * ps + ro) = rnB[c];
              *reinterpret_cast<double2*>(pout + c * ps + ro) = pnA[c];
            }
          } else {
            if (on0) {
              rr = fma(rnB[c].x, rnB[c].x, rr);
              wr = fma(w[c].x, rnB[c].x, wr);
              xbase[c * N + xo] = xn.x;
              rout[c * ps + ro] = rnB[c].x;
              pout[c * ps + ro] = pnA[c].x;
            }
            if (on1) {
              rr = fma(rnB[c].y, rnB[c].y, rr);
              wr = fma(w[c].y, rnB[c].y, wr);
              xbase[c * N + xo + 1] = xn.y;
              rout[c * ps + ro + 1] = rnB[c].y;
              pout[c * ps + ro + 1] = pnA[c].y;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < K; ++c) {
        rnA[c] = rnB[c];
        rnB[c] = rnC[c];
      }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      pnA[c] = pnB[c];
      pnB[c] = pnC[c];
      rprev[c] = rcur[c];
    }
  }
  rr = warp_sum(rr);
  wr = warp_sum(wr);
  if (lane == 0) {
    part_out[0] = rr;
    part_out[1] = wr;
  }
}

template <int K, bool HITS>
__global__ void __launch_bounds__(32 * march_warps(K), 1) cg_march_kernel(const CgArgs a, const __grid_constant__ CgMaps maps) {
  constexpr int BW = 64, TY = MARCH_TY, BR = TY + 4, CR = march_cr(K), NB = march_nb(K), W = march_warps(K);
  constexpr int NCH = BR / CR;
  constexpr int CHUNK = 2 * K * CR * BW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring_all = reinterpret_cast<double*>(smem_raw);
  SysState* st = reinterpret_cast<SysState*>(smem_raw + (size_t)W * NB * CHUNK * 8);
  int* act = reinterpret_cast<int*>(st + a.n_sys);
  __shared__ __align__(8) uint64_t mbar[W * NB];
  __shared__ double Msh[W][KCG_KMAX * KCG_KMAX + KCG_KMAX];
  __shared__ double red[2][32];
  __shared__ int s_nact;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tps = a.tiles_per_sys;
  const int gwarp = blockIdx.x * W + warp, nwarps_total = gridDim.x * W;
  cg::grid_group grid = cg::this_grid();

  for (int s = tid; s < a.n_sys; s += blockDim.x) {
    SysState z;
    z.bnorm2 = 0.0; z.gamma = 0.0; z.alpha = 0.0; z.beta = 0.0; z.rel = 1.0;
    z.iters = 0; z.status = ST_RUNNING; z.parity = 0; z.pad = 0;
    st[s] = z;
  }
  if (tid < W * NB) mbar_init(&mbar[tid], 1);
  if (tid == 0) fence_mbar_init();
  __syncthreads();

  MarchWarp mw;
  mw.bar = &mbar[warp * NB];
  mw.ring = ring_all + (size_t)warp * NB * CHUNK;
  mw.seq = 0;
  int it = -1;

  while (true) {
    if (tid == 0) {
      int n = 0;
      for (int s = 0; s < a.n_sys; ++s)
        if (st[s].status == ST_RUNNING) act[n++] = s;
      s_nact = n;
    }
    __syncthreads();
    const int nact = s_nact;
    if (nact == 0) break;
    const int ntiles = nact * tps;
    const int par_out = (it + 1) & 1;
    const int my_tiles = gwarp < ntiles ? (ntiles - gwarp + nwarps_total - 1) / nwarps_total : 0;
    const int total_chunks = my_tiles * NCH;
    int issued = 0;
    for (int i = 0; i < my_tiles; ++i) {
      const int t = gwarp + i * nwarps_total;
      const int s = act[t / tps];
      const int tile = t - (t / tps) * tps;
      const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
      const SysParams* sp = a.params + s;
      for (int e = lane; e < K * K; e += 32) Msh[warp][e] = __ldg(&sp->M[e]);
      if (lane < K) Msh[warp][K * K + lane] = __ldg(&sp->tau[lane]);
      __syncwarp();
      const int y0 = ty * TY, x0 = tx * MARCH_TX;
      const double* hp = HITS ? a.hits + (size_t)__ldg(&sp->hits_plane) * ((size_t)a.side * a.side) : nullptr;
      double* part = a.partials + (((size_t)par_out * a.n_sys + s) * tps + tile) * 2;
      const bool interior = x0 >= 2 && x0 + MARCH_TX + 2 <= a.side && y0 >= 2 && y0 + TY + 2 <= a.side;
      if (interior)
        march_tile<K, false, HITS>(a, maps, mw, Msh[warp], s, y0, x0, st[s].parity, st[s].alpha, st[s].beta,
                                   __ldg(&sp->kappa2), hp, part, lane, issued, total_chunks, i * NCH, act, st, tps,
                                   gwarp, nwarps_total);
      else
        march_tile<K, true, HITS>(a, maps, mw, Msh[warp], s, y0, x0, st[s].parity, st[s].alpha, st[s].beta,
                                  __ldg(&sp->kappa2), hp, part, lane, issued, total_chunks, i * NCH, act, st, tps,
                                  gwarp, nwarps_total);
      __syncwarp();
    }
    mw.seq += total_chunks;

    fence_proxy_async_global();
    grid.sync();
    fence_proxy_async_global();

    reduce_update_systems<32 * W>(a, st, act, nact, par_out, it, red);
    if (blockIdx.x == 0 && tid == 0 && it >= 0 && it < a.history_cap) {
      double m = 0.0;
      for (int ii = 0; ii < nact; ++ii) m = fmax(m, st[act[ii]].rel);
      a.history[it] = m;
    }
    ++it;
  }
  if (blockIdx.x == 0)
    for (int s = tid; s < a.n_sys; s += blockDim.x) a.state_out[s] = st[s];
}

// --------------------------------------------------------------------------- apply / residual
constexpr int AP_TY = 16, AP_TX = 64, AP_NT = 256;

int apply_tiles_per_sys(int side) {
  return ((side + AP_TY - 1) / AP_TY) * ((side + AP_TX - 1) / AP_TX);
}

// RESID = false: y = G x.   RESID = true: partials[s][tile] = (||b - G x||^2, ||b||^2) over the
// tile, with b = h Y E recomputed from the data (E = T A).
template <int K, bool RESID>
__global__ void __launch_bounds__(AP_NT) apply_kernel(const SysParams* __restrict__ params,
                                                      const double* __restrict__ x, double* __restrict__ y,
                                                      const double* __restrict__ Y, const double* __restrict__ E,
                                                      const double* __restrict__ hits,
                                                      double* __restrict__ partials, int n, int side) {
  constexpr int BW = AP_TX + 2, BH = AP_TY + 2, PLANE = BW * BH;
  extern __shared__ double xs[];  // [K][BH][BW], then E [n][K] if RESID
  __shared__ double red[2][AP_NT / 32];
  const int s = blockIdx.y;
  const int tiles_x = (side + AP_TX - 1) / AP_TX;
  const int tile = blockIdx.x;
  const int ty0 = (tile / tiles_x) * AP_TY, tx0 = (tile % tiles_x) * AP_TX;
  const size_t N = (size_t)side * side;
  const SysParams* sp = params + s;
  for (int e = threadIdx.x; e < K * PLANE; e += AP_NT) {
    const int c = e / PLANE, r = e - c * PLANE;
    const int gy = ty0 - 1 + r / BW, gx = tx0 - 1 + r % BW;
    xs[e] = (gy >= 0 && gy < side && gx >= 0 && gx < side) ? x[((size_t)(s * K + c) * side + gy) * side + gx] : 0.0;
  }
  double* Es = xs + K * PLANE;
  if (RESID)
    for (int e = threadIdx.x; e < n * K; e += AP_NT) Es[e] = E[(size_t)s * n * K + e];
  __syncthreads();
  double M[K * K], tau[K];
#pragma unroll
  for (int e = 0; e < K * K; ++e) M[e] = sp->M[e];
#pragma unroll
  for (int c = 0; c < K; ++c) tau[c] = sp->tau[c];
  const double kappa2 = sp->kappa2;
  const double* hp = hits ? hits + (size_t)sp->hits_plane * N : nullptr;
  double acc0 = 0.0, acc1 = 0.0;
  for (int pt = threadIdx.x; pt < AP_TY * AP_TX; pt += AP_NT) {
    const int gy = ty0 + pt / AP_TX, gx = tx0 + pt % AP_TX;
    if (gy >= side || gx >= side) continue;
    const int o = (pt / AP_TX + 1) * BW + pt % AP_TX + 1;
    const double deg = 4.0 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1);
    const double h = hp ? hp[(size_t)gy * side + gx] : 1.0;
    double xc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) xc[c] = xs[c * PLANE + o];
    double bq[K];
    if (RESID) {
#pragma unroll
      for (int c = 0; c < K; ++c) bq[c] = 0.0;
      const double* yp = Y + (size_t)s * n * N + (size_t)gy * side + gx;
      for (int f = 0; f < n; ++f) {
        const double yv = yp[(size_t)f * N];
#pragma unroll
        for (int c = 0; c < K; ++c) bq[c] = fma(yv, Es[f * K + c], bq[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double* xl = xs + c * PLANE + o;
      const double nb = (xl[-BW] + xl[BW]) + (xl[-1] + xl[1]);
      double mix = 0.0;
#pragma unroll
      for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], xc[d], mix);
      const double q = fma(h, mix, tau[c] * fma(kappa2 + deg, xc[c], -nb));
      if (RESID) {
        const double b = h * bq[c];
        const double rres = b - q;
        acc0 = fma(rres, rres, acc0);
        acc1 = fma(b, b, acc1);
      } else {
        y[((size_t)(s * K + c) * side + gy) * side + gx] = q;
      }
    }
  }
  if (RESID) {
    acc0 = warp_sum(acc0);
    acc1 = warp_sum(acc1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { red[0][warp] = acc0; red[1][warp] = acc1; }
    __syncthreads();
    if (warp == 0) {
      double v0 = lane < AP_NT / 32 ? red[0][lane] : 0.0;
      double v1 = lane < AP_NT / 32 ? red[1][lane] : 0.0;
      v0 = warp_sum(v0);
      v1 = warp_sum(v1);
      if (lane == 0) {
        partials[((size_t)s * gridDim.x + tile) * 2] = v0;
        partials[((size_t)s * gridDim.x + tile) * 2 + 1] = v1;
      }
    }
  }
}

// out[s] = fixed-order sums of partials[s][0..tps)
__global__ void __launch_bounds__(256) reduce_pairs_kernel(const double* __restrict__ partials,
                                                           double* __restrict__ out, int tps) {
  __shared__ double red[2][8];
  const int s = blockIdx.x;
  double a0 = 0.0, a1 = 0.0;
  for (int t = threadIdx.x; t < tps; t += 256) {
    a0 += partials[((size_t)s * tps + t) * 2];
    a1 += partials[((size_t)s * tps + t) * 2 + 1];
  }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[0][warp] = a0; red[1][warp] = a1; }
  __syncthreads();
  if (warp == 0) {
    double v0 = lane < 8 ? red[0][lane] : 0.0, v1 = lane < 8 ? red[1][lane] : 0.0;
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    if (lane == 0) { out[2 * s] = v0; out[2 * s + 1] = v1; }
  }
}

// --------------------------------------------------------------------------- back-transform
// x[p][c][j] = sum_i W[p][c][i] xt[p][i][j]   (X = Xt W^T), in place.
template <int K>
__global__ void __launch_bounds__(256) backtransform_kernel(const double* __restrict__ W, double* __restrict__ x,
                                                            int side) {
  __shared__ double Ws[K * K];
  const int p = blockIdx.y;
  if (threadIdx.x < K * K) Ws[threadIdx.x] = W[(size_t)p * K * K + threadIdx.x];
  __syncthreads();
  const size_t N = (size_t)side * side;
  double* xp = x + (size_t)p * K * N;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x) {
    double t[K];
#pragma unroll
    for (int i = 0; i < K; ++i) t[i] = xp[(size_t)i * N + j];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) v = fma(Ws[c * K + i], t[i], v);
      xp[(size_t)c * N + j] = v;
    }
  }
}

// --------------------------------------------------------------------------- launchers
#define KCG_DISPATCH(K, CALL)                 \
  switch (K) {                                \
    case 1: { constexpr int KK = 1; CALL; } break; \
    case 2: { constexpr int KK = 2; CALL; } break; \
    case 3: { constexpr int KK = 3; CALL; } break; \
    case 4: { constexpr int KK = 4; CALL; } break; \
    case 5: { constexpr int KK = 5; CALL; } break; \
    case 6: { constexpr int KK = 6; CALL; } break; \
    case 7: { constexpr int KK = 7; CALL; } break; \
    case 8: { constexpr int KK = 8; CALL; } break; \
    default: return cudaErrorInvalidValue;    \
  }

static int grid_for(size_t N) {
  size_t b = (N + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return (int)(b ? b : 1);
}

cudaError_t launch_rhs(int K, cudaStream_t s, const double* Y, const double* E, const double* hits, double* r0,
                       double* p0, double* x, int P, int n, int side, int pitch) {
  const size_t N = (size_t)side * side;
  dim3 g(grid_for(N), P);
  const size_t sm = (size_t)n * K * sizeof(double);
  KCG_DISPATCH(K, (rhs_kernel<KK><<<g, 256, sm, s>>>(Y, E, hits, r0, p0, x, n, side, pitch)));
  return cudaGetLastError();
}

template <int K, bool HITS>
static cudaError_t cg_config_t(int n_sys, int* max_grid, size_t* smem) {
  const size_t sm = cg_stages(K) * (size_t)cg_stage_bytes(K) +
                    (size_t)n_sys * (sizeof(SysState) + sizeof(int));
  cudaError_t e = cudaFuncSetAttribute(cg_persistent_kernel<K, HITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int nb = 0, dev = 0, nsm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, cg_persistent_kernel<K, HITS>, cg_threads(K), sm);
  if (e != cudaSuccess) return e;
  e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  *max_grid = nb * nsm;
  *smem = sm;
  return nb > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t cg_kernel_config(int K, bool hits, int n_sys, int* max_grid, size_t* smem) {
  if (hits) { KCG_DISPATCH(K, return (cg_config_t<KK, true>(n_sys, max_grid, smem))); }
  else { KCG_DISPATCH(K, return (cg_config_t<KK, false>(n_sys, max_grid, smem))); }
  return cudaErrorInvalidValue;
}

cudaError_t launch_cg(int K, cudaStream_t s, const CgArgs& a, const CgMaps& m, int grid, size_t smem) {
  void* args[2] = {(void*)&a, (void*)&m};
  if (a.hits) {
    KCG_DISPATCH(K, return cudaLaunchCooperativeKernel((const void*)cg_persistent_kernel<KK, true>, dim3(grid),
                                                        dim3(cg_threads(KK)), args, smem, s));
  } else {
    KCG_DISPATCH(K, return cudaLaunchCooperativeKernel((const void*)cg_persistent_kernel<KK, false>, dim3(grid),
                                                        dim3(cg_threads(KK)), args, smem, s));
  }
  return cudaErrorInvalidValue;
}

template <int K, bool HITS>
static cudaError_t march_config_t(int n_sys, int* max_grid, size_t* smem) {
  const size_t sm = (size_t)march_warps(K) * march_nb(K) * march_chunk_bytes(K) +
                    (size_t)n_sys * (sizeof(SysState) + sizeof(int));
  cudaError_t e = cudaFuncSetAttribute(cg_march_kernel<K, HITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int nb = 0, dev = 0, nsm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, cg_march_kernel<K, HITS>, 32 * march_warps(K), sm);
  if (e != cudaSuccess) return e;
  e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  *max_grid = nb * nsm;
  *smem = sm;
  return nb > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t march_kernel_config(int K, bool hits, int n_sys, int* max_grid, size_t* smem) {
  if (hits) { KCG_DISPATCH(K, return (march_config_t<KK, true>(n_sys, max_grid, smem))); }
  else { KCG_DISPATCH(K, return (march_config_t<KK, false>(n_sys, max_grid, smem))); }
  return cudaErrorInvalidValue;
}

cudaError_t launch_march(int K, cudaStream_t s, const CgArgs& a, const CgMaps& m, int grid, size_t smem) {
  void* args[2] = {(void*)&a, (void*)&m};
  if (a.hits) {
    KCG_DISPATCH(K, return cudaLaunchCooperativeKernel((const void*)cg_march_kernel<KK, true>, dim3(grid),
                                                        dim3(32 * march_warps(KK)), args, smem, s));
  } else {
    KCG_DISPATCH(K, return cudaLaunchCooperativeKernel((const void*)cg_march_kernel<KK, false>, dim3(grid),
                                                        dim3(32 * march_warps(KK)), args, smem, s));
  }
  return cudaErrorInvalidValue;
}

template <int K, bool R>
static cudaError_t apply_t(cudaStream_t s, const SysParams* params, const double* x, double* y, const double* Y,
                           const double* E, const double* hits, double* partials, int n_sys, int n, int side) {
  const size_t sm = ((size_t)K * (AP_TX + 2) * (AP_TY + 2) + (R ? (size_t)n * K : 0)) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(apply_kernel<K, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  dim3 g(apply_tiles_per_sys(side), n_sys);
  apply_kernel<K, R><<<g, AP_NT, sm, s>>>(params, x, y, Y, E, hits, partials, n, side);
  return cudaGetLastError();
}

cudaError_t launch_apply(int K, cudaStream_t s, const SysParams* params, const double* x, double* y,
                         const double* hits, int n_sys, int side) {
  KCG_DISPATCH(K, return (apply_t<KK, false>(s, params, x, y, nullptr, nullptr, hits, nullptr, n_sys, 0, side)));
  return cudaErrorInvalidValue;
}

cudaError_t launch_resid(int K, cudaStream_t s, const SysParams* params, const double* x, const double* Y,
                         const double* E, const double* hits, double* partials, double* out, int n_sys, int n,
                         int side) {
  cudaError_t e = cudaSuccess;
  KCG_DISPATCH(K, e = (apply_t<KK, true>(s, params, x, nullptr, Y, E, hits, partials, n_sys, n, side)));
  if (e != cudaSuccess) return e;
  reduce_pairs_kernel<<<n_sys, 256, 0, s>>>(partials, out, apply_tiles_per_sys(side));
  return cudaGetLastError();
}

cudaError_t launch_backtransform(int K, cudaStream_t s, const double* W, double* x, int P, int side) {
  const size_t N = (size_t)side * side;
  dim3 g(grid_for(N), P);
  KCG_DISPATCH(K, (backtransform_kernel<KK><<<g, 256, 0, s>>>(W, x, side)));
  return cudaGetLastError();
}

}  // namespace kcg
