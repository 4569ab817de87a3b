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
__device__ __forceinline__ void tma_prefetch_l2_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
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
    z.alpha_last = z.alpha;  // the step this pass used
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

// ---------------------------------------------------------------------- per-iteration reduction
// Canonical order of a system's reduction, used by every mode below so that the scalars -- and
// hence the iterates -- are bitwise independent of the mode, the grid size and the batch
// composition: slot t in [0, NT) sums the tile partials t, t+NT, t+2NT, ... in order; the slots of a
// warp are combined by the xor-shuffle tree; the NW warp sums are added in warp order.
#define KCG_RB 8  // systems reduced per CTA pass (shared slots [KCG_RB][2][NW])

// The CTA reduces systems act[ii], ii = ii0, ii0 + step, ... and applies the CG scalar update.
// Results go to st_smem[s] (redundant mode: every CTA computes the same values) or a.state_out[s].
template <int NT>
__device__ __forceinline__ void reduce_systems_cta(const CgArgs& a, SysState* st, const int* act, int nact, int ii0,
                                                   int step, int par_out, int it, double (*rs)[2][NT / 32],
                                                   bool to_global) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tps = a.tiles_per_sys;
  for (int first = ii0; first < nact; first += KCG_RB * step) {
    int nb = 0;
#pragma unroll 2
    for (int b = 0; b < KCG_RB; ++b) {
      const int ii = first + b * step;
      if (ii >= nact) break;
      const int s = act[ii];
      const double2* base = reinterpret_cast<const double2*>(a.partials + ((size_t)par_out * a.n_sys + s) * tps * 2);
      double rr = 0.0, wr = 0.0;
      for (int t = tid; t < tps; t += NT) {
        const double2 v = __ldcg(base + t);
        rr += v.x;
        wr += v.y;
      }
      rr = warp_sum(rr);
      wr = warp_sum(wr);
      if (lane == 0) { rs[b][0][warp] = rr; rs[b][1][warp] = wr; }
      ++nb;
    }
    __syncthreads();
    if (tid < nb) {
      const int s = act[first + tid * step];
      double r2 = 0.0, w2 = 0.0;
      for (int w = 0; w < NW; ++w) { r2 += rs[tid][0][w]; w2 += rs[tid][1][w]; }
      const SysState z = cg_update(st[s], r2, w2, it, a);
      if (to_global) a.state_out[s] = z;
      else st[s] = z;
    }
    __syncthreads();
  }
}

// Every CTA pulls the states published in a.state_out by the reducing CTA(s).
template <int NT>
__device__ __forceinline__ void pull_states(const CgArgs& a, SysState* st, const int* act, int nact) {
  for (int ii = threadIdx.x; ii < nact; ii += NT) {
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
    z.alpha_last = __ldcg(&g->alpha_last);
    st[s] = z;
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until_geq(const unsigned* p, unsigned target) {
  if (ld_acquire_u32(p) >= target) return;
  const long long t0 = clock64();
  while (ld_acquire_u32(p) < target) {
    if (clock64() - t0 > (1LL << 34)) __trap();  // ~8 s: a lost arrival, never a legal wait
  }
}

// The iteration's barrier + reduction.  Modes (chosen per iteration, all in the canonical order):
//  REDUNDANT  (nact <= KCG_RB and nact*tps <= KCG_RED_MAX): one grid barrier, then every CTA reduces
//             every active system itself -- no second barrier, no state broadcast.
//  ONEBAR     (KCG_ONEBAR): CTAs arrive on a monotonic counter a.sync[0]; the LAST to arrive reduces
//             all systems, publishes the states and releases the generation flag a.sync[1].
//  otherwise  grid barrier; CTA b reduces systems b, b+grid, ...; second grid barrier; pull.
// a.sync is zeroed before each launch.  `after_count` runs on thread 0 once every CTA's stores of the pass are visible (the speculative
// TMA of the next pass).
template <int NT, typename F>
__device__ __forceinline__ void iteration_reduce(const CgArgs& a, SysState* st, const int* act, int nact,
                                                 int par_out, int it, double (*rs)[2][NT / 32], unsigned& epoch,
                                                 F after_count) {
  __shared__ int s_last;
  const int tid = threadIdx.x;
  const bool small = nact <= KCG_RB && nact * a.tiles_per_sys <= KCG_RED_MAX;
  if (small || !KCG_ONEBAR) {
    fence_proxy_async_global();
    cg::this_grid().sync();
    fence_proxy_async_global();
    if (tid == 0) after_count();
    if (small) {
      reduce_systems_cta<NT>(a, st, act, nact, 0, 1, par_out, it, rs, false);
    } else {
      reduce_systems_cta<NT>(a, st, act, nact, blockIdx.x, gridDim.x, par_out, it, rs, true);
      __threadfence();
      cg::this_grid().sync();
      pull_states<NT>(a, st, act, nact);
    }
    return;
  }
  ++epoch;  // ONEBAR iterations so far (uniform across CTAs: the mode choice is)
  const unsigned target = epoch * gridDim.x;
  __syncthreads();  // every partial / state store of this CTA is issued
  if (tid == 0) {
    fence_proxy_async_global();
    __threadfence();
    const unsigned prev = atomicAdd(a.sync, 1u);
    s_last = prev + 1 == target;
    if (!s_last) spin_until_geq(a.sync, target);
    __threadfence();
    fence_proxy_async_global();
    after_count();
  }
  __syncthreads();
  if (s_last) {
#if KCG_ONEBAR == 2
    {  // EXPERIMENT: warp per system, lanes in order (not the canonical order)
      constexpr int NW = NT / 32, U = 8;
      const int lane = tid & 31, warp = tid >> 5, tps = a.tiles_per_sys;
      for (int ii = warp; ii < nact; ii += NW) {
        const int s = act[ii];
        const double2* base = reinterpret_cast<const double2*>(a.partials + ((size_t)par_out * a.n_sys + s) * tps * 2);
        double rr = 0.0, wr = 0.0;
        for (int t0 = lane; t0 < tps; t0 += U * 32) {
          double2 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = t0 + u * 32 < tps ? __ldcg(base + t0 + u * 32) : make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < U; ++u) { rr += v[u].x; wr += v[u].y; }
        }
        rr = warp_sum(rr);
        wr = warp_sum(wr);
        if (lane == 0) a.state_out[s] = cg_update(st[s], rr, wr, it, a);
      }
      __syncthreads();
    }
#else
    reduce_systems_cta<NT>(a, st, act, nact, 0, 1, par_out, it, rs, true);
#endif
    if (tid == 0) {
      __threadfence();
      st_release_u32(a.sync + 1, epoch);
    }
  } else if (tid == 0) {
    spin_until_geq(a.sync + 1, epoch);
  }
  __syncthreads();
  pull_states<NT>(a, st, act, nact);
}

// --------------------------------------------------------------------------- persistent CG
// One tile of one system: box = tile + 2-pixel halo, K planes of r and p staged by TMA (zero fill
// outside the face).  Warp w owns T rows w, w+NW, ...; lane l owns the pixel PAIR at tile columns
// 2l, 2l+1 (double2 in shared and global memory); horizontal neighbours come from shuffles.
//   Phase A  p_new = r + beta p                    whole box (elementwise)
//   Phase B  q = G p_new, r_new = r - alpha q      T rows (pairs) + the 1-pixel ring (scalars)
//   Phase C  w = G r_new on T; (r,r), (w,r); x += alpha p_new (+ alpha_prev p_old, X2)
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
  bool xpass;         // this pass updates x (every pass without KCG_X2; even passes >= 2 with it)
  double alpha, beta, kappa2;
  double alpha_prev;  // X2: alpha of the previous pass (its p_new is this pass's p_old), else 0
  const double* hp;   // hits plane or nullptr
  uint64_t* bar;      // stage mbarrier
  uint32_t phase;
  double* part_out;
};

template <int K, bool EDGE, bool HITS, bool XTMA>
__device__ __forceinline__ void cg_tile(const CgArgs& a, const TileCtx& tc, double (*tred)[cg_threads(K) / 32]) {
  constexpr int TY = cg_tile_y(K), TX = KCG_TX, H = KCG_HALO;
  constexpr int BW = TX + 2 * H, BH = TY + 2 * H, PLANE = BW * BH;
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

  // Phase A: p_new = r + beta p over the whole box.  The tile interior is done in the pair
  // mapping of phases B/C, so on x passes the thread keeps its pairs' x increment
  //   xinc = alpha_prev p_old + alpha p_new   (X2: x is updated every other pass, see cg_update)
  // in registers; the 2-pixel frame of the box is a flat loop over double2 units.
  double2 xinc[RPW][K];
  {
    double2* P2 = reinterpret_cast<double2*>(Pp);
    const double2* R2 = reinterpret_cast<const double2*>(R);
    const double ap = tc.alpha_prev;
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int ly = warp + j * NW + H;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const int e = (c * PLANE + ly * BW + H) / 2 + lane;
        const double2 r = R2[e], po = P2[e];
        double2 pn;
        pn.x = fma(beta, po.x, r.x);
        pn.y = fma(beta, po.y, r.y);
        P2[e] = pn;
        xinc[j][c].x = fma(alpha, pn.x, ap * po.x);
        xinc[j][c].y = fma(alpha, pn.y, ap * po.y);
      }
    }
    constexpr int FR = 4 * (BW / 2) + 2 * TY;  // frame double2 units per plane
    for (int u = tid; u < K * FR; u += NT) {
      const int c = u / FR, v = u - c * FR;
      int e;
      if (v < 4 * (BW / 2)) {
        const int rr = v / (BW / 2);
        e = (rr < 2 ? rr : BH - 4 + rr) * (BW / 2) + (v - rr * (BW / 2));
      } else {
        const int w = v - 4 * (BW / 2);
        e = (H + (w >> 1)) * (BW / 2) + ((w & 1) ? BW / 2 - 1 : 0);
      }
      e += c * (PLANE / 2);
      const double2 r = R2[e], po = P2[e];
      double2 pn;
      pn.x = fma(beta, po.x, r.x);
      pn.y = fma(beta, po.y, r.y);
      P2[e] = pn;
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
    if (tc.xpass) {
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
      xn.x = xj[c].x + xinc[j][c].x;
      xn.y = xj[c].y + xinc[j][c].y;
      if (!EDGE || (in0 && in1)) {
        rr = fma(rc[c].x, rc[c].x, rr);
        wr = fma(w0, rc[c].x, wr);
        rr = fma(rc[c].y, rc[c].y, rr);
        wr = fma(w1, rc[c].y, wr);
        if (tc.xpass) *reinterpret_cast<double2*>(xp + c * N) = xn;
        *reinterpret_cast<double2*>(rout + c * ps) = rc[c];
        *reinterpret_cast<double2*>(pout + c * ps) = pn;
      } else {
        if (in0) {
          rr = fma(rc[c].x, rc[c].x, rr);
          wr = fma(w0, rc[c].x, wr);
          if (tc.xpass) xp[c * N] = xn.x;
          rout[c * ps] = rc[c].x;
          pout[c * ps] = pn.x;
        }
        if (in1) {
          rr = fma(rc[c].y, rc[c].y, rr);
          wr = fma(w1, rc[c].y, wr);
          if (tc.xpass) xp[c * N + 1] = xn.y;
          rout[c * ps + 1] = rc[c].y;
          pout[c * ps + 1] = pn.y;
        }
      }
    }
  }
  rr = warp_sum(rr);
  wr = warp_sum(wr);
  // per-warp partials; warp 0 sums them (fixed order) after the next CTA barrier (flush_tile_partial)
  if (lane == 0) { tred[0][warp] = rr; tred[1][warp] = wr; }
  if (!KCG_DEFER) {
    __syncthreads();
    if (warp == 0) {
      double v0 = lane < NW ? tred[0][lane] : 0.0;
      double v1 = lane < NW ? tred[1][lane] : 0.0;
      v0 = warp_sum(v0);
      v1 = warp_sum(v1);
      if (lane == 0) { tc.part_out[0] = v0; tc.part_out[1] = v1; }
    }
  }
}

// Tile partial (r,r), (w,r) of a finished tile: the fixed-order sum of its per-warp values, written
// by warp 0 after a barrier that follows the tile (deferred, so a tile needs no barrier of its own).
template <int NW>
__device__ __forceinline__ void flush_tile_partial(const double (*tred)[NW], double* part_out, int warp, int lane) {
  if (warp == 0) {
    double v0 = lane < NW ? tred[0][lane] : 0.0;
    double v1 = lane < NW ? tred[1][lane] : 0.0;
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    if (lane == 0) { part_out[0] = v0; part_out[1] = v1; }
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
  __shared__ double tred[2][2][NW];  // per-warp tile partials, double-buffered by tile parity
  // per-warp system sums of the iteration reduction: aliased onto pipeline stage 1, which is idle
  // from the end of a pass's last tile until the first prefetch of the next pass
  double (*rs)[2][NW] = reinterpret_cast<double (*)[2][NW]>(smem_raw + STAGE_BYTES);
  static_assert(NS == 2 && (size_t)KCG_RB * 2 * NW * 8 <= (size_t)STAGE_BYTES, "rs alias");  // per-warp tile partials, double-buffered by tile parity
  __shared__ double Ms[KCG_KMAX * KCG_KMAX + KCG_KMAX];
  __shared__ int s_nact;
  __shared__ int s_sched[2][2];  // [buffer][current tile, next tile]
  __shared__ int s_info[2][4];   // [stage][system, tile, tile row, tile col] of the tile in that stage

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tps = a.tiles_per_sys;
  const bool xtma = cg_xtma(K) && a.x_tma != 0;
  unsigned epoch = 0;  // ONEBAR barrier generations

  for (int s = tid; s < a.n_sys; s += NT) {
    SysState z;
    z.bnorm2 = 0.0; z.gamma = 0.0; z.alpha = 0.0; z.beta = 0.0; z.rel = 1.0;
    z.iters = 0; z.status = ST_RUNNING; z.parity = 0; z.pad = 0; z.alpha_last = 0.0;
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
  // pass q = it + 1 updates x iff xpass_of(q) (KCG_X2: even passes >= 2; else every pass >= 1)
  auto xpass_of = [](int q) { return KCG_X2 ? (q >= 2 && (q & 1) == 0) : (q >= 1); };
  // Thread 0: TMA of (physical) tile t into stage sidx (parity flipped for the speculative load of
  // the next pass) and its coordinates into s_info[sidx] for all threads.  On x passes the x block
  // comes with the boxes (XTMA) or is prefetched into L2 (read by phase C).
  auto issue = [&](int t, int sidx, int flip) {
    const int s = act[t / tps];
    const int tile = t - (t / tps) * tps;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    s_info[sidx][0] = s; s_info[sidx][1] = tile; s_info[sidx][2] = ty; s_info[sidx][3] = tx;
    const int par = st[s].parity ^ flip;
    double* dst = reinterpret_cast<double*>(smem_raw + sidx * STAGE_BYTES);
    const bool xp = xpass_of(it + 1 + flip);
    const bool xl = xtma && xp;
    mbar_arrive_expect_tx(&mbar[sidx], xl ? STAGE_BYTES : 2 * FIELD * 8);
    if (xl) tma_load_3d(dst + 2 * FIELD, &maps.x, &mbar[sidx], tx * TX, ty * TY, s * K);
    else if (xp && a.x_tma && KCG_XPF) tma_prefetch_l2_3d(&maps.x, tx * TX, ty * TY, s * K);
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

    // serpentine order: odd passes walk the active-tile list backwards, so the first tiles of a
    // pass are the ones the previous pass wrote last (still L2-resident when the state fits)
    const bool rev = KCG_SERP && (par_out != 0);
    if (!spec && (int)blockIdx.x < ntiles && tid == 0) issue(rev ? ntiles - 1 - (int)blockIdx.x : (int)blockIdx.x, 0, 0);
    spec = false;
    // Tile schedule (logical indices into the active-tile list): CTA b starts with tiles b and
    // b + grid; with KCG_DYN the rest are claimed from the pass's counter a.sync[2 + par_out]
    // (starting at 2 grid), one claim ahead so the atomic's latency hides behind a whole tile;
    // without it, b + 2 grid, b + 3 grid, ...  Both buffers of s_sched are written by thread 0 one
    // tile ahead of their readers (separated by the top-of-tile barrier).
    unsigned* ctr = a.sync + 2 + par_out;
    const int G = gridDim.x;
    if (tid == 0) { s_sched[0][0] = blockIdx.x; s_sched[0][1] = blockIdx.x + G; }
    int i = 0;
    double* prev_part = nullptr;  // partial slot of the previous tile, flushed after the next barrier
    for (;; ++i) {
      const int sidx = i & 1;
      __syncthreads();
      const int t = s_sched[i & 1][0], tn = s_sched[i & 1][1];
      if (prev_part) flush_tile_partial<NW>(tred[(i - 1) & 1], prev_part, warp, lane);
      if (t >= ntiles) break;
      unsigned claim = 0;
      if (tid == 0) {
        if (tn < ntiles) {
          fence_proxy_async_smem();
          issue(rev ? ntiles - 1 - tn : tn, sidx ^ 1, 0);
        }
        if (KCG_DYN && tn < ntiles) claim = atomicAdd(ctr, 1u);
      }
      const int s = s_info[sidx][0], tile = s_info[sidx][1], ty = s_info[sidx][2], tx = s_info[sidx][3];
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
      tc.xpass = xpass_of(it + 1);
      tc.alpha_prev = KCG_X2 ? st[s].alpha_last : 0.0;
      tc.kappa2 = __ldg(&sp->kappa2);
      tc.hp = HITS ? a.hits + (size_t)__ldg(&sp->hits_plane) * ((size_t)a.side * a.side) : nullptr;
      tc.bar = &mbar[sidx];
      tc.phase = sidx ? phase1 : phase0;
      tc.part_out = a.partials + (((size_t)par_out * a.n_sys + s) * tps + tile) * 2;
      const bool interior = tc.x0 >= H && tc.x0 + TX + H <= a.side && tc.y0 >= H && tc.y0 + TY + H <= a.side;
      if (cg_xtma(K) && xtma) {
        if (interior) cg_tile<K, false, HITS, cg_xtma(K)>(a, tc, tred[i & 1]);
        else cg_tile<K, true, HITS, cg_xtma(K)>(a, tc, tred[i & 1]);
      } else {
        if (interior) cg_tile<K, false, HITS, false>(a, tc, tred[i & 1]);
        else cg_tile<K, true, HITS, false>(a, tc, tred[i & 1]);
      }
      if (sidx) phase1 ^= 1u; else phase0 ^= 1u;
      if (KCG_DEFER) prev_part = tc.part_out;
      if (tid == 0) {  // the tile after tn (the claim's value is consumed only now)
        s_sched[(i + 1) & 1][0] = tn;
        s_sched[(i + 1) & 1][1] = tn >= ntiles ? ntiles : (KCG_DYN ? 2 * G + (int)claim : tn + G);
      }
    }  // (the loop exits at a top-of-tile barrier, after flushing the last tile's partial)

    if (tr && tid == 0 && blockIdx.x < KCG_TRACE_COLS - 3)
      a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 3 + blockIdx.x] = globaltimer();
    // speculative first load of the next iteration (same active set, flipped parity and order)
    // overlaps the reduction; verified against the new active count at the top of the loop
    const int spec_t = (KCG_SERP && !rev) ? ntiles - 1 - (int)blockIdx.x : (int)blockIdx.x;
    const bool do_spec = it >= 0 && (int)blockIdx.x < ntiles;
    iteration_reduce<NT>(a, st, act, nact, par_out, it, rs, epoch, [&]() {
      if (tr && blockIdx.x == 0) a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 1] = globaltimer();
      if (KCG_DYN && blockIdx.x == 0) *ctr = 0u;  // quiescent now; next used two passes later
      if (do_spec) issue(spec_t, 0, 1);
    });
    spec = do_spec;
    nact_prev = nact;

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

// --------------------------------------------------------------------------- X2 fix-up
// x += alpha_last p for every system whose last pass left its x increment pending (odd `iters`,
// KCG_X2); p = the system's current p planes (buffer `parity`, row pitch `pitch`).
template <int K>
__global__ void __launch_bounds__(256) xfix_kernel(const SysState* __restrict__ st, const double* __restrict__ p0,
                                                   const double* __restrict__ p1, double* __restrict__ x, int side,
                                                   int pitch) {
  const int s = blockIdx.y;
  const SysState z = st[s];
  if (!KCG_X2 || (z.iters & 1) == 0) return;
  const double al = z.alpha_last;
  const double* p = (z.parity ? p1 : p0) + (size_t)s * K * pitch * side;
  double* xs = x + (size_t)s * K * side * side;
  const size_t N = (size_t)side * side;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x) {
    const size_t gy = j / side, gx = j - gy * side;
#pragma unroll
    for (int c = 0; c < K; ++c) xs[c * N + j] = fma(al, p[(size_t)c * pitch * side + gy * pitch + gx], xs[c * N + j]);
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

cudaError_t launch_xfix(int K, cudaStream_t s, const SysState* st, const double* p0, const double* p1, double* x,
                        int n_sys, int side, int pitch) {
  const size_t N = (size_t)side * side;
  dim3 g(grid_for(N), n_sys);
  KCG_DISPATCH(K, (xfix_kernel<KK><<<g, 256, 0, s>>>(st, p0, p1, x, side, pitch)));
  return cudaGetLastError();
}

cudaError_t launch_backtransform(int K, cudaStream_t s, const double* W, double* x, int P, int side) {
  const size_t N = (size_t)side * side;
  dim3 g(grid_for(N), P);
  KCG_DISPATCH(K, (backtransform_kernel<KK><<<g, 256, 0, s>>>(W, x, side)));
  return cudaGetLastError();
}

}  // namespace kcg
