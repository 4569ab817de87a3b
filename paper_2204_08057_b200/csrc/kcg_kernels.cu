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

// --------------------------------------------------------------------------- persistent CG
template <int K>
__global__ void __launch_bounds__(KCG_NT, 1) cg_persistent_kernel(const CgArgs a, const __grid_constant__ CgMaps maps) {
  constexpr int TY = cg_tile_y(K), TX = KCG_TX, H = KCG_HALO;
  constexpr int BW = TX + 2 * H, BH = TY + 2 * H;
  constexpr int PLANE = BW * BH;
  constexpr int FIELD = K * PLANE;  // doubles of one field box
  constexpr int STAGE_BYTES = 2 * FIELD * 8;
  constexpr int NW = KCG_NT / 32;
  constexpr int PTS = TY * TX / KCG_NT;  // T-region points per thread
  static_assert(PTS >= 1 && TY * TX % KCG_NT == 0, "tile/threads mismatch");
  static_assert(STAGE_BYTES == cg_stage_bytes(K), "stage size");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  SysState* st = reinterpret_cast<SysState*>(smem_raw + 2 * STAGE_BYTES);
  int* act = reinterpret_cast<int*>(st + a.n_sys);
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double red[2][NW];
  __shared__ int s_nact;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int side = a.side, pitch = a.pitch;
  const size_t N = (size_t)side * side;
  const size_t ps = (size_t)pitch * side;
  const int tps = a.tiles_per_sys;
  cg::grid_group grid = cg::this_grid();

  for (int s = tid; s < a.n_sys; s += KCG_NT) {
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

  auto issue = [&](int t, int sidx) {
    const int s = act[t / tps];
    const int tile = t - (t / tps) * tps;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int par = st[s].parity;
    double* dst = reinterpret_cast<double*>(smem_raw + sidx * STAGE_BYTES);
    mbar_arrive_expect_tx(&mbar[sidx], STAGE_BYTES);
    tma_load_3d(dst, &maps.r[par], &mbar[sidx], tx * TX - H, ty * TY - H, s * K);
    tma_load_3d(dst + FIELD, &maps.p[par], &mbar[sidx], tx * TX - H, ty * TY - H, s * K);
  };

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

    int sidx = 0;
    if ((int)blockIdx.x < ntiles && tid == 0) issue(blockIdx.x, 0);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, sidx ^= 1) {
      const int tn = t + gridDim.x;
      if (tn < ntiles && tid == 0) {
        fence_proxy_async_smem();
        issue(tn, sidx ^ 1);
      }
      const int s = act[t / tps];
      const int tile = t - (t / tps) * tps;
      const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
      const int ty0 = ty * TY, tx0 = tx * TX;
      const SysParams* sp = a.params + s;
      double M[K * K], tau[K];
#pragma unroll
      for (int e = 0; e < K * K; ++e) M[e] = __ldg(&sp->M[e]);
#pragma unroll
      for (int c = 0; c < K; ++c) tau[c] = __ldg(&sp->tau[c]);
      const double kappa2 = __ldg(&sp->kappa2);
      const double* hp = a.hits ? a.hits + (size_t)__ldg(&sp->hits_plane) * N : nullptr;
      const double alpha = st[s].alpha, beta = st[s].beta;
      const int par = st[s].parity;

      // prefetch x of this thread's T-region points
      double xv[PTS][K];
#pragma unroll
      for (int j = 0; j < PTS; ++j) {
        const int pt = tid + j * KCG_NT;
        const int gy = ty0 + pt / TX, gx = tx0 + pt % TX;
        const bool in = gy < side && gx < side;
#pragma unroll
        for (int c = 0; c < K; ++c)
          xv[j][c] = in ? __ldcg(a.x + ((size_t)(s * K + c) * side + gy) * side + gx) : 0.0;
      }

      if (sidx == 0) { mbar_wait(&mbar[0], phase0); phase0 ^= 1u; }
      else           { mbar_wait(&mbar[1], phase1); phase1 ^= 1u; }
      double* R = reinterpret_cast<double*>(smem_raw + sidx * STAGE_BYTES);
      double* Pp = R + FIELD;

      // Phase A: p_new = r + beta p_old on the whole haloed box (zero outside the face).
      {
        double2* P2 = reinterpret_cast<double2*>(Pp);
        const double2* R2 = reinterpret_cast<const double2*>(R);
        if (beta == 0.0) {
          for (int e = tid; e < FIELD / 2; e += KCG_NT) P2[e] = R2[e];
        } else {
          for (int e = tid; e < FIELD / 2; e += KCG_NT) {
            const double2 r = R2[e];
            double2 p = P2[e];
            p.x = fma(beta, p.x, r.x);
            p.y = fma(beta, p.y, r.y);
            P2[e] = p;
          }
        }
      }
      __syncthreads();

      // Phase B: q = G p_new and r_new = r - alpha q on the tile + 1-pixel ring (in-face only).
      {
        constexpr int RW = BW - 2, RH = BH - 2;
        for (int pt = tid; pt < RW * RH; pt += KCG_NT) {
          const int ly = pt / RW + 1, lx = pt % RW + 1;
          const int gy = ty0 - H + ly, gx = tx0 - H + lx;
          if (gy < 0 || gy >= side || gx < 0 || gx >= side) continue;
          const double deg = 4.0 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1);
          const double h = hp ? __ldg(hp + (size_t)gy * side + gx) : 1.0;
          const int o = ly * BW + lx;
          double pc[K];
#pragma unroll
          for (int c = 0; c < K; ++c) pc[c] = Pp[c * PLANE + o];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            const double* pl = Pp + c * PLANE + o;
            const double nb = (pl[-BW] + pl[BW]) + (pl[-1] + pl[1]);
            double mix = 0.0;
#pragma unroll
            for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], pc[d], mix);
            const double q = fma(h, mix, tau[c] * (fma(kappa2 + deg, pc[c], -nb)));
            R[c * PLANE + o] = fma(-alpha, q, R[c * PLANE + o]);
          }
        }
      }
      __syncthreads();

      // Phase C: w = G r_new on the tile, partial (r,r), (w,r); x += alpha p; store x, r, p.
      double rr = 0.0, wr = 0.0;
#pragma unroll
      for (int j = 0; j < PTS; ++j) {
        const int pt = tid + j * KCG_NT;
        const int ly = pt / TX + H, lx = pt % TX + H;
        const int gy = ty0 + pt / TX, gx = tx0 + pt % TX;
        if (gy < side && gx < side) {
          const double deg = 4.0 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1);
          const double h = hp ? __ldg(hp + (size_t)gy * side + gx) : 1.0;
          const int o = ly * BW + lx;
          double rc[K];
#pragma unroll
          for (int c = 0; c < K; ++c) rc[c] = R[c * PLANE + o];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            const double* rl = R + c * PLANE + o;
            const double nb = (rl[-BW] + rl[BW]) + (rl[-1] + rl[1]);
            double mix = 0.0;
#pragma unroll
            for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], rc[d], mix);
            const double w = fma(h, mix, tau[c] * (fma(kappa2 + deg, rc[c], -nb)));
            rr = fma(rc[c], rc[c], rr);
            wr = fma(w, rc[c], wr);
            const double pn = Pp[c * PLANE + o];
            const size_t plane = (size_t)(s * K + c);
            a.x[(plane * side + gy) * side + gx] = fma(alpha, pn, xv[j][c]);
            a.rbuf[par ^ 1][plane * ps + (size_t)gy * pitch + gx] = rc[c];
            a.pbuf[par ^ 1][plane * ps + (size_t)gy * pitch + gx] = pn;
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
        if (lane == 0) {
          double* dst = a.partials + (((size_t)par_out * a.n_sys + s) * tps + tile) * 2;
          dst[0] = v0;
          dst[1] = v1;
        }
      }
      __syncthreads();
    }

    fence_proxy_async_global();
    grid.sync();
    fence_proxy_async_global();

    // Per-system reduction of the tile partials (fixed order -> deterministic, independent of the
    // grid size and of which other systems are in the batch), then the CG scalar recurrences.
    for (int i = warp; i < nact; i += NW) {
      const int s = act[i];
      const double* base = a.partials + ((size_t)par_out * a.n_sys + s) * tps * 2;
      double rr = 0.0, wr = 0.0;
      for (int tl = lane; tl < tps; tl += 32) {
        rr += __ldcg(base + 2 * tl);
        wr += __ldcg(base + 2 * tl + 1);
      }
      rr = warp_sum(rr);
      wr = warp_sum(wr);
      if (lane == 0) {
        SysState z = st[s];
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
        st[s] = z;
      }
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0 && it >= 0 && it < a.history_cap) {
      double m = 0.0;
      for (int i = 0; i < nact; ++i) m = fmax(m, st[act[i]].rel);
      a.history[it] = m;
    }
    ++it;
  }
  if (blockIdx.x == 0)
    for (int s = tid; s < a.n_sys; s += KCG_NT) a.state_out[s] = st[s];
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

template <int K>
static cudaError_t cg_config_t(int n_sys, int* max_grid, size_t* smem) {
  const size_t sm = 2 * (size_t)cg_stage_bytes(K) + (size_t)n_sys * (sizeof(SysState) + sizeof(int));
  cudaError_t e = cudaFuncSetAttribute(cg_persistent_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int nb = 0, dev = 0, nsm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, cg_persistent_kernel<K>, KCG_NT, sm);
  if (e != cudaSuccess) return e;
  e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  *max_grid = nb * nsm;
  *smem = sm;
  return nb > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

cudaError_t cg_kernel_config(int K, int n_sys, int* max_grid, size_t* smem) {
  KCG_DISPATCH(K, return cg_config_t<KK>(n_sys, max_grid, smem));
  return cudaErrorInvalidValue;
}

cudaError_t launch_cg(int K, cudaStream_t s, const CgArgs& a, const CgMaps& m, int grid, size_t smem) {
  void* args[2] = {(void*)&a, (void*)&m};
  KCG_DISPATCH(K, return cudaLaunchCooperativeKernel((const void*)cg_persistent_kernel<KK>, dim3(grid),
                                                      dim3(KCG_NT), args, smem, s));
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
