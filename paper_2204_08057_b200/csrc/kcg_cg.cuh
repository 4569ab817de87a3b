#pragma once
// sm_100a fp64 kernels of the Kronecker CG / Sylvester hot path (arxiv 2204.08057): the persistent
// CG kernel templates (instantiated per K in kcg_cg_k<K>.cu, so the build compiles them in parallel).
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

#include <algorithm>
#include <type_traits>

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

// --------------------------------------------------------------------------- NESTED order
// HEALPix NESTED pixel index inside a face (reading R1): bit b of x -> bit 2b, bit b of y -> 2b+1.
__device__ __forceinline__ uint32_t part1by1(uint32_t v) {
  v &= 0xffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__device__ __forceinline__ uint32_t nest_of(uint32_t x, uint32_t y) { return part1by1(x) | (part1by1(y) << 1); }

// --------------------------------------------------------------------------- rhs
// b[p][c][j] = h_j sum_f Y[p][f][j] E[p][f][c];  r0 = b (internal pitch), p0 = 0, x = 0.
// E == nullptr (b given, kron_cg_solve_b): Y holds b itself, [p][K][j] (n == K), copied as is.
template <int K>
__global__ void __launch_bounds__(256) rhs_kernel(const double* __restrict__ Y, const double* __restrict__ E,
                                                  const double* __restrict__ hits, double* __restrict__ r0,
                                                  double* __restrict__ p0, double* __restrict__ x, int n,
                                                  int side, int rows, int pitch, int ghost, int hghost,
                                                  int nested) {
  extern __shared__ double Es[];  // [n][K]
  const int p = blockIdx.y;
  if (E)
    for (int e = threadIdx.x; e < n * K; e += blockDim.x) Es[e] = E[(size_t)p * n * K + e];
  __syncthreads();
  const size_t N = (size_t)rows * side;                 // local pixels (a row slab in slab mode)
  const size_t ps = (size_t)pitch * (rows + 2 * ghost);  // r/p plane incl. ghost rows
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x) {
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    const size_t jy = nested ? nest_of((uint32_t)(j % side), (uint32_t)(j / side)) : j;  // Y's pixel index
    const double* yp = Y + (size_t)p * n * N + jy;
    if (E) {
      for (int f = 0; f < n; ++f) {
        const double y = __ldg(yp + (size_t)f * N);
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = fma(y, Es[f * K + c], acc[c]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < K; ++c) acc[c] = __ldg(yp + (size_t)c * N);
    }
    const size_t gy = j / side, gx = j - gy * side;
    const double h = (hits && E) ? __ldg(hits + (size_t)p * (rows + 2 * hghost) * side + (gy + hghost) * side + gx) : 1.0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const size_t plane = (size_t)p * K + c;
      r0[plane * ps + (gy + ghost) * pitch + gx] = h * acc[c];
      if (p0) p0[plane * ps + (gy + ghost) * pitch + gx] = 0.0;
      if (x) x[plane * N + j] = 0.0;
    }
  }
}

// --------------------------------------------------------------------------- CG scalar update
// One CG scalar step for a system from its reduced partials (Chronopoulos-Gear single-reduction
// CG, preconditioned form; reading R9/R10): rr = (r,r), ru = (r,u), wu = (w,u) with u = K^{-1} r,
// w = G u (u = r, ru = rr without a preconditioner).  The start pass (it < 0) gives ||b||^2,
// gamma_0 = (b,u_0) and alpha_0 = gamma_0/delta_0; afterwards beta = gamma'/gamma,
// alpha = gamma'/(delta - beta gamma'/alpha); stop on ||r|| <= tol ||b|| (reading R8).
// Warm start (a.bnorm2 != nullptr, reading R37): the start pass sees r_0 = b - G x_0, so ||b||^2 of
// system s comes from the host-launched residual kernel (a.bnorm2[2 s + 1]); the stopping rule
// stays ||r_j|| <= tol ||b|| (||r_0|| when b = 0), and x_0 may already satisfy it (0 iterations).
__device__ __forceinline__ SysState cg_update(SysState z, double rr, double ru, double wu, int it, const CgArgs& a,
                                              int s) {
  if (it < 0) {
    const double b2 = a.bnorm2 ? a.bnorm2[2 * s + 1] : rr;
    z.bnorm2 = b2 > 0.0 ? b2 : rr;
    z.gamma = ru;
    z.rel = z.bnorm2 > 0.0 ? sqrt(rr / z.bnorm2) : 0.0;
    if (!isfinite(rr) || !isfinite(ru) || !isfinite(wu)) z.status = ST_NONFINITE;
    else if (rr == 0.0 || (a.bnorm2 && rr <= a.tol2 * z.bnorm2)) z.status = ST_CONVERGED;
    else if (!(wu > 0.0) || !(ru > 0.0)) z.status = ST_BREAKDOWN;
    else if (a.max_iter <= 0) z.status = ST_MAXIT;
    else { z.alpha = ru / wu; z.beta = 0.0; }
  } else {
    z.alpha_last = z.alpha;  // the step this pass used
    z.iters = it + 1;
    z.rel = sqrt(rr / z.bnorm2);
    if (!isfinite(rr) || !isfinite(ru) || !isfinite(wu)) z.status = ST_NONFINITE;
    else if (rr <= a.tol2 * z.bnorm2) z.status = ST_CONVERGED;
    else if (z.iters >= a.max_iter) z.status = ST_MAXIT;
    else {
      const double beta = ru / z.gamma;
      const double den = wu - beta * ru / z.alpha;
      if (!(den > 0.0) || !(ru > 0.0)) z.status = ST_BREAKDOWN;
      else { z.beta = beta; z.alpha = ru / den; z.gamma = ru; }
    }
  }
  z.parity ^= 1;
  return z;
}

// ---------------------------------------------------------------------- per-iteration reduction
// Tile partials: NP doubles per tile, (rr, wr) without a preconditioner, (rr, ru, wu) with one.
// Canonical order of a system's reduction, used by every mode below so that the scalars -- and
// hence the iterates -- are bitwise independent of the mode, the grid size and the batch
// composition: slot t in [0, NT) sums the tile partials t, t+NT, t+2NT, ... in order; the slots of a
// warp are combined by the xor-shuffle tree; the NW warp sums are added in warp order.
#define KCG_RB 8  // systems reduced per CTA pass (shared slots [KCG_RB][3][NW])

template <int NP>
__device__ __forceinline__ void load_partial(const double* base, int t, double (&v)[3]) {
  if (NP == 2) {
    const double2 d = __ldcg(reinterpret_cast<const double2*>(base) + t);
    v[0] = d.x; v[1] = d.y; v[2] = 0.0;
  } else {
    v[0] = __ldcg(base + 3 * t); v[1] = __ldcg(base + 3 * t + 1); v[2] = __ldcg(base + 3 * t + 2);
  }
}

// Thread tid's canonical slot sum acc += partials t = tid, tid + NT, ... (in this order), the loads
// issued four at a time (one L2 round trip per four partials; the sum, and so the iterate, is the
// same as with one load at a time).
template <int NT, int NP>
__device__ __forceinline__ void sum_slot(const double* base, int tps, int tid, double (&acc)[3]) {
  int t = tid;
  for (; t + 3 * NT < tps; t += 4 * NT) {
    double v0[3], v1[3], v2[3], v3[3];
    load_partial<NP>(base, t, v0);
    load_partial<NP>(base, t + NT, v1);
    load_partial<NP>(base, t + 2 * NT, v2);
    load_partial<NP>(base, t + 3 * NT, v3);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      acc[q] += v0[q];
      acc[q] += v1[q];
      acc[q] += v2[q];
      acc[q] += v3[q];
    }
  }
  for (; t < tps; t += NT) {
    double v[3];
    load_partial<NP>(base, t, v);
#pragma unroll
    for (int q = 0; q < NP; ++q) acc[q] += v[q];
  }
}

// Scalar update from the NP reduced sums (without a preconditioner ru = rr, wu = wr).
template <int NP>
__device__ __forceinline__ SysState update_from(SysState z, const double (&v)[3], int it, const CgArgs& a, int s) {
  return NP == 2 ? cg_update(z, v[0], v[0], v[1], it, a, s) : cg_update(z, v[0], v[1], v[2], it, a, s);
}

// The CTA reduces systems act[ii], ii = ii0, ii0 + step, ... and applies the CG scalar update.
// Results go to st[s] (redundant mode: every CTA computes the same values) or a.state_out[s].
template <int NT, int NP>
__device__ __forceinline__ void reduce_systems_cta(const CgArgs& a, SysState* st, const int* act, int nact, int ii0,
                                                   int step, int par_out, int it, double (*rs)[3][NT / 32],
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
      const double* base = a.partials + ((size_t)par_out * a.n_sys + s) * tps * NP;
      double acc[3] = {0.0, 0.0, 0.0};
      sum_slot<NT, NP>(base, tps, tid, acc);
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        acc[q] = warp_sum(acc[q]);
        if (lane == 0) rs[b][q][warp] = acc[q];
      }
      ++nb;
    }
    __syncthreads();
    if (tid < nb) {
      const int s = act[first + tid * step];
      double v[3] = {0.0, 0.0, 0.0};
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int q = 0; q < NP; ++q) v[q] += rs[tid][q][w];
      const SysState z = update_from<NP>(st[s], v, it, a, s);
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

// ------------------------------------------------------------------ row-slab cross-rank protocol
// System-scope release/acquire on 64-bit flags in (peer) global memory, and a barrier over the CTAs
// of one rank's group (a monotonic counter zeroed before each launch).
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Bounded spins: a wait that is never satisfied (a lost peer) traps after ~8 s instead of hanging.
__device__ __forceinline__ void spin_geq_u32(const unsigned* p, unsigned target) {
  const long long t0 = clock64();
  while (ld_acquire_gpu_u32(p) < target)
    if (clock64() - t0 > (1LL << 34)) __trap();
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Cross-rank rendezvous on `tag` by one thread: ONE system-scope fence, then relaxed stores of the
// tag into every rank's flag array (release by fence + store); waiting polls the flags with relaxed
// system-scope loads and fences once after all of them (acquire).  A release / acquire per flag
// would serialise G fences.
__device__ __forceinline__ void xrank_signal(const CgArgs& a, unsigned long long tag) {
  __threadfence_system();
  for (int q = 0; q < a.nranks; ++q) st_relaxed_sys_u64(a.flags[q] + a.rank, tag);
}
// The G flags are loaded together each round (one memory round trip per poll, not G).
__device__ __forceinline__ void xrank_wait(const CgArgs& a, unsigned long long tag) {
  const long long t0 = clock64();
  while (true) {
    unsigned long long f[KCG_GMAX];
#pragma unroll
    for (int q = 0; q < KCG_GMAX; ++q) f[q] = q < a.nranks ? ld_relaxed_sys_u64(a.my_flags + q) : tag;
    bool ok = true;
#pragma unroll
    for (int q = 0; q < KCG_GMAX; ++q) ok &= f[q] >= tag;
    if (ok) break;
    if (clock64() - t0 > (1LL << 34)) __trap();
  }
  __threadfence_system();
}

// The iteration's barrier + reduction (all modes in the canonical order):
//  REDUNDANT  (nact <= KCG_RB and nact*tps <= KCG_RED_MAX): one grid barrier, then every CTA reduces
//             every active system itself -- no second barrier, no state broadcast.
//  DISTRIBUTED grid barrier; CTA b reduces systems b, b+grid, ...; second grid barrier; pull.
//  SLAB       (row-slab decomposition, the exchange step of SURVEY 8(e)): the rank's last-arriving
//             CTA reduces every active system over the rank's tiles (canonical order) and stores
//             the sums into slot [par][s][rank] of EVERY rank (peer stores), then releases its flag
//             on every rank; every CTA acquires all ranks' flags (one poll round trip for all G) and
//             adds the ranks' sums in rank order (the same on every rank) before the scalar update.
// `after_count` runs on thread 0 once every CTA's stores of the pass are visible (the speculative
// TMA of the next pass).
template <int NT, int NP, bool SLAB, typename F>
__device__ __forceinline__ void iteration_reduce(const CgArgs& a, SysState* st, const int* act, int nact,
                                                 int par_out, int it, double (*rs)[3][NT / 32], int cta, int ncta,
                                                 unsigned& gepoch, F after_count) {
  if constexpr (SLAB) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = a.nranks;
    const unsigned long long tag = a.tag0 + (unsigned long long)(it + 2);
    // The LAST CTA of the rank to arrive reduces (no group barrier: the others go straight to the
    // cross-rank flags).  Arrival = system fence (publishes the CTA's ghost-row peer stores and tile
    // partials) + one atomic on the rank's counter; the last arrival acquires every partial.
    __shared__ int s_last;
    __syncwarp();
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      const unsigned old = atomicAdd(a.group, 1u);
      ++gepoch;
      s_last = old == gepoch * (unsigned)ncta - 1u;
      if (s_last) __threadfence();
    }
    __syncthreads();
    if (s_last) {
      const int tps = a.tiles_per_sys;
      for (int first = 0; first < nact; first += KCG_RB) {
        const int nb = min(KCG_RB, nact - first);
        for (int b = 0; b < nb; ++b) {
          const double* base = a.partials + ((size_t)par_out * a.n_sys + act[first + b]) * tps * NP;
          double acc[3] = {0.0, 0.0, 0.0};
          sum_slot<NT, NP>(base, tps, tid, acc);
#pragma unroll
          for (int q = 0; q < NP; ++q) {
            acc[q] = warp_sum(acc[q]);
            if (lane == 0) rs[b][q][warp] = acc[q];
          }
        }
        __syncthreads();
        for (int e = tid; e < nb * G; e += NT) {  // (system, destination rank) pairs
          const int b = e / G, g = e - b * G;
          const int s = act[first + b];
          double v[3] = {0.0, 0.0, 0.0};
          for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int q = 0; q < NP; ++q) v[q] += rs[b][q][w];
          double* dst = a.slots[g] + (((size_t)par_out * a.n_sys + s) * G + a.rank) * NP;
#pragma unroll
          for (int q = 0; q < NP; ++q) dst[q] = v[q];
        }
        __syncthreads();
      }
      if (tid == 0) xrank_signal(a, tag);
    }
    if (tid == 0) {
      xrank_wait(a, tag);
      fence_proxy_async_global();
      after_count();
    }
    __syncthreads();
    for (int ii = tid; ii < nact; ii += NT) {
      const int s = act[ii];
      const double* src = a.my_slots + ((size_t)par_out * a.n_sys + s) * G * NP;
      double v[3] = {0.0, 0.0, 0.0};
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int q = 0; q < NP; ++q) v[q] += __ldcg(src + g * NP + q);
      st[s] = update_from<NP>(st[s], v, it, a, s);
    }
    __syncthreads();
    return;
  }
  const bool small = nact <= KCG_RB && nact * a.tiles_per_sys <= KCG_RED_MAX;
  fence_proxy_async_global();
  cg::this_grid().sync();
  fence_proxy_async_global();
  if (threadIdx.x == 0) after_count();
  if (small) {
    reduce_systems_cta<NT, NP>(a, st, act, nact, 0, 1, par_out, it, rs, false);
  } else {
    reduce_systems_cta<NT, NP>(a, st, act, nact, cta, ncta, par_out, it, rs, true);
    __threadfence();
    cg::this_grid().sync();
    pull_states<NT>(a, st, act, nact);
  }
}

// --------------------------------------------------------------------------- the operator
// Per pixel j and plane c (G = M (x) N_h + P (x) (kappa2 I + L), Alg.MatvecD/MatvecQ/MatvecBCBT):
//   (G v)_c(j) = h_j sum_d M[c][d] v_d(j) + tau_c ((kappa2 + deg_j) v_c(j) - sum_{nbr} v_c(nbr))
// `nb` = the neighbour sum, `kd` = kappa2 + deg_j, `mix` = sum_d M[c][d] v_d(j).
template <bool HITS>
__device__ __forceinline__ double op_point(double h, double mix, double tau, double kd, double v, double nb) {
  return HITS ? fma(h, mix, tau * fma(kd, v, -nb)) : fma(tau, fma(kd, v, -nb), mix);
}

// Pixel-block Jacobi (reading R10): u = K_j^{-1} r with K_j = h_j M + (kappa2 + deg_j) diag(tau),
// the k x k diagonal block of G at pixel j.  hits = 1: the three inverses (deg 2, 3, 4) are
// precomputed on the host (Kinv, shared); with hits K_j is factorised per pixel (Cholesky).
template <int K, bool HITS>
__device__ __forceinline__ void precond_pixel(const double* Kinv, const double* M,
                                              const double* tau, double kappa2, double h, int deg,
                                              const double (&r)[K], double (&u)[K], bool d2 = false) {
  if (!HITS) {
    const double* Ki = Kinv + kinv_slot(deg) * K * K;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double v = 0.0;
#pragma unroll
      for (int d = 0; d < K; ++d) v = fma(Ki[c * K + d], r[d], v);
      u[c] = v;
    }
  } else {
    double L[K][K];
    const double kd = kappa2 + (d2 ? (double)(deg * deg + deg) : (double)deg);  // diag(Q0)_jj
#pragma unroll
    for (int c = 0; c < K; ++c)
#pragma unroll
      for (int d = 0; d <= c; ++d) L[c][d] = fma(h, M[c * K + d], c == d ? kd * tau[c] : 0.0);
#pragma unroll
    for (int j = 0; j < K; ++j) {  // in-register Cholesky, K = L L^T
      double dsum = L[j][j];
#pragma unroll
      for (int m = 0; m < j; ++m) dsum = fma(-L[j][m], L[j][m], dsum);
      const double ljj = sqrt(dsum), inv = 1.0 / ljj;
      L[j][j] = ljj;
#pragma unroll
      for (int i = j + 1; i < K; ++i) {
        double v = L[i][j];
#pragma unroll
        for (int m = 0; m < j; ++m) v = fma(-L[i][m], L[j][m], v);
        L[i][j] = v * inv;
      }
    }
    double y[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double v = r[i];
#pragma unroll
      for (int m = 0; m < i; ++m) v = fma(-L[i][m], y[m], v);
      y[i] = v / L[i][i];
    }
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      double v = y[i];
#pragma unroll
      for (int m = i + 1; m < K; ++m) v = fma(-L[m][i], u[m], v);
      u[i] = v / L[i][i];
    }
  }
}

// --------------------------------------------------------------------------- persistent CG
// One tile of one system: box = tile + 2-pixel halo, K planes of r and p staged by TMA (zero fill
// outside the face; in row-slab mode the rows beyond the slab are the ghost rows its neighbours
// wrote).  Warp w owns tile rows w, w+NW, ...; lane l owns the pixel PAIR at tile columns 2l, 2l+1
// (double2 in shared and global memory); horizontal neighbours come from shuffles.
//   Phase A  p_new = u + beta p, u = K^{-1} r        whole box; interior pairs keep the x increment
//   Phase B  q = G p_new, r_new = r - alpha q         tile rows (pairs) + the 1-pixel ring (scalars)
//   Phase B' u_new = K^{-1} r_new on tile + ring      (PREC only, into the U box)
//   Phase C  w = G u_new on the tile; (r,r), (r,u), (w,u); x += xinc on x passes; store r, p, x
// Geometry: the tile origin (y0 local row of the slab, x0 column); global face row = a.row0 + local
// row; the face is side x side; the slab holds a.rows local rows (= side without slabs).
// EDGE = the box touches the face border or the slab end (bounds checks, degree 2/3).
struct TileCtx {
  double* R;          // r box (stage)
  double* Pp;         // p box (stage)
  double* U;          // PREC: u box [K][TY+2][BW] (tile + ring; shared by both stages)
  double* xs;         // x block of the tile in the stage [K][TY][TX] (XTMA)
  const double* Ms;   // M (K*K), tau (K), Kinv (3 K*K) of this tile's system, shared (valid after
                      // the phase-A barrier: written at the top of the tile by other threads)
  const SysParams* sp;  // the same parameters in global memory (read before that barrier)
  int s, y0, x0, par;
  bool xpass;         // this pass updates x (every pass without KCG_X2; even passes >= 2 with it)
  double alpha, beta, kappa2;
  double alpha_prev;  // X2: alpha of the previous pass (its p_new is this pass's p_old), else 0
  const double* hp;   // hits plane (slab rows) or nullptr
  uint64_t* bar;      // stage mbarrier
  uint32_t phase;
  double* part_out;
  double* dump;       // KCG_TRACE == 2 diagnostic builds: smem snapshots of one tile (else nullptr)
};

// KCG_TRACE == 2: copy n doubles of shared memory to dst (all threads; barrier after)
__device__ __forceinline__ void dump_smem(double* dst, const double* src, int n) {
  if (dst)
    for (int e0 = 0; e0 < n; e0 += blockDim.x)
      if (e0 + (int)threadIdx.x < n) dst[e0 + threadIdx.x] = src[e0 + threadIdx.x];
  __syncwarp();
  __syncthreads();
}

template <int K, bool EDGE, bool HITS, bool XTMA, bool PREC, bool SLAB>
__device__ __forceinline__ void cg_tile(const CgArgs& a, const TileCtx& tc, double (*tred)[cg_threads(K) / 32]) {
  constexpr int TY = cg_tile_y(K), TX = KCG_TX, H = KCG_HALO;
  constexpr int BW = TX + 2 * H, BH = TY + 2 * H, PLANE = BW * BH;
  constexpr int UPLANE = BW * (TY + 2);
  constexpr int NT = cg_threads(K), NW = NT / 32, RPW = TY / NW;
  constexpr int RP = 2 * (TX + 2) + 2 * TY;  // ring points
  static_assert(TX == 64 && RPW * NW == TY, "pair mapping needs TX = 64 and NW | TY");
  constexpr bool FUSE = cg_fuse(K, PREC);  // phases A and B fused, r_new into the U box (KCG_FUSEAB)
  static_assert(!FUSE || KCG_ROWMAP, "the fused phases need consecutive rows per warp");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int side = a.side, rows = SLAB ? a.rows : side, row0 = SLAB ? a.row0 : 0, ghost = SLAB ? a.ghost : 0;
  const size_t N = (size_t)rows * side;                   // pixels of one local plane
  const size_t ps = (size_t)a.pitch * (rows + 2 * ghost);  // one r/p buffer plane
  double* __restrict__ R = tc.R;
  double* __restrict__ Pp = tc.Pp;
  const int s = tc.s, y0 = tc.y0, x0 = tc.x0;
  const double alpha = tc.alpha, beta = tc.beta, kappa2 = tc.kappa2;
  const int gx = x0 + 2 * lane;
  const double* __restrict__ M = tc.Ms;
#if KCG_PREC_SMEM_A
  const double* Mg = tc.Ms;              // phase A: the shared copy (a barrier follows its writes)
  const double* Kinvg = tc.Ms + K * K + K;
#else
  const double* Mg = tc.sp->M;           // phase A (before the barrier): global copies
  const double* Kinvg = &tc.sp->Kinv[0][0];
#endif
  // degree of a pixel from its global face coordinates (free boundary, reading R2)
  auto degree = [&](int gyg, int gxx) { return 4 - (gyg == 0) - (gyg == side - 1) - (gxx == 0) - (gxx == side - 1); };
  auto in_face = [&](int gyg, int gxx) { return gyg >= 0 && gyg < side && gxx >= 0 && gxx < side; };
  // hits planes carry the ghost rows too in slab mode ([rows + 2 ghost][side], local row 0 at +ghost)
  auto hit = [&](int ly, int gxx) { return HITS ? __ldg(tc.hp + (size_t)(ly + ghost) * side + gxx) : 1.0; };

  mbar_wait(tc.bar, tc.phase);
  if (KCG_TRACE == 2) dump_smem(tc.dump, R, K * PLANE);

  double tau[K];  // PREC: needed in phase A (global copy); else read from shared after the barrier
  if (PREC)
#pragma unroll
    for (int c = 0; c < K; ++c) tau[c] = KCG_PREC_SMEM_A ? tc.Ms[K * K + c] : __ldg(&tc.sp->tau[c]);

  // x of tile row j (x passes; phase C): TMA-staged (XTMA), else from L2 (prefetched there by the issue)
  auto load_x = [&](int j, double2 (&xj)[K]) {
    const int ly = KCG_ROWMAP ? warp * RPW + j : warp + j * NW;
    bool in0 = true, in1 = true;
    if (EDGE) {
      const bool rin = y0 + ly < rows;
      in0 = rin && gx < side;
      in1 = rin && gx + 1 < side;
    }
    const double* xp = a.x + ((size_t)s * K * rows + y0 + ly) * side + gx;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      if (XTMA) {
        xj[c] = reinterpret_cast<const double2*>(tc.xs + ((size_t)c * TY + ly) * TX)[lane];
      } else if (!EDGE || (in0 && in1)) {
        xj[c] = __ldcg(reinterpret_cast<const double2*>(xp + c * N));
      } else {
        xj[c].x = in0 ? __ldcg(xp + c * N) : 0.0;
        xj[c].y = in1 ? __ldcg(xp + c * N + 1) : 0.0;
      }
    }
  };
  // KCG_XEARLY (L2 x only): rows 0 .. XE-1 of x are requested before the phase-B barrier, so their L2
  // latency overlaps the ring phase and the barrier instead of stalling phase C
  constexpr int XE = XTMA ? 0 : (KCG_XEARLY >= 2 ? RPW : KCG_XEARLY);
  double2 xe[XE > 0 ? XE : 1][K];
  double2 xinc[RPW][K];
  if constexpr (FUSE) {
    // ---- Phase AB (KCG_FUSEAB, no preconditioner; no CTA barrier between A and B): warp w owns the
    // tile rows ly = w RPW + j.  p_new = r + beta p of its rows and of the rows just above / below (the
    // neighbour warps' rows, recomputed) sits in registers, the edge columns -1 / TX come from broadcast
    // loads; r_new of its rows goes to the U box (tile + 1 ring, row pitch BW, U row = tile row + 1)
    // -- the R and P boxes stay read-only, so the ring phase below can form p_new itself; p_new is
    // final here and is stored at once; the x increment waits in registers for phase C.
    const double* __restrict__ Mg = tc.sp->M;  // (the shared copy is written per tile without a barrier)
    double taug[K];
#pragma unroll
    for (int c = 0; c < K; ++c) taug[c] = __ldg(&tc.sp->tau[c]);
    const double ap = tc.alpha_prev;
    const double2* R2 = reinterpret_cast<const double2*>(R);
    const double2* P2 = reinterpret_cast<const double2*>(Pp);
    double2* U2 = reinterpret_cast<double2*>(tc.U);
    double2 pr[RPW + 2][K];  // p_new of box rows warp RPW + H - 1 + i
#pragma unroll
    for (int i = 0; i < RPW + 2; ++i) {
      const int by = warp * RPW + H - 1 + i;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const int e = by * (BW / 2) + 1 + lane + c * (PLANE / 2);
        const double2 r = R2[e], po = P2[e];
        pr[i][c] = make_double2(fma(beta, po.x, r.x), fma(beta, po.y, r.y));
        if (i >= 1 && i <= RPW) {
          xinc[i - 1 < RPW ? i - 1 : 0][c] = make_double2(fma(alpha, pr[i][c].x, ap * po.x), fma(alpha, pr[i][c].y, ap * po.y));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int ly = warp * RPW + j;  // local tile row
      const int by = ly + H;          // box row
      const int gyg = row0 + y0 + ly;
      bool in0 = true, in1 = true;
      double kd0 = kappa2 + 4.0, kd1 = kappa2 + 4.0;
      if (EDGE) {
        const bool rin = y0 + ly < rows;
        in0 = rin && gx < side;
        in1 = rin && gx + 1 < side;
        kd0 = kappa2 + degree(gyg, gx);
        kd1 = kappa2 + degree(gyg, gx + 1);
      }
      bool up0 = in0, up1 = in1;
      if (EDGE && SLAB) {
        const bool rin1 = y0 + ly <= rows;
        up0 = rin1 && in_face(gyg, gx);
        up1 = rin1 && in_face(gyg, gx + 1);
      }
      const double h0 = HITS && up0 ? hit(y0 + ly, gx) : 1.0, h1 = HITS && up1 ? hit(y0 + ly, gx + 1) : 1.0;
      const size_t ro = ((size_t)s * K) * ps + (size_t)(y0 + ly + ghost) * a.pitch + gx;
      double* pout = (tc.par ? a.pbuf[0] : a.pbuf[1]) + ro;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const double2 pc = pr[j + 1][c], up = pr[j][c], dn = pr[j + 2][c];
        const double* rowR = R + c * PLANE + by * BW;
        const double* rowP = Pp + c * PLANE + by * BW;
        const double el = fma(beta, rowP[H - 1], rowR[H - 1]), er = fma(beta, rowP[H + TX], rowR[H + TX]);
        double left = __shfl_up_sync(0xffffffffu, pc.y, 1);
        double right = __shfl_down_sync(0xffffffffu, pc.x, 1);
        left = lane == 0 ? el : left;
        right = lane == 31 ? er : right;
        const double nb0 = (up.x + dn.x) + (left + pc.y);
        const double nb1 = (up.y + dn.y) + (pc.x + right);
        double mix0 = 0.0, mix1 = 0.0;
#pragma unroll
        for (int d = 0; d < K; ++d) {
          const double m = __ldg(&Mg[c * K + d]);
          mix0 = fma(m, pr[j + 1][d].x, mix0);
          mix1 = fma(m, pr[j + 1][d].y, mix1);
        }
        const double q0 = op_point<HITS>(h0, mix0, taug[c], kd0, pc.x, nb0);
        const double q1 = op_point<HITS>(h1, mix1, taug[c], kd1, pc.y, nb1);
        const double2 r = R2[by * (BW / 2) + 1 + lane + c * (PLANE / 2)];
        double2 rn = r;
        if (up0) rn.x = fma(-alpha, q0, r.x);
        if (up1) rn.y = fma(-alpha, q1, r.y);
        U2[(ly + 1) * (BW / 2) + 1 + lane + c * (UPLANE / 2)] = rn;
        if constexpr (SLAB) {  // boundary rows of p_new also land in the neighbour's ghost rows
          const int lyy = y0 + ly;
          const int bsel = tc.par ? 0 : 1;
          const size_t so = ((size_t)s * K + c) * ps + gx;
#pragma unroll
          for (int dir = 0; dir < 2; ++dir) {
            if (a.nb_p[dir][bsel] == nullptr) continue;
            const int nrow = dir == 0 ? rows + ghost + lyy : lyy - (rows - ghost);
            if (dir == 0 ? lyy >= ghost : lyy < rows - ghost) continue;
            double* npp = a.nb_p[dir][bsel] + so + (size_t)nrow * a.pitch;
            if (!EDGE || (in0 && in1)) {
              *reinterpret_cast<double2*>(npp) = pc;
            } else {
              if (in0) npp[0] = pc.x;
              if (in1) npp[1] = pc.y;
            }
          }
        }
        if (!EDGE || (in0 && in1)) {
          *reinterpret_cast<double2*>(pout + c * ps) = pc;
        } else {
          if (in0) pout[c * ps] = pc.x;
          if (in1) pout[c * ps + 1] = pc.y;
        }
      }
    }
    if (XE > 0 && tc.xpass)
#pragma unroll
      for (int j = 0; j < XE; ++j) load_x(j, xe[j]);
    // Phase B2 (fused form): r_new on the 1-pixel ring into the U box; p_new of a ring point and of
    // its four neighbours formed from the read-only R and P boxes.  Ring pixels outside the face get 0.
    for (int t0 = 0; t0 < RP; t0 += NT) {
      const int t = t0 + tid;
      if (t >= RP) continue;
      int by, bx;
      if (t < TX + 2) { by = H - 1; bx = H - 1 + t; }
      else if (t < 2 * (TX + 2)) { by = H + TY; bx = H - 1 + (t - (TX + 2)); }
      else { const int u = t - 2 * (TX + 2); by = H + (u >> 1); bx = (u & 1) ? H + TX : H - 1; }
      const int ly = y0 - H + by, gxr = x0 - H + bx, gyg = row0 + ly;
      double* uo = tc.U + (by - 1) * BW + bx;
      double kd = kappa2 + 4.0;
      if (EDGE) {
        if (!in_face(gyg, gxr)) {
#pragma unroll
          for (int c = 0; c < K; ++c) uo[c * UPLANE] = 0.0;
          continue;
        }
        kd = kappa2 + degree(gyg, gxr);
      }
      const double h = HITS ? hit(ly, gxr) : 1.0;
      const int o = by * BW + bx;
      auto pnew = [&](int c, int off) { return fma(beta, Pp[c * PLANE + o + off], R[c * PLANE + o + off]); };
      double pcs[K];
#pragma unroll
      for (int c = 0; c < K; ++c) pcs[c] = pnew(c, 0);
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const double nb = (pnew(c, -BW) + pnew(c, BW)) + (pnew(c, -1) + pnew(c, 1));
        double mix = 0.0;
#pragma unroll
        for (int d = 0; d < K; ++d) mix = fma(__ldg(&Mg[c * K + d]), pcs[d], mix);
        uo[c * UPLANE] = fma(-alpha, op_point<HITS>(h, mix, taug[c], kd, pcs[c], nb), R[c * PLANE + o]);
      }
    }
    __syncwarp();
    __syncthreads();
#pragma unroll
    for (int c = 0; c < K; ++c) tau[c] = M[K * K + c];
  } else {
  // Phase A.  Interior pairs in the pair mapping (the thread keeps its pairs' x increment
  //   xinc = alpha_prev p_old + alpha p_new   (X2: x is updated every other pass)
  // in registers); the 2-pixel frame of the box as a flat loop over double2 units (pixel pairs).
  {
    double2* P2 = reinterpret_cast<double2*>(Pp);
    const double2* R2 = reinterpret_cast<const double2*>(R);
    const double ap = tc.alpha_prev;
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int ly = KCG_ROWMAP ? warp * RPW + j : warp + j * NW;
      const int e0 = ((ly + H) * BW + H) / 2 + lane;
      if constexpr (!PREC) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const int e = e0 + c * (PLANE / 2);
          const double2 r = R2[e], po = P2[e];
          double2 pn;
          pn.x = fma(beta, po.x, r.x);
          pn.y = fma(beta, po.y, r.y);
          P2[e] = pn;
          xinc[j][c].x = fma(alpha, pn.x, ap * po.x);
          xinc[j][c].y = fma(alpha, pn.y, ap * po.y);
        }
      } else {
      double2 uu[K];
#pragma unroll
      for (int c = 0; c < K; ++c) uu[c] = R2[e0 + c * (PLANE / 2)];
      if (PREC) {
        const int gyg = row0 + y0 + ly;
        const bool f0 = !EDGE || in_face(gyg, gx), f1 = !EDGE || in_face(gyg, gx + 1);
        const int d0 = EDGE ? (f0 ? degree(gyg, gx) : 4) : 4, d1 = EDGE ? (f1 ? degree(gyg, gx + 1) : 4) : 4;
        const double h0 = HITS && f0 ? hit(y0 + ly, gx) : 1.0, h1 = HITS && f1 ? hit(y0 + ly, gx + 1) : 1.0;
        double r0[K], r1[K], u0[K], u1[K];
#pragma unroll
        for (int c = 0; c < K; ++c) { r0[c] = uu[c].x; r1[c] = uu[c].y; }
        precond_pixel<K, HITS>(Kinvg, Mg, tau, kappa2, h0, d0, r0, u0);
        precond_pixel<K, HITS>(Kinvg, Mg, tau, kappa2, h1, d1, r1, u1);
#pragma unroll
        for (int c = 0; c < K; ++c) uu[c] = make_double2(u0[c], u1[c]);
      }
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const int e = e0 + c * (PLANE / 2);
        const double2 po = P2[e];
        double2 pn;
        pn.x = fma(beta, po.x, uu[c].x);
        pn.y = fma(beta, po.y, uu[c].y);
        P2[e] = pn;
        xinc[j][c].x = fma(alpha, pn.x, ap * po.x);
        xinc[j][c].y = fma(alpha, pn.y, ap * po.y);
      }
      }  // PREC
    }
    constexpr int FR = 4 * (BW / 2) + 2 * TY;  // frame double2 units per plane
    constexpr int NFR = PREC ? FR : K * FR;
    // uniform trip count (every warp arrives converged at the barrier below)
    for (int v0 = 0; v0 < NFR; v0 += NT) {
      const int v = v0 + tid;
      if (v >= NFR) continue;
      const int c0 = PREC ? 0 : v / FR, w0 = PREC ? v : v - c0 * FR;
      int by, bu;  // box row, double2 column unit
      if (w0 < 4 * (BW / 2)) {
        const int rr = w0 / (BW / 2);
        by = rr < 2 ? rr : BH - 4 + rr;
        bu = w0 - rr * (BW / 2);
      } else {
        const int w = w0 - 4 * (BW / 2);
        by = H + (w >> 1);
        bu = (w & 1) ? BW / 2 - 1 : 0;
      }
      const int e = by * (BW / 2) + bu;
      if (!PREC) {
        const double2 r = R2[e + c0 * (PLANE / 2)], po = P2[e + c0 * (PLANE / 2)];
        P2[e + c0 * (PLANE / 2)] = make_double2(fma(beta, po.x, r.x), fma(beta, po.y, r.y));
      } else {
        const int gyg = row0 + y0 - H + by, gxx = x0 - H + 2 * bu;
        const bool f0 = in_face(gyg, gxx), f1 = in_face(gyg, gxx + 1);
        const int d0 = f0 ? degree(gyg, gxx) : 4, d1 = f1 ? degree(gyg, gxx + 1) : 4;
        const double h0 = HITS && f0 ? hit(y0 - H + by, gxx) : 1.0, h1 = HITS && f1 ? hit(y0 - H + by, gxx + 1) : 1.0;
        double r0[K], r1[K], u0[K], u1[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double2 r = R2[e + c * (PLANE / 2)];
          r0[c] = r.x; r1[c] = r.y;
        }
        precond_pixel<K, HITS>(Kinvg, Mg, tau, kappa2, h0, d0, r0, u0);
        precond_pixel<K, HITS>(Kinvg, Mg, tau, kappa2, h1, d1, r1, u1);
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double2 po = P2[e + c * (PLANE / 2)];
          P2[e + c * (PLANE / 2)] = make_double2(fma(beta, po.x, u0[c]), fma(beta, po.y, u1[c]));
        }
      }
    }
  }
  __syncwarp();
  __syncthreads();

  if (!PREC)
#pragma unroll
    for (int c = 0; c < K; ++c) tau[c] = M[K * K + c];

  // Phase B1: tile rows, pairs.  With consecutive rows per warp (KCG_ROWMAP) the centre rows of all
  // RPW rows are loaded once and serve as the up / down neighbours of the adjacent rows.
  double2 pcs[KCG_ROWMAP ? RPW : 1][K];
  if (KCG_ROWMAP)
#pragma unroll
    for (int j = 0; j < RPW; ++j)
#pragma unroll
      for (int c = 0; c < K; ++c)
        pcs[KCG_ROWMAP ? j : 0][c] =
            reinterpret_cast<const double2*>(Pp + c * PLANE + (warp * RPW + j + H) * BW)[1 + lane];
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    const int ly = KCG_ROWMAP ? warp * RPW + j : warp + j * NW;  // local tile row
    const int by = ly + H;                   // box row
    const int gyg = row0 + y0 + ly;
    bool in0 = true, in1 = true;
    double kd0 = kappa2 + 4.0, kd1 = kappa2 + 4.0;
    if (EDGE) {
      const bool rin = y0 + ly < rows;
      in0 = rin && gx < side;
      in1 = rin && gx + 1 < side;
      kd0 = kappa2 + degree(gyg, gx);
      kd1 = kappa2 + degree(gyg, gx + 1);
    }
    // r_new is also needed on the row just below the slab (the 1-ring of the last output row): in
    // slab mode that row is a ghost row inside a partially filled tile, so it is updated here too
    bool up0 = in0, up1 = in1;
    if (EDGE && SLAB) {
      const bool rin1 = y0 + ly <= rows;
      up0 = rin1 && in_face(gyg, gx);
      up1 = rin1 && in_face(gyg, gx + 1);
    }
    const double h0 = HITS && up0 ? hit(y0 + ly, gx) : 1.0, h1 = HITS && up1 ? hit(y0 + ly, gx + 1) : 1.0;
    double2 pc[K];
#pragma unroll
    for (int c = 0; c < K; ++c)
      pc[c] = KCG_ROWMAP ? pcs[KCG_ROWMAP ? j : 0][c] : reinterpret_cast<const double2*>(Pp + c * PLANE + by * BW)[1 + lane];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double* row = Pp + c * PLANE + by * BW;
      const double2 up = (KCG_ROWMAP && j > 0) ? pcs[KCG_ROWMAP ? j - 1 : 0][c]
                                                : reinterpret_cast<const double2*>(row - BW)[1 + lane];
      const double2 dn = (KCG_ROWMAP && j + 1 < RPW) ? pcs[KCG_ROWMAP ? j + 1 : 0][c]
                                                      : reinterpret_cast<const double2*>(row + BW)[1 + lane];
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
      const double q0 = op_point<HITS>(h0, mix0, tau[c], kd0, pc[c].x, nb0);
      const double q1 = op_point<HITS>(h1, mix1, tau[c], kd1, pc[c].y, nb1);
      double2* rp = reinterpret_cast<double2*>(R + c * PLANE + by * BW) + 1 + lane;
      double2 rv = *rp;
      if (up0) rv.x = fma(-alpha, q0, rv.x);
      if (up1) rv.y = fma(-alpha, q1, rv.y);
      *rp = rv;
    }
  }
  if (XE > 0 && tc.xpass)
#pragma unroll
    for (int j = 0; j < XE; ++j) load_x(j, xe[j]);
  // Phase B2: the 1-pixel ring around the tile (scalars).  Ring pixels outside the face are
  // skipped (their r stays 0); in slab mode ring rows beyond the slab are real (ghost) pixels.
  for (int t0 = 0; t0 < RP; t0 += NT) {
    const int t = t0 + tid;
    if (t >= RP) continue;
    int by, bx;
    if (t < TX + 2) { by = H - 1; bx = H - 1 + t; }
    else if (t < 2 * (TX + 2)) { by = H + TY; bx = H - 1 + (t - (TX + 2)); }
    else { const int u = t - 2 * (TX + 2); by = H + (u >> 1); bx = (u & 1) ? H + TX : H - 1; }
    const int ly = y0 - H + by, gxr = x0 - H + bx, gyg = row0 + ly;
    double kd = kappa2 + 4.0;
    if (EDGE) {
      if (!in_face(gyg, gxr)) continue;
      kd = kappa2 + degree(gyg, gxr);
    }
    const double h = HITS ? hit(ly, gxr) : 1.0;
    const int o = by * BW + bx;
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
      R[c * PLANE + o] = fma(-alpha, op_point<HITS>(h, mix, tau[c], kd, pcs[c], nb), R[c * PLANE + o]);
    }
  }
  __syncwarp();
  __syncthreads();
  }  // FUSE

  if (KCG_TRACE == 2) dump_smem(tc.dump ? tc.dump + 8192 : nullptr, R, K * PLANE);
  // Phase B' (PREC): u_new = K^{-1} r_new on tile + ring into U (row by of the R box = U row by-1).
  if (PREC) {
    constexpr int UPTS = (TY + 2) * (TX + 2);
    for (int t0 = 0; t0 < UPTS; t0 += NT) {
      const int t = t0 + tid;
      if (t >= UPTS) continue;
      const int uy = t / (TX + 2), ux = t - uy * (TX + 2);  // U row (tile row uy-1), column ux-1
      const int ly = y0 - 1 + uy, gxr = x0 - 1 + ux, gyg = row0 + ly;
      const int o = (uy + 1) * BW + (ux + 1);
      const bool f = in_face(gyg, gxr) && ly <= rows;  // beyond: r = 0 and unused
      double r[K], u[K];
#pragma unroll
      for (int c = 0; c < K; ++c) r[c] = R[c * PLANE + o];
      if (f) {
        precond_pixel<K, HITS>(tc.Ms + K * K + K, M, tau, kappa2, HITS ? hit(ly, gxr) : 1.0, degree(gyg, gxr), r, u);
      } else {
#pragma unroll
        for (int c = 0; c < K; ++c) u[c] = 0.0;
      }
#pragma unroll
      for (int c = 0; c < K; ++c) tc.U[c * UPLANE + uy * BW + ux + 1] = u[c];
    }
    __syncwarp();
    __syncthreads();
  }

  if (KCG_TRACE == 2) {
    dump_smem(tc.dump ? tc.dump + 2 * 8192 : nullptr, R, K * PLANE);
    if (PREC) dump_smem(tc.dump ? tc.dump + 3 * 8192 : nullptr, tc.U, K * UPLANE);
  }
  // Phase C.  Stencil source S = r_new (R box) or u_new (U box, same indexing: U = S + BW).
  constexpr bool USEU = PREC || FUSE;  // (FUSE: the U box holds r_new itself)
  const double* __restrict__ S = USEU ? tc.U - BW : R;
  constexpr int SPLANE = USEU ? UPLANE : PLANE;
  double rr = 0.0, ru = 0.0, wu = 0.0;
  double2 scs[KCG_ROWMAP ? RPW : 1][K];  // (KCG_ROWMAP) the S centre rows of all RPW rows, loaded once
  if (KCG_ROWMAP)
#pragma unroll
    for (int j = 0; j < RPW; ++j)
#pragma unroll
      for (int c = 0; c < K; ++c)
        scs[KCG_ROWMAP ? j : 0][c] =
            reinterpret_cast<const double2*>(S + c * SPLANE + (warp * RPW + j + H) * BW)[1 + lane];
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    const int ly = KCG_ROWMAP ? warp * RPW + j : warp + j * NW;
    const int by = ly + H;
    const int gyg = row0 + y0 + ly;
    bool in0 = true, in1 = true;
    double kd0 = kappa2 + 4.0, kd1 = kappa2 + 4.0;
    if (EDGE) {
      const bool rin = y0 + ly < rows;
      in0 = rin && gx < side;
      in1 = rin && gx + 1 < side;
      kd0 = kappa2 + degree(gyg, gx);
      kd1 = kappa2 + degree(gyg, gx + 1);
    }
    const double h0 = HITS && in0 ? hit(y0 + ly, gx) : 1.0, h1 = HITS && in1 ? hit(y0 + ly, gx + 1) : 1.0;
    double* xp = a.x + ((size_t)s * K * rows + y0 + ly) * side + gx;
    double2 xj[K];
    if (tc.xpass) {
      if (j < XE) {
#pragma unroll
        for (int c = 0; c < K; ++c) xj[c] = xe[j < XE ? j : 0][c];
      } else {
        load_x(j, xj);
      }
    }
    double2 rc[K], sc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      if (KCG_ROWMAP && (!USEU || FUSE)) {
        rc[c] = scs[KCG_ROWMAP ? j : 0][c];
        sc[c] = rc[c];
      } else {
        rc[c] = reinterpret_cast<const double2*>(R + c * PLANE + by * BW)[1 + lane];
        sc[c] = USEU ? (KCG_ROWMAP ? scs[KCG_ROWMAP ? j : 0][c]
                                   : reinterpret_cast<const double2*>(S + c * SPLANE + by * BW)[1 + lane])
                     : rc[c];
      }
    }
    const size_t ro = ((size_t)s * K) * ps + (size_t)(y0 + ly + ghost) * a.pitch + gx;
    double* rout = (tc.par ? a.rbuf[0] : a.rbuf[1]) + ro;  // select, not a dynamic param index
    double* pout = (tc.par ? a.pbuf[0] : a.pbuf[1]) + ro;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double* row = S + c * SPLANE + by * BW;
      const double2 up = (KCG_ROWMAP && j > 0) ? scs[KCG_ROWMAP ? j - 1 : 0][c]
                                                : reinterpret_cast<const double2*>(row - BW)[1 + lane];
      const double2 dn = (KCG_ROWMAP && j + 1 < RPW) ? scs[KCG_ROWMAP ? j + 1 : 0][c]
                                                      : reinterpret_cast<const double2*>(row + BW)[1 + lane];
      const double el = row[H - 1], er = row[H + TX];
      double left = __shfl_up_sync(0xffffffffu, sc[c].y, 1);
      double right = __shfl_down_sync(0xffffffffu, sc[c].x, 1);
      left = lane == 0 ? el : left;
      right = lane == 31 ? er : right;
      const double nb0 = (up.x + dn.x) + (left + sc[c].y);
      const double nb1 = (up.y + dn.y) + (sc[c].x + right);
      double mix0 = 0.0, mix1 = 0.0;
#pragma unroll
      for (int d = 0; d < K; ++d) {
        mix0 = fma(M[c * K + d], sc[d].x, mix0);
        mix1 = fma(M[c * K + d], sc[d].y, mix1);
      }
      const double w0 = op_point<HITS>(h0, mix0, tau[c], kd0, sc[c].x, nb0);
      const double w1 = op_point<HITS>(h1, mix1, tau[c], kd1, sc[c].y, nb1);
      const double2 pn = FUSE ? make_double2(0.0, 0.0)  // (FUSE: p_new stored in phase AB)
                              : reinterpret_cast<const double2*>(Pp + c * PLANE + by * BW)[1 + lane];
      double2 xn;
      xn.x = xj[c].x + xinc[j][c].x;
      xn.y = xj[c].y + xinc[j][c].y;
      if (in0) {
        rr = fma(rc[c].x, rc[c].x, rr);
        if (PREC) ru = fma(rc[c].x, sc[c].x, ru);
        wu = fma(w0, sc[c].x, wu);
      }
      if (in1) {
        rr = fma(rc[c].y, rc[c].y, rr);
        if (PREC) ru = fma(rc[c].y, sc[c].y, ru);
        wu = fma(w1, sc[c].y, wu);
      }
      if constexpr (SLAB) {  // boundary rows also land in the neighbour's ghost rows (peer stores)
        const int lyy = y0 + ly;
        const int bsel = tc.par ? 0 : 1;
        const size_t so = ((size_t)s * K + c) * ps + gx;
#pragma unroll
        for (int dir = 0; dir < 2; ++dir) {
          double* nr = a.nb_r[dir][bsel];
          if (nr == nullptr) continue;
          const int nrow = dir == 0 ? rows + ghost + lyy : lyy - (rows - ghost);  // row in its buffer
          if (dir == 0 ? lyy >= ghost : lyy < rows - ghost) continue;
          double* nrp = nr + so + (size_t)nrow * a.pitch;
          double* npp = a.nb_p[dir][bsel] + so + (size_t)nrow * a.pitch;
          if (!EDGE || (in0 && in1)) {
            *reinterpret_cast<double2*>(nrp) = rc[c];
            if (!FUSE) *reinterpret_cast<double2*>(npp) = pn;
          } else {
            if (in0) { nrp[0] = rc[c].x; if (!FUSE) npp[0] = pn.x; }
            if (in1) { nrp[1] = rc[c].y; if (!FUSE) npp[1] = pn.y; }
          }
        }
      }
      if (!EDGE || (in0 && in1)) {
        if (tc.xpass) *reinterpret_cast<double2*>(xp + c * N) = xn;
        *reinterpret_cast<double2*>(rout + c * ps) = rc[c];
        if (!FUSE) *reinterpret_cast<double2*>(pout + c * ps) = pn;
      } else {
        if (in0) {
          if (tc.xpass) xp[c * N] = xn.x;
          rout[c * ps] = rc[c].x;
          if (!FUSE) pout[c * ps] = pn.x;
        }
        if (in1) {
          if (tc.xpass) xp[c * N + 1] = xn.y;
          rout[c * ps + 1] = rc[c].y;
          if (!FUSE) pout[c * ps + 1] = pn.y;
        }
      }
    }
  }
  rr = warp_sum(rr);
  wu = warp_sum(wu);
  if (PREC) ru = warp_sum(ru);
  // per-warp partials; warp 0 sums them (fixed order) after the next CTA barrier (flush_tile_partial)
  if (lane == 0) {
    tred[0][warp] = rr;
    if (PREC) { tred[1][warp] = ru; tred[2][warp] = wu; }
    else tred[1][warp] = wu;
  }
  if (KCG_TRACE == 2) {
    __syncthreads();
    dump_smem(tc.dump ? tc.dump + 4 * 8192 : nullptr, &tred[0][0], 3 * NW);
  }
}

// Tile partials of a finished tile: the fixed-order sums of its per-warp values, written by warp 0
// after a barrier that follows the tile (deferred, so a tile needs no barrier of its own).
template <int NW, int NP>
__device__ __forceinline__ void flush_tile_partial(const double (*tred)[NW], double* part_out, int warp, int lane) {
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      double v = lane < NW ? tred[q][lane] : 0.0;
      v = warp_sum(v);
      if (lane == 0) part_out[q] = v;
    }
  }
}

// The persistent CG iteration of one CTA group: `cta` of `ncta` CTAs working on the systems of
// `a` (the whole grid without slabs; one rank's group in row-slab mode, where the launch may carry
// several emulated ranks).
template <int K, bool HITS, bool PREC, bool SLAB>
__device__ __forceinline__ void cg_body(const CgArgs& a, const CgMaps& maps, const int cta, const int ncta) {
  constexpr int TY = cg_tile_y(K), TX = KCG_TX, H = KCG_HALO;
  constexpr int BW = TX + 2 * H, BH = TY + 2 * H;
  constexpr int FIELD = K * BW * BH;  // doubles of one field box
  constexpr int XBYTES = cg_xstage_bytes(K);  // x block, TMA-staged with the boxes (0 if disabled)
  constexpr int STAGE_BYTES = 2 * FIELD * 8 + XBYTES;
  constexpr int UBYTES = (PREC || cg_fuse(K, PREC)) ? cg_ubox_bytes(K) : 0;
  constexpr int NT = cg_threads(K), NW = NT / 32, NS = cg_stages(K);
  constexpr int NP = PREC ? 3 : 2;  // partials per tile
  constexpr int MSZ = K * K + K + (PREC ? 4 * K * K : 0);
  static_assert(STAGE_BYTES == cg_stage_bytes(K), "stage size");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ubox = reinterpret_cast<double*>(smem_raw + NS * STAGE_BYTES);
  SysState* st = reinterpret_cast<SysState*>(smem_raw + NS * STAGE_BYTES + UBYTES);
  int* act = reinterpret_cast<int*>(st + a.n_sys);
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double tred[2][3][NW];  // per-warp tile partials, double-buffered by tile parity
  // per-warp system sums of the iteration reduction: aliased onto pipeline stage 1, which is idle
  // from the end of a pass's last tile until the first prefetch of the next pass
  double (*rs)[3][NW] = reinterpret_cast<double (*)[3][NW]>(smem_raw + STAGE_BYTES);
  static_assert(NS == 2 && (size_t)KCG_RB * 3 * NW * 8 <= (size_t)STAGE_BYTES, "rs alias");
  __shared__ double Ms[MSZ];
  __shared__ int s_nact;
  __shared__ int s_sched[2][2];  // [buffer][current tile, next tile]
  __shared__ int s_info[2][4];   // [stage][system, tile, tile row, tile col] of the tile in that stage

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tps = a.tiles_per_sys;
  const bool xtma = cg_xtma(K) && a.x_tma != 0;

  if (tid == 0) {  // the launch must provide the dynamic shared memory this layout assumes
    unsigned dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if ((size_t)dyn < (size_t)NS * STAGE_BYTES + UBYTES + (size_t)a.n_sys * (sizeof(SysState) + sizeof(int)))
      __trap();
  }
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
  int it = -1;  // -1 = start pass (alpha = beta = 0): p <- u_0 = K^{-1} b, (b,b), (b,u_0), (G u_0, u_0)
  unsigned gepoch = 0;  // slab mode: generations of the rank's group barrier
  if constexpr (SLAB) {  // every rank's rhs and ghost fill are complete before the first box is read
    if (cta == 0 && tid == 0) xrank_signal(a, a.tag0);
    if (tid == 0) {
      xrank_wait(a, a.tag0);
      fence_proxy_async_global();
    }
    __syncthreads();
  }

  // pass q = it + 1 updates x on tile `tile` iff cg_xpass(q, tile) (KCG_X2 + KCG_XMIX: the tile class
  // tile & 1 picks the even or the odd passes; without KCG_X2 every pass >= 1)
  // Thread 0: TMA of (physical) tile t into stage sidx (parity flipped for the speculative load of
  // the next pass) and its coordinates into s_info[sidx] for all threads.  On x passes the x block
  // comes with the boxes (XTMA) or is prefetched into L2 (read by phase C).  r/p buffers carry
  // a.ghost ghost rows above and below the slab (row-slab mode), hence the + ghost.
  auto issue = [&](int t, int sidx, int flip) {
    const int s = act[t / tps];
    const int tile = t - (t / tps) * tps;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    s_info[sidx][0] = s; s_info[sidx][1] = tile; s_info[sidx][2] = ty; s_info[sidx][3] = tx;
    const int par = st[s].parity ^ flip;
    double* dst = reinterpret_cast<double*>(smem_raw + sidx * STAGE_BYTES);
    const bool xp = cg_xpass(it + 1 + flip, cg_xclass(ty, tx, a.tiles_x));
    const bool xl = xtma && xp;
    mbar_arrive_expect_tx(&mbar[sidx], xl ? STAGE_BYTES : 2 * FIELD * 8);
    if (xl) tma_load_3d(dst + 2 * FIELD, &maps.x, &mbar[sidx], tx * TX, ty * TY, s * K);
    else if (xp && a.x_tma && KCG_XPF) tma_prefetch_l2_3d(&maps.x, tx * TX, ty * TY, s * K);
    tma_load_3d(dst, &maps.r[par], &mbar[sidx], tx * TX - H, ty * TY - H + (SLAB ? a.ghost : 0), s * K);
    tma_load_3d(dst + FIELD, &maps.p[par], &mbar[sidx], tx * TX - H, ty * TY - H + (SLAB ? a.ghost : 0), s * K);
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
    const bool tr = KCG_TRACE == 1 && a.trace && it + 1 < KCG_TRACE_ITERS;
    if (tr && cta == 0 && tid == 0) a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 0] = globaltimer();

    // serpentine order: odd passes walk the active-tile list backwards, so the first tiles of a
    // pass are the ones the previous pass wrote last (still L2-resident when the state fits)
    const bool rev = KCG_SERP && (par_out != 0);
    if (!spec && cta < ntiles && tid == 0) issue(rev ? ntiles - 1 - cta : cta, 0, 0);
    spec = false;
    // Tile schedule (logical indices into the active-tile list): CTA b starts with tiles b and
    // b + grid; with KCG_DYN the rest are claimed from the pass's counter a.sync[2 + par_out]
    // (starting at 2 grid), one claim ahead so the atomic's latency hides behind a whole tile;
    // without it, b + 2 grid, b + 3 grid, ...  Both buffers of s_sched are written by thread 0 one
    // tile ahead of their readers (separated by the top-of-tile barrier).
    unsigned* ctr = a.sync + 2 + par_out;
    const int G = ncta;
    if (tid == 0) { s_sched[0][0] = cta; s_sched[0][1] = cta + G; }
    int i = 0;
    double* prev_part = nullptr;  // partial slot of the previous tile, flushed after the next barrier
    for (;; ++i) {
      const int sidx = i & 1;
      __syncthreads();
      const int t = s_sched[i & 1][0], tn = s_sched[i & 1][1];
      if (prev_part) flush_tile_partial<NW, NP>(tred[(i - 1) & 1], prev_part, warp, lane);
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
      else if (PREC && tid < MSZ) Ms[tid] = __ldg(&sp->Kinv[0][0] + (tid - K * K - K));
#if KCG_PREC_SMEM_A
      if constexpr (PREC) __syncthreads();  // phase A of the PCG tile reads the shared copy
#endif
      TileCtx tc;
      tc.R = reinterpret_cast<double*>(smem_raw + sidx * STAGE_BYTES);
      tc.Pp = tc.R + FIELD;
      tc.xs = tc.R + 2 * FIELD;
      tc.U = ubox;
      tc.Ms = Ms;
      tc.sp = sp;
      tc.s = s;
      tc.y0 = ty * TY;
      tc.x0 = tx * TX;
      tc.par = st[s].parity;
      tc.alpha = st[s].alpha;
      tc.beta = st[s].beta;
      tc.xpass = cg_xpass(it + 1, cg_xclass(ty, tx, a.tiles_x));
      tc.alpha_prev = KCG_X2 ? st[s].alpha_last : 0.0;
      tc.kappa2 = __ldg(&sp->kappa2);
      tc.hp = HITS ? a.hits + (size_t)__ldg(&sp->hits_plane) * ((size_t)(SLAB ? a.rows + 2 * a.ghost : a.side) * a.side)
                   : nullptr;
      tc.bar = &mbar[sidx];
      tc.phase = sidx ? phase1 : phase0;
      tc.part_out = a.partials + (((size_t)par_out * a.n_sys + s) * tps + tile) * NP;
      tc.dump = (KCG_TRACE == 2 && a.trace && it < 0 && cta == 0 && i == 0)
                    ? reinterpret_cast<double*>(a.trace) : nullptr;
      const int gy0 = (SLAB ? a.row0 : 0) + tc.y0;
      const bool interior = tc.x0 >= H && tc.x0 + TX + H <= a.side && gy0 >= H && gy0 + TY + H <= a.side &&
                            tc.y0 + TY <= (SLAB ? a.rows : a.side);
      if (cg_xtma(K) && xtma) {
        if (interior) cg_tile<K, false, HITS, cg_xtma(K), PREC, SLAB>(a, tc, tred[i & 1]);
        else cg_tile<K, true, HITS, cg_xtma(K), PREC, SLAB>(a, tc, tred[i & 1]);
      } else {
        if (interior) cg_tile<K, false, HITS, false, PREC, SLAB>(a, tc, tred[i & 1]);
        else cg_tile<K, true, HITS, false, PREC, SLAB>(a, tc, tred[i & 1]);
      }
      if (sidx) phase1 ^= 1u; else phase0 ^= 1u;
      prev_part = tc.part_out;
      if (tid == 0) {  // the tile after tn (the claim's value is consumed only now)
        s_sched[(i + 1) & 1][0] = tn;
        s_sched[(i + 1) & 1][1] = tn >= ntiles ? ntiles : (KCG_DYN ? 2 * G + (int)claim : tn + G);
      }
    }  // (the loop exits at a top-of-tile barrier, after flushing the last tile's partial)

    if (tr && tid == 0 && cta < KCG_TRACE_COLS - 3)
      a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 3 + cta] = globaltimer();
    // speculative first load of the next iteration (same active set, flipped parity and order)
    // overlaps the reduction; verified against the new active count at the top of the loop
    const int spec_t = (KCG_SERP && !rev) ? ntiles - 1 - cta : cta;
    const bool do_spec = it >= 0 && cta < ntiles;
    iteration_reduce<NT, NP, SLAB>(a, st, act, nact, par_out, it, rs, cta, ncta, gepoch, [&]() {
      if (tr && cta == 0) a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 1] = globaltimer();
      if (KCG_DYN && cta == 0) *ctr = 0u;  // quiescent now; next used two passes later
      if (do_spec) issue(spec_t, 0, 1);
    });
    spec = do_spec;
    nact_prev = nact;

    if (tr && cta == 0 && tid == 0) a.trace[(size_t)(it + 1) * KCG_TRACE_COLS + 2] = globaltimer();
    if (cta == 0 && tid == 0 && it >= 0 && it < a.history_cap) {
      double m = 0.0;
      for (int ii = 0; ii < nact; ++ii) m = fmax(m, st[act[ii]].rel);
      a.history[it] = m;
    }
    ++it;
  }
  if (cta == 0)
    for (int s = tid; s < a.n_sys; s += NT) a.state_out[s] = st[s];
}

template <int K, bool HITS, bool PREC>
__global__ void __launch_bounds__(cg_threads(K), cg_min_blocks(K))
    cg_persistent_kernel(const CgArgs a, const __grid_constant__ CgMaps maps) {
  cg_body<K, HITS, PREC, false>(a, maps, blockIdx.x, gridDim.x);
}

// Row-slab mode: CTA group r (blocks [r ctas, (r+1) ctas)) runs local rank r of the launch.
template <int K, bool HITS, bool PREC>
__global__ void __launch_bounds__(cg_threads(K), cg_min_blocks(K)) cg_slab_kernel(const __grid_constant__ CgSlabLaunch L) {
  const int rl = blockIdx.x / L.ctas;
  cg_body<K, HITS, PREC, true>(L.a[rl], L.m[rl], blockIdx.x - rl * L.ctas, L.ctas);
}


}  // namespace kcg
#include "kcg_march.cuh"
namespace kcg {

// --------------------------------------------------------------------------- per-K entry points
// Defined here, explicitly instantiated once per K in kcg_cg_k<K>.cu; the dispatchers in
// kcg_kernels.cu see them as extern templates.
template <int K>
struct CgEntry {
  static cudaError_t config(bool hits, bool prec, bool slab, bool d2, int n_sys, int* max_grid, size_t* smem);
  static cudaError_t launch(bool prec, bool d2, cudaStream_t s, const CgArgs& a, const CgMaps& m, int grid,
                            size_t smem);
  static cudaError_t launch_slab(bool prec, cudaStream_t s, const CgSlabLaunch& L, size_t smem);
};

// Dynamic shared memory of one CTA (Laplacian tile kernel): two stages, the PREC u box (+ the states).
template <int K, bool PREC>
constexpr size_t cg_dyn_smem_fixed() {
  return cg_stages(K) * (size_t)cg_stage_bytes(K) + ((PREC || cg_fuse(K, PREC)) ? (size_t)cg_ubox_bytes(K) : 0);
}

template <int K, bool HITS, bool PREC>
static cudaError_t cg_config_t(bool slab, bool d2, int n_sys, int* max_grid, size_t* smem) {
  const void* kern = nullptr;
  size_t sm = (size_t)n_sys * (sizeof(SysState) + sizeof(int));
  int nt = cg_threads(K);
  if (d2) {  // the row-march kernel (kcg_march.cuh)
    if constexpr (K <= 4) kern = (const void*)cg_march_kernel<K, HITS, PREC>;
    sm += (size_t)m_groups(K, HITS) * m_group_doubles(K, PREC, HITS) * 8;
    nt = m_threads(K, HITS);
  } else {
    kern = slab ? (const void*)cg_slab_kernel<K, HITS, PREC> : (const void*)cg_persistent_kernel<K, HITS, PREC>;
    sm += cg_dyn_smem_fixed<K, PREC>();
  }
  if (!kern) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int nb = 0, dev = 0, nsm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, nt, sm);
  if (e != cudaSuccess) return e;
  e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  *max_grid = nb * nsm;
  *smem = sm;
  return nb > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

// Built: PREC for K <= 7 (u box), the D2 prior (row-march kernel) for K <= 4 without slabs.
template <int K>
cudaError_t CgEntry<K>::config(bool hits, bool prec, bool slab, bool d2, int n_sys, int* max_grid, size_t* smem) {
  if (d2 && (K > 4 || slab)) return cudaErrorInvalidValue;
  if (prec) {
    if constexpr (K <= 7)
      return hits ? cg_config_t<K, true, true>(slab, d2, n_sys, max_grid, smem)
                  : cg_config_t<K, false, true>(slab, d2, n_sys, max_grid, smem);
    return cudaErrorInvalidValue;
  }
  return hits ? cg_config_t<K, true, false>(slab, d2, n_sys, max_grid, smem)
              : cg_config_t<K, false, false>(slab, d2, n_sys, max_grid, smem);
}

template <int K>
cudaError_t CgEntry<K>::launch(bool prec, bool d2, cudaStream_t s, const CgArgs& a, const CgMaps& m, int grid,
                               size_t smem) {
  void* args[2] = {(void*)&a, (void*)&m};
  const bool hits = a.hits != nullptr;
  const void* f = nullptr;
  if (d2) {
    if constexpr (K <= 4) {
      if (prec) f = hits ? (const void*)cg_march_kernel<K, true, true> : (const void*)cg_march_kernel<K, false, true>;
      else f = hits ? (const void*)cg_march_kernel<K, true, false> : (const void*)cg_march_kernel<K, false, false>;
    }
  } else if (prec) {
    if constexpr (K <= 7) f = hits ? (const void*)cg_persistent_kernel<K, true, true> : (const void*)cg_persistent_kernel<K, false, true>;
  } else {
    f = hits ? (const void*)cg_persistent_kernel<K, true, false> : (const void*)cg_persistent_kernel<K, false, false>;
  }
  if (!f) return cudaErrorInvalidValue;
  return cudaLaunchCooperativeKernel(f, dim3(grid), dim3(d2 ? m_threads(K, hits) : cg_threads(K)), args, smem, s);
}

template <int K>
cudaError_t CgEntry<K>::launch_slab(bool prec, cudaStream_t s, const CgSlabLaunch& L, size_t smem) {
  void* args[1] = {(void*)&L};
  const bool hits = L.a[0].hits != nullptr;
  const void* f = nullptr;
  if (prec) {
    if constexpr (K <= 7) f = hits ? (const void*)cg_slab_kernel<K, true, true> : (const void*)cg_slab_kernel<K, false, true>;
  } else {
    f = hits ? (const void*)cg_slab_kernel<K, true, false> : (const void*)cg_slab_kernel<K, false, false>;
  }
  if (!f) return cudaErrorInvalidValue;
  return cudaLaunchCooperativeKernel(f, dim3(L.nlocal * L.ctas), dim3(cg_threads(K)), args, smem, s);
}

}  // namespace kcg
