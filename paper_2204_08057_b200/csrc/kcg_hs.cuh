#pragma once
// sm_100a fp64: the textbook (Hestenes-Stiefel) CG variant, KCG_CG_HS -- the second of the paper's
// "two variants of the conjugate gradient approach" (reading R9), i.e. Alg. CG (P:L225-241,
// reading R7) with its two inner products per iteration kept as two grid-wide reductions:
//
//   pass A (stencil)   p_j = z_j + beta_{j-1} p_{j-1}  (z = K^{-1} r, on the tile + operator halo)
//                      q_j = G p_j  (tile);  x += alpha_{j-1} p_{j-1}  (x folded into this pass)
//                      partials (p_j, q_j)  [and (r_0, r_0), (r_0, z_0) at j = 0]
//   grid barrier -> alpha_j = (r_j, z_j) / (p_j, q_j)
//   pass B (pointwise) r_{j+1} = r_j - alpha_j q_j, z_{j+1} = K^{-1} r_{j+1};  (r, r), (r, z)
//   grid barrier -> stop on ||r_{j+1}|| <= tol ||b||, beta_j = (r_{j+1}, z_{j+1}) / (r_j, z_j)
//
// The last step's x += alpha p is applied by hs_xfix_kernel after the loop.  Bytes per iteration
// and system: pass A reads r, p, x and writes p (ping-pong), q, x; pass B reads r, q and writes r:
// 9 vectors = 72 K N B (SURVEY 8(d) "two-kernel HS"), against 48 (6 vectors) of the single-pass
// kernel.  Tiles are staged by plain coalesced loads (the variant is for like-for-like parity with
// the oracle's HS-CG and as the measured baseline of the single-pass design, not the headline);
// CTA partial sums follow a static tile order, so results are deterministic for a given batch.
#include "kcg_cg.cuh"

namespace kcg {

template <int K, bool D2>
struct HsGeom {
  static constexpr int R = D2 ? 2 : 1;  // operator radius
  static constexpr int TX = 64;
  static constexpr int TY = hs_tile_y(K);
  static constexpr int BW = TX + 2 * R, BH = TY + 2 * R, PLANE = BW * BH;
  static constexpr int SW = TX + 2, SH = TY + 2, SPLANE = SW * SH;  // D2 scratch: D p on tile + 1 ring
  static constexpr int NT = 256, NW = NT / 32;
  static constexpr size_t smem_fixed() { return (size_t)(2 * K * PLANE + (D2 ? K * SPLANE : 0)) * 8; }
};

// Block-wide sums of NV values (fixed order: warp shuffle tree, then warps in order); result in
// out[0..NV) on every thread.  Two barriers.
template <int NV, int NW>
__device__ __forceinline__ void block_sums(double (&v)[NV], double (*red)[NW], double (&out)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double s = warp_sum(v[q]);
    if (lane == 0) red[q][warp] = s;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[q][w];
    out[q] = s;
  }
  __syncthreads();
}

// CTA partial sums [slot][cta][system][3] -> every CTA sums over the CTAs in CTA order (lane-strided,
// then the warp's shuffle tree: deterministic); warp w handles systems act[w], act[w + NW], ...
template <int NW>
__device__ __forceinline__ void hs_reduce(const double* part, int ncta, int n_sys, const int* act, int nact,
                                          double (*sums)[3]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int ii = warp; ii < nact; ii += NW) {
    const int s = act[ii];
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int b = lane; b < ncta; b += 32) {
      const double* p = part + ((size_t)b * n_sys + s) * 3;
      v0 += __ldcg(p);
      v1 += __ldcg(p + 1);
      v2 += __ldcg(p + 2);
    }
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    v2 = warp_sum(v2);
    if (lane == 0) { sums[ii][0] = v0; sums[ii][1] = v1; sums[ii][2] = v2; }
  }
  __syncthreads();
}

template <int K, bool HITS, bool PREC, bool D2>
__global__ void __launch_bounds__(256) cg_hs_kernel(const CgArgs a, double* __restrict__ q_buf,
                                                    double* __restrict__ hs_part) {
  using Gm = HsGeom<K, D2>;
  constexpr int R = Gm::R, TX = Gm::TX, TY = Gm::TY, BW = Gm::BW, PLANE = Gm::PLANE;
  constexpr int SW = Gm::SW, SPLANE = Gm::SPLANE, NT = Gm::NT, NW = Gm::NW;
  extern __shared__ __align__(16) double hs_smem[];
  double* Rs = hs_smem;              // [K][BH][BW] r box
  double* Ps = hs_smem + K * PLANE;  // [K][BH][BW] p_old box, then p_new in place
  double* Ss = hs_smem + 2 * K * PLANE;  // D2: [K][SH][SW] D p_new
  SysState* st = reinterpret_cast<SysState*>(hs_smem + Gm::smem_fixed() / 8);
  int* act = reinterpret_cast<int*>(st + a.n_sys);
  double (*sums)[3] = reinterpret_cast<double (*)[3]>(act + ((a.n_sys + 1) & ~1));  // [n_sys][3]
  double* acc = &sums[0][0] + 3 * a.n_sys;  // this CTA's partials [n_sys][3]
  __shared__ double red[3][NW];
  __shared__ int s_nact;
  __shared__ double Msh[K * K + K + 4 * K * K];

  const int tid = threadIdx.x, cta = blockIdx.x, ncta = gridDim.x;
  const int side = a.side, pitch = a.pitch;
  const size_t N = (size_t)side * side, ps = (size_t)pitch * side;
  const int tps = a.tiles_per_sys, tiles_x = a.tiles_x;
  cg::grid_group grid = cg::this_grid();

  for (int s = tid; s < a.n_sys; s += NT) {
    SysState z;
    z.bnorm2 = 0.0; z.gamma = 0.0; z.alpha = 0.0; z.beta = 0.0; z.rel = 1.0;
    z.iters = 0; z.status = ST_RUNNING; z.parity = 0; z.pad = 0; z.alpha_last = 0.0;
    st[s] = z;
  }
  __syncthreads();

  auto degree = [&](int gy, int gx) { return 4 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1); };
  auto in_face = [&](int gy, int gx) { return gy >= 0 && gy < side && gx >= 0 && gx < side; };

  for (int it = 0;; ++it) {
    if (tid == 0) {
      int n = 0;
      for (int s = 0; s < a.n_sys; ++s)
        if (st[s].status == ST_RUNNING) act[n++] = s;
      s_nact = n;
    }
    __syncthreads();
    const int nact = s_nact;
    if (nact == 0) break;
    for (int e = tid; e < 3 * a.n_sys; e += NT) acc[e] = 0.0;
    __syncthreads();

    // ------------------------------------------------------------------ pass A (static tile order)
    const int ntiles = nact * tps;
    for (int t = cta; t < ntiles; t += ncta) {
      const int s = act[t / tps], tile = t - (t / tps) * tps;
      const int y0 = (tile / tiles_x) * TY, x0 = (tile - (tile / tiles_x) * tiles_x) * TX;
      const SysParams* sp = a.params + s;
      const SysState z = st[s];
      const double beta = z.beta, ap = z.alpha_last, kappa2 = __ldg(&sp->kappa2);
      const bool xupd = it > 0;
      const double* rg = a.rbuf[0] + (size_t)s * K * ps;
      const double* pg = (z.parity ? a.pbuf[1] : a.pbuf[0]) + (size_t)s * K * ps;
      double* pn_g = (z.parity ? a.pbuf[0] : a.pbuf[1]) + (size_t)s * K * ps;
      double* qg = q_buf + (size_t)s * K * ps;
      double* xg = a.x + (size_t)s * K * N;
      const double* hp = HITS ? a.hits + (size_t)__ldg(&sp->hits_plane) * N : nullptr;
      if (tid < K * K) Msh[tid] = __ldg(&sp->M[tid]);
      else if (tid < K * K + K) Msh[tid] = __ldg(&sp->tau[tid - K * K]);
      else if (PREC && tid < K * K + K + 4 * K * K) Msh[tid] = __ldg(&sp->Kinv[0][0] + (tid - K * K - K));
      // stage the r and p_old boxes (zero outside the face)
      for (int e = tid; e < K * PLANE; e += NT) {
        const int c = e / PLANE, rem = e - c * PLANE, by = rem / BW, bx = rem - by * BW;
        const int gy = y0 - R + by, gx = x0 - R + bx;
        double rv = 0.0, pv = 0.0;
        if (in_face(gy, gx)) {
          const size_t o = (size_t)c * ps + (size_t)gy * pitch + gx;
          rv = __ldcg(rg + o);
          pv = it > 0 ? __ldcg(pg + o) : 0.0;
        }
        Rs[e] = rv;
        Ps[e] = pv;
      }
      __syncthreads();
      const double* M = Msh;
      const double* tau = Msh + K * K;
      // p_new = z + beta p_old on the box; x += alpha_prev p_old on the tile; (r, r), (r, z) at j = 0
      double v[3] = {0.0, 0.0, 0.0};  // (p, q), (r, r), (r, z)
      for (int e = tid; e < PLANE; e += NT) {
        const int by = e / BW, bx = e - by * BW, gy = y0 - R + by, gx = x0 - R + bx;
        if (!in_face(gy, gx)) continue;  // p_new stays 0 outside the face
        double r[K], u[K];
#pragma unroll
        for (int c = 0; c < K; ++c) r[c] = Rs[c * PLANE + e];
        if (PREC) {
          double tv[K];
#pragma unroll
          for (int c = 0; c < K; ++c) tv[c] = tau[c];
          precond_pixel<K, HITS>(Msh + K * K + K, M, tv, kappa2, HITS ? __ldg(hp + (size_t)gy * side + gx) : 1.0,
                                 side == 1 ? 0 : degree(gy, gx), r, u, D2);
        } else {
#pragma unroll
          for (int c = 0; c < K; ++c) u[c] = r[c];
        }
        const bool tile_px = by >= R && by < R + TY && bx >= R && bx < R + TX;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double po = Ps[c * PLANE + e];
          Ps[c * PLANE + e] = fma(beta, po, u[c]);
          if (tile_px) {
            if (it == 0) { v[1] = fma(r[c], r[c], v[1]); v[2] = fma(r[c], u[c], v[2]); }
            if (xupd) {
              double* xp = xg + (size_t)c * N + (size_t)gy * side + gx;
              *xp = fma(ap, po, __ldcg(xp));
            }
          }
        }
      }
      __syncthreads();
      if constexpr (D2) {  // S = D p_new on tile + 1 ring, zero outside the face
        for (int e = tid; e < SPLANE; e += NT) {
          const int sy = e / SW, sx = e - sy * SW;
          const int by = sy + R - 1, bx = sx + R - 1, gy = y0 + sy - 1, gx = x0 + sx - 1;
          const bool f = in_face(gy, gx);
          const int deg = f ? (side == 1 ? 0 : degree(gy, gx)) : 0;
#pragma unroll
          for (int c = 0; c < K; ++c) {
            const double* pc = Ps + c * PLANE + by * BW + bx;
            Ss[c * SPLANE + e] = f ? ((pc[-BW] + pc[BW]) + (pc[-1] + pc[1])) - deg * pc[0] : 0.0;
          }
        }
        __syncthreads();
      }
      // q = G p_new on the tile; store p_new, q; (p, q)
      for (int e = tid; e < TY * TX; e += NT) {
        const int ty = e / TX, tx = e - ty * TX, gy = y0 + ty, gx = x0 + tx;
        if (gy >= side || gx >= side) continue;
        const int by = ty + R, bx = tx + R;
        const int deg = side == 1 ? 0 : degree(gy, gx);
        const double h = HITS ? __ldg(hp + (size_t)gy * side + gx) : 1.0;
        double pc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) pc[c] = Ps[c * PLANE + by * BW + bx];
        const size_t o = (size_t)gy * pitch + gx;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          double mix = 0.0;
#pragma unroll
          for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], pc[d], mix);
          double qp;
          if constexpr (D2) {
            const double* sc = Ss + c * SPLANE + (ty + 1) * SW + (tx + 1);
            qp = fma(kappa2, pc[c], ((sc[-SW] + sc[SW]) + (sc[-1] + sc[1])) - deg * sc[0]);
          } else {
            const double* pp = Ps + c * PLANE + by * BW + bx;
            qp = fma(kappa2 + deg, pc[c], -((pp[-BW] + pp[BW]) + (pp[-1] + pp[1])));
          }
          const double q = fma(h, mix, tau[c] * qp);
          pn_g[(size_t)c * ps + o] = pc[c];
          qg[(size_t)c * ps + o] = q;
          v[0] = fma(pc[c], q, v[0]);
        }
      }
      double out[3];
      block_sums<3, NW>(v, red, out);  // (its barriers also retire this tile's smem)
      if (tid == 0) { acc[3 * s] += out[0]; acc[3 * s + 1] += out[1]; acc[3 * s + 2] += out[2]; }
    }
    __syncthreads();
    double* partA = hs_part;                                  // slot 0
    double* partB = hs_part + (size_t)ncta * a.n_sys * 3;     // slot 1
    for (int ii = tid; ii < nact; ii += NT) {
      const int s = act[ii];
      double* d = partA + ((size_t)cta * a.n_sys + s) * 3;
      d[0] = acc[3 * s]; d[1] = acc[3 * s + 1]; d[2] = acc[3 * s + 2];
    }
    __threadfence();
    grid.sync();
    hs_reduce<NW>(partA, ncta, a.n_sys, act, nact, sums);
    if (tid < nact) {  // alpha_j = (r_j, z_j) / (p_j, q_j)
      const int s = act[tid];
      SysState z = st[s];
      const double pq = sums[tid][0];
      if (it == 0) {
        z.bnorm2 = sums[tid][1];
        z.gamma = sums[tid][2];
        z.rel = z.bnorm2 > 0.0 ? 1.0 : 0.0;
      }
      if (!isfinite(pq) || !isfinite(z.bnorm2) || !isfinite(z.gamma)) z.status = ST_NONFINITE;
      else if (it == 0 && z.bnorm2 == 0.0) z.status = ST_CONVERGED;
      else if (it == 0 && a.max_iter <= 0) z.status = ST_MAXIT;
      else if (!(pq > 0.0) || !(z.gamma > 0.0)) z.status = ST_BREAKDOWN;
      else z.alpha = z.gamma / pq;
      z.alpha_last = 0.0;  // x now holds every step before j
      st[s] = z;
    }
    __syncthreads();
    for (int e = tid; e < 3 * a.n_sys; e += NT) acc[e] = 0.0;
    __syncthreads();

    // ------------------------------------------------------------------ pass B (pointwise)
    const size_t gtid = (size_t)cta * NT + tid, gstride = (size_t)ncta * NT;
    for (int ii = 0; ii < nact; ++ii) {
      const int s = act[ii];
      const SysState z = st[s];
      double v[3] = {0.0, 0.0, 0.0};  // (r, r), (r, z), unused
      if (z.status == ST_RUNNING) {
        const SysParams* sp = a.params + s;
        const double alpha = z.alpha, kappa2 = __ldg(&sp->kappa2);
        double* rg = a.rbuf[0] + (size_t)s * K * ps;
        const double* qg = q_buf + (size_t)s * K * ps;
        const double* hp = HITS ? a.hits + (size_t)__ldg(&sp->hits_plane) * N : nullptr;
        double tv[K];
#pragma unroll
        for (int c = 0; c < K; ++c) tv[c] = __ldg(&sp->tau[c]);
        const double* Mg = sp->M;              // PREC: read through L1 (constant per system)
        const double* Ki = &sp->Kinv[0][0];
        for (size_t j = gtid; j < N; j += gstride) {
          const int gy = (int)(j / side), gx = (int)(j - (size_t)gy * side);
          const size_t o = (size_t)gy * pitch + gx;
          double r[K], u[K];
#pragma unroll
          for (int c = 0; c < K; ++c) {
            r[c] = fma(-alpha, __ldcg(qg + c * ps + o), __ldcg(rg + c * ps + o));
            rg[c * ps + o] = r[c];
          }
          if (PREC) {
            precond_pixel<K, HITS>(Ki, Mg, tv, kappa2, HITS ? __ldg(hp + j) : 1.0, side == 1 ? 0 : degree(gy, gx), r,
                                   u, D2);
          } else {
#pragma unroll
            for (int c = 0; c < K; ++c) u[c] = r[c];
          }
#pragma unroll
          for (int c = 0; c < K; ++c) {
            v[0] = fma(r[c], r[c], v[0]);
            v[1] = fma(r[c], u[c], v[1]);
          }
        }
      }
      double out[3];
      block_sums<3, NW>(v, red, out);
      if (tid == 0) { acc[3 * s] = out[0]; acc[3 * s + 1] = out[1]; }
    }
    __syncthreads();
    for (int ii = tid; ii < nact; ii += NT) {
      const int s = act[ii];
      double* d = partB + ((size_t)cta * a.n_sys + s) * 3;
      d[0] = acc[3 * s]; d[1] = acc[3 * s + 1]; d[2] = 0.0;
    }
    __threadfence();
    grid.sync();
    hs_reduce<NW>(partB, ncta, a.n_sys, act, nact, sums);
    if (tid < nact) {  // stop test on the recursive residual; beta_j = (r_{j+1}, z_{j+1}) / (r_j, z_j)
      const int s = act[tid];
      SysState z = st[s];
      if (z.status == ST_RUNNING) {
        const double rr = sums[tid][0], rz = sums[tid][1];
        z.iters = it + 1;
        z.alpha_last = z.alpha;  // alpha_j p_j pending in x
        z.parity ^= 1;           // p_j now lives in buffer `parity`
        z.rel = sqrt(rr / z.bnorm2);
        if (!isfinite(rr) || !isfinite(rz)) z.status = ST_NONFINITE;
        else if (rr <= a.tol2 * z.bnorm2) z.status = ST_CONVERGED;
        else if (z.iters >= a.max_iter) z.status = ST_MAXIT;
        else if (!(rz > 0.0)) z.status = ST_BREAKDOWN;
        else { z.beta = rz / z.gamma; z.gamma = rz; }
        st[s] = z;
      }
    }
    __syncthreads();
    if (cta == 0 && tid == 0 && it < a.history_cap) {
      double m = 0.0;
      for (int ii = 0; ii < nact; ++ii) m = fmax(m, st[act[ii]].rel);
      a.history[it] = m;
    }
  }
  if (cta == 0)
    for (int s = tid; s < a.n_sys; s += NT) a.state_out[s] = st[s];
}

// x += alpha_last p (buffer `parity`) for every system: the step of its last iteration.
template <int K>
__global__ void __launch_bounds__(256) hs_xfix_kernel(const SysState* __restrict__ st, const double* __restrict__ p0,
                                                      const double* __restrict__ p1, double* __restrict__ x, int side,
                                                      int pitch) {
  const int s = blockIdx.y;
  const SysState z = st[s];
  if (z.iters < 1 || z.alpha_last == 0.0) return;
  const size_t N = (size_t)side * side, ps = (size_t)pitch * side;
  const double* p = (z.parity ? p1 : p0) + (size_t)s * K * ps;
  double* xs = x + (size_t)s * K * N;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x) {
    const size_t gy = j / side, gx = j - gy * side;
#pragma unroll
    for (int c = 0; c < K; ++c) xs[c * N + j] = fma(z.alpha_last, p[(size_t)c * ps + gy * pitch + gx], xs[c * N + j]);
  }
}

template <int K>
struct HsEntry {
  static cudaError_t config(bool hits, bool prec, bool d2, int n_sys, int* max_grid, size_t* smem);
  static cudaError_t launch(bool prec, bool d2, cudaStream_t s, const CgArgs& a, double* q, double* part, int grid,
                            size_t smem);
  static cudaError_t xfix(cudaStream_t s, const SysState* st, const double* p0, const double* p1, double* x, int n_sys,
                          int side, int pitch);
};

template <int K, bool HITS, bool PREC, bool D2>
static const void* hs_fn() {
  if constexpr ((D2 && K > 4) || (PREC && K > 7)) return nullptr;
  else return (const void*)cg_hs_kernel<K, HITS, PREC, D2>;
}
template <int K>
static const void* hs_pick(bool hits, bool prec, bool d2) {
  if (d2) {
    if (prec) return hits ? hs_fn<K, true, true, true>() : hs_fn<K, false, true, true>();
    return hits ? hs_fn<K, true, false, true>() : hs_fn<K, false, false, true>();
  }
  if (prec) return hits ? hs_fn<K, true, true, false>() : hs_fn<K, false, true, false>();
  return hits ? hs_fn<K, true, false, false>() : hs_fn<K, false, false, false>();
}

template <int K>
cudaError_t HsEntry<K>::config(bool hits, bool prec, bool d2, int n_sys, int* max_grid, size_t* smem) {
  const void* f = hs_pick<K>(hits, prec, d2);
  if (!f) return cudaErrorInvalidValue;
  const size_t fixed = d2 ? HsGeom<K, true>::smem_fixed() : HsGeom<K, false>::smem_fixed();
  const size_t sm = fixed + (size_t)n_sys * (sizeof(SysState) + sizeof(int)) + 8 + (size_t)n_sys * 6 * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int nb = 0, dev = 0, nsm = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, 256, sm)) != cudaSuccess) return e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  *max_grid = nb * nsm;
  *smem = sm;
  return nb > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

template <int K>
cudaError_t HsEntry<K>::launch(bool prec, bool d2, cudaStream_t s, const CgArgs& a, double* q, double* part, int grid,
                               size_t smem) {
  const void* f = hs_pick<K>(a.hits != nullptr, prec, d2);
  if (!f) return cudaErrorInvalidValue;
  void* args[3] = {(void*)&a, (void*)&q, (void*)&part};
  // the attribute is per function and shared by the routes (contexts) that launch it: set it to
  // this launch's size every time
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(f, dim3(grid), dim3(256), args, smem, s);
}

template <int K>
cudaError_t HsEntry<K>::xfix(cudaStream_t s, const SysState* st, const double* p0, const double* p1, double* x,
                             int n_sys, int side, int pitch) {
  const size_t N = (size_t)side * side;
  const int gx = (int)std::min<size_t>((N + 255) / 256, 1184);
  hs_xfix_kernel<K><<<dim3(std::max(gx, 1), n_sys), 256, 0, s>>>(st, p0, p1, x, side, pitch);
  return cudaGetLastError();
}

}  // namespace kcg
