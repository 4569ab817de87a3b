#pragma once
// sm_100a fp64: the small-problem regime of the CG iteration (SURVEY 8(d) "size regimes"; the paper's
// experiments run HEALPix levels 1-10, most of which are latency- not bandwidth-bound on a
// B200).  When a batch's CG state fits in the SMs' shared memory, the solve keeps x, r and p ON CHIP
// for the whole iteration instead of streaming them through HBM every pass:
//
//   * CTA = one row strip of RS rows (full face width) of one system, resident for the whole solve
//     (cooperative launch, n_sys * side / RS CTAs, one per SM);
//   * per pass the same single-pass (Chronopoulos-Gear) iteration as cg_persistent_kernel, with the
//     same scalars (cg_update) and stopping rule: p = u + beta p on strip + 2 rows, q = G p and
//     r -= alpha q on strip + 1 row, w = G u on the strip, x += alpha p, partials (r,r), (r,u), (w,u)
//     -- the 2 halo rows above / below are the neighbouring strips' r and p, published every pass
//     into the r / p ping-pong buffers (L2-resident rows) and read back after the pass's ONE grid
//     barrier, which also carries the reduction (every CTA sums every system's strip partials in
//     strip order: deterministic, identical on every CTA);
//   * RS = side ("single" mode, small faces: one CTA per system) needs no grid barrier at all: each
//     CTA iterates its own system with __syncthreads only.
// Global traffic per pass: 4 halo rows of r and p per strip read + written (L2), 3 partials per CTA;
// b read once, x written once.  Laplacian prior (radius 1), with hits and block-Jacobi.
#include "kcg_cg.cuh"

namespace kcg {

template <int K, bool HITS, bool PREC>
__global__ void __launch_bounds__(256, 1) cg_resident_kernel(const CgArgs a, double* __restrict__ part) {
  constexpr int NT = 256, NW = NT / 32;
  const int side = a.side, pitch = a.pitch, nstrip = a.tiles_per_sys, RS = side / nstrip;
  const int BW = side + 2, BH = RS + 4;
  const int cta = blockIdx.x, ncta = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = cta / nstrip, strip = cta - s * nstrip, y0 = strip * RS;
  const int lside = 31 - __clz(side);  // side = 2^L
  const bool gmode = nstrip > 1;
  const size_t N = (size_t)side * side, ps = (size_t)pitch * side;
  const int BOX = BH * BW, UBOX = (RS + 2) * BW;
  const SysParams* sp = a.params + s;

  extern __shared__ __align__(16) double rs_smem[];
  double* Rb = rs_smem;                    // [K][BH][BW]: r (rows y0-2 .. y0+RS+1, column pads)
  double* Pb = Rb + K * BOX;               // [K][BH][BW]: p
  double* Ub = Pb + K * BOX;               // [K][RS+2][BW]: u = K^{-1} r_new (PREC)
  double* Xb = Ub + (PREC ? K * UBOX : 0);  // [K][RS][side]: x
  double* Hb = Xb + K * RS * side;         // [BH][BW]: hits (HITS)
  SysState* st = reinterpret_cast<SysState*>(Hb + (HITS ? BOX : 0));  // [n_sys]
  double* Pq = reinterpret_cast<double*>(st + a.n_sys);  // grid mode: every CTA's partials [ncta][3]
  __shared__ double Msh[K * K + K + 4 * K * K];
  __shared__ double red[3][NW];
  cg::grid_group grid = cg::this_grid();

  // ---------------------------------------------------------------- set-up: b and the constants
  const int total = (2 * K * BOX + (PREC ? K * UBOX : 0) + K * RS * side + (HITS ? BOX : 0));
  for (int e = tid; e < total; e += NT) rs_smem[e] = 0.0;
  for (int t = tid; t < a.n_sys; t += NT) {
    SysState z;
    z.bnorm2 = 0.0; z.gamma = 0.0; z.alpha = 0.0; z.beta = 0.0; z.rel = 1.0;
    z.iters = 0; z.status = ST_RUNNING; z.parity = 0; z.pad = 0; z.alpha_last = 0.0;
    st[t] = z;
  }
  if (tid < K * K) Msh[tid] = __ldg(&sp->M[tid]);
  else if (tid < K * K + K) Msh[tid] = __ldg(&sp->tau[tid - K * K]);
  else if (PREC && tid < K * K + K + 4 * K * K) Msh[tid] = __ldg(&sp->Kinv[0][0] + (tid - K * K - K));
  __syncthreads();
  const double kappa2 = __ldg(&sp->kappa2);
  const double* hp = HITS ? a.hits + (size_t)__ldg(&sp->hits_plane) * N : nullptr;
  // rows [b0, b1) of the box from the global planes g (b: ping-pong buffer 0 holds b at start)
  auto load_rows = [&](double* box, const double* g, int b0, int b1) {
    const int n = (b1 - b0) * side;
    for (int c = 0; c < K; ++c)
      for (int e = tid; e < n; e += NT) {
        const int by = b0 + e / side, gx = e - (e / side) * side, gy = y0 - 2 + by;
        if (gy >= 0 && gy < side) box[(c * BH + by) * BW + gx + 1] = __ldcg(g + (s * K + c) * ps + (size_t)gy * pitch + gx);
      }
  };
  load_rows(Rb, a.rbuf[0], 0, BH);
  if (a.bnorm2)  // warm start: the strip's x starts at x_0 (a.x holds it), not at 0
    for (int c = 0; c < K; ++c)
      for (int e = tid; e < RS * side; e += NT) Xb[c * RS * side + e] = a.x[(s * K + c) * N + (size_t)y0 * side + e];
  if (HITS)
    for (int e = tid; e < BH * side; e += NT) {
      const int by = e / side, gx = e - by * side, gy = y0 - 2 + by;
      if (gy >= 0 && gy < side) Hb[by * BW + gx + 1] = __ldg(hp + (size_t)gy * side + gx);
    }
  __syncthreads();
  const double* M = Msh;
  const double* tau = Msh + K * K;
  const double* Kinv = Msh + K * K + K;
  auto degree = [&](int gy, int gx) { return 4 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1); };
  auto hit = [&](int by, int gx) { return HITS ? Hb[by * BW + gx + 1] : 1.0; };
  // rows [b0, b1) inside the face
  auto rows_in = [&](int b0, int b1, int& lo, int& hi) {
    lo = max(b0, 2 - y0);
    hi = min(b1, side - y0 + 2);
  };

  // KCG_TRACE builds: per pass q, [0] CTA 0 start, [1..3] after phases A, B, C (+ halo publish),
  // [4] after the grid barrier, [5] after the reduction, [6 + b] CTA b at the barrier
  const bool trc = KCG_TRACE == 1 && a.trace != nullptr;
  auto stamp = [&](int q, int col) {
    if (trc && q < KCG_TRACE_ITERS && tid == 0 && (cta == 0 || col >= 6) && col < KCG_TRACE_COLS)
      a.trace[(size_t)q * KCG_TRACE_COLS + col] = globaltimer();
  };
  for (int it = -1;; ++it) {
    const int q = it + 1;  // pass number; writes ping-pong buffer (q + 1) & 1
    stamp(q, 0);
    const SysState z = st[s];
    double v[3] = {0.0, 0.0, 0.0};  // (r, r), (r, u), (w, u)
    if (z.status == ST_RUNNING) {
      const double alpha = z.alpha, beta = z.beta;
      int lo, hi;
      // Phase A: p = u + beta p, u = K^{-1} r, on every in-face box row
      rows_in(0, BH, lo, hi);
      for (int e = tid; e < (hi - lo) * side; e += NT) {
        const int by = lo + e / side, gx = e - (e / side) * side;
        const int o = by * BW + gx + 1;
        double r[K], u[K];
#pragma unroll
        for (int c = 0; c < K; ++c) r[c] = Rb[c * BOX + o];
        if (PREC) precond_pixel<K, HITS>(Kinv, M, tau, kappa2, hit(by, gx), degree(y0 - 2 + by, gx), r, u);
        else
#pragma unroll
          for (int c = 0; c < K; ++c) u[c] = r[c];
#pragma unroll
        for (int c = 0; c < K; ++c) Pb[c * BOX + o] = fma(beta, Pb[c * BOX + o], u[c]);
      }
      __syncthreads();
      stamp(q, 1);
      // Phase B: q = G p, r -= alpha q on strip + 1 row
      rows_in(1, BH - 1, lo, hi);
      for (int e = tid; e < (hi - lo) * side; e += NT) {
        const int by = lo + e / side, gx = e - (e / side) * side;
        const int o = by * BW + gx + 1;
        const double kd = kappa2 + degree(y0 - 2 + by, gx), h = hit(by, gx);
        double pc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) pc[c] = Pb[c * BOX + o];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double* pp = Pb + c * BOX + o;
          const double nb = (pp[-BW] + pp[BW]) + (pp[-1] + pp[1]);
          double mix = 0.0;
#pragma unroll
          for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], pc[d], mix);
          Rb[c * BOX + o] = fma(-alpha, op_point<HITS>(h, mix, tau[c], kd, pc[c], nb), Rb[c * BOX + o]);
        }
      }
      __syncthreads();
      stamp(q, 2);
      if (PREC) {  // Phase B': u = K^{-1} r_new on strip + 1 row (U row = box row - 1)
        for (int e = tid; e < (hi - lo) * side; e += NT) {
          const int by = lo + e / side, gx = e - (e / side) * side;
          double r[K], u[K];
#pragma unroll
          for (int c = 0; c < K; ++c) r[c] = Rb[c * BOX + by * BW + gx + 1];
          precond_pixel<K, HITS>(Kinv, M, tau, kappa2, hit(by, gx), degree(y0 - 2 + by, gx), r, u);
#pragma unroll
          for (int c = 0; c < K; ++c) Ub[c * UBOX + (by - 1) * BW + gx + 1] = u[c];
        }
        __syncthreads();
      }
      // Phase C: w = G u on the strip; partials; x += alpha p
      const double* Vb = PREC ? Ub - BW : Rb;  // addressed with box rows
      const int VBOX = PREC ? UBOX : BOX;
      rows_in(2, RS + 2, lo, hi);
      for (int e = tid; e < (hi - lo) * side; e += NT) {
        const int by = lo + e / side, gx = e - (e / side) * side;
        const int o = by * BW + gx + 1;
        const double kd = kappa2 + degree(y0 - 2 + by, gx), h = hit(by, gx);
        double uc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) uc[c] = Vb[c * VBOX + o];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double* up = Vb + c * VBOX + o;
          const double nb = (up[-BW] + up[BW]) + (up[-1] + up[1]);
          double mix = 0.0;
#pragma unroll
          for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], uc[d], mix);
          const double w = op_point<HITS>(h, mix, tau[c], kd, uc[c], nb);
          const double r = Rb[c * BOX + o];
          v[0] = fma(r, r, v[0]);
          if (PREC) v[1] = fma(r, uc[c], v[1]);
          v[2] = fma(w, uc[c], v[2]);
          double* xp = Xb + (c * RS + by - 2) * side + gx;
          *xp = fma(alpha, Pb[c * BOX + o], *xp);
        }
      }
      if (!PREC) v[1] = v[0];
      if (gmode) {  // publish the strip's first and last two rows of r and p (the neighbours' halo)
        double* rg = (q & 1) ? a.rbuf[0] : a.rbuf[1];
        double* pg = (q & 1) ? a.pbuf[0] : a.pbuf[1];
        const int nb4 = min(4, RS);
        for (int c = 0; c < K; ++c)
          for (int e = tid; e < nb4 * side; e += NT) {
            const int k4 = e / side, gx = e - k4 * side;
            const int ly = (RS <= 4) ? k4 : (k4 < 2 ? k4 : RS - 4 + k4);  // strip row
            if (y0 + ly >= side) continue;
            const int o = (ly + 2) * BW + gx + 1;
            const size_t go = (s * K + c) * ps + (size_t)(y0 + ly) * pitch + gx;
            rg[go] = Rb[c * BOX + o];
            pg[go] = Pb[c * BOX + o];
          }
      }
    }
    // block sums of the partials (fixed order)
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const double w = warp_sum(v[t]);
      if (lane == 0) red[t][warp] = w;
    }
    __syncthreads();
    if (gmode) {
      if (tid < 3) {
        double acc = 0.0;
        for (int w = 0; w < NW; ++w) acc += red[tid][w];
        part[((size_t)(q & 1) * ncta + cta) * 3 + tid] = acc;
      }
      stamp(q, 3);  // (grid.sync orders the halo / partial stores of every thread before it)
      stamp(q, 6 + cta);
      grid.sync();
      stamp(q, 4);
      // The next pass's halo rows (box rows 0, 1, RS + 2, RS + 3 of r and p, written by the
      // neighbouring strips this pass) are loaded into registers in batches of HC per thread, their
      // L2 latency overlapped with the reduction below; element e = ((f K + c) 4 + row) side + x.
      constexpr int HC = 24;
      const bool halo = z.status == ST_RUNNING;
      const int nh = halo ? 8 * K * side : 0;
      const double* rg = (q & 1) ? a.rbuf[0] : a.rbuf[1];
      const double* pg = (q & 1) ? a.pbuf[0] : a.pbuf[1];
      auto decode = [&](int e, int& so, size_t& go) {  // false: outside the face (stays 0)
        const int gx = e & (side - 1), t4 = e >> lside, hr = t4 & 3, fc = t4 >> 2, c = fc % K, f = fc / K;
        const int by = hr < 2 ? hr : RS + hr, gy = y0 - 2 + by;
        so = (f * K + c) * BOX + by * BW + gx + 1;  // Pb = Rb + K * BOX
        go = (size_t)(s * K + c) * ps + (size_t)gy * pitch + gx;
        return gy >= 0 && gy < side;
      };
      double hv[HC];
#pragma unroll
      for (int j = 0; j < HC; ++j) {
        const int e = j * NT + tid;
        int so;
        size_t go;
        hv[j] = (e < nh && decode(e, so, go)) ? __ldcg(((e / (4 * side * K)) ? pg : rg) + go) : 0.0;
      }
      // every CTA: every system's sums over its strips in strip order, then the CG scalar update.
      // All partials come in ONE round of loads (batches of PC per thread) into shared memory.
      const double* pq = part + (size_t)(q & 1) * ncta * 3;
      constexpr int PC = 12;
      for (int e0 = 0; e0 < ncta * 3; e0 += PC * NT) {
        double pv[PC];
#pragma unroll
        for (int j = 0; j < PC; ++j) {
          const int e = e0 + j * NT + tid;
          pv[j] = e < ncta * 3 ? __ldcg(pq + e) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PC; ++j) {
          const int e = e0 + j * NT + tid;
          if (e < ncta * 3) Pq[e] = pv[j];
        }
      }
      __syncthreads();
      for (int t = warp; t < a.n_sys; t += NW) {
        if (st[t].status != ST_RUNNING) continue;
        double w0 = 0.0, w1 = 0.0, w2 = 0.0;
        for (int b = lane; b < nstrip; b += 32) {
          const double* p3 = Pq + ((size_t)t * nstrip + b) * 3;
          w0 += p3[0];
          w1 += p3[1];
          w2 += p3[2];
        }
        w0 = warp_sum(w0);
        w1 = warp_sum(w1);
        w2 = warp_sum(w2);
        if (lane == 0) st[t] = cg_update(st[t], w0, w1, w2, it, a, t);
      }
#pragma unroll
      for (int j = 0; j < HC; ++j) {
        const int e = j * NT + tid;
        int so;
        size_t go;
        if (e < nh && decode(e, so, go)) rs_smem[so] = hv[j];
      }
      for (int e0 = HC * NT; e0 < nh; e0 += HC * NT) {  // wide faces: further batches
#pragma unroll
        for (int j = 0; j < HC; ++j) {
          const int e = e0 + j * NT + tid;
          int so;
          size_t go;
          hv[j] = (e < nh && decode(e, so, go)) ? __ldcg(((e / (4 * side * K)) ? pg : rg) + go) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < HC; ++j) {
          const int e = e0 + j * NT + tid;
          int so;
          size_t go;
          if (e < nh && decode(e, so, go)) rs_smem[so] = hv[j];
        }
      }
      __syncthreads();
      stamp(q, 5);
      bool done = true;  // every thread reads the same states: uniform
      double m = 0.0;
      for (int t = 0; t < a.n_sys; ++t) {
        done &= st[t].status != ST_RUNNING;
        m = fmax(m, st[t].rel);
      }
      if (cta == 0 && tid == 0 && it >= 0 && it < a.history_cap) a.history[it] = m;
      if (done) break;
    } else {
      if (tid == 0 && z.status == ST_RUNNING) {
        double w0 = 0.0, w1 = 0.0, w2 = 0.0;
        for (int w = 0; w < NW; ++w) { w0 += red[0][w]; w1 += red[1][w]; w2 += red[2][w]; }
        st[s] = cg_update(st[s], w0, w1, w2, it, a, s);
        if (it >= 0 && it < a.history_cap)  // max over the systems: positive doubles order as integers
          atomicMax(reinterpret_cast<unsigned long long*>(a.history + it), __double_as_longlong(st[s].rel));
      }
      __syncthreads();
      if (st[s].status != ST_RUNNING) break;
    }
  }
  // x of the strip; the final states
  for (int c = 0; c < K; ++c)
    for (int e = tid; e < RS * side; e += NT)
      a.x[(s * K + c) * N + (size_t)y0 * side + e] = Xb[c * RS * side + e];
  if (gmode) {
    if (cta == 0)
      for (int t = tid; t < a.n_sys; t += NT) a.state_out[t] = st[t];
  } else if (tid == 0) {
    a.state_out[s] = st[s];
  }
}

// Dynamic shared memory of the resident kernel for strips of RS rows (0 if it cannot fit).
__host__ __device__ constexpr size_t res_smem_bytes(int K, int RS, int side, bool hits, bool prec, int n_sys) {
  return 8 * ((size_t)2 * K * (RS + 4) * (side + 2) + (prec ? (size_t)K * (RS + 2) * (side + 2) : 0) +
              (size_t)K * RS * side + (hits ? (size_t)(RS + 4) * (side + 2) : 0)) +
         (size_t)n_sys * sizeof(SysState) + (RS < side ? (size_t)n_sys * (side / RS) * 3 * 8 : 0);
}

template <int K>
struct ResEntry {
  static cudaError_t config(bool hits, bool prec, size_t smem, int* blocks_per_sm);
  static cudaError_t launch(bool prec, cudaStream_t s, const CgArgs& a, double* part, int grid, size_t smem);
};

template <int K>
static const void* res_pick(bool hits, bool prec) {
  if constexpr (K > 7) {
    if (prec) return nullptr;
    return hits ? (const void*)cg_resident_kernel<K, true, false> : (const void*)cg_resident_kernel<K, false, false>;
  } else {
    if (prec) return hits ? (const void*)cg_resident_kernel<K, true, true> : (const void*)cg_resident_kernel<K, false, true>;
    return hits ? (const void*)cg_resident_kernel<K, true, false> : (const void*)cg_resident_kernel<K, false, false>;
  }
}

template <int K>
cudaError_t ResEntry<K>::config(bool hits, bool prec, size_t smem, int* blocks_per_sm) {
  const void* f = res_pick<K>(hits, prec);
  if (!f) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, 256, smem);
}

template <int K>
cudaError_t ResEntry<K>::launch(bool prec, cudaStream_t s, const CgArgs& a, double* part, int grid, size_t smem) {
  const void* f = res_pick<K>(a.hits != nullptr, prec);
  if (!f) return cudaErrorInvalidValue;
  void* args[2] = {(void*)&a, (void*)&part};
  // the attribute is per function and shared by the routes (contexts) that launch it: set it to
  // this launch's size every time
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(f, dim3(grid), dim3(256), args, smem, s);
}

}  // namespace kcg
