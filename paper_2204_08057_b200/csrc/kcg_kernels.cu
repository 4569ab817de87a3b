// sm_100a fp64 kernels of the Kronecker CG / Sylvester hot path (arxiv 2204.08057): the small
// kernels (rhs, apply / residual, x fix-up, back-transform, row-slab helpers) and the launchers.
// The persistent CG kernel templates live in kcg_cg.cuh (instantiated per K in kcg_cg_k<K>.cu).
#include "kcg_cg.cuh"

namespace kcg {

extern template struct CgEntry<1>;
extern template struct CgEntry<2>;
extern template struct CgEntry<3>;
extern template struct CgEntry<4>;
extern template struct CgEntry<5>;
extern template struct CgEntry<6>;
extern template struct CgEntry<7>;
extern template struct CgEntry<8>;

// --------------------------------------------------------------------------- apply / residual
constexpr int AP_TX = 64, AP_NT = 256;
#ifndef KCG_AP_TYD2
#define KCG_AP_TYD2 8   // apply / residual tile rows with the D2 prior (two boxes in shared memory per block: 52 KB at 8 rows, 4 blocks per SM; 16 rows: 87 KB, 2 blocks -- paper workload residual pass 0.43 ms slower)
#endif
constexpr int ap_ty(bool d2) { return d2 ? KCG_AP_TYD2 : 16; }
#ifndef KCG_AP_MINB
#define KCG_AP_MINB 4  // resident blocks per SM for apply_kernel, K <= 4 (64 registers: 2.8x faster than 1 under ncu); 2 above
#endif

int apply_tiles_per_sys(int rows, int side, bool d2) {
  return ((rows + ap_ty(d2) - 1) / ap_ty(d2)) * ((side + AP_TX - 1) / AP_TX);
}

// RESID = false: y = G x.   RESID = true: partials[s][tile] = (||b - G x||^2, ||b||^2) over the
// tile, with b = h Y E recomputed from the data (E = T A), or b = Y itself when E == nullptr.  Slab geometry: `rows` local rows from
// global face row `row0`; the halo rows beyond the slab come from xg_top / xg_bot ([planes][side],
// the neighbours' boundary rows; nullptr or outside the face -> 0).  D2: Q0 = D^2 + kappa2 I, the
// tile's x is staged with a 2-pixel halo and D x is formed on tile + 1-ring first (no slabs).
template <int K, bool RESID, bool D2>
__global__ void __launch_bounds__(AP_NT, (K <= 4 ? KCG_AP_MINB : 2)) apply_kernel(const SysParams* __restrict__ params,
                                                      const double* __restrict__ x, double* __restrict__ y,
                                                      const double* __restrict__ Y, const double* __restrict__ E,
                                                      const double* __restrict__ hits,
                                                      double* __restrict__ partials, int n, int side, int rows,
                                                      int row0, int ghost, int nested,
                                                      const double* __restrict__ xg_top,
                                                      const double* __restrict__ xg_bot) {
  constexpr int HA = D2 ? 2 : 1, AP_TY = ap_ty(D2);
  constexpr int BW = AP_TX + 2 * HA, BH = AP_TY + 2 * HA, PLANE = BW * BH;
  extern __shared__ double xs[];  // [K][BH][BW], then (D2) D x [K][BH][BW], then E [n][K] if RESID
  __shared__ double red[2][AP_NT / 32];
  const int s = blockIdx.y;
  const int tiles_x = (side + AP_TX - 1) / AP_TX;
  const int tile = blockIdx.x;
  const int ty0 = (tile / tiles_x) * AP_TY, tx0 = (tile % tiles_x) * AP_TX;  // local rows
  const size_t N = (size_t)rows * side;
  const SysParams* sp = params + s;
  for (int e = threadIdx.x; e < K * PLANE; e += AP_NT) {
    const int c = e / PLANE, r = e - c * PLANE;
    const int ly = ty0 - HA + r / BW, gx = tx0 - HA + r % BW, gyg = row0 + ly;
    double v = 0.0;
    if (gx >= 0 && gx < side && gyg >= 0 && gyg < side) {
      const size_t plane = (size_t)(s * K + c);
      if (ly >= 0 && ly < rows) v = x[(plane * rows + ly) * side + gx];
      else if (ly == -1 && xg_top) v = xg_top[plane * side + gx];
      else if (ly == rows && xg_bot) v = xg_bot[plane * side + gx];
    }
    xs[e] = v;
  }
  double* Ds = xs + K * PLANE;                  // D2: D x on tile + 1-ring (zero outside the face)
  double* Es = xs + (D2 ? 2 : 1) * K * PLANE;
  if (RESID && E)
    for (int e = threadIdx.x; e < n * K; e += AP_NT) Es[e] = E[(size_t)s * n * K + e];
  __syncthreads();
  auto degf = [&](int gy, int gx) { return 4 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1); };
  if (D2) {
    for (int e = threadIdx.x; e < K * PLANE; e += AP_NT) {
      const int c = e / PLANE, r = e - c * PLANE, by = r / BW, bx = r % BW;
      const int gy = row0 + ty0 - HA + by, gx = tx0 - HA + bx;
      double v = 0.0;
      if (by >= 1 && by < BH - 1 && bx >= 1 && bx < BW - 1 && gy >= 0 && gy < side && gx >= 0 && gx < side) {
        const double* xl = xs + e;
        v = ((xl[-BW] + xl[BW]) + (xl[-1] + xl[1])) - degf(gy, gx) * xl[0];
      }
      Ds[e] = v;
    }
    __syncthreads();
  }
  double M[K * K], tau[K];
#pragma unroll
  for (int e = 0; e < K * K; ++e) M[e] = sp->M[e];
#pragma unroll
  for (int c = 0; c < K; ++c) tau[c] = sp->tau[c];
  const double kappa2 = sp->kappa2;
  // hits planes [rows + 2 ghost][side] (ghost rows present in slab mode), local row 0 at +ghost
  const double* hp = hits ? hits + (size_t)sp->hits_plane * (rows + 2 * ghost) * side + (size_t)ghost * side : nullptr;
  double acc0 = 0.0, acc1 = 0.0;
  for (int pt = threadIdx.x; pt < AP_TY * AP_TX; pt += AP_NT) {
    const int ly = ty0 + pt / AP_TX, gx = tx0 + pt % AP_TX, gyg = row0 + ly;
    if (ly >= rows || gx >= side) continue;
    const int o = (pt / AP_TX + HA) * BW + pt % AP_TX + HA;
    const int deg = degf(gyg, gx);
    const double h = hp ? hp[(size_t)ly * side + gx] : 1.0;
    double xc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) xc[c] = xs[c * PLANE + o];
    double bq[K];
    if (RESID) {
#pragma unroll
      for (int c = 0; c < K; ++c) bq[c] = 0.0;
      const double* yp = Y + (size_t)s * n * N + (nested ? (size_t)nest_of(gx, ly) : (size_t)ly * side + gx);
      if (E) {
        for (int f = 0; f < n; ++f) {
          const double yv = yp[(size_t)f * N];
#pragma unroll
          for (int c = 0; c < K; ++c) bq[c] = fma(yv, Es[f * K + c], bq[c]);
        }
      } else {  // b given (n == K): Y holds b, no N_h factor
#pragma unroll
        for (int c = 0; c < K; ++c) bq[c] = yp[(size_t)c * N];
      }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      double q0;  // (Q0 x)_c without the kappa2 term: (L x) or (D^2 x)
      if (D2) {
        const double* dl = Ds + c * PLANE + o;
        q0 = ((dl[-BW] + dl[BW]) + (dl[-1] + dl[1])) - deg * dl[0];
      } else {
        const double* xl = xs + c * PLANE + o;
        q0 = deg * xl[0] - ((xl[-BW] + xl[BW]) + (xl[-1] + xl[1]));
      }
      double mix = 0.0;
#pragma unroll
      for (int d = 0; d < K; ++d) mix = fma(M[c * K + d], xc[d], mix);
      const double q = fma(h, mix, tau[c] * fma(kappa2, xc[c], q0));
      if (RESID) {
        const double b = E ? h * bq[c] : bq[c];
        const double rres = b - q;
        acc0 = fma(rres, rres, acc0);
        acc1 = fma(b, b, acc1);
      } else {
        y[((size_t)(s * K + c) * rows + ly) * side + gx] = q;
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
// x += alpha_last p for every pixel whose tile's last pass left its x increment pending
// (cg_xpending, KCG_X2); p = the system's current p planes (buffer `parity`, row pitch `pitch`).
// tile_y > 0: the tile CG kernel's per-tile schedule (tiles KCG_TX x tile_y, local rows; KCG_XMIX);
// tile_y = 0: every pixel in class 0 (the row-march kernel's uniform schedule).
template <int K>
__global__ void __launch_bounds__(256) xfix_kernel(const SysState* __restrict__ st, const double* __restrict__ p0,
                                                   const double* __restrict__ p1, double* __restrict__ x, int side,
                                                   int rows, int pitch, int ghost, int tile_y) {
  const int s = blockIdx.y;
  const SysState z = st[s];
  if (!KCG_X2 || z.iters == 0) return;
  const bool pend0 = cg_xpending(z.iters, 0), pend1 = cg_xpending(z.iters, 1);
  if (!pend0 && !(tile_y > 0 && pend1)) return;
  const int tiles_x = (side + KCG_TX - 1) / KCG_TX;
  const double al = z.alpha_last;
  const size_t ps = (size_t)pitch * (rows + 2 * ghost);
  const double* p = (z.parity ? p1 : p0) + (size_t)s * K * ps + (size_t)ghost * pitch;
  const size_t N = (size_t)rows * side;
  double* xs = x + (size_t)s * K * N;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x) {
    const size_t gy = j / side, gx = j - gy * side;
    const int cls = tile_y > 0 ? cg_xclass((int)(gy / tile_y), (int)(gx / KCG_TX), tiles_x) : 0;
    if (!(cls ? pend1 : pend0)) continue;
#pragma unroll
    for (int c = 0; c < K; ++c) xs[c * N + j] = fma(al, p[(size_t)c * ps + gy * pitch + gx], xs[c * N + j]);
  }
}

// --------------------------------------------------------------------------- back-transform
// x[p][c][j] = sum_i W[p][c][i] xt[p][i][j]   (X = Xt W^T), in place.
template <int K>
__global__ void __launch_bounds__(256) backtransform_kernel(const double* __restrict__ W, double* __restrict__ x,
                                                            size_t N) {
  __shared__ double Ws[K * K];
  const int p = blockIdx.y;
  if (threadIdx.x < K * K) Ws[threadIdx.x] = W[(size_t)p * K * K + threadIdx.x];
  __syncthreads();
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

// --------------------------------------------------------------------------- row-slab helpers
// Ghost fill at solve start: this rank's first / last `ghost` rows of r0 and p0 (buffer 0) into the
// up neighbour's bottom ghost rows and the down neighbour's top ghost rows (peer stores).
__global__ void __launch_bounds__(256) ghost_fill_kernel(const double* __restrict__ r0, const double* __restrict__ p0,
                                                         double* up_r, double* up_p, double* dn_r, double* dn_p,
                                                         int planes, int side, int rows, int pitch, int ghost) {
  const size_t ps = (size_t)pitch * (rows + 2 * ghost);
  const int per = ghost * side;  // elements of one plane's ghost band
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < planes * per; e += gridDim.x * blockDim.x) {
    const int pl = e / per, w = e - pl * per, gr = w / side, gx = w - gr * side;
    const size_t base = (size_t)pl * ps + gx;
    if (up_r) {  // my local rows [0, ghost) -> its buffer rows [rows + ghost, rows + 2 ghost)
      const size_t src = base + (size_t)(ghost + gr) * pitch, dst = base + (size_t)(rows + ghost + gr) * pitch;
      up_r[dst] = r0[src];
      up_p[dst] = p0[src];
    }
    if (dn_r) {  // my local rows [rows - ghost, rows) -> its buffer rows [0, ghost)
      const size_t src = base + (size_t)(rows + gr) * pitch, dst = base + (size_t)gr * pitch;
      dn_r[dst] = r0[src];
      dn_p[dst] = p0[src];
    }
  }
}

// x boundary rows for the slab residual: my row 0 -> up neighbour's xg_bot, my row rows-1 -> down
// neighbour's xg_top (both [planes][side]).
__global__ void __launch_bounds__(256) xghost_kernel(const double* __restrict__ x, double* up_xg_bot,
                                                     double* dn_xg_top, int planes, int side, int rows) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < planes * side; e += gridDim.x * blockDim.x) {
    const int pl = e / side, gx = e - pl * side;
    if (up_xg_bot) up_xg_bot[e] = x[((size_t)pl * rows) * side + gx];
    if (dn_xg_top) dn_xg_top[e] = x[((size_t)pl * rows + rows - 1) * side + gx];
  }
}

// dst[g][rank * count + i] = src[i] for every rank g (peer stores of this rank's small results).
__global__ void __launch_bounds__(256) put_kernel(XrankPut P) {
  for (int e = threadIdx.x; e < P.count * P.nranks; e += blockDim.x) {
    const int g = e / P.count, i = e - g * P.count;
    P.dst[g][(size_t)P.rank * P.count + i] = P.src[i];
  }
}

// Cross-rank rendezvous of the local ranks [rank0, rank0 + nlocal) on `tag` (one thread): every
// local rank publishes the tag on every rank, then waits for every rank's tag.
__global__ void xrank_sync_kernel(XrankSync X) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int j = 0; j < X.nlocal; ++j)
    for (int q = 0; q < X.nranks; ++q) st_relaxed_sys_u64(X.flags[q] + X.rank0 + j, X.tag);
  const long long t0 = clock64();
  for (int j = 0; j < X.nlocal; ++j)
    for (int q = 0; q < X.nranks; ++q)
      while (ld_relaxed_sys_u64(X.flags[X.rank0 + j] + q) < X.tag)
        if (clock64() - t0 > (1LL << 34)) __trap();
  __threadfence_system();
}

// --------------------------------------------------------------------------- NESTED permutation
__global__ void __launch_bounds__(256) permute_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                      size_t planes, int side, int to_nested) {
  const size_t N = (size_t)side * side;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < planes * N; e += (size_t)gridDim.x * blockDim.x) {
    const size_t pl = e / N, j = e - pl * N;
    const size_t jn = nest_of((uint32_t)(j % side), (uint32_t)(j / side));
    if (to_nested) dst[pl * N + jn] = src[e];
    else dst[e] = src[pl * N + jn];
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
                       double* p0, double* x, int P, int n, const SlabGeom& g) {
  const size_t N = (size_t)g.rows * g.side;
  dim3 gr(grid_for(N), P);
  const size_t sm = (size_t)n * K * sizeof(double);
  KCG_DISPATCH(K, (rhs_kernel<KK><<<gr, 256, sm, s>>>(Y, E, hits, r0, p0, x, n, g.side, g.rows, g.pitch, g.ghost,
                                                     g.hits_ghost, g.nested)));
  return cudaGetLastError();
}

cudaError_t cg_kernel_config(int K, bool hits, bool prec, bool slab, bool d2, int n_sys, int* max_grid,
                             size_t* smem) {
  KCG_DISPATCH(K, return CgEntry<KK>::config(hits, prec, slab, d2, n_sys, max_grid, smem));
  return cudaErrorInvalidValue;
}

cudaError_t launch_cg(int K, bool prec, bool d2, cudaStream_t s, const CgArgs& a, const CgMaps& m, int grid,
                      size_t smem) {
  KCG_DISPATCH(K, return CgEntry<KK>::launch(prec, d2, s, a, m, grid, smem));
  return cudaErrorInvalidValue;
}

cudaError_t launch_cg_slab(int K, bool prec, cudaStream_t s, const CgSlabLaunch& L, size_t smem) {
  KCG_DISPATCH(K, return CgEntry<KK>::launch_slab(prec, s, L, smem));
  return cudaErrorInvalidValue;
}

template <int K, bool R, bool D2>
static cudaError_t apply_t(cudaStream_t s, const SysParams* params, const double* x, double* y, const double* Y,
                           const double* E, const double* hits, double* partials, int n_sys, int n, const SlabGeom& g,
                           const double* xg_top, const double* xg_bot) {
  constexpr int HA = D2 ? 2 : 1;
  const size_t plane = (size_t)(AP_TX + 2 * HA) * (ap_ty(D2) + 2 * HA);
  const size_t sm = ((D2 ? 2 : 1) * (size_t)K * plane + (R ? (size_t)n * K : 0)) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(apply_kernel<K, R, D2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  dim3 gr(apply_tiles_per_sys(g.rows, g.side, D2), n_sys);
  apply_kernel<K, R, D2><<<gr, AP_NT, sm, s>>>(params, x, y, Y, E, hits, partials, n, g.side, g.rows, g.row0,
                                               g.hits_ghost, g.nested, xg_top, xg_bot);
  return cudaGetLastError();
}

cudaError_t launch_apply(int K, cudaStream_t s, const SysParams* params, const double* x, double* y,
                         const double* hits, int n_sys, const SlabGeom& g, const double* xg_top,
                         const double* xg_bot) {
  if (g.d2) { KCG_DISPATCH(K, return (apply_t<KK, false, true>(s, params, x, y, nullptr, nullptr, hits, nullptr, n_sys, 0, g, xg_top, xg_bot))); }
  KCG_DISPATCH(K, return (apply_t<KK, false, false>(s, params, x, y, nullptr, nullptr, hits, nullptr, n_sys, 0, g,
                                                    xg_top, xg_bot)));
  return cudaErrorInvalidValue;
}

cudaError_t launch_resid(int K, cudaStream_t s, const SysParams* params, const double* x, const double* Y,
                         const double* E, const double* hits, double* partials, double* out, int n_sys, int n,
                         const SlabGeom& g, const double* xg_top, const double* xg_bot) {
  cudaError_t e = cudaSuccess;
  if (g.d2) { KCG_DISPATCH(K, e = (apply_t<KK, true, true>(s, params, x, nullptr, Y, E, hits, partials, n_sys, n, g, xg_top, xg_bot))); }
  else { KCG_DISPATCH(K, e = (apply_t<KK, true, false>(s, params, x, nullptr, Y, E, hits, partials, n_sys, n, g, xg_top, xg_bot))); }
  if (e != cudaSuccess) return e;
  reduce_pairs_kernel<<<n_sys, 256, 0, s>>>(partials, out, apply_tiles_per_sys(g.rows, g.side, g.d2));
  return cudaGetLastError();
}

// r[plane][y pitch + x] -= v[plane][y side + x] (warm start: r_0 = b - G x_0 in the pitched r buffer)
__global__ void __launch_bounds__(256) sub_pitched_kernel(double* __restrict__ r, const double* __restrict__ v,
                                                          size_t planes, int side, int pitch) {
  const size_t N = (size_t)side * side, tot = planes * N;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const size_t pl = e / N, j = e - pl * N, y = j / side, x = j - y * side;
    r[pl * pitch * side + y * pitch + x] -= v[e];
  }
}

cudaError_t launch_sub_pitched(cudaStream_t s, double* r, const double* v, size_t planes, int side, int pitch) {
  sub_pitched_kernel<<<grid_for(planes * (size_t)side * side), 256, 0, s>>>(r, v, planes, side, pitch);
  return cudaGetLastError();
}

cudaError_t launch_xfix(int K, int tile_y, cudaStream_t s, const SysState* st, const double* p0, const double* p1,
                        double* x, int n_sys, const SlabGeom& g) {
  const size_t N = (size_t)g.rows * g.side;
  dim3 gr(grid_for(N), n_sys);
  KCG_DISPATCH(K, (xfix_kernel<KK><<<gr, 256, 0, s>>>(st, p0, p1, x, g.side, g.rows, g.pitch, g.ghost, tile_y)));
  return cudaGetLastError();
}

cudaError_t launch_backtransform(int K, cudaStream_t s, const double* W, double* x, int P, size_t N) {
  dim3 gr(grid_for(N), P);
  KCG_DISPATCH(K, (backtransform_kernel<KK><<<gr, 256, 0, s>>>(W, x, N)));
  return cudaGetLastError();
}

cudaError_t launch_ghost_fill(cudaStream_t s, const double* r0, const double* p0, double* up_r, double* up_p,
                              double* dn_r, double* dn_p, int planes, const SlabGeom& g) {
  const int n = planes * g.ghost * g.side;
  ghost_fill_kernel<<<std::max(1, std::min((n + 255) / 256, 148 * 4)), 256, 0, s>>>(r0, p0, up_r, up_p, dn_r, dn_p,
                                                                                    planes, g.side, g.rows, g.pitch,
                                                                                    g.ghost);
  return cudaGetLastError();
}

cudaError_t launch_xghost(cudaStream_t s, const double* x, double* up_xg_bot, double* dn_xg_top, int planes,
                          const SlabGeom& g) {
  const int n = planes * g.side;
  xghost_kernel<<<std::max(1, std::min((n + 255) / 256, 148 * 4)), 256, 0, s>>>(x, up_xg_bot, dn_xg_top, planes,
                                                                                g.side, g.rows);
  return cudaGetLastError();
}

cudaError_t launch_put(cudaStream_t s, const XrankPut& P) {
  put_kernel<<<1, 256, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_xrank_sync(cudaStream_t s, const XrankSync& X) {
  xrank_sync_kernel<<<1, 32, 0, s>>>(X);
  return cudaGetLastError();
}

}  // namespace kcg

namespace kcg {
cudaError_t launch_permute(cudaStream_t s, const double* src, double* dst, size_t planes, int side, bool to_nested) {
  const size_t n = planes * (size_t)side * side;
  permute_kernel<<<(unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 148 * 8)), 256, 0, s>>>(
      src, dst, planes, side, to_nested ? 1 : 0);
  return cudaGetLastError();
}
// ------------------------------------------------------------------ posterior variances (NEXT-3)
// SplitMix64 (Steele, Lea & Flood 2014; Vigna's reference constants): the counter-based generator
// of the Hutchinson probes (the header documents the key; the CPU reference implements it too).
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) probe_kernel(double* __restrict__ z, int P, int K, int side, int nested,
                                                    unsigned long long seed, int probe) {
  const size_t N = (size_t)side * side, tot = (size_t)P * K * N;
  const unsigned long long s0 = splitmix64(seed);
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const size_t pc = e / N, px = e - pc * N;  // pc = p K + c
    const size_t gy = px / side, gx = px - gy * side;
    const size_t j = nested ? (size_t)nest_of((uint32_t)gx, (uint32_t)gy) : px;
    const unsigned long long key = ((unsigned long long)probe * P * K + pc) * N + j;
    z[e] = (splitmix64(s0 + key) >> 63) ? -1.0 : 1.0;
  }
}

__global__ void __launch_bounds__(256) var_accum_kernel(const double* __restrict__ z, const double* __restrict__ x,
                                                        double* __restrict__ var, size_t n, int first, double scale) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const double v = first ? z[e] * x[e] : fma(z[e], x[e], var[e]);
    var[e] = v * scale;
  }
}

cudaError_t launch_probe(cudaStream_t s, double* z, int P, int K, int side, bool nested, unsigned long long seed,
                         int probe) {
  probe_kernel<<<grid_for((size_t)P * K * side * side), 256, 0, s>>>(z, P, K, side, nested ? 1 : 0, seed, probe);
  return cudaGetLastError();
}

cudaError_t launch_var_accum(cudaStream_t s, const double* z, const double* x, double* var, size_t n, bool first,
                             double scale) {
  var_accum_kernel<<<grid_for(n), 256, 0, s>>>(z, x, var, n, first ? 1 : 0, scale);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Alg. Kohler (NEXT-4)
// Column i of every patch: b = h (Y E[:, i] - sum_{k<i} R[k][i] Xh_k) into r0 plane p (internal
// pitch), p0 = 0, x = 0.  E = T A P^{-1} W (F^ = Y^ W), R the upper-triangular Schur factor, Xh the
// columns solved so far ([P][K][N], working row-major layout), Y in the user layout (NESTED gather).
template <int K>
__global__ void __launch_bounds__(256) kohler_rhs_kernel(const double* __restrict__ Y, const double* __restrict__ E,
                                                         const double* __restrict__ Rk, const double* __restrict__ Xh,
                                                         const double* __restrict__ hits, double* __restrict__ r0,
                                                         double* __restrict__ p0, double* __restrict__ x, int n, int i,
                                                         int side, int pitch, int nested) {
  __shared__ double Ec[64], Rc[KCG_KMAX];
  const int p = blockIdx.y;
  for (int f = threadIdx.x; f < n; f += blockDim.x) Ec[f] = E[((size_t)p * n + f) * K + i];
  if (threadIdx.x < K) Rc[threadIdx.x] = Rk[((size_t)p * K + threadIdx.x) * K + i];
  __syncthreads();
  const size_t N = (size_t)side * side;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x) {
    const size_t gy = j / side, gx = j - gy * side;
    const size_t jy = nested ? nest_of((uint32_t)gx, (uint32_t)gy) : j;
    const double* yp = Y + (size_t)p * n * N + jy;
    double f = 0.0;
    for (int q = 0; q < n; ++q) f = fma(__ldg(yp + (size_t)q * N), Ec[q], f);
    for (int k = 0; k < i; ++k) f = fma(-Rc[k], Xh[((size_t)p * K + k) * N + j], f);
    const double h = hits ? __ldg(hits + (size_t)p * N + j) : 1.0;
    r0[(size_t)p * pitch * side + gy * pitch + gx] = h * f;
    p0[(size_t)p * pitch * side + gy * pitch + gx] = 0.0;
    x[(size_t)p * N + j] = 0.0;
  }
}

// dst[p][K][N] plane i <- src[p][N]
__global__ void __launch_bounds__(256) column_copy_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                          int K, int i, size_t N) {
  const int p = blockIdx.y;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (size_t)gridDim.x * blockDim.x)
    dst[((size_t)p * K + i) * N + j] = src[(size_t)p * N + j];
}

cudaError_t launch_kohler_rhs(int K, cudaStream_t s, const double* Y, const double* E, const double* Rk,
                              const double* Xh, const double* hits, double* r0, double* p0, double* x, int P, int n,
                              int i, int side, int pitch, bool nested) {
  const size_t N = (size_t)side * side;
  dim3 gr(grid_for(N), P);
  KCG_DISPATCH(K, (kohler_rhs_kernel<KK><<<gr, 256, 0, s>>>(Y, E, Rk, Xh, hits, r0, p0, x, n, i, side, pitch,
                                                            nested ? 1 : 0)));
  return cudaGetLastError();
}

cudaError_t launch_column_copy(cudaStream_t s, const double* src, double* dst, int P, int K, int i, size_t N) {
  column_copy_kernel<<<dim3(grid_for(N), P), 256, 0, s>>>(src, dst, K, i, N);
  return cudaGetLastError();
}



// --------------------------------------------------------------------------- argument checks
// Count of entries that are not finite and > 0 (hit counts must be positive): one atomic
// per block, launched once at create.
__global__ void __launch_bounds__(256) count_nonpositive_kernel(const double* __restrict__ v, size_t n,
                                                                unsigned* __restrict__ bad) {
  unsigned c = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double h = __ldg(v + i);
    c += (h > 0.0 && isfinite(h)) ? 0u : 1u;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, c);
}

cudaError_t launch_count_nonpositive(cudaStream_t s, const double* v, size_t n, unsigned* bad) {
  const int grid = (int)std::min<size_t>((n + 255) / 256, 1184);
  count_nonpositive_kernel<<<std::max(grid, 1), 256, 0, s>>>(v, n, bad);
  return cudaGetLastError();
}

}  // namespace kcg
