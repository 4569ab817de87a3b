#pragma once
// sm_100a fp64: the single-pass CG iteration for the paper's own prior Q0 = D^2 + kappa2 I
// (reading R3 "d2"; Alg.MatvecD P:L128-138 applied twice) as a ROW MARCH in registers.
//
// Why not the CTA tiles of the Laplacian kernel: with a radius-2 operator the single-pass recompute
// needs p on the tile + 4 rings, so a 64 x 8 tile staged a 72 x 16 box (2.25x) and evaluated five
// shared-memory stencil phases over it -- the round-1 kernel was shared-memory-wavefront and barrier
// bound (ncu: smem pipe ~58% busy, issue active 25%, 0.22 of HBM).  Here:
//
//   * a GROUP of K warps owns a strip of 24 output columns (lane l = box column x0 - 4 + l, 4-column
//     halo each side), warp c of the group component plane c, and marches DOWN a segment of rows;
//     everything a pixel needs from its vertical neighbours sits in small per-lane register rings
//     (3 rows per quantity), its horizontal neighbours come from the adjacent lanes by shuffles --
//     no shared-memory stencil at all; the planes meet only in the k x k mixing, through 4-row
//     shared rings of p_new / r_new (/ u_new) and one named barrier of the group per row, no CTA
//     barrier inside a pass (one plane per warp: ~60 registers, 16 warps per SM);
//   * the rows of r, p (and x on x passes, hits with N_h) are staged by TMA one row (32 columns x K
//     planes) per stage into a per-group ring of m_stages(K, HITS) shared-memory stages (own mbarriers),
//     prefetched continuously across the warp's units (zero fill outside the face = the free
//     boundary); a stage is held until its r feeds r_old two rows later;
//   * per input row y the warp evaluates, pipelined by one row per phase,
//         A   p_new(y)   = u(y) + beta p(y)          (u = r, or K^{-1} r with block-Jacobi)
//         B0  S1(y-1)    = D p_new                   (0 outside the face)
//         B1  r_new(y-2) = r - alpha (h M p_new + tau (kappa2 p_new + D S1))
//         C0  S2(y-3)    = D u_new                   (u_new = r_new, or K^{-1} r_new)
//         C1  w(y-4)     = h M u_new + tau (kappa2 u_new + D S2);  (r,r), (r,u), (w,u)
//     p_new, x (+= alpha_prev p_old + alpha p_new on x passes) and r_new are final when computed and
//     are stored at once (valid columns / segment rows only);
//   * work unit = (system, strip, segment of `seg` rows, re-planned every pass from the number of
//     systems still running), claimed dynamically per warp group; the segment
//     starts 4 rows early (warm-up: the halo rows are recomputed -- bitwise identical to the
//     neighbouring unit's values, so the iterate does not depend on the decomposition);
//   * partials per (system, strip, 16-row block, plane): the reduction order is fixed by the face
//     geometry, independent of the segment length, the grid and the batch composition.
//   * block-Jacobi: u = K^{-1} r mixes the planes too -- A reads every plane of r from the stage;
//     u_new is formed one row later from the shared r_new ring (C0 / C1 one row further behind).
// Global traffic per pass = the Laplacian kernel's (r, p read + written, x every other pass) plus
// the re-read halo columns (L2) and 8 warm-up rows per segment.
// Edge cases: faces narrower than a strip (one strip, masked lanes), level 0 (deg 0), x / hits
// without a TMA descriptor (side 1: direct loads).

namespace kcg {

__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int K, bool HITS, bool PREC>
__global__ void __launch_bounds__(m_threads(K, HITS), 1) cg_march_kernel(const CgArgs a, const __grid_constant__ CgMaps maps) {
  constexpr int NG = m_groups(K, HITS), NT = m_threads(K, HITS), NW = NT / 32, NS = m_stages(K, HITS), SD = m_stage_doubles(K);
  constexpr int KP = m_kp(K, HITS), GW = m_gw(K, HITS), CP = m_cp(K);  // planes per warp, warps per group, columns per lane
  constexpr int BW = 32 * CP;                                 // box width (one stage row of a plane)
  constexpr int XR = 4 * K * BW, GD = m_group_doubles(K, PREC, HITS);
  constexpr int MO = m_out(K), MH = KCG_MHALO, PB = KCG_MPB;
  constexpr int NP = PREC ? 3 : 2;
  constexpr int DL = PREC ? 5 : 4;  // row of C1 behind the input row
  constexpr int MSZ = K * K + K + (PREC ? 4 * K * K : 0);
  constexpr unsigned FULL = 0xffffffffu;
  static_assert((NS & (NS - 1)) == 0 && NS >= 4 && KCG_MCH == 1 && (GW == 1 || NG <= 15) && GW * KP == K, "geometry");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  SysState* st = reinterpret_cast<SysState*>(smem_raw + (size_t)NG * GD * 8);
  int* act = reinterpret_cast<int*>(st + a.n_sys);
  __shared__ __align__(8) uint64_t mbar[NG][NS];
  __shared__ double rs[KCG_RB][3][NW];
  __shared__ double Mw[NW][MSZ];  // per-warp constants of the system being marched
  __shared__ int uq[NG][4];       // units claimed by each group's issuing warp, in order
  __shared__ int s_nact, s_seg;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp / GW, wg = warp - g * GW, c0 = wg * KP;  // group, warp in the group, its first plane
  const bool issuer = wg == 0;                                 // the group's TMA / claim warp
  const int cta = blockIdx.x, ncta = gridDim.x;
  const int side = a.side, pitch = a.pitch;
  const int nstrips = a.tiles_x, tps = a.tiles_per_sys;
  int seg = a.seg, nsegs = 1, ups = 1;  // rows per unit (planned per pass), segments and units per system
  const size_t N = (size_t)side * side, ps = (size_t)pitch * side;
  double* gsm = reinterpret_cast<double*>(smem_raw) + (size_t)g * GD;
  double* stg = gsm;                 // [NS][SD]: r [K][BW], p [K][BW], x [K][BW], hits [BW]
  double* PX = gsm + NS * SD;        // [4][K][BW] p_new rows
  double* RX = PX + XR;              // [4][K][BW] r_new rows
  double* UX = RX + XR;              // [4][K][BW] u_new rows (block-Jacobi)
  auto gsync = [&]() {
    if constexpr (GW == 1) __syncwarp();
    else group_bar(1 + g, GW * 32);
  };

  if (tid == 0) {  // the launch must provide the dynamic shared memory this layout assumes
    unsigned dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if ((size_t)dyn < (size_t)NG * GD * 8 + (size_t)a.n_sys * (sizeof(SysState) + sizeof(int))) __trap();
  }
  for (int s = tid; s < a.n_sys; s += NT) {
    SysState z;
    z.bnorm2 = 0.0; z.gamma = 0.0; z.alpha = 0.0; z.beta = 0.0; z.rel = 1.0;
    z.iters = 0; z.status = ST_RUNNING; z.parity = 0; z.pad = 0; z.alpha_last = 0.0;
    st[s] = z;
  }
  if (tid == 0) {
    for (int w = 0; w < NG; ++w)
      for (int i = 0; i < NS; ++i) mbar_init(&mbar[w][i], 1);
    fence_mbar_init();
  }
  // r_old of a unit's first two rows reads stages of the previous unit (masked): keep them finite
  for (int e = tid; e < NG * GD; e += NT) reinterpret_cast<double*>(smem_raw)[e] = 0.0;
  __syncthreads();

  auto xpass_of = [](int q) { return KCG_X2 ? (q >= 2 && (q & 1) == 0) : (q >= 1); };
  struct Unit { int s, x0, ys, ye, nsteps, par, hpl; };
  auto unit_of = [&](int u) {  // a unit's geometry from its index in the pass's active-unit list
    Unit U;
    const int i = u / ups, rem = u - i * ups, sg = rem / nstrips;
    U.s = act[i];
    U.x0 = (rem - sg * nstrips) * MO;
    U.ys = sg * seg;
    U.ye = min(side, U.ys + seg);
    U.nsteps = (U.ye - U.ys + MH + DL + 2) / 3 * 3;  // rows ys-4 .. >= ye-1+DL, a multiple of the ring period
    U.par = st[U.s].parity;
    U.hpl = HITS ? (int)__ldg(&a.params[U.s].hits_plane) : 0;
    return U;
  };

  // per-group stage sequence numbers (uniform in the group): issued / waited for / freed
  uint32_t gi = 0, gr = 0, gf = 0;
  int it = -1;
  unsigned gepoch = 0;
  while (true) {
    if (tid == 0) {
      int n = 0;
      for (int s = 0; s < a.n_sys; ++s)
        if (st[s].status == ST_RUNNING) act[n++] = s;
      s_nact = n;
      // the partials are per 16-row block, so the segment length never changes the iterate
      s_seg = a.seg > 0 ? a.seg : (int)a.seg_tab[min(n, KCG_MSEGTAB) - 1];
    }
    __syncthreads();
    const int nact = s_nact;
    if (nact == 0) break;
    seg = s_seg;  // (nact > 0 here, so the table index is valid)
    nsegs = (side + seg - 1) / seg;
    ups = nstrips * nsegs;
    const int units = nact * ups;
    const int par_out = (it + 1) & 1;
    const bool xpass = xpass_of(it + 1);
    const bool xl = xpass && a.x_tma;  // x rows staged with r and p
    const bool hl = HITS && a.h_tma;
    const uint32_t tx_bytes = (2 * K + (xl ? K : 0) + (hl ? 1 : 0)) * BW * 8;
    unsigned* ctr = a.sync + 2 + par_out;
    const int ngt = ncta * NG;

    // ---- the group's row stream (issuing warp only): unit iu, next row ic; claims published in uq
    int iu = cta * NG + g, ic = 0, kq = 0;
    Unit I{};
    if (issuer && iu < units) I = unit_of(iu);
    auto advance_issue = [&]() {
      if (iu >= units) return;
      if (ic == I.nsteps) {  // the issuing unit is exhausted: claim the next one
        unsigned cl = 0;
        if (lane == 0) cl = atomicAdd(ctr, 1u);
        iu = ngt + (int)__shfl_sync(FULL, cl, 0);
        ic = 0;
        ++kq;
        if (lane == 0) uq[g][kq & 3] = iu;
        if (iu >= units) return;
        I = unit_of(iu);
      }
      if (lane == 0) {
        const int slot = gi & (NS - 1);
        double* d = stg + slot * SD;
        uint64_t* bar = &mbar[g][slot];
        const int r0 = I.ys - MH + ic, c0 = I.x0 - MH;
        mbar_arrive_expect_tx(bar, tx_bytes);
        tma_load_3d(d, &maps.r[I.par], bar, c0, r0, I.s * K);
        tma_load_3d(d + K * BW, &maps.p[I.par], bar, c0, r0, I.s * K);
        if (xl) tma_load_3d(d + 2 * K * BW, &maps.x, bar, c0, r0, I.s * K);
        if (hl) tma_load_3d(d + 3 * K * BW, &maps.h, bar, c0, r0, I.hpl);
      }
      ++ic;
      ++gi;
    };
    if (issuer) {
      // generic-proxy writes to the stages (the zero fill at kernel start) before the async-proxy
      // TMA writes; afterwards the stages are only read by the generic proxy, and a stage is
      // refilled after the group barrier that follows its last reads (WAR: no proxy fence needed)
      if (lane == 0) fence_proxy_async_smem();
      for (int j = 0; j < NS; ++j) advance_issue();
    }

    int cu = cta * NG + g, ku = 0;
    while (cu < units) {
      const Unit C = unit_of(cu);
      const SysParams* sp = a.params + C.s;
      __syncwarp();
      for (int e = lane; e < MSZ; e += 32)
        Mw[warp][e] = e < K * K ? __ldg(&sp->M[e]) : (e < K * K + K ? __ldg(&sp->tau[e - K * K]) : __ldg(&sp->Kinv[0][0] + (e - K * K - K)));
      __syncwarp();
      double Mrow[KP][K], tau_c[KP];  // rows c0 .. c0+KP-1 of M, their prior scales
#pragma unroll
      for (int i = 0; i < KP; ++i) {
#pragma unroll
        for (int d = 0; d < K; ++d) Mrow[i][d] = Mw[warp][(c0 + i) * K + d];
        tau_c[i] = Mw[warp][K * K + c0 + i];
      }
      const SysState z = st[C.s];
      const double alpha = z.alpha, beta = z.beta, ap = KCG_X2 ? z.alpha_last : 0.0;
      const double kappa2 = __ldg(&sp->kappa2);
      const double* hp = HITS ? a.hits + (size_t)C.hpl * N : nullptr;
      // this lane's CP face columns gx + cc (CP = 2: a double2 in the stage rows and the stores)
      const int gx = C.x0 - MH + CP * lane;
      bool colin[CP], outc[CP];
      int degx[CP];
#pragma unroll
      for (int cc = 0; cc < CP; ++cc) {
        const int xx = gx + cc, l = CP * lane + cc;
        colin[cc] = xx >= 0 && xx < side;
        outc[cc] = l >= MH && l < MH + MO && xx < side;
        degx[cc] = 4 - (xx == 0) - (xx == side - 1);
      }
      const bool pair_out = CP == 2 && outc[0] && outc[CP - 1];  // both columns stored (aligned double2)
      const size_t pc = ((size_t)C.s * K + c0);  // this warp's first plane
      double* rout = (C.par ? a.rbuf[0] : a.rbuf[1]) + pc * ps + gx;  // select, not a dynamic index
      double* pout = (C.par ? a.pbuf[0] : a.pbuf[1]) + pc * ps + gx;
      double* xo = a.x + pc * N + gx;
      const int strip = C.x0 / MO;
      double* part = a.partials + ((size_t)par_out * a.n_sys + C.s) * tps * NP + ((size_t)strip * GW + wg) * NP;
      // the full K x K block-Jacobi solve of a pixel: every plane of v, planes c0.. of K^{-1} v
      auto prec_w = [&](const double (&v)[K], double h, double dg, double (&uo)[KP]) {
        double u[K];
        double tau[K];
#pragma unroll
        for (int d = 0; d < K; ++d) tau[d] = Mw[warp][K * K + d];
        precond_pixel<K, HITS>(&Mw[warp][K * K + K], &Mw[warp][0], tau, kappa2, h, (int)dg, v, u, true);
#pragma unroll
        for (int i = 0; i < KP; ++i) {
          double ui = u[0];
#pragma unroll
          for (int d = 1; d < K; ++d) ui = d == c0 + i ? u[d] : ui;
          uo[i] = ui;
        }
      };
      // left + right neighbours of this lane's CP columns of a row (shuffles across lanes)
      auto lr = [&](const double (&v)[CP], double (&o)[CP]) {
        if constexpr (CP == 1) {
          o[0] = __shfl_up_sync(FULL, v[0], 1) + __shfl_down_sync(FULL, v[0], 1);
        } else {
          const double L = __shfl_up_sync(FULL, v[CP - 1], 1), R = __shfl_down_sync(FULL, v[0], 1);
          o[0] = L + v[1];
          o[CP - 1] = v[0] + R;
        }
      };
      // row `row` of a shared ring, plane d, this lane's columns
      auto xr = [&](const double* X, int row, int d, int cc) { return X[((row & 3) * K + d) * BW + CP * lane + cc]; };
      auto ld = [&](const double* src, double (&v)[CP]) {  // this lane's columns of a stage / ring row
        if constexpr (CP == 1) v[0] = src[lane];
        else { const double2 t = reinterpret_cast<const double2*>(src)[lane]; v[0] = t.x; v[CP - 1] = t.y; }
      };
      // x is the caller's buffer: double2 stores only if it is 16-byte aligned (r / p: the workspace)
      const bool x16 = (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
      auto stv = [&](double* dst, const double (&v)[CP], bool al = true) {  // this lane's valid columns
        if constexpr (CP == 2) {  // outc[1] implies outc[0] (even halo, even box start): one test per store
          if (pair_out) {
            if (al) *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[CP - 1]);
            else { dst[0] = v[0]; dst[CP - 1] = v[CP - 1]; }
          } else if (outc[0]) dst[0] = v[0];  // (side 1 only)
        } else {
          if (outc[0]) dst[0] = v[0];
        }
      };

      // register rings of this warp's planes and columns (slot of row y = (y - ys + 4) mod 3)
      double pn[3][KP][CP], s1[3][KP][CP], rn[3][KP][CP], s2[3][KP][CP], un[3][KP][CP];
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < KP; ++i)
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) {
            pn[j][i][cc] = 0.0; s1[j][i][cc] = 0.0; rn[j][i][cc] = 0.0; s2[j][i][cc] = 0.0; un[j][i][cc] = 0.0;
          }
      // per-row values of rows y-1 .. y-5, shifted by one every step: in-face row, degree offset, hits
      bool r1 = false, r2 = false, r3 = false, r4 = false, r5 = false;
      int e1 = 0, e2 = 0, e3 = 0, e4 = 0, e5 = 0;  // -(row == 0) - (row == side - 1)
      double h1[CP], h2[CP], h3[CP], h4[CP], h5[CP];
#pragma unroll
      for (int cc = 0; cc < CP; ++cc) { h1[cc] = 1.0; h2[cc] = 1.0; h3[cc] = 1.0; h4[cc] = 1.0; h5[cc] = 1.0; }
      double prr = 0.0, pru = 0.0, pwu = 0.0;  // partials of the current 16-row block
      const uint32_t q0 = gr;                 // the unit's first stage
      auto free_stage = [&]() {               // issuing warp: the oldest held stage is consumed, refill it
        ++gf;
        if (KCG_MFENCE && lane == 0) fence_proxy_async_smem();
        advance_issue();
      };

      // one input row: y = ys - 4 + t, ring period 3 (J = t mod 3 at compile time)
      // IN (KCG_MINT): every row and column the unit touches lies strictly inside the face (degree 4,
      // no border masks); the rows before the warm-up then hold finite values no valid output reads
      auto step = [&](auto Jc, auto INc, int t) {
        constexpr int J = decltype(Jc)::value, J1 = (J + 2) % 3, J2 = (J + 1) % 3;  // rows y-1 | y-4, y-2 | y-5
        constexpr bool IN = decltype(INc)::value;
        auto on = [&](bool row, int cc) { return IN || (row && colin[cc]); };       // pixel inside the face
        auto mdeg = [&](int cc, int e) { return IN ? -4.0 : -(double)(degx[cc] + e); };  // -(degree)
        const int y = C.ys - MH + t;
        const uint32_t q = gr++;
        const int slot = q & (NS - 1);
        mbar_wait(&mbar[g][slot], (q / NS) & 1u);
        const double* sg = stg + slot * SD;
        const double* sg2 = stg + ((q - 2) & (NS - 1)) * SD;  // row y - 2 (held)
        double r_c[KP][CP], p_c[KP][CP], ro_c[KP][CP];
#pragma unroll
        for (int i = 0; i < KP; ++i) {
          ld(sg + (c0 + i) * BW, r_c[i]);
          ld(sg + (K + c0 + i) * BW, p_c[i]);
          ld(sg2 + (c0 + i) * BW, ro_c[i]);
        }
        const bool r0 = IN || (unsigned)y < (unsigned)side;
        const int e0 = IN ? 0 : -(y == 0) - (y == side - 1);
        const bool vA = y >= C.ys && y < C.ye;
        double xv[KP][CP];
#pragma unroll
        for (int i = 0; i < KP; ++i)
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) xv[i][cc] = 0.0;
        if (xpass) {
#pragma unroll
          for (int i = 0; i < KP; ++i) {
            if (xl) ld(sg + (2 * K + c0 + i) * BW, xv[i]);
            else
#pragma unroll
              for (int cc = 0; cc < CP; ++cc)
                xv[i][cc] = (vA && outc[cc]) ? __ldcg(xo + i * N + (size_t)y * side + cc) : 0.0;
          }
        }
        double h0[CP];
#pragma unroll
        for (int cc = 0; cc < CP; ++cc) h0[cc] = 1.0;
        if (HITS) {
          if (hl) ld(sg + 3 * K * BW, h0);
          else
#pragma unroll
            for (int cc = 0; cc < CP; ++cc) h0[cc] = on(r0, cc) ? __ldg(hp + (size_t)y * side + gx + cc) : 1.0;
        }
        // A: p_new(y)
#pragma unroll
        for (int cc = 0; cc < CP; ++cc) {
          double u_c[KP];
#pragma unroll
          for (int i = 0; i < KP; ++i) u_c[i] = r_c[i][cc];
          if (PREC) {
            double rv[K];
#pragma unroll
            for (int d = 0; d < K; ++d) rv[d] = sg[d * BW + CP * lane + cc];
            if (on(r0, cc)) prec_w(rv, h0[cc], -mdeg(cc, e0), u_c);
            else
#pragma unroll
              for (int i = 0; i < KP; ++i) u_c[i] = 0.0;
          }
#pragma unroll
          for (int i = 0; i < KP; ++i) pn[J][i][cc] = fma(beta, p_c[i][cc], u_c[i]);
        }
#pragma unroll
        for (int i = 0; i < KP; ++i) {
          if (GW > 1)
#pragma unroll
            for (int cc = 0; cc < CP; ++cc) PX[((y & 3) * K + c0 + i) * BW + CP * lane + cc] = pn[J][i][cc];
          if (vA) {
            stv(pout + i * ps + (size_t)y * pitch, pn[J][i]);
            if (xpass) {
              double xn[CP];
#pragma unroll
              for (int cc = 0; cc < CP; ++cc) xn[cc] = xv[i][cc] + fma(alpha, pn[J][i][cc], ap * p_c[i][cc]);
              stv(xo + i * N + (size_t)y * side, xn, x16);
            }
          }
        }
        // B0: S1(y-1) = D p_new
#pragma unroll
        for (int i = 0; i < KP; ++i) {
          double o[CP];
          lr(pn[J1][i], o);
#pragma unroll
          for (int cc = 0; cc < CP; ++cc)
            s1[J1][i][cc] = on(r1, cc) ? fma(mdeg(cc, e1), pn[J1][i][cc], (pn[J2][i][cc] + pn[J][i][cc]) + o[cc])
                                                : 0.0;
        }
        // B1: r_new(y-2)
        {
          const int y2 = y - 2;
          const bool st2 = y2 >= C.ys && y2 < C.ye;
#pragma unroll
          for (int i = 0; i < KP; ++i) {
            double o[CP];
            lr(s1[J2][i], o);
#pragma unroll
            for (int cc = 0; cc < CP; ++cc) {
              const double d2p = fma(mdeg(cc, e2), s1[J2][i][cc], (s1[J][i][cc] + s1[J1][i][cc]) + o[cc]);
              double mix = 0.0;
#pragma unroll
              for (int d = 0; d < K; ++d)  // p_new of row y-2, plane d (GW == 1: every plane is this warp's)
                mix = fma(Mrow[i][d], GW == 1 ? pn[J2][GW == 1 ? d : 0][cc] : xr(PX, y2, d, cc), mix);
              const double qv = fma(h2[cc], mix, tau_c[i] * fma(kappa2, pn[J2][i][cc], d2p));
              rn[J2][i][cc] = on(r2, cc) ? fma(-alpha, qv, ro_c[i][cc]) : 0.0;
              if (GW > 1 || PREC) RX[((y2 & 3) * K + c0 + i) * BW + CP * lane + cc] = rn[J2][i][cc];
            }
            if (st2) stv(rout + i * ps + (size_t)y2 * pitch, rn[J2][i]);
          }
        }
        // B' (block-Jacobi): u_new(y-3) = K^{-1} r_new from the shared r_new row
        if (PREC) {
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) {
            double rv[K];
#pragma unroll
            for (int d = 0; d < K; ++d) rv[d] = GW == 1 ? rn[J][GW == 1 ? d : 0][cc] : xr(RX, y - 3, d, cc);
            double uo[KP];
            if (on(r3, cc)) prec_w(rv, h3[cc], -mdeg(cc, e3), uo);
            else
#pragma unroll
              for (int i = 0; i < KP; ++i) uo[i] = 0.0;
#pragma unroll
            for (int i = 0; i < KP; ++i) {
              un[J][i][cc] = uo[i];
              if (GW > 1) UX[(((y - 3) & 3) * K + c0 + i) * BW + CP * lane + cc] = uo[i];
            }
          }
        }
        // C0: S2 = D u_new at row y-3 (u = r_new) or y-4 (block-Jacobi)
#pragma unroll
        for (int i = 0; i < KP; ++i) {
          double o[CP];
          if (!PREC) {
            lr(rn[J][i], o);
#pragma unroll
            for (int cc = 0; cc < CP; ++cc)
              s2[J][i][cc] = on(r3, cc) ? fma(mdeg(cc, e3), rn[J][i][cc], (rn[J1][i][cc] + rn[J2][i][cc]) + o[cc])
                                               : 0.0;
          } else {  // u_new rows: y-3 -> J, y-4 -> J1, y-5 -> J2; S2 row y-4 -> J1
            lr(un[J1][i], o);
#pragma unroll
            for (int cc = 0; cc < CP; ++cc)
              s2[J1][i][cc] = on(r4, cc) ? fma(mdeg(cc, e4), un[J1][i][cc], (un[J2][i][cc] + un[J][i][cc]) + o[cc])
                                                : 0.0;
          }
        }
        // C1: w at row yc = y - DL and the partials
        {
          const int yc = y - DL;
          double lrr = 0.0, lru = 0.0, lwu = 0.0;
#pragma unroll
          for (int i = 0; i < KP; ++i) {
            double o[CP];
            lr(PREC ? s2[J2][i] : s2[J1][i], o);
#pragma unroll
            for (int cc = 0; cc < CP; ++cc) {
              double w, uc, rc;
              double mix = 0.0;
              if (!PREC) {  // S2 rows y-5 (J2), y-4 (J1), y-3 (J); u = r_new row y-4 (J1)
                const double d2v = fma(mdeg(cc, e4), s2[J1][i][cc], (s2[J2][i][cc] + s2[J][i][cc]) + o[cc]);
#pragma unroll
                for (int d = 0; d < K; ++d) mix = fma(Mrow[i][d], GW == 1 ? rn[J1][GW == 1 ? d : 0][cc] : xr(RX, yc, d, cc), mix);
                uc = rn[J1][i][cc];
                rc = uc;
                w = fma(h4[cc], mix, tau_c[i] * fma(kappa2, uc, d2v));
              } else {      // S2 rows y-6 (J), y-5 (J2), y-4 (J1); u_new row y-5 (J2); r_new row y-5 (RX)
                const double d2v = fma(mdeg(cc, e5), s2[J2][i][cc], (s2[J][i][cc] + s2[J1][i][cc]) + o[cc]);
#pragma unroll
                for (int d = 0; d < K; ++d) mix = fma(Mrow[i][d], GW == 1 ? un[J2][GW == 1 ? d : 0][cc] : xr(UX, yc, d, cc), mix);
                uc = un[J2][i][cc];
                rc = xr(RX, yc, c0 + i, cc);
                w = fma(h5[cc], mix, tau_c[i] * fma(kappa2, uc, d2v));
              }
              if (outc[cc]) {
                lrr = fma(rc, rc, lrr);
                if (PREC) lru = fma(rc, uc, lru);
                lwu = fma(w, uc, lwu);
              }
            }
          }
          const bool inc = yc >= C.ys && yc < C.ye;
          if (inc) { prr += lrr; pru += lru; pwu += lwu; }
          // the 16-row block of yc ends (or the segment does): flush this warp's partials
          if (inc && (((yc + 1) % PB) == 0 || yc == C.ye - 1)) {
            const double sr = warp_sum(prr), sw = warp_sum(pwu), su = PREC ? warp_sum(pru) : 0.0;
            if (lane == 0) {
              double* o = part + (size_t)(yc / PB) * nstrips * GW * NP;
              o[0] = sr;
              if (PREC) { o[1] = su; o[2] = sw; }
              else o[1] = sw;
            }
            prr = 0.0; pru = 0.0; pwu = 0.0;
          }
        }
        // shift the per-row values
        r5 = r4; r4 = r3; r3 = r2; r2 = r1; r1 = r0;
        e5 = e4; e4 = e3; e3 = e2; e2 = e1; e1 = e0;
        if (HITS)
#pragma unroll
          for (int cc = 0; cc < CP; ++cc) { h5[cc] = h4[cc]; h4[cc] = h3[cc]; h3[cc] = h2[cc]; h2[cc] = h1[cc]; h1[cc] = h0[cc]; }
        // Group barrier: the shared rows of this step are written, stage y-2 is read by every warp.
        // (A barrier every other step -- enough for the read distances without block-Jacobi --
        // measured 5% slower: the issuing warp then refills two stages at once.)
        gsync();
        if (issuer && q >= q0 + 2) free_stage();
      };
      const bool interior = KCG_MINT && C.x0 - MH >= 1 && C.x0 - MH + BW <= side - 1 && C.ys - MH >= 1 &&
                            C.ys - MH + C.nsteps <= side - 1;
      if (KCG_MINT && interior) {
        for (int t = 0; t < C.nsteps; t += 3) {
          step(std::integral_constant<int, 0>{}, std::true_type{}, t);
          step(std::integral_constant<int, 1>{}, std::true_type{}, t + 1);
          step(std::integral_constant<int, 2>{}, std::true_type{}, t + 2);
        }
      } else {
        for (int t = 0; t < C.nsteps; t += 3) {
          step(std::integral_constant<int, 0>{}, std::false_type{}, t);
          step(std::integral_constant<int, 1>{}, std::false_type{}, t + 1);
          step(std::integral_constant<int, 2>{}, std::false_type{}, t + 2);
        }
      }
      gsync();  // every warp is done with the unit's stages
      if (issuer)
        while (gf < q0 + C.nsteps) free_stage();  // the unit's last held stages
      gsync();  // uq of the next unit is published
      cu = uq[g][++ku & 3];
    }
    __syncwarp();

    iteration_reduce<NT, NP, false>(a, st, act, nact, par_out, it, rs, cta, ncta, gepoch, [&]() {
      if (cta == 0) *ctr = 0u;  // quiescent now; next used two passes later
    });
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

}  // namespace kcg
