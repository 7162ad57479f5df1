// Fused single-pass PDHG iteration ("sweep") and the check-iteration kernels.
//
// One CTA owns a tile of TX columns x rows_per_block rows and walks it top to
// bottom, one row per step, so every word of the state is read once from HBM
// and written once (27 words per cell for 3-channel vector transport, the
// compulsory traffic of S/solver.py:220-240).  Per row step:
//
//   1. prefetch phi(i+1), u(i), w(i), diff(i)               (HBM -> registers)
//   2. u' = prox_u(u + mu grad phi)      (S/solver.py:221-224, S/spatial.py:80-86)
//   3. ubar = 2u' - u                    (:225-226)
//   4. exchange phi(i, j+1) and ubar_y(i, j-1) with the neighbour threads
//      through shared memory (double-buffered, one barrier per row)
//   5. w' = prox_w(w + nu grad_c phi), wbar = 2w' - w        (:230-236)
//   6. phi' = phi + tau (div ubar - diff + div_c wbar)      (:228-229, 237-240)
//
// ubar_x(i-1, j) is carried in registers from the previous step.  The tile's
// first row re-derives u'(r0-1) from the read-only iterate (one halo row per
// tile) and thread 0 re-derives u'(i, c0-1) for the left halo column, so tiles
// are independent and iterates do not depend on the tiling.  State is
// ping-ponged (read A, write B): the kernel never reads what it writes.
//
// The CHECK variant additionally accumulates the fixed-point residual R^k
// (S/solver.py:282-291) from the registers it already holds, so a check
// iteration needs no snapshot copies (the reference copies u, w, phi at
// :306-308).
#pragma once

#include "payload.cuh"

namespace otfx {

template <class P, typename T>
struct Cell {
  static constexpr int NP = P::NP;
  // u' for one cell from phi(i,j), phi(i+1,j), phi(i,j+1) and u(i,j)
  template <class PA>
  __device__ static __forceinline__ void flux(const T (&ph)[NP], const T (&phx)[NP],
                                              const T (&phy)[NP], bool hasx, bool hasy,
                                              const T (&uo)[2][NP], T (&un)[2][NP],
                                              const PA& A) {
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      const T gx = hasx ? (phx[c] - ph[c]) * A.inv_dx : T(0);
      const T gy = hasy ? (phy[c] - ph[c]) * A.inv_dx : T(0);
      un[0][c] = gx * A.mu + uo[0][c];
      un[1][c] = gy * A.mu + uo[1][c];
    }
    P::prox_u(un, A);
  }
  // forward-difference gradient with zero ghost entries (S/spatial.py:80-86)
  template <class PA>
  __device__ static __forceinline__ void grad(const T (&ph)[NP], const T (&phx)[NP],
                                              const T (&phy)[NP], bool hasx, bool hasy,
                                              T (&g)[2][NP], const PA& A) {
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      g[0][c] = hasx ? (phx[c] - ph[c]) * A.inv_dx : T(0);
      g[1][c] = hasy ? (phy[c] - ph[c]) * A.inv_dx : T(0);
    }
  }
  // u' = prox_u(g mu + u)  (S/solver.py:221-224)
  template <class PA>
  __device__ static __forceinline__ void flux_g(const T (&g)[2][NP], const T (&uo)[2][NP],
                                                T (&un)[2][NP], const PA& A) {
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      un[0][c] = g[0][c] * A.mu + uo[0][c];
      un[1][c] = g[1][c] * A.mu + uo[1][c];
    }
    P::prox_u(un, A);
  }
};

template <typename T>
__device__ __forceinline__ int64_t cell_off(const SweepArgs<T>& A, int g, int col) {
  return int64_t(g - A.row_begin + 1) * A.pitch + col;
}

// Scalar / vector payloads with k <= 3 are held to 4 resident CTAs per SM
// (<= 128 registers): small grids run one row per CTA and need every CTA of a
// 256^2 grid (512) resident in one wave.
template <class P, typename T, bool CHECK>
__global__ void __launch_bounds__(128, ((P::NCOEF > 0 || !P::HAS_W) && P::K <= 3) ? 4 : 0)
    sweep_kernel(const __grid_constant__ SweepArgs<T> A) {
  constexpr int NP = P::NP;
  constexpr int NWA = P::NWA;
  constexpr int NARR = CHECK ? 3 : 2;
  const int TX = blockDim.x;
  const int SW = TX + 1;  // smem row width
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sphi = reinterpret_cast<T*>(smem_raw);  // [2][NP][SW]: phi(row, c0 + t), t in [0, TX]
  T* subar = sphi + 2 * NP * SW;             // [2][NP][SW]: ubar_y(row, c0 - 1 + t)
  T* sdu = subar + 2 * NP * SW;              // [2][NP][SW]: du_y(row, c0 - 1 + t) (CHECK)
  double* sred = reinterpret_cast<double*>(
      smem_raw + ((size_t(NARR) * 2 * NP * SW * sizeof(T) + 15) & ~size_t(15)));

  const int t = threadIdx.x;
  const int c0 = blockIdx.x * TX;
  const int j = c0 + t;
  const int n = A.n;
  const bool live = j < n;
  const bool hasy = j + 1 < n;
  const int band = A.band0 + int(blockIdx.y) * A.band_step;
  const int gr0 = A.row_begin + band * A.rows_per_block;
  const int gr1 = min(gr0 + A.rows_per_block, A.row_end);
  const int64_t pl = A.plane;
  const bool halo_l = (t == 0) && (c0 > 0);
  const bool halo_r = (t == TX - 1) && (c0 + TX < n);

  auto S = [&](T* base, int buf, int comp, int idx) -> T& {
    return base[(buf * NP + comp) * SW + idx];
  };

  T phc[NP];        // phi(i, j)
  T uxb_prev[NP];   // ubar_x(i-1, j)
  T dux_prev[NP];   // (CHECK) du_x(i-1, j)
  T hph[NP];        // thread 0: phi(i, c0-1)

  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // SDU, SDW, SDPHI, SCROSS

  // inputs of one row step: phi(i+1), u(i), diff(i), w(i) of this column, and
  // for the edge threads the halo columns (thread 0: phi(i+1, c0-1),
  // u(i, c0-1); thread TX-1: phi(i+1, c0+TX))
  struct RowIn {
    T phn[NP], uo[2][NP], df[NP], wo[NWA], hphn[NP], huo[2][NP], phr[NP];
  };
  auto load_row = [&](int i, RowIn& r) {
    const bool hasx = i + 1 < n;
    const int64_t o = cell_off(A, i, j);
    const int64_t on = cell_off(A, i + 1, j);
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      r.phn[c] = (live && hasx) ? ldg(A.a.phi + c * pl + on) : T(0);
      r.uo[0][c] = live ? ldg(A.a.u + c * pl + o) : T(0);
      r.uo[1][c] = live ? ldg(A.a.u + (NP + c) * pl + o) : T(0);
      r.df[c] = live ? ldg(A.diff + c * pl + o) : T(0);
    }
    if (P::HAS_W) {
#pragma unroll
      for (int e = 0; e < NWA; ++e)
        r.wo[e] = (live && e < A.ell * P::NWS) ? ldg(A.a.w + e * pl + o) : T(0);
    }
    if (halo_l) {
      const int64_t oh = cell_off(A, i, c0 - 1), ohn = cell_off(A, i + 1, c0 - 1);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        r.hphn[c] = hasx ? ldg(A.a.phi + c * pl + ohn) : T(0);
        r.huo[0][c] = ldg(A.a.u + c * pl + oh);
        r.huo[1][c] = ldg(A.a.u + (NP + c) * pl + oh);
      }
    }
    if (halo_r) {
#pragma unroll
      for (int c = 0; c < NP; ++c)
        r.phr[c] = hasx ? ldg(A.a.phi + c * pl + cell_off(A, i + 1, c0 + TX)) : T(0);
    }
  };

  // ---------------------------------------------------------------- prologue
  // Every global load of the tile's first step is issued up front (first
  // row's inputs, phi of rows gr0 and gr0-1, u of row gr0-1): small grids run
  // one row per CTA, where a chain of dependent load rounds is the latency.
  RowIn in;
  pdl_wait();  // the previous sweep has finished reading what this one writes
  pdl_launch_dependents();
  load_row(gr0, in);
  {
    const int64_t o = cell_off(A, gr0, j);
    const int gm = gr0 - 1;
    const int64_t om = cell_off(A, gm, j);
    T pm[NP], uom[2][NP], pmr[NP], phr0[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      phc[c] = live ? ldg(A.a.phi + c * pl + o) : T(0);
      if (halo_r) phr0[c] = ldg(A.a.phi + c * pl + cell_off(A, gr0, c0 + TX));
      if (halo_l) hph[c] = ldg(A.a.phi + c * pl + cell_off(A, gr0, c0 - 1));
      if (gr0 > 0) {
        pm[c] = live ? ldg(A.a.phi + c * pl + om) : T(0);
        if (halo_r) pmr[c] = ldg(A.a.phi + c * pl + cell_off(A, gm, c0 + TX));
        uom[0][c] = live ? ldg(A.a.u + c * pl + om) : T(0);
        uom[1][c] = live ? ldg(A.a.u + (NP + c) * pl + om) : T(0);
      }
    }
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      S(sphi, gr0 & 1, c, t) = phc[c];
      if (halo_r) S(sphi, gr0 & 1, c, TX) = phr0[c];
      uxb_prev[c] = T(0);
      dux_prev[c] = T(0);
    }
    if (gr0 > 0) {
      // halo row gr0-1: recompute u'(gr0-1, j) from the read-only iterate
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        S(sphi, gm & 1, c, t) = pm[c];
        if (halo_r) S(sphi, gm & 1, c, TX) = pmr[c];
      }
      __syncthreads();
      if (live) {
        T un[2][NP], py[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) py[c] = hasy ? S(sphi, gm & 1, c, t + 1) : T(0);
        Cell<P, T>::flux(pm, phc, py, true, hasy, uom, un, A);
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          uxb_prev[c] = (un[0][c] + un[0][c]) - uom[0][c];
          dux_prev[c] = un[0][c] - uom[0][c];
        }
      }
    }
    __syncthreads();
  }

  // ---------------------------------------------------------------- sweep
  for (int i = gr0; i < gr1; ++i) {
    const int b = i & 1, bn = (i + 1) & 1;
    const bool hasx = i + 1 < n;
    const int64_t o = cell_off(A, i, j);
    if (i > gr0) load_row(i, in);
    const T (&phn)[NP] = in.phn;
    const T (&uo)[2][NP] = in.uo;
    const T (&df)[NP] = in.df;
    const T (&wo)[NWA] = in.wo;
    const T (&hphn)[NP] = in.hphn;
    const T (&huo)[2][NP] = in.huo;
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      S(sphi, bn, c, t) = phn[c];
      if (halo_r) S(sphi, bn, c, TX) = in.phr[c];
    }

    // spatial flux of this cell
    T un[2][NP], ub[2][NP];
    {
      T py[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) py[c] = hasy ? S(sphi, b, c, t + 1) : T(0);
      Cell<P, T>::flux(phc, phn, py, hasx, hasy, uo, un, A);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        ub[0][c] = (un[0][c] + un[0][c]) - uo[0][c];
        ub[1][c] = (un[1][c] + un[1][c]) - uo[1][c];
        S(subar, b, c, t + 1) = ub[1][c];
        if (CHECK) S(sdu, b, c, t + 1) = un[1][c] - uo[1][c];
      }
    }
    if (t == 0) {
      if (halo_l) {
        T hun[2][NP];
        Cell<P, T>::flux(hph, hphn, phc, hasx, true, huo, hun, A);
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          S(subar, b, c, 0) = (hun[1][c] + hun[1][c]) - huo[1][c];
          if (CHECK) S(sdu, b, c, 0) = hun[1][c] - huo[1][c];
          hph[c] = hphn[c];
        }
      } else {
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          S(subar, b, c, 0) = T(0);
          if (CHECK) S(sdu, b, c, 0) = T(0);
        }
      }
    }
    __syncthreads();

    if (live) {
      // phi update: rhs = div(ubar) - diff (+ div_c wbar), rhs *= tau, phi + rhs
      T rhs[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        T d = ub[0][c];
        if (i > 0) d = d - uxb_prev[c];
        d = d + ub[1][c];
        if (j > 0) d = d - S(subar, b, c, t);
        d = d * A.inv_dx;
        rhs[c] = d - df[c];
      }
      T wn[NWA];
      T dwv[NWA];
      if (P::HAS_W) {
        T g[NWA];
        P::grad_c(phc, g, A);
#pragma unroll
        for (int e = 0; e < NWA; ++e) wn[e] = g[e] * A.nu + wo[e];
        P::prox_w(wn, A);
        T wb[NWA], dv[NP];
#pragma unroll
        for (int e = 0; e < NWA; ++e) {
          wb[e] = (wn[e] + wn[e]) - wo[e];
          dwv[e] = wn[e] - wo[e];
        }
        P::div_c(wb, dv, A);
#pragma unroll
        for (int c = 0; c < NP; ++c) rhs[c] = rhs[c] + dv[c];
      }
      T phnew[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        rhs[c] = rhs[c] * A.tau;
        phnew[c] = phc[c] + rhs[c];
      }
      // stores (iterate k+1)
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        A.b.u[c * pl + o] = un[0][c];
        A.b.u[(NP + c) * pl + o] = un[1][c];
        A.b.phi[c * pl + o] = phnew[c];
      }
      if (P::HAS_W) {
#pragma unroll
        for (int e = 0; e < NWA; ++e)
          if (e < A.ell * P::NWS) A.b.w[e * pl + o] = wn[e];
      }
      if (CHECK) {
        // R^k terms (S/solver.py:282-291)
        T cross[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const T dx = un[0][c] - uo[0][c];
          const T dy = un[1][c] - uo[1][c];
          acc[0] += P::wp(c) * (double(dx) * double(dx) + double(dy) * double(dy));
          T d = dx;
          if (i > 0) d = d - dux_prev[c];
          d = d + dy;
          if (j > 0) d = d - S(sdu, b, c, t);
          cross[c] = d * A.inv_dx;
          dux_prev[c] = dx;
        }
        if (P::HAS_W) {
          T dv[NP];
          P::div_c(dwv, dv, A);
#pragma unroll
          for (int c = 0; c < NP; ++c) cross[c] = cross[c] + dv[c];
#pragma unroll
          for (int e = 0; e < NWA; ++e) acc[1] += P::ww(e) * double(dwv[e]) * double(dwv[e]);
        }
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const T dp = phnew[c] - phc[c];
          acc[2] += P::wp(c) * double(dp) * double(dp);
          acc[3] += P::wp(c) * double(dp) * double(cross[c]);
        }
      }
    }
    // carry to the next row
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      uxb_prev[c] = ub[0][c];
      phc[c] = phn[c];
    }
  }

  if (CHECK) {
    block_sum<4>(acc, sred);
    if (t == 0) {
      double* dst = A.partials + (size_t(band) * gridDim.x + blockIdx.x) * 10;
#pragma unroll
      for (int s = 0; s < 4; ++s) dst[s] = acc[s];
#pragma unroll
      for (int s = 4; s < 10; ++s) dst[s] = 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// evaluate(): primal, dual, feasibility terms of the current iterate
// (S/solver.py:242-280).  One thread per cell; neighbours come through L1.
// ---------------------------------------------------------------------------
template <class P, typename T>
__global__ void __launch_bounds__(128) evaluate_kernel(const __grid_constant__ SweepArgs<T> A) {
  constexpr int NP = P::NP;
  constexpr int NWA = P::NWA;
  __shared__ double sred[32 * 8];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const int64_t pl = A.plane;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // PU PW SU2 SW2 SCON SPHID PENU PENW
  double mx[2] = {0.0, 0.0};
  for (int i = A.row_begin + blockIdx.y; j < n && i < A.row_end; i += gridDim.y) {
    const int64_t o = cell_off(A, i, j);
    T u[2][NP], ph[NP], df[NP], w[NWA];
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      u[0][c] = ldg(A.a.u + c * pl + o);
      u[1][c] = ldg(A.a.u + (NP + c) * pl + o);
      ph[c] = ldg(A.a.phi + c * pl + o);
      df[c] = ldg(A.diff + c * pl + o);
    }
    if (P::HAS_W) {
#pragma unroll
      for (int e = 0; e < NWA; ++e) w[e] = (e < A.ell * P::NWS) ? ldg(A.a.w + e * pl + o) : T(0);
    }
    s[0] += P::norm_u(u, A.norm_u);
    double su = 0.0;
#pragma unroll
    for (int c = 0; c < NP; ++c)
      su += P::wp(c) * (double(u[0][c]) * double(u[0][c]) + double(u[1][c]) * double(u[1][c]));
    s[2] += su;
    // constraint residual: div u - diff + div_c w
    T con[NP];
    const int64_t oxm = cell_off(A, i - 1, j), oym = o - 1;
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      T d = u[0][c];
      if (i > 0) d = d - ldg(A.a.u + c * pl + oxm);
      d = d + u[1][c];
      if (j > 0) d = d - ldg(A.a.u + (NP + c) * pl + oym);
      con[c] = d * A.inv_dx - df[c];
    }
    if (P::HAS_W) {
      s[1] += P::norm_w(w, A.norm_w);  // inactive channel blocks are zero
      double sw = 0.0;
#pragma unroll
      for (int e = 0; e < NWA; ++e) sw += P::ww(e) * double(w[e]) * double(w[e]);
      s[3] += sw;
      T dv[NP];
      P::div_c(w, dv, A);
#pragma unroll
      for (int c = 0; c < NP; ++c) con[c] = con[c] + dv[c];
    }
    double sc = 0.0, sp = 0.0;
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      sc += P::wp(c) * double(con[c]) * double(con[c]);
      sp += P::wp(c) * double(ph[c]) * double(df[c]);
    }
    s[4] += sc;
    s[5] += sp;
    // dual norms of grad phi and grad_c phi
    T g[2][NP];
    const bool hx = i + 1 < n, hy = j + 1 < n;
    const int64_t oxp = cell_off(A, i + 1, j);
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      g[0][c] = hx ? (ldg(A.a.phi + c * pl + oxp) - ph[c]) * A.inv_dx : T(0);
      g[1][c] = hy ? (ldg(A.a.phi + c * pl + o + 1) - ph[c]) * A.inv_dx : T(0);
    }
    P::dual_u(g, A.norm_u, mx[0], s[6]);
    if (P::HAS_W) {
      T gc[NWA];
      P::grad_c(ph, gc, A);
      P::dual_w(gc, A.norm_w, A.ell, A.alpha, mx[1], s[7]);
    }
  }
  block_sum<8>(s, sred);
  block_max<2>(mx, sred);
  if (threadIdx.x == 0) {
    const size_t bid = size_t(blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
    for (int q = 0; q < 8; ++q) A.partials[bid * 8 + q] = s[q];
    A.maxes[bid * 2] = mx[0];
    A.maxes[bid * 2 + 1] = mx[1];
  }
}

}  // namespace otfx

namespace otfx {

// ---------------------------------------------------------------------------
// residual between two given iterates A.a (k) and A.b (k+1), for the
// standalone residual_Rk helper (S/solver.py:501-526).  Partials go to
// A.partials[block][8] slots 0..3 = |du|^2, |dw|^2, |dphi|^2, <dphi, cross>.
// ---------------------------------------------------------------------------
template <class P, typename T>
__global__ void __launch_bounds__(128) residual_kernel(const __grid_constant__ SweepArgs<T> A) {
  constexpr int NP = P::NP;
  constexpr int NWA = P::NWA;
  __shared__ double sred[32 * 4];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const int64_t pl = A.plane;
  double s[4] = {0, 0, 0, 0};
  for (int i = A.row_begin + blockIdx.y; j < n && i < A.row_end; i += gridDim.y) {
    const int64_t o = cell_off(A, i, j), oxm = cell_off(A, i - 1, j);
    auto du = [&](int comp, int64_t off) { return A.b.u[comp * pl + off] - A.a.u[comp * pl + off]; };
    T cross[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      const T dx = du(c, o), dy = du(NP + c, o);
      s[0] += P::wp(c) * (double(dx) * double(dx) + double(dy) * double(dy));
      T d = dx;
      if (i > 0) d = d - du(c, oxm);
      d = d + dy;
      if (j > 0) d = d - du(NP + c, o - 1);
      cross[c] = d * A.inv_dx;
    }
    if (P::HAS_W) {
      T dw[NWA];
#pragma unroll
      for (int e = 0; e < NWA; ++e)
        dw[e] = (e < A.ell * P::NWS) ? A.b.w[e * pl + o] - A.a.w[e * pl + o] : T(0);
#pragma unroll
      for (int e = 0; e < NWA; ++e) s[1] += P::ww(e) * double(dw[e]) * double(dw[e]);
      T dv[NP];
      P::div_c(dw, dv, A);
#pragma unroll
      for (int c = 0; c < NP; ++c) cross[c] = cross[c] + dv[c];
    }
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      const T dp = A.b.phi[c * pl + o] - A.a.phi[c * pl + o];
      s[2] += P::wp(c) * double(dp) * double(dp);
      s[3] += P::wp(c) * double(dp) * double(cross[c]);
    }
  }
  block_sum<4>(s, sred);
  if (threadIdx.x == 0) {
    const size_t bid = size_t(blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) A.partials[bid * 8 + q] = s[q];
#pragma unroll
    for (int q = 4; q < 8; ++q) A.partials[bid * 8 + q] = 0.0;
    A.maxes[bid * 2] = 0.0;
    A.maxes[bid * 2 + 1] = 0.0;
  }
}

}  // namespace otfx
