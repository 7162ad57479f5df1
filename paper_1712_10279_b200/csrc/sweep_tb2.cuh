// Temporal blocking: two PDHG iterations per HBM pass (SURVEY.md §8(f)
// rank 1).  Same arithmetic as sweep.cuh / sweep_tma.cuh, so the iterates are
// bit-identical to two single sweeps; the intermediate iterate X^{k+1} never
// leaves registers.
//
// Each thread owns one column and walks the CTA's rows with two levels:
//   level A: X^k     -> X^{k+1} at row a      (inputs from the TMA row ring)
//   level B: X^{k+1} -> X^{k+2} at row a - 1  (inputs from A's registers)
// B at row b needs X^{k+1} at rows b and b+1, so it lags A by one row and
// reads A's current outputs for b+1; column neighbours come by warp shuffle.
// All dependencies stay inside a warp: lane 0 only contributes A's flux,
// lane 31 only A's full update, lanes 1..30 B's flux, lanes 2..30 B's
// outputs -- 29 output columns per warp, warps overlap by 3 columns, and no
// barrier is needed anywhere in the row loop.
//
// Rows: outputs [gr0, gr1) need X^{k+1} on [gr0-1, gr1] and A's flux on
// gr0-2, i.e. X^k on rows [gr0-2, gr1+1]:
//   stage q <-> global row gr0 - 2 + q, q = 0 (u, phi), 1 .. R+2 (all),
//   R+3 (phi); stages outside the grid complete with a plain arrive.
#pragma once

#include "sweep_tma.cuh"

namespace otfx {

template <class P, typename T>
struct TB2Shape {
  static constexpr int H = 16 / int(sizeof(T));  // staged columns left of c0 (16 B)
  static constexpr int TILE = 29 * 4;            // output columns per CTA
  // staged columns: c0-H .. c0+117  (lane 31 of warp 3 reads phi at c0+117)
  static constexpr int TW = ((118 + H) + H - 1) / H * H;
  static constexpr int ROW = TW * int(sizeof(T));
  static constexpr int R128(int x) { return (x + 127) / 128 * 128; }
  static constexpr int OFF_W = R128(2 * P::NP * ROW);
  static constexpr int OFF_D = OFF_W + R128((P::NWA > 0 ? P::NWA : 1) * ROW);
  static constexpr int OFF_P = OFF_D + R128(P::NP * ROW);
  static constexpr int BYTES = OFF_P + R128(P::NP * ROW);
};

template <typename T>
__device__ __forceinline__ T shfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T>
__device__ __forceinline__ T shfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <class P, typename T>
__global__ void __launch_bounds__(160, 2) sweep_tb2_kernel(const __grid_constant__ TmaSweepArgs<T> G,
                                                          const __grid_constant__ TmaSet M) {
  using SS = TB2Shape<P, T>;
  constexpr int NP = P::NP;
  constexpr int NWA = P::NWA;
  constexpr int TW = SS::TW;
  const SweepArgs<T>& A = G.s;
  const StageLayout& L = G.L;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [S]
  uint64_t* empty = full + 8;                          // [S]
  unsigned char* stages = smem + 128;

  const int CW = 4;
  const int S = L.S;
  const int t = threadIdx.x;
  const int warp = t >> 5, lane = t & 31;
  const bool producer = warp >= CW;
  const int c0 = blockIdx.x * SS::TILE;
  const int sc = SS::H - 2 + 29 * warp + lane;  // staged column of this thread's column
  const int j = c0 - 2 + 29 * warp + lane;
  const int n = A.n;
  const bool outB = !producer && lane >= 2 && lane <= 30 && j < n;
  const bool hasy = j + 1 < n;
  const int gr0 = A.row_begin + blockIdx.y * A.rows_per_block;
  const int gr1 = min(gr0 + A.rows_per_block, A.row_end);
  const int qmax = gr1 - gr0 + 3;
  auto qrow = [&](int r) { return r - gr0 + 2; };

  if (t == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (producer) {
    if (lane == 0) {
      const int cx = c0 - SS::H;
      for (int q = 0; q <= qmax; ++q) {
        const int slot = q % S;
        if (q >= S) mbar_wait(&empty[slot], ((q / S) - 1) & 1);
        uint64_t* bar = &full[slot];
        const int r = gr0 - 2 + q;
        const int lrow = r - A.row_begin + 1;
        unsigned char* st = stages + slot * SS::BYTES;
        if (r < 0 || r >= n) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
        } else if (q == 0) {
          mbar_expect_tx(bar, L.bytes_flux);
          tma_load_3d(st, &M.u, bar, cx, lrow, 0);
          tma_load_3d(st + SS::OFF_P, &M.phi, bar, cx, lrow, 0);
        } else if (q == qmax) {
          mbar_expect_tx(bar, L.bytes_phi);
          tma_load_3d(st + SS::OFF_P, &M.phi, bar, cx, lrow, 0);
        } else {
          mbar_expect_tx(bar, L.bytes_full);
          tma_load_3d(st, &M.u, bar, cx, lrow, 0);
          if (P::HAS_W) tma_load_3d(st + SS::OFF_W, &M.w, bar, cx, lrow, 0);
          tma_load_3d(st + SS::OFF_D, &M.diff, bar, cx, lrow, 0);
          tma_load_3d(st + SS::OFF_P, &M.phi, bar, cx, lrow, 0);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  HotArgs<P, T> H;
  H.load(A);
  const int nwp = H.ell * P::NWS;
  const int64_t pl = A.plane;
  auto sbase = [&](int q) -> const unsigned char* {
    return stages + (q % S) * SS::BYTES + sc * int(sizeof(T));
  };
  auto wait_q = [&](int q) { mbar_wait(&full[q % S], (q / S) & 1); };
  int rel = 0;  // next stage to release
  auto release_upto = [&](int qlim) {
    while (rel < qlim) {
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[rel % S]))
                     : "memory");
      ++rel;
    }
  };

  // level carries
  T aub_prev[NP];                   // ubar^A_x(a-1)
  T bub_prev[NP];                   // ubar^B_x(b-1)
  T xu[2][NP], xw[NWA], xp[NP];     // X^{k+1}(a-1, j): u, w, phi
#pragma unroll
  for (int c = 0; c < NP; ++c) {
    aub_prev[c] = T(0);
    bub_prev[c] = T(0);
  }

  // A's flux on the halo row gr0-2 (only ubar^A_x is needed)
  if (gr0 - 2 >= 0) {
    wait_q(0);
    wait_q(1);
    const T* sU = reinterpret_cast<const T*>(sbase(0));
    const T* sP = reinterpret_cast<const T*>(sbase(0) + SS::OFF_P);
    const T* sPn = reinterpret_cast<const T*>(sbase(1) + SS::OFF_P);
    T ph[NP], px[NP], py[NP], uo[2][NP], un[2][NP], g[2][NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      ph[c] = sP[c * TW];
      py[c] = sP[c * TW + 1];
      px[c] = sPn[c * TW];
      uo[0][c] = sU[c * TW];
      uo[1][c] = sU[(NP + c) * TW];
    }
    Cell<P, T>::grad(ph, px, py, true, hasy, g, H);
    Cell<P, T>::flux_g(g, uo, un, H);
#pragma unroll
    for (int c = 0; c < NP; ++c) aub_prev[c] = (un[0][c] + un[0][c]) - uo[0][c];
  }
  release_upto(1);

  const int a0 = max(gr0 - 1, 0);
  for (int a = a0; a <= gr1; ++a) {
    const int q = qrow(a);
    T nu_[2][NP], nw_[NWA], np_[NP];  // X^{k+1}(a, j)
    // ---------------------------------------------------------- level A (row a)
    if (a < n) {
      wait_q(q);
      wait_q(q + 1);
      const T* sU = reinterpret_cast<const T*>(sbase(q));
      const T* sW = reinterpret_cast<const T*>(sbase(q) + SS::OFF_W);
      const T* sD = reinterpret_cast<const T*>(sbase(q) + SS::OFF_D);
      const T* sP = reinterpret_cast<const T*>(sbase(q) + SS::OFF_P);
      const T* sPn = reinterpret_cast<const T*>(sbase(q + 1) + SS::OFF_P);
      const bool hasx = a + 1 < n;
      T ph[NP], px[NP], py[NP], uo[2][NP], g[2][NP], ub[2][NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        ph[c] = sP[c * TW];
        py[c] = sP[c * TW + 1];
        px[c] = sPn[c * TW];
        uo[0][c] = sU[c * TW];
        uo[1][c] = sU[(NP + c) * TW];
      }
      Cell<P, T>::grad(ph, px, py, hasx, hasy, g, H);
      Cell<P, T>::flux_g(g, uo, nu_, H);
      T rhs[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        ub[0][c] = (nu_[0][c] + nu_[0][c]) - uo[0][c];
        ub[1][c] = (nu_[1][c] + nu_[1][c]) - uo[1][c];
        const T lub = shfl_up1(ub[1][c]);
        T d = ub[0][c];
        if (a > 0) d = d - aub_prev[c];
        d = d + ub[1][c];
        if (j > 0) d = d - lub;
        d = d * H.inv_dx;
        rhs[c] = d - sD[c * TW];
        aub_prev[c] = ub[0][c];
      }
      if (P::HAS_W) {
        T wo[NWA], gc[NWA], wb[NWA], dv[NP];
#pragma unroll
        for (int e = 0; e < NWA; ++e) wo[e] = e < nwp ? sW[e * TW] : T(0);
        P::grad_c(ph, gc, H);
#pragma unroll
        for (int e = 0; e < NWA; ++e) nw_[e] = gc[e] * H.nu + wo[e];
        P::prox_w(nw_, H);
#pragma unroll
        for (int e = 0; e < NWA; ++e) wb[e] = (nw_[e] + nw_[e]) - wo[e];
        P::div_c(wb, dv, H);
#pragma unroll
        for (int c = 0; c < NP; ++c) rhs[c] = rhs[c] + dv[c];
      }
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        rhs[c] = rhs[c] * H.tau;
        np_[c] = ph[c] + rhs[c];
      }
    } else {
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        np_[c] = T(0);
        nu_[0][c] = nu_[1][c] = T(0);
      }
#pragma unroll
      for (int e = 0; e < NWA; ++e) nw_[e] = T(0);
    }

    // ---------------------------------------------------------- level B (row a-1)
    const int b = a - 1;
    if (b >= max(gr0 - 1, 0)) {
      const bool hasx = b + 1 < n;
      T pr[NP], g[2][NP], un[2][NP], ub[2][NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) pr[c] = shfl_dn1(xp[c]);  // phi^{k+1}(b, j+1)
      Cell<P, T>::grad(xp, np_, pr, hasx, hasy, g, H);
      Cell<P, T>::flux_g(g, xu, un, H);
      T lub[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        ub[0][c] = (un[0][c] + un[0][c]) - xu[0][c];
        ub[1][c] = (un[1][c] + un[1][c]) - xu[1][c];
        lub[c] = shfl_up1(ub[1][c]);
      }
      if (b >= gr0) {
        const T* sD = reinterpret_cast<const T*>(sbase(q - 1) + SS::OFF_D);
        T rhs[NP], wn[NWA];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          T d = ub[0][c];
          if (b > 0) d = d - bub_prev[c];
          d = d + ub[1][c];
          if (j > 0) d = d - lub[c];
          d = d * H.inv_dx;
          rhs[c] = d - sD[c * TW];
        }
        if (P::HAS_W) {
          T gc[NWA], wb[NWA], dv[NP];
          P::grad_c(xp, gc, H);
#pragma unroll
          for (int e = 0; e < NWA; ++e) wn[e] = gc[e] * H.nu + xw[e];
          P::prox_w(wn, H);
#pragma unroll
          for (int e = 0; e < NWA; ++e) wb[e] = (wn[e] + wn[e]) - xw[e];
          P::div_c(wb, dv, H);
#pragma unroll
          for (int c = 0; c < NP; ++c) rhs[c] = rhs[c] + dv[c];
        }
        if (outB) {
          const int64_t o = cell_off(A, b, j);
          T* pu = A.b.u + o;
          T* pp = A.b.phi + o;
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            rhs[c] = rhs[c] * H.tau;
            pu[c * pl] = un[0][c];
            pu[(NP + c) * pl] = un[1][c];
            pp[c * pl] = xp[c] + rhs[c];
          }
          if (P::HAS_W) {
            T* pw = A.b.w + o;
#pragma unroll
            for (int e = 0; e < NWA; ++e)
              if (e < nwp) pw[e * pl] = wn[e];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NP; ++c) bub_prev[c] = ub[0][c];
    }
    // shift X^{k+1}(a) into the carry
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      xu[0][c] = nu_[0][c];
      xu[1][c] = nu_[1][c];
      xp[c] = np_[c];
    }
#pragma unroll
    for (int e = 0; e < NWA; ++e) xw[e] = nw_[e];
    release_upto(q);  // rows < a are done (B(a-1) read its diff above)
  }
  release_upto(qmax + 1);
}

}  // namespace otfx
