// On-chip solve for small grids: the whole PDHG run loop (S/solver.py:294-337)
// in ONE thread-block cluster, the state resident on chip.
//
// Below ~100^2 cells an iteration is a few µs of dependent latency, and the
// streamed sweeps pay a kernel boundary plus L2 round trips per iteration.
// Here the grid's rows are split over the C CTAs of one cluster (C <= 16, one
// row band each) and every thread owns one cell for the whole run: its u, w,
// phi and diff live in registers.  Shared memory only carries what neighbours
// exchange (phi, ubar, and on check iterations du and u').  Per iteration, in
// the reference's order (S/solver.py:220-240):
//
//   phase A  u' = prox_u(u + mu grad phi), ubar = 2u' - u          (own cells)
//            + the row above the band, recomputed from the upper
//              neighbour's published rows (so ubar_x(r0-1) needs no exchange)
//   __syncthreads
//   phase B  w' = prox_w(w + nu grad_c phi); phi' = phi + tau (div ubar - diff
//            + div_c wbar)
//   publish  the band's first phi row to CTA r-1, its last (phi, u) rows to
//            CTA r+1, with st.async into their double-buffered halo slots;
//            each slot's mbarrier counts the bytes (complete_tx)
//
// So the CTAs synchronise point to point with their two neighbours only; the
// ring of two slots covers the write-after-read hazard (a CTA can run at most
// one iteration ahead of a neighbour).  Check iterations add the R^k terms
// (S/solver.py:282-291) from the values at hand, then an evaluate phase
// (S/solver.py:242-280) on the new iterate, a fixed-order cluster reduction
// (CTA 0 sums the CTAs' partials in rank order), the reference's scalar
// algebra (finalize) and the termination test, all on the device: one launch
// per solve, the history written to global memory.  Per-cell arithmetic is the
// sweeps' (same operation order), so iterates are bit-identical to the
// streamed path; only the reduction order of the check scalars differs.
#pragma once

#include <cooperative_groups.h>

#include "sweep_tma.cuh"

namespace otfx {

namespace cg = cooperative_groups;

constexpr int kClusterThreads = 384;  // launch bound: one thread per cell + one halo row

template <typename T>
struct ClusterArgs {
  SweepArgs<T> s;          // s.a = the engine's current iterate (global planes)
  double tol_gap, tol_feas;
  double diff_norm;        // ||diff|| for the feasibility residual
  double mu, nu, tau;      // fp64 step sizes for the R^k algebra
  long long max_iters, check_every;
  int checks;              // 0: max_iters plain iterations, no evaluation
  int ctas;                // cluster size C
  int rows_max;            // rows of the tallest band
  int has_w;
  double* hist;            // [hist_cap][6]: it, primal, dual, gap, feas, R^k
  long long hist_cap;
  long long* result;       // iterations, history points, converged
};

// shared-memory layout (elements of T unless noted), per CTA
template <class P, typename T>
struct ClusterSmem {
  static constexpr int NP = P::NP;
  int rb, n;  // rows_max, n
  __host__ __device__ ClusterSmem(int rows_max, int n_) : rb(rows_max), n(n_) {}
  __host__ __device__ size_t band() const { return size_t(rb) * n; }
  // bands: PHI [NP], UB [2NP], DU [2NP], U1 [2NP]; halo rows UBH [NP], DUH [NP];
  // two slots of { PRVPHI [NP], PRVU [2NP], NXTPHI [NP] } rows
  __host__ __device__ size_t phi() const { return 0; }
  __host__ __device__ size_t ub() const { return NP * band(); }
  __host__ __device__ size_t du() const { return ub() + 2 * NP * band(); }
  __host__ __device__ size_t u1() const { return du() + 2 * NP * band(); }
  __host__ __device__ size_t ubh() const { return u1() + 2 * NP * band(); }
  __host__ __device__ size_t duh() const { return ubh() + size_t(NP) * n; }
  __host__ __device__ size_t slot(int s) const { return duh() + size_t(NP) * n + size_t(s) * 4 * NP * n; }
  __host__ __device__ size_t elems() const { return slot(2); }
  // byte offsets after the element area
  __host__ __device__ size_t off_bar() const { return (elems() * sizeof(T) + 15) & ~size_t(15); }
  __host__ __device__ size_t off_red() const { return off_bar() + 16; }
  __host__ __device__ size_t off_slots() const { return off_red() + 32 * 12 * sizeof(double); }
  __host__ __device__ size_t off_flag() const { return off_slots() + 16 * 14 * sizeof(double); }
  __host__ __device__ size_t bytes() const { return off_flag() + 16; }
};

__host__ __device__ inline int band_begin(int n, int C, int r) {
  const int base = n / C, extra = n % C;
  return r * base + (r < extra ? r : extra);
}

// ---- cluster / async-store primitives --------------------------------------
__device__ __forceinline__ uint32_t cl_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void cl_arm(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cl_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// full cluster barrier with release / acquire (check points only)
__device__ __forceinline__ void cl_sync() {
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// reference scalar algebra of the check (engine.cu finalize, S/solver.py:242-291)
__device__ inline void finalize_dev(const double* raw, bool has_w, double alpha, double eps,
                                    double diff_norm, double mu, double nu, double tau,
                                    double out[5]) {
  double p = raw[R_PU];
  if (has_w) p += alpha * raw[R_PW];
  if (eps > 0) {
    p += eps * raw[R_SU2];
    if (has_w) p += eps * raw[R_SW2];
  }
  const double rawd = -raw[R_SPHID];
  double dual;
  if (eps == 0) {
    double s = dmax(1.0, raw[R_GU]);
    if (has_w) s = dmax(s, raw[R_GW] / alpha);
    dual = rawd / s;
  } else {
    double pen = raw[R_PENU] / (4.0 * eps);
    if (has_w) pen += raw[R_PENW] / (4.0 * eps);
    dual = rawd - pen;
  }
  const double gap = (p - dual) / dmax(p, 1e-30);
  const double feas = sqrt(raw[R_SCON]) / dmax(diff_norm, 2.2250738585072014e-308);
  double r = raw[R_SDU] / mu + raw[R_SDPHI] / tau;
  if (has_w) r += raw[R_SDW] / nu;
  r = r - 2.0 * raw[R_SCROSS];
  out[0] = p;
  out[1] = dual;
  out[2] = gap;
  out[3] = feas;
  out[4] = r;
}

template <class P, typename T>
__global__ void __launch_bounds__(kClusterThreads) cluster_run_kernel(
    const __grid_constant__ ClusterArgs<T> G) {
  constexpr int NP = P::NP;
  constexpr int NWA = P::NWA;
  const SweepArgs<T>& A = G.s;
  const int C = G.ctas;
  const int rank = int(cg::this_cluster().block_rank());
  const int n = A.n;
  const int r0 = band_begin(n, C, rank), r1 = band_begin(n, C, rank + 1);
  const int rows = r1 - r0;
  const bool has_prev = rank > 0, has_next = rank + 1 < C;
  const int t = threadIdx.x;
  const ClusterSmem<P, T> L(G.rows_max, n);
  const int band = G.rows_max * n;

  // thread role: one own cell (li, j), or one cell of the halo row r0-1
  const bool own = t < rows * n;
  const bool halo = !own && t >= band && t < band + n && has_prev;
  const int li = own ? t / n : -1;
  const int j = own ? t - li * n : (halo ? t - band : 0);
  const int i = own ? r0 + li : r0 - 1;
  const bool hasx = i + 1 < n, hasy = j + 1 < n;
  const bool first = own && li == 0, last = own && li == rows - 1;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.off_bar());
  double* sred = reinterpret_cast<double*>(smem_raw + L.off_red());
  double* sslot = reinterpret_cast<double*>(smem_raw + L.off_slots());
  volatile int* sflag = reinterpret_cast<volatile int*>(smem_raw + L.off_flag());
  T* PHI = sm + L.phi();
  T* UB = sm + L.ub();
  T* DU = sm + L.du();
  T* U1 = sm + L.u1();
  T* UBH = sm + L.ubh();
  T* DUH = sm + L.duh();
  // 32-bit index arithmetic: a band is at most a few thousand elements
  auto bandp = [&](T* base, int c, int row, int col) -> T& { return base[c * band + row * n + col]; };
  auto rowp = [&](T* base, int c, int col) -> T& { return base[c * n + col]; };
  // halo slot s: PRVPHI rows [0, NP), PRVU [NP, 3NP), NXTPHI [3NP, 4NP)
  T* const slot0 = sm + L.slot(0);
  T* const slot1 = sm + L.slot(1);
  auto slotp = [&](int s, int r, int col) -> T& { return (s ? slot1 : slot0)[r * n + col]; };
  const uint32_t sbase = uint32_t(__cvta_generic_to_shared(sm));
  const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(bars));
  auto slot_addr = [&](int s, int r, int col) -> uint32_t {
    return sbase + uint32_t((L.slot(s) + size_t(r) * n + col) * sizeof(T));
  };
  // bytes a CTA receives per iteration
  const uint32_t in_bytes = uint32_t(((has_prev ? 3 * NP : 0) + (has_next ? NP : 0)) * n * sizeof(T));

  HotArgs<P, T> H;
  H.load(A);
  const int nwp = H.ell * P::NWS;
  const int64_t pl = A.plane;

  // ---- load: the cell's state into registers
  T u[2][NP], w[NWA], ph[NP], df[NP];
#pragma unroll
  for (int c = 0; c < NP; ++c) {
    u[0][c] = u[1][c] = ph[c] = df[c] = T(0);
  }
#pragma unroll
  for (int e = 0; e < NWA; ++e) w[e] = T(0);
  if (own) {
    const int64_t o = cell_off(A, i, j);
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      u[0][c] = A.a.u[c * pl + o];
      u[1][c] = A.a.u[(NP + c) * pl + o];
      ph[c] = A.a.phi[c * pl + o];
      df[c] = A.diff[c * pl + o];
      bandp(PHI, c, li, j) = ph[c];
      bandp(U1, c, li, j) = u[0][c];
      bandp(U1, NP + c, li, j) = u[1][c];
    }
    if (P::HAS_W) {
#pragma unroll
      for (int e = 0; e < NWA; ++e) w[e] = e < nwp ? A.a.w[e * pl + o] : T(0);
    }
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl_sync();  // every CTA's barriers exist before anyone stores into them

  // publish the boundary rows of the iterate that iteration k reads into the
  // neighbours' slot k & 1 (phi rows: both neighbours; u row: the next CTA)
  const uint32_t prev_rank = uint32_t(rank - 1), next_rank = uint32_t(rank + 1);
  auto publish_phi = [&](int k, const T (&p)[NP]) {
    const int s = k & 1;
    if (first && has_prev) {
      const uint32_t rb = cl_mapa(bar0 + 8 * s, prev_rank);
#pragma unroll
      for (int c = 0; c < NP; ++c) st_async(cl_mapa(slot_addr(s, 3 * NP + c, j), prev_rank), p[c], rb);
    }
    if (last && has_next) {
      const uint32_t rb = cl_mapa(bar0 + 8 * s, next_rank);
#pragma unroll
      for (int c = 0; c < NP; ++c) st_async(cl_mapa(slot_addr(s, c, j), next_rank), p[c], rb);
    }
  };
  auto publish_u = [&](int k, const T (&uu)[2][NP]) {
    if (last && has_next) {
      const int s = k & 1;
      const uint32_t rb = cl_mapa(bar0 + 8 * s, next_rank);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        st_async(cl_mapa(slot_addr(s, NP + c, j), next_rank), uu[0][c], rb);
        st_async(cl_mapa(slot_addr(s, 2 * NP + c, j), next_rank), uu[1][c], rb);
      }
    }
  };
  // arm slot k & 1 for iteration k (one arrival + the expected bytes)
  auto arm = [&](unsigned k) {
    if (t == 0) cl_arm(bar0 + 8 * uint32_t(k & 1), in_bytes);
  };
  auto wait_slot = [&](unsigned k) {
    if (in_bytes) cl_wait(bar0 + 8 * uint32_t(k & 1), uint32_t((k >> 1) & 1));
  };

  arm(0);
  publish_u(0, u);
  publish_phi(0, ph);

  // ---- one PDHG iteration k; CHECK accumulates the R^k terms into acc
  auto iterate = [&](unsigned k, bool check, double (&acc)[4]) {
    const int s = int(k & 1);
    // phase A: spatial flux
    if (own || halo) {
      if (last || halo) wait_slot(k);
      T phx[NP], phy[NP], pc[NP], uo[2][NP], un[2][NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        if (own) {
          pc[c] = ph[c];
          phy[c] = hasy ? bandp(PHI, c, li, j + 1) : T(0);
          phx[c] = hasx ? (li + 1 < rows ? bandp(PHI, c, li + 1, j) : slotp(s, 3 * NP + c, j)) : T(0);
          uo[0][c] = u[0][c];
          uo[1][c] = u[1][c];
        } else {  // halo row r0-1 from the upper neighbour's published rows
          pc[c] = slotp(s, c, j);
          phy[c] = hasy ? slotp(s, c, j + 1) : T(0);
          phx[c] = bandp(PHI, c, 0, j);
          uo[0][c] = slotp(s, NP + c, j);
          uo[1][c] = slotp(s, 2 * NP + c, j);
        }
      }
      Cell<P, T>::flux(pc, phx, phy, hasx, hasy, uo, un, H);
      if (own) {
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          bandp(UB, c, li, j) = (un[0][c] + un[0][c]) - uo[0][c];
          bandp(UB, NP + c, li, j) = (un[1][c] + un[1][c]) - uo[1][c];
          if (check) {
            bandp(DU, c, li, j) = un[0][c] - uo[0][c];
            bandp(DU, NP + c, li, j) = un[1][c] - uo[1][c];
            bandp(U1, c, li, j) = un[0][c];
            bandp(U1, NP + c, li, j) = un[1][c];
          }
          u[0][c] = un[0][c];
          u[1][c] = un[1][c];
        }
        publish_u(int(k + 1), un);
      } else {
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          rowp(UBH, c, j) = (un[0][c] + un[0][c]) - uo[0][c];
          if (check) rowp(DUH, c, j) = un[0][c] - uo[0][c];
        }
      }
    }
    if (t == 0) cl_arm(bar0 + 8 * uint32_t((k + 1) & 1), in_bytes);  // arm iteration k+1
    __syncthreads();
    // phase B: channel flux and potential (own cells)
    if (own) {
      T rhs[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        T d = bandp(UB, c, li, j);
        if (i > 0) d = d - (li > 0 ? bandp(UB, c, li - 1, j) : rowp(UBH, c, j));
        d = d + bandp(UB, NP + c, li, j);
        if (j > 0) d = d - bandp(UB, NP + c, li, j - 1);
        d = d * H.inv_dx;
        rhs[c] = d - df[c];
      }
      T dwv[NWA];
      if (P::HAS_W) {
        T gc[NWA], wn[NWA], wb[NWA], dv[NP];
        P::grad_c(ph, gc, H);
#pragma unroll
        for (int e = 0; e < NWA; ++e) wn[e] = gc[e] * H.nu + w[e];
        P::prox_w(wn, H);
#pragma unroll
        for (int e = 0; e < NWA; ++e) {
          wb[e] = (wn[e] + wn[e]) - w[e];
          dwv[e] = wn[e] - w[e];
          w[e] = e < nwp ? wn[e] : T(0);
        }
        P::div_c(wb, dv, H);
#pragma unroll
        for (int c = 0; c < NP; ++c) rhs[c] = rhs[c] + dv[c];
      }
      T phnew[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        rhs[c] = rhs[c] * H.tau;
        phnew[c] = ph[c] + rhs[c];
      }
      if (check) {
        T cross[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const T dx = bandp(DU, c, li, j);
          const T dy = bandp(DU, NP + c, li, j);
          acc[0] += P::wp(c) * (double(dx) * double(dx) + double(dy) * double(dy));
          T d = dx;
          if (i > 0) d = d - (li > 0 ? bandp(DU, c, li - 1, j) : rowp(DUH, c, j));
          d = d + dy;
          if (j > 0) d = d - bandp(DU, NP + c, li, j - 1);
          cross[c] = d * H.inv_dx;
        }
        if (P::HAS_W) {
          T dv[NP];
          P::div_c(dwv, dv, H);
#pragma unroll
          for (int c = 0; c < NP; ++c) cross[c] = cross[c] + dv[c];
#pragma unroll
          for (int e = 0; e < NWA; ++e) acc[1] += P::ww(e) * double(dwv[e]) * double(dwv[e]);
        }
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          const T dp = phnew[c] - ph[c];
          acc[2] += P::wp(c) * double(dp) * double(dp);
          acc[3] += P::wp(c) * double(dp) * double(cross[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        ph[c] = phnew[c];
        bandp(PHI, c, li, j) = phnew[c];
      }
      publish_phi(int(k + 1), phnew);
    }
    __syncthreads();  // PHI complete before the next phase A reads it
  };

  // ---- evaluate iterate `it` (+ the R^k terms of the iteration that made
  // it), cluster reduction in rank order; returns the stop decision
  long long nh = 0;
  auto check_point = [&](long long it, bool with_res, const double (&acc)[4]) -> bool {
    double sacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // raw order R_PU .. R_SCROSS
    double mx[2] = {0.0, 0.0};
    if (with_res) {
      sacc[R_SDU] = acc[0];
      sacc[R_SDW] = acc[1];
      sacc[R_SDPHI] = acc[2];
      sacc[R_SCROSS] = acc[3];
    }
    const int s = int(it & 1);
    if (own) {
      if (first || last) wait_slot(unsigned(it));
      sacc[R_PU] += P::norm_u(u, H.norm_u);
      double su = 0.0;
#pragma unroll
      for (int c = 0; c < NP; ++c)
        su += P::wp(c) * (double(u[0][c]) * double(u[0][c]) + double(u[1][c]) * double(u[1][c]));
      sacc[R_SU2] += su;
      T con[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        T d = u[0][c];
        if (i > 0) d = d - (li > 0 ? bandp(U1, c, li - 1, j) : slotp(s, NP + c, j));
        d = d + u[1][c];
        if (j > 0) d = d - bandp(U1, NP + c, li, j - 1);
        con[c] = d * H.inv_dx - df[c];
      }
      if (P::HAS_W) {
        sacc[R_PW] += P::norm_w(w, H.norm_w);
        double sw = 0.0;
#pragma unroll
        for (int e = 0; e < NWA; ++e) sw += P::ww(e) * double(w[e]) * double(w[e]);
        sacc[R_SW2] += sw;
        T dv[NP];
        P::div_c(w, dv, H);
#pragma unroll
        for (int c = 0; c < NP; ++c) con[c] = con[c] + dv[c];
      }
      double sc = 0.0, sp = 0.0;
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        sc += P::wp(c) * double(con[c]) * double(con[c]);
        sp += P::wp(c) * double(ph[c]) * double(df[c]);
      }
      sacc[R_SCON] += sc;
      sacc[R_SPHID] += sp;
      T g[2][NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const T px = hasx ? (li + 1 < rows ? bandp(PHI, c, li + 1, j) : slotp(s, 3 * NP + c, j)) : T(0);
        g[0][c] = hasx ? (px - ph[c]) * H.inv_dx : T(0);
        g[1][c] = hasy ? (bandp(PHI, c, li, j + 1) - ph[c]) * H.inv_dx : T(0);
      }
      P::dual_u(g, H.norm_u, mx[0], sacc[R_PENU]);
      if (P::HAS_W) {
        T gc[NWA];
        P::grad_c(ph, gc, H);
        P::dual_w(gc, H.norm_w, H.ell, H.alpha, mx[1], sacc[R_PENW]);
      }
    }
    block_sum<12>(sacc, sred);
    block_max<2>(mx, sred);
    if (t == 0) {
      double* dst = cg::this_cluster().map_shared_rank(sslot, 0) + rank * 14;
#pragma unroll
      for (int q = 0; q < 12; ++q) dst[q] = sacc[q];
      dst[12] = mx[0];
      dst[13] = mx[1];
    }
    cl_sync();
    if (rank == 0 && t == 0) {
      double raw[R_NRAW];
#pragma unroll
      for (int q = 0; q < R_NRAW; ++q) raw[q] = 0.0;
      for (int r = 0; r < C; ++r) {
        for (int q = 0; q < 12; ++q) raw[q] += sslot[r * 14 + q];
        raw[R_GU] = dmax(raw[R_GU], sslot[r * 14 + 12]);
        raw[R_GW] = dmax(raw[R_GW], sslot[r * 14 + 13]);
      }
      double out[5];
      finalize_dev(raw, G.has_w != 0, A.alpha, A.eps, G.diff_norm, G.mu, G.nu, G.tau, out);
      const bool conv = out[2] <= G.tol_gap && out[3] <= G.tol_feas;
      if (nh < G.hist_cap) {
        double* h = G.hist + nh * 6;
        h[0] = double(it);
        h[1] = out[0];
        h[2] = out[1];
        h[3] = out[2];
        h[4] = out[3];
        h[5] = with_res ? out[4] : __longlong_as_double(0x7ff8000000000000LL);
      }
      for (int r = 0; r < C; ++r)
        *cg::this_cluster().map_shared_rank(const_cast<int*>(sflag), r) = conv ? 1 : 0;
    }
    ++nh;
    cl_sync();
    return *sflag != 0;
  };

  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  long long it = 0;
  bool conv = false;
  if (G.checks) {
    conv = check_point(0, false, acc);
    const long long ce = G.check_every, mxi = G.max_iters;
    while (!conv && it < mxi) {
      long long nxt = (it / ce + 1) * ce;
      if (nxt > mxi) nxt = mxi;
      const int plain = int(nxt - 1 - it);
      for (int q = 0; q < plain; ++q) iterate(unsigned(it) + unsigned(q), false, acc);
      it = nxt - 1;
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = 0.0;
      iterate(unsigned(it), true, acc);
      it = nxt;
      conv = check_point(it, true, acc);
    }
  } else {
    const int plain = int(G.max_iters);
    for (int q = 0; q < plain; ++q) iterate(unsigned(q), false, acc);
    it = G.max_iters;
  }

  // ---- store the cell back (in place: the engine's current iterate)
  if (own) {
    const int64_t o = cell_off(A, i, j);
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      A.a.u[c * pl + o] = u[0][c];
      A.a.u[(NP + c) * pl + o] = u[1][c];
      A.a.phi[c * pl + o] = ph[c];
    }
    if (P::HAS_W) {
#pragma unroll
      for (int e = 0; e < NWA; ++e)
        if (e < nwp) A.a.w[e * pl + o] = w[e];
    }
  }
  if (rank == 0 && t == 0) {
    G.result[0] = it;
    G.result[1] = nh;
    G.result[2] = conv ? 1 : 0;
  }
  // the rows published for iteration `it` have landed before anyone exits
  wait_slot(unsigned(it));
  cl_sync();
}

// shared memory bytes of one CTA of the on-chip solve
template <class P, typename T>
inline size_t cluster_smem_bytes(int rows_max, int n) {
  return ClusterSmem<P, T>(rows_max, n).bytes();
}

}  // namespace otfx
