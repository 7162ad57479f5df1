// TMA-streamed, warp-specialised variant of the fused PDHG sweep (same
// arithmetic as sweep.cuh, same results bit for bit).
//
// The register-streaming sweep issues its row loads and immediately waits on
// them, and a CTA-wide barrier per row ties its warps together, so memory
// parallelism per SM is bounded by the warps that happen to be in their load
// phase.  Here one producer warp per CTA drives a ring of S row stages in
// shared memory: one 3-D TMA box per field group (u: 2NP planes, w, diff,
// phi) of TW = tile + 2h columns (cols c0-h .. c0+tile+h-1, zero-filled outside
// the grid by the tensor map; h makes the box start 16-byte aligned, which the
// TMA unit requires) lands on a "full" mbarrier; every consumer warp
// releases a stage through an "empty" mbarrier when it is done with it.
// Consumer warps overlap by one column: lane 0 of each warp only computes
// the spatial flux of the column left of the warp's 31 output columns, and
// ubar_y(i, j-1) reaches lane l from lane l-1 by a warp shuffle.  Consumers
// therefore never wait for each other (no block barrier in the row loop) and
// the redundant work is 1/32 of the flux.
//
// Stage q of a CTA holds global row qbase + q with qbase = gr0 - 1:
//   q = 0            halo row gr0-1: u, phi          (skipped when gr0 == 0)
//   q = 1 .. R       rows gr0 .. gr1-1: u, w, diff, phi
//   q = R + 1        row gr1: phi only               (skipped when gr1 == n)
// Skipped stages complete their mbarrier with a plain arrive so the phase
// bookkeeping (parity = (q / S) & 1) stays uniform.
#pragma once

#include "sweep.cuh"
#include "tma.cuh"

namespace otfx {

struct alignas(64) TmaSet {
  CUtensorMap u, w, phi, diff;
};

struct StageLayout {
  int cw;          // consumer warps per CTA (a producer warp follows them)
  int tile;        // output columns per CTA = 31 * cw
  int h;           // halo columns staged each side: 16 B worth (TMA needs the box
                   // start column 16-byte aligned), 2 for fp64, 4 for fp32
  int tw;          // staged columns = tile + 2h (cols c0-h .. c0+tile+h-1)
  int S;           // ring depth
  int off_w, off_d, off_p;  // byte offsets inside a stage
  int stage_bytes;
  int bytes_full, bytes_flux, bytes_phi;  // expect-tx per stage kind
  int off_stages, off_xchg, off_red;      // byte offsets in dynamic smem
  int total;
};

template <typename T>
struct TmaSweepArgs {
  SweepArgs<T> s;
  StageLayout L;
};

// Channel coefficients as the kernels read them: the small vector D/c matrix
// is pulled into registers once per CTA; the Lindblad stacks stay in the
// (constant-cached) parameter space.
template <class P, typename T, bool REG = (P::NCOEF > 0 && P::NCOEF <= 64)>
struct CoefView;
template <class P, typename T>
struct CoefView<P, T, true> {
  T c[P::NCOEF];
  __device__ __forceinline__ void load(const SweepArgs<T>& A) {
#pragma unroll
    for (int q = 0; q < P::NCOEF; ++q) c[q] = T(A.coef[q]);
  }
  __device__ __forceinline__ T operator[](int q) const { return c[q]; }
};
template <class P, typename T>
struct CoefView<P, T, false> {
  const double* c;
  __device__ __forceinline__ void load(const SweepArgs<T>& A) { c = A.coef; }
  __device__ __forceinline__ double operator[](int q) const { return c[q]; }
};

// The scalars the per-cell math reads, held in registers for the whole CTA
// (the policies are duck-typed on these field names).
template <class P, typename T>
struct HotArgs {
  T mu, thr_w, nu, tau, inv_dx, den_u, den_w;
  int has_eps, norm_u, norm_w, ell, real_l;
  double alpha;
  CoefView<P, T> coef;
  __device__ __forceinline__ void load(const SweepArgs<T>& A) {
    mu = A.mu; thr_w = A.thr_w; nu = A.nu; tau = A.tau; inv_dx = A.inv_dx;
    den_u = A.den_u; den_w = A.den_w; has_eps = A.has_eps; real_l = A.real_l;
    norm_u = A.norm_u; norm_w = A.norm_w; ell = A.ell; alpha = A.alpha;
    coef.load(A);
  }
};

// compile-time shared-memory layout of one TMA row stage
template <class P, typename T, int CW_ = 4>
struct StageShape {
  static constexpr int CW = CW_;                    // consumer warps per CTA
  static constexpr int H = 16 / int(sizeof(T));     // halo columns (16 B)
  static constexpr int TILE = 31 * CW;              // output columns per CTA
  // staged columns, a multiple of 16 bytes (TMA box rows; an odd warp count
  // stages one spare column)
  static constexpr int TW = (TILE + 2 * H + H - 1) / H * H;
  static constexpr int ROW = TW * int(sizeof(T));
  static constexpr int R128(int x) { return (x + 127) / 128 * 128; }
  static constexpr int OFF_W = R128(2 * P::NP * ROW);
  static constexpr int OFF_D = OFF_W + R128((P::NWA > 0 ? P::NWA : 1) * ROW);
  static constexpr int OFF_P = OFF_D + R128(P::NP * ROW);
  static constexpr int BYTES = OFF_P + R128(P::NP * ROW);
};

// Loads of ring stage q (global row qbase + q) into `slot`: the halo row
// (u, phi), the R owned rows (u, w, diff, phi), the phi-only tail row -- each
// a set of 3-D TMA boxes completing on full[slot].
template <class SS, class P, typename T>
__device__ __forceinline__ void tma_issue_stage(const SweepArgs<T>& A, const StageLayout& L,
                                                const TmaSet& M, uint64_t* full,
                                                unsigned char* stages, int c0, int gr0, int qbase,
                                                int qmax, int q, int slot) {
  const int n = A.n;
  const int cx = c0 - SS::H;
  uint64_t* bar = &full[slot];
  const int r = qbase + q;
  const int lrow = r - A.row_begin + 1;
  unsigned char* st = stages + slot * SS::BYTES;
  if (q == 0 || q == qmax) {
    const bool load = (q == 0) ? (gr0 > 0) : (r < n);
    if (!load) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    } else {
      if (q == 0) {
        mbar_expect_tx(bar, L.bytes_flux);
        tma_load_3d(st, &M.u, bar, cx, lrow, 0);
      } else {
        mbar_expect_tx(bar, L.bytes_phi);
      }
      tma_load_3d(st + SS::OFF_P, &M.phi, bar, cx, lrow, 0);
    }
  } else {
    mbar_expect_tx(bar, L.bytes_full);
    tma_load_3d(st, &M.u, bar, cx, lrow, 0);
    if (P::HAS_W) tma_load_3d(st + SS::OFF_W, &M.w, bar, cx, lrow, 0);
    tma_load_3d(st + SS::OFF_D, &M.diff, bar, cx, lrow, 0);
    tma_load_3d(st + SS::OFF_P, &M.phi, bar, cx, lrow, 0);
  }
}

// The producer warp's loop (one elected lane): stage q of the ring is reused
// once every consumer warp has arrived on empty[slot].
template <class SS, class P, typename T>
__device__ __forceinline__ void tma_produce(const SweepArgs<T>& A, const StageLayout& L,
                                            const TmaSet& M, uint64_t* full, uint64_t* empty,
                                            unsigned char* stages, int c0, int gr0, int gr1,
                                            int qbase, int qmax) {
  const int S = L.S;
  int slot = 0, use = 0;
  for (int q = 0; q <= qmax; ++q) {
    if (q >= S) mbar_wait(&empty[slot], (use - 1) & 1);
    tma_issue_stage<SS, P, T>(A, L, M, full, stages, c0, gr0, qbase, qmax, q, slot);
    if (++slot == S) {
      slot = 0;
      ++use;
    }
  }
}

#ifndef OTFX_HEAVY_SELF
#define OTFX_HEAVY_SELF 1
#endif
#ifndef OTFX_SELF_NARROW
#define OTFX_SELF_NARROW 0
#endif
// Thread roles of a TMA sweep CTA: CW consumer warps plus one producer warp,
// except (OTFX_HEAVY_SELF, default on) the wide heavy complex-Hermitian payloads, whose
// 255-register consumers fit at most 8 warps per SM (2 per sub-partition's
// register file): there the last consumer warp to release a ring slot issues
// the slot's next loads itself, and all 8 warps compute.
template <class P, typename T, int CW>
struct TmaRoles {
  static constexpr bool HEAVY = sizeof(T) == 8 && P::NCOEF == 0 && P::NP == P::K * P::K && P::K >= 3;
  // (OTFX_SELF_NARROW: the 2x2 complex payload's 4-warp CTAs too, so four
  // of them fit an SM on a 2-stage ring)
  static constexpr bool C2X2 = sizeof(T) == 8 && P::NCOEF == 0 && P::NP == P::K * P::K && P::K == 2;
  static constexpr bool SELF = (OTFX_HEAVY_SELF != 0 && HEAVY && CW == 8) ||
                               (OTFX_SELF_NARROW != 0 && C2X2 && CW == 4);
  static constexpr int THREADS = 32 * (CW + (SELF ? 0 : 1));
};

// FL bit 0 (CHECK): this sweep ends on a check iteration -- accumulate the
//   R^k terms (S/solver.py:282-291) from the old and new values in registers;
// FL bit 1 (DUAL): the INPUT iterate is a checked one -- accumulate its
//   evaluate terms (S/solver.py:242-280): primal, feasibility and <phi, diff>
//   from the staged input, and the dual norms of its gradients, which this
//   sweep computes anyway for the flux and channel updates.  (Splitting the
//   check work over the two sweeps keeps both close to a plain sweep.)
template <class P, typename T, int FL, int CWT = 4>
//
// Occupancy hints, measured on B200 (profiles/README.md): the wide check and
// dual sweeps are held to two resident CTAs per SM (<= 96 registers; at their
// natural 126-156 the check sweep ran one CTA per SM and took 2.6x a plain
// sweep), and the plain sweep states minBlocks = 1 explicitly, which steers
// ptxas to a 70-register schedule for fp32 (12 % faster than the 56-register
// one it picks without the hint; fp64 unchanged).
// The 4-warp instantiations (matrix payloads) keep ptxas' default (0 = no
// hint): stating minBlocks = 1 there raises the 3x3 real payload from 156 to
// 196 registers and halves its occupancy.
#ifndef OTFX_DUAL_MINB
#define OTFX_DUAL_MINB 2
#endif
__global__ void __launch_bounds__(TmaRoles<P, T, CWT>::THREADS,
                                  (CWT == 8 && (P::NCOEF > 0 || !P::HAS_W))
                                      ? (FL == 0 ? 1 : (FL == 2 ? OTFX_DUAL_MINB : 2))
                                      : 0)
    sweep_tma_kernel(
    const __grid_constant__ TmaSweepArgs<T> G, const __grid_constant__ TmaSet M) {
  constexpr bool CHECK = (FL & 1) != 0;
  constexpr bool DUAL = (FL & 2) != 0;
  using SS = StageShape<P, T, CWT>;
  constexpr int NP = P::NP;
  constexpr int NWA = P::NWA;
  constexpr int TW = SS::TW;
  const SweepArgs<T>& A = G.s;
  const StageLayout& L = G.L;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [S]
  uint64_t* empty = full + 8;                          // [S]
  unsigned char* stages = smem + 128;
  double* sred = reinterpret_cast<double*>(smem + L.off_red);

  constexpr int CW = CWT;
  const int S = L.S;
  const int t = threadIdx.x;
  const int warp = t >> 5, lane = t & 31;
  constexpr bool SELF = TmaRoles<P, T, CWT>::SELF;
  const bool producer = !SELF && warp >= CW;
  int* cnt = reinterpret_cast<int*>(empty);  // SELF: releases per slot
  const int c0 = blockIdx.x * SS::TILE;
  const int sc = SS::H + 31 * warp + lane - 1;  // staged column index of this thread's column
  const int j = c0 - SS::H + sc;                // = c0 + 31 warp + lane - 1
  const int n = A.n;
  const bool out = !producer && lane > 0 && j < n;  // lane 0 is the overlap column
  const bool hasy = j + 1 < n;
  const int band = A.band0 + int(blockIdx.y) * A.band_step;
  const int gr0 = A.row_begin + band * A.rows_per_block;
  const int gr1 = min(gr0 + A.rows_per_block, A.row_end);
  const int qbase = gr0 - 1;
  const int qmax = gr1 - qbase;  // index of the phi-only tail stage

  if (t == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      if (SELF) cnt[2 * s] = 0;
      else mbar_init(&empty[s], CW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // the previous sweep has finished reading what this one writes
  pdl_launch_dependents();
  if (SELF && t == 0) {
    for (int q = 0; q < S && q <= qmax; ++q)
      tma_issue_stage<SS, P, T>(A, L, M, full, stages, c0, gr0, qbase, qmax, q, q);
  }

  // CHECK: SDU SDW SDPHI SCROSS;  DUAL: PU PW SU2 SW2 SCON SPHID PENU PENW | GU GW
  double acc[4] = {0, 0, 0, 0};
  double dsum[8] = {0, 0, 0, 0, 0, 0, 0, 0}, dmx[2] = {0.0, 0.0};
  if (producer) {
    if (lane == 0) tma_produce<SS, P, T>(A, L, M, full, empty, stages, c0, gr0, gr1, qbase, qmax);
  } else {
    // ------------------------------------------------------------ consumers
    HotArgs<P, T> H;
    H.load(A);
    const int nwp = H.ell * P::NWS;
    const int64_t pl = A.plane;
    // ring cursor for stage q (slot, phase parity) and stage q+1
    int s0 = 0, ph0 = 0;
    auto adv = [&](int& s, int& ph) {
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    };
    auto base = [&](int s) -> const T* {
      return reinterpret_cast<const T*>(stages + s * SS::BYTES) + sc;
    };
    int qrel = 0;  // ring stage released next
    auto release = [&](int s) {
      __syncwarp();
      if (lane == 0) {
        if constexpr (SELF) {
          // the last warp out refills the slot with stage qrel + S
          __threadfence_block();
          if (atomicAdd(&cnt[2 * s], 1) == CW - 1) {
            atomicExch(&cnt[2 * s], 0);
            const int qn = qrel + S;
            if (qn <= qmax) {
              fence_proxy_async();
              tma_issue_stage<SS, P, T>(A, L, M, full, stages, c0, gr0, qbase, qmax, qn, s);
            }
          }
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s]))
                       : "memory");
        }
      }
      ++qrel;
    };
    T uxb_prev[NP], dux_prev[NP], uox_prev[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      uxb_prev[c] = T(0);
      dux_prev[c] = T(0);
      uox_prev[c] = T(0);
    }
    int s1 = 1, ph1 = 0;  // cursor of stage q+1
    if (S == 1) s1 = 0;
    // halo row gr0-1: ubar_x(gr0-1, j) from the read-only iterate
    mbar_wait(&full[s0], ph0);
    if (gr0 > 0) {
      mbar_wait(&full[s1], ph1);
      const T* b0 = base(s0);
      const T* b1 = base(s1);
      T pm[NP], px[NP], py[NP], uo[2][NP], un[2][NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const T* pp = reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(b0) + SS::OFF_P);
        pm[c] = pp[c * TW];
        py[c] = pp[c * TW + 1];
        px[c] = reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(b1) + SS::OFF_P)[c * TW];
        uo[0][c] = b0[c * TW];
        uo[1][c] = b0[(NP + c) * TW];
      }
      Cell<P, T>::flux(pm, px, py, true, hasy, uo, un, H);
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        uxb_prev[c] = (un[0][c] + un[0][c]) - uo[0][c];
        dux_prev[c] = un[0][c] - uo[0][c];
        uox_prev[c] = uo[0][c];
      }
    }
    release(s0);
    adv(s0, ph0);  // stage 0 -> stage 1 becomes "q"
    s1 = s0;
    ph1 = ph0;
    adv(s1, ph1);

    T* gu = A.b.u;
    T* gphi = A.b.phi;
    T* gw = A.b.w;
    for (int i = gr0; i < gr1; ++i) {
      const bool hasx = i + 1 < n;
      mbar_wait(&full[s0], ph0);
      mbar_wait(&full[s1], ph1);
      const unsigned char* st0 = reinterpret_cast<const unsigned char*>(base(s0));
      const unsigned char* st1 = reinterpret_cast<const unsigned char*>(base(s1));
      const T* sU = reinterpret_cast<const T*>(st0);
      const T* sW = reinterpret_cast<const T*>(st0 + SS::OFF_W);
      const T* sD = reinterpret_cast<const T*>(st0 + SS::OFF_D);
      const T* sP = reinterpret_cast<const T*>(st0 + SS::OFF_P);
      const T* sPn = reinterpret_cast<const T*>(st1 + SS::OFF_P);
      T phc[NP], un[2][NP], ub[2][NP], uo[2][NP], lub[NP], ldu[NP], luo[NP];
      {
        T phx[NP], phy[NP], g[2][NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          phc[c] = sP[c * TW];
          phy[c] = sP[c * TW + 1];
          phx[c] = sPn[c * TW];
          uo[0][c] = sU[c * TW];
          uo[1][c] = sU[(NP + c) * TW];
        }
        Cell<P, T>::grad(phc, phx, phy, hasx, hasy, g, H);
        if (DUAL && out) P::dual_u(g, H.norm_u, dmx[0], dsum[6]);
        Cell<P, T>::flux_g(g, uo, un, H);
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          ub[0][c] = (un[0][c] + un[0][c]) - uo[0][c];
          ub[1][c] = (un[1][c] + un[1][c]) - uo[1][c];
          // ubar_y / du_y / u'_y of the left neighbour (i, j-1) from lane - 1
          lub[c] = __shfl_up_sync(0xffffffffu, ub[1][c], 1);
          if (CHECK) ldu[c] = __shfl_up_sync(0xffffffffu, un[1][c] - uo[1][c], 1);
          if (DUAL) luo[c] = __shfl_up_sync(0xffffffffu, uo[1][c], 1);
        }
      }
      // u' is final: store it now, so its registers are free for the channel
      // half of the row (the heavy complex payloads run at the register cap)
      if (out) {
        T* pu = gu + cell_off(A, i, j);
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          pu[c * pl] = un[0][c];
          pu[(NP + c) * pl] = un[1][c];
        }
      }
      T df[NP], wo[NWA];
#pragma unroll
      for (int c = 0; c < NP; ++c) df[c] = sD[c * TW];
      if (P::HAS_W) {
#pragma unroll
        for (int e = 0; e < NWA; ++e) wo[e] = e < nwp ? sW[e * TW] : T(0);
      }
      release(s0);  // stage q fully consumed (stage q+1 stays for the next row)
      if (out) {
        const int64_t o = cell_off(A, i, j);
        T rhs[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          T d = ub[0][c];
          if (i > 0) d = d - uxb_prev[c];
          d = d + ub[1][c];
          if (j > 0) d = d - lub[c];
          d = d * H.inv_dx;
          rhs[c] = d - df[c];
        }
        T wn[NWA], dwv[NWA];
        if (P::HAS_W) {
          T gc[NWA];
          P::grad_c(phc, gc, H);
          if (DUAL) P::dual_w(gc, H.norm_w, H.ell, H.alpha, dmx[1], dsum[7]);
#pragma unroll
          for (int e = 0; e < NWA; ++e) wn[e] = gc[e] * H.nu + wo[e];
          P::prox_w(wn, H);
          T wb[NWA], dv[NP];
#pragma unroll
          for (int e = 0; e < NWA; ++e) {
            wb[e] = (wn[e] + wn[e]) - wo[e];
            dwv[e] = wn[e] - wo[e];
          }
          T* pw = gw + o;
#pragma unroll
          for (int e = 0; e < NWA; ++e)
            if (e < nwp) pw[e * pl] = wn[e];
          P::div_c(wb, dv, H);
#pragma unroll
          for (int c = 0; c < NP; ++c) rhs[c] = rhs[c] + dv[c];
        }
        T phnew[NP];
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          rhs[c] = rhs[c] * H.tau;
          phnew[c] = phc[c] + rhs[c];
        }
        T* pp = gphi + o;
#pragma unroll
        for (int c = 0; c < NP; ++c) pp[c * pl] = phnew[c];
        if (CHECK) {
          T cross[NP];
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            const T dx = un[0][c] - uo[0][c];
            const T dy = un[1][c] - uo[1][c];
            acc[0] += P::wp(c) * (double(dx) * double(dx) + double(dy) * double(dy));
            T d = dx;
            if (i > 0) d = d - dux_prev[c];
            d = d + dy;
            if (j > 0) d = d - ldu[c];
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
            const T dp = phnew[c] - phc[c];
            acc[2] += P::wp(c) * double(dp) * double(dp);
            acc[3] += P::wp(c) * double(dp) * double(cross[c]);
          }
        }
        if (DUAL) {
          // evaluate terms of the input (checked) iterate, same order as
          // evaluate_kernel (S/solver.py:242-256)
          dsum[0] += P::norm_u(uo, H.norm_u);
          T con[NP];
          double su = 0.0, sc2 = 0.0, sp = 0.0;
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            su += P::wp(c) * (double(uo[0][c]) * double(uo[0][c]) +
                              double(uo[1][c]) * double(uo[1][c]));
            T d = uo[0][c];
            if (i > 0) d = d - uox_prev[c];
            d = d + uo[1][c];
            if (j > 0) d = d - luo[c];
            con[c] = d * H.inv_dx - df[c];
          }
          dsum[2] += su;
          if (P::HAS_W) {
            T wa[NWA];
#pragma unroll
            for (int e = 0; e < NWA; ++e) wa[e] = e < nwp ? wo[e] : T(0);
            dsum[1] += P::norm_w(wa, H.norm_w);
            double sw = 0.0;
#pragma unroll
            for (int e = 0; e < NWA; ++e) sw += P::ww(e) * double(wa[e]) * double(wa[e]);
            dsum[3] += sw;
            T dv[NP];
            P::div_c(wa, dv, H);
#pragma unroll
            for (int c = 0; c < NP; ++c) con[c] = con[c] + dv[c];
          }
#pragma unroll
          for (int c = 0; c < NP; ++c) {
            sc2 += P::wp(c) * double(con[c]) * double(con[c]);
            sp += P::wp(c) * double(phc[c]) * double(df[c]);
          }
          dsum[4] += sc2;
          dsum[5] += sp;
        }
      }
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        uxb_prev[c] = ub[0][c];
        if (CHECK) dux_prev[c] = un[0][c] - uo[0][c];
        if (DUAL) uox_prev[c] = uo[0][c];
      }
      s0 = s1;
      ph0 = ph1;
      adv(s1, ph1);
    }
  }

  const size_t bid = size_t(band) * gridDim.x + blockIdx.x;
  if (CHECK) {
    block_sum<4>(acc, sred);
    if (t == 0) {
      double* dst = A.partials + bid * 10;
#pragma unroll
      for (int s = 0; s < 4; ++s) dst[s] = acc[s];
#pragma unroll
      for (int s = 4; s < 10; ++s) dst[s] = 0.0;
    }
  }
  if (DUAL) {
    block_sum<8>(dsum, sred);
    block_max<2>(dmx, sred);
    if (t == 0) {
      double* dst = A.dualp + bid * 10;
#pragma unroll
      for (int s = 0; s < 8; ++s) dst[s] = dsum[s];
      dst[8] = dmx[0];
      dst[9] = dmx[1];
    }
  }
}

}  // namespace otfx
