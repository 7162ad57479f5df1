// Runtime-size vector payload: k-channel transport on a graph with k and ell
// known only at run time (k up to DYN_KMAX, ell up to DYN_LMAX).
//
// The reference's TransportGraph takes any connected graph on k nodes
// (S/graph.py:23-70); the compiled policies (payload.cuh VecPolicy) cover
// k <= 8 with the state in registers.  Wider graphs run here: the same
// per-cell arithmetic in the same operation order (VecPolicy, S/solver.py:
// 220-240), with runtime loops over channels and edges, the cell's payload in
// local memory, and the graph D/c read from a device buffer (too large for the
// kernel parameters).  One thread per cell walks a band of rows as the
// register sweep does (sweep.cuh), but instead of exchanging ubar with its
// neighbours through shared memory it recomputes their flux (a third of the
// throughput; this is the coverage path, the compiled policies are the fast
// one).  Iterates are bit-identical to the reference's order for every k,
// like the compiled vector path (tests/test_gpu_channel_counts.py).
#pragma once

#include "sweep.cuh"

namespace otfx {

// local memory per thread ~7 KB (fp64) at these capacities; the complete
// graph on 16 channels has 120 edges
constexpr int DYN_KMAX = 32;
constexpr int DYN_LMAX = 128;

template <typename T>
struct DynVec {
  // NumPy einsum sum of squares (np_sumsq in payload.cuh) for a runtime length
  __device__ static T sumsq(const T* x, int len) {
    T a0 = T(0), a1 = T(0);
    int b = 0;
#pragma unroll 1
    for (; b + 8 <= len; b += 8) {
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        a0 = x[b + 2 * q] * x[b + 2 * q] + a0;
        a1 = x[b + 2 * q + 1] * x[b + 2 * q + 1] + a1;
      }
    }
#pragma unroll 1
    for (int i = b; i < len; i += 2) {
      a0 = x[i] * x[i] + a0;
      if (i + 1 < len) a1 = x[i + 1] * x[i + 1] + a1;
    }
    return a0 + a1;
  }

  __device__ static T coef(const SweepArgs<T>& A, int c, int e) {
    return T(__ldg(A.chan_dev + size_t(c) * A.ell + e));
  }

  // u payload x[d * K + c] (the reference's (2, k) block in C order)
  __device__ static void prox_u(T* x, const SweepArgs<T>& A) {
    const int K = A.nchan;
    const T thr = A.mu;
    if (A.norm_u == NORM_L2) {
      const T f = soft_factor(sqrt(sumsq(x, 2 * K)), thr);
#pragma unroll 1
      for (int q = 0; q < 2 * K; ++q) x[q] = x[q] * f;
    } else if (A.norm_u == NORM_L12) {
#pragma unroll 1
      for (int c = 0; c < K; ++c) {
        const T f = soft_factor(sqrt(x[c] * x[c] + x[K + c] * x[K + c]), thr);
        x[c] = x[c] * f;
        x[K + c] = x[K + c] * f;
      }
    } else {
#pragma unroll 1
      for (int q = 0; q < 2 * K; ++q) x[q] = x[q] * soft_factor(fabs(x[q]), thr);
    }
    if (A.has_eps) {
#pragma unroll 1
      for (int q = 0; q < 2 * K; ++q) x[q] = x[q] / A.den_u;
    }
  }

  // diag(1/c) D^T phi: the reference's (n^2, k) @ (k, ell) BLAS product, one
  // ascending fused multiply-add chain over k per edge (VecPolicy::grad_c)
  __device__ static void grad_c(const T* p, T* g, const SweepArgs<T>& A) {
    const int K = A.nchan;
#pragma unroll 1
    for (int e = 0; e < A.ell; ++e) {
      T s = T(0);
      if (K == 2) {
        s = fma(p[1], coef(A, 1, e), s);
        s = fma(p[0], coef(A, 0, e), s);
      } else {
#pragma unroll 1
        for (int c = 0; c < K; ++c) s = fma(p[c], coef(A, c, e), s);
      }
      g[e] = s;
    }
  }

  // -D diag(1/c) y: (n^2, ell) @ (ell, k), ascending chain over ell
  __device__ static void div_c(const T* y, T* d, const SweepArgs<T>& A) {
#pragma unroll 1
    for (int c = 0; c < A.nchan; ++c) {
      T s = T(0);
#pragma unroll 1
      for (int e = 0; e < A.ell; ++e) s = fma(y[e], -coef(A, c, e), s);
      d[c] = s;
    }
  }

  __device__ static void prox_w(T* x, const SweepArgs<T>& A) {
    const int L = A.ell;
    const T thr = A.thr_w;
    if (A.norm_w == NORM_L2) {
      const T f = soft_factor(sqrt(sumsq(x, L)), thr);
#pragma unroll 1
      for (int e = 0; e < L; ++e) x[e] = x[e] * f;
    } else {
#pragma unroll 1
      for (int e = 0; e < L; ++e) x[e] = x[e] * soft_factor(fabs(x[e]), thr);
    }
    if (A.has_eps) {
#pragma unroll 1
      for (int e = 0; e < L; ++e) x[e] = x[e] / A.den_w;
    }
  }

  // per-cell norm values and dual norms (VecPolicy::norm_u ... dual_w)
  __device__ static double norm_u(const T* x, const SweepArgs<T>& A) {
    const int K = A.nchan;
    T s = T(0);
    if (A.norm_u == NORM_L2) {
#pragma unroll 1
      for (int q = 0; q < 2 * K; ++q) s = s + x[q] * x[q];
      return double(sqrt(s));
    }
    if (A.norm_u == NORM_L12) {
#pragma unroll 1
      for (int c = 0; c < K; ++c) s = s + sqrt(x[c] * x[c] + x[K + c] * x[K + c]);
      return double(s);
    }
#pragma unroll 1
    for (int q = 0; q < 2 * K; ++q) s = s + fabs(x[q]);
    return double(s);
  }

  __device__ static double norm_w(const T* x, const SweepArgs<T>& A) {
    T s = T(0);
    if (A.norm_w == NORM_L2) {
#pragma unroll 1
      for (int e = 0; e < A.ell; ++e) s = s + x[e] * x[e];
      return double(sqrt(s));
    }
#pragma unroll 1
    for (int e = 0; e < A.ell; ++e) s = s + fabs(x[e]);
    return double(s);
  }

  __device__ static void dual_u(const T* g, const SweepArgs<T>& A, double& gmax, double& pen) {
    const int K = A.nchan;
    if (A.norm_u == NORM_L2) {
      T s = T(0);
#pragma unroll 1
      for (int q = 0; q < 2 * K; ++q) s = s + g[q] * g[q];
      const double v = double(sqrt(s));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - 1.0, 0.0));
    } else if (A.norm_u == NORM_L12) {
#pragma unroll 1
      for (int c = 0; c < K; ++c) {
        const double v = double(sqrt(g[c] * g[c] + g[K + c] * g[K + c]));
        gmax = dmax(gmax, v);
        pen += sq(dmax(v - 1.0, 0.0));
      }
    } else {
#pragma unroll 1
      for (int q = 0; q < 2 * K; ++q) {
        const double v = double(fabs(g[q]));
        gmax = dmax(gmax, v);
        pen += sq(dmax(v - 1.0, 0.0));
      }
    }
  }

  __device__ static void dual_w(const T* g, const SweepArgs<T>& A, double& gmax, double& pen) {
    if (A.norm_w == NORM_L2) {
      T s = T(0);
#pragma unroll 1
      for (int e = 0; e < A.ell; ++e) s = s + g[e] * g[e];
      const double v = double(sqrt(s));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - A.alpha, 0.0));
    } else {
#pragma unroll 1
      for (int e = 0; e < A.ell; ++e) {
        const double v = double(fabs(g[e]));
        gmax = dmax(gmax, v);
        pen += sq(dmax(v - A.alpha, 0.0));
      }
    }
  }

  // phi(i, j) of the read iterate into p (zeros off the grid)
  __device__ static void load_phi(const SweepArgs<T>& A, int i, int j, T* p) {
    const int K = A.nchan;
    const bool in = i < A.n && j < A.n;
    const int64_t o = cell_off(A, i, j);
#pragma unroll 1
    for (int c = 0; c < K; ++c) p[c] = in ? ldg(A.a.phi + c * A.plane + o) : T(0);
  }

  // u'(i, j) = prox_u(grad phi * mu + u) of the read iterate
  // (S/solver.py:221-224, S/spatial.py:80-86); uo = u(i, j)
  __device__ static void flux(const SweepArgs<T>& A, int i, int j, T* uo, T* un, T* ph, T* pn) {
    const int K = A.nchan;
    const int64_t o = cell_off(A, i, j), pl = A.plane;
    const bool hasx = i + 1 < A.n, hasy = j + 1 < A.n;
    load_phi(A, i, j, ph);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      uo[c] = ldg(A.a.u + c * pl + o);
      uo[K + c] = ldg(A.a.u + (K + c) * pl + o);
    }
    load_phi(A, i + 1, j, pn);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      const T gx = hasx ? (pn[c] - ph[c]) * A.inv_dx : T(0);
      un[c] = gx * A.mu + uo[c];
    }
    load_phi(A, i, j + 1, pn);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      const T gy = hasy ? (pn[c] - ph[c]) * A.inv_dx : T(0);
      un[K + c] = gy * A.mu + uo[K + c];
    }
    prox_u(un, A);
  }
};

// One PDHG iteration (CHECK: + the R^k partials), same band / partial layout
// as sweep_kernel so the engine launches it in its place.
template <typename T, bool CHECK>
__global__ void __launch_bounds__(128) dyn_sweep_kernel(const __grid_constant__ SweepArgs<T> A) {
  using D = DynVec<T>;
  __shared__ double sred[32 * 4];
  const int K = A.nchan, L = A.ell;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const bool live = j < n;
  const int band = A.band0 + int(blockIdx.y) * A.band_step;
  const int gr0 = A.row_begin + band * A.rows_per_block;
  const int gr1 = min(gr0 + A.rows_per_block, A.row_end);
  const int64_t pl = A.plane;

  T ph[DYN_KMAX], pn[DYN_KMAX], uo[2 * DYN_KMAX], un[2 * DYN_KMAX];
  T nuo[2 * DYN_KMAX], nun[2 * DYN_KMAX];  // a neighbour cell's flux
  T uxb_prev[DYN_KMAX], dux_prev[DYN_KMAX], lub[DYN_KMAX], ldu[DYN_KMAX], rhs[DYN_KMAX];
  T wo[DYN_LMAX], wn[DYN_LMAX], wt[DYN_LMAX];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};

  if (live && gr0 > 0 && gr0 < gr1) {
    // ubar_x / du_x of the row above the band, from the read-only iterate
    D::flux(A, gr0 - 1, j, nuo, nun, pn, rhs);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      uxb_prev[c] = (nun[c] + nun[c]) - nuo[c];
      dux_prev[c] = nun[c] - nuo[c];
    }
  }
  for (int i = gr0; live && i < gr1; ++i) {
    const int64_t o = cell_off(A, i, j);
    D::flux(A, i, j, uo, un, ph, pn);
    if (j > 0) {
      D::flux(A, i, j - 1, nuo, nun, pn, rhs);
#pragma unroll 1
      for (int c = 0; c < K; ++c) {
        lub[c] = (nun[K + c] + nun[K + c]) - nuo[K + c];
        ldu[c] = nun[K + c] - nuo[K + c];
      }
    }
    // phi update: rhs = div(ubar) - diff (+ div_c wbar), rhs *= tau
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      const T ubx = (un[c] + un[c]) - uo[c];
      const T uby = (un[K + c] + un[K + c]) - uo[K + c];
      T d = ubx;
      if (i > 0) d = d - uxb_prev[c];
      d = d + uby;
      if (j > 0) d = d - lub[c];
      d = d * A.inv_dx;
      rhs[c] = d - ldg(A.diff + c * pl + o);
      uxb_prev[c] = ubx;
    }
#pragma unroll 1
    for (int e = 0; e < L; ++e) wo[e] = ldg(A.a.w + e * pl + o);
    D::grad_c(ph, wt, A);
#pragma unroll 1
    for (int e = 0; e < L; ++e) wn[e] = wt[e] * A.nu + wo[e];
    D::prox_w(wn, A);
#pragma unroll 1
    for (int e = 0; e < L; ++e) wt[e] = (wn[e] + wn[e]) - wo[e];
    D::div_c(wt, pn, A);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      rhs[c] = rhs[c] + pn[c];
      rhs[c] = rhs[c] * A.tau;
    }
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      const T phnew = ph[c] + rhs[c];
      A.b.u[c * pl + o] = un[c];
      A.b.u[(K + c) * pl + o] = un[K + c];
      A.b.phi[c * pl + o] = phnew;
      rhs[c] = phnew - ph[c];  // dphi (CHECK)
    }
#pragma unroll 1
    for (int e = 0; e < L; ++e) A.b.w[e * pl + o] = wn[e];
    if (CHECK) {
      // R^k terms (S/solver.py:282-291), as sweep_kernel accumulates them
#pragma unroll 1
      for (int e = 0; e < L; ++e) wt[e] = wn[e] - wo[e];
      D::div_c(wt, pn, A);
#pragma unroll 1
      for (int c = 0; c < K; ++c) {
        const T dx = un[c] - uo[c];
        const T dy = un[K + c] - uo[K + c];
        acc[0] += double(dx) * double(dx) + double(dy) * double(dy);
        T d = dx;
        if (i > 0) d = d - dux_prev[c];
        d = d + dy;
        if (j > 0) d = d - ldu[c];
        const T cross = d * A.inv_dx + pn[c];
        dux_prev[c] = dx;
        acc[2] += double(rhs[c]) * double(rhs[c]);
        acc[3] += double(rhs[c]) * double(cross);
      }
#pragma unroll 1
      for (int e = 0; e < L; ++e) acc[1] += double(wt[e]) * double(wt[e]);
    }
  }
  if (CHECK) {
    block_sum<4>(acc, sred);
    if (threadIdx.x == 0) {
      double* dst = A.partials + (size_t(band) * gridDim.x + blockIdx.x) * 10;
#pragma unroll
      for (int s = 0; s < 4; ++s) dst[s] = acc[s];
#pragma unroll
      for (int s = 4; s < 10; ++s) dst[s] = 0.0;
    }
  }
}

// evaluate terms of the read iterate (evaluate_kernel, S/solver.py:242-280)
template <typename T>
__global__ void __launch_bounds__(128) dyn_evaluate_kernel(const __grid_constant__ SweepArgs<T> A) {
  using D = DynVec<T>;
  __shared__ double sred[32 * 8];
  const int K = A.nchan, L = A.ell;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const int64_t pl = A.plane;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // PU PW SU2 SW2 SCON SPHID PENU PENW
  double mx[2] = {0.0, 0.0};
  T u[2 * DYN_KMAX], ph[DYN_KMAX], pn[DYN_KMAX], con[DYN_KMAX], w[DYN_LMAX];
  for (int i = A.row_begin + blockIdx.y; j < n && i < A.row_end; i += gridDim.y) {
    const int64_t o = cell_off(A, i, j), oxm = cell_off(A, i - 1, j);
#pragma unroll 1
    for (int q = 0; q < 2 * K; ++q) u[q] = ldg(A.a.u + q * pl + o);
#pragma unroll 1
    for (int e = 0; e < L; ++e) w[e] = ldg(A.a.w + e * pl + o);
    D::load_phi(A, i, j, ph);
    s[0] += D::norm_u(u, A);
    double su = 0.0;
#pragma unroll 1
    for (int c = 0; c < K; ++c)
      su += double(u[c]) * double(u[c]) + double(u[K + c]) * double(u[K + c]);
    s[2] += su;
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      T d = u[c];
      if (i > 0) d = d - ldg(A.a.u + c * pl + oxm);
      d = d + u[K + c];
      if (j > 0) d = d - ldg(A.a.u + (K + c) * pl + o - 1);
      con[c] = d * A.inv_dx - ldg(A.diff + c * pl + o);
    }
    s[1] += D::norm_w(w, A);
    double sw = 0.0;
#pragma unroll 1
    for (int e = 0; e < L; ++e) sw += double(w[e]) * double(w[e]);
    s[3] += sw;
    D::div_c(w, pn, A);
    double sc = 0.0, sp = 0.0;
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      con[c] = con[c] + pn[c];
      sc += double(con[c]) * double(con[c]);
      sp += double(ph[c]) * double(ldg(A.diff + c * pl + o));
    }
    s[4] += sc;
    s[5] += sp;
    // dual norms of grad phi (u[] reused for the gradient) and grad_c phi
    const bool hx = i + 1 < n, hy = j + 1 < n;
    D::load_phi(A, i + 1, j, pn);
#pragma unroll 1
    for (int c = 0; c < K; ++c) u[c] = hx ? (pn[c] - ph[c]) * A.inv_dx : T(0);
    D::load_phi(A, i, j + 1, pn);
#pragma unroll 1
    for (int c = 0; c < K; ++c) u[K + c] = hy ? (pn[c] - ph[c]) * A.inv_dx : T(0);
    D::dual_u(u, A, mx[0], s[6]);
    D::grad_c(ph, w, A);
    D::dual_w(w, A, mx[1], s[7]);
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

// R^k between the iterates A.a and A.b (residual_kernel)
template <typename T>
__global__ void __launch_bounds__(128) dyn_residual_kernel(const __grid_constant__ SweepArgs<T> A) {
  using D = DynVec<T>;
  __shared__ double sred[32 * 4];
  const int K = A.nchan, L = A.ell;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const int64_t pl = A.plane;
  double s[4] = {0, 0, 0, 0};
  T dw[DYN_LMAX], dv[DYN_KMAX];
  for (int i = A.row_begin + blockIdx.y; j < n && i < A.row_end; i += gridDim.y) {
    const int64_t o = cell_off(A, i, j), oxm = cell_off(A, i - 1, j);
    auto du = [&](int comp, int64_t off) { return A.b.u[comp * pl + off] - A.a.u[comp * pl + off]; };
#pragma unroll 1
    for (int e = 0; e < L; ++e) {
      dw[e] = A.b.w[e * pl + o] - A.a.w[e * pl + o];
      s[1] += double(dw[e]) * double(dw[e]);
    }
    D::div_c(dw, dv, A);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      const T dx = du(c, o), dy = du(K + c, o);
      s[0] += double(dx) * double(dx) + double(dy) * double(dy);
      T d = dx;
      if (i > 0) d = d - du(c, oxm);
      d = d + dy;
      if (j > 0) d = d - du(K + c, o - 1);
      const T cross = d * A.inv_dx + dv[c];
      const T dp = A.b.phi[c * pl + o] - A.a.phi[c * pl + o];
      s[2] += double(dp) * double(dp);
      s[3] += double(dp) * double(cross);
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
