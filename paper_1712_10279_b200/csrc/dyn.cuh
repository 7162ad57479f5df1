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
  static constexpr int NPMAX = DYN_KMAX;  // reals per potential
  static constexpr int NWMAX = DYN_LMAX;  // reals of the channel flux
  __device__ static int np(const SweepArgs<T>& A) { return A.nchan; }
  __device__ static int nw(const SweepArgs<T>& A) { return A.ell; }
  __device__ static double wp(const SweepArgs<T>&, int) { return 1.0; }
  __device__ static double ww(const SweepArgs<T>&, int) { return 1.0; }

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

};

// Runtime-size matrix payloads: the real-symmetric (CPLX = false, SymPolicy)
// and complex-Hermitian (CPLX = true, HermPolicy) paths for k and ell beyond
// the compiled instantiations (k up to DYN_MKMAX, ell * block reals up to
// DYN_MNWMAX).  Same packed layouts, same per-entry arithmetic; the Jacobi
// eigensolver runs on runtime-indexed local arrays.
constexpr int DYN_MKMAX = 8;
constexpr int DYN_MNWMAX = 256;

template <typename T, bool CPLX>
struct DynMat {
  static constexpr int NPMAX = DYN_MKMAX * DYN_MKMAX;
  static constexpr int NWMAX = DYN_MNWMAX;
  using M = T[DYN_MKMAX][DYN_MKMAX];

  __device__ static int npk(int K) { return CPLX ? K * K : K * (K + 1) / 2; }
  __device__ static int nws(int K) { return CPLX ? K * K : K * (K - 1) / 2; }
  __device__ static int np(const SweepArgs<T>& A) { return npk(A.nchan); }
  __device__ static int nw(const SweepArgs<T>& A) { return A.ell * nws(A.nchan); }
  __device__ static double wp(const SweepArgs<T>& A, int c) { return c < A.nchan ? 1.0 : 2.0; }
  __device__ static double ww(const SweepArgs<T>& A, int e) {
    return CPLX ? ((e % nws(A.nchan)) < A.nchan ? 1.0 : 2.0) : 2.0;
  }
  __device__ static int pair(int K, int a, int b) { return a * K - a * (a + 1) / 2 + (b - a - 1); }
  // packed index of the (re) entry of pair (a < b)
  __device__ static int poff(int K, int a, int b) { return K + (CPLX ? 2 : 1) * pair(K, a, b); }
  __device__ static cpx<T> L(const SweepArgs<T>& A, int s, int a, int b) {
    const int o = ((s * A.nchan + a) * A.nchan + b) * 2;
    return {T(__ldg(A.chan_dev + o)), T(__ldg(A.chan_dev + o + 1))};
  }

  // weighted sum of squares / of entry moduli of one packed block
  __device__ static T ssq_p(const T* x, int K) {
    T s = T(0), o = T(0);
#pragma unroll 1
    for (int i = 0; i < K; ++i) s = s + x[i] * x[i];
#pragma unroll 1
    for (int i = K; i < npk(K); ++i) o = o + x[i] * x[i];
    return s + (o + o);
  }
  __device__ static T ssq_w(const T* x, int K) {  // real path: strict upper triangle
    T o = T(0);
#pragma unroll 1
    for (int i = 0; i < nws(K); ++i) o = o + x[i] * x[i];
    return o + o;
  }
  __device__ static T abs_p(const T* x, int K) {
    T s = T(0), o = T(0);
#pragma unroll 1
    for (int i = 0; i < K; ++i) s = s + fabs(x[i]);
    if (CPLX) {
#pragma unroll 1
      for (int q = K; q < npk(K); q += 2) o = o + hypot(x[q], x[q + 1]);
    } else {
#pragma unroll 1
      for (int i = K; i < npk(K); ++i) o = o + fabs(x[i]);
    }
    return s + (o + o);
  }
  __device__ static void soft_entries(T* x, int K, T thr) {  // complex blocks
#pragma unroll 1
    for (int i = 0; i < K; ++i) x[i] = x[i] * soft_factor(fabs(x[i]), thr);
#pragma unroll 1
    for (int q = K; q < K * K; q += 2) {
      const T f = soft_factor(hypot(x[q], x[q + 1]), thr);
      x[q] = x[q] * f;
      x[q + 1] = x[q + 1] * f;
    }
  }

  // packed Hermitian block <-> full re / im matrices; skew Z <-> H = -i Z
  __device__ static void unpack_h(const T* x, int K, M& mr, M& mi) {
#pragma unroll 1
    for (int a = 0; a < K; ++a) {
      mr[a][a] = x[a];
      mi[a][a] = T(0);
#pragma unroll 1
      for (int b = a + 1; b < K; ++b) {
        const int q = poff(K, a, b);
        mr[a][b] = x[q];
        mi[a][b] = x[q + 1];
        mr[b][a] = x[q];
        mi[b][a] = -x[q + 1];
      }
    }
  }
  __device__ static void pack_h(const M& mr, const M& mi, int K, T* x) {
#pragma unroll 1
    for (int a = 0; a < K; ++a) {
      x[a] = mr[a][a];
#pragma unroll 1
      for (int b = a + 1; b < K; ++b) {
        const int q = poff(K, a, b);
        x[q] = mr[a][b];
        x[q + 1] = mi[a][b];
      }
    }
  }
  __device__ static void skew_to_h(const T* z, int K, M& mr, M& mi) {
#pragma unroll 1
    for (int a = 0; a < K; ++a) {
      mr[a][a] = z[a];
      mi[a][a] = T(0);
#pragma unroll 1
      for (int b = a + 1; b < K; ++b) {
        const int q = poff(K, a, b);
        mr[a][b] = z[q + 1];
        mi[a][b] = -z[q];
        mr[b][a] = z[q + 1];
        mi[b][a] = z[q];
      }
    }
  }
  __device__ static void h_to_skew(const M& mr, const M& mi, int K, T* z) {
#pragma unroll 1
    for (int a = 0; a < K; ++a) {
      z[a] = mr[a][a];
#pragma unroll 1
      for (int b = a + 1; b < K; ++b) {
        const int q = poff(K, a, b);
        z[q] = -mi[a][b];
        z[q + 1] = mr[a][b];
      }
    }
  }

  // cyclic Jacobi on the upper triangle (herm_jacobi, payload.cuh) with
  // runtime K: eigenvalues on the diagonal of ar, eigenvectors in (vr, vi)
  __device__ static cpx<T> hget(const M& ar, const M& ai, int a, int b) {
    return a < b ? cpx<T>{ar[a][b], ai[a][b]} : cpx<T>{ar[b][a], -ai[b][a]};
  }
  __device__ static void hset(M& ar, M& ai, int a, int b, cpx<T> v) {
    if (a < b) {
      ar[a][b] = v.r;
      ai[a][b] = v.i;
    } else {
      ar[b][a] = v.r;
      ai[b][a] = -v.i;
    }
  }
  __device__ static void jacobi(M& ar, M& ai, M& vr, M& vi, int K, bool want_v) {
    if (want_v) {
#pragma unroll 1
      for (int a = 0; a < K; ++a)
#pragma unroll 1
        for (int b = 0; b < K; ++b) {
          vr[a][b] = (a == b) ? T(1) : T(0);
          vi[a][b] = T(0);
        }
    }
    const T eps = sizeof(T) == 8 ? T(1e-17) : T(1e-9);
#pragma unroll 1
    for (int sweep = 0; sweep < 16; ++sweep) {
      T off = T(0), dia = T(0);
#pragma unroll 1
      for (int p = 0; p < K; ++p) {
        dia = dia + fabs(ar[p][p]);
#pragma unroll 1
        for (int q = p + 1; q < K; ++q) off = off + fabs(ar[p][q]) + fabs(ai[p][q]);
      }
      if (!(off > eps * dia)) break;
#pragma unroll 1
      for (int p = 0; p < K - 1; ++p) {
#pragma unroll 1
        for (int q = p + 1; q < K; ++q) {
          const T r = hypot(ar[p][q], ai[p][q]);
          if (!(r > T(0))) continue;
          const T rinv = T(1) / r;
          // a subnormal |a_pq| (fp32 flux blocks decaying to 0) overflows 1/r:
          // the pair is already diagonal to working precision
          if (!(rinv <= FLT_MAX_OF<T>())) continue;
          const T er = ar[p][q] * rinv, ei = -ai[p][q] * rinv;
          const T zeta = (ar[q][q] - ar[p][p]) * (T(0.5) * rinv);
          const T t = (zeta >= T(0) ? T(1) : T(-1)) / (fabs(zeta) + sqrt(T(1) + zeta * zeta));
          const T c = T(1) / sqrt(T(1) + t * t);
          const T s = t * c;
          const cpx<T> uqp = {-s * er, -s * ei}, uqq = {c * er, c * ei};
          const T tr = t * r;
          ar[p][p] = ar[p][p] - tr;
          ar[q][q] = ar[q][q] + tr;
#pragma unroll 1
          for (int k = 0; k < K; ++k) {
            if (k == p || k == q) continue;
            const cpx<T> xp = hget(ar, ai, k, p), xq = hget(ar, ai, k, q);
            hset(ar, ai, k, p, cmac(cpx<T>{c * xp.r, c * xp.i}, xq, uqp));
            hset(ar, ai, k, q, cmac(cpx<T>{s * xp.r, s * xp.i}, xq, uqq));
          }
          ar[p][q] = T(0);
          ai[p][q] = T(0);
          if (want_v) {
#pragma unroll 1
            for (int k = 0; k < K; ++k) {
              const cpx<T> xp = {vr[k][p], vi[k][p]}, xq = {vr[k][q], vi[k][q]};
              const cpx<T> np_ = cmac(cpx<T>{c * xp.r, c * xp.i}, xq, uqp);
              const cpx<T> nq_ = cmac(cpx<T>{s * xp.r, s * xp.i}, xq, uqq);
              vr[k][p] = np_.r;
              vi[k][p] = np_.i;
              vr[k][q] = nq_.r;
              vi[k][q] = nq_.i;
            }
          }
        }
      }
    }
  }
  // nuclear prox of a Hermitian matrix (herm_nuc_prox): V diag(f(lambda)) V^H
  __device__ static void nuc_prox(M& hr, M& hi, int K, T thr) {
    M ar, ai, vr, vi;
#pragma unroll 1
    for (int a = 0; a < K; ++a)
#pragma unroll 1
      for (int b = 0; b < K; ++b) {
        ar[a][b] = hr[a][b];
        ai[a][b] = hi[a][b];
      }
    jacobi(ar, ai, vr, vi, K, true);
#pragma unroll 1
    for (int a = 0; a < K; ++a)
#pragma unroll 1
      for (int b = a; b < K; ++b) {
        T sr = T(0), si = T(0);
#pragma unroll 1
        for (int k = 0; k < K; ++k) {
          const T f = soft_eig(ar[k][k], thr);
          const T pr = fma(vr[a][k], vr[b][k], vi[a][k] * vi[b][k]);
          const T pi = fma(vi[a][k], vr[b][k], -(vr[a][k] * vi[b][k]));
          sr = fma(f, pr, sr);
          si = fma(f, pi, si);
        }
        hr[a][b] = sr;
        hi[a][b] = (a == b) ? T(0) : si;
        if (a != b) {
          hr[b][a] = sr;
          hi[b][a] = -si;
        }
      }
  }
  // sum and max of the eigenvalue moduli (herm_abs_eigs)
  __device__ static void abs_eigs(M& hr, M& hi, int K, double& sum, double& mx) {
    M vr, vi;
    jacobi(hr, hi, vr, vi, K, false);
    sum = 0.0;
    mx = 0.0;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
      const double e = fabs(double(hr[k][k]));
      sum += e;
      mx = dmax(mx, e);
    }
  }

  // ---- prox, channel operators, norms (SymPolicy / HermPolicy order) -----
  __device__ static void prox_u(T* x, const SweepArgs<T>& A) {
    const int K = A.nchan, NP = npk(K);
    const T thr = A.mu;
    if (A.norm_u == NORM_L2) {
      const T f = soft_factor(sqrt(ssq_p(x, K) + ssq_p(x + NP, K)), thr);
#pragma unroll 1
      for (int i = 0; i < 2 * NP; ++i) x[i] = x[i] * f;
    } else if (A.norm_u == NORM_L12) {
#pragma unroll 1
      for (int d = 0; d < 2; ++d) {
        const T f = soft_factor(sqrt(ssq_p(x + d * NP, K)), thr);
#pragma unroll 1
        for (int i = 0; i < NP; ++i) x[d * NP + i] = x[d * NP + i] * f;
      }
    } else if (A.norm_u == NORM_L1) {
      if (CPLX) {
        soft_entries(x, K, thr);
        soft_entries(x + NP, K, thr);
      } else {
#pragma unroll 1
        for (int i = 0; i < 2 * NP; ++i) x[i] = x[i] * soft_factor(fabs(x[i]), thr);
      }
    } else if (CPLX) {
#pragma unroll 1
      for (int d = 0; d < 2; ++d) {
        M mr, mi;
        unpack_h(x + d * NP, K, mr, mi);
        nuc_prox(mr, mi, K, thr);
        pack_h(mr, mi, K, x + d * NP);
      }
    }
    if (A.has_eps) {
#pragma unroll 1
      for (int i = 0; i < 2 * NP; ++i) x[i] = x[i] / A.den_u;
    }
  }

  // [L_s, X] = P - P^H with P = L_s X (S/lindblad.py:87-107)
  __device__ static void grad_c(const T* p, T* g, const SweepArgs<T>& A) {
    const int K = A.nchan, NWS = nws(K);
    M xr, xi, pr, pi;
    if (CPLX) {
      unpack_h(p, K, xr, xi);
    } else {
#pragma unroll 1
      for (int a = 0; a < K; ++a) {
        xr[a][a] = p[a];
#pragma unroll 1
        for (int b = a + 1; b < K; ++b) xr[a][b] = xr[b][a] = p[poff(K, a, b)];
      }
    }
#pragma unroll 1
    for (int s = 0; s < A.ell; ++s) {
#pragma unroll 1
      for (int a = 0; a < K; ++a)
#pragma unroll 1
        for (int b = 0; b < K; ++b) {
          if (CPLX) {
            cpx<T> acc = {T(0), T(0)};
#pragma unroll 1
            for (int c = 0; c < K; ++c) acc = cmac(acc, L(A, s, a, c), cpx<T>{xr[c][b], xi[c][b]});
            pr[a][b] = acc.r;
            pi[a][b] = acc.i;
          } else {
            T acc = T(0);
#pragma unroll 1
            for (int c = 0; c < K; ++c) acc = fma(L(A, s, a, c).r, xr[c][b], acc);
            pr[a][b] = acc;
          }
        }
      T* z = g + s * NWS;
      if (CPLX) {
#pragma unroll 1
        for (int a = 0; a < K; ++a) z[a] = pi[a][a] + pi[a][a];
      }
#pragma unroll 1
      for (int a = 0; a < K; ++a)
#pragma unroll 1
        for (int b = a + 1; b < K; ++b) {
          if (CPLX) {
            const int q = poff(K, a, b);
            z[q] = pr[a][b] - pr[b][a];
            z[q + 1] = pi[a][b] + pi[b][a];
          } else {
            z[pair(K, a, b)] = pr[a][b] - pr[b][a];
          }
        }
    }
  }

  // T + T^H with T = sum_s Z_s L_s (S/lindblad.py:110-129)
  __device__ static void div_c(const T* y, T* d, const SweepArgs<T>& A) {
    const int K = A.nchan, NWS = nws(K);
    M tr, ti, zr, zi;
#pragma unroll 1
    for (int a = 0; a < K; ++a)
#pragma unroll 1
      for (int b = 0; b < K; ++b) tr[a][b] = ti[a][b] = T(0);
#pragma unroll 1
    for (int s = 0; s < A.ell; ++s) {
      const T* z = y + s * NWS;
#pragma unroll 1
      for (int a = 0; a < K; ++a) {
        zr[a][a] = T(0);
        zi[a][a] = CPLX ? z[a] : T(0);
#pragma unroll 1
        for (int b = a + 1; b < K; ++b) {
          if (CPLX) {
            const int q = poff(K, a, b);
            zr[a][b] = z[q];
            zi[a][b] = z[q + 1];
            zr[b][a] = -z[q];
            zi[b][a] = z[q + 1];
          } else {
            zr[a][b] = z[pair(K, a, b)];
            zr[b][a] = -zr[a][b];
          }
        }
      }
#pragma unroll 1
      for (int a = 0; a < K; ++a)
#pragma unroll 1
        for (int b = 0; b < K; ++b) {
          if (CPLX) {
            cpx<T> acc = {tr[a][b], ti[a][b]};
#pragma unroll 1
            for (int c = 0; c < K; ++c) acc = cmac(acc, cpx<T>{zr[a][c], zi[a][c]}, L(A, s, c, b));
            tr[a][b] = acc.r;
            ti[a][b] = acc.i;
          } else {
            T acc = tr[a][b];
#pragma unroll 1
            for (int c = 0; c < K; ++c) acc = fma(zr[a][c], L(A, s, c, b).r, acc);
            tr[a][b] = acc;
          }
        }
    }
#pragma unroll 1
    for (int a = 0; a < K; ++a) {
      d[a] = tr[a][a] + tr[a][a];
#pragma unroll 1
      for (int b = a + 1; b < K; ++b) {
        if (CPLX) {
          const int q = poff(K, a, b);
          d[q] = tr[a][b] + tr[b][a];
          d[q + 1] = ti[a][b] - ti[b][a];
        } else {
          d[poff(K, a, b)] = tr[a][b] + tr[b][a];
        }
      }
    }
  }

  __device__ static void prox_w(T* x, const SweepArgs<T>& A) {
    const int K = A.nchan, NWS = nws(K), NW = A.ell * NWS;
    const T thr = A.thr_w;
    if (A.norm_w == NORM_L2) {
      T s = T(0);
#pragma unroll 1
      for (int q = 0; q < A.ell; ++q) s = s + (CPLX ? ssq_p(x + q * NWS, K) : ssq_w(x + q * NWS, K));
      const T f = soft_factor(sqrt(s), thr);
#pragma unroll 1
      for (int i = 0; i < NW; ++i) x[i] = x[i] * f;
    } else if (A.norm_w == NORM_L1) {
      if (CPLX) {
#pragma unroll 1
        for (int q = 0; q < A.ell; ++q) soft_entries(x + q * NWS, K, thr);
      } else {
#pragma unroll 1
        for (int i = 0; i < NW; ++i) x[i] = x[i] * soft_factor(fabs(x[i]), thr);
      }
    } else if (CPLX) {
#pragma unroll 1
      for (int q = 0; q < A.ell; ++q) {
        M mr, mi;
        skew_to_h(x + q * NWS, K, mr, mi);
        nuc_prox(mr, mi, K, thr);
        h_to_skew(mr, mi, K, x + q * NWS);
      }
    }
    if (A.has_eps) {
#pragma unroll 1
      for (int i = 0; i < NW; ++i) x[i] = x[i] / A.den_w;
    }
  }

  __device__ static double norm_u(const T* x, const SweepArgs<T>& A) {
    const int K = A.nchan, NP = npk(K);
    const int nid = A.norm_u;
    if (nid == NORM_L2) return double(sqrt(ssq_p(x, K) + ssq_p(x + NP, K)));
    if (nid == NORM_L12) return double(sqrt(ssq_p(x, K)) + sqrt(ssq_p(x + NP, K)));
    if (nid == NORM_L1 || !CPLX) return double(abs_p(x, K) + abs_p(x + NP, K));
    double tot = 0.0;
#pragma unroll 1
    for (int d = 0; d < 2; ++d) {
      M mr, mi;
      unpack_h(x + d * NP, K, mr, mi);
      double s, m;
      abs_eigs(mr, mi, K, s, m);
      tot += s;
    }
    return tot;
  }

  __device__ static double norm_w(const T* x, const SweepArgs<T>& A) {
    const int K = A.nchan, NWS = nws(K);
    const int nid = A.norm_w;
    if (!CPLX) {
      T s = T(0);
      if (nid == NORM_L2) {
#pragma unroll 1
        for (int q = 0; q < A.ell; ++q) s = s + ssq_w(x + q * NWS, K);
        return double(sqrt(s));
      }
#pragma unroll 1
      for (int i = 0; i < A.ell * NWS; ++i) s = s + fabs(x[i]);
      return double(s + s);
    }
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll 1
      for (int q = 0; q < A.ell; ++q) s = s + ssq_p(x + q * NWS, K);
      return double(sqrt(s));
    }
    if (nid == NORM_L1) {
      T s = T(0);
#pragma unroll 1
      for (int q = 0; q < A.ell; ++q) s = s + abs_p(x + q * NWS, K);
      return double(s);
    }
    double tot = 0.0;
#pragma unroll 1
    for (int q = 0; q < A.ell; ++q) {
      M mr, mi;
      skew_to_h(x + q * NWS, K, mr, mi);
      double s, m;
      abs_eigs(mr, mi, K, s, m);
      tot += s;
    }
    return tot;
  }

  __device__ static void dual_u(const T* g, const SweepArgs<T>& A, double& gmax, double& pen) {
    const int K = A.nchan, NP = npk(K);
    const int nid = A.norm_u;
    if (nid == NORM_L2) {
      const double v = double(sqrt(ssq_p(g, K) + ssq_p(g + NP, K)));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - 1.0, 0.0));
    } else if (nid == NORM_L12) {
#pragma unroll 1
      for (int d = 0; d < 2; ++d) {
        const double v = double(sqrt(ssq_p(g + d * NP, K)));
        gmax = dmax(gmax, v);
        pen += sq(dmax(v - 1.0, 0.0));
      }
    } else if (nid == NORM_L1 || !CPLX) {
#pragma unroll 1
      for (int d = 0; d < 2; ++d) {
        const T* b = g + d * NP;
        if (CPLX) {
#pragma unroll 1
          for (int i = 0; i < K; ++i) {
            const double v = double(fabs(b[i]));
            gmax = dmax(gmax, v);
            pen += sq(dmax(v - 1.0, 0.0));
          }
#pragma unroll 1
          for (int q = K; q < NP; q += 2) {
            const double v = double(hypot(b[q], b[q + 1]));
            gmax = dmax(gmax, v);
            pen += 2.0 * sq(dmax(v - 1.0, 0.0));
          }
        } else {
#pragma unroll 1
          for (int i = 0; i < NP; ++i) {
            const double v = double(fabs(b[i]));
            gmax = dmax(gmax, v);
            pen += (i < K ? 1.0 : 2.0) * sq(dmax(v - 1.0, 0.0));
          }
        }
      }
    } else {
#pragma unroll 1
      for (int d = 0; d < 2; ++d) {
        M mr, mi;
        unpack_h(g + d * NP, K, mr, mi);
        double s, m;
        abs_eigs(mr, mi, K, s, m);
        gmax = dmax(gmax, m);
        pen += sq(dmax(m - 1.0, 0.0));
      }
    }
  }

  __device__ static void dual_w(const T* g, const SweepArgs<T>& A, double& gmax, double& pen) {
    const int K = A.nchan, NWS = nws(K);
    const int nid = A.norm_w;
    const double alpha = A.alpha;
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll 1
      for (int q = 0; q < A.ell; ++q) s = s + (CPLX ? ssq_p(g + q * NWS, K) : ssq_w(g + q * NWS, K));
      const double v = double(sqrt(s));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - alpha, 0.0));
      return;
    }
    if (!CPLX) {
#pragma unroll 1
      for (int i = 0; i < A.ell * NWS; ++i) {
        const double v = double(fabs(g[i]));
        gmax = dmax(gmax, v);
        pen += 2.0 * sq(dmax(v - alpha, 0.0));
      }
      return;
    }
#pragma unroll 1
    for (int q = 0; q < A.ell; ++q) {
      const T* z = g + q * NWS;
      if (nid == NORM_L1) {
#pragma unroll 1
        for (int i = 0; i < K; ++i) {
          const double v = double(fabs(z[i]));
          gmax = dmax(gmax, v);
          pen += sq(dmax(v - alpha, 0.0));
        }
#pragma unroll 1
        for (int p = K; p < NWS; p += 2) {
          const double v = double(hypot(z[p], z[p + 1]));
          gmax = dmax(gmax, v);
          pen += 2.0 * sq(dmax(v - alpha, 0.0));
        }
      } else {
        M mr, mi;
        skew_to_h(z, K, mr, mi);
        double s, m;
        abs_eigs(mr, mi, K, s, m);
        gmax = dmax(gmax, m);
        pen += sq(dmax(m - alpha, 0.0));
      }
    }
  }
};

// cell-level steps shared by the runtime-size payloads D (DynVec, DynMat)
template <class D, typename T>
struct DynCell {
  // phi(i, j) of the read iterate into p (zeros off the grid)
  __device__ static void load_phi(const SweepArgs<T>& A, int i, int j, T* p) {
    const int K = D::np(A);
    const bool in = i < A.n && j < A.n;
    const int64_t o = cell_off(A, i, j);
#pragma unroll 1
    for (int c = 0; c < K; ++c) p[c] = in ? ldg(A.a.phi + c * A.plane + o) : T(0);
  }

  // u'(i, j) = prox_u(grad phi * mu + u) of the read iterate
  // (S/solver.py:221-224, S/spatial.py:80-86); uo = u(i, j)
  __device__ static void flux(const SweepArgs<T>& A, int i, int j, T* uo, T* un, T* ph, T* pn) {
    const int K = D::np(A);
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
    D::prox_u(un, A);
  }
};

// One PDHG iteration (CHECK: + the R^k partials), same band / partial layout
// as sweep_kernel so the engine launches it in its place.
template <class D, typename T, bool CHECK>
__global__ void __launch_bounds__(128) dyn_sweep_kernel(const __grid_constant__ SweepArgs<T> A) {
  using C = DynCell<D, T>;
  __shared__ double sred[32 * 4];
  const int K = D::np(A), L = D::nw(A);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const bool live = j < n;
  const int band = A.band0 + int(blockIdx.y) * A.band_step;
  const int gr0 = A.row_begin + band * A.rows_per_block;
  const int gr1 = min(gr0 + A.rows_per_block, A.row_end);
  const int64_t pl = A.plane;

  constexpr int NPM = D::NPMAX, NWM = D::NWMAX;
  T ph[NPM], pn[NPM], uo[2 * NPM], un[2 * NPM];
  T nuo[2 * NPM], nun[2 * NPM];  // a neighbour cell's flux
  T uxb_prev[NPM], dux_prev[NPM], lub[NPM], ldu[NPM], rhs[NPM];
  T wo[NWM], wn[NWM], wt[NWM];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};

  if (live && gr0 > 0 && gr0 < gr1) {
    // ubar_x / du_x of the row above the band, from the read-only iterate
    C::flux(A, gr0 - 1, j, nuo, nun, pn, rhs);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      uxb_prev[c] = (nun[c] + nun[c]) - nuo[c];
      dux_prev[c] = nun[c] - nuo[c];
    }
  }
  for (int i = gr0; live && i < gr1; ++i) {
    const int64_t o = cell_off(A, i, j);
    C::flux(A, i, j, uo, un, ph, pn);
    if (j > 0) {
      C::flux(A, i, j - 1, nuo, nun, pn, rhs);
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
        acc[0] += D::wp(A, c) * (double(dx) * double(dx) + double(dy) * double(dy));
        T d = dx;
        if (i > 0) d = d - dux_prev[c];
        d = d + dy;
        if (j > 0) d = d - ldu[c];
        const T cross = d * A.inv_dx + pn[c];
        dux_prev[c] = dx;
        acc[2] += D::wp(A, c) * double(rhs[c]) * double(rhs[c]);
        acc[3] += D::wp(A, c) * double(rhs[c]) * double(cross);
      }
#pragma unroll 1
      for (int e = 0; e < L; ++e) acc[1] += D::ww(A, e) * double(wt[e]) * double(wt[e]);
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
template <class D, typename T>
__global__ void __launch_bounds__(128) dyn_evaluate_kernel(const __grid_constant__ SweepArgs<T> A) {
  using C = DynCell<D, T>;
  __shared__ double sred[32 * 8];
  const int K = D::np(A), L = D::nw(A);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const int64_t pl = A.plane;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // PU PW SU2 SW2 SCON SPHID PENU PENW
  double mx[2] = {0.0, 0.0};
  T u[2 * D::NPMAX], ph[D::NPMAX], pn[D::NPMAX], con[D::NPMAX], w[D::NWMAX];
  for (int i = A.row_begin + blockIdx.y; j < n && i < A.row_end; i += gridDim.y) {
    const int64_t o = cell_off(A, i, j), oxm = cell_off(A, i - 1, j);
#pragma unroll 1
    for (int q = 0; q < 2 * K; ++q) u[q] = ldg(A.a.u + q * pl + o);
#pragma unroll 1
    for (int e = 0; e < L; ++e) w[e] = ldg(A.a.w + e * pl + o);
    C::load_phi(A, i, j, ph);
    s[0] += D::norm_u(u, A);
    double su = 0.0;
#pragma unroll 1
    for (int c = 0; c < K; ++c)
      su += D::wp(A, c) * (double(u[c]) * double(u[c]) + double(u[K + c]) * double(u[K + c]));
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
    for (int e = 0; e < L; ++e) sw += D::ww(A, e) * double(w[e]) * double(w[e]);
    s[3] += sw;
    D::div_c(w, pn, A);
    double sc = 0.0, sp = 0.0;
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      con[c] = con[c] + pn[c];
      sc += D::wp(A, c) * double(con[c]) * double(con[c]);
      sp += D::wp(A, c) * double(ph[c]) * double(ldg(A.diff + c * pl + o));
    }
    s[4] += sc;
    s[5] += sp;
    // dual norms of grad phi (u[] reused for the gradient) and grad_c phi
    const bool hx = i + 1 < n, hy = j + 1 < n;
    C::load_phi(A, i + 1, j, pn);
#pragma unroll 1
    for (int c = 0; c < K; ++c) u[c] = hx ? (pn[c] - ph[c]) * A.inv_dx : T(0);
    C::load_phi(A, i, j + 1, pn);
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
template <class D, typename T>
__global__ void __launch_bounds__(128) dyn_residual_kernel(const __grid_constant__ SweepArgs<T> A) {
  __shared__ double sred[32 * 4];
  const int K = D::np(A), L = D::nw(A);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = A.n;
  const int64_t pl = A.plane;
  double s[4] = {0, 0, 0, 0};
  T dw[D::NWMAX], dv[D::NPMAX];
  for (int i = A.row_begin + blockIdx.y; j < n && i < A.row_end; i += gridDim.y) {
    const int64_t o = cell_off(A, i, j), oxm = cell_off(A, i - 1, j);
    auto du = [&](int comp, int64_t off) { return A.b.u[comp * pl + off] - A.a.u[comp * pl + off]; };
#pragma unroll 1
    for (int e = 0; e < L; ++e) {
      dw[e] = A.b.w[e * pl + o] - A.a.w[e * pl + o];
      s[1] += D::ww(A, e) * double(dw[e]) * double(dw[e]);
    }
    D::div_c(dw, dv, A);
#pragma unroll 1
    for (int c = 0; c < K; ++c) {
      const T dx = du(c, o), dy = du(K + c, o);
      s[0] += D::wp(A, c) * (double(dx) * double(dx) + double(dy) * double(dy));
      T d = dx;
      if (i > 0) d = d - du(c, oxm);
      d = d + dy;
      if (j > 0) d = d - du(K + c, o - 1);
      const T cross = d * A.inv_dx + dv[c];
      const T dp = A.b.phi[c * pl + o] - A.a.phi[c * pl + o];
      s[2] += D::wp(A, c) * double(dp) * double(dp);
      s[3] += D::wp(A, c) * double(dp) * double(cross);
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
