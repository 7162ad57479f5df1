// Per-cell payload policies: how one grid cell's flux / potential payload is
// shrunk (prox), mapped by the channel operator and measured.  The sweep
// kernel (sweep.cuh) is generic over these.
//
//   VecPolicy<T,K,HASW>   scalar (K=1, no w) and k-channel vector transport
//                         (S/shrink.py:120-136, S/graph.py:105-123)
//   SymPolicy<T,K>        real-symmetric matrix path (S/solver.py:415-423,
//                         S/lindblad.py:87-129): phi/u/diff packed upper
//                         triangles, w packed strict upper (antisymmetric)
//   HermPolicy<T,K>       complex Hermitian matrix path incl. the nuclear
//                         eigen-shrink (S/shrink.py:161-196)
//
// Packed storage keeps the Hermitian / skew structure exact by construction
// (the reference enforces it with hermitian_part/skew_part, S/fields.py:66-79);
// sums of squares and inner products weight off-diagonal reals by 2 so they
// equal the full-matrix quantities.
#pragma once

#include "common.cuh"

namespace otfx {

template <typename T>
__device__ __forceinline__ T soft_factor(T r, T thr) {
  // S/shrink.py:120-136: r = max(r, tiny); r = thr / r; r = 1 - r; r = max(r, 0).
  // For r <= thr the reference's value is exactly 0 (thr/r >= 1 rounds to >= 1,
  // and thr/tiny or the fp32 thr/0 = inf give 0 too), so the division only runs
  // where it matters; for r > thr, 1 - thr/r >= 0 and the max is a no-op.
  // Bit-identical to the reference's sequence, without fp32 div-by-zero slow paths.
  const T q = thr / (r > thr ? r : T(1));
  return r > thr ? T(1) - q : T(0);
}

template <typename T>
__device__ __forceinline__ T sq(T x) { return x * x; }

// Sum of squares in NumPy's einsum order.  The reference's block norms are
// np.einsum("...i,...i->...", x, x) over the contiguous payload
// (S/shrink.py:88-104), whose inner loop (sum_of_products_contig_contig_
// outstride0_two, baseline SSE2 build: two double lanes, multiply then add)
// runs blocks of 8 elements as  lane += x[6+l]^2, x[4+l]^2, x[2+l]^2, x[l]^2,
// then the rest two at a time, and returns lane0 + lane1.  `len` (<= N) is
// the runtime block length; entries past it are not touched.
// tools/einsum_order.py checks this model against NumPy.
template <int N, typename T>
__device__ __forceinline__ T np_sumsq(const T* x, int len) {
  T a0 = T(0), a1 = T(0);
  int done = 0;
#pragma unroll
  for (int b = 0; b + 8 <= N; b += 8) {
    if (b + 8 <= len) {
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        a0 = x[b + 2 * q] * x[b + 2 * q] + a0;
        a1 = x[b + 2 * q + 1] * x[b + 2 * q + 1] + a1;
      }
      done = b + 8;
    }
  }
#pragma unroll
  for (int i = 0; i < N; i += 2) {
    if (i >= done && i < len) a0 = x[i] * x[i] + a0;
    if (i + 1 < N && i + 1 >= done && i + 1 < len) a1 = x[i + 1] * x[i + 1] + a1;
  }
  return a0 + a1;
}

// ===========================================================================
// vector / scalar payloads
// ===========================================================================

// LC_: edge capacity of the instantiation (0 = the complete graph's
// k(k-1)/2); sparse graphs (chains, cycles, stars: ell <= k) get LC_ = k, so
// the edge loops and the coefficient block are sized for the graph they run
template <typename T, int K_, bool HASW, int LC_ = 0>
struct VecPolicy {
  static constexpr int K = K_;
  static constexpr int NP = K;
  static constexpr int LMAX =
      HASW ? (LC_ > 0 ? LC_ : (K * (K - 1) / 2 > 0 ? K * (K - 1) / 2 : 1)) : 1;
  static constexpr int NWS = 1;                 // reals per channel block (edge)
  static constexpr int NW = HASW ? LMAX : 0;
  static constexpr int NWA = HASW ? LMAX : 1;   // array extent
  static constexpr bool HAS_W = HASW;
  static constexpr int NCOEF = K * LMAX;        // graph D/c entries the kernels read

  __device__ static __forceinline__ double wp(int) { return 1.0; }
  __device__ static __forceinline__ double ww(int) { return 1.0; }

  // u payload x[dir][c]; prox of mu*||.|| then the eps scaling (S/shrink.py:208-240)
  template <class PA>
  __device__ static void prox_u(T (&x)[2][NP], const PA& A) {
    const T thr = A.mu;
    if (A.norm_u == NORM_L2) {
      // the (2, k) payload block in C order (S/shrink.py:107-108)
      const T s = np_sumsq<2 * K>(&x[0][0], 2 * K);
      const T f = soft_factor(sqrt(s), thr);
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int c = 0; c < K; ++c) x[d][c] = x[d][c] * f;
    } else if (A.norm_u == NORM_L12) {
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const T f = soft_factor(sqrt(x[0][c] * x[0][c] + x[1][c] * x[1][c]), thr);
        x[0][c] = x[0][c] * f;
        x[1][c] = x[1][c] * f;
      }
    } else {
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int c = 0; c < K; ++c) x[d][c] = x[d][c] * soft_factor(fabs(x[d][c]), thr);
    }
    if (A.has_eps) {
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int c = 0; c < K; ++c) x[d][c] = x[d][c] / A.den_u;
    }
  }

  // graph gradient diag(1/c) D^T phi  (S/graph.py:105-114).  The reference
  // computes it as the matmul (n^2, k) @ (k, ell), which NumPy hands to
  // OpenBLAS: dgemm accumulates every output with a fused multiply-add chain
  // over k in ascending order from 0, and for ell = 1 (k = 2, a single edge)
  // the matrix-vector kernel runs the chain in descending order
  // (tools/blas_order.py checks both against NumPy).  The same chains here
  // make the channel update bit-identical to the reference.
  template <class PA>
  __device__ static void grad_c(const T (&p)[NP], T (&g)[NWA], const PA& A) {
#pragma unroll
    for (int e = 0; e < NWA; ++e) {
      T s = T(0);
      if constexpr (K == 2) {
        s = fma(p[1], T(A.coef[1 * LMAX + e]), s);
        s = fma(p[0], T(A.coef[0 * LMAX + e]), s);
      } else {
#pragma unroll
        for (int c = 0; c < K; ++c) s = fma(p[c], T(A.coef[c * LMAX + e]), s);
      }
      g[e] = s;
    }
  }

  // graph divergence -D diag(1/c) y  (S/graph.py:117-123): the matmul
  // (n^2, ell) @ (ell, k), an ascending fused multiply-add chain over ell
  template <class PA>
  __device__ static void div_c(const T (&y)[NWA], T (&d)[NP], const PA& A) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      T s = T(0);
#pragma unroll
      for (int e = 0; e < NWA; ++e) s = fma(y[e], T(-A.coef[c * LMAX + e]), s);
      d[c] = s;
    }
  }

  template <class PA>
  __device__ static void prox_w(T (&x)[NWA], const PA& A) {
    const T thr = A.thr_w;
    if (A.norm_w == NORM_L2) {
      const T s = np_sumsq<NWA>(x, A.ell);
      const T f = soft_factor(sqrt(s), thr);
#pragma unroll
      for (int e = 0; e < NWA; ++e) x[e] = x[e] * f;
    } else {
#pragma unroll
      for (int e = 0; e < NWA; ++e) x[e] = x[e] * soft_factor(fabs(x[e]), thr);
    }
    if (A.has_eps) {
#pragma unroll
      for (int e = 0; e < NWA; ++e) x[e] = x[e] / A.den_w;
    }
  }

  // per-cell norm value (S/shrink.py:243-259)
  __device__ static double norm_u(const T (&x)[2][NP], int nid) {
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int c = 0; c < K; ++c) s = s + x[d][c] * x[d][c];
      return double(sqrt(s));
    }
    if (nid == NORM_L12) {
      T s = T(0);
#pragma unroll
      for (int c = 0; c < K; ++c) s = s + sqrt(x[0][c] * x[0][c] + x[1][c] * x[1][c]);
      return double(s);
    }
    T s = T(0);
#pragma unroll
    for (int d = 0; d < 2; ++d)
#pragma unroll
      for (int c = 0; c < K; ++c) s = s + fabs(x[d][c]);
    return double(s);
  }

  __device__ static double norm_w(const T (&x)[NWA], int nid) {
    T s = T(0);
    if (nid == NORM_L2) {
#pragma unroll
      for (int e = 0; e < NWA; ++e) s = s + x[e] * x[e];
      return double(sqrt(s));
    }
#pragma unroll
    for (int e = 0; e < NWA; ++e) s = s + fabs(x[e]);
    return double(s);
  }

  // dual norms of the shrink blocks of grad phi (S/shrink.py:262-283):
  // running max and the eps penalty sum of (g - bound)_+^2
  __device__ static void dual_u(const T (&g)[2][NP], int nid, double& gmax, double& pen) {
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int c = 0; c < K; ++c) s = s + g[d][c] * g[d][c];
      const double v = double(sqrt(s));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - 1.0, 0.0));
    } else if (nid == NORM_L12) {
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const double v = double(sqrt(g[0][c] * g[0][c] + g[1][c] * g[1][c]));
        gmax = dmax(gmax, v);
        pen += sq(dmax(v - 1.0, 0.0));
      }
    } else {
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double v = double(fabs(g[d][c]));
          gmax = dmax(gmax, v);
          pen += sq(dmax(v - 1.0, 0.0));
        }
    }
  }

  __device__ static void dual_w(const T (&g)[NWA], int nid, int ell, double alpha, double& gmax,
                                double& pen) {
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int e = 0; e < NWA; ++e) s = s + g[e] * g[e];
      const double v = double(sqrt(s));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - alpha, 0.0));
    } else {
#pragma unroll
      for (int e = 0; e < NWA; ++e) {
        if (e < ell) {
          const double v = double(fabs(g[e]));
          gmax = dmax(gmax, v);
          pen += sq(dmax(v - alpha, 0.0));
        }
      }
    }
  }
};

// ===========================================================================
// small complex helpers for the matrix payloads
// ===========================================================================

template <typename T>
struct cpx {
  T r, i;
};
template <typename T>
__device__ __forceinline__ cpx<T> cmul(cpx<T> a, cpx<T> b) {
  return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r};
}
template <typename T>
__device__ __forceinline__ cpx<T> cadd(cpx<T> a, cpx<T> b) { return {a.r + b.r, a.i + b.i}; }
// acc + a*b with fused multiply-adds (4 FMA instead of 4 MUL + 4 ADD).  The
// library is built with --fmad=false so the vector and scalar paths round
// exactly like the NumPy reference (bit-identical iterates); the matrix
// payloads, whose reference runs einsum / LAPACK with their own summation
// orders (parity 1e-10), opt in for the Lindblad commutators and the
// eigensolver.
template <typename T>
__device__ __forceinline__ cpx<T> cmac(cpx<T> acc, cpx<T> a, cpx<T> b) {
  return {fma(a.r, b.r, fma(-a.i, b.i, acc.r)), fma(a.r, b.i, fma(a.i, b.r, acc.i))};
}

// packed index of the pair (a<b) in row-major order over the strict upper triangle
template <int K>
__host__ __device__ constexpr int pair_index(int a, int b) {
  return a * K - a * (a + 1) / 2 + (b - a - 1);
}

// Cyclic Jacobi eigensolver for a K x K complex Hermitian matrix held in
// registers (re/im arrays).  Only the diagonal and the strict upper triangle
// are read or maintained (the lower triangle is dead: A stays Hermitian, so a
// rotation of the (p, q) plane updates a_pp, a_qq in closed form and each
// off-plane pair (a_kp, a_kq) once — a third of the flops and half the live
// registers of updating A U and U^H A in full).  On return ar[k][k] hold the
// eigenvalues and (vr, vi) the eigenvectors (columns) when WANT_V.  The
// reference calls LAPACK *heevd (S/shrink.py:164); eigenvalues and the
// reconstructed prox agree to rounding, the GPU tests bound it at 1e-10.
template <typename T, int K>
__device__ __forceinline__ cpx<T> herm_get(const T (&ar)[K][K], const T (&ai)[K][K], int a, int b) {
  // A_ab from the upper triangle (a != b; indices are compile-time after unrolling)
  return a < b ? cpx<T>{ar[a][b], ai[a][b]} : cpx<T>{ar[b][a], -ai[b][a]};
}
template <typename T, int K>
__device__ __forceinline__ void herm_set(T (&ar)[K][K], T (&ai)[K][K], int a, int b, cpx<T> v) {
  if (a < b) {
    ar[a][b] = v.r;
    ai[a][b] = v.i;
  } else {
    ar[b][a] = v.r;
    ai[b][a] = -v.i;
  }
}

template <typename T, int K, bool WANT_V>
__device__ void herm_jacobi(T (&ar)[K][K], T (&ai)[K][K], T (&vr)[K][K], T (&vi)[K][K]) {
  if (WANT_V) {
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) {
        vr[a][b] = (a == b) ? T(1) : T(0);
        vi[a][b] = T(0);
      }
  }
  const T eps = sizeof(T) == 8 ? T(1e-17) : T(1e-9);
  for (int sweep = 0; sweep < 16; ++sweep) {
    T off = T(0), dia = T(0);
#pragma unroll
    for (int p = 0; p < K; ++p) {
      dia = dia + fabs(ar[p][p]);
#pragma unroll
      for (int q = p + 1; q < K; ++q) off = off + fabs(ar[p][q]) + fabs(ai[p][q]);
    }
    if (!(off > eps * dia)) break;
#pragma unroll
    for (int p = 0; p < K - 1; ++p) {
#pragma unroll
      for (int q = p + 1; q < K; ++q) {
        const T r = hypot(ar[p][q], ai[p][q]);
        if (!(r > T(0))) continue;
        // phase e^{-i phi} = conj(a_pq)/r
        const T rinv = T(1) / r;
        // a subnormal |a_pq| (fp32 flux blocks decaying to 0) overflows 1/r:
        // the pair is already diagonal to working precision
        if (!(rinv <= FLT_MAX_OF<T>())) continue;
        const T er = ar[p][q] * rinv, ei = -ai[p][q] * rinv;
        const T zeta = (ar[q][q] - ar[p][p]) * (T(0.5) * rinv);
        const T t = (zeta >= T(0) ? T(1) : T(-1)) / (fabs(zeta) + sqrt(T(1) + zeta * zeta));
        const T c = T(1) / sqrt(T(1) + t * t);
        const T s = t * c;
        // U on columns (p,q): U_pp=c, U_pq=s, U_qp=-s e, U_qq=c e   (e = e^{-i phi})
        const cpx<T> uqp = {-s * er, -s * ei}, uqq = {c * er, c * ei};
        // A' = U^H A U: a'_pp = a_pp - t r, a'_qq = a_qq + t r, a'_pq = 0, and
        // for k outside the plane (a'_kp, a'_kq) = (a_kp, a_kq) U restricted to (p, q)
        const T tr = t * r;
        ar[p][p] = ar[p][p] - tr;
        ar[q][q] = ar[q][q] + tr;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (k == p || k == q) continue;
          const cpx<T> xp = herm_get(ar, ai, k, p), xq = herm_get(ar, ai, k, q);
          herm_set(ar, ai, k, p, cmac(cpx<T>{c * xp.r, c * xp.i}, xq, uqp));
          herm_set(ar, ai, k, q, cmac(cpx<T>{s * xp.r, s * xp.i}, xq, uqq));
        }
        ar[p][q] = T(0);
        ai[p][q] = T(0);
        if (WANT_V) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const cpx<T> xp = {vr[k][p], vi[k][p]}, xq = {vr[k][q], vi[k][q]};
            const cpx<T> np_ = cmac(cpx<T>{c * xp.r, c * xp.i}, xq, uqp);
            const cpx<T> nq_ = cmac(cpx<T>{s * xp.r, s * xp.i}, xq, uqq);
            vr[k][p] = np_.r; vi[k][p] = np_.i;
            vr[k][q] = nq_.r; vi[k][q] = nq_.i;
          }
        }
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ T soft_eig(T lam, T thr) {
  // np.sign(lam) * max(|lam| - thr, 0)  (S/shrink.py:167)
  const T m = maxT(fabs(lam) - thr, T(0));
  return lam > T(0) ? m : (lam < T(0) ? -m : T(0));
}

// Nuclear prox of a Hermitian K x K matrix given as full re/im arrays; the
// result overwrites (hr, hi) and is exactly Hermitian.
template <typename T, int K>
__device__ void herm_nuc_prox(T (&hr)[K][K], T (&hi)[K][K], T thr) {
  if constexpr (K == 2) {
    // closed form: f(X) = (f+ + f-)/2 I + (f+ - f-)/(2r) (X - m I)
    const T a = hr[0][0], d = hr[1][1];
    const T m = (a + d) * T(0.5);
    const T h = (a - d) * T(0.5);
    const T r = hypot(h, hypot(hr[0][1], hi[0][1]));
    const T fp = soft_eig(m + r, thr), fm = soft_eig(m - r, thr);
    const T al = (fp + fm) * T(0.5);
    T be;
    if (r > T(0)) {
      if (m - r > thr) be = T(1);               // both eigenvalues shifted by -thr
      else if (m + r < -thr) be = T(1);         // both shifted by +thr
      else be = (fp - fm) / (r + r);
    } else {
      be = T(0);
    }
    hr[0][0] = al + be * h;
    hr[1][1] = al - be * h;
    hr[0][1] = be * hr[0][1];
    hi[0][1] = be * hi[0][1];
    hr[1][0] = hr[0][1];
    hi[1][0] = -hi[0][1];
    hi[0][0] = hi[1][1] = T(0);
  } else {
  // Spectral enclosure first: with m = tr X / K every eigenvalue lies within
  // rho = sqrt((K-1)/K) ||X - m I||_F of m.  When the whole interval
  // [m - rho, m + rho] is on one piece of the soft threshold, the prox is
  // X - thr I, X + thr I or 0 without an eigensolve (the reference's
  // V diag(f) V^H equals these to rounding).  The enclosure is widened by a
  // relative 1e-12 so rounding in rho cannot put a boundary eigenvalue on
  // the wrong piece; cells on the boundary take the Jacobi path.
#ifndef OTFX_NUC_ENCLOSURE
#define OTFX_NUC_ENCLOSURE 1
#endif
  if (OTFX_NUC_ENCLOSURE) {
    T tr = T(0);
#pragma unroll
    for (int a = 0; a < K; ++a) tr = tr + hr[a][a];
    const T m = tr * (T(1) / T(K));
    T f2 = T(0);
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const T d = hr[a][a] - m;
      f2 = fma(d, d, f2);
#pragma unroll
      for (int b = a + 1; b < K; ++b) f2 = fma(T(2) * hr[a][b], hr[a][b], fma(T(2) * hi[a][b], hi[a][b], f2));
    }
    const T rho = sqrt(f2 * (T(K - 1) / T(K))) * T(1 + 1e-12) + fabs(m) * T(1e-12);
    const int piece = (m - rho > thr) ? 1 : ((m + rho < -thr) ? -1 : ((m + rho < thr && m - rho > -thr) ? 0 : 2));
    if (piece != 2) {
      const T sh = piece == 1 ? -thr : thr;
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          if (piece == 0) {
            hr[a][b] = T(0);
            hi[a][b] = T(0);
          } else if (a == b) {
            hr[a][b] = hr[a][b] + sh;
            hi[a][b] = T(0);
          }
        }
      return;
    }
  }
  T ar[K][K], ai[K][K], vr[K][K], vi[K][K];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) {
      ar[a][b] = hr[a][b];
      ai[a][b] = hi[a][b];
    }
  herm_jacobi<T, K, true>(ar, ai, vr, vi);
  T f[K];
#pragma unroll
  for (int k = 0; k < K; ++k) f[k] = soft_eig(ar[k][k], thr);
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = a; b < K; ++b) {
      T sr = T(0), si = T(0);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        // f_k V_ak conj(V_bk)
        const T pr = fma(vr[a][k], vr[b][k], vi[a][k] * vi[b][k]);
        const T pi = fma(vi[a][k], vr[b][k], -(vr[a][k] * vi[b][k]));
        sr = fma(f[k], pr, sr);
        si = fma(f[k], pi, si);
      }
      hr[a][b] = sr;
      hi[a][b] = (a == b) ? T(0) : si;
      if (a != b) {
        hr[b][a] = sr;
        hi[b][a] = -si;
      }
    }
  }
}

// eigenvalue magnitudes of a Hermitian matrix: sum and max (norm / dual norm)
template <typename T, int K>
__device__ void herm_abs_eigs(const T (&hr)[K][K], const T (&hi)[K][K], double& sum, double& mx) {
  if constexpr (K == 2) {
    const T m = (hr[0][0] + hr[1][1]) * T(0.5);
    const T h = (hr[0][0] - hr[1][1]) * T(0.5);
    const T r = hypot(h, hypot(hr[0][1], hi[0][1]));
    const double e1 = fabs(double(m + r)), e2 = fabs(double(m - r));
    sum = e1 + e2;
    mx = dmax(e1, e2);
  } else {
  T ar[K][K], ai[K][K], vr[K][K], vi[K][K];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) {
      ar[a][b] = hr[a][b];
      ai[a][b] = hi[a][b];
    }
  herm_jacobi<T, K, false>(ar, ai, vr, vi);
  sum = 0.0;
  mx = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double e = fabs(double(ar[k][k]));
    sum += e;
    mx = dmax(mx, e);
  }
  }
}

// ===========================================================================
// matrix payloads
// ===========================================================================

// Real-symmetric path.  phi/diff/u-direction block: NP = K(K+1)/2 reals
// (diagonal first, then the strict upper triangle row-major); w block:
// K(K-1)/2 reals (strict upper triangle of an antisymmetric matrix).
template <typename T, int K_, int LM_ = 4>
struct SymPolicy {
  static constexpr int K = K_;
  static constexpr int NP = K * (K + 1) / 2;
  static constexpr int NWS = K * (K - 1) / 2;
  static constexpr int LMAX = LM_;  // Lindblad-matrix capacity (2 or 4)
  static constexpr int NW = LMAX * NWS;
  static constexpr int NWA = NW;
  static constexpr bool HAS_W = true;
  static constexpr int NCOEF = 0;  // Lindblad stack stays in parameter space

  __device__ static __forceinline__ double wp(int i) { return i < K ? 1.0 : 2.0; }
  __device__ static __forceinline__ double ww(int) { return 2.0; }

  __device__ static __forceinline__ void unpack(const T (&x)[NP], T (&m)[K][K]) {
#pragma unroll
    for (int a = 0; a < K; ++a) m[a][a] = x[a];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) m[a][b] = m[b][a] = x[K + pair_index<K>(a, b)];
  }

  // weighted sum of squares of one packed block (full-matrix Frobenius^2)
  __device__ static __forceinline__ T ssq_p(const T* x) {
    T s = T(0);
#pragma unroll
    for (int i = 0; i < K; ++i) s = s + x[i] * x[i];
    T o = T(0);
#pragma unroll
    for (int i = K; i < NP; ++i) o = o + x[i] * x[i];
    return s + (o + o);
  }
  __device__ static __forceinline__ T ssq_w(const T* x) {
    T o = T(0);
#pragma unroll
    for (int i = 0; i < NWS; ++i) o = o + x[i] * x[i];
    return o + o;
  }
  __device__ static __forceinline__ T abs_p(const T* x) {
    T s = T(0), o = T(0);
#pragma unroll
    for (int i = 0; i < K; ++i) s = s + fabs(x[i]);
#pragma unroll
    for (int i = K; i < NP; ++i) o = o + fabs(x[i]);
    return s + (o + o);
  }

  template <class PA>
  __device__ static void prox_u(T (&x)[2][NP], const PA& A) {
    const T thr = A.mu;
    if (A.norm_u == NORM_L2) {
      const T f = soft_factor(sqrt(ssq_p(x[0]) + ssq_p(x[1])), thr);
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int i = 0; i < NP; ++i) x[d][i] = x[d][i] * f;
    } else if (A.norm_u == NORM_L12) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const T f = soft_factor(sqrt(ssq_p(x[d])), thr);
#pragma unroll
        for (int i = 0; i < NP; ++i) x[d][i] = x[d][i] * f;
      }
    } else {
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int i = 0; i < NP; ++i) x[d][i] = x[d][i] * soft_factor(fabs(x[d][i]), thr);
    }
    if (A.has_eps) {
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int i = 0; i < NP; ++i) x[d][i] = x[d][i] / A.den_u;
    }
  }

  template <class PA>
  __device__ static __forceinline__ T L(const PA& A, int s, int a, int b) {
    return T(A.coef[((s * K + a) * K + b) * 2]);
  }

  // [L_s, X] = P - P^T with P = L_s X  (S/lindblad.py:87-107)
  template <class PA>
  __device__ static void grad_c(const T (&p)[NP], T (&g)[NWA], const PA& A) {
    T X[K][K];
    unpack(p, X);
#pragma unroll
    for (int s = 0; s < LMAX; ++s) {
      T P[K][K];
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          T acc = T(0);
#pragma unroll
          for (int c = 0; c < K; ++c) acc = fma(L(A, s, a, c), X[c][b], acc);
          P[a][b] = acc;
        }
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = a + 1; b < K; ++b) g[s * NWS + pair_index<K>(a, b)] = P[a][b] - P[b][a];
    }
  }

  // sum_s Z_s L_s + (.)^T  (S/lindblad.py:110-129)
  template <class PA>
  __device__ static void div_c(const T (&y)[NWA], T (&d)[NP], const PA& A) {
    T Tm[K][K];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) Tm[a][b] = T(0);
#pragma unroll
    for (int s = 0; s < LMAX; ++s) {
      T Z[K][K];
#pragma unroll
      for (int a = 0; a < K; ++a) Z[a][a] = T(0);
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = a + 1; b < K; ++b) {
          Z[a][b] = y[s * NWS + pair_index<K>(a, b)];
          Z[b][a] = -Z[a][b];
        }
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          T acc = Tm[a][b];
#pragma unroll
          for (int c = 0; c < K; ++c) acc = fma(Z[a][c], L(A, s, c, b), acc);
          Tm[a][b] = acc;
        }
    }
#pragma unroll
    for (int a = 0; a < K; ++a) d[a] = Tm[a][a] + Tm[a][a];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) d[K + pair_index<K>(a, b)] = Tm[a][b] + Tm[b][a];
  }

  template <class PA>
  __device__ static void prox_w(T (&x)[NWA], const PA& A) {
    const T thr = A.thr_w;
    if (A.norm_w == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < LMAX; ++q) s = s + ssq_w(&x[q * NWS]);
      const T f = soft_factor(sqrt(s), thr);
#pragma unroll
      for (int i = 0; i < NW; ++i) x[i] = x[i] * f;
    } else {
#pragma unroll
      for (int i = 0; i < NW; ++i) x[i] = x[i] * soft_factor(fabs(x[i]), thr);
    }
    if (A.has_eps) {
#pragma unroll
      for (int i = 0; i < NW; ++i) x[i] = x[i] / A.den_w;
    }
  }

  __device__ static double norm_u(const T (&x)[2][NP], int nid) {
    if (nid == NORM_L2) return double(sqrt(ssq_p(x[0]) + ssq_p(x[1])));
    if (nid == NORM_L12) return double(sqrt(ssq_p(x[0])) + sqrt(ssq_p(x[1])));
    return double(abs_p(x[0]) + abs_p(x[1]));
  }

  __device__ static double norm_w(const T (&x)[NWA], int nid) {
    T s = T(0);
    if (nid == NORM_L2) {
#pragma unroll
      for (int q = 0; q < LMAX; ++q) s = s + ssq_w(&x[q * NWS]);
      return double(sqrt(s));
    }
#pragma unroll
    for (int i = 0; i < NW; ++i) s = s + fabs(x[i]);
    return double(s + s);
  }

  __device__ static void dual_u(const T (&g)[2][NP], int nid, double& gmax, double& pen) {
    if (nid == NORM_L2) {
      const double v = double(sqrt(ssq_p(g[0]) + ssq_p(g[1])));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - 1.0, 0.0));
    } else if (nid == NORM_L12) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const double v = double(sqrt(ssq_p(g[d])));
        gmax = dmax(gmax, v);
        pen += sq(dmax(v - 1.0, 0.0));
      }
    } else {
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const double v = double(fabs(g[d][i]));
          gmax = dmax(gmax, v);
          pen += (i < K ? 1.0 : 2.0) * sq(dmax(v - 1.0, 0.0));
        }
    }
  }

  __device__ static void dual_w(const T (&g)[NWA], int nid, int ell, double alpha, double& gmax,
                                double& pen) {
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < LMAX; ++q) s = s + ssq_w(&g[q * NWS]);
      const double v = double(sqrt(s));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - alpha, 0.0));
    } else {
      // full (ell,k,k) entries: the zero diagonal contributes |0| blocks
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        if (i < ell * NWS) {
          const double v = double(fabs(g[i]));
          gmax = dmax(gmax, v);
          pen += 2.0 * sq(dmax(v - alpha, 0.0));
        }
      }
    }
  }
};

// Complex Hermitian path.  A Hermitian block is K^2 reals: K real diagonal
// entries, then (re, im) of the strict upper triangle row-major.  A skew
// block is stored the same way with the diagonal holding imaginary parts.
template <typename T, int K_, int LM_ = 4>
struct HermPolicy {
  static constexpr int K = K_;
  static constexpr int NP = K * K;
  static constexpr int NWS = K * K;
  static constexpr int LMAX = LM_;  // Lindblad-matrix capacity (2 or 4)
  static constexpr int NW = LMAX * NWS;
  static constexpr int NWA = NW;
  static constexpr bool HAS_W = true;
  static constexpr int NCOEF = 0;  // Lindblad stack stays in parameter space

  __device__ static __forceinline__ double wp(int i) { return i < K ? 1.0 : 2.0; }
  __device__ static __forceinline__ double ww(int i) { return (i % NWS) < K ? 1.0 : 2.0; }

  __device__ static __forceinline__ void unpack_h(const T* x, T (&mr)[K][K], T (&mi)[K][K]) {
#pragma unroll
    for (int a = 0; a < K; ++a) {
      mr[a][a] = x[a];
      mi[a][a] = T(0);
    }
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) {
        const int q = K + 2 * pair_index<K>(a, b);
        mr[a][b] = x[q];
        mi[a][b] = x[q + 1];
        mr[b][a] = x[q];
        mi[b][a] = -x[q + 1];
      }
  }
  __device__ static __forceinline__ void pack_h(const T (&mr)[K][K], const T (&mi)[K][K], T* x) {
#pragma unroll
    for (int a = 0; a < K; ++a) x[a] = mr[a][a];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) {
        const int q = K + 2 * pair_index<K>(a, b);
        x[q] = mr[a][b];
        x[q + 1] = mi[a][b];
      }
  }
  // skew block Z -> Hermitian H = -i Z  (diag: im -> real; pair (re,im) -> (im,-re))
  __device__ static __forceinline__ void skew_to_h(const T* z, T (&mr)[K][K], T (&mi)[K][K]) {
#pragma unroll
    for (int a = 0; a < K; ++a) {
      mr[a][a] = z[a];
      mi[a][a] = T(0);
    }
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) {
        const int q = K + 2 * pair_index<K>(a, b);
        mr[a][b] = z[q + 1];
        mi[a][b] = -z[q];
        mr[b][a] = z[q + 1];
        mi[b][a] = z[q];
      }
  }
  // Hermitian Y -> skew i Y
  __device__ static __forceinline__ void h_to_skew(const T (&mr)[K][K], const T (&mi)[K][K], T* z) {
#pragma unroll
    for (int a = 0; a < K; ++a) z[a] = mr[a][a];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) {
        const int q = K + 2 * pair_index<K>(a, b);
        z[q] = -mi[a][b];
        z[q + 1] = mr[a][b];
      }
  }

  __device__ static __forceinline__ T ssq_p(const T* x) {
    T s = T(0), o = T(0);
#pragma unroll
    for (int i = 0; i < K; ++i) s = s + x[i] * x[i];
#pragma unroll
    for (int i = K; i < NP; ++i) o = o + x[i] * x[i];
    return s + (o + o);
  }
  // sum of entry moduli of the full matrix
  __device__ static __forceinline__ T abs_p(const T* x) {
    T s = T(0), o = T(0);
#pragma unroll
    for (int i = 0; i < K; ++i) s = s + fabs(x[i]);
#pragma unroll
    for (int q = K; q < NP; q += 2) o = o + hypot(x[q], x[q + 1]);
    return s + (o + o);
  }
  __device__ static __forceinline__ void soft_entries(T* x, int len, T thr) {
    // complex soft threshold with modulus; diagonal entries are real
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = x[i] * soft_factor(fabs(x[i]), thr);
#pragma unroll
    for (int q = K; q < NWS; q += 2) {
      const T f = soft_factor(hypot(x[q], x[q + 1]), thr);
      x[q] = x[q] * f;
      x[q + 1] = x[q + 1] * f;
    }
    (void)len;
  }

  template <class PA>
  __device__ static void prox_u(T (&x)[2][NP], const PA& A) {
    const T thr = A.mu;
    if (A.norm_u == NORM_L2) {
      const T f = soft_factor(sqrt(ssq_p(x[0]) + ssq_p(x[1])), thr);
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int i = 0; i < NP; ++i) x[d][i] = x[d][i] * f;
    } else if (A.norm_u == NORM_L12) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const T f = soft_factor(sqrt(ssq_p(x[d])), thr);
#pragma unroll
        for (int i = 0; i < NP; ++i) x[d][i] = x[d][i] * f;
      }
    } else if (A.norm_u == NORM_L1) {
      soft_entries(x[0], NP, thr);
      soft_entries(x[1], NP, thr);
    } else if constexpr (K == 2) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        T mr[K][K], mi[K][K];
        unpack_h(x[d], mr, mi);
        herm_nuc_prox<T, K>(mr, mi, thr);
        pack_h(mr, mi, x[d]);
      }
    } else {
      // one rolled loop over the two direction blocks: a single inlined copy
      // of the eigensolver (K >= 3 unrolls to thousands of instructions; two
      // copies per prox overflowed the instruction cache -- ncu stall
      // "no_instructions").  Blocks are selected with compile-time-indexed
      // selects, so nothing moves to local memory.
#pragma unroll 1
      for (int d = 0; d < 2; ++d) {
        T blk[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) blk[i] = d == 0 ? x[0][i] : x[1][i];
        T mr[K][K], mi[K][K];
        unpack_h(blk, mr, mi);
        herm_nuc_prox<T, K>(mr, mi, thr);
        pack_h(mr, mi, blk);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          if (d == 0) x[0][i] = blk[i];
          else x[1][i] = blk[i];
        }
      }
    }
    if (A.has_eps) {
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int i = 0; i < NP; ++i) x[d][i] = x[d][i] / A.den_u;
    }
  }

  template <class PA>
  __device__ static __forceinline__ cpx<T> L(const PA& A, int s, int a, int b) {
    const int o = ((s * K + a) * K + b) * 2;
    return {T(A.coef[o]), T(A.coef[o + 1])};
  }

  // L_s(a, b) times x (lmac) or x times L_s(a, b) (macl).  RL: the stack is
  // real (A.real_l), so the imaginary parts are not read and their
  // multiply-adds are not issued -- the same values as the complex form,
  // whose terms with a zero imaginary part add exactly 0 (up to the sign of
  // a zero)
  template <bool RL, class PA>
  __device__ static __forceinline__ cpx<T> lmac(cpx<T> acc, const PA& A, int s, int a, int b,
                                                cpx<T> x) {
    if constexpr (RL) {
      const T lr = T(A.coef[((s * K + a) * K + b) * 2]);
      return {fma(lr, x.r, acc.r), fma(lr, x.i, acc.i)};
    } else {
      return cmac(acc, L(A, s, a, b), x);
    }
  }
  template <bool RL, class PA>
  __device__ static __forceinline__ cpx<T> macl(cpx<T> acc, cpx<T> z, const PA& A, int s, int a,
                                                int b) {
    if constexpr (RL) {
      const T lr = T(A.coef[((s * K + a) * K + b) * 2]);
      return {fma(z.r, lr, acc.r), fma(z.i, lr, acc.i)};
    } else {
      return cmac(acc, z, L(A, s, a, b));
    }
  }

  // [L_s, X] = P - P^H, P = L_s X
  template <class PA>
  __device__ static void grad_c(const T (&p)[NP], T (&g)[NWA], const PA& A) {
    if (A.real_l) grad_c_impl<true>(p, g, A);
    else grad_c_impl<false>(p, g, A);
  }
  template <bool RL, class PA>
  __device__ static __forceinline__ void grad_c_impl(const T (&p)[NP], T (&g)[NWA], const PA& A) {
    T xr[K][K], xi[K][K];
    unpack_h(p, xr, xi);
#pragma unroll
    for (int s = 0; s < LMAX; ++s) {
      cpx<T> P[K][K];
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          cpx<T> acc = {T(0), T(0)};
#pragma unroll
          for (int c = 0; c < K; ++c) acc = lmac<RL>(acc, A, s, a, c, cpx<T>{xr[c][b], xi[c][b]});
          P[a][b] = acc;
        }
      T* z = &g[s * NWS];
#pragma unroll
      for (int a = 0; a < K; ++a) z[a] = P[a][a].i + P[a][a].i;
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = a + 1; b < K; ++b) {
          const int q = K + 2 * pair_index<K>(a, b);
          z[q] = P[a][b].r - P[b][a].r;
          z[q + 1] = P[a][b].i + P[b][a].i;
        }
    }
  }

  // T + T^H, T = sum_s Z_s L_s
  template <class PA>
  __device__ static void div_c(const T (&y)[NWA], T (&d)[NP], const PA& A) {
    if (A.real_l) div_c_impl<true>(y, d, A);
    else div_c_impl<false>(y, d, A);
  }
  template <bool RL, class PA>
  __device__ static __forceinline__ void div_c_impl(const T (&y)[NWA], T (&d)[NP], const PA& A) {
    cpx<T> Tm[K][K];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) Tm[a][b] = {T(0), T(0)};
#pragma unroll
    for (int s = 0; s < LMAX; ++s) {
      const T* z = &y[s * NWS];
      cpx<T> Z[K][K];
#pragma unroll
      for (int a = 0; a < K; ++a) Z[a][a] = {T(0), z[a]};
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = a + 1; b < K; ++b) {
          const int q = K + 2 * pair_index<K>(a, b);
          Z[a][b] = {z[q], z[q + 1]};
          Z[b][a] = {-z[q], z[q + 1]};
        }
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          cpx<T> acc = Tm[a][b];
#pragma unroll
          for (int c = 0; c < K; ++c) acc = macl<RL>(acc, Z[a][c], A, s, c, b);
          Tm[a][b] = acc;
        }
    }
#pragma unroll
    for (int a = 0; a < K; ++a) d[a] = Tm[a][a].r + Tm[a][a].r;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = a + 1; b < K; ++b) {
        const int q = K + 2 * pair_index<K>(a, b);
        d[q] = Tm[a][b].r + Tm[b][a].r;
        d[q + 1] = Tm[a][b].i - Tm[b][a].i;
      }
  }

  template <class PA>
  __device__ static void prox_w(T (&x)[NWA], const PA& A) {
    const T thr = A.thr_w;
    if (A.norm_w == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < LMAX; ++q) s = s + ssq_p(&x[q * NWS]);
      const T f = soft_factor(sqrt(s), thr);
#pragma unroll
      for (int i = 0; i < NW; ++i) x[i] = x[i] * f;
    } else if (A.norm_w == NORM_L1) {
#pragma unroll
      for (int q = 0; q < LMAX; ++q) soft_entries(&x[q * NWS], NWS, thr);
    } else if constexpr (K == 2) {
#pragma unroll
      for (int q = 0; q < LMAX; ++q) {
        if (q < A.ell) {
          T mr[K][K], mi[K][K];
          skew_to_h(&x[q * NWS], mr, mi);
          herm_nuc_prox<T, K>(mr, mi, thr);
          h_to_skew(mr, mi, &x[q * NWS]);
        }
      }
    } else {
      // rolled over the Lindblad blocks for the same reason as prox_u
      const int nb = A.ell < LMAX ? A.ell : LMAX;
#pragma unroll 1
      for (int q = 0; q < nb; ++q) {
        T blk[NWS];
#pragma unroll
        for (int i = 0; i < NWS; ++i) {
          T v = x[i];
#pragma unroll
          for (int s = 1; s < LMAX; ++s)
            if (q == s) v = x[s * NWS + i];
          blk[i] = v;
        }
        T mr[K][K], mi[K][K];
        skew_to_h(blk, mr, mi);
        herm_nuc_prox<T, K>(mr, mi, thr);
        h_to_skew(mr, mi, blk);
#pragma unroll
        for (int s = 0; s < LMAX; ++s)
          if (q == s) {
#pragma unroll
            for (int i = 0; i < NWS; ++i) x[s * NWS + i] = blk[i];
          }
      }
    }
    if (A.has_eps) {
#pragma unroll
      for (int i = 0; i < NW; ++i) x[i] = x[i] / A.den_w;
    }
  }

  __device__ static double norm_u(const T (&x)[2][NP], int nid) {
    if (nid == NORM_L2) return double(sqrt(ssq_p(x[0]) + ssq_p(x[1])));
    if (nid == NORM_L12) return double(sqrt(ssq_p(x[0])) + sqrt(ssq_p(x[1])));
    if (nid == NORM_L1) return double(abs_p(x[0]) + abs_p(x[1]));
    double tot = 0.0;
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      T mr[K][K], mi[K][K];
      unpack_h(x[d], mr, mi);
      double s, m;
      herm_abs_eigs<T, K>(mr, mi, s, m);
      tot += s;
    }
    return tot;
  }

  __device__ static double norm_w_ell(const T (&x)[NWA], int nid, int ell) {
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < LMAX; ++q) s = s + ssq_p(&x[q * NWS]);
      return double(sqrt(s));
    }
    if (nid == NORM_L1) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < LMAX; ++q) s = s + abs_p(&x[q * NWS]);
      return double(s);
    }
    double tot = 0.0;
#pragma unroll
    for (int q = 0; q < LMAX; ++q) {
      if (q < ell) {
        T mr[K][K], mi[K][K];
        skew_to_h(&x[q * NWS], mr, mi);
        double s, m;
        herm_abs_eigs<T, K>(mr, mi, s, m);
        tot += s;
      }
    }
    return tot;
  }
  __device__ static double norm_w(const T (&x)[NWA], int nid) { return norm_w_ell(x, nid, LMAX); }

  __device__ static void dual_u(const T (&g)[2][NP], int nid, double& gmax, double& pen) {
    if (nid == NORM_L2) {
      const double v = double(sqrt(ssq_p(g[0]) + ssq_p(g[1])));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - 1.0, 0.0));
    } else if (nid == NORM_L12) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const double v = double(sqrt(ssq_p(g[d])));
        gmax = dmax(gmax, v);
        pen += sq(dmax(v - 1.0, 0.0));
      }
    } else if (nid == NORM_L1) {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const double v = double(fabs(g[d][i]));
          gmax = dmax(gmax, v);
          pen += sq(dmax(v - 1.0, 0.0));
        }
#pragma unroll
        for (int q = K; q < NP; q += 2) {
          const double v = double(hypot(g[d][q], g[d][q + 1]));
          gmax = dmax(gmax, v);
          pen += 2.0 * sq(dmax(v - 1.0, 0.0));
        }
      }
    } else {
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        T mr[K][K], mi[K][K];
        unpack_h(g[d], mr, mi);
        double s, m;
        herm_abs_eigs<T, K>(mr, mi, s, m);
        gmax = dmax(gmax, m);
        pen += sq(dmax(m - 1.0, 0.0));
      }
    }
  }

  __device__ static void dual_w(const T (&g)[NWA], int nid, int ell, double alpha, double& gmax,
                                double& pen) {
    if (nid == NORM_L2) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < LMAX; ++q) s = s + ssq_p(&g[q * NWS]);
      const double v = double(sqrt(s));
      gmax = dmax(gmax, v);
      pen += sq(dmax(v - alpha, 0.0));
      return;
    }
#pragma unroll
    for (int q = 0; q < LMAX; ++q) {
      if (q >= ell) continue;
      const T* z = &g[q * NWS];
      if (nid == NORM_L1) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const double v = double(fabs(z[i]));
          gmax = dmax(gmax, v);
          pen += sq(dmax(v - alpha, 0.0));
        }
#pragma unroll
        for (int p = K; p < NWS; p += 2) {
          const double v = double(hypot(z[p], z[p + 1]));
          gmax = dmax(gmax, v);
          pen += 2.0 * sq(dmax(v - alpha, 0.0));
        }
      } else {
        T mr[K][K], mi[K][K];
        skew_to_h(z, mr, mi);
        double s, m;
        herm_abs_eigs<T, K>(mr, mi, s, m);
        gmax = dmax(gmax, m);
        pen += sq(dmax(m - alpha, 0.0));
      }
    }
  }
};

}  // namespace otfx
