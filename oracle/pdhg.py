"""TEST INFRASTRUCTURE ONLY -- NumPy restatement of the reference PDHG engine.

This is the parity oracle for the CUDA path (see ``oracle/__init__.py``).  It
re-derives, operation by operation and in the same floating-point order, the
iteration of ``/root/reference/pkg/src/otflux/solver.py`` so that its iterates
agree bit-for-bit with the reference on the golden vectors under
``tests/golden`` (checked by ``tests/test_oracle_golden.py``).

Array layout is the reference one (AoS, C-contiguous):
  scalar  u (n,n,2)        phi/diff (n,n)
  vector  u (n,n,2,k)      w (n,n,ell)          phi/diff (n,n,k)
  matrix  u (n,n,2,k,k)    w (n,n,ell,k,k)      phi/diff (n,n,k,k)

Citations are ``S/<file>:<line>`` with ``S/`` = ``pkg/src/otflux/`` of the
reference.
"""

from __future__ import annotations

import math

import numpy as np

TINY = np.finfo(np.float64).tiny  # S/shrink.py:30, S/solver.py:62

# payload rank of every (kind, role) pair -- S/shrink.py:40-46
PAYLOAD_RANK = {
    ("scalar", "u"): 1,
    ("vector", "u"): 2,
    ("matrix", "u"): 3,
    ("vector", "w"): 1,
    ("matrix", "w"): 3,
}

_ABC = "abcdefghijklmnop"


# ---------------------------------------------------------------------------
# reductions (S/shrink.py:88-104, S/solver.py:167-172)
# ---------------------------------------------------------------------------


def sumsq_axes(x, axes, keepdims=False):
    """Sum of |x|^2 over ``axes`` through einsum; complex arrays add the
    real-plane and imaginary-plane sums (S/shrink.py:88-104)."""
    nd = x.ndim
    axes = tuple(a % nd for a in axes)
    src = _ABC[:nd]
    dst = "".join(s for a, s in enumerate(src) if a not in axes)
    spec = src + "," + src + "->" + dst
    if np.iscomplexobj(x):
        r = np.einsum(spec, x.real, x.real) + np.einsum(spec, x.imag, x.imag)
    else:
        r = np.einsum(spec, x, x)
    if keepdims:
        r = r.reshape([1 if a in axes else s for a, s in enumerate(x.shape)])
    return r


def total_sumsq(x):
    """S/solver.py:167-168."""
    return float(sumsq_axes(x, tuple(range(x.ndim))))


def real_inner(a, b):
    """S/solver.py:171-172."""
    return float(np.real(np.sum(a * np.conj(b))))


# ---------------------------------------------------------------------------
# spatial operators (S/spatial.py:30-37, 80-90)
# ---------------------------------------------------------------------------


def grad_stack(phi, inv_dx):
    """Forward differences, ghost row/column zero (S/spatial.py:80-86)."""
    out = np.empty(phi.shape[:2] + (2,) + phi.shape[2:], dtype=phi.dtype)
    out[:-1, :, 0] = (phi[1:] - phi[:-1]) * inv_dx
    out[-1, :, 0] = 0.0
    out[:, :-1, 1] = (phi[:, 1:] - phi[:, :-1]) * inv_dx
    out[:, -1, 1] = 0.0
    return out


def div_stack(u, inv_dx):
    """Backward-difference divergence, (((ux - ux[i-1]) + uy) - uy[j-1]) * inv_dx
    (S/spatial.py:30-37, 89-90)."""
    ux = u[:, :, 0]
    uy = u[:, :, 1]
    d = ux.copy()
    d[1:] -= ux[:-1]
    d += uy
    d[:, 1:] -= uy[:, :-1]
    d *= inv_dx
    return d


# ---------------------------------------------------------------------------
# shrink / prox families (S/shrink.py:120-240) and norms (:243-283)
# ---------------------------------------------------------------------------


def _payload_axes(kind, role, nd):
    r = PAYLOAD_RANK[(kind, role)]
    return tuple(range(nd - r, nd))


def _l12_axes(kind, nd):
    # S/shrink.py:111-117
    if kind == "vector":
        return (nd - 2,)
    if kind == "matrix":
        return (nd - 2, nd - 1)
    return (nd - 1,)


def block_soft(x, thr, axes):
    """Block soft threshold (S/shrink.py:120-127)."""
    r = sumsq_axes(x, axes, keepdims=True)
    np.sqrt(r, out=r)
    np.maximum(r, TINY, out=r)
    np.divide(thr, r, out=r)
    np.subtract(1.0, r, out=r)
    np.maximum(r, 0.0, out=r)
    return x * r


def entry_soft(x, thr):
    """Elementwise (complex: modulus) soft threshold (S/shrink.py:130-136)."""
    r = np.abs(x)
    np.maximum(r, TINY, out=r)
    np.divide(thr, r, out=r)
    np.subtract(1.0, r, out=r)
    np.maximum(r, 0.0, out=r)
    return x * r


def herm(x):
    """(X + X^H)/2 over the trailing axes (S/fields.py:66-71)."""
    xt = np.swapaxes(x, -1, -2)
    if np.iscomplexobj(x):
        xt = np.conj(xt)
    return 0.5 * (x + xt)


def skew(x):
    """(X - X^H)/2 (S/fields.py:74-79)."""
    xt = np.swapaxes(x, -1, -2)
    if np.iscomplexobj(x):
        xt = np.conj(xt)
    return 0.5 * (x - xt)


def eig_soft(x, thr):
    """Sign-preserving eigenvalue soft threshold of Hermitian blocks
    (S/shrink.py:161-169)."""
    lam, vec = np.linalg.eigh(x)
    lt = np.sign(lam) * np.maximum(np.abs(lam) - thr, 0.0)
    y = np.einsum("...ab,...b,...cb->...ac", vec, lt.astype(np.complex128), np.conj(vec))
    return herm(y)


def nuc_shrink(x, thr, role):
    """S/shrink.py:172-196 with the structure chosen as in :199-200."""
    x = np.asarray(x, dtype=np.complex128)
    if role == "u":
        return eig_soft(x, thr)
    return skew(1j * eig_soft(-1j * x, thr))


def prox(x, thr, family, kind, role):
    """shrink_norm dispatch (S/shrink.py:208-221)."""
    if family == "l2":
        return block_soft(x, thr, _payload_axes(kind, role, x.ndim))
    if family == "l12":
        return block_soft(x, thr, _l12_axes(kind, x.ndim))
    if family == "l1":
        return entry_soft(x, thr)
    return nuc_shrink(x, thr, role)


def prox_reg(x, thr, eps, family, kind, role):
    """S/shrink.py:224-240: plain prox divided by (1 + 2 thr eps)."""
    if eps == 0:
        return prox(x, thr, family, kind, role)
    return prox(x, thr, family, kind, role) / (1.0 + 2.0 * thr * eps)


def cell_norms(x, family, kind, role):
    """Per-cell norm value (S/shrink.py:243-259)."""
    axes = _payload_axes(kind, role, x.ndim)
    if family == "l2":
        return np.sqrt(sumsq_axes(x, axes))
    if family == "l12":
        rows = np.sqrt(sumsq_axes(x, _l12_axes(kind, x.ndim), keepdims=True))
        return np.sum(rows, axis=axes)
    if family == "l1":
        return np.sum(np.abs(x), axis=axes)
    h = x if role == "u" else -1j * np.asarray(x, dtype=np.complex128)
    return np.sum(np.abs(np.linalg.eigvalsh(h)), axis=(-2, -1))


def dual_blocks(x, family, kind, role):
    """Dual norm of every shrink block, (cells..., blocks) (S/shrink.py:262-283)."""
    r = PAYLOAD_RANK[(kind, role)]
    lead = x.shape[: x.ndim - r]
    if family == "l2":
        return np.sqrt(sumsq_axes(x, _payload_axes(kind, role, x.ndim)))[..., None]
    if family == "l12":
        return np.sqrt(sumsq_axes(x, _l12_axes(kind, x.ndim))).reshape(lead + (-1,))
    if family == "l1":
        return np.abs(x).reshape(lead + (-1,))
    h = x if role == "u" else -1j * np.asarray(x, dtype=np.complex128)
    return np.max(np.abs(np.linalg.eigvalsh(h)), axis=-1).reshape(lead + (-1,))


# ---------------------------------------------------------------------------
# channel operators
# ---------------------------------------------------------------------------


def graph_coef(k, edges, costs, orientations=None):
    """D / c of S/graph.py:96-102 and :69 (k x ell)."""
    ell = len(edges)
    if orientations is None:
        orientations = np.ones(ell)
    D = np.zeros((k, ell))
    for e, (i, j) in enumerate(edges):
        D[i, e] = orientations[e]
        D[j, e] = -orientations[e]
    return D / np.asarray(costs, dtype=np.float64)


def graph_lambda_max(k, edges, costs, orientations=None):
    """S/graph.py:126-134."""
    ell = len(edges)
    if orientations is None:
        orientations = np.ones(ell)
    D = np.zeros((k, ell))
    for e, (i, j) in enumerate(edges):
        D[i, e] = orientations[e]
        D[j, e] = -orientations[e]
    lap = -(D / np.asarray(costs, dtype=np.float64) ** 2) @ D.T
    return float(np.linalg.eigvalsh(-lap).max())


def graph_grad(coef, x):
    """S/graph.py:105-114 (BLAS matmul)."""
    k, ell = coef.shape
    return (x.reshape(-1, k) @ coef).reshape(x.shape[:-1] + (ell,))


def graph_div(coef, y):
    """S/graph.py:117-123."""
    k, ell = coef.shape
    return (y.reshape(-1, ell) @ (-coef.T)).reshape(y.shape[:-1] + (k,))


def _ct(x):
    xt = np.swapaxes(x, -1, -2)
    return np.conj(xt) if np.iscomplexobj(x) else xt


def comm_grad(mats, x):
    """[L_s, X] as P - P^H, P = L_s X (S/lindblad.py:87-107)."""
    if np.iscomplexobj(x) != np.iscomplexobj(mats):
        x = x.astype(np.complex128)
        mats = mats.astype(np.complex128)
    p = np.einsum("sab,...bc->...sac", mats, x, optimize=True)
    return p - _ct(p)


def comm_div(mats, z):
    """T + T^H, T = sum_s Z_s L_s (S/lindblad.py:110-129)."""
    if np.iscomplexobj(z) != np.iscomplexobj(mats):
        z = z.astype(np.complex128)
        mats = mats.astype(np.complex128)
    t = np.einsum("...sab,sbc->...ac", z, mats, optimize=True)
    return t + _ct(t)


def hermitian_basis(k):
    """S/lindblad.py:132-152."""
    out = np.zeros((k * k, k, k), dtype=np.complex128)
    s = 1.0 / math.sqrt(2.0)
    m = 0
    for i in range(k):
        out[m, i, i] = 1.0
        m += 1
    for i in range(k):
        for j in range(i + 1, k):
            out[m, i, j] = s
            out[m, j, i] = s
            m += 1
            out[m, i, j] = 1j * s
            out[m, j, i] = -1j * s
            m += 1
    return out


def comm_lambda_max(mats):
    """S/lindblad.py:155-174."""
    mats = np.asarray(mats, dtype=np.complex128)
    B = hermitian_basis(mats.shape[-1])
    g = (np.einsum("sab,...bc->...sac", mats, B, optimize=True)
         - np.einsum("...ab,sbc->...sac", B, mats, optimize=True))
    M = np.real(np.einsum("aspq,bspq->ab", g, np.conj(g)))
    M = 0.5 * (M + M.T)
    return float(np.linalg.eigvalsh(M).max())


# ---------------------------------------------------------------------------
# the engine (S/solver.py:175-291) and its driver loop (:294-337)
# ---------------------------------------------------------------------------


class OracleEngine:
    """CPU restatement of ``_Engine``.

    kind: "scalar" | "vector" | "matrix".  ``chan`` is the k x ell graph
    coefficient matrix D/c (vector) or the (ell,k,k) Lindblad stack (matrix);
    for the matrix kind ``dtype`` selects the real or complex path exactly as
    S/solver.py:412-426 does (the caller decides).
    """

    def __init__(self, kind, diff, n, tau, norm_u="l2", norm_w="l1", alpha=1.0,
                 eps=0.0, chan=None, lam_chan=None, dtype=np.float64):
        self.kind = kind
        self.n = n
        self.inv_dx = 1.0 / (1.0 / (n - 1))  # S/solver.py:183 with dx of S/fields.py:48-49
        self.diff = diff
        self.diff_norm = float(np.sqrt(total_sumsq(diff)))
        self.tau = tau
        self.norm_u = norm_u
        self.norm_w = norm_w
        self.alpha = alpha
        self.eps = eps
        self.chan = chan
        has_w = kind != "scalar"
        p = diff.shape[2:]
        self.u = np.zeros((n, n, 2) + p, dtype=dtype)
        self.phi = np.zeros((n, n) + p, dtype=dtype)
        if kind == "vector":
            self.w = np.zeros((n, n, chan.shape[1]), dtype=dtype)
        elif kind == "matrix":
            self.w = np.zeros((n, n, chan.shape[0]) + p, dtype=dtype)
        else:
            self.w = None
        self.mu = 1.0 / ((32.0 if has_w else 16.0) * tau * (n - 1) ** 2)  # :199
        self.nu = None if not has_w else 1.0 / (4.0 * tau * lam_chan)  # :205

    # channel operator closures (S/solver.py:388-390, 429-431)
    def cgrad(self, phi):
        if self.kind == "vector":
            return graph_grad(self.chan, phi)
        return comm_grad(self.chan, phi)

    def cdiv(self, w):
        if self.kind == "vector":
            return graph_div(self.chan, w)
        return comm_div(self.chan, w)

    def _prox_u(self, x):  # :207-210
        return prox_reg(x, self.mu, self.eps, self.norm_u, self.kind, "u")

    def _prox_w(self, x):  # :212-218
        thr = self.alpha * self.nu
        return prox_reg(x, thr, self.eps / self.alpha if self.eps > 0 else 0.0,
                        self.norm_w, self.kind, "w")

    def step(self):
        """One PDHG iteration, same op order as S/solver.py:220-240."""
        a = grad_stack(self.phi, self.inv_dx)
        a *= self.mu
        a += self.u
        un = self._prox_u(a)
        ubar = un + un
        ubar -= self.u
        self.u = un
        rhs = div_stack(ubar, self.inv_dx)
        rhs -= self.diff
        if self.w is not None:
            b = self.cgrad(self.phi)
            b *= self.nu
            b += self.w
            wn = self._prox_w(b)
            wbar = wn + wn
            wbar -= self.w
            rhs += self.cdiv(wbar)
            self.w = wn
        rhs *= self.tau
        self.phi = self.phi + rhs

    def feas(self):  # :242-246
        con = div_stack(self.u, self.inv_dx) - self.diff
        if self.w is not None:
            con += self.cdiv(self.w)
        return float(np.sqrt(total_sumsq(con)) / max(self.diff_norm, TINY))

    def primal(self):  # :248-256
        p = float(np.sum(cell_norms(self.u, self.norm_u, self.kind, "u")))
        if self.w is not None:
            p += self.alpha * float(np.sum(cell_norms(self.w, self.norm_w, self.kind, "w")))
        if self.eps > 0:
            p += self.eps * total_sumsq(self.u)
            if self.w is not None:
                p += self.eps * total_sumsq(self.w)
        return p

    def dual(self):  # :258-274
        raw = -real_inner(self.phi, self.diff)
        gu = dual_blocks(grad_stack(self.phi, self.inv_dx), self.norm_u, self.kind, "u")
        gw = None
        if self.w is not None:
            gw = dual_blocks(self.cgrad(self.phi), self.norm_w, self.kind, "w")
        if self.eps == 0:
            s = max(1.0, float(gu.max(initial=0.0)))
            if gw is not None:
                s = max(s, float(gw.max(initial=0.0)) / self.alpha)
            return raw / s
        pen = float(np.sum(np.maximum(gu - 1.0, 0.0) ** 2)) / (4.0 * self.eps)
        if gw is not None:
            pen += float(np.sum(np.maximum(gw - self.alpha, 0.0) ** 2)) / (4.0 * self.eps)
        return raw - pen

    def evaluate(self):  # :276-280
        p = self.primal()
        d = self.dual()
        return p, d, (p - d) / max(p, 1e-30), self.feas()

    def residual_from(self, u0, w0, phi0):  # :282-291
        du = self.u - u0
        dphi = self.phi - phi0
        r = total_sumsq(du) / self.mu + total_sumsq(dphi) / self.tau
        cross = div_stack(du, self.inv_dx)
        if self.w is not None:
            dw = self.w - w0
            r += total_sumsq(dw) / self.nu
            cross += self.cdiv(dw)
        return r - 2.0 * real_inner(dphi, cross)


def oracle_run(eng: OracleEngine, tol_gap=1e-3, tol_feas=1e-5, max_iters=200_000,
               check_every=100):
    """The ``_run`` loop (S/solver.py:294-337).  Returns
    (converged, iterations, history) with history rows
    (iteration, primal, dual, gap, feas, residual)."""
    hist = []
    p, d, g, f = eng.evaluate()
    hist.append((0, p, d, g, f, float("nan")))
    conv = g <= tol_gap and f <= tol_feas
    it = 0
    while not conv and it < max_iters:
        chk = ((it + 1) % check_every == 0) or (it + 1 == max_iters)
        if chk:
            u0 = eng.u.copy()
            w0 = None if eng.w is None else eng.w.copy()
            p0 = eng.phi.copy()
        eng.step()
        it += 1
        if chk:
            rk = eng.residual_from(u0, w0, p0)
            p, d, g, f = eng.evaluate()
            hist.append((it, p, d, g, f, rk))
            conv = g <= tol_gap and f <= tol_feas
    return conv, it, hist
