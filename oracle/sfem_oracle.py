"""oracle/sfem_oracle.py -- TEST INFRASTRUCTURE, not product code.

A numpy restatement of the reference's algorithm for the hot path (algorithm
(a) full diagonalisation and the standalone 1D expand/unexpand), used ONLY by
tests/, __graft_entry__.smoke() and bench.py's cpu legs as the checker.  The
product path (paper_1701_03967_b200) never imports it.

Parity pin: this restatement is checked (tests/test_oracle.py) against
  * the reference's own known-answer tests, restated: closed-form interior
    spectra (test_element.cpp:87-99), exact n=1/n=2 element matrices
    (test_element.cpp:23-39), the n=1 theta-equation root
    (test_spectral.cpp:13-25), trig impulse responses (test_trig.cpp:30-91),
    the 1D diagonal action (test_poisson.cpp:90-115);
  * golden vectors produced by the reference itself, compiled from its
    sources into oracle/_ref (tests/golden/make_golden.py).

Every function cites the reference file:line it restates (paths relative to
/root/reference/proj).  Layout conventions: a 1D "line" is the interleaved
dof vector of length n*K-1 (dof t = e*n + c is interior component c of
element e, t = j*n - 1 is node j; banded.cpp:9-15), coefficients are in
frequency-major order (grid1d.hpp:41-58).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# L0 numeric kit
# ----------------------------------------------------------------------------


def _legendre_eval(m: int, x: float):
    """quadrature.hpp:18-33."""
    p0, p1 = 1.0, x
    if m == 0:
        return 1.0, 0.0
    for k in range(2, m + 1):
        pk = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
        p0, p1 = p1, pk
    return p1, m * (x * p1 - p0) / (x * x - 1.0)


def gauss_legendre(m: int):
    """Gauss-Legendre rule, half solved then mirrored (quadrature.hpp:40-74)."""
    nodes = [0.0] * m
    weights = [0.0] * m
    eps = np.finfo(float).eps
    half = m // 2
    for i in range(half):
        x = math.cos(math.pi * (i + 0.75) / (m + 0.5))
        for _ in range(200):
            p, dp = _legendre_eval(m, x)
            dx = p / dp
            x -= dx
            if abs(dx) <= 2 * eps * (1 + abs(x)):
                break
        p, dp = _legendre_eval(m, x)
        w = 2.0 / ((1.0 - x * x) * dp * dp)
        nodes[m - 1 - i] = x
        nodes[i] = -x
        weights[i] = w
        weights[m - 1 - i] = w
    if m % 2 == 1:
        p, dp = _legendre_eval(m, 0.0)
        nodes[half] = 0.0
        weights[half] = 2.0 / (dp * dp)
    return nodes, weights


def equispaced_nodes(n: int):
    """lagrange.hpp:11-17: (2k - n)/n."""
    return [(2 * k - n) / n for k in range(n + 1)]


def lagrange_value(nodes, l, x):
    """lagrange.hpp:20-27."""
    v = 1.0
    for m, xm in enumerate(nodes):
        if m == l:
            continue
        v *= (x - xm) / (nodes[l] - xm)
    return v


def lagrange_derivative(nodes, l, x):
    """lagrange.hpp:31-47 (product-rule form)."""
    s = 0.0
    denom = 1.0
    for m, xm in enumerate(nodes):
        if m == l:
            continue
        denom *= nodes[l] - xm
        term = 1.0
        for r, xr in enumerate(nodes):
            if r == l or r == m:
                continue
            term *= x - xr
        s += term
    return s / denom


def _jacobi_eigensymm(a: np.ndarray):
    """Cyclic Jacobi (smallmat.hpp:125-170)."""
    m = a.copy()
    n = m.shape[0]
    vecs = np.eye(n)
    eps = np.finfo(float).eps
    for _ in range(128):
        diag = np.abs(np.diag(m)).sum()
        off = np.abs(np.triu(m, 1)).sum()
        if not (off > eps * (diag + off)):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = m[p, q]
                if abs(apq) <= eps * eps * (abs(m[p, p]) + abs(m[q, q])):
                    continue
                tau = (m[q, q] - m[p, p]) / (2.0 * apq)
                if tau >= 0:
                    t = 1.0 / (tau + math.sqrt(1.0 + tau * tau))
                else:
                    t = -1.0 / (-tau + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                mkp = m[:, p].copy()
                mkq = m[:, q].copy()
                m[:, p] = c * mkp - s * mkq
                m[:, q] = s * mkp + c * mkq
                mpk = m[p, :].copy()
                mqk = m[q, :].copy()
                m[p, :] = c * mpk - s * mqk
                m[q, :] = s * mpk + c * mqk
                vkp = vecs[:, p].copy()
                vkq = vecs[:, q].copy()
                vecs[:, p] = c * vkp - s * vkq
                vecs[:, q] = s * vkp + c * vkq
    return np.diag(m).copy(), vecs


def _matmul(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Loop order of smallmat.hpp:36-44 (kept exact so tables match the reference bit-closely)."""
    z = np.zeros((x.shape[0], y.shape[1]))
    for i in range(x.shape[0]):
        for k in range(x.shape[1]):
            xik = x[i, k]
            for j in range(y.shape[1]):
                z[i, j] += xik * y[k, j]
    return z


def _dot(x, y) -> float:
    """smallmat.hpp:57-62."""
    s = 0.0
    for a, b in zip(x, y):
        s += a * b
    return s


def _cholesky_lower(m: np.ndarray) -> np.ndarray:
    """smallmat.hpp:72-89."""
    n = m.shape[0]
    l = np.zeros((n, n))
    for j in range(n):
        d = m[j, j]
        for k in range(j):
            d -= l[j, k] * l[j, k]
        if not (d > 0):
            raise ValueError("cholesky: matrix not positive definite")
        l[j, j] = math.sqrt(d)
        for i in range(j + 1, n):
            s = m[i, j]
            for k in range(j):
                s -= l[i, k] * l[j, k]
            l[i, j] = s / l[j, j]
    return l


def _solve_lower(l: np.ndarray, b) -> list:
    """smallmat.hpp:92-100."""
    b = list(b)
    for i in range(len(b)):
        for k in range(i):
            b[i] -= l[i, k] * b[k]
        b[i] /= l[i, i]
    return b


def _solve_lower_transposed(l: np.ndarray, b) -> list:
    """smallmat.hpp:102-110."""
    b = list(b)
    n = len(b)
    for i in range(n - 1, -1, -1):
        for k in range(i + 1, n):
            b[i] -= l[k, i] * b[k]
        b[i] /= l[i, i]
    return b


def _pencil_eigensymm(a: np.ndarray, b: np.ndarray):
    """A x = lambda B x through the Cholesky factor of B (smallmat.hpp:175-214)."""
    n = a.shape[0]
    if n == 0:
        return np.zeros(0), np.zeros((0, 0))
    l = _cholesky_lower(b)
    m = np.zeros((n, n))
    for j in range(n):
        m[:, j] = _solve_lower(l, a[:, j])
    for i in range(n):
        m[i, :] = _solve_lower(l, m[i, :])
    for i in range(n):
        for j in range(i + 1, n):
            v = (m[i, j] + m[j, i]) / 2.0
            m[i, j] = v
            m[j, i] = v
    w, y = _jacobi_eigensymm(m)
    order = sorted(range(n), key=lambda i: w[i])
    vecs = np.zeros((n, n))
    vals = np.zeros(n)
    for j in range(n):
        vecs[:, j] = _solve_lower_transposed(l, y[:, order[j]])
        vals[j] = w[order[j]]
    return vals, vecs


# ----------------------------------------------------------------------------
# L1 reference element
# ----------------------------------------------------------------------------


def _symmetrize_bisymmetric(m: np.ndarray):
    """element.hpp:85-100: symmetrise, then copy the canonical half onto the flip image."""
    n = m.shape[0] - 1
    for i in range(n + 1):
        for j in range(i, n + 1):
            v = (m[i, j] + m[j, i]) / 2.0
            m[i, j] = v
            m[j, i] = v
    for i in range(n + 1):
        for j in range(n + 1):
            fi, fj = n - i, n - j
            if (fi, fj) > (i, j):
                m[fi, fj] = m[i, j]


@dataclass
class Blocks:
    """ElementBlocks (element.hpp:25-32)."""
    corner: float
    cross: float
    edge: np.ndarray
    edge_rev: np.ndarray
    interior: np.ndarray


def _carve_blocks(m: np.ndarray) -> Blocks:
    """element.hpp:102-118."""
    n = m.shape[0] - 1
    return Blocks(m[0, 0], m[0, n], m[1:n, 0].copy(), m[1:n, n].copy(), m[1:n, 1:n].copy())


@dataclass
class Element:
    order: int
    stiffness: np.ndarray
    mass: np.ndarray
    stiff: Blocks
    massb: Blocks


def build_element_matrices(n: int, order_cap: int = 9) -> Element:
    """(n+1)-point Gauss stiffness/mass of the order-n Lagrange basis (element.hpp:258-295)."""
    if not (1 <= n <= order_cap):
        raise ValueError(f"build_element_matrices: order {n} outside [1, {order_cap}]")
    nodes = equispaced_nodes(n)
    gn, gw = gauss_legendre(n + 1)
    vals = np.array([[lagrange_value(nodes, l, g) for g in gn] for l in range(n + 1)])
    ders = np.array([[lagrange_derivative(nodes, l, g) for g in gn] for l in range(n + 1)])
    st = np.zeros((n + 1, n + 1))
    ma = np.zeros((n + 1, n + 1))
    for k in range(n + 1):
        for l in range(n + 1):
            sa = 0.0
            sc = 0.0
            for g in range(n + 1):
                sa += gw[g] * ders[k, g] * ders[l, g]
                sc += gw[g] * vals[k, g] * vals[l, g]
            st[k, l] = sa
            ma[k, l] = sc
    _symmetrize_bisymmetric(st)
    _symmetrize_bisymmetric(ma)
    return Element(n, st, ma, _carve_blocks(st), _carve_blocks(ma))


def _parity_basis(m: int, sign: int) -> np.ndarray:
    """element.hpp:122-135."""
    half = m // 2
    dim = (m + 1) // 2 if sign > 0 else m // 2
    u = np.zeros((m, dim))
    r = 1.0 / math.sqrt(2.0)
    for i in range(half):
        u[i, i] = r
        u[m - 1 - i, i] = r if sign > 0 else -r
    if sign > 0 and m % 2 == 1:
        u[half, dim - 1] = 1.0
    return u


def parity_pencil_eig(a: np.ndarray, b: np.ndarray):
    """Parity-split pencil eigenpairs, sorted, first nonzero entry positive (element.hpp:140-198)."""
    m = a.shape[0]
    pairs = []
    for sign in (+1, -1):
        u = _parity_basis(m, sign)
        if u.shape[1] == 0:
            continue
        ut = u.T.copy()
        ar = _matmul(ut, _matmul(a, u))
        br = _matmul(ut, _matmul(b, u))
        w, y = _pencil_eigensymm(ar, br)
        for j in range(u.shape[1]):
            v = np.zeros(m)
            for i in range(m):
                s = 0.0
                for k in range(u.shape[1]):
                    s += u[i, k] * y[k, j]
                v[i] = s
            pairs.append((w[j], v, sign))
    pairs.sort(key=lambda p: p[0])  # std::sort on distinct values
    values = np.zeros(m)
    vecs = np.zeros((m, m))
    parity = np.zeros(m, dtype=int)
    for j, (w, v, s) in enumerate(pairs):
        peak = np.max(np.abs(v))
        for i in range(m):
            if abs(v[i]) > peak / 1048576.0:
                if v[i] < 0:
                    v = -v
                break
        values[j] = w
        vecs[:, j] = v
        parity[j] = s
    return values, vecs, parity


@dataclass
class InteriorEigenSystem:
    """InteriorEigenSystemT (element.hpp:43-62)."""
    order: int
    values: np.ndarray
    vectors: np.ndarray  # column l-1 = e^(l)
    parity: np.ndarray
    edge_stiff: np.ndarray
    edge_mass: np.ndarray


def interior_eigensystem(em: Element) -> InteriorEigenSystem:
    """element.hpp:313-347."""
    values, vecs, parity = parity_pencil_eig(em.stiff.interior, em.massb.interior)
    for j in range(len(values) - 1):
        gap = values[j + 1] - values[j]
        if not (gap > 1e-12 * (1 + abs(values[j + 1]))):
            raise ValueError("interior_eigensystem: eigenvalue multiplicity")
    m = len(values)
    es = np.array([_dot(em.stiff.edge, vecs[:, l]) for l in range(m)])
    ms = np.array([_dot(em.massb.edge, vecs[:, l]) for l in range(m)])
    return InteriorEigenSystem(em.order, values, vecs, parity, es, ms)


# ----------------------------------------------------------------------------
# L2 spectral table
# ----------------------------------------------------------------------------


class ThetaEquation:
    """Frequency equation in pole/residue form (spectral.hpp:26-80)."""

    def __init__(self, es: InteriorEigenSystem, em: Element, theta: float):
        self.affine_a = em.stiff.corner + theta * em.stiff.cross
        self.affine_b = em.massb.corner + theta * em.massb.cross
        self.pole = list(es.values)
        self.coef = [1.0 + theta * float(p) for p in es.parity]
        self.num_a = list(es.edge_stiff)
        self.num_c = list(es.edge_mass)

    def value(self, x):
        s = self.affine_a - x * self.affine_b
        for l in range(len(self.pole)):
            d = self.num_a[l] - x * self.num_c[l]
            s += self.coef[l] * d * d / (x - self.pole[l])
        return s

    def derivative(self, x):
        s = -self.affine_b
        for l in range(len(self.pole)):
            d = self.num_a[l] - x * self.num_c[l]
            u = x - self.pole[l]
            s += self.coef[l] * (-2.0 * self.num_c[l] * d * u - d * d) / (u * u)
        return s


def _refine_root(eq: ThetaEquation, lo: float, hi: float) -> float:
    """Bracketed Newton/bisection (spectral.hpp:84-105)."""
    eps = np.finfo(float).eps
    x = (lo + hi) / 2.0
    for _ in range(500):
        g = eq.value(x)
        if g > 0:
            lo = x
        elif g < 0:
            hi = x
        else:
            return x
        width = hi - lo
        if not (width > 4.0 * eps * (abs(lo) + abs(hi))):
            break
        dg = eq.derivative(x)
        nxt = x - g / dg
        if not (nxt > lo) or not (nxt < hi):
            nxt = (lo + hi) / 2.0
        x = nxt
    return (lo + hi) / 2.0


def solve_theta_equation(es, em: Element, theta: float):
    """n roots of the frequency equation (spectral.hpp:112-193)."""
    n = em.order
    if n == 1:
        return [(em.stiff.corner + theta * em.stiff.cross) / (em.massb.corner + theta * em.massb.cross)]
    eq = ThetaEquation(es, em, theta)
    m = n - 1

    def right_of_pole(l):
        p = eq.pole[l]
        gap = (eq.pole[l + 1] if l + 1 < m else 2.0 * p + 1.0) - p
        d = gap / 8.0
        for _ in range(2000):
            if eq.value(p + d) > 0:
                return p + d
            d /= 2.0
            if not (p + d > p):
                break
        raise ValueError("no positive bracket right of pole")

    def left_of_pole(l):
        p = eq.pole[l]
        gap = p - (eq.pole[l - 1] if l > 0 else 0.0)
        d = gap / 8.0
        for _ in range(2000):
            if eq.value(p - d) < 0:
                return p - d
            d /= 2.0
            if not (p - d < p):
                break
        raise ValueError("no negative bracket left of pole")

    roots = []
    lo = 0.0
    if not (eq.value(lo) > 0):
        step = eq.pole[0] / 4.0
        found = False
        for _ in range(64):
            lo = -step
            found = eq.value(lo) > 0
            if found:
                break
            step *= 2.0
        if not found:
            raise ValueError("no positive bracket below the first pole")
    roots.append(_refine_root(eq, lo, left_of_pole(0)))
    for l in range(m - 1):
        roots.append(_refine_root(eq, right_of_pole(l), left_of_pole(l + 1)))
    hi = 4.0 * eq.pole[m - 1] + 4.0 * abs(eq.affine_a) + 4.0
    cap = 64.0 * hi
    while not (eq.value(hi) < 0):
        hi *= 2.0
        if hi > cap:
            raise ValueError("outer bracket cap reached")
    roots.append(_refine_root(eq, right_of_pole(m - 1), hi))
    return roots


def interior_solution(es: InteriorEigenSystem, lam: float) -> np.ndarray:
    """spectral.hpp:198-213."""
    m = es.order - 1
    p = [0.0] * m
    for l in range(m):
        d = lam - es.values[l]
        w = (es.edge_stiff[l] - lam * es.edge_mass[l]) / d
        for i in range(m):
            p[i] += w * es.vectors[i, l]
    return np.array(p)


@dataclass
class Table:
    """SpectralTable1D (spectral.hpp:281-312) plus the finalize_table fields (spectral.cpp:21-79)."""
    order: int
    elements: int
    element: Element
    interior: InteriorEigenSystem | None
    theta: np.ndarray
    half_cos: np.ndarray
    half_sin: np.ndarray
    values: np.ndarray        # (K-1, n)
    norm_sq: np.ndarray       # (K-1, n)
    nodal_weight: np.ndarray  # (K-1, n)
    p: np.ndarray             # (K-1, n, m)
    q: np.ndarray             # (K-1, n, m)
    p_even: np.ndarray = field(default=None)
    p_odd: np.ndarray = field(default=None)
    q_even: np.ndarray = field(default=None)
    q_odd: np.ndarray = field(default=None)

    @property
    def interior_dim(self):
        return self.order - 1

    def eigenvalues_coeff_order(self) -> np.ndarray:
        """spectral.cpp:10-17."""
        head = self.interior.values if self.order > 1 else np.zeros(0)
        return np.concatenate([head, self.values.reshape(-1)])


def build_spectral_table(n: int, K: int) -> Table:
    """build_table_primaries (spectral.hpp:228-277) + finalize_table (spectral.cpp:21-79)."""
    if K < 2:
        raise ValueError("spectral table: need at least two elements")
    em = build_element_matrices(n)
    es = interior_eigensystem(em) if n >= 2 else None
    m = n - 1
    theta = np.array([math.cos(math.pi * k / K) for k in range(1, K)])
    values = np.zeros((K - 1, n))
    norm_sq = np.zeros((K - 1, n))
    p = np.zeros((K - 1, n, m))
    mb = em.massb
    for k in range(1, K):
        th = theta[k - 1]
        roots = solve_theta_equation(es, em, th)
        for l in range(n):
            lam = roots[l]
            values[k - 1, l] = lam
            pv = interior_solution(es, lam) if m > 0 else np.zeros(0)
            p[k - 1, l] = pv
            cp = [_dot(mb.interior[i, :], pv) for i in range(m)]
            term_direct = mb.corner
            term_rev = mb.cross
            for i in range(m):
                w = cp[i] + 2.0 * mb.edge[i]
                term_direct += w * pv[i]
                term_rev += w * pv[m - 1 - i]
            ns = K * (term_direct + th * term_rev)
            if not (ns > 0):
                raise ValueError("spectral table: nonpositive squared norm")
            norm_sq[k - 1, l] = ns
    half_cos = np.array([math.cos(math.pi * k / (2.0 * K)) for k in range(1, K)])
    half_sin = np.array([math.sin(math.pi * k / (2.0 * K)) for k in range(1, K)])
    q = np.zeros_like(p)
    nodal_weight = np.zeros((K - 1, n))
    half = m // 2
    ne, no = n // 2, (n - 1) // 2
    p_even = np.zeros((K - 1, n, ne))
    p_odd = np.zeros((K - 1, n, no))
    q_even = np.zeros((K - 1, n, ne))
    q_odd = np.zeros((K - 1, n, no))
    for k in range(1, K):
        th = theta[k - 1]
        for l in range(n):
            pv = p[k - 1, l]
            edge_dot = 0.0
            edge_dot_rev = 0.0
            qv = np.zeros(m)
            for i in range(m):
                s = mb.edge[i]
                for j in range(m):
                    s += mb.interior[i, j] * pv[j]
                qv[i] = s
                edge_dot += mb.edge[i] * pv[i]
                edge_dot_rev += mb.edge[i] * pv[m - 1 - i]
            q[k - 1, l] = qv
            nodal_weight[k - 1, l] = 2.0 * (mb.corner + edge_dot + th * (mb.cross + edge_dot_rev))
            for i in range(half):
                p_even[k - 1, l, i] = 0.5 * (pv[i] + pv[m - 1 - i])
                p_odd[k - 1, l, i] = 0.5 * (pv[i] - pv[m - 1 - i])
                q_even[k - 1, l, i] = 0.5 * (qv[i] + qv[m - 1 - i])
                q_odd[k - 1, l, i] = 0.5 * (qv[i] - qv[m - 1 - i])
            if m % 2 == 1:
                p_even[k - 1, l, half] = pv[half]
                q_even[k - 1, l, half] = qv[half]
    return Table(n, K, em, es, theta, half_cos, half_sin, values, norm_sq, nodal_weight, p, q,
                 p_even, p_odd, q_even, q_odd)


_TABLES: dict = {}


def table(n: int, K: int) -> Table:
    """Memoised table set (TableSet::get, poisson.cpp:49-73, without the file cache)."""
    key = (n, K)
    if key not in _TABLES:
        _TABLES[key] = build_spectral_table(n, K)
    return _TABLES[key]


# ----------------------------------------------------------------------------
# L3 trig transforms (trig.hpp:3-7 conventions), batched over leading axes
# ----------------------------------------------------------------------------


# Short transforms are the O(K^2) sums themselves; from FAST_K on they go
# through scipy.fft's r2r transforms, whose unnormalised type-I/II/III
# definitions are FFTW's (the functions the reference binds, trig.cpp:43-48),
# rescaled exactly as Plan::execute does (trig.cpp:71-92).  Both forms are
# checked against each other and against the reference's trig KATs in
# tests/test_oracle.py; the fast form makes 1e9-unknown full-size checks
# feasible (C5 n=1, which the reference itself cannot run in 2-D/3-D).
FAST_K = 48


def _sfft():
    try:
        import scipy.fft as sf
        return sf
    except Exception:  # scipy absent: the direct sums only
        return None


def _sin_matrix(K):
    j = np.arange(1, K)
    return np.sin(np.pi * np.outer(j, j) / K)


def dst1(x: np.ndarray, direct: bool = False) -> np.ndarray:
    """X_k = sum_{j=1}^{K-1} x_j sin(pi j k / K) over the last axis (trig.hpp:4).
    FFTW RODFT00 output times 1/2 (trig.cpp:76-78)."""
    K = x.shape[-1] + 1
    if K == 1:
        return x.copy()
    sf = _sfft()
    if sf is not None and not direct and K >= FAST_K:
        return 0.5 * sf.dst(x, type=1, axis=-1, workers=-1)
    return x @ _sin_matrix(K).T


def dst3_synthesis(b: np.ndarray, direct: bool = False) -> np.ndarray:
    """w_j = sum_{k=1}^{K} b_k sin(pi k (j-1/2)/K) (trig.hpp:5).
    FFTW RODFT01 of the input halved except the last (trig.cpp:83-91)."""
    K = b.shape[-1]
    sf = _sfft()
    if sf is not None and not direct and K >= FAST_K:
        h = 0.5 * b
        h[..., -1] = b[..., -1]
        return sf.dst(h, type=3, axis=-1, workers=-1)
    j = np.arange(1, K + 1)
    k = np.arange(1, K + 1)
    return b @ np.sin(np.pi * np.outer(k, j - 0.5) / K)


def dct3_synthesis(a: np.ndarray, direct: bool = False) -> np.ndarray:
    """w_j = sum_{k=0}^{K-1} a_k cos(pi k (j-1/2)/K) (trig.hpp:6).
    FFTW REDFT01 of the input halved except the first (trig.cpp:83-91)."""
    K = a.shape[-1]
    sf = _sfft()
    if sf is not None and not direct and K >= FAST_K:
        h = 0.5 * a
        h[..., 0] = a[..., 0]
        return sf.dct(h, type=3, axis=-1, workers=-1)
    j = np.arange(1, K + 1)
    k = np.arange(0, K)
    return a @ np.cos(np.pi * np.outer(k, j - 0.5) / K)


# ----------------------------------------------------------------------------
# L4 line transforms on a batch of dof-layout lines, shape (..., nK-1)
# ----------------------------------------------------------------------------


def split_line(y: np.ndarray, n: int, K: int):
    """dof line -> (nodal[..., K+1], interior[..., K, n-1]) (banded.cpp:98-109)."""
    m = n - 1
    lead = y.shape[:-1]
    nodal = np.zeros(lead + (K + 1,))
    full = np.concatenate([y, np.zeros(lead + (1,))], axis=-1).reshape(lead + (K, n))
    nodal[..., 1:K] = full[..., :K - 1, n - 1]
    interior = full[..., :, :m].copy()
    return nodal, interior


def join_line(nodal: np.ndarray, interior: np.ndarray, n: int, K: int) -> np.ndarray:
    """(nodal, interior) -> dof line (banded.cpp:87-96)."""
    lead = nodal.shape[:-1]
    full = np.zeros(lead + (K, n))
    full[..., :, :n - 1] = interior
    full[..., :K - 1, n - 1] = nodal[..., 1:K]
    return full.reshape(lead + (K * n,))[..., :K * n - 1]


def _centre(interior, m, K):
    """accumulate_alternating (eigenbasis.cpp:31-40): sum_j (-P)^(j-1) v_{j-1/2}."""
    odd = interior[..., 0::2, :].sum(axis=-2)
    even = interior[..., 1::2, :].sum(axis=-2)
    return odd - even[..., ::-1]


def _folds(interior, m, K):
    """build_folds (eigenbasis.cpp:46-59): even slots 0..ne-1 then odd slots; shape (..., m, K-1)."""
    half, ne = m // 2, (m + 1) // 2
    a = interior[..., :K - 1, :]
    b = interior[..., 1:, :]
    lead = interior.shape[:-2]
    fold = np.zeros(lead + (m, K - 1))
    for i in range(half):
        u_i = a[..., i] + b[..., i]
        u_r = a[..., m - 1 - i] + b[..., m - 1 - i]
        v_i = b[..., i] - a[..., i]
        v_r = b[..., m - 1 - i] - a[..., m - 1 - i]
        fold[..., i, :] = u_i + u_r
        fold[..., ne + i, :] = v_i - v_r
    if m % 2 == 1:
        fold[..., half, :] = a[..., half] + b[..., half]
    return fold


def decompose_weighted(y: np.ndarray, t: Table) -> np.ndarray:
    """FC_n (lines::decompose_weighted, eigenbasis.cpp:63-101) on dof lines -> coefficients."""
    return _analysis(y, t, weighted=True)


def decompose(y: np.ndarray, t: Table) -> np.ndarray:
    """F_n (lines::decompose, eigenbasis.cpp:103-142)."""
    return _analysis(y, t, weighted=False)


def _analysis(y, t: Table, weighted: bool):
    n, K = t.order, t.elements
    m = n - 1
    ne, no = n // 2, (n - 1) // 2
    nodal, interior = split_line(y, n, K)
    lead = y.shape[:-1]
    out = np.zeros(lead + (n * K - 1,))
    if m > 0:
        centre = _centre(interior, m, K)
        if not weighted:
            centre = centre @ t.element.massb.interior.T  # matvec(C~, centre)
        out[..., :m] = (centre @ t.interior.vectors) / K
    nodal_hat = dst1(nodal[..., 1:K])                      # (..., K-1)
    if m > 0:
        fold_hat = dst1(_folds(interior, m, K))            # (..., m, K-1)
    pe = t.p_even if weighted else t.q_even
    po = t.p_odd if weighted else t.q_odd
    num = np.empty(lead + (K - 1, n))
    for l in range(n):
        base = nodal_hat * (1.0 if weighted else t.nodal_weight[:, l])
        acc = base.copy()
        for i in range(ne):
            acc = acc + pe[:, l, i] * fold_hat[..., i, :]
        for i in range(no):
            acc = acc + po[:, l, i] * fold_hat[..., ne + i, :]
        num[..., l] = acc / t.norm_sq[:, l]
    out[..., m:] = num.reshape(lead + ((K - 1) * n,))
    return out


def synthesize(c: np.ndarray, t: Table) -> np.ndarray:
    """Inverse F_n (lines::synthesize, eigenbasis.cpp:144-225): coefficients -> dof lines."""
    n, K = t.order, t.elements
    m = n - 1
    half = m // 2
    ne, no = n // 2, (n - 1) // 2
    lead = c.shape[:-1]
    ck = c[..., m:].reshape(lead + (K - 1, n))
    nodal = np.zeros(lead + (K + 1,))
    nodal[..., 1:K] = dst1(ck.sum(axis=-1))
    interior = np.zeros(lead + (K, m))
    if m > 0:
        centre = c[..., :m] @ t.interior.vectors.T       # centre_i = sum_l c0l e_i^(l)
        interior[..., 0::2, :] = centre[..., None, :]
        interior[..., 1::2, :] = -centre[..., None, ::-1]
        d = np.einsum("...kl,kli->...ki", ck, t.p)       # (..., K-1, m)
        for i in range(ne):
            de = 0.5 * (d[..., i] + d[..., m - 1 - i]) if i < half else d[..., half]
            b = np.zeros(lead + (K,))
            b[..., :K - 1] = 2.0 * t.half_cos * de
            e = dst3_synthesis(b)                        # (..., K)
            if i < half:
                interior[..., :, i] += e
                interior[..., :, m - 1 - i] += e
            else:
                interior[..., :, half] += e
        for i in range(no):
            a = np.zeros(lead + (K,))
            a[..., 1:] = -2.0 * t.half_sin * (0.5 * (d[..., i] - d[..., m - 1 - i]))
            o = dct3_synthesis(a)
            interior[..., :, i] += o
            interior[..., :, m - 1 - i] -= o
    return join_line(nodal, interior, n, K)


# ----------------------------------------------------------------------------
# L5 algorithm (a): axis sweeps + symbol divide on a dof tensor
# ----------------------------------------------------------------------------


def _along(x: np.ndarray, axis: int, fn):
    moved = np.moveaxis(x, axis, -1)
    return np.moveaxis(fn(moved), -1, axis)


def scale_by_symbol(coef: np.ndarray, eigs, factors, shift: float) -> np.ndarray:
    """coef /= alpha + sum_i f_i lambda_i[t_i] (poisson.cpp:573-600); fails on denom <= 0."""
    N = coef.ndim
    denom = np.full(coef.shape, shift)
    for i in range(N):
        shape = [1] * N
        shape[i] = -1
        denom = denom + factors[i] * np.asarray(eigs[i]).reshape(shape)
    if not np.all(denom > 0):
        raise ValueError("solve: nonpositive denominator; shift too negative")
    return coef / denom


def axis_scale_factors(lengths, elements):
    """f_i = 4 / h_i^2 (poisson.cpp:398-405)."""
    return [4.0 / ((X / K) ** 2) for X, K in zip(lengths, elements)]


def solve_full_diagonalization(load: np.ndarray, orders, elements, lengths, shift,
                               coefficients=None) -> np.ndarray:
    """run_full_diagonalization (poisson.cpp:637-669) on a dof-layout load tensor.

    `coefficients` (a_i, default 1) multiplies axis i's factor: the operator
    -sum a_i d_i^2 u + alpha u.  The reference has a_i = 1; a_i = 2 equals the
    reference with X_i / sqrt(2), which the golden tests use.
    """
    N = load.ndim
    tabs = [table(orders[i], elements[i]) for i in range(N)]
    x = np.array(load, dtype=np.float64, copy=True)
    for axis in range(N):
        x = _along(x, axis, lambda v, t=tabs[axis]: decompose_weighted(v, t))
    f = axis_scale_factors(lengths, elements)
    if coefficients is not None:
        f = [fi * ai for fi, ai in zip(f, coefficients)]
    x = scale_by_symbol(x, [t.eigenvalues_coeff_order() for t in tabs], f, shift)
    for axis in range(N - 1, -1, -1):
        x = _along(x, axis, lambda v, t=tabs[axis]: synthesize(v, t))
    return x


# ----------------------------------------------------------------------------
# Dense references (oracle.hpp:13-55), small sizes only
# ----------------------------------------------------------------------------


def assemble_global_1d(n: int, K: int):
    """Dense A, C over the interleaved dof order (oracle.cpp:13-41)."""
    em = build_element_matrices(n)
    dim = n * K - 1

    def dof(e, loc):
        if loc == 0:
            return -1 if e == 0 else e * n - 1
        if loc == n:
            return -1 if e == K - 1 else (e + 1) * n - 1
        return e * n + loc - 1

    A = np.zeros((dim, dim))
    C = np.zeros((dim, dim))
    for e in range(K):
        for li in range(n + 1):
            gi = dof(e, li)
            if gi < 0:
                continue
            for lj in range(n + 1):
                gj = dof(e, lj)
                if gj < 0:
                    continue
                A[gi, gj] += em.stiffness[li, lj]
                C[gi, gj] += em.mass[li, lj]
    return A, C


def dense_solve(load: np.ndarray, orders, elements, lengths, shift, coefficients=None):
    """Kronecker-assembled direct solve (oracle.cpp:146-184)."""
    N = load.ndim
    mats = [assemble_global_1d(orders[i], elements[i]) for i in range(N)]
    f = axis_scale_factors(lengths, elements)
    if coefficients is not None:
        f = [fi * ai for fi, ai in zip(f, coefficients)]
    system = 0.0
    for t in range(N + 1):
        term = np.ones((1, 1))
        for i in range(N):
            term = np.kron(term, mats[i][0] if i == t else mats[i][1])
        system = system + (shift if t == N else f[t]) * term
    return np.linalg.solve(system, load.reshape(-1)).reshape(load.shape)


# ----------------------------------------------------------------------------
# The steps either side of the solve: operator application,
# FEM load averaging, the manufactured cases.  Small sizes only.
# ----------------------------------------------------------------------------


def _along_axis_matmul(mat: np.ndarray, x: np.ndarray, axis: int) -> np.ndarray:
    return np.moveaxis(np.tensordot(mat, x, axes=([1], [axis])), 0, axis)


def apply_operator(v: np.ndarray, orders, elements, lengths, shift, coefficients=None) -> np.ndarray:
    """A v with A = sum_t f_t (x)_{u!=t} C_u (x) A_t + shift (x)_u C_u (apply_operator,
    poisson.cpp:749-769; f_t = a_t 4/h_t^2, axis_scale_factors 398-405), using the
    assembled 1-D matrices of oracle.cpp:13-41 (assemble_global_1d)."""
    N = v.ndim
    mats = [assemble_global_1d(orders[i], elements[i]) for i in range(N)]
    f = axis_scale_factors(lengths, elements)
    if coefficients is not None:
        f = [fi * ai for fi, ai in zip(f, coefficients)]
    out = np.zeros_like(v)
    for t in range(N + 1):
        tmp = v
        for u in range(N):
            tmp = _along_axis_matmul(mats[u][0] if u == t else mats[u][1], tmp, u)
        out = out + (shift if t == N else f[t]) * tmp
    return out


def _axis_quad(n: int):
    """axis_quad (poisson.cpp:481-495): Gauss nodes and w_g * phi_loc(xi_g)."""
    gn, gw = gauss_legendre(n + 1)
    nodes = equispaced_nodes(n)
    wq = np.array([[gw[g] * lagrange_value(nodes, loc, gn[g]) for g in range(n + 1)] for loc in range(n + 1)])
    return np.array(gn), wq


def fem_load_average(orders, elements, lengths, rhs) -> np.ndarray:
    """fem_load_average (poisson.cpp:499-569) into the dof layout: per element,
    rhs on the tensor Gauss grid, one weighted-basis contraction per axis, the
    local load added into the dofs with the boundary contributions dropped.
    `rhs(x)` takes a list of coordinate arrays (broadcasting)."""
    N = len(orders)
    quad = [_axis_quad(n) for n in orders]
    h = [L / K for L, K in zip(lengths, elements)]
    ext = [n * K - 1 for n, K in zip(orders, elements)]
    out = np.zeros(ext)
    for e in np.ndindex(*elements):
        grids = np.meshgrid(*[(e[i] + 0.5 * (quad[i][0] + 1.0)) * h[i] for i in range(N)], indexing="ij")
        vals = rhs(grids)
        for ax in range(N - 1, -1, -1):
            vals = _along_axis_matmul(quad[ax][1], vals, ax)
        # scatter (dof coordinate t = e*n - 1 + loc; boundary dropped)
        idx = []
        keep = []
        for i in range(N):
            t = e[i] * orders[i] - 1 + np.arange(orders[i] + 1)
            idx.append(t)
            keep.append((t >= 0) & (t < ext[i]))
        sub = vals[np.ix_(*keep)]
        out[np.ix_(*[t[k] for t, k in zip(idx, keep)])] += sub
    return out


def case_functions(name: str, shift: float):
    """The reference's manufactured cases (cases.cpp:11-55, make_problem 81-95):
    (rhs, exact) as functions of a coordinate list; exact None for constantNd."""
    pi = math.pi
    if name == "sin1d":
        def u(x):
            return np.sin(pi * x[0]) * np.exp(x[0])

        def lap(x):
            return ((1.0 - pi * pi) * np.sin(pi * x[0]) + 2.0 * pi * np.cos(pi * x[0])) * np.exp(x[0])
    elif name == "poisson2d":
        def u(x):
            return np.sin(2 * pi * x[0]) * np.sin(3 * pi * x[1]) * np.cosh(math.sqrt(2.0) * x[0] - x[1])

        def lap(x):
            s1, c1 = np.sin(2 * pi * x[0]), np.cos(2 * pi * x[0])
            s2, c2 = np.sin(3 * pi * x[1]), np.cos(3 * pi * x[1])
            w = math.sqrt(2.0) * x[0] - x[1]
            return ((-13.0 * pi * pi + 3.0) * s1 * s2 * np.cosh(w)
                    + 2.0 * np.sinh(w) * (2.0 * math.sqrt(2.0) * pi * c1 * s2 - 3.0 * pi * s1 * c2))
    elif name == "poisson3d":
        def u(x):
            w = math.sqrt(2.0) * x[0] - x[1] + x[2] / math.sqrt(3.0)
            return np.sin(2 * pi * x[0]) * np.sin(3 * pi * x[1]) * np.sin(4 * pi * x[2]) * np.cosh(w)

        def lap(x):
            s1, c1 = np.sin(2 * pi * x[0]), np.cos(2 * pi * x[0])
            s2, c2 = np.sin(3 * pi * x[1]), np.cos(3 * pi * x[1])
            s3, c3 = np.sin(4 * pi * x[2]), np.cos(4 * pi * x[2])
            w = math.sqrt(2.0) * x[0] - x[1] + x[2] / math.sqrt(3.0)
            return ((-29.0 * pi * pi + 10.0 / 3.0) * s1 * s2 * s3 * np.cosh(w)
                    + 2.0 * np.sinh(w) * (2.0 * math.sqrt(2.0) * pi * c1 * s2 * s3 - 3.0 * pi * s1 * c2 * s3
                                          + 4.0 * pi / math.sqrt(3.0) * s1 * s2 * c3))
    elif name in ("constant1d", "constant2d", "constant3d"):
        return (lambda x: np.ones_like(x[0])), None
    else:
        raise ValueError(f"unknown case '{name}'")
    return (lambda x: -lap(x) + shift * u(x)), u


def dof_coordinates(orders, elements, lengths):
    """Per-axis coordinate of every dof (axis_coordinate, ndgrid.cpp:71-78)."""
    out = []
    for n, K, L in zip(orders, elements, lengths):
        h = L / K
        t = np.arange(n * K - 1)
        node = (t + 1) % n == 0
        x = np.where(node, h * ((t + 1) // n), h * (t // n + (t % n + 1) / n))
        out.append(x)
    return out
