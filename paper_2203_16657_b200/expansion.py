"""P2 expansion fitting on the host.

Represents a coupling function in a basis whose structure separates x_l from
x_m, so the E1 observables (order parameters / moments) can replace the pair
sums.  The fused device path consumes the real Fourier-difference form
(``fit_real_fourier_diff`` -> d_cos[0..p], d_sin[0..p]: the harmonics the
HigherHarmonicsKuramoto engine evaluates, p <= 8) and the polynomial forms
(``cs.fit_eta`` is the config-4 specialisation of ``fit_poly_diff``).

Kinds: complex_fourier_diff, real_fourier_diff,
complex_fourier_2d, real_fourier_2d, poly_diff, poly_2d.  Quadrature as the
SPEC's design decisions state: trapezoidal rule on a uniform periodic grid of
4(2p+1) points per axis for Fourier kinds (exact for trigonometric
polynomials of degree <= p), least squares in the monomials (x - x0)^a on
2(p+1) Chebyshev nodes per axis for polynomial kinds.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import CommdynError, InputError

KINDS = ("complex_fourier_diff", "real_fourier_diff", "complex_fourier_2d", "real_fourier_2d",
         "poly_diff", "poly_2d")


class ExpansionError(CommdynError):
    """Fitting failed (non-finite sample, order limit)."""


@dataclass(frozen=True)
class Expansion:
    kind: str
    p: int
    L: float = math.pi  # half width (Fourier kinds); interval half-length (poly kinds)
    x0: float = 0.0  # shift (poly kinds; centre of the interval)
    coef: np.ndarray = None  # see the fit_* docstrings for the layout
    y0: float = 0.0  # poly_2d second-axis shift

    # real_fourier_diff views (the device path's tables)
    @property
    def d_cos(self) -> np.ndarray:
        assert self.kind == "real_fourier_diff"
        return np.asarray(self.coef[0])

    @property
    def d_sin(self) -> np.ndarray:
        assert self.kind == "real_fourier_diff"
        return np.asarray(self.coef[1])


def _samples(f, pts, what):
    v = np.asarray(f(*pts) if isinstance(pts, tuple) else f(pts), dtype=np.float64)
    bad = ~np.isfinite(v)
    if bad.any():
        k = np.argwhere(bad)[0]
        at = tuple(float(np.asarray(p)[tuple(k)]) for p in pts) if isinstance(pts, tuple) else \
            float(np.asarray(pts)[tuple(k)])
        raise ExpansionError(f"{what}: non-finite sample at grid point {at}")
    return v


def _periodic_grid(p: int, L: float) -> np.ndarray:
    m = 4 * (2 * p + 1)
    return -L + 2.0 * L * np.arange(m) / m


def fit_fourier_diff(h, p: int, L: float = math.pi) -> Expansion:
    """d_alpha = (1/2L) int_{-L}^{L} h(x) e^{-i pi alpha x / L} dx, alpha = -p..p,
    stored at index alpha + p; conjugate symmetry enforced."""
    if p < 0 or L <= 0:
        raise InputError("need p >= 0 and L > 0")
    x = _periodic_grid(p, L)
    v = _samples(h, x, "fit_fourier_diff")
    a = np.arange(-p, p + 1)
    d = (v[None, :] * np.exp(-1j * math.pi * a[:, None] * x[None, :] / L)).mean(axis=1)
    d = 0.5 * (d + np.conj(d[::-1]))  # d_-a = conj(d_a)
    return Expansion("complex_fourier_diff", p, float(L), 0.0, d)


def fit_real_fourier_diff(h, p: int, L: float = math.pi) -> Expansion:
    """coef = (d_cos[0..p], d_sin[0..p]) with h(x) ~ sum_a d_cos[a] cos(pi a x/L)
    + d_sin[a] sin(pi a x/L): d_cos[a] = 2 Re d_a, d_sin[a] = -2 Im d_a (a >= 1),
    d_cos[0] = Re d_0, d_sin[0] = 0."""
    c = fit_fourier_diff(h, p, L).coef
    dcos = np.empty(p + 1)
    dsin = np.zeros(p + 1)
    dcos[0] = c[p].real
    for a in range(1, p + 1):
        dcos[a] = 2.0 * c[p + a].real
        dsin[a] = -2.0 * c[p + a].imag
    return Expansion("real_fourier_diff", p, float(L), 0.0, np.stack([dcos, dsin]))


def fit_fourier_2d(g, p: int, L: float = math.pi, kind: str = "real") -> Expansion:
    """g(x, y) on [-L, L]^2.  complex: c[a+p, b+p] of
    e^{i pi (a x + b y)/L}; real: coef[k][a, b], k = 0..3 the tables
    c11 (cos a x cos b y), c12 (cos a x sin b y), c21 (sin a x cos b y),
    c22 (sin a x sin b y), a, b = 0..p."""
    if p < 0 or L <= 0:
        raise InputError("need p >= 0 and L > 0")
    x = _periodic_grid(p, L)
    X, Y = np.meshgrid(x, x, indexing="ij")
    v = _samples(g, (X, Y), "fit_fourier_2d")
    a = np.arange(-p, p + 1)
    ex = np.exp(-1j * math.pi * a[:, None] * x[None, :] / L)  # [2p+1, m]
    c = ex @ v @ ex.T / (x.size * x.size)  # c[a, b]
    c = 0.5 * (c + np.conj(c[::-1, ::-1]))
    if kind == "complex":
        return Expansion("complex_fourier_2d", p, float(L), 0.0, c)
    if kind != "real":
        raise InputError("kind must be 'real' or 'complex'")
    # e^{i(ax+by)} + e^{-i(ax+by)} and e^{i(ax-by)} + e^{-i(ax-by)} pairs -> real tables
    tab = np.zeros((4, p + 1, p + 1))
    for ia in range(p + 1):
        for ib in range(p + 1):
            cpp = c[p + ia, p + ib]
            cpm = c[p + ia, p - ib]
            # sum over (+-a, +-b): 2Re(cpp e^{i(ax+by)}) + 2Re(cpm e^{i(ax-by)}), halved at a=0 or b=0
            w = (1.0 if ia == 0 else 2.0) * (1.0 if ib == 0 else 2.0) / 2.0
            if ia == 0 and ib == 0:
                tab[0, 0, 0] = cpp.real
                continue
            # Re(c e^{i(ax+by)}) = Re c (cos cos - sin sin) - Im c (sin cos + cos sin)
            tab[0, ia, ib] = w * (cpp.real + cpm.real)
            tab[3, ia, ib] = w * (-cpp.real + cpm.real)
            tab[2, ia, ib] = w * (-cpp.imag - cpm.imag)
            tab[1, ia, ib] = w * (-cpp.imag + cpm.imag)
    return Expansion("real_fourier_2d", p, float(L), 0.0, tab)


def _cheb(p: int, lo: float, hi: float) -> np.ndarray:
    m = 2 * (p + 1)
    k = np.arange(m)
    return 0.5 * (lo + hi) + 0.5 * (hi - lo) * np.cos((2 * k + 1) * math.pi / (2 * m))


def fit_poly_diff(h, p: int, interval=(-1.0, 1.0), x0: float | None = None) -> Expansion:
    """h(x) ~ sum_a c[a] (x - x0)^a, least squares on 2(p+1) Chebyshev nodes of
    ``interval``; x0 defaults to the midpoint."""
    lo, hi = (float(interval[0]), float(interval[1]))
    if p < 0 or not lo < hi:
        raise InputError("need p >= 0 and lo < hi")
    x0 = 0.5 * (lo + hi) if x0 is None else float(x0)
    x = _cheb(p, lo, hi)
    v = _samples(h, x, "fit_poly_diff")
    V = np.vander(x - x0, p + 1, increasing=True)
    c, *_ = np.linalg.lstsq(V, v, rcond=None)
    return Expansion("poly_diff", p, 0.5 * (hi - lo), x0, c)


def fit_poly_2d(g, p: int, domain=((-1.0, 1.0), (-1.0, 1.0))) -> Expansion:
    """g(x, y) ~ sum_{a,b <= p} c[a, b] (x - x0)^a (y - y0)^b on the Chebyshev
    tensor grid (2(p+1) nodes per axis)."""
    (xl, xh), (yl, yh) = domain
    if p < 0 or not (xl < xh and yl < yh):
        raise InputError("need p >= 0 and a nonempty domain")
    x0, y0 = 0.5 * (xl + xh), 0.5 * (yl + yh)
    xs, ys = _cheb(p, xl, xh), _cheb(p, yl, yh)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    v = _samples(g, (X, Y), "fit_poly_2d").reshape(-1)
    Vx = np.vander(X.reshape(-1) - x0, p + 1, increasing=True)
    Vy = np.vander(Y.reshape(-1) - y0, p + 1, increasing=True)
    A = (Vx[:, :, None] * Vy[:, None, :]).reshape(v.size, -1)
    c, *_ = np.linalg.lstsq(A, v, rcond=None)
    return Expansion("poly_2d", p, 0.5 * (xh - xl), x0, c.reshape(p + 1, p + 1), y0)


def eval_expansion(e: Expansion, x, y=None):
    """Finite-series value; complex kinds assert the
    imaginary residue <= 1e-9 (1 + |value|)."""
    x = np.asarray(x, dtype=np.float64)
    two_d = e.kind.endswith("_2d")
    if two_d != (y is not None):
        raise InputError(f"{e.kind} takes {'two arguments' if two_d else 'one argument'}")
    if e.kind == "complex_fourier_diff":
        a = np.arange(-e.p, e.p + 1)
        v = (e.coef[None, :] * np.exp(1j * math.pi * np.multiply.outer(x.reshape(-1), a) / e.L)
             ).sum(axis=1).reshape(x.shape)
        if np.any(np.abs(v.imag) > 1e-9 * (1.0 + np.abs(v.real))):
            raise ExpansionError("imaginary residue above 1e-9")
        return v.real
    if e.kind == "real_fourier_diff":
        a = np.arange(e.p + 1)
        t = math.pi * np.multiply.outer(x, a) / e.L
        return (np.cos(t) * e.coef[0] + np.sin(t) * e.coef[1]).sum(axis=-1)
    if e.kind == "poly_diff":
        return np.polynomial.polynomial.polyval(x - e.x0, e.coef)
    y = np.asarray(y, dtype=np.float64)
    if e.kind == "complex_fourier_2d":
        a = np.arange(-e.p, e.p + 1)
        ex = np.exp(1j * math.pi * np.multiply.outer(x.reshape(-1), a) / e.L)
        ey = np.exp(1j * math.pi * np.multiply.outer(y.reshape(-1), a) / e.L)
        v = np.einsum("na,ab,nb->n", ex, e.coef, ey).reshape(x.shape)
        if np.any(np.abs(v.imag) > 1e-9 * (1.0 + np.abs(v.real))):
            raise ExpansionError("imaginary residue above 1e-9")
        return v.real
    if e.kind == "real_fourier_2d":
        a = np.arange(e.p + 1)
        tx = math.pi * np.multiply.outer(x.reshape(-1), a) / e.L
        ty = math.pi * np.multiply.outer(y.reshape(-1), a) / e.L
        cx, sx, cy, sy = np.cos(tx), np.sin(tx), np.cos(ty), np.sin(ty)
        v = (np.einsum("na,ab,nb->n", cx, e.coef[0], cy) + np.einsum("na,ab,nb->n", cx, e.coef[1], sy)
             + np.einsum("na,ab,nb->n", sx, e.coef[2], cy)
             + np.einsum("na,ab,nb->n", sx, e.coef[3], sy))
        return v.reshape(x.shape)
    if e.kind == "poly_2d":
        return np.polynomial.polynomial.polyval2d(x - e.x0, y - e.y0, e.coef)
    raise InputError(f"unknown kind {e.kind!r}")


def expansion_sup_error(e: Expansion, f, grid_density: int = 1001) -> float:
    """max |eval_expansion - f| on a uniform grid of the expansion's domain."""
    if e.kind.endswith("_2d"):
        lo_x, hi_x = (-e.L, e.L) if "fourier" in e.kind else (e.x0 - e.L, e.x0 + e.L)
        g = np.linspace(lo_x, hi_x, int(math.sqrt(grid_density)) + 1)
        X, Y = np.meshgrid(g, g if "fourier" in e.kind else g - e.x0 + e.y0, indexing="ij")
        return float(np.abs(eval_expansion(e, X, Y) - np.asarray(f(X, Y))).max())
    lo, hi = (-e.L, e.L) if "fourier" in e.kind else (e.x0 - e.L, e.x0 + e.L)
    x = np.linspace(lo, hi, grid_density)
    return float(np.abs(eval_expansion(e, x) - np.asarray(f(x))).max())


def auto_order(fit, f, tol: float, max_p: int = 64, **kw) -> Expansion:
    """Double p from 1 until expansion_sup_error <= tol; error at
    p = max_p."""
    p = 1
    while True:
        e = fit(f, p, **kw)
        if expansion_sup_error(e, f) <= tol:
            return e
        if p >= max_p:
            raise ExpansionError(f"sup error above {tol} at p = {max_p}")
        p = min(2 * p, max_p)


def dump_csv(e: Expansion, path: str) -> None:
    """Header ``kind,p,L,x0`` then rows ``alpha[,beta],re,im``."""
    with open(path, "w") as f:
        f.write("kind,p,L,x0\n")
        f.write(f"{e.kind},{e.p},{float(e.L)!r},{float(e.x0)!r}\n")
        c = np.asarray(e.coef)
        if e.kind == "complex_fourier_diff":
            for i, v in enumerate(c):
                f.write(f"{i - e.p},{float(v.real)!r},{float(v.imag)!r}\n")
        elif e.kind == "real_fourier_diff":  # alpha, cos, sin
            for a in range(e.p + 1):
                f.write(f"{a},{float(c[0, a])!r},{float(c[1, a])!r}\n")
        elif e.kind == "poly_diff":
            for a, v in enumerate(c):
                f.write(f"{a},{float(v)!r},0.0\n")
        elif e.kind == "complex_fourier_2d":
            for i in range(c.shape[0]):
                for j in range(c.shape[1]):
                    f.write(f"{i - e.p},{j - e.p},{float(c[i, j].real)!r},{float(c[i, j].imag)!r}\n")
        else:
            raise InputError(f"dump_csv: {e.kind} not supported")


def load_csv(path: str) -> Expansion:
    with open(path) as f:
        lines = [ln.strip() for ln in f if ln.strip()]
    kind, p, L, x0 = lines[1].split(",")
    p = int(p)
    rows = [[float(t) for t in ln.split(",")] for ln in lines[2:]]
    if kind == "complex_fourier_diff":
        coef = np.array([r[1] + 1j * r[2] for r in rows])
    elif kind == "real_fourier_diff":
        coef = np.array([[r[1] for r in rows], [r[2] for r in rows]])
    elif kind == "poly_diff":
        coef = np.array([r[1] for r in rows])
    elif kind == "complex_fourier_2d":
        coef = np.array([r[2] + 1j * r[3] for r in rows]).reshape(2 * p + 1, 2 * p + 1)
    else:
        raise InputError(f"load_csv: {kind} not supported")
    return Expansion(kind, p, float(L), float(x0), coef)
