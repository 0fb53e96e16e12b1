"""P2 expansion fitters against the SPEC's examples and
invariants (host code, CPU)."""

import math

import numpy as np
import pytest

from paper_2203_16657_b200 import expansion as X


def test_fourier_diff_sin_exact():
    e = X.fit_fourier_diff(np.sin, 1, math.pi)
    np.testing.assert_allclose(e.coef, [-1 / 2j, 0, 1 / 2j], atol=1e-12)


def test_fourier_diff_const_and_cos2():
    e = X.fit_fourier_diff(lambda x: np.ones_like(x), 0)
    np.testing.assert_allclose(e.coef, [1.0], atol=1e-12)
    e = X.fit_fourier_diff(lambda x: np.cos(2 * x), 3)
    want = np.zeros(7, complex)
    want[3 + 2] = want[3 - 2] = 0.5
    np.testing.assert_allclose(e.coef, want, atol=1e-12)


def test_real_fourier_diff_examples():
    e = X.fit_real_fourier_diff(np.sin, 1)
    np.testing.assert_allclose(e.d_sin, [0, 1], atol=1e-12)
    np.testing.assert_allclose(e.d_cos, [0, 0], atol=1e-12)
    e = X.fit_real_fourier_diff(np.cos, 1)
    np.testing.assert_allclose(e.d_cos, [0, 1], atol=1e-12)
    e = X.fit_real_fourier_diff(lambda x: np.zeros_like(x), 3)
    assert np.all(e.coef == 0)


def test_random_trig_polynomial_reproduced_and_symmetric():
    rng = np.random.default_rng(0)
    for p in (1, 2, 4, 8):
        dc, ds = rng.standard_normal(p + 1), rng.standard_normal(p + 1)
        ds[0] = 0.0
        h = lambda x: sum(dc[a] * np.cos(a * x) + ds[a] * np.sin(a * x) for a in range(p + 1))  # noqa: E731
        e = X.fit_real_fourier_diff(h, p)
        np.testing.assert_allclose(e.d_cos, dc, atol=1e-10)
        np.testing.assert_allclose(e.d_sin, ds, atol=1e-10)
        c = X.fit_fourier_diff(h, p).coef
        np.testing.assert_allclose(c, np.conj(c[::-1]), atol=1e-12)
        x = rng.uniform(-math.pi, math.pi, 1000)
        np.testing.assert_allclose(X.eval_expansion(e, x), h(x), atol=1e-10)
        assert X.expansion_sup_error(e, h) <= 1e-10


def test_fourier_2d_examples():
    e = X.fit_fourier_2d(lambda x, y: np.sin(x - y), 1)
    t = e.coef
    assert abs(t[2, 1, 1] - 1) < 1e-12 and abs(t[1, 1, 1] + 1) < 1e-12
    t2 = t.copy()
    t2[2, 1, 1] = t2[1, 1, 1] = 0
    assert np.abs(t2).max() < 1e-12
    e = X.fit_fourier_2d(lambda x, y: np.cos(x) * np.cos(y), 1)
    assert abs(e.coef[0, 1, 1] - 1) < 1e-12
    e = X.fit_fourier_2d(lambda x, y: 3.0 + 0 * x, 2, kind="complex")
    assert abs(e.coef[2, 2] - 3) < 1e-12 and np.abs(e.coef).sum() - 3 < 1e-10
    rng = np.random.default_rng(1)
    x, y = rng.uniform(-math.pi, math.pi, (2, 200))
    g = lambda a, b: np.sin(a - 2 * b) + 0.3 * np.cos(2 * a) * np.sin(b)  # noqa: E731
    for kind in ("real", "complex"):
        e = X.fit_fourier_2d(g, 2, kind=kind)
        np.testing.assert_allclose(X.eval_expansion(e, x, y), g(x, y), atol=1e-10)


def test_poly_examples():
    e = X.fit_poly_diff(lambda x: x, 1, (-1, 1), x0=0.0)
    np.testing.assert_allclose(e.coef, [0, 1], atol=1e-10)
    e = X.fit_poly_diff(lambda x: x * x, 2, (-1, 1), x0=0.0)
    np.testing.assert_allclose(e.coef, [0, 0, 1], atol=1e-10)
    e = X.fit_poly_diff(np.exp, 4, (-1, 1))
    assert X.expansion_sup_error(e, np.exp, 1000) <= 1e-3
    assert X.eval_expansion(X.fit_poly_diff(lambda x: x, 1, (-1, 1)), 0.3) == pytest.approx(0.3)
    e = X.fit_poly_2d(lambda x, y: x * y + 2 * y * y, 2)
    rng = np.random.default_rng(2)
    x, y = rng.uniform(-1, 1, (2, 50))
    np.testing.assert_allclose(X.eval_expansion(e, x, y), x * y + 2 * y * y, atol=1e-10)


def test_convergence_and_auto_order():
    f = lambda x: np.exp(np.cos(x))  # noqa: E731
    errs = [X.expansion_sup_error(X.fit_real_fourier_diff(f, p), f) for p in (2, 4, 8, 16)]
    assert all(b <= a for a, b in zip(errs, errs[1:]))
    e = X.auto_order(X.fit_real_fourier_diff, f, 1e-8)
    assert e.p in (8, 16) and X.expansion_sup_error(e, f) <= 1e-8
    with pytest.raises(X.ExpansionError):
        X.auto_order(X.fit_real_fourier_diff, lambda x: np.abs(x), 1e-12, max_p=8)


def test_errors_and_csv_roundtrip(tmp_path):
    with pytest.raises(X.ExpansionError, match="grid point"):
        X.fit_fourier_diff(lambda x: 1.0 / (x - x[5]), 2)
    with pytest.raises(X.InputError):
        X.eval_expansion(X.fit_fourier_diff(np.sin, 1), 0.1, 0.2)
    for e in (X.fit_fourier_diff(np.sin, 2), X.fit_real_fourier_diff(np.cos, 3),
              X.fit_poly_diff(np.exp, 3, (0, 2))):
        p = tmp_path / f"{e.kind}.csv"
        X.dump_csv(e, str(p))
        assert p.read_text().splitlines()[0] == "kind,p,L,x0"
        e2 = X.load_csv(str(p))
        assert (e2.kind, e2.p) == (e.kind, e.p)
        np.testing.assert_allclose(e2.coef, e.coef, rtol=0, atol=0)
