"""SURVEY §8(f) rank 4 model paths on the device (composed of the kernel
twins pinned in tests/test_f4_kernels.py): Desai–Zwanzig CIA vs naive and vs
the oracle's composition of the reference kernels, the Appendix-B rank-one
and nearest-neighbour fast paths vs direct sums, Bornholdt–Rohlf fast path
vs the literal double loop (exact)."""

import math

import numpy as np
import pytest

from oracle import kernels as K
from paper_2203_16657_b200 import graph as G

pytestmark = pytest.mark.gpu


def _dz_oracle(dec, x, coef, v_prime, n):
    """The same CIA composition over the oracle's reference-kernel restatement."""
    from math import comb

    out = -np.polynomial.polynomial.polyval(x, v_prime)
    p = len(coef) - 1
    w = K.moments_blocks(x, dec.offsets, p, 0.0, n)
    tbl = np.zeros((w.shape[0], p + 1))
    for b in range(p + 1):
        acc = sum(coef[a] * comb(a, b) * w[:, a - b] for a in range(b, p + 1))
        tbl[:, b] = acc if b % 2 == 0 else -acc
    K.dense_poly(x, dec.offsets, tbl, 1.0, 0.0, out)
    s = dec.correction
    K.pairs_poly(s.iu, s.iv, x, 1.0 / n, np.asarray(coef, float), 0.0, s.sgn, out)
    return out


def test_desai_zwanzig_cia_naive_oracle():
    from paper_2203_16657_b200.appendix_models import DesaiZwanzig, DzEngine

    g, part = G.planted_partition_graph([20, 15, 15], 0.8, 0.05, 3)
    dec = G.decompose(g, part)
    gp = dec.graph()
    rng = np.random.default_rng(0)
    for coef in ([0.0, 1.0], [0.0, 1.0, 0.0, 0.3]):  # h(x) = x (§A.4) and h(x) = x + 0.3 x^3
        model = DesaiZwanzig(50, np.array(coef))
        cia_e, naive_e = DzEngine(model, dec), DzEngine(model, gp)
        for _ in range(10):
            x = rng.uniform(-1.5, 1.5, 50)
            kc = cia_e.rhs(x).cpu().numpy()
            kn = naive_e.rhs(x).cpu().numpy()
            assert np.abs(kc - kn).max() <= 1e-11
            ko = _dz_oracle(dec, x, coef, model.v_prime, 50)
            assert np.abs(kc - ko).max() <= 1e-12
    # V' = 0, linear coupling on a complete graph: the mean is conserved
    gc, pc = G.planted_partition_graph([30], 1.0, 0.0, 1)
    dc = G.decompose(gc, pc)
    m0 = DesaiZwanzig(30, np.array([0.0, 1.0]), v_prime=(0.0,))
    x = rng.standard_normal(30)
    assert abs(float(DzEngine(m0, dc).rhs(x).sum())) <= 1e-13
    xs = DzEngine(m0, dc).rk4(x, 0.01, 50).cpu().numpy()
    assert abs(xs.mean() - x.mean()) <= 1e-12


def test_rank_one_and_nearest_neighbour():
    from paper_2203_16657_b200.appendix_models import nearest_neighbor_rhs, rank_one_rhs

    rng = np.random.default_rng(1)
    n = 50
    a, b, x = rng.standard_normal(n), rng.standard_normal(n), rng.uniform(-math.pi, math.pi, n)
    direct = a * ((b * np.exp(1j * x)).sum() / n) * np.exp(-1j * x)
    assert np.abs(rank_one_rhs(a, b, x) - direct).max() <= 1e-12
    assert np.abs(rank_one_rhs(a, np.zeros(n), x)).max() == 0.0
    # alpha = beta = 1: the single-community dense Kuramoto harmonic
    r = np.exp(1j * x).mean()
    assert np.abs(rank_one_rhs(np.ones(n), np.ones(n), x) - r * np.exp(-1j * x)).max() <= 1e-12
    for nn, k in ((6, 2), (5000, 7), (3001, 40)):
        x = rng.uniform(-math.pi, math.pi, nn)
        z = np.exp(1j * x)
        idx = (np.arange(nn)[:, None] + np.arange(-k, k + 1)[None, :]) % nn
        direct = z[idx].sum(1) / nn * np.exp(-1j * x)
        assert np.abs(nearest_neighbor_rhs(k, x) - direct).max() <= 1e-12
    x = np.full(4, 0.3)
    f = nearest_neighbor_rhs(1, x) * np.exp(1j * x)  # F_m = (3/4) e^{i theta}
    assert np.abs(f - 0.75 * np.exp(0.3j)).max() <= 1e-15


def test_bornholdt_rohlf_fast_equals_double_loop():
    from paper_2203_16657_b200.appendix_models import BornholdtRohlf, iterate_map

    rng = np.random.default_rng(2)
    v0 = np.where(rng.random(301) < 0.5, -1, 1)
    model = BornholdtRohlf(mu=-0.7, sigma=3.0)
    fast = iterate_map(model, v0, 50, seed=11)
    # literal double loop (oracle C restatement of _spin_field_sums_nb), same noise stream
    noise_rng = np.random.Generator(np.random.PCG64(11))
    v = v0.astype(np.int64)
    for step in range(50):
        f = K.spin_field_sums(v).astype(np.float64) + model.mu * v + model.sigma * \
            noise_rng.standard_normal(v.shape[0])
        v = np.where(f >= 0.0, 1, -1)
        assert np.array_equal(fast[step + 1], v), step
    # sigma = 0, all up, mu = 1: fixed point; balanced spins with mu = -1 all flip
    assert np.all(iterate_map(BornholdtRohlf(1.0, 0.0), np.ones(10, int), 100) == 1)
    vb = np.array([1, -1] * 5)
    assert np.array_equal(iterate_map(BornholdtRohlf(-1.0, 0.0), vb, 1)[1], -vb)
