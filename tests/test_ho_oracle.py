"""Higher-order (triadic) Kuramoto, CPU side: the CIA restatement (oracle/ho.py)
against the literal triangle sum, the reference's ho_naive_block pinning the
dense part, and the host triangle preparation."""

import math

import numpy as np
import pytest

from oracle import ho as oh
from oracle import kernels as K
from paper_2203_16657_b200 import configs
from paper_2203_16657_b200 import graph as G
from paper_2203_16657_b200 import ho


def _with_pool(g, part, rng, k):
    a = part.assignment.copy()
    a[rng.choice(a.shape[0], k, replace=False)] = -1
    used = np.unique(a[a >= 0])
    remap = -np.ones(a.max() + 2, dtype=np.int64)
    remap[used] = np.arange(used.size)
    return G.Partition.from_assignment(np.where(a >= 0, remap[a], -1))


@pytest.mark.parametrize("seed,pool", [(0, 0), (1, 0), (2, 12)])
def test_cia_restatement_equals_triangle_sum(seed, pool):
    rng = np.random.default_rng(seed)
    g, part = G.planted_partition_graph([35, 20, 50, 4, 1], 0.8, 0.08, seed)
    if pool:
        part = _with_pool(g, part, rng, pool)
    dec = G.decompose(g, part)
    A = g.dense()[np.ix_(part.perm, part.perm)]
    th = rng.uniform(-math.pi, math.pi, g.n_nodes)
    om = rng.standard_normal(g.n_nodes)
    kd = oh.ho_rhs_direct(th, om, A, 1.0, 0.5)
    kc = oh.ho_rhs_cia(th, om, dec, 1.0, 0.5, inter_triangles=ho.spanning_triangles(dec))
    assert np.abs(kd - kc).max() <= 1e-12


def test_dense_part_pinned_by_reference_ho_naive_block():
    """Complete community block: the CIA dense part Im(Z^2 conj z_m^2)/lam^2 is
    the reference's all-to-all block sum ho_naive_block(theta, (1,1,0,-2))
    (_kernels.py:398-428; fixture from the real reference in kernels_small.npz)."""
    import os

    ks = np.load(os.path.join(os.path.dirname(__file__), "golden", "kernels_small.npz"))
    th = ks["ho_theta"]
    z = np.exp(1j * th)
    Z = z.sum()
    dense = np.imag(Z * Z * np.conj(z) ** 2) / th.shape[0] ** 2
    assert np.abs(dense - ks["ho_1102"]).max() <= 1e-13
    assert np.abs(dense - K.ho_naive_block(th, (1, 1, 0, -2))).max() <= 1e-13


def test_triangle_preparation_counts():
    dec = G.planted_partition_decomposition([60, 60, 60], 0.9, 0.02, 4)
    mt = ho.missing_triangles(dec)
    # brute force on the missing graph
    s = dec.correction
    m = (s.sgn < 0) & (s.iu != s.iv)
    n = dec.n_nodes
    M = np.zeros((n, n), dtype=np.int64)
    M[s.iu[m], s.iv[m]] = 1
    M = M + M.T
    assert len(mt) == int(np.trace(M @ M @ M)) // 6
    assert np.all(mt[:, 0] < mt[:, 1]) and np.all(mt[:, 1] < mt[:, 2])
    assert np.all(M[mt[:, 0], mt[:, 1]] & M[mt[:, 1], mt[:, 2]] & M[mt[:, 0], mt[:, 2]])


@pytest.mark.slow
def test_config3_scaled_oracles_agree():
    c = configs.scaled_config3(m=6, lam=100, p_out=3e-3)
    dec = c.decomposition()
    omega, theta0 = c.state()
    rows, cols, sg = dec.directed()
    n = c.n
    A = np.ones((n, n))
    off = dec.offsets
    A[:] = 0
    for k in range(len(c.sizes)):
        A[off[k]:off[k + 1], off[k]:off[k + 1]] = 1
    np.fill_diagonal(A, 0)
    A[rows, cols] += sg
    kd = oh.ho_rhs_direct(theta0, omega, A, c.k1, c.k2)
    kc = oh.ho_rhs_cia(theta0, omega, dec, c.k1, c.k2, inter_triangles=ho.spanning_triangles(dec))
    assert np.abs(kd - kc).max() <= 1e-12


@pytest.mark.parametrize("seed,pool", [(0, 0), (5, 9)])
def test_precomputed_cia_oracle_equals_restatement(seed, pool):
    """oracle.ho.HoCia (enumerated missing and spanning triangles, used for
    the long-horizon config-3 fixture) equals ho_rhs_cia and the literal sum."""
    rng = np.random.default_rng(seed)
    g, part = G.planted_partition_graph([45, 30, 50, 4, 1], 0.7, 0.1, seed)
    if pool:
        part = _with_pool(g, part, rng, pool)
    dec = G.decompose(g, part)
    orc = oh.HoCia(dec)
    span = ho.spanning_triangles(dec)
    assert {tuple(t) for t in orc.span.tolist()} == {tuple(t) for t in span.tolist()}
    mt = ho.missing_triangles(dec)
    assert {tuple(t) for t in orc.tri.tolist()} == {tuple(t) for t in mt.tolist()}
    A = g.dense()[np.ix_(part.perm, part.perm)]
    th = rng.uniform(-math.pi, math.pi, g.n_nodes)
    om = rng.standard_normal(g.n_nodes)
    kd = oh.ho_rhs_direct(th, om, A, 1.0, 0.5)
    kc = orc.rhs(th, om, 1.0, 0.5)
    assert np.abs(kd - kc).max() <= 1e-12
    assert np.abs(kc - oh.ho_rhs_cia(th, om, dec, 1.0, 0.5, inter_triangles=span)).max() <= 1e-13
