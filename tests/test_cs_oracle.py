"""Cucker-Smale (config 4), CPU side: the P2 fit, the same-basis CIA
restatement against the direct sum through the reference kernel pairs_cs,
and the SPEC invariants."""

import numpy as np
import pytest

from oracle import cs as ocs
from oracle import kernels as K
from paper_2203_16657_b200 import configs, cs
from paper_2203_16657_b200 import graph as G


def _case(seed=0, sizes=(60, 80, 40), p_in=0.9, p_out=0.02):
    rng = np.random.default_rng(seed)
    g, part = G.planted_partition_graph(list(sizes), p_in, p_out, seed + 1)
    dec = G.decompose(g, part)
    n = g.n_nodes
    pos = rng.uniform(0, 10, (n, 2))
    vel = rng.standard_normal((n, 2))
    inv = part.inv_perm
    return g, dec, pos, vel, inv[g.edges[:, 0]], inv[g.edges[:, 1]]


def test_fit_exact_for_polynomial_coupling():
    """a coupling that is a polynomial of degree <= p is reproduced."""
    m = cs.CuckerSmale(K=1.0, sigma=1.0, beta=-3.0)  # eta = (1 + y)^3
    c, sup = cs.fit_eta(m, L=2.0)
    ref = np.array([1, 12, 48, 64, 0, 0, 0, 0, 0], dtype=float)  # (1 + 4u)^3
    np.testing.assert_allclose(c, ref, atol=1e-8)
    assert sup < 1e-8


def test_cia_restatement_bounded_error_vs_direct():
    """|cia - naive| <= sup_err * max|v_l - v_m| (+1e-9)."""
    g, dec, pos, vel, eu, ev = _case()
    model = cs.CuckerSmale()
    n = g.n_nodes
    plan = cs.cs_plan(model, dec, pos, vel, t_end=1.0)
    kd = ocs.cs_rhs_direct(K, pos, vel, eu, ev, 1.0, 1.0, 0.25, n)
    kc = ocs.cs_rhs_cia(K, pos, vel, dec, plan, 1.0, 1.0, 0.25, n)
    dv = np.sqrt(((vel[:, None, :] - vel[None, :, :]) ** 2).sum(-1)).max()
    lam_max = max(np.diff(dec.offsets))
    bound = plan.sup_err.max() * dv * lam_max / n + 1e-9
    assert np.abs(kd - kc).max() <= bound


def test_cia_exact_when_eta_is_polynomial():
    g, dec, pos, vel, eu, ev = _case(seed=3)
    n = g.n_nodes
    model = cs.CuckerSmale(beta=-2.0)  # eta = (1 + y)^2: exactly representable
    plan = cs.cs_plan(model, dec, pos, vel, t_end=1.0)
    kd = ocs.cs_rhs_direct(K, pos, vel, eu, ev, 1.0, 1.0, -2.0, n)
    kc = ocs.cs_rhs_cia(K, pos, vel, dec, plan, 1.0, 1.0, -2.0, n)
    assert np.abs(kd - kc).max() <= 1e-9 * np.abs(kd).max()


def test_momentum_conservation_direct_complete_graph():
    """sum v' = 0 on a complete graph (naive)."""
    rng = np.random.default_rng(1)
    n = 40
    iu, iv = np.triu_indices(n, 1)
    pos = rng.uniform(0, 10, (n, 2))
    vel = rng.standard_normal((n, 2))
    kd = ocs.cs_rhs_direct(K, pos, vel, iu, iv, 1.0, 1.0, 0.25, n)
    assert np.abs(kd.sum(0)).max() <= 1e-12


def test_config4_plan_domain():
    c = configs.config4()
    dec = c.decomposition()
    pos, vel = c.state()
    plan = cs.cs_plan(cs.CuckerSmale(c.K, c.sigma, c.beta), dec, pos, vel, c.t_end)
    assert plan.T.shape == (100, cs.NMON, cs.NMON)
    assert np.all(plan.L > 0)


def test_bank_spread_order_keeps_rows_and_spreads_banks():
    """cs._csr_bank_spread: every row keeps its set of missing columns; a pair
    of consecutive rows reading 4 consecutive entries each (one quarter-warp
    step of cs_sparse_win_kernel) meets fewer shared-memory bank conflicts
    than with sorted columns."""
    from paper_2203_16657_b200 import cs as CS
    from paper_2203_16657_b200 import graph as G
    from paper_2203_16657_b200.plan import build_layout

    dec = G.planted_partition_decomposition([600, 333], 0.9, 1e-3, 5)
    n = dec.n_nodes
    lay = build_layout(dec)
    rows, cols, sg = dec.directed()
    comm = dec.partition.comm_of_permuted()
    base = np.where(comm >= 0, dec.offsets[np.maximum(comm, 0)], 0).astype(np.int64)
    rb = np.searchsorted(lay.rblk_row0, np.arange(n), side="right") - 1
    par = ((np.arange(n) - lay.rblk_row0[np.minimum(rb, lay.n_rblk - 1)]) & 1).astype(np.int64)
    p0, c0 = CS._csr(rows[sg < 0], cols[sg < 0], n)
    p1, c1 = CS._csr_bank_spread(rows[sg < 0], cols[sg < 0], n, base, par)
    assert np.array_equal(p0, p1)
    for r in range(n):
        assert np.array_equal(np.sort(c1[p1[r]:p1[r + 1]]), c0[p0[r]:p0[r + 1]])

    def load(ptr, col):
        tot = steps = 0
        for r in range(0, 600 - 1, 2):  # pairs inside the first community's rblocks
            a = (col[ptr[r]:ptr[r + 1]] - base[r]) & 7
            b = (col[ptr[r + 1]:ptr[r + 2]] - base[r + 1]) & 7
            for k in range(0, max(len(a), len(b)), 4):
                q = np.r_[a[k:k + 4], b[k:k + 4]]
                tot += np.bincount(q, minlength=8).max()
                steps += 1
        return tot / steps

    assert load(p1, c1) < 0.8 * load(p0, c0)
