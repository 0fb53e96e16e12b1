"""Pin the oracle (C restatement + SPEC orchestration) against fixtures made by
the REAL reference kernels (tests/golden/make_golden.py), plus the SPEC KATs
the oracle must satisfy.  CPU only."""

import hashlib
import math
import os

import numpy as np
import pytest

from oracle import cia
from oracle import kernels as K
from paper_2203_16657_b200 import configs

TOL = 1e-13


@pytest.fixture(scope="module")
def ks(golden_dir):
    return dict(np.load(os.path.join(golden_dir, "kernels_small.npz")))


def dec_hash(dec):
    h = hashlib.sha256()
    s = dec.correction
    for a in (s.iu, s.iv, s.sgn, dec.offsets):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_order_params_vs_reference(ks):
    x, off = ks["x"], ks["offsets"]
    n = x.shape[0]
    for p in (1, 2, 3):
        np.testing.assert_allclose(K.order_params_blocks(x, off, p, math.pi, n), ks[f"op_p{p}"],
                                   rtol=0, atol=TOL)
        np.testing.assert_allclose(K.order_params_blocks(x, off, p, 2.0, 13.0),
                                   ks[f"op_l2_p{p}"], rtol=0, atol=TOL)


def test_dense_complex_vs_reference(ks):
    x, off = ks["x"], ks["offsets"]
    o = ks["dc_out0"].copy()
    nv, mi = K.dense_complex(x, off, ks["dc_tbl"], math.pi, o)
    np.testing.assert_allclose(o, ks["dc_out"], rtol=0, atol=TOL)
    assert nv == int(ks["dc_nviol"]) == 0
    o = np.zeros_like(o)
    nv, mi = K.dense_complex(x, off, ks["dcbad_tbl"], math.pi, o)
    assert nv == int(ks["dcbad_nviol"]) > 0
    assert abs(mi - float(ks["dcbad_maximag"])) < TOL
    np.testing.assert_allclose(o, ks["dcbad_out"], rtol=0, atol=TOL)


def test_dense_real_vs_reference(ks):
    o = np.zeros_like(ks["x"])
    K.dense_real(ks["x"], ks["offsets"], ks["dr_tc"], ks["dr_ts"], math.pi, o)
    np.testing.assert_allclose(o, ks["dr_out"], rtol=0, atol=TOL)


@pytest.mark.parametrize("threads", [1, 3])
def test_pairs_trig_vs_reference(ks, threads):
    K.set_threads(threads)
    try:
        x = ks["x"]
        o = np.zeros_like(x)
        K.pairs_trig(ks["pt_iu"], ks["pt_iv"], x, 1.0 / x.shape[0], ks["pt_dcos"], ks["pt_dsin"],
                     math.pi, ks["pt_sgn"], o)
        np.testing.assert_allclose(o, ks["pt_out"], rtol=0, atol=TOL)
    finally:
        K.set_threads(1)


@pytest.mark.parametrize("threads", [1, 4])
def test_pairs_cs_vs_reference(ks, threads):
    K.set_threads(threads)
    try:
        o = np.zeros_like(ks["cs_pos"])
        n = o.shape[0]
        K.pairs_cs(ks["pt_iu"], ks["pt_iv"], ks["cs_pos"], ks["cs_vel"], 1.0 / n, 1.0, 1.0, 0.25,
                   ks["pt_sgn"], o)
        np.testing.assert_allclose(o, ks["cs_out"], rtol=0, atol=TOL)
    finally:
        K.set_threads(1)


def test_moments_poly_ho_vs_reference(ks):
    x, off = ks["x"], ks["offsets"]
    np.testing.assert_allclose(K.moments_blocks(x, off, 5, 0.3, x.shape[0]), ks["mom"],
                               rtol=1e-14, atol=TOL)
    o = np.zeros_like(x)
    K.dense_poly(x, off, ks["dp_tbl"], 0.5, -0.1, o)
    np.testing.assert_allclose(o, ks["dp_out"], rtol=0, atol=TOL)
    np.testing.assert_allclose(K.ho_naive_block(ks["ho_theta"], (1, 1, 0, -2)), ks["ho_1102"],
                               rtol=0, atol=TOL)
    np.testing.assert_allclose(K.ho_naive_block(ks["ho_theta"], (1, 1, -1, -1)),
                               ks["ho_11m1m1"], rtol=0, atol=TOL)


def test_cfg1_trajectory_vs_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "cfg1.npz"))
    c = configs.config1()
    dec = c.decomposition()
    assert dec_hash(dec) == str(g["dec_sha256"]), "generator drifted from the fixture"
    omega, theta0 = c.state()
    s = dec.correction

    def rhs(x):
        return cia.kuramoto_rhs_cia(K, x, omega, dec.offsets, s.iu, s.iv, s.sgn, c.coupling, c.n)

    np.testing.assert_allclose(rhs(theta0), g["rhs0_cia"], rtol=0, atol=1e-14)
    fin, snaps = cia.rk4_integrate(rhs, theta0, c.dt, c.steps, record_every=100)
    assert cia.circ_dist(fin, g["final_cia"]).max() <= 1e-12
    assert cia.circ_dist(fin, g["final_naive"]).max() <= 1e-9
    for (st, x), gs, gx in zip(snaps, g["snap_steps"], g["snaps"]):
        assert st == gs and cia.circ_dist(x, gx).max() <= 1e-12


@pytest.mark.slow
def test_cfg2_rhs_vs_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "cfg2_sample.npz"))
    c = configs.config2()
    dec = c.decomposition()
    assert dec_hash(dec) == str(g["dec_sha256"])
    omega, theta0 = c.state()
    s = dec.correction
    K.set_threads(K.max_threads())
    try:
        k0 = cia.kuramoto_rhs_cia(K, theta0, omega, dec.offsets, s.iu, s.iv, s.sgn, c.coupling, c.n)
    finally:
        K.set_threads(1)
    np.testing.assert_allclose(k0[g["idx"]], g["rhs0"], rtol=0, atol=1e-13)
    assert abs(k0.sum() - float(g["rhs0_sum"])) < 1e-8


def test_spec_kats_oracle():
    # SPEC.md:261-262 order parameters
    r = K.order_params_blocks(np.zeros(5), np.array([0, 5]), 2, math.pi, 5)
    np.testing.assert_allclose(r, np.ones((1, 5)), atol=1e-15)
    r = K.order_params_blocks(np.array([0.0, math.pi]), np.array([0, 2]), 2, math.pi, 2)
    assert abs(r[0, 3]) < 1e-15 and abs(r[0, 4] - 1) < 1e-15
    # SPEC.md:356 sparse KAT: S={(0,3,+1)}, theta0=0, theta3=pi/2, N=4
    o = np.zeros(4)
    K.pairs_trig(np.array([0]), np.array([3]), np.array([0, 0, 0, math.pi / 2]), 0.25,
                 np.zeros(2), np.array([0.0, 1.0]), math.pi, np.array([1.0]), o)
    np.testing.assert_allclose(o, [0.25, 0, 0, -0.25], atol=1e-16)
    # SPEC.md:373 naive K2: theta=(0, pi/2), omega=0 -> (0.5, -0.5)
    k = cia.kuramoto_rhs_naive(K, np.array([0.0, math.pi / 2]), np.zeros(2), np.array([0]),
                               np.array([1]), 1.0, 2)
    np.testing.assert_allclose(k, [0.5, -0.5], atol=1e-16)
    # SPEC.md:546 RK4 order ratio on x' = -x
    def err(dt):
        x, _ = cia.rk4_integrate(lambda x: -x, np.array([1.0]), dt, int(round(1 / dt)), wrap=False)
        return abs(x[0] - math.exp(-1))
    ratio = err(0.1) / err(0.05)
    assert 12 <= ratio <= 20
    # SPEC.md:535 Euler one step
    assert abs(cia.euler_integrate(lambda x: -x, np.array([1.0]), 0.1, 1, wrap=False)[0] - 0.9) < 1e-15
