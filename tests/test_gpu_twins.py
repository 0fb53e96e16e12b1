"""Device twins of the reference dispatchers vs the oracle and the golden
fixtures of the real reference (tests/golden/kernels_small.npz)."""

import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-13


@pytest.fixture(scope="module")
def ks(golden_dir):
    return dict(np.load(os.path.join(golden_dir, "kernels_small.npz")))


@pytest.fixture(scope="module")
def KD():
    from paper_2203_16657_b200 import _kernels

    return _kernels


def test_order_params(ks, KD):
    x, off = ks["x"], ks["offsets"]
    for p in (1, 2, 3):
        np.testing.assert_allclose(KD.order_params_blocks(x, off, p, math.pi, x.shape[0]),
                                   ks[f"op_p{p}"], rtol=0, atol=TOL)
        np.testing.assert_allclose(KD.order_params_blocks(x, off, p, 2.0, 13.0),
                                   ks[f"op_l2_p{p}"], rtol=0, atol=TOL)


def test_dense_complex_and_guard(ks, KD):
    x, off = ks["x"], ks["offsets"]
    o = ks["dc_out0"].copy()
    nv, mi = KD.dense_complex(x, off, ks["dc_tbl"], math.pi, o)
    np.testing.assert_allclose(o, ks["dc_out"], rtol=0, atol=TOL)
    assert nv == 0
    o = np.zeros_like(o)
    nv, mi = KD.dense_complex(x, off, ks["dcbad_tbl"], math.pi, o)
    assert nv == int(ks["dcbad_nviol"]) and abs(mi - float(ks["dcbad_maximag"])) < 1e-12
    np.testing.assert_allclose(o, ks["dcbad_out"], rtol=0, atol=TOL)


def test_dense_real_poly_moments(ks, KD):
    x, off = ks["x"], ks["offsets"]
    o = np.zeros_like(x)
    KD.dense_real(x, off, ks["dr_tc"], ks["dr_ts"], math.pi, o)
    np.testing.assert_allclose(o, ks["dr_out"], rtol=0, atol=TOL)
    o = np.zeros_like(x)
    KD.dense_poly(x, off, ks["dp_tbl"], 0.5, -0.1, o)
    np.testing.assert_allclose(o, ks["dp_out"], rtol=0, atol=TOL)
    np.testing.assert_allclose(KD.moments_blocks(x, off, 5, 0.3, x.shape[0]), ks["mom"],
                               rtol=1e-13, atol=TOL)


def test_pairs(ks, KD):
    x = ks["x"]
    n = x.shape[0]
    o = np.zeros_like(x)
    KD.pairs_trig(ks["pt_iu"], ks["pt_iv"], x, 1.0 / n, ks["pt_dcos"], ks["pt_dsin"], math.pi,
                  ks["pt_sgn"], o)
    np.testing.assert_allclose(o, ks["pt_out"], rtol=0, atol=1e-12)  # atomics: order-free sum
    o = np.zeros_like(ks["cs_pos"])
    KD.pairs_cs(ks["pt_iu"], ks["pt_iv"], ks["cs_pos"], ks["cs_vel"], 1.0 / n, 1.0, 1.0, 0.25,
                ks["pt_sgn"], o)
    np.testing.assert_allclose(o, ks["cs_out"], rtol=0, atol=1e-12)


def test_spec_kats_device(KD):
    r = KD.order_params_blocks(np.array([0.0, math.pi]), np.array([0, 2]), 2, math.pi, 2)
    assert abs(r[0, 3]) < 1e-15 and abs(r[0, 4] - 1) < 1e-15
    o = np.zeros(4)
    KD.pairs_trig(np.array([0]), np.array([3]), np.array([0, 0, 0, math.pi / 2]), 0.25,
                  np.zeros(2), np.array([0.0, 1.0]), math.pi, np.array([1.0]), o)
    np.testing.assert_allclose(o, [0.25, 0, 0, -0.25], atol=1e-16)
