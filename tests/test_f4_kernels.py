"""SURVEY §8(f) rank 4 kernels — pairs_poly (Desai–Zwanzig coupling,
_kernels.py:264-294,365-369), nn_recurrence (Appendix B window sums,
:436-477), spin_field_sums (Bornholdt–Rohlf oracle, :485-509) and
ho_naive_block at a 40-node block (:398-428): the oracle C restatement (CPU)
and the device twins (GPU) against fixtures made by the REAL reference
(tests/golden/make_golden.py f4).

Bars: nn_recurrence and spin_field_sums bit-exact (the twin repeats the
reference's additions in the same order; integer sums); pairs_poly 1e-13 on
the CPU, 1e-12 on the GPU (fp64 atomic scatter); ho_naive_block
1e-13 / 1e-12 (sin ulp differences over 64 000 terms).
"""

import math
import os

import numpy as np
import pytest

from oracle import kernels as K

NN_TAGS = ("a", "b", "c", "d", "e")


@pytest.fixture(scope="module")
def f4(golden_dir):
    return dict(np.load(os.path.join(golden_dir, "kernels_f4.npz")))


@pytest.fixture(scope="module")
def KD():
    from paper_2203_16657_b200 import _kernels

    return _kernels


def _pairs_poly(mod, f4):
    o = f4["pp_out0"].copy()
    n = o.shape[0]
    mod.pairs_poly(f4["pp_iu"], f4["pp_iv"], f4["pp_x"], 1.0 / n, f4["pp_coef"], 0.2,
                   f4["pp_sgn"], o)
    return o


def test_oracle_pairs_poly(f4):
    np.testing.assert_allclose(_pairs_poly(K, f4), f4["pp_out"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("tag", NN_TAGS)
def test_oracle_nn_recurrence_bit_exact(f4, tag):
    ph = f4[f"nn_{tag}_ph"]
    got = K.nn_recurrence(ph, int(f4[f"nn_{tag}_k"]), 1.0 / ph.shape[0],
                          int(f4[f"nn_{tag}_anchor"]))
    assert np.array_equal(got, f4[f"nn_{tag}_f"])


def test_oracle_nn_recurrence_vs_direct_window(f4):
    """after N recurrence steps |F_m - direct| <= 1e-10."""
    ph = f4["nn_c_ph"]
    n, k = ph.shape[0], int(f4["nn_c_k"])
    got = K.nn_recurrence(ph, k, 1.0 / n, 10 ** 9)  # never re-anchored
    c = np.concatenate([[0], np.cumsum(np.concatenate([ph, ph, ph]))])
    m = np.arange(n) + n
    direct = (c[m + k + 1] - c[m - k]) / n
    assert np.abs(got - direct).max() <= 1e-10


def test_oracle_spin_field_sums(f4):
    assert np.array_equal(K.spin_field_sums(f4["spin"]), f4["spin_f"])


def test_oracle_ho_naive_block_40(f4):
    th = f4["ho40_theta"]
    np.testing.assert_allclose(K.ho_naive_block(th, (1, 1, 0, -2)), f4["ho40_1102"], rtol=0,
                               atol=1e-13)
    np.testing.assert_allclose(K.ho_naive_block(th, (2, -1, 1, -2)), f4["ho40_2m11m2"], rtol=0,
                               atol=1e-13)


# ---------------------------------------------------------------------------
# device twins (C ABI: cdk_pairs_poly, cdk_nn_recurrence, cdk_spin_field_sums,
# cdk_ho_naive_block)
# ---------------------------------------------------------------------------
@pytest.mark.gpu
def test_gpu_pairs_poly(f4, KD):
    np.testing.assert_allclose(_pairs_poly(KD, f4), f4["pp_out"], rtol=0, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", NN_TAGS)
def test_gpu_nn_recurrence_bit_exact(f4, KD, tag):
    ph = f4[f"nn_{tag}_ph"]
    got = KD.nn_recurrence(ph, int(f4[f"nn_{tag}_k"]), 1.0 / ph.shape[0],
                           int(f4[f"nn_{tag}_anchor"]))
    assert got.dtype == np.complex128 and np.array_equal(got, f4[f"nn_{tag}_f"])


@pytest.mark.gpu
def test_gpu_spin_field_sums(f4, KD):
    got = KD.spin_field_sums(f4["spin"])
    assert got.dtype == np.int64 and np.array_equal(got, f4["spin_f"])
    # large input, both signs, exact integer arithmetic
    rng = np.random.default_rng(3)
    s = rng.integers(-5, 6, 3_000_001).astype(np.int64)
    assert np.all(KD.spin_field_sums(s)[[0, -1]] == int(s.sum()))
    assert KD.spin_field_sums(np.zeros(0, np.int64)).shape == (0,)


@pytest.mark.gpu
def test_gpu_ho_naive_block(f4, KD):
    th = f4["ho40_theta"]
    np.testing.assert_allclose(KD.ho_naive_block(th, (1, 1, 0, -2)), f4["ho40_1102"], rtol=0,
                               atol=1e-12)
    np.testing.assert_allclose(KD.ho_naive_block(th, (2, -1, 1, -2)), f4["ho40_2m11m2"], rtol=0,
                               atol=1e-12)


@pytest.mark.gpu
def test_gpu_ho_naive_block_small_golden(golden_dir, KD):
    ks = np.load(os.path.join(golden_dir, "kernels_small.npz"))
    th = ks["ho_theta"]
    np.testing.assert_allclose(KD.ho_naive_block(th, (1, 1, 0, -2)), ks["ho_1102"], rtol=0,
                               atol=1e-12)
    np.testing.assert_allclose(KD.ho_naive_block(th, (1, 1, -1, -1)), ks["ho_11m1m1"], rtol=0,
                               atol=1e-12)
    assert math.isfinite(float(KD.ho_naive_block(th[:1], (1, 1, 0, -2))[0]))
