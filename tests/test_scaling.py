"""SPEC.md:585-591,607-609 scaling witness: kernel-evaluation counts of the
CIA path grow linearly in N on the community-structured family, the naive
counts quadratically (CPU: counts only); on the GPU, the benchmark rows,
slopes and CSV (tests marked gpu)."""

import numpy as np
import pytest

from paper_2203_16657_b200 import scaling


def test_loglog_slope_exact():
    ns = [2**k for k in range(10, 15)]
    assert abs(scaling.loglog_slope(ns, [3 * n for n in ns]) - 1.0) < 1e-12
    assert abs(scaling.loglog_slope(ns, [n * n for n in ns]) - 2.0) < 1e-12


def test_cia_count_slope_linear_naive_quadratic_cpu():
    from paper_2203_16657_b200.integrator import cia_kernel_evals_per_rhs
    from paper_2203_16657_b200.models import kuramoto_model

    ns = [2**k for k in range(10, 18)]
    cia = []
    for n in ns:
        dec = scaling.scaled_decomposition(n)
        cia.append(cia_kernel_evals_per_rhs(kuramoto_model(np.zeros(n)), dec))
    assert 0.95 <= scaling.loglog_slope(ns, cia) <= 1.05
    nn = [2**k for k in range(10, 14)]
    naive = [2 * scaling.scaled_decomposition(n).graph().edges.shape[0] for n in nn]
    assert 1.95 <= scaling.loglog_slope(nn, naive) <= 2.05


@pytest.mark.gpu
def test_bench_scaling_gpu(tmp_path):
    cia = scaling.bench_scaling("kuramoto", "cia", repeats=2, steps=10)
    naive = scaling.bench_scaling("kuramoto", "naive", repeats=2, steps=5)
    assert 0.95 <= cia[1]["count_slope"] <= 1.05
    assert 1.95 <= naive[1]["count_slope"] <= 2.05
    # corroboration: naive device time grows faster than CIA's
    assert naive[1]["wall_slope"] > cia[1]["wall_slope"]
    p = tmp_path / "scaling.csv"
    scaling.write_csv(str(p), [cia, naive])
    txt = p.read_text().splitlines()
    assert txt[0] == "model,mode,N,median_seconds,kernel_evals" and len(txt) == 1 + 8 + 4 + 4
    print(cia[1], naive[1])
