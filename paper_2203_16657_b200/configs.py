"""Frozen workload definitions for the BASELINE.json configs (seeded, synthetic).

Open decisions the SPEC/BASELINE leave are fixed here and
restated in DESIGN.md:

* coupling: theta'_m = omega_m + (K/N) sum_l A_ml sin(theta_l - theta_m), i.e.
  h = K sin with the paper's global 1/N; "K = 5/N" in BASELINE is K = 5 here.
  Configs 2 and 5 do not state K; they use the same K = 5.
* config 2 sizes: 200 draws of a power law (exponent 2) on [200, 5000],
  renormalised to sum to N by floor + largest remainders (sizes then span
  roughly 300..7500 — the renormalisation is applied as BASELINE states).
  Inter edges: each inter-community pair independently with
  p_out = 5 N / (N^2 - sum lambda^2), i.e. expected inter degree 5.
* seeds: graph seed and state seed fixed per config (below); the state stream
  draws omega then theta0 from PCG64(SeedSequence(state_seed)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .graph import planted_partition_decomposition, power_law_sizes


@dataclass(frozen=True)
class KuramotoCase:
    name: str
    sizes: tuple
    p_in: float
    p_out: float
    coupling: float
    dt: float
    steps: int
    graph_seed: int
    state_seed: int

    @property
    def n(self) -> int:
        return int(sum(self.sizes))

    def decomposition(self):
        return planted_partition_decomposition(self.sizes, self.p_in, self.p_out, self.graph_seed)

    def state(self):
        """(omega, theta0) float64[N] in permuted (= planted) order."""
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(self.state_seed)))
        omega = rng.standard_normal(self.n)
        theta0 = rng.uniform(0.0, 2.0 * math.pi, self.n)
        return omega, theta0


def _cfg2_sizes(n=200_000, m=200, seed=2002):
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    return tuple(int(s) for s in power_law_sizes(rng, m, 2.0, 200.0, 5000.0, n))


def config1() -> KuramotoCase:
    """BASELINE configs[0]: SBM N=1000, 10 x 100, p_in .9, p_out .01, RK4 dt .01 x 1000."""
    return KuramotoCase("cfg1", (100,) * 10, 0.9, 0.01, 5.0, 0.01, 1000, 1001, 1101)


def config2() -> KuramotoCase:
    """BASELINE configs[1]: N=200k, 200 power-law communities, p_in .95,
    inter degree 5, RK4 dt .01 x 2000 (the bench workload)."""
    sizes = _cfg2_sizes()
    n = sum(sizes)
    sum_sq = sum(s * s for s in sizes)
    p_out = 5.0 * n / (n * n - sum_sq)
    return KuramotoCase("cfg2", sizes, 0.95, p_out, 5.0, 0.01, 2000, 2001, 2101)


def scaled_config2(n: int, m: int, seed: int = 7) -> KuramotoCase:
    """Config-2 family at another size (tests, scaling sweeps)."""
    sizes = _cfg2_sizes(n, m, seed)
    sum_sq = sum(s * s for s in sizes)
    p_out = 5.0 * n / (n * n - sum_sq)
    return KuramotoCase(f"cfg2_n{n}", sizes, 0.95, p_out, 5.0, 0.01, 2000, seed + 1, seed + 2)


@dataclass(frozen=True)
class HOCase:
    """Higher-order (triadic) Kuramoto on 3-cliques (BASELINE configs[2])."""

    name: str
    sizes: tuple
    p_in: float
    p_out: float
    k1: float
    k2: float
    dt: float
    steps: int
    graph_seed: int
    state_seed: int

    @property
    def n(self) -> int:
        return int(sum(self.sizes))

    def decomposition(self):
        return planted_partition_decomposition(self.sizes, self.p_in, self.p_out, self.graph_seed)

    def state(self):
        """omega ~ N(0,1) (BASELINE leaves it open), theta0 ~ U[0, 2pi)."""
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(self.state_seed)))
        omega = rng.standard_normal(self.n)
        theta0 = rng.uniform(0.0, 2.0 * math.pi, self.n)
        return omega, theta0


def config3() -> HOCase:
    """SBM N=50000, 100 x 500, p_in .9, p_out 1e-4; K1=1, K2=.5; RK4 dt .005 x 1000."""
    return HOCase("cfg3", (500,) * 100, 0.9, 1e-4, 1.0, 0.5, 0.005, 1000, 3001, 3101)


def scaled_config3(m: int = 8, lam: int = 120, p_out: float = 2e-3, seed: int = 31) -> HOCase:
    """Config-3 family at a size the O(N^3) direct oracle handles."""
    return HOCase(f"cfg3_{m}x{lam}", (lam,) * m, 0.9, p_out, 1.0, 0.5, 0.005, 1000, seed,
                  seed + 1)


@dataclass(frozen=True)
class CSCase:
    """Cucker-Smale 2-D (BASELINE configs[3])."""

    name: str
    sizes: tuple
    p_in: float
    p_out: float
    K: float
    sigma: float
    beta: float
    dt: float
    steps: int
    graph_seed: int
    state_seed: int

    @property
    def n(self) -> int:
        return int(sum(self.sizes))

    @property
    def t_end(self) -> float:
        return self.dt * self.steps

    def decomposition(self):
        return planted_partition_decomposition(self.sizes, self.p_in, self.p_out, self.graph_seed)

    def state(self):
        """positions ~ U[0,10]^2, velocities ~ N(0,1)^2."""
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(self.state_seed)))
        pos = rng.uniform(0.0, 10.0, (self.n, 2))
        vel = rng.standard_normal((self.n, 2))
        return pos, vel


def config4() -> CSCase:
    """SBM N=100000, 100 x 1000, p_in .9, p_out 1e-4; psi=(1+r^2)^-1/4; RK4 dt .01 x 500."""
    return CSCase("cfg4", (1000,) * 100, 0.9, 1e-4, 1.0, 1.0, 0.25, 0.01, 500, 4001, 4101)


def scaled_config4(m: int = 5, lam: int = 80, p_out: float = 3e-3, seed: int = 41) -> CSCase:
    return CSCase(f"cfg4_{m}x{lam}", (lam,) * m, 0.9, p_out, 1.0, 1.0, 0.25, 0.01, 500, seed,
                  seed + 1)


CONFIGS = {"cfg1": config1, "cfg2": config2, "cfg3": config3, "cfg4": config4}
