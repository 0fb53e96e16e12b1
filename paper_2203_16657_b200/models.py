"""Model definitions (ModelSpec) for the models on the hot path.

* ``Kuramoto``          SPEC.md:433-438.
                        theta'_m = omega_m + (K/N) sum_l a_ml sin(theta_l - theta_m)
* ``HigherOrderKuramoto`` and ``CuckerSmale`` are defined in models_ho.py /
  models_cs.py (configs 3 and 4).

States are given in ORIGINAL node order at this API level; the engines work
in the decomposition's permuted order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Kuramoto:
    """Classical Kuramoto; h = coupling * sin, global 1/norm (default N)."""

    omega: np.ndarray
    coupling: float = 1.0
    norm: float | None = None
    state_space: str = "circle"

    def n(self) -> int:
        return int(np.asarray(self.omega).shape[0])

    def norm_value(self) -> float:
        return float(self.norm if self.norm is not None else self.n())


def kuramoto_model(omega, coupling: float = 1.0, norm: float | None = None) -> Kuramoto:
    return Kuramoto(np.asarray(omega, dtype=np.float64), float(coupling), norm)
