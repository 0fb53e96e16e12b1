"""commdyn-b200: the CIA hot path of arXiv 2203.16657 (reference package
``commdyn``) as hand-written sm_100a CUDA behind a C ABI
(include/commdyn_cuda.h, libcommdyn_cuda.so).

Public API (mirrors the reference/SPEC names):
    graph      Graph, Partition, SparseCorrection, Decomposition,
               planted_partition_graph, planted_partition_decomposition, decompose
    models     Kuramoto, kuramoto_model
    evaluator  eval_rhs_cia, eval_rhs_naive
    integrator IntegrationPlan, Trajectory, integrate
    _kernels   device twins of the reference dispatchers
    _backend   backend() == "cuda"
"""

from . import errors  # noqa: F401
from .graph import (  # noqa: F401
    Decomposition,
    Graph,
    Partition,
    SparseCorrection,
    decompose,
    planted_partition_decomposition,
    planted_partition_graph,
)
from .models import Kuramoto, kuramoto_model  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):  # lazy: these import torch / the CUDA library
    if name in ("eval_rhs_cia", "eval_rhs_naive"):
        from . import evaluator

        return getattr(evaluator, name)
    if name in ("IntegrationPlan", "Trajectory", "integrate"):
        from . import integrator

        return getattr(integrator, name)
    if name in ("HigherOrderKuramoto", "ho_kuramoto_model", "HOEngine"):
        from . import ho

        return getattr(ho, name)
    if name in ("HigherHarmonicsKuramoto", "higher_harmonics_model",
                "harmonics_model_from_coupling", "HhEngine"):
        from . import harmonics

        return getattr(harmonics, name)
    if name in ("CuckerSmale", "CSEngine"):
        from . import cs

        return getattr(cs, name)
    if name == "KuramotoEngine":
        from .engine import KuramotoEngine

        return KuramotoEngine
    raise AttributeError(name)
