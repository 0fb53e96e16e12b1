"""Evaluator: CIA right-hand side and the direct-sum RHS.

* ``eval_rhs_cia``   SPEC.md:359-366 — E1 (community observables) + E2 (signed
                     sparse correction with the exact coupling) + intrinsic term,
                     one fused kernel (cdk_kuramoto_rhs).
* ``eval_rhs_naive`` SPEC.md:368-374 — direct sum over the graph's edges with the
                     exact coupling (naive.NaiveEngine: cdk_pairs_trig /
                     cdk_pairs_cs over the full edge list, sgn = +1, plus
                     cdk_triangles_sin for the triadic model).
                     Memory guard N > 2^15 as SPEC.md:614.

Both take and return states in ORIGINAL node order (numpy).
"""

from __future__ import annotations

import numpy as np

from .engine import KuramotoEngine
from .errors import InputError
from .graph import Decomposition, Graph
from .models import Kuramoto
from .naive import NAIVE_N_CAP  # noqa: F401  (re-exported: the SPEC's memory guard)
from .plan import DeviceGraph


def perm_device(dec: Decomposition):
    """(perm, inv_perm) of the decomposition as cached int64 device tensors."""
    import torch

    t = dec._cache.get("perm_dev")
    if t is None:
        p = dec.partition
        t = dec._cache["perm_dev"] = (torch.as_tensor(p.perm, device="cuda"),
                                      torch.as_tensor(p.inv_perm, device="cuda"))
    return t


def _engine(model: Kuramoto, dec: Decomposition) -> KuramotoEngine:
    """One engine (device graph + workspace) per decomposition; a different
    model object only re-uploads omega and the coupling constants."""
    cached = dec._cache.get("engine")  # (model, engine) of the most recent model
    if cached is not None and cached[0] is model:
        return cached[1]
    perm = dec.partition.perm
    omega = np.asarray(model.omega, dtype=np.float64)
    if omega.shape != (dec.n_nodes,):
        raise InputError("omega shape does not match the decomposition")
    if cached is not None:
        eng = cached[1]
        eng.upload_permuted(eng.omega, omega, perm_device(dec)[0])
        eng.coupling = float(model.coupling)
        eng.norm = float(model.norm_value())
        eng.k_over_n = eng.coupling / eng.norm
    else:
        dg = dec._cache.get("device_graph")
        if dg is None:
            dg = dec._cache["device_graph"] = DeviceGraph(dec)
        eng = KuramotoEngine(dec, omega[perm], coupling=model.coupling,
                             norm=model.norm_value(), graph=dg)
    dec._cache["engine"] = (model, eng)
    return eng


def _ho_engine(model, dec: Decomposition):
    from .ho import HOEngine, HoDeviceGraph

    cached = dec._cache.get("ho_engine")
    eng = cached[1] if cached is not None and cached[0] is model else None
    if eng is None:
        dg = dec._cache.get("ho_graph")
        if dg is None:
            dg = dec._cache["ho_graph"] = HoDeviceGraph(dec)
        perm = dec.partition.perm
        eng = HOEngine(dec, np.asarray(model.omega)[perm], model.k1, model.k2,
                       norm=model.norm_value(), graph=dg)
        dec._cache["ho_engine"] = (model, eng)
    return eng


def _hh_engine(model, dec: Decomposition):
    from .harmonics import HhDeviceGraph, HhEngine

    cached = dec._cache.get("hh_engine")
    if cached is not None and cached[0] is model:
        return cached[1]
    dg = dec._cache.get("hh_graph")
    if dg is None:
        dg = dec._cache["hh_graph"] = HhDeviceGraph(dec)
    perm = dec.partition.perm
    eng = HhEngine(dec, np.asarray(model.omega)[perm], model.d_cos, model.d_sin,
                   norm=model.norm_value(), graph=dg)
    dec._cache["hh_engine"] = (model, eng)
    return eng


def engine_for(model, dec: Decomposition):
    """The device engine of a model (Kuramoto, higher-harmonics Kuramoto or
    higher-order Kuramoto)."""
    from .harmonics import HigherHarmonicsKuramoto
    from .ho import HigherOrderKuramoto

    if isinstance(model, Kuramoto):
        return _engine(model, dec)
    if isinstance(model, HigherHarmonicsKuramoto):
        return _hh_engine(model, dec)
    if isinstance(model, HigherOrderKuramoto):
        return _ho_engine(model, dec)
    raise InputError(f"unsupported model {type(model).__name__}")


def _cs_engine(model, dec: Decomposition, pos_perm, vel_perm, t_end: float):
    """The P2 fit (centres, scales, polynomial) depends on the initial state and
    the horizon, so the cache key carries a fingerprint of both: a cached
    engine is reused only for the same model, horizon and initial state."""
    import hashlib

    from .cs import CSEngine

    h = hashlib.sha1(np.ascontiguousarray(pos_perm, np.float64).tobytes())
    h.update(np.ascontiguousarray(vel_perm, np.float64).tobytes())
    key = ("cs_engine", id(model), float(t_end), h.hexdigest())
    cached = dec._cache.get("cs_engine")
    if cached is not None and cached[0] == key and cached[1] is model:
        eng = cached[2]
        eng.set_state(pos_perm, vel_perm)
        return eng
    eng = CSEngine(dec, model, pos_perm, vel_perm, t_end=t_end)
    dec._cache["cs_engine"] = (key, model, eng)
    return eng


def eval_rhs_cia(model, dec: Decomposition, state) -> np.ndarray:
    from .cs import CuckerSmale

    if isinstance(model, CuckerSmale):  # state [N, 4] = (s_x, s_y, v_x, v_y)
        x = np.asarray(state, dtype=np.float64)
        if x.shape != (dec.n_nodes, 4):
            raise InputError("Cucker-Smale state must have shape (N, 4)")
        perm = dec.partition.perm
        xp = x[perm]
        eng = _cs_engine(model, dec, xp[:, :2], xp[:, 2:], t_end=0.0)
        sd, vd = eng.rhs(xp[:, :2], xp[:, 2:])
        outp = np.concatenate([sd.cpu().numpy(), vd.cpu().numpy()], 1)
        out = np.empty_like(outp)
        out[perm] = outp
        return out
    x = np.asarray(state, dtype=np.float64)
    if x.shape != (dec.n_nodes,):
        raise InputError("state shape does not match the decomposition")
    perm = dec.partition.perm
    eng = engine_for(model, dec)
    out_perm = eng.rhs(x[perm]).cpu().numpy()
    out = np.empty_like(out_perm)
    out[perm] = out_perm
    return out


def eval_rhs_naive(model, graph: Graph, state) -> np.ndarray:
    """Direct sum over ``graph``'s edges with the exact coupling
    for every model on the path: Kuramoto, higher-order Kuramoto (pairs +
    3-cliques) and Cucker-Smale (state [N, 4]).  States in the graph's node
    order; device kernels (naive.NaiveEngine); MemoryGuardError above 2^15."""
    from .naive import NaiveEngine

    x = np.asarray(state, dtype=np.float64)
    eng = NaiveEngine(model, graph)
    want = (graph.n_nodes, 4) if eng.kind == "cs" else (graph.n_nodes,)
    if x.shape != want:
        raise InputError(f"state must have shape {want}")
    return eng.rhs(x).cpu().numpy()
