"""ctypes binding of libcommdyn_cuda.so (include/commdyn_cuda.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, ``lib()`` raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CDK_CUDA, CDK_INPUT, CDK_NUMERIC, CDK_OK, DeviceError, InputError, NumericError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CDK_LIB") or os.path.join(_PKG, "_build", "libcommdyn_cuda.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
D = ctypes.c_double
I = ctypes.c_int


class CdkGraph(ctypes.Structure):
    _fields_ = [
        ("n_rows", I64),
        ("n_comm", I64),
        ("comm_off", P),
        ("intra_ptr", P),
        ("intra_col", P),
        ("inter_ptr", P),
        ("inter_col", P),
        ("n_rblk", I32),
        ("n_seg", I32),
        ("n_cta", I32),
        ("cta_threads", I32),
        ("smem_nodes", I32),
        ("seg_rows_cap", I32),
        ("rblk_row0", P),
        ("rblk_comm", P),
        ("comm_rblk_off", P),
        ("seg_rblk", P),
        ("seg_win", P),
        ("seg_base", P),
        ("cta_seg", P),
        ("seg_lpr", P),
        ("intra_split", P),
        ("inter_blocks", I32),
        ("inter_block_nodes", I32),
        ("inter_split", P),
        ("xs_cap", I32),
        ("reserved0", I32),
        ("seg_xr", P),
        ("ell_off", P),
        ("ell_col", P),
        ("xell_off", P),
        ("xell_col", P),
        ("ell_units", P),
        ("seg_unit", P),
        ("ell_meta", P),
    ]


class CdkPeers(ctypes.Structure):
    _fields_ = [
        ("n_ranks", I32),
        ("rank", I32),
        ("z0", P),
        ("z1", P),
        ("bar", P),
        ("bar_base", ctypes.c_uint32),
        ("wait", I32),
    ]


class CdkHoGraph(ctypes.Structure):
    _fields_ = [
        ("n_rows", I64),
        ("n_rblk", I32),
        ("n_comm", I32),
        ("rblk_row0", P),
        ("rblk_comm", P),
        ("comm_rblk_off", P),
        ("miss_ptr", P),
        ("miss_col", P),
        ("inter_ptr", P),
        ("inter_col", P),
        ("tri_ptr", P),
        ("tri_jk", P),
    ]


class CdkHhGraph(ctypes.Structure):
    _fields_ = [
        ("n_rows", I64),
        ("n_rblk", I32),
        ("n_comm", I32),
        ("p", I32),
        ("reserved", I32),
        ("rblk_row0", P),
        ("rblk_comm", P),
        ("comm_rblk_off", P),
        ("comm_off", P),
        ("miss_ptr", P),
        ("miss_col", P),
        ("inter_ptr", P),
        ("inter_col", P),
        ("d_cos", P),
        ("d_sin", P),
    ]


class CdkCsGraph(ctypes.Structure):
    _fields_ = [
        ("n_rows", I64),
        ("n_comm", I64),
        ("n_rblk", I32),
        ("max_comm", I32),
        ("comm_off", P),
        ("rblk_row0", P),
        ("rblk_comm", P),
        ("miss_ptr", P),
        ("miss_col", P),
        ("inter_ptr", P),
        ("inter_col", P),
        ("mu", P),
        ("inv_L", P),
        ("chat", P),
        ("t_ptr", P),
        ("t_col", P),
        ("t_coef", P),
    ]


class CdkGenParams(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("n_rows", I64),
        ("n_comm", I64),
        ("comm_off", P),
        ("node_cdf", P),
        ("n_inter_edges", I64),
        ("miss_thr", ctypes.c_uint32),
        ("pass_nodes", ctypes.c_uint32),
        ("row_lo", I64),
        ("row_hi", I64),
    ]


class CdkRunStatus(ctypes.Structure):
    _fields_ = [("nonfinite", I64), ("first_bad_step", I64), ("steps_done", I64),
                ("reserved", I64)]


# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGS = {
    "cdk_kuramoto_stage_threads": [],
    "cdk_kuramoto_stage_ctas_per_sm": [],
    "cdk_order_params_blocks": [P, P, I64, I, D, D, P, P],
    "cdk_dense_complex": [P, P, I64, P, I, D, P, P, P],
    "cdk_dense_real": [P, P, I64, P, P, I, D, P, P],
    "cdk_pairs_trig": [P, P, I64, P, D, P, P, I, D, P, P, P],
    "cdk_pairs_cs": [P, P, I64, P, P, I, D, D, D, D, P, P, P],
    "cdk_moments_blocks": [P, P, I64, I, D, D, P, P],
    "cdk_dense_poly": [P, P, I64, P, I, D, D, P, P],
    "cdk_pairs_poly": [P, P, I64, P, D, P, I, D, P, P, P],
    "cdk_ho_naive_block": [P, I64, D, D, D, D, P, P],
    "cdk_nn_recurrence": [P, I64, I64, D, I64, P, P],
    "cdk_spin_field_sums": [P, I64, P, P, P],
    "cdk_triangles_sin": [P, I64, P, D, P, P],
    "cdk_rank_one": [P, P, P, I64, D, P, P, P],
    "cdk_kuramoto_workspace_bytes": [ctypes.POINTER(CdkGraph)],
    "cdk_kuramoto_prepare": [ctypes.POINTER(CdkGraph), P, P, P],
    "cdk_kuramoto_rhs": [ctypes.POINTER(CdkGraph), P, P, D, P, P, P],
    "cdk_kuramoto_rk4": [ctypes.POINTER(CdkGraph), P, P, D, D, I64, P, P],
    "cdk_kuramoto_rk4_stage": [ctypes.POINTER(CdkGraph), P, P, D, D, I, P, P],
    "cdk_kuramoto_workspace_layout": [ctypes.POINTER(CdkGraph), P],
    "cdk_kuramoto_advance": [ctypes.POINTER(CdkGraph), P, I64, P],
    "cdk_kuramoto_euler": [ctypes.POINTER(CdkGraph), P, P, D, D, I64, P, P],
    "cdk_kuramoto_status": [ctypes.POINTER(CdkGraph), P, ctypes.POINTER(CdkRunStatus), P],
    "cdk_host_bank_order": [P, P, I64, I32, I32],
    "cdk_host_ell_intra": [P, I32, P, P, P, P, I32, P, P],
    "cdk_kuramoto_ell_threads": [],
    "cdk_kuramoto_stage_cycles": [P, P, P, D, D, P, P, P],
    "cdk_kuramoto_ell_ctas_per_sm": [],
    "cdk_kuramoto_ell_window_nodes": [],
    "cdk_debug_set_profile_buffer": [P],
    "cdk_host_triangles": [P, P, I64, P, I64],
    "cdk_ho_workspace_bytes": [ctypes.POINTER(CdkHoGraph)],
    "cdk_ho_prepare": [ctypes.POINTER(CdkHoGraph), P, P, P],
    "cdk_ho_rhs": [ctypes.POINTER(CdkHoGraph), P, P, D, D, P, P, P],
    "cdk_ho_rk4": [ctypes.POINTER(CdkHoGraph), P, P, D, D, D, I64, P, P],
    "cdk_ho_status": [ctypes.POINTER(CdkHoGraph), P, ctypes.POINTER(CdkRunStatus), P],
    "cdk_hh_workspace_bytes": [ctypes.POINTER(CdkHhGraph)],
    "cdk_hh_prepare": [ctypes.POINTER(CdkHhGraph), P, P, P],
    "cdk_hh_rhs": [ctypes.POINTER(CdkHhGraph), P, P, D, P, P, P],
    "cdk_hh_rk4": [ctypes.POINTER(CdkHhGraph), P, P, D, D, I64, P, P],
    "cdk_hh_status": [ctypes.POINTER(CdkHhGraph), P, ctypes.POINTER(CdkRunStatus), P],
    "cdk_cs_workspace_bytes": [ctypes.POINTER(CdkCsGraph)],
    "cdk_cs_prepare": [ctypes.POINTER(CdkCsGraph), P, P],
    "cdk_cs_rhs": [ctypes.POINTER(CdkCsGraph), P, P, D, D, D, D, P, P, P],
    "cdk_cs_rk4": [ctypes.POINTER(CdkCsGraph), P, P, D, D, D, D, D, I64, P, P],
    "cdk_cs_status": [ctypes.POINTER(CdkCsGraph), P, ctypes.POINTER(CdkRunStatus), P],
    "cdk_gen_intra_count": [ctypes.POINTER(CdkGenParams), P, P, P, P],
    "cdk_gen_intra_fill": [ctypes.POINTER(CdkGenParams), P, P, P, P],
    "cdk_gen_inter_count": [ctypes.POINTER(CdkGenParams), P, P],
    "cdk_gen_inter_fill": [ctypes.POINTER(CdkGenParams), P, P, P],
    "cdk_gen_inter_sort": [I64, P, P, P, P],
    "cdk_gen_inter_compact": [I64, P, P, P, P, P],
    "cdk_gen_rebase": [I64, P, P, P, P],
    "cdk_inter_split": [I64, P, P, ctypes.c_int, ctypes.c_int, P, P],
    "cdk_bank_order": [I64, P, P, P, P, ctypes.c_int, P],
    "cdk_kuramoto_rk4_peers": [ctypes.POINTER(CdkGraph), P, P, ctypes.c_double, ctypes.c_double,
                               I64, P, ctypes.POINTER(CdkPeers), P],
    "cdk_kuramoto_rk4_stage_peers": [ctypes.POINTER(CdkGraph), P, P, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_int, P, ctypes.POINTER(CdkPeers),
                                     P],
    "cdk_ipc_export": [P, P, ctypes.POINTER(ctypes.c_uint64)],
    "cdk_ipc_import": [P, ctypes.c_uint64, ctypes.POINTER(P)],
    "cdk_ipc_close": [P, ctypes.c_uint64],
    "cdk_abi_version": [],
    "cdk_last_error": [],
    "cdk_launch_count": [],
    "cdk_max_smem_optin": [],
}
_RESTYPES = {
    "cdk_kuramoto_workspace_bytes": ctypes.c_size_t,
    "cdk_last_error": ctypes.c_char_p,
    "cdk_launch_count": I64,
    "cdk_debug_set_profile_buffer": None,
    "cdk_host_triangles": I64,
    "cdk_ho_workspace_bytes": ctypes.c_size_t,
    "cdk_hh_workspace_bytes": ctypes.c_size_t,
    "cdk_cs_workspace_bytes": ctypes.c_size_t,
}

EXPORTED = tuple(_SIGS)
ABI_VERSION = 17

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load the shared library and bind every declared symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback for the CUDA path)"
            )
        lib = ctypes.CDLL(path)
        for name, argtypes in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        if lib.cdk_abi_version() != ABI_VERSION:
            raise DeviceError("libcommdyn_cuda.so ABI version mismatch")
        _lib = lib
        return lib


def lib():
    """The loaded library, after checking a CUDA device is present."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the commdyn CUDA backend has no CPU fallback")
    return load_library()


def check(rc: int, what: str = "") -> None:
    if rc == CDK_OK:
        return
    msg = (_lib.cdk_last_error() or b"").decode() if _lib is not None else ""
    if rc == CDK_INPUT:
        raise InputError(f"{what}: {msg}")
    if rc == CDK_NUMERIC:
        raise NumericError(f"{what}: {msg}")
    if rc == CDK_CUDA:
        raise DeviceError(f"{what}: {msg}")
    raise DeviceError(f"{what}: unknown status {rc}")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
