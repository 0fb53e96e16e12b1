"""Every run-time knob of the planner and the multi-GPU driver in one place.

The defaults are the measured choices; the environment can
override them for experiments and tests.  ``settings()`` re-reads the
environment on each call (cheap), so a test that sets a variable sees it at
the next DeviceGraph construction.  Nothing else in the package reads
``CDK_*`` variables (the library path ``CDK_LIB`` is read by ``_lib`` at
load time; it selects an experiment build of the same ABI).

=====================  ======================  =========================================
variable               field                   meaning
=====================  ======================  =========================================
CDK_ELL                ell                     lane-per-row ELL kernels (0: row-group kernels)
CDK_ELL_CALIBRATE      ell_calibrate           measured CTA re-cuts at construction (0: off)
CDK_ELL_WINDOW         ell_window              cap on the ELL window (nodes; 0: library's)
CDK_ELL_META           ell_meta                packed per-unit metadata records
CDK_ELL_SLOT_COST ...  ell_slot_cost, ...      ELL cost model (cycles per slot / rblock / segment)
CDK_ROWS_CAP           rows_cap                rows per segment of the row-group kernels
CDK_SMEM_BUDGET        smem_budget             row-group kernels' shared-memory budget (bytes)
CDK_SEG_COST           seg_cost                row-group segment cost (model units)
CDK_XS                 xs                      staged inter columns (row-group kernels)
CDK_LPR                lpr                     lanes per row of the row-group gathers
CDK_INTER_PHASE        inter_phase             force (1) / forbid (0) the separate inter phase
CDK_INTER_BLOCKS       inter_blocks            force the block-phased inter sweep's block count
CDK_P2P                p2p                     fused NVLink exchange on multi-GPU runs (0: NCCL)
CDK_CS_BANK_SPREAD     cs_bank_spread          Cucker-Smale: missing columns ordered for the window's banks
=====================  ======================  =========================================
"""

from __future__ import annotations

import os
from dataclasses import dataclass


def _int(name: str, default: int) -> int:
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


def _float(name: str, default: float) -> float:
    v = os.environ.get(name)
    return float(v) if v not in (None, "") else default


def _flag(name: str, default: bool) -> bool:
    v = os.environ.get(name)
    return default if v in (None, "") else v != "0"


def _opt_int(name: str):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else None


@dataclass(frozen=True)
class Settings:
    ell: bool = True
    ell_calibrate: int = 4
    ell_window: int = 0
    ell_meta: bool = True
    ell_slot_cost: float = 0.144
    ell_xslot_cost: float = 0.39
    ell_rblk_cost: float = 100.0
    ell_seg_cost: float = 6500.0
    rows_cap: int = 1536
    smem_budget: int = 232448 - 2048
    seg_cost: float = 40000.0
    xs: bool = True
    lpr: int = 8
    inter_phase: int | None = None  # None: per community (mean inter degree)
    inter_blocks: int | None = None  # None: by the size of z
    p2p: bool = True
    cs_bank_spread: bool = True


def settings() -> Settings:
    d = Settings()
    return Settings(
        ell=_flag("CDK_ELL", d.ell),
        ell_calibrate=_int("CDK_ELL_CALIBRATE", d.ell_calibrate),
        ell_window=_int("CDK_ELL_WINDOW", d.ell_window),
        ell_meta=_flag("CDK_ELL_META", d.ell_meta),
        ell_slot_cost=_float("CDK_ELL_SLOT_COST", d.ell_slot_cost),
        ell_xslot_cost=_float("CDK_ELL_XSLOT_COST", d.ell_xslot_cost),
        ell_rblk_cost=_float("CDK_ELL_RBLK_COST", d.ell_rblk_cost),
        ell_seg_cost=_float("CDK_ELL_SEG_COST", d.ell_seg_cost),
        rows_cap=_int("CDK_ROWS_CAP", d.rows_cap),
        smem_budget=_int("CDK_SMEM_BUDGET", d.smem_budget),
        seg_cost=_float("CDK_SEG_COST", d.seg_cost),
        xs=_flag("CDK_XS", d.xs),
        lpr=_int("CDK_LPR", d.lpr),
        inter_phase=_opt_int("CDK_INTER_PHASE"),
        inter_blocks=_opt_int("CDK_INTER_BLOCKS"),
        p2p=_flag("CDK_P2P", d.p2p),
        cs_bank_spread=_flag("CDK_CS_BANK_SPREAD", d.cs_bank_spread),
    )
